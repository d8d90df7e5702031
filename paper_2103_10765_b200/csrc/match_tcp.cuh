// Product-form block matching on the tensor cores for patch 12 / stride 4 (BASELINE c2, the
// high-noise profile of PAPER.md:250-253).
//
// Method.  As match_tc16.cuh: d(p, q) = ||f_p||^2 + ||f_q||^2 - 2 <f_p, f_q> (Eq. (2),
// PAPER.md:82), the norms as box sums (step 1), the local cross-correlations
// (Prop. 1) as tcgen05.mma kind::f16 inner products of a 128-reference tile with
// each candidate row.  Exactness: the tile's pixels are centred on c = (min + max) / 2 and held as
// fp16 of z - c (exact for |z - c| <= 2048); every partial sum of <f_p, f_q> is an integer of
// magnitude <= P^2 M^2 (M = max |z - c|), exact in the fp32 accumulator while P^2 M^2 <= 2^24
// (M <= 341 at P = 12).  A tile above the bound takes an in-kernel exact int32 path (direct
// Eq. (1) sums from the pixel plane), so every tile is bit-exact.
//
// Layout.
//   * Tile = 16 x TX grid references in MMA M = 128 (TMEM lane m = reference 8a + b, b < TX); one
//     CTA per tile (c2's 512^2 image: 144 tiles of 16 x 7 for 148 SMs, a single wave).
//   * The union of the tile's windows is NT = 15S + 2r + 1 candidate rows x NJ = (TX-1)S + 2r + 1
//     candidate columns <= N (TX = 7, N = 64 when that fits, else TX = 8, N = 80).  One
//     candidate row = one M128 xN product over K = 12 patch rows x 16 (the last 4 fp16 of every
//     patch row are zero in A): 12 MMAs of K16.
//   * B needs no per-row building: the tile's centred fp16 plane is written once pre-shifted,
//     X[y][q][m][e] = plane[y][8q + m + e], so candidate row t's K16 step i (patch row i) is the
//     canonical K-major operand at X + (t + i) * XP with LBO = SBO = 128 B (next 8 pixels of the
//     patch row / next 8 candidates).  A (the 128 reference patches) lives in tensor memory.
//   * Warps 0-3 (one per TMEM lane quarter, lane = reference): per row, tcgen05.ld of the 80
//     accumulators, u = N_q - 2<> (one FFMA), pass masks from the sign of u - T against the
//     reference's gate T, u staged to shared memory, then insertion rounds of two keys per lane
//     into a sorted register list of the K - 1 smallest 32-bit keys (d << cb | code; key order =
//     (d, idx) order, reading R5).  Warp 4 allocates TMEM and issues the MMAs (4 accumulator
//     stages); warps 5-7 help with the prologue only.
//   * Candidate rows are visited in a scrambled order (t = t_lo + s * step mod n, step coprime to
//     n near 0.618 n) so that every warp has work in every stretch of rows and the lists fill
//     with typical distances early.
//   * Keys are exact while d <= dsat = 2^(32 - cb) - 1: the gate starts at min(dsat, tau - 1), so a
//     candidate with larger d never enters a list; when tau - 1 > dsat, a reference whose list
//     ends short is recomputed exactly with 64-bit keys (direct Eq. (1) from the tile's pixels).
#pragma once
#include <cuda_fp16.h>

#include <climits>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace gbm3d {
namespace tcp {
constexpr int TY = 16;               // reference tile rows (grid rows); 8 lanes per grid row
// Two tile shapes (template NBT): 16 x 7 references with N = 64 candidate columns when
// 6S + 2r + 1 <= 64 (c2: r = 19), else 16 x 8 with N = 80 (r <= 21).  The narrower tile scans
// a fifth fewer columns per row, holds six accumulator stages and a smaller plane, and c2's
// 144 tiles still fit one wave on 148 SMs.  Lanes with b >= TX are idle.
template <int NBT>
struct Shape {
    static constexpr int NB = NBT;                // candidate columns per MMA (N)
    static constexpr int TX = NBT == 64 ? 7 : 8;  // reference tile columns (grid cols)
    static constexpr int PW = NB + 16;            // pixel plane pitch (int16)
    // 16-byte pixel groups per pre-shifted row: 10 for both shapes -- the last candidate
    // group's second chunk (q + 1) and the exact path's reads (columns <= 77) stay in the row
    static constexpr int XQ = 10;
    static constexpr int XP = XQ * 128;           // bytes per pre-shifted row (8 shifts per group)
    static constexpr int NTS = NBT == 64 ? 6 : 5;  // accumulator stages in flight
    static constexpr int SPITCH = NB;             // TMEM columns per stage
    static constexpr int TM_A = (NTS * SPITCH + 31) / 32 * 32;  // A: 12 K16 steps x 8 columns
};
#ifndef GBM3D_TCP_NH
#define GBM3D_TCP_NH 1
#endif
// NH warps per TMEM lane quarter, each taking a part of every reference's window columns with
// its own list (the lists gate each other and are merged at the end).  Dev switch: NH = 2 is
// correct but slower on c2 (0.110 vs 0.098 ms: both warps scan every column, and they share
// the SMSP), so NH = 1.
constexpr int NH = GBM3D_TCP_NH;
constexpr int EPI_WARPS = 4 * NH, MMA_WARP = EPI_WARPS;
constexpr int NWARPS = EPI_WARPS + (NH == 1 ? 4 : 1), THREADS = 32 * NWARPS;
// floats per lane: the window part's <= 11 (NH = 1) / <= 6 (NH = 2) groups of 4 columns (lane
// pitch 44 / 28 words: conflict-free STS.128)
constexpr int STG_PITCH = NH == 1 ? 44 : 28;
constexpr uint32_t TMEM_COLS = 512;
constexpr int MAX_R = 21;            // shared memory bound (see TcpGeom)
}  // namespace tcp

// Shared-memory carve-up of one CTA (host and device agree).
struct TcpGeom {
    int NT, NJ, PR;
    int off_x, off_nq, off_raw, off_bar, total;
    template <int NBT>
    __host__ __device__ static TcpGeom make(int P, int S, int r) {
        using namespace tcp;
        using SH = Shape<NBT>;
        constexpr int NB = SH::NB, PW = SH::PW, XP = SH::XP, NTS = SH::NTS;
        TcpGeom g;
        g.NT = 15 * S + 2 * r + 1;
        g.NJ = (SH::TX - 1) * S + 2 * r + 1;
        g.PR = g.NT + P - 1;
        g.off_x = 0;                                          // X (+ one pad row); prologue: hs
        g.off_nq = (g.PR + 1) * XP;                           // candidate norms [NT][NB] fp32
        g.off_raw = g.off_nq + g.NT * NB * 4;                 // int16 plane [PR][PW] / staging
        const int raw = g.PR * PW * 2, stg = EPI_WARPS * 32 * STG_PITCH * 4;
        g.off_bar = g.off_raw + ((raw > stg ? raw : stg) + 15) / 16 * 16;
        g.total = g.off_bar + 2 * NTS * 8 + 16 + NH * 128 * 4;  // tfull, tempty; min, max, tmem;
                                                                // published gates [NH][128]
        return g;
    }
};

#if GBM3D_TCP_TRACE  // dev-only: %globaltimer stamps per CTA, read by gbm3d_dev_tcp_trace
static __device__ long long g_tcp_trace[4096][12];
static __device__ long long g_tcp_cnt[4096][4][6];  // per warp: wait, scan, rounds cycles; rounds, rows, dense rows
#define TCP_CLK(v) (v) = clock64()
#define TCP_ADD(i, v)                                                                          \
    do {                                                                                       \
        const int c_ = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;         \
        if (c_ < 4096 && lane == 0) g_tcp_cnt[c_][warp & 3][i] += (v);                         \
    } while (0)
#define TCP_TR(k)                                                                          \
    do {                                                                                   \
        long long t_;                                                                      \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                             \
        const int c_ = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;     \
        if (c_ < 4096) g_tcp_trace[c_][k] = t_;                                            \
    } while (0)
#else
#define TCP_TR(k) \
    do {          \
    } while (0)
#define TCP_CLK(v) \
    do {           \
    } while (0)
#define TCP_ADD(i, v) \
    do {              \
    } while (0)
#endif

namespace tcp {
// Sorted list of the KL smallest keys: insert lo <= hi (KEY_INF = none).  The k-th smallest of
// L u {lo, hi} is min(L[k], max(L[k-1], lo), max(L[k-2], hi)).
template <int KL>
static __device__ __forceinline__ void ins2(uint32_t (&L)[KL], uint32_t lo, uint32_t hi) {
#pragma unroll
    for (int k = KL - 1; k >= 2; --k) L[k] = min(L[k], min(max(L[k - 1], lo), max(L[k - 2], hi)));
    if (KL >= 2) L[1] = min(L[1], min(max(L[0], lo), hi));
    L[0] = min(L[0], lo);
}
template <int KL, typename KT>
static __device__ __forceinline__ void ins1(KT (&L)[KL], KT x) {
#pragma unroll
    for (int k = KL - 1; k >= 1; --k) L[k] = min(L[k], max(L[k - 1], x));
    L[0] = min(L[0], x);
}
// step coprime to n near 0.618 n (scrambled row order)
static __device__ __forceinline__ int row_step(int n) {
    int st = max(1, (int)(0.618f * (float)n));
    for (;; ++st) {
        int x = st, y = n;
        while (y) {
            const int t = x % y;
            x = y;
            y = t;
        }
        if (x == 1) return st;
    }
}
static __device__ __forceinline__ uint32_t win_bits(int lo, int hi, int k) {
    const int a0 = max(lo, 32 * k), a1 = min(hi, 32 * k + 31);
    if (a0 > a1) return 0u;
    const int nb = a1 - a0 + 1;
    return (nb == 32 ? 0xffffffffu : ((1u << nb) - 1u)) << (a0 - 32 * k);
}
}  // namespace tcp

template <int P, int S, int KL, int NBT>
__global__ void __launch_bounds__(tcp::THREADS, 1) match_tcp_kernel(MatchParams p, int mmax) {
    using namespace tcp;
    using SH = Shape<NBT>;
    constexpr int NB = SH::NB, TX = SH::TX, PW = SH::PW, XQ = SH::XQ, XP = SH::XP;
    constexpr int NTS = SH::NTS, SPITCH = SH::SPITCH, TM_A = SH::TM_A;
    static_assert(S % 4 == 0, "window staging in groups of 4 columns needs bS = S b aligned to 4");
    static_assert(TM_A + 8 * P <= (int)TMEM_COLS, "TMEM: accumulator stages + A");
    extern __shared__ __align__(1024) unsigned char sm[];
    const TcpGeom g = TcpGeom::make<NBT>(P, S, p.r);
    const int r = p.r, cb = p.cb;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kr1 = min(p.row_end, p.Ry_reg);
    const int gy0 = p.row_begin + TY * (int)blockIdx.y, gx0 = TX * (int)blockIdx.x;
    const int bimg = blockIdx.z;
    const int cy0 = gy0 * S - r, cx0 = gx0 * S - r;  // image position of candidate (t, j) = (0, 0)
    const int ylo = max(0, p.slab_y0), yhi = min(p.H, p.slab_y1);
    const int16_t* __restrict__ img = p.img + (int64_t)bimg * p.img_bstride;
    int16_t* const raw = reinterpret_cast<int16_t*>(sm + g.off_raw);
    float* const nq = reinterpret_cast<float*>(sm + g.off_nq);
    int* const hs = reinterpret_cast<int*>(sm + g.off_x);
    uint64_t* const tfull = reinterpret_cast<uint64_t*>(sm + g.off_bar);
    uint64_t* const tempty = tfull + NTS;
    int* const misc = reinterpret_cast<int*>(tempty + NTS);  // zmin, zmax, TMEM address
    volatile uint32_t* const gpub = reinterpret_cast<volatile uint32_t*>(misc + 4);  // [NH][128]
    for (int i = threadIdx.x; i < NH * 128; i += THREADS) gpub[i] = KEY_INF;

    if (threadIdx.x == 0) {
        TCP_TR(0);
        for (int i = 0; i < NTS; ++i) {
            tc::mbar_init(&tfull[i], 1);
            tc::mbar_init(&tempty[i], EPI_WARPS);
        }
        misc[0] = INT_MAX;
        misc[1] = INT_MIN;
        tc::fence_mbar_init();
    }
    if (warp == MMA_WARP) tc::tmem_alloc<TMEM_COLS>(reinterpret_cast<uint32_t*>(misc + 2));
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = static_cast<uint32_t>(misc[2]);

    // (1) int16 pixel plane of the tile (0 outside the image / slab and beyond the used columns)
    // and the range of the used pixels
    const int ucols = g.NJ + P - 1;
    {
        int lo = INT_MAX, hi = INT_MIN;
        // 8 loads in flight per thread (the image is L2-resident: latency, not bandwidth)
        for (int i0 = threadIdx.x; i0 < g.PR * PW; i0 += 8 * THREADS) {
            int v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = i0 + k * THREADS;
                const int y = i / PW, x = i - y * PW;
                const int gy = cy0 + y, gx = cx0 + x;
                v[k] = INT_MIN;
                if (i < g.PR * PW && x < ucols && gy >= ylo && gy < yhi && gx >= 0 && gx < p.W)
                    v[k] = __ldg(img + (int64_t)(gy - p.slab_y0) * p.W + gx);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = i0 + k * THREADS;
                if (i < g.PR * PW) {
                    const bool in = v[k] != INT_MIN;
                    if (in) {
                        lo = min(lo, v[k]);
                        hi = max(hi, v[k]);
                    }
                    raw[i] = (int16_t)(in ? v[k] : 0);
                }
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            atomicMin(&misc[0], lo);
            atomicMax(&misc[1], hi);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) TCP_TR(1);
    const int zmin = misc[0], zmax = misc[1];
    const int cz = (zmin + zmax) >> 1;
    const bool fast = max(zmax - cz, cz - zmin) <= mmax;

    // the tile's candidate rows: in the image (slab) and in some valid reference's window
    const int amax = min(TY, kr1 - gy0) - 1;
    const int t_lo = max(0, ylo - cy0);
    const int t_hi = min(min(g.NT - 1, (yhi - P) - cy0), amax * S + 2 * r);
    const int nrow = t_hi - t_lo + 1;

    if (fast) {
        // (2) the centred fp16 plane in place of the int16 one (pixels outside the used area
        // become -c: finite, they only feed masked candidates or the zero columns of A)
        __half* const pl = reinterpret_cast<__half*>(raw);
        for (int i = threadIdx.x; i < g.PR * PW / 8; i += THREADS) {
            const uint4 v = *reinterpret_cast<const uint4*>(raw + 8 * i);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            uint32_t h[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int v0 = (int)(int16_t)(w[e] & 0xffffu) - cz, v1 = (int)(int16_t)(w[e] >> 16) - cz;
                const __half2 h2 = __halves2half2(__int2half_rn(v0), __int2half_rn(v1));
                h[e] = *reinterpret_cast<const uint32_t*>(&h2);
            }
            *reinterpret_cast<uint4*>(raw + 8 * i) = make_uint4(h[0], h[1], h[2], h[3]);
        }
        __syncthreads();
        // (3) horizontal sums of squares hs[y][j] = sum_{jj < P} plane[y][j + jj]^2 (fp32, exact:
        // integers < 2^24 for every used column) into the X region, four columns per task by a
        // running sum
        float* const hsf = reinterpret_cast<float*>(hs);
        for (int i = threadIdx.x; i < g.PR * (NB / 4); i += THREADS) {
            const int y = i / (NB / 4), gq = i - y * (NB / 4);
            const uint2* rp = reinterpret_cast<const uint2*>(pl + y * PW + 4 * gq);
            float sq[16];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint2 v = rp[k];
                const float2 f0 = __half22float2(*reinterpret_cast<const __half2*>(&v.x));
                const float2 f1 = __half22float2(*reinterpret_cast<const __half2*>(&v.y));
                sq[4 * k] = f0.x * f0.x;
                sq[4 * k + 1] = f0.y * f0.y;
                sq[4 * k + 2] = f1.x * f1.x;
                sq[4 * k + 3] = f1.y * f1.y;
            }
            float s0 = 0.f;
#pragma unroll
            for (int k = 0; k < P; ++k) s0 += sq[k];
            float o[4];
            o[0] = s0;
#pragma unroll
            for (int k = 1; k < 4; ++k) {
                s0 += sq[P - 1 + k] - sq[k - 1];
                o[k] = s0;
            }
            *reinterpret_cast<float4*>(hsf + y * NB + 4 * gq) = make_float4(o[0], o[1], o[2], o[3]);
        }
        __syncthreads();
        if (threadIdx.x == 0) TCP_TR(8);
        // (4) candidate norms N_q (vertical running P-row sums per column and row segment;
        // integers <= 2^24, exact in fp32); +inf for candidates outside the image or the tile's
        // columns (they never pass)
        {
            constexpr int NSEG = 3;
            const int seg = (g.NT + NSEG - 1) / NSEG;
            for (int task = threadIdx.x; task < NB * NSEG; task += THREADS) {
                const int j = task % NB, sg = task / NB;
                const int t0 = sg * seg, t1 = min(g.NT, t0 + seg);
                const int cx = cx0 + j;
                const bool colok = j < g.NJ && cx >= 0 && cx <= p.W - P;
                float acc = 0.f;
#pragma unroll
                for (int ii = 0; ii < P - 1; ++ii) acc += hsf[(t0 + ii) * NB + j];
                for (int t = t0; t < t1; ++t) {
                    acc += hsf[(t + P - 1) * NB + j];
                    const int cy = cy0 + t;
                    nq[t * NB + j] = (colok && cy >= ylo && cy <= yhi - P) ? acc : __int_as_float(0x7f800000);
                    acc -= hsf[t * NB + j];
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) TCP_TR(9);
        // (5) X: pre-shifted rows, X[y][q][m] = plane[y][8q + m .. 8q + m + 7]: a lane per
        // 16-byte output (consecutive lanes write consecutive chunks: conflict-free), five
        // 4-byte loads and a byte permute for odd shifts
        for (int i = threadIdx.x; i < (g.PR + 1) * XQ * 8; i += THREADS) {
            const int y = i / (XQ * 8), rem = i - y * (XQ * 8);
            const int q = rem >> 3, m = rem & 7;
            uint32_t o[4] = {0u, 0u, 0u, 0u};
            if (y < g.PR) {
                const uint32_t* wp = reinterpret_cast<const uint32_t*>(pl + y * PW) + ((8 * q + m) >> 1);
                const uint32_t sel = (m & 1) ? 0x5432u : 0x3210u;
                uint32_t w[5];
#pragma unroll
                for (int k = 0; k < 5; ++k) w[k] = wp[k];
#pragma unroll
                for (int k = 0; k < 4; ++k) o[k] = __byte_perm(w[k], w[k + 1], sel);
            }
            *reinterpret_cast<uint4*>(sm + g.off_x + y * XP + q * 128 + m * 16) = make_uint4(o[0], o[1], o[2], o[3]);
        }
        __syncthreads();
        // (6) A: TMEM lane m = reference m holds its patch, K = 16 i + j (j >= P zero), two fp16
        // per column, read from X (patch row i = the 8 pixels at the reference column and the
        // next P - 8); epilogue warp w writes its lane quarter
        if (warp < 4) {
            static_assert(P > 8 && P <= 16 && P % 2 == 0, "A rows: one full and one partial 8-pixel chunk");
            const int m = 32 * warp + lane, a = m >> 3, b = m & 7;
            const int col = b * S + r;
            const unsigned char* xa0 = sm + g.off_x + (a * S + r) * XP + (col >> 3) * 128 + (col & 7) * 16;
#pragma unroll
            for (int c3 = 0; c3 < (P * 8 + 31) / 32; ++c3) {
                uint32_t av[32];
#pragma unroll
                for (int ii = 0; ii < 4; ++ii) {
                    const int i = 4 * c3 + ii;
                    uint4 c0 = make_uint4(0u, 0u, 0u, 0u), c1 = c0;
                    if (i < P) {
                        c0 = *reinterpret_cast<const uint4*>(xa0 + i * XP);
                        c1 = *reinterpret_cast<const uint4*>(xa0 + i * XP + 128);
                    }
                    const uint32_t cw[8] = {c0.x, c0.y, c0.z, c0.w, c1.x, c1.y, c1.z, c1.w};
#pragma unroll
                    for (int e = 0; e < 8; ++e) av[8 * ii + e] = (2 * e < P) ? cw[e] : 0u;
                }
                tc::tmem_st32(tmem + TM_A + 32 * c3 + ((uint32_t)(32 * warp) << 16), av);
            }
            tc::tmem_wait_st();
        }
        tc::fence_proxy_async_smem();  // generic-proxy X stores -> the tensor core
        tc::tc_fence_before();
    }
    __syncthreads();
    tc::tc_fence_after();
    if (threadIdx.x == 0) TCP_TR(2);

    if (warp == MMA_WARP) {
        // ---------------- MMA issuer: 12 x (M128 N80 K16) per candidate row; lane 0 issues
        if (fast && nrow > 0) {
            const uint32_t idesc = tc::idesc_f16f16_f32(128, NB);
            const uint32_t xa = tc::smem_u32(sm + g.off_x);
            const int step = row_step(nrow);
            int tc_ = 0;
            for (int s = 0; s < nrow; ++s) {
                const int ts = s % NTS, t = t_lo + tc_;
                tc_ += step;
                if (tc_ >= nrow) tc_ -= nrow;
                if (s >= NTS) tc::mbar_wait(&tempty[ts], ((s / NTS) - 1) & 1);
                tc::tc_fence_after();
                if (lane == 0) {
#pragma unroll
                    for (int i = 0; i < P; ++i)
                        tc::mma_f16_ts(tmem + (uint32_t)(ts * SPITCH), tmem + TM_A + 8 * i,
                                       tc::smem_desc(xa + (uint32_t)((t + i) * XP), 128, 128), idesc,
                                       i > 0 ? 1u : 0u);
                    tc::mma_commit(&tfull[ts]);
                }
                __syncwarp();
            }
        }
    } else if (warp < EPI_WARPS) {
        // ---------------- warp w: references of TMEM lane quarter w & 3 (lane = reference),
        // window part h = w >> 2
        const int wq = warp & 3, h = warp >> 2;
        const int m = 32 * wq + lane, a = m >> 3, b = m & 7;
        const int ky = gy0 + a, kx = gx0 + b;
        const bool active = b < TX && ky < kr1 && kx < p.Rx_reg;
        const int ry = ky * S, rx = kx * S;  // regular grid positions
        const int nfill = KL - (p.K - 1);    // sentinel zeros below the real keys
        uint32_t L[KL];
#pragma unroll
        for (int i = 0; i < KL; ++i) L[i] = i < nfill ? 0u : KEY_INF;
        const int tdr0 = p.tdr0;
        if (fast) {
            const float Np = nq[(a * S + r) * NB + b * S + r];
            const int wn = 2 * r + 1;         // window columns (<= 43)
            const int nwg = (2 * r) / 4 + 1;  // groups of 4 columns from bS = 4b
            // this warp's part of the window: columns bS + [klo, khi), groups [b + glo, b + ghi)
            const int gsplit = (nwg + 1) / 2;
            const int glo = (NH == 2 && h == 1) ? gsplit : 0;
            const int ghi = (NH == 2 && h == 0) ? gsplit : nwg;
            const int klo = 4 * glo, khi = min(wn, 4 * ghi);
            const uint64_t wmask = active ? (((1ull << khi) - 1ull) & ~((1ull << klo) - 1ull)) : 0ull;
            float* const stg = reinterpret_cast<float*>(sm + g.off_raw) + (32 * warp + lane) * STG_PITCH;
            float* const stgb = stg - 4 * (b + glo);
            const uint32_t taddr = tmem + ((uint32_t)(32 * wq) << 16);
            const int trow0 = 4 * wq * S, trow1 = (4 * wq + 3) * S + 2 * r;
            float T = (float)(tdr0 + 1) - Np;
            const int step = nrow > 0 ? row_step(nrow) : 1;
            int s = 0, tc_ = 0;
            // the warp's next row (rows visited in the scrambled order; the stages of rows no
            // reference of this warp uses are released at once); -1 after the last
            auto next_row = [&](int& ts_out) -> int {
                while (s < nrow) {
                    const int ts = s % NTS, t = t_lo + tc_;
                    tc::mbar_wait(&tfull[ts], (s / NTS) & 1);
                    tc::tc_fence_after();
                    ++s;
                    tc_ += step;
                    if (tc_ >= nrow) tc_ -= nrow;
                    if (t >= trow0 && t <= trow1) {
                        ts_out = ts;
                        return t;
                    }
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive(&tempty[ts]);
                }
                return -1;
            };
            uint32_t acc[NB];
            auto load_acc = [&](int tsx) {
#pragma unroll
                for (int c = 0; c < NB / 16; ++c)
                    tc::tmem_ld16p(taddr + (uint32_t)(tsx * SPITCH + 16 * c), acc + 16 * c);
            };
            // the row's candidate norms in registers, loaded with its accumulators (ahead of use)
            float4 nqv[NB / 4];
            auto load_nq = [&](int tx) {
                const float4* nqr = reinterpret_cast<const float4*>(nq + tx * NB);
#pragma unroll
                for (int c = 0; c < NB / 4; ++c) nqv[c] = nqr[c];
            };
            int ts = 0;
            int t = next_row(ts);
            if (t >= 0) {
                load_acc(ts);
                load_nq(t);
            }
            while (t >= 0) {
                long long k0 = 0, k1 = 0, k2 = 0, k3 = 0;
                (void)k0; (void)k1; (void)k2; (void)k3;
                TCP_CLK(k0);
                tc::tmem_wait_ld();
#pragma unroll
                for (int c = 0; c < NB / 16; ++c) tc::tmem_tie16(acc + 16 * c);
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&tempty[ts]);
                // u = N_q - 2 <f_p, f_q> (exact for every passing candidate); the lane's groups
                // staged; pass bits = sign of u - T, bit j of word j / 32
                uint32_t mk[3] = {0u, 0u, 0u};
#pragma unroll
                for (int c = NB / 4 - 1; c >= 0; --c) {
                    const float nv[4] = {nqv[c].x, nqv[c].y, nqv[c].z, nqv[c].w};
                    float u[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) u[e] = fmaf(-2.f, __uint_as_float(acc[4 * c + e]), nv[e]);
                    if ((unsigned)(c - b - glo) < (unsigned)(ghi - glo))
                        *reinterpret_cast<float4*>(stgb + 4 * c) = make_float4(u[0], u[1], u[2], u[3]);
#pragma unroll
                    for (int e = 3; e >= 0; --e) {
                        const int j = 4 * c + e;
                        mk[j >> 5] = __funnelshift_l(__float_as_uint(u[e] - T), mk[j >> 5], 1);
                    }
                }
                // window-relative 64-bit mask: bit k = column bS + k = displacement dx + r
                const int tt = t - a * S;
                const int bs = b * S;
                uint64_t mw = (((uint64_t)mk[1] << 32) | mk[0]) >> bs;
                if (bs > 0) mw |= (uint64_t)mk[2] << (64 - bs);
                mw &= ((unsigned)tt <= (unsigned)(2 * r)) ? wmask : 0ull;
                if (tt == r) mw &= ~(1ull << r);  // the reference itself (slot 0)
                TCP_CLK(k1);
                // the next row's accumulators load while this row's keys are inserted
                int tsn = 0;
                const int tn = next_row(tsn);
                if (tn >= 0) {
                    load_acc(tsn);
                    load_nq(tn);
                }
                TCP_CLK(k2);
                const uint32_t cbase = (uint32_t)(tt * p.side);
                auto pop = [&]() -> uint32_t {
                    const int j = __ffsll((long long)mw) - 1;
                    mw &= mw - 1ull;
                    const uint32_t key =
                        (__float2uint_rn(stg[max(j - klo, 0)] + Np) << cb) | (cbase + (uint32_t)j);
                    return j >= 0 ? key : KEY_INF;
                };
                int nr_ = 0;
                (void)nr_;
                while (__any_sync(0xffffffffu, mw != 0ull)) {
#if GBM3D_TCP_TRACE
                    ++nr_;
#endif
                    const uint32_t k1 = pop(), k2 = pop();
                    ins2<KL>(L, min(k1, k2), max(k1, k2));
                }
                TCP_CLK(k3);
                TCP_ADD(0, k2 - k1);
                TCP_ADD(1, k1 - k0);
                TCP_ADD(2, k3 - k2);
                TCP_ADD(3, nr_);
                TCP_ADD(4, 1);
                // gate: the (K-1)-th key of this list or of the partner's (either bounds the
                // union's (K-1)-th)
                uint32_t gk = L[KL - 1];
                if (NH == 2) {
                    gpub[h * 128 + m] = gk;
                    gk = min(gk, gpub[(1 - h) * 128 + m]);
                }
                const int gd = min((int)(gk >> cb), tdr0);
                T = (float)(gd + 1) - Np;
                t = tn;
                ts = tsn;
            }
            if (NH == 2) {
                // merge: part 1 hands its list over (through the norms' buffer, dead once every
                // row is scanned; X stays intact), part 0 inserts the partner's K - 1 real keys
                asm volatile("bar.sync 1, %0;" ::"r"(32 * EPI_WARPS) : "memory");
                uint32_t* const mb = reinterpret_cast<uint32_t*>(sm + g.off_nq);
                if (h == 1) {
#pragma unroll
                    for (int i = 0; i < KL; ++i) mb[i * 128 + m] = L[i];
                }
                asm volatile("bar.sync 1, %0;" ::"r"(32 * EPI_WARPS) : "memory");
                if (h == 0) {
                    for (int i = nfill; i < KL; i += 2) {
                        const uint32_t lo = mb[i * 128 + m], hi = i + 1 < KL ? mb[(i + 1) * 128 + m] : KEY_INF;
                        if (!__any_sync(0xffffffffu, lo < L[KL - 1])) break;
                        ins2<KL>(L, lo, hi);
                    }
                }
            }
        } else if (active && h == 0) {
            // ---------------- exact int32 path for a tile above the fp16 bound: direct Eq. (1)
            const int pa = a * S + r, pb = b * S + r;  // the reference's plane position
            for (int dy = -r; dy <= r; ++dy) {
                const int cy = ry + dy;
                if (cy < ylo || cy > yhi - P) continue;
                for (int dx = -r; dx <= r; ++dx) {
                    const int cx = rx + dx;
                    if (cx < 0 || cx > p.W - P || (dy == 0 && dx == 0)) continue;
                    int d = 0;
                    for (int i = 0; i < P; ++i) {
                        const int16_t* r0 = raw + (pa + i) * PW + pb;
                        const int16_t* r1 = raw + (pa + dy + i) * PW + pb + dx;
#pragma unroll
                        for (int jj = 0; jj < P; ++jj) {
                            const int df = (int)r0[jj] - (int)r1[jj];
                            d += df * df;
                        }
                    }
                    if (d <= tdr0)
                        ins1<KL, uint32_t>(L, ((uint32_t)d << cb) | (uint32_t)((dy + r) * p.side + dx + r));
                }
            }
        }
        // ---------------- tau - 1 above the 32-bit key's d range (dsat): keys stop at d <= dsat,
        // so a list that ended short may miss valid candidates with larger d; such a reference
        // is recomputed exactly (direct Eq. (1) in int32, 64-bit keys d << 32 | code) from the
        // pixels still in shared memory (X in the fp16 path, the int16 plane otherwise)
        bool exact64 = false;
        uint64_t L64[KL];
        if (p.tau_above_dsat && active && h == 0) {
            int nreal = 0;
#pragma unroll
            for (int i = 0; i < KL; ++i) nreal += (i >= nfill && L[i] != KEY_INF) ? 1 : 0;
            if (nreal < p.K - 1) {
                exact64 = true;
#pragma unroll
                for (int i = 0; i < KL; ++i) L64[i] = i < nfill ? 0ull : ~0ull;
                const int pa = a * S + r, pb = b * S + r;
                auto pix = [&](int y, int x) -> int {
                    if (fast)
                        return __half2int_rn(*reinterpret_cast<const __half*>(
                            sm + g.off_x + y * XP + (x >> 3) * 128 + (x & 7) * 16));
                    return (int)raw[y * PW + x];
                };
                for (int dy = -r; dy <= r; ++dy) {
                    const int cy = ry + dy;
                    if (cy < ylo || cy > yhi - P) continue;
                    for (int dx = -r; dx <= r; ++dx) {
                        const int cx = rx + dx;
                        if (cx < 0 || cx > p.W - P || (dy == 0 && dx == 0)) continue;
                        int d = 0;
                        for (int i = 0; i < P; ++i)
                            for (int jj = 0; jj < P; ++jj) {
                                const int df = pix(pa + i, pb + jj) - pix(pa + dy + i, pb + dx + jj);
                                d += df * df;
                            }
                        if ((int64_t)d < p.tau)
                            ins1<KL, uint64_t>(L64, ((uint64_t)(uint32_t)d << 32) |
                                                        (uint64_t)((dy + r) * p.side + dx + r));
                    }
                }
            }
        }
        if (lane == 0 && warp < 4) TCP_TR(3 + warp);
        // ---------------- output (part 0): slot 0 = self, ranks 1 .. K-1, pads (self, -1)
        if (active && h == 0) {
            const int self = ry * p.W + rx;
            const int64_t ref = (int64_t)bimg * p.out_bstride + (int64_t)(ky - p.row_begin) * p.Rx + kx;
            int32_t* const oi = p.idx + ref * p.K;
            int32_t* const od = p.dist + ref * p.K;
            oi[0] = self;
            od[0] = 0;
            int cnt = 0;
            const uint32_t cmask = (1u << cb) - 1u;
#pragma unroll
            for (int i = 0; i < KL; ++i) {
                const int s = i - nfill + 1;
                if (s >= 1) {
                    const bool valid = exact64 ? L64[i] != ~0ull : L[i] != KEY_INF;
                    if (valid) {
                        const int code = exact64 ? (int)(uint32_t)L64[i] : (int)(L[i] & cmask);
                        const int dy = code / p.side - r, dx = code - (code / p.side) * p.side - r;
                        oi[s] = (ry + dy) * p.W + rx + dx;
                        od[s] = exact64 ? (int)(L64[i] >> 32) : (int)(L[i] >> cb);
                        ++cnt;
                    } else {
                        oi[s] = self;
                        od[s] = -1;
                    }
                }
            }
            if (p.nvalid) p.nvalid[ref] = 1 + cnt;
        }
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (warp == MMA_WARP) tc::tmem_dealloc<TMEM_COLS>(tmem);
    if (threadIdx.x == 0) TCP_TR(7);
}

// Largest tile half-range M with P^2 M^2 <= 2^24 (and |z - c| <= 2048 for fp16).
static inline int tcp_default_mmax(int P) {
    int M = 0;
    while (M < 2048 && (long long)P * P * (M + 1) * (M + 1) <= (1LL << 24)) ++M;
    return M;
}

template <int P, int S, int KL, int NBT>
cudaError_t launch_tcp(const MatchParams& p, cudaStream_t stream, int* launches) {
    const int kr0 = p.row_begin, kr1 = p.row_end < p.Ry_reg ? p.row_end : p.Ry_reg;
    if (kr1 <= kr0 || p.Rx_reg <= 0) return cudaSuccess;
    const TcpGeom g = TcpGeom::make<NBT>(P, S, p.r);
    constexpr int TX = tcp::Shape<NBT>::TX;
    auto kern = match_tcp_kernel<P, S, KL, NBT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, g.total);
    if (e != cudaSuccess) return e;
    // dev / test switch: a lower bound forces tiles onto the exact int32 path
    static const int mmax_env = getenv("GBM3D_TCP_MMAX") ? atoi(getenv("GBM3D_TCP_MMAX")) : -1;
    const int mmax = mmax_env >= 0 ? mmax_env : tcp_default_mmax(P);
    dim3 grid((p.Rx_reg + TX - 1) / TX, (kr1 - kr0 + tcp::TY - 1) / tcp::TY, p.B);
    kern<<<grid, tcp::THREADS, g.total, stream>>>(p, mmax);
    if (launches) ++*launches;
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    static const bool dbg = getenv("GBM3D_DEBUG") != nullptr;
    if (dbg) {
        e = cudaStreamSynchronize(stream);
        fprintf(stderr, "gbm3d: tcp P%d S%d N%d grid %u x %u x %u smem %d: %s\n", P, S, NBT, grid.x,
                grid.y, grid.z, g.total, cudaGetErrorString(e));
    }
    return e;
}

}  // namespace gbm3d
