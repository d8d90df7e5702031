// Product-form block matching on the tensor cores, fp16 operands.
//
// Same method as match_tc.cuh (Eq. (2): d = ||f_p||^2 + ||f_q||^2 - 2 <f_p, f_q>),
// but one MMA per candidate row instead of four byte-plane products:
//   * each CTA centres its pixel tile on c = (min + max) / 2 of the tile (the SSD is translation
//     invariant) and stores z - c as fp16, exact for |z - c| <= 2048;
//   * <f_p, f_q> = sum of 64 integer products runs as tcgen05.mma kind::f16 with an fp32
//     accumulator.  Every partial sum is an integer of magnitude <= 64 M^2 (M = max |z - c|);
//     for M <= TC16_MMAX = 362 that is < 2^23, and so are the norms and u = N_q - 2 <f_p, f_q>,
//     so all of it is exact in fp32 (the accumulator is checked exact for integer dot products
//     up to 2^24 by tools/dev/mma_f16_test.cu).  The gate test u < gate - N_p is exact, and so
//     is d = u + N_p for every candidate that passes it (d < gate <= 2^21).
//   * a tile whose range exceeds the bound is not computed here: its first reference gets
//     dist slot 0 = TC_TILE_MARK and the exact int8 kernel (match_tc.cuh) redoes such tiles.
//
// Work mapping: CTA = 16 x 8 grid references (M = 128, TMEM lane m =
// reference 8a + b).  The B operand needs no per-row building: the prologue writes the tile's
// fp16 plane once in a pre-shifted layout X[y][q][m][0..7] = plane[y][8q + m + 0..7] (each
// 16-byte chunk is candidate column 8q + m's patch row at image row y), so candidate row t's
// 64 patches are the K-major canonical operand at X + t * 1 KB with LBO = 1 KB (next patch row)
// and SBO = 128 B (next 8 candidates).  One thread issues 4 MMAs (M128 N64 K16) per candidate
// row into one of NTS = 8 TMEM stages (64 columns each, one fp32 accumulator); epilogue warp w
// (lane quarter w) turns its 32 x 64 accumulators into u and a pass mask and stages them;
// selector warp w keeps the 32 per-lane sorted top-(K-1) register lists (insertion network,
// one round per pass).
#pragma once
#include <cuda_fp16.h>

#include "match_tc.cuh"

namespace gbm3d {

namespace tc16 {
constexpr int TY = 16, TX = 8;
constexpr int NB = 64;           // candidate columns per MMA tile (N)
constexpr int PCH = 72;          // fp16 plane pitch in elements (64 + 7 + pad)
constexpr int NTS = 8;           // TMEM stages (64 columns each)
constexpr int EPI_WARPS = 4, SEL_WARP0 = 4, MMA_WARP = 8;  // epilogue w, selector 4 + w, MMA
constexpr int THREADS = 32 * (MMA_WARP + 1);
constexpr int NSLOT = 2;         // staged rows per lane quarter (epilogue one row ahead)
constexpr int STG_PITCH = 68;    // words per lane and staged row: u[64], mask lo/hi, gate, row
constexpr int A_BYTES = 128 * 128;
constexpr int XP = (NB / 8) * 128;  // bytes per pre-shifted plane row (8 chunks of 8 x 16 B)
constexpr uint32_t TMEM_COLS = 512;
constexpr int MMAX = 362;        // exactness bound on max |z - c| (see header)
#ifndef GBM3D_TC16_BULK_MIN
#define GBM3D_TC16_BULK_MIN 16
#endif
constexpr int BULK_MIN = GBM3D_TC16_BULK_MIN;
#ifndef GBM3D_TC16_PREFETCH
#define GBM3D_TC16_PREFETCH 1
#endif  // rows with this many passes (max over lanes) merge in bulk
}  // namespace tc16

struct Tc16Geom {
    int NT, PR, NJ;
    int off_a, off_x, off_nc, off_stg, off_bar, total;
    __host__ __device__ static Tc16Geom make(int S, int r) {
        using namespace tc16;
        Tc16Geom g;
        g.NT = 15 * S + 2 * r + 1;
        g.PR = g.NT + 7;
        g.NJ = 7 * S + 2 * r + 1;
        g.off_a = 0;
        g.off_x = A_BYTES;                 // pre-shifted plane
        g.off_nc = g.off_x + g.PR * XP;
        g.off_stg = g.off_nc + g.NT * NB * 4;  // raw tile, fp16 plane, squares before the loop
        g.off_bar = g.off_stg + EPI_WARPS * NSLOT * 32 * STG_PITCH * 4;
        // tfull/tempty[NTS], sfull/sempty[EPI_WARPS*NSLOT]; gates[128], consumed[EPI_WARPS],
        // range scratch[2], TMEM address
        g.total = g.off_bar + (2 * NTS + 2 * EPI_WARPS * NSLOT) * 8 +
                  (EPI_WARPS * 32 + EPI_WARPS + 2 + 1) * 4 + 16;
        return g;
    }
};

// Two keys into a sorted list of N in one pass: the k-th smallest of L and {lo <= hi} is
// min(L[k], max(L[k-1], lo), max(L[k-2], hi)) (merge of sorted lists), i.e. two max and one
// 3-input min (VIMNMX3) per element -- 1.5 ALU ops per key and element instead of 2, and the
// two keys share one dependency chain (tools/dev/insert_bench.cu: 1.5x keys per cycle).
template <int N>
static __device__ __forceinline__ void list_insert2(uint32_t (&L)[N], uint32_t x, uint32_t y) {
    const uint32_t lo = min(x, y), hi = max(x, y);
#pragma unroll
    for (int i = N - 1; i >= 2; --i) L[i] = __vimin3_u32(L[i], max(L[i - 1], lo), max(L[i - 2], hi));
    L[1] = __vimin3_u32(L[1], max(L[0], lo), hi);
    L[0] = min(L[0], lo);
}

// Ascending bitonic sort of N (power of two) register keys; fully unrolled min/max network.
template <int N>
static __device__ __forceinline__ void bitonic_sort(uint32_t (&B)[N]) {
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
            for (int i = 0; i < N; ++i) {
                const int l = i ^ j;
                if (l > i) {
                    const uint32_t lo = min(B[i], B[l]), hi = max(B[i], B[l]);
                    const bool asc = (i & k) == 0;
                    B[i] = asc ? lo : hi;
                    B[l] = asc ? hi : lo;
                }
            }
        }
    }
}
// L (ascending, N keys) <- the N smallest of L and B (any order): sort B, take the lower half
// of the bitonic sequence L ++ reverse(B) (min(L[i], B[N-1-i])), then one bitonic clean-up.
template <int N>
static __device__ __forceinline__ void bulk_merge(uint32_t (&L)[N], uint32_t (&B)[N]) {
    bitonic_sort<N>(B);
#pragma unroll
    for (int i = 0; i < N; ++i) L[i] = min(L[i], B[N - 1 - i]);
#pragma unroll
    for (int j = N >> 1; j > 0; j >>= 1) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const int l = i ^ j;
            if (l > i) {
                const uint32_t lo = min(L[i], L[l]), hi = max(L[i], L[l]);
                L[i] = lo;
                L[l] = hi;
            }
        }
    }
}

// L (ascending, N keys) <- the N smallest of L and 8 more keys B (any order).
template <int N>
static __device__ __forceinline__ void bulk_merge8(uint32_t (&L)[N], uint32_t (&B)[8]) {
    bitonic_sort<8>(B);
#pragma unroll
    for (int i = N - 8; i < N; ++i) L[i] = min(L[i], B[N - 1 - i]);
#pragma unroll
    for (int j = N >> 1; j > 0; j >>= 1) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            const int l = i ^ j;
            if (l > i) {
                const uint32_t lo = min(L[i], L[l]), hi = max(L[i], L[l]);
                L[i] = lo;
                L[l] = hi;
            }
        }
    }
}

// 8 consecutive fp16 (16 bytes) starting at element c of a 4-byte aligned shared row.
static __device__ __forceinline__ uint4 load16h(const __half* row, int c) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(row) + (c >> 1);
    const uint32_t sh = (uint32_t)(c & 1) * 16u;
    const uint32_t a0 = w[0], a1 = w[1], a2 = w[2], a3 = w[3], a4 = w[4];
    return make_uint4(__funnelshift_r(a0, a1, sh), __funnelshift_r(a1, a2, sh),
                      __funnelshift_r(a2, a3, sh), __funnelshift_r(a3, a4, sh));
}

// Canonical K-major offset of (row, patch row i) for 128-byte K rows (64 fp16): core matrix
// (row/8, i) at (row/8)*1024 + i*128, row-in-core * 16; patch row i = 8 fp16 = 16 bytes.
static __device__ __forceinline__ int kmaj16_off(int row, int i) {
    return (row >> 3) * 1024 + i * 128 + (row & 7) * 16;
}

// Candidate-row order of a tile.  Two "fill" rows first: f1 lies in the search window of every
// reference of warps 0-2 and is outside warp 3's rows, f2 lies in every window of warp 3 and
// outside warps 0-1's rows.  A warp's lists then all fill on the same row (one 39-round burst
// per warp instead of one per reference row), after which the scrambled order follows.
struct RowSeq {
    int lo, n, step, off, f[2], npre, pre;
    __device__ void init(int S, int r, int t_lo, int t_hi) {
        lo = t_lo;
        n = t_hi - t_lo + 1;
        step = tc_step(n);
        off = 0;
        pre = 0;
        npre = 0;
        const int a1 = 11 * S, b1 = min(2 * r, 12 * S - 1);
        const int a2 = max(15 * S, 7 * S + 2 * r + 1), b2 = 12 * S + 2 * r;
        const int f1 = (a1 + b1) / 2, f2 = (a2 + b2) / 2;
        if (a1 <= b1 && a2 <= b2 && f1 >= t_lo && f2 <= t_hi) {
            f[0] = f1;
            f[1] = f2;
            npre = 2;
        }
    }
    __device__ int next() {
        if (pre < npre) return f[pre++];
        for (;;) {
            const int t = lo + off;
            off = tc_next(off, n, step);
            if (npre == 0 || (t != f[0] && t != f[1])) return t;
        }
    }
};

template <int S, int KL>
__global__ void __launch_bounds__(tc16::THREADS, 1) match_tc16_kernel(MatchParams p) {
    using namespace tc16;
    extern __shared__ __align__(1024) unsigned char sm[];
    if (threadIdx.x == 0) TC_TR(2, clock64());
    if (threadIdx.x == 0) { TC_SPAN(0, gtimer()); TC_SPAN(2, (long long)smid()); }
    const Tc16Geom g = Tc16Geom::make(S, p.r);
    constexpr int P = 8;
    const int r = p.r;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bimg = blockIdx.z;
    const int kr1 = min(p.row_end, p.Ry_reg);
    const int ky0 = p.row_begin + (int)blockIdx.y * TY, kx0 = (int)blockIdx.x * TX;
    const int gy0 = S * ky0 - r, gx0 = S * kx0 - r;
    const int16_t* __restrict__ img = p.img + (int64_t)bimg * p.img_bstride;

    // raw int16 tile and the fp16 plane live in the (not yet used) staging area
    int16_t* const raw = reinterpret_cast<int16_t*>(sm + g.off_stg);
    __half* const pl = reinterpret_cast<__half*>(sm + g.off_stg + g.PR * PCH * 2);
    float* const nc = reinterpret_cast<float*>(sm + g.off_nc);
    uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + g.off_bar);
    uint64_t* const tfull = bars;
    uint64_t* const tempty = tfull + NTS;
    uint64_t* const sfull = tempty + NTS;
    uint64_t* const sempty = sfull + EPI_WARPS * NSLOT;
    volatile int* const gate_pub = reinterpret_cast<volatile int*>(sempty + EPI_WARPS * NSLOT);
    // rows taken by selector (w, h)
    volatile int* const consumed = gate_pub + EPI_WARPS * 32;    // rows taken by selector w
    int* const rng = const_cast<int*>(consumed + EPI_WARPS);     // tile min, max
    uint32_t* const tslot = reinterpret_cast<uint32_t*>(rng + 2);

    const int t_lo = max(0, -gy0), t_hi = min(g.NT - 1, (p.H - P) - gy0);
    const int j_lo = max(0, -gx0), j_hi = min(g.NJ - 1, (p.W - P) - gx0);
    const int nseq = t_hi - t_lo + 1;

    // ---- prologue.  Work items are (row, 8-column segment) of the PR x 72 pixel tile: raw
    // int16 (pitch 144 B), the centred fp16 plane, the horizontal squares and the norms all live
    // in the staging area, which the main loop only uses afterwards.
    constexpr int SEG = PCH / 8;                                // 9 segments of 8 columns
    constexpr int NIT = (95 * SEG + THREADS - 1) / THREADS;     // PR <= 95 (radius <= 21)
    int* const hs = reinterpret_cast<int*>(sm + g.off_stg + 2 * g.PR * PCH * 2);
    const int ylo = max(0, p.slab_y0), yhi = min(p.H, p.slab_y1);
    {
        // L2 prefetch of the rows a tile two tile-rows below needs (likely a CTA of a later
        // wave): its first touch of HBM overlaps this tile's work instead of its own prologue
        if (GBM3D_TC16_PREFETCH && threadIdx.x < 2 * g.PR) {
            const int gy = gy0 + 2 * TY * S + (threadIdx.x >> 1);
            const int gx = max(0, gx0) + 64 * (threadIdx.x & 1);
            if (gy >= ylo && gy < yhi && gx < p.W)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(img + (int64_t)(gy - p.slab_y0) * p.W + gx));
        }
        if (threadIdx.x == 0) {
            rng[0] = INT_MAX;
            rng[1] = INT_MIN;
        }
        __syncthreads();
        int lo = INT_MAX, hi = INT_MIN;
        int16_t z[NIT][8];
#pragma unroll
        for (int k = 0; k < NIT; ++k) {  // all loads of a thread in flight together
            const int task = threadIdx.x + k * THREADS;
            const int row = task / SEG, seg = task - row * SEG;
            const int gy = gy0 + row, gx = gx0 + 8 * seg;
            const bool rowok = task < g.PR * SEG && gy >= ylo && gy < yhi;
            const int16_t* src = img + (int64_t)(gy - p.slab_y0) * p.W;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const bool in = rowok && gx + j >= 0 && gx + j < p.W;
                z[k][j] = in ? src[gx + j] : (int16_t)0;
                if (in) {
                    lo = min(lo, (int)z[k][j]);
                    hi = max(hi, (int)z[k][j]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < NIT; ++k) {
            const int task = threadIdx.x + k * THREADS;
            if (task < g.PR * SEG) {
                uint4 v;
                v.x = (uint32_t)(uint16_t)z[k][0] | ((uint32_t)(uint16_t)z[k][1] << 16);
                v.y = (uint32_t)(uint16_t)z[k][2] | ((uint32_t)(uint16_t)z[k][3] << 16);
                v.z = (uint32_t)(uint16_t)z[k][4] | ((uint32_t)(uint16_t)z[k][5] << 16);
                v.w = (uint32_t)(uint16_t)z[k][6] | ((uint32_t)(uint16_t)z[k][7] << 16);
                *reinterpret_cast<uint4*>(raw + task * 8) = v;  // row * PCH + 8 seg == 8 task
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        if (lane == 0) {
            atomicMin(&rng[0], lo);
            atomicMax(&rng[1], hi);
        }
        __syncthreads();
        if (threadIdx.x == 0) TC_TR(3, clock64());
    }
    const int zlo = rng[0], zhi = rng[1];
    const int cz = (zlo + zhi) >> 1;
    if (max(zhi - cz, cz - zlo) > MMAX) {  // outside the fp16/fp32 exactness bound
        if (threadIdx.x == 0) {
            const int64_t ref = (int64_t)bimg * p.out_bstride + (int64_t)(ky0 - p.row_begin) * p.Rx + kx0;
            p.dist[ref * p.K] = TC_TILE_MARK;
        }
        return;
    }
    {
        // centre on cz; pixels outside the image only feed masked candidates: 0 (= cz)
        for (int task = threadIdx.x; task < g.PR * SEG; task += THREADS) {
            const int row = task / SEG, seg = task - row * SEG;
            const int gy = gy0 + row, gx = gx0 + 8 * seg;
            const bool rowok = gy >= ylo && gy < yhi;
            const uint4 rv = *reinterpret_cast<const uint4*>(raw + task * 8);
            const uint32_t rw[4] = {rv.x, rv.y, rv.z, rv.w};
            uint32_t iw[4], hw[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int j = 2 * q;
                const bool in0 = rowok && gx + j >= 0 && gx + j < p.W;
                const bool in1 = rowok && gx + j + 1 >= 0 && gx + j + 1 < p.W;
                const int v0 = in0 ? (int)(int16_t)(rw[q] & 0xffffu) - cz : 0;
                const int v1 = in1 ? (int)(int16_t)(rw[q] >> 16) - cz : 0;
                iw[q] = (uint32_t)(uint16_t)v0 | ((uint32_t)(uint16_t)v1 << 16);
                const __half2 h2 = __halves2half2(__int2half_rn(v0), __int2half_rn(v1));
                hw[q] = *reinterpret_cast<const uint32_t*>(&h2);
            }
            *reinterpret_cast<uint4*>(raw + task * 8) = make_uint4(iw[0], iw[1], iw[2], iw[3]);
            *reinterpret_cast<uint4*>(pl + task * 8) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
        }
        if (threadIdx.x == 0) {
            for (int i = 0; i < NTS; ++i) {
                tc::mbar_init(&tfull[i], 1);
                tc::mbar_init(&tempty[i], EPI_WARPS);
            }
            for (int i = 0; i < EPI_WARPS * NSLOT; ++i) {
                tc::mbar_init(&sfull[i], 1);
                tc::mbar_init(&sempty[i], 1);
            }
            tc::fence_mbar_init();
        }
        if (warp == MMA_WARP) tc::tmem_alloc<TMEM_COLS>(tslot);
        if (threadIdx.x < EPI_WARPS * 32) gate_pub[threadIdx.x] = p.tdr0 + 1;
        if (threadIdx.x < EPI_WARPS) consumed[threadIdx.x] = 0;
        __syncthreads();  // centred raw values and the fp16 plane complete
        if (threadIdx.x == 0) TC_TR(4, clock64());
        // horizontal P-sums of squares hs[y][n] (n < 64), 8 columns per item (sliding sum)
        for (int task = threadIdx.x; task < g.PR * 8; task += THREADS) {
            const int y = task >> 3, k = task & 7;
            const uint4 r0 = *reinterpret_cast<const uint4*>(raw + y * PCH + 8 * k);
            const uint4 r1 = *reinterpret_cast<const uint4*>(raw + y * PCH + 8 * k + 8);
            const uint32_t rw[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
            int sq[16];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const int a0 = (int)(int16_t)(rw[q] & 0xffffu), a1 = (int)(int16_t)(rw[q] >> 16);
                sq[2 * q] = a0 * a0;
                sq[2 * q + 1] = a1 * a1;
            }
            int o[8];
            int sacc = 0;
#pragma unroll
            for (int j = 0; j < P; ++j) sacc += sq[j];
            o[0] = sacc;
#pragma unroll
            for (int i = 1; i < 8; ++i) {
                sacc += sq[i + P - 1] - sq[i - 1];
                o[i] = sacc;
            }
            *reinterpret_cast<int4*>(hs + y * NB + 8 * k) = make_int4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<int4*>(hs + y * NB + 8 * k + 4) = make_int4(o[4], o[5], o[6], o[7]);
        }
        // pre-shifted plane X[y][q][m] = plane[y][8q + m .. 8q + m + 7]; one 16-byte chunk per
        // item, consecutive lanes on consecutive chunks (conflict-free stores)
        uint8_t* const xop = sm + g.off_x;
        for (int u = threadIdx.x; u < g.PR * NB; u += THREADS) {
            const int y = u >> 6, n = u & 63;
            *reinterpret_cast<uint4*>(xop + y * XP + n * 16) = load16h(pl + y * PCH, n);
        }
        // A operand (K-major core matrices): reference m's patch row i
        uint8_t* const a_op = sm + g.off_a;
        for (int u = threadIdx.x; u < 128 * P; u += THREADS) {
            const int i = u >> 7, m = u & 127;
            const int row = r + S * (m >> 3) + i, col = r + S * (m & 7);
            *reinterpret_cast<uint4*>(a_op + kmaj16_off(m, i)) = load16h(pl + row * PCH, col);
        }
        tc::fence_proxy_async_smem();  // X and A (generic-proxy stores) -> the tensor core
        tc::tc_fence_before();
        __syncthreads();
        tc::tc_fence_after();
        if (threadIdx.x == 0) TC_TR(5, clock64());
    }
    const uint32_t tmem = *tslot;
    if (threadIdx.x == 0) TC_TR(0, clock64());

    if (warp != MMA_WARP) {
        // candidate norms N_q = vertical P-sums of hs (<= 64 M^2 < 2^24: exact in fp32), only
        // read by the epilogue: warps 0-7 make them while the MMA warp starts the first rows;
        // a named barrier over those 256 threads closes the phase (hs lives in the staging
        // area the epilogue overwrites afterwards)
        for (int task = threadIdx.x; task < g.NT * 8; task += 32 * MMA_WARP) {
            const int t = task >> 3, k = task & 7;
            int o[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
            for (int i = 0; i < P; ++i) {
                const int4 a0 = *reinterpret_cast<const int4*>(hs + (t + i) * NB + 8 * k);
                const int4 a1 = *reinterpret_cast<const int4*>(hs + (t + i) * NB + 8 * k + 4);
                o[0] += a0.x; o[1] += a0.y; o[2] += a0.z; o[3] += a0.w;
                o[4] += a1.x; o[5] += a1.y; o[6] += a1.z; o[7] += a1.w;
            }
            *reinterpret_cast<float4*>(nc + t * NB + 8 * k) =
                make_float4((float)o[0], (float)o[1], (float)o[2], (float)o[3]);
            *reinterpret_cast<float4*>(nc + t * NB + 8 * k + 4) =
                make_float4((float)o[4], (float)o[5], (float)o[6], (float)o[7]);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(32 * MMA_WARP) : "memory");
    }

    if (warp == MMA_WARP) {
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_f16f16_f32(128, NB);
            const uint32_t aa = tc::smem_u32(sm + g.off_a);
            const uint32_t xa = tc::smem_u32(sm + g.off_x);
            RowSeq seq;
            seq.init(S, r, t_lo, t_hi);
            for (int s = 0; s < nseq; ++s) {
                const int ts = s % NTS;
                const int t = seq.next();
                if (s >= NTS) tc::mbar_wait(&tempty[ts], ((s / NTS) - 1) & 1);
                tc::tc_fence_after();
                const uint32_t bb = xa + (uint32_t)(t * XP);
#pragma unroll
                for (int ks = 0; ks < 4; ++ks)
                    tc::mma_f16(tmem + (uint32_t)(ts * NB), tc::smem_desc(aa + ks * 256, 128, 1024),
                                tc::smem_desc(bb + ks * 2 * XP, XP, 128), idesc, ks);
                tc::mma_commit(&tfull[ts]);
                TC_TR(16 + s, clock64());
            }
        }
        __syncwarp();
    } else {
        const bool is_sel = warp >= SEL_WARP0;
        const int w = is_sel ? warp - SEL_WARP0 : warp;
        const int a = 4 * w + (lane >> 3), bb = lane & 7;
        const bool refok = (ky0 + a < kr1) && (kx0 + bb < p.Rx_reg) && (p.K > 1);
        const int ty = r + S * a, tx = r + S * bb;
        const bool warp_active = __any_sync(0xffffffffu, refok);
        const int wt0 = S * 4 * w, wt1 = S * (4 * w + 3) + 2 * r;
        const uint32_t side = (uint32_t)p.side;
        const int cb = p.cb;
        const float Nr = nc[ty * NB + tx];
        uint32_t* const stg0 = reinterpret_cast<uint32_t*>(sm + g.off_stg) +
                               (w * NSLOT * 32 + lane) * STG_PITCH;
        int used = 0;
        if (!is_sel) {
            const int c0 = max(S * bb, j_lo), c1 = min(S * bb + 2 * r, j_hi);
            const uint64_t cm = (c1 >= c0) ? ((c1 >= 63 ? ~0ull : ((2ull << c1) - 1ull)) &
                                              ~((1ull << c0) - 1ull))
                                           : 0ull;
            const uint32_t taddr = tmem + ((uint32_t)(32 * w) << 16);
            const int gate0 = p.tdr0 + 1;
            RowSeq seq;
            seq.init(S, r, t_lo, t_hi);
            for (int s = 0; s < nseq; ++s) {
                const int ts = s % NTS;
                const int t = seq.next();
                tc::mbar_wait(&tfull[ts], (s / NTS) & 1);
                if (lane == 0) TC_TR(1000 + w * 200 + s, clock64());
                if (!(warp_active && t >= wt0 && t <= wt1)) {
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive(&tempty[ts]);
                    continue;
                }
                const int slot = used % NSLOT;
                if (used >= NSLOT) tc::mbar_wait(&sempty[w * NSLOT + slot], ((used / NSLOT) - 1) & 1);
                // while the lists fill (gates still at their start value) stage one row at a
                // time: a row staged against an unset gate passes its whole window
                int gate = gate_pub[w * 32 + lane];
                if (used > 0 && __any_sync(0xffffffffu, gate == gate0 && refok)) {
                    while (consumed[w] < used) {
                    }
                    gate = gate_pub[w * 32 + lane];
                }
                // u = N_q - 2 <f_p, f_q> passes iff u < T = gate - N_p; stage v = u - T (exact for
                // every passing candidate, sign-correct for the rest): d = v + gate
                const float T = (float)(gate - __float2int_rn(Nr));
                uint32_t* const stg = stg0 + slot * 32 * STG_PITCH;
                tc::tc_fence_after();
                uint32_t msk[2] = {0u, 0u};
                const uint32_t tb = taddr + (uint32_t)(ts * NB);
                uint32_t acc[64];
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) tc::tmem_ld16p(tb + ch * 16, acc + ch * 16);
                tc::tmem_wait_ld();
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) tc::tmem_tie16(acc + ch * 16);
#pragma unroll
                for (int cc = 0; cc < 4; ++cc) {
                    const int ch = cc ^ 1;  // per 32-column half, the upper 16 columns first
                    const float4* ncv = reinterpret_cast<const float4*>(nc + t * NB + ch * 16);
                    float v[16];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float4 n4 = ncv[q];
                        v[4 * q + 0] = fmaf(__uint_as_float(acc[16 * ch + 4 * q + 0]), -2.f, n4.x - T);
                        v[4 * q + 1] = fmaf(__uint_as_float(acc[16 * ch + 4 * q + 1]), -2.f, n4.y - T);
                        v[4 * q + 2] = fmaf(__uint_as_float(acc[16 * ch + 4 * q + 2]), -2.f, n4.z - T);
                        v[4 * q + 3] = fmaf(__uint_as_float(acc[16 * ch + 4 * q + 3]), -2.f, n4.w - T);
                    }
                    // shift the sign bits in, highest column first: bit j of msk = column j passes
                    uint32_t& m = msk[ch >> 1];
#pragma unroll
                    for (int j = 15; j >= 0; --j) m = __funnelshift_l(__float_as_uint(v[j]), m, 1);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        *reinterpret_cast<float4*>(stg + ch * 16 + 4 * q) =
                            make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&tempty[ts]);

                const bool rowin = refok && t >= S * a && t <= S * a + 2 * r;
                uint64_t mm = rowin ? ((((uint64_t)msk[1]) << 32 | msk[0]) & cm) : 0ull;
                if (t == ty) mm &= ~(1ull << tx);  // the reference itself is slot 0
                *reinterpret_cast<uint4*>(stg + 64) =
                    make_uint4((uint32_t)mm, (uint32_t)(mm >> 32), (uint32_t)gate, (uint32_t)t);
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&sfull[w * NSLOT + slot]);
                if (lane == 0) TC_TR(2000 + w * 200 + s, clock64());
                ++used;
            }
        } else {
            // sorted list of the KP = KL + 1 smallest keys (a power of two for the bulk merge;
            // the extra slot is never output, the gate is the (K-1)-th key L[KL - 1])
            constexpr int KP = KL + 1;
            static_assert((KP & (KP - 1)) == 0 && KP <= 32, "list length must be a power of two");
            uint32_t L[KP];
#pragma unroll
            for (int i = 0; i < KP; ++i) L[i] = KEY_INF;
            int nrel = 0;
            if (warp_active) {
                const int lo = max(wt0, t_lo), hi = min(wt1, t_hi);
                nrel = hi >= lo ? hi - lo + 1 : 0;
            }
            // d + 2^23 as an fp32 bit pattern is 0x4B000000 + d (exact for d < 2^23), and
            // 0x4B000000 << cb == 0 (mod 2^32) for cb >= 8: key = bits(v + gate + 2^23) << cb | code
            const uint32_t kmul = 1u << cb;
            for (used = 0; used < nrel; ++used) {
                const int slot = used % NSLOT;
                if (lane == 0) TC_TR(5000 + w * 200 + used, clock64());
                tc::mbar_wait(&sfull[w * NSLOT + slot], (used / NSLOT) & 1);
                if (lane == 0) TC_TR(6000 + w * 200 + used, clock64());
                const uint32_t* const stg = stg0 + slot * 32 * STG_PITCH;
                const uint4 hdr = *reinterpret_cast<const uint4*>(stg + 64);
                uint32_t mlo = hdr.x, mhi = hdr.y;
                const float GB = (float)(int)hdr.z + 8388608.0f;  // d + 2^23 = v + gate + 2^23
                const uint32_t code_row = (uint32_t)((int)hdr.w - S * a) * side - (uint32_t)(S * bb);
                int R = (int)__reduce_max_sync(0xffffffffu, (unsigned)(__popc(mlo) + __popc(mhi)));
                if (R >= BULK_MIN) {
                    // dense row (lists filling): window columns j0 .. j0 + 31 by sort + merge,
                    // the rest (if any) by the insertion rounds below
                    const int j0 = S * bb;
                    const uint64_t mw = ((((uint64_t)mhi) << 32) | mlo) >> j0;
#pragma unroll
                    for (int c = 0; c < 32 / KP; ++c) {
                        uint32_t B[KP];
#pragma unroll
                        for (int jj = 0; jj < KP; ++jj) {
                            const int col = c * KP + jj;
                            const uint32_t bits =
                                __float_as_uint(__uint_as_float(stg[j0 + col]) + GB);
                            B[jj] = ((mw >> col) & 1ull) ? bits * kmul + code_row + (uint32_t)(j0 + col)
                                                         : KEY_INF;
                        }
                        bulk_merge<KP>(L, B);
                    }
                    uint64_t rest = ((((uint64_t)mhi) << 32) | mlo) & ~(0xffffffffull << j0);
                    if (2 * r + 1 <= 40) {  // the (at most 8) window columns left: one more batch
                        uint32_t B8[8];
#pragma unroll
                        for (int jj = 0; jj < 8; ++jj) {
                            const int col = 32 + jj;
                            const uint32_t bits =
                                __float_as_uint(__uint_as_float(stg[j0 + col]) + GB);
                            B8[jj] = ((mw >> col) & 1ull) ? bits * kmul + code_row + (uint32_t)(j0 + col)
                                                          : KEY_INF;
                        }
                        bulk_merge8<KP>(L, B8);
                        rest = 0ull;
                    }
                    mlo = (uint32_t)rest;
                    mhi = (uint32_t)(rest >> 32);
                    R = (int)__reduce_max_sync(0xffffffffu, (unsigned)(__popc(mlo) + __popc(mhi)));
                }
                // next pending candidate (highest column first), software-pipelined one round
                // ahead of the insertion network
                auto next_key = [&]() -> uint32_t {
                    const bool hi = mhi != 0u;
                    const uint32_t m = hi ? mhi : mlo;
                    const int jb = 31 - __clz(m);  // -1 when nothing is pending
                    const int j = (hi ? 32 : 0) + max(jb, 0);
                    const uint32_t clr = m ^ (jb >= 0 ? (1u << jb) : 0u);
                    if (hi) mhi = clr; else mlo = clr;
                    const uint32_t bits = __float_as_uint(__uint_as_float(stg[j]) + GB);
                    return jb >= 0 ? bits * kmul + code_row + (uint32_t)j : KEY_INF;
                };
                if (lane == 0) TC_TR(7000 + w * 200 + used, clock64());
                // two pending keys per round (the second is KEY_INF when a lane has run out)
                uint32_t ka = next_key(), kb = next_key();
                for (int q = 0; q < (R + 1) >> 1; ++q) {
                    const uint32_t ca = ka, cb2 = kb;
                    ka = next_key();
                    kb = next_key();
                    list_insert2<KP>(L, ca, cb2);
                }
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&sempty[w * NSLOT + slot]);
                if (lane == 0) TC_TR(3000 + w * 200 + used, clock64());
                if (lane == 0) TC_TR(4000 + w * 200 + used, R);
                const uint32_t top = L[KL - 1];
                gate_pub[w * 32 + lane] =
                    ((top == KEY_INF) ? p.tdr0 : min((int)(top >> cb), p.tdr0)) + 1;
                __syncwarp();
                if (lane == 0) consumed[w] = used + 1;
            }
            if (threadIdx.x == 32 * SEL_WARP0) TC_TR(7, clock64());
            // ---- output: slot 0 = self, ranks 1.. = list, pads (self, -1); coalesced rows
            const int Kout = p.K;
            const int ry = S * (ky0 + a), rx = S * (kx0 + bb);
            const int self = ry * p.W + rx;
            const uint32_t cmask = (1u << cb) - 1u;
            // idx = self + dy W + dx with code = (dy + r) side + (dx + r): with q = code / side
            // (exact through the fp32 reciprocal: code < 2^13, side <= 65),
            // idx = self - r (W + 1) + code + q (W - side)
            const float inv_side = 1.0f / (float)side;
            const int ibase = self - r * (p.W + 1), wms = p.W - (int)side;
            int cnt = 0;
            const int64_t ref0 = (int64_t)bimg * p.out_bstride;
            // per-warp output block: idx [4 rows][8 refs][Kout], then dist likewise
            uint32_t* const ob = reinterpret_cast<uint32_t*>(sm + g.off_stg) + w * NSLOT * 32 * STG_PITCH;
            auto slot_val = [&](int i, int32_t& vi, int32_t& vd) {  // i = slot (static)
                vi = self;
                vd = i == 0 ? 0 : -1;
                if (i > 0) {
                    const uint32_t key = L[i - 1];
                    if (key != KEY_INF) {
                        const uint32_t code = key & cmask;
                        const int q = (int)(((float)code + 0.5f) * inv_side);
                        vi = ibase + (int)code + q * wms;
                        vd = (int32_t)(key >> cb);
                    }
                }
            };
#pragma unroll
            for (int i = 0; i < KL; ++i) cnt += (i + 1 < Kout && L[i] != KEY_INF) ? 1 : 0;
            __syncwarp();
            const int nref = min(8, p.Rx_reg - kx0);
            if ((Kout & 3) == 0) {
                // 16-byte chunks c of a reference row stored at chunk c ^ (b & swz): conflict-free
                // stores (lanes b = 0..7 of a phase hit distinct banks) and contiguous reads
                const int nch = Kout >> 2;
                const int swz = (nch & (nch - 1)) == 0 ? nch - 1 : 0;
                uint32_t* const oi = ob + (lane >> 3) * 8 * Kout + bb * Kout;
                uint32_t* const od = oi + 32 * Kout;
#pragma unroll
                for (int c = 0; c < (KL + 1) / 4; ++c) {
                    if (4 * c < Kout) {
                        int32_t i0, i1, i2, i3, d0, d1, d2, d3;
                        slot_val(4 * c + 0, i0, d0);
                        slot_val(4 * c + 1, i1, d1);
                        slot_val(4 * c + 2, i2, d2);
                        slot_val(4 * c + 3, i3, d3);
                        const int cs = (c ^ (bb & swz)) * 4;
                        *reinterpret_cast<int4*>(oi + cs) = make_int4(i0, i1, i2, i3);
                        *reinterpret_cast<int4*>(od + cs) = make_int4(d0, d1, d2, d3);
                    }
                }
                __syncwarp();
                if (threadIdx.x == 32 * SEL_WARP0) TC_TR(8, clock64());
                const int n16 = nref * nch;
#pragma unroll
                for (int al = 0; al < 4; ++al) {
                    if (ky0 + 4 * w + al >= kr1) break;
                    const int64_t row = ref0 + (int64_t)(ky0 + 4 * w + al - p.row_begin) * p.Rx + kx0;
                    int4* const gi = reinterpret_cast<int4*>(p.idx + row * Kout);
                    int4* const gd = reinterpret_cast<int4*>(p.dist + row * Kout);
                    const uint32_t* const si = ob + al * 8 * Kout;
                    for (int u = lane; u < n16; u += 32) {
                        const int b2 = u / nch, c = u - b2 * nch;
                        const int off = b2 * Kout + ((c ^ (b2 & swz)) << 2);
                        gi[u] = *reinterpret_cast<const int4*>(si + off);
                        gd[u] = *reinterpret_cast<const int4*>(si + 32 * Kout + off);
                    }
                }
            } else {
                // general K: one word per slot, each reference row written by the warp
                uint32_t* const oi = ob + lane * Kout;
                uint32_t* const od = oi + 32 * Kout;
#pragma unroll
                for (int i = 0; i < KL + 1; ++i) {
                    if (i < Kout) {
                        int32_t vi, vd;
                        slot_val(i, vi, vd);
                        oi[i] = (uint32_t)vi;
                        od[i] = (uint32_t)vd;
                    }
                }
                __syncwarp();
                for (int l = 0; l < 32; ++l) {
                    const int la = 4 * w + (l >> 3), lb = l & 7;
                    if (ky0 + la >= kr1 || lb >= nref) continue;
                    const int64_t ref = ref0 + (int64_t)(ky0 + la - p.row_begin) * p.Rx + (kx0 + lb);
                    for (int s2 = lane; s2 < Kout; s2 += 32) {
                        p.idx[ref * Kout + s2] = (int32_t)ob[l * Kout + s2];
                        p.dist[ref * Kout + s2] = (int32_t)ob[32 * Kout + l * Kout + s2];
                    }
                }
            }
            __syncwarp();
            if (threadIdx.x == 32 * SEL_WARP0) TC_TR(9, clock64());
            if (refok && p.tau_above_dsat && cnt < Kout - 1) {
                const int wy = min(p.H - P, ry + r) - max(0, ry - r) + 1;
                const int wx = min(p.W - P, rx + r) - max(0, rx - r) + 1;
                if (cnt < wy * wx - 1) {
                    const int64_t ref = ref0 + (int64_t)(ky0 + a - p.row_begin) * p.Rx + (kx0 + bb);
                    cnt = tc_exact_ref(p.img + (int64_t)bimg * p.img_bstride, p.slab_y0, p.H, p.W,
                                       P, r, ry, rx, Kout, p.tau, p.idx + ref * Kout,
                                       p.dist + ref * Kout);
                }
            }
            if (refok && p.nvalid) {
                const int64_t ref = ref0 + (int64_t)(ky0 + a - p.row_begin) * p.Rx + (kx0 + bb);
                p.nvalid[ref] = 1 + cnt;
            }
        }
    }

    tc::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) TC_TR(1, clock64());
    if (threadIdx.x == 0) TC_SPAN(1, gtimer());
    if (warp == MMA_WARP) {
        tc::tc_fence_after();
        tc::tmem_dealloc<tc16::TMEM_COLS>(tmem);
    }
}

template <int S, int KL>
cudaError_t launch_tc16(const MatchParams& p, cudaStream_t stream, int* launches) {
    const int kr0 = p.row_begin, kr1 = p.row_end < p.Ry_reg ? p.row_end : p.Ry_reg;
    if (kr1 <= kr0 || p.Rx_reg <= 0) return cudaSuccess;
    const Tc16Geom g = Tc16Geom::make(S, p.r);
    static_assert(tc16::NB == 64, "pre-shifted plane layout assumes 64 candidate columns");
    auto kern = match_tc16_kernel<S, KL>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, g.total);
    if (e != cudaSuccess) return e;
    dim3 grid((p.Rx_reg + tc16::TX - 1) / tc16::TX, (kr1 - kr0 + tc16::TY - 1) / tc16::TY, p.B);
    kern<<<grid, tc16::THREADS, g.total, stream>>>(p);
    if (launches) ++*launches;
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    // exact int8 kernel for the tiles the fp16 kernel marked (usually none: those CTAs exit)
    return launch_tc<S, KL>(p, stream, launches, 1);
}

}  // namespace gbm3d
