// Generic exact block matching, one CTA per reference: direct Eq. (1) SSD for every candidate
// of the clamped window and an exact selection of the K - 1 smallest 64-bit keys (d << 32 | idx)
// by warp-wide bitonic merges (no block-wide sort).
// Used for the appended last reference row/column of the grid (reading R3), for shapes the
// fast kernels do not instantiate (e.g. the paper's stage-1 tiling, patch 16 / stride 16,
// PAPER.md:232), and as GBM3D_METHOD_DIRECT.
//
// The candidate window's pixels (2r + P rows and columns at most: 80 x 80) are staged in shared
// memory once as int32; each thread computes eight horizontally adjacent candidates at a time,
// streaming one window row of P + 7 pixels through registers per patch row with 16-byte loads
// (every pixel feeds up to eight differences) against the reference row read as a broadcast.
// int32 arithmetic: the range precondition P^2 (max - min)^2 <= 2^31 - 1 (reading R10) bounds
// every d.
#pragma once
#include "common.cuh"

namespace gbm3d {

constexpr int DIRECT_THREADS = 256;
constexpr int DIRECT_CG = 8;               // candidates per thread task (adjacent along x)
constexpr int DIRECT_ROWS = 2 * 32 + 16;   // window rows: 2 r + P with r <= 32, P <= 16
constexpr int DIRECT_WIN = DIRECT_ROWS + DIRECT_CG;  // int32 row pitch (+ zero columns of a group)

// SSD of the reference (ref: shared, P rows of 16 ints) with the DIRECT_CG candidates whose
// top-left pixels are window columns x .. x + 7 of window row y (win: shared int32, pitch
// DIRECT_WIN, 16-byte aligned rows; x a multiple of 8).  Per patch row: 16-byte loads of the
// P + 7 window pixels and of the reference row (a broadcast), then 8 P ISUB + IMAD.
//
// Compile-time patch 12 or 16: Eq. (2), d = ||f_p||^2 + ||f_q||^2 - 2 <f_p, f_q>,
// in uint32 arithmetic modulo 2^32 -- one IMAD per pixel pair for the inner products, the
// candidates' norms from sliding row sums of the squared window row (P + 7 squares and 2 ops
// per candidate per row) -- instead of ISUB + IMAD per pair.  Exact: the true d is < 2^31
// (range precondition R10), so the wrapped value is d.  `np` = ||f_p||^2 mod 2^32.  (At P = 8
// the saving per row is smaller than the longer dependency chains cost: 1.76 -> 1.87 ms.)
template <int PT>
static __device__ __forceinline__ void direct_ssd8(const int* __restrict__ ref,
                                                   const int* __restrict__ win, int P, int y,
                                                   int x, int (&acc)[DIRECT_CG], uint32_t np) {
    constexpr int PM = PT > 0 ? PT : 16;
    constexpr int NW = (PM + DIRECT_CG - 1 + 3) / 4;  // 16-byte window loads per row
    const int Pn = PT > 0 ? PT : P;
    if (PT >= 12) {
        uint32_t ip[DIRECT_CG], nq[DIRECT_CG];
#pragma unroll
        for (int c = 0; c < DIRECT_CG; ++c) ip[c] = nq[c] = 0u;
#pragma unroll 1
        for (int i = 0; i < PM; ++i) {
            const int4* row = reinterpret_cast<const int4*>(win + (y + i) * DIRECT_WIN + x);
            uint32_t w[4 * NW];
#pragma unroll
            for (int q = 0; q < NW; ++q) {
                const int4 v = row[q];
                w[4 * q] = (uint32_t)v.x;
                w[4 * q + 1] = (uint32_t)v.y;
                w[4 * q + 2] = (uint32_t)v.z;
                w[4 * q + 3] = (uint32_t)v.w;
            }
            const int4* rr = reinterpret_cast<const int4*>(ref + i * 16);
#pragma unroll
            for (int q = 0; q < PM / 4; ++q) {
                const int4 a4 = rr[q];
                const uint32_t av[4] = {(uint32_t)a4.x, (uint32_t)a4.y, (uint32_t)a4.z, (uint32_t)a4.w};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj)
#pragma unroll
                    for (int c = 0; c < DIRECT_CG; ++c) ip[c] += av[jj] * w[c + 4 * q + jj];
            }
            uint32_t sq[PM + DIRECT_CG - 1];
#pragma unroll
            for (int k = 0; k < PM + DIRECT_CG - 1; ++k) sq[k] = w[k] * w[k];
            uint32_t rs = 0u;
#pragma unroll
            for (int k = 0; k < PM; ++k) rs += sq[k];
            nq[0] += rs;
#pragma unroll
            for (int c = 1; c < DIRECT_CG; ++c) {
                rs += sq[c + PM - 1] - sq[c - 1];
                nq[c] += rs;
            }
        }
#pragma unroll
        for (int c = 0; c < DIRECT_CG; ++c) acc[c] = (int)(np + nq[c] - 2u * ip[c]);
        return;
    }
#pragma unroll 1
    for (int i = 0; i < Pn; ++i) {
        const int4* row = reinterpret_cast<const int4*>(win + (y + i) * DIRECT_WIN + x);
        int w[4 * NW];
#pragma unroll
        for (int q = 0; q < NW; ++q) {
            const int4 v = row[q];
            w[4 * q] = v.x;
            w[4 * q + 1] = v.y;
            w[4 * q + 2] = v.z;
            w[4 * q + 3] = v.w;
        }
        const int4* rr = reinterpret_cast<const int4*>(ref + i * 16);
#pragma unroll
        for (int q = 0; q < PM / 4; ++q) {
            if (PT > 0 || 4 * q < Pn) {
                const int4 a4 = rr[q];
                const int av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) {
                    const int j = 4 * q + jj;
                    if (PT > 0 || j < Pn) {
#pragma unroll
                        for (int c = 0; c < DIRECT_CG; ++c) {
                            const int df = av[jj] - w[c + j];
                            acc[c] += df * df;
                        }
                    }
                }
            }
        }
    }
}

// Warp-wide selection helpers: a warp holds a sorted list of the 64 smallest keys seen so far
// (lane l keeps ranks l and l + 32) and folds in 32 new keys (one per lane) per round: the new
// keys are bitonic-sorted across the lanes, the lower half of Q ++ reverse(new) is bitonic, and a
// bitonic clean-up of 64 restores the order (DIRECT_KP = 64 >= K - 1 for every K <= 64).
typedef unsigned long long dkey;
static __device__ __forceinline__ dkey dmin(dkey a, dkey b) { return a < b ? a : b; }
static __device__ __forceinline__ dkey dmax(dkey a, dkey b) { return a < b ? b : a; }

static __device__ __forceinline__ dkey warp_sort32(dkey x, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const dkey y = __shfl_xor_sync(0xffffffffu, x, j);
            const bool lower = (lane & j) == 0, asc = (lane & k) == 0;
            x = (lower == asc) ? dmin(x, y) : dmax(x, y);
        }
    }
    return x;
}
// (q0, q1) = ranks (lane, lane + 32) of a sorted 64-list; s = ascending 32-list (rank lane).
static __device__ __forceinline__ void warp_merge64(dkey& q0, dkey& q1, dkey s, int lane) {
    const dkey srev = __shfl_sync(0xffffffffu, s, 31 - lane);  // rank 31 - lane
    q1 = dmin(q1, srev);                                      // rank lane + 32 vs s[63 - (lane+32)]
    // bitonic clean-up of 64: stride 32 inside the lane, then strides 16 .. 1 across lanes
    const dkey lo = dmin(q0, q1), hi = dmax(q0, q1);
    q0 = lo;
    q1 = hi;
#pragma unroll
    for (int j = 16; j > 0; j >>= 1) {
        const dkey y0 = __shfl_xor_sync(0xffffffffu, q0, j);
        const dkey y1 = __shfl_xor_sync(0xffffffffu, q1, j);
        const bool lower = (lane & j) == 0;
        q0 = lower ? dmin(q0, y0) : dmax(q0, y0);
        q1 = lower ? dmin(q1, y1) : dmax(q1, y1);
    }
}

// References [k_begin, k_end) x [m_begin, m_begin + m_count) of the grid (grid indices), every
// image (grid.z).  PT = compile-time patch (8, 12, 16) or 0 (any P <= 16).
template <int PT>
__global__ void __launch_bounds__(DIRECT_THREADS) match_direct_kernel(MatchParams p, int k_begin,
                                                                      int m_begin, int m_count) {
    __shared__ __align__(16) int refpatch[16 * 16];
    __shared__ __align__(16) int win[DIRECT_ROWS * DIRECT_WIN];
    __shared__ dkey wq[DIRECT_THREADS / 32][64];  // every warp's 64 best keys
    const int P = PT > 0 ? PT : p.P;
    const int r = p.r, W = p.W;
    const int k = k_begin + (int)(blockIdx.x / (unsigned)m_count);
    const int m = m_begin + (int)(blockIdx.x % (unsigned)m_count);
    const int b = blockIdx.z;
    const int16_t* __restrict__ img = p.img + (int64_t)b * p.img_bstride;
    const int ry = grid_pos(k, p.Ry_reg, p.S, p.H - P);
    const int rx = grid_pos(m, p.Rx_reg, p.S, p.W - P);
    const int cy0 = max(0, ry - r), cy1 = min(p.H - P, ry + r);
    const int cx0 = max(0, rx - r), cx1 = min(p.W - P, rx + r);
    const int wy = cy1 - cy0 + 1, wx = cx1 - cx0 + 1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    // stage the window's pixels as int32 (rows cy0 .. cy1 + P - 1, columns cx0 .. cx1 + P - 1;
    // the columns after them read as 0 and only feed candidates past the window, not kept)
    const int prow = wy + P - 1, pcol = wx + P - 1;
    const int gx = (wx + DIRECT_CG - 1) / DIRECT_CG;
    const int wcols = DIRECT_CG * gx + P - 1;  // columns a task row may read
    for (int y0 = warp; y0 < prow; y0 += 4 * nw) {  // a thread's 12 loads in flight together
        int v[4][3];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int yy = y0 + u * nw;
            const int16_t* src = img + (int64_t)(cy0 + yy - p.slab_y0) * W + cx0;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const int xx = lane + 32 * q;
                v[u][q] = (yy < prow && xx < pcol) ? (int)__ldg(src + xx) : 0;
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int yy = y0 + u * nw;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const int xx = lane + 32 * q;
                if (yy < prow && xx < wcols) win[yy * DIRECT_WIN + xx] = v[u][q];
            }
        }
    }
    for (int i = threadIdx.x; i < P * P; i += blockDim.x)
        refpatch[(i / P) * 16 + i % P] = img[(int64_t)(ry + i / P - p.slab_y0) * W + rx + i % P];
    __shared__ uint32_t s_np;  // ||f_p||^2 mod 2^32 (Eq. (2) path)
    if (threadIdx.x == 0) s_np = 0u;
    __syncthreads();
    if (PT >= 12) {
        uint32_t v = 0u;
        for (int i = threadIdx.x; i < P * P; i += blockDim.x) {
            const uint32_t z = (uint32_t)refpatch[(i / P) * 16 + i % P];
            v += z * z;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) atomicAdd(&s_np, v);
        __syncthreads();
    }
    const uint32_t np = s_np;
    // every warp: tasks of 8 candidates along x, then one selection round per candidate slot
    // (keys (d << 32 | idx); INF for d >= tau, the reference itself and the padding)
    dkey q0 = ~0ull, q1 = ~0ull;
    const int ntask = wy * gx;
    for (int t0 = warp * 32; t0 < ntask; t0 += 32 * nw) {
        const int task = t0 + lane;
        dkey key[DIRECT_CG];
#pragma unroll
        for (int c = 0; c < DIRECT_CG; ++c) key[c] = ~0ull;
        if (task < ntask) {
            const int yy = task / gx, x8 = DIRECT_CG * (task - yy * gx);
            int acc[DIRECT_CG] = {0, 0, 0, 0, 0, 0, 0, 0};
            direct_ssd8<PT>(refpatch, win, P, yy, x8, acc, np);
#pragma unroll
            for (int c = 0; c < DIRECT_CG; ++c) {
                const int cy = cy0 + yy, cx = cx0 + x8 + c;
                if (x8 + c < wx && !(cy == ry && cx == rx) && (int64_t)acc[c] < p.tau)
                    key[c] = ((dkey)(uint32_t)acc[c] << 32) | (uint32_t)(cy * W + cx);
            }
        }
#pragma unroll
        for (int c = 0; c < DIRECT_CG; ++c) {  // rounds with no key below the 64th best: skipped
            const dkey qmax = __shfl_sync(0xffffffffu, q1, 31);
            if (__any_sync(0xffffffffu, key[c] < qmax))
                warp_merge64(q0, q1, warp_sort32(key[c], lane), lane);
        }
    }
    wq[warp][lane] = q0;
    wq[warp][lane + 32] = q1;
    __syncthreads();
    if (warp != 0) return;
    for (int o = 1; o < nw; ++o) {  // warp 0 folds in the other warps' lists (32 keys at a time)
        const dkey a = wq[o][lane], c = wq[o][lane + 32];
        const dkey qmax = __shfl_sync(0xffffffffu, q1, 31);
        if (__any_sync(0xffffffffu, a < qmax)) warp_merge64(q0, q1, a, lane);
        if (__any_sync(0xffffffffu, c < __shfl_sync(0xffffffffu, q1, 31))) warp_merge64(q0, q1, c, lane);
    }
    // ranks 0 .. 63 of the window, ascending: slot s (1 .. K-1) = rank s - 1
    const int64_t ref = (int64_t)b * p.out_bstride + (int64_t)(k - p.row_begin) * p.Rx + m;
    int32_t* oi = p.idx + ref * p.K;
    int32_t* od = p.dist + ref * p.K;
    const int self = ry * W + rx;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const int s = 1 + lane + 32 * h;
        const dkey key = h ? q1 : q0;
        if (s < p.K) {
            oi[s] = key != ~0ull ? (int32_t)(uint32_t)(key & 0xffffffffu) : self;
            od[s] = key != ~0ull ? (int32_t)(key >> 32) : -1;
        }
    }
    if (lane == 0) {
        oi[0] = self;
        od[0] = 0;
    }
    const int cnt = __popc(__ballot_sync(0xffffffffu, q0 != ~0ull && 1 + lane < p.K)) +
                    __popc(__ballot_sync(0xffffffffu, q1 != ~0ull && 33 + lane < p.K));
    if (p.nvalid && lane == 0) p.nvalid[ref] = 1 + cnt;
}

}  // namespace gbm3d
