// Fast exact block-matching kernel, organised by search displacement (SSD form).
//
// Method (section II): for a fixed displacement delta = (dy, dx) the distance of every
// reference rho on the strided grid is the P x P box sum of the shifted-difference image
//     e_delta(y, x) = (Z[y][x] - Z[y+dy][x+dx])^2                          (Eq. (1))
// i.e. Prop. 1 with an all-ones block applied to e_delta, the box-filter step
// of PAPER.md:113.  The box sum is separable: vertical sums at reference rows, then horizontal
// sums at reference columns.  Everything is exact int32 arithmetic (reading R10).
//
// Work mapping:
//   * CTA = NS strips stacked vertically, two warps per strip.  The CTA stages its image region
//     (tile + radius halo) into shared memory once, as int16, zero outside the image.
//   * strip = RC = 32 - HL reference columns x TRY reference rows.  Lane l of both warps of the
//     strip owns the S pixel columns of reference column m0+l and keeps that column strip's
//     pixels (NR rows x S) in registers for the whole kernel (the "a" side of every difference).
//   * displacements are visited in blocks of D consecutive dy at one dx; the two warps of a strip
//     take alternate blocks.  For one block a lane streams the NR + D - 1 shifted rows ("b" side)
//     from shared memory once; each shifted row feeds D displacements (register reuse across dy).
//   * vertical box sums per column use chunk sums of S rows (C) and of the first P%S rows (A):
//       V_k = C_k + ... + C_{k+Q-1} + A_{k+Q},   Q = P / S,
//     horizontal sums combine the lane's column sums with Q neighbouring lanes via shuffles.
//   * selection (arg_K min): per reference a max-heap of the K-1 smallest 32-bit
//     keys (d << cb | code) in shared memory, shared by the strip's two warps.  The per-eval
//     gate is one compare against a register copy of the heap root; passing candidates go to a
//     per-(warp, ref) queue with predicated stores.  After each pair of blocks the warps merge
//     both queues into the heaps (each warp owns half of the reference rows), then refresh the
//     gates.  At the end an in-place heapsort orders each heap and the strip writes the tables
//     with coalesced 128-byte rows.
#pragma once
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"

namespace gbm3d {

constexpr int HEAP_STRIDE = 33;  // words per heap row: conflict-free per-lane AND per-ref access

template <int P_, int S_, int TRY_, int D_, int CB_, int WPS_ = 2, int LV_ = 4>
struct StripCfg {
    static constexpr int P = P_, S = S_, TRY = TRY_, D = D_;
    static constexpr int LV = LV_;                // heap sift levels: heap = 2^(LV+1) - 1 slots
    static constexpr int LP = (2 << LV_) - 1;
    static constexpr int WPS = WPS_;  // warps per strip: 2 = paired (shared heaps), 1 = solo
    static constexpr int CB = CB_;  // key = d << CB | code; 2^CB > (2r+1)^2
    static constexpr int Q = P / S, REM = P % S;
    static constexpr int HL = (P + S - 1) / S - 1;       // helper lanes (no references)
    static constexpr int RC = 32 - HL;                   // reference columns per warp
    static constexpr int NR = S * (TRY - 1) + P;         // pixel rows of a strip
    static constexpr int NCH = TRY - 1 + Q + (REM > 0);  // row chunks of a strip
    static constexpr int COLS = 32 * S;                  // pixel columns covered by a warp
    static_assert(S <= P, "fast path needs stride <= patch");
    static_assert(WPS == 1 || WPS == 2, "one or two warps per strip");
    static_assert(TRY % WPS == 0, "the warps of a strip split the reference rows");
    static_assert(D <= 15, "queue lengths are packed in 4 bits");
};

// Heap capacity: the smallest perfect binary tree (2^h - 1 nodes) holding n keys.  The slots
// beyond n hold 0-valued pads, which never rise above a real key, so the root stays the n-th
// smallest key seen and the sift-down has a fixed depth h - 1.
__host__ __device__ inline int heap_pad(int n) {
    int c = 0;
    while (c < n) c = 2 * c + 1;
    return c;
}
__host__ __device__ inline int heap_levels(int npad) {  // sift levels = h - 1
    int h = 0;
    while ((1 << h) - 1 < npad) ++h;
    return h > 0 ? h - 1 : 0;
}

// Shared-memory geometry of one CTA (host and device agree on it).
struct StripSmem {
    int pitch, rows, img_bytes, heap_words, queue_words, count_bytes;
    __host__ __device__ static StripSmem make(int COLS, int S, int P, int TRY, int D, int NS, int r,
                                              int K, int WPS, int LP) {
        StripSmem g;
        g.pitch = (COLS + 2 * r + 1) & ~1;
        g.rows = S * (TRY * NS - 1) + P + 2 * r + (D - 1);  // + D-1 rows read by the dy tail block
        g.img_bytes = ((g.rows * g.pitch * 2) + 15) & ~15;
        g.heap_words = NS * TRY * LP * HEAP_STRIDE;
        (void)K;
        g.queue_words = WPS * NS * TRY * D * 32;
        g.count_bytes = WPS * NS * TRY * 32 * 2;  // pair mode: u8 lengths; solo: u16 task list
        return g;
    }
    __host__ __device__ int bytes() const {
        return img_bytes + 4 * (heap_words + queue_words) + ((count_bytes + 15) & ~15);
    }
};

// Max-heap (perfect tree, `levels` = h - 1) of one reference: slot i at byte offset i * ROWB
// from Hb.  Replace the root by key (key < root) and sift down, branch-free, fixed depth.
constexpr int HEAP_ROWB = HEAP_STRIDE * 4;
static __device__ __forceinline__ uint32_t lds32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
    return v;
}
static __device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
static __device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Returns the new root.
template <int LEVELS>
static __device__ __forceinline__ uint32_t heap_replace_root(uint32_t base, uint32_t key) {
    // 32-bit shared addresses: child(a) = 2a - base + ROWB, sibling = child + ROWB
    const uint32_t cofs = HEAP_ROWB - base;
    uint32_t a = base;
    uint32_t root = key;
#pragma unroll
    for (int lv = 0; lv < LEVELS; ++lv) {
        const uint32_t c = 2 * a + cofs;
        const uint32_t v1 = lds32(c);
        const uint32_t v2 = lds32(c + HEAP_ROWB);
        const bool right = v2 > v1;
        const uint32_t big = right ? v2 : v1;
        const bool go = big > key;
        const uint32_t w = go ? big : key;
        if (lv == 0) root = w;
        sts32(a, w);
        const uint32_t nx = right ? c + HEAP_ROWB : c;
        a = go ? nx : a;
    }
    sts32(a, key);
    return root;
}

// In-place heapsort of a max-heap of n keys -> ascending order.
static __device__ void heap_sort(uint32_t* H, int n) {
    for (int end = n - 1; end > 0; --end) {
        const uint32_t top = H[0];
        const uint32_t key = H[end * HEAP_STRIDE];
        H[end * HEAP_STRIDE] = top;
        int i = 0;
        for (;;) {
            const int c = 2 * i + 1;
            if (c >= end) break;
            const uint32_t v1 = H[c * HEAP_STRIDE];
            const uint32_t v2 = (c + 1 < end) ? H[(c + 1) * HEAP_STRIDE] : 0u;
            const bool right = v2 > v1;
            const uint32_t big = right ? v2 : v1;
            if (big <= key) break;
            H[i * HEAP_STRIDE] = big;
            i = right ? c + 1 : c;
        }
        H[i * HEAP_STRIDE] = key;
    }
}

// i-th element of the centre-out sequence c, c+1, c-1, c+2, c-2, ... over [0, n).
static __device__ __forceinline__ int center_out(int i, int c, int n) {
    if (i == 0) return c;
    const int lo = c, hi = n - 1 - c, m = min(lo, hi);
    if (i <= 2 * m) {
        const int s = (i + 1) >> 1;
        return (i & 1) ? c + s : c - s;
    }
    const int extra = i - 2 * m;
    return hi > lo ? c + m + extra : c - m - extra;
}

static __device__ __forceinline__ void pair_sync(int strip) {
    asm volatile("bar.sync %0, 64;" ::"r"(strip + 1) : "memory");
}

// One displacement block: D consecutive dy at a fixed dx, all TRY reference rows of the lane.
template <class Cfg>
__device__ __forceinline__ void strip_block(const int16_t* __restrict__ sm_img, int pitch, int brow,
                                            int bcol, const int (&a)[Cfg::NR][Cfg::S],
                                            const int (&tdr)[Cfg::TRY], uint32_t* (&qp)[Cfg::TRY],
                                            const uint32_t (&mk)[Cfg::TRY],
                                            const uint32_t (&codej)[Cfg::D]) {
    constexpr int S = Cfg::S, P = Cfg::P, D = Cfg::D, NR = Cfg::NR, TRY = Cfg::TRY;
    constexpr int Q = Cfg::Q, REM = Cfg::REM, NCH = Cfg::NCH;
    int Cc[D][NCH][S];
    int Ac[D][NCH][S];
#pragma unroll
    for (int t = 0; t < NR + D - 1; ++t) {
        int bv[S];
        const int16_t* rowp = sm_img + (brow + t) * pitch + bcol;
#pragma unroll
        for (int c = 0; c < S; ++c) bv[c] = rowp[c];
#pragma unroll
        for (int j = 0; j < D; ++j) {
            const int y = t - j;
            if (y < 0 || y >= NR) continue;
            const int ch = y / S, pos = y % S;
#pragma unroll
            for (int c = 0; c < S; ++c) {
                const int df = a[y][c] - bv[c];
                if (pos == 0)
                    Cc[j][ch][c] = df * df;
                else
                    Cc[j][ch][c] += df * df;
                if (REM > 0 && pos == REM - 1) Ac[j][ch][c] = Cc[j][ch][c];
            }
            // reference row k is complete once its last pixel row y = S k + P - 1 is in
            if (y >= P - 1 && (y - (P - 1)) % S == 0 && (y - (P - 1)) / S < TRY) {
                const int k = (y - (P - 1)) / S;
                int hc = 0, ha = 0;
#pragma unroll
                for (int c = 0; c < S; ++c) {
                    int v = 0;
#pragma unroll
                    for (int q = 0; q < Q; ++q) v += Cc[j][k + q][c];
                    if (REM > 0) v += Ac[j][k + Q][c];
                    if (c < REM) ha += v;
                    hc += v;
                }
                int d = hc;
#pragma unroll
                for (int q = 1; q < Q; ++q) d += __shfl_down_sync(0xffffffffu, hc, q);
                if (REM > 0) d += __shfl_down_sync(0xffffffffu, ha, Q);
                // gate: one compare with the heap-root copy, AND the border/self mask bit
                const bool pass = (d <= tdr[k]) && ((mk[k] >> j) & 1u);
                if (pass) {
                    *qp[k] = ((uint32_t)d << Cfg::CB) + codej[j];
                    qp[k] += 32;
                }
            }
        }
    }
}

// Exact per-reference recomputation with 64-bit keys, used only for references whose 32-bit
// key range may have dropped a valid candidate (tau - 1 > dsat and the heap is not full).
// The list lives directly in the output slots 1..K-1.  Returns the number of matches.
static __device__ __noinline__ int strip_exact_ref(const int16_t* __restrict__ sm_img, int pitch,
                                                   int sy, int sx, int ry, int rx, int H, int W,
                                                   int P, int r, int K, int64_t tau, int32_t* oi,
                                                   int32_t* od) {
    const int L = K - 1;
    int cnt = 0;
    const int cy0 = max(0, ry - r), cy1 = min(H - P, ry + r);
    const int cx0 = max(0, rx - r), cx1 = min(W - P, rx + r);
    for (int cy = cy0; cy <= cy1; ++cy) {
        for (int cx = cx0; cx <= cx1; ++cx) {
            if (cy == ry && cx == rx) continue;
            int64_t d = 0;
            for (int i = 0; i < P; ++i) {
                const int16_t* ra = sm_img + (sy + i) * pitch + sx;
                const int16_t* rb = sm_img + (sy + cy - ry + i) * pitch + sx + (cx - rx);
                for (int jj = 0; jj < P; ++jj) {
                    const int64_t df = (int64_t)ra[jj] - (int64_t)rb[jj];
                    d += df * df;
                }
            }
            if (d >= tau) continue;
            const uint64_t key = ((uint64_t)d << 32) | (uint32_t)(cy * W + cx);
            int pos;
            if (cnt < L) {
                pos = cnt++;
            } else {
                const uint64_t last = ((uint64_t)(uint32_t)od[L] << 32) | (uint32_t)oi[L];
                if (key >= last) continue;
                pos = L - 1;
            }
            while (pos > 0) {
                const uint64_t prev = ((uint64_t)(uint32_t)od[pos] << 32) | (uint32_t)oi[pos];
                if (prev < key) break;
                od[pos + 1] = od[pos];
                oi[pos + 1] = oi[pos];
                --pos;
            }
            od[pos + 1] = (int32_t)d;
            oi[pos + 1] = cy * W + cx;
        }
    }
    const int self = ry * W + rx;
    oi[0] = self;
    od[0] = 0;
    for (int i = cnt; i < L; ++i) {
        oi[1 + i] = self;
        od[1 + i] = -1;
    }
    return cnt;
}

// nsplit > 1 (small images): the CTAs of a cluster of nsplit along z share one strip tile and
// take interleaved subsets of the displacement blocks; cluster rank 0 merges the others' sorted
// heaps through distributed shared memory and writes the tables (more CTAs fill the GPU).
#ifndef GBM3D_S12_MINB
#define GBM3D_S12_MINB 3  // patch-12 shape: 3 resident CTAs per SM (168 registers; c2 0.31 -> 0.28 ms)
#endif
template <class Cfg>
__global__ void __launch_bounds__(128, Cfg::P == 12 ? GBM3D_S12_MINB : 1)
    match_strip_kernel(MatchParams p, int NS, int nsplit) {
    constexpr int S = Cfg::S, P = Cfg::P, D = Cfg::D, NR = Cfg::NR, TRY = Cfg::TRY;
    constexpr int RC = Cfg::RC, CB = Cfg::CB, WPS = Cfg::WPS, HALF = TRY / WPS;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int r = p.r;
    const int L = p.K - 1;
    constexpr int LP = Cfg::LP;          // heap slots (perfect tree; >= K-1, checked on host)
    const StripSmem g = StripSmem::make(Cfg::COLS, S, P, TRY, D, NS, r, p.K, WPS, LP);
    int16_t* sm_img = reinterpret_cast<int16_t*>(smem_raw);
    uint32_t* sm_heap = reinterpret_cast<uint32_t*>(smem_raw + g.img_bytes);
    uint32_t* sm_q = sm_heap + g.heap_words;
    uint8_t* sm_cnt = reinterpret_cast<uint8_t*>(sm_q + g.queue_words);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int strip = warp / WPS, half = warp % WPS;
    const int b = (int)blockIdx.z / nsplit, split = (int)blockIdx.z % nsplit;
    const int kr0 = p.row_begin, kr1 = min(p.row_end, p.Ry_reg);  // regular rows in this call
    const int k0 = kr0 + (int)blockIdx.y * TRY * NS;
    const int m0 = (int)blockIdx.x * RC;
    const int16_t* __restrict__ img = p.img + (int64_t)b * p.img_bstride;

    // ---- stage tile + halo (int16, zero outside the image / slab); heaps: INF keys, 0 pads
    {
        const int gy0 = S * k0 - r, gx0 = S * m0 - r;
        const int ylo = max(0, p.slab_y0), yhi = min(p.H, p.slab_y1);
        for (int yy = warp; yy < g.rows; yy += blockDim.x >> 5) {
            const int gy = gy0 + yy;
            const bool rowok = gy >= ylo && gy < yhi;
            const int16_t* src = img + (int64_t)(gy - p.slab_y0) * p.W;
            for (int xx = lane; xx < g.pitch; xx += 32) {
                const int gx = gx0 + xx;
                sm_img[yy * g.pitch + xx] = (rowok && gx >= 0 && gx < p.W) ? src[gx] : (int16_t)0;
            }
        }
        for (int i = threadIdx.x; i < g.heap_words; i += blockDim.x) {
            const int slot = (i / HEAP_STRIDE) % (LP > 0 ? LP : 1);
            sm_heap[i] = slot < L ? KEY_INF : 0u;
        }
    }
    __syncthreads();

    const int kw = k0 + TRY * strip;  // first reference row of this strip
    const int m = m0 + lane;
    const int nk = min(TRY, kr1 - kw);
    const int nm = min(RC, p.Rx_reg - m0);
    // strip without references (only pair barriers follow); with a split it still walks the
    // loop (no passes) so that every thread reaches the cluster barriers
    if ((nk <= 0 || nm <= 0) && nsplit == 1) return;
    const bool lane_ok = (lane < RC) && (m < p.Rx_reg);

    const int arow0 = r + S * TRY * strip;  // smem row of strip row 0
    int a[NR][S];
#pragma unroll
    for (int y = 0; y < NR; ++y)
#pragma unroll
        for (int c = 0; c < S; ++c) a[y][c] = sm_img[(arow0 + y) * g.pitch + r + S * lane + c];

    uint32_t* const heap0 = sm_heap + (strip * TRY) * LP * HEAP_STRIDE + lane;  // + k*LP*33
    uint32_t* const qw = sm_q + (warp * TRY * D) * 32 + lane;                  // own queues
    uint8_t* const cw = sm_cnt + (warp * TRY) * 32 + lane;

    int tdr[TRY];
    bool refok[TRY];
    uint32_t* qp[TRY];
#pragma unroll
    for (int k = 0; k < TRY; ++k) {
        refok[k] = lane_ok && (k < nk) && (L > 0);
        tdr[k] = refok[k] ? p.tdr0 : -1;
        qp[k] = qw + k * D * 32;
    }
    const int ry_first = S * kw, ry_last = S * (kw + nk - 1);
    const int rx_first = S * m0, rx_last = S * (m0 + nm - 1);
    const int ylast = p.H - P, xlast = p.W - P;
    const uint32_t side = (uint32_t)p.side;
    const int nDY = (p.side + D - 1) / D;
    const int NB = p.side * nDY;  // displacement blocks (dx-major)
    const int NBs = (NB + nsplit - 1) / nsplit;  // this CTA's blocks: every nsplit-th

    if (L > 0) {
        for (int it = 0; it < NBs; it += WPS) {
            const int blk = (it + half) * nsplit + split;
            if (blk < NB) {
                // centre-out visiting order (dx: 0, +1, -1, +2, ...; dy blocks likewise): the
                // nearest displacements usually match best, so the heap gates tighten early
                const int dx = center_out(blk / nDY, r, 2 * r + 1) - r;
                const int dy0 = -r + center_out(blk % nDY, r / D, nDY) * D;
                const int bcol = r + S * lane + dx;
                const int brow = arow0 + dy0;
                const uint32_t code0 = (uint32_t)((dy0 + r) * p.side + (dx + r));
                const bool interior = (rx_first + dx >= 0) && (rx_last + dx <= xlast) &&
                                      (ry_first + dy0 >= 0) && (ry_last + dy0 + D - 1 <= ylast) &&
                                      (dy0 + D - 1 <= r) && !(dx == 0 && dy0 <= 0 && dy0 + D > 0);
                uint32_t mk[TRY];
                if (interior) {
#pragma unroll
                    for (int k = 0; k < TRY; ++k) mk[k] = 0xffffffffu;
                } else {  // border / window-tail / self: per (row, dy) validity bits
                    const bool xvalid = (S * m + dx >= 0) && (S * m + dx <= xlast);
                    uint32_t jx = 0;
#pragma unroll
                    for (int j = 0; j < D; ++j) {
                        const int dy = dy0 + j;
                        const bool ok = (dy <= r) && !(dx == 0 && dy == 0) && xvalid;
                        jx |= (ok ? 1u : 0u) << j;
                    }
#pragma unroll
                    for (int k = 0; k < TRY; ++k) {
                        const int ry = S * (kw + k);
                        const int lo = max(-(ry + dy0), 0), hi = min(ylast - ry - dy0, D - 1);
                        const uint32_t ym =
                            hi >= lo ? (((2u << hi) - 1u) & ~((1u << lo) - 1u)) : 0u;
                        mk[k] = jx & ym;
                    }
                }
                uint32_t codej[D];
#pragma unroll
                for (int j = 0; j < D; ++j) codej[j] = code0 + (uint32_t)j * side;
                strip_block<Cfg>(sm_img, g.pitch, brow, bcol, a, tdr, qp, mk, codej);
            }
            if constexpr (WPS == 1) {
                // Solo merge with work redistribution: the warp lists its non-empty queues
                // (one task = one heap and its queue) and lane t takes tasks t, t+32, ...  so the
                // sifts are spread evenly over the lanes instead of following the reference
                // that owns them.
                uint16_t* const tl = reinterpret_cast<uint16_t*>(sm_cnt) + warp * TRY * 32;
                const uint32_t ltm = (1u << lane) - 1u;
                int E = 0;
#pragma unroll
                for (int k = 0; k < TRY; ++k) {
                    const int q = (int)((qp[k] - (qw + k * D * 32)) >> 5);
                    qp[k] = qw + k * D * 32;
                    const uint32_t m = __ballot_sync(0xffffffffu, q > 0);
                    if (q > 0) tl[E + __popc(m & ltm)] = (uint16_t)((k << 9) | (lane << 4) | q);
                    E += __popc(m);
                }
                __syncwarp();
                const uint32_t heapw = smem_addr(sm_heap + (strip * TRY) * LP * HEAP_STRIDE);
                const uint32_t qbase = smem_addr(sm_q + (warp * TRY * D) * 32);
#pragma unroll 1
                for (int t = lane; t < E; t += 32) {
                    const uint32_t task = tl[t];
                    const uint32_t k = task >> 9, l = (task >> 4) & 31u, q = task & 15u;
                    const uint32_t hb = heapw + (k * LP * HEAP_STRIDE + l) * 4;
                    uint32_t qa = qbase + (k * D * 32 + l) * 4;
                    uint32_t thr = min(lds32(hb), p.thr0);
#pragma unroll 1
                    for (uint32_t i = 0; i < q; ++i, qa += 128) {
                        const uint32_t key = lds32(qa);
                        if (key < thr) thr = min(heap_replace_root<Cfg::LV>(hb, key), p.thr0);
                    }
                }
                __syncwarp();
#pragma unroll
                for (int k = 0; k < TRY; ++k) {
                    if (refok[k]) {
                        const uint32_t thr = min(heap0[k * LP * HEAP_STRIDE], p.thr0);
                        tdr[k] = thr == p.thr0 ? p.tdr0 : (int)(thr >> CB);
                    }
                }
                continue;
            }
            // publish queue lengths; this warp merges reference rows k = half (mod 2)
#pragma unroll
            for (int k = 0; k < TRY; ++k) {
                cw[k * 32] = (uint8_t)((qp[k] - (qw + k * D * 32)) >> 5);
                qp[k] = qw + k * D * 32;
            }
            if (WPS == 2) pair_sync(strip); else __syncwarp();
            {
                // flattened per-thread task loop over groups g = 2*kk + src.  Thread (half, lane)
                // merges rows k = half + 2 kk, each in column (lane + 5 k) mod 32: spreading a
                // thread's heaps over distant columns decorrelates their task counts.
                uint32_t packed = 0, nonempty = 0;
                int T = 0;
#pragma unroll
                for (int kk = 0; kk < HALF; ++kk) {
                    const int k = half + WPS * kk;
                    const int col = (lane + 5 * k) & 31;
#pragma unroll
                    for (int src = 0; src < WPS; ++src) {
                        const uint32_t n = sm_cnt[((warp ^ src) * TRY + k) * 32 + col];
                        packed |= n << (4 * (WPS * kk + src));
                        nonempty |= (n ? 1u : 0u) << (WPS * kk + src);
                        T += (int)n;
                    }
                }
                if (T > 0) {
                    char* const heapb = reinterpret_cast<char*>(sm_heap + (strip * TRY) * LP * HEAP_STRIDE);
                    int gq = __ffs(nonempty) - 1;
                    int n = (packed >> (4 * gq)) & 15u, i = 0;
                    int k = half + WPS * (gq / WPS), col = (lane + 5 * k) & 31;
                    uint32_t Hb = smem_addr(heapb + (k * LP * HEAP_STRIDE + col) * 4);
                    const uint32_t* q = sm_q + (((warp ^ (gq % WPS)) * TRY + k) * D) * 32 + col;
                    uint32_t thr = min(lds32(Hb), p.thr0);
                    for (int t = 0; t < T; ++t) {
                        const uint32_t key = q[i * 32];
                        if (key < thr) thr = min(heap_replace_root<Cfg::LV>(Hb, key), p.thr0);
                        if (++i == n) {
                            nonempty &= ~(1u << gq);
                            if (nonempty) {
                                gq = __ffs(nonempty) - 1;
                                n = (packed >> (4 * gq)) & 15u;
                                i = 0;
                                k = half + WPS * (gq / WPS);
                                col = (lane + 5 * k) & 31;
                                Hb = smem_addr(heapb + (k * LP * HEAP_STRIDE + col) * 4);
                                q = sm_q + (((warp ^ (gq % WPS)) * TRY + k) * D) * 32 + col;
                                thr = min(lds32(Hb), p.thr0);
                            }
                        }
                    }
                }
            }
            if (WPS == 2) pair_sync(strip); else __syncwarp();
#pragma unroll
            for (int k = 0; k < TRY; ++k) {
                if (refok[k]) {
                    const uint32_t thr = min(heap0[k * LP * HEAP_STRIDE], p.thr0);
                    tdr[k] = thr == p.thr0 ? p.tdr0 : (int)(thr >> CB);
                }
            }
        }
        // ---- order each heap ascending (in place), each warp its own reference rows
#pragma unroll 1
        for (int k = half; k < TRY; k += WPS)
            if (refok[k]) heap_sort(heap0 + k * LP * HEAP_STRIDE, LP);
        if (WPS == 2) pair_sync(strip); else __syncwarp();
    }
    if (nsplit > 1) {
        // rank 0 keeps, per reference, the L smallest of its sorted list and the other ranks'
        // (distinct displacements: distinct keys), read through distributed shared memory; the
        // merged list goes through this lane's queue slots (L <= TRY D, checked on the host)
        namespace cg = cooperative_groups;
        cg::cluster_group cl = cg::this_cluster();
        cl.sync();
        if (split == 0 && L > 0) {
            const int off0 = LP - L;
#pragma unroll 1
            for (int k = half; k < nk; k += WPS) {
                if (!refok[k]) continue;
                uint32_t* const mine = heap0 + (k * LP + off0) * HEAP_STRIDE;
#pragma unroll 1
                for (int rk = 1; rk < nsplit; ++rk) {
                    const uint32_t* peer = cl.map_shared_rank(mine, rk);
                    int ia = 0, ib = 0;
#pragma unroll 1
                    for (int o = 0; o < L; ++o) {
                        const uint32_t va = mine[ia * HEAP_STRIDE], vb = peer[ib * HEAP_STRIDE];
                        const bool ta = va < vb;
                        qw[o * 32] = ta ? va : vb;
                        ia += ta ? 1 : 0;
                        ib += ta ? 0 : 1;
                    }
#pragma unroll 1
                    for (int o = 0; o < L; ++o) mine[o * HEAP_STRIDE] = qw[o * 32];
                }
            }
        }
        cl.sync();  // the other ranks' heaps are read: they may exit
        if (split != 0 || nk <= 0) return;
    }

    // ---- epilogue: coalesced rows; slot 0 = self (d = 0), ranks 1.. sorted keys, pads (self,-1)
    const uint32_t cmask = (1u << CB) - 1u;
    const int off = LP - L;  // sorted heap: LP - L zero pads first, then the L keys ascending
#pragma unroll 1
    for (int k = half; k < nk; k += WPS) {
        const int kk = kw + k, ry = S * kk;
        const uint32_t* Hk = sm_heap + (strip * TRY + k) * LP * HEAP_STRIDE;
#pragma unroll 1
        for (int l = 0; l < nm; ++l) {
            const int rx = S * (m0 + l);
            const int64_t ref =
                (int64_t)b * p.out_bstride + (int64_t)(kk - p.row_begin) * p.Rx + (m0 + l);
            int32_t* oi = p.idx + ref * p.K;
            int32_t* od = p.dist + ref * p.K;
            const int self = ry * p.W + rx;
            int cnt = 0;
            for (int s0 = 0; s0 < p.K; s0 += 32) {
                const int s = s0 + lane;
                uint32_t key = KEY_INF;
                if (s >= 1 && s < p.K) key = Hk[(off + s - 1) * HEAP_STRIDE + l];
                cnt += __popc(__ballot_sync(0xffffffffu, key != KEY_INF));
                if (s < p.K) {
                    int32_t vi = self, vd = (s == 0) ? 0 : -1;
                    if (key != KEY_INF) {
                        const uint32_t code = key & cmask;
                        vi = (ry + (int)(code / side) - r) * p.W + rx + (int)(code % side) - r;
                        vd = (int32_t)(key >> CB);
                    }
                    oi[s] = vi;
                    od[s] = vd;
                }
            }
            if (p.tau_above_dsat && cnt < L) {
                const int wy = min(ylast, ry + r) - max(0, ry - r) + 1;
                const int wx = min(xlast, rx + r) - max(0, rx - r) + 1;
                if (cnt < wy * wx - 1) {
                    __syncwarp();
                    if (lane == 0)
                        cnt = strip_exact_ref(sm_img, g.pitch, arow0 + S * k, r + S * l, ry, rx,
                                              p.H, p.W, P, r, p.K, p.tau, oi, od);
                    cnt = __shfl_sync(0xffffffffu, cnt, 0);
                }
            }
            if (p.nvalid && lane == 0) p.nvalid[ref] = 1 + cnt;
        }
    }
}

// Host launcher: picks the strips per CTA (1 or 2; two warps each) that maximise resident
// warps per SM under the shared-memory budget, then launches over the regular grid rows.
template <class Cfg>
cudaError_t launch_strip(const MatchParams& p, cudaStream_t stream, int* launches) {
    const int kr0 = p.row_begin, kr1 = p.row_end < p.Ry_reg ? p.row_end : p.Ry_reg;
    if (kr1 <= kr0 || p.Rx_reg <= 0) return cudaSuccess;
    if (p.K - 1 > Cfg::LP) return cudaErrorInvalidValue;  // dispatcher picks LV with 2^(LV+1)-1 >= K-1
    int dev = 0, max_optin = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    e = cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (e != cudaSuccess) return e;
    auto kern = match_strip_kernel<Cfg>;
    int best_ns = 0, best_warps = -1, best_smem = 0;
    for (int ns : {4 / Cfg::WPS, 2 / Cfg::WPS, 1}) {
        const int smem = StripSmem::make(Cfg::COLS, Cfg::S, Cfg::P, Cfg::TRY, Cfg::D, ns, p.r, p.K,
                                         Cfg::WPS, Cfg::LP).bytes();
        if (smem > max_optin) continue;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        int nb = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, 32 * Cfg::WPS * ns, smem);
        if (e != cudaSuccess) return e;
        if (nb * Cfg::WPS * ns > best_warps) {
            best_warps = nb * Cfg::WPS * ns;
            best_ns = ns;
            best_smem = smem;
        }
    }
    if (best_ns == 0 || best_warps <= 0) return cudaErrorInvalidConfiguration;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, best_smem);
    if (e != cudaSuccess) return e;
    dim3 grid((p.Rx_reg + Cfg::RC - 1) / Cfg::RC,
              (kr1 - kr0 + Cfg::TRY * best_ns - 1) / (Cfg::TRY * best_ns), p.B);
    // a grid that fills less than half the GPU's resident warps (small images): split the
    // displacement blocks over a cluster of CTAs per tile (the merge needs L <= TRY D and the
    // 32-bit keys to be exact, i.e. no 64-bit fallback)
    int n_sm = 0;
    e = cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return e;
    const long long ctas = (long long)grid.x * grid.y * grid.z;
    const long long cap = (long long)n_sm * (best_warps / (Cfg::WPS * best_ns));
    int nsplit = 1;
    if (!p.tau_above_dsat && p.K - 1 <= Cfg::TRY * Cfg::D && ctas < cap) {
        // the split (<= 4) whose CTAs fill their waves of resident slots best, ties to fewer
        // splits (c2 measured, 3 CTAs/SM = 444 slots for 160 CTAs: 1 / 2 / 3 / 4 splits 0.406 /
        // 0.283 / 0.331 / 0.314 ms -> 2; at 2 CTAs/SM (296 slots) 3 splits won, 0.309 ms)
        double best = 0.0;
        for (int ns = 1; ns <= 4; ++ns) {
            const long long n = ctas * ns, waves = (n + cap - 1) / cap;
            const double eff = (double)n / (double)(waves * cap);
            if (eff > best + 1e-9) {
                best = eff;
                nsplit = ns;
            }
        }
    }
    static const int split_env = getenv("GBM3D_STRIP_SPLIT") ? atoi(getenv("GBM3D_STRIP_SPLIT")) : 0;
    if (split_env > 0 && !p.tau_above_dsat && p.K - 1 <= Cfg::TRY * Cfg::D) nsplit = split_env;  // dev
    static const bool dbg = getenv("GBM3D_DEBUG") != nullptr;
    if (dbg)
        fprintf(stderr, "gbm3d: strip P%d S%d grid %u x %u x %u, %d strips/CTA, %lld CTAs, cap %lld, split %d\n",
                Cfg::P, Cfg::S, grid.x, grid.y, grid.z, best_ns, ctas, cap, nsplit);
    if (nsplit == 1) {
        kern<<<grid, 32 * Cfg::WPS * best_ns, best_smem, stream>>>(p, best_ns, 1);
    } else {
        grid.z *= nsplit;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(32 * Cfg::WPS * best_ns);
        cfg.dynamicSmemBytes = best_smem;
        cfg.stream = stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = nsplit;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, p, best_ns, nsplit);
        if (e != cudaSuccess) return e;
    }
    if (launches) ++*launches;
    return cudaGetLastError();
}

#define GBM3D_INSTANTIATE_STRIP_LV(P, S, TRY, D, WPS, LV)                                      \
    template cudaError_t launch_strip<StripCfg<P, S, TRY, D, 11, WPS, LV>>(const MatchParams&, \
                                                                          cudaStream_t, int*); \
    template cudaError_t launch_strip<StripCfg<P, S, TRY, D, 13, WPS, LV>>(const MatchParams&, \
                                                                          cudaStream_t, int*);
// heaps of 15 / 31 / 63 slots: K <= 16, K <= 32, K <= 64
#define GBM3D_INSTANTIATE_STRIP(P, S, TRY, D, WPS)  \
    GBM3D_INSTANTIATE_STRIP_LV(P, S, TRY, D, WPS, 3) \
    GBM3D_INSTANTIATE_STRIP_LV(P, S, TRY, D, WPS, 4) \
    GBM3D_INSTANTIATE_STRIP_LV(P, S, TRY, D, WPS, 5)

}  // namespace gbm3d
