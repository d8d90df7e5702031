// Product-form block matching on the tensor cores, fp16 operands.
//
// Same method as match_tc.cuh (Eq. (2): d = ||f_p||^2 + ||f_q||^2 - 2 <f_p, f_q>),
// but one MMA per candidate row instead of four byte-plane products:
//   * each tile centres its pixels on c = (min + max) / 2 of the tile (the SSD is translation
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
// Work mapping: a tile = 16 x 8 grid references (M = 128, TMEM lane m =
// reference 8a + b).  The B operand needs no per-row building: the tile's fp16 plane is written
// once in a pre-shifted layout X[y][q][m][0..7] = plane[y][8q + m + 0..7] (each 16-byte chunk is
// candidate column 8q + m's patch row at image row y), so candidate row t's 64 patches are the
// K-major canonical operand at X + t * 1 KB with LBO = 1 KB (next patch row) and SBO = 128 B
// (next 8 candidates).
//
// Persistent CTAs (one per SM), warp-specialised, tiles streamed through a pipeline:
//   * producer warps (4): TMA load of the next tile's PR x 80 int16 pixel box
//     (cp.async.bulk.tensor, zero fill outside the image) while the current tile is matched;
//     range, centring, fp16 plane; X and A once the MMAs of the previous tile completed; the
//     candidate norms once the epilogue left the previous tile;
//   * MMA warp: one thread issues 4 MMAs (M128 N64 K16) per candidate row into one of NTS = 7
//     TMEM stages (a ring that runs on across tiles); A (the tile's 128 reference patches) lives
//     in tensor memory beside the stages, B in shared memory;
//   * epilogue warp w (TMEM lane quarter w): accumulators -> u and a pass mask, staged in SMEM;
//   * selector warp w: per-lane sorted top-(K-1) register lists (insertion network, one round
//     per pass; bulk bitonic merges for dense rows), then the output rows straight from the
//     registers -- so the next tile's prologue and this tile's output overlap the main loop.
#pragma once
#include <cuda.h>
#include <cuda_fp16.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "match_tc.cuh"

namespace gbm3d {

#if GBM3D_TC_TRACE  // dev-only timeline of persistent CTA 10 (clock64), read by gbm3d_dev_tc_trace
#define TC_TRP(i, v)                                              \
    do {                                                          \
        if (blockIdx.x == 10 && (i) < 8192) g_tc_trace[i] = (v);  \
    } while (0)
#else
#define TC_TRP(i, v) \
    do {             \
    } while (0)
#endif

namespace tc16 {
constexpr int TY = 16, TX = 8;
constexpr int NB = 64;           // candidate columns per MMA tile (N)
constexpr int PCH = 80;          // pixel box / fp16 plane width: 64 + 7 columns from a 16-byte
                                 // aligned start (TMA needs 16-byte aligned box coordinates)
constexpr int NTS = 7;           // TMEM stages (64 columns each)
constexpr uint32_t TM_A = NTS * 64;  // TMEM column of the A operand (128 lanes x 32 columns)
constexpr int EPI_WARPS = 4, SEL_WARP0 = 4, MMA_WARP = 8, PRO_WARP0 = 9, NPRO_MAX = 4;
// Warp roles by list length.  K = 32 (KL = 31): epilogue (0-3), selectors (4-7), MMA (8),
// producers (9-12, each writes the A rows of its lane quarter warp % 4 into TMEM); 13 warps.
// K <= 16: the selector runs fast enough to wait on one epilogue warp per quarter, so each
// quarter gets a second epilogue warp (12-15) and the two take its staged rows alternately;
// 16 warps keep 128 registers per thread (4 per SMSP), so there are 3 producers (9-11) and
// lane quarter 0's A rows go through a small shared buffer that the MMA warp copies in.  For
// K = 32 the second epilogue warp costs the selector more issue slots than it saves (measured,
// DESIGN.md).
#ifndef GBM3D_TC16_EARLY15
#define GBM3D_TC16_EARLY15 1  // K <= 16: u and the TMEM release before the slot / gate wait
#endif
#ifndef GBM3D_TC16_GATEFLAG15
#define GBM3D_TC16_GATEFLAG15 1  // K <= 16: no vote once the quarter's lists are full
#endif
#ifndef GBM3D_TC16_BULK_MIN15
#define GBM3D_TC16_BULK_MIN15 20
#endif
constexpr bool EARLY15 = GBM3D_TC16_EARLY15, GATEFLAG15 = GBM3D_TC16_GATEFLAG15;
#ifndef GBM3D_TC16_EH31
#define GBM3D_TC16_EH31 1  // dev switch: epilogue warps per lane quarter for K = 32
#endif
template <int KL>
struct Tc16Cfg {
    static constexpr int EH = KL <= 15 ? 2 : GBM3D_TC16_EH31;  // epilogue warps per lane quarter
    static constexpr int NPRO = EH == 2 ? 3 : 4;         // producer warps
    static constexpr int EPI_WARP1 = PRO_WARP0 + NPRO;   // first warp of epilogue half 1
    static constexpr int THREADS = 32 * (EPI_WARP1 + (EH == 2 ? EPI_WARPS : 0));
};
constexpr int NSLOT = 2;         // staged rows per lane quarter (epilogue one row ahead)
constexpr int STG_PITCH = 68;    // words per lane and staged row: u[64], mask lo/hi, gate, row
constexpr int XP = (NB / 8) * 128;  // bytes per pre-shifted plane row (8 chunks of 8 x 16 B)
constexpr uint32_t TMEM_COLS = 512;
constexpr int MMAX = 362;        // exactness bound on max |z - c| (see header)
constexpr int NINFO = 4;         // per-tile info ring (producer -> MMA, epilogue, selectors)
constexpr int INFO_W = 8;        // words per entry: tile (-1 = no more), image, ky0, kx0, row step, skip
constexpr int NSCHED = 64;       // tile-counter slots (concurrent launches use different slots)
constexpr int PRO_BAR = 2;       // named barrier of the producer warps
constexpr int MMA_PRO_BAR = 3;   // MMA warp -> producers: the tile's MMAs completed (X, A free)
constexpr int EPI_PRO_BAR = 4;   // [2] epilogue -> producers: the epilogue left a tile (by parity)
#ifndef GBM3D_TC16_BULK_MIN
#define GBM3D_TC16_BULK_MIN 16
#endif
constexpr int BULK_MIN = GBM3D_TC16_BULK_MIN;  // rows with this many passes (max over lanes) merge in bulk
}  // namespace tc16

struct Tc16Geom {
    int NT, PR, NJ;
    int off_x, off_nc, off_stg, off_pl, off_a0, off_bar, total;
    __host__ __device__ static Tc16Geom make(int S, int r) {
        using namespace tc16;
        Tc16Geom g;
        g.NT = 15 * S + 2 * r + 1;
        g.PR = g.NT + 7;
        g.NJ = 7 * S + 2 * r + 1;
        g.off_x = 0;                       // pre-shifted plane
        g.off_nc = g.off_x + g.PR * XP;    // candidate norms [2][NT][64] fp32 (tile parity)
        g.off_stg = g.off_nc + 2 * g.NT * NB * 4;
        g.off_pl = (g.off_stg + EPI_WARPS * NSLOT * 32 * STG_PITCH * 4 + 1023) & ~1023;  // TMA box
        g.off_a0 = (g.off_pl + g.PR * PCH * 2 + 15) & ~15;  // A rows of lane quarter 0 [32][32]
        g.off_bar = g.off_a0 + 32 * 32 * 4;
        // tfull/tempty[NTS], sfull/sempty[EPI_WARPS*NSLOT], raw, xa_ready, mma_done,
        // nc_ready[2], epi_done[2], info_full/info_empty[NINFO]; gates[128], consumed[EPI_WARPS],
        // info[NINFO][INFO_W], producer scratch[2*NPRO_MAX + 1], TMEM address
        g.total = g.off_bar + (2 * NTS + 2 * EPI_WARPS * NSLOT + 7 + 2 * NINFO) * 8 +
                  (EPI_WARPS * 32 + EPI_WARPS + NINFO * INFO_W + 2 * NPRO_MAX + 2) * 4 + 16;
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

// Candidate-row order of a tile.  Two "fill" rows first: f1 lies in the search window of every
// reference of warps 0-2 and is outside warp 3's rows, f2 lies in every window of warp 3 and
// outside warps 0-1's rows.  A warp's lists then all fill on the same row (one 39-round burst
// per warp instead of one per reference row), after which the scrambled order follows.
struct RowSeq {
    int lo, n, step, off, f0, f1, npre, pre;
    __device__ void init(int S, int r, int t_lo, int t_hi, int step_) {  // step_ = tc_step(n)
        lo = t_lo;
        n = t_hi - t_lo + 1;
        step = step_;
        off = 0;
        pre = 0;
        npre = 0;
        f0 = f1 = -1;
        const int a1 = 11 * S, b1 = min(2 * r, 12 * S - 1);
        const int a2 = max(15 * S, 7 * S + 2 * r + 1), b2 = 12 * S + 2 * r;
        const int g1 = (a1 + b1) / 2, g2 = (a2 + b2) / 2;
        if (a1 <= b1 && a2 <= b2 && g1 >= t_lo && g2 <= t_hi) {
            f0 = g1;
            f1 = g2;
            npre = 2;
        }
    }
    __device__ int next() {
        if (pre < npre) return pre++ == 0 ? f0 : f1;
        for (;;) {
            const int t = lo + off;
            off = tc_next(off, n, step);
            if (npre == 0 || (t != f0 && t != f1)) return t;
        }
    }
};


namespace tc {
// expect `bytes` of async-proxy (TMA) writes on a barrier, counting as this thread's arrival
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
// 3-D tiled TMA load of a box at element coordinates (x, y, z) (may be negative or past the
// end: those elements are zero-filled) into shared memory; completion counted on `bar`
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void named_bar(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
}  // namespace tc

// Dynamic tile counters: [2 * slot] = tiles handed out beyond the first wave, [2 * slot + 1] =
// CTAs finished; the last CTA of a launch zeroes both, so each slot starts every launch at 0.
static __device__ unsigned int g_tc16_sched[2 * tc16::NSCHED];

// MMA warp, after the tile's last commit: wait until the tile's MMAs completed, then let the
// producers (blocked on the named barrier) overwrite X and A (the whole warp arrives).
static __device__ __forceinline__ void tc_release_producers(uint64_t* b_mma, int it, int npro,
                                                            int lane, unsigned wm) {
    tc::mbar_wait(b_mma, it & 1);
    asm volatile("bar.arrive %0, %1;" ::"r"(tc16::MMA_PRO_BAR), "r"(32 * (npro + 1)) : "memory");
}

// Tile i of a call: image, first grid row and column of its 16 x 8 references.
struct Tc16Tile {
    int bimg, ky0, kx0;
    __device__ Tc16Tile(const MatchParams& p, int i) {
        const int kr1 = min(p.row_end, p.Ry_reg);
        const int nx = (p.Rx_reg + tc16::TX - 1) / tc16::TX;
        const int ny = (kr1 - p.row_begin + tc16::TY - 1) / tc16::TY;
        bimg = i / (nx * ny);
        const int rem = i - bimg * nx * ny;
        const int by = rem / nx;
        ky0 = p.row_begin + by * tc16::TY;
        kx0 = (rem - by * nx) * tc16::TX;
    }
};

// Insert one staged row's passing candidates into the lane's sorted list L: dense rows (R =
// max pass count over the warp >= BULK_MIN) by bitonic sort + merge of the window columns
// j0 .. j0 + 39, the rest by insertion rounds of two keys (list_insert2).  stg = the lane's
// staged v values (d = v + gate), GB = gate + 2^23 as fp32: bits(v + GB) = 0x4B000000 + d, whose
// 0x4B000000 part vanishes in the shift by cb >= 8.  
template <int KP>
static __device__ __forceinline__ void tc16_insert_row(uint32_t (&L)[KP], const uint32_t* stg,
                                                       uint32_t mlo, uint32_t mhi, float GB,
                                                       uint32_t code_row, uint32_t kmul, int j0,
                                                       int r, int R) {
    if (R >= (KP <= 16 ? GBM3D_TC16_BULK_MIN15 : tc16::BULK_MIN)) {
        // dense row (lists filling): window columns j0 .. j0 + 31 by sort + merge,
        // the rest (if any) by the insertion rounds below
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
    // two pending keys per round (the second is KEY_INF when a lane has run out)
    uint32_t ka = next_key(), kb = next_key();
    for (int q = 0; q < (R + 1) >> 1; ++q) {
        const uint32_t ca = ka, cb2 = kb;
        ka = next_key();
        kb = next_key();
        list_insert2<KP>(L, ca, cb2);
    }
}

// A lane's reference after its tile: slot 0 = self, ranks 1.. = the list (keys decoded to image
// indices and distances), pads; n_valid; the exact 64-bit recompute when tau exceeds the key
// range and the list did not fill.
template <int S, int KL>
static __device__ __forceinline__ void tc16_write_refs(const MatchParams& p, const uint32_t (&L)[KL + 1],
                                                       int a, int bb, int ky0, int kx0, int bimg,
                                                       int cb, uint32_t side) {
    constexpr int P = 8;
    const int r = p.r;
    const int Kout = p.K;
    const int ry = S * (ky0 + a), rx = S * (kx0 + bb);
    const int self = ry * p.W + rx;
    const uint32_t cmask = (1u << cb) - 1u;
    // idx = self + dy W + dx with code = (dy + r) side + (dx + r): with q = code / side
    // (exact through the fp32 reciprocal: code < 2^13, side <= 65),
    // idx = self - r (W + 1) + code + q (W - side)
    const float inv_side = 1.0f / (float)side;
    const int ibase = self - r * (p.W + 1), wms = p.W - (int)side;
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
    int cnt = 0;
#pragma unroll
    for (int i = 0; i < KL; ++i) cnt += (i + 1 < Kout && L[i] != KEY_INF) ? 1 : 0;
    const int64_t ref = (int64_t)bimg * p.out_bstride +
                        (int64_t)(ky0 + a - p.row_begin) * p.Rx + (kx0 + bb);
    int32_t* const oi = p.idx + ref * Kout;
    int32_t* const od = p.dist + ref * Kout;
    if ((Kout & 3) == 0) {
#pragma unroll
        for (int c = 0; c < (KL + 1) / 4; ++c) {
            if (4 * c < Kout) {
                int32_t i0, i1, i2, i3, d0, d1, d2, d3;
                slot_val(4 * c + 0, i0, d0);
                slot_val(4 * c + 1, i1, d1);
                slot_val(4 * c + 2, i2, d2);
                slot_val(4 * c + 3, i3, d3);
                *reinterpret_cast<int4*>(oi + 4 * c) = make_int4(i0, i1, i2, i3);
                *reinterpret_cast<int4*>(od + 4 * c) = make_int4(d0, d1, d2, d3);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < KL + 1; ++i) {
            if (i < Kout) {
                int32_t vi, vd;
                slot_val(i, vi, vd);
                oi[i] = vi;
                od[i] = vd;
            }
        }
    }
    if (p.tau_above_dsat && cnt < Kout - 1) {
        const int wy = min(p.H - P, ry + r) - max(0, ry - r) + 1;
        const int wx = min(p.W - P, rx + r) - max(0, rx - r) + 1;
        if (cnt < wy * wx - 1)
            cnt = tc_exact_ref(p.img + (int64_t)bimg * p.img_bstride, p.slab_y0, p.H,
                               p.W, P, r, ry, rx, Kout, p.tau, oi, od);
    }
    if (p.nvalid) p.nvalid[ref] = 1 + cnt;
}

template <int S, int KL>
__global__ void __launch_bounds__(tc16::Tc16Cfg<KL>::THREADS, 1)
    match_tc16_kernel(MatchParams p, const __grid_constant__ CUtensorMap tmap, int use_tma, int ntiles,
                      int sslot) {
    using namespace tc16;
    constexpr int EPI_HALVES = Tc16Cfg<KL>::EH, NPRO = Tc16Cfg<KL>::NPRO;
    constexpr int EPI_WARP1 = Tc16Cfg<KL>::EPI_WARP1;
    extern __shared__ __align__(1024) unsigned char sm[];
    const Tc16Geom g = Tc16Geom::make(S, p.r);
    constexpr int P = 8;
    constexpr int SEG = PCH / 8;  // 16-byte segments per pixel-box row
    const int r = p.r;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int kr1 = min(p.row_end, p.Ry_reg);
    const int ylo = max(0, p.slab_y0), yhi = min(p.H, p.slab_y1);

    float* const nc2 = reinterpret_cast<float*>(sm + g.off_nc);  // nc of tile it: nc2 + (it & 1) NT NB
    __half* const pl = reinterpret_cast<__half*>(sm + g.off_pl);
    uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + g.off_bar);
    uint64_t* const tfull = bars;
    uint64_t* const tempty = tfull + NTS;
    uint64_t* const sfull = tempty + NTS;
    uint64_t* const sempty = sfull + EPI_WARPS * NSLOT;
    uint64_t* const b_raw = sempty + EPI_WARPS * NSLOT;  // TMA box landed
    uint64_t* const b_xa = b_raw + 1;                    // X and A of the tile built
    uint64_t* const b_mma = b_raw + 2;                   // the tile's MMAs completed
    uint64_t* const b_nc = b_raw + 3;                    // [2] candidate norms built (by tile parity)
    uint64_t* const info_full = b_raw + 7;
    uint64_t* const info_empty = info_full + NINFO;
    volatile int* const gate_pub = reinterpret_cast<volatile int*>(info_empty + NINFO);
    volatile int* const consumed = gate_pub + EPI_WARPS * 32;  // rows taken by selector w (all tiles)
    volatile int* const info = consumed + EPI_WARPS;            // [NINFO][INFO_W]
    int* const red = const_cast<int*>(info + NINFO * INFO_W);
    volatile int* const sched = red + 2 * NPRO_MAX;             // tile fetched by the producers
    uint32_t* const tslot = reinterpret_cast<uint32_t*>(const_cast<int*>(sched + 1));

    if (threadIdx.x == 0) {
        for (int i = 0; i < NTS; ++i) {
            tc::mbar_init(&tfull[i], 1);
            tc::mbar_init(&tempty[i], EPI_WARPS * EPI_HALVES);
        }
        for (int i = 0; i < EPI_WARPS * NSLOT; ++i) {
            tc::mbar_init(&sfull[i], 1);
            tc::mbar_init(&sempty[i], 1);
        }
        tc::mbar_init(b_raw, 1);
        tc::mbar_init(b_xa, NPRO);
        tc::mbar_init(b_mma, 1);
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&b_nc[i], NPRO);
        }
        for (int i = 0; i < NINFO; ++i) {
            tc::mbar_init(&info_full[i], 1);
            tc::mbar_init(&info_empty[i], 1 + (1 + EPI_HALVES) * EPI_WARPS);  // MMA, epilogue, selectors
        }
        tc::fence_mbar_init();
    }
    if (threadIdx.x < EPI_WARPS) consumed[threadIdx.x] = 0;
    if (warp == MMA_WARP) tc::tmem_alloc<TMEM_COLS>(tslot);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tmem = *tslot;

    if (warp >= PRO_WARP0 && warp < PRO_WARP0 + NPRO) {
        // ---------------- producers: the next tile's operands while the current one is matched
        const int tp = threadIdx.x - 32 * PRO_WARP0, pw = warp - PRO_WARP0;
        for (int it = 0;; ++it) {
            // tiles are handed out dynamically (first one = blockIdx.x), one tile ahead of the
            // matching, so CTAs whose tiles ran long take fewer
            if (tp == 0) sched[0] = it == 0 ? (int)blockIdx.x : (int)gridDim.x + (int)atomicAdd(&g_tc16_sched[2 * sslot], 1u);
            tc::named_bar(PRO_BAR, 32 * NPRO);
            const int tile = sched[0];
            if (tile >= ntiles) {
                if (tp == 0) {
                    const int slot = it % NINFO;
                    if (it >= NINFO) tc::mbar_wait_long(&info_empty[slot], ((it / NINFO) - 1) & 1, 256);
                    info[slot * INFO_W] = -1;
                    tc::mbar_arrive(&info_full[slot]);
                }
                for (int j = max(0, it - 2); j < it; ++j)  // the epilogue's last two arrivals
                    tc::named_bar(EPI_PRO_BAR + (j & 1), 32 * (NPRO + EPI_WARPS * EPI_HALVES));
                break;
            }
            const Tc16Tile T(p, tile);
            const int gy0 = S * T.ky0 - r, gx0 = S * T.kx0 - r;
            // the box starts at the 8-column boundary at or left of gx0 (TMA box coordinates
            // are 16-byte aligned); plane column c + sh is candidate-area column c
            const int sh = gx0 & 7, xb = gx0 - sh;
            const int slot = it % NINFO;
            const bool tr = tp == 0 && it < 40;
            if (tr) TC_TRP(2000 + it * 8, clock64());
            // (1) the PR x 80 pixel box; every read of the plane by the previous tile ended at
            // the producer barrier that closed its iteration
            if (use_tma) {
                if (tp == 0) {
                    tc::fence_proxy_async_smem();
                    tc::mbar_expect_tx(b_raw, (uint32_t)(g.PR * PCH * 2));
                    tc::tma_load_3d(pl, &tmap, xb, gy0 - p.slab_y0, T.bimg, b_raw);
                }
                tc::mbar_wait(b_raw, it & 1);
            } else {
                const int16_t* __restrict__ img = p.img + (int64_t)T.bimg * p.img_bstride;
                for (int task = tp; task < g.PR * SEG; task += 32 * NPRO) {
                    const int row = task / SEG, seg = task - row * SEG;
                    const int gy = gy0 + row, gx = xb + 8 * seg;
                    const bool rowok = gy >= ylo && gy < yhi;
                    const int16_t* src = img + (int64_t)(gy - p.slab_y0) * p.W;
                    uint32_t wv[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int x0 = gx + 2 * q, x1 = x0 + 1;
                        const uint32_t v0 = (rowok && x0 >= 0 && x0 < p.W) ? (uint16_t)src[x0] : 0u;
                        const uint32_t v1 = (rowok && x1 >= 0 && x1 < p.W) ? (uint16_t)src[x1] : 0u;
                        wv[q] = v0 | (v1 << 16);
                    }
                    *reinterpret_cast<uint4*>(pl + task * 8) = make_uint4(wv[0], wv[1], wv[2], wv[3]);
                }
                tc::named_bar(PRO_BAR, 32 * NPRO);
            }
            if (tr) TC_TRP(2000 + it * 8 + 1, clock64());
            // (2) range of the in-image pixels -> centre, fp16 exactness bound
            int lo = INT_MAX, hi = INT_MIN;
            for (int task = tp; task < g.PR * SEG; task += 32 * NPRO) {
                const int row = task / SEG, seg = task - row * SEG;
                const int gy = gy0 + row, gx = xb + 8 * seg;
                if (gy < ylo || gy >= yhi) continue;
                const uint4 v = *reinterpret_cast<const uint4*>(pl + task * 8);
                const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int z = (int)(int16_t)(wv[j >> 1] >> (16 * (j & 1)));
                    const int c = 8 * seg + j - sh;  // column of the 72-column area
                    if (gx + j >= 0 && gx + j < p.W && c >= 0 && c < 72) {
                        lo = min(lo, z);
                        hi = max(hi, z);
                    }
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
                hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            }
            if (lane == 0) {
                red[pw] = lo;
                red[NPRO + pw] = hi;
            }
            tc::named_bar(PRO_BAR, 32 * NPRO);
#pragma unroll
            for (int i = 0; i < NPRO; ++i) {
                lo = min(lo, red[i]);
                hi = max(hi, red[NPRO + i]);
            }
            const int cz = (lo + hi) >> 1;
            const bool skip = max(hi - cz, cz - lo) > MMAX;
            if (tp == 0) {
                if (it >= NINFO) tc::mbar_wait_long(&info_empty[slot], ((it / NINFO) - 1) & 1, 256);
                volatile int* const in = info + slot * INFO_W;
                in[0] = tile;
                in[1] = T.bimg;
                in[2] = T.ky0;
                in[3] = T.kx0;
                in[4] = tc_step(min(g.NT - 1, (p.H - P) - gy0) - max(0, -gy0) + 1);
                in[5] = skip ? 1 : 0;
                if (skip) {  // the int8 kernel redoes this tile
                    const int64_t ref = (int64_t)T.bimg * p.out_bstride +
                                        (int64_t)(T.ky0 - p.row_begin) * p.Rx + T.kx0;
                    p.dist[ref * p.K] = TC_TILE_MARK;
                }
                tc::mbar_arrive(&info_full[slot]);
            }
            if (tr) TC_TRP(2000 + it * 8 + 2, clock64());
            // (3) centred fp16 plane in place (pixels outside the image only feed masked
            // candidates: 0 = cz)
            if (!skip) {
                for (int task = tp; task < g.PR * SEG; task += 32 * NPRO) {
                    const int row = task / SEG, seg = task - row * SEG;
                    const int gy = gy0 + row, gx = xb + 8 * seg;
                    const bool rowok = gy >= ylo && gy < yhi;
                    const uint4 rv = *reinterpret_cast<const uint4*>(pl + task * 8);
                    const uint32_t rw[4] = {rv.x, rv.y, rv.z, rv.w};
                    uint32_t hw[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int j = 2 * q;
                        const bool in0 = rowok && gx + j >= 0 && gx + j < p.W;
                        const bool in1 = rowok && gx + j + 1 >= 0 && gx + j + 1 < p.W;
                        const int v0 = in0 ? (int)(int16_t)(rw[q] & 0xffffu) - cz : 0;
                        const int v1 = in1 ? (int)(int16_t)(rw[q] >> 16) - cz : 0;
                        const __half2 h2 = __halves2half2(__int2half_rn(v0), __int2half_rn(v1));
                        hw[q] = *reinterpret_cast<const uint32_t*>(&h2);
                    }
                    *reinterpret_cast<uint4*>(pl + task * 8) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                }
            }
            tc::named_bar(PRO_BAR, 32 * NPRO);
            // (4) candidate norms N_q = P x P box sums of squares (integers < 2^24: exact in
            // fp32) into the buffer of this tile's parity, free once the epilogue left tile it - 2
            // (long ago: built during the previous tile); a thread per (column, half)
            // (a named barrier per tile parity: the producers sleep in hardware; the epilogue
            // cannot leave tile it before these norms exist, so the arrivals alternate)
            if (it > 1) tc::named_bar(EPI_PRO_BAR + (it & 1), 32 * (NPRO + EPI_WARPS * EPI_HALVES));
            float* const nc = nc2 + (it & 1) * g.NT * NB;
            if (tr) TC_TRP(2000 + it * 8 + 6, clock64());
            for (int task = tp; !skip && task < 2 * NB; task += 32 * NPRO) {
                const int n = task & 63, h = task >> 6;
                const int t0 = h ? (g.NT + 1) >> 1 : 0, t1 = h ? g.NT : (g.NT + 1) >> 1;
                auto hsq = [&](int y) -> float {
                    const uint4 v = load16h(pl + y * PCH, n + sh);
                    const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
                    float s0 = 0.f, s1 = 0.f;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float f0 = __half2float(__ushort_as_half((unsigned short)(wv[q] & 0xffffu)));
                        const float f1 = __half2float(__ushort_as_half((unsigned short)(wv[q] >> 16)));
                        s0 = fmaf(f0, f0, s0);
                        s1 = fmaf(f1, f1, s1);
                    }
                    return s0 + s1;
                };
                float ring[8];
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k < 7; ++k) {
                    ring[k] = hsq(t0 + k);
                    acc += ring[k];
                }
                ring[7] = 0.f;
                for (int tb = t0; tb < t1; tb += 8) {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const int t = tb + k;
                        if (t < t1) {
                            const int k7 = (k + 7) & 7;
                            ring[k7] = hsq(t + 7);
                            acc += ring[k7];
                            nc[t * NB + n] = acc;
                            acc -= ring[k];
                        }
                    }
                }
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&b_nc[it & 1]);
            if (tr) TC_TRP(2000 + it * 8 + 7, clock64());
            // (5) X and A, once the previous tile's MMAs no longer read them
            if (tr) TC_TRP(2000 + it * 8 + 3, clock64());
            // wait for the MMA warp's word that the previous tile's MMAs completed: a named
            // barrier, so the producers sleep in hardware instead of polling for a whole tile
            if (it > 0) tc::named_bar(MMA_PRO_BAR, 32 * (NPRO + 1));
            if (tr) TC_TRP(2000 + it * 8 + 4, clock64());
            if (!skip) {
                uint8_t* const xop = sm + g.off_x;
                for (int u = tp; u < g.PR * NB; u += 32 * NPRO) {
                    const int y = u >> 6, n = u & 63;
                    *reinterpret_cast<uint4*>(xop + y * XP + n * 16) = load16h(pl + y * PCH, n + sh);
                }
                tc::fence_proxy_async_smem();  // generic-proxy stores -> the tensor core
                // A: TMEM lane m = reference m = 8 a + b holds its patch, K = 8 i + j, two fp16
                // per column; producer warp q writes its lane quarter (warp % 4)
                const bool with_q0 = NPRO == 3 && (warp & 3) == 1;  // quarter 0 has no producer warp
                for (int q = with_q0 ? 0 : (warp & 3); q <= (warp & 3); q += with_q0 ? 1 : 4) {
                    const int m = 32 * q + lane;
                    const int row = r + S * (m >> 3), col = r + S * (m & 7) + sh;
                    uint32_t av[32];
#pragma unroll
                    for (int i = 0; i < P; ++i) {
                        const uint4 v = load16h(pl + (row + i) * PCH, col);
                        av[4 * i + 0] = v.x;
                        av[4 * i + 1] = v.y;
                        av[4 * i + 2] = v.z;
                        av[4 * i + 3] = v.w;
                    }
                    if (with_q0 && q == 0) {  // copied into TMEM by the MMA warp (quarter 0)
                        uint32_t* const a0 = reinterpret_cast<uint32_t*>(sm + g.off_a0);
#pragma unroll
                        for (int c = 0; c < 32; ++c) a0[c * 32 + lane] = av[c];
                    } else {
                        tc::tmem_st32(tmem + TM_A + ((uint32_t)(32 * q) << 16), av);
                        tc::tmem_wait_st();
                    }
                }
                tc::tc_fence_before();
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(b_xa);
            if (tr) TC_TRP(2000 + it * 8 + 5, clock64());
            tc::named_bar(PRO_BAR, 32 * NPRO);  // plane reads done before the next box lands
        }
    } else if (warp == MMA_WARP) {
        // ---------------- MMA issuer: 4 x (M128 N64 K16) per candidate row (lane 0 issues; the
        // whole warp copies lane quarter 0's A rows into TMEM when NPRO == 3 and releases the
        // producers after each tile)
        const unsigned wm = 0xffffffffu;
        {
            const uint32_t idesc = tc::idesc_f16f16_f32(128, NB);
            const uint32_t xa = tc::smem_u32(sm + g.off_x);
            int s = 0;
            for (int it = 0;; ++it) {
                const int slot = it % NINFO;
                tc::mbar_wait(&info_full[slot], (it / NINFO) & 1);
                const volatile int* const in = info + slot * INFO_W;
                const int tile = in[0], ky0 = in[2], step = in[4], skip = in[5];
                __syncwarp(wm);
                if (lane == 0) tc::mbar_arrive(&info_empty[slot]);
                if (tile < 0) break;
                tc::mbar_wait(b_xa, it & 1);
                if (lane == 0 && it < 40) TC_TRP(3000 + it * 4, clock64());
                if (skip) {
                    __syncwarp(wm);
                    if (lane == 0) tc::mbar_arrive(b_mma);
                    __syncwarp(wm);
                    tc_release_producers(b_mma, it, NPRO, lane, wm);
                    continue;
                }
                if (NPRO == 3) {  // A rows of lane quarter 0: shared buffer -> TMEM (this warp's quarter)
                    const uint32_t* const a0 = reinterpret_cast<const uint32_t*>(sm + g.off_a0);
                    uint32_t av[32];
#pragma unroll
                    for (int c = 0; c < 32; ++c) av[c] = a0[c * 32 + lane];
                    tc::tmem_st32(tmem + TM_A, av);
                    tc::tmem_wait_st();
                    tc::tc_fence_before();
                    __syncwarp(wm);
                }
                tc::tc_fence_after();
                // the whole warp walks the rows (converged: the waits are warp-wide), lane 0 issues
                const int gy0 = S * ky0 - r;
                const int t_lo = max(0, -gy0), t_hi = min(g.NT - 1, (p.H - P) - gy0);
                RowSeq seq;
                seq.init(S, r, t_lo, t_hi, step);
                const int nseq = t_hi - t_lo + 1;
                for (int k = 0; k < nseq; ++k, ++s) {
                    const int ts = s % NTS;
                    const int t = seq.next();
                    if (s >= NTS) tc::mbar_wait(&tempty[ts], ((s / NTS) - 1) & 1);
                    tc::tc_fence_after();
                    if (lane == 0) {
                        const uint32_t bb = xa + (uint32_t)(t * XP);
#pragma unroll
                        for (int ks = 0; ks < 4; ++ks)
                            tc::mma_f16_ts(tmem + (uint32_t)(ts * NB), tmem + TM_A + ks * 8,
                                           tc::smem_desc(bb + ks * 2 * XP, XP, 128), idesc, ks);
                        tc::mma_commit(&tfull[ts]);
                    }
                    __syncwarp(wm);
                }
                if (lane == 0) tc::mma_commit(b_mma);  // X and A free once these MMAs completed
                if (lane == 0 && it < 40) TC_TRP(3000 + it * 4 + 1, clock64());
                __syncwarp(wm);  // the warp stays converged for the next tile's TMEM copy
                tc_release_producers(b_mma, it, NPRO, lane, wm);
            }
        }
    } else if (warp < EPI_WARPS || (EPI_HALVES == 2 && warp >= EPI_WARP1)) {
        // ---------------- epilogue warp w: accumulators of lane quarter w -> staged rows
        const int w = warp & 3, half = warp >= EPI_WARP1 ? 1 : 0;
        const int a = 4 * w + (lane >> 3), bb = lane & 7;
        const uint32_t taddr = tmem + ((uint32_t)(32 * w) << 16);
        const int gate0 = p.tdr0 + 1;
        uint32_t* const stg0 = reinterpret_cast<uint32_t*>(sm + g.off_stg) +
                               (w * NSLOT * 32 + lane) * STG_PITCH;
        int s = 0, used = 0;
        for (int it = 0;; ++it) {
            const int slot_i = it % NINFO;
            tc::mbar_wait(&info_full[slot_i], (it / NINFO) & 1);
            const volatile int* const in = info + slot_i * INFO_W;
            const int tile = in[0], ky0 = in[2], kx0 = in[3], step = in[4], skip = in[5];
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&info_empty[slot_i]);
            if (tile < 0) break;
            // the tile's constants before its norms are ready
            const int gy0 = S * ky0 - r, gx0 = S * kx0 - r;
            const int t_lo = max(0, -gy0), t_hi = min(g.NT - 1, (p.H - P) - gy0);
            const int j_lo = max(0, -gx0), j_hi = min(g.NJ - 1, (p.W - P) - gx0);
            const bool refok = (ky0 + a < kr1) && (kx0 + bb < p.Rx_reg);
            const int ty = r + S * a, tx = r + S * bb;
            const bool warp_active = __any_sync(0xffffffffu, refok);
            const int wt0 = S * 4 * w, wt1 = S * (4 * w + 3) + 2 * r;
            const int c0 = max(S * bb, j_lo), c1 = min(S * bb + 2 * r, j_hi);
            const uint64_t cm = (c1 >= c0) ? ((c1 >= 63 ? ~0ull : ((2ull << c1) - 1ull)) &
                                              ~((1ull << c0) - 1ull))
                                           : 0ull;
            RowSeq seq;
            seq.init(S, r, t_lo, t_hi, step);
            tc::mbar_wait(&b_nc[it & 1], (it >> 1) & 1);
            const float* const nc = nc2 + (it & 1) * g.NT * NB;
            if (lane == 0 && it < 40) TC_TRP(4000 + it * 16 + w * 4, clock64());
            if (!skip) {
                const float Nr = nc[ty * NB + tx];
                const int tile_start = used;
                bool lists_full = false;
                if (lane == 0 && it < 40) TC_TRP(4400 + it * 8 + w, clock64());
                const int nseq = t_hi - t_lo + 1;
                for (int k = 0; k < nseq; ++k, ++s) {
                    const int ts = s % NTS;
                    const int t = seq.next();
                    if (lane == 0 && it == 5 && w == 0) TC_TRP(6400 + (used - tile_start), clock64());
                    tc::mbar_wait(&tfull[ts], (s / NTS) & 1);
                    if (!(warp_active && t >= wt0 && t <= wt1)) {
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive(&tempty[ts]);
                        continue;
                    }
                    if (lane == 0 && it == 5 && w == 0) TC_TRP(6500 + (used - tile_start), clock64());
                    const int slot = used % NSLOT;
                    static_assert(NSLOT == 2, "half h stages the rows of slot h");
                    if (EPI_HALVES == 2 && slot != half) {  // the other half stages this row
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive(&tempty[ts]);
                        ++used;
                        continue;
                    }
                    // EARLY (two epilogue halves): the gate-independent half first -- TMEM
                    // load, u = N_q - 2 <f_p, f_q>, TMEM stage released -- then the staging slot
                    // and the gate; otherwise v = u - T in one pass after the gate is known
                    constexpr bool EARLY = EPI_HALVES == 2 && EARLY15;
                    const uint32_t tb = taddr + (uint32_t)(ts * NB);
                    uint32_t acc[64];
                    if (EARLY) {
                        tc::tc_fence_after();
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) tc::tmem_ld16p(tb + ch * 16, acc + ch * 16);
                        tc::tmem_wait_ld();
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) tc::tmem_tie16(acc + ch * 16);
                        tc::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive(&tempty[ts]);
                        const float4* ncv = reinterpret_cast<const float4*>(nc + t * NB);
#pragma unroll
                        for (int q = 0; q < 16; ++q) {
                            const float4 n4 = ncv[q];
                            uint32_t* const u = acc + 4 * q;
                            u[0] = __float_as_uint(fmaf(__uint_as_float(u[0]), -2.f, n4.x));
                            u[1] = __float_as_uint(fmaf(__uint_as_float(u[1]), -2.f, n4.y));
                            u[2] = __float_as_uint(fmaf(__uint_as_float(u[2]), -2.f, n4.z));
                            u[3] = __float_as_uint(fmaf(__uint_as_float(u[3]), -2.f, n4.w));
                        }
                    }
                    if (used >= NSLOT) tc::mbar_wait(&sempty[w * NSLOT + slot], ((used / NSLOT) - 1) & 1);
                    int gate = gate0;
                    if (used > tile_start) {
                        // (once every list of the quarter is full in this tile, no more votes)
                        const bool check = !(EPI_HALVES == 2 && GATEFLAG15 && lists_full);
                        if (check) while (consumed[w] <= tile_start) __nanosleep(32);
                        gate = gate_pub[w * 32 + lane];
                        if (check) {
                            if (__any_sync(0xffffffffu, gate == gate0 && refok)) {
                                while (consumed[w] < used) __nanosleep(32);
                                gate = gate_pub[w * 32 + lane];
                            } else {
                                lists_full = true;
                            }
                        }
                    }
                    if (lane == 0 && it == 5 && w == 0) TC_TRP(6600 + (used - tile_start), clock64());
                    const float Tg = (float)(gate - __float2int_rn(Nr));
                    uint32_t* const stg = stg0 + slot * 32 * STG_PITCH;
                    uint32_t msk[2] = {0u, 0u};
                    if (!EARLY) {
                        tc::tc_fence_after();
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) tc::tmem_ld16p(tb + ch * 16, acc + ch * 16);
                        tc::tmem_wait_ld();
#pragma unroll
                        for (int ch = 0; ch < 4; ++ch) tc::tmem_tie16(acc + ch * 16);
                        if (lane == 0 && it == 5 && w == 0) TC_TRP(6900 + (used - tile_start), clock64());
                    }
#pragma unroll
                    for (int cc = 0; cc < 4; ++cc) {
                        const int ch = cc ^ 1;  // per 32-column half, the upper 16 columns first
                        float v[16];
                        if (EARLY) {
#pragma unroll
                            for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(acc[16 * ch + j]) - Tg;
                        } else {
                            const float4* ncv = reinterpret_cast<const float4*>(nc + t * NB + ch * 16);
#pragma unroll
                            for (int q = 0; q < 4; ++q) {
                                const float4 n4 = ncv[q];
                                v[4 * q + 0] = fmaf(__uint_as_float(acc[16 * ch + 4 * q + 0]), -2.f, n4.x - Tg);
                                v[4 * q + 1] = fmaf(__uint_as_float(acc[16 * ch + 4 * q + 1]), -2.f, n4.y - Tg);
                                v[4 * q + 2] = fmaf(__uint_as_float(acc[16 * ch + 4 * q + 2]), -2.f, n4.z - Tg);
                                v[4 * q + 3] = fmaf(__uint_as_float(acc[16 * ch + 4 * q + 3]), -2.f, n4.w - Tg);
                            }
                        }
                        uint32_t& m = msk[ch >> 1];
#pragma unroll
                        for (int j = 15; j >= 0; --j) m = __funnelshift_l(__float_as_uint(v[j]), m, 1);
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            *reinterpret_cast<float4*>(stg + ch * 16 + 4 * q) =
                                make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                    }
                    if (lane == 0 && it == 5 && w == 0) TC_TRP(7000 + (used - tile_start), clock64());
                    if (!EARLY) {
                        tc::tc_fence_before();
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive(&tempty[ts]);
                    }
                    const bool rowin = refok && t >= S * a && t <= S * a + 2 * r;
                    uint64_t mm = rowin ? ((((uint64_t)msk[1]) << 32 | msk[0]) & cm) : 0ull;
                    if (t == ty) mm &= ~(1ull << tx);  // the reference itself is slot 0
                    *reinterpret_cast<uint4*>(stg + 64) =
                        make_uint4((uint32_t)mm, (uint32_t)(mm >> 32), (uint32_t)gate, (uint32_t)t);
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive(&sfull[w * NSLOT + slot]);
                    if (lane == 0 && it == 5 && w == 0) TC_TRP(6700 + (used - tile_start), clock64());
                    if (lane == 0 && it < 40 && used == tile_start) TC_TRP(4000 + it * 16 + w * 4 + 1, clock64());
                    ++used;
                }
            }
            __syncwarp();
            // nc buffer (it & 1) free again
            asm volatile("bar.arrive %0, %1;" ::"r"(EPI_PRO_BAR + (it & 1)),
                         "r"(32 * (NPRO + EPI_WARPS * EPI_HALVES)) : "memory");
            if (lane == 0 && it < 40) TC_TRP(4000 + it * 16 + w * 4 + 2, clock64());
        }
    } else if (warp >= SEL_WARP0 && warp < SEL_WARP0 + EPI_WARPS) {
        // ---------------- selector warp w: per-lane top-(K-1) lists, then the output rows
        const int w = warp - SEL_WARP0;
        const int a = 4 * w + (lane >> 3), bb = lane & 7;
        const uint32_t side = (uint32_t)p.side;
        const int cb = p.cb;
        const uint32_t* const stg0 = reinterpret_cast<const uint32_t*>(sm + g.off_stg) +
                                     (w * NSLOT * 32 + lane) * STG_PITCH;
        constexpr int KP = KL + 1;
        static_assert((KP & (KP - 1)) == 0 && KP <= 32, "list length must be a power of two");
        // d + 2^23 as an fp32 bit pattern is 0x4B000000 + d (exact for d < 2^23), and
        // 0x4B000000 << cb == 0 (mod 2^32) for cb >= 8: key = bits(v + gate + 2^23) << cb | code
        const uint32_t kmul = 1u << cb;
        int used = 0;
        for (int it = 0;; ++it) {
            const int slot_i = it % NINFO;
            tc::mbar_wait(&info_full[slot_i], (it / NINFO) & 1);
            const volatile int* const in = info + slot_i * INFO_W;
            const int tile = in[0], bimg = in[1], ky0 = in[2], kx0 = in[3], skip = in[5];
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&info_empty[slot_i]);
            if (tile < 0) break;
            if (lane == 0 && it < 40) TC_TRP(5000 + it * 16 + w * 4, clock64());
            if (skip) continue;
            const int gy0 = S * ky0 - r;
            const int t_lo = max(0, -gy0), t_hi = min(g.NT - 1, (p.H - P) - gy0);
            const bool refok = (ky0 + a < kr1) && (kx0 + bb < p.Rx_reg);
            const bool warp_active = __any_sync(0xffffffffu, refok);
            const int wt0 = S * 4 * w, wt1 = S * (4 * w + 3) + 2 * r;
            uint32_t L[KP];
#pragma unroll
            for (int i = 0; i < KP; ++i) L[i] = KEY_INF;
            int nrel = 0;
            if (warp_active) {
                const int lo = max(wt0, t_lo), hi = min(wt1, t_hi);
                nrel = hi >= lo ? hi - lo + 1 : 0;
            }
            for (int k = 0; k < nrel; ++k, ++used) {
                const int slot = used % NSLOT;
                if (lane == 0 && it == 5 && w == 0) TC_TRP(6200 + k, clock64());
                tc::mbar_wait(&sfull[w * NSLOT + slot], (used / NSLOT) & 1);
                if (lane == 0 && it == 5 && w == 0) TC_TRP(6300 + k, clock64());
                const uint32_t* const stg = stg0 + slot * 32 * STG_PITCH;
                const uint4 hdr = *reinterpret_cast<const uint4*>(stg + 64);
                uint32_t mlo = hdr.x, mhi = hdr.y;
                const float GB = (float)(int)hdr.z + 8388608.0f;  // d + 2^23 = v + gate + 2^23
                const uint32_t code_row = (uint32_t)((int)hdr.w - S * a) * side - (uint32_t)(S * bb);
                int R = (int)__reduce_max_sync(0xffffffffu, (unsigned)(__popc(mlo) + __popc(mhi)));
                tc16_insert_row<KP>(L, stg, mlo, mhi, GB, code_row, kmul, S * bb, r, R);
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&sempty[w * NSLOT + slot]);
                const uint32_t top = L[KL - 1];
                gate_pub[w * 32 + lane] = ((top == KEY_INF) ? p.tdr0 : min((int)(top >> cb), p.tdr0)) + 1;
                __syncwarp();
                if (lane == 0) consumed[w] = used + 1;
                if (lane == 0 && it < 40 && k == 0) TC_TRP(5000 + it * 16 + w * 4 + 1, clock64());
                if (lane == 0 && it == 5 && w == 0) {
                    TC_TRP(6000 + k, clock64());
                    TC_TRP(6100 + k, R);
                }
            }
            if (lane == 0 && it < 40) TC_TRP(5000 + it * 16 + w * 4 + 2, clock64());
            // ---- output straight from the registers: slot 0 = self, ranks 1.. = list, pads
            if (refok) tc16_write_refs<S, KL>(p, L, a, bb, ky0, kx0, bimg, cb, side);
            __syncwarp();
            if (lane == 0 && it < 40) TC_TRP(5000 + it * 16 + w * 4 + 3, clock64());
        }
    }

    tc::tc_fence_before();
    __syncthreads();
    if (warp == MMA_WARP) {
        tc::tc_fence_after();
        tc::tmem_dealloc<tc16::TMEM_COLS>(tmem);
    }
    // the last CTA out resets the launch's tile counter (every fetch has happened by now)
    if (threadIdx.x == 0 && atomicAdd(&g_tc16_sched[2 * sslot + 1], 1u) == gridDim.x - 1) {
        g_tc16_sched[2 * sslot] = 0u;
        g_tc16_sched[2 * sslot + 1] = 0u;
    }
}

// cuTensorMapEncodeTiled from the driver (no link-time libcuda dependency)
typedef CUresult (*Tc16EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static inline Tc16EncodeTiled tc16_encode_fn() {
    static const Tc16EncodeTiled fn = []() -> Tc16EncodeTiled {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        return reinterpret_cast<Tc16EncodeTiled>(f);
    }();
    return fn;
}
// Tensor map of the call's pixels [B][slab rows][W] (int16 bits as uint16) with the producer's PR x 80 box;
// false when TMA cannot address it (row pitch or base not 16-byte aligned): plain loads then.
static inline bool tc16_make_tmap(const MatchParams& p, int PR, CUtensorMap* m) {
    if ((p.W % 8) != 0 || (reinterpret_cast<uintptr_t>(p.img) & 15u) != 0) return false;
    const Tc16EncodeTiled enc = tc16_encode_fn();
    if (!enc) return false;
    const int rows = p.slab_y1 - p.slab_y0;
    const cuuint64_t dims[3] = {(cuuint64_t)p.W, (cuuint64_t)rows, (cuuint64_t)p.B};
    const cuuint64_t strides[2] = {(cuuint64_t)p.W * 2, (cuuint64_t)p.img_bstride * 2};
    const cuuint32_t box[3] = {(cuuint32_t)tc16::PCH, (cuuint32_t)PR, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, const_cast<int16_t*>(p.img), dims, strides, box,
               estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static inline int tc16_sm_count() {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
        n = 148;
    return n;
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
    const long long nx = (p.Rx_reg + tc16::TX - 1) / tc16::TX, ny = (kr1 - kr0 + tc16::TY - 1) / tc16::TY;
    const long long ntiles = nx * ny * p.B;
    if (ntiles >= (1LL << 31)) return cudaErrorInvalidValue;
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    static const int no_tma = getenv("GBM3D_TC16_NO_TMA") != nullptr;  // dev switch
    const int use_tma = (!no_tma && tc16_make_tmap(p, g.PR, &tm)) ? 1 : 0;
    const int nsm = tc16_sm_count();
    const int grid = (int)(ntiles < nsm ? ntiles : nsm);
    static std::atomic<unsigned> calls{0};
    const int sslot = (int)(calls.fetch_add(1u) % tc16::NSCHED);
    kern<<<grid, tc16::Tc16Cfg<KL>::THREADS, g.total, stream>>>(p, tm, use_tma, (int)ntiles, sslot);
    if (launches) ++*launches;
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    static const bool dbg = getenv("GBM3D_DEBUG") != nullptr;
    if (dbg) {
        e = cudaStreamSynchronize(stream);
        fprintf(stderr, "gbm3d: tc16 grid %d tiles %lld tma %d smem %d: %s\n", grid, ntiles, use_tma,
                g.total, cudaGetErrorString(e));
        if (e != cudaSuccess) return e;
    }
    // exact int8 kernel for the tiles the fp16 kernel marked (usually none)
    return launch_tc<S, KL>(p, stream, launches, 1);
}

}  // namespace gbm3d
