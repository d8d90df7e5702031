// Product-form block matching on the 5th-generation tensor cores.
//
// Method.  For integer patches the SSD of Eq. (1) splits as Eq. (2):
//     d(p, q) = ||f_p||^2 + ||f_q||^2 - 2 <f_p, f_q>,
// the form the paper evaluates with local cross-correlations (Prop. 1; the box
// filter of the norms is step 1).  Here every term is computed exactly in int32
// arithmetic modulo 2^32: the true d is < 2^31 (range precondition, R10), so the
// wrapped sum equals d bit for bit.  Pixels are offset to z' = z + 32768 (0..65535; the SSD is
// translation invariant) and split into bytes z' = 256 h + l, so
//     <f_p, f_q> = 65536 <h_p, h_q> + 256 (<h_p, l_q> + <l_p, h_q>) + <l_p, l_q>,
// four u8 x u8 -> s32 inner products, i.e. tcgen05.mma kind::i8 (exact integer MMA).
//
// Work mapping:
//   * CTA = a tile of 16 x 8 grid references (M = 128 MMA rows; TMEM lane m = reference
//     8a + b at grid offset (a, b)).  Warp w (0..3) owns TMEM lanes 32w.. = grid rows 4w..4w+3.
//   * The union of the tile's search windows is NT = 15S + 2r + 1 candidate rows x NJ = 7S + 2r
//     + 1 (<= 64) candidate columns.  One candidate row = one MMA N-tile of 64 columns: builder
//     warps write the row's 64 candidate patches (both byte planes, canonical K-major layout) into
//     a 4-stage shared-memory ring; one thread issues 8 MMAs (hh, mid, ll accumulators, K = 64 B
//     each plane) into one of two TMEM stages.
//   * Epilogue warps read the three accumulators (tcgen05.ld), form e = d - g for all 64
//     columns (g = the reference's current gate), mask the search window, and insert the
//     passing candidates into a per-lane sorted register list of the K-1 smallest 32-bit keys
//     (d << cb | displacement code, the same key order (d, idx) as the SSD kernel) with a
//     branch-free min/max insertion network, one round per passing key.
//   * Candidate rows are visited front/back interleaved (t_lo, t_hi, t_lo+1, t_hi-1, ...) so the
//     two TMEM stages in flight usually belong to disjoint sets of epilogue warps.
#pragma once
#include "common.cuh"
#include "tc_ptx.cuh"

namespace gbm3d {

#if GBM3D_TC_TRACE  // dev-only timeline of one CTA (clock64), read by gbm3d_dev_tc_trace
static __device__ long long g_tc_trace[8192];
// dev-only: per CTA (linear block id) start / end %globaltimer and SM id
static __device__ long long g_cta_span[65536][3];
__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ int smid() {
    int s;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
    return s;
}
#define TC_SPAN(k, v)                                                                      \
    do {                                                                                   \
        const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;   \
        if (cta < 65536) g_cta_span[cta][k] = (v);                                         \
    } while (0)
#else
#define TC_SPAN(k, v) \
    do {              \
    } while (0)
#endif
#if GBM3D_TC_TRACE
#define TC_TR(i, v)                                                                   \
    do {                                                                              \
        if (blockIdx.x == 10 && blockIdx.y == 10 && blockIdx.z == 0) g_tc_trace[i] = (v); \
    } while (0)
#else
#define TC_TR(i, v) \
    do {            \
    } while (0)
#endif

namespace tcm {
constexpr int TY = 16, TX = 8;  // reference tile (grid rows x grid cols) = 128 MMA rows
constexpr int NB = 64;          // candidate columns per MMA tile (N)
constexpr int PC = 72;          // byte-plane pitch: 64 candidate columns + 7 + pad
constexpr int NSTG = 4;         // B-operand ring stages
// warps 0-3: epilogue (TMEM -> e = d - gate, window masks, staged rows); 4-7: selectors (one
// per epilogue warp, same lane <-> reference map; register top-(K-1) lists); 8: MMA issuer;
// 9-10: B builders
constexpr int EPI_WARPS = 4, SEL_WARP0 = 4, MMA_WARP = 8, BLD_WARP0 = 9, NBLD = 2;
constexpr int THREADS = 32 * 11;
constexpr int NSLOT = 4;        // staged rows in flight per epilogue/selector pair
constexpr int STG_PITCH = 68;   // words per lane and staged row: e[64], mask lo/hi, gate, row
constexpr int A_BYTES = 128 * 64, B_BYTES = 64 * 64;  // one byte plane of A / of a B stage
constexpr uint32_t TMEM_COLS = 512;                   // 2 stages x (hh, mid, ll) x 64
}  // namespace tcm

// Shared-memory carve-up of one CTA (host and device agree).
struct TcGeom {
    int NT, PR, NJ;
    int off_a, off_b, off_hi, off_lo, off_nc, off_stg, off_bar, total;
    __host__ __device__ static TcGeom make(int S, int r) {
        using namespace tcm;
        TcGeom g;
        g.NT = 15 * S + 2 * r + 1;
        g.PR = g.NT + 7;
        g.NJ = 7 * S + 2 * r + 1;
        g.off_a = 0;                                    // A_hi, A_lo
        g.off_b = 2 * A_BYTES;                          // NSTG x (B_hi, B_lo)
        g.off_hi = g.off_b + NSTG * 2 * B_BYTES;        // byte planes of the pixel tile
        g.off_lo = g.off_hi + ((g.PR * PC + 15) & ~15);
        g.off_nc = g.off_lo + ((g.PR * PC + 15) & ~15);  // candidate norms [NT][64]
        g.off_stg = g.off_nc + g.NT * NB * 4;           // epilogue staging / prologue scratch
        g.off_bar = g.off_stg + EPI_WARPS * NSLOT * 32 * STG_PITCH * 4;
        // mbarriers: full/empty[NSTG], tfull/tempty[2], sfull/sempty[EPI_WARPS*NSLOT]; then the
        // published gates [EPI_WARPS*32] and the TMEM address
        g.total = g.off_bar + (2 * NSTG + 4 + 2 * EPI_WARPS * NSLOT) * 8 + EPI_WARPS * 32 * 4 + 16;
        return g;
    }
};

// 8 bytes at an arbitrary byte offset c of a 4-byte aligned shared row.
static __device__ __forceinline__ uint2 load8u(const uint8_t* row, int c) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(row) + (c >> 2);
    const uint32_t sh = (uint32_t)(c & 3) * 8u;
    const uint32_t a0 = w[0], a1 = w[1], a2 = w[2];
    return make_uint2(__funnelshift_r(a0, a1, sh), __funnelshift_r(a1, a2, sh));
}

// Canonical K-major (no swizzle) byte offset of (row, patch row i) for 64-byte K rows: core
// matrix (row/8, k/16) at (row/8)*512 + (k/16)*128, row-in-core * 16, k % 16; k = 8 i + j.
static __device__ __forceinline__ int kmaj_off(int row, int i) {
    return (row >> 3) * 512 + (i >> 1) * 128 + (row & 7) * 16 + (i & 1) * 8;
}

// Sorted list of the KL smallest keys: insert x (KEY_INF = no-op).  Branch-free network.
template <int KL>
static __device__ __forceinline__ void list_insert(uint32_t (&L)[KL], uint32_t x) {
#pragma unroll
    for (int i = KL - 1; i >= 1; --i) L[i] = min(L[i], max(L[i - 1], x));
    L[0] = min(L[0], x);
}

// Candidate rows are visited in a scrambled order t = lo + (s * step) mod n, step coprime to n
// near 0.618 n: spatially ordered visits (raster, centre-out) let the smooth image content
// keep the gates loose, a spread order fills the lists with typical distances early.
static __device__ __forceinline__ int tc_step(int n) {
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
// Running form: off_{s+1} = (off_s + step) mod n, off_0 = 0; row = lo + off.
static __device__ __forceinline__ int tc_next(int off, int n, int step) {
    off += step;
    return off >= n ? off - n : off;
}

// Exact per-reference recomputation with 64-bit keys from global memory (rare: only when tau
// exceeds the 32-bit key range and the list is not full).  Writes slots 1..K-1, returns count.
static __device__ __noinline__ int tc_exact_ref(const int16_t* __restrict__ img, int slab_y0,
                                                int H, int W, int P, int r, int ry, int rx,
                                                int K, int64_t tau, int32_t* oi, int32_t* od) {
    const int L = K - 1;
    int cnt = 0;
    const int cy0 = max(0, ry - r), cy1 = min(H - P, ry + r);
    const int cx0 = max(0, rx - r), cx1 = min(W - P, rx + r);
    for (int cy = cy0; cy <= cy1; ++cy) {
        for (int cx = cx0; cx <= cx1; ++cx) {
            if (cy == ry && cx == rx) continue;
            int64_t d = 0;
            for (int i = 0; i < P; ++i) {
                const int16_t* ra = img + (int64_t)(ry + i - slab_y0) * W + rx;
                const int16_t* rb = img + (int64_t)(cy + i - slab_y0) * W + cx;
                for (int j = 0; j < P; ++j) {
                    const int64_t df = (int64_t)ra[j] - (int64_t)rb[j];
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
    for (int i = cnt; i < L; ++i) {
        oi[1 + i] = self;
        od[1 + i] = -1;
    }
    return cnt;
}

// Tile marker written by the fp16 kernel (match_tc16.cuh) into the slot-0 distance of the
// tile's first reference when the tile's pixel range is outside its exactness bound; the int8
// kernel launched with only_marked = 1 recomputes exactly those tiles.
constexpr int32_t TC_TILE_MARK = -2;

// One reference tile (bx, by) of image bz; called by the whole CTA.
template <int S, int KL>
static __device__ __forceinline__ void tc_tile(const MatchParams& p, int bx, int by, int bz) {
    using namespace tcm;
    extern __shared__ __align__(1024) unsigned char sm[];
    const TcGeom g = TcGeom::make(S, p.r);
    constexpr int P = 8;
    const int r = p.r;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bimg = bz;
    const int kr1 = min(p.row_end, p.Ry_reg);
    const int ky0 = p.row_begin + by * TY, kx0 = bx * TX;
    const int gy0 = S * ky0 - r, gx0 = S * kx0 - r;  // global pixel of tile (0, 0)
    const int16_t* __restrict__ img = p.img + (int64_t)bimg * p.img_bstride;

    uint8_t* const pl_hi = sm + g.off_hi;
    uint8_t* const pl_lo = sm + g.off_lo;
    uint32_t* const nc = reinterpret_cast<uint32_t*>(sm + g.off_nc);
    uint64_t* const bars = reinterpret_cast<uint64_t*>(sm + g.off_bar);
    uint64_t* const full = bars;               // builders -> MMA   (count NBLD)
    uint64_t* const empty = bars + NSTG;       // MMA commit -> builders
    uint64_t* const tfull = bars + 2 * NSTG;   // MMA commit -> epilogue
    uint64_t* const tempty = tfull + 2;        // epilogue -> MMA   (count EPI_WARPS)
    uint64_t* const sfull = tempty + 2;                // epilogue warp w -> selector w
    uint64_t* const sempty = sfull + EPI_WARPS * NSLOT;  // selector w -> epilogue warp w
    volatile uint32_t* const gate_pub =
        reinterpret_cast<volatile uint32_t*>(sempty + EPI_WARPS * NSLOT);
    uint32_t* const tslot = reinterpret_cast<uint32_t*>(sempty + EPI_WARPS * NSLOT) + EPI_WARPS * 32;

    // valid candidate rows / columns of the tile (candidates lie fully inside the image)
    const int t_lo = max(0, -gy0), t_hi = min(g.NT - 1, (p.H - P) - gy0);
    const int j_lo = max(0, -gx0), j_hi = min(g.NJ - 1, (p.W - P) - gx0);
    const int nseq = t_hi - t_lo + 1;
    const int step = tc_step(nseq);

    // ---- prologue 1: pixel tile -> byte planes of z' = z + 32768, and z'^2 (mod 2^32)
    {
        uint32_t* sq = reinterpret_cast<uint32_t*>(sm + g.off_stg);
        const int ylo = max(0, p.slab_y0), yhi = min(p.H, p.slab_y1);
        for (int i = threadIdx.x; i < g.PR * PC; i += THREADS) {
            const int row = i / PC, col = i - row * PC;
            const int gy = gy0 + row, gx = gx0 + col;
            const int z = (gy >= ylo && gy < yhi && gx >= 0 && gx < p.W)
                              ? (int)img[(int64_t)(gy - p.slab_y0) * p.W + gx]
                              : 0;
            const uint32_t zu = (uint32_t)(z + 32768);
            pl_hi[i] = (uint8_t)(zu >> 8);
            pl_lo[i] = (uint8_t)(zu & 255u);
            sq[i] = zu * zu;
        }
        if (threadIdx.x == 0) {
            for (int i = 0; i < NSTG; ++i) {
                tc::mbar_init(&full[i], NBLD);
                tc::mbar_init(&empty[i], 1);
            }
            for (int i = 0; i < 2; ++i) {
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
        if (threadIdx.x < EPI_WARPS * 32) gate_pub[threadIdx.x] = (uint32_t)(p.tdr0 + 1);
        __syncthreads();
        // horizontal sums of squares over the 8 patch columns (scratch in the B ring)
        uint32_t* hs = reinterpret_cast<uint32_t*>(sm + g.off_b);
        for (int i = threadIdx.x; i < g.PR * NB; i += THREADS) {
            const int row = i >> 6, c = i & 63;
            const uint32_t* q = sq + row * PC + c;
            uint32_t s = 0;
#pragma unroll
            for (int j = 0; j < P; ++j) s += q[j];
            hs[i] = s;
        }
        __syncthreads();
        // candidate norms N(t, j) = box sum over 8 rows (mod 2^32)
        for (int i = threadIdx.x; i < g.NT * NB; i += THREADS) {
            const uint32_t* q = hs + i;
            uint32_t s = 0;
#pragma unroll
            for (int k = 0; k < P; ++k) s += q[k * NB];
            nc[i] = s;
        }
        // A operand: reference m = 8a + b at tile position (r + S a, r + S b), both planes
        uint8_t* const a_hi = sm + g.off_a;
        uint8_t* const a_lo = a_hi + A_BYTES;
        for (int u = threadIdx.x; u < 128 * P; u += THREADS) {
            const int m = u >> 3, i = u & 7;
            const int row = r + S * (m >> 3) + i, col = r + S * (m & 7);
            const int off = kmaj_off(m, i);
            *reinterpret_cast<uint2*>(a_hi + off) = load8u(pl_hi + row * PC, col);
            *reinterpret_cast<uint2*>(a_lo + off) = load8u(pl_lo + row * PC, col);
        }
        tc::fence_proxy_async_smem();
        tc::tc_fence_before();
        __syncthreads();
        tc::tc_fence_after();
    }
    const uint32_t tmem = *tslot;
    if (threadIdx.x == 0) TC_TR(0, clock64());

    if (warp >= BLD_WARP0) {
        // ---- B builders: candidate row t -> 64 candidate patches, canonical K-major
        const int n = threadIdx.x - 32 * BLD_WARP0;  // candidate column 0..63
        int off = 0;
        for (int s = 0; s < nseq; ++s, off = tc_next(off, nseq, step)) {
            const int stage = s % NSTG;
            if (s >= NSTG) tc::mbar_wait(&empty[stage], ((s / NSTG) - 1) & 1);
            const int t = t_lo + off;
            uint8_t* const bh = sm + g.off_b + stage * 2 * B_BYTES;
            uint8_t* const bl = bh + B_BYTES;
#pragma unroll
            for (int i = 0; i < P; ++i) {
                const int off = kmaj_off(n, i);
                *reinterpret_cast<uint2*>(bh + off) = load8u(pl_hi + (t + i) * PC, n);
                *reinterpret_cast<uint2*>(bl + off) = load8u(pl_lo + (t + i) * PC, n);
            }
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&full[stage]);
        }
    } else if (warp == MMA_WARP) {
        // ---- MMA issuer (one thread): 8 x (M128 N64 K32) per candidate row
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_u8u8_s32(128, NB);
            const uint32_t ah = tc::smem_u32(sm + g.off_a), al = ah + A_BYTES;
            for (int s = 0; s < nseq; ++s) {
                const int stage = s % NSTG, ts = s & 1;
                tc::mbar_wait(&full[stage], (s / NSTG) & 1);
                if (s >= 2) tc::mbar_wait(&tempty[ts], ((s >> 1) - 1) & 1);
                tc::tc_fence_after();
                const uint32_t bh = tc::smem_u32(sm + g.off_b + stage * 2 * B_BYTES);
                const uint32_t bl = bh + B_BYTES;
                const uint32_t d = tmem + (uint32_t)(ts * 3 * NB);
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const uint32_t o = ks * 256;
                    tc::mma_i8(d, tc::smem_desc(ah + o, 128, 512), tc::smem_desc(bh + o, 128, 512),
                               idesc, ks);
                }
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const uint32_t o = ks * 256;
                    tc::mma_i8(d + NB, tc::smem_desc(ah + o, 128, 512),
                               tc::smem_desc(bl + o, 128, 512), idesc, ks);
                }
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const uint32_t o = ks * 256;
                    tc::mma_i8(d + NB, tc::smem_desc(al + o, 128, 512),
                               tc::smem_desc(bh + o, 128, 512), idesc, 1);
                }
#pragma unroll
                for (int ks = 0; ks < 2; ++ks) {
                    const uint32_t o = ks * 256;
                    tc::mma_i8(d + 2 * NB, tc::smem_desc(al + o, 128, 512),
                               tc::smem_desc(bl + o, 128, 512), idesc, ks);
                }
                tc::mma_commit(&empty[stage]);
                tc::mma_commit(&tfull[ts]);
                TC_TR(16 + s, clock64());
            }
        }
        __syncwarp();
    } else {
        // ---- epilogue (warps 0-3) and selector (warps 4-7) of lane quarter w
        const bool is_sel = warp >= SEL_WARP0;
        const int w = is_sel ? warp - SEL_WARP0 : warp;
        const int a = 4 * w + (lane >> 3), bb = lane & 7;
        const bool refok = (ky0 + a < kr1) && (kx0 + bb < p.Rx_reg) && (p.K > 1);
        const int ty = r + S * a, tx = r + S * bb;  // reference position in tile coordinates
        const bool warp_active = __any_sync(0xffffffffu, refok);
        const int wt0 = S * 4 * w, wt1 = S * (4 * w + 3) + 2 * r;  // rows any lane can use
        const uint32_t side = (uint32_t)p.side;
        const int cb = p.cb;
        uint32_t* const stg0 = reinterpret_cast<uint32_t*>(sm + g.off_stg) +
                               (w * NSLOT * 32 + lane) * STG_PITCH;  // + slot * 32 * STG_PITCH
        int used = 0;  // staged rows so far (the two warps of the pair count identically)
        if (!is_sel) {
            const uint32_t Nr = nc[ty * NB + tx];
            const int c0 = max(S * bb, j_lo), c1 = min(S * bb + 2 * r, j_hi);
            const uint64_t cm = (c1 >= c0) ? ((c1 >= 63 ? ~0ull : ((2ull << c1) - 1ull)) &
                                              ~((1ull << c0) - 1ull))
                                           : 0ull;
            const uint32_t cm_lo = (uint32_t)cm, cm_hi = (uint32_t)(cm >> 32);
            const uint32_t taddr = tmem + ((uint32_t)(32 * w) << 16);
            int off = 0;
            for (int s = 0; s < nseq; ++s, off = tc_next(off, nseq, step)) {
                const int ts = s & 1;
                const int t = t_lo + off;
                tc::mbar_wait(&tfull[ts], (s >> 1) & 1);
                if (lane == 0) TC_TR(1000 + w * 200 + s, clock64());
                if (!(warp_active && t >= wt0 && t <= wt1)) {
                    __syncwarp();
                    if (lane == 0) tc::mbar_arrive(&tempty[ts]);
                    continue;
                }
                const int slot = used % NSLOT;
                if (used >= NSLOT) tc::mbar_wait(&sempty[w * NSLOT + slot], ((used / NSLOT) - 1) & 1);
                uint32_t* const stg = stg0 + slot * 32 * STG_PITCH;
                const uint32_t gate = gate_pub[w * 32 + lane];  // selector's latest gate
                tc::tc_fence_after();
                const uint32_t cl = Nr - gate;  // e = d - gate = N_c - 2 G + (N_r - gate)
                uint32_t msk[2] = {0u, 0u};
                const uint32_t tb = taddr + (uint32_t)(ts * 3 * NB);
#pragma unroll
                for (int ch = 0; ch < 4; ++ch) {
                    uint32_t hh[16], md[16], ll[16];
                    tc::tmem_ld16(tb + ch * 16, hh);
                    tc::tmem_ld16(tb + NB + ch * 16, md);
                    tc::tmem_ld16(tb + 2 * NB + ch * 16, ll);
                    tc::tmem_wait_ld(hh);
                    tc::tmem_wait_ld(md);
                    tc::tmem_wait_ld(ll);
                    const uint4* ncv = reinterpret_cast<const uint4*>(nc + t * NB + ch * 16);
                    uint32_t e[16];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint4 n4 = ncv[q];
                        const uint32_t nn[4] = {n4.x, n4.y, n4.z, n4.w};
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int j = 4 * q + u;
                            const uint32_t G = ll[j] + 256u * md[j] + 65536u * hh[j];
                            e[j] = nn[u] + cl - 2u * G;
                        }
                    }
                    uint32_t m = 0;
#pragma unroll
                    for (int j = 0; j < 16; ++j) m |= (e[j] >> 31) << j;
                    msk[ch >> 1] |= m << ((ch & 1) * 16);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        *reinterpret_cast<uint4*>(stg + ch * 16 + 4 * q) =
                            make_uint4(e[4 * q], e[4 * q + 1], e[4 * q + 2], e[4 * q + 3]);
                }
                tc::tc_fence_before();
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&tempty[ts]);

                const bool rowin = refok && t >= S * a && t <= S * a + 2 * r;
                uint32_t mlo = rowin ? (msk[0] & cm_lo) : 0u;
                uint32_t mhi = rowin ? (msk[1] & cm_hi) : 0u;
                if (t == ty) {  // the reference itself is slot 0, never a match
                    if (tx < 32) mlo &= ~(1u << tx);
                    else mhi &= ~(1u << (tx - 32));
                }
                *reinterpret_cast<uint4*>(stg + 64) = make_uint4(mlo, mhi, gate, (uint32_t)t);
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(&sfull[w * NSLOT + slot]);
                if (lane == 0) TC_TR(2000 + w * 200 + s, clock64());
                ++used;
            }
        } else {
            uint32_t L[KL];
#pragma unroll
            for (int i = 0; i < KL; ++i) L[i] = KEY_INF;
            // number of rows the epilogue warp stages (same relevance test, same order)
            int nrel = 0;
            if (warp_active) {
                const int lo = max(wt0, t_lo), hi = min(wt1, t_hi);
                nrel = hi >= lo ? hi - lo + 1 : 0;
            }
            while (used < nrel) {
                // take every staged row that is ready (at least one): fewer, fuller rounds
                tc::mbar_wait(&sfull[w * NSLOT + used % NSLOT], (used / NSLOT) & 1);
                int nb = 1;
#ifndef GBM3D_TC_BATCH
#define GBM3D_TC_BATCH 1
#endif
                if (GBM3D_TC_BATCH && lane == 0) {
                    while (nb < NSLOT && used + nb < nrel &&
                           tc::mbar_test(&sfull[w * NSLOT + (used + nb) % NSLOT],
                                         ((used + nb) / NSLOT) & 1))
                        ++nb;
                }
                nb = __shfl_sync(0xffffffffu, nb, 0);
                uint32_t mlo[NSLOT], mhi[NSLOT], g0[NSLOT], crow[NSLOT];
                int cnt = 0;
#pragma unroll
                for (int b2 = 0; b2 < NSLOT; ++b2) {
                    mlo[b2] = mhi[b2] = 0u;
                    g0[b2] = crow[b2] = 0u;
                    if (b2 < nb) {
                        const uint4 hdr = *reinterpret_cast<const uint4*>(
                            stg0 + ((used + b2) % NSLOT) * 32 * STG_PITCH + 64);
                        mlo[b2] = hdr.x;
                        mhi[b2] = hdr.y;
                        g0[b2] = hdr.z;
                        crow[b2] = (uint32_t)((int)hdr.w - S * a) * side - (uint32_t)(S * bb);
                        cnt += __popc(hdr.x) + __popc(hdr.y);
                    }
                }
                const int R = (int)__reduce_max_sync(0xffffffffu, (unsigned)cnt);
                for (int q = 0; q < R; ++q) {
                    uint32_t key = KEY_INF;
                    // first staged row with a pending candidate
                    int bsel = -1;
#pragma unroll
                    for (int b2 = NSLOT - 1; b2 >= 0; --b2)
                        if (mlo[b2] | mhi[b2]) bsel = b2;
                    if (bsel >= 0) {
                        uint32_t ml = 0, mh = 0, gg = 0, cr = 0;
#pragma unroll
                        for (int b2 = 0; b2 < NSLOT; ++b2)
                            if (b2 == bsel) {
                                ml = mlo[b2];
                                mh = mhi[b2];
                                gg = g0[b2];
                                cr = crow[b2];
                            }
                        int j;
                        if (ml) {
                            j = __ffs(ml) - 1;
                            ml &= ml - 1u;
                        } else {
                            j = 31 + __ffs(mh);
                            mh &= mh - 1u;
                        }
#pragma unroll
                        for (int b2 = 0; b2 < NSLOT; ++b2)
                            if (b2 == bsel) {
                                mlo[b2] = ml;
                                mhi[b2] = mh;
                            }
                        const uint32_t d = stg0[((used + bsel) % NSLOT) * 32 * STG_PITCH + j] + gg;
                        key = (d << cb) | (cr + (uint32_t)j);
                    }
                    list_insert<KL>(L, key);
                }
                __syncwarp();
                if (lane == 0)
                    for (int b2 = 0; b2 < nb; ++b2)
                        tc::mbar_arrive(&sempty[w * NSLOT + (used + b2) % NSLOT]);
                if (lane == 0) TC_TR(3000 + w * 200 + used, clock64());
                if (lane == 0) TC_TR(4000 + w * 200 + used, nb * 1000 + R);
                const uint32_t top = L[KL - 1];
                const int gd = (top == KEY_INF) ? p.tdr0 : min((int)(top >> cb), p.tdr0);
                gate_pub[w * 32 + lane] = (uint32_t)(gd + 1);
                used += nb;
            }

            // ---- output: slot 0 = self, ranks 1.. = list, pads (self, -1); coalesced rows
            uint32_t* const stg = stg0;  // every staged row has been consumed: reuse slot 0
            const int Kout = p.K;
            const int ry = S * (ky0 + a), rx = S * (kx0 + bb);
            const int self = ry * p.W + rx;
            const uint32_t cmask = (1u << cb) - 1u;
            int cnt = 0;
            __syncwarp();
            stg[0] = (uint32_t)self;
            stg[Kout] = 0u;
#pragma unroll
            for (int i = 0; i < KL; ++i) {
                if (i + 1 < Kout) {
                    const uint32_t key = L[i];
                    int32_t vi = self, vd = -1;
                    if (key != KEY_INF) {
                        const uint32_t code = key & cmask;
                        const int dy = (int)(code / side) - r, dx = (int)(code % side) - r;
                        vi = (ry + dy) * p.W + rx + dx;
                        vd = (int32_t)(key >> cb);
                        ++cnt;
                    }
                    stg[1 + i] = (uint32_t)vi;
                    stg[Kout + 1 + i] = (uint32_t)vd;
                }
            }
            __syncwarp();
            const int64_t ref0 = (int64_t)bimg * p.out_bstride;
            for (int l = 0; l < 32; ++l) {
                const int la = 4 * w + (l >> 3), lb = l & 7;
                if (ky0 + la >= kr1 || kx0 + lb >= p.Rx_reg) continue;
                const int64_t ref = ref0 + (int64_t)(ky0 + la - p.row_begin) * p.Rx + (kx0 + lb);
                const uint32_t* src = reinterpret_cast<uint32_t*>(sm + g.off_stg) +
                                      (w * NSLOT * 32 + l) * STG_PITCH;
                for (int s2 = lane; s2 < Kout; s2 += 32) {
                    p.idx[ref * Kout + s2] = (int32_t)src[s2];
                    p.dist[ref * Kout + s2] = (int32_t)src[Kout + s2];
                }
            }
            __syncwarp();  // the warp's row stores above precede a fallback rewrite of the same rows
            // exact fallback (tau beyond the 32-bit key range and a short list): own reference
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
    if (warp == MMA_WARP) {
        tc::tc_fence_after();
        tc::tmem_dealloc<tcm::TMEM_COLS>(tmem);
    }
}

// Host launcher over the regular grid part of the call.
// only_marked = 0: one CTA per tile.  only_marked = 1: a small persistent grid walks all tiles
// and recomputes the ones the fp16 kernel marked (usually none: a few microseconds).
template <int S, int KL>
__global__ void __launch_bounds__(tcm::THREADS, 1) match_tc_kernel(MatchParams p, int only_marked) {
    if (!only_marked) {
        tc_tile<S, KL>(p, (int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z);
        return;
    }
    // every thread checks one tile's flag (tiles interleaved over the CTAs), the marked ones
    // are collected in shared memory and recomputed by the whole CTA: one flag-load latency
    // per pass instead of one per tile
    __shared__ int nmk;
    __shared__ int mk[tcm::THREADS];
    const int kr1 = min(p.row_end, p.Ry_reg);
    const int nx = (p.Rx_reg + tcm::TX - 1) / tcm::TX, ny = (kr1 - p.row_begin + tcm::TY - 1) / tcm::TY;
    const int total = nx * ny * p.B;
    const int stride = (int)gridDim.x * (int)blockDim.x;
    for (int t0 = (int)blockIdx.x; t0 < total; t0 += stride) {
        if (threadIdx.x == 0) nmk = 0;
        __syncthreads();
        const int t = t0 + (int)threadIdx.x * (int)gridDim.x;
        if (t < total) {
            const int bx = t % nx, by = (t / nx) % ny, bz = t / (nx * ny);
            const int64_t ref = (int64_t)bz * p.out_bstride + (int64_t)(by * tcm::TY) * p.Rx + bx * tcm::TX;
            if (p.dist[ref * p.K] == TC_TILE_MARK) mk[atomicAdd(&nmk, 1)] = t;
        }
        __syncthreads();
        const int n = nmk;
        for (int i = 0; i < n; ++i) {
            const int tt = mk[i];
            tc_tile<S, KL>(p, tt % nx, (tt / nx) % ny, tt / (nx * ny));
        }
        __syncthreads();
    }
}

template <int S, int KL>
cudaError_t launch_tc(const MatchParams& p, cudaStream_t stream, int* launches, int only_marked) {
    const int kr0 = p.row_begin, kr1 = p.row_end < p.Ry_reg ? p.row_end : p.Ry_reg;
    if (kr1 <= kr0 || p.Rx_reg <= 0) return cudaSuccess;
    const TcGeom g = TcGeom::make(S, p.r);
    auto kern = match_tc_kernel<S, KL>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, g.total);
    if (e != cudaSuccess) return e;
    dim3 grid((p.Rx_reg + tcm::TX - 1) / tcm::TX, (kr1 - kr0 + tcm::TY - 1) / tcm::TY, p.B);
    if (only_marked) {
        static int n_sm = 0;
        if (n_sm == 0) {
            int dev = 0;
            if (cudaGetDevice(&dev) != cudaSuccess ||
                cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
                n_sm = 148;
        }
        const long long tiles = (long long)grid.x * grid.y * grid.z;
        grid = dim3((unsigned)(tiles < n_sm ? tiles : n_sm), 1, 1);
    }
    kern<<<grid, tcm::THREADS, g.total, stream>>>(p, only_marked);
    if (launches) ++*launches;
    return cudaGetLastError();
}

}  // namespace gbm3d
