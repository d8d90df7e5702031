// Stage-1 global volume hard thresholding of G-BM3D, float32.
//
// PAPER.md:132-206.  The matched blocks of the tiling references are stacked into one volume V
// with the image's spatial size (slice 0 = the image); the whole volume is
// transformed by a 3D wavelet transform -- 2D biorthogonal 1.5 in space, Haar along the group,
// 3 levels -- hard thresholded with lambda_l = sigma (3.6 - 0.3 l)
// (PAPER.md:173-178, :241), inverted, and averaged over the cycle spins h = 0, 1 (circular
// shifts of the volume by h along every axis).  The filtered groups are then
// aggregated with weights 1 / TV (3D total variation), the pad blocks left
// out.  Readings S1-S7 in DESIGN.md.
//
// Layout: coefficient volumes are float [B][K][H][W] (slice-major); the 2D transform uses the
// in-place Mallat layout (level l's LL band in the top-left H/2^l x W/2^l corner).  Per cycle
// spin: one fused analysis launch per level (level 1 reads V straight from the image through
// the match table, with the spin's circular shift; V is never stored), one pass along z (Haar
// cascade + threshold + inverse cascade in registers, thread per pixel), one fused synthesis
// launch per level (coarsest first; level 1 stores, then adds, 1/H x the unshifted result into
// U).  Then one launch for the TV weights and the aggregation (fp32 reductions) and the N x N
// box-sum divide.  The passes stream the volume (HBM) or are issue-bound.
#include <cmath>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/gbm3d.h"

namespace gbm3d {
namespace {

// bior1.5 (CDF(1,5)): analysis lowpass h~ = (3, -3, -22, 22, 128, 128, 22, -22, -3, 3) sqrt2/256 on
// n = -4..5, synthesis lowpass = Haar; highpasses by the biorthogonal QMF relations
// g~[n] = (-1)^n h[1-n], g[n] = (-1)^n h~[1-n].  The passes use them in sum / difference form
// (ana_step, syn_step) with the constants as instruction immediates.
constexpr float kR2 = 0.70710678118654752f;

// The z pass: 128-thread x tiles over (rows, images) grids.
constexpr int TPB = 128;

// ---- fused 2D passes: one level of analysis (x then y) or synthesis (y then x) per launch ----
// A CTA owns a 32 x 32 tile of every subband of one slice.  Analysis stages the 73 x 73 inputs of
// its outputs (rows and columns 2 i - 4 .. 2 i + 5, periodic in the band) in shared memory, runs
// the x pass into two shared 73 x 32 planes (a | d) and the y pass from those straight to the
// four subbands: one read and one write of the band per level instead of two of each.  Synthesis
// mirrors it: the 68 x 68 coefficients its 64 x 64 outputs need (a[j] and d[j-2 .. j+2] along
// both axes), y pass into a shared 64 x 68 plane, x pass into a staged 64 x 64 output tile
// written (or, at level 1, accumulated unshifted into U) row by row.
constexpr int FT = 32;                 // coefficient tile (per subband)
constexpr int FIN = 2 * FT + 9;        // 73 analysis inputs per axis
constexpr int FTHREADS = 256;
#ifndef GBM3D_S1_ANA_MINB
#define GBM3D_S1_ANA_MINB 5  // 48 registers: 5 CTAs per SM (the shared-memory limit)
#endif
#ifndef GBM3D_S1_ANA_MINB_G
#define GBM3D_S1_ANA_MINB_G 4  // the level-1 gather instance: 63 registers, no spills
#endif
constexpr int SYN_IN = FT + FT + 4;    // 68: a[j0 .. j0+31] then d[j0-2 .. j0+33]

__device__ __forceinline__ int mod_pos(int i, int n) {
    const int r = i % n;
    return r < 0 ? r + n : r;
}

// One analysis step on 5 consecutive input pairs P_m = (x_{2m}, x_{2m+1}), m = i-2 .. i+2, in the
// sum / difference form of the bior1.5 filters: with S_m = x_{2m} + x_{2m+1}, D_m = x_{2m+1} -
// x_{2m} the lowpass sum_n h~[n] x_{2i+n} (taps (3, -3, -22, 22, 128, 128, 22, -22, -3, 3) sqrt2/256)
// is sqrt2/256 (128 S_i + 22 (D_{i-1} - D_{i+1}) + 3 (D_{i+2} - D_{i-2})) and the highpass
// (x_{2i} - x_{2i+1}) / sqrt2 = -D_i / sqrt2.
constexpr float kS22 = 22.0f * 0.005524271728019903f, kS3 = 3.0f * 0.005524271728019903f;
__device__ __forceinline__ void ana_step(const float (&D)[5], float S2, float& a, float& d) {
    a = fmaf(kS3, D[4] - D[0], fmaf(kS22, D[1] - D[3], kR2 * S2));
    d = -kR2 * D[2];
}

// One synthesis step: outputs x[2j], x[2j+1] from a[j] and d[j-2 .. j+2] (D[0..4]):
// x[m] = h[m & 1] a[m >> 1] + sum_n g[n] d[(m - n) / 2] with g[n] = (-1)^n h~[1 - n] gives
// x[2j] = a/sqrt2 + P + d_j/sqrt2, x[2j+1] = a/sqrt2 + P - d_j/sqrt2,
// P = sqrt2/256 (3 (d_{j+2} - d_{j-2}) + 22 (d_{j-1} - d_{j+1})).
__device__ __forceinline__ void syn_step(const float (&D)[5], float a, float& e, float& f) {
    const float base = fmaf(kS3, D[4] - D[0], fmaf(kS22, D[1] - D[3], kR2 * a));
    e = fmaf(kR2, D[2], base);
    f = fmaf(-kR2, D[2], base);
}

// src: band [0, h) x [0, w) of slice s at row offset `src_row0` (level 1: the volume V itself,
// read as S_shift V); LL -> ll_dst (row offset ll_row0), the three detail bands -> det (at their
// in-place positions).  Slices are H x W with row pitch W.
// GATHER (level 1): the band is the volume V of matched blocks, read straight from the image:
// V[k][y][x] = Z[cy + y mod N][cx + x mod N] with (cy, cx) = idx of the tile (y / N, x / N) and
// slot k, the cycle spin's circular shift applied to (k, y, x) first; `src`
// is then unused.  Otherwise `src` holds the band (the previous level's LL).
template <bool GATHER>
__global__ void __launch_bounds__(FTHREADS, GATHER ? GBM3D_S1_ANA_MINB_G : GBM3D_S1_ANA_MINB) s1_ana_xy_kernel(const float* __restrict__ src,
        int src_row0, const int16_t* __restrict__ img, const int32_t* __restrict__ idx, int N,
        float* __restrict__ ll_dst, int ll_row0, float* __restrict__ det, int K, int H,
        int W, int h, int w, int shift) {
    __shared__ float in[FIN][FIN];            // odd pitch: row-per-lane reads conflict-free
    __shared__ float xa[FIN][FT + 1], xd[FIN][FT + 1];
    // per input row / column: offset inside the block (GATHER) or in the band, and the local
    // tile-block index; the tile's table entries idx[p][q][k] for its <= NBT x NBT blocks
    constexpr int NBT = (FIN + 3) / 4 + 1;    // blocks per axis for N >= 4
    __shared__ int rtab[FIN], rl[FIN], ctab[FIN], cl[FIN];
    __shared__ int rblk[NBT], cblk[NBT];
    __shared__ int ttab[NBT][NBT];
    const int hh = h >> 1, wh = w >> 1;
    const int i0 = blockIdx.y * FT, j0 = blockIdx.x * FT, s = blockIdx.z;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t plane = (int64_t)H * W;
    const int k = s % K, b = s / K;
    const int ks = GATHER ? mod_pos(k - shift, K) : k;
    const float* const slice = src + (int64_t)s * plane + (int64_t)src_row0 * W;
    const int16_t* const zimg = img + (int64_t)b * plane;
    const bool table = GATHER && N >= 4;
    if (tid < FIN) {
        const int y = mod_pos(mod_pos(2 * i0 - 4 + tid, h) - shift, GATHER ? H : h);
        if (GATHER) {
            const int pb = y / N;
            rtab[tid] = (y - pb * N) * W;                                  // row within the block
            // H is a multiple of N, so the block changes every N rows, across the wrap too
            const int y0 = mod_pos(2 * i0 - 4 - shift, H);
            const int lr = (tid + y0 % N) / N;
            rl[tid] = lr;
            const int blk = ((b * (H / N) + pb) * (W / N)) * K + ks;      // table row of the tile
            if (table) {
                if (tid == 0 || (y - pb * N) == 0) rblk[lr] = blk;
            } else {
                rl[tid] = blk;                                             // N < 4: direct lookups
            }
        } else {
            rtab[tid] = y * W;
        }
    } else if (tid >= 128 && tid < 128 + FIN) {
        const int c = tid - 128;
        const int x = mod_pos(mod_pos(2 * j0 - 4 + c, w) - shift, GATHER ? W : w);
        if (GATHER) {
            const int qb = x / N;
            ctab[c] = x - qb * N;
            const int x0 = mod_pos(2 * j0 - 4 - shift, W);
            const int lc = (c + x0 % N) / N;
            cl[c] = lc;
            if (table) {
                if (c == 0 || (x - qb * N) == 0) cblk[lc] = qb * K;
            } else {
                cl[c] = qb * K;
            }
        } else {
            ctab[c] = x;
        }
    }
    __syncthreads();
    if (table) {
        const int nb = (FIN - 1 + N - 1) / N + 1;   // local blocks per axis
        for (int e = tid; e < nb * nb; e += FTHREADS) {
            const int r = e / nb, c = e - r * nb;
            ttab[r][c] = __ldg(idx + rblk[r] + cblk[c]);
        }
        __syncthreads();
    }
    {
        // rows warp, warp + 8, ..; lanes on columns lane + 32 m: every load of the thread in
        // flight before its first shared store
        constexpr int RPW = (FIN + 7) / 8;
        int cofs[3], cq[3];
#pragma unroll
        for (int m = 0; m < 3; ++m) {
            const int c = min(lane + 32 * m, FIN - 1);
            cofs[m] = ctab[c];
            cq[m] = GATHER ? cl[c] : 0;
        }
        float v[RPW][3];
        if (GATHER) {
            int cpos[RPW][3];
            if (table) {
                const int* const tflat = &ttab[0][0];
#pragma unroll
                for (int q = 0; q < RPW; ++q) {
                    const int ro = rl[min(warp + 8 * q, FIN - 1)] * NBT;
#pragma unroll
                    for (int m = 0; m < 3; ++m) cpos[q][m] = tflat[ro + cq[m]];
                }
            } else {
#pragma unroll
                for (int q = 0; q < RPW; ++q) {
                    const int ro = rl[min(warp + 8 * q, FIN - 1)];
#pragma unroll
                    for (int m = 0; m < 3; ++m) cpos[q][m] = __ldg(idx + ro + cq[m]);
                }
            }
            // last column of a lane: lane + 64 < 73 only for lanes 0..8; rows: warp + 8 q < 73
            const bool m2ok = lane + 64 < FIN;
#pragma unroll
            for (int q = 0; q < RPW; ++q) {
                const int r = warp + 8 * q;
                if (q < RPW - 1 || r < FIN) {
                    const int16_t* const rp = zimg + rtab[r];
                    v[q][0] = (float)__ldg(rp + (cpos[q][0] + cofs[0]));
                    v[q][1] = (float)__ldg(rp + (cpos[q][1] + cofs[1]));
                    if (m2ok) v[q][2] = (float)__ldg(rp + (cpos[q][2] + cofs[2]));
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < RPW; ++q) {
                const int r = warp + 8 * q;
                if (r < FIN) {
                    const float* rp = slice + rtab[r];
#pragma unroll
                    for (int m = 0; m < 3; ++m)
                        if (lane + 32 * m < FIN) v[q][m] = __ldg(rp + cofs[m]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
            const int r = warp + 8 * q;
            if (r < FIN) {
#pragma unroll
                for (int m = 0; m < 3; ++m)
                    if (lane + 32 * m < FIN) in[r][lane + 32 * m] = v[q][m];
            }
        }
    }
    __syncthreads();
    // x pass: item = (row r, segment of 11 | 11 | 10 outputs), a sliding window of 5 pairs
    if (tid < 3 * FIN) {
        const int seg = tid / FIN, r = tid - seg * FIN;
        const int jb = seg * 11;
        float D[5], S2, S3;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const float x0 = in[r][2 * (jb + m)], x1 = in[r][2 * (jb + m) + 1];
            D[m] = x1 - x0;
            if (m == 2) S2 = x0 + x1;
            if (m == 3) S3 = x0 + x1;
        }
#pragma unroll
        for (int jj = 0; jj < 11; ++jj) {
            const int j = jb + jj;
            if (j >= FT) break;
            const float x0 = in[r][2 * j + 8], x1 = in[r][2 * j + 9];
            D[4] = x1 - x0;
            const float S4 = x0 + x1;
            float a, d;
            ana_step(D, S2, a, d);
            xa[r][j] = a;
            xd[r][j] = d;
#pragma unroll
            for (int t = 0; t < 4; ++t) D[t] = D[t + 1];
            S2 = S3;
            S3 = S4;
        }
    }
    __syncthreads();
    // y pass: item = (column c of [a | d], segment of 8 outputs); a warp = 32 consecutive columns
    {
        const int c = tid & 63, seg = tid >> 6;
        const int j = c & 31;
        const bool dcol = c >= 32;
        const float(*xs)[FT + 1] = dcol ? xd : xa;
        const int ib = seg * 8;
        float D[5], S2, S3;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
            const float x0 = xs[2 * (ib + m)][j], x1 = xs[2 * (ib + m) + 1][j];
            D[m] = x1 - x0;
            if (m == 2) S2 = x0 + x1;
            if (m == 3) S3 = x0 + x1;
        }
        const int xo = dcol ? wh + j0 + j : j0 + j;
        const bool colok = j0 + j < wh;
        // output pointers of this item's first row, advanced by one image row per output
        float* lo = (dcol ? det + (int64_t)s * plane : ll_dst + (int64_t)s * plane + (int64_t)ll_row0 * W) +
                    (int64_t)(i0 + ib) * W + xo;
        float* hi = det + (int64_t)s * plane + (int64_t)(hh + i0 + ib) * W + xo;
        const int nrow = colok ? min(8, hh - i0 - ib) : 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int i = ib + u;
            const float x0 = xs[2 * i + 8][j], x1 = xs[2 * i + 9][j];
            D[4] = x1 - x0;
            const float S4 = x0 + x1;
            float a, d;
            ana_step(D, S2, a, d);
            if (u < nrow) {
                *lo = a;
                *hi = d;
            }
            lo += W;
            hi += W;
#pragma unroll
            for (int t = 0; t < 4; ++t) D[t] = D[t + 1];
            S2 = S3;
            S3 = S4;
        }
    }
}

// synthesis of one level: LL (ll_src at row offset ll_row0) and the detail bands (det) of the
// band [0, h) x [0, w) -> the band's reconstruction: written to dst at row offset dst_row0, or
// (accumulate) added as scale x S_-shift into U.
__global__ void __launch_bounds__(FTHREADS) s1_syn_xy_kernel(const float* __restrict__ ll_src,
        int ll_row0, const float* __restrict__ det, float* __restrict__ dst, int dst_row0, int K,
        int H, int W, int h, int w, int shift, float scale, int accumulate) {
    __shared__ float cf[SYN_IN][SYN_IN + 1];       // [y: a rows | d rows][x: a cols | d cols]
    __shared__ float ty[2 * FT][SYN_IN + 1];       // after the y pass: 64 rows x [a | d] cols
    __shared__ int rtab[SYN_IN], ctab[SYN_IN];
    const int hh = h >> 1, wh = w >> 1;
    const int i0 = blockIdx.y * FT, j0 = blockIdx.x * FT, s = blockIdx.z;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t plane = (int64_t)H * W;
    // coefficient rows/columns: a at i0 + t (t < 32; beyond the band: unused), d at hh + (i0 - 2
    // + t - 32 mod hh)
    if (tid < SYN_IN)
        rtab[tid] = tid < FT ? min(i0 + tid, hh - 1) : hh + mod_pos(i0 - 2 + tid - FT, hh);
    else if (tid < 2 * SYN_IN) {
        const int t = tid - SYN_IN;
        ctab[t] = t < FT ? min(j0 + t, wh - 1) : wh + mod_pos(j0 - 2 + t - FT, wh);
    }
    __syncthreads();
    const float* const llp = ll_src + (int64_t)s * plane + (int64_t)ll_row0 * W;
    const float* const dp = det + (int64_t)s * plane;
    {
        // rows warp, warp + 8, ..; lanes on columns lane + 32 m: loads first, then stores
        constexpr int RPW = (SYN_IN + 7) / 8;
        int cofs[3];
#pragma unroll
        for (int m = 0; m < 3; ++m) cofs[m] = ctab[min(lane + 32 * m, SYN_IN - 1)];
        float v[RPW][3];
        // column lane (< 32: the LL block for the first 32 rows), lane + 32, lane + 64 (< 68)
        const bool m2ok = lane + 64 < SYN_IN;
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
            const int r = warp + 8 * q;
            if (q < RPW - 1 || r < SYN_IN) {
                const int64_t ro = (int64_t)rtab[r] * W;
                const float* const rd = dp + ro;
                v[q][0] = __ldg((r < FT ? llp + ro : rd) + cofs[0]);
                v[q][1] = __ldg(rd + cofs[1]);
                if (m2ok) v[q][2] = __ldg(rd + cofs[2]);
            }
        }
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
            const int r = warp + 8 * q;
            if (r < SYN_IN) {
#pragma unroll
                for (int m = 0; m < 3; ++m)
                    if (lane + 32 * m < SYN_IN) cf[r][lane + 32 * m] = v[q][m];
            }
        }
    }
    __syncthreads();
    // y pass: item = (column c, segment of 11 | 11 | 10 output pairs); x[2j] = r2 a[j] +
    // sum_u g[4 - 2u] d[j - 2 + u], x[2j+1] = r2 a[j] + sum_u g[5 - 2u] d[j - 2 + u]
    if (tid < 3 * SYN_IN) {
        const int seg = tid / SYN_IN, c = tid - seg * SYN_IN;
        const int jb = seg * 11;
        float dw[5];
#pragma unroll
        for (int t = 0; t < 4; ++t) dw[t] = cf[FT + jb + t][c];
#pragma unroll
        for (int jj = 0; jj < 11; ++jj) {
            const int j = jb + jj;
            if (j >= FT) break;
            dw[4] = cf[FT + j + 4][c];
            const float aj = cf[j][c];
            float e, f;
            syn_step(dw, aj, e, f);
            ty[2 * j][c] = e;
            ty[2 * j + 1][c] = f;
#pragma unroll
            for (int t = 0; t < 4; ++t) dw[t] = dw[t + 1];
        }
    }
    __syncthreads();
    // x pass: item = (row m, segment of 8 output pairs); the 64 x 64 result overwrites cf
    float(*const out)[SYN_IN + 1] = cf;
    {
        const int m = tid & 63, seg = tid >> 6;
        const int jb = seg * 8;
        float dw[5];
#pragma unroll
        for (int t = 0; t < 4; ++t) dw[t] = ty[m][FT + jb + t];
#pragma unroll
        for (int u8 = 0; u8 < 8; ++u8) {
            const int j = jb + u8;
            dw[4] = ty[m][FT + j + 4];
            const float aj = ty[m][j];
            float e, f;
            syn_step(dw, aj, e, f);
            out[m][2 * j] = e;
            out[m][2 * j + 1] = f;
#pragma unroll
            for (int t = 0; t < 4; ++t) dw[t] = dw[t + 1];
        }
    }
    __syncthreads();
    const int y0 = 2 * i0, x0 = 2 * j0;
    const int c = tid & 63, x = x0 + c;
    if (x >= w) return;
    constexpr int RPT = 2 * FT / (FTHREADS / 64);   // 16 rows per thread
    if (accumulate == 0) {
        float* o = dst + (int64_t)s * plane + (int64_t)(dst_row0 + y0 + (tid >> 6)) * W + x;
        const int64_t rowstep = (int64_t)(FTHREADS / 64) * W;
#pragma unroll
        for (int q = 0; q < RPT; ++q, o += rowstep) {
            const int r = (tid >> 6) + q * (FTHREADS / 64);
            if (y0 + r < h) *o = out[r][c];
        }
    } else {
        // (S_-h R)[k][y][x] = R[k + h][y + h][x + h]: this element lands at (k-h, y-h, x-h)
        // (level 1: the band is the whole slice, h = H, w = W, 0 <= shift < H, W, K).  The first
        // spin stores (accumulate = 1: U needs no clearing), later ones add (accumulate = 2),
        // every load of the thread in flight before its first store.
        const int k = s % K, b = s / K;
        const int kk = k >= shift ? k - shift : k - shift + K;
        const int xs = x >= shift ? x - shift : x - shift + W;
        float* const o = dst + (int64_t)(b * K + kk) * plane + xs;
        // row y = yb + 4 q lands at y - shift: one pointer step of 4 rows per q, except that
        // y < shift (only q = 0 can have it: yb < shift <= 1) wraps to y - shift + H
        const int yb = y0 + (tid >> 6);
        const int64_t rowstep = (int64_t)(FTHREADS / 64) * W;
        float* const pq0 = o + (int64_t)(yb >= shift ? yb - shift : yb - shift + H) * W;
        float* const pq1 = o + (int64_t)(yb + FTHREADS / 64 - shift) * W;  // q >= 1, no wrap
        auto orow = [&](int q) { return q == 0 ? pq0 : pq1 + (q - 1) * rowstep; };
        float old[RPT];
#pragma unroll
        for (int q = 0; q < RPT; ++q)
            old[q] = (accumulate == 2 && yb + q * (FTHREADS / 64) < h) ? *orow(q) : 0.f;
#pragma unroll
        for (int q = 0; q < RPT; ++q) {
            const int r = (tid >> 6) + q * (FTHREADS / 64);
            if (y0 + r < h) *orow(q) = fmaf(scale, out[r][c], old[q]);
        }
    }
}

// along z at every (b, y, x): Haar cascade (lz levels), hard threshold, inverse cascade
template <int K>
__global__ void __launch_bounds__(TPB) s1_z_kernel(float* __restrict__ C, int H, int W, int L, int lz,
                                                   const float* __restrict__ sigmas,
                                                   uint8_t* __restrict__ keep_out) {
    const int x = blockIdx.x * TPB + threadIdx.x, y = blockIdx.y, b = blockIdx.z;
    if (x >= W) return;
    const int64_t plane = (int64_t)H * W;
    // spatial level of (y, x) in the Mallat layout (reading S2): the level-l detail bands, the
    // final LL band counting as level L
    int lev = L;
    for (int l = 1; l <= L; ++l) {
        if (y >= (H >> l) || x >= (W >> l)) { lev = l; break; }
    }
    const bool ll = y < (H >> L) && x < (W >> L);
    const float lam = sigmas[b] * (3.6f - 0.3f * (float)lev);
    float v[K];
    float* base = C + (int64_t)b * K * plane + (int64_t)y * W + x;
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = base[(int64_t)k * plane];
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        const int s = 1 << t;
        if (t >= lz) break;
#pragma unroll
        for (int i = 0; i < K; i += 2 * s) {
            const float a = v[i], d = v[i + s];
            v[i] = (a + d) * kR2;
            v[i + s] = (a - d) * kR2;
        }
    }
    const int zstep = 1 << lz;
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const bool keep = fabsf(v[k]) >= lam || (ll && (k % zstep) == 0);
        v[k] = keep ? v[k] : 0.f;
        // test hook (gbm3d_stage1_denoise_keep): Upsilon's decision per coefficient
        if (keep_out) keep_out[((int64_t)b * K + k) * plane + (int64_t)y * W + x] = keep ? 1 : 0;
    }
#pragma unroll
    for (int t = 4; t >= 0; --t) {
        if (t >= lz) continue;
        const int s = 1 << t;
#pragma unroll
        for (int i = 0; i < K; i += 2 * s) {
            const float a = v[i], d = v[i + s];
            v[i] = (a + d) * kR2;
            v[i + s] = (a - d) * kR2;
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) base[(int64_t)k * plane] = v[k];
}

// TV weight and aggregation of one group per CTA (K N threads): the group's K x N x N values are
// staged in shared memory in (k, i, j) order (16-byte loads, consecutive threads on consecutive
// elements: conflict-free), TV = sum of |forward differences| along x, y and z (reading S4) with
// every thread on elements e, e + nt, ..; w = 1 / TV (1 when TV = 0) by a block reduction; then
// the first n_valid blocks add w U_pq[k] at their positions (fp32 reductions, consecutive
// threads on consecutive pixels of a block row) and their weight once at their top-left pixel
// of the weight map.
__device__ __forceinline__ void s1_split(int e, int N, int NN, bool p2, int lg, int& k, int& i, int& j) {
    if (p2) {
        k = e >> (2 * lg);
        const int r = e & (NN - 1);
        i = r >> lg;
        j = r & (N - 1);
    } else {
        k = e / NN;
        const int r = e - k * NN;
        i = r / N;
        j = r - i * N;
    }
}

// NC, KC: compile-time N and K (0 = the runtime values), so the common shapes get constant
// index arithmetic and fully unrolled loops
template <int NC, int KC>
__global__ void __launch_bounds__(512) s1_tv_aggregate_kernel(const float* __restrict__ U,
        const int32_t* __restrict__ idx, const int32_t* __restrict__ nvalid, int K_rt, int H, int W,
        int N_rt, float* __restrict__ num, float* __restrict__ wmap) {
    extern __shared__ float gsm[];              // [K][N][N], 32 partial sums, K positions
    const int N = NC > 0 ? NC : N_rt, K = KC > 0 ? KC : K_rt;
    const int Bx = W / N, By = H / N;
    const int t = threadIdx.x, nt = (NC > 0 && KC > 0) ? NC * KC : (int)blockDim.x;
    const int g = blockIdx.x, b = blockIdx.y;
    const int p = g / Bx, q = g - p * Bx;
    const int64_t gi = (int64_t)b * By * Bx + g;
    const int64_t plane = (int64_t)H * W;
    const int NN = N * N, KNN = K * NN;
    const bool p2 = (N & (N - 1)) == 0;
    const int lg = __ffs(N) - 1;
    const float* const gbase = U + (int64_t)b * K * plane + (int64_t)(p * N) * W + q * N;
    int* const pos = reinterpret_cast<int*>(gsm + KNN + 32);     // K block positions
    if (t < K) pos[t] = __ldg(idx + gi * K + t);
    if ((N & 3) == 0) {
        for (int e4 = t; e4 < KNN / 4; e4 += nt) {
            int k, i, j;
            s1_split(4 * e4, N, NN, p2, lg, k, i, j);
            const float4 v = __ldg(reinterpret_cast<const float4*>(gbase + (int64_t)k * plane + (int64_t)i * W + j));
            *reinterpret_cast<float4*>(gsm + 4 * e4) = v;
        }
    } else {
        for (int e = t; e < KNN; e += nt) {
            int k, i, j;
            s1_split(e, N, NN, p2, lg, k, i, j);
            gsm[e] = __ldg(gbase + (int64_t)k * plane + (int64_t)i * W + j);
        }
    }
    __syncthreads();
    float tv = 0.f;
    for (int e = t; e < KNN; e += nt) {
        int k, i, j;
        s1_split(e, N, NN, p2, lg, k, i, j);
        const float u = gsm[e];
        if (j + 1 < N) tv += fabsf(gsm[e + 1] - u);
        if (i + 1 < N) tv += fabsf(gsm[e + N] - u);
        if (k + 1 < K) tv += fabsf(gsm[e + NN] - u);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tv += __shfl_xor_sync(0xffffffffu, tv, o);
    float* const part = gsm + KNN;
    if ((t & 31) == 0) part[t >> 5] = tv;
    __syncthreads();
    float tot = 0.f;
    for (int wi = 0; wi < (nt + 31) / 32; ++wi) tot += part[wi];
    const float w = tot > 0.f ? 1.f / tot : 1.f;
    const int nv = __ldg(nvalid + gi);
    float* const nb = num + b * plane;
    for (int e = t; e < nv * NN; e += nt) {
        int kb, ii, jj;
        s1_split(e, N, NN, p2, lg, kb, ii, jj);
        const int c = pos[kb];                              // cy W + cx
        atomicAdd(nb + (int64_t)c + (int64_t)ii * W + jj, w * gsm[e]);
        if (ii == 0 && jj == 0) atomicAdd(wmap + b * plane + c, w);
    }
}

// out = num / (N x N box sums of the weight map over [y-N+1, y] x [x-N+1, x]): 32 x 32 output
// tiles, the map staged with its (N-1)-pixel halo, separable sums
template <int NC>  // compile-time N (0 = runtime)
__global__ void __launch_bounds__(256) s1_divide_kernel(const float* __restrict__ num,
        const float* __restrict__ wmap, float* __restrict__ out, int H, int W, int N_rt) {
    const int N = NC > 0 ? NC : N_rt;
    __shared__ float m[47][48];
    __shared__ float hs[47][33];
    const int b = blockIdx.z, y0 = blockIdx.y * 32, x0 = blockIdx.x * 32;
    const int E = 32 + N - 1;
    const int64_t plane = (int64_t)H * W;
    const float* wm = wmap + b * plane;
    for (int i = threadIdx.x; i < E * E; i += 256) {
        const int r = i / E, c = i - r * E;
        const int y = y0 - (N - 1) + r, x = x0 - (N - 1) + c;
        m[r][c] = (y >= 0 && y < H && x >= 0 && x < W) ? wm[(int64_t)y * W + x] : 0.f;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < E * 32; i += 256) {
        const int r = i >> 5, c = i & 31;
        float h = 0.f;
        for (int j = 0; j < N; ++j) h += m[r][c + j];
        hs[r][c] = h;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 32 * 32; i += 256) {
        const int r = i >> 5, c = i & 31;
        const int y = y0 + r, x = x0 + c;
        if (y >= H || x >= W) continue;
        float d = 0.f;
        for (int t = 0; t < N; ++t) d += hs[r + t][c];
        const int64_t o = b * plane + (int64_t)y * W + x;
        out[o] = d > 0.f ? num[o] / d : 0.f;
    }
}

unsigned grid1(int64_t n) {
    const int64_t b = (n + 255) / 256;
    return (unsigned)(b < 148 * 32 ? (b > 0 ? b : 1) : 148 * 32);
}

}  // namespace
}  // namespace gbm3d

using namespace gbm3d;

extern "C" size_t gbm3d_stage1_workspace_bytes(int B, int H, int W, int patch, int K) {
    if (B < 1 || H < 1 || W < 1 || patch < 1 || K < 1) return 0;
    const size_t vol = (size_t)B * K * H * W;
    return (3 * vol + 2 * (size_t)B * H * W) * sizeof(float);
}

static int stage1_run(const int16_t* noisy, int B, int H, int W, int patch, const int32_t* idx,
                      const int32_t* n_valid, int K, const float* sigmas, int levels, float* out,
                      void* workspace, size_t workspace_bytes, void* stream, uint8_t* keep) {
    if (!noisy || !idx || !n_valid || !sigmas || !out || !workspace) return GBM3D_ERR_ARG;
    if (B < 1 || patch < 1 || K < 1 || levels < 1 || H < patch || W < patch) return GBM3D_ERR_ARG;
    if (H % patch || W % patch || H % (2 << levels) || W % (2 << levels)) return GBM3D_ERR_ARG;
    if ((long long)H * W >= (1LL << 31)) return GBM3D_ERR_ARG;
    if (workspace_bytes < gbm3d_stage1_workspace_bytes(B, H, W, patch, K)) return GBM3D_ERR_ARG;
    if ((K & (K - 1)) != 0 || K > 32 || patch > 16 || levels > 5) return GBM3D_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t vol = (int64_t)B * K * H * W, plane = (int64_t)B * H * W;
    float* const C = (float*)workspace;   // coefficients
    float* const Tm = C + vol;            // separable-pass scratch
    float* const U = Tm + vol;            // filtered volume (mean of the spins)
    float* const num = U + vol;
    float* const wmap = num + plane;
    int lz = 0;  // Haar levels along z: min(L, log2 K) (reading S1)
    while ((1 << (lz + 1)) <= K && lz < levels) ++lz;
    const int BK = B * K;
    // U is stored by the first spin's last synthesis pass; the aggregation planes are cleared
    if (cudaMemsetAsync(num, 0, (size_t)(2 * plane) * sizeof(float), s) != cudaSuccess)
        return GBM3D_ERR_CUDA;
    const unsigned gx = (unsigned)((W + TPB - 1) / TPB);
    const int spins = 2;
    for (int sh = 0; sh < spins; ++sh) {
        // analysis: LL_l goes to the scratch volume at alternating row offsets (odd levels at
        // row 0, even ones at row H/2: never the rows the same launch reads), the last level's
        // to C's corner; the details to C at their in-place positions
        for (int l = 1; l <= levels; ++l) {
            const int h = H >> (l - 1), w = W >> (l - 1);
            const dim3 fg((unsigned)((w / 2 + FT - 1) / FT), (unsigned)((h / 2 + FT - 1) / FT), BK);
            float* lld = l == levels ? C : Tm;
            const int ll_row0 = l == levels ? 0 : (l & 1 ? 0 : H / 2);
            if (l == 1)
                s1_ana_xy_kernel<true><<<fg, FTHREADS, 0, s>>>(nullptr, 0, noisy, idx, patch, lld, ll_row0,
                                                               C, K, H, W, h, w, sh);
            else
                s1_ana_xy_kernel<false><<<fg, FTHREADS, 0, s>>>(Tm, (l - 1) & 1 ? 0 : H / 2, nullptr, nullptr,
                                                                patch, lld, ll_row0, C, K, H, W, h, w, 0);
        }
        const dim3 zg(gx, H, B);
        uint8_t* const kp = keep ? keep + sh * vol : nullptr;
        switch (K) {
            case 1: s1_z_kernel<1><<<zg, TPB, 0, s>>>(C, H, W, levels, lz, sigmas, kp); break;
            case 2: s1_z_kernel<2><<<zg, TPB, 0, s>>>(C, H, W, levels, lz, sigmas, kp); break;
            case 4: s1_z_kernel<4><<<zg, TPB, 0, s>>>(C, H, W, levels, lz, sigmas, kp); break;
            case 8: s1_z_kernel<8><<<zg, TPB, 0, s>>>(C, H, W, levels, lz, sigmas, kp); break;
            case 16: s1_z_kernel<16><<<zg, TPB, 0, s>>>(C, H, W, levels, lz, sigmas, kp); break;
            default: s1_z_kernel<32><<<zg, TPB, 0, s>>>(C, H, W, levels, lz, sigmas, kp); break;
        }
        // synthesis: LL_l from C's corner (l = L) or the scratch offset of level l, LL_(l-1) to
        // the scratch offset of level l - 1, level 1 accumulated unshifted into U
        for (int l = levels; l >= 1; --l) {
            const int h = H >> (l - 1), w = W >> (l - 1);
            const dim3 fg((unsigned)((w / 2 + FT - 1) / FT), (unsigned)((h / 2 + FT - 1) / FT), BK);
            const float* lls = l == levels ? C : Tm;
            const int ll_row0 = l == levels ? 0 : (l & 1 ? 0 : H / 2);
            float* dst = l == 1 ? U : Tm;
            const int dst_row0 = l == 1 ? 0 : ((l - 1) & 1 ? 0 : H / 2);
            s1_syn_xy_kernel<<<fg, FTHREADS, 0, s>>>(lls, ll_row0, C, dst, dst_row0, K, H, W, h, w, sh,
                                                     1.0f / spins, l == 1 ? (sh == 0 ? 1 : 2) : 0);
        }
    }
    {
        // whole warps: the TV reduction shuffles over full warps (extra threads idle)
        const int nt = (K * patch + 31) & ~31;
        const size_t smem = ((size_t)K * patch * patch + 32 + K) * sizeof(float);
        const dim3 grid((unsigned)((H / patch) * (W / patch)), B);
        if (patch == 8 && K == 16)
            s1_tv_aggregate_kernel<8, 16><<<grid, nt, smem, s>>>(U, idx, n_valid, K, H, W, patch, num, wmap);
        else if (patch == 8 && K == 32)
            s1_tv_aggregate_kernel<8, 32><<<grid, nt, smem, s>>>(U, idx, n_valid, K, H, W, patch, num, wmap);
        else
            s1_tv_aggregate_kernel<0, 0><<<grid, nt, smem, s>>>(U, idx, n_valid, K, H, W, patch, num, wmap);
    }
    {
        const dim3 dg((unsigned)((W + 31) / 32), (unsigned)((H + 31) / 32), B);
        if (patch == 8)
            s1_divide_kernel<8><<<dg, 256, 0, s>>>(num, wmap, out, H, W, patch);
        else
            s1_divide_kernel<0><<<dg, 256, 0, s>>>(num, wmap, out, H, W, patch);
    }
    return cudaGetLastError() == cudaSuccess ? GBM3D_OK : GBM3D_ERR_CUDA;
}

extern "C" int gbm3d_stage1_denoise(const int16_t* noisy, int B, int H, int W, int patch,
                                    const int32_t* idx, const int32_t* n_valid, int K,
                                    const float* sigmas, int levels, float* out, void* workspace,
                                    size_t workspace_bytes, void* stream) {
    return stage1_run(noisy, B, H, W, patch, idx, n_valid, K, sigmas, levels, out, workspace,
                      workspace_bytes, stream, nullptr);
}

extern "C" int gbm3d_stage1_denoise_keep(const int16_t* noisy, int B, int H, int W, int patch,
                                         const int32_t* idx, const int32_t* n_valid, int K,
                                         const float* sigmas, int levels, float* out,
                                         void* workspace, size_t workspace_bytes,
                                         uint8_t* keep, void* stream) {
    if (!keep) return GBM3D_ERR_ARG;
    return stage1_run(noisy, B, H, W, patch, idx, n_valid, K, sigmas, levels, out, workspace,
                      workspace_bytes, stream, keep);
}
