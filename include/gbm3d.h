/*
 * gbm3d.h -- C ABI of the B200 (sm_100a) block-matching library for G-BM3D
 * (Sanders & Larkin, arXiv 2103.10765).  Library: paper_2103_10765_b200/libgbm3d.so.
 *
 * What every entry computes (PAPER.md = /root/reference/PAPER.md, line numbers):
 *   For each reference patch rho = (ry, rx) on the grid R_y x R_x with
 *     R = {0, s, 2s, ... <= L-P} U {L-P}                 (tiles at (pN,qN), PAPER.md:154-156;
 *                                                         DESIGN.md reading R3)
 *   and each candidate c in the clamped window |c - rho|_inf <= radius, c != rho
 *                                                        (local search; R2)
 *     d(rho, c) = ||Z_rho - Z_c||_2^2 = sum_{i,j<P} (Z[ry+i][rx+j] - Z[cy+i][cx+j])^2
 *                                                        (Eq. (1))
 *   keep the K-1 smallest keys (d, idx(c)) with d < tau (strict, Eq. (1); R5, R6), after
 *   the reference itself in slot 0 with d = 0:  this is S^K_pq on the
 *   local window, "exactly 15 matches" for K = 16 (R4).  Missing slots are
 *   "padded with the reference block": idx = idx(rho), dist = -1 (R7).
 *   idx(c) = cy * W + cx (raster index of the candidate's top-left pixel).
 *   Two exact formulations compute d (results are bit-identical to the definition above):
 *   - product form (Eq. (2): d = ||f_p||^2 + ||f_q||^2 - 2 <f_p, f_q>), the AUTO
 *     choice for patch 8 / stride 3 / radius <= 21 / K <= 32: the inner products of a tile of
 *     128 references with each candidate row run on the tcgen05 tensor cores (fp16 operands of
 *     tile-centred pixels, fp32 accumulators; every partial sum is an integer below 2^24, so
 *     exact; tiles whose pixel range breaks that bound are redone by an int8 byte-plane
 *     kernel), norms by box sums (step 1); likewise patch 12 / stride 4 /
 *     radius <= 21 / K <= 32 (c2): 12 MMAs of K16 per candidate row, tiles above the fp16
 *     bound and references whose 32-bit-key lists end short (tau - 1 above the key's d
 *     range) take in-kernel exact int32 paths;
 *   - SSD form, organised by displacement delta = c - rho: the shifted-difference image
 *     (Z - S_delta Z)^2 box-summed over P x P (Prop. 1 with an all-ones block,
 *     PAPER.md:89-113), in int32; used for the other instantiated shapes.
 *   Anything else runs the direct per-reference kernel.
 *
 * Layouts (all row-major, contiguous):
 *   image      int16  [H][W]          batched: [B][H][W]
 *   idx, dist  int32  [Ry][Rx][K]     batched: [B][Ry][Rx][K]
 *   n_valid    int32  [Ry][Rx]        batched: [B][Ry][Rx]  (nullable)
 *   references in raster order of the grid; slots hold ranks 0..K-1.
 *
 * Ownership: the caller allocates and owns every buffer.  Device entries take DEVICE
 * pointers and enqueue on `stream` (a cudaStream_t passed as void*; NULL = legacy default
 * stream); they return after enqueueing (results are ready when the stream is).  They
 * allocate no memory and are reentrant: any number of concurrent calls on distinct streams is
 * allowed.  The only library state is a pair of side streams per host thread and device
 * (created on first use): a call whose grid has an appended last row / column runs those
 * references' direct kernel there, forked from and joined back into `stream` with events (so
 * the call stays ordered on `stream` and is capturable in a CUDA graph).  Outputs are
 * undefined after any error.
 *
 * Precondition (exactness domain, reading R10): P^2 * (max(Z) - min(Z))^2 <=
 * 2^31 - 1, so every distance fits int32.  gbm3d_check_range verifies it; the device entries
 * do not (they are the hot path).
 *
 * Supported sizes: 1 <= patch <= 16, 0 <= radius <= 32, 1 <= K <= 64, stride >= 1,
 * H, W >= patch, H*W < 2^31.  Larger patch/radius/K return GBM3D_ERR_UNSUPPORTED.
 */
#ifndef GBM3D_H
#define GBM3D_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* tau value meaning "no threshold" (d < INT64_MAX always holds). */
#define GBM3D_TAU_NONE INT64_MAX

enum {
    GBM3D_OK = 0,
    GBM3D_ERR_ARG = -1,         /* null pointer, bad size/parameter; nothing enqueued     */
    GBM3D_ERR_RANGE = -2,       /* image violates P^2 (max-min)^2 <= 2^31-1               */
    GBM3D_ERR_UNSUPPORTED = -3, /* patch > 16, radius > 32 or K > 64                      */
    GBM3D_ERR_CUDA = -4         /* a CUDA launch/copy error (async faults surface at sync) */
};

/* Matching algorithm selector for gbm3d_block_match_ex. */
enum {
    GBM3D_METHOD_AUTO = 0,     /* fastest exact kernel available for the shape            */
    GBM3D_METHOD_SSD = 1,      /* displacement-organised shifted-difference box sums      */
    GBM3D_METHOD_PRODUCT = 2,  /* Eq. (2) product form on tensor cores (fp16, exact)      */
    GBM3D_METHOD_DIRECT = 3,   /* generic per-reference direct SSD (any shape; slow)      */
    GBM3D_METHOD_PRODUCT_I8 = 4 /* product form, byte-plane int8 tensor-core kernel only   */
};

/* Reference-grid counts along both axes (host, pure, reading R3).
 * Returns GBM3D_ERR_ARG if H < patch, W < patch, patch < 1 or stride < 1. */
int gbm3d_grid_dims(int H, int W, int patch, int stride, int* n_ref_y, int* n_ref_x);

/* One image.  img: device int16 [H][W]; idx/dist: device int32 [Ry][Rx][K];
 * n_valid: device int32 [Ry][Rx] or NULL.  tau: raw SSD threshold (strict), or
 * GBM3D_TAU_NONE; tau < 0 is GBM3D_ERR_ARG. */
int gbm3d_block_match(const int16_t* img, int H, int W, int patch, int stride, int radius,
                      int K, int64_t tau, int32_t* idx, int32_t* dist, int32_t* n_valid,
                      void* stream);

/* B independent images (grid.z = image): imgs [B][H][W] -> [B][Ry][Rx][K]; idx are
 * per-image raster indices.  Byte-identical to B calls of gbm3d_block_match. */
int gbm3d_block_match_batched(const int16_t* imgs, int B, int H, int W, int patch, int stride,
                              int radius, int K, int64_t tau, int32_t* idx, int32_t* dist,
                              int32_t* n_valid, void* stream);

/* Row range of one image for spatial sharding (the paper processes overlapping image
 * patches in parallel).  `slab` holds global image rows
 * [slab_y0, slab_y0 + slab_rows) of an H x W image; the call computes reference grid rows
 * [ref_row_begin, ref_row_end) and writes idx/dist [ref_row_end - ref_row_begin][Rx][K],
 * n_valid [..][Rx], with GLOBAL raster indices.  The slab must contain every row those
 * references read: [max(0, y_first - radius), min(H, y_last + radius + patch)), where
 * y_first/y_last are the pixel rows of the first/last reference row; else GBM3D_ERR_ARG.
 * Concatenating the outputs of row ranges is byte-identical to gbm3d_block_match. */
int gbm3d_block_match_rows(const int16_t* slab, int slab_y0, int slab_rows, int H, int W,
                           int patch, int stride, int radius, int K, int64_t tau,
                           int ref_row_begin, int ref_row_end, int32_t* idx, int32_t* dist,
                           int32_t* n_valid, void* stream);

/* gbm3d_block_match_batched with an explicit method (GBM3D_METHOD_*).  B >= 1. */
int gbm3d_block_match_ex(const int16_t* imgs, int B, int H, int W, int patch, int stride,
                         int radius, int K, int64_t tau, int method, int32_t* idx,
                         int32_t* dist, int32_t* n_valid, void* stream);

/* ---- Matched-block gather (the groups the 3D filtering of both stages
 * consumes).  imgs: device int16 [B][H][W] (4-byte aligned, as cudaMalloc returns); idx:
 * device int32 tables of gbm3d_block_match* for the same (B, H, W, patch).
 *
 * gbm3d_gather_groups: the 5D tensor of PAPER.md:217 ("N x N x K x B x B": matched blocks x
 * reference grid), layout groups[b][ry][rx][k][i][j] = Z_b[cy + i][cx + j] with
 * (cy, cx) = (idx[b][ry][rx][k] / W, idx[b][ry][rx][k] % W), 0 <= i, j < patch, for the
 * table shape [B][Ry][Rx][K].  Pad slots hold the reference's own index, so they repeat the
 * reference block ("padded with the reference block").  Fast path (patch 8):
 * each CTA stages the bounding box of a 64-reference strip's candidates in shared memory.
 *
 * gbm3d_gather_volume: the paper's volume of matched blocks for tiling references
 * (stride = patch = N, N | H and N | W):
 *   vol[b][k][p N + i][q N + j] = Z_b[cy + i][cx + j],  (cy, cx) from idx[b][p Bx + q][k],
 * i.e. V[pN+i, qN+j, z] of PAPER.md:162 stored slice-major ([B][K][H][W]); slice 0 is Z.
 *
 * Both enqueue on `stream`, allocate nothing, and are bit-exact copies (an index outside the
 * image writes a zero block).  Errors: GBM3D_ERR_ARG for null pointers / bad sizes (and, for
 * the volume, H or W not a multiple of patch); GBM3D_ERR_UNSUPPORTED for patch > 16;
 * GBM3D_ERR_CUDA for a launch error. */
int gbm3d_gather_groups(const int16_t* imgs, int B, int H, int W, int patch, const int32_t* idx,
                        int Ry, int Rx, int K, int16_t* groups, void* stream);
int gbm3d_gather_volume(const int16_t* imgs, int B, int H, int W, int patch, const int32_t* idx,
                        int K, int16_t* vol, void* stream);

/* ---- Stage-2 collaborative Wiener filtering + aggregation (PAPER.md:210-217,
 * aggregation Eq. of PAPER.md:190 with the original algorithm's Wiener weights).
 * noisy: device int16 [B][H][W]; basic: device float32 [B][H][W] (the basic estimate the
 * shrinkage is computed from); idx / n_valid: device tables [B][Ry][Rx][K] / [B][Ry][Rx] of
 * gbm3d_block_match* for the same (B, H, W, patch) -- their indices must lie in the image;
 * sigmas: device float32 [B] noise standard deviations; out: device float32 [B][H][W].
 * For every group: T = Haar_K o DCT2_8x8 (orthonormal) of the noisy and of the basic blocks,
 * W = T_B^2 / (T_B^2 + sigma^2) (1 where both vanish), filtered blocks T^-1(W . T_Z), group
 * weight 1 / (sigma^2 ||W||^2) (1 if sigma = 0 or ||W|| = 0); out = weighted average of the
 * filtered blocks over every pixel, using the first n_valid blocks of each group (pad blocks
 * are left out).  fp32 arithmetic with atomic accumulation: results match a
 * float64 evaluation within DESIGN.md's tolerance, not bit for bit.
 * workspace: device buffer of gbm3d_wiener_workspace_bytes(B, H, W) bytes (2 float planes),
 * cleared by the call.  Errors: GBM3D_ERR_ARG (null pointer, sizes, small workspace),
 * GBM3D_ERR_UNSUPPORTED (patch != 8, K not a power of two or > 32), GBM3D_ERR_CUDA. */
size_t gbm3d_wiener_workspace_bytes(int B, int H, int W);
int gbm3d_wiener_stage2(const int16_t* noisy, const float* basic, int B, int H, int W, int patch,
                        const int32_t* idx, const int32_t* n_valid, int Ry, int Rx, int K,
                        const float* sigmas, float* out, void* workspace, size_t workspace_bytes,
                        void* stream);

/* ---- Stage-1 global volume hard thresholding, the
 * operator phi of PAPER.md:200-204 for one noisy image per batch entry.  References tile the
 * image (stride = patch = N; H and W multiples of N and of 2^(levels+1)); idx / n_valid are the
 * tables of gbm3d_block_match* for that grid (K a power of two <= 32).  The volume of matched
 * blocks V (slice 0 = Z) is transformed by a 3D wavelet transform -- 2D bior1.5 over (y, x),
 * periodic, `levels` Mallat levels (the paper uses 3), then Haar along the group with
 * min(levels, log2 K) levels -- hard thresholded with lambda_l = sigma (3.6 - 0.3 l) by spatial
 * level (the coarsest approximation kept), inverted, averaged over the cycle spins h = 0, 1
 * (circular shifts of V by h along all three axes), and aggregated with the group weights
 * 1 / TV(U_pq) (anisotropic 3D total variation), pad blocks left out.
 * noisy: device int16 [B][H][W]; sigmas: device float32 [B]; out: device float32 [B][H][W];
 * workspace: gbm3d_stage1_workspace_bytes(B, H, W, patch, K) bytes (3 float volumes + 2 planes).
 * fp32 with atomic accumulation: matches a float64 evaluation within DESIGN.md's tolerance.
 * The translation trials of PAPER.md:203 (match and filter circularly shifted images, shift
 * back, average) compose gbm3d_shift_trials, one batched gbm3d_block_match + this call over
 * the T x B shifted images, and gbm3d_unshift_mean.
 * Errors: GBM3D_ERR_ARG (null pointers, sizes, small workspace), GBM3D_ERR_UNSUPPORTED (K not a
 * power of two or > 32, patch > 16, levels > 5), GBM3D_ERR_CUDA. */
size_t gbm3d_stage1_workspace_bytes(int B, int H, int W, int patch, int K);
int gbm3d_stage1_denoise(const int16_t* noisy, int B, int H, int W, int patch, const int32_t* idx,
                         const int32_t* n_valid, int K, const float* sigmas, int levels, float* out,
                         void* workspace, size_t workspace_bytes, void* stream);

/* ---- Translation trials of stage 1 (Eq. (10)):
 *   Y_f = (1/T) sum_t S_-h_t( phi(S_h_t Z) ),  S_h = circular shift by h pixels along both
 * image axes (reading S8).  shifts: HOST int array of T trial offsets, each in
 * [0, min(H, W)), 1 <= T <= GBM3D_MAX_TRIALS (the paper uses h = 0, N/4, N/2).
 * gbm3d_shift_trials: imgs device int16 [B][H][W] -> out device int16 [T][B][H][W] with
 *   out[t][b][y][x] = imgs[b][(y - h_t) mod H][(x - h_t) mod W]   (a batch for the matcher);
 * gbm3d_unshift_mean: ys device float32 [T][B][H][W] (phi of each shifted image) -> out device
 *   float32 [B][H][W], out[b][y][x] = (1/T) sum_t ys[t][b][(y + h_t) mod H][(x + h_t) mod W].
 * Both enqueue on `stream` and allocate nothing; exact copies / an fp32 mean of T terms.
 * Errors: GBM3D_ERR_ARG (null pointers, sizes, T or a shift out of range, T*B > 65535),
 * GBM3D_ERR_UNSUPPORTED (H > 65535), GBM3D_ERR_CUDA. */
#define GBM3D_MAX_TRIALS 16
int gbm3d_shift_trials(const int16_t* imgs, int B, int H, int W, const int* shifts, int T,
                       int16_t* out, void* stream);
int gbm3d_unshift_mean(const float* ys, int T, int B, int H, int W, const int* shifts,
                       float* out, void* stream);

/* Test hook of the same operation: additionally writes Upsilon's keep (1) / zero (0) decision for
 * every coefficient of both cycle spins to keep: device uint8 [2][B][K][H][W] in the in-place
 * layout of the transform (spatial Mallat layout, Haar positions along the group), so that a
 * float64 evaluation can take the same decisions for the coefficients that lie within rounding
 * of their threshold.  Same errors as gbm3d_stage1_denoise (GBM3D_ERR_ARG for a null keep). */
int gbm3d_stage1_denoise_keep(const int16_t* noisy, int B, int H, int W, int patch,
                              const int32_t* idx, const int32_t* n_valid, int K,
                              const float* sigmas, int levels, float* out, void* workspace,
                              size_t workspace_bytes, uint8_t* keep, void* stream);

/* Host-buffer entry (end-to-end path): h_imgs is HOST int16 [B][H][W] (pinned for async
 * copies), outputs are HOST int32 arrays with the batched layouts.  d_workspace is a device
 * buffer of at least gbm3d_host_workspace_bytes(...) bytes.  Copies in, matches, copies out,
 * and BLOCKS until the results are on the host.  The work is pipelined in up to 16 chunks
 * (images for B > 1; for B = 1 blocks of reference rows -- a 32-row first chunk, then equal
 * multiples of 16 -- whose pixel rows are copied in as bands): copies run on two
 * library-owned streams (created once per host thread and device) overlapped with the
 * matching on `stream` and a second library stream; n_valid comes back in one copy at the
 * end.
 * Results are identical to the device entries. */
size_t gbm3d_host_workspace_bytes(int B, int H, int W, int patch, int stride, int K);
int gbm3d_block_match_host(const int16_t* h_imgs, int B, int H, int W, int patch, int stride,
                           int radius, int K, int64_t tau, int32_t* h_idx, int32_t* h_dist,
                           int32_t* h_n_valid, void* d_workspace, size_t workspace_bytes,
                           void* stream);

/* Range precondition (reading R10): *ok = 1 iff patch^2 * (max - min)^2 <= 2^31 - 1 over
 * the n device int16 values at img.  BLOCKING (synchronises `stream`).  Returns
 * GBM3D_ERR_ARG for null pointers or n < 1. */
int gbm3d_check_range(const int16_t* img, int64_t n, int patch, int* ok, void* stream);

/* ---- Integer instruction-throughput microkernels (the ALU roofline's peak is
 * measured on the box in the same run).  kind 0 = SHF + LOP3 (ALU pipe only), 1 = IMAD (FMA
 * pipe only), 2 = IMNMX min/max (ALU pipe; the selection's instruction), 3 = IMAD + IADD3 (both
 * pipes: the issue-rate bound).  gbm3d_int_peak_launch enqueues blocks x threads threads
 * (threads a multiple of 32, <= 256), each running 8 independent chains for `iters` x 16 steps
 * of two instructions; sink: device uint32 [blocks] (written only to keep the chains live).
 * gbm3d_int_peak_ops returns the lane-instructions one such launch executes (0 for a bad kind).
 * Errors: GBM3D_ERR_ARG, GBM3D_ERR_CUDA. */
double gbm3d_int_peak_ops(int kind, int blocks, int threads, int iters);
int gbm3d_int_peak_launch(int kind, int blocks, int threads, int iters, uint32_t* sink,
                          void* stream);

/* Number of kernel launches the last successful call on this thread enqueued (for the
 * bench's gpu_launches claim). */
int gbm3d_last_launch_count(void);

/* Static string for a status code. */
const char* gbm3d_strerror(int status);

/* Library version string. */
const char* gbm3d_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GBM3D_H */
