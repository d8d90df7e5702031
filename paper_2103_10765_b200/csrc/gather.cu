// Matched-block gather: the 3D groups of S^K_pq and the paper's volume V.
//
// the matched blocks of the tiling reference Z^N_pq are S^K_pq, and
//     V[p N + i, q N + j, z_x] = Z_x[i, j],   x = the z-th element of S^K_pq, 0 <= i, j < N,
// "the aggregated 3D volume of matched blocks" (Fig. 2).  PAPER.md:217: both stages stack the
// matched blocks of every reference into 5D tensors N x N x K x B x B, so that the 3D transforms
// run on all groups in one call.  Here:
//   * gbm3d_gather_groups  -> groups[b][ref][k][i][j] = Z_b[cy + i][cx + j], (cy, cx) = idx[b][ref][k]
//     (any reference grid; the layout of the matcher's tables with a P x P block per slot), and
//   * gbm3d_gather_volume  -> vol[b][k][p N + i][q N + j] (tiling references, stride = N, N | H, W):
//     slice k of V, an image, so slice 0 is Z itself (slot 0 is the reference, reading R4).
// Pad slots carry the reference's own index ("padded with the reference block"),
// so they repeat the reference block, as the paper prescribes.  An index outside the image
// (not produced by the matcher) yields a zero block rather than an out-of-bounds read.
//
// Both are pure data movement, HBM-write bound: a 4-byte index read and P^2 2-byte pixels
// (L2 hits: the image is read once from HBM) per output block.  One thread writes one 8-pixel
// row segment (16 bytes) of a block: 32 lanes write 512 contiguous bytes.
#include <climits>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/gbm3d.h"

namespace gbm3d {
namespace {

// 8 consecutive int16 starting at element e of the (4-byte aligned) image buffer as one 16-byte
// chunk, from the 32-bit aligned words that cover them (read-only path: the image is L2/L1
// resident).  For odd e the fifth word's upper half is one element past the chunk; it lies in
// the same aligned word as the chunk's last element, so it never leaves the allocation.
__device__ __forceinline__ uint4 load8(const int16_t* __restrict__ base, int64_t e) {
    const uint32_t* w = reinterpret_cast<const uint32_t*>(base + (e & ~(int64_t)1));
    const uint32_t a0 = __ldg(w), a1 = __ldg(w + 1), a2 = __ldg(w + 2), a3 = __ldg(w + 3);
    if ((e & 1) == 0) return make_uint4(a0, a1, a2, a3);
    const uint32_t a4 = __ldg(w + 4);
    return make_uint4(__funnelshift_r(a0, a1, 16), __funnelshift_r(a1, a2, 16),
                      __funnelshift_r(a2, a3, 16), __funnelshift_r(a3, a4, 16));
}

// groups, P = 8, tiled: CTA = a chunk of CH consecutive references of one grid row (CH x K
// <= 1024 slots).  The bounding box of all the chunk's candidate blocks (a strip of the search
// windows, e.g. 139 x 46 pixels for c3) is staged in shared memory with coalesced row loads,
// every slot's position is decoded once, then every 16-byte block row is assembled from shared
// memory: HBM reads the image about once and the kernel is bound by the block writes.  The
// staging buffer is small (20 KB: about 7 CTAs per SM); a chunk whose box does not fit is
// redone in halves, down to single references whose blocks come from global memory (indices
// not from a local search).
#ifndef GBM3D_GATHER_SLOTS
#define GBM3D_GATHER_SLOTS 1024
#endif
constexpr int SLOTS = GBM3D_GATHER_SLOTS;  // slots (references x K) per CTA
#ifndef GBM3D_BOX_WORDS
#define GBM3D_BOX_WORDS 5120
#endif
constexpr int BOX_WORDS = GBM3D_BOX_WORDS;  // staging words (2 pixels each)
constexpr int GATHER_SMEM = (BOX_WORDS + SLOTS) * 4;
__global__ void __launch_bounds__(256) gather_groups8_tiled_kernel(
        const int16_t* __restrict__ imgs, int H, int W, const int32_t* __restrict__ idx,
        int Ry, int Rx, int K, int CH, uint4* __restrict__ out) {
    extern __shared__ uint32_t gsm[];
    uint32_t* const box = gsm;
    uint32_t* const pos = gsm + BOX_WORDS;  // per slot: cy << 16 | cx, or ~0 when invalid
    __shared__ int bb[4];
    const int chunks_per_row = (Rx + CH - 1) / CH;
    const int ry = blockIdx.x / chunks_per_row, c0 = (blockIdx.x - ry * chunks_per_row) * CH;
    const int b = blockIdx.y;
    const int nref = min(CH, Rx - c0);
    const int64_t ref0 = ((int64_t)b * Ry + ry) * Rx + c0;
    const int32_t* __restrict__ tab = idx + ref0 * K;
    const int nslot = nref * K;
    const unsigned uW = (unsigned)W;
    // decode every slot once
    for (int q = threadIdx.x; q < nslot; q += blockDim.x) {
        const int c = __ldg(tab + q);
        const unsigned cy = (unsigned)c / uW, cx = (unsigned)c - cy * uW;
        const bool ok = c >= 0 && (int)cy <= H - 8 && (int)cx <= W - 8;
        pos[q] = ok ? (cy << 16 | cx) : ~0u;
    }
    __syncthreads();
    const int16_t* __restrict__ img = imgs + (int64_t)b * H * W;
    uint4* const o = out + ref0 * K * 8;
    // references [s0, s0 + sub) at a time: the whole chunk when its candidates' bounding box
    // fits the staging buffer (the usual case), else halves of it, down to one reference
    // whose blocks are then read straight from global memory
    int sub = nref;
    for (int s0 = 0; s0 < nref;) {
        const int s1 = min(nref, s0 + sub);
        int y0 = INT_MAX, y1 = -1, x0 = INT_MAX, x1 = -1;
        for (int q = s0 * K + (int)threadIdx.x; q < s1 * K; q += blockDim.x) {
            const uint32_t pq = pos[q];
            if (pq != ~0u) {
                const int cy = (int)(pq >> 16), cx = (int)(pq & 0xffffu);
                y0 = min(y0, cy); y1 = max(y1, cy);
                x0 = min(x0, cx); x1 = max(x1, cx);
            }
        }
        if (threadIdx.x == 0) { bb[0] = INT_MAX; bb[1] = -1; bb[2] = INT_MAX; bb[3] = -1; }
        __syncthreads();
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            y0 = min(y0, __shfl_xor_sync(0xffffffffu, y0, off));
            y1 = max(y1, __shfl_xor_sync(0xffffffffu, y1, off));
            x0 = min(x0, __shfl_xor_sync(0xffffffffu, x0, off));
            x1 = max(x1, __shfl_xor_sync(0xffffffffu, x1, off));
        }
        if ((threadIdx.x & 31) == 0) {
            atomicMin(&bb[0], y0); atomicMax(&bb[1], y1); atomicMin(&bb[2], x0); atomicMax(&bb[3], x1);
        }
        __syncthreads();
        const int by0 = bb[0], bx0 = bb[2] & ~1;  // even column: 4-byte aligned staging words
        const int rows = bb[1] - by0 + 8, cols = bb[3] + 8 - bx0;
        const int pitch = ((cols + 9) & ~1) / 2;  // words per staged row (>= cols / 2 + 1)
        const bool staged = bb[1] >= 0 && rows * pitch <= BOX_WORDS;
        if (!staged && bb[1] >= 0 && sub > 1) {  // retry these references in smaller groups
            sub = (sub + 1) >> 1;
            __syncthreads();
            continue;
        }
        if (staged) {
            // rows of the box as 32-bit words, coalesced per row: aligned word loads when W is
            // even (bx0 is even, so every staged word starts on a 4-byte boundary)
            if ((W & 1) == 0) {
                const uint32_t* img32 = reinterpret_cast<const uint32_t*>(img);
                const int W2 = W >> 1;
                for (int u = threadIdx.x; u < rows * pitch; u += blockDim.x) {
                    const int r = u / pitch, cw = u - r * pitch;
                    const int gw = (bx0 >> 1) + cw;
                    box[u] = gw < W2 ? __ldg(img32 + (int64_t)(by0 + r) * W2 + gw) : 0u;
                }
            } else {
                for (int u = threadIdx.x; u < rows * pitch; u += blockDim.x) {
                    const int r = u / pitch, cw = u - r * pitch;
                    const int gx = bx0 + 2 * cw;
                    const int16_t* src = img + (int64_t)(by0 + r) * W;
                    const uint32_t lo = gx < W ? (uint16_t)__ldg(src + gx) : 0u;
                    const uint32_t hi = gx + 1 < W ? (uint16_t)__ldg(src + gx + 1) : 0u;
                    box[u] = lo | (hi << 16);
                }
            }
        }
        __syncthreads();
        // one item = one 8-pixel block row: (slot q, row i); 32 lanes write 512 B
        for (int it = s0 * K * 8 + (int)threadIdx.x; it < s1 * K * 8; it += blockDim.x) {
            const int q = it >> 3, i = it & 7;
            const uint32_t pq = pos[q];
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (pq != ~0u) {
                const int cy = (int)(pq >> 16), cx = (int)(pq & 0xffffu);
                if (staged) {
                    const int e = cx - bx0;
                    const uint32_t* w = box + (cy - by0 + i) * pitch + (e >> 1);
                    const uint32_t a0 = w[0], a1 = w[1], a2 = w[2], a3 = w[3];
                    if ((e & 1) == 0) {
                        v = make_uint4(a0, a1, a2, a3);
                    } else {
                        const uint32_t a4 = w[4];
                        v = make_uint4(__funnelshift_r(a0, a1, 16), __funnelshift_r(a1, a2, 16),
                                       __funnelshift_r(a2, a3, 16), __funnelshift_r(a3, a4, 16));
                    }
                } else {
                    v = load8(imgs, ((int64_t)b * H + cy + i) * (int64_t)W + cx);
                }
            }
            o[it] = v;
        }
        __syncthreads();  // the box is restaged by the next group
        s0 = s1;
    }
}

// groups, any P <= 16: item = one pixel (simple and still coalesced on the output).
__global__ void gather_groups_any_kernel(const int16_t* __restrict__ imgs, int H, int W, int P,
                                         const int32_t* __restrict__ idx, int64_t n_blocks,
                                         int64_t blocks_per_img, int16_t* __restrict__ out) {
    const int64_t PP = (int64_t)P * P, n = n_blocks * PP;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t blk = e / PP;
        const int rem = (int)(e - blk * PP), i = rem / P, j = rem - i * P;
        const int64_t b = blk / blocks_per_img;
        const int c = __ldg(idx + blk);
        const int cy = c / W, cx = c - cy * W;
        int16_t v = 0;
        if (c >= 0 && cy <= H - P && cx <= W - P) v = __ldg(imgs + (b * H + cy + i) * (int64_t)W + cx + j);
        out[e] = v;
    }
}

// volume, P = 8: item = (b, k, image row y, tile column q) -> 8 pixels of vol[b][k][y][8q ..].
__global__ void gather_volume8_kernel(const int16_t* __restrict__ imgs, int B, int H, int W,
                                      const int32_t* __restrict__ idx, int K,
                                      uint4* __restrict__ vol) {
    const int Bx = W >> 3, By = H >> 3;
    const int64_t n_items = (int64_t)B * K * H * Bx;
    for (int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; it < n_items;
         it += (int64_t)gridDim.x * blockDim.x) {
        const int q = (int)(it % Bx);
        const int64_t r1 = it / Bx;
        const int y = (int)(r1 % H);
        const int64_t r2 = r1 / H;
        const int k = (int)(r2 % K);
        const int64_t b = r2 / K;
        const int p = y >> 3, i = y & 7;
        const int c = __ldg(idx + ((b * By + p) * Bx + q) * K + k);
        const int cy = c / W, cx = c - cy * W;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (c >= 0 && cy <= H - 8 && cx <= W - 8)
            v = load8(imgs, (b * H + cy + i) * (int64_t)W + cx);
        vol[it] = v;
    }
}

// volume, any P: item = one pixel of vol[b][k][y][x].
__global__ void gather_volume_any_kernel(const int16_t* __restrict__ imgs, int B, int H, int W,
                                         int P, const int32_t* __restrict__ idx, int K,
                                         int16_t* __restrict__ vol) {
    const int Bx = W / P, By = H / P;
    const int64_t n = (int64_t)B * K * H * W;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(e % W);
        const int64_t r1 = e / W;
        const int y = (int)(r1 % H);
        const int64_t r2 = r1 / H;
        const int k = (int)(r2 % K);
        const int64_t b = r2 / K;
        const int p = y / P, q = x / P, i = y - p * P, j = x - q * P;
        const int c = __ldg(idx + ((b * By + p) * Bx + q) * K + k);
        const int cy = c / W, cx = c - cy * W;
        int16_t v = 0;
        if (c >= 0 && cy <= H - P && cx <= W - P) v = __ldg(imgs + (b * H + cy + i) * (int64_t)W + cx + j);
        vol[e] = v;
    }
}

int grid_for(int64_t items) {
    // a multiple of the SM count (148) x 8 resident 256-thread CTAs, or fewer for small jobs
    const int64_t want = (items + 255) / 256;
    const int64_t cap = 148 * 8 * 4;
    return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

}  // namespace
}  // namespace gbm3d

using namespace gbm3d;

extern "C" int gbm3d_gather_groups(const int16_t* imgs, int B, int H, int W, int patch,
                                   const int32_t* idx, int Ry, int Rx, int K, int16_t* groups,
                                   void* stream) {
    if (!imgs || !idx || !groups) return GBM3D_ERR_ARG;
    if (B < 1 || H < 1 || W < 1 || patch < 1 || Ry < 0 || Rx < 0 || K < 1) return GBM3D_ERR_ARG;
    if (H < patch || W < patch || (long long)H * W >= (1LL << 31)) return GBM3D_ERR_ARG;
    if ((long long)Ry * Rx * K * 8 >= (1LL << 31)) return GBM3D_ERR_ARG;  // per image
    if (patch > 16) return GBM3D_ERR_UNSUPPORTED;
    if (Ry == 0 || Rx == 0) return GBM3D_OK;
    cudaStream_t s = (cudaStream_t)stream;
    if (patch == 8 && K <= SLOTS && W < 65536 && H < 65536) {  // (cy << 16 | cx) slot packing
        // references per CTA: at most SLOTS / K (and 128), balanced over the row's chunks
        const int chmax = SLOTS / K < 128 ? SLOTS / K : 128;
        const int nchunk = (Rx + chmax - 1) / chmax;
        const int ch = (Rx + nchunk - 1) / nchunk;
        // per call: the attribute is per device, and the call may come from any thread
        if (cudaFuncSetAttribute(gather_groups8_tiled_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 GATHER_SMEM) != cudaSuccess)
            return GBM3D_ERR_CUDA;
        dim3 grid((unsigned)(Ry * ((Rx + ch - 1) / ch)), (unsigned)B);
        gather_groups8_tiled_kernel<<<grid, 256, GATHER_SMEM, s>>>(
            imgs, H, W, idx, Ry, Rx, K, ch, reinterpret_cast<uint4*>(groups));
    } else {
        const int64_t per_img = (int64_t)Ry * Rx * K, n_blocks = per_img * B;
        gather_groups_any_kernel<<<grid_for(n_blocks * patch * patch), 256, 0, s>>>(
            imgs, H, W, patch, idx, n_blocks, per_img, groups);
    }
    return cudaGetLastError() == cudaSuccess ? GBM3D_OK : GBM3D_ERR_CUDA;
}

extern "C" int gbm3d_gather_volume(const int16_t* imgs, int B, int H, int W, int patch,
                                   const int32_t* idx, int K, int16_t* vol, void* stream) {
    if (!imgs || !idx || !vol) return GBM3D_ERR_ARG;
    if (B < 1 || H < 1 || W < 1 || patch < 1 || K < 1) return GBM3D_ERR_ARG;
    if (H < patch || W < patch || (long long)H * W >= (1LL << 31)) return GBM3D_ERR_ARG;
    if (H % patch || W % patch) return GBM3D_ERR_ARG;  // M / N = B integral
    if (patch > 16) return GBM3D_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    if (patch == 8) {
        gather_volume8_kernel<<<grid_for((int64_t)B * K * H * (W / 8)), 256, 0, s>>>(
            imgs, B, H, W, idx, K, reinterpret_cast<uint4*>(vol));
    } else {
        gather_volume_any_kernel<<<grid_for((int64_t)B * K * H * W), 256, 0, s>>>(
            imgs, B, H, W, patch, idx, K, vol);
    }
    return cudaGetLastError() == cudaSuccess ? GBM3D_OK : GBM3D_ERR_CUDA;
}
