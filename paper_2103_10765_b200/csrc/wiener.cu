// Stage-2 collaborative Wiener filtering of the matched groups and its aggregation
// (SURVEY.md §8f-3).
//
// the second estimate filters every group of matched 8 x 8 blocks with a 3D
// transform made of a 2D DCT over the block and a 1D Haar transform along the group; all groups
// at once (the 5D tensor N x N x K x B x B); "the filtering and aggregation rules in this step
// match the original algorithm precisely" (readings W1-W6):
//   T_Z, T_B = transforms of the group in the noisy image Z and in the basic estimate Ŷ,
//   W = T_B^2 / (T_B^2 + sigma^2)  (1 where both vanish),  U = T^-1(W . T_Z),
//   w = 1 / (sigma^2 ||W||^2)      (1 when sigma = 0 or ||W|| = 0),
//   Y(x) = sum w U(x) / sum w chi(x) over the first n_valid blocks of every group (
//   the pad blocks that fill short groups are left out).
//
// Mapping: one lane per block (K lanes per group, K a power of two <= 32): the block's 64
// coefficients live in the lane's registers, the 2D DCT is two in-register passes of 8 x 8
// products, the Haar transform along the group is a butterfly cascade across the K lanes
// (shfl.xor; orthonormal, coefficients in the butterfly's positions, which the elementwise
// shrinkage does not care about), and the weight's ||W||^2 is a K-lane reduction.  A CTA takes
// an 8 x 8 tile of references; their blocks lie in the union of the tile's search windows, so
// the aggregation sums go to a shared-memory copy of that region (bounding box of the tile's
// blocks) and reach global memory as one atomic add per region pixel.  fp32 arithmetic.
#include <climits>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/gbm3d.h"

namespace gbm3d {
namespace {

constexpr int WT = 8;                   // reference tile: WT x WT grid cells per CTA
constexpr int WTHREADS = 128;
constexpr int REGION_MAX = 6144;        // pixels of the shared aggregation region (3 x 24 KB)

// 8-point orthonormal DCT-II of v[0], v[st], .., v[7 st] in place, by the symmetry of its
// rows: even rows see s_j = x_j + x_{7-j}, odd rows d_j = x_j - x_{7-j} (4 products each
// instead of 8).  The inverse (DCT-III) splits the same way: x_j = E_j + O_j, x_{7-j} = E_j - O_j.
__device__ __forceinline__ void dct8_1d(float* v, int st, const float* __restrict__ C, bool inverse) {
    if (!inverse) {
        float sj[4], dj[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            sj[j] = v[j * st] + v[(7 - j) * st];
            dj[j] = v[j * st] - v[(7 - j) * st];
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float* src = (k & 1) ? dj : sj;
            float acc = 0.f;
#pragma unroll
            for (int j = 0; j < 4; ++j) acc = fmaf(C[k * 8 + j], src[j], acc);
            v[k * st] = acc;
        }
    } else {
        float e[4], o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float ae = 0.f, ao = 0.f;
#pragma unroll
            for (int k = 0; k < 8; k += 2) ae = fmaf(C[k * 8 + j], v[k * st], ae);
#pragma unroll
            for (int k = 1; k < 8; k += 2) ao = fmaf(C[k * 8 + j], v[k * st], ao);
            e[j] = ae;
            o[j] = ao;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v[j * st] = e[j] + o[j];
            v[(7 - j) * st] = e[j] - o[j];
        }
    }
}
// 2D: rows then columns (forward), columns then rows (inverse) of the 8 x 8 block x[i * 8 + j].
__device__ __forceinline__ void dct8x8(float (&x)[64], const float* __restrict__ C, bool inverse) {
    if (!inverse) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dct8_1d(x + 8 * i, 1, C, false);
#pragma unroll
        for (int l = 0; l < 8; ++l) dct8_1d(x + l, 8, C, false);
    } else {
#pragma unroll
        for (int l = 0; l < 8; ++l) dct8_1d(x + l, 8, C, true);
#pragma unroll
        for (int i = 0; i < 8; ++i) dct8_1d(x + 8 * i, 1, C, true);
    }
}

// Orthonormal Haar cascade across the K lanes of a group (lane k = block k): at stride s only
// the lanes holding approximation coefficients (k % s == 0) take part: k % 2s == 0 keeps
// (x_k + x_{k+s}) / sqrt 2, k % 2s == s keeps (x_{k-s} - x_k) / sqrt 2 (a detail coefficient,
// left alone from then on).  Forward runs s = 1, 2, .., K/2; the inverse runs the same butterfly
// (its own inverse) in the reverse order.
template <int K>
__device__ __forceinline__ void haar_lanes(float (&x)[64], int k, bool inverse) {
    const float r2 = 0.70710678118654752f;
#pragma unroll
    for (int t = 0; t < 5; ++t) {
        const int s = inverse ? (K >> 1) >> t : 1 << t;
        if (s < 1 || s >= K) continue;
        const bool act = (k & (s - 1)) == 0, lo = (k & s) == 0;
#pragma unroll
        for (int e = 0; e < 64; ++e) {
            const float p = __shfl_xor_sync(0xffffffffu, x[e], s);
            const float y = lo ? (x[e] + p) * r2 : (p - x[e]) * r2;
            x[e] = act ? y : x[e];
        }
    }
}

template <int K>
__global__ void __launch_bounds__(WTHREADS) wiener_tile_kernel(
        const int16_t* __restrict__ noisy, const float* __restrict__ basic, int H, int W,
        const int32_t* __restrict__ idx, const int32_t* __restrict__ nvalid, int Ry, int Rx,
        const float* __restrict__ sigmas, float* __restrict__ num, float* __restrict__ den) {
    extern __shared__ float wsm[];
    float* const rnum = wsm;                   // [REGION_MAX] numerator sums
    float* const rwm = wsm + REGION_MAX;       // [REGION_MAX] block weights at block top-lefts
    float* const rtmp = wsm + 2 * REGION_MAX;  // [REGION_MAX] horizontal box sums of rwm
    __shared__ float C[64];
    __shared__ int bb[4];
    const int b = blockIdx.z;
    const int ty0 = blockIdx.y * WT, tx0 = blockIdx.x * WT;
    const int ny = min(WT, Ry - ty0), nx = min(WT, Rx - tx0);
    const int64_t plane = (int64_t)H * W;
    const int16_t* __restrict__ zimg = noisy + b * plane;
    const float* __restrict__ bimg = basic + b * plane;
    const float sigma = sigmas[b];
    if (threadIdx.x < 64) {
        const int k = threadIdx.x >> 3, i = threadIdx.x & 7;
        const float a = k == 0 ? 0.35355339059327376f : 0.5f;  // sqrt(1/8), sqrt(2/8)
        C[threadIdx.x] = a * cospif((float)((2 * i + 1) * k) / 16.0f);
    }
    if (threadIdx.x == 0) { bb[0] = INT_MAX; bb[1] = -1; bb[2] = INT_MAX; bb[3] = -1; }
    __syncthreads();
    // bounding box of every block of the tile's groups
    {
        int y0 = INT_MAX, y1 = -1, x0 = INT_MAX, x1 = -1;
        for (int q = threadIdx.x; q < ny * nx * K; q += WTHREADS) {
            const int g = q / K, k = q - g * K;
            const int gy = ty0 + g / nx, gx = tx0 + g % nx;
            const int c = __ldg(idx + (((int64_t)b * Ry + gy) * Rx + gx) * K + k);
            const int cy = c / W, cx = c - cy * W;
            y0 = min(y0, cy); y1 = max(y1, cy); x0 = min(x0, cx); x1 = max(x1, cx);
        }
        atomicMin(&bb[0], y0); atomicMax(&bb[1], y1); atomicMin(&bb[2], x0); atomicMax(&bb[3], x1);
    }
    __syncthreads();
    const int by0 = bb[0], bx0 = bb[2];
    const int rh = bb[1] + 8 - by0, rw = bb[3] + 8 - bx0;
    const bool regional = rh * rw <= REGION_MAX;
    if (regional)
        for (int i = threadIdx.x; i < rh * rw; i += WTHREADS) { rnum[i] = 0.f; rwm[i] = 0.f; }
    __syncthreads();

    constexpr int GPW = 32 / K;  // groups per warp pass
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int k = lane % K, gslot = lane / K;
    const int ngroups = ny * nx;
    for (int g0 = warp * GPW; g0 < ngroups; g0 += (WTHREADS / 32) * GPW) {
        const int g = g0 + gslot;
        const bool live = g < ngroups;  // uniform per K-lane group
        const int gy = ty0 + (live ? g / nx : 0), gx = tx0 + (live ? g % nx : 0);
        const int64_t ref = ((int64_t)b * Ry + gy) * Rx + gx;
        const int c = live ? __ldg(idx + ref * K + k) : 0;
        const int nv = live ? __ldg(nvalid + ref) : 0;
        const int cy = c / W, cx = c - cy * W;
        // basic-estimate group -> T_B -> shrinkage W (kept in tb)
        float tb[64];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) tb[i * 8 + j] = __ldg(bimg + (int64_t)(cy + i) * W + cx + j);
        dct8x8(tb, C, false);
        haar_lanes<K>(tb, k, false);
        const float s2 = sigma * sigma;
        float n2 = 0.f;
#pragma unroll
        for (int e = 0; e < 64; ++e) {
            const float t2 = tb[e] * tb[e];
            const float dn = t2 + s2;
            const float wv = dn > 0.f ? t2 / dn : 1.f;
            tb[e] = wv;
            n2 = fmaf(wv, wv, n2);
        }
#pragma unroll
        for (int o = 1; o < K; o <<= 1) n2 += __shfl_xor_sync(0xffffffffu, n2, o);
        const float wgt = (sigma > 0.f && n2 > 0.f) ? 1.f / (s2 * n2) : 1.f;
        // noisy group -> T_Z, shrink, inverse
        float tz[64];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) tz[i * 8 + j] = (float)__ldg(zimg + (int64_t)(cy + i) * W + cx + j);
        dct8x8(tz, C, false);
        haar_lanes<K>(tz, k, false);
#pragma unroll
        for (int e = 0; e < 64; ++e) tz[e] *= tb[e];
        haar_lanes<K>(tz, k, true);
        dct8x8(tz, C, true);
        // aggregation of the group's real matches (slots < n_valid)
        if (live && k < nv) {
            if (regional) {
                // numerator per pixel; the denominator sum w chi is the 8 x 8 box sum of the
                // block weights placed at the blocks' top-left pixels (one add per block)
                float* const pn = rnum + (cy - by0) * rw + (cx - bx0);
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) atomicAdd(pn + i * rw + j, wgt * tz[i * 8 + j]);
                atomicAdd(rwm + (cy - by0) * rw + (cx - bx0), wgt);
            } else {
                float* const pn = num + b * plane + (int64_t)cy * W + cx;
                float* const pd = den + b * plane + (int64_t)cy * W + cx;
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        atomicAdd(pn + (int64_t)i * W + j, wgt * tz[i * 8 + j]);
                        atomicAdd(pd + (int64_t)i * W + j, wgt);
                    }
            }
        }
    }
    if (regional) {
        __syncthreads();
        for (int i = threadIdx.x; i < rh * rw; i += WTHREADS) {  // horizontal 8-box of rwm
            const int y = i / rw, x = i - y * rw;
            float h = 0.f;
#pragma unroll
            for (int j = 0; j < 8; ++j) h += x - j >= 0 ? rwm[y * rw + x - j] : 0.f;
            rtmp[i] = h;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < rh * rw; i += WTHREADS) {
            const int y = i / rw, x = i - y * rw;
            float d = 0.f;
#pragma unroll
            for (int t = 0; t < 8; ++t) d += y - t >= 0 ? rtmp[(y - t) * rw + x] : 0.f;
            if (d != 0.f) {
                const int y = by0 + i / rw, x = bx0 + i % rw;
                atomicAdd(num + b * plane + (int64_t)y * W + x, rnum[i]);
                atomicAdd(den + b * plane + (int64_t)y * W + x, d);
            }
        }
    }
}

__global__ void wiener_divide_kernel(const float* __restrict__ num, const float* __restrict__ den,
                                     float* __restrict__ out, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float d = den[i];
        out[i] = d > 0.f ? num[i] / d : 0.f;
    }
}

template <int K>
cudaError_t launch_wiener(const int16_t* noisy, const float* basic, int B, int H, int W,
                          const int32_t* idx, const int32_t* nvalid, int Ry, int Rx,
                          const float* sigmas, float* num, float* den, cudaStream_t s) {
    const int smem = 3 * REGION_MAX * 4;
    static bool attr = false;
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(wiener_tile_kernel<K>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    dim3 grid((unsigned)((Rx + WT - 1) / WT), (unsigned)((Ry + WT - 1) / WT), (unsigned)B);
    wiener_tile_kernel<K><<<grid, WTHREADS, smem, s>>>(noisy, basic, H, W, idx, nvalid, Ry, Rx,
                                                       sigmas, num, den);
    return cudaGetLastError();
}

}  // namespace
}  // namespace gbm3d

using namespace gbm3d;

extern "C" size_t gbm3d_wiener_workspace_bytes(int B, int H, int W) {
    if (B < 1 || H < 1 || W < 1) return 0;
    return (size_t)2 * B * H * W * sizeof(float);
}

extern "C" int gbm3d_wiener_stage2(const int16_t* noisy, const float* basic, int B, int H, int W,
                                   int patch, const int32_t* idx, const int32_t* n_valid, int Ry,
                                   int Rx, int K, const float* sigmas, float* out, void* workspace,
                                   size_t workspace_bytes, void* stream) {
    if (!noisy || !basic || !idx || !n_valid || !sigmas || !out || !workspace) return GBM3D_ERR_ARG;
    if (B < 1 || H < patch || W < patch || Ry < 1 || Rx < 1 || K < 1) return GBM3D_ERR_ARG;
    if ((long long)H * W >= (1LL << 31)) return GBM3D_ERR_ARG;
    if (workspace_bytes < gbm3d_wiener_workspace_bytes(B, H, W)) return GBM3D_ERR_ARG;
    if (patch != 8 || (K & (K - 1)) != 0 || K > 32) return GBM3D_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    float* num = (float*)workspace;
    float* den = num + (size_t)B * H * W;
    if (cudaMemsetAsync(workspace, 0, gbm3d_wiener_workspace_bytes(B, H, W), s) != cudaSuccess)
        return GBM3D_ERR_CUDA;
    cudaError_t e;
    switch (K) {
        case 1: e = launch_wiener<1>(noisy, basic, B, H, W, idx, n_valid, Ry, Rx, sigmas, num, den, s); break;
        case 2: e = launch_wiener<2>(noisy, basic, B, H, W, idx, n_valid, Ry, Rx, sigmas, num, den, s); break;
        case 4: e = launch_wiener<4>(noisy, basic, B, H, W, idx, n_valid, Ry, Rx, sigmas, num, den, s); break;
        case 8: e = launch_wiener<8>(noisy, basic, B, H, W, idx, n_valid, Ry, Rx, sigmas, num, den, s); break;
        case 16: e = launch_wiener<16>(noisy, basic, B, H, W, idx, n_valid, Ry, Rx, sigmas, num, den, s); break;
        default: e = launch_wiener<32>(noisy, basic, B, H, W, idx, n_valid, Ry, Rx, sigmas, num, den, s); break;
    }
    if (e != cudaSuccess) return GBM3D_ERR_CUDA;
    const int64_t n = (int64_t)B * H * W;
    const int64_t blocks = (n + 255) / 256;
    wiener_divide_kernel<<<(unsigned)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s>>>(num, den, out, n);
    return cudaGetLastError() == cudaSuccess ? GBM3D_OK : GBM3D_ERR_CUDA;
}
