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
// Layout: volumes are float [B][K][H][W] (slice-major).  The 2D transform uses the in-place
// Mallat layout (level l's LL band in the top-left H/2^l x W/2^l corner).  Passes:
//   volume build (gather, with the cycle shift folded into the first row pass's reads),
//   per level: analysis along x into a scratch volume, analysis along y back,
//   one pass along z: Haar cascade + threshold + inverse cascade in registers (thread per pixel),
//   per level (coarsest first): synthesis along y into scratch, synthesis along x back (the last
//   one adds 1/H x the unshifted result into the accumulator U),
//   TV weight per group (warp per group), aggregation (fp32 reductions) and the N x N box-sum
//   divide.  Every pass is a streaming pass over the volume: HBM bound.
#include <cmath>
#include <cstdint>

#include <cuda_runtime.h>

#include "../../include/gbm3d.h"

namespace gbm3d {
namespace {

// bior1.5 analysis lowpass on n = -4..5 (x sqrt2/256), synthesis lowpass = Haar; highpasses by
// the biorthogonal QMF relations g~[n] = (-1)^n h[1-n], g[n] = (-1)^n h~[1-n].  The constants are
// the CDF(1,5) integers; the scaling is applied in the kernels.
__constant__ float kHan[10] = {3.f, -3.f, -22.f, 22.f, 128.f, 128.f, 22.f, -22.f, -3.f, 3.f};

__device__ __forceinline__ float han(int n) {  // n in [-4, 5]
    return kHan[n + 4] * 0.005524271728019903f;  // sqrt(2) / 256
}
__device__ __forceinline__ float gsy(int n) {  // g[n] = (-1)^n h~[1 - n], n in [-4, 5]
    const float v = han(1 - n);
    return (n & 1) ? -v : v;
}
constexpr float kR2 = 0.70710678118654752f;

__device__ __forceinline__ int wrap(int i, int n) { return i < 0 ? i + n : (i >= n ? i - n : i); }

// V[b][k][y][x] = Z_b at the k-th block of the tile containing (y, x), as float
__global__ void s1_volume_kernel(const int16_t* __restrict__ noisy, const int32_t* __restrict__ idx,
                                 int B, int K, int H, int W, int N, float* __restrict__ V) {
    const int Bx = W / N, By = H / N;
    const int64_t n = (int64_t)B * K * H * W;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(e % W);
        const int64_t r1 = e / W;
        const int y = (int)(r1 % H);
        const int64_t r2 = r1 / H;
        const int k = (int)(r2 % K);
        const int64_t b = r2 / K;
        const int p = y / N, q = x / N;
        const int c = __ldg(idx + ((b * By + p) * Bx + q) * K + k);
        const int cy = c / W, cx = c - cy * W;
        V[e] = (float)__ldg(noisy + (b * H + cy + (y - p * N)) * (int64_t)W + cx + (x - q * N));
    }
}

// analysis along x of the band [0, h) x [0, w) of every slice: out row = [a | d];
// `shift` > 0 reads the source circularly shifted by `shift` along k, y and x (S_h V)
__global__ void s1_ana_x_kernel(const float* __restrict__ src, float* __restrict__ dst, int BK, int K,
                                int H, int W, int h, int w, int shift) {
    const int half = w >> 1;
    const int64_t n = (int64_t)BK * h * half;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(e % half);
        const int64_t r = e / half;
        const int y = (int)(r % h);
        const int s = (int)(r / h);  // slice index b * K + k
        const float* row;
        if (shift) {
            const int k = s % K, b = s / K;
            const int ks = wrap(k - shift, K), ys = wrap(y - shift, H);
            row = src + ((int64_t)(b * K + ks) * H + ys) * W;
        } else {
            row = src + ((int64_t)s * H + y) * W;
        }
        float a = 0.f;
#pragma unroll
        for (int t = -4; t <= 5; ++t) {
            const int xx = wrap(wrap(2 * i + t, w) - shift, shift ? W : w);
            a = fmaf(han(t), row[xx], a);
        }
        const int x0 = wrap(2 * i - shift, shift ? W : w), x1 = wrap(2 * i + 1 - shift, shift ? W : w);
        const float d = (row[x0] - row[x1]) * kR2;
        float* o = dst + ((int64_t)s * H + y) * W;
        o[i] = a;
        o[half + i] = d;
    }
}

// analysis along y of the band: out column = [a ; d]
__global__ void s1_ana_y_kernel(const float* __restrict__ src, float* __restrict__ dst, int BK, int H,
                                int W, int h, int w) {
    const int half = h >> 1;
    const int64_t n = (int64_t)BK * half * w;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(e % w);
        const int64_t r = e / w;
        const int i = (int)(r % half);
        const int s = (int)(r / half);
        const float* col = src + (int64_t)s * H * W + x;
        float a = 0.f;
#pragma unroll
        for (int t = -4; t <= 5; ++t) a = fmaf(han(t), col[(int64_t)wrap(2 * i + t, h) * W], a);
        const float d = (col[(int64_t)(2 * i) * W] - col[(int64_t)(2 * i + 1) * W]) * kR2;
        float* o = dst + (int64_t)s * H * W + x;
        o[(int64_t)i * W] = a;
        o[(int64_t)(half + i) * W] = d;
    }
}

// synthesis along y of the band: x[m] = h[m & 1] a[m >> 1] + sum_{n = m (mod 2)} g[n] d[(m - n) / 2]
__global__ void s1_syn_y_kernel(const float* __restrict__ src, float* __restrict__ dst, int BK, int H,
                                int W, int h, int w) {
    const int half = h >> 1;
    const int64_t n = (int64_t)BK * h * w;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int x = (int)(e % w);
        const int64_t r = e / w;
        const int m = (int)(r % h);
        const int s = (int)(r / h);
        const float* col = src + (int64_t)s * H * W + x;
        float v = kR2 * col[(int64_t)(m >> 1) * W];
#pragma unroll
        for (int t = -4; t <= 5; ++t) {
            if (((m - t) & 1) == 0) v = fmaf(gsy(t), col[(int64_t)(half + wrap((m - t) >> 1, half)) * W], v);
        }
        dst[(int64_t)s * H * W + (int64_t)m * W + x] = v;
    }
}

// synthesis along x; for the last level (accumulate != 0) U[S_-h] += scale * result
__global__ void s1_syn_x_kernel(const float* __restrict__ src, float* __restrict__ dst, int BK, int K,
                                int H, int W, int h, int w, int shift, float scale, int accumulate) {
    const int half = w >> 1;
    const int64_t n = (int64_t)BK * h * w;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int m = (int)(e % w);
        const int64_t r = e / w;
        const int y = (int)(r % h);
        const int s = (int)(r / h);
        const float* row = src + ((int64_t)s * H + y) * W;
        float v = kR2 * row[m >> 1];
#pragma unroll
        for (int t = -4; t <= 5; ++t) {
            if (((m - t) & 1) == 0) v = fmaf(gsy(t), row[half + wrap((m - t) >> 1, half)], v);
        }
        if (!accumulate) {
            dst[((int64_t)s * H + y) * W + m] = v;
        } else {
            // (S_-h R)[k][y][x] = R[k + h][y + h][x + h]: this R element lands at (k-h, y-h, x-h)
            const int k = s % K, b = s / K;
            const int ko = wrap(k - shift, K), yo = wrap(y - shift, H), xo = wrap(m - shift, W);
            dst[((int64_t)(b * K + ko) * H + yo) * W + xo] += scale * v;
        }
    }
}

// along z at every (b, y, x): Haar cascade (lz levels), hard threshold, inverse cascade
template <int K>
__global__ void s1_z_kernel(float* __restrict__ C, int B, int H, int W, int L, int lz,
                            const float* __restrict__ sigmas) {
    const int64_t plane = (int64_t)H * W;
    const int64_t n = (int64_t)B * plane;
    const int hL = H >> L, wL = W >> L;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / plane;
        const int64_t pix = e - b * plane;
        const int y = (int)(pix / W), x = (int)(pix - (int64_t)y * W);
        // spatial level of (y, x) in the Mallat layout: l such that it lies in the level-l detail
        // bands; the final LL band counts as level L (reading S2)
        int lev = L;
        for (int l = 1; l <= L; ++l) {
            if (y >= (H >> l) || x >= (W >> l)) { lev = l; break; }
        }
        const bool ll = y < hL && x < wL;
        const float lam = sigmas[b] * (3.6f - 0.3f * (float)lev);
        float v[K];
        float* base = C + b * K * plane + pix;
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
}

// TV of every group U_pq (K x N x N) -> weight 1 / TV (1 when TV = 0); warp per group
__global__ void s1_tv_kernel(const float* __restrict__ U, int B, int K, int H, int W, int N,
                             float* __restrict__ wout) {
    const int Bx = W / N, By = H / N;
    const int64_t ngroups = (int64_t)B * By * Bx;
    const int lane = threadIdx.x & 31;
    for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < ngroups;
         g += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t b = g / (By * Bx);
        const int pq = (int)(g - b * By * Bx), p = pq / Bx, q = pq - p * Bx;
        const float* base = U + b * K * (int64_t)H * W + (int64_t)(p * N) * W + q * N;
        float tv = 0.f;
        for (int e = lane; e < K * N * N; e += 32) {
            const int k = e / (N * N), r = e - k * N * N, i = r / N, j = r - i * N;
            const float u = base[(int64_t)k * H * W + (int64_t)i * W + j];
            if (k + 1 < K) tv += fabsf(base[(int64_t)(k + 1) * H * W + (int64_t)i * W + j] - u);
            if (i + 1 < N) tv += fabsf(base[(int64_t)k * H * W + (int64_t)(i + 1) * W + j] - u);
            if (j + 1 < N) tv += fabsf(base[(int64_t)k * H * W + (int64_t)i * W + j + 1] - u);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tv += __shfl_xor_sync(0xffffffffu, tv, o);
        if (lane == 0) wout[g] = tv > 0.f ? 1.f / tv : 1.f;
    }
}

// aggregation: block k < n_valid of group (p, q) adds w U_pq[k] at its position; the block's
// weight goes once to its top-left pixel of the weight map (the divide takes N x N box sums)
__global__ void s1_aggregate_kernel(const float* __restrict__ U, const int32_t* __restrict__ idx,
                                    const int32_t* __restrict__ nvalid, const float* __restrict__ wg,
                                    int B, int K, int H, int W, int N, float* __restrict__ num,
                                    float* __restrict__ wmap) {
    const int Bx = W / N, By = H / N;
    const int64_t n = (int64_t)B * By * Bx * K * N * N;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int r = (int)(e % (N * N));
        const int64_t gk = e / (N * N);
        const int k = (int)(gk % K);
        const int64_t g = gk / K;
        const int64_t b = g / (By * Bx);
        const int pq = (int)(g - b * By * Bx), p = pq / Bx, q = pq - p * Bx;
        if (k >= __ldg(nvalid + g)) continue;
        const int i = r / N, j = r - i * N;
        const int c = __ldg(idx + g * K + k);
        const int cy = c / W, cx = c - cy * W;
        const float w = wg[g];
        const float u = U[(b * K + k) * (int64_t)H * W + (int64_t)(p * N + i) * W + q * N + j];
        atomicAdd(num + b * (int64_t)H * W + (int64_t)(cy + i) * W + cx + j, w * u);
        if (r == 0) atomicAdd(wmap + b * (int64_t)H * W + (int64_t)cy * W + cx, w);
    }
}

// out = num / (N x N box sums of the weight map over [y-N+1, y] x [x-N+1, x])
__global__ void s1_divide_kernel(const float* __restrict__ num, const float* __restrict__ wmap,
                                 float* __restrict__ out, int B, int H, int W, int N) {
    const int64_t n = (int64_t)B * H * W;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t b = e / ((int64_t)H * W);
        const int64_t pix = e - b * (int64_t)H * W;
        const int y = (int)(pix / W), x = (int)(pix - (int64_t)y * W);
        float d = 0.f;
        for (int i = max(0, y - N + 1); i <= y; ++i)
            for (int j = max(0, x - N + 1); j <= x; ++j) d += wmap[b * (int64_t)H * W + (int64_t)i * W + j];
        out[e] = d > 0.f ? num[e] / d : 0.f;
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
    const size_t groups = (size_t)B * (H / patch) * (W / patch);
    return (4 * vol + 2 * (size_t)B * H * W + groups) * sizeof(float);
}

extern "C" int gbm3d_stage1_denoise(const int16_t* noisy, int B, int H, int W, int patch,
                                    const int32_t* idx, const int32_t* n_valid, int K,
                                    const float* sigmas, int levels, float* out, void* workspace,
                                    size_t workspace_bytes, void* stream) {
    if (!noisy || !idx || !n_valid || !sigmas || !out || !workspace) return GBM3D_ERR_ARG;
    if (B < 1 || patch < 1 || K < 1 || levels < 1 || H < patch || W < patch) return GBM3D_ERR_ARG;
    if (H % patch || W % patch || H % (2 << levels) || W % (2 << levels)) return GBM3D_ERR_ARG;
    if ((long long)H * W >= (1LL << 31)) return GBM3D_ERR_ARG;
    if (workspace_bytes < gbm3d_stage1_workspace_bytes(B, H, W, patch, K)) return GBM3D_ERR_ARG;
    if ((K & (K - 1)) != 0 || K > 32 || patch > 16 || levels > 5) return GBM3D_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t vol = (int64_t)B * K * H * W, plane = (int64_t)B * H * W;
    float* const V = (float*)workspace;   // the volume (kept for both cycle spins)
    float* const C = V + vol;             // coefficients
    float* const Tm = C + vol;            // separable-pass scratch
    float* const U = Tm + vol;            // filtered volume (mean of the spins)
    float* const num = U + vol;
    float* const wmap = num + plane;
    float* const wg = wmap + plane;
    int lz = 0;  // Haar levels along z: min(L, log2 K) (reading S1)
    while ((1 << (lz + 1)) <= K && lz < levels) ++lz;
    const int BK = B * K;
    if (cudaMemsetAsync(U, 0, (size_t)(vol + 2 * plane) * sizeof(float), s) != cudaSuccess)
        return GBM3D_ERR_CUDA;
    s1_volume_kernel<<<grid1(vol), 256, 0, s>>>(noisy, idx, B, K, H, W, patch, V);
    const int spins = 2;
    for (int sh = 0; sh < spins; ++sh) {
        for (int l = 1; l <= levels; ++l) {
            const int h = H >> (l - 1), w = W >> (l - 1);
            s1_ana_x_kernel<<<grid1((int64_t)BK * h * (w / 2)), 256, 0, s>>>(l == 1 ? V : C, Tm, BK, K, H, W,
                                                                             h, w, l == 1 ? sh : 0);
            s1_ana_y_kernel<<<grid1((int64_t)BK * (h / 2) * w), 256, 0, s>>>(Tm, C, BK, H, W, h, w);
        }
        switch (K) {
            case 1: s1_z_kernel<1><<<grid1(plane), 256, 0, s>>>(C, B, H, W, levels, lz, sigmas); break;
            case 2: s1_z_kernel<2><<<grid1(plane), 256, 0, s>>>(C, B, H, W, levels, lz, sigmas); break;
            case 4: s1_z_kernel<4><<<grid1(plane), 256, 0, s>>>(C, B, H, W, levels, lz, sigmas); break;
            case 8: s1_z_kernel<8><<<grid1(plane), 256, 0, s>>>(C, B, H, W, levels, lz, sigmas); break;
            case 16: s1_z_kernel<16><<<grid1(plane), 256, 0, s>>>(C, B, H, W, levels, lz, sigmas); break;
            default: s1_z_kernel<32><<<grid1(plane), 256, 0, s>>>(C, B, H, W, levels, lz, sigmas); break;
        }
        for (int l = levels; l >= 1; --l) {
            const int h = H >> (l - 1), w = W >> (l - 1);
            s1_syn_y_kernel<<<grid1((int64_t)BK * h * w), 256, 0, s>>>(C, Tm, BK, H, W, h, w);
            s1_syn_x_kernel<<<grid1((int64_t)BK * h * w), 256, 0, s>>>(Tm, l == 1 ? U : C, BK, K, H, W, h, w,
                                                                      sh, 1.0f / spins, l == 1);
        }
    }
    s1_tv_kernel<<<grid1((int64_t)B * (H / patch) * (W / patch) * 32), 256, 0, s>>>(U, B, K, H, W, patch, wg);
    s1_aggregate_kernel<<<grid1(vol), 256, 0, s>>>(U, idx, n_valid, wg, B, K, H, W, patch, num, wmap);
    s1_divide_kernel<<<grid1(plane), 256, 0, s>>>(num, wmap, out, B, H, W, patch);
    return cudaGetLastError() == cudaSuccess ? GBM3D_OK : GBM3D_ERR_CUDA;
}
