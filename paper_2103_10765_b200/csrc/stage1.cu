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

// All passes use 3D grids (x tiles of 128 threads, rows, slices): no integer division by
// runtime sizes in the streaming loops.
constexpr int TPB = 128;

// V[b][k][y][x] = Z_b at the k-th block of the tile containing (y, x), as float; a thread
// copies one block row (N pixels) of one tile
__global__ void __launch_bounds__(TPB) s1_volume_kernel(const int16_t* __restrict__ noisy,
        const int32_t* __restrict__ idx, int K, int H, int W, int N, float* __restrict__ V) {
    const int Bx = W / N, By = H / N;
    const int q = blockIdx.x * TPB + threadIdx.x, y = blockIdx.y, s = blockIdx.z;  // s = b K + k
    if (q >= Bx) return;
    const int k = s % K, b = s / K;
    const int p = y / N, i = y - p * N;
    const int c = __ldg(idx + (((int64_t)b * By + p) * Bx + q) * K + k);
    const int cy = c / W, cx = c - cy * W;
    const int16_t* src = noisy + ((int64_t)b * H + cy + i) * W + cx;
    float* dst = V + ((int64_t)s * H + y) * W + q * N;
    for (int j = 0; j < N; ++j) dst[j] = (float)__ldg(src + j);
}

// analysis along x of the band [0, h) x [0, w) of every slice: out row = [a | d]; a CTA makes
// TPB outputs of one row from a shared copy of the 2 TPB + 9 inputs it needs (loaded with the
// periodic wrap -- and, for the cycle spin, the circular shift -- resolved once per input);
// `shift` > 0 reads the source shifted by `shift` along k, y and x (S_h V)
__global__ void __launch_bounds__(TPB) s1_ana_x_kernel(const float* __restrict__ src,
        float* __restrict__ dst, int K, int H, int W, int w, int shift) {
    __shared__ float xs[2 * TPB + 10];
    const int half = w >> 1;
    const int i0 = blockIdx.x * TPB, y = blockIdx.y, s = blockIdx.z;
    const float* row;
    if (shift) {
        const int k = s % K, b = s / K;
        row = src + ((int64_t)(b * K + wrap(k - shift, K)) * H + wrap(y - shift, H)) * W;
    } else {
        row = src + ((int64_t)s * H + y) * W;
    }
    const int M = shift ? W : w;
    for (int j = threadIdx.x; j < 2 * TPB + 10; j += TPB) {
        const int pos = 2 * i0 - 4 + j;        // band position, in [-4, w + 6)
        int xi = wrap(min(pos, w + 5), w);
        xi = shift ? wrap(xi - shift, M) : xi;
        xs[j] = row[xi];
    }
    __syncthreads();
    const int i = i0 + threadIdx.x;
    if (i >= half) return;
    const float* q = xs + 2 * threadIdx.x + 4;  // q[t] = x[2i + t]
    float a = 0.f;
#pragma unroll
    for (int t = -4; t <= 5; ++t) a = fmaf(han(t), q[t], a);
    const float d = (q[0] - q[1]) * kR2;
    float* o = dst + ((int64_t)s * H + y) * W;
    o[i] = a;
    o[half + i] = d;
}

// analysis along y: a thread walks down one column of the band, RY outputs per CTA row, with the
// 10 input rows of the current output in a sliding register window (each input read once)
constexpr int RY = 16;
__global__ void __launch_bounds__(TPB) s1_ana_y_kernel(const float* __restrict__ src,
        float* __restrict__ dst, int H, int W, int h, int w) {
    const int half = h >> 1;
    const int x = blockIdx.x * TPB + threadIdx.x, s = blockIdx.z;
    const int i0 = blockIdx.y * RY;
    if (x >= w) return;
    const float* col = src + (int64_t)s * H * W + x;
    float* o = dst + (int64_t)s * H * W + x;
    float win[10];
#pragma unroll
    for (int t = 0; t < 8; ++t) win[t] = col[(int64_t)wrap(2 * i0 - 4 + t, h) * W];
    for (int i = i0; i < min(i0 + RY, half); ++i) {
        win[8] = col[(int64_t)wrap(2 * i + 4, h) * W];
        win[9] = col[(int64_t)wrap(2 * i + 5, h) * W];
        float a = 0.f;
#pragma unroll
        for (int t = 0; t < 10; ++t) a = fmaf(han(t - 4), win[t], a);
        o[(int64_t)i * W] = a;
        o[(int64_t)(half + i) * W] = (win[4] - win[5]) * kR2;
#pragma unroll
        for (int t = 0; t < 8; ++t) win[t] = win[t + 2];
    }
}

// synthesis along y: x[m] = h[m & 1] a[m >> 1] + sum_{n = m (mod 2)} g[n] d[(m - n) / 2];
// for an output pair (2j, 2j+1) the details d[j-2 .. j+2] and a[j] suffice: sliding window
__global__ void __launch_bounds__(TPB) s1_syn_y_kernel(const float* __restrict__ src,
        float* __restrict__ dst, int H, int W, int h, int w) {
    const int half = h >> 1;
    const int x = blockIdx.x * TPB + threadIdx.x, s = blockIdx.z;
    const int j0 = blockIdx.y * RY;
    if (x >= w) return;
    const float* col = src + (int64_t)s * H * W + x;
    float* o = dst + (int64_t)s * H * W + x;
    float dw[5];  // d[j - 2 .. j + 2]
#pragma unroll
    for (int t = 0; t < 4; ++t) dw[t] = col[(int64_t)(half + wrap(j0 - 2 + t, half)) * W];
    for (int j = j0; j < min(j0 + RY, half); ++j) {
        dw[4] = col[(int64_t)(half + wrap(j + 2, half)) * W];
        const float aj = col[(int64_t)j * W];
        // m = 2j   : n even, (m - n)/2 = j - n/2, n in {-4,-2,0,2,4} -> d[j+2], d[j+1], d[j], d[j-1], d[j-2]
        // m = 2j+1 : n odd,  (m - n)/2 = j - (n-1)/2, n in {-3,-1,1,3,5} -> d[j+2] .. d[j-2]
        float e = kR2 * aj, f = kR2 * aj;
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            e = fmaf(gsy(2 * (2 - u)), dw[u], e);       // n = 4 - 2u pairs with d[j - 2 + u]
            f = fmaf(gsy(2 * (2 - u) + 1), dw[u], f);   // n = 5 - 2u
        }
        o[(int64_t)(2 * j) * W] = e;
        o[(int64_t)(2 * j + 1) * W] = f;
#pragma unroll
        for (int t = 0; t < 4; ++t) dw[t] = dw[t + 1];
    }
}

// synthesis along x of one row segment: outputs m in [m0, m0 + 2 TPB) from shared copies of
// a[m0/2 .. m0/2 + TPB) and d[m0/2 - 2 .. m0/2 + TPB + 2); for the last level (accumulate != 0)
// U[S_-h] += scale * result
__global__ void __launch_bounds__(TPB) s1_syn_x_kernel(const float* __restrict__ src,
        float* __restrict__ dst, int K, int H, int W, int w, int shift, float scale, int accumulate) {
    __shared__ float as_[TPB], ds_[TPB + 4];
    const int half = w >> 1;
    const int j0 = blockIdx.x * TPB, y = blockIdx.y, s = blockIdx.z;
    const float* row = src + ((int64_t)s * H + y) * W;
    if (j0 + threadIdx.x < half) as_[threadIdx.x] = row[j0 + threadIdx.x];
    for (int t = threadIdx.x; t < TPB + 4; t += TPB) ds_[t] = row[half + wrap(j0 - 2 + t, half)];
    __syncthreads();
    const int j = j0 + threadIdx.x;
    if (j >= half) return;
    const float aj = as_[threadIdx.x];
    float e = kR2 * aj, f = kR2 * aj;
#pragma unroll
    for (int u = 0; u < 5; ++u) {
        const float dv = ds_[threadIdx.x + u];  // d[j - 2 + u]
        e = fmaf(gsy(2 * (2 - u)), dv, e);
        f = fmaf(gsy(2 * (2 - u) + 1), dv, f);
    }
    const int m = 2 * j;
    if (!accumulate) {
        float* o = dst + ((int64_t)s * H + y) * W;
        o[m] = e;
        o[m + 1] = f;
    } else {
        // (S_-h R)[k][y][x] = R[k + h][y + h][x + h]: this R element lands at (k-h, y-h, x-h)
        const int k = s % K, b = s / K;
        float* o = dst + ((int64_t)(b * K + wrap(k - shift, K)) * H + wrap(y - shift, H)) * W;
        o[wrap(m - shift, W)] += scale * e;
        o[wrap(m + 1 - shift, W)] += scale * f;
    }
}

// along z at every (b, y, x): Haar cascade (lz levels), hard threshold, inverse cascade
template <int K>
__global__ void __launch_bounds__(TPB) s1_z_kernel(float* __restrict__ C, int H, int W, int L, int lz,
                                                   const float* __restrict__ sigmas) {
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

// aggregation: block k < n_valid of group (p, q) adds w U_pq[k] at its position (a thread per
// block row: N reductions); the block's weight goes once to its top-left pixel of the weight
// map (the divide takes N x N box sums)
__global__ void __launch_bounds__(512) s1_aggregate_kernel(const float* __restrict__ U,
        const int32_t* __restrict__ idx, const int32_t* __restrict__ nvalid,
        const float* __restrict__ wg, int K, int H, int W, int N, float* __restrict__ num,
        float* __restrict__ wmap) {
    const int Bx = W / N, By = H / N;
    const int t = threadIdx.x;                     // (k, i) of the group: blockDim = K N
    const int g = blockIdx.x, b = blockIdx.y;      // group within image b
    const int k = t / N, i = t - k * N;
    const int64_t gi = (int64_t)b * By * Bx + g;
    if (k >= __ldg(nvalid + gi)) return;
    const int p = g / Bx, q = g - p * Bx;
    const int c = __ldg(idx + gi * K + k);
    const int cy = c / W, cx = c - cy * W;
    const float w = wg[gi];
    const int64_t plane = (int64_t)H * W;
    const float* u = U + ((int64_t)b * K + k) * plane + (int64_t)(p * N + i) * W + q * N;
    float* o = num + b * plane + (int64_t)(cy + i) * W + cx;
    for (int j = 0; j < N; ++j) atomicAdd(o + j, w * u[j]);
    if (i == 0) atomicAdd(wmap + b * plane + (int64_t)cy * W + cx, w);
}

// out = num / (N x N box sums of the weight map over [y-N+1, y] x [x-N+1, x]): 32 x 32 output
// tiles, the map staged with its (N-1)-pixel halo, separable sums
__global__ void __launch_bounds__(256) s1_divide_kernel(const float* __restrict__ num,
        const float* __restrict__ wmap, float* __restrict__ out, int H, int W, int N) {
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
    const unsigned gx = (unsigned)((W + TPB - 1) / TPB);
    s1_volume_kernel<<<dim3((unsigned)((W / patch + TPB - 1) / TPB), H, BK), TPB, 0, s>>>(
        noisy, idx, K, H, W, patch, V);
    const int spins = 2;
    for (int sh = 0; sh < spins; ++sh) {
        for (int l = 1; l <= levels; ++l) {
            const int h = H >> (l - 1), w = W >> (l - 1);
            s1_ana_x_kernel<<<dim3((unsigned)((w / 2 + TPB - 1) / TPB), h, BK), TPB, 0, s>>>(
                l == 1 ? V : C, Tm, K, H, W, w, l == 1 ? sh : 0);
            s1_ana_y_kernel<<<dim3((unsigned)((w + TPB - 1) / TPB), (unsigned)((h / 2 + RY - 1) / RY), BK),
                              TPB, 0, s>>>(Tm, C, H, W, h, w);
        }
        const dim3 zg(gx, H, B);
        switch (K) {
            case 1: s1_z_kernel<1><<<zg, TPB, 0, s>>>(C, H, W, levels, lz, sigmas); break;
            case 2: s1_z_kernel<2><<<zg, TPB, 0, s>>>(C, H, W, levels, lz, sigmas); break;
            case 4: s1_z_kernel<4><<<zg, TPB, 0, s>>>(C, H, W, levels, lz, sigmas); break;
            case 8: s1_z_kernel<8><<<zg, TPB, 0, s>>>(C, H, W, levels, lz, sigmas); break;
            case 16: s1_z_kernel<16><<<zg, TPB, 0, s>>>(C, H, W, levels, lz, sigmas); break;
            default: s1_z_kernel<32><<<zg, TPB, 0, s>>>(C, H, W, levels, lz, sigmas); break;
        }
        for (int l = levels; l >= 1; --l) {
            const int h = H >> (l - 1), w = W >> (l - 1);
            s1_syn_y_kernel<<<dim3((unsigned)((w + TPB - 1) / TPB), (unsigned)((h / 2 + RY - 1) / RY), BK),
                              TPB, 0, s>>>(C, Tm, H, W, h, w);
            s1_syn_x_kernel<<<dim3((unsigned)((w / 2 + TPB - 1) / TPB), h, BK), TPB, 0, s>>>(
                Tm, l == 1 ? U : C, K, H, W, w, sh, 1.0f / spins, l == 1);
        }
    }
    s1_tv_kernel<<<grid1((int64_t)B * (H / patch) * (W / patch) * 32), 256, 0, s>>>(U, B, K, H, W, patch, wg);
    s1_aggregate_kernel<<<dim3((unsigned)((H / patch) * (W / patch)), B), K * patch, 0, s>>>(
        U, idx, n_valid, wg, K, H, W, patch, num, wmap);
    s1_divide_kernel<<<dim3((unsigned)((W + 31) / 32), (unsigned)((H + 31) / 32), B), 256, 0, s>>>(
        num, wmap, out, H, W, patch);
    return cudaGetLastError() == cudaSuccess ? GBM3D_OK : GBM3D_ERR_CUDA;
}
