// Translation trials of stage 1 (Eq. (10)):
//   Y_f = (1/H) sum_h S_-h( phi(S_h Z) ),
// S_h = circular shift of the image by h pixels along both axes (reading S8).  The
// trials run as one batch: gbm3d_shift_trials stacks S_h Z for every trial h into a batch of
// T x B images (matched and filtered by the batched entries), gbm3d_unshift_mean shifts each
// trial's estimate back and averages them.  Pure data movement, HBM-bound: one coalesced
// pass over the inputs and outputs (a thread per 4 consecutive output pixels of a row).
#include <cstdint>

#include "../../include/gbm3d.h"
#include "common.cuh"

namespace gbm3d {

struct TrialShifts {
    int n;
    int h[GBM3D_MAX_TRIALS];
};

// out[t][b][y][x] = imgs[b][(y - h_t) mod H][(x - h_t) mod W]   (np.roll(Z, (h, h)))
__global__ void shift_trials_kernel(const int16_t* __restrict__ imgs, int B, int H, int W,
                                    TrialShifts s, int16_t* __restrict__ out) {
    const int x4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    const int y = blockIdx.y;
    const int tb = blockIdx.z;  // t * B + b
    if (x4 >= W) return;
    const int t = tb / B, b = tb - t * B;
    const int h = s.h[t];
    const int16_t* src = imgs + ((int64_t)b * H + (y - h % H + H) % H) * W;
    int16_t* dst = out + ((int64_t)tb * H + y) * W;
    const int hx = h % W;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int x = x4 + i;
        if (x < W) {
            int xs = x - hx;
            xs += xs < 0 ? W : 0;
            dst[x] = src[xs];
        }
    }
}

// out[b][y][x] = (1/T) sum_t ys[t][b][(y + h_t) mod H][(x + h_t) mod W]   (np.roll(., (-h, -h)))
__global__ void unshift_mean_kernel(const float* __restrict__ ys, int B, int H, int W,
                                    TrialShifts s, float* __restrict__ out) {
    const int x4 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    const int y = blockIdx.y;
    const int b = blockIdx.z;
    if (x4 >= W) return;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int t = 0; t < s.n; ++t) {
        const int h = s.h[t];
        const float* src = ys + ((int64_t)(t * B + b) * H + (y + h) % H) * W;
        const int hx = h % W;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int xs = x4 + i + hx;
            xs -= xs >= W ? W : 0;
            if (x4 + i < W) acc[i] += src[xs];
        }
    }
    const float inv = 1.0f / (float)s.n;
    float* dst = out + ((int64_t)b * H + y) * W;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (x4 + i < W) dst[x4 + i] = acc[i] * inv;
}

static int make_shifts(const int* shifts, int T, int H, int W, TrialShifts* s) {
    if (!shifts || T < 1 || T > GBM3D_MAX_TRIALS) return GBM3D_ERR_ARG;
    s->n = T;
    for (int t = 0; t < T; ++t) {
        if (shifts[t] < 0 || shifts[t] >= H || shifts[t] >= W) return GBM3D_ERR_ARG;
        s->h[t] = shifts[t];
    }
    return GBM3D_OK;
}

}  // namespace gbm3d

using namespace gbm3d;

extern "C" {

int gbm3d_shift_trials(const int16_t* imgs, int B, int H, int W, const int* shifts, int T,
                       int16_t* out, void* stream) {
    if (!imgs || !out || B < 1 || H < 1 || W < 1 || (int64_t)T * B > 65535) return GBM3D_ERR_ARG;
    TrialShifts s;
    const int st = make_shifts(shifts, T, H, W, &s);
    if (st != GBM3D_OK) return st;
    const dim3 block(128), grid((W + 4 * 128 - 1) / (4 * 128), H, T * B);
    if (H > 65535) return GBM3D_ERR_UNSUPPORTED;
    shift_trials_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(imgs, B, H, W, s, out);
    return cudaGetLastError() == cudaSuccess ? GBM3D_OK : GBM3D_ERR_CUDA;
}

int gbm3d_unshift_mean(const float* ys, int T, int B, int H, int W, const int* shifts,
                       float* out, void* stream) {
    if (!ys || !out || B < 1 || H < 1 || W < 1 || B > 65535) return GBM3D_ERR_ARG;
    TrialShifts s;
    const int st = make_shifts(shifts, T, H, W, &s);
    if (st != GBM3D_OK) return st;
    if (H > 65535) return GBM3D_ERR_UNSUPPORTED;
    const dim3 block(128), grid((W + 4 * 128 - 1) / (4 * 128), H, B);
    unshift_mean_kernel<<<grid, block, 0, (cudaStream_t)stream>>>(ys, B, H, W, s, out);
    return cudaGetLastError() == cudaSuccess ? GBM3D_OK : GBM3D_ERR_CUDA;
}

}  // extern "C"
