// Generic exact block matching, one CTA per reference: direct Eq. (1) SSD for every candidate
// of the clamped window, then a bitonic sort of 64-bit keys (d << 32 | idx) in shared memory.
// Used for the appended last reference row/column of the grid (reading R3), for shapes the
// fast kernels do not instantiate, and as GBM3D_METHOD_DIRECT.  Not the hot path.
#pragma once
#include "common.cuh"

namespace gbm3d {

// References [k_begin, k_end) x [m_begin, m_end) of the grid (grid indices), every image.
__global__ void __launch_bounds__(256) match_direct_kernel(MatchParams p, int k_begin, int m_begin,
                                                           int m_count, int npow2) {
    extern __shared__ __align__(16) unsigned long long keys[];
    __shared__ int refpatch[16 * 16];
    const int P = p.P, r = p.r, W = p.W;
    const int k = k_begin + (int)(blockIdx.x / (unsigned)m_count);
    const int m = m_begin + (int)(blockIdx.x % (unsigned)m_count);
    const int b = blockIdx.z;
    const int16_t* __restrict__ img = p.img + (int64_t)b * p.img_bstride;
    const int ry = grid_pos(k, p.Ry_reg, p.S, p.H - P);
    const int rx = grid_pos(m, p.Rx_reg, p.S, p.W - P);
    for (int i = threadIdx.x; i < P * P; i += blockDim.x)
        refpatch[i] = img[(int64_t)(ry + i / P - p.slab_y0) * W + rx + i % P];
    const int cy0 = max(0, ry - r), cy1 = min(p.H - P, ry + r);
    const int cx0 = max(0, rx - r), cx1 = min(p.W - P, rx + r);
    const int wx = cx1 - cx0 + 1, n = (cy1 - cy0 + 1) * wx;
    __syncthreads();
    for (int c = threadIdx.x; c < npow2; c += blockDim.x) {
        unsigned long long key = ~0ull;
        if (c < n) {
            const int cy = cy0 + c / wx, cx = cx0 + c % wx;
            if (!(cy == ry && cx == rx)) {
                int64_t d = 0;
                for (int i = 0; i < P; ++i) {
                    const int16_t* row = img + (int64_t)(cy + i - p.slab_y0) * W + cx;
                    for (int j = 0; j < P; ++j) {
                        const int64_t df = (int64_t)refpatch[i * P + j] - (int64_t)__ldg(row + j);
                        d += df * df;
                    }
                }
                if (d < p.tau) key = ((unsigned long long)d << 32) | (uint32_t)(cy * W + cx);
            }
        }
        keys[c] = key;
    }
    __syncthreads();
    // bitonic sort, ascending
    for (int size = 2; size <= npow2; size <<= 1) {
        for (int stride = size >> 1; stride > 0; stride >>= 1) {
            for (int i = threadIdx.x; i < (npow2 >> 1); i += blockDim.x) {
                const int lo = 2 * i - (i & (stride - 1));
                const int hi = lo + stride;
                const bool up = (lo & size) == 0;
                const unsigned long long x = keys[lo], y = keys[hi];
                if ((x > y) == up) {
                    keys[lo] = y;
                    keys[hi] = x;
                }
            }
            __syncthreads();
        }
    }
    const int64_t ref = (int64_t)b * p.out_bstride + (int64_t)(k - p.row_begin) * p.Rx + m;
    int32_t* oi = p.idx + ref * p.K;
    int32_t* od = p.dist + ref * p.K;
    const int self = ry * W + rx;
    for (int s = threadIdx.x; s < p.K; s += blockDim.x) {
        if (s == 0) {
            oi[0] = self;
            od[0] = 0;
        } else {
            const unsigned long long key = (s - 1 < npow2) ? keys[s - 1] : ~0ull;
            if (key != ~0ull) {
                oi[s] = (int32_t)(uint32_t)(key & 0xffffffffu);
                od[s] = (int32_t)(key >> 32);
            } else {
                oi[s] = self;
                od[s] = -1;
            }
        }
    }
    if (p.nvalid && threadIdx.x == 0) {
        int cnt = 0;
        for (int s = 0; s < p.K - 1 && s < npow2; ++s) cnt += keys[s] != ~0ull;
        p.nvalid[ref] = 1 + cnt;
    }
}

}  // namespace gbm3d
