// Shared definitions of the CUDA path (NOT shared with oracle/: see DESIGN.md "Oracle").
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gbm3d {

constexpr uint32_t KEY_INF = 0xFFFFFFFFu;  // empty list slot / "no threshold"

// Launch-wide parameters of one matching call (a batch of images, or a row range of one).
struct MatchParams {
    const int16_t* img;      // image 0; for row-range calls the slab holding rows [slab_y0, slab_y1)
    int64_t img_bstride;     // elements between consecutive images of a batch
    int H, W, P, S, r, K;
    int64_t tau;             // raw SSD threshold (strict); INT64_MAX = none
    int Ry, Rx;              // full grid counts (incl. the appended last row/col, reading R3)
    int Ry_reg, Rx_reg;      // regular part: positions 0, S, 2S, ...
    int slab_y0, slab_y1;    // global image rows present in memory
    int row_begin, row_end;  // reference grid rows computed by this call
    int32_t* idx;            // output rows [row_begin, row_end) of image 0
    int32_t* dist;
    int32_t* nvalid;         // nullable
    int64_t out_bstride;     // references between consecutive images in the outputs
    int B;
    // 32-bit key packing (fast kernels): key = d << cb | code, code = (dy+r)*side + (dx+r)
    int side;                // 2r+1
    int cb;                  // bits for the displacement code, 2^cb > side^2
    uint32_t dsat;           // largest d representable in the key: 2^(32-cb) - 1
    int tdr0;                // initial gate on d: min(dsat, tau-1) (-1 when tau == 0)
    uint32_t thr0;           // initial key threshold: tau << cb if tau <= dsat, else KEY_INF
    int tau_above_dsat;      // tau - 1 > dsat: candidates with d > dsat may be valid matches
};

__host__ __device__ inline int grid_pos(int k, int reg, int S, int last) {
    return k < reg ? k * S : last;
}

}  // namespace gbm3d
