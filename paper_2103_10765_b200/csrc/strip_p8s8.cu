// Fast-path instantiation: patch 8, stride 8 -- the tiling references of stage 1 (PAPER.md:156,
// reference blocks at (pN, qN)).  S = P: one chunk per reference row, no helper lanes.
#include "match_strip.cuh"
#include "strip_p8s8.cuh"
namespace gbm3d {
GBM3D_INSTANTIATE_STRIP(8, 8, GBM3D_S8_TRY, GBM3D_S8_D, GBM3D_S8_WPS)
}  // namespace gbm3d
