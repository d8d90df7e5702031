// Fast-path instantiation: patch 12, stride 4 (shape in strip_p12s4.cuh).
#include "match_strip.cuh"
#include "strip_p12s4.cuh"
namespace gbm3d {
GBM3D_INSTANTIATE_STRIP(12, 4, GBM3D_S12_TRY, GBM3D_S12_D, GBM3D_S12_WPS)
}  // namespace gbm3d
