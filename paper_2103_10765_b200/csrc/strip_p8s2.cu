// Fast-path instantiation: patch 8, stride 2 (TRY=8 reference rows per strip, D=5 dy per block).
#include "match_strip.cuh"
namespace gbm3d {
GBM3D_INSTANTIATE_STRIP(8, 2, 8, 5, 2)
}  // namespace gbm3d
