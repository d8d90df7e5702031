// Fast-path instantiation: patch 12, stride 4 (TRY=4 reference rows per strip, D=4 dy per block).
#include "match_strip.cuh"
namespace gbm3d {
GBM3D_INSTANTIATE_STRIP(12, 4, 4, 4, 2)
}  // namespace gbm3d
