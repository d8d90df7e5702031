// Fast-path instantiation: patch 8, stride 4 (TRY=6 reference rows per strip, D=4 dy per block).
#include "match_strip.cuh"
namespace gbm3d {
GBM3D_INSTANTIATE_STRIP(8, 4, 6, 4, 2)
}  // namespace gbm3d
