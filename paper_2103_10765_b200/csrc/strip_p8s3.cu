// Fast-path instantiation: patch 8, stride 3 (solo warps: TRY=4 reference rows, D=8 dy per block).
#include "match_strip.cuh"
namespace gbm3d {
GBM3D_INSTANTIATE_STRIP(8, 3, 4, 8, 1)
}  // namespace gbm3d
