// Tensor-core product-form instantiation: patch 8, stride 3, K-1 <= 15 / <= 31.
#include "match_tc.cuh"
namespace gbm3d {
template cudaError_t launch_tc<3, 15>(const MatchParams&, cudaStream_t, int*);
template cudaError_t launch_tc<3, 31>(const MatchParams&, cudaStream_t, int*);
}  // namespace gbm3d
