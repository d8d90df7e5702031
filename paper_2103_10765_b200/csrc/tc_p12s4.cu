// Tensor-core product-form instantiations for patch 12, stride 4 (BASELINE c2): K-1 <= 15 / <= 31.
#include "match_tcp.cuh"
namespace gbm3d {
template cudaError_t launch_tcp<12, 4, 15>(const MatchParams&, cudaStream_t, int*);
template cudaError_t launch_tcp<12, 4, 31>(const MatchParams&, cudaStream_t, int*);
}  // namespace gbm3d
