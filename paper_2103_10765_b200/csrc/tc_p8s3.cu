// Tensor-core product-form instantiations: patch 8, stride 3, K-1 <= 15 / <= 31.
#include "match_tc16.cuh"
namespace gbm3d {
template cudaError_t launch_tc<3, 15>(const MatchParams&, cudaStream_t, int*, int);
template cudaError_t launch_tc<3, 31>(const MatchParams&, cudaStream_t, int*, int);
template cudaError_t launch_tc16<3, 15>(const MatchParams&, cudaStream_t, int*);
template cudaError_t launch_tc16<3, 31>(const MatchParams&, cudaStream_t, int*);
}  // namespace gbm3d

#if GBM3D_TC_TRACE
extern "C" int gbm3d_dev_cta_spans(long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, gbm3d::g_cta_span, sizeof(long long) * 3 * (n < 65536 ? n : 65536));
}
extern "C" int gbm3d_dev_tc_trace(long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, gbm3d::g_tc_trace, sizeof(long long) * (n < 8192 ? n : 8192));
}
#endif
