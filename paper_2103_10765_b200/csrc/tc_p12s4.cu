// Tensor-core product-form instantiations for patch 12, stride 4 (BASELINE c2): K-1 <= 15 / <= 31.
#include "match_tcp.cuh"
namespace gbm3d {
template cudaError_t launch_tcp<12, 4, 15, 64>(const MatchParams&, cudaStream_t, int*);
template cudaError_t launch_tcp<12, 4, 31, 64>(const MatchParams&, cudaStream_t, int*);
template cudaError_t launch_tcp<12, 4, 15, 80>(const MatchParams&, cudaStream_t, int*);
template cudaError_t launch_tcp<12, 4, 31, 80>(const MatchParams&, cudaStream_t, int*);
}  // namespace gbm3d

#if GBM3D_TCP_TRACE
extern "C" int gbm3d_dev_tcp_trace(long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, gbm3d::g_tcp_trace, sizeof(long long) * 12 * (n < 4096 ? n : 4096));
}
extern "C" int gbm3d_dev_tcp_cnt(long long* host, int n) {
    return (int)cudaMemcpyFromSymbol(host, gbm3d::g_tcp_cnt, sizeof(long long) * 24 * (n < 4096 ? n : 4096));
}
extern "C" int gbm3d_dev_tcp_cnt_reset() {
    static long long z[4096 * 24];
    return (int)cudaMemcpyToSymbol(gbm3d::g_tcp_cnt, z, sizeof(z));
}
#endif
