// Integer instruction-throughput microkernels (SURVEY.md 8(d) "Peak P_int must be measured on
// the box in the same run"; native component N7).  bench.py times them with CUDA events on all
// SMs and uses the best as the ALU-roofline denominator.  Every thread runs NCH independent
// dependency chains, unrolled, so the pipes -- not latency -- bound the rate.  The chains are
// shaped so that ptxas cannot fuse or fold them (checked in the SASS: tools/dev/int_peak_sass.sh):
//   kind 0 "alu"    : SHF + LOP3 alternating             (ALU pipe only)
//   kind 1 "fma"    : IMAD                               (FMA pipe only)
//   kind 2 "minmax" : IMNMX (min) + IMNMX (max)          (ALU pipe: the selector's instruction)
//   kind 3 "mixed"  : IMAD + IADD3 alternating           (both pipes: the issue-rate bound)
// One "op" = one SASS instruction for one lane; gbm3d_int_peak_ops gives the op count per
// launch.
#include <cstdint>

#include "../../include/gbm3d.h"
#include "common.cuh"

namespace gbm3d {

constexpr int IP_NCH = 8;     // independent chains per thread
constexpr int IP_UNROLL = 16; // chain steps per loop iteration

template <int KIND>
__global__ void __launch_bounds__(256) int_peak_kernel(uint32_t* __restrict__ sink, int iters,
                                                       uint32_t b, uint32_t c) {
    uint32_t a[IP_NCH];
#pragma unroll
    for (int j = 0; j < IP_NCH; ++j) a[j] = threadIdx.x * 0x9E3779B9u + j * 0x85EBCA6Bu + blockIdx.x;
    const uint32_t bb = b ^ threadIdx.x, cc = c + blockIdx.x;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < IP_UNROLL; ++u) {
#pragma unroll
            for (int j = 0; j < IP_NCH; ++j) {
                if (KIND == 0) {  // (ptxas turns a lone add.u32 into IMAD.IADD on the FMA pipe)
                    asm volatile("shf.l.wrap.b32 %0, %0, %0, %1;" : "+r"(a[j]) : "r"(bb));
                    asm volatile("xor.b32 %0, %0, %1;" : "+r"(a[j]) : "r"(cc));
                } else if (KIND == 1) {
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(bb), "r"(cc));
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(cc), "r"(bb));
                } else if (KIND == 2) {
                    asm volatile("min.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(bb));
                    asm volatile("max.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(cc));
                } else {
                    asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(bb), "r"(cc));
                    asm volatile("add.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(bb));
                }
            }
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < IP_NCH; ++j) x ^= a[j];
    if (x == 0x12345678u) sink[blockIdx.x] = x;  // keeps the chains alive
}

}  // namespace gbm3d

using namespace gbm3d;

extern "C" {

double gbm3d_int_peak_ops(int kind, int blocks, int threads, int iters) {
    if (kind < 0 || kind > 3) return 0.0;
    return (double)blocks * threads * iters * IP_UNROLL * IP_NCH * 2.0;
}

int gbm3d_int_peak_launch(int kind, int blocks, int threads, int iters, uint32_t* sink,
                          void* stream) {
    if (!sink || blocks < 1 || threads < 32 || threads > 256 || (threads & 31) || iters < 1)
        return GBM3D_ERR_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    const uint32_t b = 0x2545F491u, c = 0x6C078965u;
    switch (kind) {
        case 0: int_peak_kernel<0><<<blocks, threads, 0, s>>>(sink, iters, b, c); break;
        case 1: int_peak_kernel<1><<<blocks, threads, 0, s>>>(sink, iters, b, c); break;
        case 2: int_peak_kernel<2><<<blocks, threads, 0, s>>>(sink, iters, b, c); break;
        case 3: int_peak_kernel<3><<<blocks, threads, 0, s>>>(sink, iters, b, c); break;
        default: return GBM3D_ERR_ARG;
    }
    return cudaGetLastError() == cudaSuccess ? GBM3D_OK : GBM3D_ERR_CUDA;
}

}  // extern "C"
