// Dev check: is tcgen05 kind::f16 (fp16 in, fp32 accumulate) exact for integer operands with
// all partial sums < 2^24?  Many CTAs, random and adversarial integer data, K = 64.
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "../../paper_2103_10765_b200/csrc/tc_ptx.cuh"
using namespace gbm3d;
constexpr int M = 128, N = 64, KE = 64, KB = KE * 2;  // K in elements / bytes
__device__ __forceinline__ int cm_off(int row, int kbyte) {
    return (row >> 3) * (KB / 16) * 128 + (kbyte >> 4) * 128 + (row & 7) * 16 + (kbyte & 15);
}
__device__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__device__ int val(uint32_t seed, int mode, int vmax) {
    uint32_t h = hash(seed);
    if (mode == 0) return (int)(h % (2 * vmax + 1)) - vmax;
    if (mode == 1) return (h & 1) ? vmax : -vmax;          // extremes
    if (mode == 2) return (h & 1) ? vmax : ((h >> 1) & 3);  // large + tiny mix
    return (int)(h % (vmax + 1));                           // non-negative
}
__global__ void k(int vmax, unsigned long long* bad, unsigned long long* total) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* sA = sm; uint8_t* sB = sm + M * KB;
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    __shared__ short iA[M][KE + 1];
    __shared__ short iB[N][KE + 1];
    const int t = threadIdx.x, w = t >> 5;
    const int mode = blockIdx.x & 3;
    for (int i = t; i < M * KE; i += blockDim.x) {
        const int v = val(blockIdx.x * 1000003u + i, mode, vmax);
        iA[i / KE][i % KE] = v;
        *reinterpret_cast<__half*>(sA + cm_off(i / KE, (i % KE) * 2)) = __int2half_rn(v);
    }
    for (int i = t; i < N * KE; i += blockDim.x) {
        const int v = val(blockIdx.x * 7919u + 99991u * i + 17, mode, vmax);
        iB[i / KE][i % KE] = v;
        *reinterpret_cast<__half*>(sB + cm_off(i / KE, (i % KE) * 2)) = __int2half_rn(v);
    }
    tc::fence_proxy_async_smem();
    if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
    if (w == 0) tc::tmem_alloc<64>(&tbase);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tm = tbase;
    if (t == 0) {
        const uint32_t idesc = tc::idesc_f16f16_f32(M, N);
        for (int ks = 0; ks < KB / 32; ++ks) {
            const uint64_t ad = tc::smem_desc(tc::smem_u32(sA) + ks * 256, 128, (KB / 16) * 128);
            const uint64_t bd = tc::smem_desc(tc::smem_u32(sB) + ks * 256, 128, (KB / 16) * 128);
            tc::mma_f16(tm, ad, bd, idesc, ks > 0);
        }
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::tc_fence_after();
    unsigned long long nb = 0;
    for (int c = 0; c < N; c += 16) {
        uint32_t v[16];
        tc::tmem_ld16(tm + ((uint32_t)(32 * w) << 16) + c, v);
        tc::tmem_wait_ld(v);
        const int m = 32 * w + (t & 31);
        for (int j = 0; j < 16; ++j) {
            long long s = 0;
            for (int kk = 0; kk < KE; ++kk) s += (long long)iA[m][kk] * iB[c + j][kk];
            if ((double)__uint_as_float(v[j]) != (double)s) ++nb;
        }
    }
    atomicAdd(bad, nb);
    atomicAdd(total, (unsigned long long)(N));
    tc::tc_fence_before();
    __syncthreads();
    if (w == 0) tc::tmem_dealloc<64>(tm);
}
int main() {
    unsigned long long *bad, *tot;
    cudaMallocManaged(&bad, 8); cudaMallocManaged(&tot, 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (M + N) * KB);
    for (int vmax : {255, 362, 400, 512, 1024, 2047}) {
        *bad = 0; *tot = 0;
        k<<<4096, 128, (M + N) * KB>>>(vmax, bad, tot);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
        printf("vmax %4d (64*vmax^2 = %.3g vs 2^24 = %.3g): %llu mismatches of %llu dot products\n",
               vmax, 64.0 * vmax * vmax, 16777216.0, *bad, *tot);
    }
    return 0;
}
