// Dev check of the tcgen05 kind::i8 wrappers (descriptors, TMEM layout): D = A * B^T for
// u8 A[128][64], B[64][64] in the canonical K-major no-swizzle layout, vs a host loop.
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>
#include "../../paper_2103_10765_b200/csrc/tc_ptx.cuh"
using namespace gbm3d;

constexpr int M = 128, N = 64, KB = 64;  // K in bytes
__device__ __forceinline__ int cm_off(int row, int k) {  // canonical K-major offset
    return (row >> 3) * (KB / 16) * 128 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
}
__global__ void k_mma(const uint8_t* A, const uint8_t* B, int32_t* D) {
    __shared__ __align__(128) uint8_t sA[M * KB];
    __shared__ __align__(128) uint8_t sB[N * KB];
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    const int t = threadIdx.x, w = t >> 5;
    for (int i = t; i < M * KB; i += blockDim.x) sA[cm_off(i / KB, i % KB)] = A[i];
    for (int i = t; i < N * KB; i += blockDim.x) sB[cm_off(i / KB, i % KB)] = B[i];
    tc::fence_proxy_async_smem();
    if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
    if (w == 0) tc::tmem_alloc<64>(&tbase);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tm = tbase;
    if (t == 0) {
        const uint32_t idesc = tc::idesc_u8u8_s32(M, N);
        for (int ks = 0; ks < KB / 32; ++ks) {
            const uint64_t ad = tc::smem_desc(tc::smem_u32(sA) + ks * 256, 128, (KB / 16) * 128);
            const uint64_t bd = tc::smem_desc(tc::smem_u32(sB) + ks * 256, 128, (KB / 16) * 128);
            tc::mma_i8(tm, ad, bd, idesc, ks > 0);
        }
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::tc_fence_after();
    for (int c = 0; c < N; c += 16) {
        uint32_t v[16];
        tc::tmem_ld16(tm + ((uint32_t)(32 * w) << 16) + c, v);
        tc::tmem_wait_ld(v);
        for (int j = 0; j < 16; ++j) D[(32 * w + (t & 31)) * N + c + j] = (int32_t)v[j];
    }
    tc::tc_fence_before();
    __syncthreads();
    if (w == 0) tc::tmem_dealloc<64>(tm);
}
int main() {
    uint8_t *A, *B; int32_t* D;
    cudaMallocManaged(&A, M * KB); cudaMallocManaged(&B, N * KB); cudaMallocManaged(&D, M * N * 4);
    srand(1);
    for (int i = 0; i < M * KB; ++i) A[i] = rand() & 255;
    for (int i = 0; i < N * KB; ++i) B[i] = rand() & 255;
    k_mma<<<1, 128>>>(A, B, D);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    int bad = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            int32_t s = 0;
            for (int k = 0; k < KB; ++k) s += (int32_t)A[m * KB + k] * (int32_t)B[n * KB + k];
            if (s != D[m * N + n]) { if (bad < 5) printf("m%d n%d got %d want %d\n", m, n, D[m * N + n], s); ++bad; }
        }
    printf("mma_i8 test: %s (%d bad)\n", bad ? "FAIL" : "OK", bad);
    return bad != 0;
}
