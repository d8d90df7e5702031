// Dev check: tcgen05.mma kind::f16 with the A operand in tensor memory (written by tcgen05.st,
// lane m = row m, column c = K elements 2c, 2c+1) and B in shared memory (K-major canonical).
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include "../../paper_2103_10765_b200/csrc/tc_ptx.cuh"
using namespace gbm3d;
constexpr int M = 128, N = 64, KE = 64, KB = KE * 2;
__device__ __forceinline__ int cm_off(int row, int kbyte) {
    return (row >> 3) * (KB / 16) * 128 + (kbyte >> 4) * 128 + (row & 7) * 16 + (kbyte & 15);
}
__device__ uint32_t hash(uint32_t x) { x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16; return x; }
__global__ void k(int vmax, unsigned long long* bad, unsigned long long* total) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* sB = sm;
    __shared__ __align__(8) uint64_t bar;
    __shared__ uint32_t tbase;
    __shared__ short iA[M][KE + 1];
    __shared__ short iB[N][KE + 1];
    const int t = threadIdx.x, w = t >> 5, lane = t & 31;
    for (int i = t; i < M * KE; i += blockDim.x) iA[i / KE][i % KE] = (int)(hash(blockIdx.x * 1000003u + i) % (2 * vmax + 1)) - vmax;
    for (int i = t; i < N * KE; i += blockDim.x) {
        const int v = (int)(hash(blockIdx.x * 7919u + 99991u * i + 17) % (2 * vmax + 1)) - vmax;
        iB[i / KE][i % KE] = v;
        *reinterpret_cast<__half*>(sB + cm_off(i / KE, (i % KE) * 2)) = __int2half_rn(v);
    }
    tc::fence_proxy_async_smem();
    if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_mbar_init(); }
    if (w == 0) tc::tmem_alloc<128>(&tbase);
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    const uint32_t tm = tbase;
    const uint32_t ta = tm + 64;  // A at columns 64..95
    {
        const int m = 32 * w + lane;
        uint32_t r[32];
        for (int c = 0; c < 32; ++c) {
            const __half2 h = __halves2half2(__int2half_rn(iA[m][2 * c]), __int2half_rn(iA[m][2 * c + 1]));
            r[c] = *reinterpret_cast<const uint32_t*>(&h);
        }
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(ta + ((uint32_t)(32 * w) << 16)),
            "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
            "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
            "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
            "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc::tc_fence_before();
    __syncthreads();
    tc::tc_fence_after();
    if (t == 0) {
        const uint32_t idesc = tc::idesc_f16f16_f32(M, N);
        for (int ks = 0; ks < KB / 32; ++ks) {
            const uint64_t bd = tc::smem_desc(tc::smem_u32(sB) + ks * 256, 128, (KB / 16) * 128);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
                "r"(ta + ks * 8), "l"(bd), "r"(idesc), "r"(ks)
                : "memory");
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
        const int m = 32 * w + lane;
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
    if (w == 0) tc::tmem_dealloc<128>(tm);
}
int main() {
    unsigned long long *bad, *tot;
    cudaMallocManaged(&bad, 8); cudaMallocManaged(&tot, 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, N * KB);
    for (int vmax : {3, 255, 362}) {
        *bad = 0; *tot = 0;
        k<<<1024, 128, N * KB>>>(vmax, bad, tot);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
        printf("A in TMEM, vmax %4d: %llu mismatches of %llu dot products\n", vmax, *bad, *tot);
    }
    return 0;
}
