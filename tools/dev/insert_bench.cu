// Dev microbenchmark: cycles per sorted-list insertion round (KP = 32 keys per lane) with
// 1 or 2 warps per SMSP.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 insert_bench.cu
#include <cstdio>
#include <cstdint>
template <int N>
__device__ __forceinline__ void ins(uint32_t (&L)[N], uint32_t x) {
#pragma unroll
    for (int i = N - 1; i >= 1; --i) L[i] = min(L[i], max(L[i - 1], x));
    L[0] = min(L[0], x);
}
template <int N>
__device__ __forceinline__ void ins_split(uint32_t (&L)[N], uint32_t x) {
    uint32_t m[N];
#pragma unroll
    for (int i = 1; i < N; ++i) m[i] = max(L[i - 1], x);
#pragma unroll
    for (int i = 1; i < N; ++i) L[i] = min(L[i], m[i]);
    L[0] = min(L[0], x);
}
// two keys x <= y at once: C[k] = min(A[k], max(A[k-1], x), max(A[k-2], y))  (3 ops / element)
template <int N>
__device__ __forceinline__ void ins2(uint32_t (&L)[N], uint32_t x, uint32_t y) {
    const uint32_t lo = min(x, y), hi = max(x, y);
#pragma unroll
    for (int i = N - 1; i >= 2; --i) L[i] = __vimin3_u32(L[i], max(L[i - 1], lo), max(L[i - 2], hi));
    L[1] = __vimin3_u32(L[1], max(L[0], lo), hi);
    L[0] = min(L[0], lo);
}
template <int MODE>
__global__ void k(uint32_t* out, long long* cyc, int rounds) {
    uint32_t L[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) L[i] = 0xffffffffu - (31 - i);
    uint32_t s = threadIdx.x * 2654435761u + 12345u;
    __syncthreads();
    long long t0 = clock64();
    for (int q = 0; q < rounds; ++q) {
        s ^= s << 13; s ^= s >> 17; s ^= s << 5;
        if (MODE == 0) ins<32>(L, s);
        else if (MODE == 1) ins_split<32>(L, s);
        else { const uint32_t t = s * 2654435761u; ins2<32>(L, s, t); }
    }
    long long t1 = clock64();
    uint32_t acc = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) acc += L[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
    uint32_t* out; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 4); cudaMalloc(&cyc, 148 * 8);
    long long h[148];
    for (int mode = 0; mode < 3; mode += 2)
        for (int warps : {4, 8, 12}) {
            const int rounds = 4096;
            for (int rep = 0; rep < 2; ++rep) {
                if (mode == 0) k<0><<<148, 32 * warps>>>(out, cyc, rounds);
                else k<2><<<148, 32 * warps>>>(out, cyc, rounds);
            }
            cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
            printf("mode %d warps/SM %2d: %.1f cycles per round per warp (%s)\n", mode, warps,
                   (double)h[0] / rounds, mode == 0 ? "1 key/round" : "2 keys/round");
        }
    return 0;
}
