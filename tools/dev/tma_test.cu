// Dev: standalone check of the 3-D TMA box load used by match_tc16 (int16 image, 72 x PR box).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cstdlib>
typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                        const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                        CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tm, int x, int y, int z, int16_t* out, int PR, int mode, int BX) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) uint64_t bar;
    int16_t* box = (int16_t*)(sm + 1024);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(BX * PR * 2) : "memory");
        if (mode == 0)
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(sa(box)), "l"((uint64_t)&tm), "r"(x), "r"(y), "r"(z), "r"(sa(&bar)) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                         ::"r"(sa(box)), "l"((uint64_t)&tm), "r"(x), "r"(y), "r"(z), "r"(sa(&bar)) : "memory");
    }
    uint32_t ok = 0;
    while (!ok) {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}" : "=r"(ok) : "r"(sa(&bar)) : "memory");
    }
    for (int i = threadIdx.x; i < BX * PR; i += blockDim.x) out[i] = box[i];
}
int main(int argc, char** argv) {
    const int W = 64, H = 64, B = 1; const int BX = atoi(argv[1]), PR = atoi(argv[2]); const int X0 = atoi(argv[3]), Y0 = atoi(argv[4]);
    std::vector<int16_t> h(W * H * B);
    for (int i = 0; i < W * H * B; ++i) h[i] = (int16_t)(i % 1000 - 300);
    int16_t *d, *o;
    cudaMalloc(&d, h.size() * 2);
    cudaMalloc(&o, 256 * 256 * 2);
    cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    CUtensorMap tm;
    cuuint64_t dims[3] = {W, H, B}, str[2] = {W * 2, (cuuint64_t)W * H * 2};
    cuuint32_t box[3] = {(cuuint32_t)BX, (cuuint32_t)PR, 1}, es[3] = {1, 1, 1};
    CUresult r = ((Enc)f)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT16, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    for (int mode = 0; mode < 2; ++mode) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 + BX * PR * 2);
        k<<<1, 128, 1024 + BX * PR * 2>>>(tm, X0, Y0, 0, o, PR, mode, BX);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d: %s\n", mode, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        std::vector<int16_t> ob(BX * PR);
        cudaMemcpy(ob.data(), o, ob.size() * 2, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int yy = 0; yy < PR; ++yy)
            for (int xx = 0; xx < BX; ++xx) {
                const int gy = yy + Y0, gx = xx + X0;
                const int16_t e2 = (gy >= 0 && gy < H && gx >= 0 && gx < W) ? h[gy * W + gx] : 0;
                bad += ob[yy * BX + xx] != e2;
            }
        printf("mode %d mismatches %d\n", mode, bad);
    }
    return 0;
}
