// Standalone reproduction of the stats-kernel TMA pattern (development aid).
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include "../../paper_2403_16438_b200/csrc/tma.cuh"

__global__ void k(const __grid_constant__ CUtensorMap tmap, int bw, int bh, int bhc, int x0, int y0, float* out, int smem_pad) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) { vb::mbar_init(&bar, 1); vb::fence_mbar_init(); }
    __syncthreads();
    if (threadIdx.x == 0) {
        int nck = (bh + bhc - 1) / bhc;
        vb::mbar_expect_tx(&bar, bw * bhc * nck * 4);
        for (int c = 0; c < nck; ++c) vb::tma_load_3d(smem + (size_t)c * bhc * bw * 4, &tmap, x0, y0 + c * bhc, 0, &bar);
    }
    vb::mbar_wait(&bar, 0);
    float s = 0; for (int i = threadIdx.x; i < bw * bh; i += blockDim.x) s += ((float*)smem)[i];
    atomicAdd(out, s);
}
int main(int argc, char** argv) {
    int W = 128, H = 128;
    float* d; cudaMalloc(&d, W * H * 4); cudaMemset(d, 0, W * H * 4);
    float* out; cudaMalloc(&out, 4);
    void* fn = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    struct C { int bw, bh, bhc, x0, y0, smem; } cs[] = {
        {64, 32, 32, 42, 0, 40000}, {64, 32, 32, 40, 0, 40000}, {104, 32, 32, 40, 0, 40000}, {64, 32, 32, 41, 0, 40000},
        {64, 32, 32, 44, 0, 40000}, {64, 32, 32, 1, 0, 40000}, {104, 32, 32, 4, 0, 40000}, {104, 32, 32, 24, 0, 40000}};
    int only = argc > 1 ? atoi(argv[1]) : -1; int idx = -1;
    for (auto c : cs) { ++idx; if (only >= 0 && idx != only) continue;
        CUtensorMap m; memset(&m, 0, sizeof m);
        cuuint64_t dims[3] = {(cuuint64_t)W, (cuuint64_t)H, 1}; cuuint64_t str[2] = {(cuuint64_t)W * 4, (cuuint64_t)W * H * 4};
        cuuint32_t box[3] = {(cuuint32_t)c.bw, (cuuint32_t)c.bhc, 1}, es[3] = {1, 1, 1};
        CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, c.smem);
        k<<<1, 256, c.smem>>>(m, c.bw, c.bh, c.bhc, c.x0, c.y0, out, 0);
        cudaError_t e = cudaDeviceSynchronize();
        printf("bw=%d bh=%d bhc=%d x0=%d y0=%d smem=%d encode=%d -> %s\n", c.bw, c.bh, c.bhc, c.x0, c.y0, c.smem, (int)r, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
    }
}
