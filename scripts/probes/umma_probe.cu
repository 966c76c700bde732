// Probe: one tcgen05.mma kind::tf32 (M=128, N=16 or 64, K=8) with K-major
// SWIZZLE_NONE shared-memory descriptors, accumulator in TMEM, read back with
// tcgen05.ld 32x32b -- checks the descriptor / layout conventions the U-Net
// kernels use.  nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o umma_probe umma_probe.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (Blackwell)
    return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4)        // D f32
         | (2u << 7)        // A tf32
         | (2u << 10)       // B tf32
         | ((uint32_t)(N >> 3) << 17)
         | ((uint32_t)(M >> 4) << 24);
}

template <int N>
__global__ void probe(const float* A, const float* B, float* D, int swap) {
    constexpr int M = 128, K = 8;
    __shared__ __align__(1024) float sA[M * K];
    __shared__ __align__(1024) float sB[N * K];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // K-major interleave: (m, k) -> (k/4)*LBO + (m/8)*SBO + (m%8)*16 + (k%4)*4 bytes
    const uint32_t SBO = 128, LBO_A = M * 16, LBO_B = N * 16;
    for (int i = tid; i < M * K; i += blockDim.x) {
        const int m = i / K, k = i % K;
        const uint32_t off = (k / 4) * LBO_A + (m / 8) * SBO + (m % 8) * 16 + (k % 4) * 4;
        sA[off / 4] = A[m * K + k];
    }
    for (int i = tid; i < N * K; i += blockDim.x) {
        const int n = i / K, k = i % K;
        const uint32_t off = (k / 4) * LBO_B + (n / 8) * SBO + (n % 8) * 16 + (k % 4) * 4;
        sB[off / 4] = B[n * K + k];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                     "n"(N < 32 ? 32 : N));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic smem writes -> async proxy
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    if (tid == 0) {
        const uint32_t la = swap ? SBO : LBO_A, sa = swap ? LBO_A : SBO;
        const uint32_t lb = swap ? SBO : LBO_B, sb = swap ? LBO_B : SBO;
        const uint64_t da = sdesc(smem_u32(sA), la, sa), db = sdesc(smem_u32(sB), lb, sb);
        const uint32_t id = idesc_tf32(M, N);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(id), "r"(0));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&bar)));
    }
    // wait for the MMA
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                : "=r"(done)
                : "r"(smem_u32(&bar)));
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // warp w reads TMEM lanes 32w..32w+31; 16 columns at a time
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        const int m = warp * 32 + lane;
        for (int j = 0; j < 16; ++j) D[m * N + c0 + j] = __uint_as_float(v[j]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(N < 32 ? 32 : N));
}

template <int N>
int run(int swap) {
    const int M = 128, K = 8;
    float hA[M * K], hB[N * K], hD[M * N];
    srand(1);
    for (int i = 0; i < M * K; ++i) hA[i] = (float)((rand() % 17) - 8) / 4.0f;  // exact in tf32
    for (int i = 0; i < N * K; ++i) hB[i] = (float)((rand() % 13) - 6) / 2.0f;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, sizeof hA);
    cudaMalloc(&dB, sizeof hB);
    cudaMalloc(&dD, sizeof hD);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0, sizeof hD);
    probe<N><<<1, 128>>>(dA, dB, dD, swap);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("N=%d swap=%d: CUDA error %s\n", N, swap, cudaGetErrorString(e));
        return 1;
    }
    cudaMemcpy(hD, dD, sizeof hD, cudaMemcpyDeviceToHost);
    int bad = 0;
    double maxd = 0;
    for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
            double s = 0;
            for (int k = 0; k < K; ++k) s += (double)hA[m * K + k] * hB[n * K + k];
            const double d = fabs(s - hD[m * N + n]);
            maxd = fmax(maxd, d);
            bad += d > 1e-6;
        }
    printf("N=%d swap=%d: %d / %d wrong, max diff %g  (D[0]=%g D[last]=%g)\n", N, swap, bad, M * N, maxd, hD[0],
           hD[M * N - 1]);
    return bad != 0;
}

int main() {
    int rc = 0;
    rc |= run<16>(0);
    rc |= run<64>(0);
    if (rc) {
        run<16>(1);
        run<64>(1);
    }
    return rc;
}
