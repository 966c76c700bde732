// Microbenchmark: FP64 DADD/DMUL/DFMA and FP32 FFMA dependent-chain throughput,
// plus F2F conversions.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void k(double* out, int iters, double a) {
    double acc[8];
    for (int i = 0; i < 8; ++i) acc[i] = threadIdx.x * 1e-9 + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (OP == 0) acc[i] = __dadd_rn(acc[i], a);
            if (OP == 1) acc[i] = __dmul_rn(acc[i], a);
            if (OP == 2) acc[i] = fma(acc[i], a, 1e-9);
            if (OP == 3) acc[i] = (double)(float)acc[i] + a;
        }
    }
    double s = 0; for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 1.2345) out[0] = s;
}
int main() {
    double* o; cudaMalloc(&o, 8);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const char* names[4] = {"DADD", "DMUL", "DFMA", "F2F+DADD"};
    for (int op = 0; op < 4; ++op) {
        int blocks = 148 * 8, threads = 256, iters = 2048; float best = 1e9;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(a);
            if (op == 0) k<0><<<blocks, threads>>>(o, iters, 1.0000001);
            if (op == 1) k<1><<<blocks, threads>>>(o, iters, 1.0000001);
            if (op == 2) k<2><<<blocks, threads>>>(o, iters, 1.0000001);
            if (op == 3) k<3><<<blocks, threads>>>(o, iters, 1.0000001);
            cudaEventRecord(b); cudaEventSynchronize(b); float t; cudaEventElapsedTime(&t, a, b); if (t < best) best = t;
        }
        double ops = (double)blocks * threads * iters * 8;
        printf("%-10s %.2f Tops/s  (%.1f ops/clk/SM at 1.965 GHz)\n", names[op], ops / best / 1e9, ops / best / 1e9 * 1e12 / 148 / 1.965e9);
    }
}
