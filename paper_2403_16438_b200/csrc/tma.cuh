// TMA (cp.async.bulk.tensor) + mbarrier helpers for sm_100a, and the host
// side tensor-map encoder (driver entry point, no libcuda link dependency).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace vb {

// Frames [T][H][W] of u16/f32 as a 3-D tensor {W, H, T} with a box of
// {bw, bh, 1}.  Returns false (and the kernels fall back to plain loads) when
// the layout violates TMA's 16-byte alignment rules.
// bt > 1: boxes of bt consecutive frames ({bw, bh, bt}).
bool make_frames_tmap(CUtensorMap* map, const void* base, int dtype, int64_t t, int h, int w, int bh, int bw,
                      int bt = 1);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(smem_u32(bar)), "r"(phase)
            : "memory");
    } while (!done);
}

// 3-D tile load {x, y, z} -> shared memory, completion counted on `bar`.
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// 1-D bulk copy global -> shared (bytes and both addresses 16-byte multiples),
// completion counted on `bar`.
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// u16 -> f32 minus an integer centre, exactly, on the FMA pipe instead of the
// (16/clk/SM) conversion unit: 2^23 + v is an exact float; subtracting
// 2^23 + c (also exact for |c| < 2^23) is exact by Sterbenz.
__device__ __forceinline__ float u16_minus(uint32_t v, float magic_c /* 8388608 + c */) {
    return __fsub_rn(__uint_as_float(0x4B000000u | v), magic_c);
}

}  // namespace vb
