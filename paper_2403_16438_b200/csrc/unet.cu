// Summary normalisation + lightweight U-Net tiles, sm_100a.
//
// Reference (paths under /root/reference/pkg/src/voltseg):
//   normalize_pair   unet.py:186-196  (1st/99th percentiles, numpy "linear"
//                    method; (x - p1) / (p99 - p1) in float64, clipped, f32)
//   forward_batch    unet.py:154-178  (enc 16/32/64, two 3x3 conv + ReLU per
//                    level, 2x2 max-pool, nearest upsample + skip concat,
//                    1x1 conv + sigmoid; zero padding per 64x64 patch)
//   tile_and_merge   unet.py:212-245  (64x64 tiles at `stride`, last tile
//                    flush to the edge, numpy "reflect" pad for small frames,
//                    tent-weighted float64 blend, clip)
//
// B200 design: one CTA computes a 16x16 output tile of one patch for ALL
// output channels (<= 64 accumulators per thread), staging 8 input channels
// x 18x18 halo and their [ci][tap][cout] weights in shared memory; weights
// are read as float4 broadcasts.  Input staging fuses the layer's source:
// the normalised summary images at the tile origin (first layer, no patch
// copy), a plain NCHW tensor, or nearest-upsample(low) ++ skip (decoder).
// Epilogues fuse ReLU, the 2x2 max-pool (warp shuffles) and the final 1x1
// conv + sigmoid.  FP32 throughout (the reference is float32 numpy; parity
// target <= 1e-4 absolute, test_acceptance.py:152-163).
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "tma.cuh"
#include "vb.cuh"

namespace vb {

namespace {

constexpr int kPatch = 64;
constexpr int kCK = 8;  // input channels staged per round

// numpy float32 key order (same as the median's fkey)
__device__ __forceinline__ uint32_t fkey_u(float f) {
    const uint32_t u = __float_as_uint(f);
    return u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv_u(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k ^ 0x80000000u) : ~k);
}

struct ConvArgs {
    int n, h, w, cin, cout;
    // source of input channels [0, c0): mode 0 NCHW [n][c0][h][w]; mode 1 nearest
    // upsample of [n][c0][h/2][w/2]; mode 2 image tiles img[c0][ih][iw] at origins
    const float* x0;
    int c0, mode;
    const float* x1;  // channels [c0, cin): skip [n][cin-c0][h][w] (concat) or null
    const int2* origins;  // mode 2: patch (x, y) origins in the image
    int ih, iw;
    int64_t img_stride;  // mode 2: floats between consecutive images (blocks)
    int tiles_per_img;   // mode 2: patches per image
    const float* wt;     // [cout][cin][3][3]
    const float* wtc;    // tensor-core copy: [ceil(cin/8)][hi, lo][tap][half][cout][4] (3xTF32 split)
    const float* bias;   // [cout]
    float* out;          // [n][cout][h][w] or null
    float* pooled;       // [n][cout][h/2][w/2] or null
    const float* w1;     // final 1x1 kernel [cout] (cout -> 1) or null
    const float* b1;     // final 1x1 bias [1]
    float* prob;         // [n][h][w] sigmoid(1x1) or null
    int dbg;             // experiment build: 1 skip the MMAs, 2 skip the activation/weight staging
};

// Register-blocked tile geometry per output width: every thread owns a
// horizontal strip of 4 pixels x 16 output channels (64 accumulators); per
// (input channel, kernel row) it loads the 6 samples its 3 taps x 4 pixels
// need and 3 x 16 weights (float4 broadcasts, warps are uniform in their
// channel group): 192 FFMA per 18 shared loads.
//   COUT 16: 32x32 tile, 1 channel group;  COUT 32: 16x32 tile, 2 groups;
//   COUT 64: 16x16 tile, 4 groups  -> 256 threads each.
template <int COUT>
struct ConvGeom {
    static constexpr int kGroups = COUT / 16;
    static constexpr int TW = COUT == 64 ? 16 : 32;
    static constexpr int TH = COUT == 16 ? 32 : 16;
    static constexpr int kStrips = TW / 4;
    static constexpr int kPx = TH * kStrips;  // pixel strips per tile
    static constexpr int kThreads = kPx * kGroups;
    static constexpr int IW = TW + 2 + 1;     // padded input row
    static_assert(kThreads == 256, "256 threads per conv CTA");
};

__device__ __forceinline__ void cp_async4(void* dst, const float* src, bool valid) {
    // 4-byte global -> shared copy; src-size 0 zero-fills (padding / absent channels)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

template <int COUT>
__global__ void __launch_bounds__(256) conv3x3_kernel(ConvArgs a) {
    using G = ConvGeom<COUT>;
    // double-buffered stages: chunk k+1's cp.async copies fly while chunk k computes
    extern __shared__ __align__(16) float conv_smem[];
    using InTile = float[kCK][G::TH + 2][G::IW];
    float (*s_w)[kCK * 9 * COUT] = reinterpret_cast<float (*)[kCK * 9 * COUT]>(conv_smem);  // [ci][tap][cout]
    InTile* s_in = reinterpret_cast<InTile*>(conv_smem + 2 * kCK * 9 * COUT);
    const int tid = threadIdx.x;
    const int cg = tid / G::kPx;          // channel group (warp-uniform)
    const int g = tid - cg * G::kPx;
    const int ty = g / G::kStrips, sx = (g % G::kStrips) * 4;
    const int tiles_x = a.w / G::TW;
    const int tile = blockIdx.x, n = blockIdx.y;
    const int oy0 = (tile / tiles_x) * G::TH, ox0 = (tile % tiles_x) * G::TW;
    float acc[4][16];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int c = 0; c < 16; ++c) acc[j][c] = 0.0f;
    const int hw = a.h * a.w;
    auto stage = [&](int buf, int c0) {
        const int nck = min(kCK, a.cin - c0);
        constexpr int kIn = kCK * (G::TH + 2) * (G::TW + 2);
        for (int i = tid; i < kIn; i += 256) {
            const int ci = i / ((G::TH + 2) * (G::TW + 2));
            const int r = i % ((G::TH + 2) * (G::TW + 2));
            const int yy = r / (G::TW + 2), xx = r % (G::TW + 2);
            const int y = oy0 + yy - 1, x = ox0 + xx - 1;
            const int c = c0 + ci;
            const bool valid = ci < nck && y >= 0 && y < a.h && x >= 0 && x < a.w;
            const float* src = a.wt;  // any valid address when zero-filling
            if (valid) {
                if (c < a.c0) {
                    if (a.mode == 0) {
                        src = a.x0 + ((int64_t)n * a.c0 + c) * hw + y * a.w + x;
                    } else if (a.mode == 1) {
                        const int lw = a.w >> 1, lh = a.h >> 1;
                        src = a.x0 + ((int64_t)n * a.c0 + c) * lh * lw + (y >> 1) * lw + (x >> 1);
                    } else {
                        const int img = n / a.tiles_per_img;
                        const int2 o = a.origins[n];
                        src = a.x0 + (int64_t)img * a.img_stride + ((int64_t)c * a.ih + o.y + y) * a.iw + o.x + x;
                    }
                } else {
                    src = a.x1 + ((int64_t)n * (a.cin - a.c0) + (c - a.c0)) * hw + y * a.w + x;
                }
            }
            cp_async4(&s_in[buf][ci][yy][xx], src, valid);
        }
        for (int i = tid; i < kCK * 9 * COUT; i += 256) {
            const int co = i % COUT, r = i / COUT;
            const int ci = r / 9, tap = r % 9;
            const bool valid = ci < nck && co < a.cout;
            cp_async4(&s_w[buf][i], valid ? a.wt + ((int64_t)co * a.cin + c0 + ci) * 9 + tap : a.wt, valid);
        }
        cp_async_commit();
    };
    stage(0, 0);
    int buf = 0;
    for (int c0 = 0; c0 < a.cin; c0 += kCK, buf ^= 1) {
        const int nck = min(kCK, a.cin - c0);
        if (c0 + kCK < a.cin) {
            stage(buf ^ 1, c0 + kCK);
            cp_async_wait<1>();
        } else {
            cp_async_wait<0>();
        }
        __syncthreads();
        for (int ci = 0; ci < nck; ++ci) {
#pragma unroll
            for (int ky = 0; ky < 3; ++ky) {
                float xin[6];
#pragma unroll
                for (int j = 0; j < 6; ++j) xin[j] = s_in[buf][ci][ty + ky][sx + j];
#pragma unroll
                for (int kx = 0; kx < 3; ++kx) {
                    const float4* wv = reinterpret_cast<const float4*>(&s_w[buf][(ci * 9 + ky * 3 + kx) * COUT + cg * 16]);
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const float4 w4 = wv[q];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float xv = xin[j + kx];
                            acc[j][4 * q] = fmaf(xv, w4.x, acc[j][4 * q]);
                            acc[j][4 * q + 1] = fmaf(xv, w4.y, acc[j][4 * q + 1]);
                            acc[j][4 * q + 2] = fmaf(xv, w4.z, acc[j][4 * q + 2]);
                            acc[j][4 * q + 3] = fmaf(xv, w4.w, acc[j][4 * q + 3]);
                        }
                    }
                }
            }
        }
        __syncthreads();  // buffer `buf` is restaged two chunks later
    }
    const int y = oy0 + ty, x = ox0 + sx;
#pragma unroll
    for (int c = 0; c < 16; ++c) {
        const int co = cg * 16 + c;
        const float b = co < a.cout ? __ldg(a.bias + co) : 0.0f;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j][c] = co < a.cout ? fmaxf(__fadd_rn(acc[j][c], b), 0.0f) : 0.0f;
    }
    if (a.out) {
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            const int co = cg * 16 + c;
            if (co < a.cout)
                *reinterpret_cast<float4*>(a.out + ((int64_t)n * a.cout + co) * hw + y * a.w + x) =
                    make_float4(acc[0][c], acc[1][c], acc[2][c], acc[3][c]);
        }
    }
    if (a.pooled) {  // 2x2 blocks: pixel pairs inside the strip, row pairs = lanes l, l ^ kStrips
        const int ph = a.h >> 1, pw = a.w >> 1;
#pragma unroll
        for (int c = 0; c < 16; ++c) {
            float m0 = fmaxf(acc[0][c], acc[1][c]), m1 = fmaxf(acc[2][c], acc[3][c]);
            m0 = fmaxf(m0, __shfl_xor_sync(0xffffffffu, m0, G::kStrips));
            m1 = fmaxf(m1, __shfl_xor_sync(0xffffffffu, m1, G::kStrips));
            const int co = cg * 16 + c;
            if (co < a.cout && !(ty & 1))
                *reinterpret_cast<float2*>(a.pooled + ((int64_t)n * a.cout + co) * ph * pw + (y >> 1) * pw + (x >> 1)) =
                    make_float2(m0, m1);
        }
    }
    if (a.prob) {  // final 1x1 conv + sigmoid (unet.py:129-134, :149-150); COUT 16 = one group
        float4 pv;
        float* pp = &pv.x;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float sum = 0.0f;
#pragma unroll
            for (int c = 0; c < 16; ++c)
                if (c < a.cout) sum = fmaf(acc[j][c], __ldg(a.w1 + c), sum);
            sum = __fadd_rn(sum, __ldg(a.b1));
            pp[j] = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-sum)));
        }
        *reinterpret_cast<float4*>(a.prob + (int64_t)n * hw + y * a.w + x) = pv;
    }
}

template <int COUT>
int launch_conv(const ConvArgs& a, cudaStream_t s) {
    using G = ConvGeom<COUT>;
    if (a.h % G::TH || a.w % G::TW) return fail(VB_EINVAL, "U-Net tile size");
    if (a.prob && COUT != 16) return fail(VB_EINVAL, "fused output conv needs one channel group");
    dim3 grid((unsigned)((a.h / G::TH) * (a.w / G::TW)), (unsigned)a.n);
    const size_t smem = sizeof(float) * 2 * ((size_t)kCK * 9 * COUT + (size_t)kCK * (G::TH + 2) * G::IW);
    VB_CUDA(cudaFuncSetAttribute(conv3x3_kernel<COUT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    {
        ProfScope ps(kProfOther, s);
        conv3x3_kernel<COUT><<<grid, 256, smem, s>>>(a);
    }
    VB_LAUNCHED();
    return VB_OK;
}

// ---------------------------------------------------------- tcgen05 path
// Implicit-GEMM 3x3 conv on the 5th-generation tensor cores, 3xTF32 split so
// the float32 parity bound holds (a*b ~ ah*bh + ah*bl + al*bh, error ~2^-22).
// A CTA (4 warps) owns a 16x16 output tile of one patch = two M=128 tiles of
// 16 rows x 8 columns; D[128 px][N = cout] accumulates in TMEM.  Per chunk of
// 8 input channels the padded 18x18 input tile is staged K-major without any
// im2col copy: stored as [channel half][padded row][padded col][4 channels],
// the A operand of tap (ky, kx) and column block cb is just a descriptor at
// pixel (ky, kx + 8 cb) with SBO = one padded row and LBO = one channel-half
// plane (core matrix = 8 consecutive pixels of one output row).  Weights of
// the chunk are staged [tap][half][cout][4].  One elected thread issues
// 9 taps x 2 blocks x 3 MMAs (M=128, N=cout, K=8) and commits to an mbarrier;
// the epilogue reads TMEM (tcgen05.ld 32x32b: warp w owns pixel rows
// 4w..4w+3) and fuses bias, ReLU, max-pool and the 1x1 + sigmoid.
constexpr int kTcTH = 16, kTcTW = 16, kTcCB = kTcTW / 8;
constexpr int kTcPH = kTcTH + 2, kTcPW = kTcTW + 2;
// bytes of one 4-channel plane, padded so the second channel-half plane starts
// 28 banks further: the staging stores of 8 channels x 4 rows per warp then
// hit 32 distinct banks
constexpr int kTcPlane = kTcPH * kTcPW * 16 + 48;

__device__ __forceinline__ uint64_t umma_sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);  // SWIZZLE_NONE, K-major
}
__host__ __device__ constexpr uint32_t umma_idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ float tf32_hi(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

template <int N>
__global__ void __launch_bounds__(128) conv3x3_tc_kernel(ConvArgs a) {
    constexpr int kWBytes = 9 * 2 * N * 16;           // weights of one chunk, one split
    constexpr int kCols = kTcCB * N < 32 ? 32 : kTcCB * N;
    extern __shared__ __align__(1024) unsigned char tc_smem[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar[2];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tiles_x = a.w / kTcTW;
    const int tile = blockIdx.x, n = blockIdx.y;
    const int oy0 = (tile / tiles_x) * kTcTH, ox0 = (tile % tiles_x) * kTcTW;
    const int hw = a.h * a.w;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                     "n"(kCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = tmem_base;
    const int nchunks = (a.cin + 7) / 8;
    // Input chunks are software-pipelined through registers: the padded rows
    // of chunk ch+1 are loaded (float4 interior, scalar halo) right after
    // chunk ch's MMAs are issued, so their global latency hides behind the
    // tensor cores; once those MMAs retire the rows are split hi / lo and
    // stored K-major.  Weights cp.async from their pre-split copy.
    constexpr int kRowsPerThread = (8 * kTcPH + 127) / 128;
    float rows[kRowsPerThread][kTcPW];
    auto load_rows = [&](int ch) {
        const int c0 = ch * 8;
#pragma unroll
        for (int k = 0; k < kRowsPerThread; ++k) {
            const int pr = tid + 128 * k;
#pragma unroll
            for (int j = 0; j < kTcPW; ++j) rows[k][j] = 0.0f;
            if (pr >= 8 * kTcPH) continue;
            const int ci = pr & 7, yy = pr >> 3;  // lanes: 8 channels x 4 rows (conflict-free stores)
            const int y = oy0 + yy - 1, c = c0 + ci;
            if (c >= a.cin || y < 0 || y >= a.h) continue;
            const float* src = nullptr;
            int step = 1;
            if (c < a.c0) {
                if (a.mode == 0) {
                    src = a.x0 + ((int64_t)n * a.c0 + c) * hw + (int64_t)y * a.w;
                } else if (a.mode == 1) {
                    const int lw = a.w >> 1, lh = a.h >> 1;
                    src = a.x0 + ((int64_t)n * a.c0 + c) * lh * lw + (int64_t)(y >> 1) * lw;
                    step = 2;  // nearest upsample: column x reads x / 2
                } else {
                    const int img = n / a.tiles_per_img;
                    const int2 o = a.origins[n];
                    src = a.x0 + (int64_t)img * a.img_stride + ((int64_t)c * a.ih + o.y + y) * a.iw + o.x;
                    step = 0;  // image tiles: arbitrary alignment
                }
            } else {
                src = a.x1 + ((int64_t)n * (a.cin - a.c0) + (c - a.c0)) * hw + (int64_t)y * a.w;
            }
            if (step == 1) {  // NCHW rows: ox0 % 16 == 0 and w % 16 == 0 -> aligned float4
                const float4* v4 = reinterpret_cast<const float4*>(src + ox0);
#pragma unroll
                for (int q = 0; q < kTcTW / 4; ++q) {
                    const float4 t = __ldg(v4 + q);
                    rows[k][1 + 4 * q] = t.x;
                    rows[k][2 + 4 * q] = t.y;
                    rows[k][3 + 4 * q] = t.z;
                    rows[k][4 + 4 * q] = t.w;
                }
                if (ox0 > 0) rows[k][0] = __ldg(src + ox0 - 1);
                if (ox0 + kTcTW < a.w) rows[k][kTcPW - 1] = __ldg(src + ox0 + kTcTW);
            } else if (step == 2) {  // nearest upsample: 8 low-res samples (two float4, each used twice) + halo
                const int lx0 = ox0 >> 1;  // a multiple of 8: aligned
                const float4* v4 = reinterpret_cast<const float4*>(src + lx0);
                const float4 t0 = __ldg(v4), t1 = __ldg(v4 + 1);
                const float lr[8] = {t0.x, t0.y, t0.z, t0.w, t1.x, t1.y, t1.z, t1.w};
#pragma unroll
                for (int j = 0; j < 8; ++j) rows[k][1 + 2 * j] = rows[k][2 + 2 * j] = lr[j];
                if (ox0 > 0) rows[k][0] = __ldg(src + lx0 - 1);
                if (ox0 + kTcTW < a.w) rows[k][kTcPW - 1] = __ldg(src + lx0 + kTcTW / 2);
            } else {
#pragma unroll
                for (int j = 0; j < kTcPW; ++j) {
                    const int x = ox0 + j - 1;
                    if (x >= 0 && x < a.w) rows[k][j] = __ldg(src + (step == 2 ? (x >> 1) : x));
                }
            }
        }
    };
    auto store_rows = [&]() {
        unsigned char* sb = tc_smem;
#pragma unroll
        for (int k = 0; k < kRowsPerThread; ++k) {
            const int pr = tid + 128 * k;
            if (pr >= 8 * kTcPH) continue;
            const int ci = pr & 7, yy = pr >> 3;
            unsigned char* dst = sb + (ci >> 2) * kTcPlane + yy * kTcPW * 16 + (ci & 3) * 4;
#pragma unroll
            for (int j = 0; j < kTcPW; ++j) {
                const float hi = tf32_hi(rows[k][j]);
                *reinterpret_cast<float*>(dst + j * 16) = hi;
                *reinterpret_cast<float*>(dst + 2 * kTcPlane + j * 16) = rows[k][j] - hi;
            }
        }
    };
    // the chunk's pre-split weights: one bulk copy issued by thread 0, completing on bar[1]
    auto fetch_w = [&](int ch) {
        if (tid == 0) {
            mbar_expect_tx(&bar[1], 2 * kWBytes);
            bulk_load(tc_smem + 4 * kTcPlane, a.wtc + (size_t)ch * (2 * kWBytes / 4), 2 * kWBytes, &bar[1]);
        }
    };
    uint32_t wph = 0;
    auto issue = [&](int ch) {
        const uint32_t sb = smem_u32(tc_smem);
        constexpr uint32_t idesc = umma_idesc_tf32(128, N);
        const uint32_t sbo_a = kTcPW * 16, lbo_a = kTcPlane;
        const uint32_t sbo_b = 128, lbo_b = N * 16;
#pragma unroll 1
        for (int tap = 0; tap < 9; ++tap) {
            const int ky = tap / 3, kx = tap % 3;
            const uint64_t bh = umma_sdesc(sb + 4 * kTcPlane + tap * 2 * N * 16, lbo_b, sbo_b);
            const uint64_t bl = umma_sdesc(sb + 4 * kTcPlane + kWBytes + tap * 2 * N * 16, lbo_b, sbo_b);
#pragma unroll
            for (int cb = 0; cb < kTcCB; ++cb) {
                const uint32_t a_off = (uint32_t)((ky * kTcPW + kx + 8 * cb) * 16);
                const uint64_t ah = umma_sdesc(sb + a_off, lbo_a, sbo_a);
                const uint64_t al = umma_sdesc(sb + 2 * kTcPlane + a_off, lbo_a, sbo_a);
                const uint32_t d = tmem + cb * N;
                umma_tf32(d, ah, bh, idesc, (ch > 0 || tap > 0) ? 1u : 0u);
                umma_tf32(d, ah, bl, idesc, 1u);
                umma_tf32(d, al, bh, idesc, 1u);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&bar[0])));
    };
#ifdef VB_EXPERIMENTS
    const int dbg = a.dbg;  // time the staging and the MMAs separately (scripts/ab_unet_dbg.sh)
#else
    constexpr int dbg = 0;
#endif
    uint32_t ph = 0;
    if (dbg != 2) load_rows(0);
    for (int ch = 0; ch < nchunks; ++ch) {
        if (ch > 0) {  // the previous chunk's MMAs have read the K-major planes and weights
            mbar_wait(&bar[0], ph);
            ph ^= 1u;
        }
        if (dbg != 2) {
            fetch_w(ch);
            store_rows();
            if (tid == 0) {  // only the MMA-issuing thread reads the weights (async proxy, after this wait)
                mbar_wait(&bar[1], wph);
                wph ^= 1u;
            }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;\n");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;\n");
        if (tid == 0) {
            if (dbg != 1)
                issue(ch);
            else
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(&bar[0])) : "memory");
        }
        if (ch + 1 < nchunks && dbg != 2) load_rows(ch + 1);  // in flight during this chunk's MMAs
    }
    mbar_wait(&bar[0], ph);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    // epilogue: warp w <-> TMEM lanes 32w..32w+31 <-> tile rows 4w..4w+3 of each column block
    const int m = warp * 32 + lane;
    const int ty = m >> 3, tx = m & 7;
#pragma unroll 1
    for (int cb = 0; cb < kTcCB; ++cb) {
        float acc[N];
#pragma unroll
        for (int c0 = 0; c0 < N; c0 += 16) {
            uint32_t v[16];
            const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + cb * N + c0;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
                : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                  "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
                : "r"(taddr));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n");
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[c0 + j] = __uint_as_float(v[j]);
        }
        const int y = oy0 + ty, x = ox0 + cb * 8 + tx;
#pragma unroll
        for (int c = 0; c < N; ++c) acc[c] = c < a.cout ? fmaxf(__fadd_rn(acc[c], __ldg(a.bias + c)), 0.0f) : 0.0f;
        if (a.out) {
#pragma unroll
            for (int c = 0; c < N; ++c)
                if (c < a.cout) a.out[((int64_t)n * a.cout + c) * hw + y * a.w + x] = acc[c];
        }
        if (a.pooled) {  // 2x2 block = lanes {l, l^1, l^8, l^9}
            const int ph = a.h >> 1, pw = a.w >> 1;
#pragma unroll
            for (int c = 0; c < N; ++c) {
                float mx = fmaxf(acc[c], __shfl_xor_sync(0xffffffffu, acc[c], 1));
                mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
                if (c < a.cout && !(tx & 1) && !(ty & 1))
                    a.pooled[((int64_t)n * a.cout + c) * ph * pw + (y >> 1) * pw + (x >> 1)] = mx;
            }
        }
        if (a.prob) {
            float sum = 0.0f;
#pragma unroll
            for (int c = 0; c < N; ++c)
                if (c < a.cout) sum = fmaf(acc[c], __ldg(a.w1 + c), sum);
            sum = __fadd_rn(sum, __ldg(a.b1));
            a.prob[(int64_t)n * hw + y * a.w + x] = __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-sum)));
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(kCols));
}

template <int N>
int launch_conv_tc(const ConvArgs& a, cudaStream_t s) {
    if (a.h % kTcTH || a.w % kTcTW) return fail(VB_EINVAL, "U-Net tile size");
    if (!a.wtc) return fail(VB_EINVAL, "tensor-core weights missing");
    const size_t smem = 4 * (size_t)kTcPlane + 2 * (size_t)(9 * 2 * N * 16);
    VB_CUDA(cudaFuncSetAttribute(conv3x3_tc_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((unsigned)((a.h / kTcTH) * (a.w / kTcTW)), (unsigned)a.n);
    {
        ProfScope ps(kProfOther, s);
        conv3x3_tc_kernel<N><<<grid, 128, smem, s>>>(a);
    }
    VB_LAUNCHED();
    return VB_OK;
}

int conv(const ConvArgs& a0, cudaStream_t s) {
    ConvArgs a = a0;
    a.dbg = knob("VB_UNET_DBG", 0);
    if (!knob("VB_UNET_SIMT", 0)) {  // experiment: FP32 SIMT kernels
        if (a.cout <= 16) return launch_conv_tc<16>(a, s);
        if (a.cout <= 32) return launch_conv_tc<32>(a, s);
        if (a.cout <= 64) return launch_conv_tc<64>(a, s);
    }
    if (a.cout <= 16) return launch_conv<16>(a, s);
    if (a.cout <= 32) return launch_conv<32>(a, s);
    if (a.cout <= 64) return launch_conv<64>(a, s);
    return fail(VB_EINVAL, "U-Net layer wider than 64 channels");
}

// ------------------------------------------------------------- percentiles
// numpy "linear" quantile (np.percentile default): virtual index
// n*q + (alpha + q*(1 - alpha - beta)) - 1 with alpha = beta = 1
// (_compute_virtual_index), neighbours floor / floor + 1 clamped like
// _get_indexes, gamma = index - floor.
struct PctIdx {
    int64_t prev, next;
    double gamma;
};
PctIdx pct_index(int64_t n, double q) {
    const double vi = (double)n * q + (1.0 + q * (1.0 - 1.0 - 1.0)) - 1.0;
    PctIdx p;
    double pv = floor(vi);
    p.gamma = vi - pv;
    if (vi >= (double)(n - 1)) {
        p.prev = p.next = n - 1;
    } else if (vi < 0) {
        p.prev = p.next = 0;
    } else {
        p.prev = (int64_t)pv;
        p.next = p.prev + 1;
    }
    return p;
}

struct PctArgs {
    const float* data;  // channel c at data + c * stride  (c = 2*block + {0: spatial, 1: temporal})
    const float* data2; // temporal base (channel odd) ; spatial base for even
    int64_t stride;     // floats between consecutive blocks
    int64_t n;          // values per channel
    int64_t rank[4];    // prev/next of p1, prev/next of p99
    double gamma[2];
    double* out;        // [2K][3]: p1, p99, constant flag
};

// One CTA per channel: exact order statistics by 8-bit radix select for the
// four ranks at once, then numpy's _lerp in float64 (diff of the float32
// neighbours in float32, as numpy subtracts the two float32 values).
__global__ void __launch_bounds__(1024) percentile_kernel(PctArgs a) {
    __shared__ uint32_t hist[4][256];
    __shared__ uint32_t s_prefix[4], s_rank[4];
    const int ch = blockIdx.x;
    const float* x = (ch & 1 ? a.data2 : a.data) + (int64_t)(ch >> 1) * a.stride;
    if (threadIdx.x < 4) {
        s_prefix[threadIdx.x] = 0;
        s_rank[threadIdx.x] = (uint32_t)a.rank[threadIdx.x];
    }
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = 24 - 8 * pass;
        for (int i = threadIdx.x; i < 4 * 256; i += blockDim.x) (&hist[0][0])[i] = 0;
        __syncthreads();
        uint32_t pre[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) pre[j] = s_prefix[j];
        const uint32_t hmask = pass == 0 ? 0u : (0xffffffffu << (32 - 8 * pass));
        for (int64_t i = threadIdx.x; i < a.n; i += blockDim.x) {
            const uint32_t k = fkey_u(x[i]);
            const uint32_t d = (k >> shift) & 255u;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if ((k & hmask) == pre[j]) atomicAdd(&hist[j][d], 1u);
        }
        __syncthreads();
        if (threadIdx.x < 4) {
            const int j = threadIdx.x;
            uint32_t r = s_rank[j], c = 0;
            int d = 0;
            for (; d < 255; ++d) {
                if (r < c + hist[j][d]) break;
                c += hist[j][d];
            }
            s_rank[j] = r - c;
            s_prefix[j] = pre[j] | ((uint32_t)d << shift);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double p[2];
        for (int q = 0; q < 2; ++q) {
            const float lo = fkey_inv_u(s_prefix[2 * q]), hi = fkey_inv_u(s_prefix[2 * q + 1]);
            const double t = a.gamma[q];
            const double diff = (double)__fsub_rn(hi, lo);  // float32 subtract (numpy: b - a on f32)
            double r = (double)lo + diff * t;
            if (t >= 0.5) r = (double)hi - diff * (1.0 - t);
            p[q] = r;
        }
        a.out[3 * ch] = p[0];
        a.out[3 * ch + 1] = p[1];
        a.out[3 * ch + 2] = p[1] <= p[0] ? 1.0 : 0.0;
    }
}

// out[b][c][i] = float32(clip((x - p1) / (p99 - p1), 0, 1)) in float64, or 0
// for a constant channel (unet.py:190-195)
__global__ void normalize_kernel(const float* __restrict__ sp, const float* __restrict__ tp, int64_t stride,
                                 int64_t n, int nblk, const double* __restrict__ pct, float* __restrict__ out) {
    const int64_t total = (int64_t)nblk * 2 * n;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t chn = i / n, j = i - chn * n;
        const int b = (int)(chn >> 1), c = (int)(chn & 1);
        const double p1 = pct[3 * chn], p99 = pct[3 * chn + 1];
        float v = 0.0f;
        if (pct[3 * chn + 2] == 0.0) {
            const double x = (double)(c ? tp : sp)[(int64_t)b * stride + j];
            double r = (x - p1) / (p99 - p1);
            r = r < 0.0 ? 0.0 : (r > 1.0 ? 1.0 : r);
            v = (float)r;
        }
        out[i] = v;
    }
}

// numpy np.pad(..., mode="reflect") index (mirror without repeating the edge)
__host__ __device__ __forceinline__ int np_reflect(int i, int n) {
    if (n == 1) return 0;
    const int period = 2 * (n - 1);
    int m = i % period;
    if (m < 0) m += period;
    return m < n ? m : period - m;
}

__global__ void pad_kernel(const float* __restrict__ in, int nimg, int h, int w, int ph, int pw,
                           float* __restrict__ out) {
    const int64_t total = (int64_t)nimg * ph * pw;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t img = i / ((int64_t)ph * pw);
        const int r = (int)(i - img * ph * pw);
        const int y = r / pw, x = r % pw;
        out[i] = in[img * h * w + (int64_t)np_reflect(y, h) * w + np_reflect(x, w)];
    }
}

struct MergeArgs {
    const float* probs;  // [K * tiles][64][64]
    const float* tent;   // [64][64]
    const int* ys;
    const int* xs;
    int nys, nxs;
    int h, w;            // output (cropped)
    int nblk;
    float* out;          // [K][h][w]
};

// Tent-weighted float64 blend in the reference's tile order (unet.py:236-244)
__global__ void merge_kernel(MergeArgs a) {
    const int64_t total = (int64_t)a.nblk * a.h * a.w;
    const int tiles = a.nys * a.nxs;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int b = (int)(i / ((int64_t)a.h * a.w));
        const int r = (int)(i - (int64_t)b * a.h * a.w);
        const int y = r / a.w, x = r % a.w;
        double acc = 0.0, nrm = 0.0;
        for (int iy = 0; iy < a.nys; ++iy) {
            const int y0 = a.ys[iy];
            if (y < y0 || y >= y0 + kPatch) continue;
            for (int ix = 0; ix < a.nxs; ++ix) {
                const int x0 = a.xs[ix];
                if (x < x0 || x >= x0 + kPatch) continue;
                const int t = (y - y0) * kPatch + (x - x0);
                const float tw = a.tent[t];
                const float pv = a.probs[((int64_t)b * tiles + iy * a.nxs + ix) * kPatch * kPatch + t];
                acc += (double)__fmul_rn(pv, tw);
                nrm += (double)tw;
            }
        }
        float m = (float)(acc / nrm);
        m = m < 0.0f ? 0.0f : (m > 1.0f ? 1.0f : m);
        a.out[i] = m;
    }
}

int grid_for(int64_t total) { return (int)std::min<int64_t>((total + 255) / 256, 148 * 16); }

}  // namespace

// Canonical parameter order = unet.architecture() (unet.py:34-54).
struct UNetLayer {
    int cin, cout;
    int64_t kofs, bofs;
};

}  // namespace vb

using namespace vb;

struct vb_unet {
    float* params = nullptr;  // device copy, canonical order
    std::vector<UNetLayer> layers;  // enc1.c1, enc1.c2, enc2.c1, enc2.c2, enc3.c1, enc3.c2, dec2.c1, dec2.c2, dec1.c1, dec1.c2, out
    float* tent = nullptr;          // [64][64] device
    // activation scratch owned by the handle, grown on demand (a per-call
    // stream-ordered allocation of ~1.6 GB was measured to cost up to 190 ms
    // when the pool had to remap after other large allocations); one call at
    // a time per handle
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    // per-call work (normalised pairs, padding, tile outputs, percentiles) and
    // the tile-origin tables of the last geometry, also owned by the handle: a
    // pageable host->device copy per call would block the host thread until the
    // stream drains and serialise the stage executor's chunk pipeline
    void* work = nullptr;
    size_t work_bytes = 0;
    int g_h = -1, g_w = -1, g_stride = -1, g_nys = 0, g_nxs = 0;
    int64_t g_nblk = 0;
    int2* d_org = nullptr;
    int* d_pos = nullptr;
    // 3x3 conv weights pre-split for the tensor cores (ConvArgs::wtc layout)
    float* tcw = nullptr;
    std::vector<int64_t> tc_ofs;
};

namespace vb {
namespace {
int grow(void** buf, size_t* have, size_t bytes, cudaStream_t s) {
    if (bytes > *have) {
        VB_CUDA(cudaStreamSynchronize(s));  // the old buffer may still be in use by queued work
        cudaFree(*buf);
        *buf = nullptr;
        *have = 0;
        VB_CUDA(cudaMalloc(buf, bytes));
        *have = bytes;
    }
    return VB_OK;
}

int net_scratch(vb_unet* net, size_t bytes, cudaStream_t s, void** out) {
    if (bytes > net->scratch_bytes) {
        VB_CUDA(cudaStreamSynchronize(s));  // the old buffer may still be in use by queued work
        cudaFree(net->scratch);
        net->scratch = nullptr;
        net->scratch_bytes = 0;
        VB_CUDA(cudaMalloc(&net->scratch, bytes));
        net->scratch_bytes = bytes;
    }
    *out = net->scratch;
    return VB_OK;
}
}  // namespace
}  // namespace vb

namespace {

int64_t unet_param_count(std::vector<UNetLayer>* layers) {
    const int widths[3] = {16, 32, 64};
    std::vector<std::pair<int, int>> convs;  // (cin, cout)
    int cin = 2;
    for (int l = 0; l < 3; ++l) {
        convs.push_back({cin, widths[l]});
        convs.push_back({widths[l], widths[l]});
        cin = widths[l];
    }
    for (int l = 2; l >= 1; --l) {
        const int cout = widths[l - 1];
        convs.push_back({cin + cout, cout});
        convs.push_back({cout, cout});
        cin = cout;
    }
    int64_t off = 0;
    for (size_t i = 0; i < convs.size(); ++i) {
        UNetLayer L{convs[i].first, convs[i].second, off, off + (int64_t)convs[i].first * convs[i].second * 9};
        off = L.bofs + convs[i].second;
        if (layers) layers->push_back(L);
    }
    UNetLayer out{cin, 1, off, off + cin};
    off = out.bofs + 1;
    if (layers) layers->push_back(out);
    return off;
}

// unet.py:_tent_weights (float64 ramp outer product, floor 1e-3, float32)
void tent_host(float* t) {
    double ramp[kPatch];
    for (int i = 0; i < kPatch; ++i) ramp[i] = 1.0 - fabs((double)i - (kPatch - 1) / 2.0) / (kPatch / 2.0);
    for (int y = 0; y < kPatch; ++y)
        for (int x = 0; x < kPatch; ++x) t[y * kPatch + x] = (float)std::max(ramp[y] * ramp[x], 1e-3);
}

std::vector<int> tile_positions(int extent, int stride) {  // unet.py:199-203
    std::vector<int> pos;
    for (int p = 0; p <= extent - kPatch; p += stride) pos.push_back(p);
    if (pos.empty() || pos.back() != extent - kPatch) pos.push_back(extent - kPatch);
    return pos;
}

// Forward over n patches whose first layer reads `src` per ConvArgs mode 0/2.
int unet_forward(vb_unet* net, ConvArgs first, int64_t n, float* probs, cudaStream_t s) {
    if (n <= 0) return VB_OK;
    const int64_t P2 = (int64_t)kPatch * kPatch;
    // scratch: e1a e1 p1 e2a e2 p2 e3a e3 d2a d2 d1a (floats per patch)
    const int64_t sz[11] = {16 * P2, 16 * P2, 16 * P2 / 4, 32 * P2 / 4, 32 * P2 / 4, 32 * P2 / 16,
                            64 * P2 / 16, 64 * P2 / 16, 32 * P2 / 4, 32 * P2 / 4, 16 * P2};
    int64_t per = 0;
    for (int i = 0; i < 11; ++i) per += sz[i];
    // patches per pass: bound the scratch to ~2 GB
    int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n, ((int64_t)2 << 30) / (per * 4)));
    if (first.mode == 2 && chunk < n)  // tile batches start on an image boundary
        chunk = std::max<int64_t>(first.tiles_per_img, chunk / first.tiles_per_img * first.tiles_per_img);
    float* scratch = nullptr;
    {
        void* p = nullptr;
        const int rc0 = net_scratch(net, (size_t)(per * chunk) * sizeof(float), s, &p);
        if (rc0) return rc0;
        scratch = static_cast<float*>(p);
    }
    float* buf[11];
    {
        float* p = scratch;
        for (int i = 0; i < 11; ++i) {
            buf[i] = p;
            p += sz[i] * chunk;
        }
    }
    float *e1a = buf[0], *e1 = buf[1], *p1 = buf[2], *e2a = buf[3], *e2 = buf[4], *p2 = buf[5], *e3a = buf[6],
          *e3 = buf[7], *d2a = buf[8], *d2 = buf[9], *d1a = buf[10];
    const float* P = net->params;
    auto L = [&](int i) { return net->layers[i]; };
    int rc = VB_OK;
    for (int64_t n0 = 0; n0 < n && rc == VB_OK; n0 += chunk) {
        const int nb = (int)std::min<int64_t>(chunk, n - n0);
        auto base = [&](int li, int h, const float* x0, int c0, int mode, const float* x1, float* out, float* pooled) {
            ConvArgs a;
            memset(&a, 0, sizeof(a));
            a.n = nb;
            a.h = a.w = h;
            a.cin = L(li).cin;
            a.cout = L(li).cout;
            a.x0 = x0;
            a.c0 = c0;
            a.mode = mode;
            a.x1 = x1;
            a.wt = P + L(li).kofs;
            a.wtc = net->tcw + net->tc_ofs[li];
            a.bias = P + L(li).bofs;
            a.out = out;
            a.pooled = pooled;
            return a;
        };
        ConvArgs a0 = first;
        a0.n = nb;
        if (a0.mode == 2) {
            a0.origins = first.origins + n0;
            // images advance with the tiles: the kernel derives the image from the patch index
            // relative to this chunk, so pass the chunk's first image explicitly
            const int64_t img0 = n0 / first.tiles_per_img;
            a0.x0 = first.x0 + img0 * first.img_stride;
            a0.tiles_per_img = first.tiles_per_img;
            if (n0 % first.tiles_per_img) {  // chunk starts mid-image: fall back to one image per pass
                rc = fail(VB_EINVAL, "U-Net chunk must start on an image boundary");
                break;
            }
        } else {
            a0.x0 = first.x0 + n0 * 2 * P2;
        }
        a0.h = a0.w = kPatch;
        a0.cin = L(0).cin;
        a0.cout = L(0).cout;
        a0.c0 = L(0).cin;
        a0.x1 = nullptr;
        a0.wt = P + L(0).kofs;
        a0.wtc = net->tcw + net->tc_ofs[0];
        a0.bias = P + L(0).bofs;
        a0.out = e1a;
        a0.pooled = nullptr;
        a0.prob = nullptr;
        rc = conv(a0, s);
        if (!rc) rc = conv(base(1, 64, e1a, 16, 0, nullptr, e1, p1), s);
        if (!rc) rc = conv(base(2, 32, p1, 16, 0, nullptr, e2a, nullptr), s);
        if (!rc) rc = conv(base(3, 32, e2a, 32, 0, nullptr, e2, p2), s);
        if (!rc) rc = conv(base(4, 16, p2, 32, 0, nullptr, e3a, nullptr), s);
        if (!rc) rc = conv(base(5, 16, e3a, 64, 0, nullptr, e3, nullptr), s);
        if (!rc) rc = conv(base(6, 32, e3, 64, 1, e2, d2a, nullptr), s);
        if (!rc) rc = conv(base(7, 32, d2a, 32, 0, nullptr, d2, nullptr), s);
        if (!rc) rc = conv(base(8, 64, d2, 32, 1, e1, d1a, nullptr), s);
        if (!rc) {
            ConvArgs a = base(9, 64, d1a, 16, 0, nullptr, nullptr, nullptr);
            a.w1 = P + L(10).kofs;
            a.b1 = P + L(10).bofs;
            a.prob = probs + n0 * P2;
            rc = conv(a, s);
        }
    }
    return rc;
}

int percentiles(const float* sp, const float* tp, int64_t stride, int64_t n, int64_t nblk, double* pct,
                cudaStream_t s) {
    const PctIdx q1 = pct_index(n, 0.01), q99 = pct_index(n, 0.99);  // np.percentile(.., (1, 99)) -> q/100
    PctArgs a;
    a.data = sp;
    a.data2 = tp;
    a.stride = stride;
    a.n = n;
    a.rank[0] = q1.prev;
    a.rank[1] = q1.next;
    a.rank[2] = q99.prev;
    a.rank[3] = q99.next;
    a.gamma[0] = q1.gamma;
    a.gamma[1] = q99.gamma;
    a.out = pct;
    {
        ProfScope ps(kProfOther, s);
        percentile_kernel<<<(unsigned)(2 * nblk), 1024, 0, s>>>(a);
    }
    VB_LAUNCHED();
    return VB_OK;
}

}  // namespace

extern "C" {

int vb_unet_create(vb_unet** out, const float* params_host, int64_t n_params) {
    if (!out || !params_host) return fail(VB_EINVAL, "null argument");
    *out = nullptr;
    auto* net = new vb_unet();
    const int64_t want = unet_param_count(&net->layers);
    if (n_params != want) {
        delete net;
        return fail(VB_EINVAL, "U-Net parameter count " + std::to_string(n_params) + ", expected " +
                                   std::to_string(want));
    }
    float tent[kPatch * kPatch];
    tent_host(tent);
    // tensor-core weight copies: per 3x3 layer, per 8-channel chunk,
    // [hi, lo][tap][half][cout][4] with hi = tf32 round-to-nearest-away (cvt.rna), lo = w - hi
    std::vector<float> tcw;
    for (size_t li = 0; li + 1 < net->layers.size(); ++li) {
        const UNetLayer& L = net->layers[li];
        const int N = L.cout, nch = (L.cin + 7) / 8;
        net->tc_ofs.push_back((int64_t)tcw.size());
        const size_t base = tcw.size();
        tcw.resize(base + (size_t)nch * 2 * 9 * 2 * N * 4, 0.0f);
        for (int ch = 0; ch < nch; ++ch)
            for (int tap = 0; tap < 9; ++tap)
                for (int ci = 0; ci < 8 && ch * 8 + ci < L.cin; ++ci)
                    for (int co = 0; co < N; ++co) {
                        const float wv = params_host[L.kofs + ((int64_t)co * L.cin + ch * 8 + ci) * 9 + tap];
                        uint32_t u;
                        memcpy(&u, &wv, 4);
                        if ((u & 0x7f800000u) != 0x7f800000u) u += 0x1000u;
                        u &= 0xffffe000u;
                        float hi;
                        memcpy(&hi, &u, 4);
                        const size_t o = ((size_t)tap * 2 + (ci >> 2)) * N * 4 + (size_t)co * 4 + (ci & 3);
                        const size_t chunk = base + (size_t)ch * 2 * 9 * 2 * N * 4;
                        tcw[chunk + o] = hi;
                        tcw[chunk + (size_t)9 * 2 * N * 4 + o] = wv - hi;
                    }
    }
    net->tc_ofs.push_back((int64_t)tcw.size());
    cudaError_t e = cudaMalloc(&net->params, (size_t)want * sizeof(float));
    e = e ? e : cudaMalloc(&net->tcw, tcw.size() * sizeof(float));
    e = e ? e : cudaMemcpy(net->tcw, tcw.data(), tcw.size() * sizeof(float), cudaMemcpyHostToDevice);
    e = e ? e : cudaMalloc(&net->tent, sizeof(tent));
    e = e ? e : cudaMemcpy(net->params, params_host, (size_t)want * sizeof(float), cudaMemcpyHostToDevice);
    e = e ? e : cudaMemcpy(net->tent, tent, sizeof(tent), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(net->params);
        cudaFree(net->tent);
        cudaFree(net->tcw);
        delete net;
        return cuda_fail(e, "vb_unet_create");
    }
    *out = net;
    return VB_OK;
}

int64_t vb_unet_param_count(void) { return unet_param_count(nullptr); }

int vb_unet_forward(vb_unet* net, const float* patches_dev, int64_t n, float* probs_dev, void* stream) {
    if (!net || (n > 0 && (!patches_dev || !probs_dev))) return fail(VB_EINVAL, "null argument");
    ConvArgs a;
    memset(&a, 0, sizeof(a));
    a.x0 = patches_dev;
    a.mode = 0;
    return unet_forward(net, a, n, probs_dev, (cudaStream_t)stream);
}

}  // extern "C"

namespace {

int normalize_impl(const float* sp, const float* tp, int64_t n_blocks, int height, int width, float* out, double* pct,
                   cudaStream_t s) {
    const int64_t n = (int64_t)height * width;
    int rc = percentiles(sp, tp, n, n, n_blocks, pct, s);
    if (rc) return rc;
    normalize_kernel<<<grid_for(n_blocks * 2 * n), 256, 0, s>>>(sp, tp, n, n, (int)n_blocks, pct, out);
    VB_LAUNCHED();
    return VB_OK;
}

size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

// tile origins of (h, w, stride) for n_blocks images, cached on the handle
int tile_tables(vb_unet* net, int ph, int pw, int stride, int64_t n_blocks, cudaStream_t s) {
    if (net->g_h == ph && net->g_w == pw && net->g_stride == stride && net->g_nblk >= n_blocks) return VB_OK;
    const std::vector<int> ys = tile_positions(ph, stride), xs = tile_positions(pw, stride);
    const int tiles = (int)(ys.size() * xs.size());
    const int64_t nb = std::max<int64_t>(n_blocks, net->g_nblk);
    std::vector<int2> org((size_t)nb * tiles);
    for (int64_t b = 0; b < nb; ++b)
        for (size_t iy = 0; iy < ys.size(); ++iy)
            for (size_t ix = 0; ix < xs.size(); ++ix) org[(size_t)b * tiles + iy * xs.size() + ix] = make_int2(xs[ix], ys[iy]);
    std::vector<int> pos(ys);
    pos.insert(pos.end(), xs.begin(), xs.end());
    VB_CUDA(cudaStreamSynchronize(s));  // the old tables may still be read by queued work
    cudaFree(net->d_org);
    cudaFree(net->d_pos);
    net->d_org = nullptr;
    net->d_pos = nullptr;
    net->g_h = -1;
    VB_CUDA(cudaMalloc(&net->d_org, org.size() * sizeof(int2)));
    VB_CUDA(cudaMalloc(&net->d_pos, pos.size() * sizeof(int)));
    VB_CUDA(cudaMemcpy(net->d_org, org.data(), org.size() * sizeof(int2), cudaMemcpyHostToDevice));
    VB_CUDA(cudaMemcpy(net->d_pos, pos.data(), pos.size() * sizeof(int), cudaMemcpyHostToDevice));
    net->g_h = ph;
    net->g_w = pw;
    net->g_stride = stride;
    net->g_nblk = nb;
    net->g_nys = (int)ys.size();
    net->g_nxs = (int)xs.size();
    return VB_OK;
}

// normalised pairs (device) -> probability maps; `work` holds padding + tile outputs
int tile_merge_impl(vb_unet* net, const float* normalized, int64_t n_blocks, int height, int width, int stride,
                    float* prob_dev, char* work, cudaStream_t s) {
    const int ph = std::max(height, kPatch), pw = std::max(width, kPatch);
    int rc = tile_tables(net, ph, pw, stride, n_blocks, s);
    if (rc) return rc;
    const int tiles = net->g_nys * net->g_nxs;
    const bool pad = ph != height || pw != width;
    float* padded = reinterpret_cast<float*>(work);
    float* probs = reinterpret_cast<float*>(work + (pad ? align256((size_t)n_blocks * 2 * ph * pw * sizeof(float)) : 0));
    const float* img = normalized;
    if (pad) {
        pad_kernel<<<grid_for(n_blocks * 2 * ph * pw), 256, 0, s>>>(normalized, (int)n_blocks * 2, height, width, ph, pw,
                                                                   padded);
        VB_LAUNCHED();
        img = padded;
    }
    ConvArgs a;
    memset(&a, 0, sizeof(a));
    a.x0 = img;
    a.mode = 2;
    a.origins = net->d_org;
    a.ih = ph;
    a.iw = pw;
    a.img_stride = (int64_t)2 * ph * pw;
    a.tiles_per_img = tiles;
    rc = unet_forward(net, a, n_blocks * tiles, probs, s);
    if (rc) return rc;
    MergeArgs m;
    m.probs = probs;
    m.tent = net->tent;
    m.ys = net->d_pos;
    m.xs = net->d_pos + net->g_nys;
    m.nys = net->g_nys;
    m.nxs = net->g_nxs;
    m.h = height;
    m.w = width;
    m.nblk = (int)n_blocks;
    m.out = prob_dev;
    {
        ProfScope ps(kProfOther, s);
        merge_kernel<<<grid_for(n_blocks * height * width), 256, 0, s>>>(m);
    }
    VB_LAUNCHED();
    return VB_OK;
}

size_t tile_merge_work(int64_t n_blocks, int height, int width, int stride) {
    const int ph = std::max(height, kPatch), pw = std::max(width, kPatch);
    const size_t tiles = tile_positions(ph, stride).size() * tile_positions(pw, stride).size();
    const bool pad = ph != height || pw != width;
    return (pad ? align256((size_t)n_blocks * 2 * ph * pw * sizeof(float)) : 0) +
           align256((size_t)n_blocks * tiles * kPatch * kPatch * sizeof(float));
}

}  // namespace

extern "C" {

int vb_normalize_pair(const float* spatial_dev, const float* temporal_dev, int64_t n_blocks, int height, int width,
                      float* out_dev, void* stream) {
    if (!spatial_dev || !temporal_dev || !out_dev) return fail(VB_EINVAL, "null argument");
    if (n_blocks < 1 || height < 1 || width < 1) return fail(VB_EINVAL, "empty summary images");
    cudaStream_t s = (cudaStream_t)stream;
    // percentile scratch: a per-thread, per-device buffer grown on demand (a
    // stream-ordered pool allocation here was measured at up to 100 ms right
    // after the stage's multi-GB pool allocations)
    static thread_local void* buf[64] = {};
    static thread_local size_t have[64] = {};
    int dev = 0;
    VB_CUDA(cudaGetDevice(&dev));
    if (dev >= 64) return fail(VB_EINVAL, "device ordinal >= 64");
    int rc = grow(&buf[dev], &have[dev], (size_t)n_blocks * 2 * 3 * sizeof(double), s);
    if (rc) return rc;
    return normalize_impl(spatial_dev, temporal_dev, n_blocks, height, width, out_dev, static_cast<double*>(buf[dev]), s);
}

int vb_unet_tile_merge(vb_unet* net, const float* normalized_dev, int64_t n_blocks, int height, int width, int stride,
                       float* prob_dev, void* stream) {
    if (!net || !normalized_dev || !prob_dev) return fail(VB_EINVAL, "null argument");
    if (n_blocks < 1 || height < 1 || width < 1) return fail(VB_EINVAL, "empty summary images");
    if (stride < 1) return fail(VB_EINVAL, "stride must be >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    int rc = grow(&net->work, &net->work_bytes, tile_merge_work(n_blocks, height, width, stride), s);
    if (rc) return rc;
    return tile_merge_impl(net, normalized_dev, n_blocks, height, width, stride, prob_dev,
                           static_cast<char*>(net->work), s);
}

int vb_unet_segment(vb_unet* net, const float* spatial_dev, const float* temporal_dev, int64_t n_blocks, int height,
                    int width, int stride, float* normalized_dev, float* prob_dev, void* stream) {
    if (!net || !spatial_dev || !temporal_dev || !prob_dev) return fail(VB_EINVAL, "null argument");
    if (n_blocks < 1 || height < 1 || width < 1) return fail(VB_EINVAL, "empty summary images");
    if (stride < 1) return fail(VB_EINVAL, "stride must be >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    // work: [pct][normalised pairs (unless the caller keeps them)][tile-merge work]
    const size_t pct_b = align256((size_t)n_blocks * 6 * sizeof(double));
    const size_t norm_b = normalized_dev ? 0 : align256((size_t)n_blocks * 2 * height * width * sizeof(float));
    int rc = grow(&net->work, &net->work_bytes, pct_b + norm_b + tile_merge_work(n_blocks, height, width, stride), s);
    if (rc) return rc;
    char* w = static_cast<char*>(net->work);
    float* norm = normalized_dev ? normalized_dev : reinterpret_cast<float*>(w + pct_b);
    rc = normalize_impl(spatial_dev, temporal_dev, n_blocks, height, width, norm, reinterpret_cast<double*>(w), s);
    if (rc == VB_OK)
        rc = tile_merge_impl(net, norm, n_blocks, height, width, stride, prob_dev, w + pct_b + norm_b, s);
    return rc;
}

int vb_unet_destroy(vb_unet* net) {
    if (!net) return VB_OK;
    cudaFree(net->params);
    cudaFree(net->tent);
    cudaFree(net->scratch);
    cudaFree(net->work);
    cudaFree(net->tcw);
    cudaFree(net->d_org);
    cudaFree(net->d_pos);
    delete net;
    return VB_OK;
}

}  // extern "C"
