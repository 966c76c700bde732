// Motion estimation kernels (sm_100a).
//
// Reference algorithm (paths under /root/reference/pkg/src/voltseg):
//   make_reference           motion.py:211-214
//   mean ZNCC score grid     kernels.py:23-75 (float64 semantics), _native.pyx:22-118
//   argmax + tie-break       motion.py:127-135, :143-150
//   quadratic sub-pixel fit  motion.py:136-139, :153-160
//
// B200 design:
//  * One CTA per (patch group, frame).  A patch group is a run of up to ~8
//    patches on one patch row; the union of their search windows
//    ((P+2R) rows x (G*P+2R) cols) is staged ONCE in shared memory as f32.
//  * Window statistics (sum f, sum f^2 over every candidate window) are
//    float64 sliding sums over the staged union (exact for integer samples,
//    like the reference's float64 summed-area tables).
//  * The cross term uses the centred template r~ = r - mean_p (f32, prepared
//    once per recording), so cov = sum f * r~ never forms the catastrophic
//    difference sum(f r) - sum f sum r / n that the reference's float32 cross
//    sum suffers from (_native_impl.h:18-35).  Each thread owns one (patch,
//    dy) row of 2R+1 candidates in registers: per template row it loads
//    S+P-1 frame samples and P template taps (float4 broadcast) and issues
//    S*P FFMAs.  At r = 8 (S = 17) a half-warp owns a patch (16 rows + a
//    shared middle row, cross_row_split17) and each thread carries two
//    frames through FFMA2 (zncc_group_kernel<21,17,2,true>).
//  * Per-CTA partial sums of ZNCC over its patches are written in fixed
//    order (float64) and a finalize kernel sums the groups in fixed order,
//    divides by N and runs the tie-broken argmax + quadratic fit: fully
//    deterministic, no atomics.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <type_traits>
#include <vector>

#include "tma.cuh"
#include "vb.cuh"

namespace vb {

// ---------------------------------------------------------------- template
__global__ void template_sum_kernel(const void* __restrict__ frames, int dtype, int64_t n, int64_t hw,
                                    double* __restrict__ sum, int accumulate) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x) {
        double acc = accumulate ? sum[i] : 0.0;
        for (int64_t t = 0; t < n; ++t) acc += (double)load_sample(frames, dtype, t * hw + i);
        sum[i] = acc;
    }
}

__global__ void template_finish_kernel(const double* __restrict__ sum, double n, int64_t hw,
                                       float* __restrict__ ref) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x)
        ref[i] = (float)(sum[i] / n);
}

int launch_template_sum(const void* frames, int dtype, int64_t n, int64_t hw, double* sum, int accumulate,
                        cudaStream_t s) {
    int blocks = (int)std::min<int64_t>((hw + 255) / 256, 148 * 16);
    if (blocks < 1) blocks = 1;
    template_sum_kernel<<<blocks, 256, 0, s>>>(frames, dtype, n, hw, sum, accumulate);
    VB_LAUNCHED();
    return VB_OK;
}

int launch_template_finish(const double* sum, int64_t n_total, int64_t hw, float* ref, cudaStream_t s) {
    int blocks = (int)std::min<int64_t>((hw + 255) / 256, 148 * 16);
    if (blocks < 1) blocks = 1;
    template_finish_kernel<<<blocks, 256, 0, s>>>(sum, (double)n_total, hw, ref);
    VB_LAUNCHED();
    return VB_OK;
}

// One CTA per template patch: float64 sums in the native kernel's row-major
// order (_native.pyx:84-97), then the centred f32 patch r - rsum/n.
__global__ void prep_templates_kernel(const float* __restrict__ ref, int w, int patch, int tp,
                                      const int32_t* __restrict__ origins, float* __restrict__ tmpl,
                                      double* __restrict__ rvar_out, double* __restrict__ rmean_out) {
    const int p = blockIdx.x;
    const int px = origins[2 * p], py = origins[2 * p + 1];
    __shared__ double s_mean;
    if (threadIdx.x == 0) {
        double rsum = 0.0, rsq = 0.0;
        for (int yy = 0; yy < patch; ++yy)
            for (int xx = 0; xx < patch; ++xx) {
                double v = (double)ref[(size_t)(py + yy) * w + px + xx];
                rsum += v;
                rsq += v * v;
            }
        double n = (double)patch * (double)patch;
        rvar_out[p] = rsq - rsum * rsum / n;
        s_mean = rsum / n;
        rmean_out[p] = s_mean;
    }
    __syncthreads();
    const double mean = s_mean;
    float* out = tmpl + (size_t)p * patch * tp;
    for (int i = threadIdx.x; i < patch * tp; i += blockDim.x) {
        int yy = i / tp, xx = i % tp;
        out[i] = xx < patch ? (float)((double)ref[(size_t)(py + yy) * w + px + xx] - mean) : 0.0f;
    }
}

int launch_prep_templates(const float* ref, int h, int w, int patch, const Templates& t, cudaStream_t s) {
    (void)h;
    prep_templates_kernel<<<t.n, 128, 0, s>>>(ref, w, patch, t.tp, t.origins, t.tmpl, t.rvar, t.rmean);
    VB_LAUNCHED();
    return VB_OK;
}

// ---------------------------------------------------------------- ZNCC
struct ZnccArgs {
    const void* frames;  // first frame of this launch
    int dtype;
    int64_t hw;
    int w;
    int P, R, S, tp;
    int nch;        // dx chunks per (patch, dy) item (1 on the fast path)
    int rows;       // lanes per patch in the item space: S, or 16 for the split S = 17 kernel
    int pitch_cap;  // f32 region pitch (odd, >= max wu)
    int bw, bh;     // raw box width / height in samples (bh = P + 2R)
    int bhc;        // TMA box height (the raw box is fetched as ceil(bh/bhc) row chunks)
    int use_tma;
    int tma_z0;     // tensor-map frame index of this launch's frame 0
    int off_reg, off_z, off_t;  // shared-memory carve-up (bytes); raw box at 0
    int ss_pad;     // inv row stride per patch: S*S rounded to 4 floats (16-byte bulk copies)
    int off_inv;    // search kernel: shared buffer receiving the group's inv rows (bulk copy), -1 = none
    int conv_batch; // batched u16 -> f32 region conversion (all loads of a row first)
    int n_patches;
    const float* tmpl;
    const double* rvar;
    const double* rmean;
    const int32_t* patch_col;
    const PatchGroup* groups;
    int n_groups;
    int64_t n_frames;
    float* inv;       // [n_frames][N][S*S]  1/sqrt(fvar*rvar) (0 where the reference skips)
    double* partial;  // [n_frames][n_groups][S*S]
    const float* cov;  // COMBINE statistics: [n_frames][N][ss_pad] window covariances (zncc_mma_kernel)
    int off_sinv;      // COMBINE statistics: shared [G][ss_pad] inv rows
};

constexpr int kGenericDXB = 8;

// Frame samples are centred on an integer c close to the group's template
// level, so the f32 cross sums accumulate O(100) instead of O(1000)
// products.  Integer samples stay exact; the window variance is shift
// invariant.  (Small-valued float data, |mean| < 64, is left uncentred.)
__device__ __forceinline__ float group_centre(const ZnccArgs& a, const PatchGroup& grp) {
    double m = 0.0;
    for (int p = 0; p < grp.count; ++p) m += a.rmean[grp.first + p];
    m /= (double)grp.count;
    return fabs(m) >= 64.0 ? (float)rint(m) : 0.0f;
}

// Column offset of the group window inside its raw box: TMA tile loads on
// sm_100a fault (illegal instruction) unless the innermost start coordinate
// is 16-byte aligned, so boxes start at the aligned column below x0.
__device__ __forceinline__ int box_off(const ZnccArgs& a, const PatchGroup& grp) {
    return grp.x0 & (a.dtype == VB_U16 ? 7 : 3);
}

// Raw box [bh][bw] of frame t (group union window) -> shared memory.  With
// TMA one elected thread issues cp.async.bulk.tensor row chunks completing on
// `bar`; otherwise all threads copy (caller synchronises).
__device__ __forceinline__ void fetch_box(const ZnccArgs& a, const CUtensorMap* tmap, const PatchGroup& grp,
                                          int64_t t, void* raw, uint64_t* bar) {
    const size_t esz = a.dtype == VB_U16 ? 2 : 4;
    if (a.use_tma) {
        if (threadIdx.x == 0) {
            const int nck = (a.bh + a.bhc - 1) / a.bhc;
            mbar_expect_tx(bar, (uint32_t)((size_t)a.bw * a.bhc * nck * esz));
            for (int k = 0; k < nck; ++k)
                tma_load_3d((char*)raw + (size_t)k * a.bhc * a.bw * esz, tmap, grp.x0 - box_off(a, grp),
                            grp.y0 + k * a.bhc, a.tma_z0 + (int)t, bar);
        }
        return;
    }
    const int64_t fbase = t * a.hw;
    const int wu = grp.wu, off = box_off(a, grp);
    for (int i = threadIdx.x; i < a.bh * wu; i += blockDim.x) {
        const int r = i / wu, cc = i - r * wu;
        const int64_t idx = fbase + (int64_t)(grp.y0 + r) * a.w + grp.x0 + cc;
        if (a.dtype == VB_U16)
            reinterpret_cast<uint16_t*>(raw)[r * a.bw + cc + off] =
                __ldg(reinterpret_cast<const uint16_t*>(a.frames) + idx);
        else
            reinterpret_cast<float*>(raw)[r * a.bw + cc + off] = __ldg(reinterpret_cast<const float*>(a.frames) + idx);
    }
}

__device__ __forceinline__ void box_ready(const ZnccArgs& a, uint64_t* bar, uint32_t& phase) {
    if (a.use_tma) {
        mbar_wait(bar, phase);
        phase ^= 1u;
    }
}

// Window statistics for one (patch group, frame): sliding sums of f and f^2
// over every candidate window, then inv = 1/sqrt(fvar * rvar) (kernels.py:60-72;
// 0 where the reference skips a dead patch or a flat window).  Camera (u16)
// samples use exact integer arithmetic (int32 sums, int64 sums of squares,
// n*fvar = n*S2 - S1^2 exactly) straight from the TMA-staged raw box; float32
// input uses float64 sums.  One thread per union column slides its vertical
// sums down all S rows (a single round for groups up to 256 columns wide),
// then one thread per (patch, dy) row slides horizontally.  The next frame's
// box is fetched while this frame's horizontal pass runs.
#ifndef VB_FAST_RSQRT
#define VB_FAST_RSQRT 0  // measured: the MUFU seed + Newton step was slower (2.06 vs 1.99 ms per 4000 C2 frames)
#endif
constexpr bool kFastRsqrt = VB_FAST_RSQRT;
// 1/sqrt(x) for positive normal x: f32 MUFU seed + one float64 Newton step
// (relative error ~2^-46; the result is rounded to f32 anyway), branch-free
// unlike the library's double rsqrt.  Falls back when x leaves the f32 range.
__device__ __forceinline__ double rsqrt_pos(double x) {
    if (x < 1e-30 || x > 1e30) return rsqrt(x);
    const double y = (double)rsqrtf((float)x);
    return y * fma(-0.5 * x * y, y, 1.5);
}

// One inv row of S values whose first element sits K floats past a 16-byte
// boundary (inv rows are dense, S floats apart; per-patch blocks start
// 16-byte aligned): (4 - K) & 3 scalar stores, float4 stores, scalar tail --
// 6 stores instead of 17 for S = 17 (measured: the scalar stores, each warp
// store touching 32 sectors, were 18 % of the statistics kernel).
template <int S, int K>
__device__ __forceinline__ void store_row(float* out, const float (&v)[S]) {
    constexpr int head = (4 - K) & 3, nv = (S - head) / 4;
#pragma unroll
    for (int i = 0; i < head && i < S; ++i) out[i] = v[i];
#pragma unroll
    for (int q = 0; q < nv; ++q)
        reinterpret_cast<float4*>(out + head)[q] =
            make_float4(v[head + 4 * q], v[head + 4 * q + 1], v[head + 4 * q + 2], v[head + 4 * q + 3]);
#pragma unroll
    for (int i = head + 4 * nv; i < S; ++i) out[i] = v[i];
}

// COMBINE (tensor-core path, uint16): the kernel finishes the search -- the
// inv rows stay in shared memory and partial[t][group][c] = sum over the
// group's patches q (in order) of cov[t][q][c] * inv[q][c] in float64, the
// covariances coming from zncc_mma_kernel (no inv round trip through HBM).
template <bool INT, int P_CT, int S_CT = 0, bool COMBINE = false>
__global__ void __launch_bounds__(256) zncc_stats_kernel(ZnccArgs a, const __grid_constant__ CUtensorMap tmap) {
    using T1 = typename std::conditional<INT, int, double>::type;        // sample / sum of f
    using T2 = typename std::conditional<INT, long long, double>::type;  // sum of f^2
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    const int P = P_CT ? P_CT : a.P;  // compile-time patch: fully unrolled window sums
    const int S = S_CT ? S_CT : a.S, SS = S * S;
    const PatchGroup grp = a.groups[blockIdx.x];
    const int G = grp.count, wu = grp.wu, vp = wu | 1;
    const double nn = (double)P * (double)P;
    T2* v2 = reinterpret_cast<T2*>(smem + a.off_z);                                         // [S][vp]
    T1* v1 = reinterpret_cast<T1*>(smem + a.off_z + (size_t)S * a.pitch_cap * sizeof(T2));  // [S][vp]
    const float cg = group_centre(a, grp);
    const int cgi = (int)cg;
    const int boff = box_off(a, grp);
    if (threadIdx.x == 0 && a.use_tma) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmap);
    }
    __syncthreads();
    uint32_t phase = 0;
    int64_t t = blockIdx.y;
    if (t < a.n_frames) fetch_box(a, &tmap, grp, t, smem, &bar);
    for (; t < a.n_frames; t += gridDim.y) {
        __syncthreads();  // box visible (plain path) / V free (previous horizontal pass done)
        box_ready(a, &bar, phase);
        // vertical window sums: one thread per union column, sliding down all S rows
        for (int c = threadIdx.x; c < wu; c += blockDim.x) {
            auto sample = [&](int r) -> T1 {
                if constexpr (INT)
                    return (int)reinterpret_cast<const uint16_t*>(smem)[r * a.bw + c + boff] - cgi;
                else
                    return (double)__fsub_rn(reinterpret_cast<const float*>(smem)[r * a.bw + c + boff], cg);
            };
            T1 s1 = 0;
            T2 s2 = 0;
            if constexpr (P_CT != 0) {
#pragma unroll
                for (int yy = 0; yy < P_CT; ++yy) {
                    const T1 f = sample(yy);
                    s1 += f;
                    s2 += (T2)f * (T2)f;
                }
            } else {
                for (int yy = 0; yy < P; ++yy) {  // any patch size
                    const T1 f = sample(yy);
                    s1 += f;
                    s2 += (T2)f * (T2)f;
                }
            }
            v1[c] = s1;
            v2[c] = s2;
            for (int dy = 1; dy < S; ++dy) {
                const T1 fo = sample(dy - 1), fi = sample(dy - 1 + P);
                s1 += fi - fo;
                s2 += (T2)fi * (T2)fi - (T2)fo * (T2)fo;
                v1[dy * vp + c] = s1;
                v2[dy * vp + c] = s2;
            }
        }
        __syncthreads();
        if (t + gridDim.y < a.n_frames) fetch_box(a, &tmap, grp, t + gridDim.y, smem, &bar);  // raw box is free
        for (int it = threadIdx.x; it < G * S; it += blockDim.x) {
            int p, dy;
            if constexpr (S_CT != 0) {
                // items ordered by the 16-byte phase k = (dy * S) & 3 of their inv row, so a
                // warp's rows share the phase and store as (head, float4s, tail) together
                // (class k holds dy = d0, d0 + 4, ... with d0 = (k*S) & 3: S odd, S*S = 1 mod 4)
                int k = 0, idx = it;
#pragma unroll
                for (int kk = 0; kk < 3; ++kk) {
                    const int nk = (S_CT - ((kk * S_CT) & 3) + 3) / 4;
                    if (idx < G * nk) break;
                    idx -= G * nk;
                    k = kk + 1;
                }
                const int d0 = (k * S_CT) & 3, nk = (S_CT - d0 + 3) / 4;
                p = idx / nk;
                dy = d0 + 4 * (idx - p * nk);
            } else {
                p = it / S;
                dy = it - p * S;
            }
            const int gp = grp.first + p;
            const int col = a.patch_col[gp];
            const double rv = a.rvar[gp];
            const T1* r1 = v1 + dy * vp + col;
            const T2* r2 = v2 + dy * vp + col;
            T1 h1 = 0;
            T2 h2 = 0;
            if constexpr (P_CT != 0) {
#pragma unroll
                for (int xx = 0; xx < P_CT; ++xx) {
                    h1 += r1[xx];
                    h2 += r2[xx];
                }
            } else {
                for (int xx = 0; xx < P; ++xx) {  // any patch size
                    h1 += r1[xx];
                    h2 += r2[xx];
                }
            }
            float* out = COMBINE ? reinterpret_cast<float*>(smem + a.off_sinv) + (size_t)p * a.ss_pad + (size_t)dy * S
                                 : a.inv + ((size_t)t * a.n_patches + gp) * a.ss_pad + (size_t)dy * S;
            float ivs[S_CT ? S_CT : 1];
#pragma unroll
            for (int dx = 0; dx < (S_CT ? S_CT : 64); ++dx) {
                if (!S_CT && dx >= S) break;
                float iv = 0.0f;
                if constexpr (INT) {
                    // n*fvar exactly; 1/sqrt(fvar*rv) = P / sqrt(n*fvar*rv).  int64 -> f64 by
                    // the 2^52 bit trick (exact below 2^52, i.e. always for P <= 45 on u16
                    // data) instead of the conversion unit; larger values convert (rounded,
                    // like the reference's float64 sums).
                    const long long nf = (long long)P * P * h2 - (long long)h1 * h1;
                    if (rv > 0.0 && nf > 0) {
                        const double nfd = nf < (1LL << 52)
                                               ? __longlong_as_double(0x4330000000000000LL | nf) - 4503599627370496.0
                                               : (double)nf;
                        iv = (float)((double)P * (kFastRsqrt ? rsqrt_pos(nfd * rv) : rsqrt(nfd * rv)));
                    }
                } else {
                    const double fvar = h2 - h1 * h1 / nn;  // kernels.py:67
                    if (rv > 0.0 && fvar > 0.0) iv = (float)rsqrt(fvar * rv);
                }
                if constexpr (S_CT != 0)
                    ivs[dx] = iv;
                else
                    out[dx] = iv;
                if (dx + 1 < S) {
                    h1 += r1[dx + P] - r1[dx];
                    h2 += r2[dx + P] - r2[dx];
                }
            }
            if constexpr (S_CT != 0) {
                if constexpr (COMBINE) {
#pragma unroll
                    for (int dx = 0; dx < S_CT; ++dx) out[dx] = ivs[dx];
                } else {
                    switch ((dy * S_CT) & 3) {  // warp-uniform except where two phases meet
                        case 0: store_row<S_CT, 0>(out, ivs); break;
                        case 1: store_row<S_CT, 1>(out, ivs); break;
                        case 2: store_row<S_CT, 2>(out, ivs); break;
                        default: store_row<S_CT, 3>(out, ivs); break;
                    }
                }
            }
        }
        if constexpr (COMBINE) {
            __syncthreads();  // the group's inv rows are complete
            const float* sinv = reinterpret_cast<const float*>(smem + a.off_sinv);
            const float* cov = a.cov + ((size_t)t * a.n_patches + grp.first) * a.ss_pad;
            double* part = a.partial + ((size_t)t * a.n_groups + blockIdx.x) * SS;
            for (int c = threadIdx.x; c < SS; c += blockDim.x) {
                double acc = 0.0;
                for (int q = 0; q < G; ++q)
                    acc = fma((double)__ldg(cov + (size_t)q * a.ss_pad + c), (double)sinv[(size_t)q * a.ss_pad + c], acc);
                part[c] = acc;
            }
        }
    }
}

// Cross sums for one (patch, dy) row of S candidates, compile-time P and S.
// Template taps come from the prepared patch in global memory (L1-resident,
// warp-broadcast): every lane of a patch reads the same float4.
#ifndef VB_PAIR_IL
#define VB_PAIR_IL 1  // paired split kernel: the two frames' regions interleaved, one 64-bit load per window sample (measured: C2 search 5.84 -> 5.74 ms per 4000 frames; 0 = separate regions)
#endif
#ifndef VB_GEN_UNROLL
#define VB_GEN_UNROLL 1  // measured: 2 -> C3 search 13.54 -> 16.75 ms (115 registers)
#endif
constexpr int kGenUnroll = VB_GEN_UNROLL;
template <int P, int S>
__device__ __forceinline__ void cross_row(const float* __restrict__ reg, int pitch, const float* __restrict__ trow0,
                                          int tp, float (&acc)[S]) {
    constexpr bool kTapOuter = S == 21;
#pragma unroll
    for (int d = 0; d < S; ++d) acc[d] = 0.0f;
#pragma unroll kGenUnroll
    for (int yy = 0; yy < P; ++yy) {
        const float* fr = reg + yy * pitch;
        float win[S + P - 1];
#pragma unroll
        for (int i = 0; i < S + P - 1; ++i) win[i] = fr[i];
        const float4* trow = reinterpret_cast<const float4*>(trow0 + yy * tp);
        float tv[(P + 3) / 4 * 4];
#pragma unroll
        for (int q = 0; q < (P + 3) / 4; ++q) {
            const float4 t4 = __ldg(trow + q);
            tv[4 * q] = t4.x;
            tv[4 * q + 1] = t4.y;
            tv[4 * q + 2] = t4.z;
            tv[4 * q + 3] = t4.w;
        }
        // anti-diagonal order (window index i = xx + d ascending): the FMAs
        // consume window samples in the order their loads were issued, so the
        // row's LDS latency overlaps the arithmetic (and w[i] is the reused
        // operand of consecutive FFMAs).  S = 21: tap-outer order instead --
        // every accumulator once per tap, no short dependency chains at the
        // row ends (measured: C5 search 19.82 -> 19.33 ms per 1000 frames;
        // S = 17 / 25 unchanged).  Each accumulator still adds its products
        // in tap order xx = 0..P-1, so the sums are identical.
        if constexpr (kTapOuter) {
#pragma unroll
            for (int xx = 0; xx < P; ++xx) {
#pragma unroll
                for (int d = 0; d < S; ++d) acc[d] = fmaf(win[d + xx], tv[xx], acc[d]);
            }
        } else {
#pragma unroll
            for (int i = 0; i < S + P - 1; ++i) {
#pragma unroll
                for (int xx = (i - (S - 1) > 0 ? i - (S - 1) : 0); xx <= (i < P - 1 ? i : P - 1); ++xx)
                    acc[i - xx] = fmaf(win[i], tv[xx], acc[i - xx]);
            }
        }
    }
}

// S = 17 (search radius 8) with 16 lanes per patch: (G patches x 17 rows)
// would leave 8 of every 136 lanes' worth of a fifth warp busy, so each patch
// gets one half-warp.  Lane l owns candidate row d = l (< 8) or l + 1, and the
// middle row M = 8 is shared: its 21 (frame row, template row) products are
// spread over the lanes at two common iterations -- yy = 8, where lane d adds
// frame row d + 8 with template row d (16 rows), and yy = 12, where lanes
// d in {4, 13..16} add template rows {8, 17..20} -- so every window sample
// loaded for the lane's own row serves the shared row too.  The half-warp
// then sums the shared row's partials in a fixed shuffle tree.
#ifndef VB_SPLIT_UNROLL
#define VB_SPLIT_UNROLL 1  // one frame per thread, measured: 3 -> 7.41 ms, 7 -> 9.16 ms (instruction cache) vs 7.12 ms
#endif
#ifndef VB_SPLIT_UNROLL_PAIR
#define VB_SPLIT_UNROLL_PAIR 2  // two frames per thread (half the FMA instructions), measured: 6.28 -> 5.89 ms (2, 3 or 7 alike)
#endif
constexpr int kSplitUnroll = VB_SPLIT_UNROLL;
constexpr int kSplitUnrollPair = VB_SPLIT_UNROLL_PAIR;
#ifndef VB_SPLIT_PREFETCH_PAIR
#define VB_SPLIT_PREFETCH_PAIR 8  // two frames per thread (unrolled x2), measured: 0 / 4 / 8 / 12 / 16 samples 6.46 / 5.89 / 5.84 / 5.87 / 5.90 ms
#endif
#ifndef VB_SPLIT_PREFETCH
#define VB_SPLIT_PREFETCH 4  // measured: 7.57 -> 7.29 ms per 4000 C2 frames (4 or 8 samples alike)
#endif
#ifndef VB_SPLIT_PREFETCH_TAPS
#define VB_SPLIT_PREFETCH_TAPS 6  // measured: all taps of the next row carried over, 7.29 -> 7.12 ms (128 regs, still 4 CTAs)
#endif
#ifndef VB_SPLIT_MIN_BLOCKS
#define VB_SPLIT_MIN_BLOCKS 4  // measured: 113 regs x 4 CTAs beats a 96-reg cap with spills
#endif
constexpr int kSplitMinBlocks = VB_SPLIT_MIN_BLOCKS;

// Lane values: one frame (float, FFMA) or two frames of the same group
// (float2 = the pair's samples at the same region position, FFMA2 with the
// template tap broadcast).  Per frame the products and their order are the
// scalar path's, so both give identical sums.
__device__ __forceinline__ void lane_zero(float& v) { v = 0.0f; }
__device__ __forceinline__ void lane_zero(float2& v) { v = make_float2(0.0f, 0.0f); }
__device__ __forceinline__ void lane_load(float& v, const float* p, int) { v = *p; }
__device__ __forceinline__ void lane_load(float2& v, const float* p, int fstride) { v = make_float2(p[0], p[fstride]); }
__device__ __forceinline__ void lane_fma(float& acc, float w, float t) { acc = fmaf(w, t, acc); }
__device__ __forceinline__ void lane_fma(float2& acc, float2 w, float t) { acc = __ffma2_rn(w, make_float2(t, t), acc); }
__device__ __forceinline__ void lane_shfl_add(float& v, int off) { v += __shfl_down_sync(0xffffffffu, v, off, 16); }
__device__ __forceinline__ void lane_shfl_add(float2& v, int off) {
    v.x += __shfl_down_sync(0xffffffffu, v.x, off, 16);
    v.y += __shfl_down_sync(0xffffffffu, v.y, off, 16);
}

// Interleaved pair regions (CS = 2): the two frames' samples of one region
// position are adjacent, one 64-bit shared load per window sample.
template <int CS, typename V>
__device__ __forceinline__ void lane_load_cs(V& v, const float* p, int fstride) {
    if constexpr (CS == 2)
        v = *reinterpret_cast<const float2*>(p);
    else
        lane_load(v, p, fstride);
}

// fstride: floats between the two frames' regions (V = float2, CS = 1);
// CS: floats per region column (2 = interleaved pair, pitch in floats)
template <int P, typename V, int PF = VB_SPLIT_PREFETCH, int CS = 1>
__device__ __forceinline__ void cross_row_split17(const float* __restrict__ reg, int pitch, int fstride,
                                                  const float* __restrict__ trow0, int tp, int d, V (&acc)[17],
                                                  V (&accm)[17]) {
    constexpr int S = 17, M = 8;
#pragma unroll
    for (int i = 0; i < S; ++i) {
        lane_zero(acc[i]);
        lane_zero(accm[i]);
    }
    const bool second = d == 4 || d >= 13;
#if VB_SPLIT_PREFETCH
    // the next row's first taps and window samples are loaded during this
    // row's FMAs, so a row starts without waiting on L1 / shared latency
    constexpr int TQ = VB_SPLIT_PREFETCH_TAPS;  // float4 tap groups carried over (1..6)
    float4 t_next[TQ];
#pragma unroll
    for (int q = 0; q < TQ; ++q) t_next[q] = __ldg(reinterpret_cast<const float4*>(trow0) + q);
    V w_next[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) lane_load_cs<CS>(w_next[i], reg + CS * i, fstride);
#endif
    constexpr int kUnroll = std::is_same<V, float2>::value ? kSplitUnrollPair : kSplitUnroll;
#pragma unroll kUnroll
    for (int yy = 0; yy < P; ++yy) {
        const float* fr = reg + yy * pitch;
        V win[S + P - 1];
        float tv[(P + 3) / 4 * 4];
#if VB_SPLIT_PREFETCH
#pragma unroll
        for (int i = 0; i < PF; ++i) win[i] = w_next[i];
#pragma unroll
        for (int i = PF; i < S + P - 1; ++i) lane_load_cs<CS>(win[i], fr + CS * i, fstride);
#pragma unroll
        for (int q = 0; q < TQ; ++q) {
            tv[4 * q] = t_next[q].x;
            tv[4 * q + 1] = t_next[q].y;
            tv[4 * q + 2] = t_next[q].z;
            tv[4 * q + 3] = t_next[q].w;
        }
        {
            const float4* trow = reinterpret_cast<const float4*>(trow0 + yy * tp);
#pragma unroll
            for (int q = TQ; q < (P + 3) / 4; ++q) {
                const float4 t4 = __ldg(trow + q);
                tv[4 * q] = t4.x;
                tv[4 * q + 1] = t4.y;
                tv[4 * q + 2] = t4.z;
                tv[4 * q + 3] = t4.w;
            }
            const int yn = yy + 1 < P ? yy + 1 : yy;
#pragma unroll
            for (int q = 0; q < TQ; ++q) t_next[q] = __ldg(reinterpret_cast<const float4*>(trow0 + yn * tp) + q);
#pragma unroll
            for (int i = 0; i < PF; ++i) lane_load_cs<CS>(w_next[i], reg + yn * pitch + CS * i, fstride);
        }
#else
#pragma unroll
        for (int i = 0; i < S + P - 1; ++i) lane_load_cs<CS>(win[i], fr + CS * i, fstride);
        {
            const float4* trow = reinterpret_cast<const float4*>(trow0 + yy * tp);
#pragma unroll
            for (int q = 0; q < (P + 3) / 4; ++q) {
                const float4 t4 = __ldg(trow + q);
                tv[4 * q] = t4.x;
                tv[4 * q + 1] = t4.y;
                tv[4 * q + 2] = t4.z;
                tv[4 * q + 3] = t4.w;
            }
        }
#endif
#pragma unroll
        for (int i = 0; i < S + P - 1; ++i) {
#pragma unroll
            for (int xx = (i - (S - 1) > 0 ? i - (S - 1) : 0); xx <= (i < P - 1 ? i : P - 1); ++xx)
                lane_fma(acc[i - xx], win[i], tv[xx]);
        }
        if (yy == M || (yy == M + 4 && second)) {
            const float4* trow = reinterpret_cast<const float4*>(trow0 + (d + yy - M) * tp);
#pragma unroll
            for (int q = 0; q < (P + 3) / 4; ++q) {
                const float4 t4 = __ldg(trow + q);
                tv[4 * q] = t4.x;
                tv[4 * q + 1] = t4.y;
                tv[4 * q + 2] = t4.z;
                tv[4 * q + 3] = t4.w;
            }
#pragma unroll
            for (int i = 0; i < S + P - 1; ++i) {
#pragma unroll
                for (int xx = (i - (S - 1) > 0 ? i - (S - 1) : 0); xx <= (i < P - 1 ? i : P - 1); ++xx)
                    lane_fma(accm[i - xx], win[i], tv[xx]);
            }
        }
    }
}

// Search kernel: persistent over frames (blockIdx.y, +gridDim.y, ...), FPI
// frames per iteration.  Per iteration: wait for the TMA boxes, convert them to
// centred f32 regions, issue the next iteration's TMA into the now-free raw
// buffers, run the register-tiled cross sums, then z = cov * inv summed over
// the group's patches in fixed order.  An item is one (frame, patch, dy) row
// of S candidates; FPI = 2 packs G*S items of two frames into whole warps
// (G = 8, S = 17: 272 items in 9 warps = 94 % of the lanes busy, against
// 136 in 5 warps = 85 % with one frame).  The cov rows alias the region,
// which is dead once every thread holds its accumulators.
template <int P_CT, int S_CT, int FPI, bool SPLIT = false>
__global__ void __launch_bounds__(SPLIT ? 128 : 288, SPLIT ? (FPI == 2 ? 2 : kSplitMinBlocks) : 1) zncc_group_kernel(ZnccArgs a, const __grid_constant__ CUtensorMap tmap) {
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar[FPI];
    __shared__ __align__(8) uint64_t bar_inv;
    uint32_t inv_phase = 0;
    // inv bulk-copy path compiled for S = 17 (on) and S = 21 (off at run time: the variant with it
    // compiled in measured faster on C5 either way); S = 25 keeps 96 registers without it
    constexpr bool kInvPath = (S_CT == 17 || S_CT == 21) && (FPI == 1 || SPLIT);
    const int P = P_CT ? P_CT : a.P;
    const int S = S_CT ? S_CT : a.S;
    const int R = (S - 1) / 2;
    const int RH = P + 2 * R;
    const int tp = a.tp;
    const PatchGroup grp = a.groups[blockIdx.x];
    const int G = grp.count, wu = grp.wu;
    const int pitch = a.pitch_cap;
    const int SS = S * S;
    const size_t raw_slot = (size_t)a.off_reg / FPI;        // raw boxes at [0, off_reg)
    const size_t reg_slot = (size_t)(a.off_z - a.off_reg) / FPI;  // regions (cov aliased) at [off_reg, off_z)
    const int tid = threadIdx.x, nth = blockDim.x;
    const float cg = group_centre(a, grp);
    const float magic = 8388608.0f + cg;
    constexpr bool kIL = SPLIT && FPI == 2 && VB_PAIR_IL;  // interleaved pair regions
    constexpr int CS = kIL ? 2 : 1;
    // region of frame f, padded row r, column c (floats)
    auto reg_at = [&](int f, int r, int c) -> float* {
        return kIL ? reinterpret_cast<float*>(smem + a.off_reg) + 2 * (r * pitch + c) + f
                   : reinterpret_cast<float*>(smem + a.off_reg + f * reg_slot) + r * pitch + c;
    };
    const int boff = box_off(a, grp);
    if (tid == 0 && a.use_tma) {
#pragma unroll
        for (int f = 0; f < FPI; ++f) mbar_init(&bar[f], 1);
        mbar_init(&bar_inv, 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmap);
    }
    __syncthreads();
    uint32_t phase = 0;
    const int64_t gy = gridDim.y;
    auto fetch = [&](int64_t t0) {
#pragma unroll
        for (int f = 0; f < FPI; ++f)
            if (t0 + f * gy < a.n_frames) fetch_box(a, &tmap, grp, t0 + f * gy, smem + f * raw_slot, &bar[f]);
    };
    int64_t t = blockIdx.y;
    if (t < a.n_frames) fetch(t);
    for (; t < a.n_frames; t += FPI * gy) {
        int nf = 0;
#pragma unroll
        for (int f = 0; f < FPI; ++f) nf += (t + f * gy < a.n_frames) ? 1 : 0;
        __syncthreads();  // plain-path boxes visible; previous partial phase done with the cov rows
        if (a.use_tma) {
            for (int f = 0; f < nf; ++f) mbar_wait(&bar[f], phase);
            phase ^= 1u;
        }
        // raw boxes -> centred f32 regions: warps over rows, lanes over columns
        // (compile-time-S kernels: threads over (frame, column) units walking
        // all rows, sixteen loads in flight (measured vs eight: -0.2..0.3 % on
        // C2/C3/C5), no per-row index arithmetic)
        if (S_CT != 0 && a.dtype == VB_U16 && a.conv_batch >= 2) {
            constexpr int RHC = S_CT != 0 ? P_CT + S_CT - 1 : 1;
            for (int u = tid; u < nf * wu; u += nth) {
                const int f = u >= wu ? 1 : 0, c = u - f * wu;
                const uint16_t* raw = reinterpret_cast<const uint16_t*>(smem + f * raw_slot) + boff + c;
                float* reg = reg_at(f, 0, c);
#pragma unroll
                for (int r0 = 0; r0 < RHC; r0 += 16) {
                    uint32_t v[16];
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        if (r0 + k < RHC) v[k] = raw[(r0 + k) * a.bw];
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        if (r0 + k < RHC) reg[(r0 + k) * pitch * CS] = u16_minus(v[k], magic);
                }
            }
        } else {
            const int lane = tid & 31, nw = nth >> 5;
            for (int fr = tid >> 5; fr < nf * RH; fr += nw) {
                const int f = fr / RH, r = fr - f * RH;
                float* reg = reg_at(f, r, 0);
                if (SPLIT && a.dtype == VB_U16 && wu <= 256 && a.conv_batch) {  // loads first, then converts (LDS latency overlapped)
                    const uint16_t* raw = reinterpret_cast<const uint16_t*>(smem + f * raw_slot) + boff + r * a.bw;
                    uint32_t v[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) v[k] = lane + 32 * k < wu ? raw[lane + 32 * k] : 0u;
#pragma unroll
                    for (int k = 0; k < 8; ++k)
                        if (lane + 32 * k < wu) reg[CS * (lane + 32 * k)] = u16_minus(v[k], magic);
                } else if (a.dtype == VB_U16) {
                    const uint16_t* raw = reinterpret_cast<const uint16_t*>(smem + f * raw_slot) + boff + r * a.bw;
                    for (int c = lane; c < wu; c += 32) reg[CS * c] = u16_minus(raw[c], magic);
                } else {
                    const float* raw = reinterpret_cast<const float*>(smem + f * raw_slot) + boff + r * a.bw;
                    for (int c = lane; c < wu; c += 32) reg[CS * c] = __fsub_rn(raw[c], cg);
                }
            }
        }
        __syncthreads();
        if (t + FPI * gy < a.n_frames) fetch(t + FPI * gy);  // raw boxes are free
        if (kInvPath && a.off_inv >= 0 && tid == 0) {  // the frames' inv rows land during the cross phase
            const uint32_t bytes = (uint32_t)(G * a.ss_pad * 4);
            mbar_expect_tx(&bar_inv, bytes * nf);
            for (int f = 0; f < nf; ++f)
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                        smem_u32(smem + a.off_inv + (size_t)f * bytes)),
                    "l"(a.inv + ((size_t)(t + f * gy) * a.n_patches + grp.first) * a.ss_pad), "r"(bytes),
                    "r"(smem_u32(&bar_inv))
                    : "memory");
        }
        const int per_frame = G * a.rows * a.nch;
        const int nitems = nf * per_frame;
        // fast path: one item per thread, cov rows alias the dead regions;
        // generic path: items loop over the block, cov rows in their own slots
        constexpr bool kOneRound = P_CT != 0 && S_CT != 0;
        auto cov_at = [&](int f) -> float* {
            return kOneRound ? reinterpret_cast<float*>(smem + a.off_reg + f * reg_slot)
                             : reinterpret_cast<float*>(smem + a.off_z + f * (size_t)(a.off_t - a.off_z) / FPI);
        };
        if constexpr (SPLIT && FPI == 2) {
            // one (patch, lane) item per thread covering both frames of the
            // iteration (FFMA2 pairs); the second region may be stale when
            // nf == 1 -- its sums are computed and dropped
            const int it = tid;
            const bool valid = it < per_frame;
            const int p = it >> 4, l = it & 15;
            const int d = l < 8 ? l : l + 1;
            float2 acc[17], accm[17];
            if (valid) {
                const int col = a.patch_col[grp.first + p];
                const float* reg = reg_at(0, d, col);
                cross_row_split17<21, float2, VB_SPLIT_PREFETCH_PAIR, CS>(reg, pitch * CS, (int)(reg_slot / 4),
                                                                          a.tmpl + (size_t)(grp.first + p) * P * tp, tp,
                                                                          d, acc, accm);
            } else {
#pragma unroll
                for (int i = 0; i < 17; ++i) acc[i] = accm[i] = make_float2(0.0f, 0.0f);
            }
#pragma unroll
            for (int i = 0; i < 17; ++i) {
#pragma unroll
                for (int off = 8; off >= 1; off >>= 1) lane_shfl_add(accm[i], off);
            }
            __syncthreads();  // every region read: the cov rows may overwrite them
            if (valid) {
                float* z0 = cov_at(0) + (size_t)p * SS;
                float* z1 = cov_at(1) + (size_t)p * SS;
#pragma unroll
                for (int i = 0; i < 17; ++i) {
                    z0[d * 17 + i] = acc[i].x;
                    z1[d * 17 + i] = acc[i].y;
                }
                if (l == 0) {
#pragma unroll
                    for (int i = 0; i < 17; ++i) {
                        z0[8 * 17 + i] = accm[i].x;
                        z1[8 * 17 + i] = accm[i].y;
                    }
                }
            }
        } else if constexpr (SPLIT) {
            // one (frame, patch, lane) item per thread, 16 lanes per patch
            const int it = tid;
            const bool valid = it < nitems;
            const int f = valid ? it / per_frame : 0;
            const int rem = it - f * per_frame;
            const int p = rem >> 4, l = rem & 15;
            const int d = l < 8 ? l : l + 1;
            float acc[17], accm[17];
            if (valid) {
                const int col = a.patch_col[grp.first + p];
                const float* reg = reinterpret_cast<const float*>(smem + a.off_reg + f * reg_slot) + d * pitch + col;
                cross_row_split17<21>(reg, pitch, 0, a.tmpl + (size_t)(grp.first + p) * P * tp, tp, d, acc, accm);
            } else {
#pragma unroll
                for (int i = 0; i < 17; ++i) acc[i] = accm[i] = 0.0f;
            }
#pragma unroll
            for (int i = 0; i < 17; ++i) {
#pragma unroll
                for (int off = 8; off >= 1; off >>= 1) lane_shfl_add(accm[i], off);
            }
            __syncthreads();  // every region read: the cov rows may overwrite them
            if (valid) {
                float* z = cov_at(f) + (size_t)p * SS;
#pragma unroll
                for (int i = 0; i < 17; ++i) z[d * 17 + i] = acc[i];
                if (l == 0) {
#pragma unroll
                    for (int i = 0; i < 17; ++i) z[8 * 17 + i] = accm[i];
                }
            }
        } else {
        for (int it0 = 0; it0 < nitems; it0 += nth) {
                const int it = it0 + tid;
                float acc[S_CT ? S_CT : kGenericDXB];
                int f = 0, p = 0, dy = 0, ch = 0;
                if (it < nitems) {
                    f = it / per_frame;
                    const int rem = it - f * per_frame;
                    dy = rem % a.rows;
                    const int pc = rem / a.rows;
                    p = pc / a.nch;
                    ch = pc - p * a.nch;
                    const int col = a.patch_col[grp.first + p];
                    const float* reg = reinterpret_cast<const float*>(smem + a.off_reg + f * reg_slot) + dy * pitch + col;
                    const float* trow0 = a.tmpl + (size_t)(grp.first + p) * P * tp;
                    if constexpr (kOneRound) {
                        cross_row<P_CT, S_CT>(reg, pitch, trow0, tp, acc);
                    } else {
#pragma unroll
                        for (int d = 0; d < kGenericDXB; ++d) acc[d] = 0.0f;
                        const int dx0 = ch * kGenericDXB;
                        for (int yy = 0; yy < P; ++yy) {
                            const float* fr = reg + yy * pitch + dx0;
                            const float* trow = trow0 + yy * tp;
                            for (int xx = 0; xx < P; ++xx) {
                                const float tv = __ldg(trow + xx);
#pragma unroll
                                for (int d = 0; d < kGenericDXB; ++d) acc[d] = fmaf(fr[xx + d], tv, acc[d]);
                            }
                        }
                    }
                }
                if constexpr (kOneRound) __syncthreads();  // every region read: the cov rows may overwrite them
                if (it < nitems) {
                    float* z = cov_at(f) + (size_t)p * SS + dy * S;
                    const int dx0 = kOneRound ? 0 : ch * kGenericDXB;
#pragma unroll
                    for (int d = 0; d < (S_CT ? S_CT : kGenericDXB); ++d)
                        if (kOneRound || dx0 + d < S) z[dx0 + d] = acc[d];
                }
            }
        }
        __syncthreads();
        const bool inv_smem = kInvPath && a.off_inv >= 0;
        if (inv_smem) {  // the group's inv rows, bulk-copied during the cross phase
            mbar_wait(&bar_inv, inv_phase);
            inv_phase ^= 1u;
        }
        for (int c2 = tid; c2 < nf * SS; c2 += nth) {
            const int ff = c2 / SS, c = c2 - ff * SS;
            const int64_t tf = t + ff * gy;
            const float* cov = cov_at(ff);
            double* part = a.partial + ((size_t)tf * a.n_groups + blockIdx.x) * SS;
            double s = 0.0;
            if (inv_smem) {
                const float* inv = reinterpret_cast<const float*>(smem + a.off_inv) + (size_t)ff * G * a.ss_pad;
                for (int q = 0; q < G; ++q) s += (double)cov[(size_t)q * SS + c] * (double)inv[(size_t)q * a.ss_pad + c];
            } else {
                const float* inv = a.inv + ((size_t)tf * a.n_patches + grp.first) * a.ss_pad;
                for (int q = 0; q < G; ++q)
                    s += (double)cov[(size_t)q * SS + c] * (double)__ldg(inv + (size_t)q * a.ss_pad + c);
            }
            part[c] = s;
        }
    }
}

// Sum group partials in fixed order, mean over N, tie-broken argmax
// (motion.py:143-150 order (|dx|+|dy|, dy, dx)), quadratic fit (:153-160).
__global__ void finalize_kernel(const double* __restrict__ partial, int n_groups, int S, int n_patches,
                                int64_t n_frames, int subpixel, vb_motion* __restrict__ vectors,
                                double* __restrict__ scores_out) {
    extern __shared__ double s_sc[];  // [S*S]
    __shared__ double s_best[32];
    __shared__ int s_key[32];
    const int SS = S * S, R = (S - 1) / 2;
    for (int64_t t = blockIdx.x; t < n_frames; t += gridDim.x) {
        const double* part = partial + (size_t)t * n_groups * SS;
        double best = -INFINITY;
        int bkey = 0x7fffffff;
        for (int c = threadIdx.x; c < SS; c += blockDim.x) {
            double s = 0.0;
            for (int g = 0; g < n_groups; ++g) s += part[(size_t)g * SS + c];
            s /= (double)n_patches;
            s_sc[c] = s;
            if (scores_out) scores_out[(size_t)t * SS + c] = s;
            const int dyi = c / S, dxi = c - dyi * S;
            const int key = ((abs(dxi - R) + abs(dyi - R)) * S + dyi) * S + dxi;
            if (s > best || (s == best && key < bkey)) {
                best = s;
                bkey = key;
            }
        }
        // block reduce (max score, then min key)
        for (int o = 16; o > 0; o >>= 1) {
            const double ob = __shfl_xor_sync(0xffffffffu, best, o);
            const int ok = __shfl_xor_sync(0xffffffffu, bkey, o);
            if (ob > best || (ob == best && ok < bkey)) {
                best = ob;
                bkey = ok;
            }
        }
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane == 0) {
            s_best[warp] = best;
            s_key[warp] = bkey;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int nw = (blockDim.x + 31) >> 5;
            best = s_best[0];
            bkey = s_key[0];
            for (int i = 1; i < nw; ++i)
                if (s_best[i] > best || (s_best[i] == best && s_key[i] < bkey)) {
                    best = s_best[i];
                    bkey = s_key[i];
                }
            const int dxi = bkey % S, dyi = (bkey / S) % S;
            vb_motion v;
            v.dx = dxi - R;
            v.dy = dyi - R;
            v.confidence = s_sc[dyi * S + dxi];
            v.sub_dx = 0.0;
            v.sub_dy = 0.0;
            if (subpixel) {
                // _quadratic_peak(scores[dy+r, :], dx+r) and (scores[:, dx+r], dy+r)
                if (dxi > 0 && dxi < S - 1) {
                    const double l = s_sc[dyi * S + dxi - 1], m = s_sc[dyi * S + dxi], r = s_sc[dyi * S + dxi + 1];
                    const double den = __dadd_rn(__dsub_rn(l, __dmul_rn(2.0, m)), r);
                    if (den < 0) v.sub_dx = fmin(fmax(__ddiv_rn(__dmul_rn(0.5, __dsub_rn(l, r)), den), -0.999), 0.999);
                }
                if (dyi > 0 && dyi < S - 1) {
                    const double l = s_sc[(dyi - 1) * S + dxi], m = s_sc[dyi * S + dxi], r = s_sc[(dyi + 1) * S + dxi];
                    const double den = __dadd_rn(__dsub_rn(l, __dmul_rn(2.0, m)), r);
                    if (den < 0) v.sub_dy = fmin(fmax(__ddiv_rn(__dmul_rn(0.5, __dsub_rn(l, r)), den), -0.999), 0.999);
                }
            }
            vectors[t] = v;
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------- launcher
using KernelFn = void (*)(ZnccArgs, CUtensorMap);

template <int S>
static KernelFn fast_kernel_for(int fpi) {
    return fpi == 2 ? zncc_group_kernel<21, S, 2> : zncc_group_kernel<21, S, 1>;
}

static KernelFn pick_kernel(int P, int S, int fpi, bool* fast) {
    *fast = true;
    if (P == 21) {
        switch (S) {
            case 3: return fast_kernel_for<3>(fpi);
            case 5: return fast_kernel_for<5>(fpi);
            case 7: return fast_kernel_for<7>(fpi);
            case 9: return fast_kernel_for<9>(fpi);
            case 11: return fast_kernel_for<11>(fpi);
            case 13: return fast_kernel_for<13>(fpi);
            case 15: return fast_kernel_for<15>(fpi);
            case 17: return fast_kernel_for<17>(fpi);
            case 19: return fast_kernel_for<19>(fpi);
            case 21: return fast_kernel_for<21>(fpi);
            case 23: return fast_kernel_for<23>(fpi);
            case 25: return fast_kernel_for<25>(fpi);
            default: break;
        }
    }
    *fast = false;
    return fpi == 2 ? zncc_group_kernel<0, 0, 2> : zncc_group_kernel<0, 0, 1>;
}

struct SmemPlan {
    int bw, bh, bhc, pitch;
    size_t raw_bytes;          // raw box (TMA destination), offset 0
    size_t off_reg, off_z;     // search kernel: f32 region, cov buffer
    size_t off_t;              // search kernel: template patches (fast path)
    size_t total;              // search kernel
    size_t stats_off, stats_total;  // statistics kernel: raw box + [S][pitch] T2 + [S][pitch] T1
};

static SmemPlan zncc_smem(int P, int R, int max_g, int max_wu, int dtype, int fpi = 1, bool alias = true,
                          int pitch = 0) {
    const int S = 2 * R + 1, SS = S * S, RH = P + 2 * R;
    const size_t esz = dtype == VB_U16 ? 2 : 4;
    SmemPlan sp;
    sp.bh = RH;
    // TMA box rows are 16-byte multiples and start 16-byte aligned (up to
    // 16/esz - 1 extra leading columns)
    sp.bw = (int)((((max_wu + 16 / esz - 1) * esz + 15) / 16) * 16 / esz);
    sp.pitch = pitch > 0 ? pitch : (max_wu | 1);
    sp.bhc = std::min(sp.bh, 256);  // TMA box height limit (one chunk for P + 2R <= 256)
    const int rows = (sp.bh + sp.bhc - 1) / sp.bhc * sp.bhc;
    sp.raw_bytes = (((size_t)sp.bw * rows * esz) + 127) & ~(size_t)127;
    // search kernel: fpi raw boxes, fpi f32 regions (the cov rows alias a
    // region on the fast path, else fpi separate cov slots)
    const size_t region = (size_t)RH * sp.pitch * 4, cov = (size_t)max_g * SS * 4;
    const size_t reg_slot = ((alias ? std::max(region, cov) : region) + 15) & ~(size_t)15;
    const size_t cov_slot = alias ? 0 : (cov + 15) & ~(size_t)15;
    sp.off_reg = fpi * sp.raw_bytes;
    sp.off_z = sp.off_reg + fpi * reg_slot;
    sp.off_t = sp.off_z + fpi * cov_slot;
    sp.total = sp.off_t;
    sp.stats_off = sp.raw_bytes;
    sp.stats_total = sp.stats_off + (size_t)S * sp.pitch * (dtype == VB_U16 ? 8 + 4 : 8 + 8);
    return sp;
}

size_t zncc_smem_bytes(int patch, int radius, int max_g, int max_wu, int dtype) {
    SmemPlan sp = zncc_smem(patch, radius, max_g, max_wu, dtype);
    return std::max(sp.total, sp.stats_total);
}

size_t zncc_search_smem_bytes(int patch, int radius, int max_g, int max_wu, int dtype) {
    return zncc_smem(patch, radius, max_g, max_wu, dtype).total;
}

int launch_motion(const Templates& t, int h, int w, int patch, int radius, const void* frames, int dtype,
                  int64_t n_frames, int subpixel, vb_motion* vectors, double* scores, cudaStream_t s) {
    if (n_frames <= 0) return VB_OK;
    NvtxRange nv("motion search");
    const int S = 2 * radius + 1, SS = S * S;
    bool fast = false;
    pick_kernel(patch, S, 1, &fast);
    // frames per search iteration: two when that packs the (frame, patch, dy)
    // items into whole warps noticeably better and both frames fit
    const int nch = fast ? 1 : (S + kGenericDXB - 1) / kGenericDXB;
    const int items1 = t.max_g * S * nch;
    int fpi = 1;
    if (fast && 2 * items1 <= 288) {
        const double e1 = (double)items1 / (((items1 + 31) / 32) * 32);
        const double e2 = (double)(2 * items1) / (((2 * items1 + 31) / 32) * 32);
        // measured on C2 (G = 8, S = 17): 94 % vs 85 % lanes did not pay for
        // half the resident CTAs, so two frames only for a large lane gain
        if (e2 > e1 + 0.15 && zncc_smem(patch, radius, t.max_g, t.max_wu, dtype, 2, true, t.pitch).total <= 112 * 1024)
            fpi = 2;
    }
    const int force_fpi = knob("VB_FPI", 0);  // experiment
    if (fast && (force_fpi == 1 || force_fpi == 2)) fpi = force_fpi;
    // S = 17: half-warp per patch with the shared middle row (cross_row_split17)
    bool split = fast && patch == 21 && S == 17 && fpi == 1 && !knob("VB_NO_SPLIT", 0);
    // paired split kernel: each thread carries two frames through FFMA2 (half the FMA
    // instructions, 226 registers, twice the shared memory per CTA: 2 CTAs per SM).
    // Measured on C2: 6.62 -> 6.54 ms per 4000 frames; the issue rate drops from 82 % to
    // 51 % and the FMA pipe (2 cycles per FFMA2) becomes the limiter inside the cross phase
    const bool pair = split && knob("VB_SPLIT_PAIR", 1) == 1 &&
                      zncc_smem(patch, radius, t.max_g, t.max_wu, dtype, 2, true, t.pitch).total +
                              2 * (size_t)t.max_g * ((S * S + 3) & ~3) * 4 <= 112 * 1024;
    if (pair) fpi = 2;
    // (measured: prefetching 8, 12 or 16 window samples instead of 4 made no difference)
    KernelFn fn = pair    ? zncc_group_kernel<21, 17, 2, true>
                  : split ? zncc_group_kernel<21, 17, 1, true>
                          : pick_kernel(patch, S, fpi, &fast);
    void (*stats_fn)(ZnccArgs, CUtensorMap) =
        patch == 21 ? (dtype == VB_U16 ? zncc_stats_kernel<true, 21> : zncc_stats_kernel<false, 21>)
                    : (dtype == VB_U16 ? zncc_stats_kernel<true, 0> : zncc_stats_kernel<false, 0>);
    if (patch == 21 && dtype == VB_U16 && !knob("VB_NO_STATS_S", 0)) {  // compile-time S: unrolled horizontal chains
        if (S == 17) stats_fn = zncc_stats_kernel<true, 21, 17>;
        if (S == 21) stats_fn = zncc_stats_kernel<true, 21, 21>;
        if (S == 25) stats_fn = zncc_stats_kernel<true, 21, 25>;
        if (S == 11) stats_fn = zncc_stats_kernel<true, 21, 11>;
    }
    // tensor-core cross sums (zncc_mma.cu, experiment build) + combining statistics kernel
#ifdef VB_EXPERIMENTS
    const bool mma = dtype == VB_U16 && t.t16 != nullptr && mma_supported(patch, radius, dtype);
    if (mma) {
        stats_fn = zncc_stats_kernel<true, 0, 0, true>;
        if (patch == 21 && !knob("VB_NO_STATS_S", 0)) {
            if (S == 17) stats_fn = zncc_stats_kernel<true, 21, 17, true>;
            if (S == 21) stats_fn = zncc_stats_kernel<true, 21, 21, true>;
            if (S == 25) stats_fn = zncc_stats_kernel<true, 21, 25, true>;
            if (S == 11) stats_fn = zncc_stats_kernel<true, 21, 11, true>;
        } else if (patch == 21) {
            stats_fn = zncc_stats_kernel<true, 21, 0, true>;
        }
    }
#else
    const bool mma = false;
#endif
    SmemPlan sp = zncc_smem(patch, radius, t.max_g, t.max_wu, dtype, fpi, fast, t.pitch);
    const int ss_pad_c = (S * S + 3) & ~3;
    const size_t sinv_off = (sp.stats_total + 15) & ~(size_t)15;
    if (mma) sp.stats_total = sinv_off + (size_t)t.max_g * ss_pad_c * sizeof(float);
    if (std::max(sp.total, sp.stats_total) > 227 * 1024)
        return fail(VB_EINVAL, "patch group does not fit in shared memory");
    // the search kernel also receives the group's inv rows by bulk copy (fast path, one frame per iteration)
    const int ss_pad_ = (S * S + 3) & ~3;
    // measured on C2 (split kernel): 7.05 -> 6.78 ms with the conversion batching; kept to the
    // split kernel -- the extra registers cost the generic S != 17 kernels a resident CTA
    const int inv_mode = knob("VB_INV_SMEM", -1);  // experiment: 0 off, 1 all kernels
    const bool want_inv = fast && (fpi == 1 || pair) && inv_mode != 0 && ((patch == 21 && S == 17) || inv_mode == 1);
    const size_t inv_buf = want_inv ? (size_t)fpi * t.max_g * ss_pad_ * sizeof(float) : 0;
    const size_t search_smem = ((sp.total + 15) & ~(size_t)15) + inv_buf;
    if (search_smem > 227 * 1024) return fail(VB_EINVAL, "patch group does not fit in shared memory");
    if (!mma) VB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)search_smem));
    VB_CUDA(cudaFuncSetAttribute(stats_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.stats_total));

    ZnccArgs a;
    a.dtype = dtype;
    a.hw = (int64_t)h * w;
    a.w = w;
    a.P = patch;
    a.R = radius;
    a.S = S;
    a.tp = t.tp;
    a.nch = fast ? 1 : (S + kGenericDXB - 1) / kGenericDXB;
    a.ss_pad = ss_pad_;
    a.off_inv = -1;
    // 2: compile-time-S kernels convert column-major (measured per search: C2 6.90 -> 6.62 ms per
    // 4000 frames, C3 14.74 -> 13.55 ms per 2000, C5 20.91 -> 19.81 ms per 1000)
    a.conv_batch = knob("VB_CONV_BATCH", 2);
    a.pitch_cap = sp.pitch;
    a.bw = sp.bw;
    a.bh = sp.bh;
    a.bhc = sp.bhc;
    a.n_patches = t.n;
    a.tmpl = t.tmpl;
    a.rvar = t.rvar;
    a.rmean = t.rmean;
    a.patch_col = t.patch_col;
    a.groups = t.groups;
    a.n_groups = t.n_groups;
    // one tensor map over the whole launch range (frames as the z dimension)
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    a.use_tma = !knob("VB_NO_TMA", 0) && make_frames_tmap(&tmap, frames, dtype, n_frames, h, w, sp.bhc, sp.bw) ? 1 : 0;
    // tensor-core path: boxes of one window row x 128 frames
    CUtensorMap tmap_mma;
    memset(&tmap_mma, 0, sizeof(tmap_mma));
#ifdef VB_EXPERIMENTS
    const bool use_mma = mma && a.use_tma && make_frames_tmap_sw128(&tmap_mma, frames, n_frames, h, w);
#else
    const bool use_mma = false;
#endif
    if (use_mma) {
        a.off_sinv = (int)sinv_off;
    } else if (mma) {  // no tensor map for this buffer: the FFMA path
        return fail(VB_EINVAL, "tensor-core ZNCC path needs 16-byte aligned uint16 frames");
    }

    a.rows = split ? 16 : S;
    const int items = (pair ? 1 : fpi) * t.max_g * a.rows * nch;
    // statistics kernel: one thread per union column (vertical chains), then
    // one per (patch, dy) row (horizontal chains)
    const int stats_threads = std::max(64, std::min(256, (std::max(t.max_wu, t.max_g * S) + 31) / 32 * 32));
    int threads = ((items + 31) / 32) * 32;
    threads = std::max(64, std::min(threads, fast ? 288 : 256));

    // frame batches bound the float64 partials + f32 inv buffers to ~1 GB
    const size_t per_frame_part = (size_t)t.n_groups * SS * sizeof(double);
    // (the tensor-core path keeps the window covariances in this buffer instead of inv)
    const size_t per_frame_inv = (size_t)t.n * a.ss_pad * sizeof(float);
    int64_t batch = std::max<int64_t>(1, (int64_t)(((size_t)1 << 30) / (per_frame_part + per_frame_inv)));
    const int force_batch = knob("VB_ZNCC_BATCH", 0);  // experiment: frames per stats+search pair
    if (force_batch > 0) batch = force_batch;
    batch = std::min(batch, n_frames);
    double* partial = nullptr;
    float* inv = nullptr;
    keep_pool();
    VB_CUDA(cudaMallocAsync(&partial, per_frame_part * batch, s));
    cudaError_t e0 = cudaMallocAsync(&inv, per_frame_inv * batch, s);
    if (e0 != cudaSuccess) {
        cudaFreeAsync(partial, s);
        return cuda_fail(e0, "cudaMallocAsync(inv)");
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int rc = VB_OK;
    for (int64_t f0 = 0; f0 < n_frames && rc == VB_OK; f0 += batch) {
        const int64_t nb = std::min(batch, n_frames - f0);
        a.frames = (const char*)frames + (size_t)f0 * a.hw * (dtype == VB_U16 ? 2 : 4);
        a.tma_z0 = (int)f0;
        a.n_frames = nb;
        a.partial = partial;
        a.inv = inv;
        a.cov = inv;
#ifdef VB_EXPERIMENTS
        if (use_mma) {
            rc = launch_zncc_mma(t, patch, radius, nb, (int)f0, tmap_mma, inv, a.ss_pad, s);
            if (rc) break;
        }
#endif
        // persistent CTAs: each walks frames y, y+gy, ... (about 8 frames per CTA)
        const int64_t want_y = std::max<int64_t>(1, (int64_t)sms * 8 * 4 / std::max(1, t.n_groups));
        const unsigned gy = (unsigned)std::min<int64_t>(std::min<int64_t>(nb, 65535), std::max<int64_t>(want_y, (nb + 7) / 8));
        dim3 grid(t.n_groups, gy);
        {
            ZnccArgs as = a;
            as.off_reg = 0;
            as.off_z = (int)sp.stats_off;
            ProfScope ps(kProfOther, s);
            stats_fn<<<grid, stats_threads, sp.stats_total, s>>>(as, tmap);
        }
        launches().fetch_add(1, std::memory_order_relaxed);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { rc = cuda_fail(e, "zncc_stats_kernel"); break; }
        if (!use_mma) {
            {
                ZnccArgs as = a;
                as.off_reg = (int)sp.off_reg;
                as.off_z = (int)sp.off_z;
                as.off_t = (int)sp.off_t;
                as.off_inv = (inv_buf && a.use_tma) ? (int)((sp.total + 15) & ~(size_t)15) : -1;
                ProfScope ps(kProfZncc, s);
                fn<<<grid, threads, search_smem, s>>>(as, tmap);
            }
            launches().fetch_add(1, std::memory_order_relaxed);
            e = cudaGetLastError();
            if (e != cudaSuccess) { rc = cuda_fail(e, "zncc_group_kernel"); break; }
        }
        const int fin_blocks = (int)std::min<int64_t>(nb, 148 * 8);
        {
            ProfScope ps(kProfFinalize, s);
            finalize_kernel<<<fin_blocks, 256, SS * sizeof(double), s>>>(
                partial, t.n_groups, S, t.n, nb, subpixel, vectors + f0, scores ? scores + (size_t)f0 * SS : nullptr);
        }
        launches().fetch_add(1, std::memory_order_relaxed);
        e = cudaGetLastError();
        if (e != cudaSuccess) { rc = cuda_fail(e, "finalize_kernel"); break; }
    }
    cudaFreeAsync(partial, s);
    cudaFreeAsync(inv, s);
    return rc;
}

}  // namespace vb
