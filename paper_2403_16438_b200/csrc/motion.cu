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
//    S*P FFMAs.
//  * Per-CTA partial sums of ZNCC over its patches are written in fixed
//    order (float64) and a finalize kernel sums the groups in fixed order,
//    divides by N and runs the tie-broken argmax + quadratic fit: fully
//    deterministic, no atomics.
#include <math.h>

#include <algorithm>
#include <vector>

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
    const void* frames;
    int dtype;
    int64_t hw;
    int w;
    int P, R, S, tp;
    int dyc;  // dy rows per statistics chunk
    int nch;  // dx chunks per (patch, dy) item (1 on the fast path)
    int pitch_cap;
    int off_inv, off_reg, off_scr;  // shared-memory carve-up (bytes)
    const float* tmpl;
    const double* rvar;
    const double* rmean;
    const int32_t* patch_col;
    const PatchGroup* groups;
    int n_groups;
    int64_t n_frames;
    double* partial;  // [n_frames][n_groups][S*S]
};

constexpr int kGenericDXB = 8;

// Cross sums for one (patch, dy) row of S candidates, compile-time P and S.
template <int P, int S>
__device__ __forceinline__ void cross_row(const float* __restrict__ reg, int pitch, const float* __restrict__ trow0,
                                          int tp, float (&acc)[S]) {
#pragma unroll
    for (int d = 0; d < S; ++d) acc[d] = 0.0f;
#pragma unroll 1
    for (int yy = 0; yy < P; ++yy) {
        const float* fr = reg + yy * pitch;
        float win[S + P - 1];
#pragma unroll
        for (int i = 0; i < S + P - 1; ++i) win[i] = fr[i];
        const float4* trow = reinterpret_cast<const float4*>(trow0 + yy * tp);
#pragma unroll
        for (int q = 0; q < (P + 3) / 4; ++q) {
            const float4 t4 = trow[q];
            const float tv[4] = {t4.x, t4.y, t4.z, t4.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if (4 * q + k < P) {
#pragma unroll
                    for (int d = 0; d < S; ++d) acc[d] = fmaf(win[4 * q + k + d], tv[k], acc[d]);
                }
            }
        }
    }
}

template <int P_CT, int S_CT>
__global__ void __launch_bounds__(512, 1) zncc_group_kernel(ZnccArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int P = P_CT ? P_CT : a.P;
    const int S = S_CT ? S_CT : a.S;
    const int R = (S - 1) / 2;
    const int RH = P + 2 * R;
    const int tp = a.tp;
    const PatchGroup grp = a.groups[blockIdx.x];
    const int G = grp.count;
    const int wu = grp.wu;
    const int pitch = a.pitch_cap;  // odd, >= max wu
    const int SS = S * S;
    const double nn = (double)P * (double)P;

    // shared-memory carve-up (zncc_smem)
    float* s_tmpl = reinterpret_cast<float*>(smem);                   // [G][P][tp]
    float* s_inv = reinterpret_cast<float*>(smem + a.off_inv);        // [G][S*S]
    float* s_reg = reinterpret_cast<float*>(smem + a.off_reg);        // [RH][pitch]
    double* s_scr = reinterpret_cast<double*>(smem + a.off_scr);      // stats / z scratch
    const int tid = threadIdx.x, nth = blockDim.x;

    // templates + per-patch constants are frame independent
    {
        const float4* src = reinterpret_cast<const float4*>(a.tmpl + (size_t)grp.first * P * tp);
        float4* dst = reinterpret_cast<float4*>(s_tmpl);
        const int nv = G * P * tp / 4;
        for (int i = tid; i < nv; i += nth) dst[i] = src[i];
    }
    // Frame samples are staged centred on an integer c close to the group's
    // template level, so the f32 cross sums accumulate O(100) instead of
    // O(1000) products.  Integer samples stay exact, and the window variance
    // is shift invariant, so the float64 statistics use the centred samples
    // directly.  (Small-valued float data, |mean| < 64, is left uncentred.)
    float cg;
    {
        double m = 0.0;
        for (int p = 0; p < G; ++p) m += a.rmean[grp.first + p];
        m /= (double)G;
        cg = fabs(m) >= 64.0 ? (float)rint(m) : 0.0f;
    }

    for (int64_t t = blockIdx.y; t < a.n_frames; t += gridDim.y) {
        __syncthreads();  // previous frame fully consumed
        // ---- stage the union window (raw samples, f32) ----
        const int64_t fbase = t * a.hw;
        for (int i = tid; i < RH * wu; i += nth) {
            const int r = i / wu, c = i - r * wu;
            s_reg[r * pitch + c] =
                __fsub_rn(load_sample(a.frames, a.dtype, fbase + (int64_t)(grp.y0 + r) * a.w + grp.x0 + c), cg);
        }
        __syncthreads();

        // ---- window statistics: float64 sliding sums, DYC rows of dy at a time ----
        for (int d0 = 0; d0 < S; d0 += a.dyc) {
            const int nd = min(a.dyc, S - d0);
            double* v1 = s_scr;                 // [dyc][wu]
            double* v2 = s_scr + a.dyc * wu;    // [dyc][wu]
            for (int c = tid; c < wu; c += nth) {
                double s1 = 0.0, s2 = 0.0;
                for (int yy = 0; yy < P; ++yy) {
                    const double f = (double)s_reg[(d0 + yy) * pitch + c];
                    s1 += f;
                    s2 += f * f;
                }
                v1[c] = s1;
                v2[c] = s2;
                for (int k = 1; k < nd; ++k) {
                    const double fo = (double)s_reg[(d0 + k - 1) * pitch + c];
                    const double fi = (double)s_reg[(d0 + k - 1 + P) * pitch + c];
                    s1 += fi - fo;
                    s2 += fi * fi - fo * fo;
                    v1[k * wu + c] = s1;
                    v2[k * wu + c] = s2;
                }
            }
            __syncthreads();
            for (int it = tid; it < G * nd; it += nth) {
                const int p = it / nd, k = it - p * nd;
                const int col = a.patch_col[grp.first + p];
                const double rv = a.rvar[grp.first + p];
                const double* r1 = v1 + k * wu + col;
                const double* r2 = v2 + k * wu + col;
                double h1 = 0.0, h2 = 0.0;
                for (int xx = 0; xx < P; ++xx) {
                    h1 += r1[xx];
                    h2 += r2[xx];
                }
                float* out = s_inv + (size_t)p * SS + (size_t)(d0 + k) * S;
                for (int dx = 0; dx < S; ++dx) {
                    const double fvar = h2 - h1 * h1 / nn;  // kernels.py:67
                    out[dx] = (rv > 0.0 && fvar > 0.0) ? (float)(1.0 / sqrt(fvar * rv)) : 0.0f;
                    if (dx + 1 < S) {
                        h1 += r1[dx + P] - r1[dx];
                        h2 += r2[dx + P] - r2[dx];
                    }
                }
            }
            __syncthreads();
        }

        // ---- cross term + normalisation ----
        float* zbuf = reinterpret_cast<float*>(s_scr);  // [G][S*S]
        const int nitems = G * S * a.nch;
        for (int it = tid; it < nitems; it += nth) {
            const int dy = it % S;
            const int pc = it / S;
            const int p = pc / a.nch, ch = pc - p * a.nch;
            const int col = a.patch_col[grp.first + p];
            const float* reg = s_reg + dy * pitch + col;
            const float* trow0 = s_tmpl + (size_t)p * P * tp;
            const float* inv = s_inv + (size_t)p * SS + dy * S;
            float* z = zbuf + (size_t)p * SS + dy * S;
            if constexpr (P_CT != 0 && S_CT != 0) {
                float acc[S_CT];
                cross_row<P_CT, S_CT>(reg, pitch, trow0, tp, acc);
#pragma unroll
                for (int d = 0; d < S_CT; ++d) z[d] = acc[d] * inv[d];
            } else {
                float acc[kGenericDXB];
#pragma unroll
                for (int d = 0; d < kGenericDXB; ++d) acc[d] = 0.0f;
                const int dx0 = ch * kGenericDXB;
                for (int yy = 0; yy < P; ++yy) {
                    const float* fr = reg + yy * pitch + dx0;
                    const float* trow = trow0 + yy * tp;
                    for (int xx = 0; xx < P; ++xx) {
                        const float tv = trow[xx];
#pragma unroll
                        for (int d = 0; d < kGenericDXB; ++d) acc[d] = fmaf(fr[xx + d], tv, acc[d]);
                    }
                }
#pragma unroll
                for (int d = 0; d < kGenericDXB; ++d)
                    if (dx0 + d < S) z[dx0 + d] = acc[d] * inv[dx0 + d];
            }
        }
        __syncthreads();
        double* part = a.partial + ((size_t)t * a.n_groups + blockIdx.x) * SS;
        for (int c = tid; c < SS; c += nth) {
            double s = 0.0;
            for (int p = 0; p < G; ++p) s += (double)zbuf[(size_t)p * SS + c];
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
using KernelFn = void (*)(ZnccArgs);

template <int S>
static KernelFn fast_kernel_for() {
    return zncc_group_kernel<21, S>;
}

static KernelFn pick_kernel(int P, int S, bool* fast) {
    *fast = true;
    if (P == 21) {
        switch (S) {
            case 3: return fast_kernel_for<3>();
            case 5: return fast_kernel_for<5>();
            case 7: return fast_kernel_for<7>();
            case 9: return fast_kernel_for<9>();
            case 11: return fast_kernel_for<11>();
            case 13: return fast_kernel_for<13>();
            case 15: return fast_kernel_for<15>();
            case 17: return fast_kernel_for<17>();
            case 19: return fast_kernel_for<19>();
            case 21: return fast_kernel_for<21>();
            case 23: return fast_kernel_for<23>();
            case 25: return fast_kernel_for<25>();
            default: break;
        }
    }
    *fast = false;
    return zncc_group_kernel<0, 0>;
}

struct SmemPlan {
    size_t off_inv, off_reg, off_scr, total;
    int pitch, dyc;
};

static SmemPlan zncc_smem(int P, int R, int tp, int max_g, int max_wu) {
    const int S = 2 * R + 1, SS = S * S, RH = P + 2 * R;
    SmemPlan sp;
    sp.pitch = max_wu | 1;
    sp.dyc = std::min(S, 4);
    size_t off = 0;
    off += (size_t)max_g * P * tp * 4;  // templates
    sp.off_inv = off;
    off += (size_t)max_g * SS * 4;      // inv
    off = (off + 15) & ~(size_t)15;
    sp.off_reg = off;
    off += (size_t)RH * sp.pitch * 4;
    off = (off + 15) & ~(size_t)15;
    sp.off_scr = off;
    size_t scr = std::max((size_t)2 * sp.dyc * max_wu * 8, (size_t)max_g * SS * 4);
    off += scr;
    sp.total = off;
    return sp;
}

size_t zncc_smem_bytes(int patch, int radius, int max_g, int max_wu) {
    return zncc_smem(patch, radius, (patch + 3) & ~3, max_g, max_wu).total;
}

int launch_motion(const Templates& t, int h, int w, int patch, int radius, const void* frames, int dtype,
                  int64_t n_frames, int subpixel, vb_motion* vectors, double* scores, cudaStream_t s) {
    (void)h;
    if (n_frames <= 0) return VB_OK;
    const int S = 2 * radius + 1, SS = S * S;
    bool fast = false;
    KernelFn fn = pick_kernel(patch, S, &fast);
    SmemPlan sp = zncc_smem(patch, radius, t.tp, t.max_g, t.max_wu);
    if (sp.total > 227 * 1024) return fail(VB_EINVAL, "patch group does not fit in shared memory");
    VB_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sp.total));

    ZnccArgs a;
    a.off_inv = (int)sp.off_inv;
    a.off_reg = (int)sp.off_reg;
    a.off_scr = (int)sp.off_scr;
    a.frames = frames;
    a.dtype = dtype;
    a.hw = (int64_t)h * w;
    a.w = w;
    a.P = patch;
    a.R = radius;
    a.S = S;
    a.tp = t.tp;
    a.dyc = sp.dyc;
    a.nch = fast ? 1 : (S + kGenericDXB - 1) / kGenericDXB;
    a.pitch_cap = sp.pitch;
    a.tmpl = t.tmpl;
    a.rvar = t.rvar;
    a.rmean = t.rmean;
    a.patch_col = t.patch_col;
    a.groups = t.groups;
    a.n_groups = t.n_groups;

    const int items = t.max_g * S * a.nch;
    int threads = ((items + 31) / 32) * 32;
    threads = std::max(64, std::min(threads, 512));

    // frame batches bound the float64 partial buffer to ~256 MB
    const size_t per_frame = (size_t)t.n_groups * SS * sizeof(double);
    int64_t batch = std::max<int64_t>(1, (int64_t)((256u << 20) / per_frame));
    batch = std::min(batch, n_frames);
    double* partial = nullptr;
    keep_pool();
    VB_CUDA(cudaMallocAsync(&partial, per_frame * batch, s));
    int rc = VB_OK;
    for (int64_t f0 = 0; f0 < n_frames && rc == VB_OK; f0 += batch) {
        const int64_t nb = std::min(batch, n_frames - f0);
        a.frames = (const char*)frames + (size_t)f0 * a.hw * (dtype == VB_U16 ? 2 : 4);
        a.n_frames = nb;
        a.partial = partial;
        dim3 grid(t.n_groups, (unsigned)std::min<int64_t>(nb, 65535));
        {
            ProfScope ps(kProfZncc, s);
            fn<<<grid, threads, sp.total, s>>>(a);
        }
        launches().fetch_add(1, std::memory_order_relaxed);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) { rc = cuda_fail(e, "zncc_group_kernel"); break; }
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
    return rc;
}

}  // namespace vb
