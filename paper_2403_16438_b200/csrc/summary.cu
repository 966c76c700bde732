// Motion warp + per-block summary images (sm_100a).
//
// Reference algorithm (paths under /root/reference/pkg/src/voltseg):
//   warp                motion.py:163-200 translate/_translate_int, :235-240, :244-248
//   blocks              summarize.py:44-52 split_segments (ceil(T/L) blocks)
//   spatial summary     summarize.py:55-57  (float64 sequential mean -> f32)
//   smoothing           summarize.py:70-73  (scipy gaussian_filter1d, sigma=3,
//                       radius 9, mode "reflect", H pass then W pass, float64
//                       accumulation, f32 rounding after each pass)
//   temporal summary    summarize.py:76-92  (max - median over time; midpoint
//                       median for even counts)
//
// B200 design:
//  K3 warp_smooth_kernel: one CTA per (block, 32x64 pixel tile) walks the
//     block's frames in order.  Per frame it evaluates the corrected frame on
//     the tile plus a reflect-mapped 9-pixel halo straight from the raw
//     (u16/f32) frame, keeps the float64 running spatial sum of its own pixels
//     in registers, optionally streams the corrected tile out, and runs the
//     two separable 19-tap passes in shared memory (float64 accumulate in
//     scipy's symmetric-pair order, unfused mul/add).  The smoothed tile is
//     written time-major for K4.
//  K4 median_kernel: one CTA per (block, 16 consecutive pixels) stages the
//     block's smoothed column in shared memory; one warp per pixel holds up to
//     32 samples per lane in registers and selects the exact median by radix
//     bisection on the float bit pattern (non-negative floats order like
//     uint32), with warp REDUX counts -- no sorting, no atomics.
#include <math.h>

#include <algorithm>

#include <stdlib.h>
#include <string.h>

#include <type_traits>

#include "tma.cuh"
#include "vb.cuh"

namespace vb {

// ------------------------------------------------------------------ warp
struct WarpOp {
    int mode;  // 0 identity, 1 integer shift, 2 bilinear
    int ix, iy;
    float fx, fy, omx, omy;
};

__device__ __forceinline__ WarpOp make_warp(const vb_motion* vec, int64_t t) {
    WarpOp op;
    op.mode = 0;
    op.ix = op.iy = 0;
    op.fx = op.fy = 0.f;
    op.omx = op.omy = 1.f;
    if (!vec) return op;  // identity: the bilinear formula with zero weights returns the sample
    const vb_motion v = vec[t];
    const double vx = (double)v.dx + v.sub_dx, vy = (double)v.dy + v.sub_dy;  // MotionVector.x/.y
    if (vx == 0.0 && vy == 0.0) return op;                                     // motion.py:237-238
    const double sx = -vx, sy = -vy;                                           // translate(f, -x, -y)
    const double x0 = floor(sx), y0 = floor(sy);
    op.ix = (int)x0;
    op.iy = (int)y0;
    if (sx == x0 && sy == y0) {  // motion.py:166-167 integer path
        op.mode = 1;
        return op;
    }
    op.mode = 2;
    op.fx = (float)(sx - x0);  // frame.dtype.type(dx - x0)
    op.fy = (float)(sy - y0);
    op.omx = __fsub_rn(1.0f, op.fx);
    op.omy = __fsub_rn(1.0f, op.fy);
    return op;
}

// out[y,x] of translate(frame, sx, sy): samples frame[y - y0 (+1)][x - x0 (+1)]
// with clamping; f32 ops in numpy's order, never fused.
__device__ __forceinline__ float warp_sample(const void* f, int dtype, int64_t base, int h, int w, const WarpOp& op,
                                             int y, int x) {
    if (op.mode == 0) return load_sample(f, dtype, base + (int64_t)y * w + x);
    const int ya = clampi(y - op.iy, 0, h - 1), xa = clampi(x - op.ix, 0, w - 1);
    if (op.mode == 1) return load_sample(f, dtype, base + (int64_t)ya * w + xa);
    const int yc = clampi(y - op.iy - 1, 0, h - 1), xb = clampi(x - op.ix - 1, 0, w - 1);
    const float a = load_sample(f, dtype, base + (int64_t)ya * w + xa);
    const float b = load_sample(f, dtype, base + (int64_t)ya * w + xb);
    const float c = load_sample(f, dtype, base + (int64_t)yc * w + xa);
    const float d = load_sample(f, dtype, base + (int64_t)yc * w + xb);
    const float top = __fadd_rn(__fmul_rn(op.omx, a), __fmul_rn(op.fx, b));
    const float bot = __fadd_rn(__fmul_rn(op.omx, c), __fmul_rn(op.fx, d));
    return __fadd_rn(__fmul_rn(op.omy, top), __fmul_rn(op.fy, bot));
}

static int launch_correct_rows(const void* frames, int dtype, int64_t n, int h, int w, const vb_motion* vec,
                               const float* gain, float* out, cudaStream_t s);

// Corrected frames (translate, motion.py:163-200; + A17 gain, opt-in):
// the row-strip kernel correct_rows_kernel below.
int launch_correct(const void* frames, int dtype, int64_t n, int h, int w, const vb_motion* vec,
                   const float* gain, float* out, cudaStream_t s) {
    if (n <= 0) return VB_OK;
    return launch_correct_rows(frames, dtype, n, h, w, vec, gain, out, s);
}

// Trace extraction fused with the warp: per (ROI, frame)
// the corrected samples of the ROI's pixels only are interpolated from the
// raw frame (warp_sample, + shading gain) and averaged in float64 in
// traces_kernel's lane order and shuffle tree, so the traces equal those of
// vb_extract_traces on the corrected video without materialising it.
__global__ void traces_raw_kernel(const void* __restrict__ frames, int dtype, int64_t n, int h, int w,
                                  const vb_motion* __restrict__ vec, const float* __restrict__ gain,
                                  const int32_t* __restrict__ roi_ptr, const int32_t* __restrict__ roi_idx,
                                  double* __restrict__ out) {
    const int roi = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int p0 = roi_ptr[roi], p1 = roi_ptr[roi + 1];
    const double inv_n = 1.0 / (double)(p1 - p0);
    const int64_t hw = (int64_t)h * w;
    for (int64_t t = (int64_t)blockIdx.y * nw + warp; t < n; t += (int64_t)gridDim.y * nw) {
        const WarpOp op = make_warp(vec, t);
        double s = 0.0;
        for (int i = p0 + lane; i < p1; i += 32) {
            const int idx = roi_idx[i], y = idx / w, x = idx - y * w;
            float v = warp_sample(frames, dtype, t * hw, h, w, op, y, x);
            if (gain) v = __fdiv_rn(v, __ldg(gain + idx));
            s += (double)v;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[(int64_t)roi * n + t] = s * inv_n;
    }
}

int launch_traces_raw(const void* frames, int dtype, int64_t n, int h, int w, const vb_motion* vec,
                      const float* gain, const int32_t* roi_ptr, const int32_t* roi_idx, int n_rois, double* out,
                      cudaStream_t s) {
    if (n <= 0 || n_rois <= 0) return VB_OK;
    const int threads = 256, warps = threads / 32;
    const int64_t ychunks = std::min<int64_t>((n + warps - 1) / warps, 65535);
    dim3 grid((unsigned)n_rois, (unsigned)ychunks);
    {
        ProfScope ps(kProfOther, s);
        traces_raw_kernel<<<grid, threads, 0, s>>>(frames, dtype, n, h, w, vec, gain, roi_ptr, roi_idx, out);
    }
    VB_LAUNCHED();
    return VB_OK;
}

// ------------------------------------------------------------------ K3
constexpr int kTY = 32, kTX = 64, kK3Threads = 256;
constexpr int kMaxWR = 16;

struct Weights {
    double w[2 * kMaxWR + 1];  // centre at index wr (scipy weights reversed == same, symmetric)
};

struct K3Args {
    const void* frames;
    int dtype;
    const vb_motion* vec;  // may be null: frames are taken as they are (already corrected)
    int64_t n;             // frames in this launch
    int h, w, wr;
    Weights wt;
    float* corrected;  // [n][h][w] or null
    float* smoothed;   // [n][h][w]
    const float* gain; // [h][w] shading gain (A17, opt-in): corrected = warped / gain; null = off
};

// scipy correlate1d symmetric kernel: o = x0*w0; for j=-r..-1: o += (x[j]+x[-j])*w[j]
// (float64, unfused multiply/add as in the compiled C loop).
__device__ __forceinline__ double corr_sym(const double* line, int stride, const double* wc, int r) {
    double o = __dmul_rn(line[0], wc[0]);
    for (int j = -r; j < 0; ++j) {
        const double pr = __dadd_rn(line[j * stride], line[-j * stride]);
        o = __dadd_rn(o, __dmul_rn(pr, wc[j]));
    }
    return o;
}

static size_t k3_smem_bytes(int wr) {
    const int EH = kTY + 2 * wr, EW = kTX + 2 * wr, EWP = EW | 1;
    const size_t c = (size_t)EH * EWP * sizeof(double);
    const size_t v = std::max((size_t)kTY * EWP * sizeof(double), (size_t)(EH + 1) * (EW + 1) * sizeof(float));
    return c + v;
}

// One CTA per (frame, 32x64 tile).  Per frame: reflect/clamp index tables for
// the tile + halo, the raw source box staged in shared memory, the corrected
// samples (float32 bilinear in numpy's operation order; identity and integer
// shifts are the same formula with zero weights), then the two separable
// float64 passes.  The raw box aliases the vertical-pass buffer.
// Register-blocked symmetric pass: VR consecutive outputs along `stride` from
// VR + 2*WR loaded samples (3.25 loads/output instead of 19), same float64
// operation order as corr_sym.
template <int WR, int VR>
__device__ __forceinline__ void corr_sym_block(const double* line, int stride, const double* wc, double (&o)[VR]) {
    double x[VR + 2 * WR];
#pragma unroll
    for (int i = 0; i < VR + 2 * WR; ++i) x[i] = line[i * stride];
#pragma unroll
    for (int j = 0; j < VR; ++j) {
        double acc = __dmul_rn(x[j + WR], wc[0]);
#pragma unroll
        for (int k = WR; k >= 1; --k) acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(x[j + WR - k], x[j + WR + k]), wc[-k]));
        o[j] = acc;
    }
}

template <int WR_CT>
__global__ void __launch_bounds__(kK3Threads, 3) warp_smooth_kernel(K3Args a) {
    extern __shared__ __align__(16) double sm3[];
    const int wr = WR_CT ? WR_CT : a.wr;
    const int EH = kTY + 2 * wr, EW = kTX + 2 * wr, EWP = EW | 1;
    double* sC = sm3;                                  // [EH][EWP] corrected tile + halo
    double* sV = sm3 + (size_t)EH * EWP;               // [kTY][EWP] after the H pass
    float* sRaw = reinterpret_cast<float*>(sV);        // raw source box (before sV is written)
    __shared__ double s_w[2 * kMaxWR + 1];
    __shared__ int s_ra[kTY + 2 * kMaxWR], s_rc[kTY + 2 * kMaxWR];
    __shared__ int s_xa[kTX + 2 * kMaxWR], s_xb[kTX + 2 * kMaxWR];
    __shared__ int s_gy[kTY + 2 * kMaxWR], s_gx[kTX + 2 * kMaxWR];  // reflected output coordinates
    __shared__ int s_box[4];
    const int tid = threadIdx.x;
    if (tid < 2 * wr + 1) s_w[tid] = a.wt.w[tid];
    const double* wc = s_w + wr;
    const int ty0 = blockIdx.y * kTY, tx0 = blockIdx.x * kTX;
    const int64_t hw = (int64_t)a.h * a.w;

    for (int64_t t = blockIdx.z; t < a.n; t += gridDim.z) {
        const WarpOp op = make_warp(a.vec, t);
        if (tid < 4) s_box[tid] = (tid & 1) ? -1 : 0x7fffffff;
        __syncthreads();
        // 1. index tables: ext row ey -> source rows (ya, yc) of translate's a/c taps
        for (int i = tid; i < EH + EW; i += kK3Threads) {
            if (i < EH) {
                const int y = reflect_index(ty0 - wr + i, a.h);
                const int ya = clampi(y - op.iy, 0, a.h - 1), yc = clampi(y - op.iy - 1, 0, a.h - 1);
                s_gy[i] = y;
                s_ra[i] = ya;
                s_rc[i] = yc;
                atomicMin(&s_box[0], min(ya, yc));
                atomicMax(&s_box[1], max(ya, yc));
            } else {
                const int e = i - EH;
                const int x = reflect_index(tx0 - wr + e, a.w);
                const int xa = clampi(x - op.ix, 0, a.w - 1), xb = clampi(x - op.ix - 1, 0, a.w - 1);
                s_gx[e] = x;
                s_xa[e] = xa;
                s_xb[e] = xb;
                atomicMin(&s_box[2], min(xa, xb));
                atomicMax(&s_box[3], max(xa, xb));
            }
        }
        __syncthreads();
        const int by0 = s_box[0], bx0 = s_box[2];
        const int bh = s_box[1] - by0 + 1, bw = s_box[3] - bx0 + 1;
        // 2. stage the raw source box (<= (EH+1) x (EW+1) samples)
        const int64_t fb = t * hw;
        for (int i = tid; i < bh * bw; i += kK3Threads) {
            const int r = i / bw, c = i - r * bw;
            sRaw[i] = load_sample(a.frames, a.dtype, fb + (int64_t)(by0 + r) * a.w + bx0 + c);
        }
        __syncthreads();
        // 3. corrected samples on tile + halo
        for (int i = tid; i < EH * EW; i += kK3Threads) {
            const int ey = i / EW, ex = i - ey * EW;
            const float* ra = sRaw + (s_ra[ey] - by0) * bw - bx0;
            const float* rc = sRaw + (s_rc[ey] - by0) * bw - bx0;
            const int xa = s_xa[ex], xb = s_xb[ex];
            const float top = __fadd_rn(__fmul_rn(op.omx, ra[xa]), __fmul_rn(op.fx, ra[xb]));
            const float bot = __fadd_rn(__fmul_rn(op.omx, rc[xa]), __fmul_rn(op.fx, rc[xb]));
            float v = __fadd_rn(__fmul_rn(op.omy, top), __fmul_rn(op.fy, bot));
            if (a.gain) v = __fdiv_rn(v, __ldg(a.gain + (int64_t)s_gy[ey] * a.w + s_gx[ex]));
            sC[ey * EWP + ex] = (double)v;
        }
        __syncthreads();
        // 4. corrected output (interior) and the H (vertical) pass, rounded to f32
        if (a.corrected) {
            for (int i = tid; i < kTY * kTX; i += kK3Threads) {
                const int ly = i / kTX, lx = i - ly * kTX;
                const int gy = ty0 + ly, gx = tx0 + lx;
                if (gy < a.h && gx < a.w) a.corrected[fb + (int64_t)gy * a.w + gx] = (float)sC[(ly + wr) * EWP + lx + wr];
            }
        }
        if constexpr (WR_CT > 0) {
            constexpr int VR = 4, HR = 8;
            for (int i = tid; i < (kTY / VR) * EW; i += kK3Threads) {
                const int c = i % EW, r0 = (i / EW) * VR;
                double o[VR];
                corr_sym_block<WR_CT, VR>(sC + r0 * EWP + c, EWP, wc, o);
#pragma unroll
                for (int j = 0; j < VR; ++j) sV[(r0 + j) * EWP + c] = (double)(float)o[j];
            }
            __syncthreads();
            // 5. W pass -> smoothed frame (time-major)
            for (int i = tid; i < kTY * (kTX / HR); i += kK3Threads) {
                const int ly = i / (kTX / HR), lx0 = (i % (kTX / HR)) * HR;
                double o[HR];
                corr_sym_block<WR_CT, HR>(sV + ly * EWP + lx0, 1, wc, o);
                const int gy = ty0 + ly;
#pragma unroll
                for (int j = 0; j < HR; ++j) {
                    const int gx = tx0 + lx0 + j;
                    if (gy < a.h && gx < a.w) a.smoothed[fb + (int64_t)gy * a.w + gx] = (float)o[j];
                }
            }
        } else {
            for (int i = tid; i < kTY * EW; i += kK3Threads) {
                const int r = i / EW, c = i - r * EW;
                sV[r * EWP + c] = (double)(float)corr_sym(sC + (r + wr) * EWP + c, EWP, wc, wr);
            }
            __syncthreads();
            // 5. W pass -> smoothed frame (time-major)
            for (int i = tid; i < kTY * kTX; i += kK3Threads) {
                const int ly = i / kTX, lx = i - ly * kTX;
                const int gy = ty0 + ly, gx = tx0 + lx;
                const float sv = (float)corr_sym(sV + ly * EWP + lx + wr, 1, wc, wr);
                if (gy < a.h && gx < a.w) a.smoothed[fb + (int64_t)gy * a.w + gx] = sv;
            }
        }
        __syncthreads();
    }
}

// Rows (or columns) of the source frame that the corrected tile + halo
// touches: reflect(lo .. hi-1) shifted by -i0 and -(i0+1), clamped.  Exact
// for a single reflection (n >= the halo); otherwise the whole axis.
__device__ __forceinline__ void src_span(int lo, int hi, int n, int i0, int& a0, int& a1) {
    int mn, mx;
    if (-lo <= n && hi - n <= n) {
        mn = lo < 0 ? 0 : (hi > n ? min(lo, 2 * n - hi) : lo);
        mx = hi > n ? n - 1 : (lo < 0 ? max(hi - 1, -lo - 1) : hi - 1);
    } else {
        mn = 0;
        mx = n - 1;
    }
    a0 = clampi(mn - i0 - 1, 0, n - 1);
    a1 = clampi(mx - i0, 0, n - 1);
}

// K3 v2 (fused warp + smoothing; the fallback of the split form below for
// widths that are not a multiple of 4 and frames under 10 rows/columns):
// one CTA per (tile, frame slice), persistent over frames; the elected thread
// issues the next frame's raw box by TMA (16-byte aligned start, zero-filled
// out of bounds).  Restructured for few issued instructions:
//  A1 the bilinear warp is separable -- translate's top/bottom rows are
//     omx*a + fx*b of source rows ra and rc, and row y+1's bottom row is row
//     y's top row -- so each raw-box row is interpolated horizontally once
//     (f32, unfused, numpy's order) into sH, aliased onto sV;
//  A2 corrected = omy*sH[ra] + fy*sH[rc] (+ shading), written once as f32
//     output and once as f64 into sC;
//  B  vertical pass: one thread per (column, third of the tile's rows), up to
//     11 outputs from 29 loaded samples (2.6 loads/output instead of 5.5);
//  C  horizontal pass: 8 outputs per thread from 26 samples, float4 stores.
// The next frame's box is issued right after A1 (raw box consumed).
constexpr int kVR2 = 11;  // vertical-pass outputs per thread: kTY = 11 + 11 + 10
#ifndef VB_K3_INTERLEAVE
#define VB_K3_INTERLEAVE 1
#endif
#ifndef VB_K3V2_MIN_BLOCKS
#define VB_K3V2_MIN_BLOCKS 3  // measured: 80 regs x 3 CTAs beats a 64-reg cap (spills) x 4
#endif
constexpr int kK3V2MinBlocks = VB_K3V2_MIN_BLOCKS;
template <int WR, bool U16>
static size_t k3_v2_smem_bytes() {  // raw box | sC f32 [EH][EWP] | sV f32 [kTY][EWP] aliased by sH f32 [EH+1][EW]
    constexpr int EH = kTY + 2 * WR, EW = kTX + 2 * WR, EWP = EW | 1;
    constexpr int ALN = U16 ? 8 : 4;
    constexpr int BWB = ((EW + 1 + ALN - 1 + ALN - 1) / ALN) * ALN;
    const size_t raw = (((size_t)(EH + 1) * BWB * (U16 ? 2 : 4)) + 127) & ~(size_t)127;
    return raw + (size_t)EH * EWP * sizeof(float) + std::max((size_t)kTY * EWP, (size_t)(EH + 1) * EW) * sizeof(float);
}

template <int WR, bool U16, bool SHADE>
__global__ void __launch_bounds__(kK3Threads, kK3V2MinBlocks) warp_smooth_v2_kernel(K3Args a, const __grid_constant__ CUtensorMap tmap) {
    constexpr int EH = kTY + 2 * WR, EW = kTX + 2 * WR, EWP = EW | 1;
    constexpr int ALN = U16 ? 8 : 4;
    constexpr int BWB = ((EW + 1 + ALN - 1 + ALN - 1) / ALN) * ALN;
    constexpr int BHB = EH + 1;
    constexpr int NCS = (EW + 31) / 32;

    using S_T = typename std::conditional<U16, uint16_t, float>::type;
    extern __shared__ __align__(128) unsigned char smem[];
    S_T* sRaw = reinterpret_cast<S_T*>(smem);
    // every intermediate is an f32 value (corrected samples; the vertical pass
    // is rounded to f32 like scipy's per-pass output), so shared memory holds
    // f32 and the passes widen to f64 on load: 43 KB per CTA instead of 64
    float* sC = reinterpret_cast<float*>(smem + (((size_t)BHB * BWB * sizeof(S_T) + 127) & ~(size_t)127));  // [EH][EWP]
    float* sV = sC + (size_t)EH * EWP;  // [kTY][EWP] vertical pass
    float* sH = sV;                     // [BHB][EW] horizontal interpolations (phase A only; aliases sV)
    __shared__ double s_w[WR + 1];
    __shared__ int s_ra[EH], s_rc[EH], s_xa[EW], s_xb[EW];
    __shared__ int s_gy[SHADE ? EH : 1], s_gx[SHADE ? EW : 1];
    __shared__ int s_box[2];
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid <= WR) s_w[tid] = a.wt.w[WR - tid];  // s_w[k] = weight at offset -k (symmetric)
    const int ty0 = blockIdx.y * kTY, tx0 = blockIdx.x * kTX;
    const int64_t hw = (int64_t)a.h * a.w;
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmap);
    }
    __syncthreads();
    auto issue = [&](int64_t t) {
        const WarpOp op = make_warp(a.vec, t);
        int y0, y1, x0, x1;
        src_span(ty0 - WR, ty0 + kTY + WR, a.h, op.iy, y0, y1);
        src_span(tx0 - WR, tx0 + kTX + WR, a.w, op.ix, x0, x1);
        const int x0a = x0 & ~(ALN - 1);
        mbar_expect_tx(&bar, (uint32_t)(BWB * BHB * sizeof(S_T)));
        tma_load_3d(sRaw, &tmap, x0a, y0, (int)t, &bar);
        return make_int2(x0a, y0);
    };
    auto smp = [](S_T v) -> float {
        if constexpr (U16)
            return u16_minus(v, 8388608.0f);
        else
            return v;
    };
    int2 origin_next = make_int2(0, 0);
    int64_t t = blockIdx.z;
    if (tid == 0 && t < a.n) origin_next = issue(t);
    uint32_t phase = 0;
    const double* wk = s_w;
    for (; t < a.n; t += gridDim.z) {
        const WarpOp op = make_warp(a.vec, t);
        if (tid == 0) {
            s_box[0] = origin_next.x;
            s_box[1] = origin_next.y;
        }
        for (int i = tid; i < EH + EW; i += kK3Threads) {
            if (i < EH) {
                const int y = reflect_index(ty0 - WR + i, a.h);
                if constexpr (SHADE) s_gy[i] = y;
                s_ra[i] = clampi(y - op.iy, 0, a.h - 1);
                s_rc[i] = clampi(y - op.iy - 1, 0, a.h - 1);
            } else {
                const int e = i - EH;
                const int x = reflect_index(tx0 - WR + e, a.w);
                if constexpr (SHADE) s_gx[e] = x;
                s_xa[e] = clampi(x - op.ix, 0, a.w - 1);
                s_xb[e] = clampi(x - op.ix - 1, 0, a.w - 1);
            }
        }
        __syncthreads();  // tables + origin published; previous frame's passes done with sV/sC
        const int bx0 = s_box[0], by0 = s_box[1];
        int xa[NCS], xb[NCS];
#pragma unroll
        for (int k = 0; k < NCS; ++k) {
            const int c = lane + 32 * k;
            xa[k] = c < EW ? s_xa[c] - bx0 : 0;
            xb[k] = c < EW ? s_xb[c] - bx0 : 0;
        }
        mbar_wait(&bar, phase);
        phase ^= 1u;
        // A1: horizontal interpolation of every box row
        for (int r = warp; r < BHB; r += kK3Threads / 32) {
            const S_T* row = sRaw + r * BWB;
            float* hrow = sH + r * EW;
#pragma unroll
            for (int k = 0; k < NCS; ++k) {
                const int c = lane + 32 * k;
                if (c < EW) hrow[c] = __fadd_rn(__fmul_rn(op.omx, smp(row[xa[k]])), __fmul_rn(op.fx, smp(row[xb[k]])));
            }
        }
        __syncthreads();
        if (tid == 0 && t + gridDim.z < a.n) origin_next = issue(t + gridDim.z);  // raw box consumed
        // A2: vertical interpolation -> corrected (f32 out, f64 into sC)
        {
            float* corr_base = a.corrected ? a.corrected + t * hw : nullptr;
            int gxs[NCS];
            if constexpr (SHADE) {
#pragma unroll
                for (int k = 0; k < NCS; ++k) gxs[k] = lane + 32 * k < EW ? s_gx[lane + 32 * k] : 0;
            }
            for (int ey = warp; ey < EH; ey += kK3Threads / 32) {
                const float* ha = sH + (s_ra[ey] - by0) * EW;
                const float* hc = sH + (s_rc[ey] - by0) * EW;
                const int gy = ty0 + ey - WR;
                const bool row_out = corr_base && ey >= WR && ey < WR + kTY && gy < a.h;
                const float* grow = SHADE ? a.gain + (int64_t)s_gy[ey] * a.w : nullptr;
#pragma unroll
                for (int k = 0; k < NCS; ++k) {
                    const int c = lane + 32 * k;
                    if (c < EW) {
                        float v = __fadd_rn(__fmul_rn(op.omy, ha[c]), __fmul_rn(op.fy, hc[c]));
                        if constexpr (SHADE) v = __fdiv_rn(v, __ldg(grow + gxs[k]));
                        sC[ey * EWP + c] = v;
                        const int gx = tx0 + c - WR;
                        if (row_out && c >= WR && c < WR + kTX && gx < a.w) corr_base[(int64_t)gy * a.w + gx] = v;
                    }
                }
            }
        }
        __syncthreads();  // sC complete; sH (sV) free
        // B: vertical 19-tap pass, (column, third of the rows) per thread
        if (tid < 3 * EW) {
            const int c = tid % EW, seg = tid / EW;
            const int r0 = seg * kVR2;
            const int nout = seg < 2 ? kVR2 : kTY - 2 * kVR2;
            double x[kVR2 + 2 * WR];
#pragma unroll
            for (int q = 0; q < kVR2 + 2 * WR; ++q) x[q] = (r0 + q < EH) ? (double)sC[(r0 + q) * EWP + c] : 0.0;
#if VB_K3_INTERLEAVE
            // all outputs advance together tap by tap: kVR2 independent chains
            // per step (same per-output operation order); weights from the
            // kernel-parameter constant bank (w symmetric: w[-k] == w[+k])
            double acc[kVR2];
#pragma unroll
            for (int j = 0; j < kVR2; ++j) acc[j] = __dmul_rn(x[j + WR], a.wt.w[WR]);
#pragma unroll
            for (int k = WR; k >= 1; --k) {
#pragma unroll
                for (int j = 0; j < kVR2; ++j)
                    acc[j] = __dadd_rn(acc[j], __dmul_rn(__dadd_rn(x[j + WR - k], x[j + WR + k]), a.wt.w[WR - k]));
            }
#pragma unroll
            for (int j = 0; j < kVR2; ++j)
                if (j < nout) sV[(r0 + j) * EWP + c] = (float)acc[j];
#else
#pragma unroll
            for (int j = 0; j < kVR2; ++j) {
                if (j < nout) {
                    double acc = __dmul_rn(x[j + WR], wk[0]);
#pragma unroll
                    for (int k = WR; k >= 1; --k)
                        acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(x[j + WR - k], x[j + WR + k]), wk[k]));
                    sV[(r0 + j) * EWP + c] = (float)acc;
                }
            }
#endif
        }
        __syncthreads();
        // C: horizontal pass -> smoothed frame.  Lanes take consecutive rows.
        {
            constexpr int HR = 8;
            const int ly = tid % kTY, lx0 = (tid / kTY) * HR;
            double x[HR + 2 * WR];
#pragma unroll
            for (int q = 0; q < HR + 2 * WR; ++q) x[q] = (double)sV[ly * EWP + lx0 + q];
            float o[HR];
#if VB_K3_INTERLEAVE
            double acc[HR];
#pragma unroll
            for (int j = 0; j < HR; ++j) acc[j] = __dmul_rn(x[j + WR], a.wt.w[WR]);
#pragma unroll
            for (int k = WR; k >= 1; --k) {
#pragma unroll
                for (int j = 0; j < HR; ++j)
                    acc[j] = __dadd_rn(acc[j], __dmul_rn(__dadd_rn(x[j + WR - k], x[j + WR + k]), a.wt.w[WR - k]));
            }
#pragma unroll
            for (int j = 0; j < HR; ++j) o[j] = (float)acc[j];
#else
#pragma unroll
            for (int j = 0; j < HR; ++j) {
                double acc = __dmul_rn(x[j + WR], wk[0]);
#pragma unroll
                for (int k = WR; k >= 1; --k) acc = __dadd_rn(acc, __dmul_rn(__dadd_rn(x[j + WR - k], x[j + WR + k]), wk[k]));
                o[j] = (float)acc;
            }
#endif
            const int gy = ty0 + ly, gx0 = tx0 + lx0;
            float* dst = a.smoothed + t * hw + (int64_t)gy * a.w + gx0;
            if (gy < a.h) {
                if ((a.w & 3) == 0 && gx0 + HR <= a.w) {
#pragma unroll
                    for (int j = 0; j < HR; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
                } else {
#pragma unroll
                    for (int j = 0; j < HR; ++j)
                        if (gx0 + j < a.w) dst[j] = o[j];
                }
            }
        }
    }
}
static_assert(kK3Threads == kTY * (kTX / 8), "horizontal pass maps one thread per (row, 8 outputs)");
static_assert(3 * (kTX + 18) <= kK3Threads, "vertical pass maps one thread per (column, third)");

template <int WR, bool U16>
static int launch_k3_tma(const CUtensorMap& tmap, K3Args a, int64_t n, int h, int w, cudaStream_t s) {
    const size_t smem = k3_v2_smem_bytes<WR, U16>();
    auto kern = a.gain ? warp_smooth_v2_kernel<WR, U16, true> : warp_smooth_v2_kernel<WR, U16, false>;
    VB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int tiles = ((w + kTX - 1) / kTX) * ((h + kTY - 1) / kTY);
    // ~4 frames per CTA, at least 8 resident waves of CTAs
    const int64_t gz = std::min<int64_t>(65535, std::max<int64_t>((n + 3) / 4, ((int64_t)sms * 24 + tiles - 1) / tiles));
    a.n = n;
    dim3 grid((unsigned)((w + kTX - 1) / kTX), (unsigned)((h + kTY - 1) / kTY), (unsigned)std::min<int64_t>(gz, n));
    {
        ProfScope ps(kProfWarpSmooth, s);
        kern<<<grid, kK3Threads, smem, s>>>(a, tmap);
    }
    VB_LAUNCHED();
    return VB_OK;
}

// ---------------------------------------------------------- K3, split form
// The fused kernel above interpolates the corrected tile + halo (2x the
// tile's pixels) in every CTA, and those f32 phases cost as many issue slots
// as the float64 passes.  The split form writes the corrected frames once
// (K3a: a streaming kernel, every pixel interpolated once, in numpy's order)
// and the smoothing kernel (K3b) stages each corrected tile + halo with one
// TMA box into shared memory -- double-buffered, the next frame's box lands
// while this frame's passes run -- mirrors the reflected halo inside the box
// at the frame edges, and runs the same two float64 passes.  Same arithmetic,
// so the results are bit-identical to the fused kernel.
constexpr int kCW = 8;  // K3a: corrected outputs per thread (one row segment)
constexpr int kK3NotHandled = -100;  // launch_k3_split: use the fused kernel instead

// One thread: a strip of kCW columns x kCR rows.  translate's top row of
// output y is the bottom row of output y + 1 (both clamp(y - iy)), so each
// horizontal interpolation serves two outputs: kCR + 1 per strip.
constexpr int kCR = 16;  // rows per strip (measured: 8 -> 16, 3.28 -> 3.24 ms per 4000 C2 frames with the smoothing)

template <bool U16>
__global__ void __launch_bounds__(256) correct_rows_kernel(const void* __restrict__ frames, int64_t n, int h, int w,
                                                           const vb_motion* __restrict__ vec,
                                                           const float* __restrict__ gain, float* __restrict__ out) {
    using S_T = typename std::conditional<U16, uint16_t, float>::type;
    const int64_t hw = (int64_t)h * w;
    const int wq = (w + kCW - 1) / kCW, hq = (h + kCR - 1) / kCR;
    const int per_frame = hq * wq;
    for (int64_t t = blockIdx.y; t < n; t += gridDim.y) {
        const WarpOp op = make_warp(vec, t);
        const S_T* f = reinterpret_cast<const S_T*>(frames) + t * hw;
        float* o = out + t * hw;
        for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < per_frame; i += gridDim.x * blockDim.x) {
            const int yb = (i / wq) * kCR, x0 = (i - (i / wq) * wq) * kCW;
            // source columns x - ix - 1 + j, j = 0..kCW (b taps at j, a taps at j + 1)
            const int c0 = x0 - op.ix - 1;
            const bool inner = c0 >= 0 && c0 + kCW < w;
            // raw samples of a source row; the next row's loads are issued before
            // this row's arithmetic (one row of look-ahead)
            auto load_row = [&](int r, S_T (&raw)[kCW + 1]) {
                const S_T* row = f + (int64_t)r * w;
#pragma unroll
                for (int j = 0; j <= kCW; ++j) raw[j] = __ldg(row + (inner ? c0 + j : clampi(c0 + j, 0, w - 1)));
            };
            auto hrow = [&](const S_T (&raw)[kCW + 1], float (&hv)[kCW]) {  // horizontal interpolation
                float v[kCW + 1];
#pragma unroll
                for (int j = 0; j <= kCW; ++j) {
                    if constexpr (U16)
                        v[j] = u16_minus(raw[j], 8388608.0f);  // exact widening on the FMA pipe
                    else
                        v[j] = raw[j];
                }
#pragma unroll
                for (int k = 0; k < kCW; ++k) hv[k] = __fadd_rn(__fmul_rn(op.omx, v[k + 1]), __fmul_rn(op.fx, v[k]));
            };
            S_T rc_raw[kCW + 1], ra_raw[kCW + 1];
            load_row(clampi(yb - op.iy - 1, 0, h - 1), rc_raw);
            load_row(clampi(yb - op.iy, 0, h - 1), ra_raw);
            float hc[kCW], ha[kCW];
            hrow(rc_raw, hc);
#pragma unroll 1
            for (int y = yb; y < yb + kCR && y < h; ++y) {
                S_T cur[kCW + 1];
#pragma unroll
                for (int j = 0; j <= kCW; ++j) cur[j] = ra_raw[j];
                if (y + 1 < yb + kCR && y + 1 < h) load_row(clampi(y + 1 - op.iy, 0, h - 1), ra_raw);
                hrow(cur, ha);
                float v[kCW];
#pragma unroll
                for (int k = 0; k < kCW; ++k) {
                    v[k] = __fadd_rn(__fmul_rn(op.omy, ha[k]), __fmul_rn(op.fy, hc[k]));
                    if (gain && x0 + k < w) v[k] = __fdiv_rn(v[k], __ldg(gain + (int64_t)y * w + x0 + k));
                    hc[k] = ha[k];
                }
                float* dst = o + (int64_t)y * w + x0;
                if ((w & 3) == 0 && x0 + kCW <= w) {
#pragma unroll
                    for (int k = 0; k < kCW; k += 4)
                        *reinterpret_cast<float4*>(dst + k) = make_float4(v[k], v[k + 1], v[k + 2], v[k + 3]);
                } else {
#pragma unroll
                    for (int k = 0; k < kCW; ++k)
                        if (x0 + k < w) dst[k] = v[k];
                }
            }
        }
    }
}

static int launch_correct_rows(const void* frames, int dtype, int64_t n, int h, int w, const vb_motion* vec,
                               const float* gain, float* out, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int wq = (w + kCW - 1) / kCW;
    const int per_frame = ((h + kCR - 1) / kCR) * wq;
    const int bx = std::max(1, std::min((per_frame + 255) / 256, 64));
    const int64_t gy = std::min<int64_t>(65535, std::min<int64_t>(n, std::max<int64_t>(1, (int64_t)sms * 8 / bx)));
    dim3 grid((unsigned)bx, (unsigned)gy);
    {
        ProfScope ps(kProfWarpSmooth, s);
        if (dtype == VB_U16)
            correct_rows_kernel<true><<<grid, 256, 0, s>>>(frames, n, h, w, vec, gain, out);
        else
            correct_rows_kernel<false><<<grid, 256, 0, s>>>(frames, n, h, w, vec, gain, out);
    }
    VB_LAUNCHED();
    return VB_OK;
}

template <int WR>
struct K3bGeom {
    static constexpr int EH = kTY + 2 * WR, EW = kTX + 2 * WR, EWP = EW | 1;
    static constexpr int XO = (4 - WR % 4) % 4;      // box starts at the 16-byte aligned column tx0 - WR - XO
    static constexpr int BW = (EW + XO + 3) / 4 * 4;  // box width (f32), a 16-byte multiple
    static constexpr int BH = EH + 1;  // one spare row: the last vertical segment loads rows up to EH unguarded
    static constexpr size_t box_bytes = ((size_t)BH * BW * sizeof(float) + 127) & ~(size_t)127;  // TMA dst: 128-B aligned
    static constexpr size_t smem = 2 * box_bytes + (size_t)(kTY + 1) * EWP * sizeof(float);
};

template <int WR>
__global__ void __launch_bounds__(kK3Threads, kK3V2MinBlocks) smooth_tma_kernel(K3Args a, const __grid_constant__ CUtensorMap tmap) {
    using G = K3bGeom<WR>;
    constexpr int EH = G::EH, EW = G::EW, EWP = G::EWP, XO = G::XO, BW = G::BW;
    extern __shared__ __align__(128) unsigned char smem[];
    float* sBox = reinterpret_cast<float*>(smem);                  // 2 x [EH][BW] corrected tile + halo
    float* sV = reinterpret_cast<float*>(smem + 2 * G::box_bytes);  // [kTY][EWP] vertical pass
    __shared__ __align__(8) uint64_t bar[2];
    const int tid = threadIdx.x;
    const int ty0 = blockIdx.y * kTY, tx0 = blockIdx.x * kTX;
    const int64_t hw = (int64_t)a.h * a.w;
    const int y_lo = ty0 - WR, x_lo = tx0 - WR;
    // tiles whose halo leaves the frame mirror it inside the box (scipy "reflect")
    const bool edge = y_lo < 0 || x_lo < 0 || ty0 + kTY + WR > a.h || tx0 + kTX + WR > a.w;
    if (tid == 0) {
        mbar_init(&bar[0], 1);
        mbar_init(&bar[1], 1);
        fence_mbar_init();
        tma_prefetch_desc(&tmap);
    }
    __syncthreads();
    auto issue = [&](int64_t t, int b) {
        mbar_expect_tx(&bar[b], (uint32_t)(G::BH * BW * sizeof(float)));
        tma_load_3d(sBox + b * (G::box_bytes / sizeof(float)), &tmap, x_lo - XO, y_lo, (int)t, &bar[b]);
    };
    int64_t t = blockIdx.z;
    if (tid == 0) {
        if (t < a.n) issue(t, 0);
        if (t + gridDim.z < a.n) issue(t + gridDim.z, 1);
    }
    uint32_t phase[2] = {0u, 0u};
    for (int i = 0; t < a.n; t += gridDim.z, ++i) {
        const int b = i & 1;
        float* sC = sBox + b * (G::box_bytes / sizeof(float));
        mbar_wait(&bar[b], phase[b]);
        phase[b] ^= 1u;
        if (edge) {
            // halo columns outside the frame first (every row), then halo rows
            // (whole rows), so corners mirror twice
            const int nl = max(0, -x_lo), nr = max(0, x_lo + EW - a.w), nc = nl + nr;
            for (int k = tid; k < EH * nc; k += kK3Threads) {
                const int ey = k / nc, j = k - ey * nc;
                const int ex = j < nl ? j : EW - nr + (j - nl);
                const int sx = clampi(reflect_index(x_lo + ex, a.w) - x_lo, 0, EW - 1);
                sC[ey * BW + XO + ex] = sC[ey * BW + XO + sx];
            }
            __syncthreads();
            const int nt = max(0, -y_lo), nb = max(0, y_lo + EH - a.h), nrw = nt + nb;
            for (int k = tid; k < nrw * EW; k += kK3Threads) {
                const int j = k / EW, ex = k - j * EW;
                const int ey = j < nt ? j : EH - nb + (j - nt);
                const int sy = clampi(reflect_index(y_lo + ey, a.h) - y_lo, 0, EH - 1);
                sC[ey * BW + XO + ex] = sC[sy * BW + XO + ex];
            }
        }
        __syncthreads();  // box (mirrored) complete; the previous frame's horizontal pass is done with sV
        // B: vertical 19-tap pass, (column, third of the rows) per thread
        if (tid < 3 * EW) {
            const int c = tid % EW, seg = tid / EW;
            const int r0 = seg * kVR2;
            const int nout = seg < 2 ? kVR2 : kTY - 2 * kVR2;
            double x[kVR2 + 2 * WR];
            static_assert(2 * kVR2 + kVR2 + 2 * WR <= EH + 1, "box rows cover every segment's loads");
#pragma unroll
            for (int q = 0; q < kVR2 + 2 * WR; ++q) x[q] = (double)sC[(r0 + q) * BW + XO + c];
            double acc[kVR2];
#pragma unroll
            for (int j = 0; j < kVR2; ++j) acc[j] = __dmul_rn(x[j + WR], a.wt.w[WR]);
#pragma unroll
            for (int k = WR; k >= 1; --k) {
#pragma unroll
                for (int j = 0; j < kVR2; ++j)
                    acc[j] = __dadd_rn(acc[j], __dmul_rn(__dadd_rn(x[j + WR - k], x[j + WR + k]), a.wt.w[WR - k]));
            }
            (void)nout;  // the last segment's 11th row lands in sV's spare row
#pragma unroll
            for (int j = 0; j < kVR2; ++j) sV[(r0 + j) * EWP + c] = (float)acc[j];
        }
        __syncthreads();  // sV complete; this box is free
        if (tid == 0 && t + 2 * (int64_t)gridDim.z < a.n) issue(t + 2 * (int64_t)gridDim.z, b);
        // C: horizontal pass -> smoothed frame.  Lanes take consecutive rows.
        {
            constexpr int HR = 8;
            const int ly = tid % kTY, lx0 = (tid / kTY) * HR;
            double x[HR + 2 * WR];
#pragma unroll
            for (int q = 0; q < HR + 2 * WR; ++q) x[q] = (double)sV[ly * EWP + lx0 + q];
            double acc[HR];
#pragma unroll
            for (int j = 0; j < HR; ++j) acc[j] = __dmul_rn(x[j + WR], a.wt.w[WR]);
#pragma unroll
            for (int k = WR; k >= 1; --k) {
#pragma unroll
                for (int j = 0; j < HR; ++j)
                    acc[j] = __dadd_rn(acc[j], __dmul_rn(__dadd_rn(x[j + WR - k], x[j + WR + k]), a.wt.w[WR - k]));
            }
            float o[HR];
#pragma unroll
            for (int j = 0; j < HR; ++j) o[j] = (float)acc[j];
            const int gy = ty0 + ly, gx0 = tx0 + lx0;
            float* dst = a.smoothed + t * hw + (int64_t)gy * a.w + gx0;
            if (gy < a.h) {
                if ((a.w & 3) == 0 && gx0 + HR <= a.w) {
#pragma unroll
                    for (int j = 0; j < HR; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(o[j], o[j + 1], o[j + 2], o[j + 3]);
                } else {
#pragma unroll
                    for (int j = 0; j < HR; ++j)
                        if (gx0 + j < a.w) dst[j] = o[j];
                }
            }
        }
    }
}

// Split K3 for radius 9: K3a into `corrected` (or a scratch buffer), then K3b.
// Returns kK3NotHandled (the caller falls back to the fused kernel) when the tensor
// map cannot describe the corrected frames.
static int launch_k3_split(const void* frames, int dtype, const vb_motion* vec, int64_t n, int h, int w,
                           const K3Args& base, float* corrected, float* smoothed, cudaStream_t s) {
    using G = K3bGeom<9>;
    if ((w & 3) || n > 0x7fffffff || h < 10 || w < 10) return kK3NotHandled;
    float* corr = corrected;
    float* tmp = nullptr;
    const int64_t hw = (int64_t)h * w;
    if (!corr) {
        keep_pool();
        VB_CUDA(cudaMallocAsync(&tmp, (size_t)n * hw * sizeof(float), s));
        corr = tmp;
    }
    CUtensorMap tmap;
    memset(&tmap, 0, sizeof(tmap));
    if (!make_frames_tmap(&tmap, corr, VB_F32, n, h, w, G::BH, G::BW)) {
        if (tmp) cudaFreeAsync(tmp, s);
        return kK3NotHandled;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    {
        const int rc0 = launch_correct_rows(frames, dtype, n, h, w, vec, base.gain, corr, s);
        if (rc0) {
            if (tmp) cudaFreeAsync(tmp, s);
            return rc0;
        }
    }
    K3Args a = base;
    a.n = n;
    a.smoothed = smoothed;
    VB_CUDA(cudaFuncSetAttribute(smooth_tma_kernel<9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem));
    const int tiles = ((w + kTX - 1) / kTX) * ((h + kTY - 1) / kTY);
    const int64_t gz = std::min<int64_t>(65535, std::max<int64_t>((n + 3) / 4, ((int64_t)sms * 24 + tiles - 1) / tiles));
    dim3 grid((unsigned)((w + kTX - 1) / kTX), (unsigned)((h + kTY - 1) / kTY), (unsigned)std::min<int64_t>(gz, n));
    {
        ProfScope ps(kProfWarpSmooth, s);
        smooth_tma_kernel<9><<<grid, kK3Threads, G::smem, s>>>(a, tmap);
    }
    VB_LAUNCHED();
    if (tmp) cudaFreeAsync(tmp, s);
    return VB_OK;
}

// Spatial summary (summarize.py:55-57): per-pixel float64 mean over the
// block's corrected frames, accumulated sequentially in frame order like
// numpy's axis-0 reduction -> bit-identical.
__global__ void block_mean_kernel(const float* __restrict__ frames, int64_t n, int64_t hw, int L,
                                  float* __restrict__ spatial) {
    const int blk = blockIdx.y;
    const int64_t t0 = (int64_t)blk * L;
    const int cnt = (int)((int64_t)L < n - t0 ? (int64_t)L : n - t0);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x) {
        const float* col = frames + t0 * hw + i;
        double s = 0.0;
#pragma unroll 8
        for (int t = 0; t < cnt; ++t) s += (double)__ldcs(col + (int64_t)t * hw);
        spatial[(int64_t)blk * hw + i] = (float)(s / (double)cnt);
    }
}

// ------------------------------------------------------------------ K4
#ifndef VB_K4_PIX
#define VB_K4_PIX 16
#endif
constexpr int kK4Pix = VB_K4_PIX, kK4Threads = 256;  // pixels per median CTA (multiple of 4)
constexpr int kMaxHalfWindow = 512;  // high-pass window N = 2*hh+1 <= 1025 frames

// Order-preserving uint32 key of a float32 (total order, -0 < +0): selection
// works on keys, so the (opt-in, A17) high-passed stacks may hold negatives.
__device__ __forceinline__ uint32_t fkey(float f) {
    const uint32_t u = __float_as_uint(f);
    return u ^ ((uint32_t)((int32_t)u >> 31) | 0x80000000u);
}
__device__ __forceinline__ float fkey_inv(uint32_t k) {
    return __uint_as_float((k & 0x80000000u) ? (k ^ 0x80000000u) : ~k);
}

__host__ __device__ __forceinline__ int64_t reflect64(int64_t i, int64_t n) {
    const int64_t period = 2 * n;
    int64_t m = i % period;
    if (m < 0) m += period;
    return m >= n ? period - 1 - m : m;
}

struct K4Args {
    const float* sm;   // smoothed frames; scratch row r holds recording frame s_lo + r
    int64_t s_lo;
    int64_t g0;        // recording index of the first block's first frame
    int64_t n;         // frames summarised (blocks of L from g0; the last may be short)
    int64_t hw;
    int L;
    int hh;            // temporal high-pass half window (0 = off), window N = 2*hh + 1
    double inv_n;      // float64(1 / N)
    int64_t t_total;   // recording length: reflect boundary of the temporal filter
    float* temporal;   // [blocks][hw]
};

// k-th smallest (0-based) of the warp's keys (padding = 0xffffffff never counts).
template <int VPL>
__device__ __forceinline__ uint32_t warp_select(const uint32_t (&v)[VPL], uint32_t lo, uint32_t hi, int k) {
    // bisection over u = key - lo in [0, hi - lo]: ceil(log2(range)) rounds
    const uint32_t range = hi - lo;
    if (range == 0) return lo;
    const int nb = 32 - __clz(range);
    uint32_t u[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) u[i] = v[i] - lo;  // padding stays above any candidate
    uint32_t ans = 0;
    for (int b = nb - 1; b >= 0; --b) {
        const uint32_t cand = ans | (1u << b);
        uint32_t c = 0;
#pragma unroll
        for (int i = 0; i < VPL; ++i) c += u[i] < cand ? 1u : 0u;
        c = __reduce_add_sync(0xffffffffu, c);
        if ((int)c <= k) ans = cand;
    }
    return lo + ans;
}

// k-th smallest of the warp's keys in three steps instead of up to 32
// bisection rounds over all VPL keys per lane: a 128-bin histogram of the top
// 7 bits of key - lo (shared-memory atomics), a warp scan that finds the bin
// holding rank k, then -- when that bin holds <= 32 keys, the usual case --
// the survivors are compacted one per lane and the remaining low bits are
// bisected with one ballot per bit.  A crowded bin falls back to bisecting
// the low bits over all keys.  Exact: the same order statistic as warp_select.
constexpr int kSelBins = 128;
struct __align__(16) SelScratch {
    uint32_t hist[kSelBins];  // read as uint4 per lane
    uint32_t buf[32];
    uint32_t n, pad[3];
};

template <int VPL>
__device__ __forceinline__ uint32_t warp_select_hist(const uint32_t (&v)[VPL], uint32_t lo, uint32_t hi, int k,
                                                     SelScratch& sc) {
    const uint32_t range = hi - lo;
    if (range == 0) return lo;
    const int nb = 32 - __clz(range);
    if (nb <= 7) return warp_select<VPL>(v, lo, hi, k);
    const int shift = nb - 7;
    const int lane = threadIdx.x & 31;
    for (int i = lane; i < kSelBins; i += 32) sc.hist[i] = 0;
    if (lane == 0) sc.n = 0;
    __syncwarp();
#pragma unroll
    for (int i = 0; i < VPL; ++i)
        if (v[i] != 0xffffffffu) atomicAdd(&sc.hist[(v[i] - lo) >> shift], 1u);
    __syncwarp();
    const uint4 h = reinterpret_cast<const uint4*>(sc.hist)[lane];
    const uint32_t tot = h.x + h.y + h.z + h.w;
    uint32_t incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    const uint32_t excl = incl - tot, uk = (uint32_t)k;
    const int src = __ffs(__ballot_sync(0xffffffffu, excl <= uk && uk < incl)) - 1;
    uint32_t bin = 4 * lane, below = excl;
    if (uk >= below + h.x) {
        below += h.x;
        ++bin;
        if (uk >= below + h.y) {
            below += h.y;
            ++bin;
            if (uk >= below + h.z) {
                below += h.z;
                ++bin;
            }
        }
    }
    bin = __shfl_sync(0xffffffffu, bin, src);
    below = __shfl_sync(0xffffffffu, below, src);
    const uint32_t nbin = sc.hist[bin];
    uint32_t ans = bin << shift;
    if (nbin <= 32) {
#pragma unroll
        for (int i = 0; i < VPL; ++i)
            if (v[i] != 0xffffffffu && ((v[i] - lo) >> shift) == bin) sc.buf[atomicAdd(&sc.n, 1u)] = v[i] - lo;
        __syncwarp();
        const uint32_t sv = (uint32_t)lane < nbin ? sc.buf[lane] : 0xffffffffu;
        const uint32_t kk = uk - below;
        for (int b = shift - 1; b >= 0; --b) {
            const uint32_t cand = ans | (1u << b);
            if ((uint32_t)__popc(__ballot_sync(0xffffffffu, sv < cand)) <= kk) ans = cand;
        }
    } else {
        uint32_t u[VPL];
#pragma unroll
        for (int i = 0; i < VPL; ++i) u[i] = v[i] - lo;
        for (int b = shift - 1; b >= 0; --b) {
            const uint32_t cand = ans | (1u << b);
            uint32_t c = 0;
#pragma unroll
            for (int i = 0; i < VPL; ++i) c += (v[i] != 0xffffffffu && u[i] < cand) ? 1u : 0u;
            c = __reduce_add_sync(0xffffffffu, c);
            if (c <= uk) ans = cand;
        }
    }
    __syncwarp();  // scratch reused by the next selection
    return lo + ans;
}

// max - median over the warp's keys (numpy's midpoint for even counts).
template <int VPL>
__device__ __forceinline__ float max_minus_median(const uint32_t (&v)[VPL], uint32_t lo, uint32_t hi, int cnt,
                                                  SelScratch& sc) {
    const int mid = cnt / 2;
    constexpr bool kHist = VPL >= 4;  // histogram select pays off from ~100 keys per warp
    auto sel = [&](int k) { return kHist ? warp_select_hist<VPL>(v, lo, hi, k, sc) : warp_select<VPL>(v, lo, hi, k); };
    float med;
    if (cnt & 1) {
        med = fkey_inv(sel(mid));
    } else {
        const uint32_t a = sel(mid - 1);
        uint32_t le = 0, above = 0xffffffffu;
#pragma unroll
        for (int i = 0; i < VPL; ++i) {
            le += v[i] <= a ? 1u : 0u;
            if (v[i] > a) above = min(above, v[i]);
        }
        le = __reduce_add_sync(0xffffffffu, le);
        above = __reduce_min_sync(0xffffffffu, above);
        const uint32_t b = ((int)le >= mid + 1) ? a : above;
        med = __fmul_rn(__fadd_rn(fkey_inv(a), fkey_inv(b)), 0.5f);
    }
    return __fsub_rn(fkey_inv(hi), med);
}

// One CTA per (block, 16 consecutive pixels): stage the block's smoothed
// column (plus the high-pass halo, reflected at the recording ends) in shared
// memory, one warp per pixel.  Without the high-pass lane l holds frames
// l, l+32, ...; with it lane l owns the contiguous frames [l*VPL, (l+1)*VPL)
// and slides a float64 window sum over them (exact for camera-range data, so
// it equals the direct sum the oracle forms): hp = f32(x - sum * (1/N)).
template <int VPL, bool HP>
__global__ void __launch_bounds__(kK4Threads) median_kernel(K4Args a) {
    extern __shared__ float sm4[];  // [cnt + 2 hh][kK4Pix + 1]
    __shared__ SelScratch s_sel[kK4Threads / 32];
    constexpr int ST = kK4Pix + 1;
    const int blk = blockIdx.y;
    const int64_t t0 = a.g0 + (int64_t)blk * a.L;
    const int cnt = (int)((int64_t)a.L < a.g0 + a.n - t0 ? (int64_t)a.L : a.g0 + a.n - t0);
    const int hh = HP ? a.hh : 0;
    const int rows = cnt + 2 * hh;
    const int64_t p0 = (int64_t)blockIdx.x * kK4Pix;
    const int np = (int)((int64_t)kK4Pix < a.hw - p0 ? (int64_t)kK4Pix : a.hw - p0);
    // staging: float4 loads (4 pixels of one frame row; 4 threads per 64-byte
    // row segment), 8 independent loads in flight per thread before their
    // stores; the scalar path covers frames whose rows are not 16-byte aligned
    if ((a.hw & 3) == 0 && np == kK4Pix) {
        constexpr int kB = 8;
        const int total4 = rows * (kK4Pix / 4);
        for (int i0 = threadIdx.x; i0 < total4; i0 += kB * kK4Threads) {
            float4 vals[kB];
#pragma unroll
            for (int j = 0; j < kB; ++j) {
                const int i = i0 + j * kK4Threads;
                const int tt = i / (kK4Pix / 4), q = i % (kK4Pix / 4);
                int64_t g = t0 - hh + tt;
                if constexpr (HP) g = reflect64(g, a.t_total);
                vals[j] = i < total4 ? __ldcs(reinterpret_cast<const float4*>(a.sm + (g - a.s_lo) * a.hw + p0) + q)
                                     : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int j = 0; j < kB; ++j) {
                const int i = i0 + j * kK4Threads;
                if (i < total4) {
                    float* d = sm4 + (i / (kK4Pix / 4)) * ST + (i % (kK4Pix / 4)) * 4;
                    d[0] = vals[j].x;
                    d[1] = vals[j].y;
                    d[2] = vals[j].z;
                    d[3] = vals[j].w;
                }
            }
        }
    } else {
        constexpr int kB = 16;
        const int total = rows * kK4Pix;
        for (int i0 = threadIdx.x; i0 < total; i0 += kB * kK4Threads) {
            float vals[kB];
#pragma unroll
            for (int j = 0; j < kB; ++j) {
                const int i = i0 + j * kK4Threads;
                const int tt = i / kK4Pix, pp = i - tt * kK4Pix;
                int64_t g = t0 - hh + tt;
                if constexpr (HP) g = reflect64(g, a.t_total);
                vals[j] = (i < total && pp < np) ? __ldcs(a.sm + (g - a.s_lo) * a.hw + p0 + pp) : 0.f;
            }
#pragma unroll
            for (int j = 0; j < kB; ++j) {
                const int i = i0 + j * kK4Threads;
                if (i < total) sm4[(i / kK4Pix) * ST + (i % kK4Pix)] = vals[j];
            }
        }
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int pp = warp; pp < np; pp += kK4Threads / 32) {
        const float* col = sm4 + pp;
        uint32_t v[VPL];
        uint32_t lo = 0xffffffffu, hi = 0u;
        if constexpr (!HP) {
#pragma unroll
            for (int i = 0; i < VPL; ++i) {
                const int tt = lane + 32 * i;
                v[i] = tt < cnt ? fkey(col[tt * ST]) : 0xffffffffu;
                if (tt < cnt) {
                    lo = min(lo, v[i]);
                    hi = max(hi, v[i]);
                }
            }
        } else {
            const int tb = lane * VPL;
            double acc = 0.0;
            if (tb < cnt)
                for (int q = 0; q <= 2 * hh; ++q) acc = __dadd_rn(acc, (double)col[(tb + q) * ST]);
#pragma unroll
            for (int i = 0; i < VPL; ++i) {
                const int tt = tb + i;
                v[i] = 0xffffffffu;
                if (tt < cnt) {
                    const float x = col[(tt + hh) * ST];
                    const float hp = (float)__dsub_rn((double)x, __dmul_rn(acc, a.inv_n));
                    v[i] = fkey(hp);
                    lo = min(lo, v[i]);
                    hi = max(hi, v[i]);
                    if (tt + 1 < cnt)
                        acc = __dadd_rn(__dsub_rn(acc, (double)col[tt * ST]), (double)col[(tt + 2 * hh + 1) * ST]);
                }
            }
        }
        lo = __reduce_min_sync(0xffffffffu, lo);
        hi = __reduce_max_sync(0xffffffffu, hi);
        const float r = max_minus_median<VPL>(v, lo, hi, cnt, s_sel[warp]);
        if (lane == 0) a.temporal[(int64_t)blk * a.hw + p0 + pp] = r;
    }
}

// Fallback for blocks longer than 1024 frames (no high-pass): the column is
// re-read from global memory (L2) on each bisection step.
__global__ void median_kernel_long(K4Args a) {
    const int blk = blockIdx.y;
    const int64_t t0 = a.g0 + (int64_t)blk * a.L;
    const int cnt = (int)((int64_t)a.L < a.g0 + a.n - t0 ? (int64_t)a.L : a.g0 + a.n - t0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t p = (int64_t)blockIdx.x * (blockDim.x / 32) + warp;
    if (p >= a.hw) return;
    const float* col = a.sm + (t0 - a.s_lo) * a.hw + p;
    uint32_t lo = 0xffffffffu, hi = 0;
    for (int tt = lane; tt < cnt; tt += 32) {
        const uint32_t u = fkey(col[(int64_t)tt * a.hw]);
        lo = min(lo, u);
        hi = max(hi, u);
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    auto select = [&](int k) -> uint32_t {
        const uint32_t range = hi - lo;
        if (range == 0) return lo;
        const int nb = 32 - __clz(range);
        uint32_t ans = 0;
        for (int b = nb - 1; b >= 0; --b) {
            const uint32_t cand = ans | (1u << b);
            uint32_t c = 0;
            for (int tt = lane; tt < cnt; tt += 32) c += fkey(col[(int64_t)tt * a.hw]) - lo < cand ? 1u : 0u;
            c = __reduce_add_sync(0xffffffffu, c);
            if ((int)c <= k) ans = cand;
        }
        return lo + ans;
    };
    const int mid = cnt / 2;
    float med;
    if (cnt & 1) {
        med = fkey_inv(select(mid));
    } else {
        const uint32_t ka = select(mid - 1);
        uint32_t le = 0, above = 0xffffffffu;
        for (int tt = lane; tt < cnt; tt += 32) {
            const uint32_t u = fkey(col[(int64_t)tt * a.hw]);
            le += u <= ka ? 1u : 0u;
            if (u > ka) above = min(above, u);
        }
        le = __reduce_add_sync(0xffffffffu, le);
        above = __reduce_min_sync(0xffffffffu, above);
        const uint32_t kb = ((int)le >= mid + 1) ? ka : above;
        med = __fmul_rn(__fadd_rn(fkey_inv(ka), fkey_inv(kb)), 0.5f);
    }
    if (lane == 0) a.temporal[(int64_t)blk * a.hw + p] = __fsub_rn(fkey_inv(hi), med);
}

template <int VPL, bool HP>
static int launch_median_vpl(const K4Args& a, int nblk, cudaStream_t s) {
    const size_t smem = (size_t)(a.L + 2 * (HP ? a.hh : 0)) * (kK4Pix + 1) * sizeof(float);
    VB_CUDA(cudaFuncSetAttribute(median_kernel<VPL, HP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid((unsigned)((a.hw + kK4Pix - 1) / kK4Pix), (unsigned)nblk);
    {
        ProfScope ps(kProfMedian, s);
        median_kernel<VPL, HP><<<grid, kK4Threads, smem, s>>>(a);
    }
    VB_LAUNCHED();
    return VB_OK;
}

template <bool HP>
static int launch_median_hp(const K4Args& a, int nblk, cudaStream_t s) {
    const int vpl = (a.L + 31) / 32;
    if (vpl <= 1) return launch_median_vpl<1, HP>(a, nblk, s);
    if (vpl <= 2) return launch_median_vpl<2, HP>(a, nblk, s);
    if (vpl <= 4) return launch_median_vpl<4, HP>(a, nblk, s);
    if (vpl <= 8) return launch_median_vpl<8, HP>(a, nblk, s);
    if (vpl <= 16) return launch_median_vpl<16, HP>(a, nblk, s);
    if (vpl <= 32) return launch_median_vpl<32, HP>(a, nblk, s);
    if (HP) return fail(VB_EINVAL, "temporal high-pass needs segment_length <= 1024");
    dim3 grid((unsigned)((a.hw + 3) / 4), (unsigned)nblk);
    {
        ProfScope ps(kProfMedian, s);
        median_kernel_long<<<grid, 128, 0, s>>>(a);
    }
    VB_LAUNCHED();
    return VB_OK;
}

static int launch_median(const K4Args& a, int nblk, cudaStream_t s) {
    return a.hh > 0 ? launch_median_hp<true>(a, nblk, s) : launch_median_hp<false>(a, nblk, s);
}

static int launch_k3(const void* frames, int dtype, const vb_motion* vec, int64_t n, int h, int w,
                     const double* weights, int wradius, const float* gain, float* corrected, float* smoothed,
                     cudaStream_t s) {
    if (n <= 0) return VB_OK;
    K3Args a;
    a.dtype = dtype;
    a.h = h;
    a.w = w;
    a.wr = wradius;
    a.gain = gain;
    for (int i = 0; i < 2 * wradius + 1; ++i) a.wt.w[i] = weights[i];
    const bool no_tma = knob("VB_NO_TMA", 0) != 0;
    if (wradius == 9 && !no_tma && knob("VB_K3_SPLIT", 1) != 0) {  // experiment: 0 = fused kernel
        const int rc = launch_k3_split(frames, dtype, vec, n, h, w, a, corrected, smoothed, s);
        if (rc != kK3NotHandled) return rc;
    }
    if (wradius == 9 && !no_tma && n <= 0x7fffffff) {
        constexpr int EH = kTY + 18, EW = kTX + 18;
        CUtensorMap tmap;
        memset(&tmap, 0, sizeof(tmap));
        const int bwb = dtype == VB_U16 ? ((EW + 1 + 14) / 8) * 8 : ((EW + 1 + 6) / 4) * 4;
        if (make_frames_tmap(&tmap, frames, dtype, n, h, w, EH + 1, bwb)) {
            a.frames = frames;
            a.vec = vec;
            a.corrected = corrected;
            a.smoothed = smoothed;
            return dtype == VB_U16 ? launch_k3_tma<9, true>(tmap, a, n, h, w, s)
                                   : launch_k3_tma<9, false>(tmap, a, n, h, w, s);
        }
    }
    const size_t smem3 = k3_smem_bytes(wradius);
    void (*kern)(K3Args) = wradius == 9 ? warp_smooth_kernel<9> : warp_smooth_kernel<0>;
    VB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
    const int64_t hw = (int64_t)h * w;
    const size_t esz = dtype == VB_U16 ? 2 : 4;
    for (int64_t f0 = 0; f0 < n; f0 += 65535) {
        const int64_t nf = std::min<int64_t>(65535, n - f0);
        a.frames = (const char*)frames + (size_t)f0 * hw * esz;
        a.vec = vec ? vec + f0 : nullptr;
        a.n = nf;
        a.corrected = corrected ? corrected + (size_t)f0 * hw : nullptr;
        a.smoothed = smoothed + (size_t)f0 * hw;
        dim3 grid((unsigned)((w + kTX - 1) / kTX), (unsigned)((h + kTY - 1) / kTY), (unsigned)nf);
        {
            ProfScope ps(kProfWarpSmooth, s);
            kern<<<grid, kK3Threads, smem3, s>>>(a);
        }
        VB_LAUNCHED();
    }
    return VB_OK;
}

// Summaries of the blocks of `frames` [ioff, ioff + n) (SummaryOpts in vb.cuh).
// Batches of whole blocks bound the smoothed scratch to ~4 GB.  Per batch:
// fused warp (+ shading) + smoothing of the batch's frames -- and, with the
// temporal high-pass, of the hh-frame halo on either side (reflected at the
// recording ends; halo frames are not written to `corrected`) -- then the
// per-block mean and the (high-passed) max - median.
int launch_summarize_ex(const void* frames, int dtype, const vb_motion* vec, int64_t n_avail, int h, int w,
                        int seg_len, const double* weights, int wradius, const SummaryOpts& o, float* corrected,
                        float* spatial, float* temporal, cudaStream_t s) {
    const int64_t n = o.n_interior;
    if (n <= 0) return VB_OK;
    if (wradius > kMaxWR) return fail(VB_EINVAL, "smoothing radius too large (max 16)");
    const int hh = o.highpass_window > 1 ? o.highpass_window / 2 : 0;
    if (hh > kMaxHalfWindow) return fail(VB_EINVAL, "high-pass window too long (max 1025 frames)");
    if (hh > 0 && seg_len > 1024) return fail(VB_EINVAL, "temporal high-pass needs segment_length <= 1024");
    const int64_t hw = (int64_t)h * w;
    const size_t esz = dtype == VB_U16 ? 2 : 4;
    const int64_t nblk_total = (n + seg_len - 1) / seg_len;
    const size_t blk_bytes = (size_t)seg_len * hw * sizeof(float) * (corrected ? 1 : 2);
    int64_t per = std::max<int64_t>(1, (int64_t)((size_t)4 << 30) / (int64_t)blk_bytes);
    per = std::min(per, nblk_total);
    const size_t smooth_bytes = (size_t)(seg_len * per + 2 * hh) * hw * sizeof(float);
    const size_t corr_bytes = (size_t)seg_len * per * hw * sizeof(float);
    float* smoothed = nullptr;
    float* corr_scratch = nullptr;
    keep_pool();
    VB_CUDA(cudaMallocAsync(&smoothed, smooth_bytes, s));
    if (!corrected) {
        cudaError_t e = cudaMallocAsync(&corr_scratch, corr_bytes, s);
        if (e != cudaSuccess) {
            cudaFreeAsync(smoothed, s);
            return cuda_fail(e, "cudaMallocAsync(corrected scratch)");
        }
    }
    auto at = [&](int64_t g) { return (const char*)frames + (size_t)(g - o.t_global0) * hw * esz; };
    auto vat = [&](int64_t g) { return vec ? vec + (g - o.t_global0) : nullptr; };
    int rc = VB_OK;
    for (int64_t b0 = 0; b0 < nblk_total && rc == VB_OK; b0 += per) {
        const int nb = (int)std::min(per, nblk_total - b0);
        const int64_t gi0 = o.t_global0 + o.interior_off + b0 * seg_len;  // recording frame indices
        const int64_t nf = std::min<int64_t>((int64_t)nb * seg_len, n - b0 * seg_len);
        const int64_t gi1 = gi0 + nf;
        const int64_t sg0 = hh ? std::max<int64_t>(0, gi0 - hh) : gi0;
        const int64_t sg1 = hh ? std::min<int64_t>(o.t_total, gi1 + hh) : gi1;
        float* corr = corrected ? corrected + (size_t)(b0 * seg_len) * hw : corr_scratch;
        rc = launch_k3(at(sg0), dtype, vat(sg0), gi0 - sg0, h, w, weights, wradius, o.gain, nullptr, smoothed, s);
        if (rc == VB_OK)
            rc = launch_k3(at(gi0), dtype, vat(gi0), nf, h, w, weights, wradius, o.gain, corr,
                           smoothed + (size_t)(gi0 - sg0) * hw, s);
        if (rc == VB_OK)
            rc = launch_k3(at(gi1), dtype, vat(gi1), sg1 - gi1, h, w, weights, wradius, o.gain, nullptr,
                           smoothed + (size_t)(gi1 - sg0) * hw, s);
        if (rc) break;
        {
            dim3 grid((unsigned)std::min<int64_t>((hw + 255) / 256, 1024), (unsigned)nb);
            ProfScope ps(kProfOther, s);
            block_mean_kernel<<<grid, 256, 0, s>>>(corr, nf, hw, seg_len, spatial + (size_t)b0 * hw);
        }
        launches().fetch_add(1, std::memory_order_relaxed);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            rc = cuda_fail(e, "block_mean_kernel");
            break;
        }
        K4Args k4;
        k4.sm = smoothed;
        k4.s_lo = sg0;
        k4.g0 = gi0;
        k4.n = nf;
        k4.hw = hw;
        k4.L = seg_len;
        k4.hh = hh;
        k4.inv_n = 1.0 / (double)(2 * hh + 1);
        k4.t_total = o.t_total;
        k4.temporal = temporal + (size_t)b0 * hw;
        rc = launch_median(k4, nb, s);
    }
    cudaFreeAsync(smoothed, s);
    if (corr_scratch) cudaFreeAsync(corr_scratch, s);
    return rc;
}

// ------------------------------------------------- blocks split across time shards
// with frame-balanced shards a block may straddle ranks.  Each
// contributing rank runs launch_block_piece on its frames of the block (in
// recording order): the corrected frames continue the block's float64 running
// sum -- the same sequence of adds block_mean_kernel performs, so the chained
// sum is bit-identical -- and the smoothed frames are appended to the block's
// smoothed buffer, which travels to the rank holding the block's last frame.
// That rank runs launch_block_finish: mean = f32(sum / cnt) and the existing
// max - median selection over the assembled buffer.

// partial[i] += sum_t corrected[t][i], sequentially in frame order.
__global__ void sum_continue_kernel(const float* __restrict__ frames, int64_t n, int64_t hw,
                                    double* __restrict__ partial) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x) {
        const float* col = frames + i;
        double s = partial[i];
#pragma unroll 8
        for (int64_t t = 0; t < n; ++t) s += (double)__ldcs(col + t * hw);
        partial[i] = s;
    }
}

__global__ void mean_finish_kernel(const double* __restrict__ sum, int64_t hw, int cnt, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (float)(sum[i] / (double)cnt);
}

int launch_block_piece(const void* frames, int dtype, const vb_motion* vec, int64_t n, int h, int w,
                       const double* weights, int wradius, const float* gain, int64_t mean_off, int64_t mean_n,
                       float* corrected, float* smoothed, double* partial, cudaStream_t s) {
    if (n <= 0) return VB_OK;
    if (wradius > kMaxWR) return fail(VB_EINVAL, "smoothing radius too large (max 16)");
    const int64_t hw = (int64_t)h * w;
    const size_t esz = dtype == VB_U16 ? 2 : 4;
    auto at = [&](int64_t i) { return (const char*)frames + (size_t)i * hw * esz; };
    auto vat = [&](int64_t i) { return vec ? vec + i : nullptr; };
    float* corr = corrected;
    float* scratch = nullptr;
    keep_pool();
    if (mean_n > 0 && !corr) {
        VB_CUDA(cudaMallocAsync(&scratch, (size_t)mean_n * hw * sizeof(float), s));
        corr = scratch;
    }
    const int64_t m1 = mean_off + mean_n;
    int rc = launch_k3(at(0), dtype, vat(0), mean_off, h, w, weights, wradius, gain, nullptr, smoothed, s);
    if (rc == VB_OK && mean_n > 0)
        rc = launch_k3(at(mean_off), dtype, vat(mean_off), mean_n, h, w, weights, wradius, gain, corr,
                       smoothed + (size_t)mean_off * hw, s);
    if (rc == VB_OK)
        rc = launch_k3(at(m1), dtype, vat(m1), n - m1, h, w, weights, wradius, gain, nullptr,
                       smoothed + (size_t)m1 * hw, s);
    if (rc == VB_OK && mean_n > 0) {
        dim3 grid((unsigned)std::min<int64_t>((hw + 255) / 256, 1024));
        {
            ProfScope ps(kProfOther, s);
            sum_continue_kernel<<<grid, 256, 0, s>>>(corr, mean_n, hw, partial);
        }
        launches().fetch_add(1, std::memory_order_relaxed);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) rc = cuda_fail(e, "sum_continue_kernel");
    }
    if (scratch) cudaFreeAsync(scratch, s);
    return rc;
}

int launch_block_finish(const float* smoothed, int64_t s_lo, int64_t t0, int cnt, int64_t t_total, int hp_window,
                        int64_t hw, const double* sum, float* spatial, float* temporal, cudaStream_t s) {
    const int hh = hp_window > 1 ? hp_window / 2 : 0;
    if (hh > kMaxHalfWindow) return fail(VB_EINVAL, "high-pass window too long (max 1025 frames)");
    if (hh > 0 && cnt > 1024) return fail(VB_EINVAL, "temporal high-pass needs segment_length <= 1024");
    {
        dim3 grid((unsigned)std::min<int64_t>((hw + 255) / 256, 1024));
        ProfScope ps(kProfOther, s);
        mean_finish_kernel<<<grid, 256, 0, s>>>(sum, hw, cnt, spatial);
    }
    VB_LAUNCHED();
    K4Args k4;
    k4.sm = smoothed;
    k4.s_lo = s_lo;
    k4.g0 = t0;
    k4.n = cnt;
    k4.hw = hw;
    k4.L = cnt;
    k4.hh = hh;
    k4.inv_n = 1.0 / (double)(2 * hh + 1);
    k4.t_total = t_total;
    k4.temporal = temporal;
    return launch_median(k4, 1, s);
}

int launch_summarize(const void* frames, int dtype, const vb_motion* vec, int64_t n, int h, int w, int seg_len,
                     const double* weights, int wradius, float* corrected, float* spatial, float* temporal,
                     cudaStream_t s) {
    SummaryOpts o;
    o.t_global0 = 0;
    o.t_total = n;
    o.interior_off = 0;
    o.n_interior = n;
    return launch_summarize_ex(frames, dtype, vec, n, h, w, seg_len, weights, wradius, o, corrected, spatial,
                               temporal, s);
}

// Smoothing only (scipy gaussian_filter on each frame, summarize.py:60-73).
int launch_smooth(const void* frames, int dtype, int64_t n, int h, int w, const double* weights, int wradius,
                  float* out, cudaStream_t s) {
    if (n <= 0) return VB_OK;
    if (wradius > kMaxWR) return fail(VB_EINVAL, "smoothing radius too large (max 16)");
    return launch_k3(frames, dtype, nullptr, n, h, w, weights, wradius, nullptr, nullptr, out, s);
}

// ------------------------------------------------------------ A17 shading gain
// Flat-field gain from the template (opt-in, no reference counterpart):
// G = separable Gaussian of the template (float64 throughout, taps in order
// -r..r, "reflect" borders, vertical then horizontal), gain = f32(G / mean(G))
// with mean(G) summed in a fixed order: 1024 strided float64 partials, then
// the partials in index order (oracle/oracle.c or_shading_gain restates it).
__global__ void gain_vpass_kernel(const float* __restrict__ ref, int h, int w, const double* __restrict__ wt, int r,
                                  double* __restrict__ out) {
    const int64_t hw = (int64_t)h * w;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / w), x = (int)(i - (int64_t)y * w);
        double acc = 0.0;
        for (int j = -r; j <= r; ++j)
            acc = __dadd_rn(acc, __dmul_rn(wt[j + r], (double)ref[(int64_t)reflect_index(y + j, h) * w + x]));
        out[i] = acc;
    }
}

__global__ void gain_hpass_kernel(const double* __restrict__ in, int h, int w, const double* __restrict__ wt, int r,
                                  double* __restrict__ out) {
    const int64_t hw = (int64_t)h * w;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hw; i += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(i / w), x = (int)(i - (int64_t)y * w);
        double acc = 0.0;
        for (int j = -r; j <= r; ++j)
            acc = __dadd_rn(acc, __dmul_rn(wt[j + r], in[(int64_t)y * w + reflect_index(x + j, w)]));
        out[i] = acc;
    }
}

constexpr int kGainPartials = 1024;

__global__ void __launch_bounds__(kGainPartials) gain_norm_kernel(const double* __restrict__ g, int64_t hw,
                                                                   float* __restrict__ gain) {
    __shared__ double part[kGainPartials];
    __shared__ double mean;
    double acc = 0.0;
    for (int64_t i = threadIdx.x; i < hw; i += kGainPartials) acc = __dadd_rn(acc, g[i]);
    part[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int k = 0; k < kGainPartials; ++k) tot = __dadd_rn(tot, part[k]);
        mean = tot / (double)hw;
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < hw; i += kGainPartials) gain[i] = (float)(g[i] / mean);
}

int launch_shading_gain(const float* ref, int h, int w, const double* weights_host, int r, float* gain,
                        cudaStream_t s) {
    const int64_t hw = (int64_t)h * w;
    double *wt = nullptr, *a = nullptr, *b = nullptr;
    keep_pool();
    VB_CUDA(cudaMallocAsync(&wt, (size_t)(2 * r + 1) * sizeof(double), s));
    cudaError_t e = cudaMemcpyAsync(wt, weights_host, (size_t)(2 * r + 1) * sizeof(double), cudaMemcpyHostToDevice, s);
    e = e ? e : cudaMallocAsync(&a, (size_t)hw * sizeof(double), s);
    e = e ? e : cudaMallocAsync(&b, (size_t)hw * sizeof(double), s);
    int rc = VB_OK;
    if (e != cudaSuccess) {
        rc = cuda_fail(e, "vb_shading_gain allocation");
    } else {
        const unsigned grid = (unsigned)std::min<int64_t>((hw + 255) / 256, 4096);
        ProfScope ps(kProfOther, s);
        gain_vpass_kernel<<<grid, 256, 0, s>>>(ref, h, w, wt, r, a);
        gain_hpass_kernel<<<grid, 256, 0, s>>>(a, h, w, wt, r, b);
        gain_norm_kernel<<<1, kGainPartials, 0, s>>>(b, hw, gain);
        launches().fetch_add(3, std::memory_order_relaxed);
        e = cudaGetLastError();
        if (e != cudaSuccess) rc = cuda_fail(e, "shading gain kernels");
    }
    // the host weights must outlive the async copy
    cudaStreamSynchronize(s);
    cudaFreeAsync(wt, s);
    if (a) cudaFreeAsync(a, s);
    if (b) cudaFreeAsync(b, s);
    return rc;
}

}  // namespace vb
