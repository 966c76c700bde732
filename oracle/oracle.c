/* CPU restatement of the voltseg preprocessing stage -- TEST INFRASTRUCTURE ONLY.
 * See oracle.h for the contract and the rule that the product path never
 * links this file.  Compile with -ffp-contract=off: several functions restate
 * numpy/scipy float32/float64 expressions operation by operation, and a fused
 * multiply-add would change their rounding.
 *
 * Reference sources restated (paths under /root/reference/pkg/src/voltseg):
 *   motion.py:24, :52-75, :113-160, :163-200, :211-248
 *   kernels.py:23-86
 *   summarize.py:44-102 (+ scipy.ndimage.gaussian_filter1d, scipy 1.18.1:
 *   _gaussian_kernel1d weights, correlate1d symmetric-kernel loop, "reflect")
 */
#include "oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef double v4d __attribute__((vector_size(32)));  /* lane-wise IEEE double ops */

static inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* motion.py:211-214: video.data[:n].mean(axis=0, dtype=float64).astype(float32).
 * numpy reduces axis 0 of a C-contiguous stack frame by frame (sequential
 * float64 adds), then true_divide by the integer count. */
void or_make_reference(const float* frames, int n, int h, int w, float* out) {
    size_t px = (size_t)h * (size_t)w;
    double* acc = (double*)calloc(px, sizeof(double));
    for (int t = 0; t < n; t++) {
        const float* f = frames + (size_t)t * px;
        for (size_t i = 0; i < px; i++) acc[i] += (double)f[i];
    }
    for (size_t i = 0; i < px; i++) out[i] = (float)(acc[i] / (double)n);
    free(acc);
}

/* motion.py:71-75 _positions: range(lo, hi+1, stride) plus a final flush to hi. */
static int positions(int lo, int hi, int stride, int* out) {
    int k = 0;
    for (int p = lo; p <= hi; p += stride) { if (out) out[k] = p; k++; }
    int last = lo + (k - 1) * stride;
    if (last != hi) { if (out) out[k] = hi; k++; }
    return k;
}

/* motion.py:52-68 PatchGrid.cover. */
int or_patch_grid(int h, int w, int patch, int stride, int margin, int32_t* origins) {
    if (stride <= 0) stride = patch;
    int lo_x = margin, hi_x = w - margin - patch;
    int lo_y = margin, hi_y = h - margin - patch;
    if (hi_x < lo_x || hi_y < lo_y) return -1;
    int nx = positions(lo_x, hi_x, stride, NULL);
    int ny = positions(lo_y, hi_y, stride, NULL);
    if (origins) {
        int* xs = (int*)malloc(sizeof(int) * (size_t)nx);
        int* ys = (int*)malloc(sizeof(int) * (size_t)ny);
        positions(lo_x, hi_x, stride, xs);
        positions(lo_y, hi_y, stride, ys);
        int k = 0;
        for (int j = 0; j < ny; j++)
            for (int i = 0; i < nx; i++) { origins[2 * k] = xs[i]; origins[2 * k + 1] = ys[j]; k++; }
        free(xs); free(ys);
    }
    return nx * ny;
}

/* kernels.py:23-75.  Float64 throughout.  The reference obtains the window sums
 * from summed-area tables; the direct sums below are the same quantities. */
int or_mean_zncc_scores(const float* frame, const float* ref, int h, int w,
                        const int32_t* origins, int n, int patch, int radius,
                        double* out) {
    int side = 2 * radius + 1;
    for (int i = 0; i < n; i++) {   /* kernels.py:39-42 */
        int x = origins[2 * i], y = origins[2 * i + 1];
        if (x - radius < 0 || y - radius < 0 || x + patch + radius > w || y + patch + radius > h)
            return -1;
    }
    double nn = (double)patch * (double)patch;
    memset(out, 0, sizeof(double) * (size_t)side * (size_t)side);
    for (int i = 0; i < n; i++) {
        int px = origins[2 * i], py = origins[2 * i + 1];
        double rsum = 0.0, rsq = 0.0;   /* kernels.py:49-51 */
        for (int yy = 0; yy < patch; yy++)
            for (int xx = 0; xx < patch; xx++) {
                double v = (double)ref[(size_t)(py + yy) * w + px + xx];
                rsum += v; rsq += v * v;
            }
        double rvar = rsq - rsum * rsum / nn;
        if (!(rvar > 0.0)) continue;    /* kernels.py:52 live mask; z stays 0 */
        for (int dy = -radius; dy <= radius; dy++) {
            int dx = -radius;
            /* four candidates dx..dx+3 at a time: each lane accumulates its own
             * candidate's sums in the same (yy, xx) order as the scalar loop
             * below, so the results are bit-identical to it (speed only) */
            for (; dx + 3 <= radius; dx += 4) {
                v4d cross = {0, 0, 0, 0}, fs = {0, 0, 0, 0}, fq = {0, 0, 0, 0};
                for (int yy = 0; yy < patch; yy++) {
                    const float* fr = frame + (size_t)(py + dy + yy) * w + px + dx;
                    const float* rr = ref + (size_t)(py + yy) * w + px;
                    for (int xx = 0; xx < patch; xx++) {
                        v4d f = {(double)fr[xx], (double)fr[xx + 1], (double)fr[xx + 2], (double)fr[xx + 3]};
                        double r = (double)rr[xx];
                        v4d rv = {r, r, r, r};
                        cross += rv * f; fs += f; fq += f * f;
                    }
                }
                for (int l = 0; l < 4; l++) {
                    double fvar = fq[l] - fs[l] * fs[l] / nn;
                    if (!(fvar > 0.0)) continue;
                    double cov = cross[l] - fs[l] * rsum / nn;
                    out[(size_t)(dy + radius) * side + dx + l + radius] += cov / sqrt(fvar * rvar);
                }
            }
            for (; dx <= radius; dx++) {
                double cross = 0.0, fs = 0.0, fq = 0.0;
                for (int yy = 0; yy < patch; yy++) {
                    const float* fr = frame + (size_t)(py + dy + yy) * w + px + dx;
                    const float* rr = ref + (size_t)(py + yy) * w + px;
                    for (int xx = 0; xx < patch; xx++) {
                        double f = (double)fr[xx];
                        cross += (double)rr[xx] * f; fs += f; fq += f * f;
                    }
                }
                double fvar = fq - fs * fs / nn;          /* kernels.py:67 */
                if (!(fvar > 0.0)) continue;              /* kernels.py:69 */
                double cov = cross - fs * rsum / nn;      /* kernels.py:68 */
                out[(size_t)(dy + radius) * side + dx + radius] += cov / sqrt(fvar * rvar);
            }
        }
    }
    for (int k = 0; k < side * side; k++) out[k] /= (double)n;   /* kernels.py:73 z.sum()/N */
    return 0;
}

/* motion.py:153-160 _quadratic_peak. */
static double quadratic_peak(const double* line, int stride, int len, int i) {
    if (i <= 0 || i >= len - 1) return 0.0;
    double a = line[(size_t)(i - 1) * stride], b = line[(size_t)i * stride], c = line[(size_t)(i + 1) * stride];
    double denom = a - 2.0 * b + c;
    if (denom >= 0) return 0.0;
    double off = 0.5 * (a - c) / denom;
    if (off < -0.999) off = -0.999;
    if (off > 0.999) off = 0.999;
    return off;
}

/* motion.py:113-150: argmax over candidates visited in (|dx|+|dy|, dy, dx)
 * order (first maximum wins), then the two 1-D quadratic fits. */
void or_pick_motion(const double* scores, int radius, int subpixel,
                    int32_t* dxdy, double* sub_conf) {
    int side = 2 * radius + 1;
    int best_dx = 0, best_dy = 0;
    double best = -INFINITY;
    int found = 0;
    for (int l1 = 0; l1 <= 2 * radius; l1++)
        for (int dy = -radius; dy <= radius; dy++)
            for (int dx = -radius; dx <= radius; dx++) {
                if (abs(dx) + abs(dy) != l1) continue;
                double s = scores[(size_t)(dy + radius) * side + dx + radius];
                if (!found || s > best) { best = s; best_dx = dx; best_dy = dy; found = 1; }
            }
    double sdx = 0.0, sdy = 0.0;
    if (subpixel) {
        sdx = quadratic_peak(scores + (size_t)(best_dy + radius) * side, 1, side, best_dx + radius);
        sdy = quadratic_peak(scores + (best_dx + radius), side, side, best_dy + radius);
    }
    dxdy[0] = best_dx; dxdy[1] = best_dy;
    sub_conf[0] = sdx; sub_conf[1] = sdy; sub_conf[2] = best;
}

/* motion.py:163-200 translate / _translate_int: out[y,x] samples the frame at
 * (y - dy, x - dx) with edge replication (== index clamping). */
void or_translate(const float* frame, int h, int w, double dx, double dy, float* out) {
    if (dx == floor(dx) && dy == floor(dy)) {
        int ix = (int)dx, iy = (int)dy;
        for (int y = 0; y < h; y++) {
            int sy = clampi(y - iy, 0, h - 1);
            for (int x = 0; x < w; x++) out[(size_t)y * w + x] = frame[(size_t)sy * w + clampi(x - ix, 0, w - 1)];
        }
        return;
    }
    double fx0 = floor(dx), fy0 = floor(dy);
    int x0 = (int)fx0, y0 = (int)fy0;
    float fx = (float)(dx - fx0), fy = (float)(dy - fy0);
    float one = 1.0f;
    float omx = one - fx, omy = one - fy;
    for (int y = 0; y < h; y++) {
        int ya = clampi(y - y0, 0, h - 1), yc = clampi(y - y0 - 1, 0, h - 1);
        for (int x = 0; x < w; x++) {
            int xa = clampi(x - x0, 0, w - 1), xb = clampi(x - x0 - 1, 0, w - 1);
            float a = frame[(size_t)ya * w + xa], b = frame[(size_t)ya * w + xb];
            float c = frame[(size_t)yc * w + xa], d = frame[(size_t)yc * w + xb];
            float top = omx * a + fx * b;     /* ((1-fx)*a + fx*b) */
            float bot = omx * c + fx * d;
            out[(size_t)y * w + x] = omy * top + fy * bot;
        }
    }
}

/* motion.py:235-240 / :244-248. */
void or_correct_frame(const float* frame, int h, int w, double vx, double vy, float* out) {
    if (vx == 0.0 && vy == 0.0) { memcpy(out, frame, sizeof(float) * (size_t)h * w); return; }
    or_translate(frame, h, w, -vx, -vy, out);
}

/* summarize.py:55-57. */
void or_spatial_summary(const float* frames, int n, int h, int w, float* out) {
    or_make_reference(frames, n, h, w, out);
}

/* scipy "reflect" extension (d c b a | a b c d | d c b a), any overhang. */
static inline int reflect_index(int i, int n) {
    int period = 2 * n;
    int m = i % period;
    if (m < 0) m += period;
    return m >= n ? period - 1 - m : m;
}

/* One scipy correlate1d pass with an odd symmetric kernel: float64 line
 * buffer, o = x[0]*w[0]; for j = -r..-1: o += (x[j] + x[-j]) * w[j]. */
static double corr_sym(const double* line, int stride, int n, int i, const double* wc, int r) {
    double o = line[(size_t)i * stride] * wc[0];
    for (int j = -r; j < 0; j++) {
        double lo = line[(size_t)reflect_index(i + j, n) * stride];
        double hi = line[(size_t)reflect_index(i - j, n) * stride];
        o += (lo + hi) * wc[j];
    }
    return o;
}

void or_smooth_frame(const float* in, int h, int w, const double* weights, int radius,
                     float* out, double* scratch) {
    const double* wc = weights + radius;
    size_t px = (size_t)h * w;
    double* buf = scratch ? scratch : (double*)malloc(sizeof(double) * px);
    float* mid = (float*)malloc(sizeof(float) * px);
    for (size_t i = 0; i < px; i++) buf[i] = (double)in[i];
    /* axis 1 (H) first: summarize.py:72 */
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++) mid[(size_t)y * w + x] = (float)corr_sym(buf + x, w, h, y, wc, radius);
    for (size_t i = 0; i < px; i++) buf[i] = (double)mid[i];
    /* then axis 2 (W): summarize.py:73 */
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++) out[(size_t)y * w + x] = (float)corr_sym(buf + (size_t)y * w, 1, w, x, wc, radius);
    free(mid);
    if (!scratch) free(buf);
}

static int cmp_float(const void* a, const void* b) {
    float x = *(const float*)a, y = *(const float*)b;
    return (x > y) - (x < y);
}

/* summarize.py:76-92. */
int or_temporal_summary(const float* frames, int n, int h, int w,
                        const double* weights, int radius, float* out) {
    if (n < 2) return -1;
    size_t px = (size_t)h * w;
    float* sm = (float*)malloc(sizeof(float) * px * (size_t)n);
    double* scratch = (double*)malloc(sizeof(double) * px);
    for (int t = 0; t < n; t++) or_smooth_frame(frames + (size_t)t * px, h, w, weights, radius, sm + (size_t)t * px, scratch);
    float* col = (float*)malloc(sizeof(float) * (size_t)n);
    int mid = n / 2;
    for (size_t i = 0; i < px; i++) {
        float peak = sm[i];
        for (int t = 0; t < n; t++) { col[t] = sm[(size_t)t * px + i]; if (col[t] > peak) peak = col[t]; }
        qsort(col, (size_t)n, sizeof(float), cmp_float);
        float med = (n % 2) ? col[mid] : (col[mid - 1] + col[mid]) * 0.5f;
        out[i] = peak - med;
    }
    free(col); free(scratch); free(sm);
    return 0;
}

/* traces.py:23-34.  numpy reduces the gathered row with pairwise summation;
 * the sequential float64 sum differs only at ~1e-15 relative. */
void or_extract_trace(const float* frames, int t, int h, int w, const int32_t* idx, int n, double* out) {
    size_t px = (size_t)h * w;
    for (int k = 0; k < t; k++) {
        double s = 0.0;
        for (int i = 0; i < n; i++) s += (double)frames[(size_t)k * px + idx[i]];
        out[k] = s / (double)n;
    }
}

/* ---- A17 extensions ------------------------------------------------------
 * The north-star's shading correction and temporal high-pass have NO code in
 * the reference; the two functions below are their
 * DEFINITION (parity unpinned to the reference), restated from
 * include/voltb200.h vb_shading_gain / vb_summary_opts.highpass_window. */

/* gain = f32(G / mean(G)); G = float64 Gaussian of ref, vertical then
 * horizontal, taps j = -r..r in order (acc += w[j+r] * x), "reflect";
 * mean = (sum of 1024 strided partials, in index order) / (h*w). */
void or_shading_gain(const float* ref, int h, int w, const double* wt, int r, float* gain) {
    size_t px = (size_t)h * w;
    double* a = (double*)malloc(sizeof(double) * px);
    double* g = (double*)malloc(sizeof(double) * px);
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++) {
            double acc = 0.0;
            for (int j = -r; j <= r; j++) acc += wt[j + r] * (double)ref[(size_t)reflect_index(y + j, h) * w + x];
            a[(size_t)y * w + x] = acc;
        }
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++) {
            double acc = 0.0;
            for (int j = -r; j <= r; j++) acc += wt[j + r] * a[(size_t)y * w + reflect_index(x + j, w)];
            g[(size_t)y * w + x] = acc;
        }
    enum { NP = 1024 };
    double part[NP];
    for (int k = 0; k < NP; k++) {
        double s = 0.0;
        for (size_t i = (size_t)k; i < px; i += NP) s += g[i];
        part[k] = s;
    }
    double tot = 0.0;
    for (int k = 0; k < NP; k++) tot += part[k];
    double mean = tot / (double)px;
    for (size_t i = 0; i < px; i++) gain[i] = (float)(g[i] / mean);
    free(a); free(g);
}

/* Temporal summaries with the high-pass: sm = smoothed frames of the whole
 * recording (summarize.py:70-73 per frame); for every frame t
 *   hp[t] = f32( f64(sm[t]) - (sum_{tau=-hh..hh} f64(sm[reflect(t+tau, T)])) * (1/N) ),
 * N = window = 2*hh+1, the sum taken in tau order; then per block of L frames
 * max - median of hp (summarize.py:76-92 with hp in place of sm). */
int or_highpass_summary(const float* corrected, int T, int h, int w, const double* weights, int radius,
                        int segment_length, int window, float* temporal) {
    if (T < 1 || segment_length < 2 || window < 3 || window % 2 == 0) return -1;
    size_t px = (size_t)h * w;
    int hh = window / 2;
    double inv_n = 1.0 / (double)window;
    float* sm = (float*)malloc(sizeof(float) * px * (size_t)T);
    double* scratch = (double*)malloc(sizeof(double) * px);
    for (int t = 0; t < T; t++) or_smooth_frame(corrected + (size_t)t * px, h, w, weights, radius, sm + (size_t)t * px, scratch);
    float* col = (float*)malloc(sizeof(float) * (size_t)segment_length);
    int nseg = (T + segment_length - 1) / segment_length;
    for (int s = 0; s < nseg; s++) {
        int lo = s * segment_length, n = (lo + segment_length < T ? lo + segment_length : T) - lo;
        if (n < 2) { free(col); free(scratch); free(sm); return -2; }
        int mid = n / 2;
        for (size_t i = 0; i < px; i++) {
            float peak = 0.f;
            for (int k = 0; k < n; k++) {
                int t = lo + k;
                double acc = 0.0;
                for (int tau = -hh; tau <= hh; tau++) acc += (double)sm[(size_t)reflect_index(t + tau, T) * px + i];
                float hp = (float)((double)sm[(size_t)t * px + i] - acc * inv_n);
                col[k] = hp;
                if (k == 0 || hp > peak) peak = hp;
            }
            qsort(col, (size_t)n, sizeof(float), cmp_float);
            float med = (n % 2) ? col[mid] : (col[mid - 1] + col[mid]) * 0.5f;
            temporal[(size_t)s * px + i] = peak - med;
        }
    }
    free(col); free(scratch); free(sm);
    return 0;
}

/* ---- whole stage ------------------------------------------------------- */

/* ---- threaded drivers (same per-frame / per-pixel arithmetic) ------------ */

typedef struct {
    void (*fn)(void* ctx, long lo, long hi);
    void* ctx;
    long lo, hi;
} range_job;

static void* range_worker(void* arg) {
    range_job* j = (range_job*)arg;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}

/* fn(ctx, lo, hi) over [0, n) split into nthreads contiguous ranges. */
static void parallel_for(long n, int nthreads, void (*fn)(void*, long, long), void* ctx) {
    if (nthreads > n) nthreads = (int)n;
    if (nthreads <= 1) { if (n > 0) fn(ctx, 0, n); return; }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)nthreads);
    range_job* jobs = (range_job*)malloc(sizeof(range_job) * (size_t)nthreads);
    for (int k = 0; k < nthreads; k++) {
        range_job j = {fn, ctx, n * k / nthreads, n * (k + 1) / nthreads};
        jobs[k] = j;
        pthread_create(&th[k], NULL, range_worker, &jobs[k]);
    }
    for (int k = 0; k < nthreads; k++) pthread_join(th[k], NULL);
    free(th); free(jobs);
}

typedef struct {
    const float* frames; const float* ref; const int32_t* origins;
    int h, w, n, patch, radius, subpixel;
    int32_t* dxdy; double* sub_conf; float* corrected; double* scores;
} motion_ctx;

static void motion_range(void* arg, long t0, long t1) {
    motion_ctx* j = (motion_ctx*)arg;
    int side = 2 * j->radius + 1;
    double* own = (double*)malloc(sizeof(double) * (size_t)side * side);
    size_t px = (size_t)j->h * j->w;
    for (long t = t0; t < t1; t++) {
        const float* f = j->frames + (size_t)t * px;
        double* scores = j->scores ? j->scores + (size_t)t * side * side : own;
        or_mean_zncc_scores(f, j->ref, j->h, j->w, j->origins, j->n, j->patch, j->radius, scores);
        or_pick_motion(scores, j->radius, j->subpixel, j->dxdy + 2 * t, j->sub_conf + 3 * t);
        if (j->corrected) {
            double vx = (double)j->dxdy[2 * t] + j->sub_conf[3 * t];
            double vy = (double)j->dxdy[2 * t + 1] + j->sub_conf[3 * t + 1];
            or_correct_frame(f, j->h, j->w, vx, vy, j->corrected + (size_t)t * px);
        }
    }
    free(own);
}

int or_motion_frames(const float* frames, int t, int h, int w, const float* ref,
                     const int32_t* origins, int n, int patch, int radius, int subpixel, int nthreads,
                     int32_t* dxdy, double* sub_conf, float* corrected, double* scores) {
    if (radius < 1) return -1;
    for (int i = 0; i < n; i++) {
        int x = origins[2 * i], y = origins[2 * i + 1];
        if (x - radius < 0 || y - radius < 0 || x + patch + radius > w || y + patch + radius > h) return -1;
    }
    motion_ctx c = {frames, ref, origins, h, w, n, patch, radius, subpixel, dxdy, sub_conf, corrected, scores};
    parallel_for(t, nthreads, motion_range, &c);
    return 0;
}

typedef struct {
    const float* in; float* out; int h, w, n; const double* weights; int radius;
    float* spatial; float* temporal;
} summ_ctx;

static void smooth_range(void* arg, long t0, long t1) {
    summ_ctx* c = (summ_ctx*)arg;
    size_t px = (size_t)c->h * c->w;
    double* scratch = (double*)malloc(sizeof(double) * px);
    for (long t = t0; t < t1; t++)
        or_smooth_frame(c->in + (size_t)t * px, c->h, c->w, c->weights, c->radius, c->out + (size_t)t * px, scratch);
    free(scratch);
}

/* summarize.py:55-57 and :76-92 per pixel (the smoothed stack in c->out). */
static void pixel_range(void* arg, long i0, long i1) {
    summ_ctx* c = (summ_ctx*)arg;
    size_t px = (size_t)c->h * c->w;
    int n = c->n, mid = n / 2;
    float* col = (float*)malloc(sizeof(float) * (size_t)n);
    for (long i = i0; i < i1; i++) {
        double acc = 0.0;
        for (int t = 0; t < n; t++) acc += (double)c->in[(size_t)t * px + i];
        c->spatial[i] = (float)(acc / (double)n);
        if (n < 2) continue;
        const float* sm = c->out;
        float peak = sm[i];
        for (int t = 0; t < n; t++) { col[t] = sm[(size_t)t * px + i]; if (col[t] > peak) peak = col[t]; }
        qsort(col, (size_t)n, sizeof(float), cmp_float);
        float med = (n % 2) ? col[mid] : (col[mid - 1] + col[mid]) * 0.5f;
        c->temporal[i] = peak - med;
    }
    free(col);
}

/* summarize.py:95-102 over corrected frames [t][h][w]: one (spatial, temporal)
 * pair per block of segment_length frames; a 1-frame tail returns -1 (the
 * reference raises).  Frames are smoothed in parallel, pixels reduced in
 * parallel; the arithmetic per frame / pixel is or_smooth_frame /
 * or_spatial_summary / or_temporal_summary's. */
int or_summaries(const float* corrected, int t, int h, int w, int segment_length,
                 const double* weights, int wradius, int nthreads, float* spatial, float* temporal) {
    if (segment_length < 2) return -1;
    size_t px = (size_t)h * w;
    int nseg = (t + segment_length - 1) / segment_length;
    if (t - (nseg - 1) * segment_length < 2) return -1;
    float* sm = (float*)malloc(sizeof(float) * px * (size_t)(t < segment_length ? t : segment_length));
    for (int s = 0; s < nseg; s++) {
        int lo = s * segment_length, hi = lo + segment_length < t ? lo + segment_length : t;
        summ_ctx c = {corrected + (size_t)lo * px, sm, h, w, hi - lo, weights, wradius,
                      spatial + (size_t)s * px, temporal + (size_t)s * px};
        parallel_for(hi - lo, nthreads, smooth_range, &c);
        parallel_for((long)px, nthreads, pixel_range, &c);
    }
    free(sm);
    return 0;
}

int or_preprocess(const float* frames, int t, int h, int w, int patch, int radius,
                  int subpixel, int ref_frames, int segment_length,
                  const double* weights, int wradius, int nthreads,
                  int32_t* dxdy, double* sub_conf, float* corrected,
                  float* spatial, float* temporal) {
    if (radius < 1 || segment_length < 2) return -1;
    size_t px = (size_t)h * w;
    int n = or_patch_grid(h, w, patch, patch, radius, NULL);
    if (n < 0) return -1;
    int32_t* origins = (int32_t*)malloc(sizeof(int32_t) * 2 * (size_t)n);
    or_patch_grid(h, w, patch, patch, radius, origins);
    float* ref = (float*)malloc(sizeof(float) * px);
    or_make_reference(frames, t < ref_frames ? t : ref_frames, h, w, ref);
    int own = corrected == NULL;
    float* corr = own ? (float*)malloc(sizeof(float) * px * (size_t)t) : corrected;
    if (nthreads < 1) nthreads = 1;
    or_motion_frames(frames, t, h, w, ref, origins, n, patch, radius, subpixel, nthreads, dxdy, sub_conf, corr, NULL);
    int nseg = (t + segment_length - 1) / segment_length;
    for (int s = 0; s < nseg; s++) {
        int lo = s * segment_length, hi = lo + segment_length < t ? lo + segment_length : t;
        if (spatial) or_spatial_summary(corr + (size_t)lo * px, hi - lo, h, w, spatial + (size_t)s * px);
        if (temporal && hi - lo >= 2)
            or_temporal_summary(corr + (size_t)lo * px, hi - lo, h, w, weights, wradius, temporal + (size_t)s * px);
    }
    if (own) free(corr);
    free(ref); free(origins);
    return 0;
}
