// C-ABI entry points and the host runtime (plans, chunked stage executor).
// See include/voltb200.h for the contract and the reference interfaces each
// entry point replaces.
#include <cuda_runtime.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <string>
#include <vector>

#include <cudaTypedefs.h>

#include "tma.cuh"
#include "vb.cuh"

namespace vb {

// cuTensorMapEncodeTiled through the runtime's driver entry point.
bool make_frames_tmap(CUtensorMap* map, const void* base, int dtype, int64_t t, int h, int w, int bh, int bw,
                      int bt) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        cudaGetLastError();
    }
    if (!encode || !base) return false;
    const size_t esz = dtype == VB_U16 ? 2 : 4;
    if ((reinterpret_cast<uintptr_t>(base) & 15) || ((size_t)w * esz) % 16 || ((size_t)h * w * esz) % 16) return false;
    if (bw < 1 || bh < 1 || bt < 1 || bw > 256 || bh > 256 || bt > 256 || ((size_t)bw * esz) % 16) return false;
    cuuint64_t dims[3] = {(cuuint64_t)w, (cuuint64_t)h, (cuuint64_t)(t > 0 ? t : 1)};
    cuuint64_t strides[2] = {(cuuint64_t)(w * esz), (cuuint64_t)((size_t)h * w * esz)};
    cuuint32_t box[3] = {(cuuint32_t)bw, (cuuint32_t)bh, (cuuint32_t)bt};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = encode(map, dtype == VB_U16 ? CU_TENSOR_MAP_DATA_TYPE_UINT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                        const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}
int cuda_fail(cudaError_t e, const char* where) {
    g_err = std::string("CUDA error in ") + where + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? VB_ENOMEM : VB_ECUDA;
}
std::atomic<int64_t>& launches() { return g_launches; }

// Scratch (partials, smoothed blocks) comes from the stream-ordered pool;
// keep freed blocks cached instead of unmapping them at every sync.
void keep_pool() {
    static std::atomic<uint64_t> done_mask{0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return;
    const uint64_t bit = 1ull << dev;
    if (done_mask.load() & bit) return;
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    done_mask.fetch_or(bit);
}

// motion.py:71-75
static std::vector<int> positions(int lo, int hi, int stride) {
    std::vector<int> pos;
    for (int p = lo; p <= hi; p += stride) pos.push_back(p);
    if (pos.back() != hi) pos.push_back(hi);
    return pos;
}

static int check_origins(int h, int w, const int32_t* origins, int n, int patch, int radius) {
    for (int i = 0; i < n; ++i) {  // _native.pyx:41-46, kernels.py:39-42
        const int px = origins[2 * i], py = origins[2 * i + 1];
        if (px - radius < 0 || py - radius < 0 || px + patch + radius > w || py + patch + radius > h)
            return fail(VB_EINVAL, "patch origin too close to border for search radius");
    }
    if (radius > kMaxRadius) return fail(VB_EINVAL, "search radius too large (max 31)");  // _native.pyx:65-66
    if (radius < 0) return fail(VB_EINVAL, "search_radius must be >= 1");
    if (patch < 1) return fail(VB_EINVAL, "patch size must be >= 1");
    // exact integer window sums: sum(f - c) in int32 and P^2*sum((f - c)^2) in int64
    if (patch > kMaxPatch) return fail(VB_EINVAL, "patch size too large (max 180)");
    return VB_OK;
}

}  // namespace vb

using namespace vb;

// ---------------------------------------------------------------- plan
struct vb_motion_plan {
    int h = 0, w = 0, patch = 0, radius = 0;
    Templates t;
    std::vector<int32_t> origins;
    bool have_ref = false;
};

static void free_templates(Templates& t) {
    cudaFree(t.t16);
    cudaFree(t.tscale);
    cudaFree(t.tmpl);
    cudaFree(t.rvar);
    cudaFree(t.origins);
    cudaFree(t.patch_col);
    cudaFree(t.groups);
    t = Templates();
}

// Group consecutive patches that share an origin row into CTA work units:
// each run of equal-y patches is split into ceil(run / max_g) groups of
// near-equal size (balanced CTAs).
static void build_groups(const std::vector<int32_t>& o, int patch, int radius, int max_g,
                         std::vector<PatchGroup>& groups, std::vector<int32_t>& col) {
    const int n = (int)o.size() / 2;
    col.assign(n, 0);
    int i = 0;
    while (i < n) {
        // run of patches on the same row whose union stays compact
        int run = 1;
        int rmin = o[2 * i], rmax = o[2 * i];
        while (i + run < n && o[2 * (i + run) + 1] == o[2 * i + 1]) {
            const int x = o[2 * (i + run)];
            const int nmin = std::min(rmin, x), nmax = std::max(rmax, x);
            if (nmax - nmin > (run + 1) * patch) break;
            rmin = nmin;
            rmax = nmax;
            ++run;
        }
        const int k = (run + max_g - 1) / max_g;
        for (int q = 0, start = i; q < k; ++q) {
            const int cnt = run / k + (q < run % k ? 1 : 0);
            PatchGroup g;
            memset(&g, 0, sizeof(g));
            g.first = start;
            g.count = cnt;
            int minx = o[2 * start], maxx = o[2 * start];
            for (int j = start; j < start + cnt; ++j) {
                minx = std::min(minx, (int)o[2 * j]);
                maxx = std::max(maxx, (int)o[2 * j]);
            }
            g.x0 = minx - radius;
            g.y0 = o[2 * start + 1] - radius;
            g.wu = maxx - minx + patch + 2 * radius;
            for (int j = start; j < start + cnt; ++j) col[j] = o[2 * j] - minx;
            groups.push_back(g);
            start += cnt;
        }
        i += run;
    }
}

// Pick the group size: lane efficiency of the (patch, dy[, dx-chunk]) item
// loop times an occupancy factor, subject to the shared-memory budget.
static int choose_group_size(const std::vector<int32_t>& o, int patch, int radius) {
    const int S = 2 * radius + 1;
    const int nch = (patch == 21 && S <= 25) ? 1 : (S + 7) / 8;
    double best = -1.0;
    int best_g = 1;
    std::vector<PatchGroup> groups;
    std::vector<int32_t> col;
    for (int g = 1; g <= kMaxGroup; ++g) {
        groups.clear();
        build_groups(o, patch, radius, g, groups, col);
        int mg = 0, mw = 0;
        long long items = 0;
        for (auto& x : groups) {
            mg = std::max(mg, (int)x.count);
            mw = std::max(mw, (int)x.wu);
            items += (long long)x.count * S * nch;
        }
        // feasibility with the larger (f32-input) layout; occupancy for camera (u16) input
        if (zncc_smem_bytes(patch, radius, mg, mw, VB_F32) > 160 * 1024 && g > 1) break;
        const size_t smem = zncc_search_smem_bytes(patch, radius, mg, mw, VB_U16);
        const int max_items = mg * S * nch;
        const int threads = std::max(64, std::min(256, (max_items + 31) / 32 * 32));
        const int rounds = (max_items + threads - 1) / threads;
        const double lane_eff = (double)items / ((double)groups.size() * rounds * threads);
        // measured (G sweep, C2): >= 4 resident CTAs per SM with L1 headroom for
        // the broadcast template taps beats larger groups with fewer CTAs
        const int by_smem = (int)((228 * 1024) / (smem + 1024));
        const int by_regs = 65536 / (threads * 72);
        const int ctas = std::max(1, std::min(std::min(by_smem, by_regs), 32));
        const double occ = std::min(1.0, ctas / 4.0);
        const double score = lane_eff * occ;
        if (score >= best - 1e-9) {  // ties: larger groups (fewer CTAs, less per-group overhead; measured)
            best = score;
            best_g = g;
        }
    }
    return best_g;
}

// Row pitch of the search kernel's f32 region.  A warp's lanes are (patch,
// dy) items reading region[dy * pitch + col_p + i] in lock step (the same i),
// so the shared-memory wavefronts per LDS are fixed by the residues of
// dy * pitch + col_p mod 32.  Pick the odd pitch in [max_wu, max_wu + 64)
// with the fewest wavefronts over every warp of every group (ties: smallest).
static int choose_pitch(const std::vector<PatchGroup>& groups, const std::vector<int32_t>& col, int S,
                        int max_wu, bool split17) {
    int best_pitch = max_wu | 1;
    long long best = -1;
    for (int pitch = max_wu | 1; pitch < max_wu + 64; pitch += 2) {
        long long cost = 0;
        for (const auto& g : groups) {
            // lanes -> (patch, candidate row): S rows per patch, or the split
            // search kernel's 16 lanes per patch over rows {0..16} \ {8}
            const int per = split17 ? 16 : S;
            const int items = g.count * per;
            for (int w0 = 0; w0 < items; w0 += 32) {
                int addr[32], n = 0;
                for (int it = w0; it < std::min(items, w0 + 32); ++it) {
                    const int p = it / per, l = it % per;
                    const int dy = split17 ? (l < 8 ? l : l + 1) : l;
                    addr[n++] = dy * pitch + col[g.first + p];
                }
                int worst = 0;
                for (int b = 0; b < 32; ++b) {
                    int m = 0;
                    for (int i = 0; i < n; ++i) {
                        if (((addr[i] % 32) + 32) % 32 != b) continue;
                        bool dup = false;
                        for (int j = 0; j < i; ++j) dup |= addr[j] == addr[i];
                        m += dup ? 0 : 1;
                    }
                    worst = std::max(worst, m);
                }
                cost += worst;
            }
        }
        if (best < 0 || cost < best) {
            best = cost;
            best_pitch = pitch;
        }
    }
    return best_pitch;
}

extern "C" {

const char* vb_version(void) { return "voltb200 0.1 (sm_100a)"; }
const char* vb_last_error(void) { return g_err.c_str(); }
int64_t vb_launch_count(void) { return g_launches.load(); }

// ---- peer memory for the frame-balanced shards' block exchange ----
int vb_ipc_alloc(int64_t bytes, void** dev_ptr, unsigned char* handle) {
    if (!dev_ptr || !handle || bytes <= 0) return fail(VB_EINVAL, "null argument");
    *dev_ptr = nullptr;
    VB_CUDA(cudaMalloc(dev_ptr, (size_t)bytes));
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, *dev_ptr);
    if (e != cudaSuccess) {
        cudaFree(*dev_ptr);
        *dev_ptr = nullptr;
        return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    static_assert(sizeof(cudaIpcMemHandle_t) == VB_IPC_HANDLE_BYTES, "IPC handle size");
    memcpy(handle, &h, sizeof(h));
    return VB_OK;
}

int vb_ipc_open(const unsigned char* handle, void** dev_ptr) {
    if (!handle || !dev_ptr) return fail(VB_EINVAL, "null argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    VB_CUDA(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return VB_OK;
}

int vb_ipc_close(void* dev_ptr) {
    if (dev_ptr) VB_CUDA(cudaIpcCloseMemHandle(dev_ptr));
    return VB_OK;
}

int vb_ipc_free(void* dev_ptr) {
    if (dev_ptr) VB_CUDA(cudaFree(dev_ptr));
    return VB_OK;
}

int vb_memset_async(void* dst, int value, int64_t bytes, void* stream) {
    if (!dst && bytes > 0) return fail(VB_EINVAL, "null argument");
    if (bytes > 0) VB_CUDA(cudaMemsetAsync(dst, value, (size_t)bytes, (cudaStream_t)stream));
    return VB_OK;
}

int vb_copy_async(void* dst, const void* src, int64_t bytes, void* stream) {
    if ((!dst || !src) && bytes > 0) return fail(VB_EINVAL, "null argument");
    if (bytes > 0) VB_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, (cudaStream_t)stream));
    return VB_OK;
}

int vb_patch_grid(int height, int width, int patch, int margin, int32_t* origins, int* n_origins) {
    const int lo_x = margin, hi_x = width - margin - patch;
    const int lo_y = margin, hi_y = height - margin - patch;
    if (patch < 1 || hi_x < lo_x || hi_y < lo_y) {
        return fail(VB_EINVAL, "frame " + std::to_string(height) + "x" + std::to_string(width) +
                                   " too small for patch " + std::to_string(patch) + " with margin " +
                                   std::to_string(margin));
    }
    const std::vector<int> xs = positions(lo_x, hi_x, patch), ys = positions(lo_y, hi_y, patch);
    const int n = (int)(xs.size() * ys.size());
    if (n_origins) *n_origins = n;
    if (origins) {
        int k = 0;
        for (int y : ys)
            for (int x : xs) {
                origins[2 * k] = x;
                origins[2 * k + 1] = y;
                ++k;
            }
    }
    return VB_OK;
}

int vb_motion_plan_create(vb_motion_plan** out, int height, int width, int patch, int radius,
                          const int32_t* origins_host, int n_origins) {
    if (!out) return fail(VB_EINVAL, "null plan pointer");
    *out = nullptr;
    if (n_origins < 1) return fail(VB_EINVAL, "no patches");
    int rc = check_origins(height, width, origins_host, n_origins, patch, radius);
    if (rc) return rc;
    auto* p = new vb_motion_plan();
    p->h = height;
    p->w = width;
    p->patch = patch;
    p->radius = radius;
    p->origins.assign(origins_host, origins_host + 2 * (size_t)n_origins);
    std::vector<PatchGroup> groups;
    std::vector<int32_t> col;
    // group width: ~8 patches keeps the CTA at <= ~80 KB of shared memory;
    // shrink the group until the search CTA fits (large radii)
    const int force_g = knob("VB_GROUP", 0);  // experiment: fixed patches per group
    const int max_g = force_g > 0 ? std::min(kMaxGroup, force_g) : choose_group_size(p->origins, patch, radius);
    build_groups(p->origins, patch, radius, max_g, groups, col);
    Templates& t = p->t;
    t.n = n_origins;
    t.n_groups = (int)groups.size();
    t.tp = (patch + 3) & ~3;
    for (auto& g : groups) {
        t.max_g = std::max(t.max_g, (int)g.count);
        t.max_wu = std::max(t.max_wu, (int)g.wu);
    }
    const int force_pitch = knob("VB_PITCH", -1);  // experiment (0 = max_wu | 1)
    t.pitch = force_pitch >= 0 ? force_pitch
                               : choose_pitch(groups, col, 2 * radius + 1, t.max_wu, patch == 21 && radius == 8);
    if (t.pitch < t.max_wu) t.pitch = t.max_wu | 1;
    cudaError_t e = cudaSuccess;
    e = e ? e : cudaMalloc(&t.tmpl, (size_t)n_origins * patch * t.tp * sizeof(float));
    e = e ? e : cudaMalloc(&t.rvar, 2 * (size_t)n_origins * sizeof(double));
    t.rmean = t.rvar ? t.rvar + n_origins : nullptr;
    e = e ? e : cudaMalloc(&t.origins, (size_t)n_origins * 2 * sizeof(int32_t));
    e = e ? e : cudaMalloc(&t.patch_col, (size_t)n_origins * sizeof(int32_t));
    e = e ? e : cudaMalloc(&t.groups, groups.size() * sizeof(PatchGroup));
    e = e ? e : cudaMemcpy(t.origins, origins_host, (size_t)n_origins * 2 * sizeof(int32_t), cudaMemcpyHostToDevice);
    e = e ? e : cudaMemcpy(t.patch_col, col.data(), col.size() * sizeof(int32_t), cudaMemcpyHostToDevice);
    e = e ? e : cudaMemcpy(t.groups, groups.data(), groups.size() * sizeof(PatchGroup), cudaMemcpyHostToDevice);
#ifdef VB_EXPERIMENTS
    if (e == cudaSuccess && mma_supported(patch, radius, VB_U16)) {  // tensor-core path tables (uint16 frames)
        const MmaGeom g = mma_geom(patch, radius);
        e = e ? e : cudaMalloc(&t.t16, (size_t)n_origins * 3 * 8 * patch * g.tpw);
        e = e ? e : cudaMalloc(&t.tscale, (size_t)n_origins * sizeof(double));
    }
#endif
    if (e != cudaSuccess) {
        free_templates(t);
        delete p;
        return cuda_fail(e, "vb_motion_plan_create");
    }
    *out = p;
    return VB_OK;
}

int vb_motion_plan_set_reference(vb_motion_plan* p, const float* ref_dev, void* stream) {
    if (!p || !ref_dev) return fail(VB_EINVAL, "null argument");
    int rc = launch_prep_templates(ref_dev, p->h, p->w, p->patch, p->t, (cudaStream_t)stream);
#ifdef VB_EXPERIMENTS
    if (rc == VB_OK && p->t.t16) rc = launch_mma_prep(p->t, p->patch, p->radius, (cudaStream_t)stream);
#endif
    if (rc == VB_OK) p->have_ref = true;
    return rc;
}

int vb_motion_estimate(vb_motion_plan* p, const void* frames_dev, int dtype, int64_t n_frames, int subpixel,
                       vb_motion* vectors_dev, double* scores_dev, void* stream) {
    if (!p || !vectors_dev || (!frames_dev && n_frames > 0)) return fail(VB_EINVAL, "null argument");
    if (!p->have_ref) return fail(VB_EINVAL, "motion plan has no reference (call vb_motion_plan_set_reference)");
    if (dtype != VB_U16 && dtype != VB_F32) return fail(VB_EINVAL, "unsupported sample type");
    return launch_motion(p->t, p->h, p->w, p->patch, p->radius, frames_dev, dtype, n_frames, subpixel, vectors_dev,
                         scores_dev, (cudaStream_t)stream);
}

int vb_motion_plan_info(const vb_motion_plan* p, int* n_patches, int* n_groups, int* max_group, int* max_width) {
    if (!p) return fail(VB_EINVAL, "null argument");
    if (n_patches) *n_patches = p->t.n;
    if (n_groups) *n_groups = p->t.n_groups;
    if (max_group) *max_group = p->t.max_g;
    if (max_width) *max_width = p->t.max_wu;
    return VB_OK;
}

int vb_motion_plan_destroy(vb_motion_plan* p) {
    if (!p) return VB_OK;
    free_templates(p->t);
    delete p;
    return VB_OK;
}

int vb_template_sum(const void* frames_dev, int dtype, int64_t n_frames, int height, int width, double* sum_dev,
                    int accumulate, void* stream) {
    if (!sum_dev) return fail(VB_EINVAL, "null argument");
    if (dtype != VB_U16 && dtype != VB_F32) return fail(VB_EINVAL, "unsupported sample type");
    return launch_template_sum(frames_dev, dtype, n_frames, (int64_t)height * width, sum_dev, accumulate,
                               (cudaStream_t)stream);
}

int vb_template_finish(const double* sum_dev, int64_t n_total, int64_t n_pixels, float* ref_dev, void* stream) {
    if (!sum_dev || !ref_dev || n_total < 1) return fail(VB_EINVAL, "invalid template arguments");
    return launch_template_finish(sum_dev, n_total, n_pixels, ref_dev, (cudaStream_t)stream);
}

int vb_make_reference(const void* frames_dev, int dtype, int64_t n_frames, int height, int width, int ref_frames,
                      float* ref_dev, void* stream) {
    if (n_frames < 1 || ref_frames < 1) return fail(VB_EINVAL, "need at least one frame");
    const int64_t n = std::min<int64_t>(n_frames, ref_frames);
    const int64_t hw = (int64_t)height * width;
    cudaStream_t s = (cudaStream_t)stream;
    double* sum = nullptr;
    VB_CUDA(cudaMallocAsync(&sum, hw * sizeof(double), s));
    int rc = launch_template_sum(frames_dev, dtype, n, hw, sum, 0, s);
    if (rc == VB_OK) rc = launch_template_finish(sum, n, hw, ref_dev, s);
    cudaFreeAsync(sum, s);
    return rc;
}

int vb_correct_frames(const void* frames_dev, int dtype, int64_t n_frames, int height, int width,
                      const vb_motion* vectors_dev, float* corrected_dev, void* stream) {
    if (dtype != VB_U16 && dtype != VB_F32) return fail(VB_EINVAL, "unsupported sample type");
    return launch_correct(frames_dev, dtype, n_frames, height, width, vectors_dev, nullptr, corrected_dev,
                          (cudaStream_t)stream);
}

int vb_correct_frames_ex(const void* frames_dev, int dtype, int64_t n_frames, int height, int width,
                         const vb_motion* vectors_dev, const float* gain_dev, float* corrected_dev, void* stream) {
    if (dtype != VB_U16 && dtype != VB_F32) return fail(VB_EINVAL, "unsupported sample type");
    return launch_correct(frames_dev, dtype, n_frames, height, width, vectors_dev, gain_dev, corrected_dev,
                          (cudaStream_t)stream);
}

int vb_shading_gain(const float* ref_dev, int height, int width, const double* weights, int wradius,
                    float* gain_dev, void* stream) {
    if (!ref_dev || !weights || !gain_dev || wradius < 0) return fail(VB_EINVAL, "null argument");
    if (height < 1 || width < 1) return fail(VB_EINVAL, "video dimensions must all be >= 1");
    return launch_shading_gain(ref_dev, height, width, weights, wradius, gain_dev, (cudaStream_t)stream);
}

int vb_summarize_ex(const void* frames_dev, int dtype, const vb_motion* vectors_dev, int64_t n_frames, int height,
                    int width, int segment_length, const double* weights, int wradius, const vb_summary_opts* opts,
                    float* corrected_dev, float* spatial_dev, float* temporal_dev, void* stream) {
    if (!opts)
        return vb_summarize(frames_dev, dtype, vectors_dev, n_frames, height, width, segment_length, weights, wradius,
                            corrected_dev, spatial_dev, temporal_dev, stream);
    if (segment_length < 2) return fail(VB_EINVAL, "segment length must be >= 2");
    if (dtype != VB_U16 && dtype != VB_F32) return fail(VB_EINVAL, "unsupported sample type");
    if (n_frames < 1) return fail(VB_EINVAL, "video dimensions must all be >= 1");
    if (!weights || wradius < 0 || !spatial_dev || !temporal_dev) return fail(VB_EINVAL, "null argument");
    const int64_t L = segment_length, T = opts->t_total;
    const int64_t g0 = opts->t_global0 + opts->interior_off, g1 = g0 + opts->n_interior;
    if (opts->t_global0 < 0 || opts->t_global0 + n_frames > T || opts->interior_off < 0 || opts->n_interior < 0 ||
        opts->interior_off + opts->n_interior > n_frames)
        return fail(VB_EINVAL, "summary interior outside the frame buffer");
    if (g0 % L != 0) return fail(VB_EINVAL, "summary interior must start on a block boundary");
    if (opts->n_interior % L != 0 && g1 != T) return fail(VB_EINVAL, "summary interior must end on a block boundary");
    if (g1 == T && T % L == 1 && opts->n_interior > 0)  // summarize.py:79-80 on the final block
        return fail(VB_EINVAL, "temporal summary needs at least 2 frames");
    const int win = opts->highpass_window;
    if (win > 1) {
        if (win % 2 == 0) return fail(VB_EINVAL, "high-pass window must be odd");
        const int64_t hh = win / 2;
        if (std::max<int64_t>(0, g0 - hh) < opts->t_global0 || std::min<int64_t>(T, g1 + hh) > opts->t_global0 + n_frames)
            return fail(VB_EINVAL, "temporal high-pass halo not in the frame buffer");
    }
    SummaryOpts o;
    o.t_global0 = opts->t_global0;
    o.t_total = T;
    o.interior_off = opts->interior_off;
    o.n_interior = opts->n_interior;
    o.highpass_window = win > 1 ? win : 0;
    o.gain = opts->gain_dev;
    return launch_summarize_ex(frames_dev, dtype, vectors_dev, n_frames, height, width, segment_length, weights,
                               wradius, o, corrected_dev, spatial_dev, temporal_dev, (cudaStream_t)stream);
}

int vb_summarize(const void* frames_dev, int dtype, const vb_motion* vectors_dev, int64_t n_frames, int height,
                 int width, int segment_length, const double* weights, int wradius, float* corrected_dev,
                 float* spatial_dev, float* temporal_dev, void* stream) {
    if (segment_length < 2) return fail(VB_EINVAL, "segment length must be >= 2");  // summarize.py:46-47
    if (dtype != VB_U16 && dtype != VB_F32) return fail(VB_EINVAL, "unsupported sample type");
    if (n_frames < 1) return fail(VB_EINVAL, "video dimensions must all be >= 1");
    if (n_frames % segment_length == 1)  // summarize.py:79-80 on the final block
        return fail(VB_EINVAL, "temporal summary needs at least 2 frames");
    if (!weights || wradius < 0 || !spatial_dev || !temporal_dev) return fail(VB_EINVAL, "null argument");
    return launch_summarize(frames_dev, dtype, vectors_dev, n_frames, height, width, segment_length, weights,
                            wradius, corrected_dev, spatial_dev, temporal_dev, (cudaStream_t)stream);
}

int vb_block_piece(const void* frames_dev, int dtype, const vb_motion* vectors_dev, int64_t n_frames, int height,
                   int width, const double* weights, int wradius, const float* gain_dev, int64_t mean_off,
                   int64_t mean_n, float* corrected_dev, float* smoothed_dev, double* partial_sum_dev,
                   void* stream) {
    if (dtype != VB_U16 && dtype != VB_F32) return fail(VB_EINVAL, "unsupported sample type");
    if (n_frames < 0 || mean_off < 0 || mean_n < 0 || mean_off + mean_n > n_frames)
        return fail(VB_EINVAL, "block piece outside the frame buffer");
    if (!weights || wradius < 0 || (n_frames > 0 && !smoothed_dev) || (mean_n > 0 && !partial_sum_dev))
        return fail(VB_EINVAL, "null argument");
    return launch_block_piece(frames_dev, dtype, vectors_dev, n_frames, height, width, weights, wradius, gain_dev,
                              mean_off, mean_n, corrected_dev, smoothed_dev, partial_sum_dev, (cudaStream_t)stream);
}

int vb_block_finish(const float* smoothed_dev, int64_t s_lo, int64_t n_smoothed, int64_t t0, int64_t count,
                    int64_t t_total, int highpass_window, int height, int width, const double* sum_dev,
                    float* spatial_dev, float* temporal_dev, void* stream) {
    if (count < 2) return fail(VB_EINVAL, "temporal summary needs at least 2 frames");  // summarize.py:79-80
    if (!smoothed_dev || !sum_dev || !spatial_dev || !temporal_dev) return fail(VB_EINVAL, "null argument");
    if (highpass_window > 1 && highpass_window % 2 == 0) return fail(VB_EINVAL, "high-pass window must be odd");
    const int64_t hh = highpass_window > 1 ? highpass_window / 2 : 0;
    const int64_t need_lo = hh ? std::max<int64_t>(0, t0 - hh) : t0;
    const int64_t need_hi = hh ? std::min<int64_t>(t_total, t0 + count + hh) : t0 + count;
    if (t0 < 0 || t0 + count > t_total || need_lo < s_lo || need_hi > s_lo + n_smoothed)
        return fail(VB_EINVAL, "block frames not in the smoothed buffer");
    return launch_block_finish(smoothed_dev, s_lo, t0, (int)count, t_total, highpass_window > 1 ? highpass_window : 0,
                               (int64_t)height * width, sum_dev, spatial_dev, temporal_dev, (cudaStream_t)stream);
}

int vb_smooth_frames(const void* frames_dev, int dtype, int64_t n_frames, int height, int width,
                     const double* weights, int wradius, float* out_dev, void* stream) {
    if (dtype != VB_U16 && dtype != VB_F32) return fail(VB_EINVAL, "unsupported sample type");
    if (!weights || wradius < 0 || !out_dev) return fail(VB_EINVAL, "null argument");
    return launch_smooth(frames_dev, dtype, n_frames, height, width, weights, wradius, out_dev,
                         (cudaStream_t)stream);
}

int vb_mean_zncc_scores(const float* frame, const float* reference, int height, int width, const int32_t* origins,
                        int n_origins, int patch, int radius, double* out_scores) {
    if (!frame || !reference || !origins || !out_scores) return fail(VB_EINVAL, "null argument");
    int rc = check_origins(height, width, origins, n_origins, patch, radius);
    if (rc) return rc;
    const int S = 2 * radius + 1;
    const size_t hw = (size_t)height * width;
    if (n_origins == 0) {  // reference: empty mean -> division by zero yields NaN
        for (int i = 0; i < S * S; ++i) out_scores[i] = NAN;
        return VB_OK;
    }
    // The operator is stateless by contract (kernels.py:98-108), but callers
    // (correct_motion) invoke it once per frame with the same geometry and
    // reference: the calling thread keeps the plan, stream and device buffers
    // of its last geometry and re-uploads / re-prepares the reference only
    // when its bytes change.
    struct OpCache {
        int dev = -1, h = 0, w = 0, patch = 0, radius = 0;
        std::vector<int32_t> origins;
        std::vector<float> ref;
        vb_motion_plan* plan = nullptr;
        cudaStream_t s = nullptr;
        float *d_frame = nullptr, *d_ref = nullptr;
        vb_motion* d_vec = nullptr;
        double* d_scores = nullptr;
        void release() {
            if (s) cudaStreamSynchronize(s);
            cudaFree(d_frame);
            cudaFree(d_ref);
            cudaFree(d_vec);
            cudaFree(d_scores);
            if (s) cudaStreamDestroy(s);
            vb_motion_plan_destroy(plan);
            d_frame = d_ref = nullptr;
            d_vec = nullptr;
            d_scores = nullptr;
            s = nullptr;
            plan = nullptr;
            ref.clear();
            dev = -1;
        }
        ~OpCache() { release(); }
    };
    static thread_local OpCache c;
    int dev = 0;
    VB_CUDA(cudaGetDevice(&dev));
    const bool same = c.plan && c.dev == dev && c.h == height && c.w == width && c.patch == patch &&
                      c.radius == radius && c.origins.size() == 2 * (size_t)n_origins &&
                      memcmp(c.origins.data(), origins, c.origins.size() * sizeof(int32_t)) == 0;
    if (!same) {
        c.release();
        rc = vb_motion_plan_create(&c.plan, height, width, patch, radius, origins, n_origins);
        if (rc) return rc;
        cudaError_t e = cudaStreamCreateWithFlags(&c.s, cudaStreamNonBlocking);
        e = e ? e : cudaMalloc(&c.d_frame, hw * 4);
        e = e ? e : cudaMalloc(&c.d_ref, hw * 4);
        e = e ? e : cudaMalloc(&c.d_vec, sizeof(vb_motion));
        e = e ? e : cudaMalloc(&c.d_scores, (size_t)S * S * 8);
        if (e != cudaSuccess) {
            c.release();
            return cuda_fail(e, "vb_mean_zncc_scores setup");
        }
        c.dev = dev;
        c.h = height;
        c.w = width;
        c.patch = patch;
        c.radius = radius;
        c.origins.assign(origins, origins + 2 * (size_t)n_origins);
    }
    cudaError_t e = cudaSuccess;
    if (c.ref.size() != hw || memcmp(c.ref.data(), reference, hw * sizeof(float)) != 0) {
        e = cudaMemcpyAsync(c.d_ref, reference, hw * 4, cudaMemcpyHostToDevice, c.s);
        if (e != cudaSuccess) return cuda_fail(e, "vb_mean_zncc_scores reference");
        rc = vb_motion_plan_set_reference(c.plan, c.d_ref, c.s);
        if (rc) {
            c.ref.clear();
            return rc;
        }
        c.ref.assign(reference, reference + hw);
    }
    e = cudaMemcpyAsync(c.d_frame, frame, hw * 4, cudaMemcpyHostToDevice, c.s);
    if (e != cudaSuccess) return cuda_fail(e, "vb_mean_zncc_scores frame");
    rc = vb_motion_estimate(c.plan, c.d_frame, VB_F32, 1, 0, c.d_vec, c.d_scores, c.s);
    if (rc == VB_OK) {
        e = cudaMemcpyAsync(out_scores, c.d_scores, (size_t)S * S * 8, cudaMemcpyDeviceToHost, c.s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(c.s);
        if (e != cudaSuccess) rc = cuda_fail(e, "vb_mean_zncc_scores");
    }
    return rc;
}

}  // extern "C"
