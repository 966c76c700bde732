// Internal shared declarations for libvoltb200 (sm_100a only).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include <nvtx3/nvToolsExt.h>

#include <atomic>
#include <string>

#include "../../include/voltb200.h"

namespace vb {

// ---- error plumbing -------------------------------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* where);
std::atomic<int64_t>& launches();
void keep_pool();

// A/B experiment switches.  Only an experiment build (build.py --experiments,
// -DVB_EXPERIMENTS) reads them from the environment; the product library
// always uses the measured defaults passed here.
inline int knob(const char* name, int dflt) {
#ifdef VB_EXPERIMENTS
    const char* e = getenv(name);
    return e ? atoi(e) : dflt;
#else
    (void)name;
    return dflt;
#endif
}

#define VB_CUDA(call)                                               \
    do {                                                            \
        cudaError_t e_ = (call);                                    \
        if (e_ != cudaSuccess) return ::vb::cuda_fail(e_, #call);   \
    } while (0)

#define VB_LAUNCHED()                                                      \
    do {                                                                   \
        ::vb::launches().fetch_add(1, std::memory_order_relaxed);          \
        cudaError_t e_ = cudaGetLastError();                               \
        if (e_ != cudaSuccess) return ::vb::cuda_fail(e_, "kernel launch"); \
    } while (0)

// ---- NVTX ranges (host timeline for nsys / ncu --nvtx; no-ops without a tool)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    explicit NvtxRange(const std::string& name) { nvtxRangePushA(name.c_str()); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// ---- per-kernel CUDA-event profiler (vb_prof_enable / vb_prof_collect) ----
enum KernelId { kProfZncc = 0, kProfFinalize = 1, kProfWarpSmooth = 2, kProfMedian = 3, kProfOther = 4,
                kProfCount = 5 };
class ProfScope {
   public:
    ProfScope(int id, cudaStream_t s);
    ~ProfScope();

   private:
    int id_;
    cudaStream_t s_;
    cudaEvent_t a_ = nullptr, b_ = nullptr;
};

// ---- geometry ---------------------------------------------------------------
// A patch group is a run of patches with the same origin y whose union window
// (all candidate offsets) is staged once in shared memory by one CTA.
struct PatchGroup {
    int32_t first;  // first patch index (patches of a group are contiguous)
    int32_t count;  // patches in the group
    int32_t x0;     // union window left column  (min px - R)
    int32_t y0;     // union window top row      (py - R)
    int32_t wu;     // union window width        (max px - min px + P + 2R)
    int32_t pad[3];
};

static constexpr int kMaxRadius = 31;  // _native.pyx:63-66 (acc[63])
static constexpr int kMaxGroup = 32;
static constexpr int kMaxPatch = 180;  // integer window-sum range (zncc_stats_kernel)

// Prepared template for one recording (device memory).
struct Templates {
    float* tmpl = nullptr;       // [N][P][TP] centred template patches r - mean_p (f32)
    double* rvar = nullptr;      // [N] n*variance of each template patch (f64)
    double* rmean = nullptr;     // [N] template patch means (aliases rvar + N)
    int32_t* origins = nullptr;  // [N][2] (x, y)
    int32_t* patch_col = nullptr;// [N] column of the patch's dx=-R window inside its group union
    PatchGroup* groups = nullptr;// [n_groups]
    int n = 0, n_groups = 0, tp = 0, max_g = 0, max_wu = 0;
    int pitch = 0;               // f32 region row pitch of the search kernel (bank-conflict tuned)
    // tensor-core path (zncc_mma.cu; uint16 frames): signed digit planes of
    // the fixed-point template [N][3][8 shifts][P][tpw] (int8), per-patch 2^-s
    void* t16 = nullptr;
    double* tscale = nullptr;
};

// Geometry of the tensor-core ZNCC path for (patch, radius) (zncc_mma.cu).
struct MmaGeom {
    int wx = 0, wxp = 0, toff = 0, tpw = 0, npass = 0, nchunks = 0, na = 0, nb = 0;
    int np[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    size_t off_a = 0, off_b = 0, b_bytes = 0, off_tq = 0, smem = 0;
};
bool mma_supported(int patch, int radius, int dtype);
MmaGeom mma_geom(int patch, int radius);
bool make_frames_tmap_sw128(CUtensorMap* map, const void* base, int64_t t, int h, int w);
int launch_mma_prep(const Templates& t, int patch, int radius, cudaStream_t s);
int launch_zncc_mma(const Templates& t, int patch, int radius, int64_t n_frames, int tma_z0, const CUtensorMap& tmap,
                    float* cov, int ss_pad, cudaStream_t s);

// Kernel entry points implemented in the .cu files (host-side launchers).
int launch_template_sum(const void* frames, int dtype, int64_t n, int64_t hw, double* sum,
                        int accumulate, cudaStream_t s);
int launch_template_finish(const double* sum, int64_t n_total, int64_t hw, float* ref, cudaStream_t s);
size_t zncc_smem_bytes(int patch, int radius, int max_g, int max_wu, int dtype);  // search + stats kernels
size_t zncc_search_smem_bytes(int patch, int radius, int max_g, int max_wu, int dtype);
int launch_prep_templates(const float* ref, int h, int w, int patch, const Templates& t, cudaStream_t s);
int launch_motion(const Templates& t, int h, int w, int patch, int radius, const void* frames, int dtype,
                  int64_t n_frames, int subpixel, vb_motion* vectors, double* scores, cudaStream_t s);
int launch_correct(const void* frames, int dtype, int64_t n, int h, int w, const vb_motion* vec,
                   const float* gain, float* out, cudaStream_t s);
int launch_summarize(const void* frames, int dtype, const vb_motion* vec, int64_t n, int h, int w,
                     int seg_len, const double* weights, int wradius, float* corrected, float* spatial,
                     float* temporal, cudaStream_t s);
// Recording context of a summarize call (vb_summary_opts in voltb200.h):
// frames[0] is recording frame t_global0; blocks of frames [interior_off,
// interior_off + n_interior) are summarised; the temporal high-pass (A17,
// opt-in) reflects at 0 and t_total and reads up to window/2 halo frames on
// either side of the interior.
struct SummaryOpts {
    int64_t t_global0 = 0;
    int64_t t_total = 0;
    int64_t interior_off = 0;
    int64_t n_interior = 0;
    int highpass_window = 0;
    const float* gain = nullptr;
};
int launch_summarize_ex(const void* frames, int dtype, const vb_motion* vec, int64_t n_avail, int h, int w,
                        int seg_len, const double* weights, int wradius, const SummaryOpts& o, float* corrected,
                        float* spatial, float* temporal, cudaStream_t s);
int launch_traces_raw(const void* frames, int dtype, int64_t n, int h, int w, const vb_motion* vec,
                      const float* gain, const int32_t* roi_ptr, const int32_t* roi_idx, int n_rois, double* out,
                      cudaStream_t s);
int launch_block_piece(const void* frames, int dtype, const vb_motion* vec, int64_t n, int h, int w,
                       const double* weights, int wradius, const float* gain, int64_t mean_off, int64_t mean_n,
                       float* corrected, float* smoothed, double* partial, cudaStream_t s);
int launch_block_finish(const float* smoothed, int64_t s_lo, int64_t t0, int cnt, int64_t t_total, int hp_window,
                        int64_t hw, const double* sum, float* spatial, float* temporal, cudaStream_t s);
int launch_shading_gain(const float* ref, int h, int w, const double* weights_host, int r, float* gain,
                        cudaStream_t s);
int launch_smooth(const void* frames, int dtype, int64_t n, int h, int w, const double* weights, int wradius,
                  float* out, cudaStream_t s);

// Device helpers ---------------------------------------------------------------
__device__ __forceinline__ float load_sample(const void* base, int dtype, int64_t idx) {
    if (dtype == VB_U16) return (float)__ldg(reinterpret_cast<const uint16_t*>(base) + idx);
    return __ldg(reinterpret_cast<const float*>(base) + idx);
}

__host__ __device__ __forceinline__ int clampi(int v, int lo, int hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

// scipy "reflect" boundary (half-sample symmetric), any overhang.
__host__ __device__ __forceinline__ int reflect_index(int i, int n) {
    int period = 2 * n;
    int m = i % period;
    if (m < 0) m += period;
    return m >= n ? period - 1 - m : m;
}

}  // namespace vb
