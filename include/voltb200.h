/* voltb200 -- B200-native preprocessing stage of the voltseg pipeline
 * (per-frame rigid motion correction -> per-time-block summary images).
 *
 * C ABI: plain pointers and sizes, no torch or numpy types.  Every entry point
 * returns VB_OK (0) or a positive VB_E* code; vb_last_error() returns the
 * calling thread's last message.  Messages for argument errors are the
 * reference's ValueError texts so a binding can re-raise them verbatim.
 *
 * Reference interfaces replaced (paths under /root/reference/pkg/src/voltseg):
 *   vb_mean_zncc_scores      <- _native.pyx:22-118 mean_zncc_scores / kernels.py:98-108
 *   vb_patch_grid            <- motion.py:52-75 PatchGrid.cover
 *   vb_make_reference        <- motion.py:211-214 make_reference
 *   vb_motion_plan_* /
 *   vb_motion_estimate       <- motion.py:113-160 estimate_motion over many frames
 *                               (ZNCC grid + tie-broken argmax + quadratic fit)
 *   vb_correct_frames        <- motion.py:235-240 / :244-248 correct_frame / translate
 *   vb_summarize             <- summarize.py:95-102 summarize / summarize_segment
 *                               (optionally fused with the motion warp)
 *   vb_stage_*               <- motion.py:217-241 correct_motion followed by
 *                               summarize.py:99-102 (pipeline.py:198-224 call pattern),
 *                               host buffers in and out (the drop-in boundary)
 */
#ifndef VOLTB200_H
#define VOLTB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VB_OK 0
#define VB_EINVAL 1 /* argument error (reference raises ValueError) */
#define VB_ECUDA 2  /* CUDA runtime / launch failure */
#define VB_ENOMEM 3 /* device or pinned allocation failed */

/* Frame sample types accepted on input.  u16 is the camera format; f32 is the
 * reference's in-memory Video type (video_io.py:28-46). */
#define VB_U16 0
#define VB_F32 1

/* motion.py:27-41 MotionVector.  x = dx + sub_dx, y = dy + sub_dy. */
typedef struct vb_motion {
    int32_t dx;
    int32_t dy;
    double sub_dx;
    double sub_dy;
    double confidence;
} vb_motion;

const char* vb_version(void);
const char* vb_last_error(void);

/* ---------------- operator level, host buffers ---------------- */

/* Mean patch ZNCC of `frame` windows at origin+(dx,dy) against `reference`
 * patches for all |dx|,|dy| <= radius.  frame/reference: float32 [height][width]
 * C-contiguous host arrays; origins: int32 [n_origins][2] of (x, y);
 * out_scores: float64 [(2r+1)][(2r+1)] indexed [dy+r][dx+r].
 * Errors: "frame and reference dimensions differ" is the caller's check (one
 * shape is passed); "patch origin too close to border for search radius";
 * "search radius too large (max 31)". */
int vb_mean_zncc_scores(const float* frame, const float* reference, int height, int width,
                        const int32_t* origins, int n_origins, int patch, int radius,
                        double* out_scores);

/* PatchGrid.cover(height, width, patch, margin=margin): origins may be NULL to
 * query *n_origins.  Error: "frame HxW too small for patch P with margin M". */
int vb_patch_grid(int height, int width, int patch, int margin, int32_t* origins, int* n_origins);

/* ---------------- device primitives (stream-ordered) ---------------- */
/* All *_dev pointers are device memory on the current device; `stream` is a
 * cudaStream_t (NULL = legacy default stream). */

/* Template: float64 per-pixel sum of n frames (sequential frame order).  With
 * accumulate != 0 the sum is added to sum_dev (for sharded recordings whose
 * partial sums are then all-reduced). */
int vb_template_sum(const void* frames_dev, int dtype, int64_t n_frames, int height, int width,
                    double* sum_dev, int accumulate, void* stream);
/* ref_dev[i] = float32(sum_dev[i] / n_total)  (motion.py:214). */
int vb_template_finish(const double* sum_dev, int64_t n_total, int64_t n_pixels, float* ref_dev,
                       void* stream);
/* make_reference in one call: mean of the first min(n_frames, ref_frames) frames. */
int vb_make_reference(const void* frames_dev, int dtype, int64_t n_frames, int height, int width,
                      int ref_frames, float* ref_dev, void* stream);

/* Motion plan: geometry + prepared template patches for one recording. */
typedef struct vb_motion_plan vb_motion_plan;
int vb_motion_plan_create(vb_motion_plan** plan, int height, int width, int patch, int radius,
                          const int32_t* origins_host, int n_origins);
int vb_motion_plan_set_reference(vb_motion_plan* plan, const float* ref_dev, void* stream);
/* Per-frame motion vectors for n frames (optionally the full score grids,
 * float64 [n][(2r+1)][(2r+1)]). */
int vb_motion_estimate(vb_motion_plan* plan, const void* frames_dev, int dtype, int64_t n_frames,
                       int subpixel, vb_motion* vectors_dev, double* scores_dev, void* stream);
/* Work decomposition of the plan: patches, CTA patch groups, the largest
 * group and its union-window width (diagnostics). */
int vb_motion_plan_info(const vb_motion_plan* plan, int* n_patches, int* n_groups, int* max_group,
                        int* max_width);
int vb_motion_plan_destroy(vb_motion_plan* plan);

/* corrected[t] = frame unchanged if the vector is (0,0), else
 * translate(frame, -x, -y)  (bit-exact float32 bilinear, edge replicated). */
int vb_correct_frames(const void* frames_dev, int dtype, int64_t n_frames, int height, int width,
                      const vb_motion* vectors_dev, float* corrected_dev, void* stream);

/* Per-block summary images of n frames split into ceil(n/L) blocks
 * (summarize.py:44-102).  If vectors_dev != NULL the motion warp is applied on
 * the fly (frames are raw) and, if corrected_dev != NULL, the corrected frames
 * are written too.  weights: host float64 [2*wradius+1] (scipy
 * _gaussian_kernel1d).  spatial_dev / temporal_dev: float32 [K][height][width].
 * Error: "segment length must be >= 2"; a final block of one frame raises
 * "temporal summary needs at least 2 frames" (summarize.py:79-80). */
int vb_summarize(const void* frames_dev, int dtype, const vb_motion* vectors_dev, int64_t n_frames,
                 int height, int width, int segment_length, const double* weights, int wradius,
                 float* corrected_dev, float* spatial_dev, float* temporal_dev, void* stream);

/* Separable Gaussian smoothing of each frame (scipy gaussian_filter with mode
 * "reflect": H pass then W pass, float64 accumulate, f32 per pass;
 * summarize.py:60-73).  out_dev: float32 [n][height][width]. */
int vb_smooth_frames(const void* frames_dev, int dtype, int64_t n_frames, int height, int width,
                     const double* weights, int wradius, float* out_dev, void* stream);

/* Trace extraction (traces.py:23-40): out_dev[r][t] =
 * float64 mean of frames_dev[t] over ROI r's pixels.  ROIs in CSR form:
 * roi_ptr_dev[n_rois+1] offsets into roi_idx_dev (flattened y*width+x pixel
 * indices, row-major like np.nonzero); device pointers. */
int vb_extract_traces(const float* frames_dev, int64_t n_frames, int height, int width,
                      const int32_t* roi_ptr_dev, const int32_t* roi_idx_dev, int n_rois, double* out_dev,
                      void* stream);

/* The same traces straight from the RAW frames and their motion vectors
 * (trace extraction fused with the warp, so the
 * corrected video is never materialised): the corrected value of each ROI
 * pixel is interpolated exactly as vb_correct_frames / the stage would
 * (motion.py:163-200, + the opt-in shading gain, nullable), then averaged like
 * vb_extract_traces -- bit-identical to it on the corrected video.
 * frames_dev: uint16 / float32 [n][h][w]; vectors_dev: vb_motion[n] (null =
 * no motion). */
int vb_extract_traces_raw(const void* frames_dev, int dtype, const vb_motion* vectors_dev, const float* gain_dev,
                          int64_t n_frames, int height, int width, const int32_t* roi_ptr_dev,
                          const int32_t* roi_idx_dev, int n_rois, double* out_dev, void* stream);

/* ---------------- A17 extensions (opt-in, default off) ----------------
 * The north-star's shading/background correction and per-pixel temporal
 * high-pass have NO code in the reference; they
 * are pinned only to this repo's CPU restatement (oracle/oracle.c
 * or_shading_gain / or_highpass_summary), never to reference outputs. */
typedef struct vb_summary_opts {
    int64_t t_global0;     /* recording index of frames_dev[0] */
    int64_t t_total;       /* frames in the whole recording (reflect boundary of the high-pass) */
    int64_t interior_off;  /* first summarised frame (index into frames_dev); t_global0 + interior_off
                              must be a multiple of segment_length */
    int64_t n_interior;    /* summarised frames: a multiple of segment_length or running to t_total */
    int highpass_window;   /* odd N >= 3: the temporal summary is taken over x - mean_N(x) (centred
                              N-frame moving average of the smoothed frames, "reflect" at 0 and
                              t_total); frames_dev must hold the N/2-frame halo; 0 or 1 = off */
    const float* gain_dev; /* [h][w] shading gain, corrected = warped / gain (IEEE f32); NULL = off */
} vb_summary_opts;

/* vb_summarize over part of a longer recording (time shards, chunks with a
 * halo) with the opt-in extensions.  vectors_dev indexes frames_dev;
 * corrected_dev receives only the interior frames.  opts == NULL is
 * vb_summarize.  Errors: those of vb_summarize, "summary interior must start
 * on a block boundary", "high-pass window must be odd",
 * "temporal high-pass halo not in the frame buffer". */
int vb_summarize_ex(const void* frames_dev, int dtype, const vb_motion* vectors_dev, int64_t n_frames,
                    int height, int width, int segment_length, const double* weights, int wradius,
                    const vb_summary_opts* opts, float* corrected_dev, float* spatial_dev,
                    float* temporal_dev, void* stream);
/* Shading gain from a template: G = separable float64 Gaussian of ref_dev
 * (host weights[2*wradius+1], taps -r..r in order, "reflect"), gain_dev =
 * float32(G / mean(G)) with the mean summed in a fixed order. */
int vb_shading_gain(const float* ref_dev, int height, int width, const double* weights, int wradius,
                    float* gain_dev, void* stream);
/* vb_correct_frames followed by division by gain_dev (NULL = no shading). */
int vb_correct_frames_ex(const void* frames_dev, int dtype, int64_t n_frames, int height, int width,
                         const vb_motion* vectors_dev, const float* gain_dev, float* corrected_dev,
                         void* stream);

/* ---------------- blocks split across time shards ----------------
 * With frame-balanced time shards a summary block (summarize.py:44-52) may
 * straddle ranks.  Every rank holding part of block b calls vb_block_piece on
 * its frames of b, in recording order: frames [mean_off, mean_off + mean_n)
 * of frames_dev are the block's own frames -- warped (vectors_dev), written to
 * corrected_dev ([mean_n][h][w], NULL = not kept) and added, frame by frame,
 * onto the float64 running sum partial_sum_dev[h][w] (zeros for the block's
 * first piece; the same adds as spatial_summary, summarize.py:55-57, so the
 * chained sum is bit-identical); all n_frames frames (own frames plus, with
 * the high-pass, halo frames) are smoothed into smoothed_dev [n_frames][h][w].
 * The running sum and the smoothed frames travel to the next contributor
 * (NCCL send/recv); the rank holding the block's last frame calls
 * vb_block_finish on the assembled buffer (recording frames [s_lo, s_lo +
 * n_smoothed)): spatial = f32(sum / count), temporal = max - median
 * (summarize.py:76-92; over x - mean_N(x) when highpass_window > 1). */
int vb_block_piece(const void* frames_dev, int dtype, const vb_motion* vectors_dev, int64_t n_frames, int height,
                   int width, const double* weights, int wradius, const float* gain_dev, int64_t mean_off,
                   int64_t mean_n, float* corrected_dev, float* smoothed_dev, double* partial_sum_dev,
                   void* stream);
int vb_block_finish(const float* smoothed_dev, int64_t s_lo, int64_t n_smoothed, int64_t t0, int64_t count,
                    int64_t t_total, int highpass_window, int height, int width, const double* sum_dev,
                    float* spatial_dev, float* temporal_dev, void* stream);

/* Peer memory for the exchange of straddling blocks between ranks (SURVEY
 * 8(e)): the receiving rank allocates its block buffers with vb_ipc_alloc and
 * shares the 64-byte handle; the sending rank opens it (vb_ipc_open, peer
 * access over NVLink when the ranks are on different GPUs) and passes the
 * mapped pointers to vb_block_piece, so the warp+smooth kernel and the running
 * sum write the block straight into the owner's memory, tile by tile, with no
 * separate copy.  vb_copy_async (cudaMemcpyDefault) relays a received prefix
 * to the next owner; vb_memset_async zeroes a (peer) running sum. */
#define VB_IPC_HANDLE_BYTES 64
int vb_ipc_alloc(int64_t bytes, void** dev_ptr, unsigned char* handle);
int vb_ipc_open(const unsigned char* handle, void** dev_ptr);
int vb_ipc_close(void* dev_ptr);
int vb_ipc_free(void* dev_ptr);
int vb_copy_async(void* dst, const void* src, int64_t bytes, void* stream);
int vb_memset_async(void* dst, int value, int64_t bytes, void* stream);

/* ---------------- summary normalisation + U-Net tiles ----------------
 * The consumer of the per-block summaries in the reference pipeline
 * (pipeline.py:222-223).  Parameters are the float32 tensors of
 * unet.architecture() (unet.py:34-54) flattened in that order (kernel
 * [cout][cin][k][k] then bias [cout] per conv): vb_unet_param_count() floats. */
typedef struct vb_unet vb_unet;
int64_t vb_unet_param_count(void);
int vb_unet_create(vb_unet** net, const float* params_host, int64_t n_params);
/* unet.forward_batch (unet.py:154-178): patches_dev float32 [n][2][64][64] ->
 * probs_dev float32 [n][64][64] (sigmoid outputs). */
int vb_unet_forward(vb_unet* net, const float* patches_dev, int64_t n, float* probs_dev, void* stream);
/* unet.normalize_pair (unet.py:186-196) for n_blocks pairs: spatial_dev /
 * temporal_dev float32 [n_blocks][h][w] -> out_dev float32 [n_blocks][2][h][w]
 * (numpy "linear" 1st/99th percentiles; a constant channel maps to 0). */
int vb_normalize_pair(const float* spatial_dev, const float* temporal_dev, int64_t n_blocks, int height, int width,
                      float* out_dev, void* stream);
/* unet.tile_and_merge (unet.py:212-245) for n_blocks normalised pairs
 * [n_blocks][2][h][w] -> prob_dev float32 [n_blocks][h][w]. */
int vb_unet_tile_merge(vb_unet* net, const float* normalized_dev, int64_t n_blocks, int height, int width, int stride,
                       float* prob_dev, void* stream);
/* normalize_pair + tile_and_merge per block (pipeline.py:222-223);
 * normalized_dev (nullable) receives the normalised pairs. */
int vb_unet_segment(vb_unet* net, const float* spatial_dev, const float* temporal_dev, int64_t n_blocks, int height,
                    int width, int stride, float* normalized_dev, float* prob_dev, void* stream);
int vb_unet_destroy(vb_unet* net);

/* ---------------- whole stage, host buffers (drop-in boundary) ---------------- */
typedef struct vb_stage_config {
    int height, width;
    int patch;          /* MotionConfig.patch_size (motion.py:203-208), default 21 */
    int radius;         /* MotionConfig.search_radius */
    int subpixel;       /* MotionConfig.subpixel */
    int ref_frames;     /* REFERENCE_FRAMES (motion.py:24) */
    int segment_length; /* summarize(..., segment_length) */
    double sigma;       /* summarize(..., sigma) */
    int device;         /* CUDA device ordinal */
    int64_t chunk_frames; /* host->device streaming granularity (0 = auto) */
} vb_stage_config;

typedef struct vb_stage vb_stage;
int vb_stage_create(vb_stage** stage, const vb_stage_config* cfg);
/* Replace the smoothing weights (default: libm exp of scipy's formula).  The
 * Python binding passes numpy-computed _gaussian_kernel1d weights so the
 * summaries are bit-identical to scipy's. */
int vb_stage_set_weights(vb_stage* stage, const double* weights, int wradius);
/* Runs correct_motion + summarize over a host recording (pinned or pageable).
 * frames_host: dtype [n][h][w]; vectors_host: [n]; spatial/temporal_host:
 * float32 [ceil(n/L)][h][w]; corrected_host: float32 [n][h][w] or NULL;
 * corrected_dev: device float32 [n][h][w] that receives the whole corrected
 * video in HBM, or NULL.  With both NULL the corrected frames are only formed
 * on the fly inside the fused warp/summary kernel.  spatial_host and
 * temporal_host both NULL: motion only (correct_motion, motion.py:217-241) --
 * vectors and the optional corrected frames, no summaries. */
int vb_stage_run_host(vb_stage* stage, const void* frames_host, int dtype, int64_t n_frames,
                      vb_motion* vectors_host, float* spatial_host, float* temporal_host,
                      float* corrected_host, float* corrected_dev);
/* A17 (opt-in): temporal high-pass window (odd >= 3; 0 = off) and shading
 * gain weights (NULL = off; the gain is rebuilt from each run's template).
 * The executor uploads each chunk with its window/2-frame halo. */
int vb_stage_set_highpass(vb_stage* stage, int window);
int vb_stage_set_shading(vb_stage* stage, const double* weights, int wradius);
/* Number of device kernels the last vb_stage_run_host launched. */
int64_t vb_stage_last_launches(const vb_stage* stage);
int vb_stage_destroy(vb_stage* stage);

/* Pipeline orchestration (SURVEY 8(f) rows 2 + 4; pipeline.py:190-258 minus
 * the footprint stage): attach a U-Net (not owned; NULL detaches) and run
 * correct_motion + summarize + normalize_pair + tile_and_merge per block.  Each
 * chunk's blocks are segmented on a separate stream while the next chunk's
 * motion search runs; prob_host: float32 [ceil(n/L)][h][w]. */
int vb_stage_set_unet(vb_stage* stage, vb_unet* net, int stride);
int vb_stage_run_host_segment(vb_stage* stage, const void* frames_host, int dtype, int64_t n_frames,
                              vb_motion* vectors_host, float* spatial_host, float* temporal_host, float* prob_host,
                              float* corrected_host, float* corrected_dev);

/* ---------------- several GPUs from one process (no torch.distributed) ----------------
 * a group of devices, one vb_stage per device and
 * one NCCL communicator per device (ncclCommInitAll; NCCL is dlopen'ed).  The
 * recording is split into block-aligned time shards (vb_group_plan: whole
 * L-frame blocks, as evenly as possible), the template is the float64 sum of
 * the first min(n, ref_frames) frames all-reduced over NCCL (each device sums
 * its own frames of that range; every device divides identically), and each
 * device then streams its shard through its executor in its own host thread.
 * Outputs land in the caller's buffers exactly as vb_stage_run_host's would
 * for the whole recording on one device (bit-identical). */
typedef struct vb_group vb_group;
/* frame_bounds[n_devices + 1]: shard d = frames [frame_bounds[d], frame_bounds[d+1]). */
int vb_group_plan(int64_t n_frames, int segment_length, int n_devices, int64_t* frame_bounds);
int vb_group_create(vb_group** group, const int* devices, int n_devices, const vb_stage_config* cfg);
int vb_group_set_weights(vb_group* group, const double* weights, int wradius);
int vb_group_run_host(vb_group* group, const void* frames_host, int dtype, int64_t n_frames,
                      vb_motion* vectors_host, float* spatial_host, float* temporal_host, float* corrected_host);
int64_t vb_group_last_launches(const vb_group* group);
int vb_group_destroy(vb_group* group);

/* Page-locked host memory (cudaHostAlloc, portable).  A corrected_host
 * buffer passed to vb_stage_run_host that is page-locked (from here or
 * cudaHostRegister) receives each chunk by a direct device->host copy; a
 * pageable one goes through the executor's pinned staging slots. */
int vb_host_alloc(int64_t bytes, void** out);
int vb_host_free(void* ptr);
/* memcpy split over n_threads host threads (<= 0: min(8, cores / 2)); the
 * executor's pageable staging copy (exported for its host-logic tests). */
int vb_host_copy(void* dst, const void* src, int64_t bytes, int n_threads);

/* Use an externally built template (e.g. all-reduced across ranks) for the
 * following runs instead of averaging the first ref_frames frames of the
 * input (phase A).  ref_dev: device float32 [h][w], copied; NULL restores the
 * default. */
int vb_stage_set_reference(vb_stage* stage, const float* ref_dev);

/* Kernel launches issued by this library since load (all entry points). */
int64_t vb_launch_count(void);

/* ---------------- measurement hooks (bench.py) ---------------- */
/* Per-kernel CUDA-event timing on the launching stream: ids 0 zncc search,
 * 1 finalize (argmax/fit), 2 fused warp+smooth, 3 median, 4 other.
 * vb_prof_enable(1) clears and starts recording; vb_prof_collect synchronises
 * the recorded events and returns total ms and launch counts per id. */
int vb_prof_enable(int on);
int vb_prof_collect(double* ms, int64_t* counts, int n_ids);
/* Measured FP32 throughput of this GPU (TFLOP/s) with packed FFMA2
 * (fma.rn.f32x2) and scalar FFMA dependency chains: the denominator of the
 * ZNCC kernel's roofline. */
int vb_fp32_peak_probe(double* tflops_ffma2, double* tflops_ffma);

#ifdef __cplusplus
}
#endif
#endif /* VOLTB200_H */
