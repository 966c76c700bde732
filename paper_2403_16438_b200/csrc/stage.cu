// Whole-stage executor over a HOST recording: the drop-in boundary for
// correct_motion (motion.py:217-241) followed by summarize (summarize.py:99-102),
// as pipeline.py:198-224 calls them.
//
// Frame-chunk scheduler: chunks of whole blocks (a multiple of L frames) are
// copied host->HBM on an H2D stream, in pieces, into a two-slot device ring;
// each piece is motion-searched, warped and smoothed as it lands (compute
// stream), each block's mean and max - median run once the block is complete,
// and the chunk before drains device->host on a D2H stream.  Pageable input is first packed into pinned staging slots by the
// host thread (pinned input DMAs directly).  Events order slot reuse.
#include <cuda_runtime.h>
#include <math.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "vb.cuh"

using namespace vb;

// Host copies between caller (pageable) memory and the pinned staging slots:
// one thread moves ~10-14 GB/s, below the ~55 GB/s PCIe stream it feeds, so
// large copies are split over a few threads (measured on C2 from a plain
// numpy recording: 53 k frames/s with one thread).
static int host_copy_threads() {
    static const int nthr = [] {
        const unsigned hc = std::thread::hardware_concurrency();
        return (int)std::max(1u, std::min(8u, hc ? hc / 2 : 1u));
    }();
    return nthr;
}

// Split [0, bytes) into nt contiguous ranges with 64-byte aligned interior
// boundaries; range i = [i*step, min(bytes, (i+1)*step)) and the last one
// always ends at `bytes` (step = ceil(bytes / nt) rounded up to 64).
static void host_copy_n(void* dst, const void* src, size_t bytes, int nthr) {
    constexpr size_t kMinPerThread = 4u << 20;
    const int nt = (int)std::min<size_t>((size_t)std::max(1, nthr), std::max<size_t>(1, bytes / kMinPerThread));
    if (nt <= 1) {
        memcpy(dst, src, bytes);
        return;
    }
    const size_t step = ((bytes + nt - 1) / nt + 63) & ~(size_t)63;
    std::vector<std::thread> pool;
    pool.reserve(nt - 1);
    for (int i = 1; i < nt; ++i) {
        const size_t o = std::min(bytes, i * step), e = (i == nt - 1) ? bytes : std::min(bytes, o + step);
        if (e > o) pool.emplace_back([=] { memcpy((char*)dst + o, (const char*)src + o, e - o); });
    }
    memcpy(dst, src, std::min(bytes, step));
    for (auto& th : pool) th.join();
}

static void host_copy(void* dst, const void* src, size_t bytes) { host_copy_n(dst, src, bytes, host_copy_threads()); }

struct vb_stage {
    vb_stage_config cfg{};
    cudaStream_t s_comp = nullptr, s_h2d = nullptr, s_d2h = nullptr;
    vb_motion_plan* plan = nullptr;
    std::vector<int32_t> origins;
    std::vector<double> weights;
    int wradius = 0;
    int64_t chunk = 0;  // frames per chunk (multiple of L)
    size_t esz = 0;     // bytes per sample of the allocated ring
    void* d_frames[2] = {nullptr, nullptr};
    vb_motion* d_vec[2] = {nullptr, nullptr};
    float* d_sp[2] = {nullptr, nullptr};
    float* d_tp[2] = {nullptr, nullptr};
    float* d_corr[2] = {nullptr, nullptr};
    void* h_stage[2] = {nullptr, nullptr};
    // pinned output staging: D2H into page-locked memory never blocks the
    // host thread; chunk k-1 is unpacked into the caller's buffers while
    // chunk k computes.
    vb_motion* h_vec[2] = {nullptr, nullptr};
    float* h_sp[2] = {nullptr, nullptr};
    float* h_tp[2] = {nullptr, nullptr};
    float* h_corr[2] = {nullptr, nullptr};
    double* d_tsum = nullptr;
    float* d_ref = nullptr;
    bool external_ref = false;
    // A17 (opt-in): temporal high-pass window and shading gain weights
    int hp_window = 0;
    std::vector<double> shade_w;
    int shade_r = 0;
    float* d_gain = nullptr;
    int64_t cap = 0;  // frames per ring slot (chunk + high-pass halo)
    cudaEvent_t ev_h2d[2]{}, ev_comp[2]{}, ev_d2h[2]{};
    // a chunk is uploaded in kSubParts pieces, each with its own event, so the
    // motion search of a chunk's first frames starts while the rest is still
    // crossing PCIe (shorter pipeline fill and drain around the H2D-bound body)
    static constexpr int kSubParts = 4;  // measured: 8 pieces no better (200.9k vs 201.3k frames/s e2e)
    cudaEvent_t ev_sub[2][kSubParts]{};
    int64_t last_launches = 0;
    // SURVEY 8(f) rows 2 + 4: per-block U-Net segmentation of each chunk's
    // summaries on its own stream (overlapping the next chunk's motion search),
    // probability maps drained with the other outputs
    vb_unet* unet = nullptr;
    int unet_stride = 32;
    cudaStream_t s_seg = nullptr;
    cudaEvent_t ev_seg[2]{};
    float* d_prob[2] = {nullptr, nullptr};
    float* h_prob[2] = {nullptr, nullptr};
    // piecewise summaries (no high-pass): each upload piece is warped and
    // smoothed as soon as its motion is known, into one chunk-sized smoothed
    // buffer, with the blocks' float64 running sums; the per-block mean and
    // max - median run once the block is complete (shorter drain after the
    // last byte lands)
    float* d_smooth = nullptr;
    double* d_bsum = nullptr;
};

static void stage_free_buffers(vb_stage* st) {
    for (int i = 0; i < 2; ++i) {
        cudaFree(st->d_frames[i]);
        cudaFree(st->d_vec[i]);
        cudaFree(st->d_sp[i]);
        cudaFree(st->d_tp[i]);
        cudaFree(st->d_corr[i]);
        cudaFreeHost(st->h_stage[i]);
        cudaFreeHost(st->h_vec[i]);
        cudaFreeHost(st->h_sp[i]);
        cudaFreeHost(st->h_tp[i]);
        cudaFreeHost(st->h_corr[i]);
        cudaFree(st->d_prob[i]);
        cudaFreeHost(st->h_prob[i]);
        st->d_prob[i] = st->h_prob[i] = nullptr;
        st->d_frames[i] = st->h_stage[i] = nullptr;
        st->h_vec[i] = nullptr;
        st->h_sp[i] = st->h_tp[i] = st->h_corr[i] = nullptr;
        st->d_vec[i] = nullptr;
        st->d_sp[i] = st->d_tp[i] = st->d_corr[i] = nullptr;
    }
    cudaFree(st->d_smooth);
    cudaFree(st->d_bsum);
    st->d_smooth = nullptr;
    st->d_bsum = nullptr;
    st->esz = 0;
    st->cap = 0;
}

extern "C" {

int vb_stage_create(vb_stage** out, const vb_stage_config* cfg) {
    if (!out || !cfg) return fail(VB_EINVAL, "null argument");
    *out = nullptr;
    if (cfg->radius < 1) return fail(VB_EINVAL, "search_radius must be >= 1");
    if (cfg->segment_length < 2) return fail(VB_EINVAL, "segment length must be >= 2");
    if (!(cfg->sigma > 0)) return fail(VB_EINVAL, "sigma must be positive");
    if (cfg->ref_frames < 1) return fail(VB_EINVAL, "ref_frames must be >= 1");
    VB_CUDA(cudaSetDevice(cfg->device));
    auto* st = new vb_stage();
    st->cfg = *cfg;
    int n = 0;
    int rc = vb_patch_grid(cfg->height, cfg->width, cfg->patch, cfg->radius, nullptr, &n);
    if (rc) {
        delete st;
        return rc;
    }
    st->origins.resize(2 * (size_t)n);
    vb_patch_grid(cfg->height, cfg->width, cfg->patch, cfg->radius, st->origins.data(), &n);
    rc = vb_motion_plan_create(&st->plan, cfg->height, cfg->width, cfg->patch, cfg->radius, st->origins.data(), n);
    if (rc) {
        delete st;
        return rc;
    }
    // scipy _gaussian_kernel1d(sigma, 0, ceil(3 sigma)) (summarize.py:71),
    // normalised by numpy's pairwise sum (eight accumulators, combined as
    // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), then the tail in order).  For the
    // default sigma = 3 libm's exp equals numpy's and the taps are bit-identical
    // to scipy's; for other sigmas numpy's exp may differ in the last ulp, so
    // vb_stage_set_weights with numpy-computed taps is the parity path.
    st->wradius = (int)ceil(3.0 * cfg->sigma);
    const int nw = 2 * st->wradius + 1;
    st->weights.resize(nw);
    for (int i = -st->wradius; i <= st->wradius; ++i)
        st->weights[i + st->wradius] = exp(-0.5 / (cfg->sigma * cfg->sigma) * (double)(i * i));
    double tot = 0.0;
    if (nw < 8) {
        for (int i = 0; i < nw; ++i) tot += st->weights[i];
    } else {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = st->weights[j];
        int i = 8;
        for (; i < nw - nw % 8; i += 8)
            for (int j = 0; j < 8; ++j) r[j] += st->weights[i + j];
        tot = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < nw; ++i) tot += st->weights[i];
    }
    for (auto& wv : st->weights) wv /= tot;
    const int L = cfg->segment_length;
    // ~1000-frame chunks: short pipeline fill/drain around the PCIe-bound body
    int64_t want = cfg->chunk_frames > 0 ? cfg->chunk_frames : 1024;
    st->chunk = std::max<int64_t>(1, (want + L / 2) / L) * L;
    cudaError_t e = cudaStreamCreateWithFlags(&st->s_comp, cudaStreamNonBlocking);
    e = e ? e : cudaStreamCreateWithFlags(&st->s_h2d, cudaStreamNonBlocking);
    e = e ? e : cudaStreamCreateWithFlags(&st->s_d2h, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
        e = cudaEventCreateWithFlags(&st->ev_h2d[i], cudaEventDisableTiming);
        for (int j = 0; j < vb_stage::kSubParts && e == cudaSuccess; ++j)
            e = cudaEventCreateWithFlags(&st->ev_sub[i][j], cudaEventDisableTiming);
        e = e ? e : cudaEventCreateWithFlags(&st->ev_comp[i], cudaEventDisableTiming);
        e = e ? e : cudaEventCreateWithFlags(&st->ev_d2h[i], cudaEventDisableTiming);
    }
    const size_t hw = (size_t)cfg->height * cfg->width;
    e = e ? e : cudaMalloc(&st->d_tsum, hw * sizeof(double));
    e = e ? e : cudaMalloc(&st->d_ref, hw * sizeof(float));
    if (e != cudaSuccess) {
        vb_stage_destroy(st);
        return cuda_fail(e, "vb_stage_create");
    }
    *out = st;
    return VB_OK;
}

int vb_stage_set_weights(vb_stage* st, const double* weights, int wradius) {
    if (!st || !weights || wradius < 0) return fail(VB_EINVAL, "null argument");
    st->weights.assign(weights, weights + 2 * wradius + 1);
    st->wradius = wradius;
    return VB_OK;
}

int vb_stage_set_reference(vb_stage* st, const float* ref_dev) {
    if (!st) return fail(VB_EINVAL, "null argument");
    if (!ref_dev) {
        st->external_ref = false;
        return VB_OK;
    }
    VB_CUDA(cudaSetDevice(st->cfg.device));
    VB_CUDA(cudaMemcpy(st->d_ref, ref_dev, (size_t)st->cfg.height * st->cfg.width * sizeof(float),
                       cudaMemcpyDeviceToDevice));
    st->external_ref = true;
    return VB_OK;
}

int vb_stage_set_highpass(vb_stage* st, int window) {
    if (!st) return fail(VB_EINVAL, "null argument");
    if (window > 1 && window % 2 == 0) return fail(VB_EINVAL, "high-pass window must be odd");
    if (window / 2 > 512) return fail(VB_EINVAL, "high-pass window too long (max 1025 frames)");
    if (window > 1 && st->cfg.segment_length > 1024)
        return fail(VB_EINVAL, "temporal high-pass needs segment_length <= 1024");
    st->hp_window = window > 1 ? window : 0;
    return VB_OK;
}

int vb_stage_set_shading(vb_stage* st, const double* weights, int wradius) {
    if (!st) return fail(VB_EINVAL, "null argument");
    if (!weights) {
        st->shade_w.clear();
        st->shade_r = 0;
        return VB_OK;
    }
    if (wradius < 0) return fail(VB_EINVAL, "null argument");
    st->shade_w.assign(weights, weights + 2 * wradius + 1);
    st->shade_r = wradius;
    if (!st->d_gain) {
        VB_CUDA(cudaSetDevice(st->cfg.device));
        VB_CUDA(cudaMalloc(&st->d_gain, (size_t)st->cfg.height * st->cfg.width * sizeof(float)));
    }
    return VB_OK;
}

int64_t vb_stage_last_launches(const vb_stage* st) { return st ? st->last_launches : 0; }

int vb_stage_set_unet(vb_stage* st, vb_unet* net, int stride) {
    if (!st) return fail(VB_EINVAL, "null argument");
    if (net && stride < 1) return fail(VB_EINVAL, "stride must be >= 1");
    VB_CUDA(cudaSetDevice(st->cfg.device));
    if (net && !st->s_seg) {
        VB_CUDA(cudaStreamCreateWithFlags(&st->s_seg, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) VB_CUDA(cudaEventCreateWithFlags(&st->ev_seg[i], cudaEventDisableTiming));
    }
    st->unet = net;
    st->unet_stride = stride;
    return VB_OK;
}

static int stage_run(vb_stage* st, const void* frames_host, int dtype, int64_t n_frames, vb_motion* vectors_host,
                     float* spatial_host, float* temporal_host, float* prob_host, float* corrected_host,
                     float* corrected_dev);

int vb_stage_run_host(vb_stage* st, const void* frames_host, int dtype, int64_t n_frames, vb_motion* vectors_host,
                      float* spatial_host, float* temporal_host, float* corrected_host, float* corrected_dev) {
    return stage_run(st, frames_host, dtype, n_frames, vectors_host, spatial_host, temporal_host, nullptr,
                     corrected_host, corrected_dev);
}

int vb_stage_run_host_segment(vb_stage* st, const void* frames_host, int dtype, int64_t n_frames,
                              vb_motion* vectors_host, float* spatial_host, float* temporal_host, float* prob_host,
                              float* corrected_host, float* corrected_dev) {
    if (!st) return fail(VB_EINVAL, "null argument");
    if (!st->unet) return fail(VB_EINVAL, "no U-Net attached (vb_stage_set_unet)");
    if (!prob_host) return fail(VB_EINVAL, "null argument");
    return stage_run(st, frames_host, dtype, n_frames, vectors_host, spatial_host, temporal_host, prob_host,
                     corrected_host, corrected_dev);
}

static int stage_run_impl(vb_stage* st, const void* frames_host, int dtype, int64_t n_frames,
                          vb_motion* vectors_host, float* spatial_host, float* temporal_host, float* prob_host,
                          float* corrected_host, float* corrected_dev);

// Every exit (including errors part-way through the chunk loop) synchronises
// all stage streams, so no copy still reads the caller's frames or writes its
// outputs after the call returns.
static int stage_sync_all(vb_stage* st) {
    cudaError_t e = cudaSuccess;
    for (cudaStream_t s : {st->s_h2d, st->s_comp, st->s_d2h, st->s_seg}) {
        if (!s) continue;
        const cudaError_t es = cudaStreamSynchronize(s);
        if (e == cudaSuccess) e = es;
    }
    return e;
}

static int stage_run(vb_stage* st, const void* frames_host, int dtype, int64_t n_frames, vb_motion* vectors_host,
                     float* spatial_host, float* temporal_host, float* prob_host, float* corrected_host,
                     float* corrected_dev) {
    if (!st || !frames_host || !vectors_host) return fail(VB_EINVAL, "null argument");
    const int64_t launches0 = launches().load();
    NvtxRange nv("vb_stage_run_host");
    int rc = stage_run_impl(st, frames_host, dtype, n_frames, vectors_host, spatial_host, temporal_host, prob_host,
                            corrected_host, corrected_dev);
    const cudaError_t e = (cudaError_t)stage_sync_all(st);
    if (rc == VB_OK && e != cudaSuccess) rc = cuda_fail(e, "vb_stage_run_host");
    st->last_launches = launches().load() - launches0;
    return rc;
}

static int stage_run_impl(vb_stage* st, const void* frames_host, int dtype, int64_t n_frames,
                          vb_motion* vectors_host, float* spatial_host, float* temporal_host, float* prob_host,
                          float* corrected_host, float* corrected_dev) {
    // motion only (correct_motion): no summary outputs requested
    const bool motion_only = !spatial_host && !temporal_host;
    if (!motion_only && (!spatial_host || !temporal_host)) return fail(VB_EINVAL, "null argument");
    if (motion_only && prob_host) return fail(VB_EINVAL, "segmentation needs the summaries");
    if (dtype != VB_U16 && dtype != VB_F32) return fail(VB_EINVAL, "unsupported sample type");
    const vb_stage_config& c = st->cfg;
    const int L = c.segment_length;
    if (n_frames < 1) return fail(VB_EINVAL, "video dimensions must all be >= 1");
    if (!motion_only && n_frames % L == 1) return fail(VB_EINVAL, "temporal summary needs at least 2 frames");
    VB_CUDA(cudaSetDevice(c.device));
    const size_t hw = (size_t)c.height * c.width;
    const size_t esz = dtype == VB_U16 ? 2 : 4;
    const int64_t C = st->chunk;
    const int64_t cblk = C / L;
    const int64_t hh = st->hp_window / 2;  // high-pass halo per side (0 = off)
    const int64_t cap = C + 2 * hh;
    const bool shade = !st->shade_w.empty();

    auto is_pinned = [](const void* p) {
        cudaPointerAttributes attr;
        const bool r = p && cudaPointerGetAttributes(&attr, p) == cudaSuccess && attr.type == cudaMemoryTypeHost;
        cudaGetLastError();
        return r;
    };
    const bool pinned = is_pinned(frames_host);
    // page-locked corrected output (cudaHostAlloc / cudaHostRegister): chunks
    // are copied device->host straight into it, no staging slot or host copy
    const bool corr_direct = corrected_host && is_pinned(corrected_host) &&
                             is_pinned((const char*)corrected_host + (size_t)n_frames * hw * sizeof(float) - 1);

    // (re)allocate the two-slot ring
    const bool ring_corr = corrected_host && !corrected_dev;  // corrected chunks need ring buffers
    const bool seg = prob_host != nullptr;
    const bool piecewise = !motion_only && hh == 0 && knob("VB_STAGE_CHUNKWISE", 0) != 1;
    if (st->esz != esz || st->cap < cap || (ring_corr && !st->d_corr[0]) || (corrected_host && !corr_direct && !st->h_corr[0]) ||
        (!pinned && !st->h_stage[0]) || (seg && !st->d_prob[0]) || (piecewise && !st->d_smooth)) {
        stage_free_buffers(st);
        cudaError_t e = cudaSuccess;
        for (int i = 0; i < 2 && e == cudaSuccess; ++i) {
            e = cudaMalloc(&st->d_frames[i], (size_t)cap * hw * esz);
            e = e ? e : cudaMalloc(&st->d_vec[i], (size_t)cap * sizeof(vb_motion));
            e = e ? e : cudaMalloc(&st->d_sp[i], (size_t)cblk * hw * sizeof(float));
            e = e ? e : cudaMalloc(&st->d_tp[i], (size_t)cblk * hw * sizeof(float));
            if (ring_corr) e = e ? e : cudaMalloc(&st->d_corr[i], (size_t)C * hw * sizeof(float));
            e = e ? e : cudaHostAlloc(&st->h_vec[i], (size_t)C * sizeof(vb_motion), cudaHostAllocDefault);
            e = e ? e : cudaHostAlloc(&st->h_sp[i], (size_t)cblk * hw * sizeof(float), cudaHostAllocDefault);
            e = e ? e : cudaHostAlloc(&st->h_tp[i], (size_t)cblk * hw * sizeof(float), cudaHostAllocDefault);
            if (corrected_host && !corr_direct)
                e = e ? e : cudaHostAlloc(&st->h_corr[i], (size_t)C * hw * sizeof(float), cudaHostAllocDefault);
            if (!pinned) e = e ? e : cudaHostAlloc(&st->h_stage[i], (size_t)cap * hw * esz, cudaHostAllocDefault);
            if (seg) {
                e = e ? e : cudaMalloc(&st->d_prob[i], (size_t)cblk * hw * sizeof(float));
                e = e ? e : cudaHostAlloc(&st->h_prob[i], (size_t)cblk * hw * sizeof(float), cudaHostAllocDefault);
            }
        }
        if (piecewise) {
            e = e ? e : cudaMalloc(&st->d_smooth, (size_t)C * hw * sizeof(float));
            e = e ? e : cudaMalloc(&st->d_bsum, (size_t)cblk * hw * sizeof(double));
        }
        if (e != cudaSuccess) {
            stage_free_buffers(st);
            return cuda_fail(e, "vb_stage_run_host allocation");
        }
        st->esz = esz;
        st->cap = cap;
    }
    // chunk k covers frames [k*C, k*C + nf); its slot holds them plus the
    // high-pass halo [a0, a1) (recomputed motion for the halo frames)
    auto avail = [&](int64_t f0, int64_t nf) {
        return std::make_pair(std::max<int64_t>(0, f0 - hh), std::min<int64_t>(n_frames, f0 + nf + hh));
    };

    // the kSubParts pieces of an nf-frame slot load: piece j = [part(j), part(j+1))
    auto nparts = [&](int64_t nf) { return (int)std::min<int64_t>(vb_stage::kSubParts, std::max<int64_t>(1, nf)); };
    // (measured: pieces shrinking toward the recording's end, 40/30/20/10 %, no e2e gain)
    auto part = [&](int64_t nf, int j) { return nf * j / nparts(nf); };
    // host->device copy of frames [f0, f0+nf) into slot, piece by piece
    auto upload = [&](int slot, int64_t f0, int64_t nf) -> int {
        NvtxRange nv_up("upload");
        if (!pinned) VB_CUDA(cudaEventSynchronize(st->ev_h2d[slot]));  // staging slot free again
        VB_CUDA(cudaStreamWaitEvent(st->s_h2d, st->ev_comp[slot], 0));  // slot no longer read by compute
        for (int j = 0; j < nparts(nf); ++j) {
            const int64_t p0 = part(nf, j), p1 = part(nf, j + 1);
            const size_t off = (size_t)p0 * hw * esz, bytes = (size_t)(p1 - p0) * hw * esz;
            const char* src = (const char*)frames_host + (size_t)f0 * hw * esz + off;
            if (!pinned) {
                host_copy((char*)st->h_stage[slot] + off, src, bytes);
                src = (const char*)st->h_stage[slot] + off;
            }
            VB_CUDA(cudaMemcpyAsync((char*)st->d_frames[slot] + off, src, bytes, cudaMemcpyHostToDevice, st->s_h2d));
            VB_CUDA(cudaEventRecord(st->ev_sub[slot][j], st->s_h2d));
        }
        VB_CUDA(cudaEventRecord(st->ev_h2d[slot], st->s_h2d));
        return VB_OK;
    };
    // fresh events so the first waits are no-ops
    for (int i = 0; i < 2; ++i) {
        VB_CUDA(cudaEventRecord(st->ev_comp[i], st->s_comp));
        VB_CUDA(cudaEventRecord(st->ev_d2h[i], st->s_d2h));
        VB_CUDA(cudaEventRecord(st->ev_h2d[i], st->s_h2d));
    }

    // ---- phase A: template = mean of the first min(n, M) frames ----
    // When the template frames lie inside chunk 0 (the usual case), chunk 0 is
    // uploaded once and the template is summed from it in place; otherwise the
    // first M frames are streamed through the ring first.
    const int64_t m = st->external_ref ? 0 : std::min<int64_t>(n_frames, c.ref_frames);
    const bool chunk0_resident = m > 0 && m <= C;
    int rc = VB_OK;
    if (chunk0_resident) {
        const int64_t n0 = avail(0, std::min<int64_t>(C, n_frames)).second;
        rc = upload(0, 0, n0);
        if (rc == VB_OK) {  // only the pieces holding the first m frames
            for (int j = 0; j < nparts(n0) && part(n0, j) < m; ++j)
                VB_CUDA(cudaStreamWaitEvent(st->s_comp, st->ev_sub[0][j], 0));
            rc = launch_template_sum(st->d_frames[0], dtype, m, (int64_t)hw, st->d_tsum, 0, st->s_comp);
        }
    } else {
        for (int64_t f0 = 0, k = 0; f0 < m && rc == VB_OK; f0 += C, ++k) {
            const int slot = (int)(k & 1);
            const int64_t nf = std::min<int64_t>(C, m - f0);
            rc = upload(slot, f0, nf);
            if (rc) break;
            VB_CUDA(cudaStreamWaitEvent(st->s_comp, st->ev_h2d[slot], 0));
            rc = launch_template_sum(st->d_frames[slot], dtype, nf, (int64_t)hw, st->d_tsum, f0 > 0, st->s_comp);
            if (rc) break;
            VB_CUDA(cudaEventRecord(st->ev_comp[slot], st->s_comp));
        }
    }
    if (rc == VB_OK && !st->external_ref) rc = launch_template_finish(st->d_tsum, m, (int64_t)hw, st->d_ref, st->s_comp);
    if (rc == VB_OK) rc = vb_motion_plan_set_reference(st->plan, st->d_ref, st->s_comp);
    if (rc == VB_OK && shade)
        rc = launch_shading_gain(st->d_ref, c.height, c.width, st->shade_w.data(), st->shade_r, st->d_gain,
                                 st->s_comp);
    if (!chunk0_resident)
        for (int i = 0; i < 2 && rc == VB_OK; ++i) VB_CUDA(cudaEventRecord(st->ev_comp[i], st->s_comp));

    // ---- phase B: chunks ----
    const int64_t nchunks = (n_frames + C - 1) / C;
    auto drain = [&](int64_t k) -> int {
        const int slot = (int)(k & 1);
        const int64_t f0 = k * C, nf = std::min<int64_t>(C, n_frames - f0);
        const int64_t b0 = f0 / L, nb = (nf + L - 1) / L;
        NvtxRange nv_dr("drain");
        VB_CUDA(cudaEventSynchronize(st->ev_d2h[slot]));
        memcpy(vectors_host + f0, st->h_vec[slot], (size_t)nf * sizeof(vb_motion));
        if (!motion_only) {
            memcpy(spatial_host + (size_t)b0 * hw, st->h_sp[slot], (size_t)nb * hw * sizeof(float));
            memcpy(temporal_host + (size_t)b0 * hw, st->h_tp[slot], (size_t)nb * hw * sizeof(float));
        }
        if (corrected_host && !corr_direct)
            host_copy(corrected_host + (size_t)f0 * hw, st->h_corr[slot], (size_t)nf * hw * sizeof(float));
        if (seg) memcpy(prob_host + (size_t)b0 * hw, st->h_prob[slot], (size_t)nb * hw * sizeof(float));
        return VB_OK;
    };
    for (int64_t k = 0; k < nchunks && rc == VB_OK; ++k) {
        NvtxRange nv_chunk("chunk " + std::to_string(k));
        const int slot = (int)(k & 1);
        const int64_t f0 = k * C, nf = std::min<int64_t>(C, n_frames - f0);
        const int64_t nb = (nf + L - 1) / L;
        const auto [a0, a1] = avail(f0, nf);
        if (k == 0 && !chunk0_resident) rc = upload(slot, a0, a1 - a0);  // later chunks are prefetched below
        if (rc) break;
        VB_CUDA(cudaStreamWaitEvent(st->s_comp, st->ev_d2h[slot], 0));  // outputs of chunk k-2 drained
        float* corr = corrected_dev ? corrected_dev + (size_t)f0 * hw : (corrected_host ? st->d_corr[slot] : nullptr);
        for (int j = 0; j < nparts(a1 - a0) && rc == VB_OK; ++j) {  // search each piece as it lands
            const int64_t p0 = part(a1 - a0, j), p1 = part(a1 - a0, j + 1);
            VB_CUDA(cudaStreamWaitEvent(st->s_comp, st->ev_sub[slot][j], 0));
            rc = vb_motion_estimate(st->plan, (const char*)st->d_frames[slot] + (size_t)p0 * hw * esz, dtype, p1 - p0,
                                    c.subpixel, st->d_vec[slot] + p0, nullptr, st->s_comp);
            if (!piecewise) continue;
            // warp + smooth the piece's frames of each block it overlaps (a0 == f0 without the halo)
            for (int64_t b = p0 / L; rc == VB_OK && b * L < p1; ++b) {
                const int64_t s0 = std::max<int64_t>(p0, b * L), s1 = std::min<int64_t>({p1, (b + 1) * L, nf});
                if (s1 <= s0) continue;
                if (s0 == b * L) VB_CUDA(cudaMemsetAsync(st->d_bsum + (size_t)b * hw, 0, hw * sizeof(double), st->s_comp));
                rc = launch_block_piece((const char*)st->d_frames[slot] + (size_t)s0 * hw * esz, dtype, st->d_vec[slot] + s0,
                                        s1 - s0, c.height, c.width, st->weights.data(), st->wradius,
                                        shade ? st->d_gain : nullptr, 0, s1 - s0, corr ? corr + (size_t)s0 * hw : nullptr,
                                        st->d_smooth + (size_t)s0 * hw, st->d_bsum + (size_t)b * hw, st->s_comp);
            }
        }
        if (rc) break;
        if (motion_only) {
            if (corr)
                rc = launch_correct((const char*)st->d_frames[slot] + (size_t)(f0 - a0) * hw * esz, dtype, nf, c.height,
                                    c.width, st->d_vec[slot] + (f0 - a0), shade ? st->d_gain : nullptr, corr, st->s_comp);
        } else if (piecewise) {
            for (int64_t b = 0; b < nb && rc == VB_OK; ++b) {
                const int cnt = (int)std::min<int64_t>(L, nf - b * L);
                rc = launch_block_finish(st->d_smooth + (size_t)b * L * hw, 0, 0, cnt, n_frames, 0, (int64_t)hw,
                                         st->d_bsum + (size_t)b * hw, st->d_sp[slot] + (size_t)b * hw,
                                         st->d_tp[slot] + (size_t)b * hw, st->s_comp);
            }
        } else {
            SummaryOpts so;
            so.t_global0 = a0;
            so.t_total = n_frames;
            so.interior_off = f0 - a0;
            so.n_interior = nf;
            so.highpass_window = st->hp_window;
            so.gain = shade ? st->d_gain : nullptr;
            rc = launch_summarize_ex(st->d_frames[slot], dtype, st->d_vec[slot], a1 - a0, c.height, c.width, L,
                                     st->weights.data(), st->wradius, so, corr, st->d_sp[slot], st->d_tp[slot],
                                     st->s_comp);
        }
        if (rc) break;
        VB_CUDA(cudaEventRecord(st->ev_comp[slot], st->s_comp));
        if (seg) {  // U-Net of this chunk's blocks overlaps the next chunk's search
            VB_CUDA(cudaStreamWaitEvent(st->s_seg, st->ev_comp[slot], 0));
            rc = vb_unet_segment(st->unet, st->d_sp[slot], st->d_tp[slot], nb, c.height, c.width, st->unet_stride,
                                 nullptr, st->d_prob[slot], st->s_seg);
            if (rc) break;
            VB_CUDA(cudaEventRecord(st->ev_seg[slot], st->s_seg));
            VB_CUDA(cudaStreamWaitEvent(st->s_d2h, st->ev_seg[slot], 0));
        }
        VB_CUDA(cudaStreamWaitEvent(st->s_d2h, st->ev_comp[slot], 0));
        VB_CUDA(cudaMemcpyAsync(st->h_vec[slot], st->d_vec[slot] + (f0 - a0), (size_t)nf * sizeof(vb_motion),
                                cudaMemcpyDeviceToHost, st->s_d2h));
        if (!motion_only) {
            VB_CUDA(cudaMemcpyAsync(st->h_sp[slot], st->d_sp[slot], (size_t)nb * hw * sizeof(float),
                                    cudaMemcpyDeviceToHost, st->s_d2h));
            VB_CUDA(cudaMemcpyAsync(st->h_tp[slot], st->d_tp[slot], (size_t)nb * hw * sizeof(float),
                                    cudaMemcpyDeviceToHost, st->s_d2h));
        }
        if (corrected_host)
            VB_CUDA(cudaMemcpyAsync(corr_direct ? corrected_host + (size_t)f0 * hw : st->h_corr[slot], corr,
                                    (size_t)nf * hw * sizeof(float), cudaMemcpyDeviceToHost, st->s_d2h));
        if (seg)
            VB_CUDA(cudaMemcpyAsync(st->h_prob[slot], st->d_prob[slot], (size_t)nb * hw * sizeof(float),
                                    cudaMemcpyDeviceToHost, st->s_d2h));
        VB_CUDA(cudaEventRecord(st->ev_d2h[slot], st->s_d2h));
        // prefetch chunk k+1 into the other slot before blocking on chunk k-1's
        // outputs: the H2D stream only waits (device side) for chunk k-1's
        // compute, so the PCIe copy never waits for the host thread
        if (k + 1 < nchunks) {
            const int64_t g0 = (k + 1) * C, gn = std::min<int64_t>(C, n_frames - g0);
            const auto [b0, b1] = avail(g0, gn);
            rc = upload(slot ^ 1, b0, b1 - b0);
            if (rc) break;
        }
        if (k >= 1) rc = drain(k - 1);
    }
    if (rc == VB_OK && nchunks >= 1) rc = drain(nchunks - 1);
    return rc;
}

int vb_stage_destroy(vb_stage* st) {
    if (!st) return VB_OK;
    cudaSetDevice(st->cfg.device);
    stage_sync_all(st);
    stage_free_buffers(st);
    vb_motion_plan_destroy(st->plan);
    cudaFree(st->d_tsum);
    cudaFree(st->d_ref);
    cudaFree(st->d_gain);
    for (int i = 0; i < 2; ++i) {
        if (st->ev_h2d[i]) cudaEventDestroy(st->ev_h2d[i]);
        for (int j = 0; j < vb_stage::kSubParts; ++j)
            if (st->ev_sub[i][j]) cudaEventDestroy(st->ev_sub[i][j]);
        if (st->ev_comp[i]) cudaEventDestroy(st->ev_comp[i]);
        if (st->ev_d2h[i]) cudaEventDestroy(st->ev_d2h[i]);
    }
    if (st->s_comp) cudaStreamDestroy(st->s_comp);
    if (st->s_h2d) cudaStreamDestroy(st->s_h2d);
    if (st->s_d2h) cudaStreamDestroy(st->s_d2h);
    if (st->s_seg) cudaStreamDestroy(st->s_seg);
    for (int i = 0; i < 2; ++i)
        if (st->ev_seg[i]) cudaEventDestroy(st->ev_seg[i]);
    delete st;
    return VB_OK;
}

int vb_host_alloc(int64_t bytes, void** out) {
    if (!out || bytes < 0) return fail(VB_EINVAL, "null argument");
    *out = nullptr;
    if (bytes == 0) return VB_OK;
    const cudaError_t e = cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return fail(VB_ENOMEM, std::string("cudaHostAlloc: ") + cudaGetErrorString(e));
    }
    return VB_OK;
}

int vb_host_free(void* p) {
    if (p) VB_CUDA(cudaFreeHost(p));
    return VB_OK;
}

int vb_host_copy(void* dst, const void* src, int64_t bytes, int n_threads) {
    if ((!dst || !src) && bytes > 0) return fail(VB_EINVAL, "null argument");
    if (bytes > 0) host_copy_n(dst, src, (size_t)bytes, n_threads > 0 ? n_threads : host_copy_threads());
    return VB_OK;
}

}  // extern "C"
