// Multi-device stage handle: one process drives
// several GPUs through the C ABI alone -- no torch.distributed.  The
// recording is split into block-aligned time shards (whole L-frame blocks per
// device, so no block straddles two devices and the summaries need no
// exchange); each device runs its own vb_stage executor on its shard from the
// caller's host buffers in its own host thread.  The only collective is the
// template (motion.py:211-214): every device sums its own frames inside
// [0, M) in float64 (exact for integer samples), one ncclAllReduce(sum) over
// the group's communicator (ncclCommInitAll), and every device divides by M
// identically -- bit-identical templates on all devices, equal to the
// single-device template.
//
// NCCL is opened with dlopen at vb_group_create, so libvoltb200 carries no
// link-time NCCL dependency (inside a PyTorch process this binds the NCCL
// torch already loaded).
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <string>
#include <thread>
#include <vector>

#include "vb.cuh"

using namespace vb;

namespace {

struct NcclApi {
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            a.why = std::string("cannot load NCCL: ") + dlerror();
            return a;
        }
        a.comm_init_all = (decltype(a.comm_init_all))dlsym(h, "ncclCommInitAll");
        a.all_reduce = (decltype(a.all_reduce))dlsym(h, "ncclAllReduce");
        a.group_start = (decltype(a.group_start))dlsym(h, "ncclGroupStart");
        a.group_end = (decltype(a.group_end))dlsym(h, "ncclGroupEnd");
        a.comm_destroy = (decltype(a.comm_destroy))dlsym(h, "ncclCommDestroy");
        a.error_string = (decltype(a.error_string))dlsym(h, "ncclGetErrorString");
        a.ok = a.comm_init_all && a.all_reduce && a.group_start && a.group_end && a.comm_destroy && a.error_string;
        if (!a.ok) a.why = "NCCL library lacks the expected symbols";
        return a;
    }();
    return api;
}

int nccl_fail(ncclResult_t r, const char* where) {
    return fail(VB_ECUDA, std::string(where) + ": " + nccl().error_string(r));
}

}  // namespace

struct vb_group {
    vb_stage_config cfg{};
    std::vector<int> devices;
    std::vector<vb_stage*> stages;
    std::vector<ncclComm_t> comms;
    std::vector<cudaStream_t> streams;
    std::vector<double*> tsum;     // per device [H*W] float64 template sums
    std::vector<float*> ref;       // per device [H*W] float32 template
    std::vector<void*> head;       // per device upload buffer for its template frames
    std::vector<size_t> head_bytes;
    std::vector<int64_t> bounds;   // shard k = frames [bounds[k], bounds[k+1]) of the last run
};

extern "C" {

int vb_group_plan(int64_t n_frames, int segment_length, int n_devices, int64_t* frame_bounds) {
    if (!frame_bounds || n_devices < 1) return fail(VB_EINVAL, "null argument");
    if (segment_length < 2) return fail(VB_EINVAL, "segment length must be >= 2");
    if (n_frames < 0) return fail(VB_EINVAL, "video dimensions must all be >= 1");
    // blocks split as evenly as possible (distributed.shard_plan)
    const int64_t k = (n_frames + segment_length - 1) / segment_length;
    for (int d = 0; d <= n_devices; ++d)
        frame_bounds[d] = std::min<int64_t>(n_frames, k * d / n_devices * segment_length);
    return VB_OK;
}

int vb_group_create(vb_group** out, const int* devices, int n_devices, const vb_stage_config* cfg) {
    if (!out || !devices || !cfg || n_devices < 1) return fail(VB_EINVAL, "null argument");
    *out = nullptr;
    for (int i = 0; i < n_devices; ++i)
        for (int j = 0; j < i; ++j)
            if (devices[i] == devices[j]) return fail(VB_EINVAL, "devices must be distinct");
    const NcclApi& api = nccl();
    if (!api.ok) return fail(VB_ECUDA, api.why);
    auto* g = new vb_group();
    g->cfg = *cfg;
    g->devices.assign(devices, devices + n_devices);
    g->stages.assign(n_devices, nullptr);
    g->streams.assign(n_devices, nullptr);
    g->tsum.assign(n_devices, nullptr);
    g->ref.assign(n_devices, nullptr);
    g->head.assign(n_devices, nullptr);
    g->head_bytes.assign(n_devices, 0);
    g->comms.assign(n_devices, nullptr);
    const size_t hw = (size_t)cfg->height * cfg->width;
    int rc = VB_OK;
    for (int i = 0; i < n_devices && rc == VB_OK; ++i) {
        vb_stage_config c = *cfg;
        c.device = devices[i];
        rc = vb_stage_create(&g->stages[i], &c);
        if (rc) break;
        cudaError_t e = cudaSetDevice(devices[i]);
        e = e ? e : cudaStreamCreateWithFlags(&g->streams[i], cudaStreamNonBlocking);
        e = e ? e : cudaMalloc(&g->tsum[i], hw * sizeof(double));
        e = e ? e : cudaMalloc(&g->ref[i], hw * sizeof(float));
        if (e != cudaSuccess) rc = cuda_fail(e, "vb_group_create");
    }
    if (rc == VB_OK) {
        const ncclResult_t r = api.comm_init_all(g->comms.data(), n_devices, devices);
        if (r != ncclSuccess) rc = nccl_fail(r, "ncclCommInitAll");
    }
    if (rc) {
        vb_group_destroy(g);
        return rc;
    }
    *out = g;
    return VB_OK;
}

int vb_group_set_weights(vb_group* g, const double* weights, int wradius) {
    if (!g) return fail(VB_EINVAL, "null argument");
    for (vb_stage* st : g->stages) {
        const int rc = vb_stage_set_weights(st, weights, wradius);
        if (rc) return rc;
    }
    return VB_OK;
}

int vb_group_run_host(vb_group* g, const void* frames_host, int dtype, int64_t n_frames, vb_motion* vectors_host,
                      float* spatial_host, float* temporal_host, float* corrected_host) {
    if (!g || !frames_host || !vectors_host || !spatial_host || !temporal_host) return fail(VB_EINVAL, "null argument");
    if (dtype != VB_U16 && dtype != VB_F32) return fail(VB_EINVAL, "unsupported sample type");
    const vb_stage_config& c = g->cfg;
    const int L = c.segment_length;
    if (n_frames < 1) return fail(VB_EINVAL, "video dimensions must all be >= 1");
    if (n_frames % L == 1) return fail(VB_EINVAL, "temporal summary needs at least 2 frames");
    const int nd = (int)g->devices.size();
    const size_t hw = (size_t)c.height * c.width, esz = dtype == VB_U16 ? 2 : 4;
    NvtxRange nv("vb_group_run_host");
    g->bounds.assign(nd + 1, 0);
    int rc = vb_group_plan(n_frames, L, nd, g->bounds.data());
    if (rc) return rc;
    const int64_t m = std::min<int64_t>(n_frames, c.ref_frames);
    // ---- template: float64 sums of each device's own frames in [0, m), all-reduced ----
    for (int i = 0; i < nd; ++i) {
        VB_CUDA(cudaSetDevice(g->devices[i]));
        const int64_t lo = std::min(g->bounds[i], m), hi = std::min(g->bounds[i + 1], m);
        VB_CUDA(cudaMemsetAsync(g->tsum[i], 0, hw * sizeof(double), g->streams[i]));
        if (hi > lo) {
            const size_t bytes = (size_t)(hi - lo) * hw * esz;
            if (g->head_bytes[i] < bytes) {
                cudaFree(g->head[i]);
                g->head[i] = nullptr;
                g->head_bytes[i] = 0;
                VB_CUDA(cudaMalloc(&g->head[i], bytes));
                g->head_bytes[i] = bytes;
            }
            VB_CUDA(cudaMemcpyAsync(g->head[i], (const char*)frames_host + (size_t)lo * hw * esz, bytes,
                                    cudaMemcpyHostToDevice, g->streams[i]));
            rc = launch_template_sum(g->head[i], dtype, hi - lo, (int64_t)hw, g->tsum[i], 0, g->streams[i]);
            if (rc) return rc;
        }
    }
    const NcclApi& api = nccl();
    ncclResult_t r = api.group_start();
    for (int i = 0; i < nd && r == ncclSuccess; ++i)
        r = api.all_reduce(g->tsum[i], g->tsum[i], hw, ncclFloat64, ncclSum, g->comms[i], g->streams[i]);
    const ncclResult_t r2 = api.group_end();
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
    if (r2 != ncclSuccess) return nccl_fail(r2, "ncclGroupEnd");
    for (int i = 0; i < nd; ++i) {
        VB_CUDA(cudaSetDevice(g->devices[i]));
        rc = launch_template_finish(g->tsum[i], m, (int64_t)hw, g->ref[i], g->streams[i]);
        if (rc) return rc;
        VB_CUDA(cudaStreamSynchronize(g->streams[i]));
        rc = vb_stage_set_reference(g->stages[i], g->ref[i]);
        if (rc) return rc;
    }
    // ---- shards: one executor per device, concurrently ----
    std::vector<int> rcs(nd, VB_OK);
    std::vector<std::string> errs(nd);
    std::vector<std::thread> pool;
    for (int i = 0; i < nd; ++i) {
        const int64_t f0 = g->bounds[i], f1 = g->bounds[i + 1];
        if (f1 <= f0) continue;
        pool.emplace_back([&, i, f0, f1] {
            const int64_t b0 = f0 / L;
            rcs[i] = vb_stage_run_host(g->stages[i], (const char*)frames_host + (size_t)f0 * hw * esz, dtype, f1 - f0,
                                       vectors_host + f0, spatial_host + (size_t)b0 * hw, temporal_host + (size_t)b0 * hw,
                                       corrected_host ? corrected_host + (size_t)f0 * hw : nullptr, nullptr);
            if (rcs[i]) errs[i] = vb_last_error();
        });
    }
    for (auto& th : pool) th.join();
    for (int i = 0; i < nd; ++i)
        if (rcs[i]) return fail(rcs[i], "device " + std::to_string(g->devices[i]) + ": " + errs[i]);
    return VB_OK;
}

int64_t vb_group_last_launches(const vb_group* g) {
    int64_t n = 0;
    if (g)
        for (const vb_stage* st : g->stages) n += vb_stage_last_launches(st);
    return n;
}

int vb_group_destroy(vb_group* g) {
    if (!g) return VB_OK;
    for (size_t i = 0; i < g->devices.size(); ++i) {
        cudaSetDevice(g->devices[i]);
        if (g->streams[i]) cudaStreamSynchronize(g->streams[i]);
        if (g->comms[i]) nccl().comm_destroy(g->comms[i]);
        vb_stage_destroy(g->stages[i]);
        cudaFree(g->tsum[i]);
        cudaFree(g->ref[i]);
        cudaFree(g->head[i]);
        if (g->streams[i]) cudaStreamDestroy(g->streams[i]);
    }
    delete g;
    return VB_OK;
}

}  // extern "C"
