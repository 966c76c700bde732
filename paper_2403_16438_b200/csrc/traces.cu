// Trace extraction: mean corrected intensity over each
// ROI for every frame -- voltseg traces.py:23-40 extract_trace / extract_all.
//
// ROIs arrive in CSR form (roi_ptr[K+1], roi_idx[nnz] = flattened pixel
// indices in row-major order, i.e. np.nonzero order).  One warp per
// (ROI, frame): lanes stride over the ROI's pixels accumulating float64, then
// a fixed-order shuffle tree -- deterministic; the reference's float64 mean
// (numpy pairwise sum) agrees to ~1e-15 relative.
#include <algorithm>

#include "vb.cuh"

namespace vb {

__global__ void traces_kernel(const float* __restrict__ frames, int64_t n, int64_t hw,
                              const int32_t* __restrict__ roi_ptr, const int32_t* __restrict__ roi_idx,
                              double* __restrict__ out) {
    const int roi = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int p0 = roi_ptr[roi], p1 = roi_ptr[roi + 1];
    const double inv_n = 1.0 / (double)(p1 - p0);
    for (int64_t t = (int64_t)blockIdx.y * nw + warp; t < n; t += (int64_t)gridDim.y * nw) {
        const float* f = frames + t * hw;
        double s = 0.0;
        for (int i = p0 + lane; i < p1; i += 32) s += (double)__ldg(f + roi_idx[i]);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[(int64_t)roi * n + t] = s * inv_n;
    }
}

int launch_traces(const float* frames, int64_t n, int64_t hw, const int32_t* roi_ptr, const int32_t* roi_idx,
                  int n_rois, double* out, cudaStream_t s) {
    if (n <= 0 || n_rois <= 0) return VB_OK;
    const int threads = 256, warps = threads / 32;
    const int64_t ychunks = std::min<int64_t>((n + warps - 1) / warps, 65535);
    dim3 grid((unsigned)n_rois, (unsigned)ychunks);
    {
        ProfScope ps(kProfOther, s);
        traces_kernel<<<grid, threads, 0, s>>>(frames, n, hw, roi_ptr, roi_idx, out);
    }
    VB_LAUNCHED();
    return VB_OK;
}

}  // namespace vb

extern "C" int vb_extract_traces(const float* frames_dev, int64_t n_frames, int height, int width,
                                 const int32_t* roi_ptr_dev, const int32_t* roi_idx_dev, int n_rois, double* out_dev,
                                 void* stream) {
    using namespace vb;
    if (!frames_dev || !roi_ptr_dev || !roi_idx_dev || !out_dev) return fail(VB_EINVAL, "null argument");
    if (n_rois < 0 || height < 1 || width < 1) return fail(VB_EINVAL, "invalid trace geometry");
    return launch_traces(frames_dev, n_frames, (int64_t)height * width, roi_ptr_dev, roi_idx_dev, n_rois, out_dev,
                         (cudaStream_t)stream);
}

extern "C" int vb_extract_traces_raw(const void* frames_dev, int dtype, const vb_motion* vectors_dev,
                                     const float* gain_dev, int64_t n_frames, int height, int width,
                                     const int32_t* roi_ptr_dev, const int32_t* roi_idx_dev, int n_rois,
                                     double* out_dev, void* stream) {
    using namespace vb;
    if (!frames_dev || !roi_ptr_dev || !roi_idx_dev || !out_dev) return fail(VB_EINVAL, "null argument");
    if (dtype != VB_U16 && dtype != VB_F32) return fail(VB_EINVAL, "unsupported sample type");
    if (n_rois < 0 || height < 1 || width < 1) return fail(VB_EINVAL, "invalid trace geometry");
    return launch_traces_raw(frames_dev, dtype, n_frames, height, width, vectors_dev, gain_dev, roi_ptr_dev,
                             roi_idx_dev, n_rois, out_dev, (cudaStream_t)stream);
}
