"""Fused preprocessing stage: correct_motion (motion.py:217-241) followed by
summarize (summarize.py:99-102), as pipeline.py:198-224 runs them -- on one
device, without materialising the corrected video unless asked.

Three entry points:
  * preprocess(video, ...)        -- numpy/Video in, numpy out (API parity).
  * DevicePreprocessor            -- device-resident recording; the bench's
                                     `value` path (inputs already in HBM).
  * HostStage                     -- vb_stage C-ABI executor over a HOST
                                     buffer: chunked pinned H2D / compute / D2H
                                     overlap; the bench's `e2e` path.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
import threading
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _device as D
from . import _lib
from . import motion as M
from .extensions import check_window, shading_gain_device, shading_weights
from .summarize import DEFAULT_SEGMENT_LENGTH, DEFAULT_SMOOTH_SIGMA, SummaryPair, gaussian_weights, summarize_device
from .video import Video


@dataclass
class StageConfig:
    patch_size: int = M.DEFAULT_PATCH_SIZE
    search_radius: int = M.DEFAULT_SEARCH_RADIUS
    subpixel: bool = True
    ref_frames: int | None = None  # None -> motion.REFERENCE_FRAMES at call time
    segment_length: int = DEFAULT_SEGMENT_LENGTH
    sigma: float = DEFAULT_SMOOTH_SIGMA
    # A17 extensions (opt-in, default off; no reference counterpart -- extensions.py)
    highpass_window: int = 0     # odd N: temporal summary over x - mean_N(x)
    shading_sigma: float = 0.0   # > 0: corrected = warped / flat-field gain of the template


@dataclass
class DeviceResult:
    vectors: torch.Tensor            # device buffer of vb_motion records
    spatial: torch.Tensor            # [K, H, W] float32
    temporal: torch.Tensor           # [K, H, W] float32
    corrected: torch.Tensor | None   # [T, H, W] float32 or None
    n_frames: int

    def vectors_numpy(self) -> np.ndarray:
        return D.motion_to_numpy(self.vectors, self.n_frames)


class DevicePreprocessor:
    """Reusable stage for recordings of one geometry already in HBM.

    run(frames) = template (f64 mean of the first M frames) -> template patch
    prep -> ZNCC motion search for every frame -> fused warp + per-block
    spatial mean / smoothing / max-minus-median.  5 + 2*ceil(T/B) kernel
    launches, all on the current stream."""

    def __init__(self, height: int, width: int, config: StageConfig | None = None):
        self.cfg = config or StageConfig()
        c = self.cfg
        if c.search_radius < 1:
            raise ValueError("search_radius must be >= 1")
        if c.segment_length < 2:
            raise ValueError("segment length must be >= 2")
        self.height, self.width = height, width
        self.grid = M.PatchGrid.cover(height, width, c.patch_size, margin=c.search_radius)
        self.plan = M.MotionPlan(height, width, self.grid.origins, c.patch_size, c.search_radius)
        self.weights, self.wradius = gaussian_weights(c.sigma)
        self.window = check_window(c.highpass_window)
        self.gain = None

    def run(self, frames: torch.Tensor, corrected_out: torch.Tensor | None = None,
            vectors_out: torch.Tensor | None = None) -> DeviceResult:
        t = frames.shape[0]
        if t % self.cfg.segment_length == 1:
            raise ValueError("temporal summary needs at least 2 frames")
        m = M.REFERENCE_FRAMES if self.cfg.ref_frames is None else self.cfg.ref_frames
        ref = M.device_reference(frames, m)
        self.plan.set_reference(ref)
        self.set_shading(ref)
        vec, sp, tp = self.search_and_summarize(frames, corrected_out, vectors_out)
        return DeviceResult(vec, sp, tp, corrected_out, t)

    # Blocks per pipelined chunk (see search_and_summarize); 0 = serial.
    # Measured on C2: 0 -> 44.3 ms/step, 1..5 -> 44.4-45.8 ms (the SMs are
    # already saturated; concurrent kernels only slow each other), so serial.
    overlap_blocks = 0

    def set_shading(self, ref: torch.Tensor) -> None:
        """Flat-field gain of this recording's template (A17; no-op when off)."""
        s = self.cfg.shading_sigma
        self.gain = shading_gain_device(ref, s) if s and s > 0 else None

    def search_and_summarize(self, frames: torch.Tensor, corrected_out: torch.Tensor | None = None,
                             vectors_out: torch.Tensor | None = None, t_global0: int = 0,
                             t_total: int | None = None, interior: tuple[int, int] | None = None):
        """Motion search then fused warp + summaries, pipelined in block-aligned
        chunks over two streams: the search of chunk k+1 (FP32-bound) runs
        while the summaries of chunk k (FP64-bound) do, so the two kernels'
        pipes overlap on the SMs.  Results are identical to the serial order."""
        c = self.cfg
        t = frames.shape[0]
        L = c.segment_length
        k_blocks = math.ceil(t / L)
        dev = frames.device
        vec = vectors_out if vectors_out is not None else D.empty_motion(t, dev)
        sp = torch.empty((k_blocks, self.height, self.width), dtype=torch.float32, device=dev)
        tp = torch.empty_like(sp)
        chunk = L * self.overlap_blocks if self.overlap_blocks > 0 else t
        if interior is not None:
            k_blocks = math.ceil(interior[1] / L)
            sp, tp = sp[:k_blocks], tp[:k_blocks]
        if chunk >= t or self.window or self.gain is not None or interior is not None:
            self.plan.estimate(frames, c.subpixel, out=vec)
            summarize_device(frames, L, c.sigma, vectors_dev=vec, corrected_out=corrected_out,
                             spatial_out=sp, temporal_out=tp, highpass_window=self.window, gain=self.gain,
                             t_global0=t_global0, t_total=t_total, interior=interior)
            return vec, sp, tp
        main = torch.cuda.current_stream(dev)
        if getattr(self, "_side", None) is None:
            self._side = torch.cuda.Stream(device=dev)
        side = self._side
        side.wait_stream(main)
        rec = _lib.MOTION_DTYPE.itemsize
        for f0 in range(0, t, chunk):
            f1 = min(t, f0 + chunk)
            v = vec[f0 * rec:f1 * rec]
            self.plan.estimate(frames[f0:f1], c.subpixel, out=v)
            ev = torch.cuda.Event()
            ev.record(main)
            with torch.cuda.stream(side):
                side.wait_event(ev)
                b0, b1 = f0 // L, math.ceil(f1 / L)
                summarize_device(frames[f0:f1], L, c.sigma, vectors_dev=v,
                                 corrected_out=None if corrected_out is None else corrected_out[f0:f1],
                                 spatial_out=sp[b0:b1], temporal_out=tp[b0:b1])
        main.wait_stream(side)
        return vec, sp, tp

    def close(self):
        self.plan.close()


def preprocess(video, config: StageConfig | None = None, return_corrected: bool = True, out=None):
    """correct_motion + summarize in one device pass.

    Returns (corrected Video | None, list[MotionVector], list[SummaryPair]) --
    the same values as the reference's correct_motion(video, MotionConfig(...))
    followed by summarize(corrected, L, sigma).

    out: optional float32 (T, H, W) C-contiguous host array that receives the
    corrected video (reused across calls; page-locked arrays -- pinned_empty()
    -- are filled by direct device->host copies).  Without it the corrected
    video lands in a page-locked array from the stage's host pool."""
    v = Video.wrap(video)
    dev = D.require_cuda()
    if not (isinstance(v.samples, torch.Tensor) and v.samples.is_cuda):
        # host recording: the C-ABI executor streams it through a two-chunk
        # device ring (bounded HBM, H2D / compute / D2H overlapped, threaded
        # host staging); bit-identical to the device-resident path below
        hs = cached_host_stage(dev, v.height, v.width, config)
        rec, sp, tp, corr = hs.run(v.samples, corrected=return_corrected, out=out)
        res = Video._trusted(corr, frame_rate=v.frame_rate) if return_corrected else None
        return res, M._vectors_from_numpy(rec), [SummaryPair(i, sp[i], tp[i]) for i in range(sp.shape[0])]
    frames = D.as_device_frames(v.samples, dev)
    pre = DevicePreprocessor(v.height, v.width, config)
    try:
        corr = torch.empty(frames.shape, dtype=torch.float32, device=dev) if return_corrected else None
        res = pre.run(frames, corrected_out=corr)
        rec = res.vectors_numpy()
        sp, tp = res.spatial.cpu().numpy(), res.temporal.cpu().numpy()
        if return_corrected:
            host = _check_out(out, tuple(frames.shape)) if out is not None else pinned_empty(tuple(frames.shape))
            torch.from_numpy(host).copy_(corr)
        out_v = Video._trusted(host, frame_rate=v.frame_rate) if return_corrected else None
    finally:
        pre.close()
    vectors = M._vectors_from_numpy(rec)
    pairs = [SummaryPair(i, sp[i], tp[i]) for i in range(sp.shape[0])]
    return out_v, vectors, pairs


# ---- per-thread executor cache (shared by preprocess and motion.correct_motion)
_stage_cache = threading.local()


def _resolved(config: StageConfig | None) -> StageConfig:
    """The configuration with call-time defaults filled in (ref_frames reads
    motion.REFERENCE_FRAMES now, as the reference does at each call)."""
    c = dataclasses.replace(config) if config is not None else StageConfig()
    if c.ref_frames is None:
        c.ref_frames = M.REFERENCE_FRAMES
    return c


def cached_host_stage(dev: torch.device, height: int, width: int, config: StageConfig | None) -> "HostStage":
    """The calling thread's executor for this geometry + resolved configuration
    (repeated calls skip the device-ring and pinned-slot allocations); a
    different key replaces it."""
    c = _resolved(config)
    key = (dev.index or 0, height, width, repr(c))
    cache = _stage_cache.__dict__
    if cache.get("key") != key:
        if cache.get("hs") is not None:
            cache["hs"].close()
        cache["hs"], cache["key"] = None, None
        cache["hs"] = HostStage(height, width, c, device=dev.index or 0)
        cache["key"] = key
    return cache["hs"]


def release_cached() -> None:
    """Free the calling thread's cached executor (device ring, pinned staging)
    and the idle page-locked output buffers of the host pool."""
    cache = _stage_cache.__dict__
    if cache.get("hs") is not None:
        cache["hs"].close()
    cache["hs"], cache["key"] = None, None
    _POOL.trim(0)


# ---- page-locked output buffers -------------------------------------------
class _PinnedBlock:
    """One vb_host_alloc block exposed through the array interface; the
    numpy arrays made from it keep it alive, and when the last one goes the
    block returns to its pool."""

    def __init__(self, pool: "PinnedPool", ptr: int, nbytes: int, shape: tuple, dtype: np.dtype):
        self.__array_interface__ = {"data": (ptr, False), "shape": shape, "typestr": dtype.str, "version": 3}
        fin = weakref.finalize(self, pool._release, ptr, nbytes)
        fin.atexit = False  # at interpreter exit the process releases page-locked memory itself


class PinnedPool:
    """Reuses page-locked host blocks of equal size: allocating and first-touching
    gigabytes of output per call costs more than the PCIe transfer into them,
    and page-locked memory is what lets the executor copy device->host straight
    into the caller's array.  At most `keep` idle blocks are retained."""

    def __init__(self, keep: int = 2):
        self.keep = keep
        self._idle: list[tuple[int, int]] = []  # (nbytes, ptr), most recent last
        self._lock = threading.Lock()

    def empty(self, shape: tuple, dtype=np.float32) -> np.ndarray:
        dtype = np.dtype(dtype)
        nbytes = int(np.prod(shape)) * dtype.itemsize
        if nbytes == 0:
            return np.empty(shape, dtype)
        ptr = None
        with self._lock:
            for i in range(len(self._idle) - 1, -1, -1):
                if self._idle[i][0] == nbytes:
                    ptr = self._idle.pop(i)[1]
                    break
        if ptr is None:
            p = C.c_void_p()
            rc = _lib.load().vb_host_alloc(nbytes, C.byref(p))
            if rc != _lib.VB_OK:
                self.trim(0)  # retry once with the idle blocks released
                _lib.call("vb_host_alloc", nbytes, C.byref(p))
            ptr = p.value
        return np.asarray(_PinnedBlock(self, ptr, nbytes, tuple(shape), dtype))

    def _release(self, ptr: int, nbytes: int) -> None:
        with self._lock:
            self._idle.append((nbytes, ptr))
        self.trim(self.keep)

    def trim(self, keep: int) -> None:
        with self._lock:
            drop = self._idle[:max(0, len(self._idle) - keep)]
            self._idle = self._idle[len(drop):]
        for _, ptr in drop:
            _lib.load().vb_host_free(ptr)


_POOL = PinnedPool()


def pinned_empty(shape: tuple, dtype=np.float32) -> np.ndarray:
    """A page-locked host array from the stage's pool (see PinnedPool)."""
    return _POOL.empty(shape, dtype)


def _check_out(out, shape: tuple) -> np.ndarray:
    if not isinstance(out, np.ndarray) or out.dtype != np.float32 or out.shape != shape \
            or not out.flags.c_contiguous or not out.flags.writeable:
        raise ValueError(f"out must be a writeable C-contiguous float32 array of shape {shape}")
    return out


class HostStage:
    """vb_stage: the C-ABI whole-stage executor over host buffers."""

    def __init__(self, height: int, width: int, config: StageConfig | None = None, device: int | None = None,
                 chunk_frames: int = 0):
        self.cfg = config or StageConfig()
        c = self.cfg
        dev = D.require_cuda() if device is None else torch.device("cuda", device)
        m = M.REFERENCE_FRAMES if c.ref_frames is None else c.ref_frames
        sc = _lib.VbStageConfig(height, width, c.patch_size, c.search_radius, int(c.subpixel), m,
                                c.segment_length, float(c.sigma), dev.index or 0, int(chunk_frames))
        h = C.c_void_p()
        _lib.call("vb_stage_create", C.byref(h), C.byref(sc))
        self._h = h
        w, r = gaussian_weights(c.sigma)
        self._w = w
        _lib.call("vb_stage_set_weights", self._h, w.ctypes.data, r)
        _lib.call("vb_stage_set_highpass", self._h, check_window(c.highpass_window))
        if c.shading_sigma and c.shading_sigma > 0:
            self._sw, sr = shading_weights(c.shading_sigma)
            _lib.call("vb_stage_set_shading", self._h, self._sw.ctypes.data, sr)
        self.height, self.width = height, width

    def run(self, frames: np.ndarray, corrected: bool = False, summaries: bool = True, out=None):
        """frames: uint16/float32 (T,H,W) host array (pinned or pageable).
        Returns (vectors record array, spatial [K,H,W], temporal [K,H,W], corrected|None);
        summaries=False: motion only (spatial / temporal are None).  The
        corrected video goes into `out` when given, else into a page-locked
        array from the host pool (direct device->host copies)."""
        a = frames
        if isinstance(a, torch.Tensor):
            assert not a.is_cuda
            dtype = D.vb_dtype(a)
            ptr, t = a.data_ptr(), a.shape[0]
        else:
            a = np.ascontiguousarray(a)
            if a.dtype not in (np.uint16, np.float32):
                a = a.astype(np.float32)
            dtype = _lib.VB_U16 if a.dtype == np.uint16 else _lib.VB_F32
            ptr, t = a.ctypes.data, a.shape[0]
        k = math.ceil(t / self.cfg.segment_length)
        vec = np.empty(t, dtype=_lib.MOTION_DTYPE)
        sp = np.empty((k, self.height, self.width), np.float32) if summaries else None
        tp = np.empty((k, self.height, self.width), np.float32) if summaries else None
        corr = None
        if corrected:
            shape = (t, self.height, self.width)
            corr = _check_out(out, shape) if out is not None else pinned_empty(shape)
        self.run_into(ptr, dtype, t, vec, sp, tp, corr)
        return vec, sp, tp, corr

    def run_into(self, frames_ptr: int, dtype: int, t: int, vec, sp, tp, corr=None,
                 corrected_dev: torch.Tensor | None = None) -> None:
        """Zero-allocation variant: outputs are caller-provided host buffers
        (numpy arrays or pinned torch tensors); corrected_dev optionally keeps
        the whole corrected video in HBM."""
        def p(x):
            if x is None:
                return None
            return x.data_ptr() if isinstance(x, torch.Tensor) else x.ctypes.data
        _lib.call("vb_stage_run_host", self._h, frames_ptr, dtype, t, p(vec), p(sp), p(tp), p(corr),
                  D.ptr(corrected_dev))

    def attach_unet(self, net, stride: int = 32) -> None:
        """Segment every block's summaries with `net` (unet.DeviceUNet or a
        WeightBundle) inside run(..., segment=True) -- SURVEY 8(f) rows 2 + 4."""
        from . import unet as U

        if net is not None and not isinstance(net, U.DeviceUNet):
            net = U.DeviceUNet(net)
        self._net = net
        _lib.call("vb_stage_set_unet", self._h, net.handle if net is not None else None, int(stride))

    def run_segment(self, frames: np.ndarray, corrected: bool = False):
        """run() plus the per-block probability maps [K,H,W] (needs attach_unet)."""
        a = np.ascontiguousarray(frames)
        if a.dtype not in (np.uint16, np.float32):
            a = a.astype(np.float32)
        dtype = _lib.VB_U16 if a.dtype == np.uint16 else _lib.VB_F32
        t = a.shape[0]
        k = math.ceil(t / self.cfg.segment_length)
        vec = np.empty(t, dtype=_lib.MOTION_DTYPE)
        sp = np.empty((k, self.height, self.width), np.float32)
        tp = np.empty_like(sp)
        prob = np.empty_like(sp)
        corr = np.empty((t, self.height, self.width), np.float32) if corrected else None
        _lib.call("vb_stage_run_host_segment", self._h, a.ctypes.data, dtype, t, vec.ctypes.data, sp.ctypes.data,
                  tp.ctypes.data, prob.ctypes.data, corr.ctypes.data if corr is not None else None, None)
        return vec, sp, tp, prob, corr

    @property
    def last_launches(self) -> int:
        return int(_lib.load().vb_stage_last_launches(self._h))

    def close(self):
        if getattr(self, "_h", None) is not None:
            _lib.load().vb_stage_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def group_plan(n_frames: int, segment_length: int, n_devices: int) -> list[tuple[int, int]]:
    """Block-aligned shards of vb_group (frames [lo, hi) per device)."""
    b = np.empty(n_devices + 1, np.int64)
    _lib.call("vb_group_plan", int(n_frames), int(segment_length), int(n_devices), b.ctypes.data)
    return [(int(b[i]), int(b[i + 1])) for i in range(n_devices)]


class GroupStage:
    """vb_group: several GPUs driven from one process through the C ABI alone
     -- block-aligned time shards, the template all-reduced
    over NCCL inside the library, one executor per device.  Outputs equal a
    single-device HostStage run of the whole recording."""

    def __init__(self, height: int, width: int, config: StageConfig | None = None, devices=(0,)):
        c = _resolved(config)
        self.cfg = c
        devs = np.ascontiguousarray(list(devices), dtype=np.int32)
        sc = _lib.VbStageConfig(height, width, c.patch_size, c.search_radius, int(c.subpixel), c.ref_frames,
                                c.segment_length, float(c.sigma), int(devs[0]), 0)
        if c.highpass_window or c.shading_sigma:
            raise ValueError("the device group runs the reference stage only (no A17 options)")
        h = C.c_void_p()
        _lib.call("vb_group_create", C.byref(h), devs.ctypes.data, len(devs), C.byref(sc))
        self._h = h
        w, r = gaussian_weights(c.sigma)
        self._w = w
        _lib.call("vb_group_set_weights", self._h, w.ctypes.data, r)
        self.height, self.width, self.devices = height, width, tuple(int(d) for d in devs)

    def run(self, frames: np.ndarray, corrected: bool = False):
        a = np.ascontiguousarray(frames)
        if a.dtype not in (np.uint16, np.float32):
            a = a.astype(np.float32)
        dtype = _lib.VB_U16 if a.dtype == np.uint16 else _lib.VB_F32
        t = a.shape[0]
        k = math.ceil(t / self.cfg.segment_length)
        vec = np.empty(t, dtype=_lib.MOTION_DTYPE)
        sp = np.empty((k, self.height, self.width), np.float32)
        tp = np.empty_like(sp)
        corr = pinned_empty((t, self.height, self.width)) if corrected else None
        _lib.call("vb_group_run_host", self._h, a.ctypes.data, dtype, t, vec.ctypes.data, sp.ctypes.data,
                  tp.ctypes.data, corr.ctypes.data if corr is not None else None)
        return vec, sp, tp, corr

    @property
    def last_launches(self) -> int:
        return int(_lib.load().vb_group_last_launches(self._h))

    def close(self):
        if getattr(self, "_h", None) is not None:
            _lib.load().vb_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

