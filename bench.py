#!/usr/bin/env python
"""Benchmark of the B200 preprocessing stage (motion correction -> per-block
summary images) on BASELINE.json's paper-scale workload (configs[1], "c2":
10,000 x 256 x 512 uint16 frames, search radius 8, patch 21, L = 1000, M = 100).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = the whole stage over one rank's 10,000-frame recording shard:
template (f64 mean of the recording's first M frames; all-reduced over NCCL
when N > 1) -> ZNCC motion search for every frame -> fused warp + per-block
spatial mean / smoothing / max-minus-median, corrected video written to HBM.
`value` = frames processed by all ranks / max-over-ranks device time (inputs
resident in HBM, CUDA events).  `e2e` = the same through the C-ABI host entry
point vb_stage_run_host with pinned host input (H2D of every frame, D2H of
vectors + summaries inside the timed region).  `e2e_dropin` = the drop-in
Python API (stage.preprocess) from a plain numpy uint16 recording to the
corrected float32 video, vectors and summaries on the host -- what the
reference's correct_motion + summarize return.

--gpus N > 1 without a torchrun environment re-launches itself under
torchrun (one process per GPU).  N > 1 defaults to strong scaling: the one
10,000-frame recording split into frame-balanced time shards, blocks that
straddle two ranks exchanged over peer memory; --scaling weak gives every rank
its own 10,000-frame shard.  `--impl reference` times the unmodified
reference (voltseg, oracle/_ref) on the host CPU cores, one full L-frame block
of the same recording per step (blocks in turn).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "frames/sec of preprocessing stage at 1/2/4/8 B200 (+% HBM roofline) vs CPU ref"
UNIT = "frames/s"
CONFIG = "c2"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--stage", choices=["preprocess", "unet", "pipeline"], default="preprocess",
                   help="preprocess: the headline stage; unet: the summaries' consumer (normalize_pair + "
                        "tile_and_merge for every block, SURVEY 8(f) row 2)")
    p.add_argument("--config", default=CONFIG)
    p.add_argument("--frames", type=int, default=0, help="override frames per rank (profiling only)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-single-thread", action="store_true",
                   help="reference arm: skip the extra threads=1 block (BASELINE.md section 3 asks for N = 1 too)")
    p.add_argument("--no-corrected", action="store_true", help="do not materialise the corrected video")
    p.add_argument("--cpu-sample", type=int, default=2000, help="frames in the CPU baseline sample (~10 s of CPU work on C2)")
    p.add_argument("--ref-step-frames", type=int, default=0,
                   help="frames per --impl reference step (default: one full block, L frames)")
    p.add_argument("--scaling", choices=["weak", "strong"], default=None,
                   help="weak: each rank owns its own T-frame recording shard; strong (default for N > 1): one "
                        "T-frame recording split into frame-balanced shards (straddling blocks exchanged over "
                        "peer memory)")
    p.add_argument("--no-dropin", action="store_true", help="skip the drop-in Python API e2e leg")
    return p.parse_args()


def free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def relaunch_under_torchrun(args) -> int | None:
    """--gpus N > 1 outside torchrun: re-run this command as N ranks (one process
    per GPU, rendezvous on 127.0.0.1); rank 0 prints the JSON line."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- workload
def workload(cfg_name: str, frames_override: int):
    from paper_2403_16438_b200 import synth

    cfg = synth.CONFIGS[cfg_name]
    if frames_override:
        cfg = cfg.with_frames(frames_override)
    return cfg


def algorithmic_numbers(cfg, n_patches: int):
    """bytes/frame = H*W*(2 u16 read + 4 f32 corrected write) + 8*H*W/L;
    ZNCC cross-term flops/frame = 2 * N_patch * (2r+1)^2 * P^2."""
    hw = cfg.height * cfg.width
    bytes_frame = hw * (2 + 4) + 8 * hw / cfg.segment_length
    flops_frame = 2.0 * n_patches * (2 * cfg.radius + 1) ** 2 * 21 * 21
    return bytes_frame, flops_frame


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return json.loads(p.read_text()), "MEASURED_PEAKS.json"
        except ValueError:
            pass
    return {"hbm_gbs": 6650.0}, "fallback B200_PROFILING.md"


# ---------------------------------------------------------------- CPU reference
def reference_stage_fps(frames_f32: np.ndarray, cfg, threads: int):
    """Time the UNMODIFIED reference stage (voltseg native backend) on host cores:
    correct_motion(video, MotionConfig(search_radius=r, threads=N)) then
    summarize(corrected, L, 3.0) -- BASELINE.md section 3."""
    from oracle import ref

    motion, summarize, kernels, video_io = ref.load()
    motion.REFERENCE_FRAMES = cfg.ref_frames  # read at call time (motion.py:213)
    video = video_io.Video(frames_f32, frame_rate=cfg.fps)
    t0 = time.perf_counter()
    corrected, _vecs = motion.correct_motion(video, motion.MotionConfig(search_radius=cfg.radius, threads=threads))
    summarize.summarize(corrected, cfg.segment_length, 3.0)
    dt = time.perf_counter() - t0
    return frames_f32.shape[0] / dt, dt, kernels.BACKEND


def oracle_port_fps(frames_f32: np.ndarray, cfg, threads: int):
    from oracle import oracle as O

    t0 = time.perf_counter()
    O.preprocess(frames_f32, 21, cfg.radius, True, cfg.ref_frames, cfg.segment_length, 3.0, threads,
                 want_corrected=False)
    dt = time.perf_counter() - t0
    return frames_f32.shape[0] / dt, dt


def host_sample(cfg, n: int) -> np.ndarray:
    """The first n frames of the (rank 0) recording, as the reference's float32 Video data."""
    import torch

    from paper_2403_16438_b200 import synth

    if torch.cuda.is_available():
        v = synth.generate(cfg, "cuda")[:n]
        arr = v.view(torch.int16).cpu().numpy().view(np.uint16)
        del v
        torch.cuda.empty_cache()
    else:
        arr = synth.generate_numpy(cfg.with_frames(n))
    return arr.astype(np.float32)


def run_reference(args):
    rank, world, _ = dist_env()
    cfg = workload(args.config, args.frames)
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    n = min(args.ref_step_frames or cfg.segment_length, cfg.frames)
    # the whole recording on the host; step i runs the reference stage on block
    # (W + i) mod K -- one full L-frame block per step, so K steps cover it all
    rec = host_sample(cfg, cfg.frames)
    nblk = max(1, cfg.frames // n)
    kind = "reference"
    try:
        from oracle import ref as _r

        if not _r.available():
            raise RuntimeError("oracle/_ref missing")
        fn = lambda x: reference_stage_fps(x, cfg, threads)[1]  # noqa: E731
    except Exception:  # reference not built: oracle port (C restatement)
        kind = "port"
        fn = lambda x: oracle_port_fps(x, cfg, threads)[1]  # noqa: E731
    it = iter(range(10 ** 9))

    def step():
        b = next(it) % nblk
        return fn(rec[b * n:(b + 1) * n])

    for _ in range(args.warmup):
        step()
    times = [step() for _ in range(args.steps)]
    total = sum(times)
    fps = n * args.steps / total
    # also N = 1 (one block, after the timed steps)
    one = None
    if not args.no_single_thread and threads > 1:
        if kind == "reference":
            fps1 = n / reference_stage_fps(rec[:n], cfg, 1)[1]
        else:
            fps1 = n / oracle_port_fps(rec[:n], cfg, 1)[1]
        one = {"value": fps1, "unit": UNIT, "cores": 1, "kind": kind,
               "sample": f"block 0 of {cfg.name} ({n} frames) with threads=1, timed after the steps"}
    line = {
        "metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32/f64", "data": "synthetic (repo generator, seed 1002)",
        "impl": "reference",
        "config": {"workload": f"{cfg.name}: {cfg.frames}x{cfg.height}x{cfg.width} uint16 (step sample: one full "
                               f"{n}-frame block, blocks in turn), r={cfg.radius}, patch=21, L={cfg.segment_length}, "
                               f"M={cfg.ref_frames}",
                   "threads": threads},
        "cpu_baseline": {"value": fps, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": f"one {n}-frame block of {cfg.name} per step (block (W+i) mod {nblk}); voltseg "
                                   f"correct_motion(threads={threads}) + summarize(L={cfg.segment_length}); the "
                                   f"template is each block's first M frames"},
        "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "cpu_baseline_1thread": one,
        "host": host_details(),
    }
    print(json.dumps(line), flush=True)
    return 0


def host_details() -> dict:
    """core count, CPU model, numpy / scipy versions."""
    d = {"cores": os.cpu_count(), "numpy": np.__version__}
    try:
        import scipy

        d["scipy"] = scipy.__version__
    except ImportError:
        d["scipy"] = None
    try:
        with open("/proc/cpuinfo") as f:
            d["cpu_model"] = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), None)
    except OSError:
        d["cpu_model"] = None
    return d


# ---------------------------------------------------------------- ours
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2403_16438_b200 import _lib, distributed, stage, synth
    from paper_2403_16438_b200 import _device as D

    rank, world, local = dist_env()
    # BENCH_DIST_BACKEND=gloo (+ ranks sharing one GPU) exercises the N>1 code
    # path on a single-GPU box: gloo all-reduces are host-mediated, so no
    # kernel waits on another rank's kernel.  Measurements use NCCL.
    backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
    ngpu = torch.cuda.device_count()
    if backend == "nccl" and local >= ngpu:
        raise SystemExit(f"rank {rank}: LOCAL_RANK {local} but only {ngpu} visible GPU(s)")
    local_dev = local % ngpu
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    cfg = workload(args.config, args.frames)
    L = _lib.load()
    scfg = stage.StageConfig(patch_size=21, search_radius=cfg.radius, subpixel=True, ref_frames=cfg.ref_frames,
                             segment_length=cfg.segment_length, sigma=3.0)
    strong = args.scaling == "strong"
    if strong:
        # strong scaling: one T-frame recording, frame-balanced shards (distributed.balanced_plan)
        full = synth.generate(cfg, dev)
        shard = distributed.balanced_plan(full.shape[0], cfg.segment_length, world, rank)
        frames = full[shard.local_lo:shard.local_hi].clone()
        del full
        torch.cuda.empty_cache()
        t = shard.frames
        runner = distributed.BalancedShardedPreprocessor(cfg.height, cfg.width, scfg)
    else:
        # weak scaling: rank r owns frames [r*T, (r+1)*T) of an N*T-frame recording
        frames = synth.generate(synth.SynthConfig(**{**cfg.__dict__, "seed": cfg.seed + rank}), dev)
        t = frames.shape[0]
        shard = distributed.shard_plan(t * world, cfg.segment_length, world, rank)
        assert shard.frames == t
        runner = distributed.ShardedPreprocessor(cfg.height, cfg.width, scfg)
    corr = None if args.no_corrected else torch.empty((t, cfg.height, cfg.width), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    def step():
        return runner.run(frames, shard, cfg.ref_frames, corrected_out=corr)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local_dev)
    clocks.start()
    time.sleep(0.3)
    L.vb_prof_enable(1)
    launches0 = _lib.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev0.record()
    for _ in range(args.steps):
        res = step()
    ev1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = _lib.launch_count() - launches0
    ms = np.zeros(5, np.float64)
    cnt = np.zeros(5, np.int64)
    _lib.check(L.vb_prof_collect(ms.ctypes.data, cnt.ctypes.data, 5))
    L.vb_prof_enable(0)
    clk = clocks.stop()
    elapsed = ev0.elapsed_time(ev1)  # ms, K steps
    t_max = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    elapsed = float(t_max.item())
    total_frames = shard.n_total if strong else t * world
    value = total_frames * args.steps / (elapsed / 1e3)

    # sanity: the stage produced finite, non-negative summaries
    vec = res.vectors_numpy()
    ok = bool(np.isfinite(res.temporal.float().cpu().numpy()).all()
              and (res.temporal.numel() == 0 or res.temporal.min().item() >= 0)
              and (np.abs(vec["dx"]) <= cfg.radius).all())

    # ---- roofline of the dominant kernel (ZNCC search), CUDA events on its stream ----
    peaks, peaks_src = measured_peaks()
    pre = runner.ops.pre if strong else runner.pre
    n_patches = pre.plan.n_patches
    bytes_frame, flops_frame = algorithmic_numbers(cfg, n_patches)
    zncc_launches = int(cnt[0])
    zncc_ms = ms[0] / max(zncc_launches, 1)
    frames_per_launch = t * args.steps / max(zncc_launches, 1)
    achieved = flops_frame * frames_per_launch / (zncc_ms / 1e3) / 1e12
    p2 = _lib.C.c_double()
    p1 = _lib.C.c_double()
    _lib.check(L.vb_fp32_peak_probe(_lib.C.byref(p2), _lib.C.byref(p1)))
    fp32_peak = max(p2.value, p1.value)
    step_ms = elapsed / args.steps
    traffic, traffic_src = None, None
    tj = ROOT / "profiles" / "ncu_traffic.json"
    if tj.exists():
        try:
            z = json.loads(tj.read_text())["zncc_group_kernel"]
            traffic = z["dram_bytes_per_frame"] * frames_per_launch
            traffic_src = z["source"] + "; scaled to this run's frames per launch"
        except (ValueError, KeyError):
            pass
    # the search kernel's algorithmic bytes are its input, the u16 frame; the
    # statistics kernel's 1/sqrt(var) per (patch, candidate) (read) and the
    # float64 group partials (written) are this design's intermediates and are
    # reported separately, so traffic / traffic_algorithmic shows their cost
    info = pre.plan.info()
    sdim = 2 * cfg.radius + 1
    frame_bytes = cfg.height * cfg.width * 2
    inter_bytes_frame = 4 * info["patches"] * sdim * sdim + 8 * info["groups"] * sdim * sdim
    kernel_ms_per_step = {n: float(ms[i] / args.steps) for i, n in
                          enumerate(["zncc_group", "finalize", "warp_smooth", "median", "other"])}
    hbm_stage = bytes_frame * total_frames / world / (step_ms / 1e3) / 1e9
    roofline = {
        "bound": "fp32",
        "bound_note": ("neither 'hbm' nor 'tensor': the dominant kernel is bound by the FP32 FMA pipe (ZNCC cross "
                       "sums, SURVEY 8(d)); the whole stage moves a few % of HBM bandwidth (roofline.hbm); a "
                       "per-patch template is an N = 1 product, so tensor cores do not apply"),
        "kernel": ("zncc_group_kernel<21,17,2,split>: half-warp per patch, shared middle row, two frames per "
                   "thread through FFMA2" if cfg.radius == 8 else f"zncc_group_kernel<21,{2 * cfg.radius + 1},1>"),
        "plan": pre.plan.info(),
        "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved / fp32_peak,
        "traffic": traffic,
        "traffic_source": traffic_src,
        "traffic_algorithmic": frame_bytes * frames_per_launch,
        "traffic_algorithmic_def": "per launch: frames x 2*H*W (the u16 frames the search reads)",
        "traffic_intermediates": inter_bytes_frame * frames_per_launch,
        "traffic_intermediates_def": "per launch: frames x (4*N*S^2 inv rows from the statistics kernel + "
                                     "8*groups*S^2 float64 group partials to the finalize kernel)",
        "peak_source": "measured live: FFMA2 (fma.rn.f32x2) probe, vb_fp32_peak_probe",
        "peak_ffma_scalar": p1.value,
        "algorithmic": f"{flops_frame:.4g} flop/frame = 2*N_patch({n_patches})*(2r+1)^2*21^2; "
                       f"{frames_per_launch:.0f} frames/launch; avg launch {zncc_ms:.3f} ms",
        "kernel_share_of_step": float(ms[0] / args.steps / step_ms),
        "kernel_ms_per_step": kernel_ms_per_step,
        "hbm": {"achieved_gbs": hbm_stage, "peak_gbs": peaks.get("hbm_gbs"), "frac": hbm_stage / peaks.get("hbm_gbs", 6552.3),
                "peak_source": peaks_src,
                "algorithmic": f"{bytes_frame:.0f} B/frame = H*W*(2+4) + 8*H*W/L (stage, whole step)"},
    }

    # ---- e2e through the C-ABI host entry point ----
    e2e = None
    if not args.no_e2e and strong:
        # each rank streams its own shard over its own PCIe link: pinned host
        # frames -> HBM in pieces on an upload stream (the motion search of a
        # piece starts as it lands), the sharded stage (template all-reduce,
        # straddling blocks over peer memory), vectors + owned summaries -> pinned host
        host = frames.view(torch.int16).cpu().pin_memory()
        dev_in = torch.empty_like(frames)
        nrec = _lib.MOTION_DTYPE.itemsize * frames.shape[0]
        kb = shard.block_hi - shard.block_lo
        vec_h = torch.empty(nrec, dtype=torch.uint8, pin_memory=True)
        sp_h = torch.empty((max(kb, 1), cfg.height, cfg.width), dtype=torch.float32, pin_memory=True)
        tp_h = torch.empty_like(sp_h)

        up = torch.cuda.Stream(device=dev)
        n_loc = frames.shape[0]
        piece = 500  # frames per upload piece: the motion search of piece k runs while k+1 uploads

        def e2e_step():
            up.wait_stream(torch.cuda.current_stream())  # last step is done with dev_in
            evs = []
            with torch.cuda.stream(up):
                for a in range(0, n_loc, piece):
                    b = min(n_loc, a + piece)
                    dev_in[a:b].view(torch.int16).copy_(host[a:b], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(up)
                    evs.append((a, b, ev))

            def arrival(a, b):
                for x, y, ev in evs:
                    if x < b and y > a:
                        torch.cuda.current_stream().wait_event(ev)

            r = runner.run(dev_in, shard, cfg.ref_frames, corrected_out=corr, arrival=arrival, chunk=piece)
            vec_h.copy_(r.vectors[:nrec], non_blocking=True)
            if kb:
                sp_h[:kb].copy_(r.spatial, non_blocking=True)
                tp_h[:kb].copy_(r.temporal, non_blocking=True)
            torch.cuda.current_stream().synchronize()

        for _ in range(max(args.warmup, 1)):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        et = torch.tensor([time.perf_counter() - w0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        hw = cfg.height * cfg.width
        e2e = {"value": shard.n_total * args.steps / float(et.item()), "unit": UNIT,
               "h2d_bytes_per_step": int(frames.shape[0] * hw * 2), "d2h_bytes_per_step": int(nrec + 2 * kb * hw * 4),
               "path": "per rank: pinned uint16 shard (+ halo) -> HBM in 500-frame pieces overlapped with the "
                       "motion search, sharded stage, vectors + owned summaries -> pinned host; rank 0's bytes; "
                       "max over ranks"}
        del host, dev_in
    elif not args.no_e2e:
        host = frames.view(torch.int16).cpu().pin_memory()
        hs = stage.HostStage(cfg.height, cfg.width, scfg, device=local_dev)
        k = math.ceil(t / cfg.segment_length)
        vec_h = np.empty(t, dtype=_lib.MOTION_DTYPE)
        sp_h = np.empty((k, cfg.height, cfg.width), np.float32)
        tp_h = np.empty((k, cfg.height, cfg.width), np.float32)
        m = cfg.ref_frames

        def e2e_step():
            if world > 1:
                # the recording's template: rank 0 uploads its first M frames, NCCL all-reduce
                ts = torch.zeros((cfg.height, cfg.width), dtype=torch.float64, device=dev)
                if rank == 0:
                    head = host[:m].to(dev, non_blocking=True).view(torch.uint16)
                    _lib.call("vb_template_sum", head.data_ptr(), _lib.VB_U16, m, cfg.height, cfg.width,
                              ts.data_ptr(), 0, D.stream_handle())
                distributed.allreduce_sum_(ts)
                ref = torch.empty((cfg.height, cfg.width), dtype=torch.float32, device=dev)
                _lib.call("vb_template_finish", ts.data_ptr(), m, cfg.height * cfg.width, ref.data_ptr(),
                          D.stream_handle())
                torch.cuda.synchronize()
                _lib.call("vb_stage_set_reference", hs._h, ref.data_ptr())
            hs.run_into(host.data_ptr(), _lib.VB_U16, t, vec_h, sp_h, tp_h, None, corrected_dev=corr)

        for _ in range(max(args.warmup, 1)):
            e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        w1 = time.perf_counter()
        et = torch.tensor([w1 - w0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e_fps = t * world * args.steps / float(et.item())
        # rank 0: the recording (+ the template head uploaded separately for the all-reduce when N > 1;
        # with N = 1 the template is summed in place from the first resident chunk)
        h2d = (t + (m if world > 1 else 0)) * cfg.height * cfg.width * 2
        d2h = t * 32 + 2 * k * cfg.height * cfg.width * 4
        e2e = {"value": e2e_fps, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "path": "vb_stage_run_host (C ABI), pinned uint16 host input, vectors+summaries to host, "
                       "corrected video kept in HBM"}
        hs.close()
        del host

    # ---- e2e through the drop-in Python API, corrected video returned ----
    dropin = None
    if not args.no_dropin and not strong:
        from paper_2403_16438_b200 import Video

        host_np = frames.view(torch.int16).cpu().numpy().view(np.uint16)  # plain (pageable) numpy recording
        hw = cfg.height * cfg.width
        k = math.ceil(t / cfg.segment_length)

        def dropin_step():
            corrected, vectors, pairs = stage.preprocess(Video(host_np), scfg, return_corrected=True)
            assert corrected.data.shape == (t, cfg.height, cfg.width) and len(vectors) == t and len(pairs) == k
            del corrected, vectors, pairs  # the caller drops the step's outputs (the pool block is reused)

        for _ in range(max(args.warmup, 1)):
            dropin_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            dropin_step()
        torch.cuda.synchronize()
        et = torch.tensor([time.perf_counter() - w0], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        dropin = {"value": t * world * args.steps / float(et.item()), "unit": UNIT,
                  "h2d_bytes_per_step": int(t * hw * 2), "d2h_bytes_per_step": int(t * hw * 4 + t * 32 + 2 * k * hw * 4),
                  "path": "stage.preprocess(Video(numpy uint16), StageConfig, return_corrected=True): pageable numpy "
                          "recording in; corrected float32 video (page-locked pool array, direct D2H), "
                          "MotionVector list and SummaryPair list out -- correct_motion + summarize's return values"}
        stage.release_cached()
        del host_np

    # ---- CPU baseline: the reference on this host's cores (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        n = min(args.cpu_sample, t)
        sample = frames[:n].view(torch.int16).cpu().numpy().view(np.uint16).astype(np.float32)
        threads = os.cpu_count() or 1
        try:
            fps_ref, dt, backend = reference_stage_fps(sample, cfg, threads)
            cpu = {"value": fps_ref, "unit": UNIT, "cores": threads, "kind": "reference",
                   "sample": f"first {n} frames of {cfg.name} ({dt:.1f} s): voltseg ({backend} backend) "
                             f"correct_motion(threads={threads}) + summarize(L={cfg.segment_length})"}
        except Exception as exc:  # noqa: BLE001
            fps_ref, dt = oracle_port_fps(sample, cfg, threads)
            cpu = {"value": fps_ref, "unit": UNIT, "cores": threads, "kind": "port",
                   "sample": f"first {n} frames of {cfg.name} ({dt:.1f} s), oracle C port; reference failed: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "impl": "ours", "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32/f64",
            "data": f"synthetic (paper_2403_16438_b200.synth, BASELINE.json configs[1], seed {cfg.seed}"
                    + (")" if strong else "+rank)"),
            "config": {"workload": (f"{cfg.name}: {total_frames}x{cfg.height}x{cfg.width} uint16 recording, frame-balanced "
                                    f"shards" if strong else f"{cfg.name}: {t}x{cfg.height}x{cfg.width} uint16 per rank")
                                   + f", r={cfg.radius}, patch=21, L={cfg.segment_length}, M={cfg.ref_frames}, sigma=3",
                       "per_rank_frames": t,
                       "straddling_blocks": (sum(distributed.balanced_plan(total_frames, cfg.segment_length, world, q)
                                                 .tail is not None for q in range(world)) if strong else 0),
                       "parallelism": (f"frame-balanced time shards x{world} (template all-reduce; straddling blocks: "
                                       f"smoothed frames + float64 running sum written into the owner's HBM over "
                                       f"peer memory)") if strong
                       else f"time-sharded x{world} (template all-reduce)",
                       "corrected_video": "written to HBM" if corr is not None else "not materialised",
                       "l2": "inputs (%.1f GB u16) larger than L2 (126 MB); no flush" % (t * cfg.height * cfg.width * 2 / 1e9)},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_dropin": dropin,
            "gpu_launches": int(launches),
            "clocks": clk,
            "outputs_sane": ok,
        }
        print(json.dumps(line), flush=True)
    runner.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def unet_flops_per_patch() -> float:
    """2 * MACs of the canonical U-Net on one 64x64 patch (unet.py:34-54, :154-178)."""
    from paper_2403_16438_b200 import unet

    side = {"enc1": 64, "enc2": 32, "enc3": 16, "dec2": 32, "dec1": 64, "out": 64}
    total = 0.0
    for name, shape in unet.architecture():
        if name.endswith(".kernel"):
            cout, cin, k, _ = shape
            total += 2.0 * cout * cin * k * k * side[name.split(".")[0]] ** 2
    return total


def run_unet(args):
    """Segmentation consumer on C2: all K blocks' summary pairs -> probability maps."""
    import torch

    from paper_2403_16438_b200 import _lib, stage, synth, unet
    from paper_2403_16438_b200.unet import _tile_count

    rank, world, local = dist_env()
    if rank != 0:
        return 0
    cfg = workload(args.config, args.frames)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    frames = synth.generate(cfg, dev)
    scfg = stage.StageConfig(search_radius=cfg.radius, segment_length=cfg.segment_length, ref_frames=cfg.ref_frames)
    pre = stage.DevicePreprocessor(cfg.height, cfg.width, scfg)
    res = pre.run(frames)
    sp, tp = res.spatial.contiguous(), res.temporal.contiguous()
    del frames
    k = sp.shape[0]
    weights = unet.WeightBundle.random(np.random.default_rng(7))
    net = unet.DeviceUNet(weights)
    prob = torch.empty_like(sp)
    tiles = _tile_count(cfg.height, cfg.width, unet.DEFAULT_STRIDE)
    for _ in range(max(args.warmup, 3)):
        net.segment_device(sp, tp, out=prob)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.3)
    launches0 = _lib.launch_count()
    ev0.record()
    for _ in range(args.steps):
        net.segment_device(sp, tp, out=prob)
    ev1.record()
    torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    clk = clocks.stop()
    ms = ev0.elapsed_time(ev1) / args.steps
    flops = unet_flops_per_patch() * k * tiles
    p2, p1 = _lib.C.c_double(), _lib.C.c_double()
    _lib.check(_lib.load().vb_fp32_peak_probe(_lib.C.byref(p2), _lib.C.byref(p1)))
    peak = max(p2.value, p1.value)
    # dense TF32 tensor-core peak: half the measured dense BF16 rate (the tcgen05 kind::tf32 rate on B200)
    peaks, psrc = measured_peaks()
    tf32_peak = peaks.get("bf16_tflops", 2250.0) / 2.0
    tf32_src = f"{psrc}: bf16_tflops / 2 (kind::tf32 issues at half the kind::f16 rate)"
    cpu = None
    if not args.no_cpu_baseline:
        try:
            from oracle import ref
            ref.load()
            import voltseg.unet as R
            spn, tpn = sp[0].cpu().numpy(), tp[0].cpu().numpy()
            t0 = time.perf_counter()
            R.tile_and_merge(weights_ref := R.WeightBundle.random(np.random.default_rng(7)), R.normalize_pair(spn, tpn))
            dt = time.perf_counter() - t0
            cpu = {"value": 1.0 / dt, "unit": "summary pairs/s", "cores": os.cpu_count(), "kind": "reference",
                   "sample": "one C2 summary pair: voltseg normalize_pair + tile_and_merge (numpy BLAS)"}
            del weights_ref
        except Exception as exc:  # noqa: BLE001
            cpu = {"unavailable": str(exc)}
    line = {
        "metric": "summary pairs/s through normalize_pair + U-Net tile_and_merge (SURVEY 8(f) row 2)",
        "value": k / (ms / 1e3), "unit": "summary pairs/s", "n_gpus": 1, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True, "scaling": "none",
        "vs_baseline": None, "dtype": "f32", "data": "summary pairs of the synthetic C2 recording; random weights",
        "config": {"workload": f"{cfg.name}: {k} blocks of {cfg.height}x{cfg.width}, {tiles} tiles/block, stride 32",
                   "patches_per_step": k * tiles},
        "roofline": {"bound": "tensor", "achieved": 3 * flops / (ms / 1e3) / 1e12, "peak": tf32_peak,
                     "unit": "TFLOP/s", "frac": 3 * flops / (ms / 1e3) / 1e12 / tf32_peak,
                     "peak_source": tf32_src,
                     "algorithmic": f"3 x {unet_flops_per_patch():.4g} flop/patch (3xTF32 split on tcgen05) x "
                                    f"{k * tiles} patches per step",
                     "fp32_equivalent": {"achieved": flops / (ms / 1e3) / 1e12, "peak_fp32_simt": peak}},
        "cpu_baseline": cpu, "gpu_launches": int(launches), "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    net.close()
    pre.close()
    return 0


def run_pipeline(args):
    """pipeline.py:190-258 without footprints, end to end through the C ABI:
    pinned uint16 host recording -> vectors, summaries and probability maps on
    the host (vb_stage_run_host_segment), against the stage alone."""
    import torch

    from paper_2403_16438_b200 import _lib, stage, synth, unet

    rank, world, local = dist_env()
    if rank != 0:
        return 0
    cfg = workload(args.config, args.frames)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    host = synth.generate(cfg, dev).view(torch.int16).cpu().pin_memory()
    t = host.shape[0]
    scfg = stage.StageConfig(search_radius=cfg.radius, segment_length=cfg.segment_length, ref_frames=cfg.ref_frames)
    hs = stage.HostStage(cfg.height, cfg.width, scfg)
    net = unet.DeviceUNet(unet.WeightBundle.random(np.random.default_rng(7)))
    hs.attach_unet(net)
    k = math.ceil(t / cfg.segment_length)
    vec = np.empty(t, dtype=_lib.MOTION_DTYPE)
    sp = np.empty((k, cfg.height, cfg.width), np.float32)
    tp, prob = np.empty_like(sp), np.empty_like(sp)

    def seg_step():
        _lib.call("vb_stage_run_host_segment", hs._h, host.data_ptr(), _lib.VB_U16, t, vec.ctypes.data,
                  sp.ctypes.data, tp.ctypes.data, prob.ctypes.data, None, None)

    def stage_step():
        hs.run_into(host.data_ptr(), _lib.VB_U16, t, vec, sp, tp)

    out = {}
    for name, fn in (("pipeline", seg_step), ("stage_only", stage_step)):
        for _ in range(max(args.warmup, 1)):
            fn()
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        for _ in range(args.steps):
            fn()
        torch.cuda.synchronize()
        out[name] = t * args.steps / (time.perf_counter() - w0)
    line = {
        "metric": "frames/s through motion correction + summaries + U-Net segmentation (pipeline.py:190-258 "
                  "minus footprints), host in / host out",
        "value": out["pipeline"], "unit": "frames/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "higher_is_better": True, "scaling": "none", "vs_baseline": None, "dtype": "f32/f64",
        "data": "synthetic C2 recording (paper_2403_16438_b200.synth); random U-Net weights",
        "config": {"workload": f"{cfg.name}: {t}x{cfg.height}x{cfg.width} uint16, L={cfg.segment_length}, "
                               f"{k} blocks segmented", "path": "vb_stage_run_host_segment (C ABI), pinned input"},
        "stage_only_fps": out["stage_only"],
        "e2e": {"value": out["pipeline"], "unit": "frames/s", "h2d_bytes_per_step": int(t * cfg.height * cfg.width * 2),
                "d2h_bytes_per_step": int(t * 32 + 3 * k * cfg.height * cfg.width * 4)},
    }
    print(json.dumps(line), flush=True)
    hs.close()
    net.close()
    return 0


def main():
    args = parse()
    rc = relaunch_under_torchrun(args)
    if rc is not None:
        return rc
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.scaling is None:
        args.scaling = "strong" if world > 1 else "weak"
    if args.stage == "unet":
        return run_unet(args)
    if args.stage == "pipeline":
        return run_pipeline(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
