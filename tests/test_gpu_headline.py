"""Parity at the headline configurations, every frame.

* C2 exactly as bench.py times it (10,000 x 256 x 512 uint16, seed 1002,
  r = 8, L = 1,000, M = 100, generated on the GPU by the same call): the CUDA
  stage (DevicePreprocessor, the bench's `value` path) against the float64 C
  oracle's OWN pipeline (oracle template -> oracle motion -> oracle warp ->
  oracle summaries), on all 10,000 frames and all 10 blocks:
    - integer shifts (dx, dy) bit-exact on every frame;
    - sub-pixel shifts within 1e-3 px;
    - corrected frames within 1e-4 relative (|a - b| / max(|b|, 1));
    - spatial summaries within 1e-4 relative; temporal summaries (max - median
      of ~1000-count frames, themselves a few counts) within 1e-4 of the
      block's spatial scale.
* Against the reference's DEFAULT backend (its compiled `_native` kernel,
  `oracle/_ref`) on every frame: the native kernel forms its cross sums in
  float32 (`-ffast-math`, _native_impl.h:18-35) and disagrees with the
  reference's own float64 backend on a few percent of C2 frames.  Required:
  every frame where the GPU's integer shift differs from native is a frame
  where native also differs from float64, and on each such frame native's
  score grid is within its float32 noise (<= 1e-3) of the float64 grid --
  the flip is native rounding at a near-tie, not a GPU error.  Reported:
  the float64 top-2 margin at those frames vs over all frames.
* C3 / C4 / C5 geometries: the same checks on two full 1,000-frame blocks.

Each configuration's table (GPU / native / float64 pairwise counts, maxima)
is written to gpurun_out/r02_parity_<cfg>.json (copied to profiles/).
"""
import json
import os
import time
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2403_16438_b200 import synth
from paper_2403_16438_b200.stage import DevicePreprocessor, StageConfig

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
THREADS = os.cpu_count() or 1


def _native_vectors(raw: np.ndarray, ref: np.ndarray, radius: int):
    """The reference's own estimate_motion with its default (native) backend,
    frames fanned over threads as its correct_motion does (motion.py:229-231)."""
    from oracle import ref as R

    motion, _s, kernels, _v = R.load("native")
    assert kernels.BACKEND == "native" and kernels.HAVE_NATIVE
    grid = motion.PatchGrid.cover(raw.shape[1], raw.shape[2], 21, margin=radius)

    def one(t):
        v = motion.estimate_motion(raw[t].astype(np.float32), ref, grid, search_radius=radius, subpixel=True)
        return v.dx, v.dy

    with ThreadPoolExecutor(THREADS) as ex:
        return np.array(list(ex.map(one, range(raw.shape[0]), chunksize=64)), dtype=np.int32)


def _check(name: str, frames: int, native: bool):
    from oracle import oracle as O

    cfg = synth.CONFIGS[name].with_frames(frames)
    r, L, M = cfg.radius, cfg.segment_length, cfg.ref_frames
    dev = torch.device("cuda", 0)
    t0 = time.time()
    frames_dev = synth.generate(cfg, dev)  # bench.py's call (seed cfg.seed at rank 0)
    pre = DevicePreprocessor(cfg.height, cfg.width, StageConfig(search_radius=r, segment_length=L, ref_frames=M))
    corr_dev = torch.empty(frames_dev.shape, dtype=torch.float32, device=dev)
    res = pre.run(frames_dev, corrected_out=corr_dev)
    rec = res.vectors_numpy()
    g_sp, g_tp = res.spatial.cpu().numpy(), res.temporal.cpu().numpy()
    pre.close()
    raw = frames_dev.view(torch.int16).cpu().numpy().view(np.uint16)
    del frames_dev
    g_dxdy = np.stack([rec["dx"], rec["dy"]], axis=1)
    g_sub = np.stack([rec["sub_dx"], rec["sub_dy"]], axis=1)

    ref = O.make_reference(raw[:M].astype(np.float32), M)
    origins = O.patch_grid(cfg.height, cfg.width, 21, r)
    tab = dict(config=name, frames=frames, height=cfg.height, width=cfg.width, radius=r, segment_length=L,
               ref_frames=M, seed=cfg.seed, patches=int(len(origins)), host_threads=THREADS,
               gpu_vs_f64_int_mismatch=0, max_subpixel_diff_px=0.0, max_corrected_rel=0.0,
               max_spatial_rel=0.0, max_temporal_abs_over_scale=0.0, max_confidence_diff=0.0, blocks=[])
    o_dxdy_all = np.empty_like(g_dxdy)
    top2 = np.empty(frames)  # float64 top-2 score margin per frame
    for b0 in range(0, frames, L):
        b1 = min(frames, b0 + L)
        m = O.motion_frames(raw[b0:b1].astype(np.float32), ref, origins, 21, r, threads=THREADS, want_scores=True)
        o_dxdy_all[b0:b1] = m["dxdy"]
        flat = np.sort(m["scores"].reshape(b1 - b0, -1), axis=1)
        top2[b0:b1] = flat[:, -1] - flat[:, -2]
        bad = np.nonzero((m["dxdy"] != g_dxdy[b0:b1]).any(axis=1))[0]
        sub = float(np.abs(m["sub_conf"][:, :2] - g_sub[b0:b1]).max())
        conf = float(np.abs(m["sub_conf"][:, 2] - rec["confidence"][b0:b1]).max())
        gc = corr_dev[b0:b1].cpu().numpy()
        crel = float((np.abs(gc - m["corrected"]) / np.maximum(np.abs(m["corrected"]), 1.0)).max())
        del gc
        sp, tp = O.summaries(m["corrected"], L, 3.0, threads=THREADS)
        k = b0 // L
        srel = float((np.abs(g_sp[k] - sp[0]) / np.maximum(np.abs(sp[0]), 1.0)).max())
        tabs = float(np.abs(g_tp[k] - tp[0]).max() / np.abs(sp[0]).max())
        tab["blocks"].append(dict(block=k, int_mismatch=[int(b0 + i) for i in bad], max_subpixel_diff_px=sub,
                                  max_corrected_rel=crel, max_spatial_rel=srel, max_temporal_abs_over_scale=tabs))
        tab["gpu_vs_f64_int_mismatch"] += int(len(bad))
        tab["max_subpixel_diff_px"] = max(tab["max_subpixel_diff_px"], sub)
        tab["max_confidence_diff"] = max(tab["max_confidence_diff"], conf)
        tab["max_corrected_rel"] = max(tab["max_corrected_rel"], crel)
        tab["max_spatial_rel"] = max(tab["max_spatial_rel"], srel)
        tab["max_temporal_abs_over_scale"] = max(tab["max_temporal_abs_over_scale"], tabs)
        del m
    del corr_dev
    torch.cuda.empty_cache()

    failures = []
    if native:
        from oracle import ref as R

        _m, _s, kernels, _v = R.load("native")
        n_dxdy = _native_vectors(raw, ref, r)
        nat_vs_gpu = np.nonzero((n_dxdy != g_dxdy).any(axis=1))[0]
        nat_vs_f64 = set(np.nonzero((n_dxdy != o_dxdy_all).any(axis=1))[0].tolist())
        rows = []
        for t in nat_vs_gpu:
            f32 = raw[t].astype(np.float32)
            s64 = O.mean_zncc_scores(f32, ref, origins, 21, r)
            snat = kernels.mean_zncc_scores(f32, ref, origins, 21, r)
            gi, ni = (g_dxdy[t][1] + r, g_dxdy[t][0] + r), (n_dxdy[t][1] + r, n_dxdy[t][0] + r)
            margin = float(s64[gi] - s64[ni])
            nerr = float(np.abs(snat - s64).max())
            explained = int(t) in nat_vs_f64 and nerr <= 1e-3 and 0.0 <= margin <= 2 * nerr
            rows.append(dict(frame=int(t), gpu=g_dxdy[t].tolist(), native=n_dxdy[t].tolist(),
                             f64=o_dxdy_all[t].tolist(), f64_margin=margin, native_grid_err=nerr,
                             native_rounding_flip=explained))
            if not explained:
                failures.append(f"frame {t}: gpu {g_dxdy[t]} native {n_dxdy[t]} f64 margin {margin:.3g} "
                                f"native err {nerr:.3g}")
        mm = np.array([row["f64_margin"] for row in rows]) if rows else np.zeros(1)
        tab["native"] = dict(
            backend="reference voltseg._native (oracle/_ref), estimate_motion, default flags",
            frames_compared=int(frames), gpu_vs_native_int_mismatch=int(len(nat_vs_gpu)),
            native_vs_f64_int_mismatch=int(len(nat_vs_f64)),
            gpu_vs_f64_int_mismatch=tab["gpu_vs_f64_int_mismatch"],
            mismatch_f64_margin_max=float(mm.max()),
            mismatch_native_grid_err_max=float(max([row["native_grid_err"] for row in rows], default=0.0)),
            all_frames_f64_top2_margin_quantiles={q: float(np.quantile(top2, q)) for q in (0.01, 0.05, 0.5)},
            frames_with_top2_margin_below_mismatch_max=int((top2 <= mm.max()).sum()),
            mismatches=rows)
    tab["wall_s"] = round(time.time() - t0, 1)
    OUT.mkdir(exist_ok=True)
    (OUT / f"r02_parity_{name}.json").write_text(json.dumps(tab, indent=1))

    assert tab["gpu_vs_f64_int_mismatch"] == 0, [b["int_mismatch"] for b in tab["blocks"]]
    assert tab["max_subpixel_diff_px"] <= 1e-3
    assert tab["max_corrected_rel"] <= 1e-4
    assert tab["max_spatial_rel"] <= 1e-4
    assert tab["max_temporal_abs_over_scale"] <= 1e-4
    assert not failures, failures


def test_c2_headline_every_frame(cuda):
    _check("c2", 10000, native=True)


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_large_configs_two_blocks(cuda, name):
    _check(name, 2000, native=True)


def test_motion_recovery_acceptance(cuda):
    """pkg/tests/test_acceptance.py:130-149 on the CUDA path: 20 seeded videos
    of the reference's own simulator (oracle/_ref voltseg.simulate), motion
    recovered by this package's correct_motion; >= 95 % exact integer shifts
    and every residual <= 1 px."""
    from oracle import ref as R

    from paper_2403_16438_b200 import Video
    from paper_2403_16438_b200.motion import MotionConfig, correct_motion

    R.load()
    from voltseg.simulate import SceneConfig, synthesize

    exact = total = 0
    worst = 0.0
    for seed in range(20):
        video, gt = synthesize(SceneConfig(frames=1000, motion_amplitude=5, noise_level=0.10, seed=300 + seed))
        _, vectors = correct_motion(Video(video.data), MotionConfig(search_radius=5))
        for t, v in enumerate(vectors):
            dx, dy = gt.motion[t]
            exact += int(v.dx == dx and v.dy == dy)
            total += 1
            residual = max(abs(v.x - dx), abs(v.y - dy))
            worst = max(worst, residual)
            assert residual <= 1.0, f"seed {seed} frame {t}: residual {residual}"
    OUT.mkdir(exist_ok=True)
    (OUT / "r02_acceptance_motion_recovery.json").write_text(
        json.dumps(dict(videos=20, frames=total, exact_frac=exact / total, worst_residual_px=worst)))
    assert exact / total >= 0.95
