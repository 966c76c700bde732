"""The operator-level drop-in inside the reference's OWN code: our
kernels.mean_zncc_scores takes the place of the compiled `_native` extension
behind voltseg.kernels' dispatcher (kernels.py:98-108 calls
`_native.mean_zncc_scores` when BACKEND == "native"), driving the unmodified
reference correct_motion (oracle/_ref, test infrastructure)."""
import types

import numpy as np
import pytest

from oracle import ref as REF
from paper_2403_16438_b200 import kernels as K, synth

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not REF.available(), reason="reference not built (oracle/build_ref.sh)")
def test_reference_correct_motion_with_b200_backend(cuda):
    motion, _summarize, kernels, video_io = REF.load()
    cfg = synth.CONFIGS["c1"].with_frames(60)
    raw = synth.generate_numpy(cfg).astype(np.float32)
    video = video_io.Video(raw, frame_rate=cfg.fps)
    old_backend, old_m, old_native = kernels.BACKEND, motion.REFERENCE_FRAMES, kernels._native
    calls = []

    def b200(*args):
        calls.append(1)
        return K.mean_zncc_scores(*args)

    try:
        motion.REFERENCE_FRAMES = 20
        runs = {}
        for name in ("b200", "python"):
            if name == "b200":  # the compiled operator replaced by ours (same signature)
                kernels._native, kernels.BACKEND = types.SimpleNamespace(mean_zncc_scores=b200), "native"
            else:
                kernels._native, kernels.BACKEND = old_native, "python"
            corrected, vecs = motion.correct_motion(video, motion.MotionConfig(search_radius=cfg.radius, threads=4))
            runs[name] = (corrected.data, vecs)
    finally:
        kernels.BACKEND, motion.REFERENCE_FRAMES, kernels._native = old_backend, old_m, old_native
    assert len(calls) == raw.shape[0]  # every frame's score grid came from the B200 operator
    (c_b, v_b), (c_p, v_p) = runs["b200"], runs["python"]
    np.testing.assert_array_equal([[v.dx, v.dy] for v in v_b], [[v.dx, v.dy] for v in v_p])
    np.testing.assert_allclose([[v.sub_dx, v.sub_dy] for v in v_b], [[v.sub_dx, v.sub_dy] for v in v_p], atol=1e-3)
    np.testing.assert_allclose([v.confidence for v in v_b], [v.confidence for v in v_p], atol=1e-6)
    rel = np.abs(c_b - c_p) / np.maximum(np.abs(c_p), 1.0)
    assert rel.max() <= 1e-4


@pytest.mark.slow
@pytest.mark.skipif(not REF.available(), reason="reference not built (oracle/build_ref.sh)")
def test_reference_correct_motion_throughput_with_b200_backend(cuda):
    """Timing record (profiles/r01_operator_dropin.json): the reference's own
    correct_motion on 400 C2 frames with its compiled operator and with ours,
    1 and all host threads; written to gpurun_out/ when run on the GPU box."""
    import json
    import os
    import time
    from pathlib import Path

    motion, _s, kernels, video_io = REF.load()
    cfg = synth.CONFIGS["c2"].with_frames(400)
    video = video_io.Video(synth.generate_numpy(cfg).astype(np.float32), frame_rate=cfg.fps)
    old = (kernels.BACKEND, motion.REFERENCE_FRAMES, kernels._native)
    threads = os.cpu_count() or 1
    out = {"config": f"c2 400x{cfg.height}x{cfg.width}, r={cfg.radius}: reference correct_motion"}
    try:
        motion.REFERENCE_FRAMES = cfg.ref_frames
        kernels.BACKEND = "native"
        ours = types.SimpleNamespace(mean_zncc_scores=K.mean_zncc_scores)
        for name, thr in (("b200", 1), ("b200", threads), ("native", 1), ("native", threads)):
            kernels._native = ours if name == "b200" else old[2]
            t0 = time.perf_counter()
            motion.correct_motion(video, motion.MotionConfig(search_radius=cfg.radius, threads=thr))
            out[f"{name}_threads{thr}_frames_per_s"] = 400 / (time.perf_counter() - t0)
    finally:
        kernels.BACKEND, motion.REFERENCE_FRAMES, kernels._native = old
    if Path("gpurun_out").is_dir():
        Path("gpurun_out/operator_dropin.json").write_text(json.dumps(out))
    assert out["b200_threads1_frames_per_s"] > out["native_threads1_frames_per_s"]
