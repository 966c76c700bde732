"""Pipeline orchestration on the GPU: the C-ABI executor
with the U-Net attached (vb_stage_run_host_segment: per-chunk segmentation
on its own stream) against (a) the reference's own pipeline hot path
(tests/golden/pipeline.npz: correct_motion -> summarize_segment ->
normalize_pair -> tile_and_merge) and (b) the separate device calls."""
from pathlib import Path

import numpy as np
import pytest

from paper_2403_16438_b200 import pipeline, unet
from paper_2403_16438_b200.stage import DevicePreprocessor, HostStage, StageConfig

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden" / "pipeline.npz"


@pytest.fixture(scope="module")
def golden():
    return np.load(G)


def test_motion_and_segment_matches_reference_pipeline(cuda, golden):
    w = unet.WeightBundle.random(np.random.default_rng(7))
    res = pipeline.run_motion_and_segment(golden["raw"], w, search_radius=int(golden["radius"]),
                                          segment_length=int(golden["L"]), ref_frames=int(golden["M"]),
                                          chunk_frames=60)
    dxdy = np.array([[v.dx, v.dy] for v in res.vectors], np.int32)
    np.testing.assert_array_equal(dxdy, golden["dxdy"])
    assert len(res.probability_maps) == golden["prob"].shape[0]
    for i, pm in enumerate(res.probability_maps):
        assert pm.segment_index == i
        np.testing.assert_allclose(res.pairs[i].spatial, golden["spatial"][i], rtol=1e-4, atol=1e-3)
        assert np.abs(pm.values - golden["prob"][i]).max() <= 1e-4
    rep = res.throughput  # pipeline.py:171-172
    assert rep.frames == golden["raw"].shape[0] and rep.total_seconds >= 1e-3
    assert rep.effective_fps == pytest.approx(rep.frames / rep.total_seconds)


@pytest.mark.parametrize("chunk", [60, 120, 0])
def test_executor_segment_equals_device_calls(cuda, golden, chunk):
    raw = golden["raw"]
    L = int(golden["L"])
    cfg = StageConfig(search_radius=int(golden["radius"]), segment_length=L, ref_frames=int(golden["M"]))
    w = unet.WeightBundle.random(np.random.default_rng(7))
    hs = HostStage(raw.shape[1], raw.shape[2], cfg, chunk_frames=chunk)
    hs.attach_unet(w)
    vec, sp, tp, prob, _ = hs.run_segment(raw)
    vec2, sp2, tp2, _ = hs.run(raw)  # the plain executor on the same handle
    hs.close()
    np.testing.assert_array_equal(sp, sp2)
    np.testing.assert_array_equal(tp, tp2)
    from paper_2403_16438_b200.summarize import SummaryPair
    maps = unet.segment_pairs(w, [SummaryPair(i, sp[i], tp[i]) for i in range(sp.shape[0])])
    for i, m in enumerate(maps):
        np.testing.assert_array_equal(prob[i], m.values)


def test_segment_without_unet_raises(cuda, golden):
    raw = golden["raw"][:60]
    hs = HostStage(raw.shape[1], raw.shape[2], StageConfig(search_radius=5, segment_length=30, ref_frames=20))
    with pytest.raises(ValueError, match="no U-Net attached"):
        hs.run_segment(raw)
    hs.close()
