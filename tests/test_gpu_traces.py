"""Trace extraction on the GPU vs the reference (golden)
and the oracle; the reference's own traces tests restated."""
import numpy as np
import pytest
import torch

from paper_2403_16438_b200 import Video, synth, traces
from paper_2403_16438_b200.stage import DevicePreprocessor, StageConfig

pytestmark = pytest.mark.gpu


def test_golden_traces_and_dff(cuda, golden):
    z = golden("traces")
    video = Video(z["video"], frame_rate=741.0)
    trs = traces.extract_all(video, [z[f"mask{k}"] for k in range(5)])
    for k, tr in enumerate(trs):
        assert tr.footprint_id == k and tr.frame_rate == 741.0
        np.testing.assert_allclose(tr.samples, z[f"trace{k}"], rtol=1e-12)
        np.testing.assert_allclose(traces.dff(tr).samples, z[f"dff{k}"], rtol=1e-9, atol=1e-12)


def test_single_and_errors(cuda, rng):
    v = Video(rng.random((30, 24, 26), dtype=np.float32))
    mask = rng.random((24, 26)) > 0.5
    tr = traces.extract_trace(v, mask, 3)
    brute = np.array([v.data[t][mask].astype(np.float64).mean() for t in range(30)])
    np.testing.assert_allclose(tr.samples, brute, rtol=1e-12)  # test_acceptance.py:120-126 (1e-6)
    with pytest.raises(ValueError, match="does not match"):
        traces.extract_trace(v, np.ones((5, 5), bool))
    with pytest.raises(ValueError, match="empty ROI"):
        traces.extract_trace(v, np.zeros((24, 26), bool))
    with pytest.raises(ValueError, match="zero baseline"):
        traces.dff(traces.Trace(0, np.zeros(10)))


def test_traces_from_device_preprocessor(cuda, oracle_mod):
    """Traces straight from the HBM-resident corrected video of the fused stage."""
    cfg = synth.CONFIGS["c1"].with_frames(200)
    raw, truth = synth.generate_numpy(cfg, return_truth=True)
    pre = DevicePreprocessor(cfg.height, cfg.width, StageConfig(search_radius=cfg.radius, segment_length=100,
                                                                 ref_frames=cfg.ref_frames))
    frames = torch.from_numpy(raw.view(np.int16)).to(cuda).view(torch.uint16)
    corr = torch.empty(frames.shape, dtype=torch.float32, device=cuda)
    pre.run(frames, corrected_out=corr)
    yy, xx = np.mgrid[:cfg.height, :cfg.width]
    masks = [((yy - cy) ** 2 + (xx - cx) ** 2) <= 16 for cx, cy in truth.centers]
    got = traces.extract_traces_device(corr, masks).cpu().numpy()
    c = corr.cpu().numpy()
    for k, m in enumerate(masks):
        np.testing.assert_allclose(got[k], oracle_mod.extract_trace(c, m), rtol=1e-12)
    pre.close()


def test_csv(cuda, tmp_path):
    trs = [traces.Trace(0, np.array([1.0, 2.0]), 500.0), traces.Trace(1, np.array([3.0, 4.5]), 500.0)]
    traces.save_traces_csv(trs, tmp_path / "t.csv")
    assert (tmp_path / "t.csv").read_text().splitlines()[1] == "0,1.000000,3.000000"
    assert "500.0" in (tmp_path / "t.json").read_text()


@pytest.mark.parametrize("as_u16", [True, False])
@pytest.mark.parametrize("shading", [0.0, 12.0])
def test_traces_from_raw_frames_equal_corrected(cuda, as_u16, shading):
    """vb_extract_traces_raw (warp fused into the trace, no corrected video)
    == vb_extract_traces on the corrected frames, bit for bit."""
    from paper_2403_16438_b200 import motion as M
    cfg = synth.CONFIGS["c1"].with_frames(160)
    raw, truth = synth.generate_numpy(cfg, return_truth=True)
    frames = (torch.from_numpy(raw.view(np.int16)).to(cuda).view(torch.uint16) if as_u16
              else torch.from_numpy(raw.astype(np.float32)).to(cuda))
    grid = M.PatchGrid.cover(cfg.height, cfg.width, 21, margin=cfg.radius)
    ref = M.device_reference(frames, 50)
    plan = M.MotionPlan(cfg.height, cfg.width, grid.origins, 21, cfg.radius)
    plan.set_reference(ref)
    vec, _ = plan.estimate(frames, True)
    gain = M.shading_gain_device(ref, shading) if shading > 0 else None
    corr = M.correct_frames_device(frames, vec, gain)
    yy, xx = np.mgrid[:cfg.height, :cfg.width]
    masks = [((yy - cy) ** 2 + (xx - cx) ** 2) <= 16 for cx, cy in truth.centers]
    masks.append(np.ones((cfg.height, cfg.width), bool))  # whole frame: edge clamping included
    want = traces.extract_traces_device(corr, masks).cpu().numpy()
    got = traces.extract_traces_raw_device(frames, vec, masks, gain).cpu().numpy()
    np.testing.assert_array_equal(got, want)
    plan.close()
