"""Motion stage on the GPU: the reference's test_motion.py cases against the
CUDA path, plus parity with the oracle / reference on camera-like video
(integer shifts bit-exact, sub-pixel <= 1e-3 px, corrected <= 1e-4 rel)."""
import hashlib

import numpy as np
import pytest
import torch
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2403_16438_b200 import Video, motion, synth
from paper_2403_16438_b200.motion import (MotionConfig, PatchGrid, correct_motion, estimate_motion,
                                          make_reference, translate)

pytestmark = pytest.mark.gpu


def _shift_with_padding(image, dx, dy, pad):
    h, w = image.shape[0] - 2 * pad, image.shape[1] - 2 * pad
    return image[pad - dy:pad - dy + h, pad - dx:pad - dx + w]


class TestEstimateMotion:  # test_motion.py:116-175
    def test_identity(self, cuda, rng):
        frame = rng.random((96, 96), dtype=np.float32)
        v = estimate_motion(frame, frame, PatchGrid.cover(96, 96, 21, margin=5), search_radius=5)
        assert (v.dx, v.dy) == (0, 0) and v.confidence == pytest.approx(1.0, abs=1e-5)

    @pytest.mark.parametrize("shift", [(3, -2), (-5, 5), (0, 4), (1, 0)])
    def test_constructed_shift_recovered(self, cuda, rng, shift):
        big = rng.random((120, 120), dtype=np.float32)
        ref = big[12:108, 12:108]
        frame = _shift_with_padding(big, *shift, 12)
        v = estimate_motion(frame, ref, PatchGrid.cover(96, 96, 21, margin=5), search_radius=5)
        assert (v.dx, v.dy) == shift and v.confidence > 0.99

    def test_shift_with_noise_monte_carlo(self, cuda):
        hits = 0
        for trial in range(100):
            r = np.random.default_rng(5000 + trial)
            big = r.random((120, 120), dtype=np.float32)
            frame = _shift_with_padding(big, 3, -2, 12).copy()
            frame = np.clip(frame + r.standard_normal(frame.shape).astype(np.float32) * 0.1, 0, None)
            v = estimate_motion(frame, big[12:108, 12:108], PatchGrid.cover(96, 96, 21, margin=5), search_radius=5)
            hits += (v.dx, v.dy) == (3, -2)
        assert hits >= 95

    def test_tie_break_prefers_origin(self, cuda):
        frame = np.full((96, 96), 5.0, dtype=np.float32)
        v = estimate_motion(frame, frame, PatchGrid.cover(96, 96, 21, margin=5), search_radius=3)
        assert (v.dx, v.dy) == (0, 0)

    def test_invalid_radius(self, cuda, rng):
        frame = rng.random((96, 96), dtype=np.float32)
        with pytest.raises(ValueError, match="search_radius"):
            estimate_motion(frame, frame, PatchGrid.cover(96, 96, 21, margin=5), search_radius=0)

    def test_subpixel_within_unit_interval(self, cuda, rng):
        frame = rng.random((96, 96), dtype=np.float32)
        v = estimate_motion(frame, frame, PatchGrid.cover(96, 96, 21, margin=5), search_radius=5)
        assert abs(v.sub_dx) < 1 and abs(v.sub_dy) < 1


class TestTranslate:  # test_motion.py:178-206
    def test_integer_shift_matches_index_arithmetic(self, cuda, rng):
        frame = rng.random((20, 24), dtype=np.float32)
        for dx, dy in [(2, -3), (-1, 1), (0, 0), (5, 5), (-25, 2), (2, 30)]:
            ys = np.clip(np.arange(20) - dy, 0, 19)
            xs = np.clip(np.arange(24) - dx, 0, 23)
            np.testing.assert_array_equal(translate(frame, dx, dy), frame[np.ix_(ys, xs)])

    def test_fractional_shift_is_bilinear(self, cuda, rng):
        frame = rng.random((16, 16), dtype=np.float32)
        out = translate(frame, 0.25, 0.0)
        np.testing.assert_allclose(out[:, 1:], 0.75 * frame[:, 1:] + 0.25 * frame[:, :-1], atol=1e-6)

    def test_round_trip_interior(self, cuda, rng):
        frame = rng.random((32, 32), dtype=np.float32)
        back = translate(translate(frame, 3, -2), -3, 2)
        np.testing.assert_array_equal(back[5:27, 5:27], frame[5:27, 5:27])

    @given(dx=st.integers(-6, 6), dy=st.integers(-6, 6), seed=st.integers(0, 2 ** 16))
    @settings(max_examples=25, deadline=None)
    def test_integer_shift_preserves_value_set(self, cuda, dx, dy, seed):
        frame = np.random.default_rng(seed).random((16, 16), dtype=np.float32)
        assert np.isin(translate(frame, dx, dy), frame).all()

    def test_golden_bit_exact(self, cuda, golden):
        z = golden("translate")
        for (dx, dy), want in zip(z["shifts"], z["out"]):
            np.testing.assert_array_equal(translate(z["frame"], dx, dy), want)

    @given(dx=st.floats(-12, 12), dy=st.floats(-12, 12))
    @settings(max_examples=40, deadline=None)
    def test_random_shift_bit_exact_vs_oracle(self, cuda, oracle_mod, dx, dy):
        frame = (np.random.default_rng(3).random((33, 47), dtype=np.float32) * 4000).astype(np.float32)
        np.testing.assert_array_equal(translate(frame, dx, dy), oracle_mod.translate(frame, dx, dy))


class TestCorrectMotion:  # test_motion.py:209-261
    def test_motion_free_video_unchanged(self, cuda, rng):
        video = Video(rng.random((30, 96, 96), dtype=np.float32))
        corrected, vectors = correct_motion(video, MotionConfig(search_radius=3, subpixel=False))
        assert len(vectors) == 30 and all((v.dx, v.dy) == (0, 0) for v in vectors)
        np.testing.assert_array_equal(corrected.data, video.data)

    def test_single_frame_video(self, cuda, rng):
        video = Video(rng.random((1, 96, 96), dtype=np.float32))
        corrected, vectors = correct_motion(video, MotionConfig(search_radius=3, subpixel=False))
        assert len(vectors) == 1 and (vectors[0].dx, vectors[0].dy) == (0, 0)
        np.testing.assert_array_equal(corrected.data, video.data)

    def test_reference_is_mean_of_first_frames(self, cuda, oracle_mod, rng):
        video = Video(rng.random((120, 64, 64), dtype=np.float32))
        np.testing.assert_array_equal(make_reference(video), oracle_mod.make_reference(video.data, 50))
        short = Video(rng.random((7, 64, 64), dtype=np.float32))
        np.testing.assert_array_equal(make_reference(short), oracle_mod.make_reference(short.data, 50))

    def test_reference_frames_is_monkeypatchable(self, cuda, oracle_mod, rng, monkeypatch):
        monkeypatch.setattr(motion, "REFERENCE_FRAMES", 100)
        video = Video(rng.random((130, 40, 40), dtype=np.float32))
        np.testing.assert_array_equal(make_reference(video), oracle_mod.make_reference(video.data, 100))

    def test_corrected_frame_realigns(self, cuda, rng):
        big = rng.random((140, 140), dtype=np.float32)
        shifts = [(0, 0)] * 10 + [(3, -2), (-4, 1), (5, 5), (-5, -5), (2, 0)]
        frames = np.stack([_shift_with_padding(big, dx, dy, 12)[:96, :96] for dx, dy in shifts])
        corrected, vectors = correct_motion(Video(frames), MotionConfig(search_radius=5, subpixel=False))
        for t, (dx, dy) in enumerate(shifts):
            assert (vectors[t].dx, vectors[t].dy) == (dx, dy), f"frame {t}"
        for t in range(len(shifts)):
            np.testing.assert_allclose(corrected.data[t][10:86, 10:86], frames[0][10:86, 10:86], atol=1e-5)

    def test_deterministic(self, cuda, rng):
        video = Video(rng.random((20, 96, 96), dtype=np.float32))
        c1, v1 = correct_motion(video, MotionConfig(search_radius=3))
        c2, v2 = correct_motion(video, MotionConfig(search_radius=3))
        assert v1 == v2
        np.testing.assert_array_equal(c1.data, c2.data)


def _regen(z, case):
    raw = synth.generate_numpy(synth.CONFIGS[case].with_frames(int(z[f"{case}__raw_spec"][0])))
    assert hashlib.sha256(raw.tobytes()).hexdigest() == str(z[f"{case}__raw_sha256"])
    return raw


@pytest.mark.parametrize("case", ["c1", "c2"])
@pytest.mark.parametrize("as_u16", [True, False])
def test_golden_correct_motion(cuda, golden, monkeypatch, case, as_u16):
    """Against the reference's correct_motion: integer shifts bit-exact vs the
    native (default) backend, sub-pixel <= 1e-3 px vs the float64 backend,
    corrected frames <= 1e-4 relative."""
    z = golden("motion")
    raw = _regen(z, case)
    p, r, m = (int(v) for v in z[f"{case}__geom"])
    monkeypatch.setattr(motion, "REFERENCE_FRAMES", m)
    corrected, vectors = correct_motion(Video(raw if as_u16 else raw.astype(np.float32)), MotionConfig(search_radius=r))
    dxdy = np.array([[v.dx, v.dy] for v in vectors])
    # bit-exact vs the reference's float64 backend on every frame ...
    np.testing.assert_array_equal(dxdy, z[f"{case}__python__dxdy"])
    # ... and vs its native (float32 cross-sum) backend wherever the reference's
    # two backends agree.  c2 frame 106 is a near-tie (top-2 margin 2.6e-5, below
    # the native kernel's ~1e-4 score noise) on which the reference disagrees with
    # itself; there we follow the float64 backend.
    nat, py = z[f"{case}__native__dxdy"], z[f"{case}__python__dxdy"]
    agree = (nat == py).all(axis=1)
    np.testing.assert_array_equal(dxdy[agree], nat[agree])
    assert (~agree).sum() <= 1
    sub = np.array([[v.sub_dx, v.sub_dy, v.confidence] for v in vectors])
    np.testing.assert_allclose(sub[:, :2], z[f"{case}__python__sub"][:, :2], atol=1e-3, rtol=0)
    assert np.abs(sub[:, :2] - z[f"{case}__python__sub"][:, :2]).max() < 2e-4  # measured margin
    np.testing.assert_allclose(sub[:, 2], z[f"{case}__python__sub"][:, 2], atol=1e-6)
    keep = z[f"{case}__python__corr_head"].shape[0]
    ref_c = z[f"{case}__python__corr_head"]
    rel = np.abs(corrected.data[:keep] - ref_c) / np.maximum(np.abs(ref_c), 1.0)
    assert rel.max() <= 1e-4
    sums = corrected.data.astype(np.float64).sum(axis=(1, 2))
    np.testing.assert_allclose(sums, z[f"{case}__python__corr_sum"], rtol=1e-6)


def test_c1_full_recording_vs_oracle(cuda, oracle_mod, monkeypatch):
    """BASELINE.json configs[0] at full size (1000 x 128 x 128, r=5, M=100)."""
    cfg = synth.CONFIGS["c1"]
    raw = synth.generate_numpy(cfg)
    monkeypatch.setattr(motion, "REFERENCE_FRAMES", cfg.ref_frames)
    corrected, vectors = correct_motion(Video(raw), MotionConfig(search_radius=cfg.radius))
    ref = oracle_mod.preprocess(raw.astype(np.float32), 21, cfg.radius, True, cfg.ref_frames, cfg.segment_length)
    dxdy = np.array([[v.dx, v.dy] for v in vectors])
    np.testing.assert_array_equal(dxdy, ref["dxdy"])
    sub = np.array([[v.sub_dx, v.sub_dy] for v in vectors])
    np.testing.assert_allclose(sub, ref["sub_conf"][:, :2], atol=1e-3, rtol=0)
    rel = np.abs(corrected.data - ref["corrected"]) / np.maximum(np.abs(ref["corrected"]), 1.0)
    assert rel.max() <= 1e-4


@pytest.mark.parametrize("n_frames", [1, 2, 3, 5, 37])
def test_c2_geometry_frame_counts_vs_oracle(cuda, oracle_mod, monkeypatch, n_frames):
    """C2 geometry (256 x 512, r = 8: the split S = 17 search kernel, two frames
    per CTA iteration) at frame counts that leave single-frame tails on some
    CTAs: shifts, sub-pixel and corrected frames against the C oracle."""
    cfg = synth.CONFIGS["c2"].with_frames(max(n_frames, 2))
    raw = synth.generate_numpy(cfg)[:n_frames]
    monkeypatch.setattr(motion, "REFERENCE_FRAMES", min(n_frames, 4))
    corrected, vectors = correct_motion(Video(raw), MotionConfig(search_radius=cfg.radius))
    ref = oracle_mod.preprocess(raw.astype(np.float32), 21, cfg.radius, True, min(n_frames, 4), 1000)
    np.testing.assert_array_equal(np.array([[v.dx, v.dy] for v in vectors]), ref["dxdy"])
    sub = np.array([[v.sub_dx, v.sub_dy] for v in vectors])
    np.testing.assert_allclose(sub, ref["sub_conf"][:, :2], atol=1e-3, rtol=0)
    rel = np.abs(corrected.data - ref["corrected"]) / np.maximum(np.abs(ref["corrected"]), 1.0)
    assert rel.max() <= 1e-4


@pytest.mark.parametrize("radius", [5, 8])
def test_high_dynamic_range_vs_oracle(cuda, oracle_mod, monkeypatch, radius):
    """Full-range uint16 frames (smooth structure spanning ~0..60000 counts,
    saturated 65535 spots, zero pixels) with sub-pixel drift: the exact integer
    window statistics (int64 sums of squares near their limits) and the
    centred float32 cross sums against the float64 oracle."""
    rng = np.random.default_rng(7)
    h, w, t = 128, 160, 24
    yy, xx = np.mgrid[0:h + 20, 0:w + 20].astype(np.float64)
    scene = 30000 + 25000 * np.sin(yy / 7.0) * np.cos(xx / 9.0) + 4000 * rng.standard_normal((h + 20, w + 20))
    scene[rng.integers(0, h + 20, 40), rng.integers(0, w + 20, 40)] = 1e9  # saturated spots
    scene[rng.integers(0, h + 20, 40), rng.integers(0, w + 20, 40)] = -1e9  # zeros
    frames = np.empty((t, h, w), np.uint16)
    for i in range(t):
        dy, dx = rng.uniform(-3, 3, 2)
        iy, ix = int(np.floor(dy)), int(np.floor(dx))
        fy, fx = dy - iy, dx - ix
        y0, x0 = 10 + iy, 10 + ix
        a = scene[y0:y0 + h, x0:x0 + w]
        b = scene[y0:y0 + h, x0 + 1:x0 + 1 + w]
        c = scene[y0 + 1:y0 + 1 + h, x0:x0 + w]
        d = scene[y0 + 1:y0 + 1 + h, x0 + 1:x0 + 1 + w]
        f = (1 - fy) * ((1 - fx) * a + fx * b) + fy * ((1 - fx) * c + fx * d)
        frames[i] = np.clip(np.rint(f + 50 * rng.standard_normal((h, w))), 0, 65535).astype(np.uint16)
    monkeypatch.setattr(motion, "REFERENCE_FRAMES", 8)
    corrected, vectors = correct_motion(Video(frames), MotionConfig(search_radius=radius))
    ref = oracle_mod.preprocess(frames.astype(np.float32), 21, radius, True, 8, 1000)
    np.testing.assert_array_equal(np.array([[v.dx, v.dy] for v in vectors]), ref["dxdy"])
    sub = np.array([[v.sub_dx, v.sub_dy] for v in vectors])
    np.testing.assert_allclose(sub, ref["sub_conf"][:, :2], atol=1e-3, rtol=0)
    np.testing.assert_allclose([v.confidence for v in vectors], ref["sub_conf"][:, 2], atol=1e-5)


def test_correct_motion_executor_equals_device_pipeline(cuda, monkeypatch):
    """correct_motion streams host recordings through the C-ABI executor in
    motion-only mode: identical vectors and frames to the device pipeline
    (template, MotionPlan.estimate, correct_frames_device), for uint16 and
    float32 recordings and the opt-in shading gain, across repeated calls."""
    raw = synth.generate_numpy(synth.CONFIGS["c1"].with_frames(130))
    monkeypatch.setattr(motion, "REFERENCE_FRAMES", 40)
    for data, shading in ((raw, 0.0), (raw.astype(np.float32), 0.0), (raw, 10.0)):
        cfg = MotionConfig(search_radius=5, shading_sigma=shading)
        got, vg = correct_motion(Video(data), cfg)
        frames = torch.from_numpy(data.view(np.int16) if data.dtype == np.uint16 else data).to(cuda)
        if data.dtype == np.uint16:
            frames = frames.view(torch.uint16)
        ref = motion.device_reference(frames, 40)
        grid = motion.PatchGrid.cover(128, 128, 21, margin=5)
        plan = motion.MotionPlan(128, 128, grid.origins, 21, 5)
        plan.set_reference(ref)
        vec, _ = plan.estimate(frames, True)
        gain = motion.shading_gain_device(ref, shading) if shading > 0 else None
        want = motion.correct_frames_device(frames, vec, gain).cpu().numpy()
        vw = motion._vectors_from_numpy(motion.D.motion_to_numpy(vec, frames.shape[0]))
        plan.close()
        assert vg == vw
        np.testing.assert_array_equal(got.data, want)


@pytest.mark.parametrize("n", [1, 2, 51, 101])
def test_correct_motion_any_length(cuda, monkeypatch, n):
    """correct_motion has no block structure: lengths that leave a one-frame
    summary block (n % L == 1) are fine in the motion-only executor mode."""
    raw = synth.generate_numpy(synth.CONFIGS["c1"].with_frames(max(n, 2)))[:n]
    monkeypatch.setattr(motion, "REFERENCE_FRAMES", 20)
    corrected, vectors = correct_motion(Video(raw), MotionConfig(search_radius=5))
    assert corrected.data.shape == raw.shape and len(vectors) == n
    again, v2 = correct_motion(Video(raw), MotionConfig(search_radius=5))
    assert v2 == vectors
    np.testing.assert_array_equal(again.data, corrected.data)
