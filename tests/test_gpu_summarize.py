"""Summary stage on the GPU: the reference's test_summarize.py cases plus
bit-exact parity with the reference's outputs (golden) and the oracle."""
import numpy as np
import pytest
from scipy import ndimage

from paper_2403_16438_b200 import Video, synth
from paper_2403_16438_b200.summarize import (TimeSegment, gaussian_smooth, spatial_summary, summarize,
                                             summarize_device, temporal_summary)

pytestmark = pytest.mark.gpu


def _segment(frames):
    return TimeSegment(0, np.asarray(frames, dtype=np.float32), 50)


class TestSpatial:  # test_summarize.py:45-72
    def test_constant(self, cuda):
        np.testing.assert_allclose(spatial_summary(_segment(np.full((50, 6, 6), 3.25))), 3.25, atol=1e-6)

    def test_single_impulse(self, cuda):
        f = np.zeros((50, 8, 8), np.float32)
        f[17, 3, 4] = 1.0
        s = spatial_summary(_segment(f))
        assert s[3, 4] == pytest.approx(1 / 50) and s.sum() == pytest.approx(1 / 50)

    def test_brute_force_bit_exact(self, cuda, rng):
        frames = rng.random((37, 12, 10), dtype=np.float32)
        want = frames.mean(axis=0, dtype=np.float64).astype(np.float32)
        np.testing.assert_array_equal(spatial_summary(_segment(frames)), want)

    def test_linearity(self, cuda, rng):
        u = rng.random((20, 8, 8), dtype=np.float32)
        v = rng.random((20, 8, 8), dtype=np.float32)
        lhs = spatial_summary(_segment(2.0 * u + 3.0 * v))
        rhs = 2.0 * spatial_summary(_segment(u)) + 3.0 * spatial_summary(_segment(v))
        np.testing.assert_allclose(lhs, rhs, atol=1e-5)


class TestGaussian:  # test_summarize.py:75-95
    def test_constant_preserved(self, cuda):
        np.testing.assert_allclose(gaussian_smooth(np.full((20, 20), 4.0), 3.0), 4.0, atol=1e-6)

    def test_impulse_ratio(self, cuda):
        img = np.zeros((31, 31))
        img[15, 15] = 1.0
        out = gaussian_smooth(img, 3.0)
        assert out[15, 15] / out[15, 16] == pytest.approx(np.exp(1 / 18.0), abs=1e-3)

    def test_corner_mass(self, cuda):
        img = np.zeros((31, 31))
        img[0, 0] = 1.0
        assert gaussian_smooth(img, 3.0).sum() == pytest.approx(1.0, rel=0.02)

    def test_rejects_bad_sigma(self, cuda):
        with pytest.raises(ValueError):
            gaussian_smooth(np.zeros((4, 4)), 0.0)

    @pytest.mark.parametrize("shape", [(31, 29), (8, 8), (4, 4), (1, 5), (256, 512), (70, 130),
                                       (70, 132), (100, 68), (36, 12), (10, 12), (9, 16), (33, 100)])
    def test_bit_exact_vs_scipy(self, cuda, rng, shape):
        x = (rng.random(shape, dtype=np.float32) * 1000).astype(np.float32)
        want = ndimage.gaussian_filter1d(ndimage.gaussian_filter1d(x, 3.0, axis=0, mode="reflect", radius=9),
                                         3.0, axis=1, mode="reflect", radius=9)
        np.testing.assert_array_equal(gaussian_smooth(x, 3.0), want)

    @pytest.mark.parametrize("kind", ["mixed_scales", "zeros_and_spikes", "signed", "tiny"])
    @pytest.mark.parametrize("shape", [(64, 128), (70, 130)])
    def test_bit_exact_adversarial(self, cuda, rng, kind, shape):
        """Inputs that put outputs near float32 rounding midpoints relative to
        the tile's largest sample (the R = 9 kernels' fused float64 passes
        must then fall back to scipy's unfused order): mixed magnitudes,
        zero fields with isolated spikes, signed values, subnormal-range data."""
        if kind == "mixed_scales":
            x = rng.standard_normal(shape) * 10.0 ** rng.integers(-6, 7, shape)
        elif kind == "zeros_and_spikes":
            x = np.zeros(shape)
            idx = rng.integers(0, x.size, x.size // 50)
            x.flat[idx] = rng.random(idx.size) * 6e4
            x[::7] += 1e-3
        elif kind == "signed":
            x = rng.standard_normal(shape) * 1000.0
        else:
            x = rng.standard_normal(shape) * 1e-36
        x = x.astype(np.float32)
        want = ndimage.gaussian_filter1d(ndimage.gaussian_filter1d(x, 3.0, axis=0, mode="reflect", radius=9),
                                         3.0, axis=1, mode="reflect", radius=9)
        np.testing.assert_array_equal(gaussian_smooth(x, 3.0), want)

    def test_golden_impulse(self, cuda, golden):
        z = golden("summary")
        np.testing.assert_array_equal(gaussian_smooth(z["gauss_impulse"], 3.0), z["gauss_impulse_out"])


class TestTemporal:  # test_summarize.py:98-147
    def test_constant_pixel_zero(self, cuda):
        np.testing.assert_allclose(temporal_summary(_segment(np.full((10, 6, 6), 2.0))), 0.0, atol=1e-7)

    def test_impulse_frame_value(self, cuda):
        frames = np.zeros((50, 21, 21), np.float32)
        frames[7, 10, 10] = 1.0
        amp = ndimage.gaussian_filter(frames[7].astype(np.float64), 3.0, mode="reflect", radius=9)[10, 10]
        assert temporal_summary(_segment(frames))[10, 10] == pytest.approx(amp, rel=1e-5)

    def test_brute_force(self, cuda, rng):
        frames = rng.random((24, 16, 14), dtype=np.float32)
        sm = np.stack([ndimage.gaussian_filter(f, 3.0, mode="reflect", radius=9) for f in frames])
        np.testing.assert_allclose(temporal_summary(_segment(frames)), sm.max(0) - np.median(sm, 0), atol=1e-5)

    def test_non_negative(self, cuda, rng):
        assert temporal_summary(_segment(rng.random((50, 20, 20), dtype=np.float32) * 100)).min() >= 0

    def test_single_frame_rejected(self, cuda, rng):
        with pytest.raises(ValueError, match="2 frames"):
            temporal_summary(_segment(rng.random((1, 8, 8))))

    def test_even_count_midpoint(self, cuda):
        frames = np.zeros((4, 6, 6), np.float32)
        for i, v in enumerate([0.0, 1.0, 2.0, 10.0]):
            frames[i] = v
        np.testing.assert_allclose(temporal_summary(_segment(frames)), 8.5, atol=1e-5)

    def test_permutation_invariant(self, cuda, rng):
        frames = rng.random((12, 10, 10), dtype=np.float32)
        np.testing.assert_array_equal(temporal_summary(_segment(frames)),
                                      temporal_summary(_segment(frames[rng.permutation(12)])))

    def test_offset_invariant(self, cuda, rng):
        frames = rng.random((12, 10, 10), dtype=np.float32)
        np.testing.assert_allclose(temporal_summary(_segment(frames)), temporal_summary(_segment(frames + 5.0)),
                                   atol=1e-4)

    @pytest.mark.parametrize("n", [2, 3, 31, 32, 33, 64, 65, 100, 257, 1000, 1023, 1024, 1025, 1500])
    def test_lengths_bit_exact_vs_oracle(self, cuda, oracle_mod, rng, n):
        """Register-resident selection for n <= 1024, global-memory path beyond."""
        frames = (rng.random((n, 9, 37), dtype=np.float32) * 500).astype(np.float32)
        if n % 7 == 0:
            frames[:, 3] = 42.0  # constant pixels -> exact zeros
        np.testing.assert_array_equal(temporal_summary(TimeSegment(0, frames, n)), oracle_mod.temporal_summary(frames))

    def test_ties_and_duplicates(self, cuda, oracle_mod, rng):
        frames = rng.integers(0, 4, size=(64, 16, 16)).astype(np.float32)  # heavy duplication
        np.testing.assert_array_equal(temporal_summary(TimeSegment(0, frames, 64)), oracle_mod.temporal_summary(frames))


class TestSummarize:  # test_summarize.py:150-187
    def test_output_length(self, cuda, rng):
        pairs = summarize(Video(rng.random((230, 16, 16), dtype=np.float32)), 50)
        assert [p.segment_index for p in pairs] == [0, 1, 2, 3, 4]

    def test_all_zero_video(self, cuda):
        for p in summarize(Video(np.zeros((100, 8, 8), np.float32)), 50):
            np.testing.assert_array_equal(p.spatial, 0)
            np.testing.assert_array_equal(p.temporal, 0)

    def test_one_frame_tail_rejected(self, cuda, rng):
        with pytest.raises(ValueError, match="2 frames"):
            summarize(Video(rng.random((101, 8, 8), dtype=np.float32)), 50)

    @pytest.mark.parametrize("case", ["rand_L50", "rand_L37", "counts_L64", "small_L4"])
    def test_golden_bit_exact(self, cuda, golden, case):
        z = golden("summary")
        pairs = summarize(Video(z[f"{case}__video"]), int(z[f"{case}__L"]))
        for i, p in enumerate(pairs):
            np.testing.assert_array_equal(p.spatial, z[f"{case}__spatial"][i])
            np.testing.assert_array_equal(p.temporal, z[f"{case}__temporal"][i])

    def test_golden_error_case(self, cuda, golden):
        z = golden("summary")
        with pytest.raises(ValueError, match="2 frames"):
            summarize(Video(z["tiny_L3__video"]), int(z["tiny_L3__L"]))

    def test_u16_input_equals_widened(self, cuda):
        raw = synth.generate_numpy(synth.CONFIGS["c1"].with_frames(100))
        a = summarize(Video(raw), 50)
        b = summarize(Video(raw.astype(np.float32)), 50)
        for p, q in zip(a, b):
            np.testing.assert_array_equal(p.spatial, q.spatial)
            np.testing.assert_array_equal(p.temporal, q.temporal)

    @pytest.mark.parametrize("shape", [(70, 131), (70, 132), (100, 68)])
    def test_large_frame_tiles_vs_oracle(self, cuda, oracle_mod, rng, shape):
        """Frame sizes that are not multiples of the 32x64 tile (w % 4 == 0:
        the split warp -> TMA smoothing path; otherwise the fused kernel)."""
        v = (rng.random((40, *shape), dtype=np.float32) * 1000).astype(np.float32)
        pairs = summarize(Video(v), 20)
        for i, p in enumerate(pairs):
            np.testing.assert_array_equal(p.spatial, oracle_mod.spatial_summary(v[20 * i:20 * (i + 1)]))
            np.testing.assert_array_equal(p.temporal, oracle_mod.temporal_summary(v[20 * i:20 * (i + 1)]))

    def test_spiking_pixels_stand_out(self, cuda):
        """test_summarize.py:161-178 on the repo's generator: pixels of neurons
        that spiked in a block rank high in that block's temporal summary."""
        cfg = synth.CONFIGS["c1"].with_frames(400)
        raw, truth = synth.generate_numpy(cfg, return_truth=True)
        pairs = summarize(Video(raw), 200)
        import torch
        scored = checked = 0
        for i, p in enumerate(pairs):
            sp = truth.spikes[200 * i:200 * (i + 1)].any(axis=0)
            for k in np.nonzero(sp)[0]:
                cx, cy = truth.centers[k]
                yy, xx = int(round(cy)), int(round(cx))
                if not (3 <= yy < 125 and 3 <= xx < 125):
                    continue
                checked += 1
                scored += p.temporal[yy, xx] > np.percentile(p.temporal, 75)
        assert checked > 0 and scored / checked >= 0.6


def test_summarize_chunked_equals_whole(cuda, monkeypatch, rng):
    """Recordings larger than a third of the free HBM are summarised in batches
    of whole blocks: identical pairs (indices, spatial, temporal)."""
    v = (rng.random((230, 24, 20), dtype=np.float32) * 1000).astype(np.float32)
    whole = summarize(Video(v), 50)
    import torch
    monkeypatch.setattr(torch.cuda, "mem_get_info", lambda *a: (50 * 24 * 20 * 4 * 6 * 2, 1 << 40))  # 2 blocks per batch
    chunked = summarize(Video(v), 50)
    assert [p.segment_index for p in chunked] == [p.segment_index for p in whole] == [0, 1, 2, 3, 4]
    for p, q in zip(whole, chunked):
        np.testing.assert_array_equal(p.spatial, q.spatial)
        np.testing.assert_array_equal(p.temporal, q.temporal)
