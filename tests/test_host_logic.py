"""Host-side logic of the stage API (geometry, bookkeeping, generator,
sharding plan) -- mirrors the reference's own unit tests; CPU only."""
import csv

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st
from scipy import ndimage

from paper_2403_16438_b200 import Video, distributed, synth
from paper_2403_16438_b200.motion import (MotionVector, PatchGrid, _candidate_order, _quadratic_peak,
                                          build_area_tables, rect_sum, save_motion_csv, zncc)
from paper_2403_16438_b200.summarize import gaussian_weights, split_segments


class TestPatchGrid:  # test_motion.py:90-113
    def test_patches_inside_margin(self):
        grid = PatchGrid.cover(128, 128, 21, margin=10)
        assert len(grid.origins) > 0
        for x, y in grid.origins:
            assert 10 <= x and x + 21 <= 118 and 10 <= y and y + 21 <= 118

    def test_covers_inset_region(self):
        grid = PatchGrid.cover(100, 90, 21, margin=5)
        covered = np.zeros((100, 90), dtype=bool)
        for x, y in grid.origins:
            covered[y:y + 21, x:x + 21] = True
        assert covered[5:95, 5:85].all()

    def test_flush_final_row_and_column(self):
        grid = PatchGrid.cover(128, 128, 21, margin=0)
        assert max(grid.origins[:, 0]) == 107 and max(grid.origins[:, 1]) == 107

    def test_too_small_frame(self):
        with pytest.raises(ValueError, match="too small"):
            PatchGrid.cover(30, 30, 21, margin=10)

    @pytest.mark.parametrize("h,w,p,m", [(128, 128, 21, 5), (256, 512, 21, 8), (512, 512, 21, 12),
                                         (1024, 1024, 21, 10), (96, 96, 16, 3), (60, 60, 15, 3)])
    def test_matches_oracle_and_c_abi(self, oracle_mod, h, w, p, m):
        import ctypes

        from paper_2403_16438_b200 import _lib
        g = PatchGrid.cover(h, w, p, margin=m).origins
        np.testing.assert_array_equal(g, oracle_mod.patch_grid(h, w, p, m))
        n = ctypes.c_int()
        _lib.call("vb_patch_grid", h, w, p, m, None, ctypes.byref(n))
        o = np.empty((n.value, 2), np.int32)
        _lib.call("vb_patch_grid", h, w, p, m, o.ctypes.data, ctypes.byref(n))
        np.testing.assert_array_equal(g, o)

    def test_survey_patch_counts(self):
        for (h, w, r), n in {(128, 128, 5): 36, (256, 512, 8): 288, (512, 512, 12): 576,
                             (1024, 1024, 10): 2304}.items():
            assert len(PatchGrid.cover(h, w, 21, margin=r).origins) == n


class TestZncc:  # test_motion.py:34-62
    def test_identical(self, rng):
        w = rng.random((21, 21))
        assert zncc(w, w) == pytest.approx(1.0, abs=1e-6)

    def test_affine_negative(self, rng):
        w = rng.random((21, 21))
        assert zncc(w, -2.0 * w + 5.0) == pytest.approx(-1.0, abs=1e-6)

    def test_constant_zero(self, rng):
        assert zncc(np.full((5, 5), 3.0), rng.random((5, 5))) == 0.0

    def test_dimension_mismatch(self):
        with pytest.raises(ValueError, match="dimensions differ"):
            zncc(np.zeros((4, 4)), np.zeros((5, 4)))

    @given(a=st.floats(0.1, 10.0), b=st.floats(-5.0, 5.0), seed=st.integers(0, 2 ** 16))
    @settings(max_examples=30, deadline=None)
    def test_affine_invariance(self, a, b, seed):
        r = np.random.default_rng(seed)
        x, y = r.random((9, 9)), r.random((9, 9))
        assert zncc(a * x + b, y) == pytest.approx(zncc(x, y), abs=1e-6)


class TestAreaTables:  # test_motion.py:65-87
    def test_random_rectangles(self, rng):
        frame = rng.random((64, 64))
        sat, sat2 = build_area_tables(frame)
        for _ in range(50):
            x0, y0 = rng.integers(0, 60, size=2)
            w, h = int(rng.integers(1, 64 - x0)), int(rng.integers(1, 64 - y0))
            assert rect_sum(sat, x0, y0, w, h) == pytest.approx(frame[y0:y0 + h, x0:x0 + w].sum(), rel=1e-9)
            assert rect_sum(sat2, x0, y0, w, h) == pytest.approx((frame[y0:y0 + h, x0:x0 + w] ** 2).sum(), rel=1e-9)


class TestCandidateOrder:
    @pytest.mark.parametrize("r", [1, 3, 8, 12])
    def test_order_and_kernel_key_agree(self, r):
        order, flat = _candidate_order(r)
        s = 2 * r + 1
        assert order[0] == (0, 0) and len(order) == s * s
        # the finalize kernel ranks candidates with key ((|dx|+|dy|)*S + dy+r)*S + dx+r
        keys = [((abs(dx) + abs(dy)) * s + dy + r) * s + dx + r for dx, dy in order]
        assert keys == sorted(keys)

    def test_quadratic_peak(self):
        line = -np.array([(-1 - 0.3) ** 2, (0 - 0.3) ** 2, (1 - 0.3) ** 2])
        assert _quadratic_peak(line, 1) == pytest.approx(0.3, abs=1e-9)
        assert _quadratic_peak(line, 0) == 0.0
        assert _quadratic_peak(np.array([1.0, 0.0, 1.0]), 1) == 0.0  # denom >= 0
        assert _quadratic_peak(np.array([0.0, 1.0, 1.0]), 1) == pytest.approx(0.5)


class TestMotionVectorCsv:  # test_motion.py:264-273
    def test_csv_format(self, tmp_path):
        vectors = [MotionVector(1, -2, 0.25, -0.5, 0.875), MotionVector(0, 0, 0.0, 0.0, 1.0)]
        path = tmp_path / "motion.csv"
        save_motion_csv(vectors, path)
        rows = list(csv.reader(path.open()))
        assert rows == [["frame", "dx", "dy", "confidence"], ["0", "1.25", "-2.5", "0.875000"], ["1", "0", "0", "1.000000"]]


class TestSegments:  # test_summarize.py:21-42
    @pytest.mark.parametrize("t,expected", [(10000, [50] * 200), (101, [50, 50, 1]), (7, [7])])
    def test_lengths(self, t, expected):
        segs = split_segments(Video(np.zeros((t, 4, 4), np.float32)), 50)
        assert [s.frames.shape[0] for s in segs] == expected
        assert [s.index for s in segs] == list(range(len(expected)))

    def test_rejects_short_length(self):
        with pytest.raises(ValueError):
            split_segments(Video(np.zeros((10, 4, 4), np.float32)), 1)


class TestWeights:
    @pytest.mark.parametrize("sigma", [3.0, 1.0, 2.5, 5.0])
    def test_weights_equal_scipy(self, sigma):
        from scipy.ndimage._filters import _gaussian_kernel1d
        import math
        w, r = gaussian_weights(sigma)
        assert r == math.ceil(3 * sigma)
        np.testing.assert_array_equal(w, _gaussian_kernel1d(sigma, 0, r)[::-1])

    def test_rejects_bad_sigma(self):
        with pytest.raises(ValueError):
            gaussian_weights(0.0)


class TestVideo:  # video_io.py:28-58
    def test_u16_kept_raw(self):
        v = Video(np.ones((3, 4, 5), np.uint16))
        assert v.raw is not None and v.data.dtype == np.float32 and v.shape == (3, 4, 5)

    @pytest.mark.parametrize("bad,msg", [(np.zeros((4, 4)), "3-D"), (np.zeros((0, 4, 4)), ">= 1"),
                                         (np.full((2, 2, 2), np.nan), "finite"), (-np.ones((2, 2, 2)), "non-negative")])
    def test_validation(self, bad, msg):
        with pytest.raises(ValueError, match=msg):
            Video(bad)


class TestSynth:
    def test_deterministic_and_shaped(self):
        cfg = synth.CONFIGS["c1"].with_frames(24)
        a, truth = synth.generate_numpy(cfg, return_truth=True)
        b = synth.generate_numpy(cfg)
        assert a.dtype == np.uint16 and a.shape == (24, 128, 128)
        np.testing.assert_array_equal(a, b)
        assert np.abs(truth.drift).max() <= cfg.drift_px
        assert 500 < a.mean() < 1200

    def test_configs_match_baseline(self):
        c = synth.CONFIGS
        assert (c["c1"].frames, c["c1"].height, c["c1"].width, c["c1"].radius, c["c1"].segment_length) == (1000, 128, 128, 5, 500)
        assert (c["c2"].frames, c["c2"].height, c["c2"].width, c["c2"].radius, c["c2"].segment_length) == (10000, 256, 512, 8, 1000)
        assert (c["c3"].frames, c["c3"].height, c["c3"].radius) == (20000, 512, 12)
        assert (c["c4"].frames, c["c5"].height) == (100000, 1024)


class TestShardPlan:
    @pytest.mark.parametrize("t,L,world", [(10000, 1000, 8), (10000, 1000, 3), (1000, 500, 2), (123, 50, 4), (7, 3, 5)])
    def test_partition_is_exact_and_block_aligned(self, t, L, world):
        shards = [distributed.shard_plan(t, L, world, r) for r in range(world)]
        assert shards[0].frame_lo == 0 and shards[-1].frame_hi == t
        for a, b in zip(shards, shards[1:]):
            assert a.frame_hi == b.frame_lo and a.block_hi == b.block_lo
        for s in shards:
            assert s.frame_lo % L == 0 and s.n_total == t
        assert sum(s.frames for s in shards) == t

    def test_template_rows(self):
        s = distributed.shard_plan(10000, 1000, 4, 0)
        assert distributed.template_rows(s, 100) == (0, 100)
        s1 = distributed.shard_plan(10000, 1000, 4, 1)
        assert distributed.template_rows(s1, 100) == (0, 0)
        s2 = distributed.shard_plan(150, 50, 3, 1)  # frames 50..100 hold template rows 50..99
        assert distributed.template_rows(s2, 100) == (0, 50)


def test_group_plan_block_aligned():
    """vb_group_plan (C ABI, host only): whole blocks per device, as even as
    possible, covering the recording (distributed.shard_plan's split)."""
    from paper_2403_16438_b200 import distributed
    from paper_2403_16438_b200.stage import group_plan

    for t, L, n in [(10000, 1000, 8), (10000, 1000, 3), (2500, 1000, 4), (7, 2, 5), (1000, 500, 1)]:
        plan = group_plan(t, L, n)
        assert plan[0][0] == 0 and plan[-1][1] == t
        for (a, b), (c, _d) in zip(plan, plan[1:]):
            assert b == c and (a % L == 0 or a == t)
        for r in range(n):
            s = distributed.shard_plan(t, L, n, r)
            assert plan[r] == (s.frame_lo, s.frame_hi)
