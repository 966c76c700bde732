"""Operator parity: libvoltb200's ZNCC score grid (vb_mean_zncc_scores) vs the
oracle and vs the reference's own outputs (golden), plus the reference's
kernel tests (test_kernels.py) run against the CUDA path."""
import numpy as np
import pytest

from paper_2403_16438_b200 import kernels
from paper_2403_16438_b200.motion import PatchGrid, zncc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("radius", [1, 3, 5, 10, 12, 16, 20, 31])
def test_random_frames_vs_oracle(cuda, oracle_mod, rng, radius):
    """test_kernels.py:13-19 geometry (reference tolerance 1e-4; we hold 1e-6)."""
    size = max(128, 21 + 2 * radius + 8)
    f = rng.random((size, size), dtype=np.float32)
    r = rng.random((size, size), dtype=np.float32)
    g = PatchGrid.cover(size, size, 21, margin=radius)
    a = kernels.mean_zncc_scores(f, r, g.origins, 21, radius)
    b = oracle_mod.mean_zncc_scores(f, r, g.origins, 21, radius)
    np.testing.assert_allclose(a, b, atol=1e-6)


@pytest.mark.parametrize("patch,radius,shape", [(15, 3, (60, 60)), (16, 3, (96, 96)), (11, 2, (40, 44)),
                                                 (5, 1, (20, 23)), (33, 4, (100, 90)), (21, 0, (50, 50)),
                                                 (65, 3, (150, 150)), (80, 2, (170, 168))])
def test_generic_patch_sizes(cuda, oracle_mod, rng, patch, radius, shape):
    f = rng.random(shape, dtype=np.float32)
    r = rng.random(shape, dtype=np.float32)
    g = PatchGrid.cover(shape[0], shape[1], patch, margin=radius)
    np.testing.assert_allclose(kernels.mean_zncc_scores(f, r, g.origins, patch, radius),
                               oracle_mod.mean_zncc_scores(f, r, g.origins, patch, radius), atol=1e-6)


def test_matches_brute_force(cuda, rng):
    """test_kernels.py:39-53: per-candidate brute-force mean ZNCC, free origins."""
    frame = rng.random((60, 60), dtype=np.float32)
    ref = rng.random((60, 60), dtype=np.float32)
    origins = np.array([[10, 12], [25, 20]], dtype=np.int32)
    patch, radius = 15, 3
    scores = kernels.mean_zncc_scores(frame, ref, origins, patch, radius)
    for dy in range(-radius, radius + 1):
        for dx in range(-radius, radius + 1):
            vals = [zncc(frame[y + dy:y + dy + patch, x + dx:x + dx + patch], ref[y:y + patch, x:x + patch])
                    for x, y in origins]
            assert scores[dy + radius, dx + radius] == pytest.approx(np.mean(vals), abs=1e-6)


def test_constant_patch_contributes_zero(cuda):
    frame = np.full((40, 40), 2.0, dtype=np.float32)
    ref = np.full((40, 40), 7.0, dtype=np.float32)
    scores = kernels.mean_zncc_scores(frame, ref, np.array([[10, 10]], np.int32), 11, 2)
    np.testing.assert_array_equal(scores, 0.0)


def test_self_score_is_one(cuda, rng):
    frame = rng.random((50, 50), dtype=np.float32)
    out = kernels.mean_zncc_scores(frame, frame, np.array([[12, 12]], np.int32), 15, 2)
    assert out.shape == (5, 5) and out[2, 2] == pytest.approx(1.0, abs=1e-6)


def test_errors_match_reference_messages(cuda, rng):
    f = rng.random((64, 64), dtype=np.float32)
    with pytest.raises(ValueError, match="border"):
        kernels.mean_zncc_scores(f, f, np.array([[0, 0]], np.int32), 21, 5)
    with pytest.raises(ValueError, match="differ"):
        kernels.mean_zncc_scores(f, rng.random((64, 60), dtype=np.float32), np.array([[10, 10]], np.int32), 21, 5)
    big = rng.random((200, 200), dtype=np.float32)
    with pytest.raises(ValueError, match="max 31"):
        kernels.mean_zncc_scores(big, big, np.array([[80, 80]], np.int32), 21, 32)


def test_golden_scores(cuda, golden):
    """Against the reference's float64 backend (tolerance 1e-6 abs; the
    reference's own two backends differ by up to 1.3e-4 on camera frames)."""
    z = golden("scores")
    for name in [str(n) for n in z["names"]]:
        f = z[f"{name}__frame"].astype(np.float32)
        p, r = (int(v) for v in z[f"{name}__geom"])
        got = kernels.mean_zncc_scores(f, z[f"{name}__ref"], z[f"{name}__origins"], p, r)
        np.testing.assert_allclose(got, z[f"{name}__py"], atol=1e-6, err_msg=name)
        # integer argmax agrees with both reference backends
        assert np.unravel_index(np.argmax(got), got.shape) == np.unravel_index(np.argmax(z[f"{name}__py"]), got.shape)


@pytest.mark.parametrize("patch,radius", [(65, 3), (80, 2)])
def test_large_patch_full_range_u16(cuda, oracle_mod, rng, patch, radius):
    """Patches beyond 64 (the window sums loop to P) on full-range uint16
    samples, where n*var exceeds 2^52 and the int64 -> double conversion
    must not use the bit trick."""
    from paper_2403_16438_b200 import _device as D
    from paper_2403_16438_b200.motion import MotionPlan

    size = patch + 2 * radius + 40
    fu = rng.integers(0, 65536, (2, size, size), dtype=np.uint16)  # integer window-sum path (u16)
    r = rng.integers(0, 65536, (size, size)).astype(np.float32)
    g = PatchGrid.cover(size, size, patch, margin=radius)
    plan = MotionPlan(size, size, g.origins, patch, radius)
    try:
        plan.set_reference(D.as_device_frames(r))
        _, sc = plan.estimate(D.as_device_frames(fu), True, scores=True)
        got = sc.cpu().numpy().reshape(2, 2 * radius + 1, 2 * radius + 1)
    finally:
        plan.close()
    for t in range(2):
        want = oracle_mod.mean_zncc_scores(fu[t].astype(np.float32), r, g.origins, patch, radius)
        np.testing.assert_allclose(got[t], want, atol=1e-6)
        np.testing.assert_allclose(kernels.mean_zncc_scores(fu[t].astype(np.float32), r, g.origins, patch, radius),
                                   want, atol=1e-6)


def test_patch_too_large_rejected(cuda, rng):
    f = rng.random((400, 400), dtype=np.float32)
    with pytest.raises(ValueError, match="max 180"):
        kernels.mean_zncc_scores(f, f, np.array([[100, 100]], np.int32), 181, 1)
