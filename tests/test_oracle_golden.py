"""The CPU oracle (oracle/oracle.c) against golden vectors produced by the
UNMODIFIED reference (tests/golden/make_golden.py).  CPU only."""
import hashlib

import numpy as np
import pytest

from paper_2403_16438_b200 import synth


def _names(z):
    return [str(n) for n in z["names"]]


def test_scores_match_reference_float64_backend(golden, oracle_mod):
    z = golden("scores")
    for name in _names(z):
        f = z[f"{name}__frame"].astype(np.float32)
        p, r = (int(v) for v in z[f"{name}__geom"])
        got = oracle_mod.mean_zncc_scores(f, z[f"{name}__ref"], z[f"{name}__origins"], p, r)
        # the reference obtains window sums from float64 summed-area tables (kernels.py:78-86)
        np.testing.assert_allclose(got, z[f"{name}__py"], rtol=0, atol=1e-10, err_msg=name)


def test_scores_constant_frame_exact_zero(golden, oracle_mod):
    z = golden("scores")
    got = oracle_mod.mean_zncc_scores(z["const40__frame"].astype(np.float32), z["const40__ref"],
                                      z["const40__origins"], 11, 2)
    assert (got == 0).all() and (z["const40__native"] == 0).all()


def test_pick_motion_matches_reference_on_both_backends(golden, oracle_mod):
    """Integer argmax (tie-break order) equals both reference backends; the
    quadratic fit equals the float64 backend's (motion.py:113-160)."""
    z = golden("scores")
    for name in _names(z):
        p, r = (int(v) for v in z[f"{name}__geom"])
        a = oracle_mod.pick_motion(z[f"{name}__py"], r)
        b = oracle_mod.pick_motion(z[f"{name}__native"], r)
        assert a[:2] == b[:2], name


def _regen(cfg_name, frames, sha):
    raw = synth.generate_numpy(synth.CONFIGS[cfg_name].with_frames(frames))
    assert hashlib.sha256(raw.tobytes()).hexdigest() == sha, \
        "seeded generator output changed; rerun tests/golden/make_golden.py"
    return raw


@pytest.mark.parametrize("case", ["c1", "c2"])
def test_correct_motion_matches_reference(golden, oracle_mod, case):
    z = golden("motion")
    raw = _regen(case, int(z[f"{case}__raw_spec"][0]), str(z[f"{case}__raw_sha256"]))
    p, r, m = (int(v) for v in z[f"{case}__geom"])
    frames = raw.astype(np.float32)
    ref = oracle_mod.make_reference(frames, m)
    origins = oracle_mod.patch_grid(frames.shape[1], frames.shape[2], p, r)
    # every frame for c1; a spread subset for the larger c2 (float64 search is slow)
    idx = range(frames.shape[0]) if case == "c1" else range(0, frames.shape[0], 9)
    keep = z[f"{case}__python__corr_head"].shape[0]
    for t in idx:
        dx, dy, sdx, sdy, conf = oracle_mod.estimate_motion(frames[t], ref, origins, p, r)
        assert (dx, dy) == tuple(z[f"{case}__native__dxdy"][t]) == tuple(z[f"{case}__python__dxdy"][t]), t
        np.testing.assert_allclose([sdx, sdy, conf], z[f"{case}__python__sub"][t], rtol=0, atol=1e-9)
        if t < keep:
            corr = oracle_mod.correct_frame(frames[t], dx + sdx, dy + sdy)
            np.testing.assert_allclose(corr, z[f"{case}__python__corr_head"][t], rtol=1e-6, atol=1e-3)


def test_translate_bit_exact(golden, oracle_mod):
    z = golden("translate")
    for (dx, dy), want in zip(z["shifts"], z["out"]):
        np.testing.assert_array_equal(oracle_mod.translate(z["frame"], dx, dy), want)


@pytest.mark.parametrize("case", ["rand_L50", "rand_L37", "counts_L64", "small_L4"])
def test_summaries_bit_exact(golden, oracle_mod, case):
    z = golden("summary")
    v, L = z[f"{case}__video"], int(z[f"{case}__L"])
    k = -(-v.shape[0] // L)
    for b in range(k):
        seg = v[b * L:(b + 1) * L]
        np.testing.assert_array_equal(oracle_mod.spatial_summary(seg), z[f"{case}__spatial"][b])
        np.testing.assert_array_equal(oracle_mod.temporal_summary(seg), z[f"{case}__temporal"][b])


def test_summary_reference_error_case(golden):
    z = golden("summary")
    assert "2 frames" in str(z["tiny_L3__error"])


def test_even_median_known_answer(golden, oracle_mod):
    z = golden("summary")
    got = oracle_mod.temporal_summary(z["even4__video"])
    np.testing.assert_array_equal(got, z["even4__temporal"][0])
    np.testing.assert_allclose(got, 8.5)


def test_gaussian_impulse(golden, oracle_mod):
    z = golden("summary")
    np.testing.assert_array_equal(oracle_mod.smooth_frame(z["gauss_impulse"]), z["gauss_impulse_out"])


def test_traces_match_reference(golden, oracle_mod):
    """traces.py:23-34 extract_trace on random ROIs (reference pairwise float64
    mean vs the oracle's sequential sum: <= 1e-12 relative)."""
    z = golden("traces")
    for k in range(5):
        got = oracle_mod.extract_trace(z["video"], z[f"mask{k}"])
        np.testing.assert_allclose(got, z[f"trace{k}"], rtol=1e-12)
