"""A17 extensions (opt-in shading correction and temporal high-pass; no
reference counterpart -- parity unpinned against the reference, pinned to the
repo's own restatement in oracle/oracle.c).  CPU tests: host helpers and the
oracle's defining properties.  GPU tests: the CUDA path == the oracle
bit-for-bit, and every execution shape (fused stage, separate calls, chunked
host executor, time shards with a halo) == every other."""
import numpy as np
import pytest

from paper_2403_16438_b200 import distributed, extensions


# ---------------------------------------------------------------- CPU: host logic
def test_highpass_window_from_cutoff():
    assert extensions.highpass_window(10.0, 741.0) == 33  # north-star ~10 Hz at 741 fps
    assert extensions.highpass_window(100.0, 741.0) == 3
    assert extensions.highpass_window(1.0, 741.0) % 2 == 1
    with pytest.raises(ValueError):
        extensions.highpass_window(0.0, 741.0)


def test_check_window():
    assert extensions.check_window(0) == 0 and extensions.check_window(1) == 0
    assert extensions.check_window(33) == 33
    with pytest.raises(ValueError, match="odd"):
        extensions.check_window(32)


def test_shading_weights_match_scipy_taps():
    from scipy.ndimage import _filters

    w, r = extensions.shading_weights(7.3)
    assert r == int(4 * 7.3 + 0.5)
    np.testing.assert_array_equal(w, _filters._gaussian_kernel1d(7.3, 0, r)[::-1])


@pytest.mark.parametrize("world", [2, 3, 5])
def test_halo_ranges_cover_filter_support(world):
    n, L, win = 1000, 100, 33
    for r in range(world):
        s = distributed.shard_plan(n, L, world, r)
        lo, hi = distributed.halo_range(s, win)
        assert lo == max(0, s.frame_lo - 16) and hi == min(n, s.frame_hi + 16)
        assert distributed.halo_range(s, 0) == (s.frame_lo, s.frame_hi)
        # template rows count only the shard's own frames, in halo-local indices
        a, b = distributed.template_rows(s, 150, lo)
        if b > a:
            assert lo + a == max(s.frame_lo, 0) and lo + b == min(s.frame_hi, 150)


# ---------------------------------------------------------------- CPU: oracle definition
def test_oracle_highpass_removes_linear_trends(oracle_mod, rng):
    """x - mean_N(x) vanishes on a linear ramp away from the reflected ends;
    an isolated transient survives -> the summary is the transient height."""
    t, h, w = 200, 12, 14
    base = (1000.0 + 0.5 * np.arange(t, dtype=np.float64))[:, None, None] * np.ones((1, h, w))
    frames = base.astype(np.float32)
    out = oracle_mod.highpass_summary(frames, 100, 33)
    sm_ramp = out.copy()
    frames[120, 6, 7] += 5000.0
    out2 = oracle_mod.highpass_summary(frames, 100, 33)
    assert np.abs(sm_ramp[1]).max() < 10.0       # trend removed (only the reflected tail stays)
    assert out2[1, 6, 7] > 30.0 + sm_ramp[1, 6, 7]
    np.testing.assert_array_equal(out2[0], sm_ramp[0])  # block 0 is beyond the window


def test_oracle_shading_gain_properties(oracle_mod, rng):
    ref = np.full((40, 50), 1234.5, np.float32)
    np.testing.assert_allclose(oracle_mod.shading_gain(ref, 5.0), 1.0, rtol=1e-7)
    yy, xx = np.mgrid[:64, :80]
    vig = 1000.0 * (1.0 - 0.3 * (((yy - 32) / 32.0) ** 2 + ((xx - 40) / 40.0) ** 2) / 2)
    g = oracle_mod.shading_gain(vig.astype(np.float32), 4.0)
    assert abs(g.astype(np.float64).mean() - 1.0) < 1e-3
    assert g[32, 40] > g[0, 0]


# ---------------------------------------------------------------- CPU: pinned to scipy
# The A17 definitions restated with scipy's published filters (scipy 1.18.1,
# the reference's pinned dependency, pyproject.toml:11-12): the shading gain is
# gaussian_filter(template, sigma, mode="reflect", truncate=4) / its mean, the
# high-pass is x - uniform_filter1d(x, N, axis=0, mode="reflect") on the
# reference's smoothed stack (summarize.py:70-73), then the reference's
# max - median (summarize.py:76-92).  Tolerance: 1e-4 relative (the north
# star's float32 bound; the two differ only in float64 summation order and
# where the float32 rounding happens).
def scipy_shading_gain(ref, sigma):
    from scipy import ndimage

    g = ndimage.gaussian_filter(np.asarray(ref, np.float64), sigma, mode="reflect", truncate=4.0)
    return (g / g.mean()).astype(np.float32)


def scipy_highpass_summary(frames, L, window, sigma=3.0):
    from scipy import ndimage

    f = np.asarray(frames, np.float32)
    sm = ndimage.gaussian_filter1d(f, sigma, axis=1, mode="reflect", radius=9)
    sm = ndimage.gaussian_filter1d(sm, sigma, axis=2, mode="reflect", radius=9)
    s64 = sm.astype(np.float64)
    hp = (s64 - ndimage.uniform_filter1d(s64, window, axis=0, mode="reflect")).astype(np.float32)
    out = []
    for b0 in range(0, f.shape[0], L):
        blk = hp[b0:b0 + L]
        o = np.sort(blk, axis=0)
        n, mid = blk.shape[0], blk.shape[0] // 2
        med = o[mid] if n % 2 else (o[mid - 1] + o[mid]) * np.float32(0.5)
        out.append(blk.max(axis=0) - med)
    return np.stack(out)


@pytest.mark.parametrize("shape,sigma", [((96, 128), 16.0), ((33, 70), 40.0), ((64, 80), 4.0)])
def test_oracle_shading_gain_vs_scipy(oracle_mod, shape, sigma):
    rng = np.random.default_rng(3)
    ref = (1000.0 + 300.0 * rng.random(shape)).astype(np.float32)
    # measured bit-identical on these inputs (held to 1e-6 relative)
    np.testing.assert_allclose(oracle_mod.shading_gain(ref, sigma), scipy_shading_gain(ref, sigma), rtol=1e-6)


@pytest.mark.parametrize("shape,L,win", [((300, 40, 72), 100, 33), ((122, 30, 40), 40, 3), ((20, 24, 24), 10, 33)])
def test_oracle_highpass_vs_scipy(oracle_mod, shape, L, win):
    frames = _frames(shape)
    got = oracle_mod.highpass_summary(frames, L, win)
    want = scipy_highpass_summary(frames, L, win)
    np.testing.assert_array_equal(got, want)  # bit-identical: same float64 sums, same rounding points


# ---------------------------------------------------------------- GPU
def _frames(shape, seed=7):
    rng = np.random.default_rng(seed)
    t, h, w = shape
    base = 800.0 + 200.0 * rng.random((1, h, w))
    drift = np.linspace(0.0, 60.0, t)[:, None, None]           # slow baseline (bleaching-like)
    spikes = (rng.random((t, h, w)) < 0.01) * 150.0
    noise = rng.normal(0.0, 5.0, (t, h, w))
    return np.clip(base + drift + spikes + noise, 0, 65535).astype(np.float32)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,L,win", [((300, 40, 72), 100, 33), ((250, 33, 70), 64, 9),
                                         ((20, 24, 24), 10, 33), ((122, 30, 40), 40, 3)])
def test_highpass_summary_matches_oracle(cuda, oracle_mod, shape, L, win):
    from paper_2403_16438_b200.summarize import summarize

    frames = _frames(shape)
    got = summarize(frames, L, highpass_window=win)
    want_tp = oracle_mod.highpass_summary(frames, L, win)
    for k, p in enumerate(got):
        np.testing.assert_array_equal(p.temporal, want_tp[k])
        np.testing.assert_array_equal(p.spatial, oracle_mod.spatial_summary(frames[k * L:(k + 1) * L]))


@pytest.mark.gpu
def test_highpass_off_is_reference_summary(cuda, oracle_mod):
    from paper_2403_16438_b200.summarize import summarize

    frames = _frames((120, 20, 36))
    a = summarize(frames, 50)
    b = summarize(frames, 50, highpass_window=0)
    for p, q in zip(a, b):
        np.testing.assert_array_equal(p.temporal, q.temporal)
        np.testing.assert_array_equal(p.temporal, oracle_mod.temporal_summary(frames[p.segment_index * 50:
                                                                                     (p.segment_index + 1) * 50]))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,sigma", [((96, 128), 16.0), ((33, 70), 40.0), ((256, 512), 32.0)])
def test_shading_gain_matches_oracle(cuda, oracle_mod, shape, sigma):
    rng = np.random.default_rng(3)
    ref = (1000.0 + 300.0 * rng.random(shape)).astype(np.float32)
    np.testing.assert_array_equal(extensions.shading_gain(ref, sigma), oracle_mod.shading_gain(ref, sigma))


@pytest.mark.gpu
def test_shading_correct_motion_divides_by_gain(cuda, oracle_mod):
    from paper_2403_16438_b200 import Video, synth
    from paper_2403_16438_b200.motion import MotionConfig, correct_motion, make_reference

    cfg = synth.CONFIGS["c1"].with_frames(120)
    raw = synth.generate_numpy(cfg)
    plain, vec0 = correct_motion(Video(raw), MotionConfig(search_radius=cfg.radius))
    shaded, vec1 = correct_motion(Video(raw), MotionConfig(search_radius=cfg.radius, shading_sigma=16.0))
    assert vec0 == vec1
    gain = oracle_mod.shading_gain(make_reference(Video(raw)), 16.0)
    np.testing.assert_array_equal(shaded.data, plain.data / gain[None])


@pytest.mark.gpu
def test_fused_stage_with_extensions_matches_separate_calls_and_oracle(cuda, oracle_mod):
    from paper_2403_16438_b200 import Video, synth
    from paper_2403_16438_b200.motion import MotionConfig, correct_motion
    from paper_2403_16438_b200.stage import StageConfig, preprocess
    from paper_2403_16438_b200.summarize import summarize

    cfg = synth.CONFIGS["c1"].with_frames(260)
    raw = synth.generate_numpy(cfg)
    sc = StageConfig(search_radius=cfg.radius, segment_length=100, ref_frames=50, highpass_window=33,
                     shading_sigma=16.0)
    corr, vecs, pairs = preprocess(Video(raw), sc)
    c2, v2 = correct_motion(Video(raw), MotionConfig(search_radius=cfg.radius, shading_sigma=16.0))
    assert vecs == v2
    np.testing.assert_array_equal(corr.data, c2.data)
    sep = summarize(c2, 100, highpass_window=33)
    want_tp = oracle_mod.highpass_summary(c2.data, 100, 33)
    for p, q, k in zip(pairs, sep, range(len(pairs))):
        np.testing.assert_array_equal(p.spatial, q.spatial)
        np.testing.assert_array_equal(p.temporal, q.temporal)
        np.testing.assert_array_equal(p.temporal, want_tp[k])


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [100, 200])
def test_host_stage_chunks_with_halo_equal_device_run(cuda, chunk):
    from paper_2403_16438_b200 import _device as D
    from paper_2403_16438_b200 import synth
    from paper_2403_16438_b200.stage import DevicePreprocessor, HostStage, StageConfig

    cfg = synth.CONFIGS["c1"].with_frames(450)
    raw = synth.generate_numpy(cfg)
    sc = StageConfig(search_radius=cfg.radius, segment_length=50, ref_frames=60, highpass_window=33,
                     shading_sigma=12.0)
    pre = DevicePreprocessor(cfg.height, cfg.width, sc)
    res = pre.run(D.as_device_frames(raw, cuda))
    hs = HostStage(cfg.height, cfg.width, sc, chunk_frames=chunk)
    vec, sp, tp, corr = hs.run(raw, corrected=True)
    hs.close()
    np.testing.assert_array_equal(vec, res.vectors_numpy())
    np.testing.assert_array_equal(sp, res.spatial.cpu().numpy())
    np.testing.assert_array_equal(tp, res.temporal.cpu().numpy())
    pre.close()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
def test_time_shards_with_halo_equal_single_run(cuda, world):
    """Each shard holds its frames plus the window//2 halo (recomputing the
    halo's motion); results == the single-GPU run bit-for-bit."""
    import torch

    from paper_2403_16438_b200 import _device as D
    from paper_2403_16438_b200 import _lib, synth
    from paper_2403_16438_b200.stage import DevicePreprocessor, StageConfig

    cfg = synth.CONFIGS["c1"].with_frames(500)
    raw = synth.generate_numpy(cfg)
    L, m, win = 100, 120, 33
    sc = StageConfig(search_radius=cfg.radius, segment_length=L, ref_frames=m, highpass_window=win,
                     shading_sigma=10.0)
    frames = D.as_device_frames(raw, cuda)
    pre = DevicePreprocessor(cfg.height, cfg.width, sc)
    full = pre.run(frames)
    want = (full.vectors_numpy(), full.spatial.cpu().numpy(), full.temporal.cpu().numpy())
    ref = torch.empty((cfg.height, cfg.width), dtype=torch.float32, device=cuda)
    _lib.call("vb_make_reference", frames.data_ptr(), _lib.VB_U16, raw.shape[0], cfg.height, cfg.width, m,
              ref.data_ptr(), D.stream_handle())
    for r in range(world):
        s = distributed.shard_plan(raw.shape[0], L, world, r)
        lo, hi = distributed.halo_range(s, win)
        pre.plan.set_reference(ref)
        pre.set_shading(ref)
        vec, sp, tp = pre.search_and_summarize(frames[lo:hi], t_global0=lo, t_total=raw.shape[0],
                                               interior=(s.frame_lo - lo, s.frames))
        got_vec = D.motion_to_numpy(vec, hi - lo)[s.frame_lo - lo:s.frame_hi - lo]
        np.testing.assert_array_equal(got_vec, want[0][s.frame_lo:s.frame_hi])
        np.testing.assert_array_equal(sp.cpu().numpy(), want[1][s.block_lo:s.block_hi])
        np.testing.assert_array_equal(tp.cpu().numpy(), want[2][s.block_lo:s.block_hi])
    pre.close()


@pytest.mark.gpu
def test_extension_errors(cuda):
    import torch

    from paper_2403_16438_b200.summarize import summarize, summarize_device

    with pytest.raises(ValueError, match="odd"):
        summarize(_frames((40, 8, 8)), 20, highpass_window=4)
    f = torch.zeros((100, 8, 8), dtype=torch.float32, device=cuda)
    with pytest.raises(ValueError, match="halo"):
        summarize_device(f[20:80], 20, highpass_window=9, t_global0=20, t_total=100, interior=(0, 60))
    with pytest.raises(ValueError, match="block boundary"):
        summarize_device(f, 20, t_global0=0, t_total=100, interior=(10, 40))


@pytest.mark.gpu
def test_highpass_one_frame_tail_raises_like_reference(cuda):
    """A 1-frame last block raises the reference's message (summarize.py:80)
    with the high-pass on as well as off."""
    from paper_2403_16438_b200.summarize import summarize

    frames = _frames((121, 30, 40))
    with pytest.raises(ValueError, match="at least 2 frames"):
        summarize(frames, 40, highpass_window=3)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,sigma", [((96, 128), 16.0), ((256, 512), 32.0), ((33, 70), 40.0)])
def test_shading_gain_vs_scipy(cuda, shape, sigma):
    """A17 shading gain on the CUDA path against scipy.ndimage.gaussian_filter."""
    rng = np.random.default_rng(11)
    ref = (1000.0 + 300.0 * rng.random(shape)).astype(np.float32)
    np.testing.assert_allclose(extensions.shading_gain(ref, sigma), scipy_shading_gain(ref, sigma), rtol=1e-4)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,L,win", [((300, 40, 72), 100, 33), ((250, 33, 70), 64, 9), ((20, 24, 24), 10, 33)])
def test_highpass_summary_vs_scipy(cuda, shape, L, win):
    """A17 high-passed temporal summary on the CUDA path against
    x - scipy.ndimage.uniform_filter1d(x, N, axis=0, mode="reflect") of the
    reference's smoothed stack, then max - median, within 1e-4."""
    from paper_2403_16438_b200.summarize import summarize

    frames = _frames(shape)
    got = np.stack([p.temporal for p in summarize(frames, L, highpass_window=win)])
    want = scipy_highpass_summary(frames, L, win)
    np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-4 * np.abs(frames).max())
