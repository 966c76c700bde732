"""VSEGV1 ingest: byte-compatible with the reference's
video_io for float32 files, the uint16 extension round-trips; CPU only."""
import numpy as np
import pytest

from paper_2403_16438_b200 import Video, io, synth


def _ref_video_io():
    from oracle import ref
    if not ref.available():
        pytest.skip("reference not built (oracle/build_ref.sh)")
    return ref.load()[3]


def test_f32_files_interchange_with_reference(tmp_path, rng):
    vio = _ref_video_io()
    data = (rng.random((7, 9, 11), dtype=np.float32) * 100).astype(np.float32)
    vio.save_video(vio.Video(data, frame_rate=741.0), tmp_path / "ref.vsegv1")
    ours = io.load_video(tmp_path / "ref.vsegv1")
    np.testing.assert_array_equal(ours.data, data)
    assert ours.frame_rate == 741.0
    io.save_video(Video(data, frame_rate=500.0), tmp_path / "ours.vsegv1", sample="f32")
    back = vio.load_video(tmp_path / "ours.vsegv1")
    np.testing.assert_array_equal(back.data, data)
    assert back.frame_rate == 500.0
    assert (tmp_path / "ref.vsegv1").read_bytes()[32:] == (tmp_path / "ours.vsegv1").read_bytes()[32:]


def test_u16_extension_round_trip_and_memmap(tmp_path):
    raw = synth.generate_numpy(synth.CONFIGS["c1"].with_frames(12))
    io.save_video(Video(raw, frame_rate=741.0), tmp_path / "c.vsegv1")
    assert (tmp_path / "c.vsegv1").stat().st_size == 32 + raw.nbytes  # 2 B/sample
    t, h, w, fmt, rate = io.read_header(tmp_path / "c.vsegv1")
    assert (t, h, w, fmt, rate) == (12, 128, 128, io.SAMPLE_U16, 741.0)
    mm, _ = io.open_raw(tmp_path / "c.vsegv1")
    assert isinstance(mm, np.memmap) and mm.dtype == np.uint16
    np.testing.assert_array_equal(mm, raw)
    v = io.load_video(tmp_path / "c.vsegv1")
    assert v.raw is not None and v.data.dtype == np.float32
    np.testing.assert_array_equal(v.data, raw.astype(np.float32))


@pytest.mark.parametrize("mutate,msg", [
    (lambda b: b[:20], "truncated"),
    (lambda b: b[:-2], "expected"),
    (lambda b: b[:20] + b"\x09\x00\x00\x00" + b[24:], "sample-format"),
    (lambda b: b"NOTVSEG\0" + b[8:], "not a VSEGV1"),
])
def test_header_errors(tmp_path, mutate, msg):
    io.save_video(Video(np.ones((2, 3, 4), np.float32)), tmp_path / "a.vsegv1")
    p = tmp_path / "b.vsegv1"
    p.write_bytes(mutate((tmp_path / "a.vsegv1").read_bytes()))
    with pytest.raises(io.VideoIOError, match=msg):
        io.read_header(p)


def test_missing_and_nonint_u16(tmp_path):
    with pytest.raises(io.VideoIOError, match="cannot read"):
        io.load_video(tmp_path / "nope.vsegv1")
    with pytest.raises(io.VideoIOError, match="16-bit"):
        io.save_video(Video(np.full((2, 2, 2), 0.5, np.float32)), tmp_path / "x.vsegv1", sample="u16")
