"""In-repo multi-page TIFF reader/writer (the reference
reads TIFF through tifffile, video_io.py:98-126, which this image lacks).
Files are also built byte by byte here (big-endian, several strips per
page, pages scattered between IFDs, BigTIFF) so the reader is checked
against the TIFF 6.0 layout, not only against its own writer.  CPU only."""
import struct

import numpy as np
import pytest

from paper_2403_16438_b200 import io, tiff


def build_tiff(pages, order="<", big=False, strips=1, extra_tags=()):
    """pages: list of 2-D arrays (or (arr, {tag: (type, values)}) overrides).
    Layout: header, then per page [gap, strips..., IFD] so data are NOT
    contiguous across pages."""
    ent, cnt, nxt, off_t = (20, "Q", "Q", 16) if big else (12, "H", "I", 4)
    out = bytearray(b"II" if order == "<" else b"MM")
    out += struct.pack(order + "HHHQ", 43, 8, 0, 0) if big else struct.pack(order + "HI", 42, 0)
    first_ptr = 8 if big else 4
    prev_next = first_ptr
    for a in pages:
        over = {}
        if isinstance(a, tuple):
            a, over = a
        a = np.asarray(a)
        h, w = a.shape[:2]
        spp = a.shape[2] if a.ndim == 3 else 1
        out += b"\xAB" * 24  # gap
        rows = -(-h // strips)
        offs, cnts = [], []
        for s in range(strips):
            chunk = a[s * rows:(s + 1) * rows]
            if chunk.size == 0:
                continue
            offs.append(len(out))
            bts = chunk.astype(chunk.dtype.newbyteorder(order)).tobytes()
            cnts.append(len(bts))
            out += bts
        if len(out) % 2:
            out += b"\0"
        kind = {"u": 1, "i": 2, "f": 3}[a.dtype.kind]
        tags = {256: (4, [w]), 257: (4, [h]), 258: (3, [a.dtype.itemsize * 8] * spp), 259: (3, [1]),
                262: (3, [1]), 273: (off_t, offs), 277: (3, [spp]), 278: (4, [rows]), 279: (off_t, cnts),
                339: (3, [kind] * spp)}
        tags.update(over)
        tags.update(dict(extra_tags))
        # out-of-line values first
        codes = {3: "H", 4: "I", 16: "Q"}
        inline = 8 if big else 4
        blobs = {}
        for tag, (typ, vals) in tags.items():
            b = struct.pack(order + codes[typ] * len(vals), *vals)
            if len(b) > inline:
                blobs[tag] = len(out)
                out += b
        ifd = len(out)
        struct.pack_into(order + ("Q" if big else "I"), out, prev_next, ifd)
        out += struct.pack(order + cnt, len(tags))
        for tag in sorted(tags):
            typ, vals = tags[tag]
            out += struct.pack(order + ("HHQ" if big else "HHI"), tag, typ, len(vals))
            if tag in blobs:
                out += struct.pack(order + ("Q" if big else "I"), blobs[tag])
            else:
                out += struct.pack(order + codes[typ] * len(vals), *vals).ljust(inline, b"\0")
        prev_next = len(out)
        out += struct.pack(order + nxt, 0)
    return bytes(out)


@pytest.mark.parametrize("dtype", [np.uint8, np.uint16, np.float32])
@pytest.mark.parametrize("t", [1, 5])
def test_writer_reader_round_trip_memmapped(tmp_path, dtype, t):
    rng = np.random.default_rng(t)
    a = (rng.random((t, 37, 53)) * 250).astype(dtype)
    p = tmp_path / "v.tif"
    tiff.write_tiff(p, a)
    b = tiff.read_tiff(p)
    assert isinstance(b, np.memmap) and b.dtype == a.dtype
    np.testing.assert_array_equal(b, a)


@pytest.mark.parametrize("order", ["<", ">"])
@pytest.mark.parametrize("big", [False, True])
@pytest.mark.parametrize("strips", [1, 3])
def test_handbuilt_layouts(tmp_path, order, big, strips):
    rng = np.random.default_rng(7)
    a = rng.integers(0, 65536, (4, 19, 23), dtype=np.uint16)
    p = tmp_path / "h.tif"
    p.write_bytes(build_tiff(list(a), order=order, big=big, strips=strips))
    b = tiff.read_tiff(p)
    assert b.dtype == np.uint16 and b.dtype.isnative
    np.testing.assert_array_equal(b, a)
    f = (rng.random((2, 8, 9)) * 1000).astype(np.float32)
    p.write_bytes(build_tiff(list(f), order=order, big=big, strips=strips))
    np.testing.assert_array_equal(tiff.read_tiff(p), f)


def _err(tmp_path, data, match):
    p = tmp_path / "bad.tif"
    p.write_bytes(data)
    with pytest.raises(io.VideoIOError, match=match):
        io.load_video(p)


def test_reference_error_texts(tmp_path):
    """video_io.py:98-126 messages."""
    a = np.zeros((6, 7), np.uint16)
    _err(tmp_path, build_tiff([]), "TIFF has no pages")
    _err(tmp_path, build_tiff([np.zeros((6, 7, 3), np.uint8)]), r"page 0 is not grayscale \(shape \(6, 7, 3\)\)")
    _err(tmp_path, build_tiff([np.zeros((6, 7), np.int16)]), "page 0 has unsupported sample format int16")
    _err(tmp_path, build_tiff([a, np.zeros((6, 8), np.uint16)]), r"page 1 has size \(6, 8\), expected \(6, 7\)")
    _err(tmp_path, build_tiff([a, np.zeros((6, 7), np.uint8)]), "page 1 has sample format uint8")
    _err(tmp_path, build_tiff([(a, {259: (3, [5])})]), "unreadable TIFF: compression 5")
    _err(tmp_path, b"II*\0" + b"\xff" * 4, "unreadable TIFF")
    _err(tmp_path, b"not a tiff at all", "unreadable TIFF")
    with pytest.raises(io.VideoIOError, match="cannot read video file"):
        io.load_video(tmp_path / "missing.tif")


def test_load_save_video_tiff_like_reference(tmp_path):
    """save_video writes float32 pages (video_io.py:154-157); load_video reads
    them back identically; a uint16 TIFF widens to the same float32 values."""
    from paper_2403_16438_b200 import Video

    rng = np.random.default_rng(3)
    raw = rng.integers(0, 4096, (9, 20, 24), dtype=np.uint16)
    v = Video(raw)
    io.save_video(v, tmp_path / "a.tif")
    back = io.load_video(tmp_path / "a.tif")
    np.testing.assert_array_equal(back.data, raw.astype(np.float32))
    io.save_video(v, tmp_path / "b.tiff", sample="u16")
    assert tiff.read_tiff(tmp_path / "b.tiff").dtype == np.uint16
    np.testing.assert_array_equal(io.load_video(tmp_path / "b.tiff").data, raw.astype(np.float32))
    rec = io.open_recording(tmp_path / "b.tiff")
    assert isinstance(rec, np.memmap) and rec.dtype == np.uint16


def test_truncated_files_raise_tiff_error(tmp_path):
    """Cuts anywhere in the file (inside an IFD entry, past the strips, in
    the header) raise TiffError, never a bare struct / index error; a cut
    that only drops the final IFD's alignment padding still reads back."""
    p = tmp_path / "a.tif"
    want = (np.arange(2 * 8 * 8) % 65535).astype(np.uint16).reshape(2, 8, 8)
    tiff.write_tiff(p, want)
    data = p.read_bytes()
    for cut in list(range(0, len(data), 7)) + [len(data) - 1]:
        q = tmp_path / "cut.tif"
        q.write_bytes(data[:cut])
        try:
            got = tiff.read_tiff(q, mmap=False)
        except tiff.TiffError:
            continue
        np.testing.assert_array_equal(got, want)
