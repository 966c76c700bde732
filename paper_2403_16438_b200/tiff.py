"""Multi-page grayscale TIFF reader / writer, so TIFF
recordings load without the `tifffile` package the reference delegates to
(video_io.py:98-126 read, :144-161 write; absent from this image).

Scope: baseline uncompressed TIFF (Compression = 1), one sample per pixel,
strips, in either byte order, classic (magic 42) or BigTIFF (43).  Sample
formats are the reference's _TIFF_DTYPES (video_io.py:21): uint8, uint16,
float32.  Reads return the native dtype (uint16 stays uint16: the stage
widens it exactly on the GPU); pages whose image data lie back to back in the
file are memory-mapped, so `io.preprocess_file` streams a recording from the page
cache into the C-ABI executor like a VSEGV1 file.  Error texts follow
video_io.py:98-126.
"""
from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

# tag numbers (TIFF 6.0)
_W, _H, _BPS, _COMP, _PHOTO, _STRIP_OFF, _SPP, _ROWS, _STRIP_CNT, _PLANAR, _SFMT = (
    256, 257, 258, 259, 262, 273, 277, 278, 279, 284, 339)
_TILE_W = 322
# field types: size in bytes and struct code
_TYPES = {1: (1, "B"), 2: (1, "c"), 3: (2, "H"), 4: (4, "I"), 5: (8, "II"), 6: (1, "b"), 7: (1, "B"),
          8: (2, "h"), 9: (4, "i"), 10: (8, "ii"), 11: (4, "f"), 12: (8, "d"), 16: (8, "Q"), 17: (8, "q"),
          18: (8, "Q")}
_SUPPORTED = (np.dtype(np.uint8), np.dtype(np.uint16), np.dtype(np.float32))  # video_io.py:21


class TiffError(Exception):
    pass


class _Page:
    __slots__ = ("shape", "dtype", "segments")

    def __init__(self, shape, dtype, segments):
        self.shape, self.dtype, self.segments = shape, dtype, segments  # segments: [(offset, nbytes)]


def _dtype(bps: int, sfmt: int, order: str) -> np.dtype:
    kind = {1: "u", 2: "i", 3: "f"}.get(sfmt)
    if kind is None or bps % 8:
        raise TiffError(f"sample format {sfmt} with {bps} bits")
    return np.dtype(f"{order}{kind}{bps // 8}")


def _pages(buf) -> list[_Page]:
    """Parse the IFD chain of a TIFF in `buf` (bytes-like or np.memmap);
    truncated structures raise TiffError."""
    try:
        return _parse(buf)
    except struct.error as exc:
        raise TiffError(f"truncated TIFF structure ({exc})") from None


def _parse(buf) -> list[_Page]:
    if len(buf) < 8:
        raise TiffError("file too short")
    bo = bytes(buf[:2])
    if bo not in (b"II", b"MM"):
        raise TiffError("not a TIFF file")
    e = "<" if bo == b"II" else ">"
    magic = struct.unpack_from(e + "H", buf, 2)[0]
    if magic == 42:
        big, off = False, struct.unpack_from(e + "I", buf, 4)[0]
    elif magic == 43:
        if len(buf) < 16:
            raise TiffError("file too short")
        bsz, _z, off = struct.unpack_from(e + "HHQ", buf, 4)
        if bsz != 8:
            raise TiffError("bad BigTIFF header")
        big = True
    else:
        raise TiffError(f"bad magic {magic}")
    cnt_fmt, ent_size, next_fmt, inline = ("Q", 20, "Q", 8) if big else ("H", 12, "I", 4)
    pages, seen = [], set()
    while off:
        if off in seen or off + 2 > len(buf):
            raise TiffError("corrupt IFD chain")
        seen.add(off)
        (n,) = struct.unpack_from(e + cnt_fmt, buf, off)
        p = off + struct.calcsize(cnt_fmt)
        tags = {}
        for i in range(n):
            q = p + i * ent_size
            if big:
                tag, typ, count = struct.unpack_from(e + "HHQ", buf, q)
                vpos = q + 12
            else:
                tag, typ, count = struct.unpack_from(e + "HHI", buf, q)
                vpos = q + 8
            if typ not in _TYPES:
                continue
            size, code = _TYPES[typ]
            total = size * count
            if total > inline:
                vpos = struct.unpack_from(e + ("Q" if big else "I"), buf, vpos)[0]
            if vpos + total > len(buf):
                raise TiffError(f"tag {tag} points past the end of the file")
            if typ in (1, 2, 6, 7):
                vals = bytes(buf[vpos:vpos + count])
            else:
                vals = struct.unpack_from(e + code * count, buf, vpos)
            tags[tag] = vals
        (off,) = struct.unpack_from(e + next_fmt, buf, p + n * ent_size)

        def one(tag, default=None):
            v = tags.get(tag)
            if v is None:
                if default is None:
                    raise TiffError(f"missing tag {tag}")
                return default
            return v[0]

        if _TILE_W in tags:
            raise TiffError("tiled TIFF is not supported")
        if one(_COMP, 1) != 1:
            raise TiffError(f"compression {one(_COMP)} is not supported (uncompressed only)")
        w, h, spp = one(_W), one(_H), one(_SPP, 1)
        bps_t = tags.get(_BPS, (1,))
        sf_t = tags.get(_SFMT, (1,))
        dt = _dtype(bps_t[0], sf_t[0], e)
        shape = (h, w) if spp == 1 else (h, w, spp)
        offs, cnts = tags.get(_STRIP_OFF), tags.get(_STRIP_CNT)
        if offs is None:
            raise TiffError("missing strip offsets")
        need = h * w * spp * dt.itemsize
        if cnts is None:  # a single strip may omit its byte count
            if len(offs) != 1:
                raise TiffError("missing strip byte counts")
            cnts = (need,)
        if sum(cnts) < need:
            raise TiffError(f"strips hold {sum(cnts)} bytes, image needs {need}")
        segs, left = [], need
        for o, c in zip(offs, cnts):
            c = min(c, left)
            if o + c > len(buf):
                raise TiffError("strip data past the end of the file")
            if c:
                segs.append((o, c))
            left -= c
        pages.append(_Page(shape, dt, segs))
    return pages


def read_tiff(path, mmap: bool = True) -> np.ndarray:
    """(T, H, W) stack of a multi-page grayscale TIFF in its sample dtype
    (native byte order).  Raises TiffError with the reference's texts
    (video_io.py:98-126) for pages that do not form one stack."""
    path = Path(path)
    raw = np.memmap(path, dtype=np.uint8, mode="r") if path.stat().st_size else b""
    pages = _pages(raw)
    if not pages:
        raise TiffError(f"{path}: TIFF has no pages")
    first = pages[0]
    if len(first.shape) != 2:
        raise TiffError(f"{path}: page 0 is not grayscale (shape {first.shape})")
    if first.dtype.newbyteorder("=") not in _SUPPORTED:
        raise TiffError(f"{path}: page 0 has unsupported sample format {first.dtype.newbyteorder('=')}")
    for i, pg in enumerate(pages[1:], 1):
        if pg.shape != first.shape:
            raise TiffError(f"{path}: page {i} has size {pg.shape}, expected {first.shape}")
        if pg.dtype != first.dtype:
            raise TiffError(f"{path}: page {i} has sample format {pg.dtype.newbyteorder('=')}")
    t, (h, w) = len(pages), first.shape
    nbytes = h * w * first.dtype.itemsize
    start = first.segments[0][0]
    contiguous = all(len(pg.segments) == 1 or _joined(pg.segments) for pg in pages) and all(
        pg.segments[0][0] == start + i * nbytes for i, pg in enumerate(pages))
    if contiguous and mmap and first.dtype.isnative:
        return np.memmap(path, dtype=first.dtype, mode="r", offset=start, shape=(t, h, w))
    out = np.empty((t, h, w), dtype=first.dtype.newbyteorder("="))
    flat = out.reshape(t, -1).view(np.uint8)
    for i, pg in enumerate(pages):
        pos = 0
        for o, c in pg.segments:
            flat[i, pos:pos + c] = raw[o:o + c]
            pos += c
        if not first.dtype.isnative:
            out[i] = out[i].byteswap()
    return out


def _joined(segs) -> bool:
    return all(segs[k][0] + segs[k][1] == segs[k + 1][0] for k in range(len(segs) - 1))


def write_tiff(path, data: np.ndarray) -> None:
    """Write (T, H, W) or (H, W) uint8 / uint16 / float32 as an uncompressed
    little-endian multi-page minisblack TIFF: image data back to back (so
    read_tiff memory-maps it), then one IFD per page; BigTIFF past 4 GB."""
    a = np.ascontiguousarray(data)
    if a.ndim == 2:
        a = a[None]
    if a.ndim != 3 or a.dtype not in _SUPPORTED:
        raise TiffError(f"cannot write a {a.ndim}-D {a.dtype} stack as TIFF")
    a = a.astype(a.dtype.newbyteorder("<"), copy=False)
    t, h, w = a.shape
    page = h * w * a.dtype.itemsize
    sfmt = 3 if a.dtype.kind == "f" else 1
    bps = a.dtype.itemsize * 8
    n_tags = 10
    big = 16 + t * page + t * (8 + 20 * n_tags + 8) >= 2 ** 32
    data_off = 16 if big else 8
    ifd0 = data_off + t * page
    ifd0 += (-ifd0) % 8  # word-aligned IFDs
    ent, cnt_fmt, nxt_fmt = (20, "<Q", "<Q") if big else (12, "<H", "<I")
    ifd_size = struct.calcsize(cnt_fmt) + n_tags * ent + struct.calcsize(nxt_fmt)
    ifd_size += (-ifd_size) % 8
    with open(path, "wb") as f:
        f.write(b"II" + (struct.pack("<HHHQ", 43, 8, 0, ifd0) if big else struct.pack("<HI", 42, ifd0)))
        f.write(a.tobytes())
        f.write(b"\0" * (ifd0 - data_off - t * page))
        for i in range(t):
            entries = [(_W, 4, w), (_H, 4, h), (_BPS, 3, bps), (_COMP, 3, 1), (_PHOTO, 3, 1),
                       (_STRIP_OFF, 16 if big else 4, data_off + i * page), (_SPP, 3, 1), (_ROWS, 4, h),
                       (_STRIP_CNT, 16 if big else 4, page), (_SFMT, 3, sfmt)]
            b = bytearray(struct.pack(cnt_fmt, len(entries)))
            for tag, typ, val in entries:
                code = _TYPES[typ][1]
                if big:
                    b += struct.pack("<HHQ", tag, typ, 1) + struct.pack("<" + code, val).ljust(8, b"\0")
                else:
                    b += struct.pack("<HHI", tag, typ, 1) + struct.pack("<" + code, val).ljust(4, b"\0")
            nxt = ifd0 + (i + 1) * ifd_size if i + 1 < t else 0
            b += struct.pack(nxt_fmt, nxt)
            b += b"\0" * (ifd_size - len(b))
            f.write(bytes(b))
