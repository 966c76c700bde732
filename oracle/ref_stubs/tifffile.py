"""Import-only stand-in for `tifffile` (absent in this image; no network).

Test infrastructure only. The reference imports tifffile at module top level
(voltseg/video_io.py:16, voltseg/summarize.py:15) but never calls it on the
motion/summary hot path. Any call raises so a stray use fails loudly.
"""


def _unavailable(*_a, **_k):
    raise RuntimeError("tifffile is not installed in this image (stub)")


imwrite = imread = _unavailable


class TiffFile:  # noqa: D401 - stub
    def __init__(self, *_a, **_k):
        _unavailable()


class TiffWriter(TiffFile):
    pass
