"""Import-only stand-in for skimage.measure (used by voltseg/footprints.py:15, off the hot path)."""


def _unavailable(*_a, **_k):
    raise RuntimeError("scikit-image is not installed in this image (stub)")


label = regionprops = _unavailable
