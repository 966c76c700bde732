"""Summary normalisation + lightweight U-Net tiles on the B200 (SURVEY 8(f)
row 2): the consumer of the per-block summary pairs in the reference pipeline
(pipeline.py:222-223).  Mirrors voltseg.unet (unet.py) name for name; the
forward pass, the percentile normalisation and the tiled merge run in
libvoltb200 (csrc/unet.cu), the weight container and the VSEGW1 format are
host code.

Reference: unet.py:1-295 (architecture :34-54, WeightBundle :69-104,
forward_batch :154-178, normalize_pair :186-196, tile_and_merge :212-245,
save/load_weights :248-295).
"""
from __future__ import annotations

import ctypes as C
import struct
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np
import torch

from . import _device as D
from . import _lib

PATCH = 64
IN_CHANNELS = 2
ENCODER_WIDTHS = (16, 32, 64)
DEFAULT_STRIDE = 32
MERGE_WEIGHT_FLOOR = 1e-3

WEIGHT_MAGIC = b"VSEGW1\0\0"


class WeightFormatError(Exception):
    """Raised when a weight file does not match the VSEGW1 format or the
    canonical architecture (unet.py:28-30)."""


def _conv_layers() -> list[tuple[str, int, int, int]]:
    """(layer name, in channels, out channels, kernel size) in graph order:
    two 3x3 convs per encoder level, two per decoder level (the first one
    reads upsample(previous) ++ skip), then the 1x1 output conv."""
    layers = []
    widths = ENCODER_WIDTHS
    prev = IN_CHANNELS
    for i, width in enumerate(widths):
        layers += [(f"enc{i + 1}.conv1", prev, width, 3), (f"enc{i + 1}.conv2", width, width, 3)]
        prev = width
    for i in reversed(range(1, len(widths))):
        skip = widths[i - 1]
        layers += [(f"dec{i}.conv1", prev + skip, skip, 3), (f"dec{i}.conv2", skip, skip, 3)]
        prev = skip
    layers.append(("out.conv", prev, 1, 1))
    return layers


def architecture() -> list[tuple[str, tuple[int, ...]]]:
    """Ordered (name, shape) list of the canonical parameter tensors
    (unet.py:34-54); kernels are (out_channels, in_channels, ky, kx), each
    followed by its bias."""
    out: list[tuple[str, tuple[int, ...]]] = []
    for name, cin, cout, k in _conv_layers():
        out.append((name + ".kernel", (cout, cin, k, k)))
        out.append((name + ".bias", (cout,)))
    return out


def architecture_fingerprint() -> str:
    """Stable identifier tying weight files to the layer graph (unet.py:57-60)."""
    body = ";".join("{}:{}".format(name, "x".join(str(d) for d in shape)) for name, shape in architecture())
    return "vseg-unet/{0}x{0}x{1};".format(PATCH, IN_CHANNELS) + body


def parameter_count() -> int:
    return int(sum(np.prod(shape) for _, shape in architecture()))


@dataclass
class WeightBundle:
    """Named parameter tensors matching the canonical architecture (unet.py:69-104)."""

    tensors: dict[str, np.ndarray]
    fingerprint: str = field(default_factory=architecture_fingerprint)

    def validate(self) -> None:
        """The reference's checks and messages, in its order: presence and
        shape per canonical tensor, no extras, finite values, fingerprint."""
        spec = dict(architecture())
        for name, shape in spec.items():
            arr = self.tensors.get(name)
            if arr is None:
                raise WeightFormatError(f"missing tensor {name!r}")
            if tuple(arr.shape) != shape:
                raise WeightFormatError(f"tensor {name!r} has shape {tuple(arr.shape)}, expected {shape}")
        unknown = sorted(set(self.tensors).difference(spec))
        if unknown:
            raise WeightFormatError(f"unexpected tensors: {unknown}")
        bad = next((n for n, v in self.tensors.items() if not np.isfinite(v).all()), None)
        if bad is not None:
            raise WeightFormatError(f"tensor {bad!r} contains non-finite values")
        if self.fingerprint != architecture_fingerprint():
            raise WeightFormatError("architecture fingerprint mismatch")

    @classmethod
    def zeros(cls) -> "WeightBundle":
        return cls({name: np.zeros(shape, np.float32) for name, shape in architecture()})

    @classmethod
    def random(cls, rng: np.random.Generator, scale: float = 0.1) -> "WeightBundle":
        """Same draws, in the same order, as the reference (standard normal x scale)."""
        tensors = {}
        for name, shape in architecture():
            tensors[name] = (rng.standard_normal(shape) * scale).astype(np.float32)
        return cls(tensors)

    def flat(self) -> np.ndarray:
        """The parameters in architecture() order (the vb_unet_create layout)."""
        self.validate()
        return np.ascontiguousarray(np.concatenate(
            [np.asarray(self.tensors[n], dtype=np.float32).ravel() for n, _ in architecture()]))


@dataclass(frozen=True)
class ProbabilityMap:
    segment_index: int
    values: np.ndarray  # (H, W) in [0, 1]


class DeviceUNet:
    """A WeightBundle uploaded once (vb_unet handle) for repeated device calls."""

    def __init__(self, weights: WeightBundle):
        flat = weights.flat()
        lib = _lib.load()
        if flat.size != int(lib.vb_unet_param_count()):
            raise WeightFormatError("parameter count mismatch with the device network")
        D.require_cuda()
        h = C.c_void_p()
        _lib.call("vb_unet_create", C.byref(h), flat.ctypes.data, flat.size)
        self._h = h

    @property
    def handle(self):
        return self._h

    def forward_device(self, patches: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        n = patches.shape[0]
        probs = out if out is not None else torch.empty((n, PATCH, PATCH), dtype=torch.float32,
                                                        device=patches.device)
        _lib.call("vb_unet_forward", self._h, patches.data_ptr(), n, probs.data_ptr(), D.stream_handle())
        return probs

    def tile_merge_device(self, normalized: torch.Tensor, stride: int = DEFAULT_STRIDE,
                          out: torch.Tensor | None = None) -> torch.Tensor:
        """normalized [K, 2, H, W] float32 device -> probability maps [K, H, W]."""
        k, _, h, w = normalized.shape
        prob = out if out is not None else torch.empty((k, h, w), dtype=torch.float32, device=normalized.device)
        _lib.call("vb_unet_tile_merge", self._h, normalized.data_ptr(), k, h, w, int(stride), prob.data_ptr(),
                  D.stream_handle())
        return prob

    def segment_device(self, spatial: torch.Tensor, temporal: torch.Tensor, stride: int = DEFAULT_STRIDE,
                       normalized_out: torch.Tensor | None = None, out: torch.Tensor | None = None) -> torch.Tensor:
        """normalize_pair + tile_and_merge for K device summary pairs [K, H, W] -> [K, H, W]
        (the pipeline.py:222-223 step for every block at once)."""
        k, h, w = spatial.shape
        prob = out if out is not None else torch.empty((k, h, w), dtype=torch.float32, device=spatial.device)
        _lib.call("vb_unet_segment", self._h, spatial.data_ptr(), temporal.data_ptr(), k, h, w, int(stride),
                  D.ptr(normalized_out), prob.data_ptr(), D.stream_handle())
        return prob

    def close(self):
        if getattr(self, "_h", None) is not None:
            _lib.load().vb_unet_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_cache: dict[int, tuple[WeightBundle, DeviceUNet]] = {}
_CACHE_MAX = 4  # device copies kept for the module-level functions (least recently used dropped)


def _device_net(weights: WeightBundle) -> DeviceUNet:
    """The uploaded copy of `weights` (keyed by identity: mutate a bundle's
    tensors in place and the cached upload is stale -- build a DeviceUNet
    explicitly for that)."""
    hit = _cache.pop(id(weights), None)
    if hit is None or hit[0] is not weights:
        hit = (weights, DeviceUNet(weights))
    _cache[id(weights)] = hit  # most recently used last
    while len(_cache) > _CACHE_MAX:
        _cache.pop(next(iter(_cache)))[1].close()
    return hit[1]


def _tile_count(height: int, width: int, stride: int = DEFAULT_STRIDE) -> int:
    """Patches tile_and_merge runs on one (height, width) image (unet.py:199-203, :223-227)."""
    def n(extent):
        extent = max(extent, PATCH)
        k = len(range(0, extent - PATCH + 1, stride))
        return k + (0 if (k - 1) * stride == extent - PATCH else 1)
    return n(height) * n(width)


def _f32_device(a) -> torch.Tensor:
    dev = D.require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=torch.float32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(dev)


def forward_batch(weights: WeightBundle, patches: np.ndarray) -> np.ndarray:
    """(N, 2, 64, 64) patches -> (N, 64, 64) probabilities (unet.py:154-178)."""
    x = np.asarray(patches, dtype=np.float32)
    if x.ndim != 4 or x.shape[1:] != (IN_CHANNELS, PATCH, PATCH):
        raise ValueError(f"expected (N, {IN_CHANNELS}, {PATCH}, {PATCH}) input, got {x.shape}")
    net = _device_net(weights)
    return net.forward_device(_f32_device(x)).cpu().numpy()


def forward(weights: WeightBundle, patch: np.ndarray) -> np.ndarray:
    """Single (2, 64, 64) patch -> (64, 64) probabilities (unet.py:181-183)."""
    return forward_batch(weights, np.asarray(patch)[None])[0]


def normalize_pair(spatial: np.ndarray, temporal: np.ndarray) -> np.ndarray:
    """Robust per-channel scaling to [0, 1] by the 1st/99th percentiles; a
    constant channel maps to all zeros (unet.py:186-196)."""
    sp, tp = _f32_device(spatial), _f32_device(temporal)
    if sp.shape != tp.shape or sp.dim() != 2:
        raise ValueError("spatial and temporal summaries must be 2-D images of one shape")
    h, w = sp.shape
    out = torch.empty((1, 2, h, w), dtype=torch.float32, device=sp.device)
    _lib.call("vb_normalize_pair", sp.data_ptr(), tp.data_ptr(), 1, h, w, out.data_ptr(), D.stream_handle())
    return out[0].cpu().numpy()


def tile_and_merge(weights: WeightBundle, normalized: np.ndarray, segment_index: int = 0,
                   stride: int = DEFAULT_STRIDE) -> ProbabilityMap:
    """Sliding 64x64 patches blended with centre-peaked tent weights into one
    frame-sized probability map (unet.py:212-245)."""
    x = _f32_device(normalized)
    if x.dim() != 3 or x.shape[0] != IN_CHANNELS:
        raise ValueError(f"expected ({IN_CHANNELS}, H, W) normalised channels, got {tuple(x.shape)}")
    prob = _device_net(weights).tile_merge_device(x[None], stride)
    return ProbabilityMap(segment_index, prob[0].cpu().numpy())


def segment_pairs(weights: WeightBundle, pairs, stride: int = DEFAULT_STRIDE) -> list[ProbabilityMap]:
    """normalize_pair + tile_and_merge for every SummaryPair at once, as
    pipeline.py:222-223 does per segment."""
    if not pairs:
        return []
    sp = _f32_device(np.stack([p.spatial for p in pairs]))
    tp = _f32_device(np.stack([p.temporal for p in pairs]))
    prob = _device_net(weights).segment_device(sp, tp, stride).cpu().numpy()
    return [ProbabilityMap(p.segment_index, prob[i]) for i, p in enumerate(pairs)]


class _Reader:
    """Bounds-checked little-endian cursor over a VSEGW1 byte string."""

    def __init__(self, raw: bytes, path):
        self.raw, self.pos, self.path = raw, 0, path

    def bytes(self, n: int, what: str) -> bytes:
        end = self.pos + n
        if end > len(self.raw):
            raise WeightFormatError(f"{self.path}: truncated reading {what} at byte {self.pos}")
        out, self.pos = self.raw[self.pos:end], end
        return out

    def u32(self, what: str, count: int = 1):
        vals = struct.unpack(f"<{count}I", self.bytes(4 * count, what))
        return vals[0] if count == 1 else vals


def save_weights(bundle: WeightBundle, path: str | Path) -> None:
    """Serialize to VSEGW1 (unet.py:248-263): magic, tensor count, fingerprint,
    then per canonical tensor its name, rank, dims and little-endian f32 data."""
    bundle.validate()
    out = bytearray(WEIGHT_MAGIC)
    fp = bundle.fingerprint.encode()
    out += struct.pack("<II", len(bundle.tensors), len(fp)) + fp
    for name, _ in architecture():
        arr = np.ascontiguousarray(bundle.tensors[name], dtype="<f4")
        key = name.encode()
        out += struct.pack("<I", len(key)) + key
        out += struct.pack(f"<I{arr.ndim}I", arr.ndim, *arr.shape)
        out += arr.tobytes()
    Path(path).write_bytes(bytes(out))


def load_weights(path: str | Path) -> WeightBundle:
    """Read and validate a VSEGW1 weight file (unet.py:266-295; same errors)."""
    rd = _Reader(Path(path).read_bytes(), path)
    if rd.bytes(8, "magic") != WEIGHT_MAGIC:
        raise WeightFormatError(f"{path}: bad magic bytes")
    count = rd.u32("tensor count")
    fingerprint = rd.bytes(rd.u32("fingerprint length"), "fingerprint").decode()
    tensors: dict[str, np.ndarray] = {}
    for _ in range(count):
        name = rd.bytes(rd.u32("name length"), "tensor name").decode()
        ndim = rd.u32(f"ndim of {name}")
        dims = rd.u32(f"dims of {name}", ndim) if ndim != 1 else (rd.u32(f"dims of {name}"),)
        if ndim == 0:
            dims = ()
        data = rd.bytes(4 * int(np.prod(dims)), f"values of {name}")
        tensors[name] = np.frombuffer(data, dtype="<f4").reshape(dims).copy()
    if rd.pos != len(rd.raw):
        raise WeightFormatError(f"{path}: {len(rd.raw) - rd.pos} trailing bytes at byte {rd.pos}")
    bundle = WeightBundle(tensors, fingerprint)
    bundle.validate()
    return bundle
