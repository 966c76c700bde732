"""CPU restatement of voltseg.unet's inference path -- TEST INFRASTRUCTURE
ONLY (imported by tests/, never by the product package).

  forward_batch   unet.py:154-178  float64 direct 3x3 convolution (zero
                  padding per patch), ReLU, 2x2 max-pool, nearest upsample +
                  skip concat, 1x1 conv, sigmoid
  normalize_pair  unet.py:186-196  numpy "linear" percentiles (restated from
                  numpy's _quantile: virtual index n*q + (1 - q) - 1, float32
                  neighbour difference, _lerp with the t >= 0.5 branch)
  tile_and_merge  unet.py:199-245  tile positions, numpy "reflect" padding,
                  float64 tent-weighted blend in tile order, clip

Pinned against the reference by tests/golden/unet.npz (make_golden.py).
"""
from __future__ import annotations

import math

import numpy as np

PATCH = 64
WIDTHS = (16, 32, 64)


def _conv(x: np.ndarray, kernel: np.ndarray, bias: np.ndarray) -> np.ndarray:
    """x (C, H, W) float64 -> (Cout, H, W): sum over taps of shifted slices."""
    cout, cin, k, _ = kernel.shape
    c, h, w = x.shape
    r = k // 2
    xp = np.zeros((c, h + 2 * r, w + 2 * r))
    xp[:, r:r + h, r:r + w] = x
    out = np.zeros((cout, h, w))
    for ky in range(k):
        for kx in range(k):
            win = xp[:, ky:ky + h, kx:kx + w].reshape(c, -1)
            out += (kernel[:, :, ky, kx].astype(np.float64) @ win).reshape(cout, h, w)
    return out + bias.astype(np.float64)[:, None, None]


def forward(tensors: dict, patch: np.ndarray) -> np.ndarray:
    x = np.asarray(patch, dtype=np.float64)
    skips = []

    def block(x, name):
        x = np.maximum(_conv(x, tensors[f"{name}.conv1.kernel"], tensors[f"{name}.conv1.bias"]), 0)
        return np.maximum(_conv(x, tensors[f"{name}.conv2.kernel"], tensors[f"{name}.conv2.bias"]), 0)

    for level in range(1, len(WIDTHS) + 1):
        x = block(x, f"enc{level}")
        if level < len(WIDTHS):
            skips.append(x)
            c, h, w = x.shape
            x = x.reshape(c, h // 2, 2, w // 2, 2).max(axis=(2, 4))
    for level in range(len(WIDTHS) - 1, 0, -1):
        x = np.concatenate([x.repeat(2, axis=1).repeat(2, axis=2), skips.pop()], axis=0)
        x = block(x, f"dec{level}")
    z = _conv(x, tensors["out.conv.kernel"], tensors["out.conv.bias"])[0]
    return 1.0 / (1.0 + np.exp(-z))


def forward_batch(tensors: dict, patches: np.ndarray) -> np.ndarray:
    return np.stack([forward(tensors, p) for p in patches]).astype(np.float32)


def _percentile_linear(values: np.ndarray, q: float) -> float:
    a = np.sort(np.asarray(values).ravel())
    n = a.size
    vi = n * q + (1.0 + q * (1.0 - 1.0 - 1.0)) - 1.0
    prev = math.floor(vi)
    gamma = vi - prev
    if vi >= n - 1:
        lo = hi = a[-1]
    elif vi < 0:
        lo = hi = a[0]
    else:
        lo, hi = a[prev], a[prev + 1]
    diff = float(np.subtract(hi, lo))  # in the array dtype
    if gamma >= 0.5:
        return float(hi) - diff * (1.0 - gamma)
    return float(lo) + diff * gamma


def normalize_pair(spatial: np.ndarray, temporal: np.ndarray) -> np.ndarray:
    out = np.empty((2,) + np.shape(spatial), dtype=np.float32)
    for i, ch in enumerate((spatial, temporal)):
        p1, p99 = _percentile_linear(ch, 0.01), _percentile_linear(ch, 0.99)
        if p99 <= p1:
            out[i] = 0.0
        else:
            out[i] = np.clip((np.asarray(ch, dtype=np.float64) - p1) / (p99 - p1), 0.0, 1.0)
    return out


def tile_positions(extent: int, stride: int) -> list[int]:
    pos = list(range(0, extent - PATCH + 1, stride))
    if not pos or pos[-1] != extent - PATCH:
        pos.append(extent - PATCH)
    return pos


def tent() -> np.ndarray:
    ramp = 1.0 - np.abs(np.arange(PATCH) - (PATCH - 1) / 2.0) / (PATCH / 2.0)
    return np.maximum(np.outer(ramp, ramp), 1e-3).astype(np.float32)


def _np_reflect(i: int, n: int) -> int:
    if n == 1:
        return 0
    period = 2 * (n - 1)
    m = i % period
    return m if m < n else period - m


def tile_and_merge(tensors: dict, normalized: np.ndarray, stride: int = 32) -> np.ndarray:
    c, h, w = normalized.shape
    ph, pw = max(h, PATCH), max(w, PATCH)
    ry = np.array([_np_reflect(i, h) for i in range(ph)])
    rx = np.array([_np_reflect(i, w) for i in range(pw)])
    img = np.asarray(normalized, dtype=np.float32)[:, ry][:, :, rx]
    ys, xs = tile_positions(ph, stride), tile_positions(pw, stride)
    probs = forward_batch(tensors, np.stack([img[:, y:y + PATCH, x:x + PATCH] for y in ys for x in xs]))
    t = tent()
    acc = np.zeros((ph, pw))
    nrm = np.zeros((ph, pw))
    i = 0
    for y in ys:
        for x in xs:
            acc[y:y + PATCH, x:x + PATCH] += probs[i] * t
            nrm[y:y + PATCH, x:x + PATCH] += t
            i += 1
    return np.clip((acc / nrm).astype(np.float32)[:h, :w], 0.0, 1.0)
