"""Seeded synthetic voltage-imaging recordings (BASELINE.json `configs`).

The paper's recordings are not available offline, so the
bench and the parity tests use this generator.  Model:
  tissue_t = smooth Gaussian-field background (~1000 counts, +-100)
           + sum_k amp_k * a_k(t) * footprint_k      (elliptical Gaussians)
  a_k(t)   = 1 + 1/f subthreshold (~2 %) + Poisson spikes (2-frame +spike_amp)
  frame_t  = vignetting_gain * shift(tissue_t, drift_t)   (bilinear, sub-pixel)
  counts   = round(Poisson(frame_t) + N(0, read_noise^2)) clipped to uint16
Drift is a clipped random walk with sub-pixel steps, optional jumps and jitter.
Runs with torch on CPU (tests) or CUDA (bench); each device is deterministic
for a given seed (the two devices draw different streams).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, replace

import numpy as np
import torch
import torch.nn.functional as F


@dataclass(frozen=True)
class SynthConfig:
    name: str
    frames: int
    height: int
    width: int
    neurons: int
    radius: int            # motion search radius used by the stage for this config
    segment_length: int    # summary block L
    ref_frames: int = 100  # template M
    sigma_px: tuple = (3.0, 5.0)
    overlap_frac: float = 0.0
    drift_px: float = 3.0
    drift_step: float = 0.3
    jump_prob: float = 0.0
    jump_px: float = 0.0
    jitter_px: float = 0.0
    rate_hz: tuple = (5.0, 5.0)   # (lo, hi) log-uniform per neuron
    spike_amp: float = 0.2
    neuron_amp: float = 100.0
    background: float = 1000.0
    read_noise: float = 5.0
    fps: float = 741.0
    seed: int = 1001

    def with_frames(self, frames: int) -> "SynthConfig":
        return replace(self, frames=frames)


# BASELINE.json configs[0..4] (seeds 1001..1005).
CONFIGS = {
    "c1": SynthConfig("c1", 1000, 128, 128, 8, radius=5, segment_length=500, drift_px=3.0, seed=1001),
    "c2": SynthConfig("c2", 10000, 256, 512, 30, radius=8, segment_length=1000, overlap_frac=0.2,
                      drift_px=5.0, seed=1002),
    "c3": SynthConfig("c3", 20000, 512, 512, 60, radius=12, segment_length=1000, sigma_px=(4.0, 8.0),
                      drift_px=10.0, jump_prob=0.002, jump_px=3.0, spike_amp=0.05, neuron_amp=200.0,
                      seed=1003),
    "c4": SynthConfig("c4", 100000, 512, 512, 80, radius=10, segment_length=1000, drift_px=8.0,
                      rate_hz=(2.0, 20.0), seed=1004),
    "c5": SynthConfig("c5", 20000, 1024, 1024, 300, radius=10, segment_length=1000, sigma_px=(3.0, 6.0),
                      overlap_frac=0.4, drift_px=6.0, jitter_px=0.3, seed=1005),
}


@dataclass
class SynthTruth:
    drift: np.ndarray        # (T, 2) float64 true (x, y) shift of the tissue
    centers: np.ndarray      # (K, 2)
    spikes: np.ndarray       # (T, K) bool


def _smooth_field(h, w, sigma, gen, device):
    noise = torch.randn((h, w), generator=gen, device=device)
    fy = torch.fft.fftfreq(h, device=device)[:, None]
    fx = torch.fft.fftfreq(w, device=device)[None, :]
    filt = torch.exp(-2 * (math.pi ** 2) * (sigma ** 2) * (fx ** 2 + fy ** 2))
    field = torch.fft.ifft2(torch.fft.fft2(noise) * filt).real
    field = field - field.mean()
    return field / (field.abs().max() + 1e-12)


def _drift(cfg: SynthConfig, gen, device) -> torch.Tensor:
    """Clipped random walk of the tissue position (x, y), sub-pixel steps."""
    t = cfg.frames
    steps = torch.randn((t, 2), generator=gen, device=device, dtype=torch.float64) * cfg.drift_step
    if cfg.jump_prob > 0:
        jumps = torch.rand((t, 2), generator=gen, device=device, dtype=torch.float64) < cfg.jump_prob
        sign = torch.where(torch.rand((t, 2), generator=gen, device=device, dtype=torch.float64) < 0.5, -1.0, 1.0)
        steps = steps + jumps * sign * cfg.jump_px
    st = steps.cpu().numpy()
    pos = np.zeros((t, 2))
    for i in range(1, t):  # sequential by definition; cheap on the host
        pos[i] = np.clip(pos[i - 1] + st[i], -cfg.drift_px, cfg.drift_px)
    out = torch.from_numpy(pos).to(device)
    if cfg.jitter_px > 0:
        out = out + torch.randn((t, 2), generator=gen, device=device, dtype=torch.float64) * cfg.jitter_px
    return out


def _one_over_f(t, k, gen, device):
    white = torch.randn((k, t), generator=gen, device=device)
    spec = torch.fft.rfft(white, dim=1)
    f = torch.fft.rfftfreq(t, device=device)
    f[0] = f[1] if t > 1 else 1.0
    x = torch.fft.irfft(spec / torch.sqrt(f), n=t, dim=1)
    return (x / (x.std(dim=1, keepdim=True) + 1e-12)).T  # (t, k), unit std


def generate(cfg: SynthConfig, device="cpu", chunk: int = 256, return_truth: bool = False):
    """uint16 (T, H, W) recording on `device` (torch tensor, dtype torch.uint16)."""
    device = torch.device(device)
    gen = torch.Generator(device=device)
    gen.manual_seed(cfg.seed)
    h, w, t, k = cfg.height, cfg.width, cfg.frames, cfg.neurons
    # static scene
    bg = cfg.background + 100.0 * _smooth_field(h, w, min(h, w) / 8.0, gen, device)
    yy = torch.arange(h, device=device, dtype=torch.float32)[:, None]
    xx = torch.arange(w, device=device, dtype=torch.float32)[None, :]
    rr = ((yy - (h - 1) / 2) ** 2 + (xx - (w - 1) / 2) ** 2) / (((h - 1) / 2) ** 2 + ((w - 1) / 2) ** 2)
    gain = 1.0 - 0.3 * rr  # vignetting 1.0 centre -> 0.7 corners
    u = torch.rand((k, 6), generator=gen, device=device)
    margin = 10.0
    cx = margin + u[:, 0] * (w - 2 * margin)
    cy = margin + u[:, 1] * (h - 2 * margin)
    n_ov = int(round(cfg.overlap_frac * k))
    for i in range(1, min(n_ov + 1, k)):  # place overlapping neurons next to a predecessor
        cx[i] = cx[i - 1] + (u[i, 0] - 0.5) * 2 * cfg.sigma_px[0]
        cy[i] = cy[i - 1] + (u[i, 1] - 0.5) * 2 * cfg.sigma_px[0]
    lo, hi = cfg.sigma_px
    sx = lo + u[:, 2] * (hi - lo)
    sy = lo + u[:, 3] * (hi - lo)
    th = u[:, 4] * math.pi
    dx = xx[None] - cx[:, None, None]
    dy = yy[None] - cy[:, None, None]
    c, s = torch.cos(th)[:, None, None], torch.sin(th)[:, None, None]
    xr, yr = c * dx + s * dy, -s * dx + c * dy
    foot = torch.exp(-0.5 * ((xr / sx[:, None, None]) ** 2 + (yr / sy[:, None, None]) ** 2))  # (k,h,w)
    foot = foot.reshape(k, h * w)
    # activity
    rlo, rhi = cfg.rate_hz
    rates = torch.exp(math.log(rlo) + u[:, 5] * (math.log(rhi) - math.log(rlo)))
    p = (rates / cfg.fps).clamp(max=0.5)
    ev = torch.rand((t, k), generator=gen, device=device) < p[None]
    spikes = ev.clone()
    spikes[1:] |= ev[:-1]  # 2-frame transient
    act = 1.0 + 0.02 * _one_over_f(t, k, gen, device) + cfg.spike_amp * spikes.float()  # (t,k)
    drift = _drift(cfg, gen, device)
    out = torch.empty((t, h, w), dtype=torch.int16, device=device)
    amp = cfg.neuron_amp
    for t0 in range(0, t, chunk):
        t1 = min(t, t0 + chunk)
        n = t1 - t0
        tissue = (bg.reshape(1, h * w) + amp * (act[t0:t1] @ foot)).reshape(n, 1, h, w)
        # frame(x, y) = tissue(x - sx, y - sy): sample with border clamp
        theta = torch.zeros((n, 2, 3), device=device)
        theta[:, 0, 0] = 1.0
        theta[:, 1, 1] = 1.0
        theta[:, 0, 2] = (-drift[t0:t1, 0] * 2.0 / max(w - 1, 1)).float()
        theta[:, 1, 2] = (-drift[t0:t1, 1] * 2.0 / max(h - 1, 1)).float()
        grid = F.affine_grid(theta, (n, 1, h, w), align_corners=True)
        shifted = F.grid_sample(tissue, grid, mode="bilinear", padding_mode="border", align_corners=True)
        lam = (shifted[:, 0] * gain).clamp(min=0)
        counts = torch.poisson(lam, generator=gen) + cfg.read_noise * torch.randn(lam.shape, generator=gen,
                                                                                  device=device)
        counts = counts.round().clamp(0, 65535).to(torch.int32)
        out[t0:t1] = counts.to(torch.int16)  # bit pattern of the uint16 value
    video = out.view(torch.uint16)
    if return_truth:
        return video, SynthTruth(drift.cpu().numpy(), torch.stack([cx, cy], 1).cpu().numpy(), spikes.cpu().numpy())
    return video


def generate_numpy(cfg: SynthConfig, return_truth: bool = False):
    """CPU generation -> numpy uint16 (T, H, W)."""
    r = generate(cfg, "cpu", return_truth=return_truth)
    if return_truth:
        v, truth = r
        return v.view(torch.int16).numpy().view(np.uint16), truth
    return r.view(torch.int16).numpy().view(np.uint16)
