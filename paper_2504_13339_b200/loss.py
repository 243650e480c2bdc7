"""Training loss (drop-in for ``vegsplat.loss`` on the path BASELINE.json measures).

(1 - lambda) L1 + lambda (1 - SSIM) with an 11x11 Gaussian window (sigma 1.5, K1 0.01,
K2 0.03) over valid positions, and its exact analytic adjoint
(/root/reference/pkg/src/vegsplat/loss.py:29-124,146-168), computed by the fused
``vegs_loss_l1_ssim`` kernel pair in float32.  BASELINE.json writes the loss as
``L1 + 0.2 (1 - SSIM)`` while the reference weights L1 by (1 - lambda); ``compute_loss``
keeps the reference's convention and ``l1_weight`` selects the other.

The normal-consistency and bilateral-smoothness regularisers (loss.py:175-240) are
not on the measured path (their weights are 0 in every BASELINE config); asking for
them raises ``NotImplementedError`` instead of silently dropping them.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .device import LossKernel, require_cuda
from .images import ImageBuffer
from .raster import ImageGradients

SSIM_WINDOW = 11
SSIM_SIGMA = 1.5
SSIM_K1 = 0.01
SSIM_K2 = 0.03

_KERNEL: LossKernel | None = None


def _kernel() -> LossKernel:
    global _KERNEL
    if _KERNEL is None:
        _KERNEL = LossKernel(require_cuda())
    return _KERNEL


def gaussian_window(size: int = SSIM_WINDOW, sigma: float = SSIM_SIGMA) -> np.ndarray:
    xs = np.arange(size) - (size - 1) / 2.0
    g = np.exp(-0.5 * (xs / sigma) ** 2)
    g /= g.sum()
    return np.outer(g, g)


def l1_ssim_device(x: torch.Tensor, y: torch.Tensor, w_l1: float, lam: float,
                   d_x: torch.Tensor | None = None, sums: torch.Tensor | None = None):
    """Device entry: x, y float32 (H, W, 3) CUDA tensors.  Returns (d_x, sums) where
    sums = [sum |x - y|, sum SSIM map] (float64, accumulated into if given)."""
    if x.shape != y.shape or x.dim() != 3 or x.shape[2] != 3:
        raise ValueError(f"rendered {tuple(x.shape)} vs reference {tuple(y.shape)}")
    if x.shape[0] < SSIM_WINDOW or x.shape[1] < SSIM_WINDOW:
        raise ValueError(f"images must be at least {SSIM_WINDOW}px for SSIM")
    if d_x is None:
        d_x = torch.empty_like(x)
    if sums is None:
        sums = torch.zeros(2, dtype=torch.float64, device=x.device)
    _kernel()(x.contiguous(), y.contiguous(), w_l1, lam, d_x, sums)
    return d_x, sums


def _to_dev(a) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(require_cuda())


@dataclass
class SsimCache:
    x: torch.Tensor
    y: torch.Tensor
    n_positions: int
    dtype: np.dtype


def ssim(x: np.ndarray, y: np.ndarray) -> tuple[float, SsimCache]:
    """Mean SSIM over valid window positions of (H, W, 3) images (loss.py:80-103)."""
    if x.shape != y.shape:
        raise ValueError(f"shape mismatch {x.shape} vs {y.shape}")
    if x.shape[0] < SSIM_WINDOW or x.shape[1] < SSIM_WINDOW:
        raise ValueError(f"images must be at least {SSIM_WINDOW}px for SSIM")
    xd, yd = _to_dev(x), _to_dev(y)
    _, sums = l1_ssim_device(xd, yd, 0.0, 0.0)
    n_pos = (x.shape[0] - 10) * (x.shape[1] - 10) * x.shape[2]
    return float(sums[1].item()) / n_pos, SsimCache(xd, yd, n_pos, np.asarray(x).dtype)


def ssim_backward(cache: SsimCache, upstream: float) -> np.ndarray:
    """d(upstream * mean SSIM)/dx (loss.py:106-124)."""
    d_x, _ = l1_ssim_device(cache.x, cache.y, 0.0, -float(upstream))
    return d_x.cpu().numpy().astype(cache.dtype)


@dataclass
class LossBreakdown:
    total: float
    l1: float
    ssim_term: float
    normal: float
    smooth: float

    def as_dict(self) -> dict:
        return {"total": self.total, "l1": self.l1, "ssim": self.ssim_term,
                "normal": self.normal, "smooth": self.smooth}


def compute_loss(rendered: ImageBuffer, reference_rgb: np.ndarray, config, px_scale: float = 1.0,
                 l1_weight: float | None = None) -> tuple[float, ImageGradients, LossBreakdown]:
    """Scalar loss and dL/d rgb (loss.py:146-168)."""
    rgb = rendered.rgb
    if rgb.shape != np.shape(reference_rgb):
        raise ValueError(f"rendered {rgb.shape} vs reference {np.shape(reference_rgb)}")
    if (getattr(config, "normal_loss_weight", 0.0) > 0.0 and rendered.normal is not None
            and rendered.depth is not None) or (getattr(config, "smooth_loss_weight", 0.0) > 0.0
                                               and rendered.attrs is not None):
        raise NotImplementedError("normal/smoothness regularisers are outside the B200 hot path (SURVEY §8(f))")
    lam = float(config.lambda_ssim)
    w_l1 = (1.0 - lam) if l1_weight is None else float(l1_weight)
    d_x, sums = l1_ssim_device(_to_dev(rgb), _to_dev(reference_rgb), w_l1, lam)
    n_el = rgb.size
    n_pos = (rgb.shape[0] - 10) * (rgb.shape[1] - 10) * rgb.shape[2]
    s = sums.cpu().numpy()
    l1 = float(s[0]) / n_el
    ssim_term = 1.0 - float(s[1]) / n_pos
    total = w_l1 * l1 + lam * ssim_term
    grads = ImageGradients(rgb=d_x.cpu().numpy().astype(rgb.dtype))
    return total, grads, LossBreakdown(total=total, l1=l1, ssim_term=ssim_term, normal=0.0, smooth=0.0)
