"""Training loss (drop-in for ``vegsplat.loss`` on the path BASELINE.json measures).

(1 - lambda) L1 + lambda (1 - SSIM) with an 11x11 Gaussian window (sigma 1.5, K1 0.01,
K2 0.03) over valid positions, and its exact analytic adjoint
(/root/reference/pkg/src/vegsplat/loss.py:29-124,146-168), computed by the fused
``vegs_loss_l1_ssim`` kernel pair in float32.  BASELINE.json writes the loss as
``L1 + 0.2 (1 - SSIM)`` while the reference weights L1 by (1 - lambda); ``compute_loss``
keeps the reference's convention and ``l1_weight`` selects the other.

The normal-consistency and bilateral-smoothness regularisers (loss.py:175-240) run in
``vegs_loss_aux`` on the auxiliary planes (depth, normal, attrs) when the rendered
buffer carries them, exactly as the reference applies them (weights from the config;
0 in every BASELINE config).
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
    if x.shape[:2] != y.shape[:2] or x.dim() != 3 or x.shape[2] < 3 or y.shape[2] != 3:
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
    """Scalar loss and gradients for every rendered plane (loss.py:146-245)."""
    rgb = rendered.rgb
    if rgb.shape != np.shape(reference_rgb):
        raise ValueError(f"rendered {rgb.shape} vs reference {np.shape(reference_rgb)}")
    lam = float(config.lambda_ssim)
    w_l1 = (1.0 - lam) if l1_weight is None else float(l1_weight)
    w_n = float(getattr(config, "normal_loss_weight", 0.0))
    w_s = float(getattr(config, "smooth_loss_weight", 0.0))
    use_n = w_n > 0.0 and rendered.normal is not None and rendered.depth is not None
    use_s = w_s > 0.0 and rendered.attrs is not None
    dev = require_cuda()
    ref = _to_dev(reference_rgb)
    h, w = rgb.shape[:2]
    if use_n or use_s:  # one (H, W, 11) plane stack like the blend produces
        planes = np.zeros((h, w, 11), dtype=np.float32)
        planes[:, :, :3] = rgb
        if rendered.depth is not None:
            planes[:, :, 3] = rendered.depth
        if rendered.normal is not None:
            planes[:, :, 4:7] = rendered.normal
        if rendered.attrs is not None:
            planes[:, :, 7:11] = rendered.attrs
        x = torch.from_numpy(planes).to(dev)
    else:
        x = _to_dev(rgb)
    d_x = torch.zeros_like(x)
    d_x, sums = l1_ssim_device(x, ref, w_l1, lam, d_x)
    normal_term = smooth_term = 0.0
    if use_n or use_s:
        t = _to_dev(1.0 - np.asarray(rendered.alpha, dtype=np.float32)).contiguous()
        sums3 = torch.zeros(3, dtype=torch.float64, device=dev)
        _kernel().aux(x, t, ref, px_scale, w_n if use_n else 0.0, w_s if use_s else 0.0, d_x, sums3)
        s3 = sums3.cpu().numpy()
        if use_n and s3[1] > 0:
            normal_term = w_n * float(s3[0]) / float(s3[1])
        if use_s:
            smooth_term = w_s * float(s3[2]) / (4 * (h * (w - 1) + (h - 1) * w))
    n_el = rgb.size
    n_pos = (h - 10) * (w - 10) * 3
    s = sums.cpu().numpy()
    l1 = float(s[0]) / n_el
    ssim_term = 1.0 - float(s[1]) / n_pos
    total = w_l1 * l1 + lam * ssim_term + normal_term + smooth_term
    dx = d_x.cpu().numpy()
    grads = ImageGradients(rgb=np.ascontiguousarray(dx[:, :, :3]).astype(rgb.dtype))
    if use_n:
        grads.depth = np.ascontiguousarray(dx[:, :, 3]).astype(rgb.dtype)
        grads.normal = np.ascontiguousarray(dx[:, :, 4:7]).astype(rgb.dtype)
    if use_s:
        grads.attrs = np.ascontiguousarray(dx[:, :, 7:11]).astype(rgb.dtype)
    return total, grads, LossBreakdown(total=total, l1=l1, ssim_term=ssim_term, normal=normal_term,
                                       smooth=smooth_term)
