"""Framebuffer container (drop-in for ``vegsplat.images.ImageBuffer``,
/root/reference/pkg/src/vegsplat/images.py:12-47): rgb (H,W,3), alpha (H,W) and the
optional auxiliary planes depth (H,W), normal (H,W,3), attrs (H,W,4)."""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class ImageBuffer:
    rgb: np.ndarray
    alpha: np.ndarray = None
    depth: np.ndarray | None = None
    normal: np.ndarray | None = None
    attrs: np.ndarray | None = None

    def __post_init__(self):
        if self.rgb.ndim != 3 or self.rgb.shape[2] != 3:
            raise ValueError("rgb plane must have shape (H, W, 3)")
        if self.alpha is None:
            self.alpha = np.zeros(self.rgb.shape[:2], dtype=self.rgb.dtype)
        for name in ("alpha", "depth", "normal", "attrs"):
            plane = getattr(self, name)
            if plane is not None and plane.shape[:2] != self.rgb.shape[:2]:
                raise ValueError(f"{name} plane shape {plane.shape} mismatches rgb {self.rgb.shape}")

    @property
    def width(self) -> int:
        return self.rgb.shape[1]

    @property
    def height(self) -> int:
        return self.rgb.shape[0]

    @property
    def transmittance(self) -> np.ndarray:
        return 1.0 - self.alpha
