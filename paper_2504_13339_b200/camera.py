"""Pinhole camera (drop-in for ``vegsplat.camera.Camera``).

Same conventions as /root/reference/pkg/src/vegsplat/camera.py:22-90: right-handed
look-at, pixel centres at half-integers, ``focal_px = H/2 / tan(fov_y/2)`` (:54-57),
world->camera rotation rows (right, up, forward) with positive depth in front (:85-90).
The host computes these few doubles once per view and hands them to the preprocess
kernel in a ``VegsCamera`` struct, so the device sees bit-identical camera constants.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Camera:
    position: tuple[float, float, float]
    target: tuple[float, float, float]
    up: tuple[float, float, float] = (0.0, 1.0, 0.0)
    fov_y: float = math.radians(60.0)
    width: int = 800
    height: int = 800
    near: float = 0.01
    far: float = 1000.0

    def __post_init__(self):
        if not (0.0 < self.fov_y < math.pi):
            raise ValueError("fov_y must lie in (0, pi)")
        if self.width < 1 or self.height < 1:
            raise ValueError("resolution must be positive")
        if not (0.0 < self.near < self.far):
            raise ValueError("need 0 < near < far")
        pos = np.asarray(self.position, dtype=np.float64)
        fwd = np.asarray(self.target, dtype=np.float64) - pos
        dist = np.linalg.norm(fwd)
        if dist == 0.0:
            raise ValueError("camera position must differ from target")
        up = np.asarray(self.up, dtype=np.float64)
        if np.linalg.norm(np.cross(fwd / dist, up / np.linalg.norm(up))) < 1e-9:
            raise ValueError("up vector is parallel to the view direction")

    @property
    def aspect(self) -> float:
        return self.width / self.height

    @property
    def focal_px(self) -> float:
        return 0.5 * self.height / math.tan(0.5 * self.fov_y)

    def view_matrix(self) -> np.ndarray:
        eye = np.asarray(self.position, dtype=np.float64)
        f = np.asarray(self.target, dtype=np.float64) - eye
        f = f / np.linalg.norm(f)
        r = np.cross(f, np.asarray(self.up, dtype=np.float64))
        r = r / np.linalg.norm(r)
        u = np.cross(r, f)
        m = np.eye(4)
        m[0, :3], m[1, :3], m[2, :3] = r, u, -f
        m[:3, 3] = -m[:3, :3] @ eye
        return m

    def world_to_cam_rotation(self) -> np.ndarray:
        rot = self.view_matrix()[:3, :3].copy()
        rot[2] = -rot[2]
        return rot


def orbit_camera(direction, radius: float, width: int, height: int,
                 fov_y: float = math.radians(50.0)) -> Camera:
    """Camera on the sphere of ``radius`` along ``direction``, looking at the origin."""
    d = np.asarray(direction, dtype=np.float64)
    d = d / np.linalg.norm(d)
    up = (0.0, 1.0, 0.0)
    if abs(d[1]) > 0.999:  # keep the look-at well defined near the poles
        up = (0.0, 0.0, 1.0)
    pos = tuple(float(x) for x in radius * d)
    return Camera(position=pos, target=(0.0, 0.0, 0.0), up=up, fov_y=fov_y,
                  width=width, height=height)
