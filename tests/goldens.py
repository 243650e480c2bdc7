"""Loaders that rebuild inputs (Gaussians, TF, camera) from the committed golden .npz files."""

from __future__ import annotations

from pathlib import Path

import numpy as np

from paper_2504_13339_b200.camera import Camera
from paper_2504_13339_b200.model import PARAM_CLASSES, GaussianSet
from paper_2504_13339_b200.transfer import from_tables

GOLDEN = Path(__file__).resolve().parent / "golden"


def load(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


def gs_of(d: dict, prefix: str = "gs_") -> GaussianSet:
    return GaussianSet(**{k: d[prefix + k] for k in PARAM_CLASSES})


def tf_of(d: dict, prefix: str = "tf_"):
    return from_tables(d[prefix + "op_ts"], d[prefix + "op_vals"], d[prefix + "col_ts"], d[prefix + "col_vals"])


def cam_of(v: np.ndarray) -> Camera:
    return Camera(position=tuple(v[0:3]), target=tuple(v[3:6]), up=tuple(v[6:9]), fov_y=float(v[9]),
                  width=int(v[10]), height=int(v[11]), near=float(v[12]), far=float(v[13]))


def norm_rel(a, b) -> float:
    """||a - b||_inf / max(||b||_inf, tiny): the SURVEY §8(d) gradient metric."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)) if b.size else 0.0
