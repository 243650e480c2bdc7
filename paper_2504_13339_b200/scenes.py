"""Seeded synthetic workloads for the BASELINE.json configs.

No public dataset is involved: BASELINE.json's configs are themselves synthetic, and
these generators produce them from ``numpy.random.default_rng(seed)`` on the host so the
CPU oracle and the GPU path consume the *same* float64 arrays.  Draw order is part of
the contract (changing it changes every golden fixture):

* ``random_gaussians``: draws, in order, means U[-1,1]^3, values U[0,1] (stored as
  logit(clip(v, 1e-4, 1-1e-4)), the reference's init convention, model.py:171),
  log-scales N(-3.5, 0.3) per axis, rotations a normalised N(0, I4), normals a
  normalised N(0, I3).
  Fields BASELINE leaves open follow the reference init defaults (model.py:174-186):
  raw_weight = logit(0.1), raw_ka = raw_kd = raw_ks = 0, raw_beta = log 8.
* ``blob_gaussians`` (configs 2-4 ground truth): 64 anisotropic blobs with centres
  U[-0.8,0.8]^3, blob rotation from a normalised N(0, I4), per-axis blob sigma
  U[0.05, 0.35]; points = centre + R diag(sigma) z, z ~ N(0, I3); other fields as above.
* ``random_tf``: 256 uniform knots for both maps; opacity = clip(sum of k Gaussian bumps,
  0, 1) with centres U[0,1], widths U[0.03, 0.15], heights U[0.3, 1]; colour = a random
  piecewise-linear ramp through 2-6 anchors (sorted U[0,1] positions plus both ends)
  with U[0,1] RGB, sampled at the knots.
* ``orbit_cameras``: directions normalised N(0, I3) on the radius-3 sphere looking at the
  origin, 50 degree vertical fov.
"""

from __future__ import annotations

import math

import numpy as np

from .camera import Camera, orbit_camera
from .model import GaussianSet, logit
from .transfer import TransferFunction, from_tables

N_KNOTS = 256


def _fill(rng: np.random.Generator, position: np.ndarray, values: np.ndarray) -> GaussianSet:
    n = len(position)
    log_scale = rng.normal(-3.5, 0.3, size=(n, 3))
    rotation = _unit_quats(rng, n)
    normal = rng.normal(size=(n, 3))
    normal /= np.linalg.norm(normal, axis=1, keepdims=True)
    return GaussianSet(
        position=position,
        log_scale=log_scale,
        rotation=rotation,
        raw_value=logit(np.clip(values, 1e-4, 1.0 - 1e-4)),
        raw_weight=np.full(n, float(logit(0.1))),
        normal=normal,
        raw_ka=np.zeros(n),
        raw_kd=np.zeros(n),
        raw_ks=np.zeros(n),
        raw_beta=np.full(n, math.log(8.0)),
    )


def _unit_quats(rng: np.random.Generator, n: int) -> np.ndarray:
    q = rng.normal(size=(n, 4))
    return q / np.linalg.norm(q, axis=1, keepdims=True)


def random_gaussians(n: int, seed: int = 0) -> GaussianSet:
    rng = np.random.default_rng(seed)
    position = rng.uniform(-1.0, 1.0, size=(n, 3))
    values = rng.uniform(0.0, 1.0, size=n)
    return _fill(rng, position, values)


def blob_gaussians(n: int, seed: int = 1, n_blobs: int = 64) -> GaussianSet:
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-0.8, 0.8, size=(n_blobs, 3))
    q = _unit_quats(rng, n_blobs)
    w, x, y, z = q.T
    rot = np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], 1)
    sig = rng.uniform(0.05, 0.35, size=(n_blobs, 3))
    blob = rng.integers(0, n_blobs, size=n)
    zs = rng.normal(size=(n, 3)) * sig[blob]
    position = centres[blob] + np.einsum("nij,nj->ni", rot[blob], zs)
    values = np.clip(0.5 + 0.35 * np.tanh(rng.normal(size=n)) + 0.1 * (blob % 4) - 0.15, 0.0, 1.0)
    return _fill(rng, position, values)


def random_tf(seed: int, n_bumps: int | None = None, n_knots: int = N_KNOTS) -> TransferFunction:
    rng = np.random.default_rng(seed)
    if n_bumps is None:
        n_bumps = int(rng.integers(1, 7))
    ts = np.linspace(0.0, 1.0, n_knots)
    centres = rng.uniform(0.0, 1.0, size=n_bumps)
    widths = rng.uniform(0.03, 0.15, size=n_bumps)
    heights = rng.uniform(0.3, 1.0, size=n_bumps)
    op = np.clip((heights[None, :] * np.exp(-0.5 * ((ts[:, None] - centres[None, :]) / widths[None, :]) ** 2)).sum(1),
                 0.0, 1.0)
    n_anchor = int(rng.integers(2, 7))
    at = np.concatenate([[0.0], np.sort(rng.uniform(0.0, 1.0, size=n_anchor - 2)), [1.0]])
    ac = rng.uniform(0.0, 1.0, size=(n_anchor, 3))
    rgb = np.stack([np.interp(ts, at, ac[:, c]) for c in range(3)], axis=1)
    return from_tables(ts, op, ts, rgb)


def range_tf(seed: int, lo: float, hi: float, n_bumps: int = 2, n_knots: int = N_KNOTS) -> TransferFunction:
    """A random TF whose opacity bumps sit inside the scalar range [lo, hi] (config 4 cycles
    16 of these over disjoint ranges); colour ramp as in random_tf."""
    rng = np.random.default_rng(seed)
    ts = np.linspace(0.0, 1.0, n_knots)
    w = hi - lo
    centres = rng.uniform(lo + 0.25 * w, hi - 0.25 * w, size=n_bumps)
    widths = rng.uniform(0.05, 0.15, size=n_bumps) * w
    heights = rng.uniform(0.5, 1.0, size=n_bumps)
    op = (heights[None, :] * np.exp(-0.5 * ((ts[:, None] - centres[None, :]) / widths[None, :]) ** 2)).sum(1)
    op = np.where((ts >= lo) & (ts <= hi), np.clip(op, 0.0, 1.0), 0.0)
    n_anchor = int(rng.integers(2, 7))
    at = np.concatenate([[0.0], np.sort(rng.uniform(0.0, 1.0, size=n_anchor - 2)), [1.0]])
    ac = rng.uniform(0.0, 1.0, size=(n_anchor, 3))
    rgb = np.stack([np.interp(ts, at, ac[:, c]) for c in range(3)], axis=1)
    return from_tables(ts, op, ts, rgb)


def orbit_cameras(n: int, seed: int, width: int, height: int, radius: float = 3.0,
                  fov_deg: float = 50.0) -> list[Camera]:
    rng = np.random.default_rng(seed)
    dirs = rng.normal(size=(n, 3))
    return [orbit_camera(d, radius, width, height, math.radians(fov_deg)) for d in dirs]


# -- BASELINE.json configs ------------------------------------------------------

CONFIGS = {
    # name: (n_learned, gt_kind, n_gt, views_per_step, width, height, n_bumps)
    "c0": dict(n=4096, width=128, height=128, views=1, bumps=4),
    "c1": dict(n=100_000, gt="uniform", n_gt=100_000, width=512, height=512, views=4, bumps=4),
    "c2": dict(n=1_000_000, gt="blobs", n_gt=1_000_000, width=1024, height=1024, views=16, bumps=4),
    "c3": dict(n=3_000_000, width=1920, height=1080, views=1, tfs_per_frame=8),
    "c4": dict(n=200_000, gt="blobs", n_gt=2_000_000, width=800, height=800, views=64, tfs=16),
}


def config_scene(name: str, scale: float = 1.0):
    """(learned set, ground-truth set or None, tf, cameras) for a BASELINE config.

    ``scale`` < 1 shrinks the Gaussian counts (tests); resolution is kept."""
    cfg = CONFIGS[name]
    n = max(1, int(cfg["n"] * scale))
    learned = random_gaussians(n, seed=0)
    gt = None
    if cfg.get("gt") == "uniform":
        gt = random_gaussians(max(1, int(cfg["n_gt"] * scale)), seed=1)
    elif cfg.get("gt") == "blobs":
        gt = blob_gaussians(max(1, int(cfg["n_gt"] * scale)), seed=1)
    tf = random_tf(seed=2, n_bumps=cfg.get("bumps", 4))
    cams = orbit_cameras(cfg["views"], seed=3, width=cfg["width"], height=cfg["height"])
    return learned, gt, tf, cams
