"""Piecewise-linear transfer functions (drop-in for ``vegsplat.transfer``).

Control-point containers with the reference's validation
(/root/reference/pkg/src/vegsplat/transfer.py:21-88) and its evaluation contract:
clamp to [0, 1] then ``np.interp`` per map (:91-103), derivatives on half-open
segments [t_k, t_{k+1}) (:106-127).  Evaluation itself runs on the GPU: the knot
tables are packed into one float64 blob (``pack_tf``) that the preprocess kernel stages
in shared memory; ``eval_opacity``/``eval_color``/``d_*_dv`` below call the same device
lookup through the C-ABI (``vegs_tf_eval``) so tests can pin it bitwise against numpy.
"""

from __future__ import annotations

import json
from dataclasses import dataclass

import numpy as np

_KNOT_EPS = 1e-9
MAX_KNOTS = 1024  # per map; the device stages both maps in shared memory


def _check_knots(ts: np.ndarray, what: str) -> None:
    if ts.size < 2:
        raise ValueError(f"{what} needs at least 2 control points")
    if abs(ts[0]) > _KNOT_EPS or abs(ts[-1] - 1.0) > _KNOT_EPS:
        raise ValueError(f"{what} must have control points at t=0 and t=1")
    if np.any(np.diff(ts) <= 0):
        raise ValueError(f"{what} control points must be strictly increasing in t")
    if ts.size > MAX_KNOTS:
        raise ValueError(f"{what} has {ts.size} control points; the device table holds {MAX_KNOTS}")


@dataclass(frozen=True)
class OpacityMap:
    points: tuple[tuple[float, float], ...]

    def __post_init__(self):
        ts = np.array([p[0] for p in self.points], dtype=np.float64)
        vals = np.array([p[1] for p in self.points], dtype=np.float64)
        _check_knots(ts, "opacity map")
        if np.any(vals < -_KNOT_EPS) or np.any(vals > 1.0 + _KNOT_EPS):
            raise ValueError("opacity values must lie in [0, 1]")
        object.__setattr__(self, "_ts", ts)
        object.__setattr__(self, "_vals", vals)

    @property
    def ts(self) -> np.ndarray:
        return self._ts

    @property
    def values(self) -> np.ndarray:
        return self._vals

    def __call__(self, v):
        return eval_opacity(self, v)


@dataclass(frozen=True)
class ColorMap:
    points: tuple[tuple[float, float, float, float], ...]
    name: str | None = None

    def __post_init__(self):
        ts = np.array([p[0] for p in self.points], dtype=np.float64)
        rgb = np.array([p[1:] for p in self.points], dtype=np.float64)
        _check_knots(ts, "color map")
        if rgb.ndim != 2 or rgb.shape[1] != 3 or np.any(rgb < -_KNOT_EPS) or np.any(rgb > 1.0 + _KNOT_EPS):
            raise ValueError("color values must be rgb triples in [0, 1]")
        object.__setattr__(self, "_ts", ts)
        object.__setattr__(self, "_vals", rgb)

    @property
    def ts(self) -> np.ndarray:
        return self._ts

    @property
    def values(self) -> np.ndarray:
        return self._vals

    def __call__(self, v):
        return eval_color(self, v)


@dataclass(frozen=True)
class TransferFunction:
    color: ColorMap
    opacity: OpacityMap


def from_tables(ts_opacity, opacity, ts_color, rgb, name=None) -> TransferFunction:
    """Build a TF from knot arrays (e.g. a 256-entry RGBA table on uniform knots)."""
    op = OpacityMap(tuple((float(t), float(a)) for t, a in zip(ts_opacity, opacity)))
    col = ColorMap(tuple((float(t), float(r), float(g), float(b))
                         for t, (r, g, b) in zip(ts_color, np.asarray(rgb))), name=name)
    return TransferFunction(color=col, opacity=op)


def pack_tf(tf: TransferFunction) -> tuple[np.ndarray, int, int]:
    """Device blob: [ts_op(Ko) | op(Ko) | ts_col(Kc) | r(Kc) | g(Kc) | b(Kc)] float64."""
    o, c = tf.opacity, tf.color
    blob = np.concatenate([o.ts, o.values, c.ts, c.values[:, 0], c.values[:, 1], c.values[:, 2]])
    return np.ascontiguousarray(blob, dtype=np.float64), len(o.ts), len(c.ts)


def tf_to_dict(tf: TransferFunction) -> dict:
    return {"color": [list(p) for p in tf.color.points],
            "opacity": [list(p) for p in tf.opacity.points]}


def tf_from_dict(d: dict) -> TransferFunction:
    color = ColorMap(tuple((float(t), float(r), float(g), float(b)) for t, r, g, b in d["color"]))
    opacity = OpacityMap(tuple((float(t), float(a)) for t, a in d["opacity"]))
    return TransferFunction(color=color, opacity=opacity)


def save_tf(tf: TransferFunction, path) -> None:
    with open(path, "w") as f:
        json.dump(tf_to_dict(tf), f)


def load_tf(path) -> TransferFunction:
    with open(path) as f:
        return tf_from_dict(json.load(f))


# -- evaluation through the device lookup ------------------------------------

def _device_eval(ts: np.ndarray, vals: np.ndarray, v, derivative: bool) -> np.ndarray:
    from . import device

    return device.tf_eval(ts, vals, v, derivative)


def eval_opacity(opacity: OpacityMap, v):
    out = _device_eval(opacity.ts, opacity.values[:, None], v, False)[..., 0]
    return out if np.ndim(v) else float(out)


def eval_color(color: ColorMap, v):
    return _device_eval(color.ts, color.values, v, False)


def d_opacity_dv(opacity: OpacityMap, v):
    out = _device_eval(opacity.ts, opacity.values[:, None], v, True)[..., 0]
    return out if np.ndim(v) else float(out)


def d_color_dv(color: ColorMap, v):
    return _device_eval(color.ts, color.values, v, True)
