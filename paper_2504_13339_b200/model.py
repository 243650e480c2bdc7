"""Gaussian parameter container (drop-in for ``vegsplat.model.GaussianSet``).

Host-side structure-of-arrays record with the reference's field order and
activations (/root/reference/pkg/src/vegsplat/model.py:25-40 layout, :49-59
activations, :62-154 ``GaussianSet``).  Parameters stay float64 exactly like the
reference, so the device twin (``pack_params``) is a flat float64 buffer of
19 doubles per Gaussian laid out class-major:

    [position (n,3) | log_scale (n,3) | rotation (n,4) | raw_value (n) |
     raw_weight (n) | normal (n,3) | raw_ka (n) | raw_kd (n) | raw_ks (n) | raw_beta (n)]

The same layout is used for gradients and Adam moments, so the NCCL all-reduce
and the fused Adam kernel see one contiguous buffer (152 B/Gaussian; 152 MB at 1M).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BETA_MIN, BETA_MAX = 1.0, 128.0

FIELD_LAYOUT = (
    ("position", 3),
    ("log_scale", 3),
    ("rotation", 4),
    ("raw_value", 1),
    ("raw_weight", 1),
    ("normal", 3),
    ("raw_ka", 1),
    ("raw_kd", 1),
    ("raw_ks", 1),
    ("raw_beta", 1),
)
FLOATS_PER_GAUSSIAN = sum(w for _, w in FIELD_LAYOUT)  # 19
PARAM_CLASSES = tuple(name for name, _ in FIELD_LAYOUT)


def class_offsets(n: int) -> dict[str, tuple[int, int, int]]:
    """name -> (start, stop, width) element offsets of each class in the flat buffer."""
    out = {}
    off = 0
    for name, width in FIELD_LAYOUT:
        out[name] = (off, off + n * width, width)
        off += n * width
    return out


def sigmoid(x):
    return 1.0 / (1.0 + np.exp(-np.asarray(x, dtype=np.float64)))


def logit(p):
    p = np.asarray(p, dtype=np.float64)
    return np.log(p) - np.log1p(-p)


def activate_beta(raw):
    return np.clip(np.exp(np.asarray(raw, dtype=np.float64)), BETA_MIN, BETA_MAX)


@dataclass
class GaussianSet:
    position: np.ndarray
    log_scale: np.ndarray
    rotation: np.ndarray   # (n, 4) wxyz, normalised at use
    raw_value: np.ndarray
    raw_weight: np.ndarray
    normal: np.ndarray     # (n, 3) normalised at use
    raw_ka: np.ndarray
    raw_kd: np.ndarray
    raw_ks: np.ndarray
    raw_beta: np.ndarray

    def __post_init__(self):
        n = len(self.position)
        for name, width in FIELD_LAYOUT:
            arr = getattr(self, name)
            want = (n,) if width == 1 else (n, width)
            if arr.shape != want:
                raise ValueError(f"{name}: expected shape {want}, got {arr.shape}")

    def __len__(self) -> int:
        return len(self.position)

    # activated views (host convenience, same formulas as model.py:87-110)
    def values(self):
        return sigmoid(self.raw_value)

    def weights(self):
        return sigmoid(self.raw_weight)

    def scales(self):
        return np.exp(self.log_scale)

    def ka(self):
        return sigmoid(self.raw_ka)

    def kd(self):
        return sigmoid(self.raw_kd)

    def ks(self):
        return sigmoid(self.raw_ks)

    def beta(self):
        return activate_beta(self.raw_beta)

    def field_names(self) -> list[str]:
        return list(PARAM_CLASSES)

    def arrays(self) -> dict[str, np.ndarray]:
        return {name: getattr(self, name) for name in PARAM_CLASSES}

    def copy(self) -> "GaussianSet":
        return GaussianSet(**{k: v.copy() for k, v in self.arrays().items()})

    def select(self, index) -> "GaussianSet":
        return GaussianSet(**{k: v[index].copy() for k, v in self.arrays().items()})

    @staticmethod
    def concatenate(parts: list["GaussianSet"]) -> "GaussianSet":
        return GaussianSet(**{k: np.concatenate([getattr(p, k) for p in parts]) for k in PARAM_CLASSES})

    # device layout -------------------------------------------------------
    def pack(self) -> np.ndarray:
        """Flat float64 class-major buffer (see module docstring)."""
        return np.concatenate([np.ascontiguousarray(getattr(self, k), dtype=np.float64).ravel()
                               for k in PARAM_CLASSES])

    @staticmethod
    def unpack(flat: np.ndarray, n: int) -> "GaussianSet":
        flat = np.asarray(flat, dtype=np.float64)
        if flat.size != n * FLOATS_PER_GAUSSIAN:
            raise ValueError(f"flat buffer has {flat.size} values, expected {n * FLOATS_PER_GAUSSIAN}")
        fields = {}
        for name, (a, b, w) in class_offsets(n).items():
            chunk = flat[a:b].copy()
            fields[name] = chunk if w == 1 else chunk.reshape(n, w)
        return GaussianSet(**fields)
