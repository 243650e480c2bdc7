"""VEGS model files to and from the device (drop-in for vegsplat's model I/O).

Format (/root/reference/pkg/src/vegsplat/model.py:220-314): a 64-byte header (``VEGS``,
version 1, count, flags, f32 bbox) followed either by the 19 parameter classes as
class-major little-endian float32 blocks in FIELD_LAYOUT order -- exactly the device
parameter layout, so loading is one upload and a widening to float64 -- or, with the VQ
flag, f32 positions + a (K, 16) f32 codebook + u32 indices, decompressed on the device
by a gather.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from .model import FIELD_LAYOUT, FLOATS_PER_GAUSSIAN, GaussianSet

MAGIC = b"VEGS"
VERSION = 1
HEADER_BYTES = 64
FLAG_VQ = 1
ATTRIBUTE_DIM = FLOATS_PER_GAUSSIAN - 3


class FormatError(ValueError):
    """Malformed model file (vegsplat.errors.FormatError)."""


def _header(count: int, flags: int, lo, hi) -> bytes:
    head = MAGIC + struct.pack("<III", VERSION, count, flags) + struct.pack("<6f", *lo, *hi)
    return head.ljust(HEADER_BYTES, b"\0")


def _parse_header(blob: bytes) -> tuple[int, int]:
    if len(blob) < HEADER_BYTES or blob[:4] != MAGIC:
        raise FormatError("not a VEGS model file")
    version, count, flags = struct.unpack("<III", blob[4:16])
    if version != VERSION:
        raise FormatError(f"unsupported model version {version}")
    return count, flags


def model_file_size(n: int) -> int:
    return HEADER_BYTES + n * FLOATS_PER_GAUSSIAN * 4


def save_model(gs: GaussianSet, path) -> None:
    """Uncompressed model file (64-byte header + n * 19 little-endian f32, class-major)."""
    if len(gs):
        lo, hi = gs.position.min(axis=0), gs.position.max(axis=0)
    else:
        lo, hi = np.zeros(3), np.zeros(3)
    Path(path).write_bytes(_header(len(gs), 0, lo, hi) + gs.pack().astype("<f4").tobytes())


def _split(blob: bytes, path) -> tuple[int, int, dict]:
    count, flags = _parse_header(blob)
    off = HEADER_BYTES
    if flags & FLAG_VQ:
        need = off + count * 12 + 4
        if len(blob) < need:
            raise FormatError(f"{path}: truncated VQ model file")
        pos = np.frombuffer(blob, dtype="<f4", count=count * 3, offset=off)
        off += count * 12
        (k,) = struct.unpack_from("<I", blob, off)
        off += 4
        if len(blob) != off + k * ATTRIBUTE_DIM * 4 + count * 4:
            raise FormatError(f"{path}: VQ model file is {len(blob)} bytes, expected "
                              f"{off + k * ATTRIBUTE_DIM * 4 + count * 4}")
        book = np.frombuffer(blob, dtype="<f4", count=k * ATTRIBUTE_DIM, offset=off).reshape(k, ATTRIBUTE_DIM)
        off += k * ATTRIBUTE_DIM * 4
        idx = np.frombuffer(blob, dtype="<u4", count=count, offset=off)
        if count and int(idx.max()) >= k:
            raise FormatError(f"{path}: codebook index out of range")
        return count, flags, dict(position=pos, codebook=book, indices=idx)
    if len(blob) != model_file_size(count):
        raise FormatError(f"{path}: model file is {len(blob)} bytes, expected {model_file_size(count)}")
    return count, flags, dict(flat=np.frombuffer(blob, dtype="<f4", count=count * FLOATS_PER_GAUSSIAN, offset=off))


def _vq_flat(position: np.ndarray, attrs: np.ndarray, n: int) -> np.ndarray:
    """Class-major flat buffer from positions + (n, 16) attribute rows (model.py:136-147)."""
    parts = [position.reshape(n, 3)]
    off = 0
    for name, width in FIELD_LAYOUT[1:]:
        parts.append(attrs[:, off:off + width])
        off += width
    return np.concatenate([p.reshape(-1) for p in parts])


def load_model(path) -> GaussianSet:
    """Load an uncompressed or VQ model file (VQ is decompressed) as a host GaussianSet."""
    count, flags, d = _split(Path(path).read_bytes(), path)
    if flags & FLAG_VQ:
        attrs = d["codebook"].astype(np.float64)[d["indices"].astype(np.int64)]
        return GaussianSet.unpack(_vq_flat(d["position"].astype(np.float64), attrs, count), count)
    return GaussianSet.unpack(d["flat"].astype(np.float64), count)


def load_model_device(path, device=None):
    """(flat float64 parameter tensor on the device, n): the f32 payload is uploaded once
    and widened on the device; VQ codebooks are gathered on the device."""
    import torch

    from .device import require_cuda

    dev = device or require_cuda()
    count, flags, d = _split(Path(path).read_bytes(), path)
    if flags & FLAG_VQ:
        book = torch.from_numpy(d["codebook"].copy()).to(dev)
        idx = torch.from_numpy(d["indices"].astype(np.int64)).to(dev)
        attrs = book.index_select(0, idx).double()
        pos = torch.from_numpy(d["position"].copy()).to(dev).double().view(count, 3)
        parts, off = [pos.reshape(-1)], 0
        for _, width in FIELD_LAYOUT[1:]:
            parts.append(attrs[:, off:off + width].reshape(-1))
            off += width
        return torch.cat(parts), count
    return torch.from_numpy(d["flat"].copy()).to(dev).double(), count


def save_model_device(params, n: int, path) -> None:
    """Write a device-resident flat parameter buffer as an uncompressed model file."""
    save_model(GaussianSet.unpack(params.detach().cpu().numpy(), n), path)
