"""Drop-in replacements for the reference's two numba tile kernels.

``blend_forward`` / ``blend_backward`` take exactly the argument lists of
/root/reference/pkg/src/vegsplat/raster/kernels.py:26-33 and :103-112 (numpy arrays,
outputs written in place), and run them through the C-ABI entry points
``vegs_blend_forward`` / ``vegs_blend_backward`` (include/vegsplat_b200.h).  A maintainer
can rebind ``vegsplat.raster.kernels.blend_forward`` to this function.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from ._lib import call
from .device import _p, _stream, require_cuda


def _dev(a, dtype=None):
    a = np.ascontiguousarray(a, dtype=dtype)
    return torch.from_numpy(a).to(require_cuda())


def _store(inst_alpha) -> tuple[bool, type]:
    dt = np.asarray(inst_alpha).dtype
    if dt == np.float64:
        return True, np.float64
    if dt == np.float32:
        return False, np.float32
    raise ValueError(f"unsupported blend dtype {dt}")


def blend_forward(tile_start, tile_end, tiles_x, tile_size,
                  inst_mean2d, inst_conic, inst_alpha, inst_pmin, inst_rect, inst_channels,
                  bg, width, height, alpha_clamp, trans_stop,
                  out_img, out_t, out_last, n_contrib=None):
    f64, real = _store(inst_alpha)
    n_ch = int(np.asarray(inst_channels).shape[1])
    ts, te = _dev(tile_start, np.int64), _dev(tile_end, np.int64)
    args = [_dev(inst_mean2d, real), _dev(inst_conic, real), _dev(inst_alpha, real), _dev(inst_pmin, real),
            _dev(inst_rect, np.int32), _dev(inst_channels, real)]
    bg_h = np.ascontiguousarray(bg, dtype=real)
    dev = ts.device
    img = torch.empty(int(height) * int(width) * n_ch, dtype=torch.from_numpy(bg_h).dtype, device=dev)
    t = torch.empty(int(height) * int(width), dtype=img.dtype, device=dev)
    last = torch.empty(int(height) * int(width), dtype=torch.int64, device=dev)
    ncon = torch.empty(int(height) * int(width), dtype=torch.int32, device=dev)
    call("vegs_blend_forward", _p(ts), _p(te), len(tile_start), int(tiles_x), int(tile_size), *[_p(a) for a in args[:5]],
         _p(args[5]), n_ch, int(f64), bg_h.ctypes.data_as(ctypes.c_void_p), int(width), int(height),
         float(alpha_clamp), float(trans_stop), _p(img), _p(t), _p(last), _p(ncon), _stream())
    out_img[...] = img.cpu().numpy().reshape(out_img.shape)
    out_t[...] = t.cpu().numpy().reshape(out_t.shape)
    out_last[...] = last.cpu().numpy().reshape(out_last.shape)
    if n_contrib is not None:
        n_contrib[...] = ncon.cpu().numpy().reshape(n_contrib.shape)


def blend_backward(tile_start, tile_end, tiles_x, tile_size,
                   inst_mean2d, inst_conic, inst_alpha, inst_pmin, inst_rect, inst_channels,
                   bg, width, height, alpha_clamp, out_t, out_last, d_img, d_alpha_plane,
                   g_mean2d, g_conic, g_alpha, g_channels):
    f64, real = _store(inst_alpha)
    n_ch = int(np.asarray(inst_channels).shape[1])
    ts, te = _dev(tile_start, np.int64), _dev(tile_end, np.int64)
    args = [_dev(inst_mean2d, real), _dev(inst_conic, real), _dev(inst_alpha, real), _dev(inst_pmin, real),
            _dev(inst_rect, np.int32), _dev(inst_channels, real)]
    bg_h = np.ascontiguousarray(bg, dtype=real)
    outs = [_dev(g_mean2d, real), _dev(g_conic, real), _dev(g_alpha, real), _dev(g_channels, real)]
    # keep every device copy referenced until the launch is enqueued
    planes = [_dev(out_t, real), _dev(out_last, np.int64), _dev(d_img, real), _dev(d_alpha_plane, real)]
    call("vegs_blend_backward", _p(ts), _p(te), len(tile_start), int(tiles_x), int(tile_size),
         *[_p(a) for a in args], n_ch, int(f64), bg_h.ctypes.data_as(ctypes.c_void_p), int(width), int(height),
         float(alpha_clamp), *[_p(p) for p in planes], *[_p(o) for o in outs], _stream())
    for host, d in zip((g_mean2d, g_conic, g_alpha, g_channels), outs):
        host[...] = d.cpu().numpy().reshape(host.shape)
