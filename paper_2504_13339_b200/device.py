"""Device-side orchestration of the rasteriser: torch tensors own HBM, the C-ABI does the work.

Per view, the forward pipeline is five launches on the current CUDA stream:

    vegs_preprocess_forward  per-Gaussian TF + shading + EWA projection -> splat table
    vegs_bin_count           scan of (kept, tiles touched)        [one 16-byte readback]
    vegs_bin_sort            depth rank, duplication, (tile, rank) radix sort, ranges
    vegs_composite_forward   tile blend -> image, T, last contributor, contributor count

and the backward is two more (``vegs_composite_backward`` -> per-instance rows,
``vegs_preprocess_backward`` -> float64 per-Gaussian gradients).  The only host
synchronisation is the instance count needed to size the sort.

Nothing here computes on the CPU: if CUDA or the library is missing, ``require_cuda``
raises.
"""

from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._lib import VegsCamera, VegsError, VegsSettings, VegsSplatTable, VegsTF, call
from .constants import DEFAULT_SETTINGS, RasterSettings
from .transfer import TransferFunction, pack_tf

TILE = 16

# Kernels launched per C-ABI call (our kernels plus the CUB kernels instantiated inside
# libvegsplat_b200.so); checked against the ncu launch list in profiles/.
LAUNCHES = {
    "vegs_preprocess_forward": 1,
    "vegs_preprocess_forward_projected": 1,
    "vegs_project": 1,
    "vegs_splat_table_from_arrays": 1,
    "vegs_bin_count": 4,          # pack, CUB scan (init + sweep), unpack
    "vegs_bin_count_dev": 4,      # the same (+2 capacity-check launches counted in forward_end)
    "vegs_bin_sort_dev": 18,      # the placement path of vegs_bin_sort
    "vegs_bin_sort": 18,          # counting placement: coarse keys, CUB depth sort (hist + scan + 4 onesweep), ties,
                                  # chunk counts, group sums, group scan, CUB scan (2), chunk offsets, placement,
                                  # tile weights + single-tile CUB sort (heaviest-first tile order); +5 from 4096
                                  # tiles (two levels: tile difference array, its prefix sums, CUB scan (2), block
                                  # runs); +1 (order / inst_pid) on the API path.  Radix path (> 12288 tiles): 19.
    "vegs_composite_forward": 1,
    "vegs_composite_forward_fast": 2,  # blend + float64 fix-up of the undecidable pixels (+ a 4-byte memset)
    "vegs_composite_backward": 1,
    "vegs_preprocess_backward": 3,  # kept list + row reduction + chain (float32 blends; float64: 2)
    "vegs_loss_l1_ssim": 2,
    "vegs_loss_aux": 3,
    "vegs_adam_step": 1,
    "vegs_adam_step_sum": 1,
    "vegs_grad_pack": 1,
    "vegs_adam_step_range": 1,
    "vegs_densify_count": 3,
    "vegs_densify_apply": 1,
}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise VegsError("vegsplat_b200 needs a CUDA device (B200): there is no CPU path")
    _lib.load()
    return torch.device("cuda", torch.cuda.current_device())


def _p(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


try:  # the raw cudaStream_t of the current stream without the Stream object round trip
    from torch._C import _cuda_getCurrentRawStream as _raw_stream  # noqa: E402

    def _stream():
        return ctypes.c_void_p(_raw_stream(torch._C._cuda_getDevice()))
except ImportError:  # pragma: no cover - older torch
    def _stream():
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class use_stream:
    """``torch.cuda.stream(s)`` for the hot host path: the same stream switch without the
    current-device resolution (single device per process)."""

    __slots__ = ("s", "prev")

    def __init__(self, s):
        self.s = s

    def __enter__(self):
        self.prev = torch.cuda.current_stream(self.s.device)
        torch.cuda.set_stream(self.s)
        return self.s

    def __exit__(self, *exc):
        torch.cuda.set_stream(self.prev)
        return False


def rec_stride(n_ch: int) -> int:
    return ((7 + n_ch) + 3) & ~3


_CAMERA_CACHE: dict = {}


def camera_struct(cam) -> VegsCamera:
    """The kernels' camera block (read-only to them); cached per (frozen, hashable) Camera,
    since views repeat every step and the look-at math is numpy work on the host."""
    try:
        c = _CAMERA_CACHE.get(cam)
    except TypeError:  # a camera with unhashable fields (lists): no caching
        return _camera_struct(cam)
    if c is None:
        if len(_CAMERA_CACHE) >= 4096:
            _CAMERA_CACHE.clear()
        c = _CAMERA_CACHE[cam] = _camera_struct(cam)
    return c


def _camera_struct(cam) -> VegsCamera:
    c = VegsCamera()
    c.position[:] = [float(x) for x in cam.position]
    rot = np.asarray(cam.world_to_cam_rotation(), dtype=np.float64).ravel()
    c.rot[:] = rot.tolist()
    tan_y = math.tan(0.5 * cam.fov_y)
    c.focal = 0.5 * cam.height / tan_y
    c.tan_y = tan_y
    c.tan_x = tan_y * (cam.width / cam.height)
    c.near_z = float(cam.near)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def settings_struct(s: RasterSettings) -> VegsSettings:
    if s.tile_size != TILE:
        raise ValueError(f"tile_size {s.tile_size} unsupported: the B200 kernels use 16x16 tiles")
    v = VegsSettings()
    v.dilation, v.alpha_clamp, v.alpha_skip = s.dilation, s.alpha_clamp, s.alpha_skip
    v.transmittance_stop, v.radius_sigma, v.rect_margin_px = s.transmittance_stop, s.radius_sigma, s.rect_margin_px
    v.cull_alpha, v.frustum_limit, v.tile_size = s.cull_alpha, s.frustum_limit, s.tile_size
    return v


class DeviceTF:
    """Transfer-function knot tables resident in HBM (staged to SMEM by the kernels)."""

    def __init__(self, tf: TransferFunction, device=None):
        blob, k_op, k_col = pack_tf(tf)
        self.tf = tf
        self.blob = torch.from_numpy(blob).to(device or require_cuda())
        self.struct = VegsTF(ctypes.c_void_p(self.blob.data_ptr()), k_op, k_col)


class Pool:
    """Grow-only scratch buffers keyed by name (reused across views of a step)."""

    def __init__(self, device):
        self.device = device
        self.bufs: dict[str, torch.Tensor] = {}

    def get(self, name: str, numel: int, dtype) -> torch.Tensor:
        numel = max(int(numel), 1)
        t = self.bufs.get(name)
        if t is None or t.numel() < numel or t.dtype != dtype:
            t = torch.empty(int(numel * 1.1) + 64 if t is not None else numel, dtype=dtype, device=self.device)
            self.bufs[name] = t
        return t[:numel]


class _Fresh:
    def __init__(self, device):
        self.device = device

    def get(self, name: str, numel: int, dtype) -> torch.Tensor:
        return torch.empty(max(int(numel), 1), dtype=dtype, device=self.device)


@dataclass
class Frame:
    """Everything one forward leaves on the device for its backward."""

    n: int
    n_ch: int
    store_f64: bool
    width: int
    height: int
    cam: VegsCamera | None
    tf: DeviceTF | None
    settings: VegsSettings
    bg: ctypes.Array
    params: torch.Tensor | None
    record: torch.Tensor
    rect: torch.Tensor
    tiles: torch.Tensor
    depth_key: torch.Tensor
    offsets: torch.Tensor
    kept_idx: torch.Tensor
    n_kept: int
    n_inst: int
    sorted_gauss: torch.Tensor
    inst_pid: torch.Tensor | None  # duplicate-order index per sorted instance (API path only)
    order: torch.Tensor | None
    tile_start: torch.Tensor
    tile_end: torch.Tensor
    tile_order: torch.Tensor | None  # heaviest-first launch order of the compositing kernels
    out_img: torch.Tensor
    out_t: torch.Tensor
    out_last: torch.Tensor
    n_contrib: torch.Tensor | None
    api: dict = field(default_factory=dict)
    visited: torch.Tensor | None = None  # per-instance bitmask of the latest backward_rows
    defer: torch.Tensor | None = None  # fast-T forward: [count, pixels re-blended in float64]
    counts: torch.Tensor | None = None  # device (n_kept, n_inst)
    counts_on_device: bool = False  # device-count binning: n_kept / n_inst above are the capacity

    @property
    def n_deferred(self) -> int:
        """Pixels the fast-T forward handed to its float64 fix-up pass (host sync)."""
        return 0 if self.defer is None else int(self.defer[0].item())

    @property
    def real(self):
        return torch.float64 if self.store_f64 else torch.float32


class Rasterizer:
    """Forward / backward of the tile rasteriser on the current CUDA stream.

    ``pooled=True`` reuses scratch between calls (training loops: forward, loss and
    backward of one view complete before the next view starts); ``pooled=False``
    gives every Frame its own buffers (the reference-shaped API, where a RenderState
    may outlive later renders)."""

    def __init__(self, settings: RasterSettings = DEFAULT_SETTINGS, n_channels: int = 3,
                 store_f64: bool = False, pooled: bool = True, fast_t: bool = False, cull: bool = False):
        if n_channels not in (3, 11):
            raise ValueError("n_channels must be 3 (rgb) or 11 (rgb + aux planes)")
        self.device = require_cuda()
        self.settings = settings
        self.st = settings_struct(settings)
        self.n_ch = n_channels
        self.store_f64 = store_f64
        self.real = torch.float64 if store_f64 else torch.float32
        self.pool = Pool(self.device) if pooled else None
        self._count_slots: list = []  # free (pinned counts, event) pairs, see _bin_begin
        self.timer = None  # optional KernelTimer: CUDA events around each launch group
        self.launches = 0  # kernels launched by this rasteriser (see LAUNCHES)
        self.last_counts = (0, 0)  # (kept splats, tile instances) of the latest forward
        self.contrib_counts = True  # per-pixel contributor counts (the trainer turns them off)
        # float32 blends: carry T in float32 with exact decisions (vegs_composite_forward_fast)
        # instead of the float64 chain that reproduces the reference's T bit for bit
        self.fast_t = fast_t
        # cull=True (training and render pipelines): bin on the tight ellipse boxes (_culls)
        self.cull = cull
        # device-count binning (set by the Trainer): an int64[2] step state shared by the
        # views of a step and the instance capacity of this rasteriser's pooled buffers
        self.device_counts: torch.Tensor | None = None
        self.inst_cap = 0  # tile instances a view may have
        self.kept_cap = 0  # kept splats a view may have (sizes the placement's chunk grid)

    @staticmethod
    def _placement(width: int, height: int) -> bool:
        """Counting placement (<= 12288 tiles, VEGS_BIN_RADIX unset) -- the C library's rule."""
        tx, ty = (width + TILE - 1) // TILE, (height + TILE - 1) // TILE
        return (tx + 1) * (ty + 1) <= 12288 and os.environ.get("VEGS_BIN_RADIX", "")[:1] in ("", "0")

    @staticmethod
    def _two_level(width: int, height: int) -> bool:
        """Two-level placement (the C library's rule: from 4096 tiles, VEGS_PLACE_FLAT overrides)."""
        env = os.environ.get("VEGS_PLACE_FLAT", "")[:1]
        tiles = ((width + TILE - 1) // TILE) * ((height + TILE - 1) // TILE)
        return env == "0" if env else tiles >= 4096

    @staticmethod
    def _small_sort(n_sort: int) -> bool:
        """The one-CTA depth sort (the C library's rule: <= 16384 keys, VEGS_SMALL_SORT=0 disables)."""
        return n_sort <= 16384 and os.environ.get("VEGS_SMALL_SORT", "")[:1] != "0"

    def _culls(self) -> bool:
        """Culled binning (tight ellipse boxes, float32 tables): tile lists hold only the
        instances that can blend in their tile.  Same images and gradients; out_last and the
        tile ranges then index the shorter lists, so the reference-shaped API never culls."""
        return self.cull and not self.store_f64

    def _run(self, name: str, *args) -> None:
        if self.timer is not None:
            self.timer.mark(name, True, self)
        call(name, *args)
        if self.timer is not None:
            self.timer.mark(name, False, self)
        self.launches += LAUNCHES.get(name, 1)

    def _alloc(self):
        return self.pool if self.pool is not None else _Fresh(self.device)

    # -- forward --------------------------------------------------------------------
    def forward_begin(self, params: torch.Tensor, n: int, tf: DeviceTF, cam, background=(1.0, 1.0, 1.0),
                      want_order: bool = False, api_views: bool = False, proj: torch.Tensor | None = None) -> dict:
        """First half of a forward: preprocess + instance count, with the count copied to
        pinned host memory asynchronously.  ``forward_end`` waits for it and finishes; a
        caller can queue other streams' work in between (see Trainer)."""
        A = self._alloc()
        rs = rec_stride(self.n_ch)
        record = A.get("record", n * rs, self.real)
        rect = A.get("rect", n * 4, torch.int32)
        tiles = A.get("tiles", n, torch.int32)
        depth_key = A.get("depth_key", n, torch.int64)
        tab = VegsSplatTable(_p(record), _p(rect), _p(tiles), _p(depth_key))
        api = {}
        if api_views:
            api = dict(mean2d=A.get("a_mean2d", 2 * n, torch.float64), conic=A.get("a_conic", 3 * n, torch.float64),
                       depth=A.get("a_depth", n, torch.float64), alpha_base=A.get("a_ab", n, torch.float64),
                       color=A.get("a_color", 3 * n, torch.float64), radius=A.get("a_radius", n, torch.float64),
                       visible=A.get("a_visible", n, torch.uint8), aux=A.get("a_aux", 24 * n, torch.float64))
            for k, v in api.items():
                setattr(tab, k, _p(v))
        cs = camera_struct(cam)
        if proj is not None:  # this camera's projection, computed once for several TFs (RenderPipeline)
            if api_views:
                raise ValueError("api_views needs the full preprocess (no shared projection)")
            self._run("vegs_preprocess_forward_projected", _p(params), n, ctypes.byref(cs), ctypes.byref(tf.struct),
                      ctypes.byref(self.st), self.n_ch, int(self.store_f64), _p(proj), ctypes.byref(tab), _stream())
        else:
            self._run("vegs_preprocess_forward", _p(params), n, ctypes.byref(cs), ctypes.byref(tf.struct),
                      ctypes.byref(self.st), self.n_ch, int(self.store_f64), ctypes.byref(tab), _stream())
        return self._bin_begin(A, n, record, rect, tiles, depth_key, cam.width, cam.height, background, cs, tf,
                               params, want_order, api)

    def forward(self, params: torch.Tensor, n: int, tf: DeviceTF, cam, background=(1.0, 1.0, 1.0),
                want_order: bool = False, api_views: bool = False) -> Frame:
        return self.forward_end(self.forward_begin(params, n, tf, cam, background, want_order, api_views))

    def forward_from_splats(self, mean2d, conic, alpha_base, depth, rect, channels, width, height,
                            background, want_order: bool = True) -> Frame:
        """rasterize_forward on already-projected splats (pipeline.py:197-237)."""
        A = self._alloc()
        m = int(alpha_base.shape[0])
        rs = rec_stride(self.n_ch)
        record = A.get("record", m * rs, self.real)
        rect_d = A.get("rect", m * 4, torch.int32)
        tiles = A.get("tiles", m, torch.int32)
        depth_key = A.get("depth_key", m, torch.int64)
        tab = VegsSplatTable(_p(record), _p(rect_d), _p(tiles), _p(depth_key))
        self._run("vegs_splat_table_from_arrays", _p(mean2d), _p(conic), _p(alpha_base), _p(depth), _p(rect),
             _p(channels), m, ctypes.byref(self.st), self.n_ch, int(self.store_f64), ctypes.byref(tab), _stream())
        return self.forward_end(self._bin_begin(A, m, record, rect_d, tiles, depth_key, width, height, background,
                                                None, None, None, want_order, {}))

    def _bin_begin(self, A, n, record, rect, tiles, depth_key, width, height, background, cs, tf, params,
                   want_order, api) -> dict:
        offsets = A.get("offsets", n + 1, torch.int64)
        kept_idx = A.get("kept_idx", n + 1, torch.int64)
        counts = A.get("counts", 2, torch.int64)
        s = _stream()
        wsz = _lib.size_query("vegs_bin_count", _p(tiles), n, _p(offsets), _p(kept_idx), _p(counts), tail=(s,))
        ws = A.get("ws_count", wsz, torch.uint8)
        if self.device_counts is not None and not want_order and self._placement(width, height):
            # counts stay on the device (no host round trip: CUDA-graph capturable); a view
            # above the instance capacity is emptied and flagged in the step state
            poison = A.get("poison", 1, torch.int32)
            self._run("vegs_bin_count_dev", _p(tiles), n, _p(offsets), _p(kept_idx), _p(counts),
                      int(self.inst_cap), int(self.kept_cap), _p(self.device_counts), _p(poison), _p(ws),
                      ctypes.byref(ctypes.c_size_t(wsz)), s)
            return dict(A=A, n=n, record=record, rect=rect, tiles=tiles, depth_key=depth_key, width=width,
                        height=height, background=background, cs=cs, tf=tf, params=params, want_order=want_order,
                        api=api, offsets=offsets, kept_idx=kept_idx, counts=counts, device=True)
        self._run("vegs_bin_count", _p(tiles), n, _p(offsets), _p(kept_idx), _p(counts), _p(ws),
             ctypes.byref(ctypes.c_size_t(wsz)), s)
        # pinned count buffer + event from a free list (a pinned allocation per view costs
        # ~60 us of host time); returned in forward_end once the host has read the counts
        slot = self._count_slots.pop() if self._count_slots else (
            torch.empty(2, dtype=torch.int64, pin_memory=True), torch.cuda.Event())
        host, ev = slot
        host.copy_(counts, non_blocking=True)
        ev.record(torch.cuda.current_stream(self.device))
        return dict(slot=slot, A=A, n=n, record=record, rect=rect, tiles=tiles, depth_key=depth_key, width=width,
                    height=height, background=background, cs=cs, tf=tf, params=params, want_order=want_order,
                    api=api, offsets=offsets, kept_idx=kept_idx, host=host, event=ev)

    def forward_end(self, pend: dict) -> Frame:
        """Second half: wait for the instance count (the one host sync per view), then sort
        and composite on the current stream."""
        A, n, record, rect, tiles, depth_key = (pend[k] for k in ("A", "n", "record", "rect", "tiles", "depth_key"))
        width, height, background, cs, tf, params = (pend[k] for k in ("width", "height", "background", "cs", "tf",
                                                                       "params"))
        want_order, api, offsets, kept_idx = pend["want_order"], pend["api"], pend["offsets"], pend["kept_idx"]
        s = _stream()
        tiles_x = (width + TILE - 1) // TILE
        n_tiles = tiles_x * ((height + TILE - 1) // TILE)
        tile_start = A.get("tile_start", n_tiles, torch.int32)
        tile_end = A.get("tile_end", n_tiles, torch.int32)
        tile_order = A.get("tile_order", n_tiles, torch.int32)
        inst_pid = order = None
        if pend.get("device"):
            # capacity-sized buffers, counts read by the kernels from the device
            n_kept, n_inst = int(self.kept_cap), int(self.inst_cap)  # capacities (the counts stay on the device)
            sorted_gauss = A.get("sorted_gauss", n_inst, torch.int32)
            args = (_p(depth_key), _p(rect), _p(offsets), _p(kept_idx), n, _p(pend["counts"]), int(self.kept_cap),
                    int(self.inst_cap), width, height, TILE, _p(sorted_gauss), _p(tile_start), _p(tile_end), _p(tile_order),
                    _p(record) if self._culls() else None, self.n_ch)
            wsz = _lib.size_query("vegs_bin_sort_dev", *args, tail=(s,))
            ws = A.get("ws_sort", wsz, torch.uint8)
            self._run("vegs_bin_sort_dev", *args, _p(ws), ctypes.byref(ctypes.c_size_t(wsz)), s)
            # the capacity check of vegs_bin_count_dev (+ the binning rects, + the second placement
            # level, - the device-wide depth sort's 6 launches for one when <= 16384 splats are sorted)
            self.launches += 2 + self._culls() + 5 * self._two_level(width, height) - 5 * self._small_sort(
                min(int(self.kept_cap), n))
        else:
            pend["event"].synchronize()
            n_kept, n_inst = (int(x) for x in pend["host"].tolist())
            self._count_slots.append(pend.pop("slot"))
            sorted_gauss = A.get("sorted_gauss", n_inst, torch.int32)
            inst_pid = A.get("inst_pid", n_inst, torch.int32) if want_order else None
            order = A.get("order", n_inst, torch.int64) if want_order else None
            cull = self._culls() and not want_order and self._placement(width, height)
            args = (_p(tiles), _p(depth_key), _p(rect), _p(offsets), _p(kept_idx), n, n_kept, n_inst, width, height,
                    TILE, _p(sorted_gauss), _p(inst_pid), _p(order), _p(tile_start), _p(tile_end), _p(tile_order),
                    _p(record) if cull else None, self.n_ch)
            wsz = _lib.size_query("vegs_bin_sort", *args, tail=(s,))
            ws = A.get("ws_sort", wsz, torch.uint8)
            self._run("vegs_bin_sort", *args, _p(ws), ctypes.byref(ctypes.c_size_t(wsz)), s)
            if cull:
                self.launches += 1  # the binning rects
            if not self._placement(width, height):
                self.launches += 1  # radix path
            else:
                self.launches += 5 * self._two_level(width, height) - 5 * self._small_sort(n)
            if self._placement(width, height) and want_order:
                self.launches += 1  # order / inst_pid for the reference-shaped API
        self.last_counts = (n_kept, n_inst)
        hw = width * height
        out_img = A.get("out_img", hw * self.n_ch, self.real)
        out_t = A.get("out_t", hw, self.real)
        out_last = A.get("out_last", hw, torch.int32)
        n_contrib = A.get("n_contrib", hw, torch.int32) if self.contrib_counts else None
        bg = (ctypes.c_double * 3)(*[float(x) for x in background])
        defer = None
        if self.fast_t and not self.store_f64:
            defer = A.get("defer", hw + 1, torch.int32)
            self._run("vegs_composite_forward_fast", _p(tile_start), _p(tile_end), _p(sorted_gauss), _p(record),
                      _p(rect), self.n_ch, bg, width, height, float(self.settings.alpha_clamp),
                      float(self.settings.transmittance_stop), _p(out_img), _p(out_t), _p(out_last), _p(n_contrib),
                      _p(tile_order), _p(defer), s)
        else:
            self._run("vegs_composite_forward", _p(tile_start), _p(tile_end), _p(sorted_gauss), _p(record), _p(rect),
                      self.n_ch, int(self.store_f64), bg, width, height, float(self.settings.alpha_clamp),
                      float(self.settings.transmittance_stop), _p(out_img), _p(out_t), _p(out_last), _p(n_contrib),
                      _p(tile_order), s)
        return Frame(n=n, n_ch=self.n_ch, store_f64=self.store_f64, width=width, height=height, cam=cs, tf=tf,
                     settings=self.st, bg=bg, params=params, record=record, rect=rect, tiles=tiles,
                     depth_key=depth_key, offsets=offsets, kept_idx=kept_idx, n_kept=n_kept, n_inst=n_inst,
                     sorted_gauss=sorted_gauss, inst_pid=inst_pid, order=order, tile_start=tile_start,
                     tile_end=tile_end, tile_order=tile_order, out_img=out_img, out_t=out_t, out_last=out_last,
                     n_contrib=n_contrib, api=api, defer=defer, counts=pend.get("counts"),
                     counts_on_device=bool(pend.get("device")))

    # -- backward -------------------------------------------------------------------
    def backward_rows(self, fr: Frame, d_img: torch.Tensor, d_alpha: torch.Tensor | None = None) -> torch.Tensor:
        """Per-instance gradient rows (duplicate order) from the backward tile blend."""
        A = self._alloc()
        rs = rec_stride(fr.n_ch)
        rows = A.get("rows", max(fr.n_inst, 1) * rs, fr.real)
        if d_alpha is None:
            d_alpha = A.get("zero_alpha", fr.width * fr.height, fr.real)
            d_alpha.zero_()
        d_img, d_alpha = d_img.contiguous(), d_alpha.contiguous()  # referenced until enqueued
        fr.visited = A.get("visited", (max(fr.n_inst, 1) + 31) // 32, torch.int32)
        self._run("vegs_composite_backward", _p(fr.tile_start), _p(fr.tile_end), _p(fr.sorted_gauss), _p(fr.offsets),
             _p(fr.record), _p(fr.rect), fr.n_ch, int(fr.store_f64), fr.bg, fr.width, fr.height,
             float(self.settings.alpha_clamp), _p(fr.out_t), _p(fr.out_last), _p(d_img),
             _p(d_alpha), _p(rows), _p(fr.visited), fr.n_inst, _p(fr.tile_order), _stream())
        return rows

    def backward(self, fr: Frame, d_img: torch.Tensor, d_alpha: torch.Tensor | None = None,
                 grads: torch.Tensor | None = None, scale: float = 1.0, accumulate: bool = False,
                 viewspace_norm: torch.Tensor | None = None, visible: torch.Tensor | None = None,
                 densify_stats: torch.Tensor | None = None) -> torch.Tensor:
        """Full analytic backward into the flat float64 gradient buffer (19 n)."""
        if fr.params is None:
            raise ValueError("backward through the full chain needs a Frame from forward()")
        rows = self.backward_rows(fr, d_img, d_alpha)
        if grads is None:
            grads = torch.empty(19 * fr.n, dtype=torch.float64, device=self.device)
        args = (_p(fr.params), fr.n, ctypes.byref(fr.cam), ctypes.byref(fr.tf.struct), ctypes.byref(fr.settings),
                fr.n_ch, int(fr.store_f64), _p(fr.tiles), _p(fr.offsets), _p(rows), float(scale), int(accumulate),
                _p(grads), _p(viewspace_norm), _p(visible), _p(densify_stats), _p(fr.visited), int(fr.n_kept))
        wsz = _lib.size_query("vegs_preprocess_backward", *args, tail=(_stream(),))
        ws = self._alloc().get("ws_pbwd", wsz, torch.uint8)
        self._run("vegs_preprocess_backward", *args, _p(ws), ctypes.byref(ctypes.c_size_t(wsz)), _stream())
        return grads


# -- small device utilities -------------------------------------------------------------

def tf_eval(ts, vals, v, derivative: bool) -> np.ndarray:
    """Device TF lookup (interp or half-open slope) for host arrays; returns (..., n_cols)."""
    dev = require_cuda()
    ts = np.ascontiguousarray(ts, dtype=np.float64)
    vals = np.asarray(vals, dtype=np.float64)
    q = np.asarray(v, dtype=np.float64)
    shape = q.shape
    cols = vals.shape[1]
    ts_d = torch.from_numpy(ts).to(dev)
    vals_d = torch.from_numpy(np.ascontiguousarray(vals.T)).to(dev)  # column-major
    q_d = torch.from_numpy(np.ascontiguousarray(q.ravel())).to(dev)
    out = torch.empty(q_d.numel() * cols, dtype=torch.float64, device=dev)
    call("vegs_tf_eval", _p(ts_d), _p(vals_d), len(ts), cols, _p(q_d), q_d.numel(), int(derivative), _p(out),
         _stream())
    return out.cpu().numpy().reshape(shape + (cols,))


class LossKernel:
    """Fused L1 + SSIM forward/backward (vegs_loss_l1_ssim) and the aux-plane regularisers
    (vegs_loss_aux), with reusable workspaces."""

    def __init__(self, device=None):
        self.device = device or require_cuda()
        self.pool = Pool(self.device)
        self.timer = None  # optional KernelTimer, as on Rasterizer

    def __call__(self, x: torch.Tensor, y: torch.Tensor, w_l1: float, lam: float, d_x: torch.Tensor,
                 sums: torch.Tensor) -> None:
        """x: (H, W, S) float32 with rgb in channels 0..2 (S = 3 or 11); y: (H, W, 3)."""
        h, w, xs = int(x.shape[0]), int(x.shape[1]), int(x.shape[2])
        nbytes = _lib.size_query("vegs_loss_l1_ssim", _p(x), _p(y), h, w, xs, float(w_l1), float(lam), _p(d_x),
                                 _p(sums), tail=(_stream(),))
        ws = self.pool.get("ws", nbytes, torch.uint8)
        if self.timer is not None:
            self.timer.mark("vegs_loss_l1_ssim", True)
        call("vegs_loss_l1_ssim", _p(x), _p(y), h, w, xs, float(w_l1), float(lam), _p(d_x), _p(sums), _p(ws),
             ctypes.byref(ctypes.c_size_t(nbytes)), _stream())
        if self.timer is not None:
            self.timer.mark("vegs_loss_l1_ssim", False)

    def aux(self, planes: torch.Tensor, out_t: torch.Tensor, ref: torch.Tensor, px_scale: float, w_normal: float,
            w_smooth: float, d_planes: torch.Tensor, sums3: torch.Tensor) -> None:
        h, w = int(planes.shape[0]), int(planes.shape[1])
        nbytes = _lib.size_query("vegs_loss_aux", _p(planes), _p(out_t), _p(ref), h, w, float(px_scale),
                                 float(w_normal), float(w_smooth), _p(d_planes), _p(sums3), tail=(_stream(),))
        ws = self.pool.get("ws_aux", nbytes, torch.uint8)
        call("vegs_loss_aux", _p(planes), _p(out_t), _p(ref), h, w, float(px_scale), float(w_normal),
             float(w_smooth), _p(d_planes), _p(sums3), _p(ws), ctypes.byref(ctypes.c_size_t(nbytes)), _stream())


def adam_step_device(params, grads, m, v, n: int, lrs: torch.Tensor, grad_scale: float, step: int,
                     nonfinite: torch.Tensor, extra_grads=()) -> None:
    """Adam on grads (+ up to three more partial buffers, summed into ``grads`` first in
    a fixed order); ``params=None`` only forms the sum."""
    b1, b2 = 0.9, 0.999
    if len(extra_grads) > 3:
        raise ValueError("at most 4 partial gradient buffers")
    if params is not None and not extra_grads:
        call("vegs_adam_step", _p(params), _p(grads), _p(m), _p(v), n, _p(lrs), float(grad_scale),
             1.0 - b1 ** step, 1.0 - b2 ** step, _p(nonfinite), _stream())
        return
    ex = list(extra_grads) + [None] * (3 - len(extra_grads))
    hyper = None
    if params is not None:
        hyper = torch.cat([lrs.to(torch.float64), torch.tensor([1.0 - b1 ** step, 1.0 - b2 ** step],
                                                               dtype=torch.float64, device=lrs.device)])
    call("vegs_adam_step_sum", _p(params), _p(grads), _p(ex[0]), _p(ex[1]), _p(ex[2]), _p(m), _p(v), n, _p(hyper),
         float(grad_scale), _p(nonfinite), None, _stream())


def adam_step_sum_device(params, grads, m, v, n: int, hyper: torch.Tensor, nonfinite: torch.Tensor, extra_grads=(),
                         skip: torch.Tensor | None = None) -> None:
    """The trainer's Adam: ``hyper`` (device, 12 float64: lr per class, 1 - beta1^t,
    1 - beta2^t) is read at execution time (graph replay); ``skip`` (device int64) set by an
    overflowed view leaves everything unchanged."""
    ex = list(extra_grads) + [None] * (3 - len(extra_grads))
    call("vegs_adam_step_sum", _p(params), _p(grads), _p(ex[0]), _p(ex[1]), _p(ex[2]), _p(m), _p(v), n, _p(hyper),
         1.0, _p(nonfinite), _p(skip), _stream())


def grad_pack_device(grads, extra_grads, payload32, n: int, unit0: int, units: int) -> None:
    """Sum the lanes' partial gradients of units [unit0, unit0 + units) (fixed order) into
    ``payload32`` (float32) or, when it is None, into ``grads``."""
    ex = list(extra_grads) + [None] * (3 - len(extra_grads))
    call("vegs_grad_pack", _p(grads), _p(ex[0]), _p(ex[1]), _p(ex[2]), _p(payload32), n, unit0, units, _stream())


def adam_step_range_device(params, grads, payload32, m, v, n: int, unit0: int, units: int, hyper: torch.Tensor,
                           nonfinite: torch.Tensor, skip: torch.Tensor | None = None) -> None:
    """Adam over units [unit0, unit0 + units) on the exchanged gradient (``payload32`` when
    given, widened into ``grads``; else ``grads``)."""
    call("vegs_adam_step_range", _p(params), _p(grads), _p(payload32), _p(m), _p(v), n, unit0, units, _p(hyper),
         _p(nonfinite), _p(skip), _stream())


class RenderPipeline:
    """Forward renders of many (camera, TF) pairs pipelined over CUDA streams: the next
    render's preprocess and instance count are queued before waiting on the current one's
    count, so the small per-view kernels overlap the previous view's compositing.
    Output frames are only valid until the lane that produced them is reused."""

    def __init__(self, settings: RasterSettings = DEFAULT_SETTINGS, n_channels: int = 3, lanes: int = 4,
                 fast_t: bool = False, cull: bool = True, project_once: bool = True):
        dev = self.device = require_cuda()
        main = torch.cuda.current_stream(dev)
        self.lanes = [(main if i == 0 else torch.cuda.Stream(dev),
                       Rasterizer(settings, n_channels, pooled=True, fast_t=fast_t, cull=cull))
                      for i in range(max(1, lanes))]
        for _, rz in self.lanes:
            rz.contrib_counts = False  # images only
        # project_once: items sharing a camera object (a TF sweep) share one projection
        # (vegs_project), each TF then only shades and takes its rect; identical frames
        self.project_once = project_once
        self._proj_pool = Pool(dev)
        self.launches = 0

    def render(self, params: torch.Tensor, n: int, items, background=(1.0, 1.0, 1.0), on_frame=None) -> int:
        """items: list of (camera, DeviceTF).  on_frame(i, frame) is called (on the frame's
        stream) right after each composite.  Returns the total instance count."""
        main = torch.cuda.current_stream(self.device)
        proj = {}
        if self.project_once:  # cameras used by several items: projected once, on the caller's stream
            uses: dict = {}
            for cam, _ in items:
                uses[id(cam)] = uses.get(id(cam), 0) + 1
            st = self.lanes[0][1].st
            for cam, _ in items:
                if uses[id(cam)] > 1 and id(cam) not in proj:
                    buf = self._proj_pool.get(f"proj{len(proj)}", 8 * n, torch.float64)
                    call("vegs_project", _p(params), n, ctypes.byref(camera_struct(cam)), ctypes.byref(st), _p(buf),
                         _stream())
                    self.launches += 1
                    proj[id(cam)] = buf
        for i, (s, _) in enumerate(self.lanes):
            if i or s != main:  # lane 0 is the construction-time stream
                s.wait_stream(main)
        L = len(self.lanes)
        pend = [None] * len(items)

        def begin(i):
            s, rz = self.lanes[i % L]
            with use_stream(s):
                pend[i] = rz.forward_begin(params, n, items[i][1], items[i][0], background,
                                           proj=proj.get(id(items[i][0])))

        total = 0
        ahead = L > 1  # one lane: item i+1 must not overwrite item i's pooled table early
        if items:
            begin(0)
        for i in range(len(items)):
            if ahead and i + 1 < len(items):
                begin(i + 1)
            s, rz = self.lanes[i % L]
            with use_stream(s):
                fr = rz.forward_end(pend[i])
                pend[i] = None
                total += fr.n_inst
                if on_frame is not None:
                    on_frame(i, fr)
            if not ahead and i + 1 < len(items):
                begin(i + 1)
        for i, (s, _) in enumerate(self.lanes):
            if i or s != main:
                main.wait_stream(s)
        return total
