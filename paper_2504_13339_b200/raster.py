"""Reference-shaped rasteriser API (drop-in for ``vegsplat.raster``).

Same names, signatures, dataclasses and error behaviour as
/root/reference/pkg/src/vegsplat/raster/pipeline.py (and raster/__init__.py:3-39):
``build_splat_data``, ``rasterize_forward``, ``rasterize_backward``, ``render``,
``render_with_state``, ``SplatData``, ``BlendState``, ``RenderState``, ``ImageGradients``,
``GradientSet``.  Inputs and outputs are numpy (float64 parameters, ``dtype`` blend
planes) exactly like the reference; every computation runs on the GPU through the
C-ABI (see device.py).  Bulk arrays of the states (instance arrays, T, last
contributor) stay on the device and are copied to numpy lazily on attribute access.

For training at scale use ``paper_2504_13339_b200.train.Trainer`` (device-resident
parameters, no per-call host copies).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .camera import Camera
from .constants import DEFAULT_SETTINGS, RasterSettings
from .device import DeviceTF, Frame, Rasterizer, rec_stride, require_cuda
from .images import ImageBuffer
from .model import BETA_MAX, GaussianSet, PARAM_CLASSES
from .transfer import TransferFunction

N_AUX_CHANNELS = 11
ATTR_PLANE_NAMES = ("k_ambient", "k_diffuse", "k_specular", "shininess_norm")


def _np(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()


def _dtype_flag(dtype) -> bool:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return True
    if dt == np.float32:
        return False
    raise ValueError(f"unsupported blend dtype {dt}; use float32 or float64")


@dataclass
class SplatData:
    mean2d: np.ndarray
    conic: np.ndarray
    alpha_base: np.ndarray
    depth: np.ndarray
    rect: np.ndarray
    channels: np.ndarray


@dataclass
class ShadeResult:
    """Per-Gaussian shading outputs and caches (shading.py:30-49), float64."""

    color: np.ndarray
    alpha_base: np.ndarray
    visible: np.ndarray
    v: np.ndarray
    w: np.ndarray
    opacity: np.ndarray
    cmap: np.ndarray
    light: np.ndarray
    light_dist: np.ndarray
    n_hat: np.ndarray
    n_norm: np.ndarray
    ndotl: np.ndarray
    ka: np.ndarray
    kd: np.ndarray
    ks: np.ndarray
    beta: np.ndarray
    spec_pow: np.ndarray


@dataclass
class ProjectResult:
    """Projection outputs on the kept subset (projection.py:43-66); float64."""

    in_view: np.ndarray
    mean2d: np.ndarray
    conic: np.ndarray
    cov2d: np.ndarray
    depth: np.ndarray
    radius: np.ndarray
    rect: np.ndarray


class BlendState:
    """What the backward needs to replay the blend (pipeline.py:52-74).

    Array attributes are device tensors exposed as numpy on access (cached)."""

    def __init__(self, frame: Frame, dtype, settings: RasterSettings, n_splats: int):
        self._frame = frame
        self._cache: dict = {}
        self.width, self.height = frame.width, frame.height
        self.tile_size = settings.tile_size
        self.tiles_x = (frame.width + self.tile_size - 1) // self.tile_size
        self.n_tiles = self.tiles_x * ((frame.height + self.tile_size - 1) // self.tile_size)
        self.n_splats = n_splats
        self.settings = settings
        self.dtype = np.dtype(dtype)
        bg = np.zeros(frame.n_ch)
        bg[:3] = list(frame.bg)
        self.bg_vec = bg.astype(self.dtype)

    def _get(self, name, fn):
        if name not in self._cache:
            self._cache[name] = fn()
        return self._cache[name]

    @property
    def order(self) -> np.ndarray:
        fr = self._frame
        if fr.order is not None:
            return self._get("order", lambda: _np(fr.order[:fr.n_inst]).astype(np.int64))
        return self._get("order", lambda: _np(fr.kept_idx[fr.sorted_gauss[:fr.n_inst].long()]))

    @property
    def tile_start(self) -> np.ndarray:
        return self._get("ts", lambda: _np(self._frame.tile_start).astype(np.int64))

    @property
    def tile_end(self) -> np.ndarray:
        return self._get("te", lambda: _np(self._frame.tile_end).astype(np.int64))

    def _inst_record(self, lo, hi):
        fr = self._frame
        rs = rec_stride(fr.n_ch)
        rec = fr.record[: fr.n * rs].view(fr.n, rs)[fr.sorted_gauss[:fr.n_inst].long()]
        return _np(rec[:, lo:hi])

    @property
    def inst_mean2d(self):
        return self._get("m2", lambda: np.ascontiguousarray(self._inst_record(0, 2)))

    @property
    def inst_conic(self):
        return self._get("con", lambda: np.ascontiguousarray(self._inst_record(2, 5)))

    @property
    def inst_alpha(self):
        return self._get("al", lambda: np.ascontiguousarray(self._inst_record(5, 6)[:, 0]))

    @property
    def inst_pmin(self):
        return self._get("pm", lambda: np.ascontiguousarray(self._inst_record(6, 7)[:, 0]))

    @property
    def inst_channels(self):
        return self._get("ch", lambda: np.ascontiguousarray(self._inst_record(7, 7 + self._frame.n_ch)))

    @property
    def inst_rect(self):
        fr = self._frame
        return self._get("rect", lambda: _np(fr.rect[: 4 * fr.n].view(fr.n, 4)[fr.sorted_gauss[:fr.n_inst].long()]))

    @property
    def out_t(self):
        return self._get("t", lambda: _np(self._frame.out_t).reshape(self.height, self.width))

    @property
    def out_last(self):
        return self._get("last", lambda: _np(self._frame.out_last).reshape(self.height, self.width).astype(np.int64))

    @property
    def n_contrib(self):
        """Blended instances per pixel (not in the reference; pinned by the parity tests)."""
        return self._get("ncon", lambda: _np(self._frame.n_contrib).reshape(self.height, self.width))


# -- lazy device views of the per-Gaussian caches (render_with_state's RenderState) ----------
# The reference's ShadeResult / ProjectResult hold ~17 + 7 float64 arrays per Gaussian (270 MB
# at 1M Gaussians); here each field is copied to numpy only when it is first read, so a
# render -> loss -> backward iteration moves just the image and the gradients over PCIe.

_AUX_COLS = {"v": 0, "w": 1, "opacity": 2, "cmap": (3, 6), "light": (6, 9), "light_dist": 9, "n_hat": (10, 13),
             "n_norm": 13, "ndotl": 14, "ka": 15, "kd": 16, "ks": 17, "beta": 18, "spec_pow": 19, "cov2d": (20, 23)}
_API_COLS = {"mean2d": 2, "conic": 3, "color": 3}


class _FrameViews:
    """numpy copies of a forward's per-Gaussian api tables, column by column, cached."""

    def __init__(self, fr: Frame, n: int):
        self.fr, self.n, self.cache = fr, n, {}

    def get(self, name: str) -> np.ndarray:
        if name in self.cache:
            return self.cache[name]
        fr, n = self.fr, self.n
        if name in _AUX_COLS:
            c = _AUX_COLS[name]
            aux = fr.api["aux"][: 24 * n].view(n, 24)
            out = _np(aux[:, c[0]:c[1]] if isinstance(c, tuple) else aux[:, c]).copy()
        elif name == "visible":
            out = _np(fr.api["visible"][:n]).astype(bool)
        elif name == "kept":
            out = _np(torch.nonzero(fr.tiles[:n] != 0).flatten()).astype(np.int64)
        elif name == "rect":
            out = _np(fr.rect[: 4 * n].view(n, 4)).astype(np.int32)
        else:
            k = _API_COLS.get(name, 1)
            t = fr.api[name][: k * n]
            out = _np(t.view(n, k) if k > 1 else t)
        self.cache[name] = out
        return out


class LazyShadeResult:
    """ShadeResult (shading.py:30-49) whose float64 fields are device-resident until read."""

    FIELDS = ("color", "alpha_base", "visible", "v", "w", "opacity", "cmap", "light", "light_dist", "n_hat",
              "n_norm", "ndotl", "ka", "kd", "ks", "beta", "spec_pow")

    def __init__(self, views: _FrameViews):
        self._views = views

    def __getattr__(self, name):
        if name in LazyShadeResult.FIELDS:
            return self._views.get(name)
        raise AttributeError(name)

    def materialize(self) -> ShadeResult:
        return ShadeResult(**{k: getattr(self, k) for k in self.FIELDS})


class LazyProjectResult:
    """ProjectResult (projection.py:43-66) on the kept subset, device-resident until read."""

    FIELDS = ("in_view", "mean2d", "conic", "cov2d", "depth", "radius", "rect")

    def __init__(self, views: _FrameViews):
        self._views = views

    def __getattr__(self, name):
        v = self._views
        if name == "in_view":
            key = "_in_view"
            if key not in v.cache:
                v.cache[key] = np.isin(np.flatnonzero(v.get("visible")), v.get("kept"))
            return v.cache[key]
        if name in LazyProjectResult.FIELDS:
            key = "_p_" + name
            if key not in v.cache:
                v.cache[key] = np.ascontiguousarray(v.get(name)[v.get("kept")])
            return v.cache[key]
        raise AttributeError(name)

    def materialize(self) -> ProjectResult:
        return ProjectResult(**{k: getattr(self, k) for k in self.FIELDS})


class RenderState:
    """pipeline.py:77-90: references to gs / tf / camera plus the forward's caches.
    ``shade_cache``, ``proj`` and ``kept`` are lazy device views (see LazyShadeResult)."""

    def __init__(self, gs, tf, camera, settings, shade_cache, proj, kept, blend, with_aux, image, _frame=None,
                 _rz=None):
        self.gs, self.tf, self.camera, self.settings = gs, tf, camera, settings
        self.shade_cache, self.proj, self._kept = shade_cache, proj, kept
        self.blend, self.with_aux, self.image, self._frame, self._rz = blend, with_aux, image, _frame, _rz

    @property
    def kept(self) -> np.ndarray:
        return self._kept.get("kept") if isinstance(self._kept, _FrameViews) else self._kept


@dataclass
class ImageGradients:
    rgb: np.ndarray
    alpha: np.ndarray | None = None
    depth: np.ndarray | None = None
    normal: np.ndarray | None = None
    attrs: np.ndarray | None = None


@dataclass
class GradientSet:
    position: np.ndarray
    log_scale: np.ndarray
    rotation: np.ndarray
    raw_value: np.ndarray
    raw_weight: np.ndarray
    normal: np.ndarray
    raw_ka: np.ndarray
    raw_kd: np.ndarray
    raw_ks: np.ndarray
    raw_beta: np.ndarray
    viewspace_norm: np.ndarray
    visible: np.ndarray

    @staticmethod
    def zeros(n: int) -> "GradientSet":
        return GradientSet(
            position=np.zeros((n, 3)), log_scale=np.zeros((n, 3)), rotation=np.zeros((n, 4)),
            raw_value=np.zeros(n), raw_weight=np.zeros(n), normal=np.zeros((n, 3)),
            raw_ka=np.zeros(n), raw_kd=np.zeros(n), raw_ks=np.zeros(n), raw_beta=np.zeros(n),
            viewspace_norm=np.zeros(n), visible=np.zeros(n, dtype=bool))

    def arrays(self) -> dict[str, np.ndarray]:
        return {k: getattr(self, k) for k in PARAM_CLASSES}

    def all_finite(self) -> bool:
        return all(np.all(np.isfinite(v)) for v in self.arrays().values())

    @staticmethod
    def from_flat(flat: np.ndarray, n: int, viewspace_norm: np.ndarray, visible: np.ndarray) -> "GradientSet":
        g = GaussianSet.unpack(flat, n)
        return GradientSet(**g.arrays(), viewspace_norm=viewspace_norm, visible=visible)


# -- forward ---------------------------------------------------------------------------

def _upload_params(gs: GaussianSet, device) -> torch.Tensor:
    return torch.from_numpy(gs.pack()).to(device)


def _splat_views(fr: Frame, gs_len: int, with_aux: bool):
    kept = _np(torch.nonzero(fr.tiles[:gs_len] != 0).flatten()).astype(np.int64)
    n = gs_len
    # pool buffers hold at least one element, so cut every table column to n rows
    a = {k: _np(v) for k, v in fr.api.items()}
    cut = {"aux": 24, "color": 3, "mean2d": 2, "conic": 3}
    a = {k: (v[: n * cut[k]].reshape(n, cut[k]) if k in cut else v[:n]) for k, v in a.items()}
    aux = a["aux"]
    sh = ShadeResult(color=a["color"], alpha_base=a["alpha_base"], visible=a["visible"].astype(bool),
                     v=aux[:, 0].copy(), w=aux[:, 1].copy(), opacity=aux[:, 2].copy(), cmap=aux[:, 3:6].copy(),
                     light=aux[:, 6:9].copy(), light_dist=aux[:, 9].copy(), n_hat=aux[:, 10:13].copy(),
                     n_norm=aux[:, 13].copy(), ndotl=aux[:, 14].copy(), ka=aux[:, 15].copy(), kd=aux[:, 16].copy(),
                     ks=aux[:, 17].copy(), beta=aux[:, 18].copy(), spec_pow=aux[:, 19].copy())
    vis_idx = np.flatnonzero(sh.visible)
    in_view = np.isin(vis_idx, kept)
    rect = _np(fr.rect[: 4 * n].view(n, 4))[kept].astype(np.int32)
    proj = ProjectResult(in_view=in_view, mean2d=a["mean2d"][kept], conic=a["conic"][kept],
                         cov2d=aux[kept, 20:23].copy(), depth=a["depth"][kept], radius=a["radius"][kept], rect=rect)
    ch = np.zeros((len(kept), N_AUX_CHANNELS if with_aux else 3))
    ch[:, :3] = sh.color[kept]
    if with_aux:
        ch[:, 3] = proj.depth
        ch[:, 4:7] = sh.n_hat[kept]
        ch[:, 7], ch[:, 8], ch[:, 9] = sh.ka[kept], sh.kd[kept], sh.ks[kept]
        ch[:, 10] = sh.beta[kept] / BETA_MAX
    data = SplatData(mean2d=proj.mean2d, conic=proj.conic, alpha_base=sh.alpha_base[kept], depth=proj.depth,
                     rect=rect, channels=ch)
    return data, sh, proj, kept


def build_splat_data(gs: GaussianSet, tf: TransferFunction, camera: Camera,
                     settings: RasterSettings = DEFAULT_SETTINGS,
                     with_aux: bool = False) -> tuple[SplatData, ShadeResult, ProjectResult, np.ndarray]:
    """shade + project + channel assembly on the GPU (pipeline.py:137-160)."""
    dev = require_cuda()
    rz = Rasterizer(settings, N_AUX_CHANNELS if with_aux else 3, store_f64=True, pooled=False)
    params = _upload_params(gs, dev)
    fr = rz.forward(params, len(gs), DeviceTF(tf, dev), camera, api_views=True)
    return _splat_views(fr, len(gs), with_aux)


def _image_from_frame(fr: Frame, n_ch: int) -> ImageBuffer:
    h, w = fr.height, fr.width
    img = fr.out_img.view(h, w, n_ch)
    alpha = _np(1.0 - fr.out_t.view(h, w))
    rgb = np.ascontiguousarray(_np(img[:, :, :3]))
    if n_ch == 3:
        return ImageBuffer(rgb=rgb, alpha=alpha)
    return ImageBuffer(rgb=rgb, alpha=alpha, depth=np.ascontiguousarray(_np(img[:, :, 3])),
                       normal=np.ascontiguousarray(_np(img[:, :, 4:7])),
                       attrs=np.ascontiguousarray(_np(img[:, :, 7:11])))


def rasterize_forward(data: SplatData, width: int, height: int, background,
                      settings: RasterSettings = DEFAULT_SETTINGS,
                      dtype=np.float64) -> tuple[ImageBuffer, BlendState]:
    """Tile-sorted front-to-back blending of prepared splats (pipeline.py:197-237)."""
    dev = require_cuda()
    n_ch = data.channels.shape[1]
    rz = Rasterizer(settings, n_ch, _dtype_flag(dtype), pooled=False)

    def up(a, dt):
        return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)

    fr = rz.forward_from_splats(up(data.mean2d, np.float64), up(data.conic, np.float64),
                                up(data.alpha_base, np.float64), up(data.depth, np.float64),
                                up(data.rect, np.int32), up(data.channels, np.float64), width, height,
                                np.asarray(background, dtype=np.float64)[:3], want_order=True)
    return _image_from_frame(fr, n_ch), BlendState(fr, dtype, settings, len(data.alpha_base))


def render_with_state(gs: GaussianSet, tf: TransferFunction, camera: Camera,
                      background=(1.0, 1.0, 1.0), settings: RasterSettings = DEFAULT_SETTINGS,
                      with_aux: bool = False, dtype=np.float64) -> tuple[ImageBuffer, RenderState]:
    dev = require_cuda()
    n_ch = N_AUX_CHANNELS if with_aux else 3
    rz = Rasterizer(settings, n_ch, _dtype_flag(dtype), pooled=False)
    params = _upload_params(gs, dev)
    fr = rz.forward(params, len(gs), DeviceTF(tf, dev), camera, background, want_order=True, api_views=True)
    views = _FrameViews(fr, len(gs))
    img = _image_from_frame(fr, n_ch)
    blend = BlendState(fr, dtype, settings, fr.n_kept)
    state = RenderState(gs=gs, tf=tf, camera=camera, settings=settings, shade_cache=LazyShadeResult(views),
                        proj=LazyProjectResult(views), kept=views, blend=blend, with_aux=with_aux, image=img,
                        _frame=fr, _rz=rz)
    return img, state


def render(gs: GaussianSet, tf: TransferFunction, camera: Camera,
           background=(1.0, 1.0, 1.0), settings: RasterSettings = DEFAULT_SETTINGS,
           with_aux: bool = False, dtype=np.float64) -> ImageBuffer:
    """shade -> project -> rasterize on the GPU; deterministic for fixed inputs."""
    dev = require_cuda()
    n_ch = N_AUX_CHANNELS if with_aux else 3
    rz = Rasterizer(settings, n_ch, _dtype_flag(dtype), pooled=False)
    fr = rz.forward(_upload_params(gs, dev), len(gs), DeviceTF(tf, dev), camera, background)
    return _image_from_frame(fr, n_ch)


# -- backward --------------------------------------------------------------------------

def rasterize_backward(state: RenderState, grads: ImageGradients) -> GradientSet:
    """Analytic gradients for every raw parameter (pipeline.py:272-366), float64."""
    fr, rz = state._frame, state._rz
    if fr is None:
        raise ValueError("rasterize_backward needs the RenderState returned by render_with_state")
    h, w = fr.height, fr.width
    n_ch = fr.n_ch
    real = np.float64 if fr.store_f64 else np.float32
    d_img = np.zeros((h, w, n_ch))
    d_img[:, :, :3] = grads.rgb
    if state.with_aux:
        if grads.depth is not None:
            d_img[:, :, 3] = grads.depth
        if grads.normal is not None:
            d_img[:, :, 4:7] = grads.normal
        if grads.attrs is not None:
            d_img[:, :, 7:11] = grads.attrs
    d_alpha = np.zeros((h, w)) if grads.alpha is None else np.asarray(grads.alpha, dtype=np.float64)
    dev = fr.out_t.device
    di = torch.from_numpy(np.ascontiguousarray(d_img, dtype=real)).to(dev)
    da = torch.from_numpy(np.ascontiguousarray(d_alpha, dtype=real)).to(dev)
    n = fr.n
    vs = torch.empty(n, dtype=torch.float64, device=dev)
    vis = torch.empty(n, dtype=torch.uint8, device=dev)
    flat = rz.backward(fr, di, da, viewspace_norm=vs, visible=vis)
    return GradientSet.from_flat(_np(flat), n, _np(vs), _np(vis).astype(bool))
