"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the VEG rasteriser path.

A restatement of the reference's algorithm (vegsplat, /root/reference/pkg/src/vegsplat)
in numpy float64 plus the plain-C tile kernels in ``blend.c``.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import it; the
product package never does.  It is pinned against golden vectors produced by the
reference itself (tests/golden/make_golden.py -> tests/golden/*.npz,
tests/test_oracle_golden.py).

Each function cites the reference lines it restates.  Per-Gaussian stages are written
component-wise (the same shape as the CUDA preprocess kernels) rather than with
stacked 3x3 matrices; float64 results therefore agree with the reference to the last
few ulps, which leaves every integer output (kept set, rects, sort order, last
contributor) identical in practice.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
BETA_MIN, BETA_MAX = 1.0, 128.0
N_AUX = 11

# ----------------------------------------------------------------------------- C kernels

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = HERE / "build" / "libvegs_oracle.so"
        if not path.exists():
            build()
        _LIB = ctypes.CDLL(str(path))
    return _LIB


def build() -> None:
    import subprocess

    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------------------- transfer

def tf_lookup(ts, vals, v):
    """clip to [0,1] then np.interp per column (transfer.py:91-103)."""
    v = np.clip(np.asarray(v, dtype=np.float64), 0.0, 1.0)
    vals = np.asarray(vals, dtype=np.float64)
    if vals.ndim == 1:
        return np.interp(v, ts, vals)
    return np.stack([np.interp(v, ts, vals[:, c]) for c in range(vals.shape[1])], axis=-1)


def tf_slope(ts, vals, v):
    """Slope of the half-open segment holding v (transfer.py:106-127)."""
    v = np.clip(np.asarray(v, dtype=np.float64), 0.0, 1.0)
    vals = np.asarray(vals, dtype=np.float64)
    seg = np.clip(np.searchsorted(ts, v, side="right") - 1, 0, len(ts) - 2)
    dt = ts[1:] - ts[:-1]
    dv = vals[1:] - vals[:-1]
    slopes = dv / (dt if vals.ndim == 1 else dt[:, None])
    return slopes[seg]


def _sig(x):
    return 1.0 / (1.0 + np.exp(-x))


# ----------------------------------------------------------------------------- forward

@dataclass
class Camera:
    pos: np.ndarray
    rot: np.ndarray   # rows right, up, forward (camera.py:85-90)
    focal: float
    width: int
    height: int
    near: float
    tan_y: float
    tan_x: float


def camera_of(cam) -> Camera:
    """Camera constants (camera.py:54-90) from any object with the reference fields."""
    import math

    eye = np.asarray(cam.position, dtype=np.float64)
    f = np.asarray(cam.target, dtype=np.float64) - eye
    f = f / np.linalg.norm(f)
    r = np.cross(f, np.asarray(cam.up, dtype=np.float64))
    r = r / np.linalg.norm(r)
    u = np.cross(r, f)
    rot = np.stack([r, u, f])
    tan_y = math.tan(0.5 * cam.fov_y)
    return Camera(pos=eye, rot=rot, focal=0.5 * cam.height / tan_y, width=cam.width,
                  height=cam.height, near=cam.near, tan_y=tan_y,
                  tan_x=tan_y * (cam.width / cam.height))


def quat_rot(q):
    """(n,4) unit wxyz -> 9 rotation entries r[i][j] (projection.py:27-40)."""
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    return [[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
            [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
            [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]]


def shade(gs, tf, cam: Camera, s) -> dict:
    """TF lookup + headlight Blinn-Phong + cull (shading.py:52-82)."""
    v = _sig(gs.raw_value)
    w = _sig(gs.raw_weight)
    op = tf_lookup(tf.opacity.ts, tf.opacity.values, v)
    cm = tf_lookup(tf.color.ts, tf.color.values, v)
    ab = op * w
    d = cam.pos[None, :] - gs.position
    dist = np.sqrt(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2])
    light = d / dist[:, None]
    nn = np.sqrt((gs.normal * gs.normal).sum(1))
    nh = gs.normal / np.maximum(nn, 1e-30)[:, None]
    ndl = nh[:, 0] * light[:, 0] + nh[:, 1] * light[:, 1] + nh[:, 2] * light[:, 2]
    sabs = np.abs(ndl)
    ka, kd, ks = _sig(gs.raw_ka), _sig(gs.raw_kd), _sig(gs.raw_ks)
    beta = np.clip(np.exp(gs.raw_beta), BETA_MIN, BETA_MAX)
    spec = np.where(sabs > 0.0, np.power(np.maximum(sabs, 1e-300), beta), 0.0)
    color = (ka + kd * sabs)[:, None] * cm + (ks * spec)[:, None]
    return dict(color=color, alpha_base=ab, visible=ab >= s.cull_alpha, v=v, w=w, opacity=op,
                cmap=cm, light=light, light_dist=dist, n_hat=nh, n_norm=nn, ndotl=ndl,
                ka=ka, kd=kd, ks=ks, beta=beta, spec_pow=spec)


def project(gs, idx, cam: Camera, s, alpha_base) -> dict:
    """EWA projection, level-set rect and cull on the subset idx (projection.py:69-176)."""
    pos = gs.position[idx]
    R = cam.rot
    d = pos - cam.pos[None, :]
    t = np.stack([d[:, 0] * R[i, 0] + d[:, 1] * R[i, 1] + d[:, 2] * R[i, 2] for i in range(3)], 1)
    tz = t[:, 2]
    front = tz > cam.near
    lim_x = s.frustum_limit * cam.tan_x
    lim_y = s.frustum_limit * cam.tan_y
    zs = np.where(front, tz, 1.0)
    txz, tyz = t[:, 0] / zs, t[:, 1] / zs
    xhit, yhit = np.abs(txz) > lim_x, np.abs(tyz) > lim_y
    txc = np.clip(txz, -lim_x, lim_x) * tz
    tyc = np.clip(tyz, -lim_y, lim_y) * tz
    f = cam.focal
    px = 0.5 * cam.width + f * txz
    py = 0.5 * cam.height - f * tyz

    q = gs.rotation[idx]
    qn = np.sqrt((q * q).sum(1))
    qh = q / np.maximum(qn, 1e-30)[:, None]
    r = quat_rot(qh)
    sc = np.exp(gs.log_scale[idx])
    s2 = sc * sc
    sig = [[r[i][0] * s2[:, 0] * r[j][0] + r[i][1] * s2[:, 1] * r[j][1] + r[i][2] * s2[:, 2] * r[j][2]
            for j in range(3)] for i in range(3)]
    iz = 1.0 / zs
    iz2 = iz * iz
    j00, j02 = f * iz, -f * txc * iz2
    j11, j12 = -f * iz, f * tyc * iz2
    # M = J W (2x3)
    m0 = [j00 * R[0, k] + j02 * R[2, k] for k in range(3)]
    m1 = [j11 * R[1, k] + j12 * R[2, k] for k in range(3)]

    def quad(u, vv):
        acc = 0.0
        for i in range(3):
            for k in range(3):
                acc = acc + u[i] * sig[i][k] * vv[k]
        return acc

    a = quad(m0, m0) + s.dilation
    b = quad(m0, m1)
    c = quad(m1, m1) + s.dilation
    det = a * c - b * b
    mid = 0.5 * (a + c)
    lam = mid + np.sqrt(np.maximum(mid * mid - det, 0.0))
    radius = s.radius_sigma * np.sqrt(np.maximum(lam, 0.0))
    inv_det = np.where(det > 0, 1.0 / np.where(det > 0, det, 1.0), 0.0)
    conic = np.stack([c * inv_det, -b * inv_det, a * inv_det], 1)
    ratio = np.maximum(alpha_base, s.alpha_skip) / s.alpha_skip
    rc = np.sqrt(np.maximum(lam, 0.0) * 2.0 * np.log(ratio)) + s.rect_margin_px
    x0 = np.clip(np.ceil(px - rc - 0.5).astype(np.int64), 0, cam.width)
    x1 = np.clip(np.floor(px + rc - 0.5).astype(np.int64) + 1, 0, cam.width)
    y0 = np.clip(np.ceil(py - rc - 0.5).astype(np.int64), 0, cam.height)
    y1 = np.clip(np.floor(py + rc - 0.5).astype(np.int64) + 1, 0, cam.height)
    keep = front & (det > 0) & (x1 > x0) & (y1 > y0) & np.isfinite(px) & np.isfinite(py)
    k = np.flatnonzero(keep)
    return dict(in_view=keep, mean2d=np.stack([px, py], 1)[k], conic=conic[k],
                cov2d=np.stack([a, b, c], 1)[k], depth=tz[k], radius=radius[k],
                rect=np.stack([x0, x1, y0, y1], 1)[k].astype(np.int32),
                t_cam=t[k], q_hat=qh[k], q_norm=qn[k], scale=sc[k],
                sigma=np.array([[sig[i][j][k] for j in range(3)] for i in range(3)]).transpose(2, 0, 1),
                tx_c=txc[k], ty_c=tyc[k], x_hit=xhit[k], y_hit=yhit[k], world_rot=R, focal=f)


def splat_data(gs, tf, camera, s, with_aux=False):
    """shade -> project -> channel matrix (pipeline.py:137-160)."""
    cam = camera_of(camera)
    sh = shade(gs, tf, cam, s)
    vis = np.flatnonzero(sh["visible"])
    pr = project(gs, vis, cam, s, sh["alpha_base"][vis])
    kept = vis[pr["in_view"]]
    ch = np.zeros((len(kept), N_AUX if with_aux else 3))
    ch[:, :3] = sh["color"][kept]
    if with_aux:
        ch[:, 3] = pr["depth"]
        ch[:, 4:7] = sh["n_hat"][kept]
        ch[:, 7], ch[:, 8], ch[:, 9] = sh["ka"][kept], sh["kd"][kept], sh["ks"][kept]
        ch[:, 10] = sh["beta"][kept] / BETA_MAX
    data = dict(mean2d=pr["mean2d"], conic=pr["conic"], alpha_base=sh["alpha_base"][kept],
                depth=pr["depth"], rect=pr["rect"], channels=ch)
    return data, sh, pr, kept


def instances(rect, depth, tile_size, width, height):
    """Tile duplication + lexsort((depth, tile)) + ranges (pipeline.py:163-194)."""
    tx_n = -(-width // tile_size)
    ty_n = -(-height // tile_size)
    n_tiles = tx_n * ty_n
    m = len(rect)
    if m == 0:
        z = np.zeros(n_tiles, dtype=np.int64)
        return np.zeros(0, dtype=np.int64), z, z.copy(), tx_n
    r = rect.astype(np.int64)
    a0, a1 = r[:, 0] // tile_size, (r[:, 1] - 1) // tile_size
    b0, b1 = r[:, 2] // tile_size, (r[:, 3] - 1) // tile_size
    nx, ny = a1 - a0 + 1, b1 - b0 + 1
    cnt = nx * ny
    first = np.cumsum(cnt) - cnt
    owner = np.repeat(np.arange(m, dtype=np.int64), cnt)
    j = np.arange(int(cnt.sum()), dtype=np.int64) - first[owner]
    tile = (b0[owner] + j // nx[owner]) * tx_n + a0[owner] + j % nx[owner]
    perm = np.lexsort((depth[owner], tile))
    ts = tile[perm]
    ids = np.arange(n_tiles)
    return owner[perm], np.searchsorted(ts, ids, "left"), np.searchsorted(ts, ids, "right"), tx_n


def rasterize_forward(data, width, height, background, s, dtype=np.float64):
    """Gather instance arrays in `dtype` and run the C tile kernel (pipeline.py:197-237)."""
    n_ch = data["channels"].shape[1]
    bg = np.zeros(n_ch)
    bg[:3] = np.asarray(background, dtype=np.float64)
    order, start, end, tx_n = instances(data["rect"], data["depth"], s.tile_size, width, height)
    pmin = np.log(s.alpha_skip / np.maximum(data["alpha_base"], s.alpha_skip * 1e-6))
    st = dict(order=order, tile_start=start, tile_end=end, tiles_x=tx_n, width=width,
              height=height, tile_size=s.tile_size, n_splats=len(data["alpha_base"]),
              inst_mean2d=np.ascontiguousarray(data["mean2d"][order], dtype=dtype),
              inst_conic=np.ascontiguousarray(data["conic"][order], dtype=dtype),
              inst_alpha=np.ascontiguousarray(data["alpha_base"][order], dtype=dtype),
              inst_pmin=np.ascontiguousarray(pmin[order], dtype=dtype),
              inst_rect=np.ascontiguousarray(data["rect"][order], dtype=np.int32),
              inst_channels=np.ascontiguousarray(data["channels"][order], dtype=dtype),
              bg=bg.astype(dtype), alpha_clamp=dtype(s.alpha_clamp), settings=s)
    img = np.zeros((height, width, n_ch), dtype=dtype)
    out_t = np.ones((height, width), dtype=dtype)
    last = np.full((height, width), -1, dtype=np.int64)
    ncon = np.zeros((height, width), dtype=np.int32)
    suffix = "f32" if dtype == np.float32 else "f64"
    fn = getattr(lib(), f"oracle_blend_forward_{suffix}")
    real = ctypes.c_float if dtype == np.float32 else ctypes.c_double
    fn(_p(start), _p(end), ctypes.c_int64(len(start)), ctypes.c_int64(tx_n),
       ctypes.c_int64(s.tile_size), _p(st["inst_mean2d"]), _p(st["inst_conic"]),
       _p(st["inst_alpha"]), _p(st["inst_pmin"]), _p(st["inst_rect"]),
       _p(st["inst_channels"]), ctypes.c_int64(n_ch), _p(st["bg"]), ctypes.c_int64(width),
       ctypes.c_int64(height), real(dtype(s.alpha_clamp)), real(dtype(s.transmittance_stop)),
       _p(img), _p(out_t), _p(last), _p(ncon))
    st.update(out_t=out_t, out_last=last, n_contrib=ncon, out_img=img)
    out = dict(rgb=np.ascontiguousarray(img[:, :, :3]), alpha=1.0 - out_t)
    if n_ch == N_AUX:
        out.update(depth=np.ascontiguousarray(img[:, :, 3]),
                   normal=np.ascontiguousarray(img[:, :, 4:7]),
                   attrs=np.ascontiguousarray(img[:, :, 7:11]))
    return out, st


def render_with_state(gs, tf, camera, background=(1.0, 1.0, 1.0), s=None, with_aux=False,
                      dtype=np.float64):
    """(pipeline.py:261-269)."""
    data, sh, pr, kept = splat_data(gs, tf, camera, s, with_aux)
    img, st = rasterize_forward(data, camera.width, camera.height, background, s, dtype)
    st.update(gs=gs, tf=tf, shade=sh, proj=pr, kept=kept, with_aux=with_aux, data=data)
    return img, st


# ----------------------------------------------------------------------------- backward

def blend_backward(st, d_img, d_alpha):
    """Per-instance gradients from the C tile kernel (pipeline.py:280-305)."""
    dtype = st["inst_mean2d"].dtype
    n_ch = st["inst_channels"].shape[1]
    n = len(st["order"])
    g = dict(mean2d=np.zeros((n, 2), dtype), conic=np.zeros((n, 3), dtype),
             alpha=np.zeros(n, dtype), channels=np.zeros((n, n_ch), dtype))
    suffix = "f32" if dtype == np.float32 else "f64"
    fn = getattr(lib(), f"oracle_blend_backward_{suffix}")
    real = ctypes.c_float if dtype == np.float32 else ctypes.c_double
    di = np.ascontiguousarray(d_img, dtype=dtype)
    da = np.ascontiguousarray(d_alpha, dtype=dtype)
    fn(_p(st["tile_start"]), _p(st["tile_end"]), ctypes.c_int64(len(st["tile_start"])),
       ctypes.c_int64(st["tiles_x"]), ctypes.c_int64(st["tile_size"]), _p(st["inst_mean2d"]),
       _p(st["inst_conic"]), _p(st["inst_alpha"]), _p(st["inst_pmin"]), _p(st["inst_rect"]),
       _p(st["inst_channels"]), ctypes.c_int64(n_ch), _p(st["bg"]), ctypes.c_int64(st["width"]),
       ctypes.c_int64(st["height"]), real(st["alpha_clamp"]), _p(st["out_t"]), _p(st["out_last"]),
       _p(di), _p(da), _p(g["mean2d"]), _p(g["conic"]), _p(g["alpha"]), _p(g["channels"]))
    return g


def reduce_instances(order, rows, m):
    """float64 per-splat sums in sorted-instance order (np.add.at, pipeline.py:307-316)."""
    rows = np.ascontiguousarray(rows, dtype=np.float64).reshape(len(order), -1)
    out = np.zeros((m, rows.shape[1]))
    lib().oracle_scatter_add(_p(np.ascontiguousarray(order, dtype=np.int64)),
                             ctypes.c_int64(len(order)), _p(rows), ctypes.c_int64(rows.shape[1]),
                             _p(out))
    return out


def project_backward(pr, g_m2, g_con, g_depth):
    """mean2d/conic/depth -> position, log_scale, raw quaternion (projection.py:186-277)."""
    f = pr["focal"]
    R = pr["world_rot"]
    t = pr["t_cam"]
    iz = 1.0 / t[:, 2]
    iz2 = iz * iz
    A, B, C = pr["conic"][:, 0], pr["conic"][:, 1], pr["conic"][:, 2]
    ga, gb, gc = g_con[:, 0], 0.5 * g_con[:, 1], g_con[:, 2]
    # dL/dcov = -L G L with L = [[A,B],[B,C]], G = [[ga,gb],[gb,gc]]
    l00 = A * ga + B * gb
    l01 = A * gb + B * gc
    l10 = B * ga + C * gb
    l11 = B * gb + C * gc
    G = [[-(l00 * A + l01 * B), -(l00 * B + l01 * C)],
         [-(l10 * A + l11 * B), -(l10 * B + l11 * C)]]
    j00, j02 = f * iz, -f * pr["tx_c"] * iz2
    j11, j12 = -f * iz, f * pr["ty_c"] * iz2
    M = [[j00 * R[0, k] + j02 * R[2, k] for k in range(3)],
         [j11 * R[1, k] + j12 * R[2, k] for k in range(3)]]
    S = pr["sigma"]
    # dL/dM = 2 G M Sigma ; dL/dSigma = M^T G M
    GM = [[G[i][0] * M[0][k] + G[i][1] * M[1][k] for k in range(3)] for i in range(2)]
    gM = [[2.0 * (GM[i][0] * S[:, 0, k] + GM[i][1] * S[:, 1, k] + GM[i][2] * S[:, 2, k])
           for k in range(3)] for i in range(2)]
    gS = np.empty((len(iz), 3, 3))
    for a_ in range(3):
        for b_ in range(3):
            gS[:, a_, b_] = (M[0][a_] * (G[0][0] * M[0][b_] + G[0][1] * M[1][b_])
                             + M[1][a_] * (G[1][0] * M[0][b_] + G[1][1] * M[1][b_]))
    # dL/dJ = dL/dM W^T
    gJ = [[gM[i][0] * R[j, 0] + gM[i][1] * R[j, 1] + gM[i][2] * R[j, 2] for j in range(3)]
          for i in range(2)]
    dxx = np.where(pr["x_hit"], 0.0, 1.0)
    dyy = np.where(pr["y_hit"], 0.0, 1.0)
    dxz = np.where(pr["x_hit"], pr["tx_c"] * iz, 0.0)
    dyz = np.where(pr["y_hit"], pr["ty_c"] * iz, 0.0)
    g_tx = gJ[0][2] * (-f * iz2) * dxx + g_m2[:, 0] * f * iz
    g_ty = gJ[1][2] * (f * iz2) * dyy + g_m2[:, 1] * (-f * iz)
    g_tz = (gJ[0][0] * (-f * iz2) + gJ[1][1] * (f * iz2)
            + gJ[0][2] * (2.0 * f * pr["tx_c"] * iz2 * iz - f * iz2 * dxz)
            + gJ[1][2] * (-2.0 * f * pr["ty_c"] * iz2 * iz + f * iz2 * dyz)
            + g_m2[:, 0] * (-f * t[:, 0] * iz2) + g_m2[:, 1] * (f * t[:, 1] * iz2) + g_depth)
    gt = np.stack([g_tx, g_ty, g_tz], 1)
    position = gt @ R
    q = pr["q_hat"]
    rot = np.array(quat_rot(q)).transpose(2, 0, 1)
    s2 = pr["scale"] ** 2
    rdr = np.einsum("nik,nij,njk->nk", rot, gS, rot)
    log_scale = 2.0 * s2 * rdr
    gR = 2.0 * np.einsum("nij,njk->nik", gS, rot) * s2[:, None, :]
    w, x, y, z = q[:, 0], q[:, 1], q[:, 2], q[:, 3]
    g = gR
    gw = 2.0 * (z * (g[:, 1, 0] - g[:, 0, 1]) + y * (g[:, 0, 2] - g[:, 2, 0]) + x * (g[:, 2, 1] - g[:, 1, 2]))
    gx = 2.0 * (y * (g[:, 0, 1] + g[:, 1, 0]) + z * (g[:, 0, 2] + g[:, 2, 0]) + w * (g[:, 2, 1] - g[:, 1, 2])
                - 2.0 * x * (g[:, 1, 1] + g[:, 2, 2]))
    gy = 2.0 * (x * (g[:, 0, 1] + g[:, 1, 0]) + z * (g[:, 1, 2] + g[:, 2, 1]) + w * (g[:, 0, 2] - g[:, 2, 0])
                - 2.0 * y * (g[:, 0, 0] + g[:, 2, 2]))
    gz = 2.0 * (x * (g[:, 0, 2] + g[:, 2, 0]) + y * (g[:, 1, 2] + g[:, 2, 1]) + w * (g[:, 1, 0] - g[:, 0, 1])
                - 2.0 * z * (g[:, 0, 0] + g[:, 1, 1]))
    gq = np.stack([gw, gx, gy, gz], 1)
    rotation = (gq - (gq * q).sum(1)[:, None] * q) / np.maximum(pr["q_norm"], 1e-30)[:, None]
    return position, log_scale, rotation


def shade_backward(gs, tf, sh, d_color, d_ab, d_nhat=None, d_ka=None, d_kd=None, d_ks=None,
                   d_bn=None):
    """colour/alpha/aux gradients -> raw parameters (shading.py:97-176)."""
    ndl = sh["ndotl"]
    sabs = np.abs(ndl)
    lit = sabs > 0.0
    dcc = (d_color * sh["cmap"]).sum(1)
    dcs = d_color.sum(1)
    gka, gkd, gks = dcc, dcc * sabs, dcs * sh["spec_pow"]
    if d_ka is not None:
        gka, gkd, gks = gka + d_ka, gkd + d_kd, gks + d_ks
    out = dict(raw_ka=gka * sh["ka"] * (1.0 - sh["ka"]), raw_kd=gkd * sh["kd"] * (1.0 - sh["kd"]),
               raw_ks=gks * sh["ks"] * (1.0 - sh["ks"]))
    e = np.exp(gs.raw_beta)
    active = (e > BETA_MIN) & (e < BETA_MAX)
    logs = np.where(lit, np.log(np.maximum(sabs, 1e-300)), 0.0)
    gbeta = dcs * sh["ks"] * sh["spec_pow"] * logs
    if d_bn is not None:
        gbeta = gbeta + d_bn / BETA_MAX
    out["raw_beta"] = np.where(active, gbeta * sh["beta"], 0.0)
    gsabs = dcc * sh["kd"] + np.where(lit, dcs * sh["ks"] * sh["beta"] * sh["spec_pow"]
                                      / np.maximum(sabs, 1e-300), 0.0)
    gndl = gsabs * np.sign(ndl)
    gnh = gndl[:, None] * sh["light"]
    if d_nhat is not None:
        gnh = gnh + d_nhat
    nh = sh["n_hat"]
    out["normal"] = (gnh - (gnh * nh).sum(1)[:, None] * nh) / np.maximum(sh["n_norm"], 1e-30)[:, None]
    gl = gndl[:, None] * nh
    L = sh["light"]
    out["position"] = -(gl - (gl * L).sum(1)[:, None] * L) / sh["light_dist"][:, None]
    dO = tf_slope(tf.opacity.ts, tf.opacity.values, sh["v"])
    dC = tf_slope(tf.color.ts, tf.color.values, sh["v"])
    gv = (d_color * dC).sum(1) * (sh["ka"] + sh["kd"] * sabs) + d_ab * dO * sh["w"]
    out["raw_value"] = gv * sh["v"] * (1.0 - sh["v"])
    out["raw_weight"] = d_ab * sh["opacity"] * sh["w"] * (1.0 - sh["w"])
    return out


GRAD_CLASSES = ("position", "log_scale", "rotation", "raw_value", "raw_weight", "normal",
                "raw_ka", "raw_kd", "raw_ks", "raw_beta")


def rasterize_backward(st, rgb, alpha=None, depth=None, normal=None, attrs=None):
    """Full analytic backward (pipeline.py:272-366); returns dict of float64 arrays."""
    h, w = st["height"], st["width"]
    n_ch = st["inst_channels"].shape[1]
    d_img = np.zeros((h, w, n_ch))
    d_img[:, :, :3] = rgb
    if st["with_aux"]:
        if depth is not None:
            d_img[:, :, 3] = depth
        if normal is not None:
            d_img[:, :, 4:7] = normal
        if attrs is not None:
            d_img[:, :, 7:11] = attrs
    d_alpha = np.zeros((h, w)) if alpha is None else np.asarray(alpha, dtype=np.float64)
    gi = blend_backward(st, d_img, d_alpha)
    m = st["n_splats"]
    order = st["order"]
    rows = np.concatenate([gi["mean2d"], gi["conic"], gi["alpha"][:, None], gi["channels"]], 1)
    red = reduce_instances(order, rows.astype(np.float64), m)
    g_m2, g_con, g_ab, g_ch = red[:, 0:2], red[:, 2:5], red[:, 5], red[:, 6:]
    d_depth = g_ch[:, 3] if st["with_aux"] else np.zeros(m)
    pos_p, ls_p, rot_p = project_backward(st["proj"], g_m2, g_con, d_depth)
    gs = st["gs"]
    n = len(gs.position)
    kept = st["kept"]
    dcol = np.zeros((n, 3))
    dcol[kept] = g_ch[:, :3]
    dab = np.zeros(n)
    dab[kept] = g_ab
    kw = {}
    if st["with_aux"]:
        extra = [np.zeros((n, 3))] + [np.zeros(n) for _ in range(4)]
        extra[0][kept] = g_ch[:, 4:7]
        for k in range(4):
            extra[k + 1][kept] = g_ch[:, 7 + k]
        kw = dict(d_nhat=extra[0], d_ka=extra[1], d_kd=extra[2], d_ks=extra[3], d_bn=extra[4])
    sg = shade_backward(gs, st["tf"], st["shade"], dcol, dab, **kw)
    out = {k: np.zeros_like(np.asarray(getattr(gs, k), dtype=np.float64)) for k in GRAD_CLASSES}
    out["position"] += sg["position"]
    out["position"][kept] += pos_p
    out["log_scale"][kept] = ls_p
    out["rotation"][kept] = rot_p
    for k in ("raw_value", "raw_weight", "normal", "raw_ka", "raw_kd", "raw_ks", "raw_beta"):
        out[k] = sg[k]
    vis = np.zeros(n, dtype=bool)
    vis[kept] = True
    for k in GRAD_CLASSES:
        out[k][~vis] = 0.0
    vn = np.zeros(n)
    vn[kept] = np.linalg.norm(g_m2 * np.array([0.5 * w, 0.5 * h]), axis=1)
    out["viewspace_norm"] = vn
    out["visible"] = vis
    return out


# ----------------------------------------------------------------------------- loss / adam

SSIM_WIN, SSIM_SIGMA, C1, C2 = 11, 1.5, 0.01 ** 2, 0.03 ** 2


def _gauss1d(dtype):
    xs = np.arange(SSIM_WIN) - (SSIM_WIN - 1) / 2.0
    g = np.exp(-0.5 * (xs / SSIM_SIGMA) ** 2)
    return (g / g.sum()).astype(dtype)


def _blur_valid(p):
    """Separable 11x11 Gaussian, valid positions only (loss.py:48-53)."""
    k = _gauss1d(p.dtype).astype(np.float64)
    q = p.astype(np.float64)
    v = sum(k[i] * q[i:q.shape[0] - SSIM_WIN + 1 + i] for i in range(SSIM_WIN))
    out = sum(k[i] * v[:, i:v.shape[1] - SSIM_WIN + 1 + i] for i in range(SSIM_WIN))
    return out.astype(p.dtype)


def _blur_adjoint(g, shape):
    """Exact adjoint of _blur_valid (loss.py:56-63)."""
    k = _gauss1d(g.dtype).astype(np.float64)
    q = g.astype(np.float64)
    h, w = shape
    tmp = np.zeros((q.shape[0], w))
    for i in range(SSIM_WIN):
        tmp[:, i:i + q.shape[1]] += k[i] * q
    out = np.zeros((h, w))
    for i in range(SSIM_WIN):
        out[i:i + tmp.shape[0]] += k[i] * tmp
    return out.astype(g.dtype)


def l1_ssim_loss(x, y, lam=0.2, l1_weight=None):
    """(1-lam) L1 + lam (1 - mean SSIM) and its analytic gradient (loss.py:80-168).

    l1_weight overrides the (1-lam) factor (BASELINE.json writes L1 + 0.2 (1-SSIM))."""
    x = np.asarray(x)
    y = np.asarray(y, dtype=x.dtype)
    wl1 = (1.0 - lam) if l1_weight is None else l1_weight
    diff = x - y
    l1 = float(np.abs(diff).mean())
    grad = wl1 * np.sign(diff) / diff.size
    chans = x.shape[2]
    mux = np.stack([_blur_valid(x[:, :, c]) for c in range(chans)], -1)
    muy = np.stack([_blur_valid(y[:, :, c]) for c in range(chans)], -1)
    sxx = np.stack([_blur_valid(x[:, :, c] * x[:, :, c]) for c in range(chans)], -1) - mux * mux
    syy = np.stack([_blur_valid(y[:, :, c] * y[:, :, c]) for c in range(chans)], -1) - muy * muy
    sxy = np.stack([_blur_valid(x[:, :, c] * y[:, :, c]) for c in range(chans)], -1) - mux * muy
    a1 = 2.0 * mux * muy + C1
    b1 = mux * mux + muy * muy + C1
    a2 = 2.0 * sxy + C2
    b2 = sxx + syy + C2
    smap = (a1 * a2) / (b1 * b2)
    mssim = float(smap.mean())
    coeff = -lam / smap.size
    inv = 1.0 / (b1 * b2)
    g_mu = coeff * (2.0 * muy * a2 * inv - 2.0 * mux * smap / b1 - 2.0 * muy * a1 * inv
                    + 2.0 * mux * smap / b2)
    g_xx = coeff * (-smap / b2)
    g_xy = coeff * (2.0 * a1 * inv)
    h, w = x.shape[:2]
    for c in range(chans):
        grad[:, :, c] += _blur_adjoint(g_mu[:, :, c], (h, w))
        grad[:, :, c] += 2.0 * x[:, :, c] * _blur_adjoint(g_xx[:, :, c], (h, w))
        grad[:, :, c] += y[:, :, c] * _blur_adjoint(g_xy[:, :, c], (h, w))
    total = wl1 * l1 + lam * (1.0 - mssim)
    return total, grad, l1, mssim


ADAM_B1, ADAM_B2, ADAM_EPS = 0.9, 0.999, 1e-15


def adam_update(param, grad, m, v, step, lr):
    """One bias-corrected Adam update in place (train.py:176-195); step is 1-based."""
    c1 = 1.0 - ADAM_B1 ** step
    c2 = 1.0 - ADAM_B2 ** step
    m *= ADAM_B1
    m += (1.0 - ADAM_B1) * grad
    v *= ADAM_B2
    v += (1.0 - ADAM_B2) * grad * grad
    param -= lr * ((m / c1) / (np.sqrt(v / c2) + ADAM_EPS))


def learning_rates(cfg: dict, iteration: int, extent: float = 1.0) -> dict:
    """Per-class learning rates with exponential position decay (train.py:156-173)."""
    n_it = max(cfg["iterations"], 1)
    t = min(max(iteration, 0), n_it) / n_it
    lr_pos = cfg["lr_position"] * (cfg["lr_position_final"] / cfg["lr_position"]) ** t
    if cfg.get("lr_position_scale_by_extent", False):
        lr_pos *= extent
    lit = cfg["lr_lighting"]
    return dict(position=lr_pos, log_scale=cfg["lr_scale"], rotation=cfg["lr_rotation"],
                raw_value=cfg["lr_value"], raw_weight=0.0 if cfg.get("no_weights") else cfg["lr_weight"],
                normal=lit, raw_ka=lit, raw_kd=lit, raw_ks=lit, raw_beta=lit)


# ----------------------------------------------------------------------------- densify / prune

CLASSES = ("position", "log_scale", "rotation", "raw_value", "raw_weight", "normal", "raw_ka", "raw_kd",
           "raw_ks", "raw_beta")


def tf_max_opacity(raw_value, op_maps):
    """BASELINE config 4's prune criterion: per Gaussian, the max over the training TFs of
    the opacity map at the activated value (eval_opacity, transfer.py:91-95).
    op_maps: list of (ts, values)."""
    v = np.clip(_sig(np.asarray(raw_value, dtype=np.float64)), 0.0, 1.0)
    return np.max(np.stack([np.interp(v, ts, vals) for ts, vals in op_maps]), axis=0)


def densify_and_prune(p, m, v, grad_accum, pos_accum, count, cfg, extent, rng, position_lr,
                      prune_opacity=None, max_gaussians=None):
    """train.py:237-284 on dicts of class arrays (p, m, v), with BASELINE config 4's options:
    prune_opacity (per-Gaussian max TF opacity) replaces the activated weight in the prune
    test (train.py:277-280), and max_gaussians caps the count -- when clones and splits
    would exceed it, this round densifies nothing and only prunes (the build's reconciliation,
    DESIGN.md).  Returns (p, m, v) of the new set; optimizer rows follow OptimizerState.edit_rows
    / select_rows (train.py:143-153: kept rows keep their moments, new rows start at zero)."""
    n = len(p["raw_weight"])
    cnt = np.maximum(count, 1.0)
    cand = grad_accum / cnt > cfg["densify_grad_threshold"]
    max_scale = np.exp(p["log_scale"]).max(axis=1) if n else np.zeros(0)
    small = cand & (max_scale <= cfg["percent_dense"] * extent)
    big = cand & ~small
    if cfg.get("no_weights"):
        surv_g = np.ones(n, dtype=bool)
    elif prune_opacity is not None:
        surv_g = np.asarray(prune_opacity) >= cfg["prune_weight_threshold"]
    else:
        surv_g = _sig(p["raw_weight"]) >= cfg["prune_weight_threshold"]
    if max_gaussians is not None:
        grow = int(((~big) & surv_g).sum() + (small & surv_g).sum() + 2 * (big & surv_g).sum())
        if grow > max_gaussians and (small.any() or big.any()):
            small = np.zeros(n, dtype=bool)
            big = np.zeros(n, dtype=bool)
    keep = ~big
    parts = [{k: p[k][keep] for k in CLASSES}]
    mparts = [{k: m[k][keep] for k in CLASSES}]
    vparts = [{k: v[k][keep] for k in CLASSES}]
    survive = [surv_g[keep]]
    ci = np.flatnonzero(small)
    if len(ci):
        c = {k: p[k][ci].copy() for k in CLASSES}
        g = pos_accum[ci] / cnt[ci, None]
        nrm = np.linalg.norm(g, axis=1, keepdims=True)
        d = np.where(nrm > 0, g / np.maximum(nrm, 1e-30), 0.0)
        c["position"] = c["position"] - position_lr * d
        parts.append(c)
        survive.append(surv_g[ci])
    si = np.flatnonzero(big)
    if len(si):
        for _ in range(2):
            c = {k: p[k][si].copy() for k in CLASSES}
            eps = rng.standard_normal(size=(len(si), 3))
            rot = np.moveaxis(np.array(quat_rot(c["rotation"] / np.linalg.norm(c["rotation"], axis=1,
                                                                                 keepdims=True))), 2, 0)
            off = np.einsum("nij,nj->ni", rot, np.exp(c["log_scale"]) * eps)
            c["position"] = c["position"] + off
            c["log_scale"] = c["log_scale"] - np.log(1.6)
            parts.append(c)
            survive.append(surv_g[si])
    n_new = sum(len(q["raw_weight"]) for q in parts[1:])
    zeros = {k: np.zeros((n_new,) + p[k].shape[1:]) for k in CLASSES}
    out_p = {k: np.concatenate([q[k] for q in parts]) for k in CLASSES}
    out_m = {k: np.concatenate([mparts[0][k], zeros[k]]) for k in CLASSES}
    out_v = {k: np.concatenate([vparts[0][k], zeros[k]]) for k in CLASSES}
    s = np.concatenate(survive)
    return ({k: a[s] for k, a in out_p.items()}, {k: a[s] for k, a in out_m.items()},
            {k: a[s] for k, a in out_v.items()})
