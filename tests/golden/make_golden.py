"""Generate golden vectors by running the REFERENCE (vegsplat) in this container.

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py [--ref /root/reference/pkg]

Inputs come from the build's seeded generators (paper_2504_13339_b200.scenes) and from
the reference's own test-scene generator (pkg/tests/gradcheck.py:make_scene); every
output is produced by the reference's public API (render_with_state,
rasterize_forward, rasterize_backward, compute_loss, eval_*/d_*_dv, adam_step).
The only derived quantity is the per-pixel contributor count, obtained by replaying
kernels.py:56-93 over the reference's own BlendState with the same float64
promotions; the replay must reproduce the reference's out_t and out_last exactly
before its counts are stored.

The fixtures are small (< 10 MB total) .npz files committed next to this script; the
GPU box never sees /root/reference.
"""

from __future__ import annotations

import argparse
import math
import os
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]


def _setup(ref_pkg: Path):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    sys.path.insert(0, str(ref_pkg / "src"))
    sys.path.insert(0, str(ref_pkg / "tests"))
    sys.path.insert(0, str(REPO))


def cam_fields(cam):
    return np.array(list(cam.position) + list(cam.target) + list(cam.up)
                    + [cam.fov_y, cam.width, cam.height, cam.near, cam.far], dtype=np.float64)


def tf_fields(prefix, tf):
    return {f"{prefix}op_ts": tf.opacity.ts, f"{prefix}op_vals": tf.opacity.values,
            f"{prefix}col_ts": tf.color.ts, f"{prefix}col_vals": tf.color.values}


def gs_fields(prefix, gs):
    return {f"{prefix}{k}": np.asarray(v) for k, v in gs.arrays().items()}


def to_ref_gs(vs, mine):
    return vs.model.GaussianSet(**{k: np.array(v, copy=True) for k, v in mine.arrays().items()})


def to_ref_tf(vs, mine):
    return vs.transfer.TransferFunction(
        color=vs.transfer.ColorMap(mine.color.points), opacity=vs.transfer.OpacityMap(mine.opacity.points))


def to_ref_cam(vs, mine):
    return vs.camera.Camera(position=mine.position, target=mine.target, up=mine.up, fov_y=mine.fov_y,
                            width=mine.width, height=mine.height, near=mine.near, far=mine.far)


def importlib_model(vs):
    return sys.modules["vegsplat.model"]


def replay_contributors(b, clamp, stop):
    """Contributor count per pixel by replaying kernels.py:56-93 on the BlendState."""
    h, w = b.height, b.width
    ts = b.tile_size
    t_plane = np.ones((h, w), dtype=b.inst_alpha.dtype)
    done = np.zeros((h, w), dtype=bool)
    last = np.full((h, w), -1, dtype=np.int64)
    count = np.zeros((h, w), dtype=np.int32)
    for tile in range(b.n_tiles):
        ty, tx = divmod(tile, b.tiles_x)
        x_lo, y_lo = tx * ts, ty * ts
        x_hi, y_hi = min(x_lo + ts, w), min(y_lo + ts, h)
        for i in range(b.tile_start[tile], b.tile_end[tile]):
            r = b.inst_rect[i]
            x0, x1, y0, y1 = max(r[0], x_lo), min(r[1], x_hi), max(r[2], y_lo), min(r[3], y_hi)
            if x0 >= x1 or y0 >= y1:
                continue
            ys, xs = np.mgrid[y0:y1, x0:x1]
            dx = xs + 0.5 - np.float64(b.inst_mean2d[i, 0])
            dy = ys + 0.5 - np.float64(b.inst_mean2d[i, 1])
            ca, cb, cc = (np.float64(c) for c in b.inst_conic[i])
            pw = -0.5 * (ca * dx * dx + cc * dy * dy) - cb * dx * dy
            live = ~done[y0:y1, x0:x1] & ~(pw < np.float64(b.inst_pmin[i]))
            a = np.minimum(np.float64(b.inst_alpha[i]) * np.exp(pw), np.float64(clamp))
            tt = t_plane[y0:y1, x0:x1].astype(np.float64) * (1.0 - a)
            stop_now = live & (tt < np.float64(stop))
            blend = live & ~stop_now
            done[y0:y1, x0:x1] |= stop_now
            sub_t = t_plane[y0:y1, x0:x1]
            sub_t[blend] = tt[blend].astype(t_plane.dtype)
            last[y0:y1, x0:x1][blend] = i
            count[y0:y1, x0:x1][blend] += 1
    return t_plane, last, count


def forward_fixture(vs, gs, tf, cam, bg, dtype, with_aux, probe_seed):
    rgs, rtf, rcam = to_ref_gs(vs, gs), to_ref_tf(vs, tf), to_ref_cam(vs, cam)
    img, st = vs.raster.render_with_state(rgs, rtf, rcam, bg, vs.raster.DEFAULT_SETTINGS,
                                          with_aux=with_aux, dtype=dtype)
    b = st.blend
    t_rep, last_rep, count = replay_contributors(b, dtype(0.99), dtype(1e-4))
    assert np.array_equal(last_rep, b.out_last), "contributor replay diverged (out_last)"
    if dtype == np.float32:
        assert np.array_equal(t_rep, b.out_t), "contributor replay diverged (out_t)"
    else:  # float64 T exposes numba's fast-math reassociation at the last ulp
        assert np.abs(t_rep - b.out_t).max() <= 1e-14, "contributor replay diverged (out_t)"
    rng = np.random.default_rng(probe_seed)
    h, w = cam.height, cam.width
    probe = dict(rgb=rng.uniform(-1, 1, size=(h, w, 3)), alpha=rng.uniform(-1, 1, size=(h, w)))
    if with_aux:
        probe.update(depth=rng.uniform(-1, 1, size=(h, w)), normal=rng.uniform(-1, 1, size=(h, w, 3)),
                     attrs=rng.uniform(-1, 1, size=(h, w, 4)))
    g = vs.raster.rasterize_backward(st, vs.raster.ImageGradients(**probe))
    out = dict(cam=cam_fields(cam), bg=np.asarray(bg, dtype=np.float64), **tf_fields("tf_", tf),
               **gs_fields("gs_", gs),
               kept=st.kept, rect=st.proj.rect, depth=st.proj.depth, mean2d=st.proj.mean2d,
               conic=st.proj.conic, alpha_base=st.shade_cache.alpha_base[st.kept],
               order=b.order, tile_start=b.tile_start, tile_end=b.tile_end,
               inst_pmin=b.inst_pmin, inst_channels=b.inst_channels,
               out_t=b.out_t, out_last=b.out_last, n_contrib=count, rgb=img.rgb, alpha=img.alpha)
    if with_aux:
        out.update(depth_plane=img.depth, normal_plane=img.normal, attrs_plane=img.attrs)
    out.update({f"probe_{k}": v for k, v in probe.items()})
    out.update({f"grad_{k}": v for k, v in g.arrays().items()})
    out.update(grad_viewspace_norm=g.viewspace_norm, grad_visible=g.visible)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    args = ap.parse_args()
    _setup(Path(args.ref))
    import vegsplat as vs  # noqa: E402  (the reference)
    import vegsplat.raster  # noqa: F401
    import vegsplat.loss  # noqa: F401
    import vegsplat.train  # noqa: F401
    from paper_2504_13339_b200 import scenes

    vtrain = sys.modules["vegsplat.train"]

    saved = {}

    def save(name, d):
        path = HERE / f"{name}.npz"
        np.savez_compressed(path, **d)
        saved[name] = path.stat().st_size

    # -- config 0 (BASELINE.json configs[0]) in the training dtype and the test dtype
    gs, _, tf, cams = scenes.config_scene("c0")
    cam = cams[0]
    save("c0_f32", forward_fixture(vs, gs, tf, cam, (1.0, 1.0, 1.0), np.float32, False, 7))
    save("c0_f64", forward_fixture(vs, gs, tf, cam, (1.0, 1.0, 1.0), np.float64, False, 8))
    # with auxiliary channels (C = 11, train.py:476), smaller set, random background
    small = gs.select(np.arange(1024))
    save("c0_aux_f32", forward_fixture(vs, small, tf, scenes.orbit_cameras(1, 11, 96, 80)[0],
                                       (0.2, 0.5, 0.7), np.float32, True, 9))
    # a dense near-opaque case that exercises the 0.99 clamp and 1e-4 termination
    dense = scenes.random_gaussians(3000, seed=5)
    dense.raw_weight[:] = 3.0
    dense.log_scale[:] += 0.8
    save("dense_f32", forward_fixture(vs, dense, scenes.random_tf(6, 3), scenes.orbit_cameras(1, 12, 64, 64)[0],
                                      (0.0, 0.0, 0.0), np.float32, False, 10))

    # -- reference gradient-check scenes (pkg/tests/gradcheck.py:157-180), with_aux f64
    import gradcheck

    gc = {}
    for seed in range(8):
        sc = gradcheck.make_scene(seed)
        g = gradcheck.analytic_gradients(sc)
        img, _ = vs.raster.render_with_state(sc.gs, sc.tf, sc.camera, sc.background, with_aux=True)
        p = f"s{seed}_"
        gc.update({p + "cam": cam_fields(sc.camera), p + "bg": np.asarray(sc.background)})
        gc.update(tf_fields(p + "tf_", sc.tf))
        gc.update(gs_fields(p + "gs_", sc.gs))
        gc.update({p + "probe_" + k: v for k, v in sc.probe.items()})
        gc.update({p + "grad_" + k: v for k, v in g.arrays().items()})
        gc.update({p + "rgb": img.rgb, p + "alpha": img.alpha, p + "depth_plane": img.depth})
    save("gradcheck_scenes", gc)

    # -- the raw blend boundary on reference SplatData scenes (test_rasterize.py:66-95)
    import test_rasterize

    bl = {}
    for seed in range(5):
        data, cam_s, bg, _, _ = test_rasterize.scene_splat_data(seed)
        img, b = vs.raster.rasterize_forward(data, cam_s.width, cam_s.height, bg)
        p = f"s{seed}_"
        bl.update({p + "mean2d": data.mean2d, p + "conic": data.conic, p + "alpha_base": data.alpha_base,
                   p + "depth": data.depth, p + "rect": data.rect, p + "channels": data.channels,
                   p + "bg": np.asarray(bg), p + "wh": np.array([cam_s.width, cam_s.height]),
                   p + "rgb": img.rgb, p + "alpha": img.alpha, p + "order": b.order,
                   p + "out_last": b.out_last})
    save("blend_scenes", bl)

    # -- transfer-function lookups (transfer.py:91-127) on 2..33-knot and 256-knot maps
    rng = np.random.default_rng(21)
    tfd = {}
    for j, k in enumerate((2, 3, 7, 33, 256)):
        ts = np.concatenate([[0.0], np.sort(rng.uniform(0, 1, k - 2)), [1.0]])
        if k == 256:
            ts = np.linspace(0, 1, 256)
        op = vs.transfer.OpacityMap(tuple((float(t), float(a)) for t, a in zip(ts, rng.uniform(0, 1, k))))
        cm = vs.transfer.ColorMap(tuple((float(t),) + tuple(rng.uniform(0, 1, 3)) for t in ts))
        q = np.concatenate([rng.uniform(-0.2, 1.2, 4000), ts, [0.0, 1.0, -1e-300, 1.0 + 1e-15]])
        tfd.update({f"k{j}_ts": ts, f"k{j}_op": op.values, f"k{j}_col": cm.values, f"k{j}_q": q,
                    f"k{j}_eval_op": vs.transfer.eval_opacity(op, q), f"k{j}_eval_col": vs.transfer.eval_color(cm, q),
                    f"k{j}_d_op": vs.transfer.d_opacity_dv(op, q), f"k{j}_d_col": vs.transfer.d_color_dv(cm, q)})
    save("tf_lookup", tfd)

    # -- loss (loss.py:146-168) with lambda_ssim 0.2 and the regularisers off
    class Cfg:
        lambda_ssim = 0.2
        normal_loss_weight = 0.0
        smooth_loss_weight = 0.0

    ld = {}
    for dt, name in ((np.float32, "f32"), (np.float64, "f64")):
        x = rng.uniform(0, 1, size=(40, 52, 3)).astype(dt)
        y = np.clip(x + rng.normal(scale=0.2, size=x.shape), 0, 1).astype(dt)
        total, grads, br = vs.loss.compute_loss(vs.images.ImageBuffer(rgb=x), y, Cfg())
        ld.update({f"{name}_x": x, f"{name}_y": y, f"{name}_total": np.array(total),
                   f"{name}_l1": np.array(br.l1), f"{name}_ssim": np.array(1.0 - br.ssim_term),
                   f"{name}_grad": grads.rgb})
    save("loss", ld)

    # -- loss with the auxiliary-plane regularisers on (loss.py:175-240), float32 planes
    class CfgAux:
        lambda_ssim = 0.2
        normal_loss_weight = 0.01
        smooth_loss_weight = 0.001

    rng_a = np.random.default_rng(23)
    h_a, w_a = 30, 34
    buf = dict(rgb=rng_a.uniform(0.05, 0.95, size=(h_a, w_a, 3)).astype(np.float32),
               alpha=np.where(rng_a.uniform(size=(h_a, w_a)) < 0.8, 0.9, 0.2).astype(np.float32),
               depth=(3.0 + rng_a.uniform(0, 1, size=(h_a, w_a))).astype(np.float32),
               normal=(rng_a.uniform(-1, 1, size=(h_a, w_a, 3)) + np.array([0.0, 0.0, 2.0])).astype(np.float32),
               attrs=rng_a.uniform(0.1, 0.9, size=(h_a, w_a, 4)).astype(np.float32))
    ref_a = rng_a.uniform(0, 1, size=(h_a, w_a, 3)).astype(np.float32)
    tot_a, g_a, br_a = vs.loss.compute_loss(vs.images.ImageBuffer(**buf), ref_a, CfgAux(), px_scale=0.01)
    la = {"in_" + k: v for k, v in buf.items()}
    la.update(ref=ref_a, total=np.array(tot_a), normal_term=np.array(br_a.normal), smooth_term=np.array(br_a.smooth),
              g_rgb=g_a.rgb, g_depth=g_a.depth, g_normal=g_a.normal, g_attrs=g_a.attrs)
    save("loss_aux", la)

    # -- Adam with per-class learning rates (train.py:156-195), 3 steps
    cfg = vtrain.TrainConfig(iterations=100)
    ga = scenes.random_gaussians(64, seed=31)
    rgs = to_ref_gs(vs, ga)
    opt = vtrain.OptimizerState.for_set(rgs)
    ad = {"in_" + k: np.array(v) for k, v in rgs.arrays().items()}
    for it in (1, 2, 3):
        g = vs.raster.GradientSet.zeros(len(rgs))
        for k, v in g.arrays().items():
            v[...] = rng.normal(size=v.shape)
            ad[f"g{it}_{k}"] = v.copy()
        vtrain.adam_step(rgs, g, opt, cfg, it)
    ad.update({"out_" + k: np.array(v) for k, v in rgs.arrays().items()})
    ad.update({"m_" + k: v for k, v in opt.m.items()})
    ad.update({"v_" + k: v for k, v in opt.v.items()})
    save("adam", ad)

    # -- one multi-view training step at reduced scale (render -> loss -> backward per
    #    view, mean of per-view gradients, Adam) from reference calls only
    learned = scenes.random_gaussians(2000, seed=0)
    truth = scenes.random_gaussians(2000, seed=1)
    tf2 = scenes.random_tf(2, 4)
    cams2 = scenes.orbit_cameras(2, 3, 64, 64)
    rl, rt, rtf = to_ref_gs(vs, learned), to_ref_gs(vs, truth), to_ref_tf(vs, tf2)
    ts = {}
    tot = None
    losses = []
    for v_i, c in enumerate(cams2):
        rc = to_ref_cam(vs, c)
        target = vs.raster.render(rt, rtf, rc, (1.0, 1.0, 1.0), dtype=np.float32).rgb
        img, st = vs.raster.render_with_state(rl, rtf, rc, (1.0, 1.0, 1.0), with_aux=False, dtype=np.float32)
        loss, ig, _ = vs.loss.compute_loss(img, target, Cfg())
        losses.append(loss)
        g = vs.raster.rasterize_backward(st, ig)
        ts[f"target{v_i}"] = target
        ts[f"rgb{v_i}"] = img.rgb
        if tot is None:
            tot = {k: v.copy() for k, v in g.arrays().items()}
        else:
            for k, v in g.arrays().items():
                tot[k] += v
    mean = vs.raster.GradientSet.zeros(len(rl))
    for k, v in mean.arrays().items():
        v[...] = tot[k] / len(cams2)
        ts["grad_" + k] = v.copy()
    opt = vtrain.OptimizerState.for_set(rl)
    vtrain.adam_step(rl, mean, opt, cfg, 1)
    ts.update({"out_" + k: np.array(v) for k, v in rl.arrays().items()})
    ts["losses"] = np.array(losses)
    save("train_step", ts)

    # -- the reference's own training iteration with aux planes + regularisers on
    #    (train.py:476-483, TrainConfig defaults: normal 0.01, smooth 0.001), 2 views
    cfg_aux = vtrain.TrainConfig(iterations=100)
    rl = to_ref_gs(vs, learned)
    tsa, tot, losses = {}, None, []
    for v_i, c in enumerate(cams2):
        rc = to_ref_cam(vs, c)
        target = vs.raster.render(rt, rtf, rc, (1.0, 1.0, 1.0), dtype=np.float32).rgb
        img, st = vs.raster.render_with_state(rl, rtf, rc, (1.0, 1.0, 1.0), with_aux=True, dtype=np.float32)
        px_scale = 2.0 * math.tan(0.5 * rc.fov_y) / rc.height
        loss, ig, _ = vs.loss.compute_loss(img, target, cfg_aux, px_scale=px_scale)
        losses.append(loss)
        g = vs.raster.rasterize_backward(st, ig)
        tsa[f"target{v_i}"] = target
        tot = {k: v.copy() for k, v in g.arrays().items()} if tot is None else {k: tot[k] + v for k, v in g.arrays().items()}
    mean = vs.raster.GradientSet.zeros(len(rl))
    for k, v in mean.arrays().items():
        v[...] = tot[k] / len(cams2)
        tsa["grad_" + k] = v.copy()
    opt = vtrain.OptimizerState.for_set(rl)
    vtrain.adam_step(rl, mean, opt, cfg_aux, 1)
    tsa.update({"out_" + k: np.array(v) for k, v in rl.arrays().items()})
    tsa["losses"] = np.array(losses)
    save("train_step_aux", tsa)

    # -- densify / prune (train.py:237-284): clones, splits (seeded rng) and weight pruning
    rng_d = np.random.default_rng(42)
    gd = scenes.random_gaussians(600, seed=41)
    gd.raw_weight[:] = rng_d.normal(-2.0, 2.5, size=600)
    gd.log_scale[:] += rng_d.uniform(-1.0, 2.0, size=(600, 1))
    rgd = to_ref_gs(vs, gd)
    opt = vtrain.OptimizerState.for_set(rgd)
    for d_ in (opt.m, opt.v):
        for k in d_:
            d_[k][...] = rng_d.normal(size=d_[k].shape)
    stats = vtrain.DensifyStats.zeros(600)
    stats.grad_accum[:] = rng_d.uniform(0.0, 1e-3, size=600)
    stats.pos_accum[:] = rng_d.normal(size=(600, 3))
    stats.count[:] = rng_d.integers(0, 5, size=600)
    dd = {"in_" + k: np.array(v) for k, v in rgd.arrays().items()}
    dd.update({"in_m_" + k: v.copy() for k, v in opt.m.items()})
    dd.update({"in_v_" + k: v.copy() for k, v in opt.v.items()})
    dd.update(stats_grad=stats.grad_accum.copy(), stats_pos=stats.pos_accum.copy(), stats_count=stats.count.copy())
    cfg_d = vtrain.TrainConfig(iterations=100)
    out = vtrain.densify_and_prune(rgd, opt, stats, cfg_d, 3.0, np.random.default_rng(7), 1e-3)
    dd.update({"out_" + k: np.array(v) for k, v in out.arrays().items()})
    dd.update({"out_m_" + k: v for k, v in opt.m.items()})
    dd.update({"out_v_" + k: v for k, v in opt.v.items()})
    save("densify", dd)

    # -- VEGS model files written by the reference (model.py:236-282)
    import tempfile

    vm = importlib_model(vs)
    with tempfile.TemporaryDirectory() as td:
        small_gs = to_ref_gs(vs, scenes.random_gaussians(300, seed=51))
        vm.save_model(small_gs, f"{td}/m.vegs")
        vq = vm.vq_compress(small_gs, k=16, iters=4, seed=0)
        vm.save_vq_model(vq, f"{td}/q.vegs")
        vqd = vm.load_model(f"{td}/q.vegs")  # decompressed from the file (f32 payload)
        mio = {"plain_bytes": np.frombuffer(open(f"{td}/m.vegs", "rb").read(), dtype=np.uint8),
               "vq_bytes": np.frombuffer(open(f"{td}/q.vegs", "rb").read(), dtype=np.uint8)}
        mio.update({"in_" + k: np.array(v) for k, v in small_gs.arrays().items()})
        mio.update({"plain_" + k: np.array(v) for k, v in vm.load_model(f"{td}/m.vegs").arrays().items()})
        mio.update({"vq_" + k: np.array(v) for k, v in vqd.arrays().items()})
    save("model_io", mio)

    for k, v in saved.items():
        print(f"{k:20s} {v / 1e3:9.1f} kB")


if __name__ == "__main__":
    main()
