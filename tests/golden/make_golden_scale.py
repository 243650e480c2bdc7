"""Golden vectors at the BENCHMARK's scale, produced by running the REFERENCE (vegsplat).

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden_scale.py [--ref /root/reference/pkg] [--only c2,c3,dstats]

make_golden.py pins the oracle and the CUDA path with full arrays at <= 4,096 Gaussians.
This script pins them where the benchmark runs: one config-2 view (1M Gaussians,
1024 x 1024, float32 blend, the reference's training dtype) and one config-3-shaped frame
(1920 x 1080, 500k blob Gaussians, one of the sweep's random TFs).  Full arrays at that
size would be ~100 MB, so the fixture keeps

* SHA-256 digests of every integer output that must be bit-exact (kept, rect, order,
  tile ranges, last contributor, contributor count) and of the float32 T plane;
* the tile ranges in full (4096 / 8160 entries) and a seeded sample of pixels
  (rgb, alpha, T, last contributor, contributor count) for diagnostics;
* for the gradients of a seeded image-space probe: per class the full-array inf-norm,
  sum and sum of magnitudes, plus every row of a seeded sample of Gaussians and of each
  class's 64 largest-magnitude rows.

The per-pixel contributor count is not a reference output.  It is derived exactly as
make_golden.py does, but with the C replay (oracle/blend.c, the same kernels.py:56-93
float64 promotions) run on the reference's OWN BlendState instance arrays; the replay
must reproduce the reference's out_t and out_last bit for bit before its counts are
stored.

``dstats``: the reference's DensifyStats.add (train.py:210-214) over the two views of
make_golden.py's training-step scene, for the fused statistics in the device backward.
"""

from __future__ import annotations

import argparse
import hashlib
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE))

import make_golden as MG  # noqa: E402

N_PIX_SAMPLE = 32768
N_ROW_SAMPLE = 8192
N_TOP = 64


def digest(a: np.ndarray, dtype) -> np.ndarray:
    """SHA-256 of the little-endian bytes of `a` cast to `dtype`, as a uint8 array."""
    b = np.ascontiguousarray(np.asarray(a).astype(np.dtype(dtype).newbyteorder("<"), copy=False)).tobytes()
    return np.frombuffer(hashlib.sha256(b).digest(), dtype=np.uint8).copy()


def contributor_counts(b, dtype):
    """Replay the reference BlendState through the C oracle kernel (kernels.py:56-93)."""
    import ctypes

    from oracle import vegs_oracle as O

    h, w = b.height, b.width
    n_ch = b.inst_channels.shape[1]
    img = np.zeros((h, w, n_ch), dtype=dtype)
    out_t = np.ones((h, w), dtype=dtype)
    last = np.full((h, w), -1, dtype=np.int64)
    ncon = np.zeros((h, w), dtype=np.int32)
    real = ctypes.c_float if dtype == np.float32 else ctypes.c_double
    fn = getattr(O.lib(), "oracle_blend_forward_f32" if dtype == np.float32 else "oracle_blend_forward_f64")
    arr = {k: np.ascontiguousarray(getattr(b, k)) for k in ("inst_mean2d", "inst_conic", "inst_alpha", "inst_pmin",
                                                           "inst_channels")}
    rect = np.ascontiguousarray(b.inst_rect, dtype=np.int32)
    bg = np.ascontiguousarray(b.bg_vec, dtype=dtype)
    start = np.ascontiguousarray(b.tile_start, dtype=np.int64)
    end = np.ascontiguousarray(b.tile_end, dtype=np.int64)
    fn(O._p(start), O._p(end), ctypes.c_int64(len(start)), ctypes.c_int64(b.tiles_x), ctypes.c_int64(b.tile_size),
       O._p(arr["inst_mean2d"]), O._p(arr["inst_conic"]), O._p(arr["inst_alpha"]), O._p(arr["inst_pmin"]),
       O._p(rect), O._p(arr["inst_channels"]), ctypes.c_int64(n_ch), O._p(bg), ctypes.c_int64(w),
       ctypes.c_int64(h), real(dtype(0.99)), real(dtype(1e-4)), O._p(img), O._p(out_t), O._p(last), O._p(ncon))
    return out_t, last, ncon


def forward_scale_fixture(vs, gs, tf, cam, dtype, probe_seed: int | None, sample_seed: int):
    bg = (1.0, 1.0, 1.0)
    rgs, rtf, rcam = MG.to_ref_gs(vs, gs), MG.to_ref_tf(vs, tf), MG.to_ref_cam(vs, cam)
    t0 = time.perf_counter()
    img, st = vs.raster.render_with_state(rgs, rtf, rcam, bg, vs.raster.DEFAULT_SETTINGS, with_aux=False,
                                          dtype=dtype)
    t_fwd = time.perf_counter() - t0
    b = st.blend
    t_rep, last_rep, count = contributor_counts(b, dtype)
    assert np.array_equal(last_rep, b.out_last), "C replay diverged from the reference (out_last)"
    assert np.array_equal(t_rep, b.out_t), "C replay diverged from the reference (out_t)"
    h, w = cam.height, cam.width
    rng = np.random.default_rng(sample_seed)
    pix = np.sort(rng.choice(h * w, size=min(N_PIX_SAMPLE, h * w), replace=False))
    out = dict(cam=MG.cam_fields(cam), bg=np.asarray(bg), n_gaussians=np.array(len(gs)),
               kept_sha=digest(st.kept, np.int64), n_kept=np.array(len(st.kept)),
               rect_sha=digest(st.proj.rect, np.int32), order_sha=digest(b.order, np.int64),
               n_inst=np.array(len(b.order)), tile_start=b.tile_start.astype(np.int64),
               tile_end=b.tile_end.astype(np.int64), out_last_sha=digest(b.out_last, np.int64),
               n_contrib_sha=digest(count, np.int32), out_t_sha=digest(b.out_t, np.float32),
               pix=pix, pix_rgb=img.rgb.reshape(-1, 3)[pix], pix_alpha=img.alpha.reshape(-1)[pix],
               pix_t=b.out_t.reshape(-1)[pix], pix_last=b.out_last.reshape(-1)[pix],
               pix_ncon=count.reshape(-1)[pix], rgb_sum=np.array(img.rgb.astype(np.float64).sum()),
               ncon_sum=np.array(count.astype(np.int64).sum()), t_ref_forward_s=np.array(t_fwd))
    if probe_seed is None:
        return out
    prng = np.random.default_rng(probe_seed)
    probe = dict(rgb=prng.uniform(-1, 1, size=(h, w, 3)), alpha=prng.uniform(-1, 1, size=(h, w)))
    t0 = time.perf_counter()
    g = vs.raster.rasterize_backward(st, vs.raster.ImageGradients(**probe))
    out["t_ref_backward_s"] = np.array(time.perf_counter() - t0)
    n = len(gs)
    rows = set(rng.choice(n, size=min(N_ROW_SAMPLE, n), replace=False).tolist())
    for k, v in g.arrays().items():
        mag = np.abs(v.reshape(n, -1)).max(axis=1)
        rows.update(np.argsort(mag)[-N_TOP:].tolist())
    rows = np.array(sorted(rows), dtype=np.int64)
    out["grad_rows"] = rows
    for k, v in g.arrays().items():
        out[f"grad_{k}_inf"] = np.array(np.abs(v).max())
        out[f"grad_{k}_sum"] = np.array(v.sum())
        out[f"grad_{k}_abssum"] = np.array(np.abs(v).sum())
        out[f"grad_{k}_rows"] = v.reshape(n, -1)[rows]
    out["visible_sha"] = digest(g.visible, np.uint8)
    out["vsn_rows"] = g.viewspace_norm[rows]
    out["vsn_inf"] = np.array(np.abs(g.viewspace_norm).max())
    return out


def dstats_fixture(vs):
    """Reference training-step scene of make_golden.py (2 views, 2000 Gaussians, 64x64):
    per-view rasterize_backward of the L1+SSIM loss gradient, DensifyStats.add per view."""
    from paper_2504_13339_b200 import scenes

    vtrain = sys.modules["vegsplat.train"]

    class Cfg:
        lambda_ssim = 0.2
        normal_loss_weight = 0.0
        smooth_loss_weight = 0.0

    learned = scenes.random_gaussians(2000, seed=0)
    truth = scenes.random_gaussians(2000, seed=1)
    tf2 = scenes.random_tf(2, 4)
    cams2 = scenes.orbit_cameras(2, 3, 64, 64)
    rl, rt, rtf = MG.to_ref_gs(vs, learned), MG.to_ref_gs(vs, truth), MG.to_ref_tf(vs, tf2)
    stats = vtrain.DensifyStats.zeros(len(rl))
    out = {}
    for v_i, c in enumerate(cams2):
        rc = MG.to_ref_cam(vs, c)
        target = vs.raster.render(rt, rtf, rc, (1.0, 1.0, 1.0), dtype=np.float32).rgb
        img, st = vs.raster.render_with_state(rl, rtf, rc, (1.0, 1.0, 1.0), with_aux=False, dtype=np.float32)
        _, ig, _ = vs.loss.compute_loss(img, target, Cfg())
        g = vs.raster.rasterize_backward(st, ig)
        stats.add(g)
        out[f"target{v_i}"] = target
    out.update(grad_accum=stats.grad_accum, pos_accum=stats.pos_accum, count=stats.count)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    ap.add_argument("--only", default="c2,c3,dstats")
    args = ap.parse_args()
    MG._setup(Path(args.ref))
    import vegsplat as vs  # noqa: E402  (the reference)
    import vegsplat.loss  # noqa: F401
    import vegsplat.raster  # noqa: F401
    import vegsplat.train  # noqa: F401
    from paper_2504_13339_b200 import scenes

    only = set(args.only.split(","))

    def save(name, d):
        path = HERE / f"{name}.npz"
        np.savez_compressed(path, **d)
        print(f"{name:20s} {path.stat().st_size / 1e3:9.1f} kB", flush=True)

    if "c2" in only:  # view 0 of the benchmark's step (bench.py: scenes.config_scene("c2"))
        gs, _, tf, cams = scenes.config_scene("c2")
        save("scale_c2_f32", forward_scale_fixture(vs, gs, tf, cams[0], np.float32, probe_seed=6, sample_seed=60))
    if "c3" in only:  # a config-3 frame at 500k Gaussians: the sweep's first frame and TF
        gs = scenes.blob_gaussians(500_000, seed=1)
        cam = scenes.orbit_cameras(1, 5, 1920, 1080)[0]
        save("scale_c3_f32", forward_scale_fixture(vs, gs, scenes.random_tf(1000), cam, np.float32, probe_seed=None,
                                                   sample_seed=61))
    if "dstats" in only:
        save("densify_stats", dstats_fixture(vs))


if __name__ == "__main__":
    main()
