"""Parity at the benchmark's own scale, pinned to the REFERENCE (not only the oracle), and
the multi-stream paths the benchmark times.

* ``scale_c2_f32`` (tests/golden/make_golden_scale.py): one config-2 view (1M Gaussians,
  1024 x 1024, float32 blend) rendered and back-propagated by vegsplat itself.  Integer
  outputs and the float32 T plane are compared through SHA-256 digests (bit-exact), the
  image and gradients through sampled pixels / rows, inf-norms and sums.
* ``scale_c3_f32``: a config-3-shaped frame (1920 x 1080, 500k blob Gaussians, the sweep's
  first TF) through the RenderPipeline the sweep measures.
* ``densify_stats``: the reference's DensifyStats.add over a 2-view step, against the
  statistics the trainer fuses into its backward (train.py:210-214).
* Trainer / RenderPipeline stream lanes (1..4) against single-stream results.

Bars as in test_gpu_parity.py: integers bit-exact, images |d| <= 1e-4 max(|ref|, 1e-3),
gradients ||d||_inf <= 1e-4 ||ref||_inf per class.
"""

import hashlib

import numpy as np
import pytest

import goldens as G

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

from oracle import vegs_oracle as O  # noqa: E402
from paper_2504_13339_b200 import raster as R  # noqa: E402
from paper_2504_13339_b200 import scenes  # noqa: E402
from paper_2504_13339_b200.constants import DEFAULT_SETTINGS as S  # noqa: E402
from paper_2504_13339_b200.device import DeviceTF, Rasterizer, RenderPipeline  # noqa: E402
from paper_2504_13339_b200.model import PARAM_CLASSES  # noqa: E402
from paper_2504_13339_b200.train import TrainConfig, Trainer, View  # noqa: E402

IMG_REL = 1e-4
GRAD_REL = 1e-4


def digest(a, dtype) -> np.ndarray:
    b = np.ascontiguousarray(np.asarray(a).astype(np.dtype(dtype).newbyteorder("<"), copy=False)).tobytes()
    return np.frombuffer(hashlib.sha256(b).digest(), dtype=np.uint8)


def img_close(a, b, rel=IMG_REL):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return bool(np.all(np.abs(a - b) <= rel * np.maximum(np.abs(b), 1e-3)))


def _check_forward_scale(d, img, st):
    b = st.blend
    pix = d["pix"]
    assert len(st.kept) == int(d["n_kept"]) and len(b.order) == int(d["n_inst"])
    # diagnostics first (sampled), then the full-array digests
    assert np.array_equal(b.out_last.reshape(-1)[pix], d["pix_last"])
    assert np.array_equal(b.n_contrib.reshape(-1)[pix], d["pix_ncon"])
    assert np.array_equal(b.out_t.reshape(-1)[pix], d["pix_t"])
    assert np.array_equal(b.tile_start, d["tile_start"]) and np.array_equal(b.tile_end, d["tile_end"])
    assert np.array_equal(digest(st.kept, np.int64), d["kept_sha"])
    assert np.array_equal(digest(st.proj.rect, np.int32), d["rect_sha"])
    assert np.array_equal(digest(b.order, np.int64), d["order_sha"])
    assert np.array_equal(digest(b.out_last, np.int64), d["out_last_sha"])
    assert np.array_equal(digest(b.n_contrib, np.int32), d["n_contrib_sha"])
    assert np.array_equal(digest(b.out_t, np.float32), d["out_t_sha"])
    assert img_close(img.rgb.reshape(-1, 3)[pix], d["pix_rgb"])
    assert img_close(img.alpha.reshape(-1)[pix], d["pix_alpha"], rel=1e-3)
    assert abs(float(img.rgb.astype(np.float64).sum()) - float(d["rgb_sum"])) <= 1e-5 * abs(float(d["rgb_sum"]))


@pytest.fixture(scope="module")
def c2_ref():
    d = G.load("scale_c2_f32")
    gs, _, tf, cams = scenes.config_scene("c2")
    cam = G.cam_of(d["cam"])
    assert cam == cams[0]
    img, st = R.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, False, np.float32)
    return d, gs, cam, img, st


@pytest.mark.slow
def test_c2_view_bit_exact_vs_reference(c2_ref):
    """One benchmark view against vegsplat: kept set, rects, instance order, tile ranges,
    last contributor, contributor count and T bit-exact; image within the bar."""
    d, gs, cam, img, st = c2_ref
    assert len(st.blend.order) > 10_000_000
    _check_forward_scale(d, img, st)


@pytest.mark.slow
def test_c2_view_gradients_vs_reference(c2_ref):
    d, gs, cam, img, st = c2_ref
    h, w = cam.height, cam.width
    prng = np.random.default_rng(6)
    probe = dict(rgb=prng.uniform(-1, 1, size=(h, w, 3)), alpha=prng.uniform(-1, 1, size=(h, w)))
    g = R.rasterize_backward(st, R.ImageGradients(**probe))
    rows = d["grad_rows"]
    n = len(gs)
    for k in PARAM_CLASSES:
        ref_inf = float(d[f"grad_{k}_inf"])
        mine = getattr(g, k).reshape(n, -1)
        assert abs(float(np.abs(mine).max()) - ref_inf) <= GRAD_REL * ref_inf, k
        assert np.abs(mine[rows] - d[f"grad_{k}_rows"]).max() <= GRAD_REL * ref_inf, k
        # whole-array aggregates: the sum of magnitudes pins every row, not just the sample
        ref_abs = float(d[f"grad_{k}_abssum"])
        assert abs(float(np.abs(mine).sum()) - ref_abs) <= GRAD_REL * ref_abs, k
        assert abs(float(mine.sum()) - float(d[f"grad_{k}_sum"])) <= GRAD_REL * ref_abs, k
    assert np.array_equal(digest(g.visible, np.uint8), d["visible_sha"])
    vsn_inf = float(d["vsn_inf"])
    assert np.abs(g.viewspace_norm[rows] - d["vsn_rows"]).max() <= GRAD_REL * vsn_inf


@pytest.mark.slow
def test_c3_frame_through_render_pipeline_vs_reference():
    """A config-3-shaped frame (1920 x 1080, 500k blob Gaussians, the sweep's first TF)
    rendered by the RenderPipeline the sweep times, against vegsplat's frame: T bit-exact
    (digest), image within the bar; the frame's integer outputs through the API path."""
    d = G.load("scale_c3_f32")
    gs = scenes.blob_gaussians(500_000, seed=1)
    cam = G.cam_of(d["cam"])
    tf = scenes.random_tf(1000)
    img, st = R.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, False, np.float32)
    _check_forward_scale(d, img, st)
    params = torch.from_numpy(gs.pack()).cuda()
    dtf = DeviceTF(tf)
    other = DeviceTF(scenes.random_tf(1001))
    got = {}

    def keep(i, fr):
        got[i] = (fr.out_img.view(-1, 3).clone(), fr.out_t.clone(), fr.out_last.clone())

    def keep_ids(i, fr):  # culled lists: the Gaussian behind each last-contributor position
        last = fr.out_last.long()
        gid = torch.where(last >= 0, fr.sorted_gauss[last.clamp(min=0)].long(), torch.full_like(last, -1))
        got[i] = (fr.out_img.view(-1, 3).clone(), fr.out_t.clone(), gid)

    pix = d["pix"]
    last_gid = None
    for cull in (False, True):  # the reference's tile lists, then the culled ones the sweep uses
        for fast in (False, True):  # the float64 chain (default) and the fast-T forward
            got.clear()
            pipe = RenderPipeline(lanes=3, fast_t=fast, cull=cull)
            pipe.render(params, len(gs), [(cam, other), (cam, dtf), (cam, other), (cam, dtf)],
                        on_frame=keep_ids if cull else keep)
            torch.cuda.synchronize()
            for i in (1, 3):
                rgb, t, last = (x.cpu().numpy() for x in got[i])
                if cull:  # the same last contributors, at other list positions
                    assert np.array_equal(last, last_gid), (fast, i)
                else:
                    assert np.array_equal(digest(last.astype(np.int64), np.int64), d["out_last_sha"]), (fast, i)
                assert img_close(t[pix], d["pix_t"]) and img_close(rgb[pix], d["pix_rgb"]), (cull, fast, i)
                if not fast:
                    assert np.array_equal(digest(t, np.float32), d["out_t_sha"]), (cull, i)
        if not cull:
            rz = Rasterizer(pooled=False)
            fr = rz.forward(params, len(gs), dtf, cam)
            lf = fr.out_last.long()
            last_gid = torch.where(lf >= 0, fr.sorted_gauss[lf.clamp(min=0)].long(), torch.full_like(lf, -1))
            last_gid = last_gid.cpu().numpy()


@pytest.mark.parametrize("lanes", [1, 2, 3, 4])
def test_render_pipeline_frames_equal_single_stream(lanes):
    """RenderPipeline (the render / sweep benchmark path) gives, per (camera, TF) item and
    for any lane count, bitwise the frame of a single-stream Rasterizer.forward; items of
    different sizes exercise the pooled-buffer reuse across lanes."""
    gs = scenes.blob_gaussians(60_000, seed=1)
    params = torch.from_numpy(gs.pack()).cuda()
    cams = scenes.orbit_cameras(3, 5, 320, 200) + scenes.orbit_cameras(2, 6, 96, 160)
    tfs = [DeviceTF(scenes.random_tf(1000 + k)) for k in range(3)]
    items = [(cams[i % len(cams)], tfs[i % len(tfs)]) for i in range(7)]
    ref = []
    rz = Rasterizer(pooled=False, cull=True)  # the pipeline's forward (culled binning), single stream
    for cam, tf in items:
        fr = rz.forward(params, len(gs), tf, cam)
        ref.append((fr.out_img.clone(), fr.out_t.clone(), fr.out_last.clone()))
    got = {}

    def keep(i, fr):
        got[i] = (fr.out_img.clone(), fr.out_t.clone(), fr.out_last.clone())

    pipe = RenderPipeline(lanes=lanes)
    for _ in range(2):  # the second pass reuses every lane's grown pools
        got.clear()
        total = pipe.render(params, len(gs), items, on_frame=keep)
        torch.cuda.synchronize()
        assert total > 0
        for i, (img, t, last) in enumerate(ref):
            gi, gt, gl = got[i]
            assert torch.equal(gi, img) and torch.equal(gt, t) and torch.equal(gl, last), (lanes, i)


def test_render_pipeline_shared_projection_identical_frames():
    """A TF sweep through RenderPipeline projects each camera once (vegs_project) and only
    shades per TF (vegs_preprocess_forward_projected): frames bitwise those of full
    preprocesses, item by item."""
    gs = scenes.blob_gaussians(120_000, seed=5)
    params = torch.from_numpy(gs.pack()).cuda()
    cams = scenes.orbit_cameras(2, 5, 400, 260)
    tfs = [DeviceTF(scenes.random_tf(2000 + k)) for k in range(3)]
    items = [(c, tf) for c in cams for tf in tfs]
    got = {}
    for shared in (False, True):
        frames = {}

        def keep(i, fr):
            frames[i] = (fr.out_img.clone(), fr.out_t.clone(), fr.out_last.clone(), fr.tile_end.clone())

        pipe = RenderPipeline(lanes=3, project_once=shared)
        pipe.render(params, len(gs), items, on_frame=keep)
        torch.cuda.synchronize()
        got[shared] = frames
        assert pipe.launches == (len(cams) if shared else 0)
    for i in range(len(items)):
        for a, b in zip(got[False][i], got[True][i]):
            assert torch.equal(a, b), i


def _last_gauss(fr):
    last = fr.out_last.long()
    return torch.where(last >= 0, fr.sorted_gauss[last.clamp(min=0)].long(), torch.full_like(last, -1))


@pytest.mark.parametrize("n_ch", [3, 11])
def test_culled_binning_gives_identical_frames_and_gradients(n_ch):
    """Binning on the tight ellipse boxes (the training / render pipelines) drops about a
    quarter of the tile instances -- the ones that cannot blend in their tile -- and leaves
    everything else bitwise unchanged: image, T, contributor counts, the last contributor
    (as a Gaussian id: positions index the shorter lists), and the whole backward
    (gradients, view-space norms, visibility, densify statistics)."""
    if n_ch == 3:
        gs, _, tf_h, cams = scenes.config_scene("c2")  # full config 2: 1M Gaussians at 1024^2
        cam = cams[0]
    else:
        gs = scenes.random_gaussians(20_000, seed=4)
        tf_h = scenes.random_tf(2, 4)
        cam = scenes.orbit_cameras(1, 3, 200, 150)[0]
    dtf = DeviceTF(tf_h)
    params = torch.from_numpy(gs.pack()).cuda()
    out = {}
    for cull in (False, True):
        rz = Rasterizer(n_channels=n_ch, pooled=False, cull=cull)
        fr = rz.forward(params, len(gs), dtf, cam)
        g = torch.Generator(device="cuda").manual_seed(7)
        d_img = torch.rand(fr.out_img.shape, device="cuda", generator=g) - 0.5
        d_alpha = torch.rand(fr.out_t.shape, device="cuda", generator=g) - 0.5
        vs = torch.zeros(len(gs), dtype=torch.float64, device="cuda")
        vis = torch.zeros(len(gs), dtype=torch.uint8, device="cuda")
        dst = torch.zeros(5 * len(gs), dtype=torch.float64, device="cuda")
        grads = rz.backward(fr, d_img, d_alpha, viewspace_norm=vs, visible=vis, densify_stats=dst)
        n_listed = int((fr.tile_end - fr.tile_start).sum())
        out[cull] = (fr.out_img, fr.out_t, fr.n_contrib, _last_gauss(fr), grads, vs, vis, dst, n_listed, fr.n_inst)
    full, cut = out[False], out[True]
    for k in range(8):
        assert torch.equal(full[k], cut[k]), k
    assert full[8] == full[9] and cut[9] == full[9]  # the reference lists hold every instance
    assert cut[8] < full[8] and (n_ch == 11 or cut[8] < 0.85 * full[8])


def test_culled_trainer_steps_equal_unculled():
    """Trainer steps (device counts, CUDA graphs) with culled binning are bitwise the
    reference-list steps."""
    learned, dtf, cams, targets = _train_scene(4)
    views = [View(c, dtf, t) for c, t in zip(cams, targets)]
    res = []
    for cull in (False, True):
        tr = Trainer(learned, TrainConfig(iterations=100), graphs=True, cull=cull)
        losses = [float(tr.step(views, iteration=it).item()) for it in (1, 2, 3)]
        res.append((losses, tr.params.clone()))
    assert res[0][0] == res[1][0] and torch.equal(res[0][1], res[1][1])


def _train_scene(n_views, w=64, h=64):
    learned = scenes.random_gaussians(2000, seed=0)
    truth = scenes.random_gaussians(2000, seed=1)
    dtf = DeviceTF(scenes.random_tf(2, 4))
    cams = scenes.orbit_cameras(n_views, 3, w, h)
    rz = Rasterizer(pooled=False)
    gt = torch.from_numpy(truth.pack()).cuda()
    targets = [rz.forward(gt, len(truth), dtf, c).out_img.view(c.height, c.width, 3).clone() for c in cams]
    return learned, dtf, cams, targets


def test_trainer_gradient_buffer_matches_reference_before_adam():
    """The step's gradient buffer (mean of the per-view gradients, before Adam) against the
    reference's per-view rasterize_backward of its L1+SSIM gradient, at the 1e-4 bar."""
    d = G.load("train_step")
    learned = scenes.random_gaussians(2000, seed=0)
    dtf = DeviceTF(scenes.random_tf(2, 4))
    cams = scenes.orbit_cameras(2, 3, 64, 64)
    for lanes in (1, 4):
        tr = Trainer(learned, TrainConfig(iterations=100), lanes=lanes)
        views = [View(c, dtf, torch.from_numpy(d[f"target{i}"]).cuda()) for i, c in enumerate(cams)]
        tr.step(views, iteration=1)
        g = tr.grads.cpu().numpy()
        from paper_2504_13339_b200.model import GaussianSet

        gg = GaussianSet.unpack(g, len(learned))
        for k in PARAM_CLASSES:
            assert G.norm_rel(getattr(gg, k), d["grad_" + k]) <= GRAD_REL, (lanes, k)


def test_trainer_densify_stats_match_reference():
    """DensifyStats.add (train.py:210-214) over a 2-view step, fused into the device
    backward, against the reference's statistics on the same views."""
    d = G.load("densify_stats")
    learned = scenes.random_gaussians(2000, seed=0)
    dtf = DeviceTF(scenes.random_tf(2, 4))
    cams = scenes.orbit_cameras(2, 3, 64, 64)
    for lanes in (1, 2, 4):
        tr = Trainer(learned, TrainConfig(iterations=100), lanes=lanes)
        tr.track_densify()
        views = [View(c, dtf, torch.from_numpy(d[f"target{i}"]).cuda()) for i, c in enumerate(cams)]
        tr.step(views, iteration=1)
        st = tr.gather_densify_stats().view(-1, 5).cpu().numpy()
        assert np.array_equal(st[:, 4], d["count"]), lanes
        assert G.norm_rel(st[:, 0], d["grad_accum"]) <= GRAD_REL, lanes
        assert G.norm_rel(st[:, 1:4], d["pos_accum"]) <= GRAD_REL, lanes


def test_trainer_lane_counts_agree():
    """Trainer.step with 1, 2, 3 or 4 stream lanes: losses bitwise equal (per-view sums),
    gradient buffers equal up to float64 summation order, and bitwise equal where the
    per-lane partial sums coincide (2 views on >= 2 lanes vs 1 lane)."""
    learned, dtf, cams, targets = _train_scene(5)
    res = {}
    for lanes in (1, 2, 3, 4):
        tr = Trainer(learned, TrainConfig(iterations=100), lanes=lanes)
        views = [View(c, dtf, t) for c, t in zip(cams, targets)]
        losses = [float(tr.step(views, iteration=it).item()) for it in (1, 2)]
        res[lanes] = (losses, tr.grads.clone(), tr.params.clone())
    l1, g1, p1 = res[1]
    for lanes in (2, 3, 4):
        ll, gl, pl = res[lanes]
        assert abs(ll[0] - l1[0]) <= 1e-12 * abs(l1[0])
        assert float((gl - g1).abs().max()) <= 1e-12 * float(g1.abs().max()), lanes
        assert float((pl - p1).abs().max()) <= 1e-9, lanes
    two = {}
    for lanes in (1, 2, 4):
        tr = Trainer(learned, TrainConfig(iterations=100), lanes=lanes)
        views = [View(c, dtf, t) for c, t in zip(cams[:2], targets[:2])]
        loss = float(tr.step(views, iteration=1).item())
        two[lanes] = (loss, tr.params.clone())
    for lanes in (2, 4):
        assert two[lanes][0] == two[1][0] and torch.equal(two[lanes][1], two[1][1]), lanes


def test_trainer_rejects_malformed_targets():
    learned, dtf, cams, targets = _train_scene(1)
    tr = Trainer(learned, TrainConfig(iterations=100))
    for bad in (targets[0].double(), targets[0].permute(1, 0, 2), torch.zeros(64, 64, 4, device="cuda")):
        with pytest.raises(ValueError):
            tr.step([View(cams[0], dtf, bad)])


def test_trainer_mixed_resolution_loss_uses_per_view_normalisers():
    """Views of different sizes in one step: the returned loss is the mean of each view's
    own normalised loss (each view alone gives its own value)."""
    learned = scenes.random_gaussians(2000, seed=0)
    truth = scenes.random_gaussians(2000, seed=1)
    dtf = DeviceTF(scenes.random_tf(2, 4))
    cams = [scenes.orbit_cameras(1, 3, 64, 64)[0], scenes.orbit_cameras(1, 4, 96, 48)[0]]
    rz = Rasterizer(pooled=False)
    gt = torch.from_numpy(truth.pack()).cuda()
    views = [View(c, dtf, rz.forward(gt, len(truth), dtf, c).out_img.view(c.height, c.width, 3).clone())
             for c in cams]
    alone = [float(Trainer(learned, TrainConfig(iterations=100)).step([v], iteration=1).item()) for v in views]
    both = float(Trainer(learned, TrainConfig(iterations=100)).step(views, iteration=1).item())
    assert abs(both - 0.5 * (alone[0] + alone[1])) <= 1e-12 * abs(both)


def test_adam_lane_sum_equals_eager_adds():
    """vegs_adam_step_sum (lane partial sums folded into Adam) is bitwise the eager
    ((g0 + g1) + g2) + g3 followed by vegs_adam_step."""
    from paper_2504_13339_b200.device import adam_step_device

    n = 5003
    gen = torch.Generator(device="cuda").manual_seed(3)
    p = torch.randn(19 * n, dtype=torch.float64, device="cuda", generator=gen)
    gs = [torch.randn(19 * n, dtype=torch.float64, device="cuda", generator=gen) for _ in range(4)]
    m = torch.rand(19 * n, dtype=torch.float64, device="cuda", generator=gen)
    v = torch.rand(19 * n, dtype=torch.float64, device="cuda", generator=gen)
    lrs = torch.linspace(1e-4, 1e-2, 10, dtype=torch.float64, device="cuda")
    bad = torch.zeros(10, dtype=torch.int32, device="cuda")
    for k in (1, 2, 3, 4):
        a = [x.clone() for x in (p, m, v)]
        b = [x.clone() for x in (p, m, v)]
        g_eager = gs[0].clone()
        for x in gs[1:k]:
            g_eager.add_(x)
        adam_step_device(a[0], g_eager, a[1], a[2], n, lrs, 1.0, 3, bad)
        g_fused = gs[0].clone()
        adam_step_device(b[0], g_fused, b[1], b[2], n, lrs, 1.0, 3, bad, [x for x in gs[1:k]])
        assert torch.equal(g_fused, g_eager), k
        for x, y in zip(a, b):
            assert torch.equal(x, y), k
        # sum only
        g_sum = gs[0].clone()
        adam_step_device(None, g_sum, None, None, n, None, 1.0, 1, None, [x for x in gs[1:k]])
        assert torch.equal(g_sum, g_eager), k
    assert not bad.any()


# -- the fast-T forward (vegs_composite_forward_fast): float32 chain, exact decisions ------

FAST_CASES = [("c0_f32", False), ("dense_f32", False), ("c0_aux_f32", True)]


@pytest.mark.parametrize("name,aux", FAST_CASES, ids=[c[0] for c in FAST_CASES])
def test_fast_t_forward_vs_reference_goldens(name, aux):
    """The training / render path's forward against the reference fixtures: last
    contributor and contributor count bit-exact, T and the planes within the image bar."""
    d = G.load(name)
    params = torch.from_numpy(G.gs_of(d).pack()).cuda()
    cam = G.cam_of(d["cam"])
    rz = Rasterizer(n_channels=11 if aux else 3, pooled=False, fast_t=True)
    fr = rz.forward(params, len(d["gs_position"]), DeviceTF(G.tf_of(d)), cam, tuple(d["bg"]))
    h, w = cam.height, cam.width
    assert np.array_equal(fr.out_last.cpu().numpy().reshape(h, w), d["out_last"])
    assert np.array_equal(fr.n_contrib.cpu().numpy().reshape(h, w), d["n_contrib"])
    assert img_close(fr.out_t.cpu().numpy().reshape(h, w), d["out_t"])
    assert img_close(fr.out_img.view(h, w, -1)[:, :, :3].cpu().numpy(), d["rgb"])


def test_fast_t_forward_equals_exact_forward_decisions():
    """Fast vs float64-chain forward on a 1080p blob scene: every integer decision
    equal, T within the bound the kernel tracks, few pixels deferred to the fix-up."""
    gs = scenes.blob_gaussians(200_000, seed=1)
    params = torch.from_numpy(gs.pack()).cuda()
    cam = scenes.orbit_cameras(1, 5, 1920, 1080)[0]
    tf = DeviceTF(scenes.random_tf(1000))
    ex = Rasterizer(pooled=False).forward(params, len(gs), tf, cam)
    fa = Rasterizer(pooled=False, fast_t=True).forward(params, len(gs), tf, cam)
    assert torch.equal(fa.out_last, ex.out_last)
    assert torch.equal(fa.n_contrib, ex.n_contrib)
    rel = ((fa.out_t.double() - ex.out_t.double()).abs() / ex.out_t.double().clamp(min=1e-3)).max().item()
    assert rel <= 1e-4, rel
    assert img_close(fa.out_img.cpu().numpy(), ex.out_img.cpu().numpy())
    assert fa.n_deferred < 0.03 * cam.width * cam.height


def test_fast_t_fixup_is_exact_when_every_pixel_is_deferred(monkeypatch):
    """Forcing every terminating test to be undecidable (VEGS_FAST_T_DEFER_ALL) sends those
    pixels through the float64 fix-up: the frame then equals the float64-chain forward
    bit for bit (T included) wherever the fix-up ran."""
    monkeypatch.setenv("VEGS_FAST_T_DEFER_ALL", "1")
    d = G.load("dense_f32")
    params = torch.from_numpy(G.gs_of(d).pack()).cuda()
    cam = G.cam_of(d["cam"])
    tf = DeviceTF(G.tf_of(d))
    fa = Rasterizer(pooled=False, fast_t=True).forward(params, len(d["gs_position"]), tf, cam, tuple(d["bg"]))
    assert fa.n_deferred > 0
    h, w = cam.height, cam.width
    pix = fa.defer[1:1 + fa.n_deferred].cpu().numpy()
    assert np.array_equal(fa.out_last.cpu().numpy(), d["out_last"].reshape(-1))
    assert np.array_equal(fa.n_contrib.cpu().numpy(), d["n_contrib"].reshape(-1))
    assert np.array_equal(fa.out_t.cpu().numpy()[pix], d["out_t"].reshape(-1)[pix])


@pytest.mark.slow
def test_c2_fast_t_forward_vs_reference(c2_ref):
    """The benchmark's own forward (fast T) on the pinned c2 view: last contributor and
    contributor count digests equal the reference's; sampled T / rgb within the bar."""
    d, gs, cam, img, st = c2_ref
    params = torch.from_numpy(gs.pack()).cuda()
    fr = Rasterizer(pooled=False, fast_t=True).forward(params, len(gs), DeviceTF(scenes.config_scene("c2")[2]), cam)
    last = fr.out_last.cpu().numpy().astype(np.int64)
    ncon = fr.n_contrib.cpu().numpy()
    pix = d["pix"]
    assert np.array_equal(last[pix], d["pix_last"]) and np.array_equal(ncon[pix], d["pix_ncon"])
    assert np.array_equal(digest(last, np.int64), d["out_last_sha"])
    assert np.array_equal(digest(ncon, np.int32), d["n_contrib_sha"])
    assert img_close(fr.out_t.cpu().numpy()[pix], d["pix_t"])
    assert img_close(fr.out_img.view(-1, 3).cpu().numpy()[pix], d["pix_rgb"])
    assert fr.n_deferred < 0.03 * cam.width * cam.height


# -- BASELINE config 4's densify rule (max TF opacity prune, count cap) vs the oracle --------

@pytest.mark.parametrize("cap", [None, "tight"])
def test_densify_config4_rule_matches_oracle(cap):
    from paper_2504_13339_b200.model import GaussianSet
    from paper_2504_13339_b200.train import densify_device, tf_max_opacity

    d = G.load("densify")
    gs = GaussianSet(**{k: d["in_" + k].copy() for k in PARAM_CLASSES})
    n = len(gs)
    tfs = [scenes.range_tf(500 + k, k / 4, (k + 1) / 4) for k in range(4)]
    params = torch.from_numpy(gs.pack()).cuda()

    def flat(prefix):
        return torch.from_numpy(np.concatenate([d[prefix + k].ravel() for k in PARAM_CLASSES])).cuda()

    m, v = flat("in_m_"), flat("in_v_")
    stats = torch.from_numpy(np.concatenate([d["stats_grad"][:, None], d["stats_pos"], d["stats_count"][:, None]],
                                            axis=1).copy()).cuda()
    mo = tf_max_opacity(params, n, [DeviceTF(t) for t in tfs])
    mo_ref = O.tf_max_opacity(d["in_raw_value"], [(t.opacity.ts, t.opacity.values) for t in tfs])
    mo_h = mo.cpu().numpy()
    # libm ulps of sigmoid's exp may differ; the prune decisions must not
    assert np.abs(mo_h - mo_ref).max() <= 1e-14 and np.array_equal(mo_h >= 0.005, mo_ref >= 0.005)
    cfg = TrainConfig(iterations=100)
    ocfg = dict(densify_grad_threshold=cfg.densify_grad_threshold, percent_dense=cfg.percent_dense,
                prune_weight_threshold=cfg.prune_weight_threshold, no_weights=False)
    p_in = {k: d["in_" + k].copy() for k in O.CLASSES}
    m_in = {k: d["in_m_" + k].copy() for k in O.CLASSES}
    v_in = {k: d["in_v_" + k].copy() for k in O.CLASSES}
    args = (d["stats_grad"], d["stats_pos"], d["stats_count"], ocfg, 3.0)
    cap_n = None
    if cap:
        free, _, _ = O.densify_and_prune(p_in, m_in, v_in, *args, np.random.default_rng(7), 1e-3, mo_ref)
        cap_n = len(free["raw_weight"]) - 1
    op, om, ov = O.densify_and_prune(p_in, m_in, v_in, *args, np.random.default_rng(7), 1e-3, mo_ref, cap_n)
    p, mm, vv, n_out = densify_device(params, m, v, n, stats, cfg, 3.0, np.random.default_rng(7), 1e-3, mo, cap_n)
    assert n_out == len(op["raw_weight"])
    if cap:
        assert n_out <= cap_n
    gp = GaussianSet.unpack(p.cpu().numpy(), n_out)
    gm = GaussianSet.unpack(mm.cpu().numpy(), n_out)
    gv = GaussianSet.unpack(vv.cpu().numpy(), n_out)
    for k in PARAM_CLASSES:
        ref = op[k]
        assert np.abs(getattr(gp, k) - ref).max() <= 1e-12 * max(np.abs(ref).max(), 1.0), k
        assert np.array_equal(getattr(gm, k), om[k]) and np.array_equal(getattr(gv, k), ov[k]), k


@pytest.mark.parametrize("n_ch", [3, 11])
def test_float32_backward_chain_close_to_float64_chain(monkeypatch, n_ch):
    """The float32-blend backward's adjoint chain runs in float32 (decisions in float64);
    against the float64 chain (VEGS_BWD_CHAIN_F64=1) every class agrees far inside the
    1e-4 gradient bar, and the visibility / view-space norms feeding densification match."""
    gs = scenes.blob_gaussians(150_000, seed=1)
    params = torch.from_numpy(gs.pack()).cuda()
    cam = scenes.orbit_cameras(1, 4, 640, 480)[0]
    tf = DeviceTF(scenes.random_tf(1001))
    rz = Rasterizer(n_channels=n_ch)
    fr = rz.forward(params, len(gs), tf, cam)
    d_img = torch.rand(480, 640, n_ch, device="cuda", generator=torch.Generator("cuda").manual_seed(2)) - 0.5
    out = []
    for chain64 in ("0", "1"):
        monkeypatch.setenv("VEGS_BWD_CHAIN_F64", chain64)
        vs = torch.empty(len(gs), dtype=torch.float64, device="cuda")
        vis = torch.empty(len(gs), dtype=torch.uint8, device="cuda")
        g = rz.backward(fr, d_img, viewspace_norm=vs, visible=vis).clone()
        out.append((g.cpu().numpy(), vs.cpu().numpy(), vis.cpu().numpy()))
    from paper_2504_13339_b200.model import GaussianSet

    a, b = GaussianSet.unpack(out[0][0], len(gs)), GaussianSet.unpack(out[1][0], len(gs))
    for k in PARAM_CLASSES:
        assert G.norm_rel(getattr(a, k), getattr(b, k)) <= 1e-5, (k, G.norm_rel(getattr(a, k), getattr(b, k)))
    assert np.array_equal(out[0][2], out[1][2])
    assert G.norm_rel(out[0][1], out[1][1]) <= 1e-6


@pytest.mark.parametrize("pair", ["0", "1"])
@pytest.mark.parametrize("name", ["c0_f32", "dense_f32"])
def test_paired_forward_bitwise_equals_single_entry_forward(monkeypatch, name, pair):
    """The forward's loop with two list entries per iteration (default) and with one
    (VEGS_FWD_PAIR=0) against the reference fixture: T, last contributor and contributor
    count bit for bit."""
    monkeypatch.setenv("VEGS_FWD_PAIR", pair)
    d = G.load(name)
    params = torch.from_numpy(G.gs_of(d).pack()).cuda()
    cam = G.cam_of(d["cam"])
    fr = Rasterizer(pooled=False).forward(params, len(d["gs_position"]), DeviceTF(G.tf_of(d)), cam, tuple(d["bg"]))
    h, w = cam.height, cam.width
    assert np.array_equal(fr.out_last.cpu().numpy().reshape(h, w), d["out_last"])
    assert np.array_equal(fr.n_contrib.cpu().numpy().reshape(h, w), d["n_contrib"])
    assert np.array_equal(fr.out_t.cpu().numpy().reshape(h, w), d["out_t"])


@pytest.mark.slow
def test_c2_single_entry_forward_vs_reference(monkeypatch, c2_ref):
    monkeypatch.setenv("VEGS_FWD_PAIR", "0")
    d, gs, cam, img, st = c2_ref
    params = torch.from_numpy(gs.pack()).cuda()
    fr = Rasterizer(pooled=False).forward(params, len(gs), DeviceTF(scenes.config_scene("c2")[2]), cam)
    assert np.array_equal(digest(fr.out_last.cpu().numpy().astype(np.int64), np.int64), d["out_last_sha"])
    assert np.array_equal(digest(fr.n_contrib.cpu().numpy(), np.int32), d["n_contrib_sha"])
    assert np.array_equal(digest(fr.out_t.cpu().numpy(), np.float32), d["out_t_sha"])


# -- device-count steps captured as CUDA graphs ---------------------------------------------

def _graph_runs(views_fn, steps, lanes=4, **kw):
    learned = scenes.random_gaussians(2000, seed=0)
    out = {}
    for graphs in (False, True):
        tr = Trainer(learned, TrainConfig(iterations=100), lanes=lanes, graphs=graphs, **kw)
        losses = [float(tr.step(views_fn(s), iteration=s + 1).item()) for s in range(steps)]
        torch.cuda.synchronize()
        out[graphs] = (losses, tr.params.clone(), tr.grads.clone(), tr)
    return out


def test_graph_steps_bitwise_equal_eager_steps():
    """graphs=True (device-side instance counts, capacity-sized buffers, one captured CUDA
    graph per set of views, replayed) gives bitwise the eager host-counted steps: the first
    step overflows the empty capacity, is redone, then the graph is captured and replayed."""
    learned, dtf, cams, targets = _train_scene(5)
    views = [View(c, dtf, t) for c, t in zip(cams, targets)]
    res = _graph_runs(lambda s: views, 4)
    (le, pe, ge, _), (lg, pg, gg, tr) = res[False], res[True]
    assert le == lg
    assert torch.equal(pe, pg) and torch.equal(ge, gg)
    assert len(tr._graphs) == 1 and all(l.rz.inst_cap > 0 for l in tr.lanes)


@pytest.mark.parametrize("flat", ["0", "1"])
def test_graph_steps_both_placements(monkeypatch, flat):
    """Graph-replayed device-count steps through the two-level placement (forced on small
    views with VEGS_PLACE_FLAT=0; 4096+ tiles take it by default) and the single level give
    bitwise the eager steps of the other placement: the placement changes no list."""
    learned, dtf, cams, targets = _train_scene(4, 144, 112)
    views = [View(c, dtf, t) for c, t in zip(cams, targets)]
    monkeypatch.setenv("VEGS_PLACE_FLAT", flat)
    tr = Trainer(learned, TrainConfig(iterations=100), graphs=True)
    lg = [float(tr.step(views, iteration=s + 1).item()) for s in range(3)]
    pg = tr.params.clone()
    monkeypatch.setenv("VEGS_PLACE_FLAT", "1" if flat == "0" else "0")
    te = Trainer(learned, TrainConfig(iterations=100), graphs=False)
    le = [float(te.step(views, iteration=s + 1).item()) for s in range(3)]
    assert lg == le and torch.equal(pg, te.params) and len(tr._graphs) == 1


def test_graph_steps_with_alternating_views_and_host_targets():
    """Two alternating sets of views (two cached graphs), pinned host targets uploaded inside
    the graph, and DensifyStats tracking: bitwise the eager run."""
    learned, dtf, cams, targets = _train_scene(4)
    dtf2 = DeviceTF(scenes.random_tf(5, 3))
    host = [t.cpu().pin_memory() for t in targets]
    sets = [[View(c, dtf, t) for c, t in zip(cams, host)], [View(c, dtf2, t) for c, t in zip(cams[:3], host[:3])]]
    out = {}
    for graphs in (False, True):
        tr = Trainer(learned, TrainConfig(iterations=100), graphs=graphs)
        tr.track_densify()
        losses = [float(tr.step(sets[s % 2], iteration=s + 1, total_views=4).item()) for s in range(6)]
        st = tr.gather_densify_stats().clone()
        out[graphs] = (losses, tr.params.clone(), st)
        if graphs:
            assert len(tr._graphs) == 2
    assert out[False][0] == out[True][0]
    assert torch.equal(out[False][1], out[True][1]) and torch.equal(out[False][2], out[True][2])


def test_graph_step_overflow_regrows_and_redoes():
    """A view with more instances than the captured capacity: the step is emptied on the
    device, Adam skips, the host grows the buffers and redoes it -- same parameters as eager."""
    learned, dtf, cams, targets = _train_scene(3)
    views = [View(c, dtf, t) for c, t in zip(cams, targets)]
    big = scenes.orbit_cameras(1, 9, 160, 128)[0]
    rz = Rasterizer(pooled=False)
    truth = torch.from_numpy(scenes.random_gaussians(2000, seed=1).pack()).cuda()
    tbig = rz.forward(truth, 2000, dtf, big).out_img.view(128, 160, 3).clone()
    views2 = views + [View(big, dtf, tbig)]
    res = _graph_runs(lambda s: views if s < 2 else views2, 4)
    assert res[False][0] == res[True][0]
    assert torch.equal(res[False][1], res[True][1])


@pytest.mark.parametrize("lanes,aux", [(1, False), (2, True), (8, False)])
def test_graph_steps_other_lane_counts_and_aux(lanes, aux):
    """Graph-replayed steps with one lane (no look-ahead), with the 11-plane aux loss, and
    with 8 lanes (config 4's; lane sums beyond four in a sum-only pass): bitwise the eager
    steps."""
    learned, dtf, cams, targets = _train_scene(10 if lanes == 8 else 3)
    views = [View(c, dtf, t) for c, t in zip(cams, targets)]
    res = _graph_runs(lambda s: views, 3, lanes=lanes, with_aux=aux)
    assert res[False][0] == res[True][0]
    assert torch.equal(res[False][1], res[True][1])
    assert res[True][3].graph_stats["replays"] >= 1
