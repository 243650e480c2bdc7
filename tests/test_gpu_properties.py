"""Property tests of the CUDA rasteriser, after the reference's own (pkg/tests/
test_rasterize.py:98-206): permutation invariance, colour-map independence of alpha,
determinism, zero / inert / occluded gradients, f32 vs f64 agreement, and edge cases
(empty set, everything culled, partial tiles, tiny images)."""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2504_13339_b200 import raster as R  # noqa: E402
from paper_2504_13339_b200 import scenes  # noqa: E402
from paper_2504_13339_b200.camera import Camera  # noqa: E402
from paper_2504_13339_b200.model import GaussianSet, logit  # noqa: E402
from paper_2504_13339_b200.transfer import ColorMap, OpacityMap, TransferFunction  # noqa: E402


def small_scene(seed, n=400, res=48):
    gs = scenes.random_gaussians(n, seed=seed)
    gs.log_scale[:] += 1.0  # splats a few pixels wide at this resolution
    tf = scenes.random_tf(seed + 100, 3)
    cam = scenes.orbit_cameras(1, seed + 200, res, res)[0]
    return gs, tf, cam


def test_permuting_input_order_changes_nothing():
    gs, tf, cam = small_scene(1)
    a = R.render(gs, tf, cam, (0.3, 0.4, 0.5), dtype=np.float32)
    perm = np.random.default_rng(0).permutation(len(gs))
    b = R.render(gs.select(perm), tf, cam, (0.3, 0.4, 0.5), dtype=np.float32)
    assert np.array_equal(a.rgb, b.rgb) and np.array_equal(a.alpha, b.alpha)


def test_colour_map_swap_keeps_alpha_bitwise():
    gs, tf, cam = small_scene(2)
    planes = []
    for seed in range(4):
        rng = np.random.default_rng(seed)
        ts = np.concatenate([[0.0], np.sort(rng.uniform(0, 1, 5)), [1.0]])
        cm = ColorMap(tuple((float(t),) + tuple(rng.uniform(0, 1, 3)) for t in ts))
        planes.append(R.render(gs, TransferFunction(color=cm, opacity=tf.opacity), cam, dtype=np.float32).alpha)
    assert all(np.array_equal(planes[0], p) for p in planes[1:])


def test_render_and_backward_deterministic():
    gs, tf, cam = small_scene(3)
    d = np.random.default_rng(1).uniform(-1, 1, size=(cam.height, cam.width, 3))
    outs = []
    for _ in range(2):
        img, st = R.render_with_state(gs, tf, cam, dtype=np.float32)
        outs.append((img, R.rasterize_backward(st, R.ImageGradients(rgb=d))))
    assert np.array_equal(outs[0][0].rgb, outs[1][0].rgb)
    for k, v in outs[0][1].arrays().items():
        assert np.array_equal(v, getattr(outs[1][1], k)), k


def test_zero_image_gradient_gives_zero_parameter_gradients():
    gs, tf, cam = small_scene(4)
    _, st = R.render_with_state(gs, tf, cam, with_aux=True, dtype=np.float32)
    g = R.rasterize_backward(st, R.ImageGradients(rgb=np.zeros((cam.height, cam.width, 3))))
    for k, v in g.arrays().items():
        assert np.all(v == 0.0), k


def test_subthreshold_splat_is_inert():
    data = R.SplatData(mean2d=np.array([[16.0, 16.0], [10.0, 12.0]]),
                       conic=np.array([[0.5, 0.0, 0.5], [0.3, 0.05, 0.4]]),
                       alpha_base=np.array([0.6, 0.5 / 255.0]), depth=np.array([1.0, 0.5]),
                       rect=np.array([[0, 32, 0, 32], [0, 32, 0, 32]], dtype=np.int32),
                       channels=np.array([[0.2, 0.4, 0.6], [1.0, 1.0, 1.0]]))
    with_low, _ = R.rasterize_forward(data, 32, 32, (0.1, 0.1, 0.1), dtype=np.float32)
    only = R.SplatData(**{k: getattr(data, k)[:1] for k in ("mean2d", "conic", "alpha_base", "depth", "rect",
                                                            "channels")})
    without, _ = R.rasterize_forward(only, 32, 32, (0.1, 0.1, 0.1), dtype=np.float32)
    assert np.array_equal(with_low.rgb, without.rgb)


def test_fully_occluded_splat_gets_zero_gradient():
    n_wall = 10
    pos = [[0.0, 0.0, 0.5 + 0.05 * i] for i in range(n_wall)] + [[0.0, 0.0, -2.0]]
    n = n_wall + 1
    gs = GaussianSet(position=np.array(pos), log_scale=np.full((n, 3), math.log(4.0)),
                     rotation=np.tile([1.0, 0.0, 0.0, 0.0], (n, 1)), raw_value=np.full(n, float(logit(0.5))),
                     raw_weight=np.full(n, float(logit(0.97))), normal=np.tile([0.0, 0.0, 1.0], (n, 1)),
                     raw_ka=np.zeros(n), raw_kd=np.zeros(n), raw_ks=np.zeros(n), raw_beta=np.full(n, math.log(8.0)))
    tf = TransferFunction(color=ColorMap(((0.0, 0.2, 0.3, 0.4), (1.0, 0.9, 0.8, 0.1))),
                          opacity=OpacityMap(((0.0, 0.95), (1.0, 0.95))))
    cam = Camera(position=(0.0, 0.0, 4.0), target=(0.0, 0.0, 0.0), width=32, height=32, fov_y=math.radians(45.0))
    img, st = R.render_with_state(gs, tf, cam, (0.0, 0.0, 0.0), with_aux=True, dtype=np.float32)
    wall = R.render(gs.select(np.arange(n_wall)), tf, cam, (0.0, 0.0, 0.0), with_aux=True, dtype=np.float32)
    assert np.array_equal(img.rgb, wall.rgb)
    g = R.rasterize_backward(st, R.ImageGradients(rgb=np.ones((32, 32, 3))))
    for k, v in g.arrays().items():
        assert np.all(v[n_wall] == 0.0), k
    assert np.abs(g.raw_value[n_wall - 3:n_wall]).max() > 0.0


def test_rgb_only_render_has_no_aux_planes():
    gs, tf, cam = small_scene(5)
    img = R.render(gs, tf, cam, with_aux=False)
    assert img.depth is None and img.normal is None and img.attrs is None


def test_float32_close_to_float64():
    gs, tf, cam = small_scene(6)
    a = R.render(gs, tf, cam, dtype=np.float64)
    b = R.render(gs, tf, cam, dtype=np.float32)
    assert np.abs(a.rgb - b.rgb).max() < 1e-4


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_empty_set_is_background(dtype):
    gs = scenes.random_gaussians(1, seed=0).select(np.arange(0))
    tf = scenes.random_tf(1, 2)
    cam = scenes.orbit_cameras(1, 0, 40, 24)[0]
    img, st = R.render_with_state(gs, tf, cam, (0.25, 0.5, 0.75), dtype=dtype)
    assert np.allclose(img.rgb, [0.25, 0.5, 0.75]) and np.all(img.alpha == 0.0)
    assert len(st.blend.order) == 0 and np.all(st.blend.out_last == -1)
    g = R.rasterize_backward(st, R.ImageGradients(rgb=np.ones((24, 40, 3))))
    assert g.position.shape == (0, 3)


def test_everything_culled():
    gs = scenes.random_gaussians(200, seed=3)
    gs.raw_weight[:] = -20.0  # alpha_base far below 1/255: every splat culled before projection
    tf = scenes.random_tf(3, 2)
    cam = scenes.orbit_cameras(1, 4, 33, 17)[0]
    img, st = R.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), dtype=np.float32)
    assert len(st.kept) == 0 and np.all(img.rgb == 1.0)
    g = R.rasterize_backward(st, R.ImageGradients(rgb=np.ones((17, 33, 3))))
    assert all(np.all(v == 0) for v in g.arrays().values()) and not g.visible.any()


@pytest.mark.parametrize("wh", [(1, 1), (5, 3), (17, 33), (250, 130)])
def test_partial_tiles_match_oracle(wh):
    from oracle import vegs_oracle as O
    from paper_2504_13339_b200.constants import DEFAULT_SETTINGS as S

    gs = scenes.random_gaussians(3000, seed=7)
    tf = scenes.random_tf(7, 4)
    cam = scenes.orbit_cameras(1, 8, wh[0], wh[1])[0]
    img, st = R.render_with_state(gs, tf, cam, (0.5, 0.5, 0.5), S, False, np.float32)
    img_o, st_o = O.render_with_state(gs, tf, cam, (0.5, 0.5, 0.5), S, False, np.float32)
    assert np.array_equal(st.blend.order, st_o["order"])
    assert np.array_equal(st.blend.out_last, st_o["out_last"])
    assert np.array_equal(st.blend.n_contrib, st_o["n_contrib"])
    assert np.abs(img.rgb - img_o["rgb"]).max() < 1e-5


def test_depth_ties_follow_float64_then_index_order():
    """Splats whose depths collide in float32 (but not float64), plus exact float64
    duplicates: the instance order must still be np.lexsort((depth, tile))'s."""
    from oracle import vegs_oracle as O
    from paper_2504_13339_b200.constants import DEFAULT_SETTINGS as S

    gs = scenes.random_gaussians(600, seed=11)
    gs.log_scale[:] += 1.0
    rng = np.random.default_rng(5)
    # camera on the +z axis looking at the origin: depth = 3 - z
    base = rng.uniform(-0.5, 0.5, size=(200, 1))
    z = np.concatenate([base, base + 3e-9, base + 1.5e-8]).ravel()  # same float32 depth, distinct float64
    gs.position[:, 2] = z[rng.permutation(600)]
    gs.position[:50] = gs.position[50:100]  # exact duplicates (equal float64 depth): index order
    tf = scenes.random_tf(11, 4)
    cam = Camera(position=(0.0, 0.0, 3.0), target=(0.0, 0.0, 0.0), up=(0.0, 1.0, 0.0),
                 fov_y=math.radians(50.0), width=64, height=64)
    img, st = R.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, False, np.float32)
    img_o, st_o = O.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, False, np.float32)
    assert np.array_equal(st.blend.order, st_o["order"])
    assert np.array_equal(st.blend.out_last, st_o["out_last"])
    assert np.array_equal(st.blend.n_contrib, st_o["n_contrib"])


@pytest.mark.parametrize("wh", [(512, 512), (1920, 1080)])
def test_counting_placement_equals_radix_binning(wh, monkeypatch):
    """The counting-placement binning and the radix-sort binning produce the same instance
    order, ranges and images (both equal np.lexsort((depth, tile)))."""
    from paper_2504_13339_b200.device import DeviceTF, Rasterizer

    gs = scenes.random_gaussians(100_000, seed=21)
    tf = scenes.random_tf(21, 4)
    cam = scenes.orbit_cameras(1, 22, wh[0], wh[1])[0]
    params = torch.from_numpy(gs.pack()).cuda()
    dtf = DeviceTF(tf)
    out = []
    for radix in (False, True):
        if radix:
            monkeypatch.setenv("VEGS_BIN_RADIX", "1")
        rz = Rasterizer(pooled=False)
        fr = rz.forward(params, len(gs), dtf, cam, want_order=True)
        out.append({k: getattr(fr, k).cpu().clone() for k in
                    ("sorted_gauss", "inst_pid", "order", "tile_start", "tile_end", "out_last", "out_img", "out_t")})
    a, b = out
    assert a["sorted_gauss"].numel() > 1000
    for k in a:
        assert torch.equal(a[k], b[k]), k


def test_rgb_multi_pixel_kernels_match_one_pixel_kernels_and_oracle(monkeypatch):
    """The float32 rgb path's two-pixel forward / four-pixel backward against the one-pixel
    kernels (VEGS_GENERIC_COMPOSITE=1, the reference's loop order per pixel): forward planes
    bitwise equal, gradients equal to float32 rounding (different summation order), both
    equal to the oracle."""
    from oracle import vegs_oracle as O
    from paper_2504_13339_b200.constants import DEFAULT_SETTINGS as S

    gs = scenes.random_gaussians(20_000, seed=31)
    tf = scenes.random_tf(31, 4)
    cam = scenes.orbit_cameras(1, 32, 256, 192)[0]
    d_rgb = np.random.default_rng(33).uniform(-1, 1, size=(192, 256, 3))
    img_o, st_o = O.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, False, np.float32)
    g_o = O.rasterize_backward(st_o, d_rgb)
    out = []
    for generic in (False, True):
        if generic:
            monkeypatch.setenv("VEGS_GENERIC_COMPOSITE", "1")
        img, st = R.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, False, np.float32)
        g = R.rasterize_backward(st, R.ImageGradients(rgb=d_rgb))
        out.append((img, st.blend.out_t, g))
        for k in O.GRAD_CLASSES:
            ref = g_o[k]
            assert np.abs(getattr(g, k) - ref).max() <= 1e-4 * max(np.abs(ref).max(), 1e-300), (generic, k)
    (ia, ta, ga), (ib, tb, gb) = out
    assert np.array_equal(ia.rgb, ib.rgb) and np.array_equal(ta, tb)
    for k in O.GRAD_CLASSES:
        a, b = getattr(ga, k), getattr(gb, k)
        assert np.abs(a - b).max() <= 1e-5 * max(np.abs(a).max(), 1e-300), k


def test_aux_multi_pixel_kernels_match_one_pixel_kernels_and_oracle(monkeypatch):
    """The 11-plane (with_aux) float32 path runs the two-pixel forward and four-pixel
    backward templated on the channel count; VEGS_GENERIC_COMPOSITE=1 routes it to the
    one-pixel kernels.  Forward planes are bitwise equal; gradients agree to float32
    rounding (different summation order; the suffix term is carried as one scalar), and
    both equal the oracle within the parity tolerance."""
    from oracle import vegs_oracle as O
    from paper_2504_13339_b200.constants import DEFAULT_SETTINGS as S

    gs = scenes.random_gaussians(20_000, seed=41)
    tf = scenes.random_tf(41, 4)
    cam = scenes.orbit_cameras(1, 42, 256, 192)[0]
    rng = np.random.default_rng(43)
    dg = dict(rgb=rng.uniform(-1, 1, size=(192, 256, 3)), alpha=rng.uniform(-1, 1, size=(192, 256)),
              depth=rng.uniform(-1, 1, size=(192, 256)), normal=rng.uniform(-1, 1, size=(192, 256, 3)),
              attrs=rng.uniform(-1, 1, size=(192, 256, 4)))
    img_o, st_o = O.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, True, np.float32)
    g_o = O.rasterize_backward(st_o, **dg)
    out = []
    for generic in (False, True):
        if generic:
            monkeypatch.setenv("VEGS_GENERIC_COMPOSITE", "1")
        img, st = R.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, True, np.float32)
        g = R.rasterize_backward(st, R.ImageGradients(**dg))
        out.append((img, g))
        for k in O.GRAD_CLASSES:
            ref = g_o[k]
            assert np.abs(getattr(g, k) - ref).max() <= 1e-4 * max(np.abs(ref).max(), 1e-300), (generic, k)
    (ia, ga), (ib, gb) = out
    for k in ("rgb", "alpha", "depth", "normal", "attrs"):
        assert np.array_equal(getattr(ia, k), getattr(ib, k)), k
    for k in ("rgb", "depth", "normal", "attrs"):
        ref = img_o[k]
        assert np.abs(getattr(ia, k) - ref).max() <= 1e-4 * max(np.abs(ref).max(), 1.0), k
    assert np.array_equal(st.blend.out_last, st_o["out_last"])
    for k in O.GRAD_CLASSES:
        a, b = getattr(ga, k), getattr(gb, k)
        assert np.abs(a - b).max() <= 1e-5 * max(np.abs(a).max(), 1e-300), k


def test_large_image_takes_radix_binning_and_matches_oracle():
    """2560 x 1600 = 16000 tiles exceeds the counting placement's SMEM cursors, so binning
    takes the radix path by default; the result is still np.lexsort((depth, tile))'s."""
    from oracle import vegs_oracle as O
    from paper_2504_13339_b200.constants import DEFAULT_SETTINGS as S

    gs = scenes.random_gaussians(4000, seed=41)
    gs.log_scale[:] += 1.5
    tf = scenes.random_tf(41, 4)
    cam = scenes.orbit_cameras(1, 42, 2560, 1600)[0]
    img, st = R.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, False, np.float32)
    img_o, st_o = O.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, False, np.float32)
    assert len(st_o["order"]) > 10000
    assert np.array_equal(st.blend.order, st_o["order"])
    assert np.array_equal(st.blend.out_last, st_o["out_last"])
    assert np.array_equal(st.blend.n_contrib, st_o["n_contrib"])
    assert np.abs(img.rgb - img_o["rgb"]).max() < 1e-5


def test_irregular_tf_knots_match_oracle():
    """The shading's TF lookup guesses the segment from uniform spacing and corrects it; with
    irregular knots (some nearly coincident) it must still be np.interp's segment."""
    from oracle import vegs_oracle as O
    from paper_2504_13339_b200.constants import DEFAULT_SETTINGS as S
    from paper_2504_13339_b200.transfer import from_tables

    rng = np.random.default_rng(51)
    ts = np.array([0.0, 0.02, 0.1, 0.1 + 1e-12, 0.35, 0.36, 0.5, 0.9, 0.97, 1.0])
    op = rng.uniform(0.0, 1.0, size=ts.size)
    ts_c = np.array([0.0, 0.3, 0.3 + 1e-9, 0.31, 1.0])
    rgb = rng.uniform(0.0, 1.0, size=(ts_c.size, 3))
    tf = from_tables(ts, op, ts_c, rgb)
    gs = scenes.random_gaussians(3000, seed=52)
    gs.log_scale[:] += 1.0
    cam = scenes.orbit_cameras(1, 53, 96, 80)[0]
    img, st = R.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, False, np.float32)
    img_o, st_o = O.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, False, np.float32)
    assert np.array_equal(st.kept, st_o["kept"])
    assert np.array_equal(st.blend.order, st_o["order"])
    assert np.array_equal(st.blend.out_last, st_o["out_last"])
    assert np.abs(img.rgb - img_o["rgb"]).max() < 1e-5
