"""Binning primitives at scale: vegs_bin_count's scan of the (kept, tiles) counters against
numpy's cumulative sums, and the compositing launch order (heaviest tiles first, ties in
tile order) against numpy's stable argsort."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs CUDA", allow_module_level=True)

from paper_2504_13339_b200 import _lib  # noqa: E402


@pytest.mark.parametrize("n", [1, 2047, 2048, 2049, 300_001, 3_000_000])
def test_bin_count_scan_matches_numpy(n):
    """vegs_bin_count: offsets, kept indices and totals against numpy's cumulative sums."""
    rng = np.random.default_rng(n)
    tiles = rng.integers(0, 40, n).astype(np.uint32)
    tiles[rng.random(n) < 0.3] = 0  # culled splats
    t = torch.from_numpy(tiles.view(np.int32)).cuda()
    offs = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    kept = torch.empty(n + 1, dtype=torch.int64, device="cuda")
    counts = torch.empty(2, dtype=torch.int64, device="cuda")
    p = lambda x: ctypes.c_void_p(x.data_ptr())  # noqa: E731
    nb = _lib.size_query("vegs_bin_count", p(t), n, p(offs), p(kept), p(counts), tail=(None,))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    _lib.call("vegs_bin_count", p(t), n, p(offs), p(kept), p(counts), p(ws), ctypes.byref(ctypes.c_size_t(nb)), None)
    torch.cuda.synchronize()
    ref_off = np.concatenate([[0], np.cumsum(tiles.astype(np.int64))])
    ref_kept = np.concatenate([[0], np.cumsum((tiles > 0).astype(np.int64))])
    assert np.array_equal(offs.cpu().numpy(), ref_off) and np.array_equal(kept.cpu().numpy(), ref_kept)
    assert counts.cpu().tolist() == [int(ref_kept[-1]), int(ref_off[-1])]


@pytest.mark.parametrize("wh", [(1024, 1024), (1920, 1080), (200, 120)])
def test_tile_launch_order_is_heaviest_first_stable(wh):
    """The compositing launch order: tiles by decreasing instance count, ties in tile
    order -- numpy's stable argsort of 0xffff - min(count, 0xffff)."""
    from paper_2504_13339_b200 import scenes
    from paper_2504_13339_b200.device import DeviceTF, Rasterizer

    gs = scenes.blob_gaussians(200_000, seed=2)
    cam = scenes.orbit_cameras(1, 5, *wh)[0]
    rz = Rasterizer(pooled=False, cull=True)
    fr = rz.forward(torch.from_numpy(gs.pack()).cuda(), len(gs), DeviceTF(scenes.random_tf(7)), cam)
    c = (fr.tile_end - fr.tile_start).cpu().numpy().astype(np.int64)
    key = 0xFFFF - np.minimum(c, 0xFFFF)
    assert np.array_equal(fr.tile_order.cpu().numpy(), np.argsort(key, kind="stable"))


@pytest.mark.parametrize("wh", [(1024, 1024), (1000, 700), (200, 120), (1920, 1080)])
@pytest.mark.parametrize("cull", [False, True])
def test_two_level_placement_equals_single_level(monkeypatch, wh, cull):
    """The two-level placement (4x4-tile blocks, then runs per tile) builds exactly the tile
    lists of the single-level placement (VEGS_PLACE_FLAT=1): same ranges, same ids in the
    same order, on grids that are and are not multiples of the block."""
    from paper_2504_13339_b200 import scenes
    from paper_2504_13339_b200.device import DeviceTF, Rasterizer

    gs = scenes.blob_gaussians(150_000, seed=3)
    gs.log_scale[:300] += 2.5  # a few splats spanning many blocks (full 16-tile masks)
    cam = scenes.orbit_cameras(1, 5, *wh)[0]
    params = torch.from_numpy(gs.pack()).cuda()
    tf = DeviceTF(scenes.random_tf(9))
    out = []
    for flat in ("1", "0"):
        monkeypatch.setenv("VEGS_PLACE_FLAT", flat)
        fr = Rasterizer(pooled=False, cull=cull).forward(params, len(gs), tf, cam)
        listed = int(fr.tile_end.max())
        out.append((fr.tile_start.clone(), fr.tile_end.clone(), fr.sorted_gauss[:listed].clone(), fr.out_img.clone()))
    for a, b in zip(out[0], out[1]):
        assert torch.equal(a, b)


@pytest.mark.parametrize("n", [5, 2000, 16_384])
def test_small_depth_sort_equals_device_wide_sort(monkeypatch, n):
    """Views with up to 16384 splats to sort take the one-CTA radix sort; its order (and so
    every tile list) equals the device-wide sort's (VEGS_SMALL_SORT=0), ties included."""
    from paper_2504_13339_b200 import scenes
    from paper_2504_13339_b200.device import DeviceTF, Rasterizer

    gs = scenes.random_gaussians(n, seed=11)
    gs.position[: n // 4] = gs.position[0]  # equal depths: the stable order decides
    cam = scenes.orbit_cameras(1, 3, 160, 120)[0]
    params = torch.from_numpy(gs.pack()).cuda()
    tf = DeviceTF(scenes.random_tf(2, 4))
    out = []
    for env in ("0", "1"):
        monkeypatch.setenv("VEGS_SMALL_SORT", env)
        fr = Rasterizer(pooled=False).forward(params, len(gs), tf, cam, want_order=True)
        out.append((fr.tile_start.clone(), fr.tile_end.clone(), fr.order.clone(), fr.out_img.clone()))
    for a, b in zip(out[0], out[1]):
        assert torch.equal(a, b)


def test_culled_binning_edge_cases():
    """Culled binning on degenerate views -- sub-pixel splats (only the footprint dilation
    gives them extent) and a camera looking away from every splat (nothing kept): the frames
    equal the reference lists', the culled lists are no longer (empty when nothing is kept),
    and graph-replayed training steps on such views equal the eager ones."""
    import dataclasses

    from paper_2504_13339_b200 import scenes
    from paper_2504_13339_b200.device import DeviceTF, Rasterizer
    from paper_2504_13339_b200.train import TrainConfig, Trainer, View

    gs = scenes.random_gaussians(3000, seed=21)
    gs.log_scale[:] = -9.0  # far below a pixel: only the footprint dilation gives extent
    tf = DeviceTF(scenes.random_tf(2, 4))
    cam = scenes.orbit_cameras(1, 3, 96, 80)[0]
    away = dataclasses.replace(cam, target=tuple(2 * p - t for p, t in zip(cam.position, cam.target)))
    params = torch.from_numpy(gs.pack()).cuda()
    for c in (cam, away):
        ref = Rasterizer(pooled=False).forward(params, len(gs), tf, c)
        cut = Rasterizer(pooled=False, cull=True).forward(params, len(gs), tf, c)
        assert torch.equal(ref.out_img, cut.out_img) and torch.equal(ref.out_t, cut.out_t)
        assert int(cut.tile_end.max()) <= int(ref.tile_end.max())
        if c is away:
            assert int(ref.tile_end.max()) == 0 and int(cut.tile_end.max()) == 0
    target = torch.rand(cam.height, cam.width, 3, device="cuda")
    views = [View(cam, tf, target), View(away, tf, target)]
    res = []
    for graphs in (False, True):
        tr = Trainer(gs, TrainConfig(iterations=100), graphs=graphs)
        losses = [float(tr.step(views, iteration=s + 1).item()) for s in range(3)]
        res.append((losses, tr.params.clone()))
    assert res[0][0] == res[1][0] and torch.equal(res[0][1], res[1][1])
