"""CPU-side checks: the C-ABI library loads and exports every symbol the header declares,
and the host logic (structs, parameter layout, sharding, generators) is right."""

import ctypes
import math
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2504_13339_b200 import _lib, scenes
from paper_2504_13339_b200.camera import Camera
from paper_2504_13339_b200.constants import DEFAULT_SETTINGS, RasterSettings
from paper_2504_13339_b200.model import FLOATS_PER_GAUSSIAN, GaussianSet, class_offsets
from paper_2504_13339_b200.parallel import shard_views

ROOT = Path(__file__).resolve().parents[1]


def header_functions():
    text = (ROOT / "include" / "vegsplat_b200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char \*)\s*(vegs_\w+)\s*\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    names = header_functions()
    assert len(names) >= 13
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(_lib.exported_symbols()) == names
    assert lib.vegs_version().startswith(b"vegsplat_b200")


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.VegsCamera) == 8 * (3 + 9 + 4) + 8
    assert ctypes.sizeof(_lib.VegsSettings) == 8 * 8 + 8
    assert ctypes.sizeof(_lib.VegsTF) == 16
    assert ctypes.sizeof(_lib.VegsSplatTable) == 12 * 8


def test_loss_workspace_query_runs_without_a_gpu():
    b3 = _lib.size_query("vegs_loss_l1_ssim", None, None, 64, 64, 3, 0.8, 0.2, None, None, tail=(None,))
    assert b3 == 4 * 9 * 54 * 54


@pytest.mark.gpu
def test_cub_workspace_queries():
    # CUB's queries read the device's properties, so they need the GPU
    n = 1000
    b = _lib.size_query("vegs_bin_count", None, n, None, None, None, tail=(None,))
    assert b > 8 * n
    args = (None, None, None, None, None, n, n, 20 * n, 512, 512, 16, None, None, None, None, None, None, None, 3)
    b2 = _lib.size_query("vegs_bin_sort", *args, tail=(None,))
    assert b2 > 4 * 4 * n


def test_bad_arguments_are_rejected_not_thrown():
    with pytest.raises(ValueError):
        _lib.call("vegs_bin_sort", None, None, None, None, None, 10, 10, 10, 64, 64, 8, None, None, None,
                  None, None, None, None, 3, None, ctypes.byref(ctypes.c_size_t(0)), None)
    with pytest.raises(ValueError):
        _lib.call("vegs_composite_forward", None, None, None, None, None, 3, 0, None, 64, 64, 0.99, 1e-4,
                  None, None, None, None, None, None)
    # more instances than int32 positions can address: refused before any CUDA call
    with pytest.raises(ValueError):
        _lib.size_query("vegs_bin_sort", None, None, None, None, None, 1000, 1000, 2**31, 512, 512, 16, None,
                        None, None, None, None, None, None, 3, tail=(None,))


def test_parameter_pack_roundtrip():
    gs = scenes.random_gaussians(17, seed=3)
    flat = gs.pack()
    assert flat.shape == (17 * FLOATS_PER_GAUSSIAN,)
    back = GaussianSet.unpack(flat, 17)
    for k, v in gs.arrays().items():
        assert np.array_equal(v, getattr(back, k))
    offs = class_offsets(17)
    assert offs["position"] == (0, 51, 3) and offs["raw_beta"][1] == 17 * 19


def test_camera_constants_match_reference_formulas():
    cam = Camera(position=(1.0, 2.0, 3.0), target=(0.0, 0.0, 0.0), fov_y=math.radians(50), width=320, height=200)
    from paper_2504_13339_b200.device import camera_struct, settings_struct

    cs = camera_struct(cam)
    assert cs.focal == 0.5 * 200 / math.tan(0.5 * cam.fov_y)
    rot = np.array(cs.rot).reshape(3, 3)
    assert np.allclose(rot @ rot.T, np.eye(3))
    # forward row points from the camera at the target: positive depth in front
    d = np.array(cam.target) - np.array(cam.position)
    assert (rot @ d)[2] > 0
    st = settings_struct(DEFAULT_SETTINGS)
    assert st.tile_size == 16 and st.alpha_clamp == 0.99
    with pytest.raises(ValueError):
        settings_struct(RasterSettings(tile_size=8))


@pytest.mark.parametrize("n,world", [(16, 1), (16, 2), (16, 8), (17, 4), (3, 8)])
def test_shard_views_partition(n, world):
    shards = [shard_views(n, r, world) for r in range(world)]
    flat = [i for s in shards for i in s]
    assert flat == list(range(n))
    sizes = [len(s) for s in shards]
    assert max(sizes) - min(sizes) <= 1


def test_scene_generators_are_deterministic():
    a = scenes.random_gaussians(100, seed=4)
    b = scenes.random_gaussians(100, seed=4)
    for k, v in a.arrays().items():
        assert np.array_equal(v, getattr(b, k))
    tf = scenes.random_tf(2, 4)
    assert len(tf.opacity.ts) == 256 and tf.opacity.values.max() <= 1.0
    blobs = scenes.blob_gaussians(5000, seed=1)
    assert np.abs(blobs.position).max() < 3.0
    cams = scenes.orbit_cameras(16, 3, 1024, 1024)
    assert all(abs(np.linalg.norm(c.position) - 3.0) < 1e-12 for c in cams)
