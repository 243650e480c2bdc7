"""World-size-2 gloo test of the view-sharded step's host logic.

Each rank computes the gradients of its view shard (oracle on the CPU stands in for the
per-rank GPU kernels, which need a device), scales by 1/total_views, and the same
``allreduce_gradients`` the Trainer calls sums them; the result must equal the
single-process mean over all views, and both ranks must end with identical buffers."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_13339_b200.parallel import allreduce_gradients, shard_views


def _scene():
    from paper_2504_13339_b200 import scenes

    gs = scenes.random_gaussians(300, seed=0)
    tf = scenes.random_tf(2, 4)
    cams = scenes.orbit_cameras(4, 3, 48, 48)
    return gs, tf, cams


def _view_grad(gs, tf, cam, seed):
    from oracle import vegs_oracle as O
    from paper_2504_13339_b200.constants import DEFAULT_SETTINGS as S

    img, st = O.render_with_state(gs, tf, cam, (1.0, 1.0, 1.0), S, False, np.float32)
    d = np.random.default_rng(seed).uniform(-1, 1, size=(cam.height, cam.width, 3))
    g = O.rasterize_backward(st, d)
    return np.concatenate([np.asarray(g[k], dtype=np.float64).ravel() for k in O.GRAD_CLASSES])


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gs, tf, cams = _scene()
    mine = shard_views(len(cams), rank, world)
    buf = torch.zeros(19 * len(gs), dtype=torch.float64)
    for v in mine:
        buf += torch.from_numpy(_view_grad(gs, tf, cams[v], v)) / len(cams)
    allreduce_gradients(buf)
    out[rank] = buf.numpy().copy()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gradients_equal_single_process_mean(world):
    """world 2: shards of 2 + 2 views; world 3: uneven shards of 2 + 1 + 1."""
    gs, tf, cams = _scene()
    full = sum(_view_grad(gs, tf, c, i) for i, c in enumerate(cams)) / len(cams)
    assert [len(shard_views(len(cams), r, world)) for r in range(world)] == ([2, 2] if world == 2 else [2, 1, 1])
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
        res = [out[r] for r in range(world)]
    for r in res[1:]:
        assert np.array_equal(r, res[0])  # replicas stay identical
    assert np.abs(res[0] - full).max() <= 1e-12 * max(np.abs(full).max(), 1.0)


def test_gradient_exchange_buckets_cover_the_units():
    """The exchange's unit ranges tile the 19 units of the class-major buffer in order."""
    from paper_2504_13339_b200.parallel import GradientExchange

    for b in (1, 2, 3, 4, 7, 19, 40):
        ex = GradientExchange(5, "cpu", payload="f64", buckets=b)
        flat = [u for lo, hi in ex.bounds for u in range(lo, hi)]
        assert flat == list(range(19)) and all(hi > lo for lo, hi in ex.bounds)
        assert len(ex.bounds) == min(b, 19) and ex.pay32 is None
    assert GradientExchange(5, "cpu", payload="f32").pay32.dtype == torch.float32
    with pytest.raises(ValueError):
        GradientExchange(5, "cpu", payload="bf16")
