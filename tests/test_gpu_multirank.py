"""Two ranks of the view-sharded training step on the one GPU a gpurun call has (SURVEY.md
§8(e)).  The ranks use gloo, whose all-reduce is host-side, so no kernel waits on another
rank and time-sharing one device cannot deadlock; the exchange path (pack, asynchronous
bucketed all-reduce, Adam per bucket) is the one NCCL runs under torchrun.  Checks: the
replicas stay bitwise identical, and the all-reduced gradient / updated parameters match
one process training on all the views."""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N_VIEWS = 4


def _setup():
    from paper_2504_13339_b200 import scenes
    from paper_2504_13339_b200.device import DeviceTF
    from paper_2504_13339_b200.train import View

    gs = scenes.random_gaussians(3000, seed=3)
    dtf = DeviceTF(scenes.random_tf(2, 4))
    cams = scenes.orbit_cameras(N_VIEWS, 3, 96, 80)
    rng = np.random.default_rng(5)
    targets = [torch.from_numpy(rng.uniform(0, 1, (c.height, c.width, 3)).astype(np.float32)).cuda() for c in cams]
    return gs, [View(c, dtf, t) for c, t in zip(cams, targets)]


def _worker(rank, world, port, payload, out):
    import torch.distributed as dist

    from paper_2504_13339_b200.parallel import shard_views
    from paper_2504_13339_b200.train import Trainer, TrainConfig

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        gs, views = _setup()
        mine = [views[i] for i in shard_views(len(views), rank, world)]
        tr = Trainer(gs, TrainConfig(iterations=100), group=dist.group.WORLD, grad_payload=payload, grad_buckets=3)
        for it in (1, 2):
            tr.step(mine, iteration=it, total_views=len(views))
        torch.cuda.synchronize()
        out[rank] = (tr.params.cpu().numpy(), tr.grads.cpu().numpy(), tr.exchange.collectives)
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("payload", ["f64", "f32"])
def test_two_rank_step_matches_one_process(payload):
    import torch.multiprocessing as mp

    from paper_2504_13339_b200.train import Trainer, TrainConfig

    gs, views = _setup()
    ref = Trainer(gs, TrainConfig(iterations=100))
    for it in (1, 2):
        ref.step(views, iteration=it)
    p_ref, g_ref = ref.params.cpu().numpy(), ref.grads.cpu().numpy()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(2, _free_port(), payload, out), nprocs=2, join=True)
        res = [out[r] for r in range(2)]
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])  # identical replicas
    assert res[0][2] == 2 * 3  # two steps, three buckets
    gmax = np.abs(g_ref).max()
    tol_g = 1e-12 if payload == "f64" else 1e-6  # per-rank partial sums vs one sequential sum (+ f32 rounding)
    assert np.abs(res[0][1] - g_ref).max() <= tol_g * gmax
    assert np.abs(res[0][0] - p_ref).max() <= 1e-5 * TrainConfig().lr_weight
