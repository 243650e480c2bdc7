"""Diagnostic: per-tile work of one c2 view (instances up to the tile's last contributor)
and the makespan of greedy scheduling onto G concurrent CTA slots, in launch order vs
heaviest-first: python scripts/tile_balance.py"""
import heapq
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_13339_b200 import scenes  # noqa: E402
from paper_2504_13339_b200.device import DeviceTF, Rasterizer  # noqa: E402


def makespan(work, slots):
    h = [0.0] * slots
    for w in work:
        t = heapq.heappop(h)
        heapq.heappush(h, t + w)
    return max(h)


def main():
    gs, truth, tf, cams = scenes.config_scene("c2")
    rz = Rasterizer()
    params = torch.from_numpy(gs.pack()).cuda()
    fr = rz.forward(params, len(gs), DeviceTF(tf), cams[0])
    ts, te = fr.tile_start.cpu().numpy(), fr.tile_end.cpu().numpy()
    last = fr.out_last.view(1024, 1024).cpu().numpy()
    t = last.reshape(64, 16, 64, 16).transpose(0, 2, 1, 3).reshape(4096, 256).max(1)
    work = np.where(t >= 0, t - ts + 1, 0).astype(np.float64) + 1.0
    n_inst = (te - ts).astype(np.float64)
    print("tiles", len(work), "work mean", work.mean(), "max", work.max(), "p50", np.median(work), "inst mean", n_inst.mean())
    out = Path("gpurun_out")
    if out.is_dir():
        np.savez(out / "tile_work.npz", work=work, n_inst=n_inst)
    by_count = work[np.argsort(-n_inst, kind="stable")]  # the order binning launches (instance counts)
    for slots in (148 * 6, 148 * 8):
        lb = work.sum() / slots
        nat, lpt = makespan(work, slots), makespan(np.sort(work)[::-1], slots)
        cnt = makespan(by_count, slots)
        print(f"slots {slots}: lower bound {lb:.0f}  launch order {nat:.0f} ({nat / lb:.3f})  heaviest-first "
              f"by work {lpt:.0f} ({lpt / lb:.3f})  by instance count {cnt:.0f} ({cnt / lb:.3f})")




def warp_imbalance():
    """Share of (warp, instance-slot) pairs a backward CTA spends above a warp's own last
    contributor (the warp has nothing to do there but waits at the batch barriers)."""
    gs, truth, tf, cams = scenes.config_scene("c2")
    rz = Rasterizer()
    params = torch.from_numpy(gs.pack()).cuda()
    fr = rz.forward(params, len(gs), DeviceTF(tf), cams[0])
    ts = fr.tile_start.cpu().numpy()
    last = fr.out_last.view(1024, 1024).cpu().numpy()
    blk = last.reshape(64, 2, 8, 64, 2, 8).transpose(0, 3, 1, 4, 2, 5).reshape(4096, 4, 64).max(2)
    rel = np.where(blk >= 0, blk - ts[:, None] + 1, 0)
    hi = rel.max(1, keepdims=True)
    print("warp-last imbalance: idle share", float((hi - rel).sum() / max(4 * hi.sum(), 1)))


if __name__ == "__main__":
    main()
    warp_imbalance()
