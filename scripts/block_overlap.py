"""Diagnostic: for one c2 view, how many (instance, 8x8 block) pairs the backward visits
versus (instance, 16x8 block) pairs -- i.e. how much a 4-pixels-per-lane backward (one
warp per 16x8 half tile) would re-use each instance: python scripts/block_overlap.py"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_13339_b200 import scenes  # noqa: E402
from paper_2504_13339_b200.device import DeviceTF, Rasterizer  # noqa: E402


def main():
    gs, truth, tf, cams = scenes.config_scene("c2")
    rz = Rasterizer()
    params = torch.from_numpy(gs.pack()).cuda()
    fr = rz.forward(params, len(gs), DeviceTF(tf), cams[0])
    rec = fr.record.view(-1, 12)
    ts, te = fr.tile_start.long(), fr.tile_end.long()
    last = fr.out_last.view(1024, 1024).long()
    yy, xx = torch.meshgrid(torch.arange(16, device="cuda"), torch.arange(16, device="cuda"), indexing="ij")
    n8 = n16 = n256 = 0
    for t in range(4096):
        s0, s1 = int(ts[t]), int(te[t])
        ty, tx = divmod(t, 64)
        lp = last[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16]
        hi = int(lp.max())
        if hi < s0:
            continue
        g = fr.sorted_gauss[s0:hi + 1].long()
        r = rec[g]
        px = (tx * 16 + xx).double().view(1, 16, 16) + 0.5
        py = (ty * 16 + yy).double().view(1, 16, 16) + 0.5
        dx = px - r[:, 0].double().view(-1, 1, 1)
        dy = py - r[:, 1].double().view(-1, 1, 1)
        pw = -0.5 * (r[:, 2].double().view(-1, 1, 1) * dx * dx + r[:, 4].double().view(-1, 1, 1) * dy * dy) \
            - r[:, 3].double().view(-1, 1, 1) * dx * dy
        ok = pw >= r[:, 6].double().view(-1, 1, 1)
        idx = torch.arange(s0, hi + 1, device="cuda").view(-1, 1, 1)
        ok &= idx <= lp.view(1, 16, 16)
        b8 = ok.view(-1, 2, 8, 2, 8).any(4).any(2)          # (inst, by, bx)
        b16 = b8.any(2)                                       # (inst, by): 16x8 halves
        n8 += int(b8.sum())
        n16 += int(b16.sum())
        n256 += int(b16.any(1).sum())
    print(f"(instance, 8x8 block) visits {n8}  (instance, 16x8 block) visits {n16}  "
          f"ratio {n8 / max(n16, 1):.3f} (2.0 = every 16x8 visit would serve both 8x8 blocks); "
          f"(instance, 16x16 tile) visits {n256}, 16x8/16x16 ratio {n16 / max(n256, 1):.3f}")


if __name__ == "__main__":
    main()
