"""Diagnostic: for one c2 view, the share of (splat, tile) instances no pixel of their tile
can blend (pw < pmin on all 256 pixels, i.e. the splat's rect touches the tile but its
ellipse does not), and the share behind every pixel's last contributor (never read by the
backward): python scripts/instance_waste.py"""
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
    ts, te = fr.tile_start.long().cpu(), fr.tile_end.long().cpu()
    last = fr.out_last.view(1024, 1024).long()
    yy, xx = torch.meshgrid(torch.arange(16, device="cuda"), torch.arange(16, device="cuda"), indexing="ij")
    n_inst = n_empty = n_behind = n_empty8 = 0
    for t in range(4096):
        s0, s1 = int(ts[t]), int(te[t])
        if s1 <= s0:
            continue
        ty, tx = divmod(t, 64)
        lp = last[ty * 16:(ty + 1) * 16, tx * 16:(tx + 1) * 16]
        g = fr.sorted_gauss[s0:s1].long()
        r = rec[g]
        px = (tx * 16 + xx).double().view(1, 16, 16) + 0.5
        py = (ty * 16 + yy).double().view(1, 16, 16) + 0.5
        dx = px - r[:, 0].double().view(-1, 1, 1)
        dy = py - r[:, 1].double().view(-1, 1, 1)
        pw = -0.5 * (r[:, 2].double().view(-1, 1, 1) * dx * dx + r[:, 4].double().view(-1, 1, 1) * dy * dy) \
            - r[:, 3].double().view(-1, 1, 1) * dx * dy
        ok = pw >= r[:, 6].double().view(-1, 1, 1)
        n_inst += s1 - s0
        n_empty += int((~ok.view(s1 - s0, -1).any(1)).sum())
        n_empty8 += int((~ok.view(-1, 2, 8, 2, 8).any(4).any(2)).sum())
        n_behind += s1 - 1 - max(int(lp.max()), s0 - 1)  # out_last: global instance index or -1
    print(f"instances {n_inst}: no pixel passes {n_empty} ({100 * n_empty / n_inst:.1f}%), "
          f"behind every last contributor {n_behind} ({100 * n_behind / n_inst:.1f}%), "
          f"empty (instance, 8x8 block) pairs {100 * n_empty8 / (4 * n_inst):.1f}%")


if __name__ == "__main__":
    main()
