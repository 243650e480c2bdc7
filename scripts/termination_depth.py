"""Diagnostic: where each tile of one c2 view terminates (every pixel's transmittance
test fired), replayed in float64 with torch: the share of instances a depth-sliced
binning could leave unplaced, and how the termination points spread over the depth
order: python scripts/termination_depth.py"""
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
    # depth rank of every splat in the kept depth order (sorted_gauss holds splat ids)
    yy, xx = torch.meshgrid(torch.arange(16, device="cuda"), torch.arange(16, device="cuda"), indexing="ij")
    stop = float(rz.settings.transmittance_stop)
    clamp = float(rz.settings.alpha_clamp)
    n_inst = n_after = n_open = 0
    term_frac = []
    for t in range(4096):
        s0, s1 = int(ts[t]), int(te[t])
        if s1 <= s0:
            continue
        ty, tx = divmod(t, 64)
        g = fr.sorted_gauss[s0:s1].long()
        r = rec[g].double()
        px = (tx * 16 + xx).double().view(1, -1) + 0.5
        py = (ty * 16 + yy).double().view(1, -1) + 0.5
        dx = px - r[:, 0:1]
        dy = py - r[:, 1:2]
        pw = -0.5 * (r[:, 2:3] * dx * dx + r[:, 4:5] * dy * dy) - r[:, 3:4] * dx * dy
        a = torch.where(pw >= r[:, 6:7], (r[:, 5:6] * torch.exp(pw)).clamp(max=clamp), torch.zeros_like(pw))
        T = torch.cumprod(1.0 - a, 0)  # transmittance after each instance (no early stop)
        hit = T < stop
        done = hit.any(0)
        n_inst += s1 - s0
        if bool(done.all()):
            first = torch.where(hit, torch.arange(s1 - s0, device="cuda").view(-1, 1), s1 - s0).min(0).values
            end = int(first.max()) + 1
            n_after += (s1 - s0) - end
            term_frac.append(end / (s1 - s0))
        else:
            n_open += 1
    tf_ = torch.tensor(term_frac)
    print(f"instances {n_inst}; tiles with every pixel terminated {len(term_frac)} of 4096 "
          f"(open {n_open}); instances after the termination point {n_after} ({100 * n_after / n_inst:.1f}%); "
          f"termination at p10/p50/p90 {tf_.quantile(0.1):.2f}/{tf_.quantile(0.5):.2f}/{tf_.quantile(0.9):.2f} "
          f"of the tile's list")


if __name__ == "__main__":
    main()
