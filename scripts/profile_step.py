"""Profiling driver: warm up, then run ONE config-2 training step (or one view) between
cudaProfilerStart/Stop so `ncu --profile-from-start off` sees exactly that step."""

import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2504_13339_b200 import scenes  # noqa: E402
from paper_2504_13339_b200.device import DeviceTF, Rasterizer  # noqa: E402
from paper_2504_13339_b200.train import TrainConfig, Trainer, View  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", type=int, default=16)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--aux", action="store_true", help="the 11-plane with_aux iteration")
    args = ap.parse_args()
    learned, truth, tf, cams = scenes.config_scene("c2")
    cams = cams[:args.views]
    dtf = DeviceTF(tf)
    rz = Rasterizer()
    gt = torch.from_numpy(truth.pack()).cuda()
    targets = [rz.forward(gt, len(truth), dtf, c).out_img.view(c.height, c.width, 3).clone() for c in cams]
    del rz, gt
    tr = Trainer(learned, TrainConfig(iterations=30000), with_aux=args.aux)
    views = [View(c, dtf, t) for c, t in zip(cams, targets)]
    for _ in range(args.warmup):
        tr.step(views, total_views=16)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    loss = tr.step(views, total_views=16)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"profiled one step over {len(views)} view(s); loss {float(loss.item()):.6f}; "
          f"launches/view {tr.rz.launches / ((args.warmup + 1) * len(views)):.1f}")


if __name__ == "__main__":
    main()
