"""Profiling driver for one config-4 training step (64 views at 800x800, 200k Gaussians)
between cudaProfilerStart/Stop: python scripts/profile_c4.py [--graphs]"""
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
    ap.add_argument("--graphs", action="store_true")
    args = ap.parse_args()
    learned, truth, _, cams = scenes.config_scene("c4")
    tf = DeviceTF(scenes.range_tf(500, 0.0, 1.0 / 16))
    rz = Rasterizer(pooled=True)
    gt = torch.from_numpy(truth.pack()).cuda()
    views = [View(c, tf, rz.forward(gt, len(truth), tf, c).out_img.view(c.height, c.width, 3).clone()) for c in cams]
    tr = Trainer(learned, TrainConfig(iterations=30000), graphs=args.graphs)
    for _ in range(3):
        tr.step(views)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    tr.step(views)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("profiled one config-4 step", tr.graph_stats, tr.rz.last_counts)


if __name__ == "__main__":
    main()
