"""Host-side profile of the config-4 training step (tiny views: the step is bound by the
Python/ctypes enqueue cost, not the GPU): python scripts/c4_host_profile.py"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_13339_b200 import scenes  # noqa: E402
from paper_2504_13339_b200.device import DeviceTF, Rasterizer  # noqa: E402
from paper_2504_13339_b200.train import TrainConfig, Trainer, View  # noqa: E402


def main():
    learned, truth, _, cams = scenes.config_scene("c4")
    tf = DeviceTF(scenes.range_tf(500, 0.0, 1 / 16))
    rz = Rasterizer(pooled=True)
    gt = torch.from_numpy(truth.pack()).cuda()
    targets = [rz.forward(gt, len(truth), tf, c).out_img.view(c.height, c.width, 3).clone() for c in cams]
    del rz, gt
    tr = Trainer(learned, TrainConfig(iterations=30000))
    views = [View(c, tf, t) for c, t in zip(cams, targets)]
    for _ in range(3):
        tr.step(views)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5):
        tr.step(views)
    torch.cuda.synchronize()
    print(f"{1000 * (time.perf_counter() - t0) / 5:.2f} ms/step wall")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(5):
        tr.step(views)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats(sys.argv[1] if len(sys.argv) > 1 else "tottime").print_stats(40)


if __name__ == "__main__":
    main()
