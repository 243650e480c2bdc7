"""Config-4 steps with and without graph replay: per-step times and graph statistics."""
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
    n_tf = 16
    tfs = [DeviceTF(scenes.range_tf(500 + k, k / n_tf, (k + 1) / n_tf)) for k in range(n_tf)]
    rz = Rasterizer(pooled=True)
    gt = torch.from_numpy(truth.pack()).cuda()
    sets = {}
    for k in range(n_tf):
        sets[k] = [View(c, tfs[k], rz.forward(gt, len(truth), tfs[k], c).out_img.view(c.height, c.width, 3).clone())
                   for c in cams]
    for graphs in (False, True):
        tr = Trainer(learned, TrainConfig(iterations=30000), graphs=graphs)
        tr.track_densify(True)
        for k in range(n_tf):
            tr.step(sets[k], total_views=len(cams))
        torch.cuda.synchronize()
        ts = []
        for s in range(20):
            t0 = time.perf_counter()
            tr.step(sets[s % n_tf], total_views=len(cams))
            torch.cuda.synchronize()
            ts.append(1000 * (time.perf_counter() - t0))
        print("graphs" if graphs else "eager", "ms/step", [round(t, 1) for t in ts], tr.graph_stats,
              [l.rz.inst_cap for l in tr.lanes], [l.rz.kept_cap for l in tr.lanes])


if __name__ == "__main__":
    main()
