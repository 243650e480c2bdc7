"""Training-step time at config 2 per lane count, rgb and aux:
python scripts/lanes_step_time.py [steps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_13339_b200 import scenes  # noqa: E402
from paper_2504_13339_b200.device import DeviceTF, Rasterizer  # noqa: E402
from paper_2504_13339_b200.train import TrainConfig, Trainer, View  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    learned, truth, tf, cams = scenes.config_scene("c2")
    dtf = DeviceTF(tf)
    rz = Rasterizer()
    gt = torch.from_numpy(truth.pack()).cuda()
    targets = [rz.forward(gt, len(truth), dtf, c).out_img.view(c.height, c.width, 3).clone() for c in cams]
    del rz, gt
    for aux in (False, True):
        for lanes in (3, 4, 3, 4):
            tr = Trainer(learned, TrainConfig(iterations=30000), with_aux=aux, lanes=lanes)
            views = [View(c, dtf, t) for c, t in zip(cams, targets)]
            tr.step(views)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(steps):
                tr.step(views)
            e1.record()
            torch.cuda.synchronize()
            print(f"with_aux={aux} lanes={lanes}: {e0.elapsed_time(e1) / steps:.1f} ms/step")
            del tr
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
