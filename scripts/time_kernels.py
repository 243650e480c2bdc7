"""Quick timing of every C-ABI call of one config-2 view (CUDA events around each call on a
single stream, forward + backward over 4 views): python scripts/time_kernels.py [reps] [channels] [f64|fast]"""
import sys
from collections import defaultdict
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2504_13339_b200 import scenes  # noqa: E402
from paper_2504_13339_b200.device import DeviceTF, LossKernel, Rasterizer  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    n_ch = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    f64 = len(sys.argv) > 3 and sys.argv[3] == "f64"  # the float64 blend (reference default dtype)
    fast = len(sys.argv) > 3 and sys.argv[3] == "fast"  # float32-T forward (training path)
    gs, truth, tf, cams = scenes.config_scene("c2")
    dtf = DeviceTF(tf)
    rz = Rasterizer(n_channels=n_ch, store_f64=f64, fast_t=fast)
    params = torch.from_numpy(gs.pack()).cuda()
    grads = torch.zeros_like(params)
    times = defaultdict(list)

    class T:
        def mark(self, name, begin, rz=None):
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            if begin:
                self.s = ev
            else:
                times[name].append((self.s, ev))

    d_img = torch.rand(1024, 1024, n_ch, device="cuda", dtype=torch.float64 if f64 else torch.float32) - 0.5
    loss = LossKernel(params.device) if n_ch == 3 and not f64 else None
    target = torch.rand(1024, 1024, 3, device="cuda")
    d_loss = torch.empty(1024, 1024, 3, device="cuda")
    sums = torch.zeros(2, dtype=torch.float64, device="cuda")
    for r in range(reps + 2):
        rz.timer = T() if r >= 2 else None
        for cam in cams[:4]:
            fr = rz.forward(params, len(gs), dtf, cam)
            if loss is not None:
                loss.timer = rz.timer
                loss(fr.out_img.view(1024, 1024, 3), target, 0.8, 0.2, d_loss, sums)
            rz.backward(fr, d_img, None, grads, accumulate=True)
            if fast and r == reps + 1:
                print("deferred pixels", fr.n_deferred)
    torch.cuda.synchronize()
    for k, v in times.items():
        ms = [a.elapsed_time(b) for a, b in v]
        print(f"{k}: {sum(ms) / len(ms):.3f} ms avg over {len(ms)}")


if __name__ == "__main__":
    main()
