"""Profiling driver for the forward render: warm up, then run ONE render between
cudaProfilerStart/Stop (ncu --profile-from-start off): --config c3 (3M blob Gaussians,
1920x1080, the sweep's first TF) or c2 (1M Gaussians, 1024^2, view 0).  Prints the
instance count so the capture can be scaled to other frames."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2504_13339_b200 import scenes  # noqa: E402
from paper_2504_13339_b200.device import DeviceTF, Rasterizer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", choices=("c2", "c3"), default="c3")
    ap.add_argument("--no-cull", action="store_true", help="the reference's tile lists (default: culled, as the sweep)")
    args = ap.parse_args()
    if args.config == "c3":
        gs = scenes.blob_gaussians(3_000_000, seed=1)
        cam = scenes.orbit_cameras(2, 5, 1920, 1080)[0]
        tf = DeviceTF(scenes.random_tf(1000))
    else:
        gs, _, tf_h, cams = scenes.config_scene("c2")
        cam, tf = cams[0], DeviceTF(tf_h)
    params = torch.from_numpy(gs.pack()).cuda()
    rz = Rasterizer(cull=not args.no_cull)
    rz.contrib_counts = False
    for _ in range(2):
        rz.forward(params, len(gs), tf, cam)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    fr = rz.forward(params, len(gs), tf, cam)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"profiled one {args.config} render: {fr.n_kept} kept splats, {fr.n_inst} instances "
          f"({int(fr.tile_end[-1])} tile-list entries)")


if __name__ == "__main__":
    main()
