"""Forward compositing work statistics (measurement build, -DVEGS_FWD_STATS): per c2 view,
warp-entries whose float64 exponent ran, passing pixels in them (of 64 per entry), blended
pairs (contributor counts) and instances.  Run with libvariants/stats.so in place."""
import ctypes
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2504_13339_b200 import _lib, scenes  # noqa: E402
from paper_2504_13339_b200.device import DeviceTF, Rasterizer  # noqa: E402


def main():
    gs, truth, tf, cams = scenes.config_scene(sys.argv[1] if len(sys.argv) > 1 else "c2")
    dtf = DeviceTF(tf)
    rz = Rasterizer()
    params = torch.from_numpy(gs.pack()).cuda()
    f = _lib.load().vegs_debug_fwd_stats
    f.argtypes = [ctypes.c_void_p, ctypes.c_int]
    buf = (ctypes.c_ulonglong * 4)()
    f(buf, 1)
    for v in range(min(4, len(cams))):
        fr = rz.forward(params, len(gs), dtf, cams[v])
        torch.cuda.synchronize()
        f(buf, 1)
        e, p, l = buf[0], buf[1], buf[2]
        nc = int(fr.n_contrib.sum().item()) if fr.n_contrib is not None else -1
        cs = _lib.load().vegs_debug_cull_stats
        cs.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        out = (ctypes.c_ulonglong * 4)()
        tx = (cams[v].width + 15) // 16
        nt = tx * ((cams[v].height + 15) // 16)
        cs(fr.tile_start.data_ptr(), fr.tile_end.data_ptr(), tx, nt, fr.sorted_gauss.data_ptr(),
           fr.record.data_ptr(), fr.rect.data_ptr(), out)
        print(f"view {v}: instances {out[0]}  tile-culled {out[1] / max(out[0], 1):.3f}  "
              f"all-8x8-culled {out[2] / max(out[0], 1):.3f}  bbox-culled {out[3] / max(out[0], 1):.3f}", flush=True)
        print(f"view {v}: entries {e}  pass/entry {p / max(e, 1):.2f} of 64  live/entry {l / max(e, 1):.2f}  "
              f"passing {p}  blended {nc}  instances {fr.n_inst}", flush=True)


if __name__ == "__main__":
    main()
