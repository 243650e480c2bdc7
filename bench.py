#!/usr/bin/env python
"""Benchmark: BASELINE.json config 2 -- the 1M-Gaussian, 16-view x 1024^2 training step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]

One step = every view of the step rendered (preprocess -> bin/sort -> composite),
scored (0.8 L1 + 0.2 (1-SSIM), the reference's convention), back-propagated (composite
backward -> per-Gaussian float64 gradients), the flat gradient buffer all-reduced across
ranks (NCCL, N > 1) and Adam applied.  The 16 views are sharded across the N ranks
(strong scaling: total work is fixed).  Inputs are synthetic (scenes.py, seeded);
targets are renders of the seed-1 64-blob ground-truth set.  The working set (152 MB
of float64 parameters, ~24M tile instances per view) is far larger than L2, so no flush
is needed between steps.

Reported on rank 0 as one JSON line: ``value`` = steps/s (device-timed, max over ranks),
``e2e`` = the same step through the public API with the step's target images copied
from pinned host memory each step and the loss read back, ``render_mpx_s`` = forward
render throughput over the same views, ``roofline`` for the dominant kernel (CUDA events
on its launching stream inside the timed region), ``cpu_baseline`` = the CPU oracle on a
bounded sample of the same workload, ``clocks`` sampled with nvidia-smi during the
timed region.

``--impl reference`` times the reference itself instead: vegsplat (pure numpy + numba, no
GPU code) installed unmodified under baseline/_ref, through its public API
on all host cores; the views of one step are timed in order within a time budget and
the step extrapolated from them (the line says how many views were timed).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "train steps/s at 1M Gaussians (config 2: 16 views/step @1024x1024)"
UNIT = "steps/s"
MAX_SM_MHZ = 1965.0  # B200 max SM clock; MEASURED_PEAKS.json sm_max_mhz overrides
WORKLOAD = "c2"
VIEWS_PER_STEP = 16


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--render-frames", type=int, default=5)
    ap.add_argument("--cpu-budget-s", type=float, default=60.0)
    ap.add_argument("--ref-budget-s", type=float, default=300.0,
                    help="--impl reference: stop timing further views of the step after this many seconds")
    ap.add_argument("--no-sweep", action="store_true", help="skip the config-3 TF-sweep render measurement")
    ap.add_argument("--no-c4", action="store_true", help="skip the config-4 densify/prune training measurement")
    ap.add_argument("--no-api", action="store_true", help="skip the numpy drop-in API timing")
    ap.add_argument("--api-views", type=int, default=3)
    ap.add_argument("--c4-steps", type=int, default=20)
    ap.add_argument("--sweep-frames", type=int, default=2)
    ap.add_argument("--lanes", type=int, default=4, help="CUDA-stream lanes of the view pipeline")
    ap.add_argument("--c4-lanes", type=int, default=8,
                    help="stream lanes of the config-4 trainer (small views: 8 lanes 70.3 steps/s, 4 lanes 65.4)")
    ap.add_argument("--no-cull", action="store_true",
                    help="bin on the reference's whole rects (default: tight ellipse boxes, identical results)")
    ap.add_argument("--no-shared-projection", action="store_true",
                    help="config-3 sweep: preprocess every (frame, TF) in full instead of projecting each frame once")
    ap.add_argument("--no-graphs", action="store_true",
                    help="host-counted eager steps instead of device-count steps replayed as CUDA graphs")
    ap.add_argument("--backend", choices=("nccl", "gloo"), default="nccl",
                    help="gradient all-reduce backend for N>1 (gloo: host-side plumbing check only)")
    ap.add_argument("--grad-payload", choices=("f32", "f64"), default="f32",
                    help="N>1: all-reduce payload of the step gradient (Adam stays float64, replicated)")
    ap.add_argument("--grad-buckets", type=int, default=4,
                    help="N>1: buckets of the pipelined pack / all-reduce / Adam exchange")
    return ap.parse_args()


def config_block(world: int, backend: str = "nccl", graphs: bool | None = True, payload: str = "f32",
                 buckets: int = 4) -> dict:
    cfg = {"workload": "c2: 1M Gaussians (seed 0) fit to renders of a 1M-Gaussian 64-blob set (seed 1); "
                        "16 views/step at 1024x1024, 256-knot TF; step = render + L1/SSIM + backward "
                        "+ all-reduce + Adam",
            "n_gaussians": 1_000_000, "views_per_step": VIEWS_PER_STEP, "width": 1024, "height": 1024,
            "loss": "0.8*L1 + 0.2*(1-SSIM) (reference (1-lambda) weighting)",
            "parallelism": f"view-sharded dp{world}" + ("" if world == 1 or backend == "nccl" else f" ({backend})"),
            "l2": "inputs larger than L2 (no flush needed)"}
    if world > 1:
        cfg["grad_exchange"] = (f"{buckets} buckets, {payload} payload all-reduce pipelined with the lane sum and "
                                "Adam per bucket")
    if graphs is not None:
        cfg["step_execution"] = ("device-side instance counts, each step one replayed CUDA graph (all views, lanes, "
                                 "Adam); one host wait per step" if graphs else "eager, one host count read per view")
    return cfg


def peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


# -- clocks sampled during the timed region ---------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=10)
        rows = [r.split(", ") for r in Path(self.path).read_text().splitlines() if r.strip()]
        os.unlink(self.path)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


# -- per-launch CUDA-event timing of the compositing kernels -----------------------------

class KernelTimer:
    """Events recorded on the current stream around each C-ABI launch group."""

    def __init__(self, rz, names=("vegs_composite_forward", "vegs_composite_forward_fast", "vegs_composite_backward")):
        import torch

        self.torch = torch
        self.rz = rz
        self.names = set(names)
        self.open: dict = {}
        self.done: dict = {n: [] for n in names}

    def mark(self, name, begin, rz=None):
        if name not in self.names:
            return
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record()  # on the current stream = the launching stream
        key = (name, id(rz))
        if begin:
            src = rz or self.rz
            self.open[key] = (ev, src.last_counts if src is not None else (0, 0))
        else:
            start, counts = self.open.pop(key)
            self.done[name].append((start, ev, counts))

    def summary(self) -> dict:
        out = {}
        for name, recs in self.done.items():
            if recs:
                ms = [a.elapsed_time(b) for a, b, _ in recs]
                out[name] = dict(launches=len(recs), avg_ms=sum(ms) / len(ms), total_ms=sum(ms),
                                 counts=[c for _, _, c in recs], events=recs)
        return out


STAGES = ("vegs_preprocess_forward", "vegs_bin_count", "vegs_bin_sort", "vegs_composite_forward",
          "vegs_composite_forward_fast",
          "vegs_loss_l1_ssim", "vegs_composite_backward", "vegs_preprocess_backward")


def stage_bytes(name: str, n: int, n_kept: int, n_inst: int, pixels: int, listed: float = 1.0) -> float | None:
    """Algorithmic HBM bytes per call (with this build's float64
    parameters and float32 splat table); None where no byte model bounds the stage.
    ``listed``: tile-list entries per reference instance (culled binning, < 1)."""
    if name == "vegs_preprocess_forward":  # params in; record 48 + rect 16 + tiles 4 + depth key 8 out
        return float(152 * n + 76 * n)
    if name == "vegs_bin_sort":  # splat ids in depth order + rects in, one id per instance out
        return float(20 * n_kept + 4 * n_inst * listed)
    if name in ("vegs_composite_forward", "vegs_composite_forward_fast", "vegs_composite_backward"):
        return algorithmic_bytes(name, n_kept, n_inst, pixels, listed=listed)
    if name == "vegs_loss_l1_ssim":  # image + target in, gradient out (fused minimum)
        return float(36 * pixels)
    if name == "vegs_preprocess_backward":  # params in, gradients read+written, row sums
        return float(152 * n + 304 * n + 72 * n_kept)
    return None


def composite_roofline(ksum: dict, pixels: int, ncu_key: str, ncu_file: str = "ncu_composite.json",
                       listed: float = 1.0) -> dict | None:
    """Roofline of the compositing forward from a KernelTimer summary: algorithmic HBM
    bytes / live CUDA-event launch time against MEASURED_PEAKS' HBM, plus
    the issue roofline (warp instructions per launch from the committed ncu capture, scaled
    by the live instance count) that actually bounds it."""
    import torch

    rec = None
    for name in ("vegs_composite_forward", "vegs_composite_forward_fast"):
        if name in ksum:
            rec = ksum[name]
            break
    if rec is None:
        return None
    peak, peak_kind = peaks()
    byts = [algorithmic_bytes("vegs_composite_forward", nk, ni, pixels, listed=listed) for nk, ni in rec["counts"]]
    achieved = sum(byts) / len(byts) / (rec["avg_ms"] / 1000.0) / 1e9
    out = {"bound": "hbm", "kernel": "vegs_composite_forward", "achieved": achieved, "peak": peak,
           "peak_source": peak_kind, "unit": "GB/s", "frac": achieved / peak, "traffic": None,
           "algorithmic_bytes_per_launch": sum(byts) / len(byts), "avg_launch_ms": rec["avg_ms"],
           "launches": rec["launches"], "avg_instances": sum(c[1] for c in rec["counts"]) / len(rec["counts"]),
           "listed_fraction": listed}
    prof = ROOT / "profiles" / ncu_file
    if prof.exists():
        r = json.loads(prof.read_text()).get(ncu_key)
        if r:
            ms_issue = rec["avg_ms"]
            scale = 1.0
            if r.get("instances"):
                # the launches of the very frame the capture profiled (same instance count):
                # their own live duration against the capture's instruction count
                same = [(a.elapsed_time(b)) for (a, b, c) in rec.get("events", []) if c[1] == int(r["instances"])]
                if same:
                    ms_issue = sum(same) / len(same)
                else:
                    scale = out["avg_instances"] / r["instances"]
            out["traffic"] = r["dram_bytes"] * scale
            mhz = MAX_SM_MHZ
            try:
                mhz = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["sm_max_mhz"])
            except Exception:
                pass
            sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
            peak_issue = sms * 4 * mhz * 1e6
            wi = r["warp_instructions"] * scale
            out["issue_roofline"] = {"bound": "issue", "achieved": wi / (ms_issue / 1000.0), "peak": peak_issue,
                                     "unit": "warp-instructions/s",
                                     "frac": wi / (ms_issue / 1000.0) / peak_issue,
                                     "warp_instructions_per_launch": wi, "launch_ms": ms_issue,
                                     "source": f"profiles/{ncu_file}[{ncu_key}]"
                                               + (" scaled by live/profiled instances" if scale != 1.0 else
                                                  (" over the live launches of the profiled frame"
                                                   if r.get("instances") else ""))}
    return out


def algorithmic_bytes(name: str, n_kept: int, n_inst: int, pixels: int, n_ch: int = 3,
                      listed: float = 1.0) -> float:
    """SURVEY.md §8(d) minimum HBM bytes per composite launch, over the instances the
    launch actually walks: n_inst reference instances x ``listed`` (the culled binning's
    tile-list entries per reference instance, measured)."""
    per_inst = 4 + 28 + 4 * n_ch
    per_px = 4 * n_ch + 4 + 4
    b = n_inst * listed * per_inst + pixels * per_px
    if name == "vegs_composite_backward":
        b += n_kept * (6 + n_ch) * 4 * 2
    return float(b)


# -- the B200 arm -------------------------------------------------------------------------

def run_b200(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2504_13339_b200 import scenes
    from paper_2504_13339_b200.device import DeviceTF, Rasterizer
    from paper_2504_13339_b200.parallel import init_from_env, local_device, shard_views
    from paper_2504_13339_b200.train import TrainConfig, Trainer, View

    rank, world, local = init_from_env(args.backend)
    local = local_device(local, args.backend)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    learned, truth, tf, cams = scenes.config_scene(WORKLOAD)
    mine = shard_views(VIEWS_PER_STEP, rank, world)
    dtf = DeviceTF(tf, dev)

    # ground-truth targets for this rank's views (setup, untimed)
    rz_gt = Rasterizer(pooled=True)
    gt_params = torch.from_numpy(truth.pack()).to(dev)
    targets = []
    for i in mine:
        fr = rz_gt.forward(gt_params, len(truth), dtf, cams[i])
        targets.append(fr.out_img.view(cams[i].height, cams[i].width, 3).clone())
    del rz_gt, gt_params
    host_targets = [t.cpu().pin_memory() for t in targets]
    torch.cuda.synchronize()

    group = dist.group.WORLD if world > 1 else None
    trainer = Trainer(learned, TrainConfig(iterations=30000), group=group, lanes=args.lanes,
                      graphs=not args.no_graphs, grad_payload=args.grad_payload, grad_buckets=args.grad_buckets,
                      cull=not args.no_cull)
    views = [View(cams[i], dtf, targets[j]) for j, i in enumerate(mine)]

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(max(args.warmup, 3)):
        trainer.step(views, total_views=VIEWS_PER_STEP)
    torch.cuda.synchronize()

    # ---- timed region: device-resident training steps (no per-kernel events inside)
    launches0 = trainer.launches
    clocks = ClockSampler(local)
    barrier()
    torch.cuda.synchronize()
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    loss = None
    for _ in range(args.steps):
        loss = trainer.step(views, total_views=VIEWS_PER_STEP)
    e1.record()
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1))
    launches = trainer.launches - launches0  # (lane sums, exchange and Adam included)
    ms_step = ms / args.steps
    value = 1000.0 / ms_step
    loss_val = float(loss.item())
    trainer.check_finite()

    # ---- kernel-timing pass: the same steps again with CUDA events around each
    # compositing launch on its lane stream (kept out of the timed region above, whose
    # host-side event records would perturb it)
    timer = KernelTimer(trainer.rz)
    trainer.set_timer(timer)
    trainer.set_graphs(False)  # eager, host-counted launches: events around each kernel, live counts
    trainer.step(views, total_views=VIEWS_PER_STEP)
    k_steps = max(min(args.steps, 5), 2)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(k_steps):
        trainer.step(views, total_views=VIEWS_PER_STEP)
    t1.record()
    torch.cuda.synchronize()
    trainer.set_timer(None)
    trainer.set_graphs(not args.no_graphs)
    ktimed_ms = t0.elapsed_time(t1)
    timer.done = {k: v[len(v) // (k_steps + 1):] for k, v in timer.done.items()}  # drop the re-warm step
    ksum = timer.summary()

    # ---- per-stage profile, serialised on one stream (the pipelined step overlaps stages,
    # which would blur per-stage timings): 4 views through every C-ABI stage of a step
    from paper_2504_13339_b200.device import LossKernel

    stage_timer = KernelTimer(None, names=STAGES)
    srz = Rasterizer(pooled=True, fast_t=trainer.fast_t, cull=trainer.cull)
    srz.contrib_counts = False
    sloss = LossKernel(dev)
    sgrads = torch.zeros_like(trainer.params)
    ssums = torch.zeros(2, dtype=torch.float64, device=dev)
    d_img = torch.empty(1024, 1024, 3, dtype=torch.float32, device=dev)
    listed_n = [0, 0]  # (tile-list entries, reference instances) of the profiled views
    for rep in range(2):  # the first pass grows the pools
        srz.timer = stage_timer if rep else None
        sloss.timer = stage_timer if rep else None
        for v in views[:4]:
            fr = srz.forward(trainer.params, trainer.n, v.tf, v.camera)
            if rep:
                listed_n[0] += int(fr.tile_end[-1])  # serialised pass: the read costs nothing timed
                listed_n[1] += int(fr.n_inst)
            sloss(fr.out_img.view(1024, 1024, 3), v.target, 0.8, 0.2, d_img, ssums)
            srz.backward(fr, d_img, None, sgrads, accumulate=True)
    torch.cuda.synchronize()
    stage_timer.rz = srz
    listed = listed_n[0] / max(listed_n[1], 1)
    peak_hbm, _ = peaks()
    stages = {}
    for name, rec in stage_timer.summary().items():
        byts = [stage_bytes(name, trainer.n, nk, ni, 1024 * 1024, listed) for nk, ni in rec["counts"]]
        st = {"avg_ms": rec["avg_ms"], "calls": rec["launches"]}
        if byts and byts[0] is not None:
            gbs = sum(byts) / len(byts) / (rec["avg_ms"] / 1000.0) / 1e9
            st.update(algorithmic_gb_s=gbs, hbm_frac=gbs / peak_hbm)
        stages[name] = st
    del srz, sloss, sgrads

    # ---- forward render throughput over the same views (the render pipeline's stream lanes)
    from paper_2504_13339_b200.device import RenderPipeline

    pipe = RenderPipeline(lanes=args.lanes, cull=not args.no_cull)
    items = [(v.camera, dtf) for v in views]
    for _ in range(2):
        pipe.render(trainer.params, trainer.n, items)
    barrier()
    torch.cuda.synchronize()
    r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    r0.record()
    for _ in range(args.render_frames):
        pipe.render(trainer.params, trainer.n, items)
    r1.record()
    torch.cuda.synchronize()
    barrier()
    rms = max_over_ranks(r0.elapsed_time(r1))
    px = args.render_frames * VIEWS_PER_STEP * 1024 * 1024
    render_mpx_s = px / (rms / 1000.0) / 1e6
    # kernel-timing pass of the render (events on each lane's stream), for its roofline
    rtimer = KernelTimer(None)
    for _, rz in pipe.lanes:
        rz.timer = rtimer
    pipe.render(trainer.params, trainer.n, items)
    torch.cuda.synchronize()
    for _, rz in pipe.lanes:
        rz.timer = None
    render_roof = composite_roofline(rtimer.summary(), 1024 * 1024, "vegs_composite_forward", listed=listed)
    del pipe

    # ---- end to end through the public API with host buffers: the views carry their
    # targets in pinned host memory; the trainer uploads them (overlapped with compute)
    # inside the timed region and the loss is read back every step
    h2d = sum(t.numel() * t.element_size() for t in host_targets)
    host_views = [View(v.camera, v.tf, t) for v, t in zip(views, host_targets)]
    trainer.step(host_views, total_views=VIEWS_PER_STEP).item()  # warm the upload path
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(args.steps):
        lv = trainer.step(host_views, total_views=VIEWS_PER_STEP).item()  # D2H of the loss
    s1.record()
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    barrier()
    e2e_ms = max_over_ranks(max(s0.elapsed_time(s1), wall * 1000.0)) / args.steps
    e2e = {"value": 1000.0 / e2e_ms, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 8,
           "ms_per_step": e2e_ms}

    # ---- the reference-shaped numpy API (the drop-in a vegsplat training loop calls,
    # train.py:469-483): render_with_state -> compute_loss -> rasterize_backward per view,
    # mean gradient, adam_step; every array crosses PCIe as numpy.  Timed on rank 0's
    # first views (host wall clock with a device sync), extrapolated to the 16-view step.
    api = None
    if rank == 0 and not args.no_api:
        api = run_api_path(learned, tf, [cams[i] for i in mine], [t.numpy() for t in host_targets], args.api_views)
    torch.cuda.empty_cache()

    # the config-3 sweep and the config-4 run have their own barriers / max-over-ranks:
    # every rank takes part
    sweep = None if args.no_sweep else run_sweep(args, dev, rank, world)
    del trainer, views, targets
    torch.cuda.empty_cache()
    c4 = None if args.no_c4 else run_c4(args, dev, rank, world)

    if rank != 0:
        dist.destroy_process_group() if world > 1 else None
        return

    # ---- roofline of the dominant kernel (largest share of the step)
    peak, peak_kind = peaks()
    dom = max(ksum, key=lambda k: ksum[k]["total_ms"]) if ksum else None
    roof = None
    if dom:
        rec = ksum[dom]
        byts = [algorithmic_bytes(dom, nk, ni, 1024 * 1024, listed=listed) for nk, ni in rec["counts"]]
        avg_bytes = sum(byts) / len(byts)
        achieved = avg_bytes / (rec["avg_ms"] / 1000.0) / 1e9
        traffic, issue = None, None
        prof = ROOT / "profiles" / "ncu_composite.json"
        if prof.exists():
            rec_ncu = json.loads(prof.read_text()).get(dom)
            if rec_ncu:
                traffic = rec_ncu["dram_bytes"]
                # the bound that actually applies: warp-instruction issue (4 schedulers per SM)
                props = torch.cuda.get_device_properties(dev)
                mhz = MAX_SM_MHZ
                try:
                    mhz = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["sm_max_mhz"])
                except Exception:
                    pass
                peak_issue = props.multi_processor_count * 4 * mhz * 1e6
                achieved_issue = rec_ncu["warp_instructions"] / (rec["avg_ms"] / 1000.0)
                issue = {"bound": "issue", "achieved": achieved_issue, "peak": peak_issue,
                         "unit": "warp-instructions/s", "frac": achieved_issue / peak_issue,
                         "warp_instructions_per_launch": rec_ncu["warp_instructions"],
                         "peak_source": f"{props.multi_processor_count} SMs x 4 schedulers x {mhz:.0f} MHz",
                         "source": "profiles/ncu_composite.json (instruction count) / live CUDA-event duration"}
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "peak_source": peak_kind,
                "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                "algorithmic_bytes_per_launch": avg_bytes, "avg_launch_ms": rec["avg_ms"],
                "listed_fraction": listed,
                "share_of_step": rec["total_ms"] / ktimed_ms,
                "timing": f"CUDA events on the launching lane stream over a separate {k_steps}-step pass "
                          "identical to the timed region",
                "note": "compositing is CUDA-core instruction-issue bound, not HBM bound (SURVEY §8(d)); "
                        "see issue_roofline", "issue_roofline": issue}
    kernels = {k: {"avg_ms": v["avg_ms"], "launches": v["launches"], "share_of_step": v["total_ms"] / ktimed_ms,
                   "avg_instances": sum(c[1] for c in v["counts"]) / len(v["counts"])}
               for k, v in ksum.items()}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(learned, tf, [cams[i] for i in mine], [t.numpy() for t in host_targets],
                                  args.cpu_budget_s)

    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32+f64", "data": "synthetic (seeded, scenes.py)",
            "config": config_block(world, args.backend, not args.no_graphs, args.grad_payload, args.grad_buckets),
            "e2e": e2e, "render_mpx_s": render_mpx_s,
            "render_roofline": render_roof, "loss": loss_val,
            "gpu_launches": int(launches), "roofline": roof, "kernels": kernels, "stages": stages,
            "render_sweep_c3": sweep,
            "api_path_c2": api,
            "train_densify_c4": c4,
            "cpu_baseline": cpu,
            "clocks": clk}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_api_path(learned, tf, cams, targets, n_views: int) -> dict:
    import torch

    from paper_2504_13339_b200 import raster as R
    from paper_2504_13339_b200.loss import compute_loss
    from paper_2504_13339_b200.train import OptimizerState, TrainConfig, adam_step

    cfg = TrainConfig(iterations=30000)

    class LossCfg:
        lambda_ssim = 0.2
        normal_loss_weight = 0.0
        smooth_loss_weight = 0.0

    gs = learned.select(np.arange(len(learned)))  # a private copy: adam_step updates it in place
    opt = OptimizerState.for_set(gs)

    def one_view(i):
        img, st = R.render_with_state(gs, tf, cams[i], (1.0, 1.0, 1.0), with_aux=False, dtype=np.float32)
        _, ig, _ = compute_loss(img, targets[i], LossCfg())
        return R.rasterize_backward(st, ig)

    one_view(0)  # warm-up (allocations)
    torch.cuda.synchronize()
    n = min(n_views, len(cams))
    view_s, acc = [], None
    for i in range(n):
        t0 = time.perf_counter()
        g = one_view(i)
        if acc is None:
            acc = g
        else:
            for k, a in g.arrays().items():
                getattr(acc, k)[...] += a
        torch.cuda.synchronize()
        view_s.append(time.perf_counter() - t0)
    for k, a in acc.arrays().items():
        a /= n
    t0 = time.perf_counter()
    adam_step(gs, acc, opt, cfg, 1)
    torch.cuda.synchronize()
    adam_s = time.perf_counter() - t0
    step_s = VIEWS_PER_STEP * statistics.mean(view_s) + adam_s
    return {"workload": "c2 through the numpy drop-in API (raster.render_with_state f32 + loss.compute_loss + "
                        "raster.rasterize_backward per view, train.adam_step), host wall clock",
            "steps_per_s": 1.0 / step_s, "ms_per_view": 1000.0 * statistics.mean(view_s),
            "adam_ms": 1000.0 * adam_s, "views_timed": n,
            "note": f"extrapolated x{VIEWS_PER_STEP}/{n}; params, gradients and Adam moments cross PCIe as float64 "
                    "numpy every call (~0.6 GB per Adam step), which the device-resident Trainer avoids"}


def run_sweep(args, dev, rank, world) -> dict:
    """Config 3: 3M Gaussians (64-blob shape), 1920x1080, 8 fresh TFs per frame, forward
    only; frames are sharded across ranks (replicas, no collective)."""
    import torch
    import torch.distributed as dist

    from paper_2504_13339_b200 import scenes
    from paper_2504_13339_b200.device import DeviceTF, Rasterizer

    gs = scenes.blob_gaussians(3_000_000, seed=1)
    params = torch.from_numpy(gs.pack()).to(dev)
    n_frames = max(args.sweep_frames, 1) * world
    cams = scenes.orbit_cameras(n_frames, 5, 1920, 1080)
    mine = [f for f in range(n_frames) if f % world == rank]
    tfs = {f: [DeviceTF(scenes.random_tf(1000 + 8 * f + k), dev) for k in range(8)] for f in mine}
    from paper_2504_13339_b200.device import RenderPipeline

    pipe = RenderPipeline(lanes=args.lanes, cull=not args.no_cull, project_once=not args.no_shared_projection)
    items = [(cams[f], tf) for f in mine for tf in tfs[f]]
    # warm-up over every (frame, TF): the scratch pools grow to the largest instance count
    # here, so no allocation happens inside the timed region
    pipe.render(params, len(gs), items)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    reps = 3
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        inst = pipe.render(params, len(gs), items)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    renders = 8 * n_frames
    stimer = KernelTimer(None)
    for _, rz in pipe.lanes:
        rz.timer = stimer
    listed = []
    pipe.render(params, len(gs), items, on_frame=lambda i, fr: listed.append((fr.tile_end[-1].clone(), fr.n_inst)))
    torch.cuda.synchronize()
    for _, rz in pipe.lanes:
        rz.timer = None
    lf = sum(int(t) for t, _ in listed) / max(sum(n for _, n in listed), 1)
    roof = composite_roofline(stimer.summary(), 1920 * 1080, "vegs_composite_forward_c3", listed=lf)
    return {"workload": "c3: 3M blob-shaped Gaussians, 1920x1080, 8 random 256-knot TFs per frame (1-6 bumps), "
                        "forward render per (frame, TF), frames sharded across ranks",
            "renders": renders, "ms_per_render": ms / (renders / world), "mpx_s": renders * 1920 * 1080 / (ms / 1e3) / 1e6,
            "tf_frames_per_s": renders / (ms / 1e3), "avg_instances": inst / max(len(mine) * 8, 1),
            "roofline": roof}


def run_c4(args, dev, rank, world) -> dict:
    """Config 4: 200k learned Gaussians fit to renders of a 2M-Gaussian 64-blob set, 64 views
    per step at 800x800 sharded across ranks, each step with the next of 16 TFs over disjoint
    scalar ranges, densify/prune every 100 steps (clone/split/prune with optimizer-row edits,
    on the device).  A bounded sample: `c4_steps` timed steps, then one densify/prune; the
    amortised rate charges 1/100 of the densify per step."""
    import torch
    import torch.distributed as dist

    from paper_2504_13339_b200 import scenes
    from paper_2504_13339_b200.device import DeviceTF, Rasterizer
    from paper_2504_13339_b200.parallel import shard_views
    from paper_2504_13339_b200.train import TrainConfig, Trainer, View

    learned, truth, _, cams = scenes.config_scene("c4")
    n_tf, steps = 16, max(args.c4_steps, 1)
    tfs = [DeviceTF(scenes.range_tf(500 + k, k / n_tf, (k + 1) / n_tf), dev) for k in range(n_tf)]
    mine = shard_views(len(cams), rank, world)
    used = [(s % n_tf) for s in range(steps + 1)]
    rz = Rasterizer(pooled=True)
    gt = torch.from_numpy(truth.pack()).to(dev)
    targets = {}
    for k in sorted(set(used)):
        for i in mine:
            fr = rz.forward(gt, len(truth), tfs[k], cams[i])
            targets[(k, i)] = fr.out_img.view(cams[i].height, cams[i].width, 3).clone()
    del rz, gt
    group = dist.group.WORLD if world > 1 else None
    tr = Trainer(learned, TrainConfig(iterations=30000), group=group, graphs=not args.no_graphs, lanes=args.c4_lanes,
                 grad_payload=args.grad_payload, grad_buckets=args.grad_buckets, cull=not args.no_cull)
    tr.track_densify(True)
    view_sets = {k: [View(cams[i], tfs[k], targets[(k, i)]) for i in mine] for k in sorted(set(used))}

    def views_for(s):
        return view_sets[used[s]]

    for _ in range(2):  # warm-up: every TF's view set twice (capacities settle, then graphs are captured)
        for k in sorted(set(used)):
            tr.step(view_sets[k], total_views=len(cams))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    for s in range(steps):
        tr.step(views_for(s + 1), total_views=len(cams))
    e1.record()
    n_before = tr.n
    # BASELINE config 4's rule: prune on the max opacity over the 16 training TFs (< 0.005),
    # densification capped at 3M Gaussians
    n_after = tr.densify_and_prune(scene_extent=1.0, rng=np.random.default_rng(7), position_lr=1.6e-4,
                                   prune_tfs=tfs, max_gaussians=3_000_000)
    e2.record()
    torch.cuda.synchronize()
    step_ms, dens_ms = e0.elapsed_time(e1) / steps, e1.elapsed_time(e2)
    if world > 1:
        t = torch.tensor([step_ms, dens_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms, dens_ms = (float(x) for x in t.tolist())
    return {"workload": "c4: 200k learned Gaussians, targets from a 2M-Gaussian 64-blob set, 64 views/step at "
                        "800x800 sharded across ranks, 16 TFs over disjoint scalar ranges cycled per step, "
                        "densify/prune every 100 steps (amortised; clone/split on view-space gradient > 2e-4, "
                        "prune on max TF opacity < 0.005 over the 16 TFs, capped at 3M)",
            "steps_per_s": 1000.0 / step_ms, "ms_per_step": step_ms, "densify_ms": dens_ms,
            "steps_per_s_amortised": 1000.0 / (step_ms + dens_ms / 100.0), "n_before": n_before,
            "n_after": n_after, "timed_steps": steps, "graph_stats": dict(tr.graph_stats), "lanes": len(tr.lanes)}


# -- the CPU arm (oracle restatement of the reference algorithm) -------------------------

def _oracle_view(O, S, learned, tf, cam, target):
    t0 = time.perf_counter()
    img, st = O.render_with_state(learned, tf, cam, (1.0, 1.0, 1.0), S, False, np.float32)
    total, grad, _, _ = O.l1_ssim_loss(img["rgb"], target, 0.2)
    O.rasterize_backward(st, grad)
    return time.perf_counter() - t0


def _oracle_adam(O, n):
    rng = np.random.default_rng(0)
    p = rng.normal(size=19 * n)
    g = rng.normal(size=19 * n)
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    t0 = time.perf_counter()
    O.adam_update(p, g, m, v, 1, 1e-3)
    return time.perf_counter() - t0


def cpu_baseline_sample(learned, tf, cams, targets, budget_s: float, max_views: int = 3) -> dict:
    """The oracle port (C + numpy) on distinct views 0, 1, ... of the step until the
    budget is spent, extrapolated to the 16-view step plus one 1M-Gaussian Adam."""
    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    from oracle import vegs_oracle as O
    from paper_2504_13339_b200.constants import DEFAULT_SETTINGS as S

    O.lib()
    times = []
    t_start = time.perf_counter()
    while len(times) < min(max_views, len(cams)) and (not times or time.perf_counter() - t_start + times[-1] < budget_s):
        v = len(times)
        times.append(_oracle_view(O, S, learned, tf, cams[v], targets[v]))
    t_view = statistics.mean(times)
    t_adam = _oracle_adam(O, len(learned))
    step_s = VIEWS_PER_STEP * t_view + t_adam
    return {"value": 1.0 / step_s, "unit": UNIT, "cores": int(os.environ.get("OMP_NUM_THREADS", "1")),
            "kind": "port", "sample": f"views 0..{len(times) - 1} of a c2 step (render+loss+backward, mean "
                                      f"{t_view:.2f} s/view) x{VIEWS_PER_STEP}/{len(times)} "
                                      f"+ 1M-Gaussian Adam ({t_adam:.2f} s); extrapolated",
            "s_per_step": step_s}


def run_reference(args) -> None:
    """The reference's own CPU implementation (vegsplat: numpy + numba, installed unmodified
    under baseline/_ref) through its public API: per view render_with_state (float32 blend,
    the training dtype) + compute_loss + rasterize_backward, the mean of the per-view
    gradients, then adam_step (train.py:176-195).  A 16-view c2 step takes ~10 min on a
    16-core host, so the views are timed in order until ``--ref-budget-s`` is spent and the
    step is extrapolated from the mean per-view time (``views_timed``, ``extrapolated``)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # the reference is single-process; other ranks exit without work
    ref_dir = ROOT / "baseline" / "_ref"
    if not (ref_dir / "vegsplat").is_dir():
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref/vegsplat not installed (see DESIGN.md §10)"}),
              flush=True)
        return
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="vegs_numba_"))
    sys.path.insert(0, str(ref_dir))
    import numba

    import vegsplat as vs  # the reference, unmodified
    import vegsplat.loss  # noqa: F401
    import vegsplat.raster  # noqa: F401
    import vegsplat.train  # noqa: F401
    vtrain = sys.modules["vegsplat.train"]  # (vegsplat.train is also a function name)
    from paper_2504_13339_b200 import scenes  # seeded numpy input generators only

    def ref_gs(g):
        return vs.model.GaussianSet(**{k: np.array(v, copy=True) for k, v in g.arrays().items()})

    def ref_tf(t):
        return vs.transfer.TransferFunction(color=vs.transfer.ColorMap(t.color.points),
                                            opacity=vs.transfer.OpacityMap(t.opacity.points))

    def ref_cam(c):
        return vs.camera.Camera(position=c.position, target=c.target, up=c.up, fov_y=c.fov_y, width=c.width,
                                height=c.height, near=c.near, far=c.far)

    class LossCfg:  # 0.8 L1 + 0.2 (1 - SSIM), regularisers off (rgb planes), as the b200 arm
        lambda_ssim = 0.2
        normal_loss_weight = 0.0
        smooth_loss_weight = 0.0

    threads = numba.get_num_threads()
    learned, truth, tf, cams = scenes.config_scene(WORKLOAD)
    rgs, rtf = ref_gs(learned), ref_tf(tf)
    cfg = vtrain.TrainConfig(iterations=30000)
    bg = (1.0, 1.0, 1.0)

    # JIT warm-up on a config-0-sized scene (numba compiles each kernel once per dtype)
    t0 = time.perf_counter()
    w_gs, _, w_tf, w_cams = scenes.config_scene("c0")
    wg, wt, wc = ref_gs(w_gs), ref_tf(w_tf), ref_cam(w_cams[0])
    img, st = vs.raster.render_with_state(wg, wt, wc, bg, with_aux=False, dtype=np.float32)
    _, ig, _ = vs.loss.compute_loss(img, img.rgb, LossCfg())
    g = vs.raster.rasterize_backward(st, ig)
    vtrain.adam_step(wg, g, vtrain.OptimizerState.for_set(wg), cfg, 1)
    jit_s = time.perf_counter() - t0

    # targets: the ground-truth set rendered on the host (untimed setup) by the oracle
    # port of the same algorithm (~3x faster than the reference, pinned to it by tests/golden)
    from oracle import vegs_oracle as O
    from paper_2504_13339_b200.constants import DEFAULT_SETTINGS as S

    os.environ.setdefault("OMP_NUM_THREADS", str(os.cpu_count() or 1))
    O.lib()
    acc = None
    view_s = []
    t_budget = time.perf_counter()
    for v in range(VIEWS_PER_STEP):
        if view_s and time.perf_counter() - t_budget > args.ref_budget_s:
            break
        target = O.render_with_state(truth, tf, cams[v], bg, S, False, np.float32)[0]["rgb"]
        t0 = time.perf_counter()
        img, st = vs.raster.render_with_state(rgs, rtf, ref_cam(cams[v]), bg, with_aux=False, dtype=np.float32)
        _, ig, _ = vs.loss.compute_loss(img, target, LossCfg())
        g = vs.raster.rasterize_backward(st, ig)
        if acc is None:
            acc = {k: a.copy() for k, a in g.arrays().items()}
        else:
            for k, a in g.arrays().items():
                acc[k] += a
        view_s.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    mean = vs.raster.GradientSet.zeros(len(rgs))
    for k, a in mean.arrays().items():
        a[...] = acc[k] / VIEWS_PER_STEP
    vtrain.adam_step(rgs, mean, vtrain.OptimizerState.for_set(rgs), cfg, 1)
    adam_s = time.perf_counter() - t0
    k = len(view_s)
    full = k == VIEWS_PER_STEP
    step_s = (sum(view_s) if full else VIEWS_PER_STEP * sum(view_s) / k) + adam_s
    value = 1.0 / step_s
    cores = int(threads)
    sample = (f"{k} of the {VIEWS_PER_STEP} views of one c2 step timed (views 0..{k - 1}: render_with_state f32 + "
              f"compute_loss + rasterize_backward, mean {sum(view_s) / k:.2f} s/view) + adam_step ({adam_s:.2f} s)"
              + ("" if full else f"; step extrapolated x{VIEWS_PER_STEP}/{k}"))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": 1 if full else 0, "warmup": 0, "ms_per_step": step_s * 1000.0, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64 (f32 blend planes)", "data": "synthetic (seeded)",
            "config": config_block(1, graphs=None), "views_timed": k, "extrapolated": not full,
            "view_s": view_s, "adam_s": adam_s, "jit_warmup_s": jit_s,
            "reference": {"package": "vegsplat 0.1.0 (baseline/_ref, unmodified)", "numba": numba.__version__,
                          "numba_threads": threads, "host_cpus": os.cpu_count()},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
