"""Optimisation on the GPU: drop-in Adam / learning rates, and the view-sharded trainer.

Reference: /root/reference/pkg/src/vegsplat/train.py:34-77 (TrainConfig), :120-173
(Adam constants, OptimizerState, learning_rates), :176-195 (adam_step), :200-219
(DensifyStats).  ``adam_step`` keeps the reference's signature and in-place numpy
semantics but runs the fused float64 Adam kernel (``vegs_adam_step``).

``Trainer`` is the B200 training step BASELINE.json measures: parameters, Adam moments
and the flat gradient buffer stay resident in HBM as one float64 class-major buffer
each (19 n values); a step renders, scores and back-propagates each of its views,
sums the per-view gradients scaled by 1/total_views into the buffer, all-reduces it
across ranks (one NCCL all-reduce over NVLink when world_size > 1; views are sharded
across ranks) and applies Adam.  Every rank then holds bit-identical
parameters.
"""

from __future__ import annotations

import math
from dataclasses import asdict, dataclass

import numpy as np
import torch

from .constants import DEFAULT_SETTINGS, RasterSettings
from .device import DeviceTF, Rasterizer, adam_step_device, adam_step_sum_device, require_cuda, use_stream
from .model import PARAM_CLASSES, GaussianSet, class_offsets
from .parallel import GradientExchange, allreduce_gradients

ADAM_BETA1 = 0.9
ADAM_BETA2 = 0.999
ADAM_EPS = 1e-15


class TrainingError(RuntimeError):
    """Non-finite loss or gradient (vegsplat.errors.TrainingError)."""


@dataclass(frozen=True)
class TrainConfig:
    iterations: int = 30000
    lambda_ssim: float = 0.2
    lr_value: float = 0.00025
    lr_weight: float = 0.025
    lr_position: float = 1.6e-4
    lr_position_final: float = 1.6e-6
    lr_scale: float = 5e-3
    lr_rotation: float = 1e-3
    lr_lighting: float = 5e-3
    prune_weight_threshold: float = 0.005
    densify_start: int = 500
    densify_end: int = 20000
    densify_interval: int = 100
    densify_grad_threshold: float = 2e-4
    percent_dense: float = 0.01
    weight_reset_interval: int = 3000
    lr_position_scale_by_extent: bool = False
    normal_loss_weight: float = 0.01
    smooth_loss_weight: float = 0.001
    seed: int = 0
    init_points: int = 30000
    init_mode: str = "volume"
    no_weights: bool = False
    checkpoint_interval: int = 500
    background: tuple[float, float, float] = (1.0, 1.0, 1.0)

    def __post_init__(self):
        for name in ("lr_value", "lr_weight", "lr_position", "lr_scale", "lr_rotation", "lr_lighting"):
            if getattr(self, name) <= 0:
                raise ValueError(f"{name} must be positive")
        if not (0.0 <= self.lambda_ssim <= 1.0):
            raise ValueError("lambda_ssim must lie in [0, 1]")
        if self.iterations > 0 and not (self.densify_start < self.densify_end):
            raise ValueError("need densify_start < densify_end")
        if self.init_mode not in ("volume", "random"):
            raise ValueError(f"unknown init_mode {self.init_mode!r}")

    def to_dict(self) -> dict:
        d = asdict(self)
        d["background"] = list(self.background)
        return d


def learning_rates(config: TrainConfig, iteration: int, scene_extent: float = 1.0) -> dict[str, float]:
    t = min(max(iteration, 0), max(config.iterations, 1)) / max(config.iterations, 1)
    lr_pos = config.lr_position * (config.lr_position_final / config.lr_position) ** t
    if config.lr_position_scale_by_extent:
        lr_pos *= scene_extent
    lr_w = 0.0 if config.no_weights else config.lr_weight
    lit = config.lr_lighting
    return {"position": lr_pos, "log_scale": config.lr_scale, "rotation": config.lr_rotation,
            "raw_value": config.lr_value, "raw_weight": lr_w, "normal": lit, "raw_ka": lit,
            "raw_kd": lit, "raw_ks": lit, "raw_beta": lit}


@dataclass
class OptimizerState:
    m: dict
    v: dict
    step: int = 0

    @staticmethod
    def for_set(gs: GaussianSet) -> "OptimizerState":
        return OptimizerState(m={k: np.zeros_like(getattr(gs, k)) for k in PARAM_CLASSES},
                              v={k: np.zeros_like(getattr(gs, k)) for k in PARAM_CLASSES})


def _lr_tensor(lrs: dict, device) -> torch.Tensor:
    return torch.tensor([lrs[k] for k in PARAM_CLASSES], dtype=torch.float64, device=device)


def adam_step(gs: GaussianSet, grads, state: OptimizerState, config: TrainConfig, iteration: int,
              scene_extent: float = 1.0) -> None:
    """One bias-corrected Adam update of ``gs`` in place (train.py:176-195), on the GPU."""
    dev = require_cuda()
    for name in PARAM_CLASSES:  # same check order and message as the reference
        if not np.all(np.isfinite(getattr(grads, name))):
            raise TrainingError(f"non-finite gradient in parameter class {name!r}")
    n = len(gs)
    lrs = learning_rates(config, iteration, scene_extent)
    state.step += 1

    def flat(d):
        return torch.from_numpy(np.concatenate([np.asarray(d[k], dtype=np.float64).ravel()
                                                for k in PARAM_CLASSES])).to(dev)

    p = torch.from_numpy(gs.pack()).to(dev)
    g = flat({k: getattr(grads, k) for k in PARAM_CLASSES})
    m, v = flat(state.m), flat(state.v)
    bad = torch.zeros(10, dtype=torch.int32, device=dev)
    adam_step_device(p, g, m, v, n, _lr_tensor(lrs, dev), 1.0, state.step, bad)
    for name, (a, b, w) in class_offsets(n).items():
        shape = getattr(gs, name).shape
        getattr(gs, name)[...] = p[a:b].cpu().numpy().reshape(shape)
        state.m[name][...] = m[a:b].cpu().numpy().reshape(shape)
        state.v[name][...] = v[a:b].cpu().numpy().reshape(shape)


@dataclass
class DensifyStats:
    grad_accum: np.ndarray
    pos_accum: np.ndarray
    count: np.ndarray

    @staticmethod
    def zeros(n: int) -> "DensifyStats":
        return DensifyStats(grad_accum=np.zeros(n), pos_accum=np.zeros((n, 3)), count=np.zeros(n))

    def add(self, grads) -> None:
        vis = grads.visible
        self.grad_accum[vis] += grads.viewspace_norm[vis]
        self.pos_accum[vis] += grads.position[vis]
        self.count[vis] += 1.0


# -- the device-resident, view-sharded training step ------------------------------------

@dataclass
class View:
    camera: object
    tf: DeviceTF
    target: torch.Tensor  # (H, W, 3) float32, on the device or in (pinned) host memory


class _Lane:
    """One CUDA stream of the view pipeline with its own scratch (see Trainer)."""

    def __init__(self, tr: "Trainer", stream):
        from .device import LossKernel

        self.stream = stream
        self.rz = Rasterizer(tr.settings, 11 if tr.with_aux else 3, store_f64=False, pooled=True, fast_t=tr.fast_t,
                             cull=tr.cull)
        self.rz.contrib_counts = False  # nobody reads them in training
        self.loss = LossKernel(tr.device)
        self.loss_launches = 0
        self.d_img = None
        self.grads = None
        self.dstats = None
        self.dstats_saved = None  # device-count steps: dstats before the step (restored on overflow)

    def prepare(self, tr: "Trainer") -> None:
        if self.grads is None or self.grads.numel() != tr.params.numel():
            self.grads = torch.zeros_like(tr.params)
        if tr.densify_stats is None:
            self.dstats = None
        elif self.dstats is None or self.dstats.numel() != tr.densify_stats.numel():
            self.dstats = torch.zeros_like(tr.densify_stats)



class Trainer:
    """Multi-view training step on device-resident float64 parameters.

    ``group``: a torch.distributed process group (NCCL) when views are sharded across
    GPUs; the gradient buffer is all-reduced once per step."""

    def __init__(self, gs: GaussianSet, config: TrainConfig, settings: RasterSettings = DEFAULT_SETTINGS,
                 background=(1.0, 1.0, 1.0), l1_weight: float | None = None, group=None, with_aux: bool = False,
                 lanes: int = 4, fast_t: bool = False, graphs: bool = False, grad_payload: str = "f64",
                 grad_buckets: int = 4, cull: bool = True):
        self.device = require_cuda()
        # cull: bin each view on the tight ellipse boxes (Rasterizer._culls): shorter tile lists,
        # the same images, losses and gradients
        self.cull = cull
        # fast_t: the forward carries T in float32 with every skip / clamp / termination
        # decision exact (vegs_composite_forward_fast).  Default: the float64 chain, which
        # also reproduces T bit for bit and measured as fast (A/B)
        self.fast_t = fast_t
        self.n = len(gs)
        self.config = config
        self.settings = settings
        self.background = tuple(float(x) for x in background)
        self.lam = float(config.lambda_ssim)
        self.w_l1 = (1.0 - self.lam) if l1_weight is None else float(l1_weight)
        self.params = torch.from_numpy(gs.pack()).to(self.device)
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.grads = torch.zeros_like(self.params)
        self.nonfinite = torch.zeros(10, dtype=torch.int32, device=self.device)
        self.step_count = 0
        # with_aux: blend the 11 planes (rgb, depth, normal, attrs) and apply the normal /
        # smoothness regularisers, as the reference's loop does (train.py:476-479)
        self.with_aux = with_aux
        self.group = group
        # with a process group: the bucketed, pipelined gradient exchange (parallel.py)
        self.exchange = (GradientExchange(self.n, self.device, group, grad_payload, grad_buckets)
                         if group is not None else None)
        self.densify_stats = None  # (n, 5) float64 when densification is tracked
        # Views are pipelined over `lanes` CUDA streams, each with its own scratch pool,
        # loss workspace and gradient buffer: one view's preprocess, count readback and
        # sort overlap the previous view's compositing.  Lane 0 runs on the caller's stream.
        self.lanes = [_Lane(self, torch.cuda.current_stream(self.device) if i == 0 else torch.cuda.Stream(self.device))
                      for i in range(max(1, lanes))]
        self.lanes[0].grads = self.grads
        self.rz = self.lanes[0].rz
        # host-resident targets are uploaded on their own stream, one event per view, so
        # the H2D copies overlap the previous views' compositing
        self._copy_stream = None
        self._target_bufs: list[torch.Tensor] = []
        # Adam's per-step constants: pinned host buffer -> device buffer on every step
        self._hyper_host = torch.zeros(12, dtype=torch.float64, pin_memory=True)
        self._hyper_dev = torch.zeros(12, dtype=torch.float64, device=self.device)
        # graphs=True: device-count binning + one CUDA graph per set of views (see step)
        self._graphs: dict = {}
        self._graph_pool = None
        self._replayed_launches = 0
        self._update_launches = 0  # lane sums, exchange and Adam launches
        self.graph_stats = {"captures": 0, "replays": 0, "redos": 0}
        # [overflow, max instances, max kept splats] of the views of the current step
        self._state = torch.zeros(3, dtype=torch.int64, device=self.device)
        self._state_host = torch.zeros(3, dtype=torch.int64, pin_memory=True)
        self._state_event = torch.cuda.Event()
        self.set_graphs(graphs)

    def set_graphs(self, on: bool) -> None:
        """Switch between device-count steps captured as CUDA graphs (on) and host-counted
        eager steps (off: per-view instance counts on the host, e.g. for per-kernel events)."""
        self.graphs = on
        if on and self._graph_pool is None:
            self._graph_pool = torch.cuda.graph_pool_handle()
        if on and self.lanes[0].stream == torch.cuda.default_stream(self.device):
            # the legacy default stream cannot join a captured graph: lane 0 gets its own
            self.lanes[0].stream = torch.cuda.Stream(self.device)
        for lane in self.lanes:
            lane.rz.device_counts = self._state if on else None

    def set_timer(self, timer) -> None:
        for lane in self.lanes:
            lane.rz.timer = timer
            lane.loss.timer = timer

    @property
    def launches(self) -> int:
        """Kernels launched by this trainer's steps (graph replays count their captured kernels)."""
        return (sum(lane.rz.launches + lane.loss_launches for lane in self.lanes) + self._replayed_launches
                + self._update_launches)

    def gaussians(self) -> GaussianSet:
        return GaussianSet.unpack(self.params.cpu().numpy(), self.n)

    def _upload_targets(self, views: list[View], main) -> list:
        """Queue the H2D copies of host-resident targets on the copy stream; returns per
        view (device target, event or None)."""
        out = []
        if all(v.target.is_cuda for v in views):
            return [(v.target, None) for v in views]
        if self._copy_stream is None:
            self._copy_stream = torch.cuda.Stream(self.device)
        cs = self._copy_stream
        cs.wait_stream(main)  # the previous step's readers of the buffers are done
        while len(self._target_bufs) < len(views):
            self._target_bufs.append(torch.empty(0, dtype=torch.float32, device=self.device))
        for i, v in enumerate(views):
            if v.target.is_cuda:
                out.append((v.target, None))
                continue
            buf = self._target_bufs[i]
            if buf.shape != v.target.shape:
                buf = self._target_bufs[i] = torch.empty(v.target.shape, dtype=v.target.dtype, device=self.device)
            ev = torch.cuda.Event()
            with torch.cuda.stream(cs):
                buf.copy_(v.target, non_blocking=True)
                ev.record(cs)
            out.append((buf, ev))
        return out

    def _loss_and_backward(self, lane, fr, view: View, scale: float, first: bool, sums: torch.Tensor,
                           target: torch.Tensor | None = None, ready=None) -> None:
        h, w = fr.height, fr.width
        img = fr.out_img.view(h, w, fr.n_ch)
        if lane.d_img is None or lane.d_img.numel() != img.numel():
            lane.d_img = torch.empty_like(img)
        target = view.target if target is None else target
        if target.dtype != torch.float32 or tuple(target.shape) != (h, w, 3) or not target.is_contiguous():
            raise ValueError(f"view target must be a contiguous ({h}, {w}, 3) float32 tensor, got "
                             f"{tuple(target.shape)} {target.dtype}{'' if target.is_contiguous() else ' (strided)'}")
        if ready is not None:
            lane.stream.wait_event(ready)
        lane.loss(img, target, self.w_l1, self.lam, lane.d_img, sums[:2])
        lane.loss_launches += 2
        if self.with_aux:
            cam = view.camera
            px_scale = 2.0 * math.tan(0.5 * cam.fov_y) / cam.height
            lane.loss.aux(img, fr.out_t.view(h, w), target, px_scale, self.config.normal_loss_weight,
                          self.config.smooth_loss_weight, lane.d_img, sums[2:5])
            lane.loss_launches += 3
        lane.rz.backward(fr, lane.d_img, None, lane.grads, scale=scale, accumulate=not first,
                         densify_stats=lane.dstats)

    def step(self, views: list[View], total_views: int | None = None, iteration: int | None = None,
             scene_extent: float = 1.0) -> torch.Tensor:
        """One optimisation step over this rank's views; returns the mean loss over
        this rank's views as a device scalar.

        Default (``graphs=False``): views are enqueued with one host read of each view's
        instance count (it sizes the view's buffers).  ``graphs=True``: the counts stay on the
        device (capacity-sized buffers, ``vegs_bin_count_dev``), so a whole step -- every view
        on every lane, the lane sum, the all-reduce, Adam -- is captured once per set of views
        as a CUDA graph and replayed; the host waits once per step, for the overflow check."""
        total = total_views if total_views is not None else len(views)
        self.step_count += 1
        it = self.step_count if iteration is None else iteration
        lrs = learning_rates(self.config, it, scene_extent)
        if self.graphs:
            return self._step_device(views, total, lrs)
        hyper = self._hyper(lrs)
        return self._step_body(views, total, hyper, None)

    def _hyper(self, lrs: dict) -> torch.Tensor:
        """[lr per class (10), 1 - beta1^t, 1 - beta2^t] in the pinned host buffer, copied to
        the device on the current stream (a graph copies it at replay time)."""
        t = self.step_count
        hh = self._hyper_host
        hh[:10] = torch.tensor([lrs[k] for k in PARAM_CLASSES], dtype=torch.float64)
        hh[10] = 1.0 - ADAM_BETA1 ** t
        hh[11] = 1.0 - ADAM_BETA2 ** t
        return self._hyper_dev

    def _step_body(self, views: list[View], total: int, hyper: torch.Tensor, state) -> torch.Tensor:
        main = torch.cuda.current_stream(self.device)
        self._hyper_dev.copy_(self._hyper_host, non_blocking=True)
        if state is not None:
            state.zero_()
        n_v = len(views)
        sums = torch.zeros(n_v, 5, dtype=torch.float64, device=self.device)
        lanes = self.lanes
        for lane in lanes[1:]:
            lane.prepare(self)
            lane.stream.wait_stream(main)  # parameters updated, sums zeroed
        if lanes[0].stream != main:  # called on another stream than the Trainer was built on
            lanes[0].stream.wait_stream(main)
        lanes[0].grads = self.grads
        lanes[0].dstats = self.densify_stats
        if state is not None and self.densify_stats is not None:  # restored if the step overflows
            for lane in lanes:
                if lane.dstats is not None:
                    if lane.dstats_saved is None or lane.dstats_saved.numel() != lane.dstats.numel():
                        lane.dstats_saved = torch.empty_like(lane.dstats)
                    lane.dstats_saved.copy_(lane.dstats)
        targets = self._upload_targets(views, main)
        pend: list = [None] * n_v
        used = [False] * len(lanes)

        def begin(i: int) -> None:
            lane = lanes[i % len(lanes)]
            with use_stream(lane.stream):
                pend[i] = lane.rz.forward_begin(self.params, self.n, views[i].tf, views[i].camera, self.background)

        # With one lane, view i+1 would reuse view i's pooled splat table before view i is
        # sorted and composited: queue it only after view i's backward is enqueued.
        ahead = len(lanes) > 1
        if n_v:
            begin(0)
        for i in range(n_v):
            if ahead and i + 1 < n_v:
                begin(i + 1)  # queue the next view's preprocess before waiting on this one's count
            k = i % len(lanes)
            lane = lanes[k]
            with use_stream(lane.stream):
                fr = lane.rz.forward_end(pend[i])
                pend[i] = None
                self._loss_and_backward(lane, fr, views[i], 1.0 / total, not used[k], sums[i], *targets[i])
            used[k] = True
            if not ahead and i + 1 < n_v:
                begin(i + 1)
        if lanes[0].stream != main:
            main.wait_stream(lanes[0].stream)
        if not used[0]:
            self.grads.zero_()
        for lane in lanes[1:]:
            main.wait_stream(lane.stream)
        # the lanes' partial sums are added inside the Adam kernel (fixed lane order), or in
        # a sum-only pass of the same kernel before a cross-rank all-reduce
        extra = [lane.grads for k, lane in enumerate(lanes) if k and used[k]]
        while len(extra) > 3:
            adam_step_device(None, self.grads, None, None, self.n, None, 1.0, 1, None, extra[:3])
            extra = extra[3:]
            self._update_launches += 1
        if self.exchange is not None:  # cross-rank: pack / all-reduce / Adam per bucket
            before = self.exchange.launches
            self.exchange.step(self.params, self.grads, extra, self.m, self.v, hyper, self.nonfinite, skip=state)
            self._update_launches += self.exchange.launches - before
        else:
            adam_step_sum_device(self.params, self.grads, self.m, self.v, self.n, hyper, self.nonfinite, extra,
                                 skip=state)
            self._update_launches += 1
        if state is not None:
            self._state_host.copy_(state, non_blocking=True)
        if not views:
            return torch.zeros((), dtype=torch.float64, device=self.device)
        # per-view normalisers (views may differ in resolution): element count, valid SSIM
        # windows, smoothness pairs (loss.py:146-168, :212-240)
        hw = [(int(v.camera.height), int(v.camera.width)) for v in views]
        if all(x == hw[0] for x in hw):
            (h, w), norm = hw[0], None
        else:
            norm = torch.tensor([[h * w * 3, (h - 10) * (w - 10) * 3, 4 * (h * (w - 1) + (h - 1) * w)]
                                 for h, w in hw], dtype=torch.float64).to(self.device, non_blocking=True)
        n_el = h * w * 3 if norm is None else norm[:, 0]
        n_pos = (h - 10) * (w - 10) * 3 if norm is None else norm[:, 1]
        n_pair = 4 * (h * (w - 1) + (h - 1) * w) if norm is None else norm[:, 2]
        per_view = self.w_l1 * sums[:, 0] / n_el + self.lam * (1.0 - sums[:, 1] / n_pos)
        if self.with_aux:
            cnt = sums[:, 3]
            per_view = per_view + torch.where(cnt > 0, self.config.normal_loss_weight * sums[:, 2] / cnt.clamp(min=1),
                                              torch.zeros_like(cnt))
            per_view = per_view + self.config.smooth_loss_weight * sums[:, 4] / n_pair
        return per_view.mean()

    def _graph_key(self, views: list[View], total: int):
        return (tuple((id(v.camera), id(v.tf), id(v.target)) for v in views), total, self.n,
                self.densify_stats is not None, torch.cuda.current_stream(self.device).cuda_stream)

    def _step_device(self, views: list[View], total: int, lrs: dict) -> torch.Tensor:
        """Device-count step: replay the captured graph of these views (capture it after the
        first eager run), then one host wait for the step state; a view that overflowed its
        instance capacity left the parameters untouched (Adam skipped), so the buffers grow
        and the step is redone."""
        self._hyper(lrs)
        key = self._graph_key(views, total)
        uniform = len({(int(v.camera.height), int(v.camera.width)) for v in views}) <= 1
        for _ in range(8):
            entry = self._graphs.get(key)
            if entry is not None:
                entry[0].replay()
                loss = entry[1]
                self._replayed_launches += entry[2]
                self.graph_stats["replays"] += 1
            else:
                loss = self._step_body(views, total, self._hyper_dev, self._state)
            self._state_event.record(torch.cuda.current_stream(self.device))
            self._state_event.synchronize()
            if not int(self._state_host[0]):
                # (with a process group the steps stay eager: device counts, no per-view sync,
                # but the NCCL all-reduce is not captured -- never exercised on one GPU)
                if entry is None and uniform and views and self.group is None:
                    self._capture(key, views, total)
                return loss
            # overflow: grow every lane's capacity to the largest view seen, forget the graphs
            # (their buffers are the old size), restore the densify statistics, redo the step
            self.graph_stats["redos"] += 1
            cap = int(int(self._state_host[1]) * 1.25) + 4096
            kcap = int(int(self._state_host[2]) * 1.25) + 1024
            for lane in self.lanes:
                lane.rz.inst_cap = max(lane.rz.inst_cap, cap)
                lane.rz.kept_cap = max(lane.rz.kept_cap, kcap)
                if self.densify_stats is not None and lane.dstats is not None:
                    lane.dstats.copy_(lane.dstats_saved)
            self._graphs.clear()
        raise RuntimeError("instance capacity did not converge")

    def _capture(self, key, views: list[View], total: int) -> None:
        main = torch.cuda.current_stream(self.device)
        cap_stream = torch.cuda.Stream(self.device)
        cap_stream.wait_stream(main)
        g = torch.cuda.CUDAGraph()
        before = self.launches
        with torch.cuda.graph(g, stream=cap_stream, pool=self._graph_pool):
            loss = self._step_body(views, total, self._hyper_dev, self._state)
        main.wait_stream(cap_stream)
        captured = self.launches - before
        self._replayed_launches -= captured  # the capture itself launched nothing; replays count them
        self._graphs[key] = (g, loss, captured)
        self.graph_stats["captures"] += 1

    def track_densify(self, on: bool = True) -> None:
        """Accumulate DensifyStats (per view, fused into the backward) from now on."""
        self.densify_stats = torch.zeros(self.n * 5, dtype=torch.float64, device=self.device) if on else None

    def gather_densify_stats(self) -> torch.Tensor:
        """Fold every lane's DensifyStats into ``densify_stats`` (n x 5) and return it."""
        main = torch.cuda.current_stream()
        for lane in self.lanes[1:]:
            main.wait_stream(lane.stream)
            if lane.dstats is not None and lane.dstats.numel() == self.densify_stats.numel():
                self.densify_stats.add_(lane.dstats)
                lane.dstats.zero_()
        return self.densify_stats

    def densify_and_prune(self, scene_extent: float, rng: np.random.Generator, position_lr: float,
                          prune_tfs=None, max_gaussians: int | None = None) -> int:
        """Device densify/prune of the resident set; the step's buffers are resized and
        the densification statistics reset.  With world_size > 1 the statistics are
        all-reduced first so every replica makes the same decision.  Returns the new n.

        ``prune_tfs`` (DeviceTFs) / ``max_gaussians``: BASELINE config 4's rule -- prune on
        the max opacity over these TFs instead of the activated weight, and cap the count
        (see ``densify_device``).  Defaults: the reference's rule, no cap."""
        if self.densify_stats is None:
            raise RuntimeError("call track_densify() before training steps to collect statistics")
        self.gather_densify_stats()
        allreduce_gradients(self.densify_stats, self.group)
        mo = tf_max_opacity(self.params, self.n, prune_tfs) if prune_tfs else None
        p, m, v, n_out = densify_device(self.params, self.m, self.v, self.n, self.densify_stats, self.config,
                                        scene_extent, rng, position_lr, mo, max_gaussians)
        self.params, self.m, self.v, self.n = p.clone(), m.clone(), v.clone(), n_out
        self._graphs.clear()  # captured with the old buffers
        self.grads = torch.zeros_like(self.params)
        self.densify_stats = torch.zeros(self.n * 5, dtype=torch.float64, device=self.device)
        if self.exchange is not None:
            ex = self.exchange
            self.exchange = GradientExchange(self.n, self.device, self.group, ex.payload, len(ex.bounds))
        return n_out

    def reset_weights(self) -> None:
        from .model import class_offsets, logit

        a, b, _ = class_offsets(self.n)["raw_weight"]
        self.params[a:b].clamp_(max=float(logit(WEIGHT_RESET_VALUE)))
        self.m[a:b].zero_()
        self.v[a:b].zero_()

    def check_finite(self) -> None:
        bad = self.nonfinite.cpu().numpy()
        if bad.any():
            raise TrainingError(f"non-finite gradient in parameter class {PARAM_CLASSES[int(np.argmax(bad))]!r}")


# -- densification (train.py:200-284) on the device --------------------------------------

SPLIT_SCALE_FACTOR = 1.6
WEIGHT_RESET_VALUE = 0.01


def _densify_struct(config: TrainConfig, scene_extent: float, position_lr: float, prune_opacity=None):
    from ._lib import VegsDensify

    return VegsDensify(config.densify_grad_threshold, config.percent_dense, float(scene_extent),
                       config.prune_weight_threshold, float(position_lr), math.log(SPLIT_SCALE_FACTOR),
                       int(config.no_weights), 0, None if prune_opacity is None else prune_opacity.data_ptr())


def tf_max_opacity(params: torch.Tensor, n: int, tfs) -> torch.Tensor:
    """Per-Gaussian max over ``tfs`` (DeviceTF) of the opacity map at sigmoid(raw_value):
    BASELINE config 4's prune criterion (vegs_tf_max_opacity, one launch per TF)."""
    import ctypes

    from . import _lib
    from .device import _p, _stream

    if not tfs:
        raise ValueError("need at least one transfer function")
    out = torch.empty(max(n, 1), dtype=torch.float64, device=params.device)
    for k, tf in enumerate(tfs):
        _lib.call("vegs_tf_max_opacity", _p(params), n, ctypes.byref(tf.struct), int(k == 0), _p(out), _stream())
    return out[:n]


def densify_device(params: torch.Tensor, m: torch.Tensor, v: torch.Tensor, n: int, stats: torch.Tensor,
                   config: TrainConfig, scene_extent: float, rng: np.random.Generator, position_lr: float,
                   prune_opacity: torch.Tensor | None = None, max_gaussians: int | None = None):
    """Clone / split / prune on device buffers; returns (params, m, v, n_out).

    The split offsets are drawn on the host from ``rng`` exactly as the reference does
    (two rounds of ``standard_normal((n_split, 3))``), so a seeded run reproduces it.

    ``prune_opacity`` (n float64, see ``tf_max_opacity``) switches the prune rule from the
    reference's activated weight (train.py:277-280) to BASELINE config 4's "max TF opacity
    < prune_weight_threshold".  ``max_gaussians`` is BASELINE config 4's cap: when clones
    and splits would take the set above it, this round densifies nothing (pruning still
    runs), so the set never grows past the cap by densification."""
    import ctypes

    from . import _lib
    from .device import _p, _stream

    dev = params.device
    dp = _densify_struct(config, scene_extent, position_lr, prune_opacity)
    flags = torch.empty(4 * (n + 1), dtype=torch.int32, device=dev)
    offs = torch.empty_like(flags)
    nbytes = _lib.size_query("vegs_densify_count", _p(params), n, _p(stats), ctypes.byref(dp), _p(flags), _p(offs),
                             tail=(_stream(),))
    ws = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=dev)

    def count():
        _lib.call("vegs_densify_count", _p(params), n, _p(stats), ctypes.byref(dp), _p(flags), _p(offs), _p(ws),
                  ctypes.byref(ctypes.c_size_t(nbytes)), _stream())
        return [int(x) for x in offs[4 * n:4 * n + 4].tolist()]

    keep, clone, split, n_split = count()
    if max_gaussians is not None and keep + clone + 2 * split > max_gaussians and clone + split > 0:
        dp.grad_threshold = math.inf  # the cap: no densification this round
        keep, clone, split, n_split = count()
    if n_split:
        eps_h = np.concatenate([rng.standard_normal(size=(n_split, 3)) for _ in range(2)])
    else:
        eps_h = np.zeros((0, 3))
    eps = torch.from_numpy(np.ascontiguousarray(eps_h, dtype=np.float64)).to(dev)
    n_out = keep + clone + 2 * split
    out = [torch.empty(19 * max(n_out, 1), dtype=torch.float64, device=dev) for _ in range(3)]
    _lib.call("vegs_densify_apply", _p(params), _p(m), _p(v), n, _p(stats), ctypes.byref(dp), _p(flags), _p(offs),
              _p(eps), n_out, _p(out[0]), _p(out[1]), _p(out[2]), _stream())
    return out[0][:19 * n_out], out[1][:19 * n_out], out[2][:19 * n_out], n_out


def densify_and_prune(gs: GaussianSet, opt: OptimizerState, stats: DensifyStats, config: TrainConfig,
                      scene_extent: float, rng: np.random.Generator, position_lr: float) -> GaussianSet:
    """Reference-signature densify/prune (train.py:237-284): numpy in/out, GPU compute."""
    dev = require_cuda()
    n = len(gs)

    def flat(d):
        return torch.from_numpy(np.concatenate([np.asarray(d[k], dtype=np.float64).ravel()
                                                for k in PARAM_CLASSES])).to(dev)

    st = torch.from_numpy(np.ascontiguousarray(np.concatenate(
        [stats.grad_accum[:, None], stats.pos_accum, stats.count[:, None]], axis=1), dtype=np.float64)).to(dev)
    p, m, v, n_out = densify_device(torch.from_numpy(gs.pack()).to(dev), flat(opt.m), flat(opt.v), n, st, config,
                                    scene_extent, rng, position_lr)
    out = GaussianSet.unpack(p.cpu().numpy(), n_out)
    mm = GaussianSet.unpack(m.cpu().numpy(), n_out)
    vv = GaussianSet.unpack(v.cpu().numpy(), n_out)
    opt.m = {k: getattr(mm, k) for k in PARAM_CLASSES}
    opt.v = {k: getattr(vv, k) for k in PARAM_CLASSES}
    stats.grad_accum, stats.pos_accum, stats.count = np.zeros(n_out), np.zeros((n_out, 3)), np.zeros(n_out)
    return out


def reset_weights(gs: GaussianSet, opt: OptimizerState) -> None:
    """Cap activated weights and clear their moments (train.py:227-234)."""
    from .model import logit

    cap = float(logit(WEIGHT_RESET_VALUE))
    np.minimum(gs.raw_weight, cap, out=gs.raw_weight)
    opt.m["raw_weight"][:] = 0.0
    opt.v["raw_weight"][:] = 0.0
