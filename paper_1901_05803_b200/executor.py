"""Real execution of a RALP / baseline-PS job on B200s (one process per GPU).

`run_job(job, steps=...)` is the measured counterpart of the reference's
`simulate_run` for one job (pkg/src/ralp/simulator.py:743-770): it lowers the
job's ModelGraph to the C ABI layer table, creates one `ralpb_model` per rank,
maps the peers' exchange arenas over CUDA IPC (handles exchanged with
torch.distributed), runs the steps natively and returns a `JobReport` with the
reference's field names (simulator.py:213-248).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .planner.costmodel import JobSpec, StrategyKind, volume_ralp_multi_ps, volumes_for
from .planner.layers import LayerKind, ModelGraph
from .report import JobReport, StepBreakdown


class ExecutorError(ValueError):
    """The job cannot be executed by this backend (unsupported layer mix etc.)."""


def infer_input_shape(model: ModelGraph) -> tuple[int, int, int]:
    """Per-sample input (h, w, c) of the first layer (a convolution): the smallest input that
    yields its recorded output shape (infer_conv, layers.py:87-103)."""
    first = model.layers[0]
    if first.kind is not LayerKind.CONVOLUTION or first.output_shape is None:
        raise ExecutorError("the first layer must be a derived convolution")
    hp = first.hyperparams
    k, s, p, cout = hp["k"], hp.get("stride", 1), hp.get("pad", 0), hp["cout"]
    cin = (first.param_count - cout) // (k * k * cout)
    o = first.output_shape
    return (o.h - 1) * s + k - 2 * p, (o.w - 1) * s + k - 2 * p, cin


def lower(model: ModelGraph, input_shape: Optional[tuple[int, int, int]] = None) -> list[dict]:
    """ModelGraph -> list of layer dicts (kind, k, stride, pad, h, w, cin, cout, relu)."""
    h, w, c = input_shape or infer_input_shape(model)
    out: list[dict] = []
    n = model.num_layers
    flat = None
    for i, L in enumerate(model.layers):
        hp = L.hyperparams
        last = i == n - 1
        if L.kind is LayerKind.CONVOLUTION:
            d = dict(kind="conv", k=hp["k"], stride=hp.get("stride", 1), pad=hp.get("pad", 0), h=h, w=w, cin=c,
                     cout=hp["cout"], relu=1)
            h, w, c = L.output_shape.h, L.output_shape.w, L.output_shape.c
        elif L.kind is LayerKind.POOLING:
            d = dict(kind="pool", k=hp["window"], stride=hp.get("stride", hp["window"]), pad=hp.get("pad", 0), h=h,
                     w=w, cin=c, cout=c, relu=0)
            if d["pad"]:
                raise ExecutorError(f"layer {L.name}: padded pooling is not implemented")
            h, w, c = L.output_shape.h, L.output_shape.w, L.output_shape.c
        elif L.kind is LayerKind.FULLY_CONNECTED:
            width = flat if flat is not None else (h * w * c if h else c)
            d = dict(kind="fc", k=0, stride=0, pad=0, h=0, w=0, cin=width, cout=hp["out"], relu=0 if last else 1)
            flat = hp["out"]
            h = w = 0
            c = flat
        elif L.kind is LayerKind.FLATTEN:
            continue
        else:
            raise ExecutorError(f"layer {L.name}: kind {L.kind.value} is not executable by this backend")
        d["name"] = L.name
        out.append(d)
    return out


def allgather_bytes(blob: bytes) -> list[bytes]:
    """Rank-ordered all-gather of equal-length byte strings over the initialised
    torch.distributed group (NCCL: via a CUDA tensor; gloo: on the CPU)."""
    import torch
    import torch.distributed as dist

    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    mine = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(dev)
    parts = [torch.empty_like(mine) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, mine)
    return [bytes(p.cpu().numpy().tobytes()) for p in parts]


_KIND = {"conv": _lib.RALPB_CONV, "pool": _lib.RALPB_POOL, "fc": _lib.RALPB_FC}


def _desc_array(layers: Sequence[dict]):
    arr = (_lib.LayerDesc * len(layers))()
    for a, L in zip(arr, layers):
        a.kind, a.k, a.stride, a.pad = _KIND[L["kind"]], L["k"], L["stride"], L["pad"]
        a.h, a.w, a.cin, a.cout, a.relu = L["h"], L["w"], L["cin"], L["cout"], L["relu"]
    return arr


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


@dataclass
class StepResult:
    loss: float
    logical_bytes: int
    physical_bytes: int
    launches: int
    ms_step: float
    ms_front_fwd: float
    ms_back: float
    ms_front_bwd: float
    ms_sync: float
    ms_gemm: float = 0.0
    gemm_launches: int = 0


class RankExecutor:
    """One rank's `ralpb_model`.  Multi-rank use needs torch.distributed initialised
    (any backend) so the IPC handles can be exchanged."""

    def __init__(self, job: JobSpec, *, rank: int = 0, world: Optional[int] = None, ps_rank: int = 0,
                 input_shape: Optional[tuple[int, int, int]] = None, ring_backend: str = "native",
                 fc_sharding: str = "single"):
        """ring_backend (StrategyKind.RING_ALLREDUCE only): "native" = the hand-written
        reduce-scatter + SGD + all-gather over NVLink peer memory inside the step; "nccl" = the
        step stops after the backward, torch.distributed (NCCL) all-reduces the gradient vector
        on the model stream, then the update runs (the comparison baseline).
        fc_sharding (StrategyKind.RALP only): "single" = the reference's single PS on rank 0;
        "multi" = the FC tail's first two layers sharded over every GPU (RALPB_STRATEGY_RALP_MPS,
        SURVEY.md 8f.1; logical bytes volume_ralp_multi_ps)."""
        world = job.worker_count if world is None else world
        if world != job.worker_count:
            raise ExecutorError("one rank per worker: world size must equal worker_count")
        kind = job.strategy.kind
        if ring_backend not in ("native", "nccl"):
            raise ExecutorError(f"unknown ring backend {ring_backend!r}")
        if fc_sharding not in ("single", "multi"):
            raise ExecutorError(f"unknown fc_sharding {fc_sharding!r}")
        self.fc_sharding = fc_sharding if kind is StrategyKind.RALP else "single"
        self.ring_backend = ring_backend if kind is StrategyKind.RING_ALLREDUCE else None
        self.job = job
        self.model = job.model
        self.rank, self.world, self.ps_rank = rank, world, ps_rank
        self.layers = lower(job.model, input_shape)
        self.in_shape = (self.layers[0]["h"], self.layers[0]["w"], self.layers[0]["cin"])
        self.classes = self.layers[-1]["cout"]
        split = job.strategy.split_index if kind is StrategyKind.RALP else 0
        if kind is StrategyKind.RALP:
            strategy = _lib.RALPB_STRATEGY_RALP if self.fc_sharding == "single" else _lib.RALPB_STRATEGY_RALP_MPS
        elif kind is StrategyKind.RING_ALLREDUCE:
            strategy = _lib.RALPB_STRATEGY_RING if ring_backend == "native" else _lib.RALPB_STRATEGY_RING_EXTERNAL
        else:
            strategy = _lib.RALPB_STRATEGY_BASELINE
        self._descs = _desc_array(self.layers)
        h = C.c_void_p()
        _lib.call("ralpb_model_create", C.cast(self._descs, C.c_void_p), len(self.layers), split,
                  job.model.batch_size, strategy, rank, world, ps_rank, job.model.bytes_per_element, C.byref(h))
        self._h = h
        if world > 1:
            self._open_peers()

    def _open_peers(self) -> None:
        buf = (C.c_char * 64)()
        _lib.call("ralpb_model_ipc_handle", self._h, C.cast(buf, C.c_void_p))
        blob = b"".join(allgather_bytes(bytes(buf)))
        arr = (C.c_char * len(blob)).from_buffer_copy(blob)
        _lib.call("ralpb_model_ipc_open", self._h, C.cast(arr, C.c_void_p))
        import torch.distributed as dist
        dist.barrier()

    # ---------------------------------------------------------------- params
    def set_params(self, params: Sequence) -> None:
        for i, p in enumerate(params):
            if p is None:
                continue
            w, b = (np.ascontiguousarray(x, dtype=np.float32) for x in p)
            _lib.call("ralpb_model_set_params", self._h, i, _ptr(w), _ptr(b), 1)

    def get_params(self) -> list:
        out = []
        for i, L in enumerate(self.layers):
            if L["kind"] == "conv":
                w = np.empty((L["cout"], L["k"], L["k"], L["cin"]), dtype=np.float32)
            elif L["kind"] == "fc":
                w = np.empty((L["cout"], L["cin"]), dtype=np.float32)
            else:
                out.append(None)
                continue
            b = np.empty(L["cout"], dtype=np.float32)
            _lib.call("ralpb_model_get_params", self._h, i, _ptr(w), _ptr(b), 1)
            out.append((w, b))
        return out

    # ---------------------------------------------------------------- step
    @property
    def stream(self) -> int:
        return _lib.lib().ralpb_model_stream(self._h)

    def step(self, images, labels, *, lr: float = 0.01, momentum: float = 0.9) -> None:
        """images/labels: numpy host arrays (pinned-ness is the caller's business) or torch
        tensors (host or cuda)."""
        on_host = 1
        if hasattr(images, "data_ptr"):
            ip, lp = images.data_ptr(), labels.data_ptr()
            on_host = 0 if images.is_cuda else 1
        else:
            images = np.ascontiguousarray(images, dtype=np.float32)
            labels = np.ascontiguousarray(labels, dtype=np.int32)
            ip, lp = _ptr(images), _ptr(labels)
        _lib.call("ralpb_model_step", self._h, ip, lp, on_host, float(lr), float(momentum))
        if self.ring_backend == "nccl":
            self._nccl_allreduce_and_apply(float(lr), float(momentum))

    def _grad_tensor(self):
        """The engine's fp32 gradient vector as a zero-copy torch tensor (CUDA array interface)."""
        if getattr(self, "_gtensor", None) is None:
            import torch
            ptr, n = C.c_void_p(), C.c_longlong()
            _lib.call("ralpb_model_grad_buffer", self._h, C.byref(ptr), C.byref(n))

            class _View:
                __cuda_array_interface__ = {"shape": (n.value,), "typestr": "<f4", "data": (ptr.value, False),
                                            "version": 3, "strides": None}
            self._gtensor = torch.as_tensor(_View(), device="cuda")
        return self._gtensor

    def _nccl_allreduce_and_apply(self, lr: float, mu: float) -> None:
        import torch
        import torch.distributed as dist
        g = self._grad_tensor()
        if self.world > 1:
            with torch.cuda.stream(torch.cuda.ExternalStream(self.stream)):
                dist.all_reduce(g)
        _lib.call("ralpb_model_apply", self._h, lr, mu)

    def stats(self) -> StepResult:
        st = _lib.StepStats()
        _lib.call("ralpb_model_stats", self._h, C.byref(st))
        return StepResult(st.loss, st.logical_bytes, st.physical_bytes, st.launches, st.ms_step, st.ms_front_fwd,
                          st.ms_back, st.ms_front_bwd, st.ms_sync, st.ms_gemm, st.gemm_launches)

    def read_loss(self, lag: int = 0) -> float:
        """Loss of the step issued `lag` steps ago; waits for that step only."""
        out = C.c_float()
        _lib.call("ralpb_model_read_loss", self._h, int(lag), C.byref(out))
        return out.value

    def timed_launches(self) -> list:
        """[(kind name, ms, flops)] of every tensor-core launch of the last profiled step."""
        recs = (_lib.LaunchRec * 512)()
        n = _lib.call_count("ralpb_model_timed_launches", self._h, recs, 512)
        return [(_lib.LAUNCH_KINDS[recs[i].kind], recs[i].ms, recs[i].flops) for i in range(min(n, 512))]

    def set_profiling(self, on: bool) -> None:
        _lib.call("ralpb_model_set_profiling", self._h, int(on))

    def close(self) -> None:
        if getattr(self, "_h", None):
            _lib.lib().ralpb_model_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass


def run_job(job: JobSpec, steps: int = 10, *, warmup: int = 0, seed: int = 0, lr: float = 0.01,
            momentum: float = 0.9, params=None, input_shape=None, name: Optional[str] = None,
            ring_backend: str = "native", fc_sharding: str = "single") -> JobReport:
    """Execute `job` for `steps` measured steps on this process's rank (RANK/WORLD_SIZE from the
    environment, torch.distributed already initialised when W > 1).  Returns the job report on
    every rank (rank 0's carries the loss)."""
    from . import synthetic

    rank = int(os.environ.get("RANK", "0"))
    ex = RankExecutor(job, rank=rank, input_shape=input_shape, ring_backend=ring_backend, fc_sharding=fc_sharding)
    try:
        if params is None:
            params = synthetic.init_params(ex.layers, seed)
        ex.set_params(params)
        b = job.model.batch_size
        records, losses = [], []
        expected = volumes_for(job).total_bytes_per_step
        if ex.fc_sharding == "multi":
            expected = volume_ralp_multi_ps(job.model, job.strategy.split_index, job.worker_count).total_bytes_per_step
        for t in range(warmup + steps):
            imgs, labs = synthetic.batch(seed, t, rank * b, b, ex.in_shape, ex.classes)
            ex.step(imgs, labs, lr=lr, momentum=momentum)
            st = ex.stats()
            if st.logical_bytes != expected:
                raise ExecutorError(f"logical bytes {st.logical_bytes} != oracle volume {expected}")
            if t >= warmup:
                losses.append(st.loss)
                records.append(_breakdown(name or job.model.name, len(records) + 1, st, job.worker_count))
        return JobReport(job=name or job.model.name, strategy=job.strategy.kind.value,
                         worker_count=job.worker_count, batch_size=b, steps=tuple(records),
                         bytes_on_wire_per_step=expected, losses=tuple(losses))
    finally:
        ex.close()


def _breakdown(name: str, step: int, st: StepResult, w: int) -> StepBreakdown:
    # per-rank device times (seconds) in the reference's four categories (simulator.py:163-210);
    # every worker is reported with this rank's timing (ranks are symmetric up to the PS role)
    s = 1e-3
    comp = (st.ms_front_fwd + st.ms_front_bwd) * s
    return StepBreakdown(job=name, step=step, worker_computation=(comp,) * w, ps_computation=(st.ms_back * s,) * w,
                         memcopy=(0.0,) * w, communication=(st.ms_sync * s,) * w)


__all__ = ["ExecutorError", "RankExecutor", "StepResult", "infer_input_shape", "lower", "run_job", "allgather_bytes"]
