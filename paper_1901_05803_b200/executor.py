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

from . import _lib, branchy, resnet
from .planner.costmodel import (JobSpec, volume_baseline, volume_ralp, volume_ralp_multi_ps,
                                 volume_ring)
from .planner.layers import ModelGraph
from .report import JobReport, StepBreakdown


class ExecutorError(ValueError):
    """The job cannot be executed by this backend (unsupported layer mix etc.)."""


def _kv(x) -> str:
    """Enum member -> its value string.  Layer and strategy kinds are compared by value so jobs
    built with the unmodified reference package (`ralp.ModelGraph`, `ralp.JobSpec`,
    pkg/src/ralp/layers.py:22-34, costmodel.py:34-37) lower exactly like the mirror's."""
    return getattr(x, "value", x)


def infer_input_shape(model: ModelGraph) -> tuple[int, int, int]:
    """Per-sample input (h, w, c) of the first layer (a convolution): the smallest input that
    yields its recorded output shape (infer_conv, layers.py:87-103)."""
    first = model.layers[0]
    if _kv(first.kind) != "conv" or first.output_shape is None:
        raise ExecutorError("the first layer must be a derived convolution")
    hp = first.hyperparams
    k, s, p, cout = hp["k"], hp.get("stride", 1), hp.get("pad", 0), hp["cout"]
    cin = (first.param_count - cout) // (k * k * cout)
    o = first.output_shape
    return (o.h - 1) * s + k - 2 * p, (o.w - 1) * s + k - 2 * p, cin


def lower(model: ModelGraph, input_shape: Optional[tuple[int, int, int]] = None) -> list[dict]:
    """ModelGraph -> list of layer dicts (kind, k, stride, pad, h, w, cin, cout, relu[, bn, width,
    downsample]).  ResNet-50's linearised catalog entries are lowered at block granularity from
    the architecture they were generated from (resnet.py, checked entry by entry); Inception-v3 /
    GoogLeNet at branch-group granularity (branchy.py, likewise checked); a later convolution that is
    not a stride-1 "same" window becomes a one-node module."""
    if resnet.is_resnet50(model):
        resnet.check_catalog(model)
        return resnet.lower_layers()[0]
    if branchy.is_branchy_graph(model):   # Inception-v3 / GoogLeNet branch groups
        branchy.check_catalog(model)
        return branchy.lower_layers(model.name, None if input_shape is None else input_shape[0])[0]
    h, w, c = input_shape or infer_input_shape(model)
    out: list[dict] = []
    n = model.num_layers
    flat = None
    for i, L in enumerate(model.layers):
        hp = L.hyperparams
        last = i == n - 1
        kind = _kv(L.kind)
        if kind == "conv":
            k, st, pd = hp["k"], hp.get("stride", 1), hp.get("pad", 0)
            if out and (st != 1 or k != 2 * pd + 1):
                # not a stride-1 'same' window (e.g. OverFeat's unpadded 5x5): a one-node module
                node = branchy.conv(L.name, -1, k, k, hp["cout"], stride=st, pad=(pd, pd), bn=False, output=True)
                d = dict(kind="module", k=0, stride=0, pad=0, h=h, w=w, cin=c, cout=hp["cout"], relu=1, nodes=[node])
            else:
                d = dict(kind="conv", k=k, stride=st, pad=pd, h=h, w=w, cin=c, cout=hp["cout"], relu=1)
            h, w, c = L.output_shape.h, L.output_shape.w, L.output_shape.c
        elif kind == "pool":
            d = dict(kind="pool", k=hp["window"], stride=hp.get("stride", hp["window"]), pad=hp.get("pad", 0), h=h,
                     w=w, cin=c, cout=c, relu=0)
            if d["pad"]:
                raise ExecutorError(f"layer {L.name}: padded pooling is not implemented")
            h, w, c = L.output_shape.h, L.output_shape.w, L.output_shape.c
        elif kind == "fc":
            width = flat if flat is not None else (h * w * c if h else c)
            d = dict(kind="fc", k=0, stride=0, pad=0, h=0, w=0, cin=width, cout=hp["out"], relu=0 if last else 1)
            flat = hp["out"]
            h = w = 0
            c = flat
        elif kind == "flatten":
            continue
        else:
            raise ExecutorError(f"layer {L.name}: kind {kind} is not executable by this backend")
        d["name"] = L.name
        out.append(d)
    return out


def block_param_counts(L: dict) -> tuple[int, int]:
    """(weights, batch-norm parameters) of a bottleneck block layer: wa [width][cin],
    wb [width][3][3][width], wc [cout][width] (, wd [cout][cin]); gamma / beta per convolution."""
    cin, width, cout, down = L["cin"], L["width"], L["cout"], L.get("downsample", 0)
    nw = width * cin + 9 * width * width + cout * width + (cout * cin if down else 0)
    nb = 2 * (2 * width + cout + (cout if down else 0))
    return nw, nb


def expected_volume(job, fc_sharding: str = "single") -> int:
    """The oracle's logical synchronised bytes per step for `job` (costmodel.py:107-162), dispatched
    on the strategy's value so a reference `ralp.JobSpec` works too."""
    kind, m, w = _kv(job.strategy.kind), job.model, job.worker_count
    if kind == "ralp":
        f = volume_ralp_multi_ps if fc_sharding == "multi" else volume_ralp
        return f(m, job.strategy.split_index, w).total_bytes_per_step
    if kind == "ring":
        return volume_ring(m, w).total_bytes_per_step
    return volume_baseline(m, w).total_bytes_per_step


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


_KIND = {"conv": _lib.RALPB_CONV, "pool": _lib.RALPB_POOL, "fc": _lib.RALPB_FC, "block": _lib.RALPB_BLOCK,
         "apool": _lib.RALPB_APOOL, "module": _lib.RALPB_MODULE}
_NODE_OP = {"conv": _lib.RALPB_NODE_CONV, "maxpool": _lib.RALPB_NODE_MAXPOOL, "avgpool": _lib.RALPB_NODE_AVGPOOL}


def _desc_array(layers: Sequence[dict]):
    """(ralpb_layer_desc array, ralpb_node_desc array or None) of a lowered layer table."""
    arr = (_lib.LayerDesc * len(layers))()
    nodes = []
    for a, L in zip(arr, layers):
        a.kind, a.k, a.stride, a.pad = _KIND[L["kind"]], L["k"], L["stride"], L["pad"]
        a.h, a.w, a.cin, a.cout, a.relu = L["h"], L["w"], L["cin"], L["cout"], L["relu"]
        a.bn, a.width, a.downsample = L.get("bn", 0), L.get("width", 0), L.get("downsample", 0)
        if L["kind"] == "module":
            a.node_begin, a.node_count = len(nodes), len(L["nodes"])
            nodes.extend(L["nodes"])
    if not nodes:
        return arr, None
    narr = (_lib.NodeDesc * len(nodes))()
    for a, nd in zip(narr, nodes):
        a.op, a.input = _NODE_OP[nd["op"]], nd["input"]
        a.kh, a.kw, a.stride, a.pad_h, a.pad_w = nd["kh"], nd["kw"], nd["stride"], nd["ph"], nd["pw"]
        a.cout, a.bn, a.output = nd["cout"], nd["bn"], nd["output"]
    return arr, narr


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
    nvlink_out_bytes: int = 0
    nvlink_in_bytes: int = 0


class RankExecutor:
    """One rank's `ralpb_model`.  Multi-rank use needs torch.distributed initialised
    (any backend) so the IPC handles can be exchanged."""

    def __init__(self, job: JobSpec, *, rank: int = 0, world: Optional[int] = None, ps_rank: int = 0,
                 input_shape: Optional[tuple[int, int, int]] = None, ring_backend: str = "native",
                 fc_sharding: str = "single", precision: str = "bf16", placement: str = "colocated",
                 shard_layout: str = "bytes"):
        """ring_backend (StrategyKind.RING_ALLREDUCE only): "native" = the hand-written
        reduce-scatter + SGD + all-gather over NVLink peer memory inside the step; "nccl" = the
        step stops after the backward, torch.distributed (NCCL) all-reduces the gradient vector
        on the model stream, then the update runs (the comparison baseline).
        fc_sharding (StrategyKind.RALP only): "single" = the reference's single PS on rank 0;
        "multi" = the FC tail's first two layers sharded over every GPU (RALPB_STRATEGY_RALP_MPS,
        SURVEY.md 8f.1; logical bytes volume_ralp_multi_ps).
        precision: "bf16" (throughput) or "fp32" (the parity mode: fp32 values as three bf16
        pieces through the same tcgen05 GEMM engine, include/ralpb.h RALPB_PRECISION_FP32).
        placement (StrategyKind.RALP only): "colocated" = W ranks, the PS role on ps_rank which is
        also a worker; "dedicated-ps" = the paper's RALP-N (costmodel.py:244-245): world = W + 1,
        ps_rank runs only the FC tail, every other rank is a worker.
        shard_layout (StrategyKind.BASELINE_PS only): "bytes" = W equal contiguous shards of the
        parameter vector (the B200-idiomatic layout); "layers" = the reference's own PS layout,
        whole weighted layers round-robin over the W shards (simulator.py:551-563) -- under
        parameter skew one shard carries most of the model, the paper's baseline hot spot."""
        kind = _kv(job.strategy.kind)
        if placement not in ("colocated", "dedicated-ps"):
            raise ExecutorError(f"unknown placement {placement!r}")
        if placement == "dedicated-ps" and (kind != "ralp" or fc_sharding != "single"):
            raise ExecutorError("a dedicated PS rank is a layer-placed (RALP, single PS) placement")
        workers = job.worker_count
        world = workers + (1 if placement == "dedicated-ps" else 0) if world is None else world
        if world != workers + (1 if placement == "dedicated-ps" else 0):
            raise ExecutorError("one rank per worker (plus the dedicated PS rank): world size must be "
                                f"{workers + (1 if placement == 'dedicated-ps' else 0)}")
        if ring_backend not in ("native", "nccl"):
            raise ExecutorError(f"unknown ring backend {ring_backend!r}")
        if fc_sharding not in ("single", "multi"):
            raise ExecutorError(f"unknown fc_sharding {fc_sharding!r}")
        if precision not in _lib.PRECISIONS:
            raise ExecutorError(f"unknown precision {precision!r}")
        if shard_layout not in ("bytes", "layers") or (shard_layout == "layers" and kind != "baseline"):
            raise ExecutorError(f"shard_layout {shard_layout!r}: 'bytes', or 'layers' for the all-on-PS baseline")
        self.shard_layout = shard_layout
        self.fc_sharding = fc_sharding if kind == "ralp" else "single"
        self.ring_backend = ring_backend if kind == "ring" else None
        self.precision, self.placement = precision, placement
        self.job = job
        self.model = job.model
        self.rank, self.world, self.ps_rank = rank, world, ps_rank
        self.workers = workers
        self.is_worker = not (placement == "dedicated-ps" and rank == ps_rank)
        # worker index (rank order, the dedicated PS skipped): its sample block of every step
        self.worker_index = rank - (1 if placement == "dedicated-ps" and rank > ps_rank else 0)
        self.layers = lower(job.model, input_shape)
        self.in_shape = (self.layers[0]["h"], self.layers[0]["w"], self.layers[0]["cin"])
        self.classes = self.layers[-1]["cout"]
        split = job.strategy.split_index if kind == "ralp" else 0
        if split and (resnet.is_resnet50(job.model) or branchy.is_branchy_graph(job.model)):
            try:   # catalog entries -> lowered layers
                split = (resnet.lowered_split(split) if resnet.is_resnet50(job.model)
                         else branchy.lowered_split(job.model.name, split))
            except ValueError as e:
                raise ExecutorError(str(e)) from None
        if kind == "ralp":
            strategy = _lib.RALPB_STRATEGY_RALP if self.fc_sharding == "single" else _lib.RALPB_STRATEGY_RALP_MPS
        elif kind == "ring":
            strategy = _lib.RALPB_STRATEGY_RING if ring_backend == "native" else _lib.RALPB_STRATEGY_RING_EXTERNAL
        elif shard_layout == "layers":
            strategy = _lib.RALPB_STRATEGY_BASELINE_LAYER_SHARDS
        else:
            strategy = _lib.RALPB_STRATEGY_BASELINE
        self.lowered_split = split   # 1-based cut over the lowered layer table (0: none)
        self._descs, self._nodes = _desc_array(self.layers)
        h = C.c_void_p()
        _lib.call("ralpb_model_create_graph", C.cast(self._descs, C.c_void_p), len(self.layers),
                  None if self._nodes is None else C.cast(self._nodes, C.c_void_p),
                  0 if self._nodes is None else len(self._nodes), split,
                  job.model.batch_size, strategy, rank, world, ps_rank, job.model.bytes_per_element,
                  _lib.PRECISIONS[precision], workers, C.byref(h))
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

    def _param_arrays(self, L: dict):
        """Host arrays (w, b) in the layout of ralpb_model_set_params for one lowered layer."""
        if L["kind"] == "conv":
            return (np.empty((L["cout"], L["k"], L["k"], L["cin"]), dtype=np.float32),
                    np.empty(L["cout"] * (2 if L.get("bn") else 1), dtype=np.float32))
        if L["kind"] == "fc":
            return np.empty((L["cout"], L["cin"]), dtype=np.float32), np.empty(L["cout"], dtype=np.float32)
        if L["kind"] == "block":
            nw, nb = block_param_counts(L)
            return np.empty(nw, dtype=np.float32), np.empty(nb, dtype=np.float32)
        if L["kind"] == "module":
            nw, nb = branchy.module_param_counts(L)
            return np.empty(nw, dtype=np.float32), np.empty(nb, dtype=np.float32)
        return None

    def get_params(self) -> list:
        out = []
        for i, L in enumerate(self.layers):
            arrs = self._param_arrays(L)
            if arrs is None:
                out.append(None)
                continue
            w, b = arrs
            _lib.call("ralpb_model_get_params", self._h, i, _ptr(w), _ptr(b), 1)
            out.append((w, b))
        return out

    def get_grads(self) -> list:
        """This rank's parameter gradients of the last step (per layer (w, b) or None), in the
        get_params layout; the FC tail's only on the rank that holds it."""
        out = []
        for i, L in enumerate(self.layers):
            arrs = self._param_arrays(L)
            if arrs is None:
                out.append(None)
                continue
            w, b = arrs
            _lib.call("ralpb_model_get_grads", self._h, i, _ptr(w), _ptr(b))
            out.append((w, b))
        return out

    def debug_buffer(self, which: int, i: int = 0) -> np.ndarray:
        """A copy of one of the last step's device buffers (include/ralpb.h RALPB_DBG_*), flat:
        fp32 for LOGITS / MPS_PARTIAL, bf16 values widened to fp32 otherwise (bf16 precision)."""
        import torch
        n = _lib.lib().ralpb_model_debug_buffer(self._h, i, which, None)
        if n < 0:
            raise ExecutorError(f"debug buffer {which}/{i} is not available")
        f32 = which in (_lib.DBG_LOGITS, _lib.DBG_MPS_PARTIAL)
        pieces = int(os.environ.get("RALPB_PIECES", "3")) if self.precision == "fp32" else 1
        elems = n * (pieces if not f32 else 1)
        t = torch.empty(elems, dtype=torch.float32 if f32 else torch.bfloat16)
        if _lib.lib().ralpb_model_debug_buffer(self._h, i, which, C.c_void_p(t.data_ptr())) != n:
            raise ExecutorError(f"debug buffer {which}/{i}: copy failed")
        return t.float().numpy()

    # ---------------------------------------------------------------- step
    @property
    def stream(self) -> int:
        return _lib.lib().ralpb_model_stream(self._h)

    def step(self, images, labels, *, lr: float = 0.01, momentum: float = 0.9) -> None:
        """images/labels: numpy host arrays (pinned-ness is the caller's business) or torch
        tensors (host or cuda); None on a dedicated PS rank (it has no batch of its own)."""
        on_host = 1
        if images is None:
            ip, lp, on_host = None, None, 0
        elif hasattr(images, "data_ptr"):
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
                          st.ms_back, st.ms_front_bwd, st.ms_sync, st.ms_gemm, st.gemm_launches,
                          st.nvlink_out_bytes, st.nvlink_in_bytes)

    def read_loss(self, lag: int = 0) -> float:
        """Loss of the step issued `lag` steps ago; waits for that step only."""
        out = C.c_float()
        _lib.call("ralpb_model_read_loss", self._h, int(lag), C.byref(out))
        return out.value

    def timed_launches(self) -> list:
        """[(kind name, ms, flops, bytes)] of every timed launch of the last profiled step (tensor-core
        kernels, exchange kernels, max-pool backward, SGD; include/ralpb.h ralpb_launch_rec)."""
        recs = (_lib.LaunchRec * 512)()
        n = _lib.call_count("ralpb_model_timed_launches", self._h, recs, 512)
        return [(_lib.LAUNCH_KINDS[recs[i].kind], recs[i].ms, recs[i].flops, recs[i].bytes) for i in range(min(n, 512))]

    STREAMS = ("main", "aux", "comm", "sync")

    def timeline(self) -> list:
        """[(kind name, stream name, start ms, duration ms)] of the last profiled step on this rank
        (start relative to the step's first event): the overlap of the act-grad scatter (comm),
        the FC update (aux) and the sync bucket (sync) with the main stream's kernels."""
        recs = (_lib.LaunchRec * 512)()
        n = _lib.call_count("ralpb_model_timed_launches", self._h, recs, 512)
        return [(_lib.LAUNCH_KINDS[recs[i].kind], self.STREAMS[recs[i].stream] if 0 <= recs[i].stream < 4 else "?",
                 recs[i].t0, recs[i].ms) for i in range(min(n, 512))]

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


def _allgather_rows(row: list[float], world: int) -> list[list[float]]:
    """Every rank's `row` (equal length), rank-ordered, over the initialised process group."""
    if world == 1:
        return [row]
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else torch.device("cpu")
    mine = torch.tensor(row, dtype=torch.float64, device=dev)
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    return [p.cpu().tolist() for p in parts]


def run_job(job: JobSpec, steps: int = 10, *, warmup: int = 0, seed: int = 0, lr: float = 0.01,
            momentum: float = 0.9, params=None, input_shape=None, name: Optional[str] = None,
            ring_backend: str = "native", fc_sharding: str = "single", precision: str = "bf16",
            placement: str = "colocated", shard_layout: str = "bytes") -> JobReport:
    """Execute `job` for `steps` measured steps on this process's rank (RANK from the environment,
    torch.distributed already initialised when more than one rank takes part).  `job` may be the
    mirror's JobSpec or the unmodified reference's `ralp.JobSpec`.  Every step checks that the
    logical bytes the ranks counted at their count_wire sites sum to the oracle's volume.  Returns
    the job report on every rank, with every worker's own measured times (rank 0's carries the
    losses)."""
    from . import synthetic

    rank = int(os.environ.get("RANK", "0"))
    ex = RankExecutor(job, rank=rank, input_shape=input_shape, ring_backend=ring_backend, fc_sharding=fc_sharding,
                      precision=precision, placement=placement, shard_layout=shard_layout)
    try:
        if params is None:
            params = synthetic.init_params(ex.layers, seed)
        ex.set_params(params)
        b = job.model.batch_size
        records, losses = [], []
        expected = expected_volume(job, ex.fc_sharding)
        for t in range(warmup + steps):
            if ex.is_worker:
                imgs, labs = synthetic.batch(seed, t, ex.worker_index * b, b, ex.in_shape, ex.classes)
                ex.step(imgs, labs, lr=lr, momentum=momentum)
            else:
                ex.step(None, None, lr=lr, momentum=momentum)
            st = ex.stats()
            rows = _allgather_rows([st.logical_bytes, st.ms_step, st.ms_front_fwd + st.ms_front_bwd, st.ms_back,
                                    1.0 if ex.is_worker else 0.0, 1.0 if rank == ex.ps_rank else 0.0], ex.world)
            total = int(round(sum(r[0] for r in rows)))
            if total != expected:
                raise ExecutorError(f"logical bytes {total} (summed over ranks) != oracle volume {expected}")
            if t >= warmup:
                losses.append(st.loss)
                records.append(_breakdown(name or job.model.name, len(records) + 1, rows, _kv(job.strategy.kind)))
        return JobReport(job=name or job.model.name, strategy=_kv(job.strategy.kind),
                         worker_count=job.worker_count, batch_size=b, steps=tuple(records),
                         bytes_on_wire_per_step=expected, losses=tuple(losses))
    finally:
        ex.close()


def _breakdown(name: str, step: int, rows: list[list[float]], kind: str) -> StepBreakdown:
    """Every worker's measured step (seconds) in the reference's four categories
    (simulator.py:163-210).  worker_computation = its front forward + backward; ps_computation =
    the back segment where the FC tail runs on that worker's GPU (the colocated PS; the dedicated
    PS's tail is charged to every worker in equal shares, like the reference's per-worker
    back_batch_s, simulator.py:695); communication = the rest of its step (cut / act-grad exchange,
    waiting, sharded-PS sync).  memcopy is 0: on this backend no cut, act-grad or parameter is
    staged through host memory (the reference models cudaMemcpy d2h/h2d, simulator.py:676,685)."""
    s = 1e-3
    worker_rows = [r for r in rows if r[4] > 0.5]
    ps_rows = [r for r in rows if r[5] > 0.5 and r[4] < 0.5]
    ps_share = (ps_rows[0][3] * s / len(worker_rows)) if ps_rows else 0.0
    comp, ps, comm = [], [], []
    for r in worker_rows:
        c = (r[2] + (r[3] if kind != "ralp" else 0.0)) * s   # baseline / ring: the FC tail is worker compute
        p = (r[3] * s if (r[5] > 0.5 and kind == "ralp") else 0.0) + ps_share
        comp.append(c)
        ps.append(p)
        comm.append(max(0.0, r[1] * s - c - (r[3] * s if (r[5] > 0.5 and kind == "ralp") else 0.0)))
    w = len(worker_rows)
    return StepBreakdown(job=name, step=step, worker_computation=tuple(comp), ps_computation=tuple(ps),
                         memcopy=(0.0,) * w, communication=tuple(comm))


__all__ = ["ExecutorError", "RankExecutor", "StepResult", "expected_volume", "infer_input_shape", "lower", "run_job",
           "allgather_bytes"]
