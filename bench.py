"""Headline benchmark: layer-placed (RALP) VGG-16 training step on 1/2/4/8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 is launched by the driver with torch.distributed.run (one process per GPU).
Metric (BASELINE.json): images/sec per step, layer-placed vs all-on-PS, plus the
synchronised bytes per step.  Workload: VGG-16 224x224 synthetic, b=128 per
worker, partitioner-chosen split (profile() -> pool5, layer 18), W = N workers,
PS role on rank 0.  `value` is whole-job images/s with inputs resident in HBM
(device-timed with CUDA events on the executor's stream, max over ranks);
`e2e` is the same through the public API with pinned host inputs copied in every
step and the loss read back every step.  The activation working set (~4.5 GB per
step per GPU) is far larger than the 126 MB L2, so no L2 flush is inserted.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

MODEL = "vgg16"
BATCH = 128
METRIC = "images/sec per step at 1/2/4/8 B200 (layer-placed vs all-on-PS); sync bytes/step"
KERNEL_NAMES = {"conv_fwd": "conv_slab_fwd_kernel (implicit-GEMM conv forward / backward-data, single CTA)",
                "conv_fwd_pair": "conv_slab_fwd_kernel (CTA pair)",
                "conv_wgrad_pair": "conv_slab_wgrad_pair_kernel (backward-filter, CTA pair)",
                "conv_wgrad": "conv_slab_wgrad_kernel (backward-filter, single CTA)",
                "first_conv_fwd": "conv_first_fwd_kernel", "first_conv_wgrad": "conv_first_wgrad_kernel",
                "gemm": "gemm_sm100_kernel (FC)"}
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None

    def __enter__(self):
        import threading
        self.lines, self._all, self._t0 = [], [], None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
            return self
        first = threading.Event()

        def reader():
            for line in self.proc.stdout:
                if line.strip():
                    self._all.append((time.perf_counter(), line))
                    first.set()
        self._thread = threading.Thread(target=reader, daemon=True)
        self._thread.start()
        first.wait(timeout=10.0)  # sampling is live before the timed region starts
        self._t0 = time.perf_counter()
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            t1 = time.perf_counter()
            # at least one sample after the region (nvidia-smi samples every 100 ms)
            deadline = t1 + 1.0
            while time.perf_counter() < deadline and not any(t >= t1 for t, _ in self._all):
                time.sleep(0.02)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=10)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            # samples from just before the region to just after it
            lo = max((t for t, _ in self._all if t <= self._t0), default=self._t0)
            self.lines = [l for t, l in self._all if lo <= t <= deadline]

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _cpu_baseline_step(sample_b: int, steps: int, warmup: int = 1):
    """Oracle port (oracle/step.py, plain fp32 torch on the host cores) of the layer-placed step,
    W=1 at per-worker batch sample_b: a bounded sample of the workload."""
    import torch
    from oracle import step as ostep
    from paper_1901_05803_b200 import synthetic
    from paper_1901_05803_b200.executor import lower
    from paper_1901_05803_b200.planner import catalog_lookup

    torch.set_num_threads(os.cpu_count() or 1)
    m = catalog_lookup(MODEL).with_batch_size(sample_b)
    layers = lower(m)
    st = ostep.OracleState(layers, synthetic.init_params(layers, 0))
    shape = (layers[0]["h"], layers[0]["w"], layers[0]["cin"])
    batches = [synthetic.batch(0, t, 0, sample_b, shape, layers[-1]["cout"]) for t in range(warmup + steps)]
    for t in range(warmup):
        ostep.train_step(st, "ralp", 1, [batches[t]])
    t0 = time.perf_counter()
    for t in range(steps):
        ostep.train_step(st, "ralp", 1, [batches[warmup + t]])
    dt = time.perf_counter() - t0
    return {"value": sample_b * steps / dt, "unit": "images/s", "cores": torch.get_num_threads(), "kind": "port",
            "cpu_model": _cpu_model(), "logical_cpus": os.cpu_count(),
            "sample": f"{MODEL} {shape[0]}x{shape[1]} layer-placed step (oracle/step.py, fp32 torch CPU), W=1, b={sample_b}, "
                      f"{steps} timed steps after {warmup} warm-up, {dt:.1f} s"}


def _overlap(timeline):
    """Per side stream (aux: FC update; comm: act-grad scatter; sync: the sync bucket), the time its
    timed kernels ran and how much of it overlapped the main stream's timed kernels (profiling
    pass, rank 0's clock)."""
    main = sorted((t0, t0 + d) for _, st, t0, d in timeline if st == "main")
    out = {}
    for _, st, t0, d in timeline:
        if st == "main" or st == "?":
            continue
        ov = sum(max(0.0, min(t0 + d, b) - max(t0, a)) for a, b in main)
        o = out.setdefault(st, {"launches": 0, "ms": 0.0, "overlapped_ms": 0.0})
        o["launches"] += 1
        o["ms"] += d
        o["overlapped_ms"] += min(ov, d)
    return {k: {kk: (round(vv, 4) if isinstance(vv, float) else vv) for kk, vv in v.items()} for k, v in out.items()}


def _headline_split():
    from paper_1901_05803_b200.planner import catalog_lookup, profile
    return profile(catalog_lookup(MODEL).with_batch_size(BATCH)).split_index


REF_MAX_STEPS = 3   # one b=128 VGG-16 step of the CPU port takes ~10 s on 16 host cores


def run_reference(args):
    """The reference arm: the reference's CPU path for this step (the oracle port -- the reference
    itself only simulates the step) on the box's host cores, on OUR arm's workload: VGG-16 224x224,
    b=128 per worker, the partitioner's split, fp32.  Each timed step is one full b=128 step; the
    run is capped at REF_MAX_STEPS timed steps (+1 warm-up) so it ends within a few minutes."""
    world, rank, _ = _dist()
    if rank != 0:
        return
    steps = max(1, min(args.steps, REF_MAX_STEPS))
    cb = _cpu_baseline_step(BATCH, steps, 1)
    line = {"impl": "reference", "metric": METRIC, "value": cb["value"],
            "unit": "images/s", "n_gpus": args.gpus, "steps": steps, "warmup": 1,
            "ms_per_step": 1e3 * BATCH / cb["value"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{MODEL} 224x224 synthetic, b={BATCH}/worker, W=1, partitioner split "
                                   f"{_headline_split()} (pool5), layer-placed (RALP) step, CPU oracle port",
                       "model": MODEL, "per_worker_batch": BATCH, "split": _headline_split(),
                       "same_config": True, "steps_requested": args.steps,
                       "note": f"timed steps capped at {REF_MAX_STEPS} (each ~10 s of host CPU); N>1: rank 0 "
                               "runs the W=1 step (the CPU path does not shard)"},
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _build_executor(strategy: str, world: int, rank: int, ring_backend: str = "native", fc_sharding: str = "single",
                    precision: str = "bf16", placement: str = "colocated", model: str | None = None,
                    shard_layout: str = "bytes"):
    from paper_1901_05803_b200 import synthetic
    from paper_1901_05803_b200.executor import RankExecutor
    from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, profile

    m = catalog_lookup(model or MODEL).with_batch_size(BATCH)
    rep = profile(m)
    workers = world - 1 if placement == "dedicated-ps" else world
    if strategy == "ralp":
        job = JobSpec(m, Strategy.ralp(rep.split_index), workers)
    elif strategy == "ring":
        job = JobSpec(m, Strategy.ring(), world, ps_count=0)
    else:
        job = JobSpec(m, Strategy.baseline(), world)
    ex = RankExecutor(job, rank=rank, world=world, ring_backend=ring_backend, fc_sharding=fc_sharding,
                      precision=precision, placement=placement, shard_layout=shard_layout)
    ex.set_params(synthetic.init_params(ex.layers, 0))
    return ex, job, rep


def _job_bytes(st, world: int) -> int:
    """Logical synchronised bytes of the job: the sum of every rank's count_wire-site counts."""
    if world == 1:
        return st.logical_bytes
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(st.logical_bytes)], dtype=torch.float64, device="cuda")
    dist.all_reduce(t)
    return int(t.item())


def _time_steps(ex, imgs, labs, steps, warmup, world, on_host=False, read_loss=False):
    """read_loss: read every step's loss back to the host (pipelined one step behind: the loss of
    step t is read after step t+1 has been enqueued, so its host inputs' copy overlaps step t)."""
    import torch
    import torch.distributed as dist

    stream = torch.cuda.ExternalStream(ex.stream)
    for t in range(warmup):
        ex.step(imgs[t % len(imgs)], labs[t % len(labs)])
    ex.stats()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for t in range(steps):
        ex.step(imgs[t % len(imgs)], labs[t % len(labs)])
        if read_loss and t > 0:
            ex.read_loss(1)  # device->host read of step t-1's loss
    if read_loss:
        ex.read_loss(0)
    e.record(stream)
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        dist.barrier()
    return ms / steps


def run_ours(args):
    import numpy as np
    import torch

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1901_05803_b200._lib import TENSOR_KINDS
    from paper_1901_05803_b200.planner import compute_load, volume_ralp

    ex, job, rep = _build_executor("ralp", world, rank)
    m = job.model
    shape = ex.in_shape
    g = torch.Generator(device="cuda").manual_seed(1234 + rank)
    dimgs = [torch.randn(BATCH, *shape, generator=g, device="cuda") for _ in range(2)]
    dlabs = [torch.randint(0, ex.classes, (BATCH,), generator=g, device="cuda", dtype=torch.int32) for _ in range(2)]

    with ClockSampler(local) as clk:
        ms = _time_steps(ex, dimgs, dlabs, args.steps, args.warmup, world)
    st = ex.stats()
    value = world * BATCH / (ms * 1e-3)
    # logical bytes: each rank counts its own count_wire sites; the job's figure is their sum
    logical_total = st.logical_bytes
    nvl = [st.nvlink_out_bytes, st.nvlink_in_bytes]
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([float(st.logical_bytes)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        logical_total = int(t.item())

    # end-to-end through the public API: pinned host inputs copied each step, loss read back each step
    himgs = [x.cpu().pin_memory() for x in dimgs]
    hlabs = [x.cpu().pin_memory() for x in dlabs]
    ms_e2e = _time_steps(ex, himgs, hlabs, args.steps, 1, world, on_host=True, read_loss=True)
    e2e_value = world * BATCH / (ms_e2e * 1e-3)
    h2d = BATCH * int(np.prod(shape)) * 4 + BATCH * 4

    # roofline: a profiling pass after the timed region brackets every tensor-core launch with
    # CUDA events on its own stream and records its algorithmic FLOPs (ralpb_model_timed_launches)
    ex.set_profiling(True)
    ex.step(dimgs[0], dlabs[0])
    prof = ex.stats()
    launches = ex.timed_launches()
    timeline = ex.timeline()
    ex.set_profiling(False)
    overlap = _overlap(timeline)
    if rank == 0 and os.environ.get("RALPB_TIMELINE_OUT"):
        Path(os.environ["RALPB_TIMELINE_OUT"]).write_text(json.dumps(
            {"world": world, "rank": rank, "launches": [dict(kind=k, stream=st, t0_ms=t0, ms=d) for k, st, t0, d in timeline]},
            indent=0))
    worker_flops, ps_flops = compute_load(m, rep.split_index, world)
    flops_rank = worker_flops + (ps_flops if rank == 0 else 0)
    peaks, peak_src = _peaks()
    by_kind, xchg, hbm = {}, {}, {}
    for kind, lms, lfl, lby in launches:
        dst = by_kind if kind in TENSOR_KINDS else (xchg if kind in ("push", "shard_update") else hbm)
        k = dst.setdefault(kind, {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0})
        k["launches"] += 1
        k["ms"] += lms
        k["flops"] += lfl
        k["bytes"] += lby
    traffic_doc = {}
    tfile = ROOT / "profiles" / f"traffic_{MODEL}.json"
    if tfile.exists():
        traffic_doc = json.loads(tfile.read_text())
    # NVLink: the hand-written exchange kernels' bytes / time, and NCCL all-reduce of the same
    # front-parameter vector as the comparison baseline (north star)
    nvlink = None
    if world > 1:
        import torch.distributed as dist
        link = peaks.get("nvlink_gbs_per_direction", 770.0)
        nvlink = {"peak_gbs": link, "peak_source": "B200_PROFILING.md measured peer copy per direction"}
        for kind, k in xchg.items():
            # bytes per direction (push: all outbound; shard update: the same number in and out)
            gbs = k["bytes"] / (k["ms"] * 1e-3) / 1e9 if k["ms"] > 0 else None
            nvlink[kind] = {"launches": k["launches"], "ms": k["ms"], "bytes_per_direction": k["bytes"],
                            "gbs_per_direction": gbs, "frac": gbs / link if gbs else None}
        p_front = m.cumulative_param_bytes(rep.split_index) // m.bytes_per_element
        buf = torch.zeros(p_front, dtype=torch.float32, device="cuda")
        for _ in range(3):
            dist.all_reduce(buf)
        torch.cuda.synchronize()
        dist.barrier()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(10):
            dist.all_reduce(buf)
        s1.record()
        torch.cuda.synchronize()
        t = torch.tensor([s0.elapsed_time(s1) / 10], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        nvlink["nccl_allreduce_front_params"] = {"ms": t.item(), "floats": p_front,
                                                 "note": "torch.distributed NCCL all_reduce of the front parameter "
                                                         "vector (what the sharded-PS RS+SGD+AG kernel replaces)"}
        del buf
    for kind, k in by_kind.items():
        k["tflops"] = k["flops"] / (k["ms"] * 1e-3) / 1e12 if k["ms"] > 0 else None
        k["frac"] = k["tflops"] / peaks["bf16_tflops_sustained"] if k["tflops"] else None
        k["gbs"] = k["bytes"] / (k["ms"] * 1e-3) / 1e9 if k["ms"] > 0 else None
        k["hbm_frac"] = k["gbs"] / peaks["hbm_gbs"] if k["gbs"] else None
    # kernels whose bound is HBM: the first conv (K = 27: pure data movement), the FC GEMMs at
    # M = W*b rows (weight-streaming), the max-pool backward, SGD
    for kind, k in hbm.items():
        k["gbs"] = k["bytes"] / (k["ms"] * 1e-3) / 1e9 if k["ms"] > 0 else None
        k["hbm_frac"] = k["gbs"] / peaks["hbm_gbs"] if k["gbs"] else None
    hbm_view = {kk: {"launches": v["launches"], "ms": round(v["ms"], 4), "gbs": round(v["gbs"], 1) if v["gbs"] else None,
                     "frac": round(v["hbm_frac"], 3) if v["hbm_frac"] else None}
                for kk, v in list(hbm.items()) + [(kk, by_kind[kk]) for kk in ("first_conv_fwd", "gemm") if kk in by_kind]}
    dominant = max(by_kind, key=lambda kk: by_kind[kk]["ms"]) if by_kind else None
    dom = by_kind.get(dominant, {})
    dom_traffic = traffic_doc.get("per_kind", {}).get(dominant, {}).get("dram_bytes_per_launch")
    step_ms = sum(k["ms"] for k in by_kind.values())
    step_achieved = flops_rank / (step_ms * 1e-3) / 1e12 if step_ms > 0 else None

    ex.close()
    cmp = not args.quick   # --quick: the headline line only (A/B runs)
    # the same layer-placed step with ONE parameter sync after the whole backward (no sync bucket
    # under the remaining backward, RALPB_SYNC_BUCKET=0): what the bucketed sync saves
    unbucketed = None
    if world > 1:
        torch.cuda.empty_cache()
        os.environ["RALPB_SYNC_BUCKET"] = "0"
        try:
            exu, _, _ = _build_executor("ralp", world, rank)
        finally:
            os.environ.pop("RALPB_SYNC_BUCKET", None)
        ms_u = _time_steps(exu, dimgs, dlabs, args.steps, args.warmup, world)
        stu = exu.stats()
        exu.close()
        unbucketed = {"value": world * BATCH / (ms_u * 1e-3), "ms_per_step": ms_u,
                      "ms_sync_rank0": stu.ms_sync,
                      "note": "RALPB_SYNC_BUCKET=0: the whole front synchronised after the backward"}
    # all-on-PS comparator (StrategyKind.BASELINE_PS): same workload, every layer on every worker
    ms_b = bytes_b = None
    if cmp:
        torch.cuda.empty_cache()
        exb, jobb, _ = _build_executor("baseline", world, rank)
        ms_b = _time_steps(exb, dimgs, dlabs, args.steps, args.warmup, world)
        stb = exb.stats()
        bytes_b = _job_bytes(stb, world)   # (a collective: every rank, outside the rank-0 block)
        exb.close()
    # ... with the reference's own PS layout: whole weighted layers round-robin over the W shards
    # (simulator.py:551-563), so fc1's 411 MB sits on one shard -- the paper's baseline hot spot
    layer_shards = None
    if world > 1 and cmp:
        torch.cuda.empty_cache()
        exl, _, _ = _build_executor("baseline", world, rank, shard_layout="layers")
        ms_l = _time_steps(exl, dimgs, dlabs, args.steps, args.warmup, world)
        stl = exl.stats()
        exl.close()
        layer_shards = {"value": world * BATCH / (ms_l * 1e-3), "ms_per_step": ms_l,
                        "logical_sync_bytes_per_step": _job_bytes(stl, world),
                        "note": "all-on-PS with whole-layer round-robin PS shards (the reference's layout)"}
    # ring all-reduce comparators (StrategyKind.RING_ALLREDUCE, the Horovod baseline of the paper):
    # the hand-written NVLink RS+SGD+AG vs NCCL all_reduce of the gradient vector (N > 1)
    ring = None
    if world > 1 and cmp:
        ring = {}
        for backend in ("native", "nccl"):
            torch.cuda.empty_cache()
            exr, _, _ = _build_executor("ring", world, rank, backend)
            ms_r = _time_steps(exr, dimgs, dlabs, args.steps, args.warmup, world)
            str_ = exr.stats()
            exr.close()
            ring[backend] = {"value": world * BATCH / (ms_r * 1e-3), "ms_per_step": ms_r,
                             "logical_sync_bytes_per_step": _job_bytes(str_, world)}
    # layer-placed with the FC tail sharded over every GPU (the paper's multi-PS)
    mps = None
    if world > 1 and cmp:
        torch.cuda.empty_cache()
        exm, _, _ = _build_executor("ralp", world, rank, fc_sharding="multi")
        ms_m = _time_steps(exm, dimgs, dlabs, args.steps, args.warmup, world)
        stm = exm.stats()
        exm.close()
        mps = {"value": world * BATCH / (ms_m * 1e-3), "ms_per_step": ms_m,
               "logical_bytes_per_step": _job_bytes(stm, world),
               "note": "FC-0 column-parallel / FC-1 row-parallel over all GPUs (volume_ralp_multi_ps)"}

    # the parity precision (fp32 values as three bf16 pieces through the same tcgen05 GEMM engine): a
    # same-precision number beside the fp32 CPU arm
    fp32 = None
    if not args.no_fp32 and cmp:
        torch.cuda.empty_cache()
        exf, _, _ = _build_executor("ralp", world, rank, precision="fp32")
        ms_f = _time_steps(exf, dimgs, dlabs, max(3, args.steps // 4), 3, world)
        stf = exf.stats()
        exf.close()
        fp32 = {"value": world * BATCH / (ms_f * 1e-3), "ms_per_step": ms_f, "dtype": "f32 (three bf16 pieces)",
                "logical_bytes_per_step": _job_bytes(stf, world),
                "note": "RALPB_PRECISION_FP32: every activation / gradient three bf16 pieces (exact in fp32), every "
                        "contraction on the tcgen05 GEMM engine over the pieces (9 products, fp32 accumulation); "
                        "tests/test_parity_fp32_gpu.py pins it to the plain fp32 oracle"}
    # RALP-N (costmodel.py:244-245): N-1 workers + a dedicated PS GPU (rank 0)
    ralp_n = None
    if world > 1 and cmp:
        torch.cuda.empty_cache()
        exn, jobn, _ = _build_executor("ralp", world, rank, placement="dedicated-ps")
        if exn.is_worker:
            ms_n = _time_steps(exn, dimgs, dlabs, args.steps, args.warmup, world)
        else:
            ms_n = _time_steps(exn, [None], [None], args.steps, args.warmup, world)
        stn = exn.stats()
        exn.close()
        ralp_n = {"value": (world - 1) * BATCH / (ms_n * 1e-3), "ms_per_step": ms_n, "workers": world - 1,
                  "logical_bytes_per_step": _job_bytes(stn, world),
                  "note": "ralp-n placement: rank 0 runs only the FC tail, ranks 1..N-1 are workers"}

    # The catalog's branchy models executed, layer-placed at the partitioner's
    # split for b=128, W = N: ResNet-50 (BASELINE.json config 5, conv-grad sync dominated; blocks with
    # batch norm and projection shortcuts), Inception-v3 (299x299, branch groups with batch norm) and
    # GoogLeNet (224x224, branch groups with biases)
    def catalog_comparator(name):
        torch.cuda.empty_cache()
        exc, jobc, repc = _build_executor("ralp", world, rank, model=name)
        gc = torch.Generator(device="cuda").manual_seed(4321 + rank)
        ci = [torch.randn(BATCH, *exc.in_shape, generator=gc, device="cuda") for _ in range(2)]
        cl = [torch.randint(0, exc.classes, (BATCH,), generator=gc, device="cuda", dtype=torch.int32) for _ in range(2)]
        ms_c = _time_steps(exc, ci, cl, args.steps, args.warmup, world)
        stc = exc.stats()
        exc.close()
        del ci, cl
        wfc, pfc = compute_load(jobc.model, repc.split_index, world)
        h, w, _ = exc.in_shape
        return {"value": world * BATCH / (ms_c * 1e-3), "ms_per_step": ms_c, "split": repc.split_index,
                "lowered_split": exc.lowered_split,
                "logical_bytes_per_step": _job_bytes(stc, world),
                "oracle_volume_ralp": volume_ralp(jobc.model, repc.split_index, world).total_bytes_per_step,
                "tensor_frac_of_step": (wfc + (pfc if rank == 0 else 0)) / (ms_c * 1e-3) / 1e12
                                       / peaks["bf16_tflops_sustained"],
                "note": f"{name} {h}x{w} synthetic, b={BATCH}/worker, layer-placed at the partitioner's split "
                        f"{repc.split_index}; tensor_frac_of_step = compute_load() FLOPs / wall step time / "
                        "sustained bf16 peak"}

    alexnet = catalog_comparator("alexnet") if cmp and MODEL != "alexnet" else None   # BASELINE config 2
    resnet50 = catalog_comparator("resnet-50") if cmp and not args.no_resnet and MODEL != "resnet-50" else None
    inception_v3 = catalog_comparator("inception-v3") if cmp and not args.no_branchy else None
    googlenet = catalog_comparator("googlenet") if cmp and not args.no_branchy else None

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and cmp:
        cpu = _cpu_baseline_step(BATCH, 1, 1)

    if rank == 0:
        line = {
            "metric": METRIC,
            "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{MODEL} {shape[0]}x{shape[1]} synthetic, b={BATCH}/worker, W={world}, partitioner split "
                                   f"{rep.split_index} ({m.layer(rep.split_index).name}), FC tail on rank 0",
                       "model": MODEL, "global_batch": world * BATCH, "per_worker_batch": BATCH,
                       "split": rep.split_index, "parallelism": f"dp{world}+fc-tail-on-ps",
                       "l2": "activation working set ~4.5 GB/GPU/step >> 126 MB L2; no flush"},
            "sync_bytes_per_step": {"logical": logical_total,
                                    "oracle_volume_ralp": volume_ralp(m, rep.split_index, world).total_bytes_per_step,
                                    "logical_counted_rank0": st.logical_bytes,
                                    "physical_nvlink_rank0": {"out": nvl[0], "in": nvl[1]}},
            "all_on_ps": None if ms_b is None else {"value": world * BATCH / (ms_b * 1e-3), "ms_per_step": ms_b,
                                                    "logical_sync_bytes_per_step": bytes_b},
            "ralp_unbucketed_sync": unbucketed,
            "all_on_ps_layer_shards": layer_shards,
            "ring_allreduce": ring,
            "ralp_fc_sharded": mps,
            "ralp_dedicated_ps": ralp_n,
            "precision_fp32": fp32,
            "alexnet": alexnet,
            "resnet50": resnet50,
            "inception_v3": inception_v3,
            "googlenet": googlenet,
            "overlap_rank0": overlap,
            "breakdown_ms_rank0": {"front_fwd": st.ms_front_fwd, "back": st.ms_back, "front_bwd": st.ms_front_bwd,
                                   "sync": st.ms_sync, "tensor_kernels_sum": prof.ms_gemm,
                                   "tensor_launches": prof.gemm_launches},
            "roofline": {"bound": "tensor", "kernel": KERNEL_NAMES.get(dominant, dominant),
                         "achieved": dom.get("tflops"), "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                         "frac": dom.get("frac"), "peak_source": f"{peak_src} bf16_tflops_sustained",
                         "traffic": dom_traffic,
                         "launches_per_step": dom.get("launches"), "ms_per_step": dom.get("ms"),
                         "flops_per_launch": dom["flops"] / dom["launches"] if dom else None,
                         "method": "algorithmic FLOPs of each launch (2*pixels*taps*Cin*Cout, 2*M*N*K) / its CUDA-event "
                                   "duration in a profiling pass on the launching stream; traffic = ncu "
                                   "dram__bytes_read+write per launch of the same kernel (profiles/traffic_vgg16.json)",
                         "by_kind": {kk: {"launches": v["launches"], "ms": round(v["ms"], 4),
                                          "tflops": round(v["tflops"], 1) if v["tflops"] else None,
                                          "frac": round(v["frac"], 3) if v["frac"] else None}
                                     for kk, v in sorted(by_kind.items(), key=lambda kv: -kv[1]["ms"])},
                         "hbm_bound": {"peak_gbs": peaks["hbm_gbs"], "peak_source": f"{peak_src} hbm_gbs",
                                       "note": "algorithmic bytes per launch (each operand once) / CUDA-event time; "
                                               "the first conv (K=27), the FC GEMMs at M=W*b rows, max-pool "
                                               "backward and SGD are HBM-bound",
                                       "by_kind": hbm_view},
                         "nvlink": nvlink,
                         "step": {"achieved": step_achieved,
                                  "frac": step_achieved / peaks["bf16_tflops_sustained"] if step_achieved else None,
                                  "flops": flops_rank, "tensor_ms": step_ms,
                                  "note": "compute_load() FLOPs of the step (reference 3x-forward convention) / "
                                          "summed durations of all tensor-core launches"}},
            "e2e": {"value": e2e_value, "unit": "images/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": 4,
                    "ms_per_step": ms_e2e},
            "gpu_launches": st.launches * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-fp32", action="store_true", help="skip the parity-precision comparator")
    ap.add_argument("--no-resnet", action="store_true", help="skip the ResNet-50 comparator")
    ap.add_argument("--no-branchy", action="store_true", help="skip the Inception-v3 / GoogLeNet comparators")
    ap.add_argument("--quick", action="store_true", help="headline line only (no comparators / CPU baseline)")
    ap.add_argument("--model", default=MODEL, help="catalog model (BASELINE configs: vgg16 headline, alexnet)")
    ap.add_argument("--batch", type=int, default=BATCH, help="per-worker batch")
    args = ap.parse_args()
    globals()["MODEL"] = args.model
    globals()["BATCH"] = args.batch
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
