"""Scenario files and the measured-run backend.

The reference drives its event simulator from `.scn` scenario documents
(pkg/src/ralp/simulator.py:827-969: `cluster`, `job`, `place`, `steps`
directives) and prints a `SimReport` (simulator.py:233-282).  Here the same
documents are parsed with the same grammar, validation and error classes, and
every job is then *executed* on this node's B200s through `run_job` (one process
per GPU, torch.distributed over NCCL + the engine's NVLink peer-memory
exchange).  The measured report keeps the reference's schema and adds, per job,
the step time predicted by the analytic model on a B200-calibrated
`ClusterSpec` (`B200_NODE`), so prediction and measurement sit side by side.

Placement on real hardware:
  * one machine: every `place` slot must name machine 0 and an existing GPU;
  * the PS of a RALP job is colocated with worker 0 (the paper's RALP-H
    accounting, costmodel.gpu_assignments); a PS slot given in the scenario is
    validated (capacity / double booking, as in the reference) but the engine
    does not occupy it.  The simulator itself cannot model the colocated PS
    (simulator.py:118-119), which is why prediction uses the same colocated
    arithmetic below rather than the reference's event model.
"""
from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
import tempfile
from dataclasses import dataclass
from pathlib import Path
from typing import Callable, Optional, Sequence

from .planner import (CostModelError, JobSpec, ModelGraph, ProfilerConfig, Strategy, StrategyKind, compute_load,
                      profile, volumes_for)
from .report import JobReport, StepBreakdown


class ScenarioError(ValueError):
    """Malformed scenario document or inconsistent job/placement (simulator.py ScenarioError)."""


class CapacityError(ScenarioError):
    """A placement names a slot outside the cluster or books one twice (simulator.py CapacityError)."""


@dataclass(frozen=True)
class ClusterSpec:
    """Same fields and validation as the reference's ClusterSpec (simulator.py:43-62)."""
    machines: int
    gpus_per_machine: int
    gpu_flops_per_sec: float
    memcopy_bytes_per_sec: float
    link_bytes_per_sec: float
    intra_machine_bytes_per_sec: float

    def __post_init__(self) -> None:
        if self.machines < 1 or self.gpus_per_machine < 1:
            raise ScenarioError("cluster needs at least one machine and one GPU per machine")
        for f in ("gpu_flops_per_sec", "memcopy_bytes_per_sec", "link_bytes_per_sec", "intra_machine_bytes_per_sec"):
            if not getattr(self, f) > 0:
                raise ScenarioError(f"cluster rate {f} must be > 0")

    @property
    def total_gpus(self) -> int:
        return self.machines * self.gpus_per_machine


# Defaults of a `cluster` line that omits keys: the reference's 8x4 testbed rates
# (simulator.py:69-76), so that scenario documents parse to the same specs.
DEFAULT_CLUSTER = ClusterSpec(machines=8, gpus_per_machine=4, gpu_flops_per_sec=8.0e12,
                              memcopy_bytes_per_sec=8.0e9, link_bytes_per_sec=2.0e9,
                              intra_machine_bytes_per_sec=6.4e10)

# One 8x B200 NVSwitch node, calibrated from this repo's own measurements
# (profiles/r01/bench_n1.json): effective tensor rate of the
# whole VGG-16 step (compute_load FLOPs / summed tcgen05 launch time ~0.99
# PFLOP/s), pinned-host->HBM copy ~50 GB/s, NVLink peer push/shard-update
# goodput ~550 GB/s per GPU (single node: no inter-machine link, same figure).
B200_NODE = ClusterSpec(machines=1, gpus_per_machine=8, gpu_flops_per_sec=0.99e15,
                        memcopy_bytes_per_sec=50e9, link_bytes_per_sec=550e9,
                        intra_machine_bytes_per_sec=550e9)


@dataclass(frozen=True)
class Placement:
    """(machine, gpu) per worker replica and PS process (simulator.py:79-84)."""
    workers: tuple[tuple[int, int], ...]
    ps: tuple[tuple[int, int], ...] = ()


@dataclass(frozen=True)
class ScenarioJob:
    name: str
    spec: JobSpec
    placement: Placement
    model_ref: str            # catalog name or absolute descriptor path (re-resolved by the rank processes)


@dataclass(frozen=True)
class Scenario:
    cluster: ClusterSpec
    jobs: tuple[ScenarioJob, ...]
    steps: int = 1

    def __post_init__(self) -> None:
        # the reference's checks, in its order (simulator.py:95-122)
        if self.steps < 1:
            raise ScenarioError("steps must be >= 1")
        if not self.jobs:
            raise ScenarioError("scenario has no jobs")
        names = [j.name for j in self.jobs]
        if len(set(names)) != len(names):
            raise ScenarioError("duplicate job names")
        seen: set[tuple[int, int]] = set()
        for j in self.jobs:
            if len(j.placement.workers) != j.spec.worker_count:
                raise ScenarioError(f"job {j.name}: placement covers {len(j.placement.workers)} workers, "
                                    f"spec wants {j.spec.worker_count}")
            if len(j.placement.ps) != j.spec.ps_count:
                raise ScenarioError(f"job {j.name}: placement covers {len(j.placement.ps)} PS processes, "
                                    f"spec wants {j.spec.ps_count}")
            for machine, gpu in (*j.placement.workers, *j.placement.ps):
                if not 0 <= machine < self.cluster.machines:
                    raise CapacityError(f"job {j.name}: machine {machine} outside cluster")
                if not 0 <= gpu < self.cluster.gpus_per_machine:
                    raise CapacityError(f"job {j.name}: gpu {gpu} outside machine")
                if (machine, gpu) in seen:
                    raise CapacityError(f"job {j.name}: slot ({machine}, {gpu}) double-booked")
                seen.add((machine, gpu))


def spread_placement(cluster: ClusterSpec, replica_counts: Sequence[tuple[int, int]],
                     taken: Sequence[tuple[int, int]] = ()) -> list[Placement]:
    """The reference's spread policy (simulator.py:123-160): workers, then PS processes, each on
    the least-loaded machine that still has a free slot (ties to the lower machine index),
    lowest free GPU index within it."""
    occupied = set(taken)
    load = [0] * cluster.machines
    for machine, _ in occupied:
        load[machine] += 1
    cursor = [0] * cluster.machines

    def claim() -> tuple[int, int]:
        for m in sorted(range(cluster.machines), key=lambda i: (load[i], i)):
            while cursor[m] < cluster.gpus_per_machine:
                slot = (m, cursor[m])
                cursor[m] += 1
                if slot not in occupied:
                    occupied.add(slot)
                    load[m] += 1
                    return slot
        raise CapacityError(f"cluster is full: {cluster.total_gpus} slots cannot host the requested replicas")

    out = []
    for w, p in replica_counts:
        ws = tuple(claim() for _ in range(w))
        out.append(Placement(workers=ws, ps=tuple(claim() for _ in range(p))))
    return out


def _kv(tokens: Sequence[str]) -> dict[str, str]:
    return dict(t.split("=", 1) for t in tokens if "=" in t)


def parse_scenario(text: str, resolve_model: Callable[[str], ModelGraph], default_steps: int = 1,
                   ref_of: Optional[Callable[[str], str]] = None) -> Scenario:
    """Parse a scenario document (grammar of simulator.py:827-969).

    `resolve_model(ref)` turns a `model=` token into a ModelGraph; `ref_of(ref)`
    (default: identity) gives the reference the rank processes re-resolve."""
    cluster: Optional[ClusterSpec] = None
    steps = default_steps
    job_lines: list[tuple[str, dict[str, str]]] = []
    explicit: dict[str, dict[str, dict[int, tuple[int, int]]]] = {}

    def fail(lineno: int, msg: str):
        raise ScenarioError(f"line {lineno}: {msg}")

    for lineno, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        tok = line.split()
        head = tok[0]
        if head == "cluster":
            kv = _kv(tok[1:])
            d = DEFAULT_CLUSTER
            try:
                cluster = ClusterSpec(machines=int(kv.get("machines", d.machines)),
                                      gpus_per_machine=int(kv.get("gpus", d.gpus_per_machine)),
                                      gpu_flops_per_sec=float(kv.get("flops", d.gpu_flops_per_sec)),
                                      memcopy_bytes_per_sec=float(kv.get("memcopy", d.memcopy_bytes_per_sec)),
                                      link_bytes_per_sec=float(kv.get("link", d.link_bytes_per_sec)),
                                      intra_machine_bytes_per_sec=float(kv.get("intra",
                                                                                 d.intra_machine_bytes_per_sec)))
            except (ValueError, ScenarioError) as exc:
                fail(lineno, f"bad cluster spec: {exc}")
        elif head == "job":
            if len(tok) < 3:
                fail(lineno, "job line needs a name and key=value pairs")
            kv = _kv(tok[2:])
            for req in ("model", "strategy", "workers"):
                if req not in kv:
                    fail(lineno, f"job {tok[1]!r} needs {req}=")
            job_lines.append((tok[1], kv))
        elif head == "place":
            if len(tok) < 3:
                fail(lineno, "place line needs a job name")
            slot = explicit.setdefault(tok[1], {"worker": {}, "ps": {}})
            if tok[2] == "spread":
                continue
            if len(tok) != 6 or tok[2] not in ("worker", "ps"):
                fail(lineno, "expected: place <job> worker|ps <idx> <machine> <gpu>")
            try:
                slot[tok[2]][int(tok[3])] = (int(tok[4]), int(tok[5]))
            except ValueError:
                fail(lineno, "place indices must be integers")
        elif head == "steps":
            if len(tok) != 2:
                fail(lineno, "expected: steps <n>")
            try:
                steps = int(tok[1])
            except ValueError:
                fail(lineno, "steps must be an integer")
            if steps < 1:
                fail(lineno, "steps must be >= 1")
        else:
            fail(lineno, f"unknown directive {head!r}")

    cluster = cluster or DEFAULT_CLUSTER
    if not job_lines:
        raise ScenarioError("scenario has no jobs")

    specs: list[tuple[str, JobSpec, str]] = []
    for name, kv in job_lines:
        model = resolve_model(kv["model"])
        if "batch" in kv:
            model = model.with_batch_size(int(kv["batch"]))
        workers = int(kv["workers"])
        kind = kv["strategy"]
        try:
            if kind == "baseline":
                spec = JobSpec(model, Strategy.baseline(), workers, int(kv.get("ps", 1)))
            elif kind == "ring":
                spec = JobSpec(model, Strategy.ring(), workers, int(kv.get("ps", 0)))
            elif kind == "ralp":
                tokn = kv.get("split", "auto")
                if tokn == "auto":
                    rep = profile(model, ProfilerConfig())
                    if rep.split_index is None:
                        raise ScenarioError(f"job {name!r}: model {model.name} is not partitionable "
                                            "(skewness gate failed); use strategy=baseline")
                    split = rep.split_index
                else:
                    split = int(tokn)
                spec = JobSpec(model, Strategy.ralp(split), workers, int(kv.get("ps", 1)))
            else:
                raise ScenarioError(f"job {name!r}: unknown strategy {kind!r}")
        except CostModelError as exc:
            raise ScenarioError(f"job {name!r}: {exc}") from exc
        specs.append((name, spec, (ref_of or (lambda r: r))(kv["model"])))

    taken = [s for n, _, _ in specs if n in explicit for grp in explicit[n].values() for s in grp.values()]
    auto = [(n, s) for n, s, _ in specs if n not in explicit]
    auto_map = dict(zip([n for n, _ in auto],
                        spread_placement(cluster, [(s.worker_count, s.ps_count) for _, s in auto], taken=taken)))
    jobs = []
    for name, spec, ref in specs:
        if name in explicit:
            w, p = explicit[name]["worker"], explicit[name]["ps"]
            if sorted(w) != list(range(spec.worker_count)):
                raise ScenarioError(f"job {name!r}: worker placements must cover 0..{spec.worker_count - 1}")
            if sorted(p) != list(range(spec.ps_count)):
                raise ScenarioError(f"job {name!r}: ps placements must cover 0..{spec.ps_count - 1}")
            placement = Placement(workers=tuple(w[i] for i in range(spec.worker_count)),
                                  ps=tuple(p[i] for i in range(spec.ps_count)))
        else:
            placement = auto_map[name]
        jobs.append(ScenarioJob(name, spec, placement, ref))
    return Scenario(cluster=cluster, jobs=tuple(jobs), steps=steps)


# ----------------------------------------------------------------------------- prediction

def predict_step(spec: JobSpec, cluster: ClusterSpec = B200_NODE) -> StepBreakdown:
    """Analytic step time of the colocated-PS execution on `cluster` (seconds per category).

    worker computation = the worker's compute_load FLOPs / gpu rate; PS computation =
    the PS FLOPs (FC tail over W·b) / gpu rate, charged to worker 0 only (colocated);
    memcopy = one batch of fp32 input images host->device; communication = the
    job's logical bytes per worker / link rate (single machine: the intra-node
    rate)."""
    m, w = spec.model, spec.worker_count
    split = spec.strategy.split_index if spec.strategy.kind is StrategyKind.RALP else None
    worker_flops, ps_flops = compute_load(m, split, w)
    link = cluster.intra_machine_bytes_per_sec if cluster.machines == 1 else cluster.link_bytes_per_sec
    comm = volumes_for(spec).total_bytes_per_step / w / link
    from .executor import ExecutorError, infer_input_shape
    try:
        h, wd, c = infer_input_shape(m)
        in_elems = h * wd * c
    except ExecutorError:
        in_elems = 0
    mem = m.batch_size * in_elems * 4 / cluster.memcopy_bytes_per_sec
    wc = worker_flops / cluster.gpu_flops_per_sec
    ps = ps_flops / cluster.gpu_flops_per_sec
    return StepBreakdown(job=m.name, step=0, worker_computation=(wc,) * w,
                         ps_computation=(ps,) + (0.0,) * (w - 1), memcopy=(mem,) * w, communication=(comm,) * w)


# ----------------------------------------------------------------------------- measured reports

@dataclass(frozen=True)
class MeasuredReport:
    """`SimReport` schema (simulator.py:233-282) for measured jobs; each job dict adds
    `predicted_step_time` (B200_NODE model) and the placement the engine used."""
    jobs: tuple[JobReport, ...]
    predicted: tuple[float, ...] = ()
    gpus: tuple[tuple[int, ...], ...] = ()

    def job(self, name: str) -> JobReport:
        for j in self.jobs:
            if j.job == name:
                return j
        raise KeyError(name)

    def to_dict(self) -> dict:
        out = []
        for i, j in enumerate(self.jobs):
            d = j.to_dict()
            if i < len(self.predicted):
                d["predicted_step_time"] = self.predicted[i]
            if i < len(self.gpus):
                d["gpus"] = list(self.gpus[i])
                d["ps_placement"] = "colocated with worker 0" if j.strategy == "ralp" else "sharded over workers"
            out.append(d)
        return {"backend": "measured-b200", "jobs": out}

    def to_json(self) -> str:
        return json.dumps(self.to_dict(), indent=2)

    def timeline_csv(self) -> str:
        lines = ["job,step,worker,worker_computation,ps_computation,memcopy,communication,step_duration"]
        for j in self.jobs:
            for s in j.steps:
                for w in range(len(s.worker_computation)):
                    lines.append(f"{j.job},{s.step},{w},{s.worker_computation[w]!r},{s.ps_computation[w]!r},"
                                 f"{s.memcopy[w]!r},{s.communication[w]!r},{s.step_duration(w)!r}")
        return "\n".join(lines) + "\n"


def job_report_from_dict(d: dict) -> JobReport:
    steps = tuple(StepBreakdown(job=s["job"], step=s["step"], worker_computation=tuple(s["worker_computation"]),
                                ps_computation=tuple(s["ps_computation"]), memcopy=tuple(s["memcopy"]),
                                communication=tuple(s["communication"])) for s in d["steps"])
    return JobReport(job=d["job"], strategy=d["strategy"], worker_count=d["worker_count"], batch_size=d["batch_size"],
                     steps=steps, bytes_on_wire_per_step=d["bytes_on_wire_per_step"], losses=tuple(d["losses"]))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def local_gpu_count() -> int:
    import torch
    return torch.cuda.device_count()


def job_gpus(job: ScenarioJob, available: int) -> tuple[int, ...]:
    """GPU indices of the job's worker slots on this node (machine 0 only)."""
    gpus = []
    for machine, gpu in job.placement.workers:
        if machine != 0:
            raise CapacityError(f"job {job.name}: measured runs use one machine; slot ({machine}, {gpu}) is remote")
        if gpu >= available:
            raise CapacityError(f"job {job.name}: gpu {gpu} not present (this node has {available})")
        gpus.append(gpu)
    return tuple(gpus)


def run_scenario(scn: Scenario, *, steps: Optional[int] = None, warmup: int = 2, seed: int = 0,
                 timeout: float = 1800.0, available: Optional[int] = None) -> MeasuredReport:
    """Execute every job of `scn` for real, one after another, each on its worker GPUs
    (one process per GPU under torch.distributed.run).  Returns the measured report."""
    steps = steps or scn.steps
    available = local_gpu_count() if available is None else available
    reports, preds, gpus_used = [], [], []
    try:
        placed = [job_gpus(j, available) for j in scn.jobs]
    except CapacityError:
        # a multi-machine scenario: re-spread the workers over this node's GPUs (jobs run one
        # after another, so each may use the whole node; PS roles are colocated)
        if max(j.spec.worker_count for j in scn.jobs) > available:
            raise
        placed = [tuple(range(j.spec.worker_count)) for j in scn.jobs]
    for job, gpus in zip(scn.jobs, placed):
        with tempfile.TemporaryDirectory() as td:
            spec_path, out_path = Path(td) / "spec.json", Path(td) / "report.json"
            spec_path.write_text(json.dumps({
                "name": job.name, "model_ref": job.model_ref, "batch": job.spec.model.batch_size,
                "strategy": job.spec.strategy.kind.value, "split": job.spec.strategy.split_index,
                "workers": job.spec.worker_count, "ps": job.spec.ps_count,
                "steps": steps, "warmup": warmup, "seed": seed}))
            env = dict(os.environ, CUDA_VISIBLE_DEVICES=",".join(str(g) for g in gpus))
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={len(gpus)}", "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
                   "-m", "paper_1901_05803_b200.scenario", str(spec_path), str(out_path)]
            r = subprocess.run(cmd, env=env, timeout=timeout, capture_output=True, text=True,
                               cwd=str(Path(__file__).resolve().parent.parent))
            if r.returncode != 0 or not out_path.is_file():
                raise RuntimeError(f"job {job.name} failed (exit {r.returncode}):\n{r.stdout[-2000:]}\n{r.stderr[-4000:]}")
            reports.append(job_report_from_dict(json.loads(out_path.read_text())))
        preds.append(predict_step(job.spec, scn.cluster).max_step_time)
        gpus_used.append(gpus)
    return MeasuredReport(jobs=tuple(reports), predicted=tuple(preds), gpus=tuple(gpus_used))


def resolve_model_ref(ref: str, batch: Optional[int] = None) -> ModelGraph:
    from .planner import catalog_lookup, parse_model
    if ref.endswith(".model") or "/" in ref:
        g = parse_model(Path(ref).read_text())
    else:
        g = catalog_lookup(ref)
    return g if batch is None else g.with_batch_size(batch)


def _rank_main(spec_path: str, out_path: str) -> int:
    """One rank of a measured job (launched by run_scenario under torch.distributed.run)."""
    import torch
    import torch.distributed as dist
    from .executor import run_job

    s = json.loads(Path(spec_path).read_text())
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    model = resolve_model_ref(s["model_ref"], s["batch"])
    strat = {"ralp": lambda: Strategy.ralp(s["split"]), "baseline": Strategy.baseline, "ring": Strategy.ring}
    spec = JobSpec(model, strat[s["strategy"]](), s["workers"], s["ps"])
    rep = run_job(spec, steps=s["steps"], warmup=s["warmup"], seed=s["seed"], name=s["name"])
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    if int(os.environ.get("RANK", "0")) == 0:
        Path(out_path).write_text(json.dumps(rep.to_dict()))
    return 0


__all__ = ["B200_NODE", "CapacityError", "ClusterSpec", "DEFAULT_CLUSTER", "MeasuredReport", "Placement", "Scenario",
           "ScenarioError", "ScenarioJob", "job_gpus", "job_report_from_dict", "parse_scenario", "predict_step",
           "resolve_model_ref", "run_scenario", "spread_placement"]

if __name__ == "__main__":
    raise SystemExit(_rank_main(sys.argv[1], sys.argv[2]))


def _as_scenario(scn) -> Scenario:
    """This module's Scenario, or the reference's (`ralp.Scenario`: jobs as (name, JobSpec, Placement)
    tuples over a catalog model) converted by value."""
    if isinstance(scn, Scenario):
        return scn
    c = scn.cluster
    cluster = ClusterSpec(**{f: getattr(c, f) for f in ClusterSpec.__dataclass_fields__ if hasattr(c, f)})
    jobs = []
    for name, spec, pl in scn.jobs:
        jobs.append(ScenarioJob(name=name, spec=spec, placement=Placement(tuple(map(tuple, pl.workers)),
                                                                         tuple(map(tuple, pl.ps))),
                                model_ref=spec.model.name))
    return Scenario(cluster=cluster, jobs=tuple(jobs), steps=scn.steps)


def simulate_run(scenario, **kw) -> MeasuredReport:
    """The drop-in for the reference's `simulate_run(Scenario) -> SimReport` (simulator.py:743-770),
    MEASURED instead of simulated: every job of the scenario (this module's, or the reference's own
    `ralp.Scenario` over catalog models) runs for real on this node's B200s (run_scenario) and the
    report has the SimReport schema (`to_dict` / `to_json` / `timeline_csv`)."""
    return run_scenario(_as_scenario(scenario), **kw)


def simulate_step(scenario, **kw) -> list:
    """`simulate_step` (simulator.py:773-776), measured: one step per job, its StepBreakdown."""
    rep = run_scenario(_as_scenario(scenario), steps=1, **kw)
    return [j.steps[0] for j in rep.jobs]


SimReport = MeasuredReport
