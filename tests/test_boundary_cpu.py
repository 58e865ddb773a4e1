"""The drop-in boundary on the CPU: jobs built with the UNMODIFIED reference package
(`ralp.ModelGraph`, `ralp.JobSpec`; pkg/src/ralp/costmodel.py:64-86) lower and are costed exactly
like the mirror's; placement arguments are validated before any device call; the per-rank report
rows are gathered over gloo (world_size 2 and 3) and folded into the reference's four categories
with every worker's own numbers."""
import os
import sys
from pathlib import Path

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1901_05803_b200.executor import ExecutorError, RankExecutor, _allgather_rows, _breakdown, expected_volume, lower
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, volume_baseline, volume_ralp, volume_ring

REF = Path("/root/reference/pkg/src")


@pytest.fixture(scope="module")
def ralp():
    if not (REF / "ralp" / "__init__.py").exists():
        pytest.skip("the reference package is not present on this machine")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.path.insert(0, str(REF))
    sys.dont_write_bytecode = True
    try:
        import ralp as mod
    finally:
        sys.path.remove(str(REF))
    return mod


@pytest.mark.parametrize("name", ["vgg11", "vgg16", "alexnet", "cifar_small", "overfeat", "lenet", "resnet-50",
                                  "inception-v3", "googlenet"])
def test_reference_model_graph_lowers_like_the_mirror(ralp, name):
    try:
        ref_model = ralp.catalog_lookup(name)
    except KeyError:
        pytest.skip(f"{name} is not in the reference catalog (mirror-only descriptor)")
    assert lower(ref_model) == lower(catalog_lookup(name))


def test_reference_jobspec_volumes(ralp):
    m = ralp.catalog_lookup("vgg11").with_batch_size(128)
    split = ralp.profile(m).split_index
    for w in (1, 2, 4, 8):
        assert expected_volume(ralp.JobSpec(m, ralp.Strategy.ralp(split), w)) == \
            ralp.volume_ralp(m, split, w).total_bytes_per_step
        assert expected_volume(ralp.JobSpec(m, ralp.Strategy.baseline(), w)) == \
            ralp.volume_baseline(m, w).total_bytes_per_step
        assert expected_volume(ralp.JobSpec(m, ralp.Strategy.ring(), w, ps_count=0)) == \
            ralp.volume_ring(m, w).total_bytes_per_step
    # and the mirror's own figures are the same numbers
    mm = catalog_lookup("vgg11").with_batch_size(128)
    assert volume_ralp(mm, split, 4).total_bytes_per_step == ralp.volume_ralp(m, split, 4).total_bytes_per_step
    assert volume_baseline(mm, 4).total_bytes_per_step == ralp.volume_baseline(m, 4).total_bytes_per_step
    assert volume_ring(mm, 4).total_bytes_per_step == ralp.volume_ring(m, 4).total_bytes_per_step


def test_placement_validation_before_any_device_call():
    m = catalog_lookup("cifar_small").with_batch_size(8)
    job = JobSpec(m, Strategy.ralp(4), 2)
    with pytest.raises(ExecutorError, match="world size"):
        RankExecutor(job, world=2, placement="dedicated-ps")     # RALP-N needs W + 1 ranks
    with pytest.raises(ExecutorError, match="world size"):
        RankExecutor(job, world=3)                               # colocated: one rank per worker
    with pytest.raises(ExecutorError, match="dedicated PS"):
        RankExecutor(JobSpec(m, Strategy.baseline(), 2), world=3, placement="dedicated-ps")
    with pytest.raises(ExecutorError, match="precision"):
        RankExecutor(job, world=2, precision="fp16")


def test_breakdown_uses_every_workers_own_times():
    # rows: [logical, ms_step, ms_front, ms_back, is_worker, is_ps]
    rows = [[10, 12.0, 9.0, 1.5, 1, 1],     # colocated PS worker
            [20, 12.0, 8.0, 3.0, 1, 0]]     # a remote worker (its "back" is waiting)
    b = _breakdown("j", 1, rows, "ralp")
    assert b.worker_computation == pytest.approx((9e-3, 8e-3))
    assert b.ps_computation == pytest.approx((1.5e-3, 0.0))
    assert b.memcopy == (0.0, 0.0)
    # categories add up to each worker's measured step
    assert b.step_durations == pytest.approx((12e-3, 12e-3))
    # dedicated PS (RALP-N): its tail is charged to the workers in equal shares
    rows = [[5, 4.0, 0.0, 3.0, 0, 1], [1, 12.0, 9.0, 2.0, 1, 0], [1, 12.0, 9.5, 1.5, 1, 0]]
    b = _breakdown("j", 1, rows, "ralp")
    assert len(b.worker_computation) == 2
    assert b.ps_computation == pytest.approx((1.5e-3, 1.5e-3))
    # all-on-PS: the FC tail is worker computation
    b = _breakdown("j", 1, [[1, 10.0, 7.0, 2.0, 1, 1]], "baseline")
    assert b.worker_computation == pytest.approx((9e-3,))


def _rows_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rows = _allgather_rows([float(rank), 10.0 + rank, 5.0, 1.0, 1.0, 1.0 if rank == 0 else 0.0], world)
    q.put((rank, rows))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_report_rows_gather_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + world * 10 + os.getpid() % 50
    procs = [ctx.Process(target=_rows_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(60)
    for r in range(world):
        rows = res[r]
        assert [row[0] for row in rows] == [float(i) for i in range(world)]     # rank order
        assert sum(row[0] for row in rows) == sum(range(world))                 # the byte total


def test_package_surface_covers_the_reference(ralp):
    """Every name the reference package exports (pkg/src/ralp/__init__.py:46-91) is importable
    from this package, except the network simulator's consolidation study (out of scope)."""
    import paper_1901_05803_b200 as pkg
    out_of_scope = {"simulate_consolidation", "ConsolidationReport"}
    missing = [n for n in ralp.__all__ if n not in out_of_scope and not hasattr(pkg, n)]
    assert not missing, missing


def test_reference_scenario_converts_by_value(ralp):
    """A scenario built with the reference's own types (ralp.Scenario of (name, JobSpec, Placement))
    is what simulate_run / simulate_step execute: converted by value, placements and checks kept."""
    from paper_1901_05803_b200.scenario import Scenario, _as_scenario
    model = ralp.catalog_lookup("vgg11").with_batch_size(32)
    split = ralp.profile(model).split_index
    spec = ralp.JobSpec(model, ralp.Strategy.ralp(split), 2)
    pl = ralp.spread_placement(ralp.DEFAULT_CLUSTER, [(2, 1)])[0]
    ref = ralp.Scenario(ralp.DEFAULT_CLUSTER, (("j0", spec, pl),), steps=3)
    mine = _as_scenario(ref)
    assert isinstance(mine, Scenario) and mine.steps == 3
    (job,) = mine.jobs
    assert job.name == "j0" and job.model_ref == "vgg11" and job.spec is spec
    assert job.placement.workers == tuple(map(tuple, pl.workers)) and job.placement.ps == tuple(map(tuple, pl.ps))
    assert mine.cluster.machines == ralp.DEFAULT_CLUSTER.machines
