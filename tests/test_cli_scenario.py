"""CLI and scenario documents (mirrors the reference's tests/test_cli.py and the
scenario parser cases of tests/test_simulator.py).  CPU tests cover the planner
commands, the scenario grammar/validation and the analytic prediction; the
`run` command executes a scenario on the GPU (marked gpu)."""
import json
from pathlib import Path

import pytest

from paper_1901_05803_b200 import scenario as S
from paper_1901_05803_b200.cli import EXIT_BAD_FLAG, EXIT_CAPACITY, EXIT_OK, EXIT_PARSE, EXIT_UNKNOWN_CATALOG, main
from paper_1901_05803_b200.planner import (JobSpec, Strategy, catalog_lookup, compute_load, volume_ralp,
                                           volumes_for)

GIB = 1 << 30


def cli(capsys, *argv):
    code = main(list(argv))
    c = capsys.readouterr()
    return code, c.out, c.err


def test_split_vgg11_and_vgg16(capsys):
    code, out, _ = cli(capsys, "split", "vgg11")
    assert code == EXIT_OK and json.loads(out)["split_index"] == 13        # reference tests/test_cli.py:65-71
    code, out, _ = cli(capsys, "split", "vgg16")
    assert json.loads(out)["split_index"] == 18 and json.loads(out)["split_cost_bytes"] == 71_703_808


def test_profile_errors(capsys, tmp_path):
    assert cli(capsys, "profile", "missing.model")[0] == EXIT_PARSE
    code, _, err = cli(capsys, "profile", "nosuchnet")
    assert code == EXIT_UNKNOWN_CATALOG and "vgg11" in err
    bad = tmp_path / "bad.model"
    bad.write_text("model x batch=1 input=4\noops\n")
    code, _, err = cli(capsys, "profile", str(bad))
    assert code == EXIT_PARSE and "line 2" in err
    assert cli(capsys, "profile", "vgg11", "--mode", "sideways")[0] == EXIT_BAD_FLAG


def test_profile_byte_stable(capsys):
    assert cli(capsys, "profile", "vgg16")[1] == cli(capsys, "profile", "vgg16")[1]


def test_volumes(capsys):
    code, out, _ = cli(capsys, "volumes", "vgg11", "--workers", "8", "--strategies", "all")
    rows = out.strip().split("\n")[1:]
    totals = {r.split(",")[1]: int(r.split(",")[3]) for r in rows}
    assert code == EXIT_OK and totals["ralp"] == min(totals.values())
    code, out, _ = cli(capsys, "volumes", "vgg16", "--workers", "1,8", "--strategies", "ralp", "--format", "json")
    assert [r["total_bytes"] for r in json.loads(out)] == [143_407_616, 1_147_260_928]
    assert cli(capsys, "volumes", "vgg11", "--strategies", "gossip")[0] == EXIT_BAD_FLAG
    assert cli(capsys, "volumes", "vgg11", "--workers", "eight")[0] == EXIT_BAD_FLAG
    code, out, _ = cli(capsys, "volumes", "--reproduce-table3")
    rows = dict(l.split(",", 1) for l in out.strip().split("\n")[1:])
    assert rows["vgg11"].endswith("6.93")                                     # reference test_cli.py:121-125


def test_catalog(capsys):
    code, out, _ = cli(capsys, "catalog", "--json")
    names = [m["name"] for m in json.loads(out)]
    assert code == EXIT_OK and {"vgg16", "alexnet", "cifar_small"} <= set(names)


SCN_16 = """# 15 workers + 1 PS across an 8x4 cluster (spread policy)
cluster machines=8 gpus=4 flops=8e12 memcopy=8e9 link=2e9 intra=6.4e10
job vgg11 model=vgg11 strategy=ralp workers=15 ps=1 split=auto
steps 3
"""


def test_scenario_spread_matches_reference_policy():
    scn = S.parse_scenario(SCN_16, catalog_lookup)
    j = scn.jobs[0]
    assert scn.steps == 3 and j.spec.strategy.split_index == 13
    # least-loaded machine first, workers before PS (simulator.py:123-160)
    assert j.placement.workers[:9] == ((0, 0), (1, 0), (2, 0), (3, 0), (4, 0), (5, 0), (6, 0), (7, 0), (0, 1))
    assert j.placement.ps == ((7, 1),)


def test_scenario_explicit_places_and_errors():
    txt = ("cluster machines=1 gpus=5\njob a model=cifar_small strategy=ralp workers=2\n"
           "place a worker 0 0 3\nplace a worker 1 0 1\nplace a ps 0 0 0\n"
           "job b model=cifar_small strategy=baseline workers=1\n")
    scn = S.parse_scenario(txt, catalog_lookup)
    assert scn.jobs[0].placement.workers == ((0, 3), (0, 1)) and scn.jobs[1].placement == S.Placement(((0, 2),), ((0, 4),))
    bad = [("job a model=vgg11 strategy=gossip workers=1", S.ScenarioError),
           ("job a model=vgg11 workers=1", S.ScenarioError),
           ("frobnicate", S.ScenarioError),
           ("steps 0\njob a model=vgg11 strategy=ring workers=1", S.ScenarioError),
           ("cluster machines=1 gpus=2\njob a model=vgg11 strategy=ring workers=3", S.CapacityError),
           ("cluster machines=1 gpus=2\njob a model=vgg11 strategy=ring workers=1\nplace a worker 0 0 5",
            S.CapacityError),
           ("job a model=vgg11 strategy=ralp workers=1 split=99", S.ScenarioError),
           ("", S.ScenarioError)]
    for text, exc in bad:
        with pytest.raises(exc):
            S.parse_scenario(text, catalog_lookup)


def test_run_cli_parse_errors(capsys, tmp_path):
    assert cli(capsys, "run", "nope.scn")[0] == EXIT_PARSE
    p = tmp_path / "x.scn"
    p.write_text("cluster machines=1 gpus=1\njob a model=vgg16 strategy=ring workers=2\n")
    assert cli(capsys, "run", str(p), "--predict-only")[0] == EXIT_CAPACITY
    assert cli(capsys, "run", "vgg16_b200_ralp.scn", "--steps", "0")[0] == EXIT_PARSE


def test_prediction_is_the_analytic_model(capsys):
    m = catalog_lookup("vgg16")
    spec = JobSpec(m, Strategy.ralp(18), 4)
    sb = S.predict_step(spec, S.B200_NODE)
    wf, pf = compute_load(m, 18, 4)
    assert sb.worker_computation[0] == pytest.approx(wf / 0.99e15)
    assert sb.ps_computation[0] == pytest.approx(pf / 0.99e15) and sb.ps_computation[1] == 0.0
    assert sb.communication[0] == pytest.approx(volume_ralp(m, 18, 4).total_bytes_per_step / 4 / 550e9)
    assert sb.memcopy[0] == pytest.approx(128 * 224 * 224 * 3 * 4 / 50e9)
    code, out, _ = cli(capsys, "run", "vgg16_b200_compare.scn", "--predict-only")
    assert code == EXIT_OK and len(out.strip().split("\n")) == 3 and "predicted_images_per_sec" in out


def test_measured_report_schema_roundtrip():
    from paper_1901_05803_b200.report import JobReport, StepBreakdown
    st = StepBreakdown(job="j", step=1, worker_computation=(0.01, 0.01), ps_computation=(0.001, 0.0),
                       memcopy=(0.0, 0.0), communication=(0.002, 0.002))
    jr = JobReport(job="j", strategy="ralp", worker_count=2, batch_size=8, steps=(st,), bytes_on_wire_per_step=5,
                   losses=(2.3,))
    rep = S.MeasuredReport(jobs=(jr,), predicted=(0.0125,), gpus=((0, 1),))
    d = json.loads(rep.to_json())
    assert d["jobs"][0]["predicted_step_time"] == 0.0125 and d["jobs"][0]["images_per_sec"] == jr.images_per_sec
    assert S.job_report_from_dict(d["jobs"][0]) == jr
    assert rep.timeline_csv().splitlines()[0].startswith("job,step,worker,")
    assert len(rep.timeline_csv().splitlines()) == 3


@pytest.mark.gpu
def test_run_scenario_on_gpu(capsys, tmp_path):
    out, tl = tmp_path / "r.json", tmp_path / "t.csv"
    code, text, err = cli(capsys, "run", "cifar_small_1gpu.scn", "--steps", "3", "--warmup", "1", "--out", str(out),
                          "--timeline", str(tl))
    assert code == EXIT_OK, err
    d = json.loads(out.read_text())["jobs"][0]
    m = catalog_lookup("cifar_small")
    assert d["bytes_on_wire_per_step"] == volumes_for(JobSpec(m, Strategy.ralp(4), 1)).total_bytes_per_step
    assert len(d["losses"]) == 3 and all(0.0 < l < 20.0 for l in d["losses"])
    assert d["images_per_sec"] > 0 and d["predicted_step_time"] > 0 and d["gpus"] == [0]
    assert len(tl.read_text().splitlines()) == 1 + 3


@pytest.mark.gpu
def test_simulate_step_measured_on_gpu():
    """The package's drop-in `simulate_step(Scenario)` (simulator.py:773-776) executes one step of
    every job for real and returns its StepBreakdown (every worker's own measured times)."""
    import paper_1901_05803_b200 as pkg
    m = catalog_lookup("cifar_small").with_batch_size(64)
    spec = JobSpec(m, Strategy.ralp(4), 1)
    cluster = pkg.ClusterSpec(machines=1, gpus_per_machine=2, gpu_flops_per_sec=1e15, memcopy_bytes_per_sec=50e9,
                              link_bytes_per_sec=450e9, intra_machine_bytes_per_sec=450e9)
    pl = pkg.spread_placement(cluster, [(1, 1)])[0]
    scn = pkg.Scenario(cluster, (S.ScenarioJob("j", spec, pl, "cifar_small"),), steps=1)
    (sb,) = pkg.simulate_step(scn, warmup=1)
    assert len(sb.worker_computation) == 1 and sb.worker_computation[0] > 0 and sb.memcopy == (0.0,)
