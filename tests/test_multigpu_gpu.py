"""Multi-GPU layer-placed step (>= 2 GPUs): launches tests/multi_rank_parity.py under
torch.distributed.run; skipped on single-GPU boxes."""
import subprocess
import sys
from pathlib import Path

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_two_rank_parity():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29611", str(ROOT / "tests" / "multi_rank_parity.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0 and "MULTI-RANK PARITY PASS" in r.stdout


def _parity(n: int, port: int, env_extra: dict) -> None:
    import os
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "tests" / "multi_rank_parity.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env={**os.environ, **env_extra})
    print(r.stdout[-4000:], r.stderr[-4000:])
    assert r.returncode == 0 and "MULTI-RANK PARITY PASS" in r.stdout


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_two_rank_parity_per_peer_pushes():
    """The per-peer push kernels (RALPB_SCATTER_FUSED=0, RALPB_PUSH_LEGACY=1) give the same result."""
    _parity(2, 29612, {"RALPB_SCATTER_FUSED": "0", "RALPB_PUSH_LEGACY": "1"})


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 4, reason="needs >= 4 GPUs")
def test_four_rank_parity_fused_scatter():
    """W=4: the act-grad return to three workers in one scatter launch (exchange.cu scatter_kernel)."""
    _parity(4, 29613, {})


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs >= 2 GPUs")
def test_cli_run_scenario_two_gpus(tmp_path):
    """`run` on a bundled two-worker scenario: layer-placed, all-on-PS and ring jobs executed on
    two B200s, each reporting the oracle's logical bytes."""
    from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, volumes_for

    out = tmp_path / "r.json"
    cmd = [sys.executable, "-m", "paper_1901_05803_b200", "run", "vgg16_b200_compare.scn", "--steps", "2",
           "--warmup", "1", "--out", str(out)]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=str(ROOT))
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0
    import json
    jobs = {j["job"]: j for j in json.loads(out.read_text())["jobs"]}
    m = catalog_lookup("vgg16").with_batch_size(128)
    want = {"ralp": volumes_for(JobSpec(m, Strategy.ralp(18), 2)).total_bytes_per_step,
            "allps": volumes_for(JobSpec(m, Strategy.baseline(), 2)).total_bytes_per_step,
            "ring": volumes_for(JobSpec(m, Strategy.ring(), 2, ps_count=0)).total_bytes_per_step}
    for name, b in want.items():
        assert jobs[name]["bytes_on_wire_per_step"] == b
        assert jobs[name]["worker_count"] == 2 and len(jobs[name]["losses"]) == 2
        assert jobs[name]["images_per_sec"] > 1000
