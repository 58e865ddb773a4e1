"""CPU tests of the host side: the C-ABI library loads and exports every symbol
include/ralpb.h declares (no compute calls without a GPU), the lowering of the
planner graph to the ABI layer table, the oracle step's schedule invariants, and
the multi-rank handle exchange over gloo (world_size 2)."""
import os
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import step as ostep
from paper_1901_05803_b200 import _lib, synthetic
from paper_1901_05803_b200.executor import allgather_bytes, lower
from paper_1901_05803_b200.planner import catalog_lookup, parse_model, volume_baseline, volume_ralp

ROOT = Path(__file__).resolve().parent.parent


def _declared():
    text = (ROOT / "include" / "ralpb.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ralpb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES), "ctypes table out of sync with include/ralpb.h"
    assert lib.ralpb_version() == 1


def _header_struct_fields(name):
    """Field names of `typedef struct { ... } name;` in include/ralpb.h, in order."""
    text = re.sub(r"/\*.*?\*/", "", (ROOT / "include" / "ralpb.h").read_text(), flags=re.S)
    body = re.search(r"typedef struct \{([^}]*)\}\s*" + name + r"\s*;", text).group(1)
    fields = []
    for decl in body.split(";"):
        decl = decl.strip()
        if not decl:
            continue
        names = decl.split(None, 1)[1] if not decl.startswith(("long long", "unsigned")) else decl.split(None, 2)[2]
        fields += [n.strip().lstrip("*") for n in names.split(",")]
    return fields


def test_abi_structs_match_header():
    for ctype, cname in ((_lib.LayerDesc, "ralpb_layer_desc"), (_lib.NodeDesc, "ralpb_node_desc"),
                         (_lib.StepStats, "ralpb_step_stats"), (_lib.LaunchRec, "ralpb_launch_rec")):
        assert [f for f, _ in ctype._fields_] == _header_struct_fields(cname), cname
    assert _lib.LayerDesc._fields_[-2:] == [("node_begin", C.c_int), ("node_count", C.c_int)]


def test_lowering_vgg16():
    layers = lower(catalog_lookup("vgg16"))
    assert [L["kind"] for L in layers].count("conv") == 13
    assert layers[0] == dict(kind="conv", k=3, stride=1, pad=1, h=224, w=224, cin=3, cout=64, relu=1, name="conv1")
    fc1 = layers[18]
    assert fc1["kind"] == "fc" and fc1["cin"] == 7 * 7 * 512 and fc1["relu"] == 1
    assert layers[-1]["relu"] == 0 and layers[-1]["cout"] == 1000
    alex = lower(catalog_lookup("alexnet"))
    assert (alex[0]["h"], alex[0]["stride"], alex[0]["k"]) == (227, 4, 11)


TINY = """model tiny batch=4 elem_bytes=4 input=16x16x3
c1 conv k=3 cout=16 pad=1
p1 pool window=2
c2 conv k=3 cout=32 pad=1
p2 pool window=2
f1 fc out=64
f2 fc out=10
"""


def _oracle_run(strategy, workers, b, steps=2, bf=False):
    m = parse_model(TINY)
    layers = lower(m)
    p0 = synthetic.init_params(layers, 3)
    st = ostep.OracleState(layers, p0)
    losses, wires = [], []
    for t in range(steps):
        batches = [synthetic.batch(3, t, r * b, b, (16, 16, 3), 10) for r in range(workers)]
        loss, wire = ostep.train_step(st, strategy, workers, batches, emulate_bf16=bf)
        losses.append(loss)
        wires.append(wire)
    return m, losses, wires, st.numpy_params()


def test_oracle_byte_counter_matches_cost_model():
    for w in (1, 2, 3):
        m, _, wires, _ = _oracle_run("ralp", w, 4)
        assert wires[0] == volume_ralp(m.with_batch_size(4), 4, w).total_bytes_per_step
        m, _, wires, _ = _oracle_run("baseline", w, 4)
        assert wires[0] == volume_baseline(m, w).total_bytes_per_step


def test_placements_are_mathematically_equivalent():
    """RALP with W workers == baseline with W workers == RALP W=1 on the concatenated batch
    (fp32, up to summation order): placement changes where the work runs, not the result."""
    _, l_r2, _, p_r2 = _oracle_run("ralp", 2, 4)
    _, l_b2, _, p_b2 = _oracle_run("baseline", 2, 4)
    np.testing.assert_allclose(l_r2, l_b2, rtol=1e-5)
    for a, b in zip(p_r2, p_b2):
        if a is not None:
            np.testing.assert_allclose(a[0], b[0], rtol=1e-4, atol=1e-6)
    # W=1 with b=8 over the same 8 global samples (worker r owns samples r*4..r*4+3)
    m = parse_model(TINY)
    layers = lower(m)
    st = ostep.OracleState(layers, synthetic.init_params(layers, 3))
    for t in range(2):
        imgs, labs = synthetic.batch(3, t, 0, 8, (16, 16, 3), 10)
        ostep.train_step(st, "ralp", 1, [(imgs, labs)])
    for a, b in zip(st.numpy_params(), p_r2):
        if a is not None:
            np.testing.assert_allclose(a[0], b[0], rtol=1e-4, atol=1e-6)


def test_synthetic_data_is_placement_independent():
    a, la = synthetic.batch(0, 5, 0, 8, (4, 4, 3), 10)
    b1, lb1 = synthetic.batch(0, 5, 0, 4, (4, 4, 3), 10)
    b2, lb2 = synthetic.batch(0, 5, 4, 4, (4, 4, 3), 10)
    np.testing.assert_array_equal(a, np.concatenate([b1, b2]))
    np.testing.assert_array_equal(la, np.concatenate([lb1, lb2]))


def _gloo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    got = allgather_bytes(bytes([rank]) * 64)
    q.put((rank, got))
    dist.destroy_process_group()


def test_handle_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + os.getpid() % 1000
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(60)
    for r in range(2):
        assert res[r] == [bytes([0]) * 64, bytes([1]) * 64]


def _report_worker(rank, world, port, q, placement):
    """One rank of run_job's report assembly (executor._allgather_rows + _breakdown) over gloo."""
    from paper_1901_05803_b200.executor import _allgather_rows, _breakdown
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # row: [step, ms_step, ms_front (fwd + bwd), ms_back, is_worker, holds_back]
    dedicated = placement == "dedicated-ps"
    is_worker = not (dedicated and rank == 0)
    row = [1.0, 10.0 + rank, 6.0 + rank if is_worker else 0.0, 2.0 if rank == 0 else 0.0, float(is_worker),
           float(rank == 0)]
    rows = _allgather_rows(row, world)
    bd = _breakdown("job", 1, rows, "ralp")
    q.put((rank, rows, bd.worker_computation, bd.ps_computation, bd.communication, bd.memcopy))
    dist.destroy_process_group()


@pytest.mark.parametrize("placement", ["colocated", "dedicated-ps"])
def test_report_rows_gloo_world2(placement):
    """run_job's per-worker report at world 2: every rank gathers every rank's measured row in rank
    order and charges times per worker (the colocated PS's back segment to worker 0; a dedicated PS's
    to the workers in equal shares)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29600 + os.getpid() % 1000 + (7 if placement == "dedicated-ps" else 0)
    procs = [ctx.Process(target=_report_worker, args=(r, 2, port, q, placement)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=120) for _ in range(2)))
    for p in procs:
        p.join(60)
    assert res[0] == res[1]   # every rank holds the same report
    rows, comp, ps, comm, mem = res[0]
    assert [r[1] for r in rows] == [10.0, 11.0]
    if placement == "colocated":
        assert comp == pytest.approx((6e-3, 7e-3)) and ps == pytest.approx((2e-3, 0.0))
        assert comm == pytest.approx((10e-3 - 6e-3 - 2e-3, 11e-3 - 7e-3))
        assert mem == (0.0, 0.0)
    else:   # one worker (rank 1); the dedicated PS's 2 ms charged to it
        assert comp == pytest.approx((7e-3,)) and ps == pytest.approx((2e-3,)) and mem == (0.0,)
