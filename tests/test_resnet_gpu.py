"""ResNet-50 executed: the catalog's linearised resnet-50 lowered at block
granularity (paper_1901_05803_b200/resnet.py: stem 7x7/2 + batch norm, 3x3/2 max pool with
padding, sixteen bottleneck blocks with batch-normalised 1x1 / 3x3(stride) / 1x1 convolutions and
identity or projection shortcuts, global average pool, FC) and run through the C ABI, against the
oracle's autograd restatement of the same graph with bf16 storage emulated at the GPU's storage
points (oracle/step.py `_train_step_branchy`).

  * split 55 (apool | fc, the partitioner's choice at b=128): the FC tail on the PS;
  * split 2 (pool1 | s1b1.., the partitioner's choice at b=64): every block runs on the PS over the
    gathered rows (a conv back segment with batch norm);
  * all-on-PS baseline.
Bytes: the ranks' count_wire-site counts == volume_ralp / volume_baseline of the catalog model.

Numerics.  At b=8 with batch norm and bf16 storage the step is chaotic: the oracle's own
fp32-vs-fp64 spread after two steps is ~1.2x the update itself, so a free-running comparison cannot
discriminate.  The free-running tests therefore check the bytes, the first step's loss (forward
only, 5e-3) and parameters within 2 * floor + 0.02 of the update; the sharp check is per block:
test_resnet50_teacher_forced_blocks recomputes every layer (stem, pool, each bottleneck block,
average pool) from the GPU's OWN stored input -- and its backward from the GPU's own upstream
gradient -- with the oracle's autograd restatement, and requires outputs within 5e-3 and input /
parameter gradients within 5e-2 relative (||.||; a wrong stride, shortcut, batch-norm statistic or
transposition is O(1)).
"""
import numpy as np
import pytest

from oracle import step as ostep
from paper_1901_05803_b200 import resnet, synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, profile, volume_baseline, volume_ralp

pytestmark = pytest.mark.gpu

# teacher-forced tolerances (||.|| relative): forward 5e-3 (observed <= 1.7e-3); backward 5e-2
# (observed <= 2.1e-2: a block's backward passes ~8 bf16 storage points and three batch-norm
# backwards, whose mean subtractions cancel most of dz and magnify the rounding differences)
FWD_TOL = 5e-3
BWD_TOL = 5e-2
# first-step loss (forward only, relative): the GPU's own step-0 loss varies run to run by up
# to ~2.5e-3 at b=8 (batch-norm statistics are float-atomic sums in nondeterministic order and the
# differences ride through 50 bf16 storage points); observed |gpu - oracle| / oracle <= 2.5e-3
LOSS_TOL = 5e-3


def _run(batch, strategy, steps, lr, split=None):
    model = catalog_lookup("resnet-50").with_batch_size(batch)
    if strategy == "ralp":
        split = profile(model).split_index if split is None else split
        job = JobSpec(model, Strategy.ralp(split), 1)
        expect = volume_ralp(model, split, 1).total_bytes_per_step
        lsplit = resnet.lowered_split(split)
    else:
        job = JobSpec(model, Strategy.baseline(), 1)
        expect = volume_baseline(model, 1).total_bytes_per_step
        lsplit = None
    ex = RankExecutor(job)
    params = synthetic.init_params(ex.layers, 0)
    ex.set_params(params)
    o32 = ostep.OracleState(ex.layers, params)
    o64 = ostep.OracleState(ex.layers, params)
    bad = []
    for t in range(steps):
        imgs, labs = synthetic.batch(0, t, 0, batch, ex.in_shape, ex.classes)
        ex.step(imgs, labs, lr=lr, momentum=0.9)
        st = ex.stats()
        lo, wire = ostep.train_step(o32, strategy, 1, [(imgs, labs)], lr=lr, emulate_bf16=True, split=lsplit)
        ostep.train_step(o64, strategy, 1, [(imgs, labs)], lr=lr, emulate_bf16=True, accum64=True, split=lsplit)
        print(f"  step {t}: loss gpu {st.loss:.6f} oracle {lo:.6f} bytes {st.logical_bytes} launches {st.launches} "
              f"ms {st.ms_step:.2f}")
        assert st.logical_bytes == wire == expect
        if t == 0 and abs(st.loss - lo) > LOSS_TOL * abs(lo):
            bad.append(f"step {t}: loss {st.loss} vs oracle {lo}")
    got = ex.get_params()
    ex.close()
    for li, (g, w, w64, p0) in enumerate(zip(got, o32.numpy_params(), o64.numpy_params(), params)):
        if g is None:
            continue
        for nm, a, o, o64_, c in zip("wb", g, w, w64, p0):
            upd = np.linalg.norm(o - c)
            if upd == 0:
                continue
            dev = np.linalg.norm(a.reshape(-1) - o.reshape(-1)) / upd
            floor = np.linalg.norm(o64_.reshape(-1) - o.reshape(-1)) / upd
            bound = 2 * floor + 0.02
            print(f"  layer {li} {ex.layers[li]['name']}.{nm}: dev {dev:.3e} floor {floor:.3e}")
            if dev > bound:
                bad.append(f"layer {li}.{nm}: dev {dev:.3e} > {bound:.3e}")
    assert not bad, "\n".join(bad)


def test_resnet50_fc_tail_split():
    model = catalog_lookup("resnet-50").with_batch_size(128)
    assert profile(model).split_index == 55 and resnet.lowered_split(55) == 19
    _run(8, "ralp", steps=2, lr=1e-3, split=55)


def test_resnet50_blocks_on_the_ps():
    # b=64's partitioner split (pool1): the sixteen blocks run on the PS over the gathered rows
    model = catalog_lookup("resnet-50").with_batch_size(64)
    assert profile(model).split_index == 2
    _run(8, "ralp", steps=2, lr=1e-3, split=2)


def test_resnet50_all_on_ps():
    _run(8, "baseline", steps=2, lr=1e-3)


def test_resnet50_teacher_forced_blocks():
    import torch
    from paper_1901_05803_b200 import _lib
    b = 8
    model = catalog_lookup("resnet-50").with_batch_size(b)
    ex = RankExecutor(JobSpec(model, Strategy.ralp(55), 1))
    params = synthetic.init_params(ex.layers, 0)
    ex.set_params(params)
    imgs, labs = synthetic.batch(0, 0, 0, b, ex.in_shape, ex.classes)
    ex.step(imgs, labs, lr=1e-3, momentum=0.9)
    grads = ex.get_grads()
    L = ex.layers
    R = ostep._Round.apply
    report, bad = [], []

    def nchw(flat, c):
        hw = flat.size // (b * c)
        side = int(round(hw ** 0.5))
        return torch.from_numpy(flat.reshape(b, side, side, c)).permute(0, 3, 1, 2).contiguous()

    def rel(name, got, ref, tol=2e-2):
        r = float((got.double() - ref.double()).norm() / ref.double().norm())
        report.append(f"{name:28s} rel {r:.2e}")
        if not r <= tol:
            bad.append(f"{name}: rel {r:.2e}")

    def layer_io(i):
        x = torch.from_numpy(imgs).permute(0, 3, 1, 2).contiguous() if i == 0 else nchw(ex.debug_buffer(_lib.DBG_ACT, i), L[i]["cin"])
        if i + 1 < 19:
            y = nchw(ex.debug_buffer(_lib.DBG_ACT, i + 1), L[i + 1]["cin"])
            dy = nchw(ex.debug_buffer(_lib.DBG_ACT_GRAD, i + 1), L[i + 1]["cin"])
        else:   # the cut: the FC input rows and their gradient
            y = torch.from_numpy(ex.debug_buffer(_lib.DBG_FC_IN).reshape(b, -1, 1, 1))
            dy = torch.from_numpy(ex.debug_buffer(_lib.DBG_FC_IN_GRAD).reshape(b, -1, 1, 1))
        return x, y, dy

    for i in range(19):   # stem, pool1, 16 blocks, apool
        d = L[i]
        x, y_gpu, dy_gpu = layer_io(i)
        xin = (R(x) if i == 0 else x).requires_grad_(True)
        p = params[i]
        pt = None if p is None else [torch.from_numpy(a).clone().requires_grad_(True) for a in p]
        y = ostep._branchy_forward([d], [pt], xin, R, torch.float32)
        rel(f"fwd {i} {d['name']}", y_gpu, y.detach(), tol=0.0 if d["kind"] == "pool" else FWD_TOL)
        # backward from the GPU's own upstream gradient
        y.backward(dy_gpu)
        if i > 0:
            ref = xin.grad
            if d["kind"] == "pool":   # the GPU folds the producer's ReLU derivative into the pool backward
                ref = ref * (x > 0)
            rel(f"dgrad {i} {d['name']}", nchw(ex.debug_buffer(_lib.DBG_ACT_GRAD, i), d["cin"]), ref, tol=BWD_TOL)
        if pt is not None:
            gw, gb = grads[i]
            rel(f"wgrad {i} {d['name']}", torch.from_numpy(gw.reshape(-1)), pt[0].grad.reshape(-1), tol=BWD_TOL)
            rel(f"bn grad {i} {d['name']}", torch.from_numpy(gb.reshape(-1)), pt[1].grad.reshape(-1), tol=BWD_TOL)
    ex.close()
    print("\n".join(report))
    assert not bad, "\n".join(bad)
