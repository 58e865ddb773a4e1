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
Numerics: loss within 2e-3 of the oracle at every step; parameters after the steps within
min(2 * floor + 0.02, 0.5) of the update, floor = the oracle's own fp32-vs-fp64 spread.
"""
import numpy as np
import pytest

from oracle import step as ostep
from paper_1901_05803_b200 import resnet, synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, profile, volume_baseline, volume_ralp

pytestmark = pytest.mark.gpu


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
        if abs(st.loss - lo) > 2e-3 * abs(lo):
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
            bound = min(2 * floor + 0.02, 0.5)
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
