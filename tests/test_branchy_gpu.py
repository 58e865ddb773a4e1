"""Branch-group models executed: Inception-v3, GoogLeNet, OverFeat and LeNet from
the reference catalog, lowered to RALPB_MODULE node DAGs (paper_1901_05803_b200/branchy.py,
csrc/graph.cu) and run through the C ABI at the partitioner's splits, against the oracle's autograd
restatement with bf16 storage emulated at the GPU's storage points (oracle/step.py _module_forward).

  * bytes: every rank's count_wire-site count == the oracle's wire == volume_ralp of the catalog model;
  * the first step's loss: 2e-3 relative (bias models), 5e-3 with batch norm (Inception: the
    statistics are float-atomic sums in nondeterministic order, as for ResNet-50);
  * parameters after two steps within 2 * floor + 0.02 of the update (floor = the bf16 pipeline's
    own fp32-vs-fp64 spread; capped at 0.5 for the bias models, whose training is not chaotic);
  * the sharp check, per lowered layer (teacher-forced): every group recomputed from the GPU's own
    stored input -- and its backward from the GPU's own upstream gradient -- by the oracle, outputs
    within 5e-3 and input / parameter gradients within 1e-1 (Inception: up to five batch-norm
    backwards chained inside one group) or 2e-2 (GoogLeNet); a wrong window, stride, padding, branch
    order or concatenation offset is O(1).
"""
import numpy as np
import pytest

from oracle import step as ostep
from paper_1901_05803_b200 import _lib, synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, volume_ralp

pytestmark = pytest.mark.gpu

BN_MODELS = {"inception-v3"}


def _run(name, batch, split, steps=2, lr=1e-3):
    model = catalog_lookup(name).with_batch_size(batch)
    ex = RankExecutor(JobSpec(model, Strategy.ralp(split), 1))
    params = synthetic.init_params(ex.layers, 0)
    ex.set_params(params)
    o32 = ostep.OracleState(ex.layers, params)
    o64 = ostep.OracleState(ex.layers, params)
    expect = volume_ralp(model, split, 1).total_bytes_per_step
    bad = []
    for t in range(steps):
        imgs, labs = synthetic.batch(0, t, 0, batch, ex.in_shape, ex.classes)
        ex.step(imgs, labs, lr=lr, momentum=0.9)
        st = ex.stats()
        lo, wire = ostep.train_step(o32, "ralp", 1, [(imgs, labs)], lr=lr, emulate_bf16=True, split=ex.lowered_split)
        ostep.train_step(o64, "ralp", 1, [(imgs, labs)], lr=lr, emulate_bf16=True, accum64=True, split=ex.lowered_split)
        print(f"  {name} split {split} step {t}: loss gpu {st.loss:.6f} oracle {lo:.6f} bytes {st.logical_bytes} "
              f"ms {st.ms_step:.2f}")
        assert st.logical_bytes == wire == expect
        tol = 5e-3 if name in BN_MODELS else 2e-3
        if t == 0 and abs(st.loss - lo) > tol * abs(lo):
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
            bound = 2 * floor + 0.02 if name in BN_MODELS else min(2 * floor + 0.02, 0.5)
            print(f"  layer {li} {ex.layers[li]['name']}.{nm}: dev {dev:.3e} floor {floor:.3e}")
            if dev > bound:
                bad.append(f"layer {li}.{nm}: dev {dev:.3e} > {bound:.3e}")
    assert not bad, "\n".join(bad)


@pytest.mark.parametrize("name,batch,split", [
    ("inception-v3", 8, 7),     # the partitioner's cut at b <= 64: pool2, every branch group on the PS
    ("inception-v3", 8, 97),    # b=128's cut: apool | fc
    ("googlenet", 8, 5),        # pool2
    ("googlenet", 8, 62),       # apool | fc
    ("overfeat", 8, 2),         # pool1: the unpadded 5x5 (a one-node module) on the PS
    ("overfeat", 8, 4),
    ("lenet", 8, 2),
])
def test_branchy_model_steps(name, batch, split):
    _run(name, batch, split)


# backward tolerance: Inception's 7x1 / 1x7 chains pass five batch-norm backwards inside one group
# (observed <= 5.3e-2; a single batch-normalised conv ~2e-3); GoogLeNet has no batch norm
@pytest.mark.parametrize("name,split,bwd_tol", [("inception-v3", 97, 1e-1), ("googlenet", 62, 2e-2)])
def test_teacher_forced_groups(name, split, bwd_tol):
    import torch
    b = 4
    model = catalog_lookup(name).with_batch_size(b)
    ex = RankExecutor(JobSpec(model, Strategy.ralp(split), 1))
    params = synthetic.init_params(ex.layers, 0)
    ex.set_params(params)
    imgs, labs = synthetic.batch(0, 0, 0, b, ex.in_shape, ex.classes)
    ex.step(imgs, labs, lr=1e-3, momentum=0.9)
    grads = ex.get_grads()
    L = ex.layers
    n_front = ex.lowered_split
    R = ostep._Round.apply
    report, bad = [], []

    def nchw(flat, c):
        hw = flat.size // (b * c)
        side = int(round(hw ** 0.5))
        assert side * side * b * c == flat.size
        return torch.from_numpy(flat.reshape(b, side, side, c)).permute(0, 3, 1, 2).contiguous()

    def rel(tag, got, ref, tol):
        r = float((got.double() - ref.double()).norm() / max(ref.double().norm(), 1e-30))
        report.append(f"{tag:34s} rel {r:.2e}")
        if not r <= tol:
            bad.append(f"{tag}: rel {r:.2e} > {tol}")

    for i in range(n_front):
        d = L[i]
        x = (torch.from_numpy(imgs).permute(0, 3, 1, 2).contiguous() if i == 0
             else nchw(ex.debug_buffer(_lib.DBG_ACT, i), d["cin"]))
        if i + 1 < n_front:
            y_gpu = nchw(ex.debug_buffer(_lib.DBG_ACT, i + 1), L[i + 1]["cin"])
            dy_gpu = nchw(ex.debug_buffer(_lib.DBG_ACT_GRAD, i + 1), L[i + 1]["cin"])
        else:
            y_gpu = torch.from_numpy(ex.debug_buffer(_lib.DBG_FC_IN).reshape(b, -1, 1, 1))
            dy_gpu = torch.from_numpy(ex.debug_buffer(_lib.DBG_FC_IN_GRAD).reshape(b, -1, 1, 1))
        xin = (R(x) if i == 0 else x).requires_grad_(True)
        p = params[i]
        pt = None if p is None else [torch.from_numpy(a).clone().requires_grad_(True) for a in p]
        y = ostep._branchy_forward([d], [pt], xin, R, torch.float32)
        rel(f"fwd {i} {d['name']}", y_gpu, y.detach(), 0.0 if d["kind"] == "pool" else 5e-3)
        y.backward(dy_gpu)
        if i > 0:
            # compared where the producer's ReLU passes gradient (x > 0): max pools -- stand-alone or a
            # module's pool branch -- route nothing where the window max is 0 (all-zero windows), the
            # oracle routes it to the first zero; the producer's ReLU discards both
            live = x > 0
            rel(f"dgrad {i} {d['name']}", nchw(ex.debug_buffer(_lib.DBG_ACT_GRAD, i), d["cin"]) * live,
                xin.grad * live, bwd_tol)
        if pt is not None:
            gw, gb = grads[i]
            rel(f"wgrad {i} {d['name']}", torch.from_numpy(gw.reshape(-1)), pt[0].grad.reshape(-1), bwd_tol)
            rel(f"bn/bias grad {i} {d['name']}", torch.from_numpy(gb.reshape(-1)), pt[1].grad.reshape(-1), bwd_tol)
    ex.close()
    print("\n".join(report))
    assert not bad, "\n".join(bad)
