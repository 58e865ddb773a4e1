"""The parity precision (RALPB_PRECISION_FP32) against the PLAIN fp32 oracle.

north_star: "loss and parameters after N steps from identical seeds and synthetic inputs must
match within a stated fp32 relative tolerance (e.g. 1e-4)".  In this mode every activation and
gradient is an fp32-accurate (hi, lo) bf16 pair and every contraction runs on the tcgen05 GEMM
engine over the pairs (hi*hi + hi*lo + lo*hi + lo*lo, fp32 accumulation; pair.cuh), so the whole
step is fp32-accurate.  The oracle runs in plain fp32 torch on the CPU (oracle/step.py,
emulate_bf16=False -- no GPU rounding emulated).  Stated tolerances, after N steps:

  loss            |loss_gpu - loss_oracle| <= 1e-4 * |loss_oracle| at every step
  parameters      ||p_gpu - p_oracle|| <= 1e-5 * ||p_oracle||          per tensor
  the update      ||p_gpu - p_oracle|| <= 1e-2 * ||p_oracle - p_0||    per weight tensor

(the last is the sharp one: the parameters themselves barely move in 10 steps at lr 0.01, so it
judges the update the GPU applied, not the initial values both sides share).
"""
import numpy as np
import pytest

from oracle import step as ostep
from paper_1901_05803_b200 import synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, parse_model, volume_baseline, volume_ralp

pytestmark = pytest.mark.gpu

LOSS_RTOL = 1e-4
PARAM_RTOL = 1e-5
UPDATE_RTOL = 1e-2

VGG_TINY = """
model vgg_tiny batch=8 elem_bytes=4 input=32x32x3
conv1 conv k=3 cout=64 pad=1
conv2 conv k=3 cout=64 pad=1
pool1 pool window=2
conv3 conv k=3 cout=128 pad=1
conv4 conv k=3 cout=128 pad=1
pool2 pool window=2
conv5 conv k=3 cout=256 pad=1
conv6 conv k=3 cout=256 pad=1
pool3 pool window=2
conv7 conv k=3 cout=512 pad=1
pool4 pool window=2
fc1 fc out=1024
fc2 fc out=1024
fc3 fc out=100
"""


def _fc_boundary(model):
    return next(i for i, l in enumerate(model.layers) if l.kind.value == "fc")


def run_fp32(model, strategy, steps, lr=0.01, seed=0):
    if strategy == "ralp":
        split = _fc_boundary(model)
        job = JobSpec(model, Strategy.ralp(split), 1)
        expect = volume_ralp(model, split, 1).total_bytes_per_step
    else:
        job = JobSpec(model, Strategy.baseline(), 1)
        expect = volume_baseline(model, 1).total_bytes_per_step
    ex = RankExecutor(job, precision="fp32")
    params = synthetic.init_params(ex.layers, seed)
    ex.set_params(params)
    orc = ostep.OracleState(ex.layers, params)
    orc64 = ostep.OracleState(ex.layers, params)   # the fp32 oracle's own floor: fp64 contractions
    b = model.batch_size
    bad = []
    for t in range(steps):
        imgs, labs = synthetic.batch(seed, t, 0, b, ex.in_shape, ex.classes)
        ex.step(imgs, labs, lr=lr, momentum=0.9)
        st = ex.stats()
        lo, wire = ostep.train_step(orc, strategy, 1, [(imgs, labs)], lr=lr, mu=0.9, emulate_bf16=False)
        l64, _ = ostep.train_step(orc64, strategy, 1, [(imgs, labs)], lr=lr, mu=0.9, emulate_bf16=False, accum64=True)
        assert st.logical_bytes == wire == expect
        rel = abs(st.loss - lo) / abs(lo)
        print(f"  step {t}: loss gpu {st.loss:.7f} oracle {lo:.7f} rel {rel:.2e}   (oracle fp32 vs fp64: "
              f"{abs(l64 - lo) / abs(lo):.2e})")
        if not rel <= LOSS_RTOL:
            bad.append(f"step {t}: loss rel {rel:.2e}")
    got = ex.get_params()
    ex.close()
    for li, (g, w, w64, p0) in enumerate(zip(got, orc.numpy_params(), orc64.numpy_params(), params)):
        if g is None:
            continue
        for nm, a, o, o64, c in zip("wb", g, w, w64, p0):
            rel = np.linalg.norm(a - o) / np.linalg.norm(o)
            upd = np.linalg.norm(o - c)
            urel = np.linalg.norm(a - o) / upd if upd > 0 else 0.0
            floor = np.linalg.norm(o64 - o) / upd if upd > 0 else 0.0
            print(f"  layer {li}.{nm}: ||dp||/||p|| {rel:.2e}  ||dp||/||update|| {urel:.2e}  "
                  f"(oracle fp32 vs fp64 ||dp||/||update|| {floor:.2e})")
            if not rel <= PARAM_RTOL and np.linalg.norm(o) > 0:
                bad.append(f"layer {li}.{nm}: ||dp||/||p|| {rel:.2e}")
            if nm == "w" and not urel <= UPDATE_RTOL:
                bad.append(f"layer {li}.{nm}: ||dp||/||update|| {urel:.2e}")
    assert not bad, "\n".join(bad)


@pytest.mark.parametrize("strategy", ["ralp", "baseline"])
def test_fp32_cifar_small_10_steps(strategy):
    run_fp32(catalog_lookup("cifar_small").with_batch_size(64), strategy, steps=10)


def test_fp32_vgg_tiny_10_steps():
    run_fp32(parse_model(VGG_TINY), "ralp", steps=10)


def test_fp32_alexnet_b4():
    run_fp32(catalog_lookup("alexnet").with_batch_size(4), "ralp", steps=3, lr=1e-3)


def test_fp32_vgg16_b4_split18():
    # the real VGG-16 geometry with the FC-tail split forced (the partitioner picks pool5 from b=95)
    run_fp32(catalog_lookup("vgg16").with_batch_size(4), "ralp", steps=2, lr=1e-3)
