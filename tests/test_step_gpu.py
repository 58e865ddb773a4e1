"""Full training-step parity: the B200 executor (through the C ABI) against the CPU
oracle restatement (oracle/step.py) on identical seeds, synthetic inputs and
initial parameters.

The split point and the per-step synchronised bytes must match exactly.

Numerics.  Both sides use bf16 operands with fp32 accumulation and the oracle
rounds to bf16 at exactly the points the GPU stores bf16.  The bf16 pipeline is
chaotic under summation-order noise (a 1-ulp re-rounding flips a ReLU/max-pool
decision and re-routes a gradient), so the tolerance is stated against the
pipeline's own noise floor, measured every time by re-running the oracle with
float64 accumulation:
  floor(layer) = ||p_oracle64 - p_oracle32|| / ||p_oracle32 - p_init||
  dev(layer)   = ||p_gpu      - p_oracle32|| / ||p_oracle32 - p_init||
  require dev <= min(2 * floor + 0.02, 0.5) for every parameter tensor after N steps: a wrong
  update (a lost gradient, a missing momentum term) is dev ~ 1; the deep nets' floor itself
  reaches 0.1-0.35 (bf16 re-rounding flips ReLU / max-pool decisions), so the per-kernel parity
  is pinned sharply elsewhere -- by the teacher-forced headline test (tests/test_headline_parity_gpu.py)
  and the fp32 parity precision (tests/test_parity_fp32_gpu.py),
  and |loss_gpu - loss_oracle| <= 2e-3 * |loss_oracle| at every step.
(The B200's tensor-core fp32 accumulation truncates per MMA, so its noise is
larger than CPU fp32's; the factor 4 covers that, and a real bug shows up as
dev ~ O(1).)
"""
import numpy as np
import pytest

from oracle import step as ostep
from paper_1901_05803_b200 import synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import (JobSpec, Strategy, catalog_lookup, parse_model, profile,
                                           volume_baseline, volume_ralp)

pytestmark = pytest.mark.gpu

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

LOSS_RTOL = 2e-3


def _fc_boundary(model):
    return next(i for i, l in enumerate(model.layers) if l.kind.value == "fc")


def _run(model, strategy, steps, seed=0, lr=0.01, split=None):
    """split (RALP): None = the FC-tail cut (the partitioner's choice at large batch); otherwise
    the partitioner's own split, which may leave conv / pool layers in the back segment (run on
    the PS over the gathered rows)."""
    wire_split = split
    if strategy == "ralp":
        split = _fc_boundary(model) if split is None else split
        job = JobSpec(model, Strategy.ralp(split), 1)
        expect_bytes = volume_ralp(model, split, 1).total_bytes_per_step
    else:
        job = JobSpec(model, Strategy.baseline(), 1)
        expect_bytes = volume_baseline(model, 1).total_bytes_per_step
    ex = RankExecutor(job)
    params = synthetic.init_params(ex.layers, seed)
    ex.set_params(params)
    o32 = ostep.OracleState(ex.layers, params)
    o64 = ostep.OracleState(ex.layers, params)
    b = model.batch_size
    losses = []
    for t in range(steps):
        imgs, labs = synthetic.batch(seed, t, 0, b, ex.in_shape, ex.classes)
        ex.step(imgs, labs, lr=lr, momentum=0.9)
        st = ex.stats()
        loss_o, wire = ostep.train_step(o32, strategy, 1, [(imgs, labs)], lr=lr, mu=0.9, emulate_bf16=True,
                                        split=wire_split)
        ostep.train_step(o64, strategy, 1, [(imgs, labs)], lr=lr, mu=0.9, emulate_bf16=True, accum64=True)
        assert st.logical_bytes == wire == expect_bytes
        losses.append((st.loss, loss_o))
    got = ex.get_params()
    ex.close()
    return losses, got, o32.numpy_params(), o64.numpy_params(), params


def _check(losses, got, want, want64, init, cap=0.5):
    bad = []
    for i, (lg, lo) in enumerate(losses):
        print(f"  step {i}: loss gpu {lg:.6f} oracle {lo:.6f}")
        if abs(lg - lo) > LOSS_RTOL * abs(lo):
            bad.append(f"step {i}: loss {lg} vs oracle {lo}")
    for li, (g, w, w64, p0) in enumerate(zip(got, want, want64, init)):
        if g is None:
            continue
        for nm, a, o, o64, c in zip("wb", g, w, w64, p0):
            upd = np.linalg.norm(o - c)
            dev = np.linalg.norm(a - o) / upd
            floor = np.linalg.norm(o64 - o) / upd
            print(f"  layer {li}.{nm}: dev {dev:.3e} floor {floor:.3e}")
            bound = min(2 * floor + 0.02, cap)
            if dev > bound:
                bad.append(f"layer {li}.{nm}: dev {dev:.3e} > min(2 * floor {floor:.3e} + 0.02, {cap})")
    assert not bad, "\n".join(bad)


@pytest.mark.parametrize("strategy", ["ralp", "baseline"])
def test_cifar_small_steps(strategy):
    model = catalog_lookup("cifar_small").with_batch_size(64)
    assert profile(model).split_index == 4
    losses, got, want, want64, init = _run(model, strategy, steps=5)
    print("cifar_small", strategy, losses)
    _check(losses, got, want, want64, init)


def test_vgg_tiny_steps():
    model = parse_model(VGG_TINY)
    losses, got, want, want64, init = _run(model, "ralp", steps=3)
    print("vgg_tiny", losses)
    _check(losses, got, want, want64, init)


def test_vgg16_one_step_b4():
    # the real VGG-16 geometry (224x224), small batch so the CPU oracle stays fast;
    # at b=4 the partitioner cuts at pool3 (conv layers in the back segment), so the FC-tail
    # executor is driven with the baseline plan here and the b=128 pool5 split is covered
    # by the planner golden tests.
    model = catalog_lookup("vgg16").with_batch_size(4)
    losses, got, want, want64, init = _run(model, "baseline", steps=1)
    print("vgg16 b=4", losses)
    _check(losses, got, want, want64, init)


def test_alexnet_steps_b4():
    # AlexNet config of BASELINE.json: 11x11/4 first conv (im2col GEMM), 5x5 conv, overlapping
    # 3/2 max-pools, FC tail on the PS; small batch so the CPU oracle stays fast.  At lr=0.01
    # the unnormalised 227x227 input makes step 1 overshoot (loss ~24, a chaotic regime), so
    # the parity run uses lr=1e-3.
    model = catalog_lookup("alexnet").with_batch_size(4)
    losses, got, want, want64, init = _run(model, "ralp", steps=3, lr=1e-3)
    print("alexnet b=4", losses)
    _check(losses, got, want, want64, init)


def test_pipelined_host_inputs_and_async_loss():
    """Host inputs go through the double-buffered copy stream and the loss ring: enqueueing
    several steps before reading their losses gives the same losses as stepping synchronously."""
    model = catalog_lookup("cifar_small").with_batch_size(64)
    job = JobSpec(model, Strategy.ralp(_fc_boundary(model)), 1)
    batches = [synthetic.batch(0, t, 0, 64, (32, 32, 3), 10) for t in range(4)]
    losses = []
    for pipelined in (False, True):
        ex = RankExecutor(job)
        ex.set_params(synthetic.init_params(ex.layers, 0))
        got = []
        for imgs, labs in batches:
            ex.step(imgs, labs)
            if not pipelined:
                got.append(ex.stats().loss)
        if pipelined:
            got = [ex.read_loss(lag) for lag in (3, 2, 1, 0)]
        ex.close()
        losses.append(got)
    np.testing.assert_allclose(losses[1], losses[0], rtol=1e-3)


@pytest.mark.parametrize("name,batch,split,steps,lr", [
    ("cifar_small", 8, 2, 4, 0.01),     # pool1 | conv2, pool2, fc1, fc2 on the PS
    ("vgg_tiny", 8, 3, 3, 0.01),        # pool1 | conv3..pool4 + FC tail on the PS
    ("vgg16", 4, 6, 1, 1e-3),           # pool2 | conv3_1..pool5 + FC tail (VGG-16 at b=4)
    ("alexnet", 4, 2, 2, 1e-3),         # pool1 | conv2 (5x5)..pool5 + FC tail
])
def test_partitioner_split_conv_back_segment(name, batch, split, steps, lr):
    """The partitioner's own split at small batch cuts inside the conv stack (profiler.py:101-134):
    the back segment's conv / pool layers run on the PS over the gathered cut rows, the act-grad
    returned is the gradient w.r.t. that intermediate feature map, and only the front before the
    cut is synchronised (volume_ralp(m, split, W) bytes)."""
    model = (parse_model(VGG_TINY) if name == "vgg_tiny" else catalog_lookup(name)).with_batch_size(batch)
    assert profile(model).split_index == split
    losses, got, want, want64, init = _run(model, "ralp", steps=steps, lr=lr, split=split)
    print(name, batch, "split", split, losses)
    _check(losses, got, want, want64, init)
