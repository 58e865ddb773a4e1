"""Per-layer parity at the headline configuration: VGG-16 224x224, b=128, the partitioner's split
18 (pool5 | fc1), one B200 (what bench.py times).

Teacher forcing: after one real step through the C ABI every layer is recomputed by the oracle's
per-layer ops (oracle/step.py) from the GPU's OWN stored inputs, so each kernel is judged alone,
not through the bf16 drift of everything before it:

  bf16 outputs (conv forward / backward-data, FC forward / backward-data, dlogits):
      |gpu - ref| <= 2^-8 |ref| + 1e-5 max|ref|   (the GPU's bf16 rounding of its fp32 result,
      plus fp32 summation-order noise), and >= 99 % of the elements bit-identical to bf16(ref)
  max pool forward / backward (routing of bf16 values), the cut rows, the act-grad rows:
      bit-identical
  parameter gradients (conv / FC weights and biases, fp32):
      ||g_gpu - g_ref|| <= 1e-3 ||g_ref||  and  max|g_gpu - g_ref| <= 1e-3 max|g_ref|
  SGD-momentum (first step, v = 0):  p1 == fl(p0 - fl(lr * g_gpu)) to 1 ulp
  loss: the GPU's mean cross-entropy == the oracle's from the GPU's logits to 1e-5

Then the same step runs free in the oracle (bf16 emulated at the GPU's rounding points) on the
same seeds: loss within 2e-3, split and synchronised bytes exact.  Reference schedule:
pkg/src/ralp/simulator.py:669-715; layer semantics layers.py:87-123.
"""
import numpy as np
import pytest
import torch

from oracle import step as ostep
from paper_1901_05803_b200 import _lib, synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, profile, volume_ralp

pytestmark = pytest.mark.gpu

B = 128
LR = 0.01


def bf16(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.bfloat16).to(torch.float32)


def nhwc_padded(flat: np.ndarray, n: int, c: int, h: int, w: int) -> torch.Tensor:
    """Padded NHWC buffer -> interior as NCHW fp32 (the pad is solved from the element count)."""
    hw = flat.size // (n * c)
    side = int(round(hw ** 0.5))
    assert side * side == hw, (flat.size, n, c)
    p = (side - h) // 2
    x = torch.from_numpy(flat.reshape(n, side, side, c))
    return x[:, p:p + h, p:p + w, :].permute(0, 3, 1, 2).contiguous()


def check_bf16(name, got, ref, report, rtol=2.0 ** -8, atol_frac=1e-5):
    got, ref = got.float(), ref.float()
    err = (got - ref).abs()
    tol = rtol * ref.abs() + atol_frac * ref.abs().max()
    bad = int((err > tol).sum())
    same = float((got == bf16(ref)).float().mean())
    report.append(f"{name:28s} bf16  max|err| {err.max():.3e}  bit-identical {same:.5f}  beyond tol {bad}")
    assert bad == 0, f"{name}: {bad} elements beyond 1 bf16 rounding (max err {err.max():.3e})"
    assert same >= 0.99, f"{name}: only {same:.4f} of the elements bit-identical"


def check_exact(name, got, ref, report):
    same = torch.equal(got.float(), ref.float())
    report.append(f"{name:28s} exact {same}")
    assert same, f"{name}: not bit-identical ({int((got.float() != ref.float()).sum())} differ)"


def check_grad(name, got, ref, report, tol=1e-3):
    got, ref = torch.as_tensor(got).double(), torch.as_tensor(ref).double()
    rel = float((got - ref).norm() / ref.norm())
    mx = float((got - ref).abs().max() / ref.abs().max())
    report.append(f"{name:28s} grad  rel {rel:.3e}  max {mx:.3e}")
    assert rel <= tol and mx <= tol, f"{name}: gradient off (rel {rel:.3e}, max {mx:.3e})"


@pytest.fixture(scope="module")
def headline():
    model = catalog_lookup("vgg16").with_batch_size(B)
    rep = profile(model)
    # split index 18 (1-based): conv1..pool5 in front, fc1 onward on the PS
    assert rep.split_index == 18 and model.layer(18).name == "pool5" and model.layer(19).name == "fc1"
    job = JobSpec(model, Strategy.ralp(rep.split_index), 1)
    ex = RankExecutor(job)
    params = synthetic.init_params(ex.layers, 0)
    ex.set_params(params)
    imgs, labs = synthetic.batch(0, 0, 0, B, ex.in_shape, ex.classes)
    ex.step(imgs, labs, lr=LR, momentum=0.9)
    st = ex.stats()
    yield dict(model=model, rep=rep, ex=ex, params=params, imgs=imgs, labs=labs, st=st, grads=ex.get_grads(),
               new=ex.get_params())
    ex.close()


def test_headline_split_and_bytes(headline):
    m, st = headline["model"], headline["st"]
    assert st.logical_bytes == volume_ralp(m, 18, 1).total_bytes_per_step == 143_407_616


def test_headline_front_forward_per_layer(headline):
    ex, params, imgs = headline["ex"], headline["params"], headline["imgs"]
    layers = ex.layers
    nfront = 18
    n = 16  # forward outputs are per-image: check 16 of the 128 images (first and last 8)
    sel = list(range(8)) + list(range(B - 8, B))
    report = []
    x = bf16(torch.from_numpy(imgs[sel]).permute(0, 3, 1, 2).contiguous())   # layer 0's bf16 patches
    cut_rows = ex.debug_buffer(_lib.DBG_CUT_ROWS).reshape(B, -1)
    for i in range(nfront):
        L = layers[i]
        h_out = L["h"] if L["kind"] == "conv" else (L["h"] - L["k"]) // L["stride"] + 1
        c_out = L["cout"]
        if i + 1 < nfront:
            full = ex.debug_buffer(_lib.DBG_ACT, i + 1)
            y_gpu = nhwc_padded(full, B, c_out, h_out, h_out)[sel]
        else:  # pool5 writes the PS's FC input rows directly (HWC flatten)
            y_gpu = torch.from_numpy(cut_rows[sel].reshape(n, h_out, h_out, c_out)).permute(0, 3, 1, 2)
        if L["kind"] == "conv":
            w, b = params[i]
            wt = bf16(torch.from_numpy(w).permute(0, 3, 1, 2).contiguous())
            bias = torch.from_numpy(b)
            if i == 0:
                bias = bf16(bias)  # the first conv's bias is a bf16 filter column (conv_first.cu)
            ref = ostep.conv_forward(x, wt, bias, L["stride"], L["pad"])
            check_bf16(f"fwd {i} conv {L['name']}", y_gpu, ref, report)
        else:
            ref = ostep.maxpool_forward(x, L["k"], L["stride"])
            check_exact(f"fwd {i} pool {L['name']}", y_gpu, ref, report)
        x = y_gpu  # teacher forcing: the next layer starts from the GPU's own output
    print("\n".join(report))


def test_headline_fc_tail_per_layer(headline):
    ex, params, labs, grads, st = headline["ex"], headline["params"], headline["labs"], headline["grads"], headline["st"]
    layers = ex.layers
    report = []
    x = torch.from_numpy(ex.debug_buffer(_lib.DBG_CUT_ROWS).reshape(B, -1))
    hs = [x]
    for j, li in enumerate(range(18, 21)):
        L = layers[li]
        w, b = params[li]
        wbf = bf16(torch.from_numpy(w))
        if j < 2:
            got = torch.from_numpy(ex.debug_buffer(_lib.DBG_FC_OUT, j).reshape(B, -1)[:, :L["cout"]])
            ref = ostep.fc_forward(hs[-1], wbf, torch.from_numpy(b), relu=True)
            check_bf16(f"fwd {li} fc {L['name']}", got, ref, report)
            hs.append(got)
        else:
            logits = torch.from_numpy(ex.debug_buffer(_lib.DBG_LOGITS).reshape(B, -1)[:, :L["cout"]])
            ref = ostep.fc_forward(hs[-1], wbf, torch.from_numpy(b), relu=False)
            rel = float((logits - ref).norm() / ref.norm())
            report.append(f"fwd {li} logits rel {rel:.3e}")
            assert rel <= 1e-5
    row, dref = ostep.softmax_xent(logits, labs, 1.0 / B)
    assert abs(st.loss - float(row.mean())) <= 1e-5 * abs(float(row.mean())), (st.loss, float(row.mean()))
    dy = torch.from_numpy(ex.debug_buffer(_lib.DBG_DLOGITS).reshape(B, -1)[:, :1000])
    check_bf16("dlogits", dy, dref, report)
    for j in (2, 1, 0):
        li = 18 + j
        w, _ = params[li]
        wbf = bf16(torch.from_numpy(w))
        gw, gb = grads[li]
        check_grad(f"wgrad {li}", gw, ostep._mm(dy.t(), hs[j]), report)
        check_grad(f"bgrad {li}", gb, dy.double().sum(0), report)
        dx = ostep._mm(dy, wbf)
        if j > 0:
            dx = dx * (hs[j] > 0)
            got = torch.from_numpy(ex.debug_buffer(_lib.DBG_FC_OUT_GRAD, j - 1).reshape(B, -1)[:, :layers[li - 1]["cout"]])
        else:
            got = torch.from_numpy(ex.debug_buffer(_lib.DBG_CUT_GRAD_ROWS).reshape(B, -1))
        check_bf16(f"dgrad {li}", got, dx, report)
        dy = got
    print("\n".join(report))


def test_headline_front_backward_per_layer(headline):
    ex, params, grads = headline["ex"], headline["params"], headline["grads"]
    layers = ex.layers
    report = []
    imgs = headline["imgs"]
    sel = list(range(8)) + list(range(B - 8, B))

    def act(i):  # input of front layer i (layer 0: the bf16 image the first conv's patches hold)
        L = layers[i]
        if i == 0:
            return bf16(torch.from_numpy(imgs).permute(0, 3, 1, 2).contiguous())
        return nhwc_padded(ex.debug_buffer(_lib.DBG_ACT, i), B, L["cin"], L["h"], L["w"])

    # gradient w.r.t. pool5's output = the act-grad rows the FC tail produced (W = 1: all rows)
    dy = torch.from_numpy(ex.debug_buffer(_lib.DBG_CUT_GRAD_ROWS).reshape(B, 7, 7, 512)).permute(0, 3, 1, 2)
    for i in reversed(range(18)):
        L = layers[i]
        x = act(i)
        if L["kind"] == "pool":
            got = nhwc_padded(ex.debug_buffer(_lib.DBG_ACT_GRAD, i), B, L["cin"], L["h"], L["w"])
            ref = ostep.maxpool_backward(x, dy, L["k"], L["stride"])
            check_exact(f"bwd {i} pool {L['name']}", got, ref, report)
        else:
            w, _ = params[i]
            wt = bf16(torch.from_numpy(w).permute(0, 3, 1, 2).contiguous())
            gw_ref, gb_ref = ostep.conv_backward_filter(x, dy, wt.shape, L["stride"], L["pad"])
            gw, gb = grads[i]
            check_grad(f"wgrad {i} {L['name']}", gw, gw_ref.permute(0, 2, 3, 1), report)
            check_grad(f"bgrad {i} {L['name']}", gb, gb_ref, report)
            if i > 0:
                mask = x[sel] if layers[i - 1]["kind"] == "conv" else None
                ref = ostep.conv_backward_data(dy[sel], wt, x[sel].shape, L["stride"], L["pad"], mask)
                got_full = nhwc_padded(ex.debug_buffer(_lib.DBG_ACT_GRAD, i), B, L["cin"], L["h"], L["w"])
                check_bf16(f"dgrad {i} {L['name']}", got_full[sel], ref, report)
                got = got_full
        dy = got if i > 0 else None
        del x
    print("\n".join(report))


def test_headline_sgd_update(headline):
    """First step, momentum 0: v = g, p1 = p0 - lr * g (one fused multiply-add on the GPU, so up to
    1 ulp from the host's two roundings)."""
    params, grads, new = headline["params"], headline["grads"], headline["new"]
    worst, where = 0.0, None
    for li, (p0, g, p1) in enumerate(zip(params, grads, new)):
        if p0 is None:
            continue
        for nm, a, gg, c in zip("wb", p0, g, p1):
            want = (a.astype(np.float64) - np.float64(np.float32(LR)) * gg.astype(np.float64))
            ulp = np.spacing(np.abs(want).astype(np.float32)).astype(np.float64)
            dev = np.abs(c.astype(np.float64) - want) / ulp
            k = int(np.argmax(dev))
            print(f"  layer {li}.{nm}: worst {dev.flat[k]:.2f} ulp (p0 {a.flat[k]:.6e} g {gg.flat[k]:.6e} "
                  f"p1 {c.flat[k]:.6e} want {want.flat[k]:.6e})")
            if dev.flat[k] > worst:
                worst, where = float(dev.flat[k]), f"{li}.{nm}"
    print("SGD step worst deviation (ulp):", worst, where)
    assert worst <= 1.0


def test_headline_free_step_vs_oracle(headline):
    """The same step run free in the oracle (bf16 emulated where the GPU stores bf16)."""
    ex, params, imgs, labs, st = headline["ex"], headline["params"], headline["imgs"], headline["labs"], headline["st"]
    torch.set_num_threads(max(1, torch.get_num_threads()))
    orc = ostep.OracleState(ex.layers, params)
    loss, wire = ostep.train_step(orc, "ralp", 1, [(imgs, labs)], lr=LR, mu=0.9, emulate_bf16=True)
    print(f"free step: loss gpu {st.loss:.6f} oracle {loss:.6f}")
    assert wire == st.logical_bytes
    assert abs(st.loss - loss) <= 2e-3 * abs(loss)
