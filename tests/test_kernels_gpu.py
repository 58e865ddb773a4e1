"""Per-kernel numerics: each sm_100a kernel against a plain PyTorch fp32
reference of the same op on the same (bf16-rounded) inputs."""
import pytest
import torch
import torch.nn.functional as F

from paper_1901_05803_b200 import ops

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _bf(*shape, scale=1.0, gen=None):
    return (torch.randn(*shape, generator=gen, device=DEV) * scale).to(torch.bfloat16)


def _close(got, ref, rtol=2e-2, atol=None):
    got = got.float()
    ref = ref.float()
    if atol is None:
        atol = 2e-2 * ref.abs().max().item() + 1e-6
    torch.testing.assert_close(got, ref, rtol=rtol, atol=atol)


@pytest.mark.parametrize("M,N,K,bn", [(128, 64, 64, 0), (256, 256, 512, 0), (300, 200, 320, 0),
                                      (1024, 1000, 4096, 0), (128, 32, 128, 32), (512, 128, 1024, 128)])
def test_gemm_kk(M, N, K, bn):
    g = torch.Generator(device=DEV).manual_seed(0)
    a, b = _bf(M, K, gen=g), _bf(N, K, gen=g)
    bias = torch.randn(N, device=DEV)
    out = ops.gemm(a, b, bias=bias, relu=True, block_n=bn)
    ref = torch.relu(a.float() @ b.float().t() + bias)
    _close(out, ref)
    out32 = ops.gemm(a, b, out_kind="f32")
    _close(out32, a.float() @ b.float().t(), rtol=1e-3, atol=1e-3 * (K ** 0.5))


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 512, 256), (1024, 4096, 1000)])
def test_gemm_k_mn(M, N, K):
    # FC dgrad shape: dX[M=rows, N=in] = dY[rows, K=out] @ W[out, in]
    g = torch.Generator(device=DEV).manual_seed(1)
    a, w = _bf(M, K, gen=g), _bf(K, N, gen=g)
    out = ops.gemm(a, w, b_mn=True, out_kind="f32")
    _close(out, a.float() @ w.float(), rtol=1e-3, atol=1e-3 * (K ** 0.5))


@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (256, 512, 1024), (1000, 4096, 512)])
def test_gemm_mn_mn(M, N, K):
    # FC wgrad shape: dW[M=out, N=in] = dY[K=rows, out]^T @ X[rows, in]
    g = torch.Generator(device=DEV).manual_seed(2)
    dy, x = _bf(K, M, gen=g), _bf(K, N, gen=g)
    out = ops.gemm(dy, x, a_mn=True, b_mn=True, out_kind="f32")
    _close(out, dy.float().t() @ x.float(), rtol=1e-3, atol=1e-3 * (K ** 0.5))
    out2 = ops.gemm(dy, x, a_mn=True, b_mn=True, out_kind="f32_atomic", k_splits=0)
    _close(out2, dy.float().t() @ x.float(), rtol=1e-3, atol=1e-3 * (K ** 0.5))


def _pad(x_nhwc, p):
    return F.pad(x_nhwc, (0, 0, p, p, p, p))


CONV_CASES = [
    # n, h, w, cin, cout, k, pad
    (2, 8, 16, 64, 64, 3, 1),
    (2, 14, 14, 128, 256, 3, 1),
    (1, 28, 28, 256, 512, 3, 1),
    (3, 20, 12, 16, 64, 3, 1),
    (2, 32, 32, 32, 64, 5, 2),
    (2, 32, 32, 16, 32, 5, 2),
    (2, 56, 56, 128, 256, 3, 1),
    (3, 30, 17, 64, 128, 3, 1),
    (1, 112, 112, 64, 64, 3, 1),
    # 64 -> 64 at w >= 128: the row-streamed kernel (conv_row.cu); 160 = 128 + a shifted block
    (2, 224, 224, 64, 64, 3, 1),
    (1, 130, 160, 64, 64, 3, 1),
    (3, 36, 128, 64, 64, 3, 1),
    # 5x5 with 64-channel blocks: slab backward-filter in two tap groups (AlexNet conv2 shape)
    (2, 27, 27, 64, 192, 5, 2),
    (1, 20, 24, 128, 64, 5, 2),
]


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_fwd(case):
    n, h, w, cin, cout, k, pad = case
    g = torch.Generator(device=DEV).manual_seed(3)
    x = _pad(_bf(n, h, w, cin, gen=g), pad).contiguous()
    wt = _bf(cout, k * k, cin, scale=(2.0 / (k * k * cin)) ** 0.5, gen=g)
    bias = torch.randn(cout, device=DEV) * 0.1
    y = ops.conv_fwd(x, wt, bias, n=n, h=h, w_=w, cin=cin, cout=cout, k=k, pad=pad, relu=True)
    xr = x[:, pad:pad + h, pad:pad + w, :].permute(0, 3, 1, 2).float()
    wr = wt.float().view(cout, k, k, cin).permute(0, 3, 1, 2)
    ref = torch.relu(F.conv2d(xr, wr, bias, padding=pad)).permute(0, 2, 3, 1)
    _close(y[:, pad:pad + h, pad:pad + w, :], ref)
    border = y.clone()
    border[:, pad:pad + h, pad:pad + w, :] = 0
    assert border.abs().max().item() == 0.0


@pytest.mark.parametrize("case", [c for c in CONV_CASES if c[3] >= 32])
def test_conv_dgrad(case):
    n, h, w, cin, cout, k, pad = case
    g = torch.Generator(device=DEV).manual_seed(4)
    dy = _pad(_bf(n, h, w, cout, gen=g), pad).contiguous()
    w32 = torch.randn(cout, k * k, cin, generator=g, device=DEV) * (2.0 / (k * k * cin)) ** 0.5
    wf, wd = ops.conv_weight_prep(w32)
    mask = _pad(torch.relu(_bf(n, h, w, cin, gen=g).float()).to(torch.bfloat16), pad).contiguous()
    colsum = torch.zeros(cin, device=DEV)
    dx = ops.conv_dgrad(dy, wd, mask, n=n, h=h, w_=w, cin=cin, cout=cout, k=k, pad=pad, colsum=colsum)
    dyr = dy[:, pad:pad + h, pad:pad + w, :].permute(0, 3, 1, 2).float()
    wr = wf.float().view(cout, k, k, cin).permute(0, 3, 1, 2)
    ref = F.conv_transpose2d(dyr, wr, padding=pad).permute(0, 2, 3, 1)
    ref = ref * (mask[:, pad:pad + h, pad:pad + w, :].float() > 0)
    _close(dx[:, pad:pad + h, pad:pad + w, :], ref)
    border = dx.clone()
    border[:, pad:pad + h, pad:pad + w, :] = 0
    assert border.abs().max().item() == 0.0
    # fused bias gradient of the producing conv: the sum of the stored bf16 dx per channel
    want = dx.float().sum(dim=(0, 1, 2))
    _close(colsum, want, rtol=1e-4, atol=1e-4 * dx.float().abs().sum(dim=(0, 1, 2)).max().item())


@pytest.mark.parametrize("case", CONV_CASES)
def test_conv_wgrad(case):
    n, h, w, cin, cout, k, pad = case
    g = torch.Generator(device=DEV).manual_seed(5)
    x = _pad(_bf(n, h, w, cin, gen=g), pad).contiguous()
    dy = _pad(_bf(n, h, w, cout, gen=g), pad).contiguous()
    db = torch.zeros(cout, device=DEV)
    dw = ops.conv_wgrad(x, dy, n=n, h=h, w_=w, cin=cin, cout=cout, k=k, pad=pad, db=db)
    xr = x[:, pad:pad + h, pad:pad + w, :].permute(0, 3, 1, 2).float()
    dyr = dy[:, pad:pad + h, pad:pad + w, :].permute(0, 3, 1, 2).float()
    ref = torch.nn.grad.conv2d_weight(xr, (cout, cin, k, k), dyr, padding=pad)  # [co, ci, k, k]
    ref = ref.permute(0, 2, 3, 1).reshape(cout, k * k, cin)
    _close(dw, ref, rtol=1e-3, atol=1e-3 * ref.abs().max().item())
    _close(db, dyr.sum(dim=(0, 2, 3)), rtol=1e-3, atol=1e-3 * dyr.abs().sum(dim=(0, 2, 3)).max().item())


@pytest.mark.parametrize("case", [c for c in CONV_CASES if c[3] >= 32])
def test_slab_matches_flat_path(case, monkeypatch):
    """The slab-tiled kernels (default) and the single-tap-load kernels agree."""
    n, h, w, cin, cout, k, pad = case
    g = torch.Generator(device=DEV).manual_seed(9)
    x = _pad(torch.relu(_bf(n, h, w, cin, gen=g).float()).to(torch.bfloat16), pad).contiguous()
    wt = _bf(cout, k * k, cin, scale=(2.0 / (k * k * cin)) ** 0.5, gen=g)
    wd = _bf(cin, k * k, cout, scale=(2.0 / (k * k * cout)) ** 0.5, gen=g)
    dy = _pad(_bf(n, h, w, cout, gen=g), pad).contiguous()
    res = {}
    for mode in ("slab", "flat"):
        monkeypatch.setenv("RALPB_CONV", mode)
        y = ops.conv_fwd(x, wt, None, n=n, h=h, w_=w, cin=cin, cout=cout, k=k, pad=pad, relu=True)
        dx = ops.conv_dgrad(dy, wd, x, n=n, h=h, w_=w, cin=cin, cout=cout, k=k, pad=pad)
        dw = ops.conv_wgrad(x, dy, n=n, h=h, w_=w, cin=cin, cout=cout, k=k, pad=pad)
        torch.cuda.synchronize()
        res[mode] = (y, dx, dw)
    for a, b in zip(res["slab"], res["flat"]):
        _close(a, b, rtol=1e-2)


def test_pool_fwd_bwd():
    n, h, w, c, pad = 2, 8, 12, 64, 1
    g = torch.Generator(device=DEV).manual_seed(6)
    x = _pad(torch.relu(_bf(n, h, w, c, gen=g).float()).to(torch.bfloat16), pad).contiguous()
    y = ops.maxpool_fwd(x, n=n, h=h, w=w, c=c, pad_in=pad, k=2, stride=2, pad_out=1)
    xr = x[:, pad:pad + h, pad:pad + w, :].permute(0, 3, 1, 2).float().requires_grad_(True)
    ref = F.max_pool2d(xr, 2)
    torch.testing.assert_close(y[:, 1:-1, 1:-1, :].float(), ref.permute(0, 2, 3, 1), rtol=0, atol=0)
    dy = _bf(n, h // 2, w // 2, c, gen=g)
    colsum = torch.zeros(c, device=DEV)
    dx = ops.maxpool_bwd(x, dy.contiguous(), n=n, h=h, w=w, c=c, pad_in=pad, k=2, stride=2, pad_out=0,
                         colsum=colsum)
    ref.backward(dy.permute(0, 3, 1, 2).float())
    refdx = xr.grad.permute(0, 2, 3, 1) * (xr.detach().permute(0, 2, 3, 1) > 0)
    torch.testing.assert_close(dx[:, pad:pad + h, pad:pad + w, :].float(), refdx, rtol=0, atol=0)
    torch.testing.assert_close(colsum, refdx.sum(dim=(0, 1, 2)), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("c", [64, 192])
def test_pool_bwd_overlapping_colsum(c):
    # AlexNet's 3/2 pools (generic kernel); c = 192 -> 24 channel groups (block size 240)
    n, h, w, pad = 2, 13, 13, 0
    g = torch.Generator(device=DEV).manual_seed(16)
    x = torch.relu(_bf(n, h, w, c, gen=g).float()).to(torch.bfloat16).contiguous()
    oh = (h - 3) // 2 + 1
    dy = _bf(n, oh, oh, c, gen=g).contiguous()
    colsum = torch.zeros(c, device=DEV)
    dx = ops.maxpool_bwd(x, dy, n=n, h=h, w=w, c=c, pad_in=0, k=3, stride=2, pad_out=0, colsum=colsum)
    xr = x.permute(0, 3, 1, 2).float().requires_grad_(True)
    F.max_pool2d(xr, 3, 2).backward(dy.permute(0, 3, 1, 2).float())
    refdx = xr.grad.permute(0, 2, 3, 1) * (x.float() > 0)
    torch.testing.assert_close(dx.float(), refdx.to(torch.bfloat16).float(), rtol=1e-2, atol=1e-2)
    torch.testing.assert_close(colsum, dx.float().sum(dim=(0, 1, 2)), rtol=1e-5, atol=1e-5)
    # the argmax-byte path (forward records, backward gathers) gives the same forward and backward
    y_i, idx = ops.maxpool_fwd_idx(x, n=n, h=h, w=w, c=c, pad_in=0, k=3, stride=2, pad_out=0)
    torch.testing.assert_close(y_i.float(), F.max_pool2d(xr.detach(), 3, 2).permute(0, 2, 3, 1), rtol=0, atol=0)
    cs2 = torch.zeros(c, device=DEV)
    dx2 = ops.maxpool_bwd_gather(idx, dy, h=h, w=w, pad_in=0, k=3, stride=2, pad_out=0, colsum=cs2)
    torch.testing.assert_close(dx2.float(), dx.float(), rtol=0, atol=0)
    torch.testing.assert_close(cs2, colsum, rtol=1e-5, atol=1e-5)


def test_softmax_xent():
    g = torch.Generator(device=DEV).manual_seed(7)
    logits = torch.randn(256, 1000, generator=g, device=DEV)
    labels = torch.randint(0, 1000, (256,), generator=g, device=DEV, dtype=torch.int32)
    row_loss, dl = ops.softmax_xent(logits, labels, 1.0 / 256)
    ref = F.cross_entropy(logits, labels.long(), reduction="none")
    torch.testing.assert_close(row_loss, ref, rtol=1e-5, atol=1e-5)
    lg = logits.clone().requires_grad_(True)
    F.cross_entropy(lg, labels.long()).backward()
    _close(dl, lg.grad, rtol=1e-2, atol=1e-6)


def test_sgd_and_colsum():
    g = torch.Generator(device=DEV).manual_seed(8)
    p = torch.randn(1001, generator=g, device=DEV)
    v = torch.randn(1001, generator=g, device=DEV)
    gr = torch.randn(1001, generator=g, device=DEV)
    p0, v0 = p.clone(), v.clone()
    ops.sgd_momentum(p, v, gr, 0.01, 0.9, 0.5)
    v_ref = 0.9 * v0 + 0.5 * gr
    torch.testing.assert_close(v, v_ref)
    torch.testing.assert_close(p, p0 - 0.01 * v_ref)
    dy = _bf(5000, 192, gen=g)
    torch.testing.assert_close(ops.colsum(dy), dy.float().sum(0), rtol=1e-4, atol=1e-3)


@pytest.mark.parametrize("k,stride,pad,po,kpad,h", [(3, 1, 1, 1, 32, 20), (5, 1, 2, 0, 128, 16), (11, 4, 0, 0, 384, 63),
                                                  (11, 4, 0, 1, 384, 35), (11, 4, 0, 0, 384, 227), (11, 4, 2, 1, 384, 224)])
def test_first_conv_im2col(k, stride, pad, po, kpad, h):
    """First (RGB) conv as pack_im2col + GEMM with the bias folded into a ones column (fwd) and
    the filter/bias gradient as one MN x MN GEMM."""
    g = torch.Generator(device=DEV).manual_seed(11)
    n, c, cout = 2, 3, 64
    x = torch.randn(n, h, h, c, generator=g, device=DEV)
    cols = ops.pack_im2col(x, k=k, stride=stride, pad=pad, po=po, kpad=kpad)
    kk = k * k * c
    w = torch.randn(cout, k, k, c, generator=g, device=DEV) * (2.0 / kk) ** 0.5
    b = torch.randn(cout, generator=g, device=DEV) * 0.1
    wp = torch.zeros(cout, kpad, device=DEV)
    wp[:, :kk] = w.reshape(cout, kk)
    wp[:, kk] = b
    wb = wp.to(torch.bfloat16)
    rows = cols.shape[0] * cols.shape[1] * cols.shape[2]
    y = ops.gemm(cols.view(rows, kpad), wb.contiguous(), relu=True).view(*cols.shape[:3], cout)
    ho = cols.shape[1] - 2 * po
    xr = x.to(torch.bfloat16).float().permute(0, 3, 1, 2)
    ref = torch.relu(F.conv2d(xr, wb[:, :kk].float().view(cout, k, k, c).permute(0, 3, 1, 2),
                              wb[:, kk].float(), stride=stride, padding=pad)).permute(0, 2, 3, 1)
    _close(y[:, po:po + ho, po:po + ho, :], ref)
    dy = _bf(*cols.shape[:3], cout, gen=g)
    dw = ops.gemm(dy.view(rows, cout), cols.view(rows, kpad), a_mn=True, b_mn=True, out_kind="f32_atomic",
                  k_splits=0)
    refdw = dy.view(rows, cout).float().t() @ cols.view(rows, kpad).float()
    _close(dw, refdw, rtol=1e-3, atol=1e-3 * refdw.abs().max().item())


@pytest.mark.parametrize("n,h,w", [(2, 32, 32), (3, 16, 48), (1, 224, 224)])
def test_first_conv_fused(n, h, w):
    """Fused im2col + first conv (conv_first.cu) against torch on the same bf16-rounded inputs,
    and its filter/bias gradient against the im2col GEMM formulation."""
    g = torch.Generator(device=DEV).manual_seed(12)
    x = torch.randn(n, h, w, 3, generator=g, device=DEV)
    wp = torch.zeros(64, 32, device=DEV)
    wp[:, :27] = torch.randn(64, 27, generator=g, device=DEV) * (2.0 / 27) ** 0.5
    wp[:, 27] = torch.randn(64, generator=g, device=DEV) * 0.1
    wb = wp.to(torch.bfloat16).contiguous()
    y = ops.conv_first_fwd(x, wb, pad_out=1)
    xr = x.to(torch.bfloat16).float().permute(0, 3, 1, 2)
    wr = wb[:, :27].float().view(64, 3, 3, 3).permute(0, 3, 1, 2)
    ref = torch.relu(F.conv2d(xr, wr, wb[:, 27].float(), padding=1)).permute(0, 2, 3, 1)
    _close(y[:, 1:-1, 1:-1, :], ref)
    border = y.clone()
    border[:, 1:-1, 1:-1, :] = 0
    assert border.abs().max().item() == 0.0
    dy = _pad(_bf(n, h, w, 64, gen=g), 1).contiguous()
    dw = ops.conv_first_wgrad(x, dy, pad_out=1)
    dyr = dy[:, 1:-1, 1:-1, :].permute(0, 3, 1, 2).float()
    refw = torch.nn.grad.conv2d_weight(xr, (64, 3, 3, 3), dyr, padding=1)  # [co, ci, r, s]
    refw = refw.permute(0, 2, 3, 1).reshape(64, 27)
    _close(dw[:, :27], refw, rtol=1e-3, atol=1e-3 * refw.abs().max().item())
    refb = dyr.sum(dim=(0, 2, 3))
    _close(dw[:, 27], refb, rtol=1e-3, atol=1e-3 * refb.abs().max().item())
    assert dw[:, 28:].abs().max().item() == 0.0


@pytest.mark.parametrize("case", [(2, 8, 16, 64, 64, 3, 1), (2, 28, 28, 256, 512, 3, 1), (1, 56, 56, 128, 256, 3, 1),
                                  (2, 14, 14, 512, 512, 3, 1), (2, 32, 32, 32, 64, 5, 2)])
def test_conv_fwd_fused_pool(case):
    """conv fwd with the 2x2/2 max pool fused into its epilogue == max_pool2d of its own output."""
    n, h, w, cin, cout, k, pad = case
    g = torch.Generator(device=DEV).manual_seed(14)
    x = _pad(_bf(n, h, w, cin, gen=g), pad).contiguous()
    wt = _bf(cout, k * k, cin, scale=(2.0 / (k * k * cin)) ** 0.5, gen=g)
    bias = torch.randn(cout, device=DEV) * 0.1
    y, pooled, idx = ops.conv_fwd_pool(x, wt, bias, n=n, h=h, w_=w, cin=cin, cout=cout, k=k, pad=pad, pool_pad=1)
    y_ref = ops.conv_fwd(x, wt, bias, n=n, h=h, w_=w, cin=cin, cout=cout, k=k, pad=pad, relu=True)
    torch.testing.assert_close(y.float(), y_ref.float(), rtol=0, atol=0)
    yi = y[:, pad:pad + h, pad:pad + w, :].permute(0, 3, 1, 2).float()
    ref = F.max_pool2d(yi, 2).permute(0, 2, 3, 1)
    torch.testing.assert_close(pooled[:, 1:-1, 1:-1, :].float(), ref, rtol=0, atol=0)
    border = pooled.clone()
    border[:, 1:-1, 1:-1, :] = 0
    assert border.abs().max().item() == 0.0
    # backward from the argmax bytes == the reference pool backward (first max, ReLU mask)
    dy = _bf(n, h // 2, w // 2, cout, gen=g).contiguous()
    colsum = torch.zeros(cout, device=DEV)
    dx = ops.maxpool_bwd_idx(idx, dy, pad_out=0, pad_in=pad, colsum=colsum)
    ref_dx = ops.maxpool_bwd(y, dy, n=n, h=h, w=w, c=cout, pad_in=pad, k=2, stride=2, pad_out=0)
    torch.testing.assert_close(dx.float(), ref_dx.float(), rtol=0, atol=0)
    torch.testing.assert_close(colsum, dx.float().sum(dim=(0, 1, 2)), rtol=1e-5, atol=1e-4)


@pytest.mark.parametrize("case", [(2, 224, 224, "1"), (1, 130, 160, "1"), (3, 36, 128, "1"), (1, 130, 160, "0")])
def test_row64_fused_pool(case, monkeypatch):
    """The row-streamed 64->64 kernel with the fused 2x2/2 pool (no argmax bytes), against torch
    (two column blocks run as a CTA pair unless RALPB_ROW64_PAIR=0)."""
    n, h, w, pair = case
    monkeypatch.setenv("RALPB_ROW64_PAIR", pair)
    g = torch.Generator(device=DEV).manual_seed(21)
    x = _pad(_bf(n, h, w, 64, gen=g), 1).contiguous()
    wt = _bf(64, 9, 64, scale=(2.0 / 576) ** 0.5, gen=g)
    bias = torch.randn(64, device=DEV) * 0.1
    y, pooled, idx = ops.conv_fwd_pool(x, wt, bias, n=n, h=h, w_=w, cin=64, cout=64, k=3, pad=1, pool_pad=1,
                                       with_idx=False)
    assert idx is None
    xr = x[:, 1:1 + h, 1:1 + w, :].permute(0, 3, 1, 2).float()
    ref = torch.relu(F.conv2d(xr, wt.float().view(64, 3, 3, 64).permute(0, 3, 1, 2), bias, padding=1))
    _close(y[:, 1:1 + h, 1:1 + w, :], ref.permute(0, 2, 3, 1))
    yi = y[:, 1:1 + h, 1:1 + w, :].permute(0, 3, 1, 2).float()
    torch.testing.assert_close(pooled[:, 1:-1, 1:-1, :].float(), F.max_pool2d(yi, 2).permute(0, 2, 3, 1), rtol=0, atol=0)
    for t, inner in ((y, (1, 1 + h, 1, 1 + w)), (pooled, (1, 1 + h // 2, 1, 1 + w // 2))):
        b = t.clone()
        b[:, inner[0]:inner[1], inner[2]:inner[3], :] = 0
        assert b.abs().max().item() == 0.0
