"""Per-kernel Python wrappers over the C ABI (device tensors in, device tensors out).

These exist for the kernel parity tests and for debugging; the training step
itself is driven natively by the executor inside libralpb200.so.  Every
function launches on torch's current CUDA stream.
"""
from __future__ import annotations

import torch

from ._lib import call

_BF16 = torch.bfloat16


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _p(t):
    return None if t is None else t.data_ptr()


def gemm(a: torch.Tensor, b: torch.Tensor, *, a_mn: bool = False, b_mn: bool = False,
         out: torch.Tensor | None = None, out_kind: str = "bf16", bias: torch.Tensor | None = None,
         relu: bool = False, mask: torch.Tensor | None = None, k_splits: int = 1,
         block_n: int = 0) -> torch.Tensor:
    """out[m, n] = sum_k A[m,k] B[n,k]; A is [M,K] (a_mn=False) or [K,M] (a_mn=True)."""
    assert a.dtype == _BF16 and b.dtype == _BF16 and a.is_contiguous() and b.is_contiguous()
    M = a.shape[1] if a_mn else a.shape[0]
    K = a.shape[0] if a_mn else a.shape[1]
    N = b.shape[1] if b_mn else b.shape[0]
    kind = {"bf16": 0, "f32": 1, "f32_atomic": 2}[out_kind]
    if out is None:
        dt = _BF16 if kind == 0 else torch.float32
        out = (torch.zeros if kind == 2 else torch.empty)(M, N, dtype=dt, device=a.device)
    call("ralpb_gemm_bf16", a.data_ptr(), a.shape[0], a.shape[1], a.stride(0), int(a_mn),
         b.data_ptr(), b.shape[0], b.shape[1], b.stride(0), int(b_mn), M, N, K, out.data_ptr(), kind,
         out.stride(0), out.stride(1), _p(bias), int(relu), _p(mask), 0 if mask is None else mask.stride(0),
         k_splits, block_n, _stream())
    return out


def conv_fwd(x_pad, w, bias, *, n, h, w_, cin, cout, k, pad, relu=True, out=None):
    if out is None:  # interior-only writes: the padded border must start at zero
        out = torch.zeros(n, h + 2 * pad, w_ + 2 * pad, cout, dtype=_BF16, device=x_pad.device)
    call("ralpb_conv_fwd", x_pad.data_ptr(), w.data_ptr(), _p(bias), out.data_ptr(), n, h, w_, cin, cout,
         k, pad, int(relu), _stream())
    return out


def conv_fwd_pool(x_pad, w, bias, *, n, h, w_, cin, cout, k, pad, relu=True, pool_pad=1, with_idx=True):
    """(y, pooled, argmax bytes or None): conv fwd and its 2x2/2 max pool from one kernel."""
    y = torch.zeros(n, h + 2 * pad, w_ + 2 * pad, cout, dtype=_BF16, device=x_pad.device)
    pooled = torch.zeros(n, h // 2 + 2 * pool_pad, w_ // 2 + 2 * pool_pad, cout, dtype=_BF16, device=x_pad.device)
    idx = torch.empty(n, h // 2, w_ // 2, cout, dtype=torch.uint8, device=x_pad.device) if with_idx else None
    call("ralpb_conv_fwd_pool", x_pad.data_ptr(), w.data_ptr(), _p(bias), y.data_ptr(), pooled.data_ptr(), pool_pad,
         _p(idx), n, h, w_, cin, cout, k, pad, int(relu), _stream())
    return y, pooled, idx


def maxpool_fwd_idx(x_pad, *, n, h, w, c, pad_in, k, stride, pad_out):
    oh, ow = (h - k) // stride + 1, (w - k) // stride + 1
    y = torch.empty(n, oh + 2 * pad_out, ow + 2 * pad_out, c, dtype=_BF16, device=x_pad.device)
    idx = torch.empty(n, oh, ow, c, dtype=torch.uint8, device=x_pad.device)
    call("ralpb_maxpool_fwd_idx", x_pad.data_ptr(), n, h, w, c, pad_in, k, stride, y.data_ptr(), pad_out,
         idx.data_ptr(), _stream())
    return y, idx


def maxpool_bwd_gather(idx, dy, *, h, w, pad_in, k, stride, pad_out, colsum=None):
    n, _, _, c = idx.shape
    dx = torch.zeros(n, h + 2 * pad_in, w + 2 * pad_in, c, dtype=_BF16, device=dy.device)
    call("ralpb_maxpool_bwd_gather", idx.data_ptr(), dy.data_ptr(), n, h, w, c, pad_in, k, stride, pad_out,
         dx.data_ptr(), _p(colsum), _stream())
    return dx


def maxpool_bwd_idx(idx, dy, *, pad_out, pad_in, colsum=None):
    n, oh, ow, c = idx.shape
    dx = torch.zeros(n, 2 * oh + 2 * pad_in, 2 * ow + 2 * pad_in, c, dtype=_BF16, device=dy.device)
    call("ralpb_maxpool_bwd_idx", idx.data_ptr(), dy.data_ptr(), n, oh, ow, c, pad_out, pad_in, dx.data_ptr(),
         _p(colsum), _stream())
    return dx


def conv_first_fwd(img, wf, *, pad_out=1):
    """Fused im2col + first conv (3x3/1/1, 3 -> 64, ReLU); img fp32 [n,h,w,3], wf bf16 [64,32]."""
    n, h, w, _ = img.shape
    y = torch.zeros(n, h + 2 * pad_out, w + 2 * pad_out, 64, dtype=_BF16, device=img.device)
    call("ralpb_conv_first_fwd", img.data_ptr(), n, h, w, wf.data_ptr(), y.data_ptr(), pad_out, _stream())
    return y


def conv_first_wgrad(img, dy_pad, *, pad_out=1, dw=None):
    n, h, w, _ = img.shape
    if dw is None:
        dw = torch.zeros(64, 32, dtype=torch.float32, device=img.device)
    call("ralpb_conv_first_wgrad", img.data_ptr(), n, h, w, dy_pad.data_ptr(), pad_out, dw.data_ptr(), _stream())
    return dw


def conv_dgrad(dy_pad, wd, mask_pad, *, n, h, w_, cin, cout, k, pad, out=None, colsum=None):
    """dx (and, if `colsum` is given, colsum += per-channel sum of the stored dx)."""
    if out is None:
        out = torch.zeros(n, h + 2 * pad, w_ + 2 * pad, cin, dtype=_BF16, device=dy_pad.device)
    call("ralpb_conv_dgrad", dy_pad.data_ptr(), wd.data_ptr(), _p(mask_pad), out.data_ptr(), _p(colsum), n, h, w_,
         cin, cout, k, pad, _stream())
    return out


def conv_wgrad(x_pad, dy_pad, *, n, h, w_, cin, cout, k, pad, out=None, db=None):
    """dW[co][t][ci] (+= into `out`) and, when `db` is given, the bias gradient (+= into db)."""
    if out is None:
        out = torch.zeros(cout, k * k, cin, dtype=torch.float32, device=x_pad.device)
    call("ralpb_conv_wgrad", x_pad.data_ptr(), dy_pad.data_ptr(), out.data_ptr(), _p(db), n, h, w_, cin, cout, k,
         pad, _stream())
    return out


def pack_input(x, cp, pad):
    n, h, w, c = x.shape
    out = torch.empty(n, h + 2 * pad, w + 2 * pad, cp, dtype=_BF16, device=x.device)
    call("ralpb_pack_input", x.data_ptr(), n, h, w, c, out.data_ptr(), cp, pad, _stream())
    return out


def pack_im2col(x, *, k, stride, pad, po, kpad):
    n, h, w, c = x.shape
    ho, wo = (h + 2 * pad - k) // stride + 1, (w + 2 * pad - k) // stride + 1
    out = torch.empty(n, ho + 2 * po, wo + 2 * po, kpad, dtype=_BF16, device=x.device)
    call("ralpb_pack_im2col", x.data_ptr(), n, h, w, c, k, stride, pad, ho, wo, po, kpad, out.data_ptr(), _stream())
    return out


def maxpool_fwd(x_pad, *, n, h, w, c, pad_in, k, stride, pad_out):
    oh, ow = (h - k) // stride + 1, (w - k) // stride + 1
    y = torch.empty(n, oh + 2 * pad_out, ow + 2 * pad_out, c, dtype=_BF16, device=x_pad.device)
    call("ralpb_maxpool_fwd", x_pad.data_ptr(), n, h, w, c, pad_in, k, stride, y.data_ptr(), pad_out, _stream())
    return y


def maxpool_bwd(x_pad, dy, *, n, h, w, c, pad_in, k, stride, pad_out, colsum=None):
    dx = torch.zeros_like(x_pad)  # borders / uncovered positions are not written
    call("ralpb_maxpool_bwd", x_pad.data_ptr(), dy.data_ptr(), n, h, w, c, pad_in, k, stride, pad_out,
         dx.data_ptr(), _p(colsum), _stream())
    return dx


def softmax_xent(logits, labels, scale):
    rows, classes = logits.shape
    row_loss = torch.empty(rows, dtype=torch.float32, device=logits.device)
    dl = torch.empty(rows, classes, dtype=_BF16, device=logits.device)
    call("ralpb_softmax_xent", logits.data_ptr(), rows, classes, logits.stride(0), labels.data_ptr(),
         float(scale), row_loss.data_ptr(), dl.data_ptr(), dl.stride(0), _stream())
    return row_loss, dl


def sgd_momentum(p, v, g, lr, mu, gscale=1.0):
    call("ralpb_sgd_momentum", p.data_ptr(), v.data_ptr(), g.data_ptr(), p.numel(), float(lr), float(mu),
         float(gscale), _stream())


def colsum(dy2d, out=None):
    rows, c = dy2d.shape
    if out is None:
        out = torch.zeros(c, dtype=torch.float32, device=dy2d.device)
    call("ralpb_colsum_bf16", dy2d.data_ptr(), rows, c, dy2d.stride(0), out.data_ptr(), _stream())
    return out


def conv_weight_prep(w32):
    co, taps, ci = w32.shape
    wf = torch.empty(co, taps, ci, dtype=_BF16, device=w32.device)
    wd = torch.empty(ci, taps, co, dtype=_BF16, device=w32.device)
    call("ralpb_conv_weight_prep", w32.data_ptr(), co, taps, ci, wf.data_ptr(), wd.data_ptr(), _stream())
    return wf, wd
