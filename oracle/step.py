"""Oracle restatement of one layer-placed (RALP) / all-on-PS (baseline) training step
on the CPU in plain PyTorch fp32 (test infrastructure only).

Schedule (pkg/src/ralp/simulator.py:669-715 for RALP, :637-665 for the baseline):
  RALP      W worker fronts (conv/pool) on their own batches -> cuts concatenated
            (W*b rows, HWC flatten, layers.py:62-66) -> FC tail once on the PS with
            FC weights fixed for the whole step -> act-grads split
            back -> W front backwards -> conv grads summed -> SGD-momentum; the FC tail
            is updated locally on the PS.
  baseline  every worker runs the whole model on its own batch; all grads summed.
Loss = mean cross-entropy over the W*b samples of the step; SGD in the PyTorch
form v = mu*v + g, p -= lr*v; ReLU after every conv/FC except the last;
max pool routes to the first maximum in row-major window order.

`emulate_bf16=True` rounds to bf16 exactly where the B200 path stores bf16
(packed input, every activation and activation-gradient, the bf16 weight copies
used by the GEMMs, dlogits) and keeps fp32 everywhere else (GEMM accumulation,
logits, gradients of parameters, master weights, momentum).

The byte counter adds the descriptor-unit (elem_bytes) size of every logical
transfer at the reference's count_wire sites (simulator.py:647,663,677,689,707,713).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as F


@dataclass
class OracleState:
    layers: list            # lowered layer dicts (kind, k, stride, pad, h, w, cin, cout, relu)
    params: list            # per layer: (w, b) fp32 numpy (conv w [cout][k][k][cin], fc w [out][in]) or None
    momentum: list = field(default_factory=list)

    def __post_init__(self):
        self.params = [None if p is None else (torch.tensor(p[0], dtype=torch.float32),
                                               torch.tensor(p[1], dtype=torch.float32)) for p in self.params]
        if not self.momentum:
            self.momentum = [None if p is None else (torch.zeros_like(p[0]), torch.zeros_like(p[1]))
                             for p in self.params]

    def numpy_params(self):
        return [None if p is None else (p[0].numpy().copy(), p[1].numpy().copy()) for p in self.params]


def _round(x: torch.Tensor, on: bool) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32) if on else x


# Accumulation precision of every contraction (float32 normally; float64 to measure the
# intrinsic sensitivity of the bf16 pipeline to summation-order noise).
_ACC = [torch.float32]


def _acc(*ts):
    return [None if t is None else t.to(_ACC[0]) for t in ts]


def _conv(x, w, b, stride, pad):
    x, w, b = _acc(x, w, b)
    return F.conv2d(x, w, b, stride=stride, padding=pad).to(torch.float32)


def _mm(a, b):
    a, b = _acc(a, b)
    return (a @ b).to(torch.float32)


def _conv_w(x, shape, g, stride, pad):
    x, g = _acc(x, g)
    return torch.nn.grad.conv2d_weight(x, shape, g, stride=stride, padding=pad).to(torch.float32)


def _conv_x(shape, w, g, stride, pad):
    w, g = _acc(w, g)
    return torch.nn.grad.conv2d_input(shape, w, g, stride=stride, padding=pad).to(torch.float32)


def _split_index(layers) -> int:
    return next(i for i, L in enumerate(layers) if L["kind"] == "fc")


def _front_forward(st: OracleState, nfront: int, imgs: np.ndarray, bf: bool):
    x = _round(torch.from_numpy(np.ascontiguousarray(imgs)).permute(0, 3, 1, 2).contiguous(), bf)
    acts = [x]
    for i in range(nfront):
        L = st.layers[i]
        if L["kind"] == "conv":
            w, b = st.params[i]
            wt = _round(w.permute(0, 3, 1, 2).contiguous(), bf)
            # the first (RGB, cin <= 4) conv runs on the B200 as an im2col GEMM whose bias is
            # a bf16 filter column multiplying a ones column
            bias = _round(b, bf) if i == 0 and L["cin"] <= 4 else b
            x = _round(torch.relu(_conv(x, wt, bias, L["stride"], L["pad"])), bf)
        else:
            x = F.max_pool2d(x, L["k"], L["stride"])
        acts.append(x)
    cut = x.permute(0, 2, 3, 1).reshape(x.shape[0], -1)  # HWC flatten
    return acts, cut


def _back(st: OracleState, nfront: int, x: torch.Tensor, labels: np.ndarray, scale: float, bf: bool):
    """FC tail fwd + CE + bwd on R rows; returns (mean loss, {layer: (gw, gb)}, d(cut))."""
    fcs = list(range(nfront, len(st.layers)))
    hs = [x]
    logits = None
    for j, li in enumerate(fcs):
        w, b = st.params[li]
        z = _mm(hs[-1], _round(w, bf).t()) + b
        if j + 1 < len(fcs):
            hs.append(_round(torch.relu(z), bf))
        else:
            logits = z
    lab = torch.from_numpy(np.asarray(labels, dtype=np.int64))
    lse = torch.logsumexp(logits, dim=1)
    row_loss = lse - logits.gather(1, lab[:, None])[:, 0]
    p = torch.exp(logits - lse[:, None])
    onehot = F.one_hot(lab, logits.shape[1]).to(torch.float32)
    dy = _round((p - onehot) * scale, bf)
    grads = {}
    for j in reversed(range(len(fcs))):
        li = fcs[j]
        w, _ = st.params[li]
        xin = hs[j]
        grads[li] = (_mm(dy.t(), xin), dy.sum(0))
        dx = _mm(dy, _round(w, bf))
        if j > 0:
            dx = dx * (xin > 0)
        dy = _round(dx, bf)
    return float(row_loss.mean()), grads, dy


def _front_backward(st: OracleState, nfront: int, acts, dcut: torch.Tensor, bf: bool):
    last = acts[-1]
    g = dcut.reshape(last.shape[0], last.shape[2], last.shape[3], last.shape[1]).permute(0, 3, 1, 2)
    grads = {}
    for i in reversed(range(nfront)):
        L = st.layers[i]
        xin = acts[i]
        if L["kind"] == "pool":
            xr = xin.detach().clone().requires_grad_(True)
            F.max_pool2d(xr, L["k"], L["stride"]).backward(g)
            g = _round(xr.grad * (xin > 0), bf)
        else:
            w, _ = st.params[i]
            wt = _round(w.permute(0, 3, 1, 2).contiguous(), bf)
            gw = _conv_w(xin, wt.shape, g, L["stride"], L["pad"])
            grads[i] = (gw.permute(0, 2, 3, 1).contiguous(), g.sum(dim=(0, 2, 3)))
            if i > 0:
                gx = _conv_x(xin.shape, wt, g, L["stride"], L["pad"])
                if st.layers[i - 1]["kind"] == "conv":
                    gx = gx * (xin > 0)
                g = _round(gx, bf)
    return grads


def _sgd(st: OracleState, idx, grad, lr, mu):
    (w, b), (vw, vb) = st.params[idx], st.momentum[idx]
    vw.mul_(mu).add_(grad[0])
    vb.mul_(mu).add_(grad[1])
    w.sub_(lr * vw)
    b.sub_(lr * vb)


def _accumulate(total: dict, part: dict):
    for k, (gw, gb) in part.items():
        if k in total:
            total[k] = (total[k][0] + gw, total[k][1] + gb)
        else:
            total[k] = (gw.clone(), gb.clone())


# ---------------------------------------------------------------- per-layer ops (teacher forcing)
# Each takes the GPU's own stored inputs (NCHW fp32 tensors holding bf16 values) and returns the
# layer's exact fp32 result before the GPU's final bf16 rounding, so a per-layer check isolates one
# kernel from the drift of everything before it.  Semantics as in the step above: infer_conv /
# infer_pool / infer_fc (pkg/src/ralp/layers.py:87-123), ReLU after every conv / hidden FC.

def conv_forward(x, w, b, stride, pad, relu=True):
    """relu(conv2d(x, w) + b); w [cout][cin][k][k] (already bf16-valued where the GPU's is)."""
    y = _conv(x, w, b, stride, pad)
    return torch.relu(y) if relu else y


def conv_backward_data(dy, w, x_shape, stride, pad, mask=None):
    """dL/dx of a convolution from its (masked) output gradient; times (mask > 0) when given."""
    gx = _conv_x(x_shape, w, dy, stride, pad)
    return gx * (mask > 0) if mask is not None else gx


def conv_backward_filter(x, dy, w_shape, stride, pad):
    """(dW [cout][cin][k][k], db [cout]) summed over the batch."""
    return _conv_w(x, w_shape, dy, stride, pad), dy.to(torch.float64).sum(dim=(0, 2, 3)).to(torch.float32)


def maxpool_forward(x, k, stride):
    return F.max_pool2d(x, k, stride)


def maxpool_backward(x, dy, k, stride):
    """Route dy to the first maximum of each window (row-major), times (x > 0): the pool input
    is a ReLU output, whose derivative the GPU folds into this producer."""
    xr = x.detach().clone().requires_grad_(True)
    F.max_pool2d(xr, k, stride).backward(dy)
    return xr.grad * (x > 0)


def fc_forward(x, w, b, relu):
    z = _mm(x, w.t()) + b
    return torch.relu(z) if relu else z


def softmax_xent(logits, labels, scale):
    """(per-row loss, dlogits = (softmax - onehot) * scale) -- the LOSS layer (layers.py:161-163)."""
    lab = torch.from_numpy(np.asarray(labels, dtype=np.int64))
    lse = torch.logsumexp(logits.double(), dim=1)
    row = lse - logits.double().gather(1, lab[:, None])[:, 0]
    p = torch.exp(logits.double() - lse[:, None])
    d = (p - F.one_hot(lab, logits.shape[1]).double()) * scale
    return row.float(), d.float()


def param_count(L) -> int:
    if L["kind"] == "conv":
        return L["k"] * L["k"] * L["cin"] * L["cout"] + L["cout"] * (2 if L.get("bn") else 1)
    if L["kind"] == "block":
        cin, width, cout, down = L["cin"], L["width"], L["cout"], L.get("downsample", 0)
        return (width * cin + 9 * width * width + cout * width + (cout * cin if down else 0)
                + 2 * (2 * width + cout + (cout if down else 0)))
    if L["kind"] == "module":
        return sum(w.numel() + b.numel() for w, b in _module_shapes(L))
    if L["kind"] == "fc":
        return L["cin"] * L["cout"] + L["cout"]
    return 0


def _module_shapes(L):
    """Per conv node of a module layer: (empty filter tensor [cout][kh][kw][cin], empty bn/bias)."""
    chans, out = [], []
    for nd in L["nodes"]:
        ci = L["cin"] if nd["input"] < 0 else chans[nd["input"]]
        chans.append(nd["cout"] if nd["op"] == "conv" else ci)
        if nd["op"] == "conv":
            out.append((torch.empty(nd["cout"], nd["kh"], nd["kw"], ci),
                        torch.empty(nd["cout"] * (2 if nd["bn"] else 1))))
    return out


def _module_forward(L, p, x, R, dtype):
    """A branch group (graph.cu): nodes in order over the module input x (NCHW), conv nodes with
    batch norm + ReLU or bias + ReLU, max pools (padding never wins), average pools (padding not
    counted); output nodes concatenated along channels.  p = (filters, bn / bias) flat, conv nodes
    in order, filters [cout][kh][kw][cin]."""
    w, b = p
    conv_ids = [j for j, nd in enumerate(L["nodes"]) if nd["op"] == "conv"]
    pw, ow, ob = {}, 0, 0
    for (wt, bt), j in zip(_module_shapes(L), conv_ids):
        pw[j] = (w[ow:ow + wt.numel()].reshape(wt.shape).permute(0, 3, 1, 2).to(dtype), b[ob:ob + bt.numel()].to(dtype))
        ow += wt.numel()
        ob += bt.numel()
    vals = []
    for j, nd in enumerate(L["nodes"]):
        src = x if nd["input"] < 0 else vals[nd["input"]]
        win, st, pad = (nd["kh"], nd["kw"]), nd["stride"], (nd["ph"], nd["pw"])
        if nd["op"] == "conv":
            wt, bt = R(pw[j][0]), pw[j][1]
            if nd["bn"]:
                c = nd["cout"]
                z = R(F.conv2d(src, wt, None, stride=st, padding=pad))
                y = R(torch.relu(_bn(z, bt[:c], bt[c:])))
            else:
                y = R(torch.relu(F.conv2d(src, wt, bt, stride=st, padding=pad)))
        elif nd["op"] == "maxpool":
            y = R(F.max_pool2d(src, win, st, pad))
        else:
            y = R(F.avg_pool2d(src, win, st, pad, count_include_pad=False))
        vals.append(y)
    return torch.cat([v for v, nd in zip(vals, L["nodes"]) if nd["output"]], dim=1)


# ---------------------------------------------------------------- branchy models (autograd restatement)
class _Round(torch.autograd.Function):
    """bf16 storage point: rounds the value on the way forward and its gradient on the way back
    (the GPU stores both the activation and the gradient w.r.t. it in bf16)."""

    @staticmethod
    def forward(ctx, x):
        return x.to(torch.bfloat16).to(x.dtype)

    @staticmethod
    def backward(ctx, g):
        return g.to(torch.bfloat16).to(g.dtype)


def _block_params(L, w, b):
    """Split a block's flat (w, b) into its tensors (executor.block_param_counts order)."""
    cin, width, cout, down = L["cin"], L["width"], L["cout"], L.get("downsample", 0)
    shapes = [(width, cin, 1, 1), (width, width, 3, 3), (cout, width, 1, 1)] + ([(cout, cin, 1, 1)] if down else [])
    ws, o = [], 0
    for sh in shapes:
        n = int(np.prod(sh))
        if len(sh) == 4 and sh[2] == 3:   # stored [co][kh][kw][ci]
            ws.append(w[o:o + n].reshape(sh[0], 3, 3, sh[1]).permute(0, 3, 1, 2))
        else:
            ws.append(w[o:o + n].reshape(sh))
        o += n
    bns, o = [], 0
    for sh in shapes:
        bns.append((b[o:o + sh[0]], b[o + sh[0]:o + 2 * sh[0]]))
        o += 2 * sh[0]
    return ws, bns


def _bn(x, gamma, beta):
    """Training-mode batch norm over the (worker's) batch, biased variance, eps 1e-5."""
    return F.batch_norm(x, None, None, gamma, beta, training=True, momentum=0.0, eps=1e-5)


def _branchy_forward(layers, params, x, R, dtype):
    """Forward of a model with blocks / batch-normalised convs / padded and average pools, bf16
    storage emulated by R at the GPU's storage points (block.cu, resnet.cu).  Returns logits."""
    for L, p in zip(layers, params):
        k = L["kind"]
        if k == "conv":
            w, b = p
            wt = R(w.permute(0, 3, 1, 2).contiguous().to(dtype))
            if L.get("bn"):
                c = L["cout"]
                pre = R(F.conv2d(x, wt, None, stride=L["stride"], padding=L["pad"]))
                x = R(torch.relu(_bn(pre, b[:c].to(dtype), b[c:].to(dtype))))
            else:   # the first (im2col) conv carries its bias in a bf16 filter column
                bias = R(b.to(dtype)) if L is layers[0] else b.to(dtype)
                x = R(torch.relu(F.conv2d(x, wt, bias, stride=L["stride"], padding=L["pad"])))
        elif k == "pool":
            x = R(F.max_pool2d(x, L["k"], L["stride"], L["pad"]))
        elif k == "block":
            ws, bns = _block_params(L, p[0].to(dtype), p[1].to(dtype))
            s = L["stride"]
            a = R(torch.relu(_bn(R(F.conv2d(x, R(ws[0]))), *bns[0])))
            bb = R(torch.relu(_bn(R(F.conv2d(a, R(ws[1]), stride=s, padding=1)), *bns[1])))
            c = _bn(R(F.conv2d(bb, R(ws[2]))), *bns[2])
            short = _bn(R(F.conv2d(x[:, :, ::s, ::s], R(ws[3]))), *bns[3]) if L.get("downsample") else x
            x = R(torch.relu(c + short))
        elif k == "module":
            x = _module_forward(L, p, x, R, dtype)
        elif k == "apool":
            x = R(x.mean(dim=(2, 3), keepdim=True))
        elif k == "fc":
            if x.dim() == 4:
                x = x.permute(0, 2, 3, 1).reshape(x.shape[0], -1)   # HWC flatten
            w, b = p
            last = L is layers[-1]
            z = x @ R(w.to(dtype)).t() + b.to(dtype)
            x = z if last else R(torch.relu(z))
    return x


def _train_step_branchy(st: OracleState, strategy: str, workers: int, batches, *, lr, mu, emulate_bf16, elem_bytes,
                        accum64, split):
    dtype = torch.float64 if accum64 else torch.float32
    R = _Round.apply if emulate_bf16 else (lambda t: t)
    leaves = []
    params = []
    for p in st.params:
        if p is None:
            params.append(None)
            continue
        w = p[0].detach().to(dtype).clone().requires_grad_(True)
        b = p[1].detach().to(dtype).clone().requires_grad_(True)
        leaves.append((w, b))
        params.append((w, b))
    b_sz = batches[0][0].shape[0]
    total = 0.0
    for imgs, labs in batches:   # every worker runs its front (and its batch norm) on its own batch
        x = R(torch.from_numpy(np.ascontiguousarray(imgs)).permute(0, 3, 1, 2).contiguous().to(dtype))
        logits = _branchy_forward(st.layers, params, x, R, dtype)
        lab = torch.from_numpy(np.asarray(labs, dtype=np.int64))
        loss = F.cross_entropy(logits, lab, reduction="sum") / (workers * b_sz)
        loss.backward()
        total += float(loss.detach())
    grads = {}
    for i, p in enumerate(params):
        if p is not None:
            grads[i] = (p[0].grad.to(torch.float32).reshape(st.params[i][0].shape), p[1].grad.to(torch.float32))
    for idx, g in grads.items():
        _sgd(st, idx, g, lr, mu)
    nfront = _split_index(st.layers)
    cut_at = nfront if split is None else split
    wire = 0
    if strategy == "ralp":
        with torch.no_grad():
            x = torch.from_numpy(np.ascontiguousarray(batches[0][0])).permute(0, 3, 1, 2).contiguous()
            for L, p in zip(st.layers[:cut_at], st.params[:cut_at]):
                x = _branchy_forward([L], [p], x, lambda t: t, torch.float32)
        cut_elems = x[0].numel()
        p_front = sum(param_count(L) for L in st.layers[:cut_at]) * elem_bytes
        wire = workers * (2 * b_sz * cut_elems * elem_bytes + 2 * p_front)
    else:
        wire = 2 * workers * sum(param_count(L) for L in st.layers) * elem_bytes
    return total, wire


def _branchy(layers) -> bool:
    return any(L["kind"] in ("block", "apool", "module") or L.get("bn") or (L["kind"] == "pool" and L.get("pad"))
               for L in layers)


def train_step(st: OracleState, strategy: str, workers: int, batches, *, lr: float = 0.01, mu: float = 0.9,
               emulate_bf16: bool = False, elem_bytes: int = 4, accum64: bool = False, split: int | None = None):
    """One step.  batches[r] = (images [b,h,w,c] fp32, labels [b] int) of worker r.
    split (RALP): the partitioner's 1-based cut index (profiler.py:101-134); None = the FC
    boundary.  A conv / pool back segment [split, first FC) runs on the PS over the gathered rows;
    those layers act on every image independently and their weights are fixed within the step, so
    the numerics equal running them on each worker (what this restatement does) -- only the cut
    shipped and the synchronised front differ, in the byte count.
    Returns (loss, logical_bytes)."""
    if _branchy(st.layers):
        return _train_step_branchy(st, strategy, workers, batches, lr=lr, mu=mu, emulate_bf16=emulate_bf16,
                                   elem_bytes=elem_bytes, accum64=accum64, split=split)
    _ACC[0] = torch.float64 if accum64 else torch.float32
    bf = emulate_bf16
    nfront = _split_index(st.layers)
    cut_at = nfront if split is None else split
    b = batches[0][0].shape[0]
    scale = 1.0 / (workers * b)
    wire = 0
    p_front = sum(param_count(L) for L in st.layers[:cut_at]) * elem_bytes
    p_all = sum(param_count(L) for L in st.layers) * elem_bytes
    total: dict = {}
    if strategy == "ralp":
        fronts = [_front_forward(st, nfront, imgs, bf) for imgs, _ in batches]
        cut_bytes = fronts[0][0][cut_at].numel() * elem_bytes   # layer cut_at-1's output (acts[cut_at])
        wire += workers * cut_bytes                        # "act" (simulator.py:677)
        x = torch.cat([c for _, c in fronts], dim=0)
        labels = np.concatenate([lab for _, lab in batches])
        loss, fc_grads, dcut = _back(st, nfront, x, labels, scale, bf)
        wire += workers * cut_bytes                        # "actgrad" (simulator.py:707)
        for r, (acts, _) in enumerate(fronts):
            _accumulate(total, _front_backward(st, nfront, acts, dcut[r * b:(r + 1) * b], bf))
        wire += 2 * workers * p_front                      # "grad" + "pull" (simulator.py:689,713)
        for idx, g in total.items():
            _sgd(st, idx, g, lr, mu)
        for idx, g in fc_grads.items():                    # PS-local FC update
            _sgd(st, idx, g, lr, mu)
        return loss, wire
    if strategy == "baseline":
        losses = []
        for imgs, lab in batches:
            acts, cut = _front_forward(st, nfront, imgs, bf)
            loss, fc_grads, dcut = _back(st, nfront, cut, lab, scale, bf)
            losses.append(loss)
            _accumulate(total, fc_grads)
            _accumulate(total, _front_backward(st, nfront, acts, dcut, bf))
        wire += 2 * workers * p_all                         # push + pull (simulator.py:647,663)
        for idx, g in total.items():
            _sgd(st, idx, g, lr, mu)
        return float(np.mean(losses)), wire
    raise ValueError(strategy)
