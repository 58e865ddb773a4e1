"""Deterministic synthetic inputs and parameter initialisation.

Every global sample index g of step t gets its own counter-based stream
(numpy Philox keyed by (seed, t, g)), so any placement (1 or W workers, any
rank order) sees identical batches.  Images are N(0,1) NHWC
fp32, labels uniform in [0, classes).  Parameters: conv He-normal with fan_in
= k*k*cin, FC N(0, 0.01), biases 0.
"""
from __future__ import annotations

import numpy as np

from .planner.layers import LayerKind, ModelGraph


def _rng(*key: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence(list(key))))


def sample(seed: int, step: int, g: int, shape: tuple[int, int, int], classes: int) -> tuple[np.ndarray, int]:
    r = _rng(seed, step, g)
    img = r.standard_normal(shape, dtype=np.float32)
    lab = int(r.integers(0, classes))
    return img, lab


def batch(seed: int, step: int, first: int, count: int, shape: tuple[int, int, int],
          classes: int) -> tuple[np.ndarray, np.ndarray]:
    """Samples first..first+count-1 of step `step`: images [count,h,w,c] fp32, labels [count] int32."""
    imgs = np.empty((count, *shape), dtype=np.float32)
    labs = np.empty(count, dtype=np.int32)
    for i in range(count):
        imgs[i], labs[i] = sample(seed, step, first + i, shape, classes)
    return imgs, labs


def init_params(layers: list[dict], seed: int) -> list[tuple[np.ndarray, np.ndarray] | None]:
    """Per lowered layer: (w, b) fp32 host arrays or None.  conv w [cout][k][k][cin], fc w [out][in]."""
    out: list = []
    for i, L in enumerate(layers):
        r = _rng(seed, 0xC0FFEE, i)
        if L["kind"] == "conv":
            fan_in = L["k"] * L["k"] * L["cin"]
            w = (r.standard_normal((L["cout"], L["k"], L["k"], L["cin"]), dtype=np.float32)
                 * np.float32(np.sqrt(2.0 / fan_in)))
            if L.get("bn"):   # batch norm: scale 1, shift 0 (no bias)
                out.append((w, np.concatenate([np.ones(L["cout"], np.float32), np.zeros(L["cout"], np.float32)])))
            else:
                out.append((w, np.zeros(L["cout"], dtype=np.float32)))
        elif L["kind"] == "block":
            # wa [width][cin], wb [width][3][3][width], wc [cout][width] (, wd [cout][cin]), He-normal;
            # batch-norm scale 1, shift 0 for each convolution
            cin, width, cout = L["cin"], L["width"], L["cout"]
            shapes = [((width, cin), cin), ((width, 3, 3, width), 9 * width), ((cout, width), width)]
            if L.get("downsample"):
                shapes.append(((cout, cin), cin))
            ws = [(r.standard_normal(sh, dtype=np.float32) * np.float32(np.sqrt(2.0 / fan))).reshape(-1)
                  for sh, fan in shapes]
            bns = []
            for sh, _ in shapes:
                bns += [np.ones(sh[0], np.float32), np.zeros(sh[0], np.float32)]
            out.append((np.concatenate(ws), np.concatenate(bns)))
        elif L["kind"] == "module":
            # conv nodes in order: filters [cout][kh][kw][cin] He-normal (fan_in kh*kw*cin), then
            # batch-norm scale 1 / shift 0, or a zero bias
            from .branchy import conv_cin, node_shapes
            shp, _ = node_shapes(L["nodes"], L["h"], L["w"], L["cin"])
            ws, bs = [], []
            for j, nd in enumerate(L["nodes"]):
                if nd["op"] != "conv":
                    continue
                ci, co = conv_cin(L["nodes"], j, L["cin"], shp), nd["cout"]
                fan = nd["kh"] * nd["kw"] * ci
                ws.append((r.standard_normal((co, nd["kh"], nd["kw"], ci), dtype=np.float32)
                           * np.float32(np.sqrt(2.0 / fan))).reshape(-1))
                bs += [np.ones(co, np.float32), np.zeros(co, np.float32)] if nd["bn"] else [np.zeros(co, np.float32)]
            out.append((np.concatenate(ws), np.concatenate(bs)))
        elif L["kind"] == "fc":
            w = r.standard_normal((L["cout"], L["cin"]), dtype=np.float32) * np.float32(0.01)
            out.append((w, np.zeros(L["cout"], dtype=np.float32)))
        else:
            out.append(None)
    return out


__all__ = ["sample", "batch", "init_params", "LayerKind"]
