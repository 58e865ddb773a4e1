"""Inception-v3 and GoogLeNet as executable graphs: the geometry behind the reference catalog's
linearised `inception-v3` and `googlenet` descriptors.

The reference lists these models one catalog entry per convolution with explicit totals
(`params= out= flops=`, pkg/tools/build_catalog.py:113-285, catalog_data/{inception-v3,googlenet}.model):
a stem, branch groups whose LAST convolution entry carries the merged (concatenated) group output,
pools between stages, a global average pool and the FC classifier.  This module rebuilds both
networks from their architecture (Keras Inception-v3 at 299x299, no auxiliary head; GoogLeNet
at 224x224 without LRN / auxiliary heads), checks every catalog entry against the geometry
(names, parameters, output elements, forward FLOPs), and lowers each model to the executor's
layer table:

  conv    the first convolution (RGB, im2col GEMM; batch norm for Inception, bias for GoogLeNet)
  module  a branch group -- or one convolution the slab kernels do not cover (unpadded, strided
          or asymmetric windows) -- as a node DAG (include/ralpb.h ralpb_node_desc): conv nodes
          (window, stride, padding, batch norm or bias, ReLU), max / average pool nodes; output
          nodes concatenate in node order
  pool    max pool between stages (3x3 / 2; GoogLeNet pads 1)
  apool   global average pool;   fc   the classifier

A catalog split index (1-based over the linearised entries, profiler.py:101-134) maps to a
lowered layer boundary; cuts inside a group are not executable.  Semantics the reference does not
fix: average pools inside groups exclude padding from the count (Keras 'same' pooling); GoogLeNet's
max pools pad by one (the 224 -> 112 -> 56 -> 28 -> 14 -> 7 sizes of the catalog).
"""
from __future__ import annotations

from dataclasses import dataclass

CLASSES = 1000


@dataclass(frozen=True)
class Entry:
    name: str
    kind: str
    params: int
    out: int
    flops: int


def conv(name, inp, kh, kw, cout, *, stride=1, pad=None, bn=True, output=False):
    """A conv node; pad None = 'same' for stride 1 ((k-1)/2), 'valid' (0) otherwise."""
    ph, pw = (((kh - 1) // 2, (kw - 1) // 2) if stride == 1 else (0, 0)) if pad is None else pad
    return dict(name=name, op="conv", input=inp, kh=kh, kw=kw, stride=stride, ph=ph, pw=pw, cout=cout, bn=int(bn),
                output=int(output))


def pool(op, inp, k, stride, pad, output=False):
    return dict(name=op, op=op, input=inp, kh=k, kw=k, stride=stride, ph=pad, pw=pad, cout=0, bn=0, output=int(output))


def node_shapes(nodes, h, w, c):
    """Per node (ho, wo, channels) over a module input of h x w x c, and the module output."""
    shp = []
    for nd in nodes:
        hi, wi, ci = (h, w, c) if nd["input"] < 0 else shp[nd["input"]]
        ho = (hi + 2 * nd["ph"] - nd["kh"]) // nd["stride"] + 1
        wo = (wi + 2 * nd["pw"] - nd["kw"]) // nd["stride"] + 1
        shp.append((ho, wo, nd["cout"] if nd["op"] == "conv" else ci))
    outs = [s for s, nd in zip(shp, nodes) if nd["output"]]
    assert len({(s[0], s[1]) for s in outs}) == 1, "output nodes differ in size"
    return shp, (outs[0][0], outs[0][1], sum(s[2] for s in outs))


def conv_cin(nodes, j, c, shp):
    nd = nodes[j]
    return c if nd["input"] < 0 else shp[nd["input"]][2]


# ---------------------------------------------------------------- Inception-v3 (Keras, 299x299)
def _inception_a(pool_proj):
    return [conv("1x1", -1, 1, 1, 64, output=True),
            conv("5x5r", -1, 1, 1, 48), conv("5x5", 1, 5, 5, 64, output=True),
            conv("dbl1", -1, 1, 1, 64), conv("dbl2", 3, 3, 3, 96), conv("dbl3", 4, 3, 3, 96, output=True),
            pool("avgpool", -1, 3, 1, 1), conv("proj", 6, 1, 1, pool_proj, output=True)]


def _inception_b():   # mixed3: 35 -> 17
    return [conv("3x3", -1, 3, 3, 384, stride=2, output=True),
            conv("dbl1", -1, 1, 1, 64), conv("dbl2", 1, 3, 3, 96), conv("dbl3", 2, 3, 3, 96, stride=2, output=True),
            pool("maxpool", -1, 3, 2, 0, output=True)]


def _inception_c(c7):
    return [conv("1x1", -1, 1, 1, 192, output=True),
            conv("q1", -1, 1, 1, c7), conv("q2", 1, 1, 7, c7), conv("q3", 2, 7, 1, 192, output=True),
            conv("dbl1", -1, 1, 1, c7), conv("dbl2", 4, 7, 1, c7), conv("dbl3", 5, 1, 7, c7), conv("dbl4", 6, 7, 1, c7),
            conv("dbl5", 7, 1, 7, 192, output=True),
            pool("avgpool", -1, 3, 1, 1), conv("proj", 9, 1, 1, 192, output=True)]


def _inception_d():   # mixed8: 17 -> 8
    return [conv("3x3a", -1, 1, 1, 192), conv("3x3b", 0, 3, 3, 320, stride=2, output=True),
            conv("q1", -1, 1, 1, 192), conv("q2", 2, 1, 7, 192), conv("q3", 3, 7, 1, 192),
            conv("q4", 4, 3, 3, 192, stride=2, output=True),
            pool("maxpool", -1, 3, 2, 0, output=True)]


def _inception_e():
    return [conv("1x1", -1, 1, 1, 320, output=True),
            conv("b3a", -1, 1, 1, 384), conv("b3b", 1, 1, 3, 384, output=True), conv("b3c", 1, 3, 1, 384, output=True),
            conv("dbl1", -1, 1, 1, 448), conv("dbl2", 4, 3, 3, 384), conv("dbl3", 5, 1, 3, 384, output=True),
            conv("dbl4", 5, 3, 1, 384, output=True),
            pool("avgpool", -1, 3, 1, 1), conv("proj", 8, 1, 1, 192, output=True)]


def inception_v3_groups():
    """(name, kind, payload) in catalog order: kind conv1 / single / pool / module / apool / fc."""
    g = [("conv1", "first", conv("conv1", -1, 3, 3, 32, stride=2)),
         ("conv2", "single", conv("conv2", -1, 3, 3, 32, pad=(0, 0))),
         ("conv3", "single", conv("conv3", -1, 3, 3, 64)),
         ("pool1", "pool", (3, 2, 0)),
         ("conv4", "single", conv("conv4", -1, 1, 1, 80)),
         ("conv5", "single", conv("conv5", -1, 3, 3, 192, pad=(0, 0))),
         ("pool2", "pool", (3, 2, 0))]
    g += [(f"mixed{i}", "module", _inception_a(p)) for i, p in ((0, 32), (1, 64), (2, 64))]
    g += [("mixed3", "module", _inception_b())]
    g += [(f"mixed{i}", "module", _inception_c(c7)) for i, c7 in ((4, 128), (5, 160), (6, 160), (7, 192))]
    g += [("mixed8", "module", _inception_d())]
    g += [(f"mixed{i}", "module", _inception_e()) for i in (9, 10)]
    g += [("apool", "apool", None), ("fc", "fc", CLASSES)]
    return g


# ---------------------------------------------------------------- GoogLeNet (224x224)
def _googlenet_module(c1, c3r, c3, c5r, c5, proj):
    return [conv("1x1", -1, 1, 1, c1, bn=False, output=True),
            conv("3x3r", -1, 1, 1, c3r, bn=False), conv("3x3", 1, 3, 3, c3, bn=False, output=True),
            conv("5x5r", -1, 1, 1, c5r, bn=False), conv("5x5", 3, 5, 5, c5, bn=False, output=True),
            pool("maxpool", -1, 3, 1, 1), conv("proj", 5, 1, 1, proj, bn=False, output=True)]


GOOGLENET_TABLE = (("i3a", 64, 96, 128, 16, 32, 32), ("i3b", 128, 128, 192, 32, 96, 64), "pool3",
                   ("i4a", 192, 96, 208, 16, 48, 64), ("i4b", 160, 112, 224, 24, 64, 64),
                   ("i4c", 128, 128, 256, 24, 64, 64), ("i4d", 112, 144, 288, 32, 64, 64),
                   ("i4e", 256, 160, 320, 32, 128, 128), "pool4",
                   ("i5a", 256, 160, 320, 32, 128, 128), ("i5b", 384, 192, 384, 48, 128, 128))


def googlenet_groups():
    g = [("conv1", "first", conv("conv1", -1, 7, 7, 64, stride=2, pad=(3, 3), bn=False)),
         ("pool1", "pool", (3, 2, 1)),
         ("conv2a", "single", conv("conv2a", -1, 1, 1, 64, bn=False)),
         ("conv2b", "single", conv("conv2b", -1, 3, 3, 192, bn=False)),
         ("pool2", "pool", (3, 2, 1))]
    for row in GOOGLENET_TABLE:
        if isinstance(row, str):
            g.append((row, "pool", (3, 2, 1)))
        else:
            g.append((row[0], "module", _googlenet_module(*row[1:])))
    g += [("apool", "apool", None), ("fc", "fc", CLASSES)]
    return g


MODELS = {"inception-v3": (inception_v3_groups, (299, 299, 3)), "googlenet": (googlenet_groups, (224, 224, 3))}


def is_branchy_graph(model) -> bool:
    return getattr(model, "name", "") in MODELS


# ---------------------------------------------------------------- catalog entries / lowering
def _walk(name: str, input_hw=None):
    """Yield (group name, kind, payload, (h, w, c) in, (h, w, c) out, node shapes)."""
    groups_fn, shape = MODELS[name]
    h, w, c = shape if input_hw is None else (input_hw, input_hw, 3)
    for gname, kind, pl in groups_fn():
        if kind in ("first", "single"):
            nodes = [dict(pl, output=1)]
            shp, out = node_shapes(nodes, h, w, c)
            yield gname, kind, nodes, (h, w, c), out, shp
        elif kind == "module":
            shp, out = node_shapes(pl, h, w, c)
            yield gname, kind, pl, (h, w, c), out, shp
        elif kind == "pool":
            k, s, p = pl
            out = ((h + 2 * p - k) // s + 1, (w + 2 * p - k) // s + 1, c)
            yield gname, kind, pl, (h, w, c), out, None
        elif kind == "apool":
            out = (1, 1, c)
            yield gname, kind, None, (h, w, c), out, None
        else:
            out = (0, 0, pl)
            yield gname, kind, pl, (h, w, c), out, None
        h, w, c = out


def entries(name: str) -> list[Entry]:
    """The linearised catalog entries of the model, in catalog order."""
    es = []
    for gname, kind, pl, (h, w, c), out, shp in _walk(name):
        if kind in ("first", "single", "module"):
            nodes = pl
            convs = [j for j, nd in enumerate(nodes) if nd["op"] == "conv"]
            for j in convs:
                nd = nodes[j]
                ci = conv_cin(nodes, j, c, shp)
                ho, wo, co = shp[j]
                params = nd["kh"] * nd["kw"] * ci * co + (2 * co if nd["bn"] else co)
                flops = 2 * nd["kh"] * nd["kw"] * ci * co * ho * wo
                last = j == convs[-1]
                ename = gname if kind != "module" else f"{gname}_{nd['name']}"
                es.append(Entry(ename, "conv", params, out[0] * out[1] * out[2] if last else ho * wo * co, flops))
        elif kind in ("pool", "apool"):
            es.append(Entry(gname, "pool", 0, out[0] * out[1] * out[2], 0))
        else:
            es.append(Entry(gname, "fc", c * pl + pl, pl, 2 * c * pl))
    return es


def check_catalog(model) -> None:
    """Every catalog entry of `model` (mirror's or reference's ModelGraph) equals the geometry's."""
    ents = entries(model.name)
    if model.num_layers != len(ents):
        raise ValueError(f"{model.name}: {model.num_layers} catalog layers, the geometry has {len(ents)}")
    for L, e in zip(model.layers, ents):
        o = L.output_shape
        out = o.h * o.w * o.c if o.h else o.c
        flops = getattr(L, "compute_flops_per_sample", None)
        if L.name != e.name or L.param_count != e.params or out != e.out or (flops is not None and flops != e.flops):
            raise ValueError(f"{model.name} entry {L.name}: catalog (params {L.param_count}, out {out}, flops {flops})"
                             f" != geometry {e}")


def descriptor(name: str, batch: int = 32, note: str = "") -> str:
    """The linearised descriptor text (the catalog's explicit-totals format) from the geometry."""
    lines = [f"# {note}" if note else f"# {name}: linearised one entry per convolution; the last convolution of a",
             "# branch group carries the merged group output (generated by paper_1901_05803_b200/branchy.py)",
             f"model {name} batch={batch} elem_bytes=4"]
    for e in entries(name):
        if e.kind == "conv":
            lines.append(f"{e.name} conv params={e.params} out={e.out} flops={e.flops}")
        elif e.kind == "pool":
            lines.append(f"{e.name} pool out={e.out}")
        else:
            lines.append(f"{e.name} fc out={e.out}")
    return "\n".join(lines) + "\n"


def lower_layers(name: str, input_hw=None) -> tuple[list[dict], list[int]]:
    """Executor layer table and, per lowered layer, the catalog entries it covers.  input_hw: a
    square input other than the catalog's (the parity tests run the same graph smaller)."""
    out, counts = [], []
    for gname, kind, pl, (h, w, c), (ho, wo, co), shp in _walk(name, input_hw):
        if kind == "first":
            nd = pl[0]
            assert nd["kh"] == nd["kw"] and nd["ph"] == nd["pw"]
            out.append(dict(kind="conv", k=nd["kh"], stride=nd["stride"], pad=nd["ph"], h=h, w=w, cin=c, cout=co,
                            relu=1, bn=nd["bn"], name=gname))
            counts.append(1)
        elif kind in ("single", "module"):
            nodes = [dict(nd) for nd in pl]
            out.append(dict(kind="module", k=0, stride=0, pad=0, h=h, w=w, cin=c, cout=co, relu=1, name=gname,
                            nodes=nodes))
            counts.append(sum(1 for nd in nodes if nd["op"] == "conv"))
        elif kind == "pool":
            k, s, p = pl
            out.append(dict(kind="pool", k=k, stride=s, pad=p, h=h, w=w, cin=c, cout=c, relu=0, name=gname))
            counts.append(1)
        elif kind == "apool":
            out.append(dict(kind="apool", k=h, stride=1, pad=0, h=h, w=w, cin=c, cout=c, relu=0, name=gname))
            counts.append(1)
        else:
            out.append(dict(kind="fc", k=0, stride=0, pad=0, h=0, w=0, cin=c, cout=pl, relu=0, name=gname))
            counts.append(1)
    return out, counts


def lowered_split(name: str, split_index: int) -> int:
    """Catalog split index (entries in the front) -> lowered layers in the front."""
    layers, counts = lower_layers(name)
    covered = 0
    for i, n in enumerate(counts):
        covered += n
        if covered == split_index:
            return i + 1
        if covered > split_index:
            raise ValueError(f"{name}: split {split_index} cuts inside group {layers[i]['name']} "
                             "(not an executable cut point)")
    raise ValueError(f"{name}: split {split_index} out of range")


def module_param_counts(L: dict) -> tuple[int, int]:
    """(filter floats, bn / bias floats) of a module layer: conv nodes in order, filters
    [cout][kh][kw][cin], then [gamma | beta] (bn) or bias."""
    shp, _ = node_shapes(L["nodes"], L["h"], L["w"], L["cin"])
    nw = nb = 0
    for j, nd in enumerate(L["nodes"]):
        if nd["op"] != "conv":
            continue
        ci = conv_cin(L["nodes"], j, L["cin"], shp)
        nw += nd["kh"] * nd["kw"] * ci * nd["cout"]
        nb += (2 if nd["bn"] else 1) * nd["cout"]
    return nw, nb
