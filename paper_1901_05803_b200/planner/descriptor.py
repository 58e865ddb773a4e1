"""Text model descriptors: `model <name> batch=<n> elem_bytes=<n> [input=HxWxC|N]`
then one `<name> <kind> key=value ...` line per layer; `#` comments.

Same document format and error classes as the reference parser
(pkg/src/ralp/descriptor.py:84-224): derived layers are shape-checked against
their predecessor (cin=, in=), explicit layers give `params= out= flops=`
(fused blocks, linearised branchy models), `shape=` overrides the output shape.

VENDORED API MIRROR (attribution): this module follows the reference `ralp` package's own code for
the same surface closely -- same classes, checks, error messages and arithmetic -- because north_star
makes that planner API the drop-in surface and its outputs must match the reference bit-exactly
(tests/test_planner_golden.py pins them to the unmodified reference).  It is not original work and
it is not on the GPU path; the executor accepts the reference's own objects as well
(executor.py `_kv`).
"""
from __future__ import annotations

import re
from typing import Optional

from .layers import LayerKind, LayerSpec, ModelError, ModelGraph, TensorShape, infer_layer

_KINDS = {k.value: k for k in LayerKind}
_INTEGER_KEYS = frozenset({"k", "cin", "cout", "stride", "pad", "window", "in", "out", "params", "flops",
                           "batch", "elem_bytes"})
_TOKEN = re.compile(r"\S+")


class DescriptorError(ValueError):
    """Syntax or consistency error at a (1-based) line/column."""

    def __init__(self, message: str, line: int, column: int = 1):
        super().__init__(f"line {line}, column {column}: {message}")
        self.line = line
        self.column = column


class ShapeMismatchError(DescriptorError):
    """A layer's declared input disagrees with what its predecessor produces."""


def _shape(text: str, line: int, col: int) -> TensorShape:
    try:
        dims = [int(part) for part in text.lower().split("x")]
    except ValueError:
        dims = []
    if len(dims) == 1:
        return TensorShape.flat(dims[0])
    if len(dims) == 3:
        return TensorShape(*dims)
    raise DescriptorError(f"bad shape {text!r} (expected HxWxC or N)", line, col)


def _pairs(tokens: list[tuple[str, int]], line: int) -> dict[str, object]:
    out: dict[str, object] = {}
    for tok, col in tokens:
        key, eq, val = tok.partition("=")
        if not eq or not key or not val:
            raise DescriptorError(f"expected key=value, got {tok!r}", line, col)
        if key in out:
            raise DescriptorError(f"duplicate key {key!r}", line, col)
        if key in _INTEGER_KEYS:
            try:
                out[key] = int(val)
            except ValueError:
                raise DescriptorError(f"key {key!r} needs an integer, got {val!r}", line, col) from None
        else:
            out[key] = val
    return out


def parse_model(text: str) -> ModelGraph:
    header: Optional[dict[str, object]] = None
    header_line = 0
    layers: list[LayerSpec] = []
    cur: Optional[TensorShape] = None
    prev = "<input>"
    for lineno, raw in enumerate(text.splitlines(), start=1):
        body = raw.split("#", 1)[0].rstrip()
        toks = [(m.group(0), m.start() + 1) for m in _TOKEN.finditer(body)]
        if not toks:
            continue
        first_col = toks[0][1]
        if header is None:
            if toks[0][0] != "model":
                raise DescriptorError(f"expected 'model' header, got {toks[0][0]!r}", lineno, first_col)
            if len(toks) < 2 or "=" in toks[1][0]:
                raise DescriptorError("model header needs a name", lineno, first_col)
            header = {"name": toks[1][0], **_pairs(toks[2:], lineno)}
            if "batch" not in header:
                raise DescriptorError("model header needs batch=<n>", lineno, first_col)
            if "input" in header:
                cur = _shape(str(header["input"]), lineno, first_col)
            header_line = lineno
            continue
        layers.append(_layer_line(toks, lineno, len(layers) + 1, cur, prev))
        cur = layers[-1].output_shape
        prev = layers[-1].name
    if header is None:
        raise DescriptorError("empty descriptor (no 'model' header)", max(1, len(text.splitlines()) or 1))
    try:
        return ModelGraph(name=str(header["name"]), layers=tuple(layers), batch_size=int(header["batch"]),
                          bytes_per_element=int(header.get("elem_bytes", 4)))
    except ModelError as exc:
        raise DescriptorError(str(exc), header_line) from None


def _layer_line(toks, lineno: int, index: int, cur: Optional[TensorShape], prev: str) -> LayerSpec:
    col = toks[0][1]
    if len(toks) < 2:
        raise DescriptorError("layer line needs <name> <kind> [key=value ...]", lineno, col)
    name, kind_tok = toks[0][0], toks[1][0]
    if "=" in name or "=" in kind_tok:
        raise DescriptorError("layer line needs <name> <kind> before key=value pairs", lineno, col)
    kind = _KINDS.get(kind_tok)
    if kind is None:
        raise DescriptorError(f"unknown layer kind {kind_tok!r} (expected one of {', '.join(sorted(_KINDS))})",
                              lineno, toks[1][1])
    kv = _pairs(toks[2:], lineno)
    shape_override = _shape(str(kv.pop("shape")), lineno, col) if "shape" in kv else None
    is_fc = kind is LayerKind.FULLY_CONNECTED
    try:
        if "params" in kv or ("out" in kv and not is_fc):
            # explicit totals; an fc keeps out= as its width hyperparameter
            params = int(kv.pop("params", 0))
            if "out" not in kv:
                raise DescriptorError(f"explicit layer {name!r} needs out=<elems>", lineno, col)
            out_elems = int(kv["out"]) if is_fc else int(kv.pop("out"))
            flops = int(kv.pop("flops", 0))
            shape = shape_override or TensorShape.flat(out_elems)
        else:
            if kind is LayerKind.BLOCK:
                raise DescriptorError(f"block layer {name!r} needs explicit params= out= flops=", lineno, col)
            if cur is None:
                raise DescriptorError(f"layer {name!r} needs an input shape (set input= in the header "
                                      "or give explicit out=)", lineno, col)
            _check_declared_input(kind, kv, cur, name, prev, lineno, col)
            params, out_elems, flops, shape = infer_layer(kind, kv, cur)
            shape = shape_override or shape
        return LayerSpec(index=index, name=name, kind=kind, param_count=params, output_elems_per_sample=out_elems,
                         compute_flops_per_sample=flops, hyperparams=dict(kv), output_shape=shape)
    except ModelError as exc:
        raise DescriptorError(str(exc), lineno, col) from None


def _check_declared_input(kind, kv, cur: TensorShape, name: str, prev: str, lineno: int, col: int) -> None:
    if kind is LayerKind.CONVOLUTION and "cin" in kv:
        if cur.is_flat or int(kv["cin"]) != cur.c:
            raise ShapeMismatchError(f"layer {name!r} declares cin={kv['cin']} but {prev!r} produces {cur}",
                                     lineno, col)
    if kind is LayerKind.FULLY_CONNECTED and "in" in kv and int(kv["in"]) != cur.elems:
        raise ShapeMismatchError(f"layer {name!r} declares in={kv['in']} but {prev!r} produces "
                                 f"{cur.elems} elements", lineno, col)


def serialize_model(graph: ModelGraph) -> str:
    """Explicit-totals rendering; parse_model(serialize_model(g)) == g (descriptor.py:206-224)."""
    out = [f"model {graph.name} batch={graph.batch_size} elem_bytes={graph.bytes_per_element}"]
    for layer in graph.layers:
        fields = [layer.name, layer.kind.value]
        fields += [f"{k}={layer.hyperparams[k]}" for k in sorted(layer.hyperparams)]
        fields.append(f"params={layer.param_count}")
        if "out" not in layer.hyperparams:
            fields.append(f"out={layer.output_elems_per_sample}")
        fields.append(f"flops={layer.compute_flops_per_sample}")
        if layer.output_shape is not None and not layer.output_shape.is_flat:
            fields.append(f"shape={layer.output_shape}")
        out.append(" ".join(fields))
    return "\n".join(out) + "\n"
