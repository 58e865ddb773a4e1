"""Time the implicit-GEMM conv kernels at VGG-16 b=128 layer shapes (CUDA events).

    python tools/probe_conv.py [--n 128] [--layer I] [--op fwd|dgrad|wgrad|all] [--iters 5]
"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_05803_b200 import ops  # noqa: E402

LAYERS = [  # h, cin, cout (distinct VGG-16 conv shapes; conv1 with cin padded to 16)
    (224, 16, 64), (224, 64, 64), (112, 64, 128), (112, 128, 128), (56, 128, 256), (56, 256, 256),
    (28, 256, 512), (28, 512, 512), (14, 512, 512)]
REPEATS = [1, 1, 1, 1, 1, 2, 1, 2, 3]  # occurrences in VGG-16


def timeit(fn, iters):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--layer", type=int, default=-1)
    ap.add_argument("--op", default="all")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--shape", default="", help="h,cin,cout: one extra shape instead of VGG-16's")
    a = ap.parse_args()
    global LAYERS, REPEATS
    if a.shape:
        LAYERS = [tuple(int(v) for v in a.shape.split(","))]
        REPEATS = [1]
    N = a.n
    tot = {"fwd": 0.0, "dgrad": 0.0, "wgrad": 0.0}
    for li, (h, cin, cout) in enumerate(LAYERS):
        if a.layer >= 0 and li != a.layer:
            continue
        x = torch.randn(N, h + 2, h + 2, cin, device="cuda").to(torch.bfloat16)
        dy = torch.randn(N, h + 2, h + 2, cout, device="cuda").to(torch.bfloat16)
        w = torch.randn(cout, 9, cin, device="cuda").to(torch.bfloat16)
        wd = torch.randn(cin, 9, cout, device="cuda").to(torch.bfloat16)
        b = torch.zeros(cout, device="cuda")
        y = torch.empty_like(dy)
        dx = torch.empty_like(x)
        dw = torch.zeros(cout, 9, cin, device="cuda")
        flops = 2 * 9 * cin * cout * h * h * N
        res = {}
        if a.op in ("all", "fwd"):
            res["fwd"] = timeit(lambda: ops.conv_fwd(x, w, b, n=N, h=h, w_=h, cin=cin, cout=cout, k=3, pad=1, out=y), a.iters)
        if a.op in ("all", "dgrad") and (li > 0 or a.shape):
            res["dgrad"] = timeit(lambda: ops.conv_dgrad(dy, wd, x, n=N, h=h, w_=h, cin=cin, cout=cout, k=3, pad=1, out=dx), a.iters)
        if a.op in ("all", "wgrad"):
            res["wgrad"] = timeit(lambda: ops.conv_wgrad(x, dy, n=N, h=h, w_=h, cin=cin, cout=cout, k=3, pad=1, out=dw), a.iters)
        msg = " | ".join(f"{k} {v:7.3f} ms {flops / v / 1e9:7.1f} TF/s" for k, v in res.items())
        print(f"h={h:3d} cin={cin:3d} cout={cout:3d} x{REPEATS[li]}  {msg}", flush=True)
        for k, v in res.items():
            tot[k] += v * REPEATS[li]
        del x, dy, w, wd, y, dx, dw
        torch.cuda.empty_cache()
    print("VGG-16 totals (ms):", {k: round(v, 3) for k, v in tot.items()}, flush=True)


if __name__ == "__main__":
    main()
