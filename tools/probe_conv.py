"""Time the implicit-GEMM conv kernels at VGG-16 b=128 layer shapes (CUDA events)."""
import sys
import torch
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_05803_b200 import ops

N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
LAYERS = [  # h, cin, cout
    (224, 16, 64), (224, 64, 64), (112, 64, 128), (112, 128, 128), (56, 128, 256), (56, 256, 256),
    (28, 256, 512), (28, 512, 512), (14, 512, 512)]


def timeit(fn, iters=5):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


tot = {"fwd": 0, "dgrad": 0, "wgrad": 0}
for h, cin, cout in LAYERS:
    x = torch.randn(N, h + 2, h + 2, cin, device="cuda").to(torch.bfloat16)
    dy = torch.randn(N, h + 2, h + 2, cout, device="cuda").to(torch.bfloat16)
    w = torch.randn(cout, 9, cin, device="cuda").to(torch.bfloat16)
    wd = torch.randn(cin, 9, cout, device="cuda").to(torch.bfloat16)
    b = torch.zeros(cout, device="cuda")
    y = torch.empty_like(dy)
    dx = torch.empty_like(x)
    dw = torch.zeros(cout, 9, cin, device="cuda")
    flops = 2 * 9 * cin * cout * h * h * N
    t_f = timeit(lambda: ops.conv_fwd(x, w, b, n=N, h=h, w_=h, cin=cin, cout=cout, k=3, pad=1, out=y))
    t_d = timeit(lambda: ops.conv_dgrad(dy, wd, x, n=N, h=h, w_=h, cin=cin, cout=cout, k=3, pad=1, out=dx))
    t_w = timeit(lambda: ops.conv_wgrad(x, dy, n=N, h=h, w_=h, cin=cin, cout=cout, k=3, pad=1, out=dw))
    print(f"h={h:3d} cin={cin:3d} cout={cout:3d}  fwd {t_f:7.3f} ms {flops/t_f/1e9:7.1f} TF/s | "
          f"dgrad {t_d:7.3f} ms {flops/t_d/1e9:7.1f} TF/s | wgrad {t_w:7.3f} ms {flops/t_w/1e9:7.1f} TF/s", flush=True)
    tot["fwd"] += t_f; tot["dgrad"] += t_d; tot["wgrad"] += t_w
    del x, dy, w, wd, y, dx, dw
    torch.cuda.empty_cache()
print(tot)
