"""Cost of the fused 2x2 pool in the conv epilogue: conv fwd with and without it at the
VGG-16 b=128 pool-preceding shapes (CUDA events)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_05803_b200 import ops  # noqa: E402


def timeit(fn, iters=10):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


n = 128
for h, c in [(224, 64), (112, 128), (56, 256), (28, 512), (14, 512)]:
    x = torch.randn(n, h + 2, h + 2, c, device="cuda").to(torch.bfloat16)
    w = (torch.randn(c, 9, c, device="cuda") * 0.05).to(torch.bfloat16)
    b = torch.zeros(c, device="cuda")
    y = torch.zeros(n, h + 2, h + 2, c, device="cuda", dtype=torch.bfloat16)
    t0 = timeit(lambda: ops.conv_fwd(x, w, b, n=n, h=h, w_=h, cin=c, cout=c, k=3, pad=1, out=y))
    pooled = torch.zeros(n, h // 2 + 2, h // 2 + 2, c, device="cuda", dtype=torch.bfloat16)
    t1 = timeit(lambda: ops.call("ralpb_conv_fwd_pool", x.data_ptr(), w.data_ptr(), b.data_ptr(), y.data_ptr(),
                                 pooled.data_ptr(), 1, 0, n, h, h, c, c, 3, 1, 1, ops._stream()))
    print(f"{h:4d}x{h:<4d} c={c:4d}: conv {t0 * 1e3:7.1f} us, conv+pool {t1 * 1e3:7.1f} us (+{(t1 / t0 - 1) * 100:5.1f} %)")
    del x, w, y
    torch.cuda.empty_cache()
