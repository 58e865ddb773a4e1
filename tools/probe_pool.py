"""Time the max-pool backward at the VGG-16 b=128 pool shapes (CUDA events)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_05803_b200 import ops  # noqa: E402

n = 128
tot = 0.0
for h, c in [(224, 64), (112, 128), (56, 256), (28, 512), (14, 512)]:
    x = torch.relu(torch.randn(n, h + 2, h + 2, c, device="cuda")).to(torch.bfloat16)
    dy = torch.randn(n, h // 2 + 2, h // 2 + 2, c, device="cuda").to(torch.bfloat16)
    cs = torch.zeros(c, device="cuda")
    dx = torch.zeros_like(x)
    f = lambda: ops.call("ralpb_maxpool_bwd", x.data_ptr(), dy.data_ptr(), n, h, h, c, 1, 2, 2, 1, dx.data_ptr(),
                         cs.data_ptr(), ops._stream())
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        f()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    gb = (9 * n * (h // 2) ** 2 * c * 2) / 1e9
    tot += ms
    print(f"pool bwd {h}x{h}x{c}: {ms * 1e3:7.1f} us  {gb / ms:6.2f} TB/s")
print(f"total {tot * 1e3:.1f} us")
