"""Time the fused first-conv kernels (conv_first.cu) at VGG-16 b=128 224x224 (CUDA events)."""
import sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_05803_b200 import ops  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
x = torch.randn(n, 224, 224, 3, device="cuda")
wf = (torch.randn(64, 32, device="cuda") * 0.1).to(torch.bfloat16)
dy = torch.randn(n, 226, 226, 64, device="cuda").to(torch.bfloat16)
y = torch.zeros(n, 226, 226, 64, device="cuda", dtype=torch.bfloat16)
dw = torch.zeros(64, 32, device="cuda")
for name, fn in [("fwd", lambda: ops.call("ralpb_conv_first_fwd", x.data_ptr(), n, 224, 224, wf.data_ptr(),
                                          y.data_ptr(), 1, ops._stream())),
                 ("wgrad", lambda: ops.conv_first_wgrad(x, dy, pad_out=1, dw=dw))]:
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    gb = (n * 224 * 224 * 3 * 4 + n * 224 * 224 * 64 * 2) / 1e9
    print(f"first conv {name}: {ms:.3f} ms, {gb / ms:.2f} TB/s algorithmic")
