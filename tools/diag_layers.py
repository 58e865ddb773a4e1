"""Per-layer exactness of the conv kernels: GPU bf16 output vs the fp64 reference of the
same bf16 inputs, rounded to bf16.  Reports the fraction of elements that differ and the
max difference in bf16 ulps, for the GPU and for torch-CPU fp32 (the oracle's arithmetic)."""
import sys
from pathlib import Path

import torch
import torch.nn.functional as F

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_05803_b200 import ops  # noqa: E402


def ulps(a, b):
    a = a.to(torch.bfloat16).view(torch.int16).to(torch.int32)
    b = b.to(torch.bfloat16).view(torch.int16).to(torch.int32)
    return (a - b).abs()


def check(n, h, cin, cout):
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.relu(torch.randn(n, h, h, cin, generator=g, device="cuda")).to(torch.bfloat16)
    xp = F.pad(x, (0, 0, 1, 1, 1, 1)).contiguous()
    w = (torch.randn(cout, 9, cin, generator=g, device="cuda") * (2 / (9 * cin)) ** 0.5).to(torch.bfloat16)
    b = torch.randn(cout, device="cuda") * 0.1
    y = ops.conv_fwd(xp, w, b, n=n, h=h, w_=h, cin=cin, cout=cout, k=3, pad=1, relu=False)[:, 1:-1, 1:-1, :]
    xr = x.permute(0, 3, 1, 2)
    wr = w.view(cout, 3, 3, cin).permute(0, 3, 1, 2)
    ref64 = F.conv2d(xr.double().cpu(), wr.double().cpu(), b.double().cpu(), padding=1).permute(0, 2, 3, 1)
    ref32 = F.conv2d(xr.float().cpu(), wr.float().cpu(), b.float().cpu(), padding=1).permute(0, 2, 3, 1)
    u_gpu = ulps(y.cpu().float(), ref64.float())
    u_cpu = ulps(ref32, ref64.float())
    rel_gpu = ((y.cpu().double() - ref64).abs() / ref64.abs().clamp_min(1e-3)).max().item()
    print(f"n={n} h={h} cin={cin} cout={cout}: GPU differs {u_gpu.ne(0).float().mean().item():.2e} "
          f"(max {u_gpu.max().item()} ulp, max rel {rel_gpu:.2e}) | CPU fp32 differs "
          f"{u_cpu.ne(0).float().mean().item():.2e} (max {u_cpu.max().item()} ulp)", flush=True)


for args in [(4, 56, 64, 64), (4, 28, 256, 256), (4, 14, 512, 512), (2, 56, 128, 256)]:
    check(*args)

# GEMM accumulation accuracy: long K
g = torch.Generator(device="cuda").manual_seed(1)
for K in (64, 512, 4096, 25088):
    a = torch.randn(256, K, generator=g, device="cuda").to(torch.bfloat16)
    bb = torch.randn(256, K, generator=g, device="cuda").to(torch.bfloat16)
    out = ops.gemm(a, bb, out_kind="f32")
    ref = (a.double() @ bb.double().t())
    r32 = (a.float().cpu() @ bb.float().cpu().t()).double()
    e_gpu = ((out.double() - ref).abs() / ref.abs().mean()).max().item()
    e_cpu = ((r32 - ref.cpu()).abs() / ref.abs().mean().cpu()).max().item()
    print(f"GEMM K={K}: max err/mean|ref| GPU {e_gpu:.2e}  CPU fp32 {e_cpu:.2e}", flush=True)
