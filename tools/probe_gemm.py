"""Micro-benchmarks of the GEMM engine: operand majorness / split-K / shapes (CUDA events)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1901_05803_b200 import ops  # noqa: E402


def timeit(fn, iters=3):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def run(tag, M, N, K, a_mn, b_mn, kind, splits, bn=0):
    a = (torch.randn(K, M, device="cuda") if a_mn else torch.randn(M, K, device="cuda")).to(torch.bfloat16)
    b = (torch.randn(K, N, device="cuda") if b_mn else torch.randn(N, K, device="cuda")).to(torch.bfloat16)
    out = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16 if kind == "bf16" else torch.float32)
    ms = timeit(lambda: ops.gemm(a, b, a_mn=a_mn, b_mn=b_mn, out=out, out_kind=kind, k_splits=splits, block_n=bn))
    print(f"{tag:40s} M={M:8d} N={N:5d} K={K:8d} {ms:8.3f} ms {2 * M * N * K / ms / 1e9:7.1f} TF/s", flush=True)
    del a, b, out
    torch.cuda.empty_cache()


K = 128 * 226 * 226
run("wgrad-like MNxMN atomic split60", 576, 64, K, True, True, "f32_atomic", 60)
run("wgrad-like MNxMN atomic split0", 576, 64, K, True, True, "f32_atomic", 0)
run("wgrad-like KxK atomic split60", 576, 64, K, False, False, "f32_atomic", 60)
run("wgrad-like MNxK atomic split60", 576, 64, K, True, False, "f32_atomic", 60)
run("wgrad-like KxMN atomic split60", 576, 64, K, False, True, "f32_atomic", 60)
run("big MNxMN atomic", 4608, 512, 128 * 30 * 30, True, True, "f32_atomic", 0)
run("big KxK atomic", 4608, 512, 128 * 30 * 30, False, False, "f32_atomic", 0)
run("square KxK bf16", 8192, 8192, 8192, False, False, "bf16", 1)
run("square KxMN bf16", 8192, 8192, 8192, False, True, "bf16", 1)
run("square MNxMN f32", 8192, 8192, 8192, True, True, "f32", 1)
run("fwd-like KxK bf16 N=64", K, 64, 576, False, False, "bf16", 1)
run("fwd-like KxK bf16 N=256", 128 * 58 * 58, 256, 2304, False, False, "bf16", 1)
