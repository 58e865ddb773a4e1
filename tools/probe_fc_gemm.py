"""The PS's FC-tail GEMM shapes at W*b = 512 / 1024 rows (fc1 forward, K-major x K-major, and
backward-data, MN-major filters) under several split-K settings; split 0 = the engine's choice."""
import sys
sys.path.insert(0, "tools")
from probe_gemm import run
for M in (512, 1024):
    for sp in (0, 1, 2, 4):
        run(f"fc1 fwd split{sp}", M, 4096, 25088, False, False, "f32_atomic", sp)
    for sp in (0, 1, 2):
        run(f"fc1 dgrad split{sp}", M, 25088, 4096, False, True, "f32_atomic", sp)
    run("fc1 dgrad bf16 nosplit", M, 25088, 4096, False, True, "bf16", 1)
