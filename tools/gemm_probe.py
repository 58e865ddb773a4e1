"""Per-launch tensor-core times of one profiled b=128 step of a catalog model (partitioner split), in
launch order, with the algorithmic rate of each and the time above its roofline:
python tools/gemm_probe.py <model> [top]."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1901_05803_b200 import synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, profile

PEAK_TF, PEAK_GBS = 1394.0, 7000.0
name = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
m = catalog_lookup(name).with_batch_size(128)
ex = RankExecutor(JobSpec(m, Strategy.ralp(profile(m).split_index), 1))
ex.set_params(synthetic.init_params(ex.layers, 0))
x = torch.randn(128, *ex.in_shape, device="cuda")
y = torch.randint(0, ex.classes, (128,), device="cuda", dtype=torch.int32)
for _ in range(3):
    ex.step(x, y)
ex.set_profiling(True)
ex.step(x, y)
recs = ex.timed_launches()
rows = []
for i, (kind, ms, flops, by) in enumerate(recs):
    if ms <= 0:
        continue
    roof = max(flops / (PEAK_TF * 1e9), by / (PEAK_GBS * 1e6))
    rows.append((ms - roof, i, kind, ms, flops / ms / 1e9, by / ms / 1e6))
tot = sum(r[3] for r in rows)
lost = sum(r[0] for r in rows)
print(f"{name}: {len(rows)} timed launches, {tot:.3f} ms, {lost:.3f} ms above roofline")
for r in sorted(rows, reverse=True)[:top]:
    print(f"  #{r[1]:4d} {r[2]:12s} {r[3] * 1e3:8.1f} us  {r[4]:7.1f} TF/s  {r[5]:7.0f} GB/s  lost {r[0] * 1e3:7.1f} us")
