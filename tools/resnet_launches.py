"""Run a few ResNet-50 b=128 layer-placed steps (split 55) on one GPU, for an ncu launch list and
per-category timing."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1901_05803_b200 import synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
b = int(sys.argv[2]) if len(sys.argv) > 2 else 128
m = catalog_lookup("resnet-50").with_batch_size(b)
ex = RankExecutor(JobSpec(m, Strategy.ralp(55), 1))
ex.set_params(synthetic.init_params(ex.layers, 0))
x = torch.randn(b, 224, 224, 3, device="cuda")
y = torch.randint(0, 1000, (b,), device="cuda", dtype=torch.int32)
for _ in range(steps):
    ex.step(x, y)
st = ex.stats()
print("launches/step", st.launches, "ms", st.ms_step, "fwd", st.ms_front_fwd, "back", st.ms_back, "bwd", st.ms_front_bwd,
      "sync", st.ms_sync)
