"""Run a few VGG-16 b=128 layer-placed steps (for an ncu launch list)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1901_05803_b200 import synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, profile

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
m = catalog_lookup("vgg16").with_batch_size(128)
ex = RankExecutor(JobSpec(m, Strategy.ralp(profile(m).split_index), 1))
ex.set_params(synthetic.init_params(ex.layers, 0))
x = torch.randn(128, 224, 224, 3, device="cuda")
y = torch.randint(0, 1000, (128,), device="cuda", dtype=torch.int32)
for _ in range(steps):
    ex.step(x, y)
st = ex.stats()
print("launches/step", st.launches, "ms", st.ms_step)
