"""Run a few b=128 layer-placed steps of a catalog model (partitioner split) on one GPU, for an ncu
launch list: python tools/model_launches.py <model> [steps]."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1901_05803_b200 import synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, profile

name = sys.argv[1]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m = catalog_lookup(name).with_batch_size(128)
ex = RankExecutor(JobSpec(m, Strategy.ralp(profile(m).split_index), 1))
ex.set_params(synthetic.init_params(ex.layers, 0))
x = torch.randn(128, *ex.in_shape, device="cuda")
y = torch.randint(0, ex.classes, (128,), device="cuda", dtype=torch.int32)
for _ in range(steps):
    ex.step(x, y)
st = ex.stats()
print(name, "launches/step", st.launches, "ms", st.ms_step, "fwd", st.ms_front_fwd, "back", st.ms_back, "bwd",
      st.ms_front_bwd, "sync", st.ms_sync)
