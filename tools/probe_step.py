"""Time the native VGG-16 step at b=128 on one GPU (CUDA events inside the library)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
from paper_1901_05803_b200 import synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, profile

name = sys.argv[1] if len(sys.argv) > 1 else "vgg16"
b = int(sys.argv[2]) if len(sys.argv) > 2 else 128
strategy = sys.argv[3] if len(sys.argv) > 3 else "ralp"
m = catalog_lookup(name).with_batch_size(b)
split = profile(m).split_index
job = JobSpec(m, Strategy.ralp(split) if strategy == "ralp" else Strategy.baseline(), 1)
ex = RankExecutor(job)
ex.set_params(synthetic.init_params(ex.layers, 0))
rng = np.random.default_rng(0)
imgs = rng.standard_normal((b, *ex.in_shape), dtype=np.float32)
labs = rng.integers(0, ex.classes, b).astype(np.int32)
import torch
dimgs = torch.from_numpy(imgs).cuda()
dlabs = torch.from_numpy(labs).cuda()
for t in range(8):
    ex.step(dimgs, dlabs)
    st = ex.stats()
    print(f"step {t}: loss {st.loss:.4f} ms {st.ms_step:.2f} (fwd {st.ms_front_fwd:.2f} back {st.ms_back:.2f} "
          f"bwd {st.ms_front_bwd:.2f} sync {st.ms_sync:.2f}) launches {st.launches} bytes {st.logical_bytes} "
          f"img/s {b / st.ms_step * 1e3:.0f}", flush=True)
