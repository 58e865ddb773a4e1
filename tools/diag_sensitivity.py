"""Intrinsic sensitivity of the bf16 pipeline: oracle(fp32 accumulation) vs oracle(fp64
accumulation), both with bf16 rounding points, after N steps (CPU only)."""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import step as ostep
from paper_1901_05803_b200 import synthetic
from paper_1901_05803_b200.executor import lower
from paper_1901_05803_b200.planner import catalog_lookup

name, b, steps, strategy = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
m = catalog_lookup(name).with_batch_size(b)
layers = lower(m)
p0 = synthetic.init_params(layers, 0)
runs = {}
for tag, bf, a64 in [("bf16/fp32acc", True, False), ("bf16/fp64acc", True, True), ("fp32", False, False)]:
    st = ostep.OracleState(layers, p0)
    losses = []
    for t in range(steps):
        imgs, labs = synthetic.batch(0, t, 0, b, (layers[0]["h"], layers[0]["w"], layers[0]["cin"]), layers[-1]["cout"])
        losses.append(ostep.train_step(st, strategy, 1, [(imgs, labs)], emulate_bf16=bf, accum64=a64)[0])
    runs[tag] = (losses, st.numpy_params())
ref_l, ref_p = runs["bf16/fp32acc"]
for tag in ("bf16/fp64acc", "fp32"):
    l, p = runs[tag]
    print(tag, "loss rel", [f"{abs(a - b_) / abs(b_):.1e}" for a, b_ in zip(l, ref_l)])
    for i, (g, w, z) in enumerate(zip(p, ref_p, p0)):
        if g is None:
            continue
        for nm, a, b_, c in zip("wb", g, w, z):
            print(f"   {tag} layer {i}.{nm}: max|d| / max|upd| {np.abs(a - b_).max() / np.abs(b_ - c).max():.3e}  "
                  f"||d||/||upd|| {np.linalg.norm(a - b_) / np.linalg.norm(b_ - c):.3e}")
