"""Compare the executor's per-layer forward activations with the oracle's (one step, W=1)."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from oracle import step as ostep
from paper_1901_05803_b200 import _lib, synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, parse_model

name, b = sys.argv[1], int(sys.argv[2])
m = catalog_lookup(name).with_batch_size(b)
ex = RankExecutor(JobSpec(m, Strategy.baseline(), 1))
params = synthetic.init_params(ex.layers, 0)
ex.set_params(params)
imgs, labs = synthetic.batch(0, 0, 0, b, ex.in_shape, ex.classes)
ex.step(imgs, labs)
ex.stats()
orc = ostep.OracleState(ex.layers, params)
nfront = next(i for i, L in enumerate(ex.layers) if L["kind"] == "fc")
acts, cut = ostep._front_forward(orc, nfront, imgs, True)
for i in range(1, nfront + 1):
    n = _lib.lib().ralpb_model_debug_buffer(ex._h, i, 0, None)
    buf = np.empty(n, dtype=np.uint16)
    _lib.lib().ralpb_model_debug_buffer(ex._h, i, 0, buf.ctypes.data)
    got = torch.from_numpy(buf.view(np.int16)).view(torch.bfloat16).float()
    ref = acts[i].permute(0, 2, 3, 1)  # n h w c
    hh, ww, cc = ref.shape[1:]
    tot = got.numel() // (b * cc)
    side = int(round(tot ** 0.5))
    pad = (side - hh) // 2
    got = got.view(b, side, side, cc)[:, pad:pad + hh, pad:pad + ww, :] if i < nfront else got.view(b, hh, ww, cc)
    err = (got - ref).abs().max().item()
    rel = ((got - ref).norm() / ref.norm()).item()
    print(f"act {i} ({ex.layers[i-1]['name']}): max|err| {err:.3e} rel {rel:.3e} |ref| {ref.abs().max().item():.3e}", flush=True)
