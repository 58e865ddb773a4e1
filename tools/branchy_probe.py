"""GPU probe: Inception-v3 / GoogLeNet / OverFeat / LeNet through the executor (b=8, two steps)
against the oracle's first-step loss, plus a b=128 timing of the partitioner's split."""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np
import torch
from oracle import step as ostep
from paper_1901_05803_b200 import synthetic
from paper_1901_05803_b200.executor import RankExecutor
from paper_1901_05803_b200.planner import JobSpec, Strategy, catalog_lookup, profile, volume_ralp

names = sys.argv[1:] or ["inception-v3", "googlenet", "overfeat", "lenet"]
for name in names:
    m = catalog_lookup(name).with_batch_size(8)
    rep = profile(m)
    split = rep.split_index or m.num_layers - 1
    job = JobSpec(m, Strategy.ralp(split), 1)
    try:
        ex = RankExecutor(job)
    except Exception as e:
        print(name, "CREATE FAILED", e, flush=True)
        continue
    params = synthetic.init_params(ex.layers, 0)
    ex.set_params(params)
    o = ostep.OracleState(ex.layers, params)
    for t in range(2):
        imgs, labs = synthetic.batch(0, t, 0, 8, ex.in_shape, ex.classes)
        try:
            ex.step(imgs, labs, lr=1e-3, momentum=0.9)
            st = ex.stats()
        except Exception as e:
            print(name, "STEP FAILED", e, flush=True)
            break
        lsplit = None
        lo, wire = ostep.train_step(o, "ralp", 1, [(imgs, labs)], lr=1e-3, emulate_bf16=True,
                                    split=ex.lowered_split)
        print(f"{name} split {split} step {t}: loss gpu {st.loss:.6f} oracle {lo:.6f} rel {abs(st.loss-lo)/lo:.2e} "
              f"bytes {st.logical_bytes} oracle {wire} catalog {volume_ralp(m, split, 1).total_bytes_per_step} "
              f"ms {st.ms_step:.2f} launches {st.launches}", flush=True)
    ex.close()
    # b=128 timing
    m = catalog_lookup(name).with_batch_size(128)
    split = profile(m).split_index or m.num_layers - 1
    try:
        ex = RankExecutor(JobSpec(m, Strategy.ralp(split), 1))
        ex.set_params(synthetic.init_params(ex.layers, 0))
        x = torch.randn(128, *ex.in_shape, device="cuda")
        y = torch.randint(0, ex.classes, (128,), device="cuda", dtype=torch.int32)
        for _ in range(3):
            ex.step(x, y)
        torch.cuda.synchronize()
        t0 = time.time()
        for _ in range(5):
            ex.step(x, y)
        torch.cuda.synchronize()
        dt = (time.time() - t0) / 5
        st = ex.stats()
        print(f"{name} b=128 split {split}: {dt*1e3:.2f} ms/step wall, {128/dt:.0f} img/s, device {st.ms_step:.2f} ms, "
              f"fwd {st.ms_front_fwd:.2f} back {st.ms_back:.2f} bwd {st.ms_front_bwd:.2f}", flush=True)
        ex.close()
    except Exception as e:
        print(name, "b=128 FAILED", e, flush=True)
