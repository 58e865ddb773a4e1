"""Multi-rank parity (run under torch.distributed.run, one process per GPU).

W ranks execute the layer-placed step (fronts on every rank, FC tail on rank 0,
cut gather / act-grad scatter and the sharded-PS sync over NVLink peer memory);
rank 0 replays the same W-worker step with the CPU oracle and checks loss,
per-step synchronised bytes and the parameters of every rank (all ranks must
hold identical front parameters after the sharded-PS all-gather).
Exit code 0 = pass.  Used by tests/test_multigpu_gpu.py.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from oracle import step as ostep  # noqa: E402
from paper_1901_05803_b200 import synthetic  # noqa: E402
from paper_1901_05803_b200.executor import RankExecutor  # noqa: E402
from paper_1901_05803_b200.planner import (JobSpec, Strategy, catalog_lookup, parse_model,  # noqa: E402
                                           volume_baseline, volume_ralp, volume_ralp_multi_ps, volume_ring)

TINY = """model vgg_tiny batch=8 elem_bytes=4 input=32x32x3
conv1 conv k=3 cout=64 pad=1
conv2 conv k=3 cout=64 pad=1
pool1 pool window=2
conv3 conv k=3 cout=128 pad=1
pool2 pool window=2
conv4 conv k=3 cout=256 pad=1
pool3 pool window=2
fc1 fc out=512
fc2 fc out=512
fc3 fc out=100
"""


def run(model, strategy, steps, rank, world, ring_backend="native", lr=0.01, floor=False):
    """strategy: "ralp", "baseline" (all-on-PS), "ring" (ring all-reduce; numerics are the
    baseline's, bytes are volume_ring's) or "ralp-mps" (layer-placed with the FC tail sharded
    over all ranks; numerics are RALP's, bytes volume_ralp_multi_ps)."""
    fc_sharding = "single"
    if strategy == "ralp-mps":
        strategy, fc_sharding = "ralp", "multi"
    split = next(i for i, l in enumerate(model.layers) if l.kind.value == "fc")
    if strategy == "ralp":
        job = JobSpec(model, Strategy.ralp(split), world)
        expect = (volume_ralp_multi_ps if fc_sharding == "multi" else volume_ralp)(model, split, world)
    elif strategy == "ring":
        job, expect = JobSpec(model, Strategy.ring(), world, ps_count=0), volume_ring(model, world)
    else:
        job, expect = JobSpec(model, Strategy.baseline(), world), volume_baseline(model, world)
    expect = expect.total_bytes_per_step
    ex = RankExecutor(job, rank=rank, world=world, ring_backend=ring_backend, fc_sharding=fc_sharding)
    params = synthetic.init_params(ex.layers, 1)
    ex.set_params(params)
    b = model.batch_size
    orc = ostep.OracleState(ex.layers, params) if rank == 0 else None
    # floor=True: judge parameter deviations against the oracle's own fp32-vs-fp64 spread (as
    # tests/test_step_gpu.py does) instead of a fixed bound -- deep nets amplify rounding
    orc64 = ostep.OracleState(ex.layers, params) if rank == 0 and floor else None
    ok = True
    for t in range(steps):
        imgs, labs = synthetic.batch(1, t, rank * b, b, ex.in_shape, ex.classes)
        ex.step(imgs, labs, lr=lr)
        st = ex.stats()
        if st.logical_bytes != expect:
            print(f"[rank {rank}] bytes {st.logical_bytes} != {expect}", flush=True)
            ok = False
        if rank == 0:
            batches = [synthetic.batch(1, t, r * b, b, ex.in_shape, ex.classes) for r in range(world)]
            lo, wire = ostep.train_step(orc, "baseline" if strategy == "ring" else strategy, world, batches, lr=lr,
                                        emulate_bf16=True)
            if orc64 is not None:
                ostep.train_step(orc64, strategy, world, batches, lr=lr, emulate_bf16=True, accum64=True)
            assert strategy == "ring" or fc_sharding == "multi" or wire == expect
            rel = abs(st.loss - lo) / abs(lo)
            tol = 2e-3 if strategy == "ralp" else 0.5  # baseline/ring: rank 0 reports its own batch's loss only
            tag = f"{strategy}-{ring_backend}" if strategy == "ring" else strategy + ("-mps" if fc_sharding == "multi" else "")
            print(f"[{model.name} {tag} W={world}] step {t}: loss gpu {st.loss:.6f} oracle {lo:.6f} "
                  f"rel {rel:.2e} ms {st.ms_step:.2f} phys {st.physical_bytes}", flush=True)
            if rel > tol:
                ok = False
    got = ex.get_params()
    ex.close()
    # every rank holds the same front (and, for the baseline, all) parameters
    for li, p in enumerate(got):
        if p is None:
            continue
        if strategy == "ralp" and li >= split:
            continue   # FC tail: on the PS (single) or sliced over the ranks (multi)
        t = torch.from_numpy(np.ascontiguousarray(p[0])).cuda()
        ref = t.clone()
        dist.broadcast(ref, 0)
        if not torch.equal(t, ref):
            print(f"[rank {rank}] layer {li} differs from rank 0 after the all-gather", flush=True)
            ok = False
    if rank == 0:
        w64s = orc64.numpy_params() if orc64 is not None else [None] * len(got)
        for li, (g, w, w64, p0) in enumerate(zip(got, orc.numpy_params(), w64s, params)):
            if g is None:
                continue
            upd = np.linalg.norm(w[0] - p0[0])
            dev = np.linalg.norm(g[0] - w[0]) / upd
            if w64 is None:
                bound = 0.25
            else:
                bound = 4 * np.linalg.norm(w64[0] - w[0]) / upd + 0.02
            print(f"   layer {li}: dev {dev:.3e} (bound {bound:.3e})", flush=True)
            if dev > bound:
                ok = False
    return ok


def main():
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    torch.cuda.set_device(int(os.environ["LOCAL_RANK"]))
    dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ["LOCAL_RANK"])))
    ok = True
    cifar = catalog_lookup("cifar_small").with_batch_size(32)
    for model, strategy, steps, backend, lr, *fl in [(cifar, "ralp", 4, "native", 0.01), (parse_model(TINY), "ralp", 3, "native", 0.01),
                                            (cifar, "baseline", 3, "native", 0.01), (cifar, "ring", 3, "native", 0.01),
                                            (cifar, "ring", 3, "nccl", 0.01), (cifar, "ralp-mps", 4, "native", 0.01),
                                            (parse_model(TINY), "ralp-mps", 3, "native", 0.01),
                                            # full VGG-16 geometry (224x224: first-conv, row-streamed
                                            # 64-channel, slab pair kernels, pool5 cut) at b=4 per rank
                                            (catalog_lookup("vgg16").with_batch_size(4), "ralp", 2, "native", 1e-3, True)]:
        ok &= run(model, strategy, steps, rank, world, backend, lr, floor=bool(fl and fl[0]))
    flag = torch.tensor([0 if ok else 1], device="cuda")
    dist.all_reduce(flag)
    dist.destroy_process_group()
    if rank == 0:
        print("MULTI-RANK PARITY", "PASS" if flag.item() == 0 else "FAIL", flush=True)
    sys.exit(0 if flag.item() == 0 else 1)


if __name__ == "__main__":
    main()
