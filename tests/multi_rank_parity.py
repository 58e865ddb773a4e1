"""Multi-rank parity (run under torch.distributed.run, one process per GPU).

W ranks execute a step placement through the C ABI; rank 0 replays the same W-worker step with
the CPU oracle.  Per configuration and step:

  bytes     the logical bytes every rank counted at its count_wire sites sum to the oracle's
            volume exactly (the NVLink bytes each rank moved are printed per direction)
  exchange  bit-exact: the PS's FC input rows of worker w == worker w's own cut, and worker w's
            received act-grad == the PS's gradient rows of worker w (RALP)
  sync      exact: after step 1 (momentum 0) every rank's front parameters == p0 - lr * sum_r g_r
            of the per-rank gradients the ranks computed (all-on-PS / ring: every parameter), and
            every rank holds identical front parameters after every step
  loss      the job's mean loss (reported on the PS rank for every strategy) within 2e-3 of the
            oracle's at every step
  params    after the last step, per layer ||p_gpu - p_oracle|| / ||p_oracle - p0|| within
            min(2 * floor + 0.02, cap), floor = the bf16 pipeline's own fp32-vs-fp64 spread (the
            oracle re-run with float64 accumulation; configurations marked floor=True), else the
            cap 0.25 (small nets, few steps) / 0.5 (VGG-16, whose bf16 drift is chaotic -- its
            per-layer parity is pinned by the teacher-forced single-GPU test and by the fp32 parity
            precision below); a wrong update is ~1
  fp32      precision="fp32" (the parity mode) against the plain fp32 oracle: loss within 1e-4
            relative at every step (+ 3x the oracle's own fp32-vs-fp64 spread) and per weight tensor
            ||p_gpu - p_oracle|| / ||p_oracle|| <= 1e-4, or within 3 * floor + 2e-2 of the update
            (the rule of tests/test_parity_fp32_gpu.py)

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
from paper_1901_05803_b200 import _lib, synthetic  # noqa: E402
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


def _dev() -> torch.device:
    return torch.device("cuda") if dist.get_backend() == "nccl" else torch.device("cpu")


def _gather(t: torch.Tensor, world: int) -> list[torch.Tensor]:
    t = t.contiguous().to(_dev())
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    return [p.cpu() for p in parts]


def _sum_over_ranks(v: float) -> float:
    t = torch.tensor([float(v)], dtype=torch.float64, device=_dev())
    dist.all_reduce(t)
    return t.item()


def _front_param_vec(params, split) -> torch.Tensor:
    return torch.cat([torch.from_numpy(np.ascontiguousarray(x)).reshape(-1) for p in params[:split] if p is not None
                      for x in p])


def run(model, strategy, steps, rank, world, ring_backend="native", lr=0.01, floor=False, cap=0.25,
        placement="colocated", precision="bf16", split=None, loss_tol=2e-3, loss_steps=None):
    """strategy: "ralp", "baseline" (all-on-PS), "ring" (ring all-reduce; numerics are the
    baseline's, bytes are volume_ring's) or "ralp-mps" (layer-placed with the FC tail sharded
    over all ranks; numerics are RALP's, bytes volume_ralp_multi_ps).  placement="dedicated-ps":
    RALP-N, rank 0 runs only the FC tail and ranks 1..world-1 are the workers."""
    fc_sharding, shard_layout = "single", "bytes"
    if strategy == "ralp-mps":
        strategy, fc_sharding = "ralp", "multi"
    if strategy == "baseline-layers":   # the reference's whole-layer round-robin PS shards
        strategy, shard_layout = "baseline", "layers"
    workers = world - 1 if placement == "dedicated-ps" else world
    fc_at = next(i for i, l in enumerate(model.layers) if l.kind.value == "fc")
    split = fc_at if split is None else split   # < fc_at: a conv back segment on the PS
    if strategy == "ralp":
        job = JobSpec(model, Strategy.ralp(split), workers)
        expect = (volume_ralp_multi_ps if fc_sharding == "multi" else volume_ralp)(model, split, workers)
    elif strategy == "ring":
        job, expect = JobSpec(model, Strategy.ring(), workers, ps_count=0), volume_ring(model, workers)
    else:
        job, expect = JobSpec(model, Strategy.baseline(), workers), volume_baseline(model, workers)
    expect = expect.total_bytes_per_step
    ex = RankExecutor(job, rank=rank, world=world, ring_backend=ring_backend, fc_sharding=fc_sharding,
                      placement=placement, precision=precision, shard_layout=shard_layout)
    params = synthetic.init_params(ex.layers, 1)
    ex.set_params(params)
    b = model.batch_size
    fp32 = precision == "fp32"
    orc = ostep.OracleState(ex.layers, params) if rank == 0 else None
    # floor: the oracle re-run with float64 contractions (the bf16 pipeline's chaos; for the fp32
    # precision the plain fp32 oracle's own sensitivity)
    orc64 = ostep.OracleState(ex.layers, params) if rank == 0 and (floor or fp32) else None
    tag = (f"{strategy}-{ring_backend}" if strategy == "ring" else strategy + ("-mps" if fc_sharding == "multi" else "")
           ) + ("-dedicated-ps" if placement == "dedicated-ps" else "") + ("-fp32" if fp32 else "") + (
        "-layer-shards" if shard_layout == "layers" else "")
    ok = True
    sync_all = strategy != "ralp"   # all-on-PS / ring synchronise every parameter
    nsync = len(params) if sync_all else ex.lowered_split   # lowered layers (branch groups: != catalog split)
    for t in range(steps):
        if ex.is_worker:
            imgs, labs = synthetic.batch(1, t, ex.worker_index * b, b, ex.in_shape, ex.classes)
            ex.step(imgs, labs, lr=lr)
        else:
            ex.step(None, None, lr=lr)
        st = ex.stats()
        total = _sum_over_ranks(st.logical_bytes)
        if int(total) != expect:
            print(f"[{tag} rank {rank}] logical bytes summed over ranks {int(total)} != {expect}", flush=True)
            ok = False
        # ---- exchange: bit-exact cut rows / act-grad rows (layer-placed, single PS)
        if strategy == "ralp" and fc_sharding == "single" and not fp32:
            ps = ex.ps_rank
            cut_local = torch.from_numpy(ex.debug_buffer(_lib.DBG_ACT, ex.lowered_split)) if (ex.is_worker and rank != ps) else None
            dcut = torch.from_numpy(ex.debug_buffer(_lib.DBG_CUT_GRAD)) if (ex.is_worker and rank != ps) else None
            n_cut = ex.debug_buffer(_lib.DBG_CUT_GRAD).size   # (the arena's act-grad slot exists on every rank)
            mine_cut = cut_local if cut_local is not None else torch.zeros(n_cut)
            mine_dcut = dcut if dcut is not None else torch.zeros(n_cut)
            cuts = _gather(mine_cut, world)
            dcuts = _gather(mine_dcut, world)
            if rank == ps:
                rows = torch.from_numpy(ex.debug_buffer(_lib.DBG_CUT_ROWS)).reshape(workers, -1)
                grows = torch.from_numpy(ex.debug_buffer(_lib.DBG_CUT_GRAD_ROWS)).reshape(workers, -1)
                wr = [r for r in range(world) if not (placement == "dedicated-ps" and r == ps)]
                for w, r in enumerate(wr):
                    if r == ps:
                        continue
                    if not torch.equal(rows[w], cuts[r]) or not torch.equal(grows[w], dcuts[r]):
                        print(f"[{tag}] step {t}: exchange rows of worker {w} (rank {r}) differ", flush=True)
                        ok = False
        # ---- sync: step 1 applies p0 - lr * sum_r g_r exactly (momentum starts at 0)
        if t == 0 and ring_backend != "nccl":  # (NCCL all-reduces the gradient buffer in place)
            g = ex.get_grads() if ex.is_worker else [None if p is None else (np.zeros_like(p[0]), np.zeros_like(p[1]))
                                                        for p in params]
            gv = _front_param_vec(g, nsync)
            g_all = _gather(gv, world)      # (collective: every rank)
            gsum = sum(g_all)
            gabs = sum(x.abs() for x in g_all)
            p1 = _front_param_vec(ex.get_params(), nsync) if ex.is_worker else None
            if p1 is not None:
                p0 = _front_param_vec(params, nsync)
                lr32 = torch.tensor(lr, dtype=torch.float32)
                want = p0 - lr32 * gsum
                # the W gradients are summed in another order by shard_update: allow a few roundings
                # of the terms' magnitudes (|p0| + lr * sum_r |g_r|), not of the (possibly cancelled) sum
                scale = (p0.abs() + lr32 * gabs) * 2.0 ** -23 + 1e-30
                dev = float(((p1 - want).abs() / scale).max())
                if dev > 4 * workers:
                    print(f"[{tag} rank {rank}] sync: p1 != p0 - lr * sum g ({dev:.1f} roundings)", flush=True)
                    ok = False
        if rank == 0:
            batches = [synthetic.batch(1, t, w * b, b, ex.in_shape, ex.classes) for w in range(workers)]
            lo, wire = ostep.train_step(orc, "baseline" if strategy == "ring" else strategy, workers, batches, lr=lr,
                                        emulate_bf16=not fp32, split=ex.lowered_split if strategy == "ralp" else None)
            l64 = None
            if orc64 is not None:
                l64, _ = ostep.train_step(orc64, "baseline" if strategy == "ring" else strategy, workers, batches, lr=lr,
                                          emulate_bf16=not fp32, accum64=True, split=ex.lowered_split if strategy == "ralp" else None)
            assert strategy == "ring" or fc_sharding == "multi" or wire == expect
            rel = abs(st.loss - lo) / abs(lo)
            # fp32: 1e-4, widened by the fp32 oracle's own fp64 spread where training is chaotic
            tol = (1e-4 + 3 * abs(l64 - lo) / abs(lo)) if fp32 else loss_tol
            if loss_steps is not None and t >= loss_steps:
                tol = float("inf")   # batch norm: only the first step's loss is sharp (test_resnet_gpu.py)
            print(f"[{model.name} {tag} W={workers}] step {t}: loss gpu {st.loss:.6f} oracle {lo:.6f} rel {rel:.2e} "
                  f"ms {st.ms_step:.2f} nvlink out {st.nvlink_out_bytes} in {st.nvlink_in_bytes}", flush=True)
            if not rel <= tol:
                ok = False
    got = ex.get_params() if ex.is_worker else None
    # every worker holds the same front (all-on-PS / ring: all) parameters
    if ex.is_worker or placement == "dedicated-ps":
        vec = _front_param_vec(got, nsync) if got is not None else torch.zeros_like(_front_param_vec(params, nsync))
        allv = _gather(vec, world)
        wr = [r for r in range(world) if not (placement == "dedicated-ps" and r == ex.ps_rank)]
        for r in wr[1:]:
            if not torch.equal(allv[r], allv[wr[0]]):
                print(f"[{tag}] rank {r} front parameters differ from rank {wr[0]} after the all-gather", flush=True)
                ok = False
    if rank == 0 and got is None:
        got = ex.get_params()   # the dedicated PS holds the FC tail; its front copy is not synced
        got = [g if i >= ex.lowered_split else None for i, g in enumerate(got)]
    ex.close()
    if rank == 0:
        w64s = orc64.numpy_params() if orc64 is not None else [None] * len(got)
        for li, (g, w, w64, p0) in enumerate(zip(got, orc.numpy_params(), w64s, params)):
            if g is None:
                continue
            if fp32:
                rel = np.linalg.norm(g[0] - w[0]) / np.linalg.norm(w[0])
                upd = np.linalg.norm(g[0] - w[0]) / np.linalg.norm(w[0] - p0[0])
                fl = np.linalg.norm(w64[0] - w[0]) / np.linalg.norm(w[0] - p0[0])
                print(f"   layer {li}: ||dp||/||p|| {rel:.3e}  ||dp||/||update|| {upd:.3e} (floor {fl:.3e})", flush=True)
                if not (rel <= 1e-4 or upd <= 3 * fl + 2e-2):   # the rule of tests/test_parity_fp32_gpu.py
                    ok = False
                continue
            upd = np.linalg.norm(w[0] - p0[0])
            dev = np.linalg.norm(g[0] - w[0]) / upd
            bound = cap if w64 is None else min(2 * np.linalg.norm(w64[0] - w[0]) / upd + 0.02, cap)
            print(f"   layer {li}: dev {dev:.3e} (bound {bound:.3e})", flush=True)
            if dev > bound:
                ok = False
    return ok


def main():
    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    # one rank per GPU only: ranks whose kernels wait on one another must never share a GPU
    # (separate processes on one B200 raised Xid 109, B200_PROFILING.md)
    dev = int(os.environ["LOCAL_RANK"])
    if dev >= torch.cuda.device_count():
        raise SystemExit("multi_rank_parity needs one GPU per rank")
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    shared = False
    ok = True
    cifar = catalog_lookup("cifar_small").with_batch_size(32)
    vgg16 = catalog_lookup("vgg16").with_batch_size(4)
    only = os.environ.get("RALPB_PARITY_ONLY")
    configs = [
        dict(model=cifar, strategy="ralp", steps=4),
        dict(model=parse_model(TINY), strategy="ralp", steps=3),
        dict(model=cifar, strategy="baseline", steps=3),
        dict(model=cifar, strategy="ring", steps=3),
        dict(model=cifar, strategy="ring", steps=3, ring_backend="nccl"),
        dict(model=cifar, strategy="ralp-mps", steps=4),
        dict(model=cifar, strategy="baseline-layers", steps=3),
        dict(model=parse_model(TINY), strategy="baseline-layers", steps=3),
        # branch groups (RALPB_MODULE) synchronised across ranks: GoogLeNet, FC-tail split
        dict(model=catalog_lookup("googlenet").with_batch_size(4), strategy="ralp", steps=2, lr=1e-3, floor=True,
             cap=0.5, split=62),
        # bottleneck blocks with per-worker batch norm synchronised across ranks (ResNet-50, FC-tail
        # split): the step is chaotic at b=4 (floor ~1 of the update), so the sharp checks are the
        # exact sync / exchange ones above, the first step's loss (5e-3) and the floor rule (no cap)
        dict(model=catalog_lookup("resnet-50").with_batch_size(4), strategy="ralp", steps=2, lr=1e-3, floor=True,
             cap=100.0, split=55, loss_tol=5e-3, loss_steps=1),
        # ... and with the sixteen blocks / eleven branch groups on the PS (splits 2 / 7, the
        # partitioner's cuts at b <= 64): the PS normalises each worker's rows with that worker's
        # own batch statistics, as the oracle's per-worker steps do
        dict(model=catalog_lookup("resnet-50").with_batch_size(4), strategy="ralp", steps=2, lr=1e-3, floor=True,
             cap=100.0, split=2, loss_tol=5e-3, loss_steps=1),
        dict(model=catalog_lookup("inception-v3").with_batch_size(4), strategy="ralp", steps=2, lr=1e-3, floor=True,
             cap=100.0, split=7, loss_tol=5e-3, loss_steps=1),
        dict(model=parse_model(TINY), strategy="ralp-mps", steps=3),
        # full VGG-16 geometry (224x224: first-conv, row-streamed 64-channel, slab pair kernels,
        # pool5 cut) at b=4 per rank
        dict(model=vgg16, strategy="ralp", steps=2, lr=1e-3, floor=True, cap=0.5),
    ]
    # the partitioner's split inside the conv stack: a conv back segment on the PS (cifar_small b=8
    # cuts at pool1; the tiny VGG at pool1), colocated and with a dedicated PS
    configs.append(dict(model=catalog_lookup("cifar_small").with_batch_size(8), strategy="ralp", steps=4, split=2))
    configs.append(dict(model=parse_model(TINY), strategy="ralp", steps=3, split=3))
    if world >= 2:
        configs.append(dict(model=catalog_lookup("cifar_small").with_batch_size(8), strategy="ralp", steps=4, split=2,
                            placement="dedicated-ps"))
    if world >= 2:  # RALP-N: a dedicated PS rank plus world-1 workers
        configs.append(dict(model=cifar, strategy="ralp", steps=4, placement="dedicated-ps"))
        configs.append(dict(model=parse_model(TINY), strategy="ralp", steps=3, placement="dedicated-ps"))
    if os.environ.get("RALPB_PARITY_FP32", "1") == "1":
        configs.append(dict(model=cifar, strategy="ralp", steps=4, precision="fp32"))
        configs.append(dict(model=cifar, strategy="baseline", steps=3, precision="fp32"))
        # lr 1e-4, two steps: VGG-16 from random init (no batch norm) at lr 1e-3 moves the loss by
        # ~2 % in ONE step and is chaotic from there (W=4: loss rel 4.6e-4 at step 2, W=2: 1.03e-4 at
        # step 1, while every weight tensor stays within 2x the fp32 oracle's own spread)
        configs.append(dict(model=vgg16, strategy="ralp", steps=2, lr=1e-4, precision="fp32"))
    for c in configs:
        name = f"{c['model'].name}:{c['strategy']}:{c.get('placement', 'colocated')}:{c.get('precision', 'bf16')}"
        if only and only not in name:
            continue
        if shared and (c["model"].name == "vgg16" or c.get("ring_backend") == "nccl"):
            continue
        ok &= run(c["model"], c["strategy"], c["steps"], rank, world, c.get("ring_backend", "native"), c.get("lr", 0.01),
                  c.get("floor", False), c.get("cap", 0.25), c.get("placement", "colocated"), c.get("precision", "bf16"),
                  c.get("split"), c.get("loss_tol", 2e-3), c.get("loss_steps"))
    flag = torch.tensor([0 if ok else 1], device=_dev())
    dist.all_reduce(flag)
    dist.destroy_process_group()
    if rank == 0:
        print("MULTI-RANK PARITY", "PASS" if flag.item() == 0 else "FAIL", flush=True)
    sys.exit(0 if flag.item() == 0 else 1)


if __name__ == "__main__":
    main()
