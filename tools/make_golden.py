"""Generate tests/golden/planner_golden.json by running the UNMODIFIED reference.

Imports `ralp` from /root/reference/pkg/src (read-only; bytecode and numba caches
are redirected to /tmp) with a catalog overlay directory built under /tmp: the
reference's own bundled descriptors plus this repo's vgg16 / cifar_small
descriptors (the reference catalog has neither; RALP_CATALOG_DIR replaces the
bundled directory, pkg/src/ralp/catalog.py:17,32-36).  Nothing from the
reference is written into the repo except these computed outputs.

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache python tools/make_golden.py
"""
from __future__ import annotations

import json
import os
import random
import shutil
import sys
import tempfile
from pathlib import Path

REPO = Path(__file__).resolve().parent.parent
REF_SRC = Path("/root/reference/pkg/src")
OUT = REPO / "tests" / "golden" / "planner_golden.json"

BATCHES = [1, 4, 8, 13, 22, 32, 64, 93, 95, 118, 119, 128, 256, 515]
WORKERS = [1, 2, 4, 8]


def main() -> None:
    sys.dont_write_bytecode = True
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    overlay = Path(tempfile.mkdtemp(prefix="ralp_catalog_"))
    for f in (REF_SRC / "ralp" / "catalog_data").glob("*.model"):
        shutil.copy(f, overlay / f.name)
    for name in ("vgg16", "cifar_small"):
        shutil.copy(REPO / "paper_1901_05803_b200" / "planner" / "catalog_data" / f"{name}.model", overlay)
    os.environ["RALP_CATALOG_DIR"] = str(overlay)
    sys.path.insert(0, str(REF_SRC))
    import ralp  # noqa: E402
    from ralp.costmodel import gpu_assignments, rows_to_csv  # noqa: E402

    out: dict = {"generator": "tools/make_golden.py", "reference": "pkg/src/ralp (unmodified)",
                 "models": {}, "find_split_cases": [], "random_models": [], "gpu_assignments": {},
                 "skew_cases": [], "cli_volumes_csv": {}}
    for name in ralp.catalog_names():
        m = ralp.catalog_lookup(name)
        table = [{"name": l.name, "kind": l.kind.value, "params": l.param_count,
                  "out": l.output_elems_per_sample, "flops": l.compute_flops_per_sample,
                  "hyperparams": dict(l.hyperparams),
                  "shape": None if l.output_shape is None else [l.output_shape.h, l.output_shape.w, l.output_shape.c]}
                 for l in m.layers]
        rec = {"default_batch": m.batch_size, "elem_bytes": m.bytes_per_element, "table": table,
               "total_params": m.total_param_count, "serialized": ralp.serialize_model(m),
               "skew_literal": ralp.compute_skewness([l.param_count * 4 for l in m.layers], "literal_values"),
               "eligible_k15": ralp.profile(m, ralp.ProfilerConfig(threshold=-1.5)).eligible,
               "batches": {}}
        for b in sorted(set(BATCHES + [m.batch_size])):
            mb = m.with_batch_size(b)
            rep = ralp.profile(mb)
            e = {"skewness": rep.skewness, "eligible": rep.eligible, "split": rep.split_index,
                 "cost": rep.split_cost_bytes, "profile_json": rep.to_json(),
                 "compute_load_none": list(ralp.compute_load(mb, None, 1)), "volumes": {}}
            if rep.split_index is not None:
                e["compute_load"] = {w: list(ralp.compute_load(mb, rep.split_index, w)) for w in WORKERS}
            for w in WORKERS:
                vb, vr = ralp.volume_baseline(mb, w), ralp.volume_ring(mb, w)
                v = {"baseline": [vb.total_bytes_per_step, vb.parameter_sync_bytes, vb.activation_bytes],
                     "ring": [vr.total_bytes_per_step, vr.parameter_sync_bytes, vr.activation_bytes]}
                if rep.split_index is not None:
                    va = ralp.volume_ralp(mb, rep.split_index, w)
                    v["ralp"] = [va.total_bytes_per_step, va.parameter_sync_bytes, va.activation_bytes]
                e["volumes"][w] = v
            rec["batches"][b] = e
        out["models"][name] = rec
        out["cli_volumes_csv"][name] = rows_to_csv(ralp.compare_strategies(m, [1, 2, 4, 8]))

    K = ralp.LayerKind
    cases = [  # literal inputs of the reference's known-answer tests (pkg/tests/test_profiler.py:144-163)
        ([10, 10, 80], [100, 50, 1], ["conv", "pool", "fc"]),
        ([10], [100], ["fc"]),
        ([1, 2, 3], [5, 5, 5], ["conv", "conv", "conv"]),
        ([1, 1, 1], [100, 100, 1], ["pool", "pool", "fc"]),
        ([10, 10], [20, 10], ["fc", "fc"]),
        ([5, 0, 100, 100], [1000, 10, 10, 1], ["conv", "pool", "fc", "fc"]),
    ]
    for pb, ob, kinds in cases:
        r = ralp.find_split(pb, ob, [K(k) for k in kinds])
        out["find_split_cases"].append({"param_bytes": pb, "output_bytes": ob, "kinds": kinds,
                                        "result": None if r is None else [r.index, r.cost_bytes]})
    rnd = random.Random(0xACCE)
    kinds_all = ["conv", "pool", "fc", "norm", "act", "block"]
    for _ in range(400):
        n = rnd.randint(1, 40)
        kinds = [rnd.choice(kinds_all) for _ in range(n)]
        pb = [rnd.randrange(1, 10 ** 6) * 4 if k in ("conv", "fc", "block") else 0 for k in kinds]
        ob = [rnd.randrange(1, 5 * 10 ** 5) * 4 for _ in kinds]
        r = ralp.find_split(pb, ob, [K(k) for k in kinds])
        skew = ralp.compute_skewness(pb) if n >= 2 and sum(pb) > 0 else None
        out["random_models"].append({"param_bytes": pb, "output_bytes": ob, "kinds": kinds, "skewness": skew,
                                     "result": None if r is None else [r.index, r.cost_bytes]})
    for total in range(2, 17):
        out["gpu_assignments"][total] = gpu_assignments(total)
    for vals in ([1, 9], [9, 1], [1, 1, 1, 1], [0, 0, 5, 0], [3, 1, 4, 1, 5, 9, 2, 6]):
        out["skew_cases"].append({"params": vals, "index_weighted": ralp.compute_skewness(vals),
                                  "literal_values": ralp.compute_skewness(vals, "literal_values")})
    OUT.parent.mkdir(parents=True, exist_ok=True)
    OUT.write_text(json.dumps(out, indent=1, sort_keys=True))
    shutil.rmtree(overlay)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
