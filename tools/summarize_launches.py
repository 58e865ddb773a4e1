"""Summarise an ncu launch list (--csv --metrics gpu__time_duration.sum[,dram__bytes_*]).

Steps are delimited by the engine's `bump_kernel` (first node of every step).  Prints
per-kernel-family time/share/DRAM bytes for step number --step (default: the 4th
step, i.e. the first timed bench step after 3 warm-ups) and optionally writes the
tensor-core kernels' DRAM traffic of that step to a JSON file for bench.py's
roofline.traffic.

usage: python tools/summarize_launches.py launches.csv [--step N] [--traffic-json out.json]
"""
import argparse
import csv
import json
import re
from collections import OrderedDict, defaultdict

TENSOR = re.compile(r"conv_slab_(fwd|wgrad)\w*_kernel|conv_row64_kernel|conv_first_\w+_kernel|gemm_sm100_kernel")


def kind_of(name: str) -> str:
    """Map a kernel name to the engine's launch kind (ralpb_launch_rec.kind names)."""
    if "conv_slab_wgrad_pair" in name:
        return "conv_wgrad_pair"
    if "conv_slab_wgrad" in name:
        return "conv_wgrad"
    if "conv_row64" in name:
        return "conv_fwd"
    if "conv_slab_fwd" in name:
        return "conv_fwd_pair" if re.search(r"\(bool\)1|, 1>|,\s*true>", name) else "conv_fwd"
    if "conv_first_fwd" in name:
        return "first_conv_fwd"
    if "conv_first_wgrad" in name:
        return "first_conv_wgrad"
    return "gemm"


def family(name: str) -> str:
    n = re.sub(r"\(.*", "", name)
    n = re.sub(r"^void ", "", n)
    n = n.replace("ralpb::", "")
    return n


def load(path):
    rows = OrderedDict()
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        k = int(r["ID"])
        d = rows.setdefault(k, {"name": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"]})
        v = r["Metric Value"].replace(",", "")
        try:
            v = float(v)
        except ValueError:
            continue
        if r["Metric Name"] == "gpu__time_duration.sum":
            d["ns"] = v * (1e3 if r["Metric Unit"] == "us" else 1e6 if r["Metric Unit"] == "ms" else 1.0)
        elif r["Metric Name"].startswith("dram__bytes"):
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(r["Metric Unit"], 1)
            d[r["Metric Name"]] = v * mult
    return list(rows.values())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--step", type=int, default=3)
    ap.add_argument("--traffic-json")
    a = ap.parse_args()
    rows = load(a.csv)
    steps, cur = [], None
    for r in rows:
        if "bump_kernel" in r["name"]:
            cur = []
            steps.append(cur)
        elif cur is not None:
            cur.append(r)
    step = steps[a.step]
    total = sum(r.get("ns", 0) for r in step)
    fam = defaultdict(lambda: [0, 0.0, 0.0])
    for r in step:
        f = fam[family(r["name"])]
        f[0] += 1
        f[1] += r.get("ns", 0)
        f[2] += r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)
    print(f"step {a.step} of {len(steps)}: {len(step) + 1} launches, serialized kernel time {total / 1e6:.3f} ms")
    print(f"{'kernel':60s} {'n':>4s} {'ms':>8s} {'share':>6s} {'DRAM GB':>8s}")
    for k, (n, ns, by) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:60]:60s} {n:4d} {ns / 1e6:8.3f} {ns / total:6.1%} {by / 1e9:8.3f}")
    print("\nper launch:")
    for r in step:
        by = r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)
        print(f"  {family(r['name'])[:70]:70s} grid {r['grid']:>14s} {r.get('ns', 0) / 1e3:9.1f} us {by / 1e6:9.1f} MB")
    if a.traffic_json:
        t = [r for r in step if TENSOR.search(r["name"])]
        per_kind = defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "ms": 0.0})
        for r in t:
            k = per_kind[kind_of(r["name"])]
            k["launches"] += 1
            k["dram_bytes"] += r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0)
            k["ms"] += r.get("ns", 0) / 1e6
        for k in per_kind.values():
            k["dram_bytes_per_launch"] = k["dram_bytes"] / k["launches"]
        out = {"source": a.csv, "step": a.step, "tensor_launches": len(t),
               "dram_bytes_per_step": sum(r.get("dram__bytes_read.sum", 0) + r.get("dram__bytes_write.sum", 0) for r in t),
               "serialized_ms": sum(r.get("ns", 0) for r in t) / 1e6,
               "per_kind": per_kind,
               "note": "ncu launch list, cold-cache serialized launches; bytes summed over the step's tcgen05 kernels"}
        with open(a.traffic_json, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
