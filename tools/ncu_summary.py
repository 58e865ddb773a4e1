"""Print the key counters of every kernel in an ncu report (run here, no GPU needed).

Tensor-pipe utilisation of the tcgen05 kernels: ncu 2025 on sm_100a reports the legacy
`sm__pipe_tensor_cycles_active_realtime...pct` near 0 for UTC*MMA work (it normalises a per-SMSP
realtime count by the wrong peak); `sm__mem_tensor_cycles_active` (= the hmma-subpipe realtime
cycles / 4 SMSPs / elapsed SM cycles, checked on the conv13 backward-filter capture: 148.8k of
187.2k cycles) is the consistent one and is what is printed.

usage: python tools/ncu_summary.py report.ncu-rep > summary.txt
"""
import csv
import io
import re
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("gpc__cycles_elapsed.max.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active % (tcgen05)"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active % of active"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem->tensor-core pipe %"),
    ("l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed", "smem bank reads %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
]


def main():
    rep = sys.argv[1]
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    idx = {h: i for i, h in enumerate(hdr)}
    print(f"# {rep}")
    for r in rows[2:]:
        name = r[idx["Kernel Name"]] if "Kernel Name" in idx else r[4]
        short = name.split("(")[0]
        print(f"\n## {short}")
        for k, label in KEYS:
            if k in idx:
                print(f"  {label:28s} {r[idx[k]]:>16s} {units[idx[k]]}")


if __name__ == "__main__":
    main()
