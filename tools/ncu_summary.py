#!/usr/bin/env python3
"""Summarise ncu captures (run HERE, no GPU needed):
    python tools/ncu_summary.py gpurun_out/fa.ncu-rep [...]  > profiles/rNN/<name>.md
Prints duration, clocks, DRAM traffic and throughput, tensor-pipe activity,
registers / smem, and the top stall reasons of the captured kernel."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "tensor hmma inst % (active)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe inst % (active)"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe active % (active)"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe active % (active)"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/block"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_dim_x", "cluster x"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [dict(zip(hdr, r)) for r in rows[2:]], dict(zip(hdr, units))


def main():
    for rep in sys.argv[1:]:
        data, units = raw(rep)
        for d in data:
            print(f"## {rep}: `{d.get('Kernel Name', '?')[:140]}`\n")
            print("| metric | value |\n|---|---|")
            for k, label in KEYS:
                if k in d:
                    print(f"| {label} (`{k}`) | {d[k]} {units.get(k, '')} |")
            stalls = sorted(((float(v.replace(',', '') or 0), k) for k, v in d.items()
                             if k.startswith("smsp__average_warps_issue_stalled_")
                             and k.endswith("_per_issue_active.ratio")
                             and v.replace(',', '').replace('.', '').isdigit()), reverse=True)
            if stalls:
                print("\ntop stall reasons (warps per issue-active cycle):\n")
                for v, k in stalls[:8]:
                    print(f"* {k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}: {v:.3f}")
            print()


if __name__ == "__main__":
    main()
