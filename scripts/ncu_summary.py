"""Summarise an ncu --set full report (one kernel launch) into the JSON kept under profiles/.

usage: python scripts/ncu_summary.py REPORT.ncu-rep [--kernel REGEX] [--launch I] > profiles/NAME.json
(stall shares come from the source page of all launches of the report matching --kernel)
"""
import csv
import io
import json
import re
import subprocess
import sys

FIELDS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct", "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]
STALLS = ["stall_long_sb", "stall_wait", "stall_barrier", "stall_selected", "stall_branch_resolving",
          "stall_short_sb", "stall_no_inst", "stall_not_selected", "stall_math", "stall_mio", "stall_dispatch"]


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def main():
    rep = sys.argv[1]
    kern = sys.argv[sys.argv.index("--kernel") + 1] if "--kernel" in sys.argv else None
    extra = ["-k", f"regex:{kern}"] if kern else []
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv", *extra))))
    idx = int(sys.argv[sys.argv.index("--launch") + 1]) if "--launch" in sys.argv else 0
    hdr, units, vals = rows[0], rows[1], rows[2 + idx]
    out = {"kernel": vals[hdr.index("Kernel Name")]}
    for f in FIELDS:
        if f in hdr:
            i = hdr.index(f)
            out[f] = {"value": vals[i], "unit": units[i]}
    src = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass", *extra)
    srows = list(csv.reader(io.StringIO(src)))
    h = srows[1]
    tot = {s: 0.0 for s in STALLS}
    for r in srows[2:]:
        for s in STALLS:
            try:
                tot[s] += float(r[h.index(s)])
            except (ValueError, IndexError):
                pass
    T = sum(tot.values()) or 1.0
    out["stall_share_pct"] = {re.sub("^stall_", "", k): round(100 * v / T, 1) for k, v in
                              sorted(tot.items(), key=lambda kv: -kv[1]) if v > 0}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
