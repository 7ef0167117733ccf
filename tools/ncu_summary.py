"""Summarise one kernel of an ncu report (--set full) into a small JSON for profiles/.

    python tools/ncu_summary.py gpurun_out/prof_skew.ncu-rep --rows 2000000 --note "..." > profiles/x.json
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
from collections import Counter

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum", "smsp__inst_executed.sum", "sm__cycles_active.avg",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__block_size",
    "launch__grid_size", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
]


def raw(rep: str, kernel: str | None):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h = rows[0]
    data = [r for r in rows[2:] if len(r) == len(h)]
    if kernel:
        data = [r for r in data if kernel in r[h.index("Kernel Name")]]
    return h, data[0]


def source_mix(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return None
    h = rows[1]
    ia, isrc = h.index("Instructions Executed"), h.index("Source")
    c = Counter()
    for r in rows[2:]:
        if len(r) <= ia or not r[ia].isdigit():
            continue
        t = r[isrc].split()
        if not t:
            continue
        op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
        c[op.split(".")[0]] += int(r[ia])
    tot = sum(c.values())
    return {k: round(v / tot, 4) for k, v in c.most_common(16)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--kernel", default=None)
    ap.add_argument("--rows", type=int, default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    h, v = raw(a.rep, a.kernel)
    d = {k: v[h.index(k)] for k in KEYS if k in h}
    st = {}
    for i, k in enumerate(h):
        if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
            try:
                st[k.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(v[i])
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    d["stall_share"] = {k: round(x / tot, 3) for k, x in sorted(st.items(), key=lambda t: -t[1])[:10]}
    d["instruction_mix"] = source_mix(a.rep)
    if a.rows:
        d["rows"] = a.rows
        try:
            d["wavefronts_ld_per_row"] = float(d["l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"]) / a.rows
            d["warp_instructions_per_row"] = float(d["smsp__inst_executed.sum"]) / a.rows
        except (KeyError, ValueError):
            pass
    d["note"] = a.note
    print(json.dumps(d, indent=1))


if __name__ == "__main__":
    main()
