"""Summarise an ncu --set full report into the JSON kept under profiles/.

python tools/ncu_summary.py REPORT.ncu-rep --alg-bytes B --source "cmd" [--launch i] > out.json

Per launch: duration, DRAM bytes, issue / FP64 / warp activity, instruction
count, registers, grid, shared-memory bank conflicts and the warp-stall
shares; ``dram_traffic_bytes_per_launch`` (read + write) is what bench.py
reports as ``roofline.traffic``.
"""

import argparse
import csv
import io
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__cycles_active.avg", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "smsp__thread_inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "launch__occupancy_limit_shared_mem",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--alg-bytes", type=float, default=None)
    ap.add_argument("--source", default="")
    ap.add_argument("--launch", type=int, default=0)
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2 + a.launch]
    col = {h: i for i, h in enumerate(hdr)}
    out = {"Kernel Name": data[col["Kernel Name"]]}
    for k in KEYS:
        if k in col:
            out[k] = f"{data[col[k]]} {units[col[k]]}".strip()
    st = {}
    for h, i in col.items():
        if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
            try:
                st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(
                    data[i].replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values()) or 1.0
    out["stall_share_pct"] = {k: round(100 * v / tot, 1) for k, v in
                              sorted(st.items(), key=lambda kv: -kv[1]) if v / tot > 0.0005}
    traffic = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = col[k]
        traffic += float(data[i].replace(",", "")) * SCALE.get(units[i], 1)
    out["dram_traffic_bytes_per_launch"] = traffic
    if a.alg_bytes:
        out["algorithmic_bytes_per_launch"] = a.alg_bytes
    if a.alg_bytes:  # warp instructions x 32 lanes per point-update (24 B each)
        upd = a.alg_bytes / 24.0
        out["thread_instructions_per_update"] = round(
            32 * float(data[col["smsp__inst_executed.sum"]].replace(",", "")) / upd, 1)
    out["source"] = a.source
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
