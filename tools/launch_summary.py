"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
the JSON kept under profiles/: per kernel launches, total and share of time.

python tools/launch_summary.py LAUNCHES.csv --command "..." > out.json
"""
import argparse
import csv
import json
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--command", default="")
    a = ap.parse_args()
    with open(a.csv) as fh:
        lines = [l for l in fh if l.startswith('"')]
    rows = list(csv.DictReader(lines))
    summ = {}
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = re.sub(r"\(.*$", "", r["Kernel Name"]).strip()
        us = float(r["Metric Value"].replace(",", "")) / (1000.0 if r["Metric Unit"] == "ns" else 1.0)
        s = summ.setdefault(name, {"launches": 0, "total_us": 0.0})
        s["launches"] += 1
        s["total_us"] += us
    tot = sum(s["total_us"] for s in summ.values()) or 1.0
    for s in summ.values():
        s["total_us"] = round(s["total_us"], 1)
        s["share_pct"] = round(100.0 * s["total_us"] / tot, 2)
    out = {"command": a.command,
           "note": "first launches of the bench command under ncu (cold-cache, serialized "
                   "per-launch times: compare shares, not absolutes); microseconds",
           "n_launches": sum(s["launches"] for s in summ.values()),
           "summary": dict(sorted(summ.items(), key=lambda kv: -kv[1]["total_us"]))}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
