"""Sum an ncu --csv launch list (one step of tools/prof_step.py) into per-kernel times and DRAM bytes.

    python tools/ncu_step.py LAUNCHES.csv [--json profiles/ncu_step_dram.json --workload long64k]
Skips torch's own launches (input generation); prints the repo kernels' share of the step.
"""
from __future__ import annotations

import argparse
import collections
import csv
import json


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--json", default=None)
    ap.add_argument("--workload", default="long64k")
    a = ap.parse_args()
    rows = [r for r in csv.reader(open(a.csv)) if len(r) > 10]
    hdr = rows[0]
    col = {h: n for n, h in enumerate(hdr)}
    per = collections.defaultdict(dict)
    for r in rows[1:]:
        if r[col["ID"]] == "ID":
            continue
        per[r[col["ID"]]]["name"] = r[col["Kernel Name"]]
        per[r[col["ID"]]][r[col["Metric Name"]]] = float(r[col["Metric Value"]].replace(",", ""))
    launches = [v for _, v in sorted(per.items(), key=lambda kv: int(kv[0])) if "onedf::" in v["name"]]
    t = collections.Counter()
    b = collections.Counter()
    n = collections.Counter()
    for v in launches:
        name = v["name"].split("(")[0].replace("void ", "").split("<")[0]
        t[name] += v.get("gpu__time_duration.sum", 0.0)
        b[name] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
        n[name] += 1
    total_t = sum(t.values())
    total_b = sum(b.values())
    print(f"{len(launches)} repo launches, {total_t / 1e6:.2f} ms (cold-cache, serialised), DRAM {total_b / 1e9:.2f} GB")
    for name, ms in t.most_common():
        print(f"  {name:40s} x{n[name]:3d}  {ms / 1e6:8.3f} ms  {ms / total_t * 100:5.1f} %  DRAM {b[name] / 1e9:7.3f} GB")
    if a.json:
        with open(a.json, "w") as f:
            json.dump({"_source": f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                                  f"--clock-control none of tools/prof_step.py --config {a.workload} --steps 1 "
                                  f"({len(launches)} repo launches; summed by tools/ncu_step.py)",
                       "workload": a.workload, "launches": len(launches), "bytes_per_step": total_b,
                       "serialised_ms": total_t / 1e6,
                       "per_kernel": {k: {"launches": n[k], "ms": t[k] / 1e6, "dram_bytes": b[k]} for k in t}},
                      f, indent=1)


if __name__ == "__main__":
    main()
