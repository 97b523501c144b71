"""Summarise an `ncu --set full` report into the per-kernel counter table kept under profiles/.

    python tools/ncu_summary.py gpurun_out/full_r01.ncu-rep > profiles/ncu_full_r01_summary.txt
    python tools/ncu_summary.py REP --traffic profiles/ncu_traffic.json   # also refresh dram bytes per launch
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem",
    "smsp__inst_executed.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum",
]
STALL = "smsp__average_warps_issue_stalled_"
# kernel name -> bench phase key (ncu_traffic.json)
PHASE = {"topk_attn_fwd_kernel": "fwd_topk", "bwd_query_kernel": "bwd_query", "bwd_key_kernel": "bwd_key",
         "csr_count_kernel": "bwd_csr_count"}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def fnum(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--traffic", default=None)
    a = ap.parse_args()
    hdr, units, data = raw(a.rep)
    col = {h: n for n, h in enumerate(hdr)}
    traffic = {}
    for r in data:
        name = r[col["Kernel Name"]]
        print("-----")
        print(f"  {'Kernel Name':70s} {name}")
        for m in METRICS:
            if m in col:
                print(f"  {m:70s} {r[col[m]]} {units[col[m]]}")
        stalls = []
        for h, n in col.items():
            if h.startswith(STALL) and h.endswith("_per_issue_active.ratio"):
                v = fnum(r[n])
                if v == v and v > 0.1:
                    stalls.append((v, h[len(STALL):-len("_per_issue_active.ratio")]))
        stalls.sort(reverse=True)
        print("  stalls: " + ", ".join(f"{k}={v:.2f}" for v, k in stalls[:8]))
        for key, phase in PHASE.items():
            if key in name and phase not in traffic:
                rd = fnum(r[col["dram__bytes_read.sum"]])
                wr = fnum(r[col["dram__bytes_write.sum"]])
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[col["dram__bytes_read.sum"]]]
                scale_w = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[units[col["dram__bytes_write.sum"]]]
                traffic[phase] = int(rd * scale + wr * scale_w)
    if a.traffic:
        d = {"_source": f"ncu --set full --clock-control none capture ({a.rep}; tools/prof_step.py long64k): "
                        "dram__bytes_read.sum + dram__bytes_write.sum per launch, bytes"}
        d.update(traffic)
        with open(a.traffic, "w") as f:
            json.dump(d, f, indent=2)
            f.write("\n")
    return 0


if __name__ == "__main__":
    sys.exit(main())
