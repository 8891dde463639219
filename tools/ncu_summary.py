"""Summarise ncu captures into the JSON committed under profiles/.

    python tools/ncu_summary.py full  gpurun_out/prof_knn.ncu-rep  > profiles/<name>.json
    python tools/ncu_summary.py launches gpurun_out/launches.csv   > profiles/<name>.json

`full` reads one `ncu --set full` report (raw page + SASS source page) and
records, per kernel: duration, DRAM bytes read/written, L1/L2 hit rates,
warp occupancy, issue activity, SIMT efficiency (threads per executed
instruction), registers and the top stall reasons.  `launches` condenses a
`--metrics gpu__time_duration.sum` launch list into per-kernel counts, mean
duration and share of total device time.
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

RAW = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", None),
    "dram_write_bytes": ("dram__bytes_write.sum", None),
    "dram_throughput_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "l1_hit_pct": ("l1tex__t_sector_hit_rate.pct", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "threads_per_inst": ("smsp__thread_inst_executed_per_inst_executed.ratio", 1),
    "registers": ("launch__registers_per_thread", 1),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
}
UNIT = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
        "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1, "ms": 1, "nsecond": 1e-6}


def _ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True,
                          text=True, check=True).stdout


def full(rep):
    rows = list(csv.reader(io.StringIO(_ncu(rep, "--page", "raw"))))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        k = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for key, (metric, _) in RAW.items():
            if metric not in hdr:
                continue
            i = hdr.index(metric)
            v = float(vals[i].replace(",", ""))
            u = units[i]
            if key.endswith("_bytes"):
                v *= UNIT.get(u, 1)
            elif key == "duration_ms":
                v *= UNIT.get(u, 1e-6)
            k[key] = round(v, 4)
        if "dram_read_bytes" in k:
            k["dram_bytes_per_launch"] = k["dram_read_bytes"] + k.get("dram_write_bytes", 0)
        out.append(k)
    # stall reasons from the SASS page (first kernel)
    try:
        src = list(csv.reader(io.StringIO(_ncu(rep, "--page", "source",
                                                "--print-source", "sass"))))
        h = src[1]
        data = src[2:]
        cols = [i for i, x in enumerate(h) if x.startswith("stall_") and "Not Issued" not in x]
        agg = {h[i][6:]: sum(int(r[i] or 0) for r in data) for i in cols}
        tot = sum(agg.values()) or 1
        top = sorted(agg.items(), key=lambda kv: -kv[1])[:6]
        out[0]["stalls_pct"] = {k: round(100 * v / tot, 1) for k, v in top}
        ie = h.index("Instructions Executed")
        out[0]["warp_instructions"] = sum(int(r[ie]) for r in data)
    except Exception as exc:  # pragma: no cover - diagnostic only
        out[0]["stalls_error"] = str(exc)
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    i_n, i_v, i_u = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[start + 1:]:
        name = r[i_n].split("(")[0].replace("void ", "")
        v = float(r[i_v].replace(",", "")) * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
                                               "usecond": 1e-3}.get(r[i_u], 1e-6)
        agg[name].append(v)
    total = sum(sum(v) for v in agg.values())
    return {"total_ms": round(total, 4), "launches": sum(len(v) for v in agg.values()),
            "kernels": {k: {"count": len(v), "mean_ms": round(sum(v) / len(v), 4),
                            "share": round(sum(v) / total, 4)}
                        for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1]))}}


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    res = full(path) if mode == "full" else launches(path)
    json.dump(res, sys.stdout, indent=1)
    print()
