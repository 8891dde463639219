"""Condense one round's GPU evidence (tools/profile_r02.sh) into profiles/:

    python tools/summarize_round.py r02

writes profiles/<tag>_bench.json, <tag>_launches.json, <tag>_knn_full.json,
<tag>_build_full.json, <tag>_radius_full.json, <tag>_sanitizer.txt and refreshes
profiles/ncu_summary.json (the measured figures bench.py reports beside its
byte model)."""
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
import ncu_summary  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r02"
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


def dump(name, obj):
    with open(os.path.join(P, name), "w") as fh:
        json.dump(obj, fh, indent=1)
        fh.write("\n")


line = open(os.path.join(G, f"{tag}_bench.json")).read().strip().splitlines()[-1]
dump(f"{tag}_bench.json", json.loads(line))
dump(f"{tag}_launches.json", ncu_summary.launches(os.path.join(G, f"{tag}_launches.csv")))
knn = ncu_summary.full(os.path.join(G, f"{tag}_knn.ncu-rep"))
dump(f"{tag}_knn_full.json", knn)
build = ncu_summary.full(os.path.join(G, f"{tag}_build.ncu-rep"))
dump(f"{tag}_build_full.json", build)
radius = {"c2_filled": ncu_summary.full(os.path.join(G, f"{tag}_c2_radius.ncu-rep")),
          "c3_hollow_sphere": ncu_summary.full(os.path.join(G, f"{tag}_c3_radius.ncu-rep"))}
dump(f"{tag}_radius_full.json", radius)
san = os.path.join(G, f"{tag}_sanitizer.txt")
if os.path.exists(san):
    keep = [ln for ln in open(san) if ln.startswith("==") or "ERROR SUMMARY" in ln]
    open(os.path.join(P, f"{tag}_sanitizer.txt"), "w").writelines(keep)

k = knn[0]
kernels = {}
for rec in knn + build + radius["c2_filled"] + radius["c3_hollow_sphere"]:
    name = rec["kernel"].split("(")[0].replace("void ", "").replace("unnamed>::", "")
    kernels.setdefault(name, {key: rec.get(key) for key in (
        "duration_ms", "dram_bytes_per_launch", "l1_hit_pct", "l2_hit_pct", "threads_per_inst",
        "issue_active_pct", "warps_active_pct", "stalls_pct", "warp_instructions")})
summary = {
    "source": f"profiles/{tag}_knn_full.json, {tag}_build_full.json, {tag}_radius_full.json "
              "(ncu --set full --clock-control none; C2 1e7/1e7 k=10, build 1e7, C3 radius)",
    "knn_kernel_dram_bytes_per_launch": k["dram_bytes_per_launch"],
    "knn_kernel_duration_ms_ncu": k["duration_ms"],
    "kernels": kernels,
    "knn_hardware": {
        "source": f"ncu --set full of knn_kernel<10> at C2 (profiles/{tag}_knn_full.json)",
        "bound": "instruction issue with SIMT divergence (not HBM)",
        "issue_active_pct": k.get("issue_active_pct"),
        "threads_per_inst": k.get("threads_per_inst"),
        "sm_throughput_pct": k.get("sm_throughput_pct"),
        "l1_hit_pct": k.get("l1_hit_pct"), "l2_hit_pct": k.get("l2_hit_pct"),
        "top_stalls_pct": k.get("stalls_pct"),
    },
}
dump("ncu_summary.json", summary)
print("wrote", tag, "summaries; knn", k["duration_ms"], "ms,", k["dram_bytes_per_launch"] / 1e9, "GB")
