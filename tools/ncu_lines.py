"""Per-source-line digest of one kernel in an ncu report (stall samples and
executed instructions by CUDA line).

    python tools/ncu_lines.py report.ncu-rep kernel_regex [top]
"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
txt = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kre}", "--page", "source",
                      "--print-source", "cuda,sass", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iI = hdr.index("Instructions Executed")
iT = hdr.index("Thread Instructions Executed")
lines = []
for r in rows[hi + 1:]:
    if len(r) <= iT or r[2] != "-":
        continue  # SASS rows carry an address; CUDA-line rows have "-"
    try:
        lines.append((int(r[0]), r[1], int(r[iS] or 0), int(r[iI] or 0), int(r[iT] or 0)))
    except ValueError:
        pass
S = sum(x[2] for x in lines) or 1
I = sum(x[3] for x in lines) or 1
T = sum(x[4] for x in lines) or 1
print(f"samples {S}  warp-inst {I}  thread-inst/warp-inst {T / I:.2f}")
key = 3 if "--by-inst" in sys.argv else 2
for ln, src, s, i, t in sorted(lines, key=lambda x: -x[key])[:top]:
    print(f"{ln:5d} {100 * s / S:5.1f}% stall {100 * i / I:5.1f}% inst {t / max(i, 1):5.1f} thr  {src.strip()[:80]}")
