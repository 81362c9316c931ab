"""Top source lines of one kernel launch in an ncu report, by instructions (with stall and
shared-memory excess): python scripts/ncu_top_lines.py REP LAUNCH_SKIP [N]"""
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, skip = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "--launch-skip", skip,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows, fname, header = [], None, None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        header = rec
        continue
    if header and rec[0] not in ("", "Function Name") and len(rec) == len(header):
        d = dict(zip(header, rec))

        def f(k):
            try:
                return float(d.get(k, 0) or 0)
            except ValueError:
                return 0.0
        rows.append((fname, int(d["Line No"]), f("Instructions Executed"), f("Warp Stall Sampling (All Samples)"),
                     f("L1 Wavefronts Shared Excessive")))
ti = sum(r[2] for r in rows) or 1
ts = sum(r[3] for r in rows) or 1
src = {}
for fn in {r[0] for r in rows}:
    p = os.path.join(ROOT, "paper_1406_1717_b200", "csrc", fn)
    if os.path.exists(p):
        src[fn] = open(p).read().splitlines()
print(f"total warp-instructions {ti:.4g}, smem excess wavefronts {sum(r[4] for r in rows):.4g}")
for r in sorted(rows, key=lambda r: -r[2])[:top]:
    line = src[r[0]][r[1] - 1].strip()[:80] if r[0] in src and r[1] <= len(src[r[0]]) else ""
    print(f"{r[0]}:{r[1]:<5d} inst {100 * r[2] / ti:5.1f}% stall {100 * r[3] / ts:5.1f}% xs {r[4] / 1e6:6.1f}M | {line}")
