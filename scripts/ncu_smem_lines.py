"""Shared-memory wavefronts per source line of one kernel launch in an ncu report (total, excess, ideal) and
the instructions that issue them: python scripts/ncu_smem_lines.py REP LAUNCH_SKIP [N]"""
import csv
import io
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep, skip = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
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
        rows.append((fname, int(d["Line No"]), f("L1 Wavefronts Shared"), f("L1 Wavefronts Shared Excessive"),
                     f("Instructions Executed")))
if header:
    print("columns:", [h for h in header if "Shared" in h or "Wavefront" in h])
tw = sum(r[2] for r in rows) or 1
src = {}
for fn in {r[0] for r in rows}:
    p = os.path.join(ROOT, "paper_1406_1717_b200", "csrc", fn)
    if os.path.exists(p):
        src[fn] = open(p).read().splitlines()
print(f"shared wavefronts {tw:.4g}, excess {sum(r[3] for r in rows):.4g}")
for r in sorted(rows, key=lambda r: -r[2])[:top]:
    line = src[r[0]][r[1] - 1].strip()[:70] if r[0] in src and r[1] <= len(src[r[0]]) else ""
    print(f"{r[0]}:{r[1]:<5d} wf {r[2] / 1e6:6.1f}M ({100 * r[2] / tw:4.1f}%) excess {r[3] / 1e6:6.1f}M | {line}")
