"""Summarise an ncu report per CUDA source line: python scripts/ncu_lines.py REP KERNEL_REGEX [N]
(ncu -i REP --page source --print-source cuda,sass; needs -lineinfo builds)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}", "--launch-skip", skip, "-c", "1"], capture_output=True, text=True).stdout
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

        def f(key):
            try:
                return float(d.get(key, 0) or 0)
            except ValueError:
                return 0.0
        rows.append((fname, d["Line No"], d["Source"][:70].strip(), f("Warp Stall Sampling (All Samples)"),
                     f("Instructions Executed"), f("L1 Wavefronts Shared Excessive"), f("stall_short_sb"),
                     f("stall_long_sb"), f("stall_barrier")))
tot_s = sum(r[3] for r in rows) or 1
tot_i = sum(r[4] for r in rows) or 1
print(f"{'file:line':28s} {'stall%':>6s} {'inst%':>6s} {'smem_excess':>12s} {'shortsb':>8s} {'longsb':>7s} {'bar':>6s}  source")
for r in sorted(rows, key=lambda r: -r[3])[:top]:
    print(f"{r[0] + ':' + r[1]:28s} {100 * r[3] / tot_s:6.1f} {100 * r[4] / tot_i:6.1f} {r[5]:12.0f} {r[6]:8.0f} {r[7]:7.0f} {r[8]:6.0f}  {r[2]}")
