"""Instruction / stall shares of the medium kernel by phase:
python scripts/ncu_phases.py REP KERNEL_REGEX SKIP.  Phase boundaries come from marker
comments in csrc/mf_medium.cuh and csrc/mf_blocksort.cuh, so they follow the code."""
import contextlib
import io
import os
import runpy
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CSRC = os.path.join(ROOT, "paper_1406_1717_b200", "csrc")


def marks(fname, pats):
    lines = open(os.path.join(CSRC, fname)).read().splitlines()
    out = []
    for name, pat in pats:
        ln = next(i + 1 for i, l in enumerate(lines) if pat in l)
        out.append((ln, name))
    return sorted(out)


MED = marks("mf_medium.cuh", [("pair-merge (key slots)", "auto merge_keys = [&]"),
                              ("tile loop / phase 1 calls", "for (uint64_t t = t_begin; t < t_end; ++t)"),
                              ("zero rows", "phase 2: per-pair postprocess"),
                              ("pair-merge (generic)", "merge path: team lane owns merged positions"),
                              ("xor prefix", "XOR prefix over chunks"),
                              ("select", "select the (h+1)-th live position"),
                              ("walk", "for (int t = 1; t < SR; ++t)"),
                              ("output", "rows are dead: reuse them")])
SORT = marks("mf_blocksort.cuh", [("sort: key network", "struct KeyU32 {"),
                                  ("sort: rank search", "constexpr uint32_t cpad5"),
                                  ("sort: team key merge + scatter", "void team_sort_keys(")])


def phase(table, ln, default):
    name = default
    for start, n in table:
        if ln >= start:
            name = n
    return name


rep, kern, skip = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "0"
sys.argv = ["x", rep, kern, "100000", skip]
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    runpy.run_path(os.path.join(ROOT, "scripts", "ncu_lines.py"), run_name="__main__")
ph = {}
for line in buf.getvalue().splitlines()[1:]:
    p = line.split()
    f, ln = p[0].rsplit(":", 1)
    ln = int(ln)
    st, ins = float(p[1]), float(p[2])
    if f.startswith("mf_medium"):
        key = phase(MED, ln, "kernel preamble / helpers")
    elif f.startswith("mf_blocksort"):
        key = phase(SORT, ln, "sort: merge-path helpers")
    elif f.startswith("mf_sortnet"):
        key = "sort: register network"
    elif f.startswith("sm_30"):
        key = "sort: shuffles"
    else:
        key = "intrinsics (" + f + ")"
    a = ph.setdefault(key, [0.0, 0.0])
    a[0] += st
    a[1] += ins
print(f"{'phase':34s} {'stall%':>7s} {'inst%':>7s}")
for k, v in sorted(ph.items(), key=lambda x: -x[1][1]):
    print(f"{k:34s} {v[0]:7.1f} {v[1]:7.1f}")
