"""Registers / shared / local memory per kernel of the built library:
python scripts/res_usage.py [REGEX] [LIB]"""
import re
import subprocess
import sys

pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_1406_1717_b200/libmedfilt_b200.so"
out = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout.splitlines()
name = None
for line in out:
    m = re.search(r"Function (\S+):", line)
    if m:
        name = m.group(1)
        continue
    if name and "REG:" in line:
        dem = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        dem = re.sub(r"\(mf::Geom.*", "", dem).replace("void ", "")
        if pat.search(dem):
            f = dict(re.findall(r"(\w+):(\d+)", line))
            print(f"{dem:55s} REG {f.get('REG'):>4s} STACK {f.get('STACK'):>3s} LOCAL {f.get('LOCAL'):>3s}")
        name = None
