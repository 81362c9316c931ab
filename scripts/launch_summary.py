"""Per-kernel totals from an ncu --csv launch list: python scripts/launch_summary.py FILE [calls]"""
import csv
import sys

calls = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
agg = {}
for r in rows:
    kn = r[4].split("(")[0].replace("void ", "")[:44]
    agg.setdefault(kn, {}).setdefault(r[12], [0.0, 0])
    a = agg[kn][r[12]]
    a[0] += float(r[14].replace(",", ""))
    a[1] += 1
tot = sum(v["gpu__time_duration.sum"][0] for v in agg.values() if "gpu__time_duration.sum" in v)
print(f"{'kernel':44s} {'launches':>8s} {'ms/call':>9s} {'share':>6s} {'dram GB/call':>12s} {'Minst/call':>10s}")
for kn, m in sorted(agg.items(), key=lambda kv: -kv[1].get("gpu__time_duration.sum", [0])[0]):
    t = m.get("gpu__time_duration.sum", [0, 0])
    db = (m.get("dram__bytes_read.sum", [0])[0] + m.get("dram__bytes_write.sum", [0])[0])
    unit = 1e9
    print(f"{kn:44s} {t[1]:8d} {t[0] / 1e6 / calls:9.3f} {t[0] / tot:6.1%} {db / unit / calls:12.3f} "
          f"{m.get('smsp__inst_executed.sum', [0])[0] / 1e6 / calls:10.1f}")
