import subprocess,sys,runpy
sys.argv=["x",sys.argv[1],sys.argv[2],"100000",sys.argv[3]]
import io,contextlib
buf=io.StringIO()
with contextlib.redirect_stdout(buf):
    runpy.run_path("scripts/ncu_lines.py",run_name="__main__")
ph={}
for l in buf.getvalue().splitlines()[1:]:
    p=l.split()
    f,ln=p[0].rsplit(":",1); ln=int(ln)
    st,ins=float(p[1]),float(p[2])
    if f.startswith("mf_medium"):
        key="med:"+("pre" if ln<130 else "zero" if ln<142 else "merge" if ln<191 else "prefix" if ln<203 else "walk" if ln<270 else "out")
    else: key=f
    a=ph.setdefault(key,[0,0]); a[0]+=st; a[1]+=ins
for k,v in sorted(ph.items(),key=lambda x:-x[1][0]): print(f"{k:30s} stall {v[0]:5.1f} inst {v[1]:5.1f}")
