"""Event timeline of a Python replica of the host pipeline (k from argv, 16 chunks)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1406_1717_b200 as mf  # noqa: E402

n = 1 << 26
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
nch = int(sys.argv[2]) if len(sys.argv) > 2 else 16
compute = (sys.argv[3] != "0") if len(sys.argv) > 3 else True
hx = mf.generate_device("uniform_f32", 2, n).cpu().pin_memory()
hy = torch.empty(n, dtype=torch.float32).pin_memory()
cs = n // nch
S = 4
dx = [torch.empty(cs + k - 1, device="cuda") for _ in range(S)]
dy = [torch.empty(cs, device="cuda") for _ in range(S)]
s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def run():
    marks = []
    ev_out = [None] * S
    for c in range(nch):
        sl = c % S
        o0 = c * cs
        no = min(cs, n - k + 1 - o0)
        m = [E() for _ in range(6)]
        with torch.cuda.stream(s_in):
            if ev_out[sl] is not None:
                s_in.wait_event(ev_out[sl])
            m[0].record(s_in)
            dx[sl][:no + k - 1].copy_(hx[o0:o0 + no + k - 1], non_blocking=True)
            m[1].record(s_in)
        with torch.cuda.stream(s_c):
            s_c.wait_event(m[1])
            m[2].record(s_c)
            if compute:
                mf.median_filter_device(dx[sl][:no + k - 1], k, out=dy[sl])
            m[3].record(s_c)
        with torch.cuda.stream(s_out):
            s_out.wait_event(m[3])
            m[4].record(s_out)
            hy[o0:o0 + no].copy_(dy[sl][:no], non_blocking=True)
            m[5].record(s_out)
        ev_out[sl] = m[5]
        marks.append(m)
    torch.cuda.synchronize()
    return marks


run()
marks = run()
t0 = marks[0][0]
print(f"k={k} chunks={nch} compute={compute}: total {t0.elapsed_time(marks[-1][5]):.2f} ms")
for c, m in enumerate(marks):
    print(f"chunk {c:2d}: h2d {t0.elapsed_time(m[0]):6.2f}-{t0.elapsed_time(m[1]):6.2f}  "
          f"comp {t0.elapsed_time(m[2]):6.2f}-{t0.elapsed_time(m[3]):6.2f}  "
          f"d2h {t0.elapsed_time(m[4]):6.2f}-{t0.elapsed_time(m[5]):6.2f}")
