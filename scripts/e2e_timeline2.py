"""Python replica of the host pipeline with H2D issued AHEAD chunks before the kernel/D2H
of the current chunk (issue order matters if copies share in-order hardware queues):
python scripts/e2e_timeline2.py K NCHUNKS AHEAD"""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1406_1717_b200 as mf  # noqa: E402

n = 1 << 26
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
nch = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ahead = int(sys.argv[3]) if len(sys.argv) > 3 else 1
hx = mf.generate_device("uniform_f32", 2, n).cpu().pin_memory()
hy = torch.empty(n, dtype=torch.float32).pin_memory()
cs = n // nch
S = 4
dx = [torch.empty(cs + k - 1, device="cuda") for _ in range(S)]
dy = [torch.empty(cs, device="cuda") for _ in range(S)]
s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731


def run():
    ev_out = [None] * S
    ev_in = [None] * nch
    t0, t1 = E(), E()
    t0.record(s_in)

    def h2d(c):
        sl = c % S
        o0 = c * cs
        no = min(cs, n - k + 1 - o0)
        with torch.cuda.stream(s_in):
            if ev_out[sl] is not None:
                s_in.wait_event(ev_out[sl])
            dx[sl][:no + k - 1].copy_(hx[o0:o0 + no + k - 1], non_blocking=True)
            ev_in[c] = E()
            ev_in[c].record(s_in)
    for c in range(min(ahead, nch)):
        h2d(c)
    for c in range(nch):
        if c + ahead < nch and (c + ahead) - S < c:  # slot of c+ahead freed by an earlier chunk
            h2d(c + ahead)
        sl = c % S
        o0 = c * cs
        no = min(cs, n - k + 1 - o0)
        with torch.cuda.stream(s_c):
            s_c.wait_event(ev_in[c])
            mf.median_filter_device(dx[sl][:no + k - 1], k, out=dy[sl])
            ed = E()
            ed.record(s_c)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ed)
            hy[o0:o0 + no].copy_(dy[sl][:no], non_blocking=True)
            eo = E()
            eo.record(s_out)
        ev_out[sl] = eo
    t1.record(s_out)
    torch.cuda.synchronize()
    return t0.elapsed_time(t1)


run()
ts = sorted(run() for _ in range(5))
print(f"k={k} chunks={nch} ahead={ahead}: total {ts[2]:.2f} ms")
