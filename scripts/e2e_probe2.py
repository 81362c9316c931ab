"""Python replica of the host pipeline: copies only vs copies + kernels (c2 signal, k=3)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1406_1717_b200 as mf  # noqa: E402

n = 1 << 26
k = int(sys.argv[1]) if len(sys.argv) > 1 else 3
hx = mf.generate_device("uniform_f32", 2, n).cpu().pin_memory()
hy = torch.empty(n, dtype=torch.float32).pin_memory()
nch = 16
cs = n // nch
dx = [torch.empty(cs + k - 1, device="cuda") for _ in range(3)]
dy = [torch.empty(cs, device="cuda") for _ in range(3)]
s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
ev_in = [torch.cuda.Event() for _ in range(3)]
ev_c = [torch.cuda.Event() for _ in range(3)]
ev_out = [torch.cuda.Event() for _ in range(3)]


def run(compute, sync_each=True):
    for c in range(nch):
        sl = c % 3
        o0 = c * cs
        no = min(cs, n - k + 1 - o0)
        with torch.cuda.stream(s_in):
            if c >= 3:
                s_in.wait_event(ev_out[sl])
            dx[sl][:no + k - 1].copy_(hx[o0:o0 + no + k - 1], non_blocking=True)
            ev_in[sl].record(s_in)
        with torch.cuda.stream(s_c):
            s_c.wait_event(ev_in[sl])
            if compute:
                mf.median_filter_device(dx[sl][:no + k - 1], k, out=dy[sl])
            ev_c[sl].record(s_c)
        with torch.cuda.stream(s_out):
            s_out.wait_event(ev_c[sl])
            hy[o0:o0 + no].copy_(dy[sl][:no], non_blocking=True)
            ev_out[sl].record(s_out)
    if sync_each:
        torch.cuda.synchronize()


for compute in (False, True):
    run(compute)
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        run(compute)
        ts.append(time.perf_counter() - t)
    print(f"k={k} compute={compute}: {1e3 * sorted(ts)[2]:.2f} ms per call", flush=True)
