"""Host-buffer pipeline per call (ms) by k and largest chunk, next to the bare PCIe ceiling
(H2D of the input and D2H of the output at once, no kernels): python scripts/e2e_sweep.py"""
import ctypes as C
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1406_1717_b200 as mf  # noqa: E402
from paper_1406_1717_b200 import _native as N  # noqa: E402
from paper_1406_1717_b200.filter import _DTYPES, _check  # noqa: E402

n = 1 << 26
xd = mf.generate_device("uniform_f32", 2, n)
hx = xd.cpu().pin_memory()
hy = torch.empty(n, dtype=torch.float32).pin_memory()
ctx = mf.Context.get(0)
L = N.lib()
x, y = hx.numpy(), hy.numpy()

# ceiling: both directions at once
d1 = torch.empty(n, device="cuda")
d2 = torch.empty(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def both():
    with torch.cuda.stream(s1):
        d1.copy_(hx, non_blocking=True)
    with torch.cuda.stream(s2):
        hy.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
both()
ts = []
for _ in range(5):
    t = time.perf_counter(); both(); ts.append(time.perf_counter() - t)
print("ceiling both directions ms", round(sorted(ts)[2] * 1e3, 3), flush=True)

def call(k):
    ylen = C.c_size_t()
    _check(L.mf_median_filter(ctx.handle, _DTYPES[x.dtype], x.ctypes.data, x.size, k, y.ctypes.data, y.size,
                              C.byref(ylen)))
for chunk in [int(a) for a in sys.argv[1:]] or [1 << 21, 1 << 22, 1 << 23, 1 << 24, 1 << 25]:
    ctx.pipeline_chunk(chunk)
    res = {}
    for k in (3, 31, 255, 1023):
        call(k)
        ts = []
        for _ in range(5):
            t = time.perf_counter(); call(k); ts.append(time.perf_counter() - t)
        res[k] = round(sorted(ts)[2] * 1e3, 3)
    print("chunk", chunk, res, "sum", round(sum(res.values()), 3), flush=True)
