"""Host-buffer pipeline timing per k and pipeline chunk size (pinned buffers, c2 signal)."""
import ctypes as C
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1406_1717_b200 as mf  # noqa: E402
from paper_1406_1717_b200 import _native as N  # noqa: E402

n = 1 << 26
x = mf.generate_device("uniform_f32", 2, n).cpu().pin_memory()
y = torch.empty(n, dtype=torch.float32).pin_memory()
ctx = mf.Context.get(0)
L = N.lib()
ks = [int(a) for a in sys.argv[1:]] or [3, 31, 255, 1023]
for chunk in (1 << 21, 1 << 22, 1 << 23, 1 << 24, 1 << 25):
    ctx.pipeline_chunk(chunk)
    row = []
    for k in ks:
        ylen = C.c_size_t()
        ts = []
        for _ in range(4):
            t = time.perf_counter()
            st = L.mf_median_filter(ctx.handle, N.MF_F32, x.data_ptr(), n, k, y.data_ptr(), n, C.byref(ylen))
            ts.append(time.perf_counter() - t)
            assert st == 0
        row.append(f"k={k}: {1e3 * sorted(ts)[1]:.2f} ms")
    print(f"chunk 2^{chunk.bit_length() - 1}: " + "  ".join(row), flush=True)
ctx.pipeline_chunk(0)
