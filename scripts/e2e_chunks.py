"""e2e (pinned host buffers, mf_median_filter) of the config-2 sweep at several pipeline chunk sizes."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1406_1717_b200 as mf  # noqa: E402
from paper_1406_1717_b200 import _native as N  # noqa: E402

ctx = mf.Context(0)
L = N.lib()
x = mf.generate_device("uniform_f32", 2, 1 << 26).cpu().pin_memory()
ks = (3, 31, 255, 1023)
ys = {k: torch.empty(x.numel() - k + 1, dtype=torch.float32).pin_memory() for k in ks}
for chunk in [int(a) for a in sys.argv[1:]] or [1 << 22, 1 << 23, 1 << 24, 1 << 25]:
    ctx.pipeline_chunk(chunk)
    def step():
        for k in ks:
            ylen = C.c_size_t()
            assert L.mf_median_filter(ctx.handle, N.MF_F32, C.c_void_p(x.data_ptr()), x.numel(), k,
                                      C.c_void_p(ys[k].data_ptr()), ys[k].numel(), C.byref(ylen)) == 0
    step()
    t = time.perf_counter()
    for _ in range(5):
        step()
    dt = (time.perf_counter() - t) / 5
    outs = sum(x.numel() - k + 1 for k in ks)
    print(f"chunk {chunk}: {dt * 1e3:.2f} ms/step, e2e {outs / dt:.4g} samples/s", flush=True)
