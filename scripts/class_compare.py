"""Time each kernel class on the config-2 signal for a list of k (device-resident)."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1406_1717_b200 as mf
from paper_1406_1717_b200 import _native as N
x = mf.generate_device("uniform_f32", 2, 1 << 26)
ctx = mf.Context.get(0)
for k in [int(a) for a in sys.argv[1:]]:
    res = {}
    for cls, name in ((N.MF_CLASS_SMALL, "S"), (N.MF_CLASS_MEDIUM, "M"), (N.MF_CLASS_LARGE, "L")):
        if (cls == N.MF_CLASS_SMALL and k > 31) or (cls == N.MF_CLASS_MEDIUM and k > 1023):
            continue
        ctx.force_class(cls)
        out = torch.empty(x.numel() - k + 1, dtype=x.dtype, device=x.device)
        for _ in range(3):
            mf.median_filter_device(x, k, out=out, ctx=ctx)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(5):
            mf.median_filter_device(x, k, out=out, ctx=ctx)
        b.record()
        torch.cuda.synchronize()
        res[name] = round(a.elapsed_time(b) / 5, 3)
    ctx.force_class(N.MF_CLASS_AUTO)
    print(k, res, flush=True)
