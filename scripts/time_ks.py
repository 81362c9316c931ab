"""Device time per k on the config-2 (or CFG=c4/c5) signal (median of 3 x 10 launches): python scripts/time_ks.py K..."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1406_1717_b200 as mf  # noqa: E402

cfg = os.environ.get("CFG", "c2")
if cfg == "c2":
    x = mf.generate_device("uniform_f32", 2, 1 << 26)
elif cfg == "c1":
    x = mf.generate_device("uniform_f64", 1, 1_000_000)
elif cfg == "c4":
    x = torch.from_numpy(mf.generate_trend_f64(4, 1 << 27)).cuda()
else:  # c5
    x = mf.generate_device("uniform_f32", 5, 1 << 30)
out = None
res = {}
for k in [int(a) for a in sys.argv[1:]] or [3, 31, 255, 1023]:
    for _ in range(3):
        out = mf.median_filter_device(x, k, out=out)
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            mf.median_filter_device(x, k, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) / 10)
    res[k] = round(sorted(ts)[1], 4)
print(os.environ.get("MF_B200_LIB", "default"), res, flush=True)
