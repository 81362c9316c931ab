"""One filter call per k on the config-2 signal (for ncu): python scripts/profile_c2.py K [K ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1406_1717_b200 as mf  # noqa: E402

cfg = os.environ.get("CFG", "c2")
ks = [int(a) for a in sys.argv[1:]] or [3, 31, 255, 1023]
if cfg == "c2":
    x = mf.generate_device("uniform_f32", 2, 1 << 26)
elif cfg == "c3":
    x = mf.generate_device("mod_i32", 3, 4096 * 65536, mod=16).view(4096, 65536)
elif cfg == "c1":
    x = mf.generate_device("uniform_f64", 1, 1_000_000)
elif cfg == "c4":
    x = torch.from_numpy(mf.generate_trend_f64(4, 1 << 27)).cuda()
else:
    x = mf.generate_device("uniform_f32", 5, 1 << 30)
for k in ks:
    for _ in range(2):
        if x.dim() == 2:
            y = mf.median_filter_rows_device(x, k)
        else:
            y = mf.median_filter_device(x, k)
torch.cuda.synchronize()
print("ok", ks)
