import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1406_1717_b200 as mf, torch
from oracle_lib import Oracle
o = Oracle()
for k in (1, 3, 31, 33, 101, 255, 1023, 2049):
    for dt in (np.int32, np.int64, np.float32, np.float64):
        x = (np.random.default_rng(k).standard_normal(5 * k + 3) * 100).astype(dt)
        try:
            y = mf.median_filter(x, k)
            ok = np.array_equal(y, o.median_filter(x, k))
        except Exception as e:
            ok = repr(e)
            try:
                torch.cuda.synchronize()
            except Exception as e2:
                ok += " | " + repr(e2)
            print(k, np.dtype(dt).name, ok, flush=True)
            sys.exit(0)
        print(k, np.dtype(dt).name, ok, flush=True)
