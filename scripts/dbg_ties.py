"""Tie-heavy parity probe: values drawn from {0, 1, type max} (max ties the padding key)."""
import sys
import numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1406_1717_b200 as mf  # noqa: E402
from paper_1406_1717_b200 import _native as N  # noqa: E402
from oracle_lib import Oracle  # noqa: E402
orc = Oracle()
ctx = mf.Context.get(0)
rng = np.random.default_rng(0)
fails = {}
only_cls = int(sys.argv[1]) if len(sys.argv) > 1 else None
only_dt = sys.argv[2] if len(sys.argv) > 2 else None
for it in range(400):
    kk = int(rng.choice([3, 31, 33, 63, 65, 127, 255, 1023]))
    n = int(rng.integers(kk, 5 * kk))
    for dt in (np.int32, np.int64):
        if only_dt and dt.__name__ != only_dt:
            continue
        vals = np.array([0, 1, np.iinfo(dt).max], dtype=dt)
        xx = vals[rng.integers(0, 3, size=n)]
        w = orc.median_filter(xx, kk)
        for cls in (N.MF_CLASS_SMALL, N.MF_CLASS_MEDIUM):
            if (cls == N.MF_CLASS_SMALL and kk > 31) or (only_cls is not None and cls != only_cls):
                continue
            ctx.force_class(cls)
            g = mf.median_filter(xx, kk, ctx=ctx)
            if not np.array_equal(g, w):
                key = (cls, kk, dt.__name__)
                fails[key] = fails.get(key, 0) + 1
                if fails[key] == 1:
                    bad = np.nonzero(g != w)[0]
                    print(key, "n", n, "bad", bad[:8], "got", g[bad[:3]], "want", w[bad[:3]], flush=True)
ctx.force_class(N.MF_CLASS_AUTO)
print("fails", fails)
