"""Small filter calls of every kernel class for compute-sanitizer (racecheck, synccheck,
memcheck, initcheck): python scripts/sanitize_cases.py.  Each call is checked against the
oracle so a run also proves the sanitized launches computed the right thing."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1406_1717_b200 as mf  # noqa: E402
from paper_1406_1717_b200 import _native as N  # noqa: E402
from oracle_lib import Oracle  # noqa: E402  (checker only)

orc = Oracle()
rng = np.random.default_rng(1)
ctx = mf.Context(0)
# (class, dtype, k, n): T (k = 3), S (k <= 31 and the 64-bit-mask range), M (R = 2..32,
# 1 and 2 warps per pair, key-only and payload sorts), L (multi-kernel pipeline)
CASES = [
    (N.MF_CLASS_AUTO, np.float32, 3, 40_003),
    (N.MF_CLASS_AUTO, np.int32, 31, 40_003),
    (N.MF_CLASS_AUTO, np.float64, 31, 20_003),
    (N.MF_CLASS_AUTO, np.float32, 45, 40_003),
    (N.MF_CLASS_AUTO, np.float32, 255, 60_001),
    (N.MF_CLASS_AUTO, np.int64, 101, 30_001),
    (N.MF_CLASS_AUTO, np.float32, 511, 60_001),
    (N.MF_CLASS_AUTO, np.float32, 1023, 60_001),
    (N.MF_CLASS_AUTO, np.float64, 1023, 30_001),
    (N.MF_CLASS_AUTO, np.float32, 2049, 30_001),
    (N.MF_CLASS_AUTO, np.float64, 10001, 50_001),
]
only = sys.argv[1:]
for i, (cls, dt, k, n) in enumerate(CASES):
    if only and str(i) not in only:
        continue
    ctx.force_class(cls)
    x = (rng.standard_normal(n) * 50).astype(dt) if dt in (np.float32, np.float64) else \
        rng.integers(-40, 40, size=n).astype(dt)
    got = mf.median_filter_device(torch.from_numpy(x).cuda(), k, ctx=ctx).cpu().numpy()
    want = orc.median_filter(x, k)
    vb = np.int32 if got.itemsize == 4 else np.int64
    ok = np.array_equal(got.view(vb), want.view(vb))
    print(f"case {i}: class {mf.kernel_class(dt, k)} {np.dtype(dt).name} k={k} n={n}: {'ok' if ok else 'MISMATCH'}",
          flush=True)
    assert ok
rows = rng.integers(0, 16, size=(6, 3000)).astype(np.int32)
got = mf.median_filter_rows_device(torch.from_numpy(rows).cuda(), 255, ctx=ctx).cpu().numpy()
assert all(np.array_equal(got[r], orc.median_filter(rows[r], 255)) for r in range(6))
print("rows ok")
