"""Run the golden small cases one by one, printing each before it runs (for compute-sanitizer)."""
import os
import sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1406_1717_b200 as mf  # noqa: E402

z = np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/small_cases.npz"))
n = len([f for f in z.files if f.endswith("_x")])
lo = int(sys.argv[1]) if len(sys.argv) > 1 else 0
for i in range(lo, n):
    x, k, y = z[f"c{i}_x"], int(z[f"c{i}_k"]), z[f"c{i}_y"]
    print("case", i, "k", k, x.dtype, x.size, flush=True)
    got = mf.median_filter(x, k)
    vb = np.int32 if y.itemsize == 4 else np.int64
    if not np.array_equal(got.view(vb), y.view(vb)):
        print("MISMATCH", i, flush=True)
        break
print("done")
