import sys, numpy as np
sys.path.insert(0, '.')
import paper_1406_1717_b200 as mf
k = int(sys.argv[1]); dt = np.dtype(sys.argv[2])
x = (np.random.default_rng(k).standard_normal(5 * k + 3) * 100).astype(dt)
print(mf.median_filter(x, k)[:4])
