import numpy as np, sys
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
print("keys", len(a.files), "differ:", bad[:20])
for k in bad[:5]:
    x, y = a[k].astype(np.float64), b[k].astype(np.float64)
    print(k, x.shape, y.shape, np.max(np.abs(x - y)) if x.shape == y.shape else "shape")
