import sys, numpy as np
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
bad = [k for k in a.files if not np.array_equal(a[k], b[k])]
print("identical" if not bad else f"DIFFER: {bad}")
for k in bad[:4]:
    x, y = a[k].astype(float), b[k].astype(float)
    print(k, np.max(np.abs(x - y)))
