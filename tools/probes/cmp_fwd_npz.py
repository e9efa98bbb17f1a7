"""Element mismatches between two cmp_fwd_builds.py npz files."""
import numpy as np, sys
a, b = np.load(sys.argv[1]), np.load(sys.argv[2])
for k in a.files:
    d = (a[k] != b[k])
    print(k, d.sum(), a[k].ravel()[:24] if k.startswith('b') else '', b[k].ravel()[:24] if k.startswith('b') else '')
