"""Compare two TT output dumps (tools/tt_dump.py) from two library builds:
rel-L2 and max|d|/max|ref| per scene and amplitude."""
import numpy as np
a = np.load("gpurun_out/tt_old.npz"); b = np.load("gpurun_out/tt_new.npz")
for k in a.files:
    x, y = a[k].astype(np.float64), b[k].astype(np.float64)
    print(k, "rel-L2 %.2e  max %.2e" % (np.linalg.norm(x - y) / np.linalg.norm(x), np.abs(x - y).max() / np.abs(x).max()))
