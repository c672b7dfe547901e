import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_19951_b200 as rb
from paper_2605_19951_b200 import mesh3d, _lib
m6, s6, _, _ = mesh3d._local_matrices(1.0, mesh3d.MU0)
lib = _lib.load()
for P in (1, 6, 1000):
    ml = np.ascontiguousarray(np.tile(m6, (P // 6 + 1, 1, 1))[:P])
    sl = np.ascontiguousarray(np.tile(s6, (P // 6 + 1, 1, 1))[:P])
    mm = np.zeros(P)
    out = np.zeros(1)
    rc = lib.rba_spectral_bound(P, ml.ctypes.data, sl.ctypes.data, mm.ctypes.data, out.ctypes.data)
    print(P, rc, out[0])
