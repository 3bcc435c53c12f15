import ctypes, sys
sys.path.insert(0, ".")
from paper_2307_11248_b200 import _lib
L = _lib.lib()
for k in range(5):
    v = ctypes.c_double(0)
    _lib.check(L.qapb_probe_int_peak(0, k, ctypes.byref(v)))
    print(k, v.value / 1e12)
