import ctypes as C, sys
sys.path.insert(0, '.')
from paper_2602_00395_b200 import _lib
L = _lib.lib()
for lo, hi in [(-760,-745),(-745,-709.8),(-709.8,-709.0),(-709,-700),(-700,-30),(-30,0),(0,1e-3),(0,10),(0,700)]:
    b = C.c_int64(-1)
    _lib.check(L.sgtr_check_fast_exp(1<<22, lo, hi, 7, C.byref(b)))
    print(lo, hi, b.value)
