import ctypes as C, sys
sys.path.insert(0, ".")
from paper_2107_13887_b200 import capi
ctx = capi.Context(0)
f = ctx.lib.im_debug_backward_phases
f.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_double)]
for n in (1024, 4096):
    out = (C.c_double * 4)()
    f(ctx.h, n, out)
    el = n * (n - 1) / 2
    print(n, "wait/A/issue/B cycles per element:", [round(v / el, 2) for v in out])
