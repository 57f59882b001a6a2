import ctypes as C, sys
sys.path.insert(0, ".")
from paper_2107_13887_b200 import capi
ctx = capi.Context(0)
f = ctx.lib.im_bench_backward_chain
f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double)]
for n in (64, 256, 1024, 2048, 4096):
    ms = C.c_double()
    assert f(ctx.h, n, 5, C.byref(ms)) == 0, ctx.lib.im_last_error(ctx.h)
    el = n * (n - 1) / 2
    print(f"n={n}: {ms.value:.3f} ms, {ms.value*1e6/el:.2f} ns/element, {ms.value*1e-3*1.96e9/el:.2f} cycles/element", flush=True)
