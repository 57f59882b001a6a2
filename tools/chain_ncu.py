"""One backward-substitution chain launch (k_backward_t, 3 axes) of size n
through im_bench_backward_chain, for ncu captures: python tools/chain_ncu.py 4096"""
import ctypes as C
import sys

sys.path.insert(0, ".")
from paper_2107_13887_b200 import capi

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ctx = capi.Context(0)
f = ctx.lib.im_bench_backward_chain
f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double)]
ms = C.c_double()
assert f(ctx.h, n, 3, C.byref(ms)) == 0, ctx.lib.im_last_error(ctx.h)
el = n * (n - 1) / 2
print(f"n={n}: {ms.value:.3f} ms, {ms.value * 1e-3 * 1.965e9 / el:.2f} cycles/element")
