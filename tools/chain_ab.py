"""A/B of the backward-chain consumer schedules in one process (diagnostic):
alternates IMB_BW_OLD_TAIL off/on so clock drift affects both alike."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_13887_b200 import capi  # noqa: E402

ctx = capi.Context(0)
f = ctx.lib.im_bench_backward_chain
f.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(C.c_double)]
for n in (1024, 2048, 4096):
    res = {"new": [], "old": []}
    for rep in range(3):
        for v in ("new", "old"):
            if v == "old":
                os.environ["IMB_BW_OLD_TAIL"] = "1"
            else:
                os.environ.pop("IMB_BW_OLD_TAIL", None)
            ms = C.c_double()
            assert f(ctx.h, n, 5, C.byref(ms)) == 0
            res[v].append(ms.value)
    el = n * (n - 1) / 2
    print(n, {k: f"{min(v) * 1e-3 * 1.965e9 / el:.2f} cyc/el" for k, v in res.items()}, flush=True)
