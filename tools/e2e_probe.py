"""Breakdown of the e2e im_update_volume call on cfg2 (diagnostic).

    IMB_TRACE=1 python tools/e2e_probe.py [devcache/cfg2_controls.npz]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_13887_b200 import capi, workloads as W  # noqa: E402


def main():
    import torch

    cache = sys.argv[1] if len(sys.argv) > 1 else "devcache/cfg2_controls.npz"
    w = W.cfg2()
    if os.path.exists(cache):
        z = np.load(cache)
        levels = [(z[f"c{l}"], z[f"a{l}"]) for l in range(int(z["n"]))]
    else:  # the reference's own cfg2 selection, seeded alphas (cost is alpha-independent)
        z = np.load(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                                 "cfg2_reference_selection.npz"))
        rng = np.random.default_rng(0)
        pos = w.nodes[w.surface]
        levels = [(pos[z[f"idx{l}"]], rng.standard_normal((len(z[f"idx{l}"]), 3)) * 1e-3)
                  for l in range(3)]
        for _, a in levels:
            a[:, 2] = 0.0
    ctx = capi.Context(0)
    plan = capi.VolumePlan(ctx, w.nodes, 2, w.surface, cutoff=w.D)
    d = plan.distances()
    nodes = w.nodes
    # raw copy bandwidths
    x = torch.from_numpy(nodes)
    for pin in (False, True):
        src = x.pin_memory() if pin else x
        dst = torch.empty_like(x, device="cuda")
        dst.copy_(src)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            dst.copy_(src)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 5
        print(f"h2d pinned={pin}: {nodes.nbytes / dt / 1e9:.1f} GB/s", file=sys.stderr)
        back = torch.empty_like(x, pin_memory=pin)
        back.copy_(dst)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(5):
            back.copy_(dst)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t) / 5
        print(f"d2h pinned={pin}: {nodes.nbytes / dt / 1e9:.1f} GB/s", file=sys.stderr)
    import ctypes
    rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
    if rt is not None:
        src = torch.from_numpy(nodes)
        dst = torch.empty_like(src, device="cuda")
        for it in range(3):
            t = time.perf_counter()
            rc = rt.cudaHostRegister(ctypes.c_void_p(nodes.ctypes.data), ctypes.c_size_t(nodes.nbytes), 0)
            t1 = time.perf_counter()
            dst.copy_(src, non_blocking=True)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            rt.cudaHostUnregister(ctypes.c_void_p(nodes.ctypes.data))
            t3 = time.perf_counter()
            print(f"register rc={rc} {1e3*(t1-t):.3f} ms, copy {1e3*(t2-t1):.3f} ms, "
                  f"unregister {1e3*(t3-t2):.3f} ms", file=sys.stderr)
    t = time.perf_counter()
    for _ in range(5):
        np.zeros((len(nodes), 3))[:] = 1.0
    print(f"np.zeros+touch 24MB: {(time.perf_counter() - t) / 5 * 1e3:.2f} ms", file=sys.stderr)
    pinned = os.environ.get("PROBE_PINNED") == "1"
    prec = capi.EXACT if os.environ.get("PROBE_EXACT") == "1" else capi.FP64
    out = None
    if pinned:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory().numpy()
        nodes, d = pin(nodes), pin(d)
        out = (torch.empty(len(nodes), dtype=torch.int64, pin_memory=True).numpy().view(np.uint64),
               torch.empty((len(nodes), 3), dtype=torch.float64, pin_memory=True).numpy())
    for it in range(3):
        t0 = time.perf_counter()
        for c, a in levels:
            t = time.perf_counter()
            idx, val = ctx.update_volume(nodes, d, c, a, w.D, 0, "c2", w.R, prec, out=out)
            print(f"  level nc={len(c)}: {(time.perf_counter() - t) * 1e3:.2f} ms "
                  f"(kernel {ctx.last_device_ms:.2f} ms, {len(idx)} entries)", file=sys.stderr)
        print(f"step {it}: {(time.perf_counter() - t0) * 1e3:.2f} ms", file=sys.stderr)


if __name__ == "__main__":
    main()
