"""Culling efficiency of the volume kernels (diagnostic; GPU): per level,
the in-support pair fraction (exact count) against the fraction of pairs the
exact kernel evaluates (IMB_COUNT_PAIRS counter).

    IMB_COUNT_PAIRS=1 python tools/culling_stats.py cfg2 [cfg3 ...]
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_13887_b200 import capi, workloads as W  # noqa: E402


def main():
    ctx = capi.Context(0)
    for name in sys.argv[1:] or ["cfg2"]:
        w = W.CONFIGS[name](1.0)
        z = np.load(f"devcache/{name}_controls.npz")
        plan = capi.VolumePlan(ctx, w.nodes, w.dim, w.surface,
                               cutoff=w.D if math.isfinite(w.D) else -1.0)
        n = int(z["n"])
        for l in range(n):
            plan.set_level(l, z[f"c{l}"], z[f"a{l}"], w.D, w.psi_kind, "c2", w.R, capi.EXACT)
        for l in range(n):
            i, t = plan.count_support(l, "c2", w.R)
            print(f"{name} level {l}: n_ctrl {len(z[f'c{l}'])}, in support {i / t:.4f}", flush=True)
        plan.run_steps(1, "c2", w.R, capi.EXACT, flush_l2=False)


if __name__ == "__main__":
    main()
