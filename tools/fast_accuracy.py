"""Accuracy of the FP64 fast volume update against the bit-exact path on the
cfg workloads' real control sets (diagnostic; GPU).

    python tools/fast_accuracy.py [cfg2 cfg3 cfg4] [--nodes N]

For each level: max |dV_fast - dV_exact| / max |dV_exact| over a random node
sample, and the amplification sum|alpha| / max|dV| that bounds how per-pair
rounding differences grow.
"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2107_13887_b200 import capi, workloads as W  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs", nargs="*", default=["cfg2", "cfg3", "cfg4"])
    ap.add_argument("--nodes", type=int, default=400000)
    args = ap.parse_args()
    ctx = capi.Context(0)
    rng = np.random.default_rng(0)
    for name in args.cfgs:
        w = W.CONFIGS[name](1.0)
        z = np.load(f"devcache/{name}_controls.npz")
        n = len(w.nodes)
        pick = np.sort(rng.choice(n, min(args.nodes, n), replace=False))
        nodes = np.ascontiguousarray(w.nodes[pick])
        # distances only matter through psi; use 0 so psi == 1 (worst case:
        # every sampled node active with full weight)
        dist = np.zeros(len(nodes))
        D = np.inf
        for l in range(int(z["n"])):
            c, a = z[f"c{l}"], z[f"a{l}"]
            i1, v1 = ctx.update_volume(nodes, dist, c, a, D, 0, "c2", w.R, capi.FP64)
            v1 = v1.copy()
            i2, v2 = ctx.update_volume(nodes, dist, c, a, D, 0, "c2", w.R, capi.EXACT)
            assert np.array_equal(i1, i2)
            scale = np.abs(v2).max()
            err = np.abs(v1 - v2).max() / scale if scale > 0 else 0.0
            amp = np.abs(a).sum(axis=0).max() / scale if scale > 0 else 0.0
            print(f"{name} level {l}: n_ctrl {len(c)}, max|dV| {scale:.3e}, "
                  f"fast-vs-exact rel {err:.3e}, sum|alpha|/max|dV| {amp:.3e}", flush=True)


if __name__ == "__main__":
    main()
