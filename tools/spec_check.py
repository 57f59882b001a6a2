"""Speculative vs sequential exact greedy on the device: identical results,
wall time and predictor statistics per case.  Run on the GPU box:
    python tools/spec_check.py [case ...]
cases: cfg1, cfg2l01 (cfg2 levels 0-1), cfg2 (3 levels), cfg3p / cfg4p
(300-point prefixes), cfg3l0, cfg4l01 (capped 5000-point levels)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2107_13887_b200 import capi, workloads as W  # noqa: E402


def case(name):
    if name.startswith("cfg1"):
        w = W.cfg1()
        return w.nodes[w.surface], w.displacement, w.tol, w.levels, w.cap, w.R
    if name.startswith("cfg2"):
        w = W.cfg2()
        lv = 2 if name == "cfg2l01" else w.levels
        return w.nodes[w.surface], w.displacement, w.tol, lv, w.cap, w.R
    pos, disp, R, tol, levels = W.wing_surface_case(name[:4])
    if name.endswith("p"):
        return pos, disp, tol, 2, 300, R
    if name == "cfg3l0":
        return pos, disp, tol, 1, 5000, R
    if name == "cfg4l01":
        return pos, disp, tol, 2, 5000, R
    return pos, disp, tol, levels, 5000, R


def run(ctx, args, spec):
    os.environ["IMB_SPEC"] = "1" if spec else "0"
    t = time.time()
    m = ctx.run_multilevel(*args[:3], args[3], args[4], "c2", args[5])
    return m, time.time() - t


def main():
    names = sys.argv[1:] or ["cfg1", "cfg2l01", "cfg3p", "cfg4p"]
    ctx = capi.Context(0)
    seq_too = os.environ.get("SPEC_SEQ", "1") == "1"
    for name in names:
        args = case(name)
        os.environ["IMB_SPEC_LOG"] = os.path.join(ROOT, "gpurun_out", f"spec_{name}.log")
        b, tb = run(ctx, args, True)
        os.environ.pop("IMB_SPEC_LOG")
        line = f"{name}: spec {tb:.2f} s levels {[len(l.control_indices) for l in b.levels]}"
        if seq_too:
            a, ta = run(ctx, args, False)
            same = len(a.levels) == len(b.levels) and all(
                np.array_equal(x.control_indices, y.control_indices) and np.array_equal(x.alpha, y.alpha)
                and np.array_equal(x.record_error, y.record_error)
                for x, y in zip(a.levels, b.levels)) and np.array_equal(a.final_residual, b.final_residual)
            line += f" | seq {ta:.2f} s | identical={same} | speedup {ta / tb:.2f}x"
        print(line, flush=True)


if __name__ == "__main__":
    main()
