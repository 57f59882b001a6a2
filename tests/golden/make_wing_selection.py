"""Greedy fixtures on the full 3-D BASELINE wing surfaces (cfg3: 40k points,
R = 0.5c, eps = 1e-3; cfg4: 100k points, R = 40 = 10b, eps = 1e-4).

Two kinds of fixture, both CPU-made here (the GPU box has no /root/reference):

* ``wing_prefix_reference.npz`` -- the UNMODIFIED reference run_multilevel
  (oracle/_ref) with max_points_per_level = 300 and 2 levels on each full
  surface: control indices, alpha, convergence record and a SHA-256 of the
  final residual bytes.  The same prefix through the plain-C port with a
  threaded sweep (oracle/_port, or_set_sweep_threads) must equal it bit for
  bit; that pins the threaded port, which then makes --

* ``wing_full_port.npz`` (``--full``) -- the whole multilevel selection at the
  reference's default cap of 5000 (capped levels included), by the pinned
  port with a threaded sweep: what a reference run would give in ~1.1 h
  (cfg3) / ~2.7 h (cfg4) per capped level on one core.

    python tests/golden/make_wing_selection.py [--full] [--threads 7]
"""
import argparse
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import Oracle  # noqa: E402

from paper_2107_13887_b200 import workloads as W  # noqa: E402

PREFIX_CAP, PREFIX_LEVELS = 300, 2


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def pack(prefix: str, m, out: dict) -> None:
    out[f"{prefix}_nlevels"] = np.array(len(m.levels))
    for l, lv in enumerate(m.levels):
        out[f"{prefix}_idx{l}"] = lv.control_indices
        out[f"{prefix}_alpha{l}"] = lv.alpha
        out[f"{prefix}_rec{l}"] = lv.record_error
        out[f"{prefix}_cap{l}"] = np.array(lv.cap_hit)
        out[f"{prefix}_ach{l}"] = np.array(lv.achieved_error)
        out[f"{prefix}_sec{l}"] = np.array(lv.elapsed_seconds)
    out[f"{prefix}_residual_sha"] = np.array(digest(m.final_residual))
    out[f"{prefix}_residual_max"] = np.array(np.abs(m.final_residual).max())


def same(a, b) -> bool:
    if len(a.levels) != len(b.levels):
        return False
    for x, y in zip(a.levels, b.levels):
        if not (np.array_equal(x.control_indices, y.control_indices)
                and np.array_equal(x.alpha, y.alpha)
                and np.array_equal(x.record_error, y.record_error)
                and x.cap_hit == y.cap_hit):
            return False
    return np.array_equal(a.final_residual, b.final_residual)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--threads", type=int, default=max(1, (os.cpu_count() or 2) - 1))
    ap.add_argument("--configs", default="cfg3,cfg4")
    ap.add_argument("--levels", type=int, default=0,
                    help="--full: run only the first N levels (0 = the config's count); cfg4's "
                         "fixture holds levels 0-1 (109 points + one capped level, ~20 min on 7 "
                         "threads; all four take ~1.5 h)")
    args = ap.parse_args()
    port = Oracle("port")
    port.set_sweep_threads(args.threads)
    if not args.full:
        ref = Oracle("ref")
        out = {}
        for name in args.configs.split(","):
            pos, disp, R, tol, _ = W.wing_surface_case(name)
            t0 = time.time()
            a = ref.run_multilevel(pos, disp, tol, PREFIX_LEVELS, PREFIX_CAP, "c2", R)
            t1 = time.time()
            b = port.run_multilevel(pos, disp, tol, PREFIX_LEVELS, PREFIX_CAP, "c2", R)
            t2 = time.time()
            assert same(a, b), f"{name}: threaded port differs from the reference"
            pack(name, a, out)
            print(f"{name}: ref {t1 - t0:.1f} s, port({args.threads} thr) {t2 - t1:.1f} s, "
                  f"levels {[len(l.control_indices) for l in a.levels]}, identical")
        np.savez_compressed(os.path.join(HERE, "wing_prefix_reference.npz"), **out)
        return
    path = os.path.join(HERE, "wing_full_port.npz")
    out = dict(np.load(path)) if os.path.exists(path) else {}
    for name in args.configs.split(","):
        pos, disp, R, tol, levels = W.wing_surface_case(name)
        if args.levels:
            levels = min(levels, args.levels)
        t0 = time.time()
        try:
            m = port.run_multilevel(pos, disp, tol, levels, 5000, "c2", R)
        except Exception as e:  # SolveError (rbf.cpp:92): keep the reference's message
            out[f"{name}_error"] = np.array(str(e))
            np.savez_compressed(path, **out)
            print(f"{name}: {time.time() - t0:.0f} s, error: {e}", flush=True)
            continue
        pack(name, m, out)
        np.savez_compressed(path, **out)
        print(f"{name}: {time.time() - t0:.0f} s, levels "
              f"{[len(l.control_indices) for l in m.levels]}, cap "
              f"{[l.cap_hit for l in m.levels]}", flush=True)


if __name__ == "__main__":
    main()
