"""Reference greedy selection on the full BASELINE cfg2 workload (2-D horn
ice: 10k surface points, R = 0.25c, eps = 1e-4, 3 levels, cap 5000).

Runs the UNMODIFIED reference run_multilevel (oracle/_ref) — about 27 min on
one core of the dev container (1.1 s + 92 s + 1531 s per level) — and stores
the control indices of every level.  They pin the device greedy at full size
(tests/test_gpu_parity.py::test_cfg2_full_selection) and give the reference
arm of bench.py its control sets without re-running the reference greedy.

    python tests/golden/make_cfg2_selection.py
"""
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


def main():
    w = W.cfg2()
    pos = w.nodes[w.surface]
    t0 = time.time()
    m = Oracle("ref").run_multilevel(pos, w.displacement, w.tol, w.levels, w.cap, w.kind, w.R)
    out = {f"idx{l}": lv.control_indices for l, lv in enumerate(m.levels)}
    out["seconds"] = np.array([lv.elapsed_seconds for lv in m.levels])
    out["cap_hit"] = np.array([lv.cap_hit for lv in m.levels])
    np.savez_compressed(os.path.join(HERE, "cfg2_reference_selection.npz"), **out)
    print("levels", [len(lv.control_indices) for lv in m.levels], "in", time.time() - t0, "s")


if __name__ == "__main__":
    main()
