"""Generate the golden fixtures of tests/golden/ from the REFERENCE itself.

Run in the dev container (needs oracle/_ref/libicemorph_ref.so, i.e. the
unmodified reference sources under /root/reference compiled by
oracle/Makefile).  Every array stored here is the reference's own output on
seeded inputs that are stored alongside, so the tests can pin both the
plain-C oracle restatement and the CUDA product on boxes where the
reference sources are absent.

    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import Oracle  # noqa: E402

from paper_2107_13887_b200 import workloads as W  # noqa: E402

sys.path.insert(0, os.path.dirname(HERE))
import meshes as M  # noqa: E402


def random_cloud(rng, n, dim, min_sep):
    """Rejection-sampled cloud with a minimum separation (test_rbf.cpp:13-30)."""
    pts = []
    while len(pts) < n:
        p = np.array([rng.random(), rng.random(), rng.random() if dim == 3 else 0.0])
        if all(np.linalg.norm(p - q) >= min_sep for q in pts):
            pts.append(p)
    return np.array(pts)


def circle_case(n):
    """test_greedy.cpp:16-26."""
    t = 2.0 * np.pi * np.arange(n) / n
    pos = np.stack([np.cos(t), np.sin(t), np.zeros(n)], 1)
    tgt = np.stack([np.zeros(n), 0.1 * np.sin(2 * t) + 0.05 * np.cos(t), np.zeros(n)], 1)
    return pos, tgt


def main():
    ref = Oracle("ref")
    out = {}
    # greedy vs dense-solve cases (test_greedy.cpp:53-81 shape): 4 clouds
    rng = np.random.default_rng(17)
    for trial in range(4):
        pos = random_cloud(rng, 30, 2, 0.04)
        tgt = np.stack([0.02 * np.sin(5 * pos[:, 0]), 0.05 * np.cos(4 * pos[:, 1]), 0 * pos[:, 0]], 1)
        g = ref.greedy_level(pos, tgt, 0.05, 5000, "c2", 1.5)
        out[f"greedy{trial}_pos"] = pos
        out[f"greedy{trial}_tgt"] = tgt
        out[f"greedy{trial}_idx"] = g.control_indices
        out[f"greedy{trial}_alpha"] = g.alpha
        out[f"greedy{trial}_err"] = g.record_error
        out[f"greedy{trial}_res"] = g.residual
    # multilevel circle (test_greedy.cpp:131-158)
    pos, tgt = circle_case(80)
    m = ref.run_multilevel(pos, tgt, 0.3, 3, 5000, "c2", 3.0)
    out["circle_pos"], out["circle_tgt"] = pos, tgt
    out["circle_nlevels"] = np.array(len(m.levels))
    for l, lv in enumerate(m.levels):
        out[f"circle_l{l}_idx"] = lv.control_indices
        out[f"circle_l{l}_alpha"] = lv.alpha
    out["circle_final"] = m.final_residual
    # solve_weights on a 3-D cloud (test_rbf.cpp:177-193 shape)
    rng = np.random.default_rng(23)
    p = random_cloud(rng, 30, 3, 0.05)
    d = rng.uniform(-1, 1, (30, 3))
    out["sw_pts"], out["sw_disp"] = p, d
    out["sw_alpha"] = ref.solve_weights(p, d, "c2", 0.9)
    # wall distance, 3-D random (test_wall_distance.cpp:12-27 shape)
    rng = np.random.default_rng(5)
    nodes = rng.uniform(-2, 2, (1500, 3))
    out["wd_nodes"] = nodes
    out["wd_dist"] = ref.build_distance_index(nodes, 3, np.arange(1000))
    # update_volume with both tapers
    ctrl = nodes[:40].copy()
    alpha = rng.standard_normal((40, 3)) * 0.01
    for psi in (0, 1):
        i, v = ref.update_volume(nodes, out["wd_dist"], ctrl, alpha, 0.35, psi, "c2", 0.5)
        out[f"uv{psi}_idx"], out[f"uv{psi}_val"] = i, v
    out["uv_alpha"] = alpha
    # cfg1 at 30% scale: multilevel + deform (reference linear taper)
    w = W.cfg1(0.3)
    surf = w.nodes[w.surface]
    m = ref.run_multilevel(surf, w.displacement, w.tol, w.levels, w.cap, w.kind, w.R)
    out["cfg1s_nlevels"] = np.array(len(m.levels))
    for l, lv in enumerate(m.levels):
        out[f"cfg1s_l{l}_idx"] = lv.control_indices
        out[f"cfg1s_l{l}_alpha"] = lv.alpha
    r = ref.deform(w.nodes, 2, w.surface, w.displacement, (), w.tol, w.levels, w.cap, w.kind, w.R,
                   5.0)
    out["cfg1s_nodes"], out["cfg1s_surface"], out["cfg1s_disp"] = w.nodes, w.surface, w.displacement
    out["cfg1s_deformed"] = r["nodes"]
    out["cfg1s_touched"] = r["touched"]
    # quality (quality.cpp:135-148): random mixed elements, about half inverted
    nodes, (k, o, c) = M.random_mixed(np.random.default_rng(11), 400, 3000)
    meas, inv = ref.signed_measures(nodes, 3, (k, o, c))
    out.update(q_nodes=nodes, q_kinds=k, q_offsets=o, q_conn=c, q_measures=meas,
               q_inverted=np.array(inv))
    # test_pipeline.cpp:216-228: a tall bump through a shallow quad grid inverts cells
    nodes, el, wall = M.quad_grid(10, 3, 1.0, 0.05)
    disp = M.wall_bump(nodes, wall, 0.5)
    r = ref.deform(nodes, 2, wall, disp, (), 0.01, 2, 5000, "c2", 0.3, 0.2, elements=el)
    out.update(inv_deformed=r["nodes"], inv_count=np.array(r["inverted_elements"]))
    np.savez_compressed(os.path.join(HERE, "reference_outputs.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
