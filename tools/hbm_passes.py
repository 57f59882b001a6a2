"""The HBM-side passes alone (wall distance K6, compaction K7) on a BASELINE
mesh: `python tools/hbm_passes.py cfg3 [scale] [cutoff]`.  Used plain for the
timings and under ncu for the captures in profiles/ (the kernels of interest
are k_wall_distance and k_compact_active)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2107_13887_b200 import capi, workloads as W  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
    scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
    cutoff = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    w = getattr(W, name)(scale)
    ctx = capi.Context(0)
    dim = 2 if name in ("cfg1", "cfg2") else 3
    plan = capi.VolumePlan(ctx, w.nodes, dim, w.surface, cutoff=cutoff)
    st = plan.bench_passes(cutoff, cutoff, reps=reps)
    n = len(w.nodes)
    st.update(workload=name, n_nodes=n, n_surface=len(w.surface), cutoff=cutoff,
              wall_distance_gbs=32.0 * n / (st["wall_distance_ms"] * 1e-3) / 1e9,
              compaction_gbs=(8.0 * n + 4.0 * st["active"]) / (st["compaction_ms"] * 1e-3) / 1e9)
    print(json.dumps(st))


if __name__ == "__main__":
    main()
