"""Exact device greedy on a BASELINE config, first `levels` levels, once:
python tools/greedy_levels.py cfg2 2 [cap]  (for ncu launch lists / captures)"""
import sys
import time

sys.path.insert(0, ".")
from paper_2107_13887_b200 import capi, workloads as W

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
levels = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cap = int(sys.argv[3]) if len(sys.argv) > 3 else None  # optional max points per level
ctx = capi.Context(0)
w = W.CONFIGS[name]()
pos = w.nodes[w.surface]
t = time.time()
m = ctx.run_multilevel(pos, w.displacement, w.tol, levels, cap or w.cap, w.kind, w.R)
print(name, time.time() - t, [len(l.control_indices) for l in m.levels],
      [round(l.elapsed_seconds, 3) for l in m.levels], flush=True)
