import sys, time
import numpy as np
sys.path.insert(0, ".")
from paper_2107_13887_b200 import capi, workloads as W
ctx = capi.Context(0)
name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
w = W.CONFIGS[name]()
pos = w.nodes[w.surface]
for rep in range(2):
    t = time.time()
    m1 = ctx.run_multilevel(pos, w.displacement, w.tol, w.levels if len(sys.argv) < 3 else int(sys.argv[2]), w.cap, w.kind, w.R)
    print(name, "multilevel", time.time() - t, [len(l.control_indices) for l in m1.levels], [l.elapsed_seconds for l in m1.levels], flush=True)
