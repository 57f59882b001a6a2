"""SU2 mesh I/O throughput: the native reader / writer
against the reference's read_su2 (oracle/_ref/ref_su2_tool, single-threaded
as the reference is) on the same files.  Prints one JSON line per mesh.

    python tools/su2_bench.py [cfg2 cfg3:0.5 ...]
"""
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2107_13887_b200 import capi, workloads as W  # noqa: E402
import meshes as M  # noqa: E402


def main():
    ctx = capi.Context(0)
    tool = os.path.join(ROOT, "oracle", "_ref", "ref_su2_tool")
    for spec in sys.argv[1:] or ["cfg2"]:
        name, _, scale = spec.partition(":")
        w = W.CONFIGS[name](float(scale or 1.0))
        nvol = w.meta["n_volume"]
        nodes, e = w.nodes[:nvol], W.elements(w)
        first = e[2][e[1][0]:e[1][1]]
        if w.dim == 2:  # wall marker: the first O-mesh ring
            ring = w.meta["ring"]
            marker = M.csr([(M.LINE, [i, (i + 1) % ring]) for i in range(ring)])
        else:  # first quad face of every hex of the first layer
            nq = w.meta["around"] * (w.meta["span"] - 1)
            marker = M.csr([(M.QUAD, [int(v) for v in e[2][8 * k:8 * k + 4]]) for k in range(nq)])
        del first
        with tempfile.TemporaryDirectory() as d:
            path = os.path.join(d, f"{name}.su2")
            t0 = time.perf_counter()
            ctx.write_su2(path, w.dim, nodes, e, [("wall", marker)])
            t_write = time.perf_counter() - t0
            size = os.path.getsize(path)
            ctx.read_su2(path)  # warm the page cache
            best = 1e30
            for _ in range(3):
                t0 = time.perf_counter()
                m = ctx.read_su2(path)
                best = min(best, time.perf_counter() - t0)
            assert len(m["nodes"]) == len(nodes)
            ref_s = None
            if os.path.exists(tool):
                r = subprocess.run([tool, "time", path, "1"], capture_output=True, text=True)
                if r.returncode == 0:
                    ref_s = float(r.stdout.split()[0])
            print(json.dumps({
                "mesh": w.name, "nodes": len(nodes), "elements": int(len(e[0])),
                "file_mb": round(size / 1e6, 1),
                "read_s": round(best, 4), "read_mb_s": round(size / best / 1e6, 1),
                "write_s": round(t_write, 4), "write_mb_s": round(size / t_write / 1e6, 1),
                "reference_read_s": ref_s,
                "read_speedup": round(ref_s / best, 1) if ref_s else None,
                "host_threads": os.cpu_count()}), flush=True)


if __name__ == "__main__":
    main()
