"""Small mesh builders for the quality / inverted-element tests (test
infrastructure).  Restate the reference test helpers make_quad_grid /
make_box_grid (tests/oracles.cpp:122-200) and wall_bump
(tests/test_pipeline.cpp:25-34); elements are returned in the C-ABI's CSR
form (kinds int32 in ElementKind order mesh.hpp:15-23, offsets uint64, node
indices uint64)."""
import math

import numpy as np

LINE, TRI, QUAD, TET, HEX, PRISM, PYRAMID = range(7)
NODE_COUNT = {LINE: 2, TRI: 3, QUAD: 4, TET: 4, HEX: 8, PRISM: 6, PYRAMID: 5}


def csr(elements):
    """[(kind, [nodes...]), ...] -> (kinds, offsets, conn)."""
    kinds = np.array([k for k, _ in elements], np.int32)
    offs = np.zeros(len(elements) + 1, np.uint64)
    offs[1:] = np.cumsum([len(n) for _, n in elements])
    conn = np.array([i for _, n in elements for i in n], np.uint64)
    return kinds, offs, conn


def quad_grid(nx, ny, lx=1.0, ly=1.0):
    """oracles.cpp:122-156: nodes, quad elements, 'wall' (j=0) marker nodes."""
    node = lambda i, j: j * (nx + 1) + i
    nodes = [(lx * i / nx, ly * j / ny, 0.0) for j in range(ny + 1) for i in range(nx + 1)]
    el = [(QUAD, [node(i, j), node(i + 1, j), node(i + 1, j + 1), node(i, j + 1)])
          for j in range(ny) for i in range(nx)]
    wall = [node(i, 0) for i in range(nx + 1)]
    return np.array(nodes), csr(el), wall


def box_grid(nx, ny, nz, lx=1.0, ly=1.0, lz=1.0):
    """oracles.cpp:158-187: nodes and hex elements."""
    node = lambda i, j, k: (k * (ny + 1) + j) * (nx + 1) + i
    nodes = [(lx * i / nx, ly * j / ny, lz * k / nz)
             for k in range(nz + 1) for j in range(ny + 1) for i in range(nx + 1)]
    el = [(HEX, [node(i, j, k), node(i + 1, j, k), node(i + 1, j + 1, k), node(i, j + 1, k),
                 node(i, j, k + 1), node(i + 1, j, k + 1), node(i + 1, j + 1, k + 1),
                 node(i, j + 1, k + 1)])
          for k in range(nz) for j in range(ny) for i in range(nx)]
    return np.array(nodes), el


def wall_bump(nodes, wall, amplitude):
    """test_pipeline.cpp:25-34: (0, A exp(-18 (x - 0.5)^2), 0) on the wall."""
    return np.array([(0.0, amplitude * math.exp(-18.0 * (nodes[n][0] - 0.5) *
                                                (nodes[n][0] - 0.5)), 0.0) for n in wall])


def random_mixed(rng, n_nodes, n_elem, kinds=tuple(range(7)), degenerate=0.05):
    """Random nodes and elements of the given kinds on random node tuples:
    about half come out inverted; a fraction repeat a node (measure +-0)."""
    nodes = rng.standard_normal((n_nodes, 3))
    kind = rng.choice(np.array(kinds, np.int32), n_elem)
    el = []
    for k in kind:
        n = list(rng.choice(n_nodes, NODE_COUNT[int(k)], replace=False))
        if rng.random() < degenerate and len(n) > 2:
            n[1] = n[0]
        el.append((int(k), [int(i) for i in n]))
    return nodes, csr(el)
