"""Host-side helpers of the reference's Python module that sit around the hot
path (not on it): the mesh / displacement generators (generators.cpp), the
VTK writer and displacement files (mesh_io.cpp:311-428) and the report
writers (pipeline.cpp:108-160).  They make ``import icemorph`` a drop-in for
the reference module's full name list (python/icemorph/__init__.py:1-24);
numpy on the host, no device work.  Every function cites the reference
lines it restates; messages and file formats are the reference's.
"""
from __future__ import annotations

import math

import numpy as np

from . import capi
from .icemorph import DeformationReport, DisplacementField, Mesh

# generators.hpp:34-35
SIN_AIRFOIL_AMPLITUDE = 0.01
SIN_AIRFOIL_WAVENUMBER = 15.0
_FARFIELD_CHORDS = 25.0      # generators.cpp:22
_FIRST_LAYER_FRACTION = 1.5e-4  # generators.cpp:23


def naca0012_half_thickness(x_over_c: float, chord: float) -> float:
    """generators.cpp:12-18 (closed trailing edge)."""
    x = min(max(x_over_c, 0.0), 1.0)
    y = (0.2969 * math.sqrt(x) - 0.1260 * x - 0.3516 * x * x + 0.2843 * x * x * x
         - 0.1036 * x * x * x * x)
    return 5.0 * 0.12 * chord * y


def _pow(g: float, e: float) -> float:
    """std::pow: +inf on overflow (math.pow raises)."""
    try:
        return math.pow(g, e)
    except OverflowError:
        return math.inf


def _solve_growth(layers: int, first_fraction: float) -> float:
    """generators.cpp:26-41: g with (g-1)/(g^M-1) = first_fraction, bisection."""
    lo, hi = 1.0 + 1e-12, 100.0

    def fraction(g):
        return (g - 1.0) / (_pow(g, float(layers)) - 1.0)

    if fraction(lo) <= first_fraction:
        return lo
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        if fraction(mid) > first_fraction:
            lo = mid
        else:
            hi = mid
    return 0.5 * (lo + hi)


def gen_airfoil_mesh(chord: float, circumferential: int, radial_layers: int) -> Mesh:
    """generators.cpp:45-128: NACA0012 O-mesh, quads, markers airfoil / farfield."""
    if not chord > 0.0:
        raise ValueError("chord must be positive")
    if circumferential < 8 or radial_layers < 8:
        raise ValueError("airfoil grid needs at least 8x8 cells")
    if circumferential % 2 != 0:
        raise ValueError("circumferential count must be even")
    n, m = int(circumferential), int(radial_layers)
    profile = []
    for j in range(n):
        theta = 2.0 * math.pi * j / n
        xc = 0.5 * (1.0 + math.cos(theta))
        y = naca0012_half_thickness(xc, chord)
        if j == 0 or 2 * j == n:
            y = 0.0
        elif 2 * j > n:
            y = -y
        profile.append((xc * chord, y))
    cx, far = 0.5 * chord, _FARFIELD_CHORDS * chord
    farfield = [(cx + far * math.cos(2.0 * math.pi * j / n), far * math.sin(2.0 * math.pi * j / n))
                for j in range(n)]
    growth = _solve_growth(m, _FIRST_LAYER_FRACTION)
    denom = _pow(growth, float(m)) - 1.0
    frac = [(_pow(growth, float(i)) - 1.0) / denom if denom > 0.0 else i / m
            for i in range(m + 1)]
    frac[0], frac[m] = 0.0, 1.0
    nodes = []
    for i in range(m + 1):
        t = frac[i]
        for j in range(n):
            # profile * (1 - t) + farfield * t, Vec3 arithmetic order
            px, py = profile[j][0] * (1.0 - t), profile[j][1] * (1.0 - t)
            fx, fy = farfield[j][0] * t, farfield[j][1] * t
            nodes.append((px + fx, py + fy, 0.0))
    quads = [("quadrilateral", (i * n + j, (i + 1) * n + j, (i + 1) * n + (j + 1) % n,
                                i * n + (j + 1) % n)) for i in range(m) for j in range(n)]

    def ring(r):
        lines = [("line", (r * n + j, r * n + (j + 1) % n)) for j in range(n)]
        seen, order = set(), []
        for _, e in lines:  # marker_nodes_from_elements (mesh.cpp:92-102)
            for v in e:
                if v not in seen:
                    seen.add(v)
                    order.append(v)
        return lines, order

    air_el, air_nodes = ring(0)
    far_el, far_nodes = ring(m)
    return Mesh(2, nodes, {"airfoil": air_nodes, "farfield": far_nodes}, quads,
                {"airfoil": capi.elements_csr(air_el), "farfield": capi.elements_csr(far_el)})


def gen_sinusoidal_displacement(mesh: Mesh, marker: str, mode: str = "airfoil",
                                amplitude: float = SIN_AIRFOIL_AMPLITUDE,
                                wavenumber: float = SIN_AIRFOIL_WAVENUMBER) -> DisplacementField:
    """generators.cpp:130-162 (bindings.cpp:165-180)."""
    if mode not in ("airfoil", "wing"):
        raise ValueError("mode must be 'airfoil' or 'wing'")
    nodes = mesh.marker_nodes(marker)
    if mode == "wing" and mesh.dim != 3:
        raise ValueError("wing mode requires a 3D mesh")
    axis = 0 if mode == "airfoil" else 2
    coords = [mesh._nodes[i][axis] for i in nodes]
    lo, hi = min(coords, default=math.inf), max(coords, default=-math.inf)
    extent = hi - lo
    if not extent > 0.0:
        raise ValueError(f"marker '{marker}' has no extent along the driving axis")
    f = DisplacementField(marker)
    for i, c in zip(nodes, coords):
        t = (c - lo) / extent
        f.set(i, 0.0, amplitude * math.sin(wavenumber * math.pi * t), 0.0)
    return f


def _marker_chain(mesh: Mesh, marker: str):
    """generators.cpp:178-213: neighbour lists of the marker's line polyline."""
    nodes = mesh.marker_nodes(marker)
    local = {g: i for i, g in enumerate(nodes)}
    kinds, offs, conn = mesh._marker_elements.get(marker, (np.zeros(0), [0], []))
    nb = [[] for _ in nodes]
    for e in range(len(kinds)):
        if int(kinds[e]) != 0:
            raise ValueError("arc positions require a line-element marker")
        a, b = local[int(conn[int(offs[e])])], local[int(conn[int(offs[e]) + 1])]
        nb[a].append(b)
        nb[b].append(a)
    ends = 0
    for x in nb:
        if len(x) > 2:
            raise ValueError("marker polyline branches; arc length undefined")
        if len(x) == 1:
            ends += 1
        if not x:
            raise ValueError("marker has an isolated node")
    closed = ends == 0
    if not closed and ends != 2:
        raise ValueError("marker polyline is not a single chain")
    return nodes, nb, closed


def _dist(a, b):
    dx, dy, dz = a[0] - b[0], a[1] - b[1], a[2] - b[2]
    return math.sqrt(dx * dx + dy * dy + dz * dz)


def marker_arc_positions(mesh: Mesh, marker: str):
    """generators.cpp:217-278: arc length along the marker, zero at the
    minimum-x node (lowest index on ties), wrapped to [-P/2, P/2) if closed."""
    if mesh.dim != 2:
        raise ValueError("arc positions are defined for 2D markers only")
    nodes, nb, closed = _marker_chain(mesh, marker)
    if len(nodes) < 2:
        raise ValueError("marker too small for arc positions")
    P = mesh._nodes
    start = 0
    if not closed:
        start = next(i for i, x in enumerate(nb) if len(x) == 1)
    cum = [0.0] * len(nodes)
    seen = [False] * len(nodes)
    cur, seen[start], length = start, True, 0.0
    for _ in range(1, len(nodes)):
        nxt = next((x for x in nb[cur] if not seen[x]), None)
        if nxt is None:
            raise ValueError("marker polyline is not a single chain")
        length += _dist(P[nodes[cur]], P[nodes[nxt]])
        cum[nxt], seen[nxt], cur = length, True, nxt
    perim = length + (_dist(P[nodes[cur]], P[nodes[start]]) if closed else 0.0)
    le = 0
    for i in range(1, len(nodes)):
        if P[nodes[i]][0] < P[nodes[le]][0]:
            le = i
    arc = []
    for i in range(len(nodes)):
        s = cum[i] - cum[le]
        if closed and perim > 0.0:
            s -= perim * math.floor(s / perim + 0.5)
        arc.append(s)
    return arc


def gen_ice_bump(mesh: Mesh, marker: str, center: float = 0.0, height: float = 0.02,
                 width: float = 0.05, horns: int = 2) -> DisplacementField:
    """generators.cpp:280-333 (bindings.cpp:181-187): Gaussian horns along the
    arc, exp(-(ds/w)^2) with a 5w cut-off, along the outward node normal."""
    if mesh.dim != 2:
        raise ValueError("ice bump generation supports 2D meshes")
    if not width > 0.0:
        raise ValueError("bump width must be positive")
    if horns < 1:
        raise ValueError("at least one horn is required")
    arc = marker_arc_positions(mesh, marker)
    hpos = [center + (k - 0.5 * (horns - 1)) * 3.0 * width for k in range(horns)]
    nodes, nb, _ = _marker_chain(mesh, marker)
    P = mesh._nodes
    cxs = cys = 0.0
    for i in nodes:
        cxs += P[i][0]
        cys += P[i][1]
    cxs *= 1.0 / len(nodes)
    cys *= 1.0 / len(nodes)

    def normalized(x, y):
        nrm = math.sqrt(x * x + y * y)
        return (x * (1.0 / nrm), y * (1.0 / nrm)) if nrm > 0.0 else (0.0, 0.0)

    def edge_normal(a, b):
        tx, ty = P[nodes[b]][0] - P[nodes[a]][0], P[nodes[b]][1] - P[nodes[a]][1]
        nx, ny = normalized(ty, -tx)
        mx = 0.5 * (P[nodes[a]][0] + P[nodes[b]][0])
        my = 0.5 * (P[nodes[a]][1] + P[nodes[b]][1])
        if nx * (mx - cxs) + ny * (my - cys) < 0.0:
            nx, ny = -nx, -ny
        return nx, ny

    f = DisplacementField(marker)
    for i in range(len(nodes)):
        nearest, mag = math.inf, 0.0
        for h in hpos:
            ds = arc[i] - h
            nearest = min(nearest, abs(ds))
            mag += math.exp(-(ds * ds) / (width * width))
        if nearest >= 5.0 * width:
            continue
        mag *= height
        if mag == 0.0:
            continue
        sx = sy = 0.0
        for j in nb[i]:
            ex, ey = edge_normal(i, j)
            sx, sy = sx + ex, sy + ey
        nx, ny = normalized(sx, sy)
        f.set(nodes[i], nx * mag, ny * mag, 0.0)
    return f


def _g17(v: float) -> str:
    return f"{v:.17g}"


_VTK = {0: 3, 1: 5, 2: 9, 3: 10, 4: 12, 5: 13, 6: 14}  # mesh.cpp:12-23


def write_vtk(mesh: Mesh, path: str) -> None:
    """mesh_io.cpp:311-359 (legacy ASCII unstructured grid)."""
    kinds, offs, conn = mesh._elements
    try:
        out = open(path, "w")
    except OSError:
        raise RuntimeError(f"cannot write mesh file '{path}'") from None
    with out:
        out.write("# vtk DataFile Version 3.0\nicemorph mesh\nASCII\nDATASET UNSTRUCTURED_GRID\n")
        out.write(f"POINTS {mesh.num_nodes} double\n")
        for p in mesh._nodes:
            out.write(f"{_g17(p[0])} {_g17(p[1])} {_g17(p[2])}\n")
        ne = len(kinds)
        size = sum(int(offs[e + 1] - offs[e]) + 1 for e in range(ne))
        out.write(f"CELLS {ne} {size}\n")
        for e in range(ne):
            nodes = conn[int(offs[e]):int(offs[e + 1])]
            out.write(" ".join([str(len(nodes))] + [str(int(v)) for v in nodes]) + "\n")
        out.write(f"CELL_TYPES {ne}\n")
        for e in range(ne):
            out.write(f"{_VTK[int(kinds[e])]}\n")


def write_displacements(field: DisplacementField, dim: int, path: str) -> None:
    """mesh_io.cpp:413-428: `node dx dy [dz]` per entry, ascending node."""
    try:
        out = open(path, "w")
    except OSError:
        raise RuntimeError(f"cannot write displacement file '{path}'") from None
    with out:
        for node in sorted(field.entries()):
            d = field.entries()[node]
            row = [str(node), _g17(d[0]), _g17(d[1])] + ([_g17(d[2])] if dim == 3 else [])
            out.write(" ".join(row) + "\n")


def read_displacements(path: str, mesh: Mesh, marker: str) -> DisplacementField:
    """mesh_io.cpp:361-411: '#' comments, `node dx dy [dz]`, node on the marker,
    finite components; errors "path:line: what"."""
    on_marker = set(mesh.marker_nodes(marker))
    try:
        lines = open(path).read().splitlines()
    except OSError:
        raise RuntimeError(f"cannot open displacement file '{path}'") from None
    f = DisplacementField(marker)

    def fail(no, what):
        raise capi.ParseError(f"{path}:{no}: {what}", no)

    for no, line in enumerate(lines, 1):
        tok = line.split("#", 1)[0].split()
        if not tok:
            continue
        if len(tok) != 1 + mesh.dim:
            fail(no, f"expected `node dx dy{' dz' if mesh.dim == 3 else ''}`, got {len(tok)} tokens")
        if not tok[0].isdigit():
            fail(no, f"bad node index '{tok[0]}'")
        node = int(tok[0])
        if node not in on_marker:
            fail(no, f"node {node} is not on marker '{marker}'")
        comps = [0.0, 0.0, 0.0]
        for c in range(mesh.dim):
            try:
                comps[c] = float(tok[c + 1])
            except ValueError:
                fail(no, f"bad displacement component '{tok[c + 1]}'")
            if not math.isfinite(comps[c]):
                fail(no, "displacement component is not finite")
        f.set(node, *comps)
    return f


def write_summary(report: DeformationReport, path: str) -> None:
    """pipeline.cpp:108-147 (the report as `key: value` lines)."""
    try:
        out = open(path, "w")
    except OSError:
        raise RuntimeError(f"cannot write summary file '{path}'") from None
    with out:
        w = out.write
        w(f"marker: {report.marker}\nlevels: {len(report.levels)}\n")
        w(f"total_control_points: {report.total_control_points}\n")
        w(f"target_max: {_g17(report.target_max)}\n")
        w(f"surface_max_error: {_g17(report.surface_max_error)}\n")
        w(f"surface_mean_error: {_g17(report.surface_mean_error)}\n")
        w(f"inverted_elements: {report.inverted_elements}\n")
        for tag, q in (("before", report.quality_before), ("after", report.quality_after)):
            if q is not None:
                w(f"min_orthogonality_{tag}_deg: {_g17(q.min_orthogonality_deg)}\n")
                w(f"mean_orthogonality_{tag}_deg: {_g17(q.mean_orthogonality_deg)}\n")
        w(f"total_seconds: {report.total_seconds:.6g}\n")
        for l in report.levels:
            p = f"level_{l.level}_"
            w(f"{p}points: {l.points}\n{p}error: {_g17(l.achieved_error)}\n")
            w(f"{p}cap_hit: {1 if l.cap_hit else 0}\n")
            w(f"{p}support_distance: {_g17(l.support_distance)}\n")
            w(f"{p}touched_nodes: {l.touched_nodes}\n{p}seconds: {l.seconds:.6g}\n")


def write_convergence_csv(report: DeformationReport, path: str) -> None:
    """pipeline.cpp:149-160 + greedy.cpp write_convergence_csv_header /
    append_convergence_csv: `level,points,error,seconds`, one row per greedy
    step of every level."""
    try:
        out = open(path, "w")
    except OSError:
        raise RuntimeError(f"cannot write report file '{path}'") from None
    with out:
        out.write("level,points,error,seconds\n")
        for l in report.levels:
            for pts, err, sec in getattr(l, "record", []):
                out.write(f"{l.level},{pts},{_g17(err)},{sec:.6g}\n")
