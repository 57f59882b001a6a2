"""Python mirror of the reference's ``icemorph`` module for the hot path
(proj/python/bindings.cpp:34-242, re-exported by proj/python/icemorph/__init__.py),
backed by the B200 C-ABI through :mod:`paper_2107_13887_b200.capi`.

Same names, argument meaning and error behaviour as the reference binding:
``eval_basis``, ``solve_weights``, ``eval_interpolant``, ``deform`` with
``Mesh`` / ``DisplacementField`` / ``DeformationConfig`` / ``DeformationReport``
/ ``LevelSummary``; ``ValueError`` for std::invalid_argument and
``RuntimeError`` (``capi.SolveError``) for icemorph::SolveError, as pybind11
maps them, plus ``orthogonality`` / ``signed_measures`` (bindings.cpp:194-197)
and the report's ``inverted_elements`` / ``quality_before`` / ``quality_after``
(pipeline.cpp:55, 101-102) on the device, and ``read_su2`` / ``write_su2``
(bindings.cpp:149-154) on the native SU2 reader / writer.  Generators are out
of scope; a ``Mesh`` can also be built from arrays (``Mesh(dim, nodes,
markers, elements)``).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import capi

_ctx = None


def _context() -> capi.Context:
    global _ctx
    if _ctx is None:
        _ctx = capi.Context(0)
    return _ctx


def _kind(name: str) -> str:
    if name not in ("c0", "c2", "c4", "c6", "C0", "C2", "C4", "C6"):
        raise ValueError(f"unknown basis function '{name}' (expected c0, c2, c4 or c6)")
    return name.lower()


def _precision(name: str) -> int:
    """DeformationConfig.precision (additive extension) -> IM_EXACT / IM_FP64 / IM_FP32."""
    codes = {"exact": capi.EXACT, "fp64": capi.FP64, "fp32": capi.FP32}
    if name not in codes:
        raise ValueError(f"unknown precision '{name}' (expected exact, fp64 or fp32)")
    return codes[name]


def eval_basis(kind: str, support_radius: float, distance: float) -> float:
    """bindings.cpp:199-204 -> eval_basis (rbf.cpp:52-54)."""
    lib = capi.load_library()
    return lib.im_eval_basis(capi.basis(_kind(kind), support_radius), float(distance))


def solve_weights(points, displacements, kind="c2", support_radius=1.0):
    """bindings.cpp:205-219 -> solve_weights (rbf.cpp:144-193); list of [x,y,z]."""
    return _context().solve_weights(points, displacements, _kind(kind), support_radius).tolist()


def eval_interpolant(points, alpha, kind, support_radius, query):
    """bindings.cpp:220-232 -> eval_interpolant (rbf.cpp:195-203) for one query."""
    out = _context().eval_interpolant(points, alpha, _kind(kind), support_radius, [query],
                                      capi.EXACT)
    return list(out[0])


class Mesh:
    """Node array + named markers + volume elements (the part of the reference
    Mesh the hot path reads, mesh.hpp:42-58).  ``elements``: list of
    (kind, node list) with kind an ElementKind index or name
    (``capi.ELEMENT_KINDS``), or a CSR triple from ``capi.elements_csr``."""

    def __init__(self, dim: int, nodes, markers: dict, elements=(), marker_elements=None):
        self.dim = int(dim)
        self._nodes = capi.xyz(nodes)
        self._markers = {k: [int(i) for i in v] for k, v in markers.items()}
        self._elements = capi.elements_csr(elements)
        # boundary elements per marker (CSR), as read_su2 returns them
        self._marker_elements = dict(marker_elements or {})

    @property
    def num_nodes(self) -> int:
        return len(self._nodes)

    @property
    def num_elements(self) -> int:
        return len(self._elements[0])

    def node(self, i):
        if not 0 <= i < len(self._nodes):
            raise IndexError(i)
        return list(self._nodes[i])

    def nodes(self):
        return [list(p) for p in self._nodes]

    def marker_names(self):
        return list(self._markers)

    def marker_nodes(self, name: str):
        if name not in self._markers:
            raise ValueError(f"mesh has no marker named '{name}'")
        return list(self._markers[name])


class DisplacementField:
    """bindings.cpp:66-85 (mesh_io.hpp:25-34)."""

    def __init__(self, patch: str):
        self.patch = patch
        self._entries: dict[int, tuple] = {}

    def set(self, node: int, dx: float, dy: float, dz: float = 0.0):
        self._entries[int(node)] = (float(dx), float(dy), float(dz))

    def entries(self):
        return dict(self._entries)

    def at(self, node: int):
        return self._entries.get(int(node), (0.0, 0.0, 0.0))

    def max_magnitude(self) -> float:
        return max((math.sqrt(x * x + y * y + z * z) for x, y, z in self._entries.values()),
                   default=0.0)


class DeformationConfig:
    """bindings.cpp:87-117 properties (pipeline.hpp:18-23) plus the additive
    fields: support_distance (None = reference D_l = volume_k * target_max_l),
    psi ('linear' | 'c2'), precision ('exact' | 'fp64' | 'fp32')."""

    def __init__(self):
        self.basis = "c2"
        self.support_radius = 1.0
        self.tolerance = 0.1
        self.levels = 5
        self.max_points_per_level = 5000
        self.volume_k = 5.0
        self.fixed_markers: list[str] = []
        self.compute_quality = True  # orthogonality before / after (needs mesh elements)
        self.support_distance = None
        self.psi = "linear"
        self.precision = "exact"


@dataclass
class LevelSummary:
    level: int
    points: int
    achieved_error: float
    cap_hit: bool
    support_distance: float
    touched_nodes: int
    seconds: float
    record: list = field(default_factory=list)  # ConvergenceRecord: (points, error, seconds)


@dataclass
class DeformationReport:
    marker: str
    levels: list = field(default_factory=list)
    target_max: float = 0.0
    surface_max_error: float = 0.0
    surface_mean_error: float = 0.0
    inverted_elements: int = 0
    quality_before: object = None
    quality_after: object = None
    total_seconds: float = 0.0

    @property
    def total_control_points(self) -> int:
        return sum(l.points for l in self.levels)


def read_su2(path: str) -> Mesh:
    """bindings.cpp:149-151 -> read_su2 (mesh_io.cpp:127-259): the reference's
    grammar, validation and ParseError ("path:line: what", ``capi.ParseError``,
    a RuntimeError with ``.line``)."""
    d = _context().read_su2(path)
    return Mesh(d["dim"], d["nodes"], {m["name"]: m["nodes"] for m in d["markers"]}, d["elements"],
                {m["name"]: m["elements"] for m in d["markers"]})


def write_su2(mesh: Mesh, path: str) -> None:
    """bindings.cpp:152-154 -> write_su2 (mesh_io.cpp:269-301)."""
    empty = (np.zeros(0, np.int32), np.zeros(1, np.uint64), np.zeros(0, np.uint64))
    markers = [(name, mesh._marker_elements.get(name, empty)) for name in mesh._markers]
    _context().write_su2(path, mesh.dim, mesh._nodes, mesh._elements, markers)


@dataclass
class QualityReport:
    """bindings.cpp:128-134 (quality.hpp QualityReport)."""
    min_orthogonality_deg: float = 90.0
    mean_orthogonality_deg: float = 90.0
    inverted_count: int = 0
    degenerate_count: int = 0
    element_orthogonality_deg: list = field(default_factory=list)
    element_signed_measure: list = field(default_factory=list)


def orthogonality(mesh: Mesh) -> QualityReport:
    """bindings.cpp:194 -> orthogonality (quality.cpp:150-236), on the device."""
    q = _context().orthogonality(mesh._nodes, mesh._elements)
    return QualityReport(q["min"], q["mean"], q["inverted"], q["degenerate"],
                         q["scores"].tolist(), q["measures"].tolist())


def signed_measures(mesh: Mesh):
    """bindings.cpp:195-197 -> signed_measures (quality.cpp:135-140)."""
    return _context().signed_measures(mesh._nodes, mesh._elements)[0].tolist()


def count_inverted(mesh: Mesh) -> int:
    """count_inverted (quality.cpp:142-148)."""
    return _context().count_inverted(mesh._nodes, mesh._elements)


def _quality(r, k):
    q = r["quality"]
    if q is None:
        return None
    return QualityReport(q[k]["min"], q[k]["mean"], q[k]["inverted"], q[k]["degenerate"])


def deform(mesh: Mesh, displacement: DisplacementField, config: DeformationConfig):
    """bindings.cpp:191-193 -> deform (pipeline.cpp:19-106).  Returns
    (deformed_mesh, report); the input mesh is left unchanged."""
    patch = mesh.marker_nodes(displacement.patch)
    if not patch:
        raise ValueError(f"marker '{displacement.patch}' has no nodes")
    pinned = [n for name in config.fixed_markers for n in mesh.marker_nodes(name)]
    disp = np.array([displacement.at(n) for n in patch], dtype=np.float64).reshape(-1, 3)
    D = -1.0 if config.support_distance is None else float(config.support_distance)
    r = _context().deform(mesh._nodes, mesh.dim, patch, disp, pinned, config.tolerance,
                          config.levels, config.max_points_per_level, _kind(config.basis),
                          config.support_radius, config.volume_k, D,
                          1 if config.psi in ("c2", "wendland_c2") else 0,
                          _precision(config.precision),
                          elements=mesh._elements,
                          compute_quality=config.compute_quality and mesh.num_elements > 0)
    out = Mesh(mesh.dim, r["nodes"], mesh._markers, mesh._elements, mesh._marker_elements)
    rep = DeformationReport(marker=displacement.patch, target_max=r["target_max"],
                            surface_max_error=r["surface_max_error"],
                            surface_mean_error=r["surface_mean_error"],
                            inverted_elements=int(r["inverted_elements"]),
                            quality_before=_quality(r, 0), quality_after=_quality(r, 1),
                            total_seconds=r["total_seconds"])
    for l in range(len(r["points"])):
        pts, err, sec = r["records"][l]
        rep.levels.append(LevelSummary(l, int(r["points"][l]), float(r["achieved"][l]),
                                       bool(r["cap_hit"][l]), float(r["support"][l]),
                                       int(r["touched"][l]), float(r["seconds"][l]),
                                       [(int(a), float(b), float(c)) for a, b, c in
                                        zip(pts, err, sec)]))
    return out, rep
