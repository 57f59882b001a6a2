"""ctypes binding of the C-ABI in include/icemorph_b200.h.

This is the thin Python door onto the CUDA library built in-tree at
``paper_2107_13887_b200/libicemorph_b200.so``.  There is no fallback: if the
library is missing, or the device is not an sm_100 GPU, every call raises.
Errors carry the reference's exception text and map onto the reference's
exception types as pybind11 would raise them (``ValueError`` for
std::invalid_argument, ``SolveError`` (a RuntimeError) for
icemorph::SolveError).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import threading
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IMB_LIB") or os.path.join(HERE, "libicemorph_b200.so")  # IMB_LIB: development override
KINDS = {"c0": 0, "c2": 1, "c4": 2, "c6": 3}
PSI = {"linear": 0, "c2": 1, "wendland_c2": 1}
EXACT, FP64, FP32 = 0, 1, 2  # IM_EXACT, IM_FP64, IM_FP32

_sz = C.c_size_t
_d = C.c_double
_pd = C.POINTER(C.c_double)
_psz = C.POINTER(C.c_size_t)
_pi = C.POINTER(C.c_int)


class SolveError(RuntimeError):
    """icemorph::SolveError (rbf.hpp:13-16)."""


class ParseError(RuntimeError):
    """icemorph::ParseError (mesh_io.hpp:14-21): "path:line: what"; .line."""

    def __init__(self, msg: str, line: int):
        super().__init__(msg)
        self.line = line


class IcemorphRuntimeError(RuntimeError):
    pass


class Basis(C.Structure):
    _fields_ = [("kind", C.c_int), ("support_radius", C.c_double)]


class GreedyConfigC(C.Structure):
    _fields_ = [("tolerance", C.c_double), ("max_levels", C.c_size_t),
                ("max_points_per_level", C.c_size_t), ("basis", Basis)]


class WallFunctionC(C.Structure):
    _fields_ = [("reduction_factor", C.c_double), ("support_distance", C.c_double),
                ("psi_kind", C.c_int)]


class DeformConfigC(C.Structure):
    _fields_ = [("greedy", GreedyConfigC), ("volume_k", C.c_double),
                ("support_distance", C.c_double), ("psi_kind", C.c_int), ("precision", C.c_int),
                ("element_kinds", C.POINTER(C.c_int)), ("element_offsets", C.POINTER(C.c_size_t)),
                ("element_nodes", C.POINTER(C.c_size_t)), ("n_elements", C.c_size_t),
                ("compute_quality", C.c_int), ("record_error", C.POINTER(C.c_double)),
                ("record_seconds", C.POINTER(C.c_double)), ("record_stride", C.c_size_t)]


class QualityReportC(C.Structure):
    _fields_ = [("min_orthogonality_deg", C.c_double), ("mean_orthogonality_deg", C.c_double),
                ("inverted_count", C.c_size_t), ("degenerate_count", C.c_size_t)]


class DeformReportC(C.Structure):
    _fields_ = [("n_levels", C.c_size_t), ("target_max", C.c_double),
                ("surface_max_error", C.c_double), ("surface_mean_error", C.c_double),
                ("total_seconds", C.c_double), ("greedy_seconds", C.c_double),
                ("distance_seconds", C.c_double), ("volume_seconds", C.c_double),
                ("inverted_elements", C.c_size_t), ("has_quality", C.c_int),
                ("quality_before", QualityReportC), ("quality_after", QualityReportC)]


_lib = None
_lib_lock = threading.Lock()


def load_library() -> C.CDLL:
    """Load libicemorph_b200.so (raises if it was not built)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise IcemorphRuntimeError(
                    f"{LIB_PATH} is missing: build it with __graft_entry__.build() or "
                    "`make -C paper_2107_13887_b200`")
            lib = C.CDLL(LIB_PATH)
            _declare(lib)
            _lib = lib
    return _lib


EXPORTS = [
    "im_context_create", "im_context_destroy", "im_last_error", "im_last_device_ms",
    "im_last_transfer_bytes", "im_count_pairs",
    "im_version", "im_eval_wendland", "im_eval_basis", "im_make_wall_function",
    "im_eval_wall_function", "im_solve_weights", "im_eval_interpolant", "im_greedy_level",
    "im_run_multilevel", "im_build_distance_index", "im_signed_measures", "im_count_inverted", "im_orthogonality",
    "im_su2_read", "im_su2_write", "im_mesh_destroy", "im_mesh_sizes", "im_mesh_nodes",
    "im_mesh_elements", "im_mesh_marker_sizes", "im_mesh_marker", "im_last_error_line", "im_update_volume", "im_deform",
    "im_volume_plan_create", "im_volume_plan_destroy", "im_volume_plan_set_controls",
    "im_volume_plan_run", "im_volume_plan_reset_field", "im_volume_plan_download_field",
    "im_volume_plan_distances", "im_volume_plan_set_level", "im_volume_plan_run_steps",
    "im_volume_plan_count_support", "im_bench_backward_chain", "im_assemble_surface_matrix",
    "im_cholesky_create", "im_cholesky_destroy", "im_cholesky_size", "im_cholesky_smallest_pivot",
    "im_cholesky_append", "im_cholesky_solve", "im_volume_plan_bench_passes",
]


def _declare(L):
    L.im_context_create.argtypes = [C.POINTER(C.c_void_p), C.c_int]
    L.im_context_destroy.argtypes = [C.c_void_p]
    L.im_last_error.argtypes = [C.c_void_p]
    L.im_last_error.restype = C.c_char_p
    L.im_last_device_ms.argtypes = [C.c_void_p]
    L.im_last_device_ms.restype = C.c_double
    L.im_last_transfer_bytes.argtypes = [C.c_void_p, C.POINTER(C.c_ulonglong),
                                         C.POINTER(C.c_ulonglong)]
    L.im_last_transfer_bytes.restype = None
    L.im_count_pairs.argtypes = [C.c_void_p, C.c_int]
    L.im_count_pairs.restype = C.c_ulonglong
    L.im_version.restype = C.c_char_p
    L.im_eval_wendland.argtypes = [C.c_int, _d]
    L.im_eval_wendland.restype = _d
    L.im_eval_basis.argtypes = [Basis, _d]
    L.im_eval_basis.restype = _d
    L.im_make_wall_function.argtypes = [_d, _d, C.POINTER(WallFunctionC)]
    L.im_eval_wall_function.argtypes = [C.POINTER(WallFunctionC), _d]
    L.im_eval_wall_function.restype = _d
    L.im_solve_weights.argtypes = [C.c_void_p, _pd, _pd, _sz, Basis, _pd]
    L.im_eval_interpolant.argtypes = [C.c_void_p, _pd, _pd, _sz, Basis, _pd, _sz, C.c_int, _pd]
    L.im_greedy_level.argtypes = [C.c_void_p, _pd, _pd, _sz, C.POINTER(GreedyConfigC), _sz,
                                  _psz, _pd, _psz, _pd, _pi, _pd, _pd, _psz, _pd, _pd, _psz, _pd]
    L.im_run_multilevel.argtypes = [C.c_void_p, _pd, _pd, _sz, C.POINTER(GreedyConfigC), _psz,
                                    _psz, _psz, _pd, _pd, _pi, _pd, _pd, _psz, _pd, _pd, _pd]
    L.im_build_distance_index.argtypes = [C.c_void_p, _pd, _sz, C.c_int, _psz, _sz, _pd]
    L.im_signed_measures.argtypes = [C.c_void_p, _pd, _sz, _pi, _psz, _psz, _sz, _pd, _psz]
    L.im_count_inverted.argtypes = [C.c_void_p, _pd, _sz, _pi, _psz, _psz, _sz, _psz]
    L.im_su2_read.argtypes = [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]
    L.im_mesh_destroy.argtypes = [C.c_void_p]
    L.im_mesh_sizes.argtypes = [C.c_void_p, _pi, _psz, _psz, _psz, _psz]
    L.im_mesh_nodes.argtypes = [C.c_void_p, _pd]
    L.im_mesh_elements.argtypes = [C.c_void_p, _pi, _psz, _psz]
    L.im_mesh_marker_sizes.argtypes = [C.c_void_p, _sz, _psz, _psz, _psz, _psz]
    L.im_mesh_marker.argtypes = [C.c_void_p, _sz, C.c_char_p, _pi, _psz, _psz, _psz]
    L.im_last_error_line.argtypes = [C.c_void_p]
    L.im_last_error_line.restype = _sz
    L.im_su2_write.argtypes = [C.c_void_p, C.c_char_p, C.c_int, _pd, _sz, _pi, _psz, _psz, _sz, _sz,
                               C.POINTER(C.c_char_p), C.POINTER(_pi), C.POINTER(_psz),
                               C.POINTER(_psz), _psz]
    L.im_orthogonality.argtypes = [C.c_void_p, _pd, _sz, _pi, _psz, _psz, _sz, _pd, _pd,
                                   C.POINTER(QualityReportC)]
    L.im_update_volume.argtypes = [C.c_void_p, _pd, _sz, _pd, _pd, _pd, _sz,
                                   C.POINTER(WallFunctionC), Basis, C.c_int, _psz, _pd, _psz]
    L.im_deform.argtypes = [C.c_void_p, _pd, _sz, C.c_int, _psz, _sz, _pd, _psz, _sz,
                            C.POINTER(DeformConfigC), _pd, C.POINTER(DeformReportC), _psz, _pd,
                            _pi, _pd, _psz, _pd]
    L.im_volume_plan_create.argtypes = [C.c_void_p, _pd, _sz, C.c_int, _psz, _sz, _d,
                                        C.POINTER(C.c_void_p)]
    L.im_volume_plan_destroy.argtypes = [C.c_void_p]
    L.im_volume_plan_set_controls.argtypes = [C.c_void_p, _pd, _pd, _sz]
    L.im_volume_plan_run.argtypes = [C.c_void_p, C.POINTER(WallFunctionC), Basis, C.c_int, _psz,
                                     _pd]
    L.im_volume_plan_reset_field.argtypes = [C.c_void_p]
    L.im_volume_plan_download_field.argtypes = [C.c_void_p, _pd]
    L.im_volume_plan_distances.argtypes = [C.c_void_p, _pd]
    L.im_volume_plan_set_level.argtypes = [C.c_void_p, C.c_int, _pd, _pd, _sz, _d, C.c_int, Basis,
                                           C.c_int]
    L.im_volume_plan_run_steps.argtypes = [C.c_void_p, Basis, C.c_int, C.c_int, C.c_int, _pd]
    L.im_volume_plan_count_support.argtypes = [C.c_void_p, C.c_int, Basis,
                                               C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong)]
    L.im_bench_backward_chain.argtypes = [C.c_void_p, C.c_int, C.c_int, _pd]
    L.im_volume_plan_bench_passes.argtypes = [C.c_void_p, _d, _d, C.c_int, _pd]
    L.im_assemble_surface_matrix.argtypes = [C.c_void_p, _pd, _sz, Basis, _pd]
    L.im_cholesky_create.argtypes = [C.c_void_p, C.POINTER(C.c_void_p)]
    L.im_cholesky_destroy.argtypes = [C.c_void_p]
    L.im_cholesky_size.argtypes = [C.c_void_p]
    L.im_cholesky_size.restype = _sz
    L.im_cholesky_smallest_pivot.argtypes = [C.c_void_p]
    L.im_cholesky_smallest_pivot.restype = _d
    L.im_cholesky_append.argtypes = [C.c_void_p, _pd, _sz]
    L.im_cholesky_solve.argtypes = [C.c_void_p, _pd, _sz, _pd, _sz]


def _dp(a):
    return None if a is None else a.ctypes.data_as(_pd)


def _szp(a):
    return None if a is None else a.ctypes.data_as(_psz)


def xyz(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.ndim == 1:
        a = a.reshape(-1, 3)
    if a.ndim != 2 or a.shape[1] != 3:
        raise ValueError("expected an (n, 3) array of points")
    return a


def basis(kind="c2", R=1.0) -> Basis:
    k = KINDS[kind.lower()] if isinstance(kind, str) else int(kind)
    return Basis(k, float(R))


@dataclass
class LevelResult:
    control_indices: np.ndarray
    alpha: np.ndarray
    achieved_error: float
    cap_hit: bool
    target_max: float
    elapsed_seconds: float
    record_points: np.ndarray
    record_error: np.ndarray
    record_seconds: np.ndarray | None
    residual: np.ndarray | None


@dataclass
class MultilevelResult:
    levels: list = field(default_factory=list)
    target_max: float = 0.0
    final_residual: np.ndarray | None = None


class Context:
    """One CUDA stream + scratch on one device (im_context)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.im_context_create(C.byref(h), device)
        self.h = h
        if rc != 0:
            msg = self.lib.im_last_error(h).decode() if h else "context creation failed"
            self.close()
            raise IcemorphRuntimeError(msg)

    def close(self):
        if getattr(self, "h", None):
            self.lib.im_context_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def _check(self, rc: int):
        if rc == 0:
            return
        msg = self.lib.im_last_error(self.h).decode()
        if rc == 1:
            raise ValueError(msg)
        if rc == 2:
            raise SolveError(msg)
        if rc == 4:
            raise ParseError(msg, int(self.lib.im_last_error_line(self.h)))
        raise IcemorphRuntimeError(msg)

    @property
    def last_device_ms(self) -> float:
        return self.lib.im_last_device_ms(self.h)

    @property
    def last_transfer_bytes(self) -> tuple:
        """(host->device, device->host) bytes of the last update_volume call."""
        a, b = C.c_ulonglong(), C.c_ulonglong()
        self.lib.im_last_transfer_bytes(self.h, C.byref(a), C.byref(b))
        return a.value, b.value

    def count_pairs(self, enable: bool) -> int:
        """Switch the exact kernels' evaluated-pair counter; returns the count
        accumulated since the previous call."""
        return int(self.lib.im_count_pairs(self.h, 1 if enable else 0))

    # -- rbf ---------------------------------------------------------------
    def solve_weights(self, points, displacements, kind="c2", R=1.0) -> np.ndarray:
        p, d = xyz(points), xyz(displacements)
        if len(p) != len(d):
            raise ValueError("point and displacement counts differ")
        out = np.zeros_like(p)
        self._check(self.lib.im_solve_weights(self.h, _dp(p), _dp(d), len(p), basis(kind, R),
                                              _dp(out)))
        return out

    def eval_interpolant(self, ctrl, alpha, kind, R, queries, precision=EXACT) -> np.ndarray:
        c, a, q = xyz(ctrl), xyz(alpha), xyz(queries)
        out = np.zeros_like(q)
        self._check(self.lib.im_eval_interpolant(self.h, _dp(c), _dp(a), len(c), basis(kind, R),
                                                 _dp(q), len(q), precision, _dp(out)))
        return out

    def assemble_surface_matrix(self, points, kind="c2", R=1.0) -> np.ndarray:
        """assemble_surface_matrix (rbf.hpp:35-36, rbf.cpp:56-69): n x n, row-major."""
        p = xyz(points)
        out = np.zeros((len(p), len(p)))
        self._check(self.lib.im_assemble_surface_matrix(self.h, _dp(p), len(p), basis(kind, R),
                                                        _dp(out)))
        return out

    def cholesky(self) -> "CholeskyFactor":
        return CholeskyFactor(self)

    # -- greedy --------------------------------------------------------------
    def greedy_level(self, pos, target, tol, cap=5000, kind="c2", R=1.0, level_index=0,
                     max_levels=1) -> LevelResult:
        pos, tgt = xyz(pos), xyz(target)
        n = len(pos)
        if len(tgt) != n:
            raise ValueError("target size does not match surface size")
        m = max(1, min(cap, n))
        cfg = GreedyConfigC(tol, max_levels, cap, basis(kind, R))
        idx = np.zeros(m, np.uint64)
        alpha = np.zeros((m, 3))
        rp = np.zeros(m, np.uint64)
        re = np.zeros(m)
        rs = np.zeros(m)
        res = np.zeros_like(pos)
        nc, nrec = _sz(), _sz()
        ach, tmax, el = _d(), _d(), _d()
        caph = C.c_int()
        self._check(self.lib.im_greedy_level(
            self.h, _dp(pos), _dp(tgt), n, C.byref(cfg), level_index, _szp(idx), _dp(alpha),
            C.byref(nc), C.byref(ach), C.byref(caph), C.byref(tmax), C.byref(el), _szp(rp),
            _dp(re), _dp(rs), C.byref(nrec), _dp(res)))
        k, r = nc.value, nrec.value
        return LevelResult(idx[:k].astype(np.int64), alpha[:k].copy(), ach.value,
                           bool(caph.value), tmax.value, el.value, rp[:r].astype(np.int64),
                           re[:r].copy(), rs[:r].copy(), res)

    def run_multilevel(self, pos, target, tol, max_levels=5, cap=5000, kind="c2",
                       R=1.0) -> MultilevelResult:
        pos, tgt = xyz(pos), xyz(target)
        n = len(pos)
        m = max(1, min(cap, n))
        L = max_levels
        cfg = GreedyConfigC(tol, max_levels, cap, basis(kind, R))
        nl = _sz()
        nc = np.zeros(L, np.uint64)
        idx = np.zeros(L * m, np.uint64)
        alpha = np.zeros((L * m, 3))
        ach = np.zeros(L)
        caph = np.zeros(L, np.int32)
        ltm = np.zeros(L)
        el = np.zeros(L)
        nrec = np.zeros(L, np.uint64)
        rerr = np.zeros(L * m)
        tmax = _d()
        res = np.zeros_like(pos)
        self._check(self.lib.im_run_multilevel(
            self.h, _dp(pos), _dp(tgt), n, C.byref(cfg), C.byref(nl), _szp(nc), _szp(idx),
            _dp(alpha), _dp(ach), caph.ctypes.data_as(_pi), _dp(ltm), _dp(el), _szp(nrec),
            _dp(rerr), C.byref(tmax), _dp(res)))
        out = MultilevelResult(target_max=tmax.value, final_residual=res)
        for l in range(nl.value):
            k, r = int(nc[l]), int(nrec[l])
            out.levels.append(LevelResult(idx[l * m:l * m + k].astype(np.int64),
                                          alpha[l * m:l * m + k].copy(), float(ach[l]),
                                          bool(caph[l]), float(ltm[l]), float(el[l]),
                                          np.arange(1, r + 1), rerr[l * m:l * m + r].copy(),
                                          None, None))
        return out

    # -- wall distance / volume ----------------------------------------------
    def build_distance_index(self, nodes, dim, surface) -> np.ndarray:
        nodes = xyz(nodes)
        s = np.ascontiguousarray(np.asarray(surface, dtype=np.uint64))
        out = np.zeros(len(nodes))
        self._check(self.lib.im_build_distance_index(self.h, _dp(nodes), len(nodes), dim,
                                                     _szp(s), len(s), _dp(out)))
        return out

    def update_volume(self, nodes, dist, ctrl, alpha, D, psi_kind=0, kind="c2", R=1.0,
                      precision=EXACT, out=None):
        """update_volume (wall_distance.cpp:46-64): (node ids, values).  ``out``
        = (uint64 ids[n], float64 values[n, 3]) reuses caller buffers (e.g.
        page-locked ones, which the library then fills by direct DMA)."""
        nodes, c, a = xyz(nodes), xyz(ctrl), xyz(alpha)
        dist = np.ascontiguousarray(dist, dtype=np.float64)
        if len(dist) != len(nodes):
            raise ValueError("distance index does not match the mesh")
        n = len(nodes)
        if out is None:
            idx = np.empty(max(n, 1), np.uint64)
            val = np.empty((max(n, 1), 3))
        else:
            idx, val = out
            if len(idx) < n or len(val) < n or idx.dtype != np.uint64 or val.dtype != np.float64:
                raise ValueError("out buffers too small or of the wrong type")
        cnt = _sz()
        wf = WallFunctionC(1.0, D, psi_kind)
        self._check(self.lib.im_update_volume(self.h, _dp(nodes), n, _dp(dist), _dp(c), _dp(a),
                                              len(c), C.byref(wf), basis(kind, R), precision,
                                              _szp(idx), _dp(val), C.byref(cnt)))
        k = cnt.value
        # views of the output buffers (no copy): node ids as int64, values (k, 3)
        return idx[:k].view(np.int64), val[:k]

    def signed_measures(self, nodes, elements):
        """quality.cpp:135-148: (measures, inverted) for ``elements`` =
        (kinds, offsets, conn) CSR (see :func:`elements_csr`)."""
        nodes = xyz(nodes)
        k, o, c = elements
        m = np.zeros(max(len(k), 1))
        inv = _sz()
        self._check(self.lib.im_signed_measures(
            self.h, _dp(nodes), len(nodes), k.ctypes.data_as(_pi), _szp(o), _szp(c), len(k),
            _dp(m), C.byref(inv)))
        return m[:len(k)].copy(), int(inv.value)

    def count_inverted(self, nodes, elements) -> int:
        nodes = xyz(nodes)
        k, o, c = elements
        inv = _sz()
        self._check(self.lib.im_count_inverted(
            self.h, _dp(nodes), len(nodes), k.ctypes.data_as(_pi), _szp(o), _szp(c), len(k),
            C.byref(inv)))
        return int(inv.value)

    def read_su2(self, path: str) -> dict:
        """read_su2 (mesh_io.cpp:127-259): dict(dim, nodes (n, 3), elements CSR,
        markers = [dict(name, elements CSR, nodes)])."""
        h = C.c_void_p()
        self._check(self.lib.im_su2_read(self.h, os.fsencode(path), C.byref(h)))
        try:
            L = self.lib
            dim, nn, ne, nc, nm = C.c_int(), _sz(), _sz(), _sz(), _sz()
            L.im_mesh_sizes(h, C.byref(dim), C.byref(nn), C.byref(ne), C.byref(nc), C.byref(nm))
            nodes = np.zeros((nn.value, 3))
            L.im_mesh_nodes(h, _dp(nodes))
            k = np.zeros(ne.value, np.int32)
            o = np.zeros(ne.value + 1, np.uint64)
            c = np.zeros(max(nc.value, 1), np.uint64)
            L.im_mesh_elements(h, k.ctypes.data_as(_pi), _szp(o), _szp(c))
            markers = []
            for m in range(nm.value):
                ln, me, mc, mn = _sz(), _sz(), _sz(), _sz()
                L.im_mesh_marker_sizes(h, m, C.byref(ln), C.byref(me), C.byref(mc), C.byref(mn))
                name = C.create_string_buffer(ln.value + 1)
                mk = np.zeros(me.value, np.int32)
                mo = np.zeros(me.value + 1, np.uint64)
                mcn = np.zeros(max(mc.value, 1), np.uint64)
                mnd = np.zeros(max(mn.value, 1), np.uint64)
                L.im_mesh_marker(h, m, name, mk.ctypes.data_as(_pi), _szp(mo), _szp(mcn), _szp(mnd))
                markers.append(dict(name=name.value.decode(), elements=(mk, mo, mcn[:mc.value]),
                                    nodes=mnd[:mn.value].astype(np.int64)))
            return dict(dim=dim.value, nodes=nodes, elements=(k, o, c[:nc.value]), markers=markers)
        finally:
            self.lib.im_mesh_destroy(h)

    def write_su2(self, path: str, dim: int, nodes, elements, markers):
        """write_su2 (mesh_io.cpp:269-301); markers = [(name, elements CSR)]."""
        nodes = xyz(nodes)
        k, o, c = elements
        k = np.ascontiguousarray(k, np.int32)
        o = np.ascontiguousarray(o, np.uint64)
        c = np.ascontiguousarray(c if len(c) else [0], np.uint64)
        n = len(markers)
        names = (C.c_char_p * max(n, 1))(*[m[0].encode() for m in markers])
        keep = [(np.ascontiguousarray(m[1][0], np.int32), np.ascontiguousarray(m[1][1], np.uint64),
                 np.ascontiguousarray(m[1][2] if len(m[1][2]) else [0], np.uint64)) for m in markers]
        mk = (_pi * max(n, 1))(*[a.ctypes.data_as(_pi) for a, _, _ in keep])
        mo = (_psz * max(n, 1))(*[_szp(b) for _, b, _ in keep])
        mc = (_psz * max(n, 1))(*[_szp(cc) for _, _, cc in keep])
        mn = np.array([len(a) for a, _, _ in keep] or [0], np.uint64)
        self._check(self.lib.im_su2_write(self.h, os.fsencode(path), int(dim), _dp(nodes), len(nodes),
                                          k.ctypes.data_as(_pi), _szp(o), _szp(c), len(k), n, names,
                                          mk, mo, mc, _szp(mn)))

    def orthogonality(self, nodes, elements):
        """quality.cpp:150-236 on the device: dict(scores, measures, min, mean,
        inverted, degenerate)."""
        nodes = xyz(nodes)
        k, o, c = elements
        sc, me = np.zeros(max(len(k), 1)), np.zeros(max(len(k), 1))
        rep = QualityReportC()
        self._check(self.lib.im_orthogonality(
            self.h, _dp(nodes), len(nodes), k.ctypes.data_as(_pi), _szp(o), _szp(c), len(k),
            _dp(sc), _dp(me), C.byref(rep)))
        return dict(scores=sc[:len(k)].copy(), measures=me[:len(k)].copy(),
                    min=rep.min_orthogonality_deg, mean=rep.mean_orthogonality_deg,
                    inverted=int(rep.inverted_count), degenerate=int(rep.degenerate_count))

    def deform(self, nodes, dim, patch, disp, pinned=(), tol=0.1, max_levels=5, cap=5000,
               kind="c2", R=1.0, volume_k=5.0, support_distance=-1.0, psi_kind=0,
               precision=EXACT, elements=None, compute_quality=False):
        nodes, disp = xyz(nodes), xyz(disp)
        patch = np.ascontiguousarray(patch, dtype=np.uint64)
        pinned = np.ascontiguousarray(np.asarray(pinned, dtype=np.uint64).reshape(-1))
        cfg = DeformConfigC(GreedyConfigC(tol, max_levels, cap, basis(kind, R)), volume_k,
                            support_distance, psi_kind, precision)
        if elements is not None and len(elements[0]):
            ek, eo, ec = elements
            cfg.element_kinds = ek.ctypes.data_as(_pi)
            cfg.element_offsets = _szp(eo)
            cfg.element_nodes = _szp(ec)
            cfg.n_elements = len(ek)
            cfg.compute_quality = int(bool(compute_quality))
        rep = DeformReportC()
        out = np.zeros_like(nodes)
        L = max_levels
        stride = max(1, min(cap, len(patch) + len(pinned)))
        rec_e, rec_s = np.zeros(L * stride), np.zeros(L * stride)
        cfg.record_error, cfg.record_seconds, cfg.record_stride = _dp(rec_e), _dp(rec_s), stride
        pts, tch = np.zeros(L, np.uint64), np.zeros(L, np.uint64)
        ach, sup, sec = np.zeros(L), np.zeros(L), np.zeros(L)
        caph = np.zeros(L, np.int32)
        self._check(self.lib.im_deform(
            self.h, _dp(nodes), len(nodes), dim, _szp(patch), len(patch), _dp(disp),
            _szp(pinned) if len(pinned) else None, len(pinned), C.byref(cfg), _dp(out),
            C.byref(rep), _szp(pts), _dp(ach), caph.ctypes.data_as(_pi), _dp(sup), _szp(tch),
            _dp(sec)))
        k = rep.n_levels
        return dict(nodes=out, points=pts[:k].astype(np.int64), touched=tch[:k].astype(np.int64),
                    support=sup[:k].copy(), achieved=ach[:k].copy(),
                    cap_hit=caph[:k].astype(bool), seconds=sec[:k].copy(),
                    target_max=rep.target_max, surface_max_error=rep.surface_max_error,
                    surface_mean_error=rep.surface_mean_error, total_seconds=rep.total_seconds,
                    greedy_seconds=rep.greedy_seconds, distance_seconds=rep.distance_seconds,
                    volume_seconds=rep.volume_seconds, inverted_elements=rep.inverted_elements,
                    records=[(np.arange(1, int(pts[l]) + 1),
                              rec_e[l * stride:l * stride + int(pts[l])].copy(),
                              rec_s[l * stride:l * stride + int(pts[l])].copy()) for l in range(k)],
                    quality=None if not rep.has_quality else tuple(
                        dict(min=q.min_orthogonality_deg, mean=q.mean_orthogonality_deg,
                             inverted=int(q.inverted_count), degenerate=int(q.degenerate_count))
                        for q in (rep.quality_before, rep.quality_after)))


ELEMENT_KINDS = ("line", "triangle", "quadrilateral", "tetrahedron", "hexahedron", "prism",
                 "pyramid")  # mesh.hpp:15-23 order


class CholeskyFactor:
    """icemorph::CholeskyFactor (rbf.hpp:41-60) resident on the device
    (im_cholesky_*): append(column) grows the factor by one row, solve(rhs)
    returns A^-1 rhs, both bit-identical to rbf.cpp:71-121."""

    def __init__(self, ctx: Context):
        self.ctx = ctx
        h = C.c_void_p()
        ctx._check(ctx.lib.im_cholesky_create(ctx.h, C.byref(h)))
        self.h = h

    def size(self) -> int:
        return int(self.ctx.lib.im_cholesky_size(self.h))

    def smallest_pivot(self) -> float:
        return float(self.ctx.lib.im_cholesky_smallest_pivot(self.h))

    def append(self, column) -> None:
        c = np.ascontiguousarray(column, dtype=np.float64).ravel()
        self.ctx._check(self.ctx.lib.im_cholesky_append(self.h, _dp(c), len(c)))

    def solve(self, rhs) -> np.ndarray:
        r = np.ascontiguousarray(rhs, dtype=np.float64).ravel()
        x = np.zeros(self.size())
        self.ctx._check(self.ctx.lib.im_cholesky_solve(self.h, _dp(r), len(r), _dp(x), len(x)))
        return x

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.im_cholesky_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def elements_csr(elements):
    """Element list -> (kinds int32, offsets uint64, conn uint64) CSR.  Accepts
    a list of (kind, nodes) pairs (kind an int or an ELEMENT_KINDS name) or an
    already-built CSR triple."""
    if isinstance(elements, tuple) and len(elements) == 3 and isinstance(elements[0], np.ndarray):
        k, o, c = elements
        return (np.ascontiguousarray(k, np.int32), np.ascontiguousarray(o, np.uint64),
                np.ascontiguousarray(c, np.uint64))
    kinds, offs, conn = [], [0], []
    for kind, nodes in elements:
        kinds.append(ELEMENT_KINDS.index(kind) if isinstance(kind, str) else int(kind))
        conn.extend(int(i) for i in nodes)
        offs.append(len(conn))
    return (np.asarray(kinds, np.int32), np.asarray(offs, np.uint64),
            np.asarray(conn if conn else [0], np.uint64))


class VolumePlan:
    """Resident volume-update plan (im_volume_plan): mesh + wall distances in
    HBM, one call per level."""

    def __init__(self, ctx: Context, nodes, dim, surface, cutoff=math.inf):
        self.ctx = ctx
        nodes = xyz(nodes)
        s = np.ascontiguousarray(np.asarray(surface, dtype=np.uint64))
        h = C.c_void_p()
        ctx._check(ctx.lib.im_volume_plan_create(ctx.h, _dp(nodes), len(nodes), dim, _szp(s),
                                                 len(s), cutoff, C.byref(h)))
        self.h = h
        self.n = len(nodes)

    def set_controls(self, ctrl, alpha):
        c, a = xyz(ctrl), xyz(alpha)
        self.ctx._check(self.ctx.lib.im_volume_plan_set_controls(self.h, _dp(c), _dp(a), len(c)))

    def run(self, D, psi_kind=0, kind="c2", R=1.0, precision=EXACT):
        wf = WallFunctionC(1.0, D, psi_kind)
        na, ms = _sz(), _d()
        self.ctx._check(self.ctx.lib.im_volume_plan_run(self.h, C.byref(wf), basis(kind, R),
                                                        precision, C.byref(na), C.byref(ms)))
        return na.value, ms.value

    def reset_field(self):
        self.ctx._check(self.ctx.lib.im_volume_plan_reset_field(self.h))

    def field(self) -> np.ndarray:
        out = np.zeros((self.n, 3))
        self.ctx._check(self.ctx.lib.im_volume_plan_download_field(self.h, _dp(out)))
        return out

    def distances(self) -> np.ndarray:
        out = np.zeros(self.n)
        self.ctx._check(self.ctx.lib.im_volume_plan_distances(self.h, _dp(out)))
        return out

    def set_level(self, level, ctrl, alpha, D, psi_kind=0, kind="c2", R=1.0, precision=EXACT):
        c, a = xyz(ctrl), xyz(alpha)
        self.ctx._check(self.ctx.lib.im_volume_plan_set_level(
            self.h, level, _dp(c), _dp(a), len(c), D, psi_kind, basis(kind, R), precision))

    def run_steps(self, steps, kind="c2", R=1.0, precision=EXACT, flush_l2=True) -> dict:
        st = np.zeros(10)
        self.ctx._check(self.ctx.lib.im_volume_plan_run_steps(
            self.h, basis(kind, R), precision, steps, int(flush_l2), _dp(st)))
        return dict(step_ms_total=st[0], kernel_ms_total=st[1], kernel_launches=int(st[2]),
                    launches_per_step=int(st[3]), active=[int(v) for v in st[4:8]])

    def bench_passes(self, cutoff, D, reps=5) -> dict:
        """Wall-distance (K6) and compaction (K7) passes on the resident mesh."""
        st = np.zeros(4)
        self.ctx._check(self.ctx.lib.im_volume_plan_bench_passes(self.h, cutoff, D, reps, _dp(st)))
        return dict(wall_distance_ms=st[0], compaction_ms=st[1], active=int(st[2]),
                    within_cutoff=int(st[3]))

    def count_support(self, level, kind="c2", R=1.0):
        a, b = C.c_ulonglong(), C.c_ulonglong()
        self.ctx._check(self.ctx.lib.im_volume_plan_count_support(self.h, level, basis(kind, R),
                                                                  C.byref(a), C.byref(b)))
        return a.value, b.value

    def close(self):
        if getattr(self, "h", None):
            self.ctx.lib.im_volume_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
