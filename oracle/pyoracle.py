"""oracle/pyoracle.py — TEST INFRASTRUCTURE ONLY (the checker, never the product).

ctypes front-end to the two CPU checkers built by oracle/Makefile:

* ``Oracle("ref")``  — oracle/_ref/libicemorph_ref.so: the UNMODIFIED reference
  sources (/root/reference/proj/src) behind our extern "C" driver ref_capi.cpp.
* ``Oracle("port")`` — oracle/_port/libicemorph_oracle.so: our plain-C
  restatement icemorph_oracle.c.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  Both libraries expose the
same results; the "ref" flavour additionally reports the reference's own
steady_clock timings.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "ref": os.path.join(HERE, "_ref", "libicemorph_ref.so"),
    "port": os.path.join(HERE, "_port", "libicemorph_oracle.so"),
}
KINDS = {"c0": 0, "c2": 1, "c4": 2, "c6": 3}

_sz = C.c_size_t
_d = C.c_double
_pd = C.POINTER(C.c_double)
_psz = C.POINTER(C.c_size_t)
_pi = C.POINTER(C.c_int)


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


def _dp(a):
    return a.ctypes.data_as(_pd) if a is not None else None


def _szp(a):
    return a.ctypes.data_as(_psz) if a is not None else None


def _xyz(a) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if a.ndim == 1:
        a = a.reshape(-1, 3)
    assert a.shape[1] == 3
    return a


def available(flavour: str) -> bool:
    return os.path.exists(LIBS[flavour])


def build(flavour: str = "all") -> None:
    """Build the checkers (the reference flavour needs /root/reference)."""
    import subprocess

    targets = ["port"] if flavour == "port" else ["port", "ref"] if flavour == "all" else [flavour]
    if "ref" in targets and not os.path.isdir(os.environ.get("REF", "/root/reference/proj")):
        targets.remove("ref")
    if targets:
        subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


@dataclass
class GreedyLevel:
    control_indices: np.ndarray
    alpha: np.ndarray
    achieved_error: float
    cap_hit: bool
    target_max: float
    record_points: np.ndarray
    record_error: np.ndarray
    residual: np.ndarray
    elapsed_seconds: float = 0.0


@dataclass
class Multilevel:
    levels: list = field(default_factory=list)  # list[GreedyLevel] (no residual)
    target_max: float = 0.0
    final_residual: np.ndarray | None = None


class Oracle:
    def __init__(self, flavour: str = "ref"):
        self.flavour = flavour
        self.lib = C.CDLL(LIBS[flavour])
        p = "ref_" if flavour == "ref" else "or_"
        self.p = p
        L = self.lib
        getattr(L, p + "last_error").restype = C.c_char_p
        getattr(L, p + "eval_wendland").restype = _d
        getattr(L, p + "eval_wendland").argtypes = [C.c_int, _d]

    def set_sweep_threads(self, n: int) -> None:
        """Port only: threads for the greedy sweep (bit-identical results)."""
        if self.flavour != "port":
            raise ValueError("the reference greedy is single-threaded")
        self.lib.or_set_sweep_threads(C.c_int(int(n)))

    # -- helpers ---------------------------------------------------------
    def _fn(self, name):
        return getattr(self.lib, self.p + name)

    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self._fn("last_error")().decode())

    # -- rbf -------------------------------------------------------------
    def eval_wendland(self, kind, eta: float) -> float:
        return self._fn("eval_wendland")(KINDS.get(kind, kind), float(eta))

    def solve_weights(self, points, disp, kind="c2", R=1.0) -> np.ndarray:
        p, d = _xyz(points), _xyz(disp)
        out = np.zeros_like(p)
        f = self._fn("solve_weights")
        f.argtypes = [_pd, _pd, _sz, C.c_int, _d, _pd]
        self._check(f(_dp(p), _dp(d), len(p), KINDS.get(kind, kind), R, _dp(out)))
        return out

    def eval_interpolant(self, ctrl, alpha, kind, R, queries) -> np.ndarray:
        c, a, q = _xyz(ctrl), _xyz(alpha), _xyz(queries)
        out = np.zeros_like(q)
        f = self._fn("eval_interpolant")
        f.argtypes = [_pd, _pd, _sz, C.c_int, _d, _pd, _sz, _pd]
        self._check(f(_dp(c), _dp(a), len(c), KINDS.get(kind, kind), R, _dp(q), len(q), _dp(out)))
        return out

    def assemble_surface_matrix(self, points, kind="c2", R=1.0) -> np.ndarray:
        """ref only: assemble_surface_matrix (rbf.cpp:56-69)."""
        p = _xyz(points)
        out = np.zeros((len(p), len(p)))
        f = self.lib.ref_assemble_surface_matrix
        f.argtypes = [_pd, _sz, C.c_int, _d, _pd]
        self._check(f(_dp(p), len(p), KINDS.get(kind, kind), R, _dp(out)))
        return out

    def cholesky(self) -> "RefCholesky":
        """ref only: the reference's own CholeskyFactor (rbf.cpp:71-121)."""
        return RefCholesky(self)

    # -- greedy ------------------------------------------------------------
    def greedy_level(self, pos, target, tol, cap=5000, kind="c2", R=1.0, level_index=0):
        pos, tgt = _xyz(pos), _xyz(target)
        n = len(pos)
        m = max(1, min(cap, n))
        idx = np.zeros(m, np.uint64)
        alpha = np.zeros((m, 3))
        nc, nrec = _sz(), _sz()
        ach, tmax, el = _d(), _d(), _d()
        caph = C.c_int()
        rp = np.zeros(m, np.uint64)
        re = np.zeros(m)
        rs = np.zeros(m)
        res = np.zeros_like(pos)
        f = self._fn("greedy_level")
        if self.flavour == "ref":
            f.argtypes = [_pd, _pd, _sz, _d, _sz, C.c_int, _d, _sz, _psz, _pd, _psz, _pd, _pi,
                          _pd, _pd, _psz, _pd, _pd, _psz, _pd]
            rc = f(_dp(pos), _dp(tgt), n, tol, cap, KINDS.get(kind, kind), R, level_index,
                   _szp(idx), _dp(alpha), C.byref(nc), C.byref(ach), C.byref(caph),
                   C.byref(tmax), C.byref(el), _szp(rp), _dp(re), _dp(rs), C.byref(nrec),
                   _dp(res))
        else:
            f.argtypes = [_pd, _pd, _sz, _d, _sz, C.c_int, _d, _sz, _psz, _pd, _psz, _pd, _pi,
                          _pd, _psz, _pd, _psz, _pd]
            rc = f(_dp(pos), _dp(tgt), n, tol, cap, KINDS.get(kind, kind), R, level_index,
                   _szp(idx), _dp(alpha), C.byref(nc), C.byref(ach), C.byref(caph),
                   C.byref(tmax), _szp(rp), _dp(re), C.byref(nrec), _dp(res))
        self._check(rc)
        k, r = nc.value, nrec.value
        return GreedyLevel(idx[:k].astype(np.int64), alpha[:k].copy(), ach.value,
                           bool(caph.value), tmax.value, rp[:r].astype(np.int64), re[:r].copy(),
                           res, el.value)

    def run_multilevel(self, pos, target, tol, max_levels=5, cap=5000, kind="c2", R=1.0):
        pos, tgt = _xyz(pos), _xyz(target)
        n = len(pos)
        m = max(1, min(cap, n))
        L = max_levels
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
        f = self._fn("run_multilevel")
        if self.flavour == "ref":
            f.argtypes = [_pd, _pd, _sz, _d, _sz, _sz, C.c_int, _d, _psz, _psz, _psz, _pd, _pd,
                          _pi, _pd, _pd, _psz, _pd, _pd, _pd]
            rc = f(_dp(pos), _dp(tgt), n, tol, max_levels, cap, KINDS.get(kind, kind), R,
                   C.byref(nl), _szp(nc), _szp(idx), _dp(alpha), _dp(ach),
                   caph.ctypes.data_as(_pi), _dp(ltm), _dp(el), _szp(nrec), _dp(rerr),
                   C.byref(tmax), _dp(res))
        else:
            f.argtypes = [_pd, _pd, _sz, _d, _sz, _sz, C.c_int, _d, _psz, _psz, _psz, _pd, _pd,
                          _pi, _pd, _psz, _pd, _pd, _pd]
            rc = f(_dp(pos), _dp(tgt), n, tol, max_levels, cap, KINDS.get(kind, kind), R,
                   C.byref(nl), _szp(nc), _szp(idx), _dp(alpha), _dp(ach),
                   caph.ctypes.data_as(_pi), _dp(ltm), _szp(nrec), _dp(rerr), C.byref(tmax),
                   _dp(res))
        self._check(rc)
        out = Multilevel(target_max=tmax.value, final_residual=res)
        for l in range(nl.value):
            k = int(nc[l])
            r = int(nrec[l])
            out.levels.append(GreedyLevel(idx[l * m:l * m + k].astype(np.int64),
                                          alpha[l * m:l * m + k].copy(), float(ach[l]),
                                          bool(caph[l]), float(ltm[l]), np.arange(1, r + 1),
                                          rerr[l * m:l * m + r].copy(), None, float(el[l])))
        return out

    # -- wall distance / volume ---------------------------------------------
    def build_distance_index(self, nodes, dim, surface, nthreads=1) -> np.ndarray:
        nodes = _xyz(nodes)
        s = np.ascontiguousarray(np.asarray(surface, dtype=np.uint64))
        out = np.zeros(len(nodes))
        f = self._fn("build_distance_index")
        if self.flavour == "ref":
            f.argtypes = [_pd, _sz, C.c_int, _psz, _sz, _pd]
            rc = f(_dp(nodes), len(nodes), dim, _szp(s), len(s), _dp(out))
        else:
            f.argtypes = [_pd, _sz, C.c_int, _psz, _sz, _pd, C.c_int]
            rc = f(_dp(nodes), len(nodes), dim, _szp(s), len(s), _dp(out), nthreads)
        self._check(rc)
        return out

    def update_volume(self, nodes, dist, ctrl, alpha, D, psi_kind=0, kind="c2", R=1.0,
                      nthreads=1):
        nodes, c, a = _xyz(nodes), _xyz(ctrl), _xyz(alpha)
        dist = np.ascontiguousarray(dist, dtype=np.float64)
        n = len(nodes)
        idx = np.zeros(max(n, 1), np.uint64)
        val = np.zeros((max(n, 1), 3))
        cnt = _sz()
        f = self._fn("update_volume")
        f.argtypes = [_pd, _sz, _pd, _pd, _pd, _sz, _d, C.c_int, C.c_int, _d, _psz, _pd, _psz,
                      C.c_int]
        self._check(f(_dp(nodes), n, _dp(dist), _dp(c), _dp(a), len(c), D, psi_kind,
                      KINDS.get(kind, kind), R, _szp(idx), _dp(val), C.byref(cnt), nthreads))
        k = cnt.value
        return idx[:k].astype(np.int64), val[:k].copy()

    def signed_measures(self, nodes, dim, elements):
        """quality.cpp:135-148: (measures, inverted) for a CSR element triple
        (kinds int32, offsets uint64, conn uint64)."""
        nodes = _xyz(nodes)
        k, o, c = elements
        k = np.ascontiguousarray(k, np.int32)
        o = np.ascontiguousarray(o, np.uint64)
        c = np.ascontiguousarray(c if len(c) else [0], np.uint64)
        out = np.zeros(max(len(k), 1))
        inv = _sz()
        f = self._fn("signed_measures")
        f.argtypes = [_pd, _sz, C.c_int, _pi, _psz, _psz, _sz, _pd, _psz]
        self._check(f(_dp(nodes), len(nodes), dim, k.ctypes.data_as(_pi), _szp(o), _szp(c),
                      len(k), _dp(out), C.byref(inv)))
        return out[:len(k)].copy(), int(inv.value)

    def read_su2(self, path: str) -> dict:
        """Reference read_su2 (ref flavour only): same dict as capi.Context.read_su2;
        a ParseError raises OracleError with .line set."""
        assert self.flavour == "ref"
        f = self.lib.ref_read_su2
        f.argtypes = [C.c_char_p, _psz, _pd, _pi, _psz, _psz, C.c_char_p, _psz, _psz, _psz, _pi,
                      _psz, _psz, _psz]
        sizes = np.zeros(6, np.uint64)
        big = np.zeros(1 << 16, np.uint64)  # per-marker counts (<= 65536 markers)
        me, mc, mn = big.copy(), big.copy(), big.copy()
        self._check_su2(f(os.fsencode(path), _szp(sizes), None, None, None, None, None, _szp(me),
                          _szp(mc), _szp(mn), None, None, None, None))
        dim, nn, ne, nc, nm, nb = (int(v) for v in sizes)
        xyz = np.zeros((max(nn, 1), 3))
        k = np.zeros(max(ne, 1), np.int32)
        o = np.zeros(ne + 1, np.uint64)
        c = np.zeros(max(nc, 1), np.uint64)
        names = C.create_string_buffer(nb + 1)
        tme, tmc, tmn = int(me[:nm].sum()), int(mc[:nm].sum()), int(mn[:nm].sum())
        mk = np.zeros(max(tme, 1), np.int32)
        mcnt = np.zeros(max(tme, 1), np.uint64)
        mconn = np.zeros(max(tmc, 1), np.uint64)
        mnodes = np.zeros(max(tmn, 1), np.uint64)
        self._check_su2(f(os.fsencode(path), _szp(sizes), _dp(xyz), k.ctypes.data_as(_pi), _szp(o),
                          _szp(c), names, _szp(me), _szp(mc), _szp(mn), mk.ctypes.data_as(_pi),
                          _szp(mcnt), _szp(mconn), _szp(mnodes)))
        markers, pe, pc, pn = [], 0, 0, 0
        for i, name in enumerate(names.raw[:nb].decode().split("\n")[:nm]):
            e, cc, nd = int(me[i]), int(mc[i]), int(mn[i])
            offs = np.zeros(e + 1, np.uint64)
            offs[1:] = np.cumsum(mcnt[pe:pe + e])
            markers.append(dict(name=name, elements=(mk[pe:pe + e].copy(), offs, mconn[pc:pc + cc].copy()),
                                nodes=mnodes[pn:pn + nd].astype(np.int64)))
            pe, pc, pn = pe + e, pc + cc, pn + nd
        return dict(dim=dim, nodes=xyz[:nn], elements=(k[:ne], o, c[:nc]), markers=markers)

    def roundtrip_su2(self, src: str, dst: str):
        """Reference write_su2(read_su2(src)) into dst, in a separate process
        (oracle/_ref/ref_su2_tool): the reference's ostream writer must not run
        in a process with numpy loaded."""
        import subprocess

        tool = os.path.join(HERE, "_ref", "ref_su2_tool")
        r = subprocess.run([tool, "roundtrip", src, dst], capture_output=True, text=True)
        if r.returncode:
            raise OracleError(3, r.stderr.strip())

    def _check_su2(self, rc):
        if rc == 4:
            e = OracleError(rc, self.lib.ref_last_error().decode())
            self.lib.ref_last_error_line.restype = C.c_size_t
            e.line = int(self.lib.ref_last_error_line())
            raise e
        self._check(rc)

    def orthogonality(self, nodes, dim, elements):
        """quality.cpp:150-236: dict(scores, measures, min, mean, inverted, degenerate)."""
        nodes = _xyz(nodes)
        k, o, c = elements
        k = np.ascontiguousarray(k, np.int32)
        o = np.ascontiguousarray(o, np.uint64)
        c = np.ascontiguousarray(c if len(c) else [0], np.uint64)
        sc, me = np.zeros(max(len(k), 1)), np.zeros(max(len(k), 1))
        mn, mean = _d(), _d()
        inv, deg = _sz(), _sz()
        f = self._fn("orthogonality")
        f.argtypes = [_pd, _sz, C.c_int, _pi, _psz, _psz, _sz, _pd, _pd, C.POINTER(_d),
                      C.POINTER(_d), _psz, _psz]
        self._check(f(_dp(nodes), len(nodes), dim, k.ctypes.data_as(_pi), _szp(o), _szp(c), len(k),
                      _dp(sc), _dp(me), C.byref(mn), C.byref(mean), C.byref(inv), C.byref(deg)))
        return dict(scores=sc[:len(k)].copy(), measures=me[:len(k)].copy(), min=mn.value,
                    mean=mean.value, inverted=int(inv.value), degenerate=int(deg.value))

    def deform(self, nodes, dim, patch, disp, pinned=(), tol=0.1, max_levels=5, cap=5000,
               kind="c2", R=1.0, volume_k=5.0, elements=None):
        """Reference deform() (ref flavour only).  With ``elements`` (CSR
        triple) the result carries ``inverted_elements`` (pipeline.cpp:101)."""
        assert self.flavour == "ref"
        nodes, disp = _xyz(nodes), _xyz(disp)
        patch = np.ascontiguousarray(patch, dtype=np.uint64)
        pinned = np.ascontiguousarray(np.asarray(pinned, dtype=np.uint64).reshape(-1))
        out = np.zeros_like(nodes)
        L = max_levels
        pts, tch = np.zeros(L, np.uint64), np.zeros(L, np.uint64)
        sup, ach = np.zeros(L), np.zeros(L)
        caph = np.zeros(L, np.int32)
        nl = _sz()
        tmax, smax, smean, tsec = _d(), _d(), _d(), _d()
        if elements is None:
            elements = (np.zeros(0, np.int32), np.zeros(1, np.uint64), np.zeros(1, np.uint64))
        ek = np.ascontiguousarray(elements[0], np.int32)
        eo = np.ascontiguousarray(elements[1], np.uint64)
        ec = np.ascontiguousarray(elements[2] if len(elements[2]) else [0], np.uint64)
        inv = _sz()
        f = self.lib.ref_deform_elements
        f.argtypes = [_pd, _sz, C.c_int, _psz, _sz, _pd, _psz, _sz, _d, _sz, _sz, C.c_int, _d,
                      _d, _pd, _psz, _psz, _psz, _pd, _pd, _pi, _pd, _pd, _pd, _pd, _pi, _psz,
                      _psz, _sz, _psz]
        self._check(f(_dp(nodes), len(nodes), dim, _szp(patch), len(patch), _dp(disp),
                      _szp(pinned) if len(pinned) else None, len(pinned), tol, max_levels, cap,
                      KINDS.get(kind, kind), R, volume_k, _dp(out), C.byref(nl), _szp(pts),
                      _szp(tch), _dp(sup), _dp(ach), caph.ctypes.data_as(_pi), C.byref(tmax),
                      C.byref(smax), C.byref(smean), C.byref(tsec), ek.ctypes.data_as(_pi),
                      _szp(eo), _szp(ec), len(ek), C.byref(inv)))
        k = nl.value
        return dict(nodes=out, points=pts[:k].astype(np.int64), touched=tch[:k].astype(np.int64),
                    support=sup[:k].copy(), achieved=ach[:k].copy(),
                    cap_hit=caph[:k].astype(bool), target_max=tmax.value,
                    surface_max_error=smax.value, surface_mean_error=smean.value,
                    total_seconds=tsec.value, inverted_elements=int(inv.value))


class RefCholesky:
    """The reference CholeskyFactor through oracle/_ref (ref_cholesky_*)."""

    def __init__(self, orc: Oracle):
        L = orc.lib
        self.o, self.L = orc, L
        L.ref_cholesky_create.restype = C.c_void_p
        L.ref_cholesky_destroy.argtypes = [C.c_void_p]
        L.ref_cholesky_size.argtypes = [C.c_void_p]
        L.ref_cholesky_size.restype = _sz
        L.ref_cholesky_smallest_pivot.argtypes = [C.c_void_p]
        L.ref_cholesky_smallest_pivot.restype = _d
        L.ref_cholesky_append.argtypes = [C.c_void_p, _pd, _sz]
        L.ref_cholesky_solve.argtypes = [C.c_void_p, _pd, _sz, _pd, _sz]
        self.h = L.ref_cholesky_create()

    def size(self) -> int:
        return int(self.L.ref_cholesky_size(self.h))

    def smallest_pivot(self) -> float:
        return float(self.L.ref_cholesky_smallest_pivot(self.h))

    def append(self, column) -> None:
        c = np.ascontiguousarray(column, dtype=np.float64).ravel()
        self.o._check(self.L.ref_cholesky_append(self.h, _dp(c), len(c)))

    def solve(self, rhs) -> np.ndarray:
        r = np.ascontiguousarray(rhs, dtype=np.float64).ravel()
        x = np.zeros(self.size())
        self.o._check(self.L.ref_cholesky_solve(self.h, _dp(r), len(r), _dp(x), len(x)))
        return x

    def __del__(self):
        try:
            self.L.ref_cholesky_destroy(self.h)
        except Exception:
            pass
