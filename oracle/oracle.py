"""CPU ORACLE for arXiv 2509.13230 -- ctypes wrapper around oracle/fmo.c.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this module.  The product package
``paper_2509_13230_b200`` never imports it, and this module never imports the product.

Every function here is a thin marshalling layer; the arithmetic lives in ``fmo.c`` (fp64,
libm ``log``/``log1p``, ``-ffp-contract=off``), which cites PAPER.md lines per step.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fmo.c")
_HDR = os.path.join(_HERE, "fmo.h")
_LIB = os.path.join(_HERE, "libfmo.so")

UBCM, ECM = 0, 1
_MODELS = {"ubcm": UBCM, "ecm": ECM, UBCM: UBCM, ECM: ECM}
UNDIRECTED, BIPARTITE, DIRECTED = 0, 1, 2
_KINDS = {"undirected": UNDIRECTED, "bipartite": BIPARTITE, "directed": DIRECTED, 0: 0, 1: 1, 2: 2}

CFLAGS = ["-O2", "-std=gnu11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread"]


def build(force: bool = False) -> str:
    """Compile libfmo.so with gcc (plain C, no FMA contraction)."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= max(os.path.getmtime(_SRC), os.path.getmtime(_HDR))):
        return _LIB
    tmp = _LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
    os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    L = C.CDLL(build())
    i32p, i64p, u32p, u64p, f64p = (C.POINTER(C.c_int32), C.POINTER(C.c_int64), C.POINTER(C.c_uint32),
                                    C.POINTER(C.c_uint64), C.POINTER(C.c_double))
    vp = C.c_void_p
    L.fmo_philox4x32_10.argtypes = [u32p, u32p, u32p]
    L.fmo_philox4x32_10.restype = None
    L.fmo_u01.argtypes = [C.c_uint32]
    L.fmo_u01.restype = C.c_double
    L.fmo_skip.argtypes = [C.c_uint32, C.c_double]
    L.fmo_skip.restype = C.c_int64
    L.fmo_plan_create.argtypes = [C.c_int, C.c_int64, f64p, f64p, C.c_int64, C.POINTER(vp)]
    L.fmo_plan_create.restype = C.c_int
    L.fmo_plan_create2.argtypes = [C.c_int, C.c_int, C.c_int64, f64p, f64p, C.c_int64, f64p, f64p, C.c_int64,
                                   C.POINTER(vp)]
    L.fmo_plan_create2.restype = C.c_int
    L.fmo_plan_nc.argtypes = [vp]
    L.fmo_plan_nc.restype = C.c_int64
    L.fmo_plan_export_cand.argtypes = [vp, i32p, f64p, f64p, f64p, i32p]
    L.fmo_plan_export_cand.restype = None
    L.fmo_bruteforce2.argtypes = [C.c_int, C.c_int, C.c_int64, f64p, f64p, C.c_int64, f64p, f64p, C.c_uint64,
                                  C.c_int64, C.POINTER(vp)]
    L.fmo_bruteforce2.restype = C.c_int
    L.fmo_expected2.argtypes = [C.c_int, C.c_int, C.c_int64, f64p, f64p, C.c_int64, f64p, f64p, f64p, f64p, f64p,
                                f64p]
    L.fmo_expected2.restype = None
    L.fmo_plan_free.argtypes = [vp]
    L.fmo_plan_free.restype = None
    L.fmo_plan_n.argtypes = [vp]
    L.fmo_plan_n.restype = C.c_int64
    L.fmo_plan_nseg.argtypes = [vp]
    L.fmo_plan_nseg.restype = C.c_int64
    L.fmo_plan_F.argtypes = [vp]
    L.fmo_plan_F.restype = C.c_int
    L.fmo_plan_export.argtypes = [vp, i32p, f64p, f64p, f64p, u64p, i32p, i32p, i32p, i32p, f64p, f64p, f64p, f64p,
                                  f64p, f64p]
    L.fmo_plan_export.restype = None
    L.fmo_sample.argtypes = [vp, C.c_uint64, C.c_int64, C.c_int64, i32p, C.c_int64, C.c_int, C.POINTER(vp)]
    L.fmo_sample.restype = C.c_int
    L.fmo_sample_ex.argtypes = [vp, C.c_uint64, C.c_int64, C.c_int64, i32p, C.c_int64, C.c_int, C.c_uint32,
                                C.POINTER(vp)]
    L.fmo_sample_ex.restype = C.c_int
    L.fmo_bruteforce.argtypes = [C.c_int, C.c_int64, f64p, f64p, C.c_uint64, C.c_int64, C.POINTER(vp)]
    L.fmo_bruteforce.restype = C.c_int
    L.fmo_result_n_samples.argtypes = [vp]
    L.fmo_result_n_samples.restype = C.c_int64
    L.fmo_result_n_edges.argtypes = [vp]
    L.fmo_result_n_edges.restype = C.c_int64
    L.fmo_result_export.argtypes = [vp, i64p, i32p, i32p, i64p, u32p]
    L.fmo_result_export.restype = None
    L.fmo_result_free.argtypes = [vp]
    L.fmo_result_free.restype = None
    L.fmo_expected.argtypes = [C.c_int, C.c_int64, f64p, f64p, i32p, C.c_int64, C.c_int, f64p, f64p, f64p, f64p]
    L.fmo_expected.restype = None
    L.fmo_expected_edges.argtypes = [C.c_int, C.c_int64, f64p, f64p, C.c_int]
    L.fmo_expected_edges.restype = C.c_double
    L.fmo_richclub_count.argtypes = [C.c_int64, i32p, C.c_int64, i32p, i64p]
    L.fmo_richclub_count.restype = None
    L.fmo_expected_richclub.argtypes = [C.c_int, C.c_int64, f64p, f64p, i32p, f64p, f64p]
    L.fmo_expected_richclub.restype = None
    _lib = L
    return L


def _p(a, ctype):
    return None if a is None else a.ctypes.data_as(C.POINTER(ctype))


def ncores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class OracleError(RuntimeError):
    pass


# ------------------------------------------------------------------------------------------
def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().fmo_philox4x32_10(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(out, C.c_uint32))
    return out


def u01(k: int) -> float:
    return lib().fmo_u01(int(k))


def skip(k: int, h: float) -> int:
    return lib().fmo_skip(int(k), float(h))


# ------------------------------------------------------------------------------------------
@dataclass
class Plan:
    model: int
    n: int
    seg_target: int
    F: int
    perm: np.ndarray
    kappa_s: np.ndarray
    y_s: np.ndarray | None
    ymax: np.ndarray | None
    P: np.ndarray
    seg_u: np.ndarray
    seg_a: np.ndarray
    seg_b: np.ndarray
    seg_sigma: np.ndarray
    seg_h0: np.ndarray
    seg_x0: np.ndarray      # numerator of the initial bound q0 = x0 / d0
    seg_d0: np.ndarray
    seg_omT: np.ndarray
    seg_iomT: np.ndarray
    ly_s: np.ndarray | None
    kind: int = UNDIRECTED
    nc: int = 0
    cperm: np.ndarray | None = None     # candidate (- set) arrays; the row arrays when undirected
    ckappa: np.ndarray | None = None
    cy: np.ndarray | None = None
    cly: np.ndarray | None = None
    excl: np.ndarray | None = None      # directed: candidate rank of each row's own node
    _h: int = 0

    @property
    def n_segments(self) -> int:
        return len(self.seg_u)

    def __del__(self):
        if self._h:
            try:
                lib().fmo_plan_free(C.c_void_p(self._h))
            except Exception:  # pragma: no cover
                pass
            self._h = 0


def sort_plan(x, y=None, seg_target: int = 256, model=None, kind=UNDIRECTED, x2=None, y2=None) -> Plan:
    """a1-a4 of the contract.  kind BIPARTITE: rows (x, y) = the + set,
    candidates (x2, y2) = the - set; DIRECTED: (x, y) out-fitness, (x2, y2) in-fitness."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    if model is None:
        model = UBCM if y is None else ECM
    model = _MODELS[model]
    kind = _KINDS[kind]
    yy = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
    if kind == UNDIRECTED:
        x2a, y2a = x, yy
    else:
        x2a = np.ascontiguousarray(x2, dtype=np.float64)
        y2a = None if y2 is None else np.ascontiguousarray(y2, dtype=np.float64)
    h = C.c_void_p()
    rc = lib().fmo_plan_create2(model, kind, len(x), _p(x, C.c_double), _p(yy, C.c_double), len(x2a),
                                _p(x2a, C.c_double), _p(y2a, C.c_double), int(seg_target), C.byref(h))
    if rc != 0:
        raise OracleError(f"fmo_plan_create failed: {rc}")
    L = lib()
    n = L.fmo_plan_n(h)
    nc = L.fmo_plan_nc(h)
    ns = L.fmo_plan_nseg(h)
    perm = np.empty(n, np.int32)
    ks = np.empty(n, np.float64)
    ys = np.empty(n, np.float64) if model == ECM else None
    ym = np.empty(nc + 1, np.float64) if model == ECM else None
    P = np.empty(nc + 1, np.uint64)
    ly = np.empty(n, np.float64) if model == ECM else None
    su, sa, sb, ss = (np.empty(ns, np.int32) for _ in range(4))
    h0, x0, d0, om, iom = (np.empty(ns, np.float64) for _ in range(5))
    L.fmo_plan_export(h, _p(perm, C.c_int32), _p(ks, C.c_double), _p(ys, C.c_double), _p(ym, C.c_double),
                      _p(P, C.c_uint64), _p(su, C.c_int32), _p(sa, C.c_int32), _p(sb, C.c_int32),
                      _p(ss, C.c_int32), _p(h0, C.c_double), _p(x0, C.c_double), _p(d0, C.c_double),
                      _p(om, C.c_double), _p(iom, C.c_double), _p(ly, C.c_double))
    cperm = np.empty(nc, np.int32)
    ck = np.empty(nc, np.float64)
    cy = np.empty(nc, np.float64) if model == ECM else None
    cly = np.empty(nc, np.float64) if model == ECM else None
    excl = np.empty(n, np.int32)
    L.fmo_plan_export_cand(h, _p(cperm, C.c_int32), _p(ck, C.c_double), _p(cy, C.c_double), _p(cly, C.c_double),
                           _p(excl, C.c_int32))
    return Plan(model, n, int(seg_target) or 256, L.fmo_plan_F(h), perm, ks, ys, ym, P, su, sa, sb, ss, h0, x0, d0,
                om, iom, ly, kind, nc, cperm, ck, cy, cly, excl, h.value)


@dataclass
class Result:
    offsets: np.ndarray           # int64 [n_samples + 1]
    edges: np.ndarray             # int32 [E, 2]  (min id, max id)
    weights: np.ndarray | None    # int32 [E] (ECM)
    draws: int
    landed: int
    accepted: int
    flags: int

    @property
    def n_samples(self) -> int:
        return len(self.offsets) - 1

    def sample(self, s: int):
        a, b = self.offsets[s], self.offsets[s + 1]
        return self.edges[a:b], (None if self.weights is None else self.weights[a:b])


def _collect(h) -> Result:
    L = lib()
    ns = L.fmo_result_n_samples(h)
    ne = L.fmo_result_n_edges(h)
    off = np.empty(ns + 1, np.int64)
    e = np.empty((ne, 2), np.int32)
    w = np.empty(ne, np.int32)
    cnt = np.zeros(3, np.int64)
    fl = np.zeros(1, np.uint32)
    L.fmo_result_export(h, _p(off, C.c_int64), _p(e, C.c_int32), _p(w, C.c_int32), _p(cnt, C.c_int64),
                        _p(fl, C.c_uint32))
    L.fmo_result_free(h)
    return Result(off, e, w, int(cnt[0]), int(cnt[1]), int(cnt[2]), int(fl[0]))


SAMPLE_BETA_REFRESH = 1


def sample(plan: Plan, seed: int, n_samples: int = 1, first_sample: int = 0, rows=None,
           nthreads: int | None = None, refresh: bool = False) -> Result:
    """a5-a6: the method step by step, canonical edge order.  refresh: the ECM
    per-candidate beta_min refresh (R17)."""
    rr = None if rows is None else np.ascontiguousarray(rows, dtype=np.int32)
    h = C.c_void_p()
    rc = lib().fmo_sample_ex(C.c_void_p(plan._h), int(seed) & 0xFFFFFFFFFFFFFFFF, int(first_sample),
                             int(n_samples), _p(rr, C.c_int32), 0 if rr is None else len(rr), int(nthreads or 1),
                             SAMPLE_BETA_REFRESH if refresh else 0, C.byref(h))
    if rc != 0:
        raise OracleError(f"fmo_sample failed: {rc}")
    res = _collect(h)
    if plan.model == UBCM:
        res.weights = None
    return res


def bruteforce(x, y=None, seed: int = 0, n_samples: int = 1, kind=UNDIRECTED, x2=None, y2=None) -> Result:
    """Level-1 oracle: independent Bernoulli per pair (plain definition, Eq. 3-5); bipartite
    pairs (+ i, - j), directed pairs (i, j != i) when kind says so."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    model = UBCM if y is None else ECM
    kind = _KINDS[kind]
    yy = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
    x2a = x if kind == UNDIRECTED else np.ascontiguousarray(x2, dtype=np.float64)
    y2a = yy if kind == UNDIRECTED else (None if y2 is None else np.ascontiguousarray(y2, dtype=np.float64))
    h = C.c_void_p()
    rc = lib().fmo_bruteforce2(model, kind, len(x), _p(x, C.c_double), _p(yy, C.c_double), len(x2a),
                               _p(x2a, C.c_double), _p(y2a, C.c_double), int(seed), int(n_samples), C.byref(h))
    if rc != 0:
        raise OracleError(f"fmo_bruteforce failed: {rc}")
    res = _collect(h)
    if model == UBCM:
        res.weights = None
    return res


def expected(x, y=None, nodes=None, nthreads: int | None = None):
    """Closed forms per node: (k, kvar, s, svar); s/svar None for UBCM."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    model = UBCM if y is None else ECM
    yy = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
    nn = None if nodes is None else np.ascontiguousarray(nodes, dtype=np.int32)
    m = len(x) if nn is None else len(nn)
    k, kv = np.empty(m), np.empty(m)
    s = np.empty(m) if model == ECM else None
    sv = np.empty(m) if model == ECM else None
    lib().fmo_expected(model, len(x), _p(x, C.c_double), _p(yy, C.c_double), _p(nn, C.c_int32), m,
                       int(nthreads or ncores()), _p(k, C.c_double), _p(kv, C.c_double), _p(s, C.c_double),
                       _p(sv, C.c_double))
    return k, kv, s, sv


def expected2(x, y, x2, y2, kind=BIPARTITE):
    """Closed forms of a bipartite/directed ensemble: (kout, kout_var) per + node and (kin, kin_var)
    per - node."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    x2 = np.ascontiguousarray(x2, dtype=np.float64)
    model = UBCM if y is None else ECM
    yy = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
    yy2 = None if y2 is None else np.ascontiguousarray(y2, dtype=np.float64)
    ko, kov = np.empty(len(x)), np.empty(len(x))
    ki, kiv = np.empty(len(x2)), np.empty(len(x2))
    lib().fmo_expected2(model, _KINDS[kind], len(x), _p(x, C.c_double), _p(yy, C.c_double), len(x2),
                        _p(x2, C.c_double), _p(yy2, C.c_double), _p(ko, C.c_double), _p(kov, C.c_double),
                        _p(ki, C.c_double), _p(kiv, C.c_double))
    return ko, kov, ki, kiv


def expected_edges(x, y=None, nthreads: int | None = None) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64)
    model = UBCM if y is None else ECM
    yy = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
    return lib().fmo_expected_edges(model, len(x), _p(x, C.c_double), _p(yy, C.c_double), int(nthreads or ncores()))


def richclub_count(order, edges) -> np.ndarray:
    """Rich club: e_top[m] = edges of the list among the first m nodes of ``order``
    (rank -> node id), m = 0..n (fmo_richclub_count)."""
    order = np.ascontiguousarray(order, dtype=np.int32)
    e = np.ascontiguousarray(np.asarray(edges, dtype=np.int32).reshape(-1, 2))
    out = np.empty(len(order) + 1, dtype=np.int64)
    lib().fmo_richclub_count(len(order), _p(order, C.c_int32), len(e), _p(e, C.c_int32), _p(out, C.c_int64))
    return out


def expected_richclub(x, y, order):
    """E[e_top[m]] and Var[e_top[m]], m = 0..n, for the top-m nodes of ``order`` (independent pairs,
    P:L90-93; fmo_expected_richclub, O(n^2))."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    model = UBCM if y is None else ECM
    yy = None if y is None else np.ascontiguousarray(y, dtype=np.float64)
    order = np.ascontiguousarray(order, dtype=np.int32)
    mean, var = np.empty(len(order) + 1), np.empty(len(order) + 1)
    lib().fmo_expected_richclub(model, len(x), _p(x, C.c_double), _p(yy, C.c_double), _p(order, C.c_int32),
                                _p(mean, C.c_double), _p(var, C.c_double))
    return mean, var


def expected_edges_binned(x, y=None, ratio: float = 1.003) -> float:
    """Approximate sum_{i<j} p_ij by geometric binning of x (and uniform binning of y for ECM).
    Used only to calibrate workload constants (scripts/calibrate_workloads.py); the exact
    expected_edges() checks it at N <= 1e5."""
    x = np.asarray(x, dtype=np.float64)
    xpos = x[x > 0]
    if len(xpos) == 0:
        return 0.0
    lo, hi = np.log(xpos.min()), np.log(xpos.max())
    nb = max(1, int(np.ceil((hi - lo) / np.log(ratio))) + 1)
    idx = np.clip(((np.log(xpos) - lo) / np.log(ratio)).astype(np.int64), 0, nb - 1)
    if y is None:
        cnt = np.bincount(idx, minlength=nb).astype(np.float64)
        sx = np.bincount(idx, weights=xpos, minlength=nb)
        keep = cnt > 0
        cnt, xm = cnt[keep], sx[keep] / cnt[keep]
        X = np.outer(xm, xm)
        P = X / (1.0 + X)
        tot = cnt @ P @ cnt
        tot -= np.sum(cnt * np.diag(P))      # remove i == j terms
        return float(tot / 2.0)
    yv = np.asarray(y, dtype=np.float64)[x > 0]
    ny = 16
    yb = np.clip((yv * ny).astype(np.int64), 0, ny - 1)
    key = idx * ny + yb
    cnt = np.bincount(key, minlength=nb * ny).astype(np.float64)
    sx = np.bincount(key, weights=xpos, minlength=nb * ny)
    sy = np.bincount(key, weights=yv, minlength=nb * ny)
    keep = cnt > 0
    cnt, xm, ym = cnt[keep], sx[keep] / cnt[keep], sy[keep] / cnt[keep]
    tot = 0.0
    B = 2048
    for a in range(0, len(cnt), B):
        xa, ya, ca = xm[a:a + B, None], ym[a:a + B, None], cnt[a:a + B, None]
        t = ya * ym[None, :]
        z = xa * xm[None, :] * t
        P = z / (1.0 - t + z)
        tot += float((ca * P * cnt[None, :]).sum())
    t = ym * ym
    z = xm * xm * t
    tot -= float(np.sum(cnt * z / (1.0 - t + z)))
    return tot / 2.0
