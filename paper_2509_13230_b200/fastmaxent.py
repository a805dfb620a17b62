"""Python binding of the C-ABI in include/fastmaxent.h (ctypes; argument marshalling only).

Every step of the sampler runs in libfastmaxent.so's sm_100a kernels.  There is no CPU fallback:
importing this module raises if the library is missing, and every call raises FastMaxEntError
on a non-OK status (e.g. FM_ERR_CUDA when no device is present).

    plan  = sort_plan(x, y=None, seg_target=256)         # fm_sort_plan   (a1-a4)
    edges = sample_ubcm(plan, seed, n_samples)           # fm_sample_ubcm (a5-a6)
    edges = sample_ecm(plan, seed, n_samples)            # fm_sample_ecm
    edges.edges   -> torch.int32 [E, 2] on the GPU (zero-copy), edges.weights -> [E] (ECM)
    edges.offsets -> numpy int64 [n_samples + 1]
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FM_LIB_VARIANT=<tag> loads libfastmaxent.<tag>.so (an in-tree experimental build, see build.py)
LIB_PATH = os.path.join(_HERE, "libfastmaxent.so" if not os.environ.get("FM_LIB_VARIANT")
                        else f"libfastmaxent.{os.environ['FM_LIB_VARIANT']}.so")

FM_UBCM, FM_ECM = 0, 1
FM_OK, FM_ERR_INVALID, FM_ERR_NOMEM, FM_ERR_CUDA, FM_ERR_BOUND, FM_ERR_STATE = 0, -1, -2, -3, -4, -5
FM_FLAG_WEIGHT_SATURATED, FM_FLAG_SCRATCH_RERUN, FM_FLAG_HOST_TRUNCATED = 1, 2, 4
STATUS_NAMES = {0: "FM_OK", -1: "FM_ERR_INVALID", -2: "FM_ERR_NOMEM", -3: "FM_ERR_CUDA", -4: "FM_ERR_BOUND",
                -5: "FM_ERR_STATE"}
FM_UNDIRECTED, FM_BIPARTITE, FM_DIRECTED = 0, 1, 2
_KINDS = {"undirected": FM_UNDIRECTED, "bipartite": FM_BIPARTITE, "directed": FM_DIRECTED}
SYMBOLS = ["fm_sort_plan", "fm_sort_plan_bipartite", "fm_plan_export_candidates", "fm_sample_degrees", "fm_sample_richclub", "fm_sample_ubcm", "fm_sample_ecm", "fm_sample_ecm_ex", "fm_edges_to_host", "fm_sample_to_host", "fm_plan_get_info",
           "fm_plan_export", "fm_free", "fm_last_error", "fm_abi_version", "fm_timing_enable", "fm_timing_get", "fm_debug_eval", "fm_expected_degrees",
           "fm_pool_trim"]


class FastMaxEntError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class _Edges(C.Structure):
    _fields_ = [("n_samples", C.c_int64), ("n_edges", C.c_int64), ("offsets", C.POINTER(C.c_int64)),
                ("edges", C.c_void_p), ("weights", C.c_void_p), ("draws", C.c_int64), ("landed", C.c_int64),
                ("accepted", C.c_int64), ("segments", C.c_int64), ("chunks", C.c_int64), ("flags", C.c_uint32),
                ("_owner", C.c_void_p)]


class _Counters(C.Structure):
    _fields_ = [("draws", C.c_int64), ("landed", C.c_int64), ("accepted", C.c_int64), ("flags", C.c_uint32)]


class _PlanInfo(C.Structure):
    _fields_ = [("model", C.c_int32), ("kind", C.c_int32), ("n_minus", C.c_int64), ("n", C.c_int64), ("seg_target", C.c_int64), ("F", C.c_int32),
                ("n_segments", C.c_int64), ("n_chunks", C.c_int64), ("est_draws", C.c_int64)]


class _Timing(C.Structure):
    _fields_ = [("plan_ms", C.c_double), ("sample_ms", C.c_double), ("write_ms", C.c_double),
                ("sample_launches", C.c_int64), ("launches", C.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise OSError(f"{LIB_PATH} is missing: build it with `python -m paper_2509_13230_b200.build` "
                      "(nvcc, sm_100a). There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    vp, i64, u64 = C.c_void_p, C.c_int64, C.c_uint64
    L.fm_sort_plan.argtypes = [C.c_int, i64, vp, vp, i64, vp, C.POINTER(vp)]
    L.fm_sort_plan.restype = C.c_int
    L.fm_sort_plan_bipartite.argtypes = [C.c_int, C.c_int, i64, vp, vp, i64, vp, vp, i64, vp, C.POINTER(vp)]
    L.fm_sort_plan_bipartite.restype = C.c_int
    L.fm_plan_export_candidates.argtypes = [vp] * 6
    L.fm_plan_export_candidates.restype = C.c_int
    for f in (L.fm_sample_ubcm, L.fm_sample_ecm):
        f.argtypes = [vp, u64, i64, i64, vp, C.POINTER(_Edges)]
        f.restype = C.c_int
    L.fm_sample_ecm_ex.argtypes = [vp, u64, i64, i64, C.c_uint32, vp, C.POINTER(_Edges)]
    L.fm_sample_ecm_ex.restype = C.c_int
    L.fm_sample_degrees.argtypes = [vp, u64, i64, i64, vp, vp, vp, vp, vp, C.POINTER(_Counters)]
    L.fm_sample_degrees.restype = C.c_int
    L.fm_sample_richclub.argtypes = [vp, u64, i64, i64, vp, vp, C.POINTER(_Counters)]
    L.fm_sample_richclub.restype = C.c_int
    if hasattr(L, "fm_expected_degrees") or not os.environ.get("FM_LIB_VARIANT"):  # (older A/B builds lack it)
        L.fm_expected_degrees.argtypes = [C.c_int, i64, vp, vp, vp, i64, vp, vp, vp, vp, vp]
        L.fm_expected_degrees.restype = C.c_int
    if hasattr(L, "fm_pool_trim") or not os.environ.get("FM_LIB_VARIANT"):
        L.fm_pool_trim.argtypes = [u64]
        L.fm_pool_trim.restype = C.c_int
    L.fm_sample_to_host.argtypes = [vp, u64, i64, i64, C.c_uint32, vp, vp, vp, i64, C.POINTER(_Edges)]
    L.fm_sample_to_host.restype = C.c_int
    L.fm_edges_to_host.argtypes = [C.POINTER(_Edges), vp, vp, vp]
    L.fm_edges_to_host.restype = C.c_int
    L.fm_plan_get_info.argtypes = [vp, C.POINTER(_PlanInfo)]
    L.fm_plan_get_info.restype = C.c_int
    L.fm_plan_export.argtypes = [vp] + [vp] * 11
    L.fm_plan_export.restype = C.c_int
    L.fm_free.argtypes = [vp]
    L.fm_free.restype = None
    L.fm_last_error.argtypes = []
    L.fm_last_error.restype = C.c_char_p
    L.fm_abi_version.argtypes = []
    L.fm_abi_version.restype = C.c_int32
    L.fm_timing_enable.argtypes = [C.c_int]
    L.fm_timing_enable.restype = C.c_int
    L.fm_timing_get.argtypes = [C.POINTER(_Timing), C.c_int]
    L.fm_timing_get.restype = C.c_int
    L.fm_debug_eval.argtypes = [C.c_int32, i64, vp, vp, vp]
    L.fm_debug_eval.restype = C.c_int
    return L


lib = _load()


def _check(status: int):
    if status != FM_OK:
        raise FastMaxEntError(status, lib.fm_last_error().decode(errors="replace"))


def _stream(stream):
    if stream is not None:
        return C.c_void_p(int(getattr(stream, "cuda_stream", stream)))
    try:
        import torch
        if torch.cuda.is_available():
            return C.c_void_p(torch.cuda.current_stream().cuda_stream)
    except ImportError:  # pragma: no cover
        pass
    return C.c_void_p(0)


def _as_f64(a):
    """(pointer, keepalive) for a float64 vector: torch tensor (CUDA or CPU) or array-like (host)."""
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64:
                a = a.to(torch.float64)
            a = a.contiguous()
            return C.c_void_p(a.data_ptr()), a, a.numel()
    except ImportError:  # pragma: no cover
        pass
    arr = np.ascontiguousarray(a, dtype=np.float64)
    return C.c_void_p(arr.ctypes.data), arr, arr.size


class _CAI:
    """__cuda_array_interface__ view of library-owned device memory; keeps its owner alive."""

    def __init__(self, ptr, shape, typestr, owner):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": shape, "typestr": typestr, "data": (int(ptr or 0), False),
                                         "version": 3, "strides": None}


class Plan:
    def __init__(self, handle, model):
        self._h = handle
        self.model = model
        info = _PlanInfo()
        _check(lib.fm_plan_get_info(self._h, C.byref(info)))
        self.n = info.n
        self.kind = info.kind
        self.n_minus = info.n_minus
        self.seg_target = info.seg_target
        self.F = info.F
        self.n_segments = info.n_segments
        self.n_chunks = info.n_chunks
        self.est_draws = info.est_draws

    def export(self) -> dict:
        n, s = self.n, self.n_segments
        ecm = self.model == FM_ECM
        keys = ("perm", "kappa_s", "y_s", "ymax", "ly_s", "seg", "seg_h0", "seg_x0", "seg_d0", "seg_omT", "seg_iomT")
        out = {"perm": np.empty(n, np.int32), "kappa_s": np.empty(n, np.float64),
               "y_s": np.empty(n, np.float64) if ecm else None,
               "ymax": np.empty(self.n_minus + 1, np.float64) if ecm else None,
               "ly_s": np.empty(n, np.float64) if ecm else None, "seg": np.empty((s, 4), np.int32)}
        for k in keys[6:]:
            out[k] = np.empty(s)
        ptr = lambda a: None if a is None else C.c_void_p(a.ctypes.data)  # noqa: E731
        _check(lib.fm_plan_export(self._h, *(ptr(out[k]) for k in keys)))
        return out

    def export_candidates(self) -> dict:
        """fm_plan_export_candidates: the candidate (- / in) set's arrays and the directed exclusions."""
        nc, n = self.n_minus, self.n
        ecm = self.model == FM_ECM
        out = {"cperm": np.empty(nc, np.int32), "ckappa": np.empty(nc), "cy": np.empty(nc) if ecm else None,
               "cly": np.empty(nc) if ecm else None, "excl": np.empty(n, np.int32)}
        ptr = lambda a: None if a is None else C.c_void_p(a.ctypes.data)  # noqa: E731
        _check(lib.fm_plan_export_candidates(self._h, *(ptr(out[k]) for k in ("cperm", "ckappa", "cy", "cly",
                                                                              "excl"))))
        return out

    def free(self):
        if self._h:
            lib.fm_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # pragma: no cover
            pass


class _EdgesOwner:
    """Owns the library buffers of one fm_edges result and releases them when the last holder -- the
    Edges object or a tensor view made from it -- goes away.  (The views must not keep the Edges
    object itself alive: it caches them, and a cycle through a torch tensor is invisible to
    Python's garbage collector -- every result whose .edges had been read used to leak.)"""

    def __init__(self, st: _Edges):
        self.st = st

    def free(self):
        if self.st is not None and self.st._owner:
            lib.fm_free(C.byref(self.st))

    def __del__(self):
        try:
            self.free()
        except Exception:  # pragma: no cover
            pass


class Edges:
    """Result of fm_sample_*: device edge list (+ weights), host offsets, counters."""

    def __init__(self, st: _Edges, stream):
        self._st = st
        self._own = _EdgesOwner(st)
        self._stream = stream
        self.n_samples = st.n_samples
        self.n_edges = st.n_edges
        self.offsets = np.ctypeslib.as_array(st.offsets, shape=(st.n_samples + 1,)).copy() if st.offsets else \
            np.zeros(1, np.int64)
        self.draws, self.landed, self.accepted = st.draws, st.landed, st.accepted
        self.segments, self.chunks, self.flags = st.segments, st.chunks, st.flags
        self._edges_t = None
        self._w_t = None

    @property
    def edges(self):
        """torch.int32 [n_edges, 2] on the GPU (zero-copy view of library memory)."""
        if self._edges_t is None:
            import torch
            self._edges_t = torch.as_tensor(_CAI(self._st.edges, (self.n_edges, 2), "<i4", self._own), device="cuda")
        return self._edges_t

    @property
    def weights(self):
        if not self._st.weights:
            return None
        if self._w_t is None:
            import torch
            self._w_t = torch.as_tensor(_CAI(self._st.weights, (self.n_edges,), "<i4", self._own), device="cuda")
        return self._w_t

    def to_host(self, edges_out=None, weights_out=None, stream=None):
        """fm_edges_to_host into (optionally caller-provided, e.g. pinned) host buffers -> numpy."""
        if edges_out is None:
            edges_out = np.empty((self.n_edges, 2), np.int32)
        has_w = bool(self._st.weights)
        if has_w and weights_out is None:
            weights_out = np.empty(self.n_edges, np.int32)
        ep = edges_out.data_ptr() if hasattr(edges_out, "data_ptr") else edges_out.ctypes.data
        wp = None
        if has_w:
            wp = weights_out.data_ptr() if hasattr(weights_out, "data_ptr") else weights_out.ctypes.data
        _check(lib.fm_edges_to_host(C.byref(self._st), C.c_void_p(ep), C.c_void_p(wp) if wp else None,
                                    _stream(stream) if stream is not None else self._stream))
        return edges_out, (weights_out if has_w else None)

    def sample(self, s: int):
        a, b = int(self.offsets[s]), int(self.offsets[s + 1])
        return self.edges[a:b], (None if self.weights is None else self.weights[a:b])

    def free(self):
        """Release the device buffers now (views made from this result become invalid)."""
        self._edges_t = None
        self._w_t = None
        self._own.free()


def sort_plan(x, y=None, seg_target: int = 256, stream=None) -> Plan:
    """fm_sort_plan: validate, sort (descending kappa), beta_min suffix max, segment plan."""
    model = FM_UBCM if y is None else FM_ECM
    xp, xk, n = _as_f64(x)
    yp = None
    yk = None
    if y is not None:
        yp, yk, ny = _as_f64(y)
        if ny != n:
            raise FastMaxEntError(FM_ERR_INVALID, f"len(y) = {ny} != len(x) = {n}")
    h = C.c_void_p()
    _check(lib.fm_sort_plan(model, n, xp, yp, int(seg_target), _stream(stream), C.byref(h)))
    del xk, yk
    return Plan(h, model)


def sort_plan_bipartite(x_plus, x_minus, y_plus=None, y_minus=None, kind: str = "bipartite",
                        seg_target: int = 256, stream=None) -> Plan:
    """fm_sort_plan_bipartite: kind "bipartite" (+ set rows vs - set candidates) or
    "directed" (x_plus/y_plus = out-fitness, x_minus/y_minus = in-fitness, no self loops)."""
    model = FM_UBCM if y_plus is None else FM_ECM
    k = _KINDS[kind]
    p1, k1, n1 = _as_f64(x_plus)
    p2, k2, n2 = _as_f64(x_minus)
    q1 = q2 = None
    keep = []
    if model == FM_ECM:
        q1, kk1, ny1 = _as_f64(y_plus)
        q2, kk2, ny2 = _as_f64(y_minus)
        keep = [kk1, kk2]
        if ny1 != n1 or ny2 != n2:
            raise FastMaxEntError(FM_ERR_INVALID, "y lengths differ from x lengths")
    h = C.c_void_p()
    _check(lib.fm_sort_plan_bipartite(model, k, n1, p1, q1, n2, p2, q2, int(seg_target), _stream(stream),
                                      C.byref(h)))
    del k1, k2, keep
    return Plan(h, model)


def _sample(fn, plan: Plan, seed: int, n_samples: int, first_sample: int, stream) -> Edges:
    st = _Edges()
    s = _stream(stream)
    _check(fn(plan._h, int(seed) & 0xFFFFFFFFFFFFFFFF, int(first_sample), int(n_samples), s, C.byref(st)))
    return Edges(st, s)


def sample_ubcm(plan: Plan, seed: int, n_samples: int = 1, first_sample: int = 0, stream=None) -> Edges:
    """fm_sample_ubcm."""
    return _sample(lib.fm_sample_ubcm, plan, seed, n_samples, first_sample, stream)


FM_SAMPLE_BETA_REFRESH = 1


def sample_ecm(plan: Plan, seed: int, n_samples: int = 1, first_sample: int = 0, stream=None,
               refresh: bool = False) -> Edges:
    """fm_sample_ecm (Algorithm 1); refresh=True: fm_sample_ecm_ex with
    FM_SAMPLE_BETA_REFRESH (per-candidate beta_min, R17)."""
    if not refresh:
        return _sample(lib.fm_sample_ecm, plan, seed, n_samples, first_sample, stream)
    st = _Edges()
    s = _stream(stream)
    _check(lib.fm_sample_ecm_ex(plan._h, int(seed) & 0xFFFFFFFFFFFFFFFF, int(first_sample), int(n_samples),
                                FM_SAMPLE_BETA_REFRESH, s, C.byref(st)))
    return Edges(st, s)


def sample_to_host(plan: Plan, seed: int, edges_out, weights_out=None, n_samples: int = 1, first_sample: int = 0,
                   stream=None, refresh: bool = False) -> Edges:
    """fm_sample_to_host: sample like sample_ubcm / sample_ecm (the plan's model) and deliver the list
    into caller-provided host buffers as well -- edges_out int32 [cap, 2], weights_out int32 [cap]
    (numpy arrays or CPU torch tensors, ideally page-locked) -- copying each group of samples while
    the next ones are generated.  Returns the Edges result (device list, offsets, counters);
    result.flags & FM_FLAG_HOST_TRUNCATED: the host buffers were too small (nothing valid in them)."""
    def ptr_cap(a, per):
        if a is None:
            return None, 0
        if hasattr(a, "data_ptr"):
            assert a.dtype.itemsize == 4 and a.is_contiguous() and not a.is_cuda
            return C.c_void_p(a.data_ptr()), a.numel() // per
        assert a.dtype == np.int32 and a.flags["C_CONTIGUOUS"]
        return C.c_void_p(a.ctypes.data), a.size // per
    ep, cap = ptr_cap(edges_out, 2)
    wp, wcap = ptr_cap(weights_out, 1)
    if wp is not None:
        cap = min(cap, wcap)
    st = _Edges()
    s = _stream(stream)
    _check(lib.fm_sample_to_host(plan._h, int(seed) & 0xFFFFFFFFFFFFFFFF, int(first_sample), int(n_samples),
                                 FM_SAMPLE_BETA_REFRESH if refresh else 0, s, ep, wp, int(cap), C.byref(st)))
    return Edges(st, s)


def sample_degrees(plan: Plan, seed: int, n_samples: int = 1, first_sample: int = 0, stream=None):
    """fm_sample_degrees: per-node degree (and ECM strength) sums over the samples, no edge list.
    Returns (deg_plus, deg_minus, str_plus, str_minus, counters) as CUDA int64 tensors (minus arrays
    None when undirected; strengths None for the UBCM)."""
    import torch
    ecm = plan.model == FM_ECM
    bip = plan.kind != FM_UNDIRECTED
    z = lambda n: torch.zeros(n, dtype=torch.int64, device="cuda")  # noqa: E731
    dp = z(plan.n)
    dm = z(plan.n_minus) if bip else None
    sp = z(plan.n) if ecm else None
    sm = z(plan.n_minus) if (ecm and bip) else None
    ptr = lambda t: None if t is None else C.c_void_p(t.data_ptr())  # noqa: E731
    c = _Counters()
    _check(lib.fm_sample_degrees(plan._h, int(seed) & 0xFFFFFFFFFFFFFFFF, int(first_sample), int(n_samples),
                                 _stream(stream), ptr(dp), ptr(dm), ptr(sp), ptr(sm), C.byref(c)))
    return dp, dm, sp, sm, {"draws": c.draws, "landed": c.landed, "accepted": c.accepted, "flags": c.flags}


def sample_richclub(plan: Plan, seed: int, n_samples: int = 1, first_sample: int = 0, stream=None):
    """fm_sample_richclub: e_top[m] = edges among the m top-ranked nodes (plan order), summed over
    the samples, m = 0..n, as a CUDA int64 tensor; plus the counters.  Undirected plans only."""
    import torch
    e = torch.zeros(plan.n + 1, dtype=torch.int64, device="cuda")
    c = _Counters()
    _check(lib.fm_sample_richclub(plan._h, int(seed) & 0xFFFFFFFFFFFFFFFF, int(first_sample), int(n_samples),
                                  _stream(stream), C.c_void_p(e.data_ptr()), C.byref(c)))
    return e, {"draws": c.draws, "landed": c.landed, "accepted": c.accepted, "flags": c.flags}


def expected_degrees(x, y=None, nodes=None, stream=None):
    """fm_expected_degrees: exact per-node sum_j p_ij and sum_j p_ij (1 - p_ij) (and, for
    the ECM, the expected strength and its variance) of the listed node ids (None: all nodes).
    Returns (k, kvar, s, svar) as CUDA float64 tensors (s, svar None for the UBCM)."""
    import torch
    px, kx, n = _as_f64(x)
    py, ky = (None, None) if y is None else _as_f64(y)[:2]
    keep_nodes = None
    m = n
    pn = None
    if nodes is not None:
        if isinstance(nodes, torch.Tensor):
            keep_nodes = nodes.to(torch.int32).contiguous()
            pn = C.c_void_p(keep_nodes.data_ptr())
        else:
            keep_nodes = np.ascontiguousarray(nodes, dtype=np.int32)
            pn = C.c_void_p(keep_nodes.ctypes.data)
        m = int(keep_nodes.numel() if isinstance(keep_nodes, torch.Tensor) else keep_nodes.size)
    out = [torch.empty(m, dtype=torch.float64, device="cuda") for _ in range(2 if y is None else 4)]
    ptr = [C.c_void_p(t.data_ptr()) for t in out] + [None] * (4 - len(out))
    _check(lib.fm_expected_degrees(FM_UBCM if y is None else FM_ECM, n, px, py, pn, m, *ptr, _stream(stream)))
    del kx, ky, keep_nodes
    return (out[0], out[1], None, None) if y is None else tuple(out)


def pool_trim(keep_bytes: int = 0) -> None:
    """fm_pool_trim: return the device pool's cached temporaries beyond keep_bytes to the device."""
    _check(lib.fm_pool_trim(int(keep_bytes)))


def abi_version() -> int:
    return int(lib.fm_abi_version())


def timing_enable(on: bool = True) -> None:
    """Record CUDA events around each library phase (fm_timing_enable)."""
    _check(lib.fm_timing_enable(1 if on else 0))


def timing_get(reset: bool = False) -> dict:
    """Accumulated device milliseconds per phase and the library's kernel-launch count."""
    t = _Timing()
    _check(lib.fm_timing_get(C.byref(t), 1 if reset else 0))
    return {"plan_ms": t.plan_ms, "sample_ms": t.sample_ms, "write_ms": t.write_ms,
            "sample_launches": t.sample_launches, "launches": t.launches}


def debug_eval(fn: int, x):
    """fm_debug_eval: the device fp64 logarithms (0 log, 1 log1p, 2 -log(u01(k))) on a CUDA float64 tensor;
    fn 3: x of shape [n, 2] -> x[:, 0] / x[:, 1] by the sampler's Markstein division."""
    import torch
    x = x.to(device="cuda", dtype=torch.float64).contiguous()
    n = x.numel() // 2 if fn == 3 else x.numel()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    _check(lib.fm_debug_eval(int(fn), n, C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr()), _stream(None)))
    return out
