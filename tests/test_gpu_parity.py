"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle on identical seeds.

Bar (BASELINE north_star): per-sample edge sets (and weights) differ on at most 1e-6 of edges;
the plan is bit-identical (h0 within libm-vs-CUDA log1p ulps); counters equal."""
import os

import numpy as np
import pytest

from paper_2509_13230_b200 import workloads as WL
from _parity import compare, hygiene

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402


def gpu_run(x, y, S, seed, n_samples, first_sample=0, host_inputs=False):
    if host_inputs:
        plan = fm.sort_plan(x, y, seg_target=S)
    else:
        plan = fm.sort_plan(torch.from_numpy(x).cuda(), None if y is None else torch.from_numpy(y).cuda(),
                            seg_target=S)
    fn = fm.sample_ubcm if y is None else fm.sample_ecm
    e = fn(plan, seed, n_samples=n_samples, first_sample=first_sample)
    torch.cuda.synchronize()
    E = e.edges.cpu().numpy()
    W = None if e.weights is None else e.weights.cpu().numpy()
    return plan, e, E, W


def check_parity(O, x, y, S, seed, n_samples, first_sample=0, exact=False, host_inputs=False):
    plan, e, E, W = gpu_run(x, y, S, seed, n_samples, first_sample, host_inputs)
    ref = O.sample(O.sort_plan(x, y, seg_target=S), seed, n_samples=n_samples, first_sample=first_sample,
                   nthreads=O.ncores())
    hygiene(E, len(x), W)
    bad, tot = compare(e.offsets, E, W, ref, len(x))
    allowed = 0 if exact else int(1e-6 * max(tot, 1))
    assert bad <= allowed, f"{bad} mismatched edges of {tot} (allowed {allowed})"
    if bad == 0:
        assert (e.draws, e.landed, e.accepted) == (ref.draws, ref.landed, ref.accepted)
        assert np.array_equal(e.offsets, ref.offsets)
        # v2 writes every lane-chunk in draw order: the GPU list is the oracle's canonical order
        assert np.array_equal(E, ref.edges)
        if W is not None:
            assert np.array_equal(W, ref.weights)
    return plan, e, ref


# ------------------------------------------------------------------------------ plan parity
@pytest.mark.parametrize("ecm", [False, True])
@pytest.mark.parametrize("n,S", [(2, 256), (3, 8), (1000, 8), (4097, 37), (100_003, 256)])
def test_plan_bit_identical(O, ecm, n, S):
    x, y = WL.random_fitness(100 + n, n, 2.3, 0.01, ecm=ecm)
    if n > 10:
        x[3] = x[9]  # a tie
    g = fm.sort_plan(torch.from_numpy(x).cuda(), None if y is None else torch.from_numpy(y).cuda(), seg_target=S)
    o = O.sort_plan(x, y, seg_target=S)
    gx = g.export()
    assert g.F == o.F and g.n_segments == o.n_segments
    assert np.array_equal(gx["perm"], o.perm)
    assert np.array_equal(gx["kappa_s"], o.kappa_s)
    if ecm:
        assert np.array_equal(gx["y_s"], o.y_s) and np.array_equal(gx["ymax"], o.ymax)
        assert np.abs(gx["ly_s"].view(np.int64) - o.ly_s.view(np.int64)).max() <= 1  # CUDA vs glibc log
    seg = gx["seg"]
    assert np.array_equal(seg[:, 0], o.seg_u) and np.array_equal(seg[:, 1], o.seg_a)
    assert np.array_equal(seg[:, 2], o.seg_b) and np.array_equal(seg[:, 3], o.seg_sigma)
    for k in ("seg_x0", "seg_d0", "seg_omT", "seg_iomT"):
        assert np.array_equal(gx[k], getattr(o, k)), k
    ulp = np.abs(gx["seg_h0"].view(np.int64) - o.seg_h0.view(np.int64))
    assert ulp.max(initial=0) <= 1  # CUDA log1p vs glibc log1p


@pytest.mark.parametrize("n", [5000, 4096 * 3, 100_003])
def test_plan_sort_big_tiles(O, monkeypatch, n):
    """The 4096-key radix tiles (used from 2^20 keys) forced at small n: ragged last tile, ties."""
    monkeypatch.setenv("FM_SORT_BIG_MIN", "0")
    x, y = WL.random_fitness(900 + n, n, 2.3, 0.01, ecm=True)
    x[3] = x[9] = x[n - 1]
    g = fm.sort_plan(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), seg_target=64).export()
    o = O.sort_plan(x, y, seg_target=64)
    assert np.array_equal(g["perm"], o.perm) and np.array_equal(g["kappa_s"], o.kappa_s)
    assert np.array_equal(g["y_s"], o.y_s)


def test_plan_constant_radix_digit(O):
    """Keys that agree in a whole radix digit (every kappa in [0.5, 2): the sign / high-exponent byte;
    and x = j / 8: the low mantissa bytes): those passes are plain copies on the device; the
    permutation is still the oracle's."""
    rng = np.random.default_rng(5)
    for x in (0.5 + 1.5 * rng.random(50_001) * (1 - 1e-12), np.arange(1, 40_000, dtype=np.float64) / 8.0):
        x[7] = x[11]  # a tie
        g = fm.sort_plan(torch.from_numpy(x).cuda(), seg_target=64).export()
        o = O.sort_plan(x, seg_target=64)
        assert np.array_equal(g["perm"], o.perm) and np.array_equal(g["kappa_s"], o.kappa_s)


# ------------------------------------------------------------------------------ small cases
@pytest.mark.parametrize("ecm", [False, True])
@pytest.mark.parametrize("n,S,R", [(2, 256, 50), (5, 8, 200), (31, 8, 100), (1000, 8, 20), (4097, 256, 5),
                                   (20_011, 64, 3)])
def test_small_parity(O, ecm, n, S, R):
    x, y = WL.random_fitness(7 * n + 1, n, 2.5, 0.3 if n < 100 else 0.03, ecm=ecm)
    check_parity(O, x, y, S, seed=1000 + n, n_samples=R, first_sample=3, exact=True)


def test_host_pointer_inputs(O):
    x, y = WL.random_fitness(3, 5000, 2.5, 0.02, ecm=True)
    check_parity(O, x, y, 256, seed=9, n_samples=2, exact=True, host_inputs=True)
    check_parity(O, x, None, 256, seed=9, n_samples=2, exact=True, host_inputs=True)


# ------------------------------------------------------------------------------ configs 1-3
def test_config1_exact_and_ensemble(O):
    w = WL.workload(1)
    x, _ = WL.fitness(w)
    check_parity(O, x, None, 256, w.seed, 1, exact=True)          # 1 sample: exact set equality
    check_parity(O, x, None, 256, w.seed, 10_000, exact=False)    # the 10,000-sample ensemble


@pytest.mark.parametrize("cfg", [2, 3])
def test_config_full_parity(O, cfg):
    w = WL.workload(cfg)
    x, y = WL.fitness(w)
    plan, e, ref = check_parity(O, x, y, 256, w.seed, w.n_samples)
    assert e.n_edges > 0.9 * w.n * w.kbar / 2 * w.n_samples


# ------------------------------------------------------------------------------ invariants
def test_batch_equals_singles_and_determinism():
    x, y = WL.random_fitness(5, 30_000, 2.3, 0.01, ecm=True)
    for yy in (None, y):
        _, e, E, W = gpu_run(x, yy, 64, 77, 5, first_sample=100)
        _, e2, E2, W2 = gpu_run(x, yy, 64, 77, 5, first_sample=100)
        assert np.array_equal(E, E2) and np.array_equal(e.offsets, e2.offsets)  # byte-identical reruns
        if W is not None:
            assert np.array_equal(W, W2)
        for s in range(5):
            _, es, Es, Ws = gpu_run(x, yy, 64, 77, 1, first_sample=100 + s)
            assert np.array_equal(np.sort(Es.view(np.int64).ravel()),
                                  np.sort(E[e.offsets[s]:e.offsets[s + 1]].view(np.int64).ravel()))


@pytest.mark.parametrize("cap", ["7", "8"])  # 8: 32-byte-aligned slots (whole-sector writes) that still overflow
def test_scratch_overflow_rerun_is_identical(monkeypatch, cap):
    x, y = WL.random_fitness(6, 20_000, 2.3, 0.02, ecm=True)
    for yy in (None, y):
        _, e, E, W = gpu_run(x, yy, 64, 5, 3)
        monkeypatch.setenv("FM_DEBUG_SCRATCH_CAP", cap)
        _, e2, E2, W2 = gpu_run(x, yy, 64, 5, 3)
        monkeypatch.delenv("FM_DEBUG_SCRATCH_CAP")
        assert e2.flags & fm.FM_FLAG_SCRATCH_RERUN
        assert np.array_equal(e.offsets, e2.offsets)
        key = lambda A: np.sort(A.view(np.int64).ravel())  # noqa: E731
        for s in range(3):
            a, b = e.offsets[s], e.offsets[s + 1]
            assert np.array_equal(key(E[a:b]), key(E2[a:b]))


@pytest.mark.parametrize("env", [{"FM_UBCM_RANK_OUT_MIN": "0"},   # kappa-only gathers, ranks mapped by the compaction
                                 {"FM_UBCM_CAND_MIN": str(1 << 40)},  # kappa and id from two arrays (no record)
                                 {"FM_SCRATCH_BUF4": "0"}])       # one 8-byte store per edge
def test_ubcm_gather_and_store_modes_identical(O, monkeypatch, env):
    """The sampler's alternative gather / store paths produce the default path's edge list byte for
    byte (and the oracle's on the small case)."""
    x, _ = WL.random_fitness(11, 30_011, 2.5, 0.02)
    _, e, E, _ = gpu_run(x, None, 64, 9, 4)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    _, e2, E2, _ = gpu_run(x, None, 64, 9, 4)
    assert np.array_equal(e.offsets, e2.offsets) and np.array_equal(E, E2)
    xs, _ = WL.random_fitness(12, 3001, 2.5, 0.05)
    check_parity(O, xs, None, 16, seed=3, n_samples=3, exact=True)
    for k in env:
        monkeypatch.delenv(k)


@pytest.mark.parametrize("ecm", [False, True])
def test_chunk_major_queue_identical(O, monkeypatch, ecm):
    """The chunk-major task queue (the samples of one lane-chunk back to back, on by default at
    N >= 2^19) only reorders work: the edge list equals the sample-major queue's byte for byte,
    and the oracle's on the small case."""
    x, y = WL.random_fitness(13, 40_009, 2.4, 0.02, ecm=True)
    yy = y if ecm else None
    res = []
    for v in ("0", str(1 << 40)):  # forced on / forced off
        monkeypatch.setenv("FM_INTERLEAVE_MIN", v)
        _, e, E, W = gpu_run(x, yy, 64, 21, 5)
        res.append((e.offsets, E, W))
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    if ecm:
        assert np.array_equal(res[0][2], res[1][2])
    monkeypatch.setenv("FM_INTERLEAVE_MIN", "0")
    xs, ys = WL.random_fitness(14, 3001, 2.5, 0.05, ecm=True)
    check_parity(O, xs, ys if ecm else None, 16, seed=4, n_samples=3, exact=True)
    monkeypatch.delenv("FM_INTERLEAVE_MIN")


def test_edge_cases(O):
    # complete graph, empty graph, N = 2, zero samples
    n = 300
    _, e, E, _ = gpu_run(np.full(n, 1e10), None, 1 << 40, 1, 2)
    assert e.n_edges == 2 * n * (n - 1) // 2
    _, e, E, _ = gpu_run(np.zeros(n), None, 256, 1, 3)
    assert e.n_edges == 0 and e.draws == 3 * (n - 1)
    _, e, E, _ = gpu_run(np.array([5.0, 5.0]), None, 256, 1, 100)
    assert 85 <= e.n_edges <= 100
    plan = fm.sort_plan(torch.ones(10, dtype=torch.float64, device="cuda"))
    e0 = fm.sample_ubcm(plan, 1, n_samples=0)
    assert e0.n_edges == 0 and list(e0.offsets) == [0]
    # ECM with y = 0: t = 0, every weight is 1
    x = np.full(50, 3.0)
    _, e, E, W = gpu_run(x, np.zeros(50), 256, 2, 4)
    assert e.n_edges == 0  # z = 0 -> p = 0
    x, y = WL.random_fitness(1, 200, 2.5, 50.0, ecm=True)
    y[:] = 1e-9
    _, e, E, W = gpu_run(x / 1e-9, y, 256, 2, 4)
    assert e.n_edges > 0 and np.all(W == 1)


def test_status_codes():
    with pytest.raises(fm.FastMaxEntError) as ex:
        fm.sort_plan(np.array([1.0]))
    assert ex.value.status == fm.FM_ERR_INVALID
    for bad in ([1.0, -1.0], [1.0, np.nan], [1.0, np.inf], [1e200, 1.0], [1e80, 1.0]):
        with pytest.raises(fm.FastMaxEntError) as ex:
            fm.sort_plan(torch.tensor(bad, dtype=torch.float64, device="cuda"))
        assert ex.value.status == fm.FM_ERR_INVALID
    with pytest.raises(fm.FastMaxEntError) as ex:
        fm.sort_plan(np.ones(4), np.array([0.5, 0.5, 1.0, 0.2]))
    assert ex.value.status == fm.FM_ERR_INVALID
    with pytest.raises(fm.FastMaxEntError) as ex:
        fm.sort_plan(np.ones(4), seg_target=4)
    assert ex.value.status == fm.FM_ERR_INVALID
    p = fm.sort_plan(np.ones(4))
    with pytest.raises(fm.FastMaxEntError) as ex:
        fm.sample_ecm(p, 1, 1)
    assert ex.value.status == fm.FM_ERR_STATE
    with pytest.raises(fm.FastMaxEntError) as ex:
        fm.sample_ubcm(p, 1, 2, first_sample=2**32 - 1)
    assert ex.value.status == fm.FM_ERR_INVALID


# ------------------------------------------------------------------------------ v3 fused write
@pytest.mark.parametrize("n,S,R", [(1000, 8, 20), (20_011, 64, 3), (100_000, 256, 7)])
def test_fused_write_option_parity(O, n, S, R):
    """FM_FUSE_WRITE=1 (opt-in v3 write path): the same lists as the default path
    and the oracle, element by element."""
    x, _ = WL.random_fitness(11 * n + 5, n, 2.4, 0.03 if n < 50_000 else 0.005)
    os.environ["FM_FUSE_WRITE"] = "1"
    try:
        plan, e, E, _ = gpu_run(x, None, S, 4242, R, first_sample=1)
    finally:
        os.environ.pop("FM_FUSE_WRITE", None)
    _, e0, E0, _ = gpu_run(x, None, S, 4242, R, first_sample=1)
    assert np.array_equal(e.offsets, e0.offsets) and np.array_equal(E, E0)
    ref = O.sample(O.sort_plan(x, seg_target=S), 4242, n_samples=R, first_sample=1, nthreads=O.ncores())
    assert np.array_equal(E, ref.edges)


# ------------------------------------------------------------------------------ round-2 scheduling options
@pytest.mark.parametrize("ecm", [False, True])
@pytest.mark.parametrize("env", [
    {"FM_SAMPLE_GROUPS": "3"},                              # pipelined sample groups on two streams
    {"FM_SAMPLE_GROUPS": "4", "FM_COMPACT_SMALL": "2"},     # ... every group through the TMA compaction
    {"FM_COMPACT_SMALL": "0"},                              # the block-staged compaction kernel
    {"FM_CHUNK_BIG_DRAWS": "0"},                            # no big lane-chunks
    {"FM_CHUNK_BIG_DRAWS": "512", "FM_TAIL_FACTOR_BIG": "0", "FM_TAIL_FACTOR": "0"},  # big chunks only
    {"FM_CHUNK_BIG_DRAWS": "300", "FM_TAIL_FACTOR_BIG": "0", "FM_SAMPLE_GROUPS": "2",
     "FM_UBCM_RANK_OUT_MIN": "0"},                          # all three ranges x groups x rank mapping
])
def test_scheduling_options_identical(O, monkeypatch, ecm, env):
    """Sample groups, the lane-chunkings (big / coarse / fine) and the compaction kernels only
    schedule work: offsets, edges and weights equal the default configuration's byte for byte, and
    the oracle's canonical order."""
    x, y = WL.random_fitness(17, 30_011, 2.4, 0.02, ecm=True)
    yy = y if ecm else None
    R = 9
    _, e0, E0, W0 = gpu_run(x, yy, 64, 31, R, first_sample=2)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    try:
        plan, e, E, W = gpu_run(x, yy, 64, 31, R, first_sample=2)
    finally:
        for k in env:
            monkeypatch.delenv(k)
    assert np.array_equal(e.offsets, e0.offsets) and np.array_equal(E, E0)
    assert (e.draws, e.landed, e.accepted) == (e0.draws, e0.landed, e0.accepted)
    if ecm:
        assert np.array_equal(W, W0)
    ref = O.sample(O.sort_plan(x, yy, seg_target=64), 31, n_samples=R, first_sample=2, nthreads=O.ncores())
    assert np.array_equal(e.offsets, ref.offsets) and np.array_equal(E, ref.edges)
    if ecm:
        assert np.array_equal(W, ref.weights)


def test_groups_with_overflow_rerun(monkeypatch):
    """Sample groups + tasks that overflow slot and spill (re-run into the final list at the group's
    base) + a final list that is too small on the first pass (whole call redone)."""
    x, _ = WL.random_fitness(6, 20_000, 2.3, 0.02)
    _, e, E, _ = gpu_run(x, None, 64, 5, 6)
    monkeypatch.setenv("FM_DEBUG_SCRATCH_CAP", "8")
    monkeypatch.setenv("FM_SAMPLE_GROUPS", "3")
    _, e2, E2, _ = gpu_run(x, None, 64, 5, 6)
    monkeypatch.delenv("FM_DEBUG_SCRATCH_CAP")
    monkeypatch.delenv("FM_SAMPLE_GROUPS")
    assert e2.flags & fm.FM_FLAG_SCRATCH_RERUN
    assert np.array_equal(e.offsets, e2.offsets)
    key = lambda A: np.sort(A.view(np.int64).ravel())  # noqa: E731
    for s in range(6):
        a, b = e.offsets[s], e.offsets[s + 1]
        assert np.array_equal(key(E[a:b]), key(E2[a:b]))


def test_queue_ending_with_empty_tasks(O):
    """Regression (found by test_gpu_fuzz.py): an almost empty graph whose total work is just above a
    multiple of the chunk target has an EMPTY last lane-chunk; in the chunk-major queue those tasks
    are the last of the call, and the warps that fetched them used to leave before recording their
    (zero) counts -- the scan then summed stale memory.  Dirty the pool first."""
    xd, _ = WL.random_fitness(1, 50_000, 2.5, 0.05)
    _ = gpu_run(xd, None, 256, 1, 8)  # leaves non-zero counts / offsets in the stream-ordered pool
    x, _ = WL.random_fitness(58, 257, 2.5, 0.001)
    for S in (37, 256):
        for R in (13, 60, 64, 100):
            check_parity(O, x, None, S, seed=342799134629, n_samples=R, first_sample=1, exact=True)
