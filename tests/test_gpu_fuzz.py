"""Seeded random sweep of the whole C-ABI surface against the oracle: model x graph kind x size x
fitness scale x segmentation target x sample range x ECM bound refresh x scheduling options, every
case element by element (offsets, edges in canonical order, weights, counters).  Small sizes: the
sweep spans the degenerate regimes (empty rows, saturated hubs, one-segment and many-segment rows,
tasks of a single draw) that the fixed-size tests only touch."""
import os

import numpy as np
import pytest

from paper_2509_13230_b200 import workloads as WL

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402

OPTIONS = [
    {},
    {"FM_SAMPLE_GROUPS": "2"},
    {"FM_SAMPLE_GROUPS": "3", "FM_COMPACT_SMALL": "2"},
    {"FM_COMPACT_SMALL": "0"},
    {"FM_CHUNK_BIG_DRAWS": "200", "FM_TAIL_FACTOR_BIG": "0", "FM_TAIL_FACTOR": "0"},
    {"FM_CHUNK_LANE_DRAWS": "16", "FM_CHUNK_FINE_DRAWS": "4", "FM_CHUNK_BIG_DRAWS": "40", "FM_TAIL_FACTOR_BIG": "0"},
    {"FM_UBCM_RANK_OUT_MIN": "0", "FM_INTERLEAVE_MIN": "0"},
    {"FM_INTERLEAVE_FINE": "0", "FM_SCRATCH_BUF4": "0"},
    {"FM_FUSE_WRITE": "1"},                                   # (UBCM undirected only; ignored elsewhere)
    {"FM_DEBUG_SCRATCH_CAP": "8", "FM_SAMPLE_GROUPS": "2"},   # slots overflow: spill regions and re-runs
    {"FM_DEBUG_SCRATCH_CAP": "12"},
]


def case(i):
    r = np.random.default_rng(9000 + i)
    ecm = bool(r.integers(2))
    kind = ("undirected", "bipartite", "directed")[int(r.integers(3))]
    n1 = int(r.choice([2, 3, 17, 64, 257, 1000, 3001, 9001]))
    n2 = n1 if kind != "bipartite" else int(r.choice([1, 5, 33, 500, 2500]))
    gamma = float(r.choice([2.1, 2.5, 3.0]))
    scale = float(r.choice([1e-3, 0.02, 0.3, 3.0])) if n1 <= 1000 else float(r.choice([1e-3, 0.02, 0.1]))
    S = int(r.choice([8, 9, 37, 256, 1 << 20]))
    R = int(r.choice([1, 2, 7, 20])) if n1 > 300 else int(r.choice([1, 13, 100]))
    first = int(r.choice([0, 1, 4_000_000_000]))
    refresh = ecm and bool(r.integers(2))
    return dict(ecm=ecm, kind=kind, n1=n1, n2=n2, gamma=gamma, scale=scale, S=S, R=R, first=first, refresh=refresh,
                env=OPTIONS[i % len(OPTIONS)], seed=int(r.integers(1 << 40)))


# FM_FUZZ_OFFSET / FM_FUZZ_N: run another (or a longer) slice of the sweep, e.g. to hunt for bugs ad hoc
_OFF, _N = int(os.environ.get("FM_FUZZ_OFFSET", "0")), int(os.environ.get("FM_FUZZ_N", "160"))


@pytest.mark.parametrize("i", range(_OFF, _OFF + _N))
def test_fuzz_case(O, monkeypatch, i):
    c = case(i)
    x1, y1 = WL.random_fitness(50 + i, c["n1"], c["gamma"], c["scale"], ecm=c["ecm"])
    x2, y2 = WL.random_fitness(150 + i, c["n2"], c["gamma"], c["scale"], ecm=c["ecm"])
    dev = lambda a: None if a is None else torch.from_numpy(a).cuda()  # noqa: E731
    for k, v in c["env"].items():
        monkeypatch.setenv(k, v)
    if c["kind"] == "undirected":
        plan = fm.sort_plan(dev(x1), dev(y1), seg_target=c["S"])
        op = O.sort_plan(x1, y1, seg_target=c["S"])
    else:
        plan = fm.sort_plan_bipartite(dev(x1), dev(x2), dev(y1), dev(y2), kind=c["kind"], seg_target=c["S"])
        op = O.sort_plan(x1, y1, seg_target=c["S"], kind=c["kind"], x2=x2, y2=y2)
    if c["ecm"]:
        e = fm.sample_ecm(plan, c["seed"], n_samples=c["R"], first_sample=c["first"], refresh=c["refresh"])
    else:
        e = fm.sample_ubcm(plan, c["seed"], n_samples=c["R"], first_sample=c["first"])
    ref = O.sample(op, c["seed"], n_samples=c["R"], first_sample=c["first"], nthreads=O.ncores(), refresh=c["refresh"])
    assert plan.n_segments == op.n_segments, c
    assert np.array_equal(e.offsets, ref.offsets), c
    assert np.array_equal(e.edges.cpu().numpy().reshape(-1, 2), ref.edges.reshape(-1, 2)), c
    if c["ecm"]:
        assert np.array_equal(e.weights.cpu().numpy(), ref.weights), c
    assert (e.draws, e.landed, e.accepted) == (ref.draws, ref.landed, ref.accepted), c
    # statistics mode on the same samples: degree sums of the oracle's lists
    if i % 3 == 0 and not c["refresh"]:  # (fm_sample_degrees has no bound-refresh option)
        out = fm.sample_degrees(plan, c["seed"], n_samples=c["R"], first_sample=c["first"])
        dp, dm = out[0], out[1]
        oe = ref.edges.reshape(-1, 2).astype(np.int64)
        o1, o2 = np.bincount(oe[:, 0], minlength=c["n1"]), np.bincount(oe[:, 1], minlength=c["n2"])
        if c["kind"] == "undirected":
            assert np.array_equal(dp.cpu().numpy(), o1 + o2), c
        else:
            assert np.array_equal(dp.cpu().numpy(), o1) and np.array_equal(dm.cpu().numpy(), o2), c


@pytest.mark.parametrize("i", range(_OFF, _OFF + max(1, _N * 36 // 160)))
def test_fuzz_medium(O, monkeypatch, i):
    """The same sweep at N = 10,000 ... 60,000 (several blocks, many warp batches, hub rows cut into
    segments), undirected and bipartite."""
    r = np.random.default_rng(7000 + i)
    ecm = bool(r.integers(2))
    bip = bool(r.integers(3) == 0)
    n1 = int(r.integers(10_000, 60_000))
    n2 = int(r.integers(5_000, 30_000)) if bip else n1
    gamma = float(r.choice([2.2, 2.5, 2.8]))
    scale = float(r.choice([0.003, 0.01, 0.03]))
    S = int(r.choice([8, 64, 256, 1000]))
    R = int(r.choice([1, 3, 9]))
    env = OPTIONS[(i * 5 + 3) % len(OPTIONS)]
    seed = int(r.integers(1 << 50))
    x1, y1 = WL.random_fitness(300 + i, n1, gamma, scale, ecm=ecm)
    x2, y2 = WL.random_fitness(400 + i, n2, gamma, scale, ecm=ecm)
    dev = lambda a: None if a is None else torch.from_numpy(a).cuda()  # noqa: E731
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    if bip:
        plan = fm.sort_plan_bipartite(dev(x1), dev(x2), dev(y1), dev(y2), kind="bipartite", seg_target=S)
        op = O.sort_plan(x1, y1, seg_target=S, kind="bipartite", x2=x2, y2=y2)
    else:
        plan = fm.sort_plan(dev(x1), dev(y1), seg_target=S)
        op = O.sort_plan(x1, y1, seg_target=S)
    e = (fm.sample_ecm if ecm else fm.sample_ubcm)(plan, seed, n_samples=R, first_sample=5)
    ref = O.sample(op, seed, n_samples=R, first_sample=5, nthreads=O.ncores())
    tag = dict(i=i, ecm=ecm, bip=bip, n1=n1, n2=n2, gamma=gamma, scale=scale, S=S, R=R, env=env)
    assert np.array_equal(e.offsets, ref.offsets), tag
    assert np.array_equal(e.edges.cpu().numpy().reshape(-1, 2), ref.edges.reshape(-1, 2)), tag
    if ecm:
        assert np.array_equal(e.weights.cpu().numpy(), ref.weights), tag
    assert (e.draws, e.landed, e.accepted) == (ref.draws, ref.landed, ref.accepted), tag
    if not bip and i % 2 == 0:  # rich-club profile of the same samples from the statistics mode
        et, cnt = fm.sample_richclub(plan, seed, n_samples=R, first_sample=5)
        want = O.richclub_count(op.perm, ref.edges.reshape(-1, 2))
        assert np.array_equal(et.cpu().numpy().astype(np.int64), np.asarray(want).astype(np.int64)), tag


def test_concurrent_host_threads(O, monkeypatch):
    """Four host threads, each with its own stream, plan and seed, calling into the library at the
    same time (ctypes releases the GIL): every result equals the oracle's.  Half of the threads
    use pipelined sample groups (they share the device's side stream)."""
    import threading

    cases = []
    for k in range(4):
        x, y = WL.random_fitness(900 + k, 20_000 + 3_000 * k, 2.4, 0.02, ecm=True)
        cases.append((x, y if k % 2 else None, 100 + k))
    refs = [O.sample(O.sort_plan(x, y, seg_target=64), seed, n_samples=6, first_sample=k, nthreads=O.ncores())
            for k, (x, y, seed) in enumerate(cases)]
    monkeypatch.setenv("FM_SAMPLE_GROUPS", "2")
    out, errs = [None] * 4, []

    def work(k):
        try:
            x, y, seed = cases[k]
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                xd = torch.from_numpy(x).cuda()
                yd = None if y is None else torch.from_numpy(y).cuda()
                st.synchronize()
                for _ in range(3):  # repeated: overlapping calls of different threads
                    plan = fm.sort_plan(xd, yd, seg_target=64, stream=st)
                    e = (fm.sample_ubcm if y is None else fm.sample_ecm)(plan, seed, n_samples=6, first_sample=k, stream=st)
                    st.synchronize()
                    out[k] = (e.offsets.copy(), e.edges.cpu().numpy().copy(),
                              None if y is None else e.weights.cpu().numpy().copy())
        except Exception as ex:  # noqa: BLE001
            errs.append((k, repr(ex)))

    ths = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errs, errs
    for k in range(4):
        off, E, W = out[k]
        assert np.array_equal(off, refs[k].offsets), k
        assert np.array_equal(E.reshape(-1, 2), refs[k].edges.reshape(-1, 2)), k
        if W is not None:
            assert np.array_equal(W, refs[k].weights), k


# ------------------------------------------------------------------------------ API surface and extremes
@pytest.mark.parametrize("i", range(24))
def test_fuzz_api_surface(O, i):
    """Host-pointer plans, fm_edges_to_host, ECM strength sums (all graph kinds), the T1 expectation
    kernel on random nodes -- against the oracle on random small cases."""
    r = np.random.default_rng(3000 + i)
    ecm = bool(r.integers(2))
    kind = ("undirected", "bipartite", "directed")[int(r.integers(3))]
    n1 = int(r.choice([5, 40, 333, 2000]))
    n2 = n1 if kind != "bipartite" else int(r.choice([3, 77, 900]))
    scale = float(r.choice([0.02, 0.2, 1.0]))
    S, R, seed = int(r.choice([8, 50, 256])), int(r.choice([1, 6, 40])), int(r.integers(1 << 30))
    x1, y1 = WL.random_fitness(500 + i, n1, 2.5, scale, ecm=ecm)
    x2, y2 = WL.random_fitness(600 + i, n2, 2.5, scale, ecm=ecm)
    if kind == "undirected":
        plan = fm.sort_plan(x1, y1, seg_target=S)  # host (numpy) inputs
        op = O.sort_plan(x1, y1, seg_target=S)
    else:
        plan = fm.sort_plan_bipartite(x1, x2, y1, y2, kind=kind, seg_target=S)
        op = O.sort_plan(x1, y1, seg_target=S, kind=kind, x2=x2, y2=y2)
    e = (fm.sample_ecm if ecm else fm.sample_ubcm)(plan, seed, n_samples=R)
    ref = O.sample(op, seed, n_samples=R, nthreads=O.ncores())
    E, W = e.to_host()
    assert np.array_equal(E.reshape(-1, 2), ref.edges.reshape(-1, 2))
    if ecm:
        assert np.array_equal(W, ref.weights)
    dp, dm, sp, sm, cnt = fm.sample_degrees(plan, seed, n_samples=R)
    oe = ref.edges.reshape(-1, 2).astype(np.int64)
    ow = ref.weights.astype(np.int64) if ecm else np.ones(len(oe), np.int64)
    d1, d2 = np.bincount(oe[:, 0], minlength=n1), np.bincount(oe[:, 1], minlength=n2)
    s1 = np.bincount(oe[:, 0], weights=ow, minlength=n1).round().astype(np.int64)
    s2 = np.bincount(oe[:, 1], weights=ow, minlength=n2).round().astype(np.int64)
    if kind == "undirected":
        assert np.array_equal(dp.cpu().numpy(), d1 + d2)
        if ecm:
            assert np.array_equal(sp.cpu().numpy(), s1 + s2)
    else:
        assert np.array_equal(dp.cpu().numpy(), d1) and np.array_equal(dm.cpu().numpy(), d2)
        if ecm:
            assert np.array_equal(sp.cpu().numpy(), s1) and np.array_equal(sm.cpu().numpy(), s2)
    assert cnt["accepted"] == len(oe)
    if kind == "undirected":  # T1: exact expectations of random nodes
        nodes = r.choice(n1, size=min(n1, 50), replace=False).astype(np.int32)
        k, kv, s, sv = fm.expected_degrees(x1, y1, nodes=nodes)
        ok, okv, os_, osv = O.expected(x1, y1, nodes=nodes)
        assert np.allclose(k.cpu().numpy(), ok, rtol=1e-12, atol=1e-300)
        assert np.allclose(kv.cpu().numpy(), okv, rtol=1e-12, atol=1e-300)
        if ecm:
            assert np.allclose(s.cpu().numpy(), os_, rtol=1e-12) and np.allclose(sv.cpu().numpy(), osv, rtol=1e-11)


def test_extremes(O):
    """Many samples of tiny graphs (task counts far above the resident lanes), saturated and empty
    fitness mixes, the largest admissible first_sample, S at both ends of its range."""
    def same(x, y, S, seed, R, first=0):
        plan = fm.sort_plan(torch.from_numpy(x).cuda(), None if y is None else torch.from_numpy(y).cuda(), seg_target=S)
        e = (fm.sample_ubcm if y is None else fm.sample_ecm)(plan, seed, n_samples=R, first_sample=first)
        ref = O.sample(O.sort_plan(x, y, seg_target=S), seed, n_samples=R, first_sample=first, nthreads=O.ncores())
        assert np.array_equal(e.offsets, ref.offsets)
        assert np.array_equal(e.edges.cpu().numpy().reshape(-1, 2), ref.edges.reshape(-1, 2))
        if y is not None:
            assert np.array_equal(e.weights.cpu().numpy(), ref.weights)
        assert (e.draws, e.landed, e.accepted) == (ref.draws, ref.landed, ref.accepted)

    same(np.array([0.7, 1.9]), None, 256, 1, 300_000)                      # N = 2, 3e5 samples
    same(np.array([0.7, 1.9, 0.0]), np.array([0.5, 0.2, 0.3]), 8, 2, 100_000)  # N = 3 ECM, an isolated node
    x = np.concatenate([np.full(40, 1e6), np.zeros(300), np.full(60, 1e-6)])   # saturated core, isolated, near-empty
    same(x, None, 8, 3, 50)
    same(x, np.full(len(x), 0.9), 1 << 40, 4, 20)                           # y close to 1: long weight tails; S = 2^40
    xs, ys = WL.random_fitness(77, 3000, 2.2, 0.05, ecm=True)
    same(xs, ys, 8, 5, 3, first=(1 << 32) - 3)                              # last admissible samples


def test_no_device_memory_leak():
    """Plans, results and the tensor views of results are released by reference counting alone (the
    views once kept their result alive in a cycle through a torch tensor, which Python's collector
    cannot see: every result whose .edges had been read leaked); the library's own temporaries go
    back to the pool.  300 plan + sample cycles over the graph kinds and scheduling options."""
    import gc

    def free_mib():
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        fm.pool_trim(0)
        return torch.cuda.mem_get_info()[0] / 2**20

    x, y = WL.random_fitness(1, 30_000, 2.4, 0.02, ecm=True)
    x2, y2 = WL.random_fitness(2, 11_000, 2.4, 0.02, ecm=True)
    xd, yd, x2d, y2d = (torch.from_numpy(a).cuda() for a in (x, y, x2, y2))
    envs = [{}, {"FM_SAMPLE_GROUPS": "3"}, {"FM_DEBUG_SCRATCH_CAP": "8"}, {"FM_FUSE_WRITE": "1"}]

    def cycle(it):
        env = envs[it % len(envs)]
        os.environ.update(env)
        try:
            yy, yy2 = (yd, y2d) if it % 3 == 0 else (None, None)
            if it % 4 == 1:
                p = fm.sort_plan_bipartite(xd, x2d, yy, yy2, kind="bipartite", seg_target=64)
            else:
                p = fm.sort_plan(xd, yy, seg_target=64)
            e = (fm.sample_ubcm if yy is None else fm.sample_ecm)(p, it, n_samples=3)
            v = e.edges[:5].clone()  # a view of the result
            w = e.weights
            fm.sample_degrees(p, it, n_samples=1)
            return int(v.sum().item()) + (0 if w is None else 1)
        finally:
            for k in env:
                del os.environ[k]

    gc.collect()
    gc.disable()
    try:
        for it in range(12):  # every path once: lazily created streams, tables, module data
            cycle(it)
        f0 = free_mib()
        for it in range(300):
            cycle(it)
        f1 = free_mib()
    finally:
        gc.enable()
    assert f0 - f1 < 64, f"device memory: {f0:.0f} MiB free before, {f1:.0f} MiB after"


@pytest.mark.parametrize("ecm", [False, True])
@pytest.mark.parametrize("env", [{}, {"FM_HOST_GROUPS": "3"}, {"FM_DEBUG_SCRATCH_CAP": "8"}, {"FM_HOST_GROUPS": "1"},
                                 {"FM_HOST_GROUPS": "3", "FM_D2H_CHUNK_KB": "4", "FM_D2H_ALIGN": "256"},  # many aligned pieces
                                 {"FM_D2H_CHUNK_MB": "0"}])
def test_sample_to_host(O, monkeypatch, ecm, env):
    """fm_sample_to_host: the host buffers hold the oracle's list (copied group by group while later
    groups are sampled), also after forced slot overflows (re-run tasks: copied again); too small
    host buffers are reported, the device list stays valid."""
    x, y = WL.random_fitness(41, 25_000, 2.4, 0.02, ecm=True)
    yy = y if ecm else None
    R = 11
    ref = O.sample(O.sort_plan(x, yy, seg_target=64), 5, n_samples=R, first_sample=2, nthreads=O.ncores())
    n_e = len(ref.edges.reshape(-1, 2))
    plan = fm.sort_plan(torch.from_numpy(x).cuda(), None if yy is None else torch.from_numpy(yy).cuda(), seg_target=64)
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    eh = torch.full((n_e + 100, 2), -7, dtype=torch.int32).pin_memory()
    wh = torch.full((n_e + 100,), -7, dtype=torch.int32).pin_memory() if ecm else None
    e = fm.sample_to_host(plan, 5, eh, wh, n_samples=R, first_sample=2)
    assert not (e.flags & fm.FM_FLAG_HOST_TRUNCATED) and e.n_edges == n_e
    assert np.array_equal(e.offsets, ref.offsets)
    assert np.array_equal(eh.numpy()[:n_e], ref.edges.reshape(-1, 2))
    assert np.all(eh.numpy()[n_e:] == -7)  # nothing written beyond the list
    assert np.array_equal(e.edges.cpu().numpy(), ref.edges.reshape(-1, 2))  # the device list as well
    if ecm:
        assert np.array_equal(wh.numpy()[:n_e], ref.weights) and np.all(wh.numpy()[n_e:] == -7)
    # pageable numpy destination, exact size
    en = np.full((n_e, 2), -7, np.int32)
    e2 = fm.sample_to_host(plan, 5, en, None, n_samples=R, first_sample=2)
    assert np.array_equal(en, ref.edges.reshape(-1, 2)) and e2.n_edges == n_e
    # too small: reported, buffers unspecified, fm_edges_to_host still works
    small = np.full((n_e // 2, 2), -7, np.int32)
    e3 = fm.sample_to_host(plan, 5, small, None, n_samples=R, first_sample=2)
    assert e3.flags & fm.FM_FLAG_HOST_TRUNCATED and e3.n_edges == n_e
    E3, _ = e3.to_host()
    assert np.array_equal(E3, ref.edges.reshape(-1, 2))
