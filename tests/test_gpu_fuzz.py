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
