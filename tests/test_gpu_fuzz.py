"""Seeded random sweep of the whole C-ABI surface against the oracle: model x graph kind x size x
fitness scale x segmentation target x sample range x ECM bound refresh x scheduling options, every
case element by element (offsets, edges in canonical order, weights, counters).  Small sizes: the
sweep spans the degenerate regimes (empty rows, saturated hubs, one-segment and many-segment rows,
tasks of a single draw) that the fixed-size tests only touch."""
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


@pytest.mark.parametrize("i", range(160))
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
