"""fm_sample_degrees (NEXT-3): per-node degree/strength sums over an ensemble without edge lists --
identical to the sums over the edge lists of the same samples, and on full-size config 5 within
5 sigma of the exact expectation (the BASELINE.json config-5 gate without materialising 12.8 GB)."""
import numpy as np
import pytest

from paper_2509_13230_b200 import workloads as WL

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402


def edge_sums(e, n1, n2, bip):
    E = e.edges.long()
    W = None if e.weights is None else e.weights.long()
    d1 = torch.bincount(E[:, 0], minlength=n1)
    d2 = torch.bincount(E[:, 1], minlength=n2)
    s1 = s2 = None
    if W is not None:
        s1 = torch.bincount(E[:, 0], weights=W.double(), minlength=n1).round().long()
        s2 = torch.bincount(E[:, 1], weights=W.double(), minlength=n2).round().long()
    if not bip:
        return d1 + d2, None, (None if W is None else s1 + s2), None
    return d1, d2, s1, s2


@pytest.mark.parametrize("ecm", [False, True])
@pytest.mark.parametrize("kind", ["undirected", "bipartite", "directed"])
def test_degrees_equal_edge_list_sums(O, kind, ecm):
    n1 = 20_000
    n2 = 15_000 if kind == "bipartite" else n1
    x1, y1 = WL.random_fitness(5, n1, 2.3, 0.01, ecm=ecm)
    x2, y2 = WL.random_fitness(6, n2, 2.3, 0.01, ecm=ecm)
    dev = lambda a: None if a is None else torch.from_numpy(a).cuda()  # noqa: E731
    if kind == "undirected":
        plan = fm.sort_plan(dev(x1), dev(y1), seg_target=64)
    else:
        plan = fm.sort_plan_bipartite(dev(x1), dev(x2), dev(y1), dev(y2), kind=kind, seg_target=64)
    fn = fm.sample_ecm if ecm else fm.sample_ubcm
    e = fn(plan, 9, n_samples=6, first_sample=4)
    dp, dm, sp, sm, cnt = fm.sample_degrees(plan, 9, n_samples=6, first_sample=4)
    assert cnt["accepted"] == e.accepted and cnt["draws"] == e.draws
    r1, r2, q1, q2 = edge_sums(e, n1, n2, kind != "undirected")
    assert torch.equal(dp, r1)
    if kind != "undirected":
        assert torch.equal(dm, r2)
    if ecm:
        assert torch.equal(sp, q1)
        if kind != "undirected":
            assert torch.equal(sm, q2)
    # ... and to the sums over the ORACLE's samples of the same seeds (not only the GPU's own lists)
    okind = {"undirected": O.UNDIRECTED, "bipartite": O.BIPARTITE, "directed": O.DIRECTED}[kind]
    if kind == "undirected":
        op = O.sort_plan(x1, y1, seg_target=64)
    else:
        op = O.sort_plan(x1, y1, seg_target=64, kind=okind, x2=x2, y2=y2)
    ref = O.sample(op, 9, n_samples=6, first_sample=4, nthreads=O.ncores())
    oe = ref.edges.astype(np.int64)
    o1, o2 = np.bincount(oe[:, 0], minlength=n1), np.bincount(oe[:, 1], minlength=n2)
    if kind == "undirected":
        assert np.array_equal(dp.cpu().numpy(), o1 + o2)
    else:
        assert np.array_equal(dp.cpu().numpy(), o1) and np.array_equal(dm.cpu().numpy(), o2)
    if ecm:
        ow = ref.weights.astype(np.int64)
        w1 = np.bincount(oe[:, 0], weights=ow, minlength=n1).round().astype(np.int64)
        w2 = np.bincount(oe[:, 1], weights=ow, minlength=n2).round().astype(np.int64)
        if kind == "undirected":
            assert np.array_equal(sp.cpu().numpy(), w1 + w2)
        else:
            assert np.array_equal(sp.cpu().numpy(), w1) and np.array_equal(sm.cpu().numpy(), w2)


def test_config5_degree_gate_without_edge_lists(O):
    w = WL.workload(5)
    x, _ = WL.fitness(w)
    plan = fm.sort_plan(torch.from_numpy(x).cuda())
    dp, _, _, _, cnt = fm.sample_degrees(plan, w.seed, n_samples=w.n_samples)
    R = w.n_samples
    assert abs(cnt["accepted"] / R / (len(x) * w.kbar / 2) - 1) < 0.02
    nodes = np.random.default_rng(3).choice(len(x), 1000, replace=False).astype(np.int32)
    k, kv, _, _ = O.expected(x, None, nodes=nodes)
    m = dp[torch.from_numpy(nodes).cuda().long()].cpu().numpy() / R
    z = (m - k) / np.sqrt(kv / R)
    assert np.max(np.abs(z[R * kv >= 25])) < 5.0
    assert abs(int(dp.sum().item()) - 2 * cnt["accepted"]) == 0


def test_rank_out_plan_without_records(O, monkeypatch):
    """A plan above the rank-out threshold holds no (kappa, id) records: the statistics mode and the
    overflow re-runs gather from the two arrays instead; all agree with the oracle's samples."""
    monkeypatch.setenv("FM_UBCM_RANK_OUT_MIN", "1000")
    n = 30_000
    x, _ = WL.random_fitness(11, n, 2.4, 0.02, ecm=False)
    plan = fm.sort_plan(torch.from_numpy(x).cuda(), seg_target=64)
    e = fm.sample_ubcm(plan, 3, n_samples=5, first_sample=2)
    dp, _, _, _, cnt = fm.sample_degrees(plan, 3, n_samples=5, first_sample=2)
    assert cnt["accepted"] == e.accepted and cnt["draws"] == e.draws
    r, _, _, _ = edge_sums(e, n, n, False)
    assert torch.equal(dp, r)
    ref = O.sample(O.sort_plan(x, None, seg_target=64), 3, n_samples=5, first_sample=2, nthreads=O.ncores())
    oe = ref.edges.astype(np.int64)
    assert np.array_equal(dp.cpu().numpy(), np.bincount(oe[:, 0], minlength=n) + np.bincount(oe[:, 1], minlength=n))
    assert np.array_equal(np.asarray(e.offsets), ref.offsets)
    # tiny scratch slots: the overflowed tasks are re-run straight into the list (record-free gathers)
    monkeypatch.setenv("FM_DEBUG_SCRATCH_CAP", "8")
    plan2 = fm.sort_plan(torch.from_numpy(x).cuda(), seg_target=64)
    e2 = fm.sample_ubcm(plan2, 3, n_samples=5, first_sample=2)
    assert torch.equal(e2.edges, e.edges) and np.array_equal(np.asarray(e2.offsets), np.asarray(e.offsets))
