"""Full-size BASELINE.json configs on the GPU, in the launch configuration bench.py times (one
fm_sample_* call over all R samples of the config):

* parity: EVERY sample of configs 4 (4 samples, N = 1e7) and 5 (64 samples, N = 1e6, 12.8 GB)
  against the oracle's sample with the same (seed, sample index), streamed one sample at a time
  (O.sample(first_sample=s)); the GPU list is compared element by element (canonical order), and
  as sets when they differ: at most 1e-6 of the edges may differ (north star; the slack is for
  libm-vs-CUDA log ulps only);
* statistical gates (SPEC acceptance 7, "every node"; P:L233 degree
  preservation): per-node degree sums over the R samples against the exact expectation
  sum_j p_ij and variance sum_j p_ij (1 - p_ij) from the T1 expectation kernel
  (fm_expected_degrees), itself checked against the oracle's closed form on 1,000 random nodes;
  5 sigma on 1,000 random nodes and the Bonferroni bound plus an aggregate chi-square over all
  nodes (tests/_stats.py: node_gate);
* configs 1 and 2: the per-node gate over their ensembles (10,000 and 100 samples), all nodes.
"""
import numpy as np
import pytest

from paper_2509_13230_b200 import workloads as WL
from _stats import node_gate

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402


def keys(e, n, w=None):
    k = e[:, 0].astype(np.int64) * n + e[:, 1]
    if w is not None:
        k = k * (1 << 31) + w.astype(np.int64)
    return np.sort(k)


def degree_sums_gpu(e, n, samples=None):
    """per-node degree summed over the samples of an Edges result (float64 CUDA tensor)."""
    D = torch.zeros(n, dtype=torch.float64, device="cuda")
    for s in (range(e.n_samples) if samples is None else samples):
        a, b = int(e.offsets[s]), int(e.offsets[s + 1])
        E = e.edges[a:b].long()
        D += torch.bincount(E[:, 0], minlength=n).double() + torch.bincount(E[:, 1], minlength=n).double()
    return D


def expected_checked(O, x, y, rng_seed, n_check=1000, nodes=None):
    """T1 expectations (all nodes, or `nodes`) checked against the oracle's closed form."""
    n = len(x)
    k, kv, s, sv = fm.expected_degrees(torch.from_numpy(x).cuda(), None if y is None else torch.from_numpy(y).cuda(),
                                       nodes=None if nodes is None else torch.from_numpy(nodes).cuda())
    pool = np.arange(n, dtype=np.int32) if nodes is None else nodes
    pick = np.random.default_rng(rng_seed).choice(len(pool), min(n_check, len(pool)), replace=False)
    ok, okv, os_, osv = O.expected(x, y, nodes=pool[pick].astype(np.int32))
    assert np.allclose(k.cpu().numpy()[pick], ok, rtol=1e-9, atol=1e-12)
    assert np.allclose(kv.cpu().numpy()[pick], okv, rtol=1e-9, atol=1e-12)
    if y is not None:
        assert np.allclose(s.cpu().numpy()[pick], os_, rtol=1e-9, atol=1e-12)
        assert np.allclose(sv.cpu().numpy()[pick], osv, rtol=1e-8, atol=1e-12)
    return k, kv, s, sv


def streamed_parity(O, x, y, w, e, perm_gpu):
    """every sample of e (one call over all samples) vs the oracle's sample s; returns (bad, total)."""
    n = len(x)
    oplan = O.sort_plan(x, y)
    assert np.array_equal(oplan.perm, perm_gpu), "sorted order differs"
    bad = tot = exact = 0
    for s in range(w.n_samples):
        a, b = int(e.offsets[s]), int(e.offsets[s + 1])
        g = e.edges[a:b].cpu().numpy()
        gw = None if e.weights is None else e.weights[a:b].cpu().numpy()
        ref = O.sample(oplan, w.seed, n_samples=1, first_sample=s, nthreads=O.ncores())
        o = ref.edges
        tot += len(o)
        if g.shape == o.shape and np.array_equal(g, o) and (gw is None or np.array_equal(gw, ref.weights)):
            exact += 1
            continue
        bad += len(np.setxor1d(keys(g, n, gw), keys(o, n, None if gw is None else ref.weights)))
    return bad, tot, exact


@pytest.mark.parametrize("cfg", [4, 5])
def test_full_config_parity_every_sample_and_all_node_gate(O, cfg):
    w = WL.workload(cfg)
    x, y = WL.fitness(w)
    n = len(x)
    plan = fm.sort_plan(torch.from_numpy(x).cuda())
    e = fm.sample_ubcm(plan, w.seed, n_samples=w.n_samples)
    torch.cuda.synchronize()
    assert e.n_edges == int(e.offsets[-1]) == e.accepted
    assert abs(e.n_edges / w.n_samples / (n * w.kbar / 2) - 1) < 0.02
    bad, tot, exact = streamed_parity(O, x, y, w, e, plan.export()["perm"])
    assert tot == e.n_edges or bad > 0
    assert bad <= int(1e-6 * tot), f"{bad} of {tot} edges differ ({exact}/{w.n_samples} samples identical)"
    # statistical gates: per-node degree sums over the R samples vs the exact T1 expectation
    D = degree_sums_gpu(e, n)
    assert int(D.sum().item()) == 2 * e.n_edges
    R = w.n_samples
    if cfg == 5:
        k, kv, _, _ = expected_checked(O, x, None, 11)                     # all 1e6 nodes
        node_gate(D.cpu().numpy(), k.cpu().numpy(), kv.cpu().numpy(), R)  # Bonferroni z* ~ 6.1 + chi2
    else:
        nodes = np.random.default_rng(12).choice(n, 200_000, replace=False).astype(np.int32)
        k, kv, _, _ = expected_checked(O, x, None, 12, nodes=nodes)
        idx = torch.from_numpy(nodes).cuda().long()
        node_gate(D[idx].cpu().numpy(), k.cpu().numpy(), kv.cpu().numpy(), R)
    # 5 sigma on 1,000 random nodes, expectation straight from the oracle
    nodes = np.random.default_rng(1).choice(n, 1000, replace=False).astype(np.int32)
    ok, okv, _, _ = O.expected(x, None, nodes=nodes)
    node_gate(D[torch.from_numpy(nodes).cuda().long()].cpu().numpy(), ok, okv, R, sigma=5.0)
    # statistics mode on the same samples: identical sums without the edge list (NEXT-3)
    dp, _, _, _, cnt = fm.sample_degrees(plan, w.seed, n_samples=R)
    assert cnt["accepted"] == e.n_edges and cnt["draws"] == e.draws
    assert torch.equal(dp.double(), D)


def test_config1_and_2_node_gates(O):
    # config 1: the 10,000-sample ensemble, every node, 5 sigma
    w = WL.workload(1)
    x, _ = WL.fitness(w)
    plan = fm.sort_plan(torch.from_numpy(x).cuda())
    e = fm.sample_ubcm(plan, w.seed, n_samples=10_000)
    E = e.edges.long()
    D = torch.bincount(E[:, 0], minlength=w.n).double() + torch.bincount(E[:, 1], minlength=w.n).double()
    k, kv, _, _ = expected_checked(O, x, None, 3)
    node_gate(D.cpu().numpy(), k.cpu().numpy(), kv.cpu().numpy(), 10_000, sigma=5.0)
    # config 2: 100 samples, all 1e5 nodes (Bonferroni) and 1,000 random nodes at 5 sigma
    w = WL.workload(2)
    x, _ = WL.fitness(w)
    plan = fm.sort_plan(torch.from_numpy(x).cuda())
    e = fm.sample_ubcm(plan, w.seed, n_samples=w.n_samples)
    D = degree_sums_gpu(e, w.n)
    k, kv, _, _ = expected_checked(O, x, None, 4)
    node_gate(D.cpu().numpy(), k.cpu().numpy(), kv.cpu().numpy(), w.n_samples)
    nodes = np.random.default_rng(5).choice(w.n, 1000, replace=False)
    node_gate(D.cpu().numpy()[nodes], k.cpu().numpy()[nodes], kv.cpu().numpy()[nodes], w.n_samples, sigma=5.0)


def test_config2_statistics_mode_equals_oracle_sums(O):
    """fm_sample_degrees (NEXT-3) against degree sums over the ORACLE's samples (same seed and
    sample indices), not only against the GPU's own edge lists."""
    w = WL.workload(2)
    x, _ = WL.fitness(w)
    plan = fm.sort_plan(torch.from_numpy(x).cuda())
    dp, _, _, _, cnt = fm.sample_degrees(plan, w.seed, n_samples=w.n_samples)
    ref = O.sample(O.sort_plan(x), w.seed, n_samples=w.n_samples, nthreads=O.ncores())
    od = np.bincount(ref.edges[:, 0], minlength=w.n) + np.bincount(ref.edges[:, 1], minlength=w.n)
    diff = int(np.abs(dp.cpu().numpy() - od).sum())
    assert diff <= 2 * int(1e-6 * ref.accepted), diff
    assert cnt["accepted"] == ref.accepted or diff > 0


def test_config3_ecm_strength_gate(O):
    w = WL.workload(3)
    x, y = WL.fitness(w)
    n = len(x)
    plan = fm.sort_plan(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    e = fm.sample_ecm(plan, w.seed, n_samples=w.n_samples)
    R = w.n_samples
    E, W = e.edges.long(), e.weights.double()
    deg = torch.bincount(E[:, 0], minlength=n).double() + torch.bincount(E[:, 1], minlength=n).double()
    st = torch.bincount(E[:, 0], weights=W, minlength=n) + torch.bincount(E[:, 1], weights=W, minlength=n)
    k, kv, s, sv = expected_checked(O, x, y, 6)
    node_gate(deg.cpu().numpy(), k.cpu().numpy(), kv.cpu().numpy(), R)   # all nodes, Bonferroni
    big = (R * sv >= 25).cpu().numpy()
    node_gate(st.cpu().numpy()[big], s.cpu().numpy()[big], sv.cpu().numpy()[big], R)
    # statistics mode == edge-list sums
    dp, _, sp, _, _ = fm.sample_degrees(plan, w.seed, n_samples=R)
    assert torch.equal(dp.double(), deg) and torch.equal(sp.double(), st)
    # pooled weight law vs Eq. 5 over all edges of sample 0, binned by t
    from scipy import stats
    a, b = int(e.offsets[0]), int(e.offsets[1])
    E0 = e.edges[a:b].cpu().numpy()
    W0 = e.weights[a:b].cpu().numpy()
    t = y[E0[:, 0]] * y[E0[:, 1]]
    for lo, hi in zip(np.quantile(t, [0, .25, .5, .75]), np.quantile(t, [.25, .5, .75, 1])):
        msk = (t >= lo) & (t <= hi)
        tt, ww = t[msk], np.minimum(W0[msk], 11)
        obs = np.bincount(ww, minlength=12)[1:]
        exp = np.array([np.sum(tt ** (j - 1) * (1 - tt)) for j in range(1, 11)] + [np.sum(tt ** 10)])
        keep = exp >= 5
        assert stats.chi2.sf(np.sum((obs[keep] - exp[keep]) ** 2 / exp[keep]), keep.sum() - 1) > 1e-4
