"""Full-size BASELINE.json configs 4 and 5 on the GPU, in the launch configuration bench.py times:
parity on sampled rows (the oracle computes chosen rows one by one) and the statistical gates
(per-node mean degree vs the exact expectation sum_j p_ij on 1,000 random nodes)."""
import math

import numpy as np
import pytest
from scipy import stats

from paper_2509_13230_b200 import workloads as WL

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402


def rows_of(edges_t, rank_t):
    """sorted-rank row of each GPU edge (the endpoint with the smaller rank)."""
    return torch.minimum(rank_t[edges_t[:, 0].long()], rank_t[edges_t[:, 1].long()])


def sampled_row_parity(O, x, y, w, samples, n_rows=600, seed=0):
    n = len(x)
    xd = torch.from_numpy(x).cuda()
    yd = None if y is None else torch.from_numpy(y).cuda()
    plan = fm.sort_plan(xd, yd)
    fn = fm.sample_ubcm if y is None else fm.sample_ecm
    e = fn(plan, w.seed, n_samples=w.n_samples)
    torch.cuda.synchronize()
    perm = torch.from_numpy(plan.export()["perm"]).cuda().long()
    rank = torch.empty_like(perm)
    rank[perm] = torch.arange(n, device="cuda")
    oplan = O.sort_plan(x, y)
    assert np.array_equal(oplan.perm, perm.cpu().numpy())
    rng = np.random.default_rng(seed)
    rows = np.unique(np.concatenate([np.arange(40), rng.choice(n - 1, n_rows, replace=False)])).astype(np.int32)
    rows_t = torch.from_numpy(rows).cuda().long()
    bad = tot = 0
    for s in samples:
        a, b = int(e.offsets[s]), int(e.offsets[s + 1])
        E = e.edges[a:b]
        r = rows_of(E, rank)
        sel = torch.isin(r, rows_t)
        g = E[sel].cpu().numpy().astype(np.int64)
        gw = None if e.weights is None else e.weights[a:b][sel].cpu().numpy()
        ref = O.sample(oplan, w.seed, n_samples=1, first_sample=s, rows=rows, nthreads=O.ncores())
        o = ref.edges.astype(np.int64)
        kg, ko = g[:, 0] * n + g[:, 1], o[:, 0] * n + o[:, 1]
        if gw is not None:
            kg, ko = kg * (1 << 31) + gw, ko * (1 << 31) + ref.weights
        bad += len(np.setxor1d(kg, ko))
        tot += len(ko)
    return e, plan, bad, tot


@pytest.mark.parametrize("cfg", [4, 5])
def test_full_config_sampled_rows_and_degrees(O, cfg):
    w = WL.workload(cfg)
    x, y = WL.fitness(w)
    n = len(x)
    samples = [0, w.n_samples - 1] if cfg == 4 else [0, 31, 63]
    e, plan, bad, tot = sampled_row_parity(O, x, y, w, samples)
    assert tot > 1000
    assert bad <= max(0, int(1e-6 * tot)) + 0, f"{bad} of {tot} sampled-row edges differ"
    # hygiene + totals
    assert e.n_edges == int(e.offsets[-1])
    mean_edges = e.n_edges / w.n_samples
    assert abs(mean_edges / (n * w.kbar / 2) - 1) < 0.02
    # statistical gate: per-node mean degree over the R samples vs exact sum_j p_ij (1,000 nodes)
    R = w.n_samples
    deg = torch.zeros(n, dtype=torch.float64, device="cuda")
    for s in range(R):
        a, b = int(e.offsets[s]), int(e.offsets[s + 1])
        E = e.edges[a:b].long()
        deg += torch.bincount(E[:, 0], minlength=n).double() + torch.bincount(E[:, 1], minlength=n).double()
    nodes = np.random.default_rng(1).choice(n, 1000, replace=False).astype(np.int32)
    k, kv, _, _ = O.expected(x, y, nodes=nodes)
    m = deg[torch.from_numpy(nodes).cuda().long()].cpu().numpy() / R
    big = R * kv >= 25
    z = (m - k) / np.sqrt(kv / R)
    assert np.max(np.abs(z[big])) < 5.0, np.max(np.abs(z[big]))
    # all chosen nodes together: chi-square of the standardised means
    stat = float(np.sum(z[kv > 0] ** 2))
    assert stats.chi2.sf(stat, int((kv > 0).sum())) > 1e-4, stat


def test_config3_ecm_strength_gate(O):
    w = WL.workload(3)
    x, y = WL.fitness(w)
    n = len(x)
    plan = fm.sort_plan(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    e = fm.sample_ecm(plan, w.seed, n_samples=w.n_samples)
    R = w.n_samples
    deg = torch.zeros(n, dtype=torch.float64, device="cuda")
    st = torch.zeros(n, dtype=torch.float64, device="cuda")
    E, W = e.edges.long(), e.weights.double()
    deg += torch.bincount(E[:, 0], minlength=n).double() + torch.bincount(E[:, 1], minlength=n).double()
    st += torch.bincount(E[:, 0], weights=W, minlength=n) + torch.bincount(E[:, 1], weights=W, minlength=n)
    nodes = np.random.default_rng(2).choice(n, 1000, replace=False).astype(np.int32)
    k, kv, s, sv = O.expected(x, y, nodes=nodes)
    idx = torch.from_numpy(nodes).cuda().long()
    mk, ms = deg[idx].cpu().numpy() / R, st[idx].cpu().numpy() / R
    zk, zs = (mk - k) / np.sqrt(kv / R), (ms - s) / np.sqrt(sv / R)
    assert np.max(np.abs(zk[R * kv >= 25])) < 5 and np.max(np.abs(zs[R * sv >= 25])) < 5
    # pooled weight law vs Eq. 5 over all edges of sample 0, binned by t
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
