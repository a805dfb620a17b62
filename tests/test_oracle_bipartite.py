"""Pins of the bipartite and directed extensions: the + set is swept
row by row against the - set sorted by its own key, with no j > i restriction; directed graphs are
the bipartite graph of out- and in-copies without the diagonal."""
import numpy as np
import pytest
from scipy import stats

from paper_2509_13230_b200 import workloads as WL
from _stats import two_sample_z

R = 100_000


def fit(seed, n, c=0.3, ecm=False):
    return WL.random_fitness(seed, n, 2.5, c, ecm=ecm)


def pcounts(res, n1, n2):
    idx = res.edges[:, 0].astype(np.int64) * n2 + res.edges[:, 1]
    return np.bincount(idx, minlength=n1 * n2).reshape(n1, n2)


def chi2_cells(c, Rn, P, mask):
    var = Rn * P * (1 - P)
    m = mask & (var >= 5)
    z = (c[m] - Rn * P[m]) / np.sqrt(var[m])
    return float(np.sum(z * z)), int(m.sum()), float(np.max(np.abs(z)))


def cross_p(x1, y1, x2, y2):
    if y1 is None:
        X = np.outer(x1, x2)
        return X / (1 + X), None
    t = np.outer(y1, y2)
    z = np.outer(x1, x2) * t
    return z / (1 - t + z), t


@pytest.mark.parametrize("ecm", [False, True])
@pytest.mark.parametrize("kind", ["bipartite", "directed"])
@pytest.mark.parametrize("S", [8, 1 << 40])
def test_pair_frequencies(O, kind, ecm, S):
    n1, n2 = (9, 7) if kind == "bipartite" else (8, 8)
    x1, y1 = fit(11, n1, 0.8, ecm)
    x2, y2 = fit(12, n2, 0.6, ecm)
    x1[0] = 30.0  # a saturated hub row: the first candidate is bounded by itself (bound position 0)
    pl = O.sort_plan(x1, y1, seg_target=S, kind=kind, x2=x2, y2=y2)
    res = O.sample(pl, seed=77 + S, n_samples=R, nthreads=O.ncores())
    c = pcounts(res, n1, n2)
    P, T = cross_p(x1, y1, x2, y2)
    mask = np.ones_like(P, bool)
    if kind == "directed":
        np.fill_diagonal(mask, False)
        assert np.all(np.diag(c) == 0)  # no self loops
    stat, dof, zmax = chi2_cells(c, R, P, mask)
    assert dof > 20 and stats.chi2.sf(stat, dof) > 1e-4 and zmax < 5.5, (stat, dof, zmax)
    bf = O.bruteforce(x1, y1, seed=5 + S, n_samples=R, kind=kind, x2=x2, y2=y2)
    cb = pcounts(bf, n1, n2)
    if kind == "directed":
        assert np.all(np.diag(cb) == 0)
    # two-sample test on all cells (square helper: embed)
    m = max(n1, n2)
    A, B = np.zeros((m, m)), np.zeros((m, m))
    A[:n1, :n2], B[:n1, :n2] = c, cb
    st2, d2, pv2 = two_sample_z(A, B, R, R)  # uses the upper triangle; check the transpose too
    st3, d3, pv3 = two_sample_z(A.T.copy(), B.T.copy(), R, R)
    assert pv2 > 1e-4 and pv3 > 1e-4
    if ecm:
        w = res.weights
        assert w.min() >= 1
        t = T[res.edges[:, 0], res.edges[:, 1]]
        for lo, hi in zip(np.quantile(t, [0, .5]), np.quantile(t, [.5, 1])):
            msk = (t >= lo) & (t <= hi)
            tt, ww = t[msk], np.minimum(w[msk], 8)
            obs = np.bincount(ww, minlength=9)[1:]
            exp = np.array([np.sum(tt ** (j - 1) * (1 - tt)) for j in range(1, 8)] + [np.sum(tt ** 7)])
            keep = exp >= 5
            assert stats.chi2.sf(np.sum((obs[keep] - exp[keep]) ** 2 / exp[keep]), keep.sum() - 1) > 1e-4


def test_full_joint_bipartite_2x3(O):
    x1, x2 = np.array([2.0, 0.4]), np.array([1.5, 0.7, 0.2])
    pl = O.sort_plan(x1, None, seg_target=8, kind="bipartite", x2=x2)
    RR = 300_000
    res = O.sample(pl, seed=3, n_samples=RR, nthreads=O.ncores())
    bit = {(i, j): 1 << (3 * i + j) for i in range(2) for j in range(3)}
    codes = np.zeros(RR, np.int64)
    sid = np.repeat(np.arange(RR), np.diff(res.offsets))
    np.add.at(codes, sid, np.array([bit[(int(a), int(b))] for a, b in res.edges]))
    obs = np.bincount(codes, minlength=64)
    P, _ = cross_p(x1, None, x2, None)
    exp = np.ones(64)
    for code in range(64):
        for (i, j), bb in bit.items():
            exp[code] *= P[i, j] if code & bb else 1 - P[i, j]
    exp *= RR
    assert stats.chi2.sf(np.sum((obs - exp) ** 2 / exp), 63) > 1e-4


@pytest.mark.parametrize("kind", ["bipartite", "directed"])
def test_degrees_closed_form(O, kind):
    n1, n2 = (300, 200) if kind == "bipartite" else (300, 300)
    x1, y1 = fit(21, n1, 0.08, True)
    x2, y2 = fit(22, n2, 0.08, True)
    RR = 2000
    pl = O.sort_plan(x1, y1, seg_target=16, kind=kind, x2=x2, y2=y2)
    res = O.sample(pl, seed=31, n_samples=RR, nthreads=O.ncores())
    ko, kov, ki, kiv = O.expected2(x1, y1, x2, y2, kind=kind)
    dout = np.bincount(res.edges[:, 0], minlength=n1) / RR
    din = np.bincount(res.edges[:, 1], minlength=n2) / RR
    zo = (dout - ko) / np.sqrt(kov / RR)
    zi = (din - ki) / np.sqrt(kiv / RR)
    assert np.max(np.abs(zo[RR * kov > 25])) < 5 and np.max(np.abs(zi[RR * kiv > 25])) < 5


def test_bipartite_plan_and_determinism(O):
    x1, y1 = fit(1, 500, 0.05, True)
    x2, y2 = fit(2, 333, 0.05, True)
    pl = O.sort_plan(x1, y1, seg_target=8, kind="bipartite", x2=x2, y2=y2)
    assert pl.nc == 333 and set(np.unique(pl.seg_u)) == set(range(500))  # every + row has candidates
    first = np.r_[True, pl.seg_u[1:] != pl.seg_u[:-1]]
    assert np.all(pl.seg_a[first] == 0) and np.all(pl.seg_b[np.r_[first[1:], True]] == 333)
    assert np.array_equal(pl.cperm, np.lexsort((np.arange(333), -(x2 * y2))))
    a = O.sample(pl, seed=4, n_samples=3, nthreads=1)
    b = O.sample(pl, seed=4, n_samples=3, nthreads=5)
    assert np.array_equal(a.edges, b.edges) and np.array_equal(a.weights, b.weights)
    # directed: exclusion map points at each row's own in-copy
    pd = O.sort_plan(x1, y1, kind="directed", x2=x1 * 0.7, y2=y1)
    assert np.array_equal(pd.cperm[pd.excl], pd.perm)
    with pytest.raises(O.OracleError):
        O.sort_plan(x1, y1, kind="directed", x2=x2, y2=y2)  # n1 != n2
