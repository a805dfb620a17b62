"""Pins of the oracle's closed forms and plan."""
import math
import os

import numpy as np
import pytest

from paper_2509_13230_b200 import workloads as WL

GOLD = os.path.join(os.path.dirname(__file__), "golden", "model_examples.txt")


def test_model_examples_closed_form(O):
    """SPEC S:L80-84, S:L92, S:L122 examples (Eq. 4) via the oracle closed forms on N=2."""
    for line in open(GOLD):
        if line.startswith("#") or not line.strip() or line.startswith("pmf"):
            continue
        model, xi, xj, yi, yj, p, ew = line.split()
        x = np.array([float(xi), float(xj)])
        y = None if model == "ubcm" else np.array([float(yi), float(yj)])
        k, kv, s, sv = O.expected(x, y)
        assert k[0] == pytest.approx(float(p), abs=1e-15) and k[1] == pytest.approx(float(p), abs=1e-15)
        assert kv[0] == pytest.approx(float(p) * (1 - float(p)), abs=1e-15)
        if ew != "-":
            assert s[0] == pytest.approx(float(ew), abs=1e-12)


def test_weight_pmf_examples(O):
    """SPEC S:L102-103 (Eq. 5): P(w = 1 | edge) = 0.5 and P(w = 3 | edge) = 0.125 at t = 1/2, on
    the sampler's own weights: N = 2, x = (1, 1), y = (sqrt(1/2), sqrt(1/2)) (so p = 0.5),
    200,000 samples; 5 sigma."""
    rows = [ln.split() for ln in open(GOLD) if ln.startswith("pmf")]
    assert len(rows) == 2
    R = 200_000
    for _, w, yi, yj, pw in rows:
        x = np.array([1.0, 1.0])
        y = np.array([float(yi), float(yj)])
        r = O.sample(O.sort_plan(x, y), seed=77, n_samples=R)
        m = len(r.weights)
        assert abs(m - 0.5 * R) < 5 * np.sqrt(0.25 * R)  # p = 0.5
        q = float(pw)
        hits = int(np.sum(r.weights == int(w)))
        assert abs(hits - q * m) < 5 * np.sqrt(q * (1 - q) * m), (w, hits, m)


def test_weight_moments_closed_form(O):
    """E[s] and Var[s] against truncated series of Eq. 3-5: sum_w w p t^{w-1}(1-t)."""
    x = np.array([0.7, 1.3, 0.2])
    y = np.array([0.6, 0.8, 0.3])
    k, kv, s, sv = O.expected(x, y)
    w = np.arange(1, 4000, dtype=np.float64)
    es = ev = 0.0
    for j in (1, 2):
        t = y[0] * y[j]
        z = x[0] * x[j] * t
        p = z / (1 - t + z)
        pmf = t ** (w - 1) * (1 - t)
        assert pmf.sum() == pytest.approx(1.0, abs=1e-12)
        m1 = p * np.sum(w * pmf)
        m2 = p * np.sum(w * w * pmf)
        es += m1
        ev += m2 - m1 * m1
    assert s[0] == pytest.approx(es, rel=1e-12)
    assert sv[0] == pytest.approx(ev, rel=1e-10)


def test_expected_edges_consistent(O):
    x, y = WL.random_fitness(3, 257, 2.5, 0.05, ecm=True)
    for yy in (None, y):
        k = O.expected(x, yy)[0]
        assert O.expected_edges(x, yy) == pytest.approx(k.sum() / 2, rel=1e-12)
        assert O.expected_edges_binned(x, yy) == pytest.approx(k.sum() / 2, rel=2e-2)


# ---------------------------------------------------------------------------------- plan
@pytest.mark.parametrize("ecm", [False, True])
@pytest.mark.parametrize("S", [8, 37, 256])
def test_plan_invariants(O, ecm, S):
    x, y = WL.random_fitness(11, 3001, 2.2, 0.02, ecm=ecm)
    x[5] = x[17]  # ties
    if ecm:
        y[5] = y[17]
    pl = O.sort_plan(x, y, seg_target=S)
    n = len(x)
    kappa = x * y if ecm else x
    # permutation, non-increasing key, ties by ascending id (R9)
    assert np.array_equal(np.sort(pl.perm), np.arange(n))
    assert np.array_equal(pl.kappa_s, kappa[pl.perm])
    assert np.all(np.diff(pl.kappa_s) <= 0)
    eq = np.diff(pl.kappa_s) == 0
    assert np.all(np.diff(pl.perm)[eq] > 0)
    order = np.lexsort((np.arange(n), -kappa))
    assert np.array_equal(pl.perm, order)
    if ecm:
        assert np.array_equal(pl.y_s, y[pl.perm])
        ref = np.maximum.accumulate(pl.y_s[::-1])[::-1]
        assert np.array_equal(pl.ymax[:-1], ref) and pl.ymax[-1] == 0.0
    # F and fixed-point prefix
    e = math.frexp(pl.kappa_s[0])[1]
    L = math.ceil(math.log2(n))
    assert pl.F == 61 - e - L
    assert pl.P[0] == 0 and np.all(np.diff(pl.P.astype(object)) >= 0)
    assert int(pl.P[-1]) < 2**61
    # segments partition every row's candidates [u+1, N) in order, sigma = 0..m-1
    su, sa, sb, ss = pl.seg_u, pl.seg_a, pl.seg_b, pl.seg_sigma
    assert np.all(np.diff(su) >= 0)
    assert set(np.unique(su)) == set(range(n - 1))
    first = np.r_[True, su[1:] != su[:-1]]
    last = np.r_[su[1:] != su[:-1], True]
    assert np.all(sa[first] == su[first] + 1)
    assert np.all(sb[last] == n)
    assert np.all(sb[~last] == sa[1:][~last[:-1]])
    assert np.all(sa < sb)
    assert np.all(ss[first] == 0) and np.all(ss[1:][~first[1:]] == ss[:-1][~first[1:]] + 1)
    # initial bounds (R3, R10): q0 = x0/d0 at the virtual position a-1 dominates every candidate
    kq = pl.kappa_s[su] * pl.kappa_s[sa - 1]
    assert np.array_equal(pl.seg_x0, kq)
    if not ecm:
        assert np.array_equal(pl.seg_d0, 1.0 + kq)
        assert np.allclose(pl.seg_h0, np.log1p(kq), rtol=4e-16, atol=0)
        q0 = kq / (1.0 + kq)
        for g in range(0, len(su), 97):
            v = np.arange(sa[g], sb[g])
            X = pl.kappa_s[su[g]] * pl.kappa_s[v]
            assert np.all(X / (1.0 + X) <= q0[g] * (1 + 2.0 ** -50))
    else:
        T = pl.y_s[su] * pl.ymax[sa]
        assert np.array_equal(pl.seg_omT, 1.0 - T)
        assert np.array_equal(pl.seg_iomT, 1.0 / (1.0 - T))
        assert np.array_equal(pl.seg_d0, (1.0 - T) + kq)
        assert np.max(np.abs(pl.ly_s.view(np.int64) - np.log(pl.y_s).view(np.int64))) <= 1  # numpy vs glibc log
        q0 = kq / ((1.0 - T) + kq)
        for g in range(0, len(su), 97):
            v = np.arange(sa[g], sb[g])
            z = pl.kappa_s[su[g]] * pl.kappa_s[v]
            t = pl.y_s[su[g]] * pl.y_s[v]
            assert np.all(z / ((1.0 - t) + z) <= q0[g] * (1 + 2.0 ** -50))


def test_plan_splits_heavy_rows(O):
    w = WL.workload(2)
    x, _ = WL.fitness(w)
    pl = O.sort_plan(x, None, seg_target=256)
    counts = np.bincount(pl.seg_u, minlength=len(x))
    assert counts[0] > 1                   # the top hub row is split
    assert pl.n_segments < 1.2 * len(x)    # ...and only a few percent extra segments
    pl2 = O.sort_plan(x, None, seg_target=1 << 40)
    assert pl2.n_segments == len(x) - 1    # S = huge: one segment per row


def test_plan_validation(O):
    with pytest.raises(O.OracleError):
        O.sort_plan(np.array([1.0]))                      # N < 2
    with pytest.raises(O.OracleError):
        O.sort_plan(np.array([1.0, -1.0]))                # x < 0
    with pytest.raises(O.OracleError):
        O.sort_plan(np.array([1.0, np.nan]))
    with pytest.raises(O.OracleError):
        O.sort_plan(np.array([1.0, np.inf]))
    with pytest.raises(O.OracleError):
        O.sort_plan(np.array([1e200, 1.0]))               # kappa_max^4 overflows (R10 products)
    with pytest.raises(O.OracleError):
        O.sort_plan(np.array([1e80, 1.0]))
    with pytest.raises(O.OracleError):
        O.sort_plan(np.array([1.0, 1.0]), np.array([0.5, 1.0]))   # y >= 1 (beta <= 0)
    with pytest.raises(O.OracleError):
        O.sort_plan(np.array([1.0, 1.0]), seg_target=4)   # S < 8
