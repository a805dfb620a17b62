"""Pins of the oracle's sampler chain against the plain definition:
brute force, exact per-pair probabilities, the full joint law, textbook special cases and
closed-form expectations.  Every plausible slip (a dropped term, a wrong sign or index, a
transposed operand, q updated in the wrong place, the Alg. 1 first-candidate bug) moves at
least one pair frequency or one invariant below."""
import math

import numpy as np
import pytest
from scipy import stats

from paper_2509_13230_b200 import workloads as WL
from _stats import chi2_binomial, ecm_p, pair_counts, two_sample_z, ubcm_p, degree_sums

R = 100_000


def _x30(kind):
    if kind == "pareto":
        return WL.random_fitness(5, 30, 2.5, 0.3)[0]                  # p in [0.09, 0.82]
    if kind == "hub":
        x = WL.random_fitness(9, 30, 2.5, 0.15)[0]
        x[:3] = [40.0, 25.0, 9.0]                                       # p up to 0.999
        return x
    raise KeyError(kind)


@pytest.mark.parametrize("S", [8, 16, 1 << 40])
@pytest.mark.parametrize("kind", ["pareto", "hub"])
def test_ubcm_pair_frequencies_n30(O, kind, S):
    x = _x30(kind)
    pl = O.sort_plan(x, seg_target=S)
    res = O.sample(pl, seed=1234 + S, n_samples=R, nthreads=O.ncores())
    c = pair_counts(res.offsets, res.edges, 30)
    stat, dof, pv, zmax = chi2_binomial(c, R, ubcm_p(x))
    assert dof > 300
    assert pv > 1e-4, (stat, dof, zmax)
    assert zmax < 5.5
    # two-sample test against the brute-force (Level 1) sampler with an unrelated RNG
    bf = O.bruteforce(x, seed=77 + S, n_samples=R)
    cb = pair_counts(bf.offsets, bf.edges, 30)
    st2, d2, pv2 = two_sample_z(c, cb, R, R)
    assert pv2 > 1e-4, (st2, d2)


@pytest.mark.parametrize("refresh", [False, True])
@pytest.mark.parametrize("S", [8, 1 << 40])
def test_ecm_pair_and_weight_law_n30(O, S, refresh):
    x, y = WL.random_fitness(6, 30, 2.5, 0.4, ecm=True)
    pl = O.sort_plan(x, y, seg_target=S)
    res = O.sample(pl, seed=99 + S, n_samples=R, nthreads=O.ncores(), refresh=refresh)
    P, T = ecm_p(x, y)
    c = pair_counts(res.offsets, res.edges, 30)
    stat, dof, pv, zmax = chi2_binomial(c, R, P)
    assert pv > 1e-4, (stat, dof, zmax)
    # pooled weight law (Eq. 5): bin edges by t, chi-square of w = 1..10, 11+ vs t^{w-1}(1-t)
    e = res.edges
    t = T[e[:, 0], e[:, 1]]
    w = res.weights
    assert w.min() >= 1
    bins = np.quantile(t, np.linspace(0, 1, 6))
    for lo, hi in zip(bins[:-1], bins[1:]):
        m = (t >= lo) & (t <= hi)
        tt = t[m]
        ww = np.minimum(w[m], 11)
        obs = np.bincount(ww, minlength=12)[1:]
        exp = np.zeros(11)
        for k in range(1, 11):
            exp[k - 1] = np.sum(tt ** (k - 1) * (1 - tt))
        exp[10] = np.sum(tt ** 10)
        keep = exp >= 5
        st = np.sum((obs[keep] - exp[keep]) ** 2 / exp[keep])
        assert stats.chi2.sf(st, keep.sum() - 1) > 1e-4, (lo, hi, obs, exp)
    bf = O.bruteforce(x, y, seed=5 + S, n_samples=R)
    cb = pair_counts(bf.offsets, bf.edges, 30)
    st2, d2, pv2 = two_sample_z(c, cb, R, R)
    assert pv2 > 1e-4
    # mean weight per edge matches brute force (Eq. 3 factorisation)
    assert abs(res.weights.mean() - bf.weights.mean()) < 6 * res.weights.std() / math.sqrt(len(res.weights)) * 1.5


@pytest.mark.parametrize("ecm,refresh", [(False, False), (True, False), (True, True)])
def test_full_joint_n4(O, ecm, refresh):
    """All 2^6 edge configurations of N=4 vs the product law (independence, incl. across segments)."""
    x = np.array([3.0, 1.2, 0.5, 0.2])
    y = np.array([0.7, 0.3, 0.8, 0.5]) if ecm else None
    pl = O.sort_plan(x, y, seg_target=8)
    RR = 400_000
    res = O.sample(pl, seed=4242, n_samples=RR, nthreads=O.ncores(), refresh=refresh)
    pairs = [(i, j) for i in range(4) for j in range(i + 1, 4)]
    bit = {pr: 1 << k for k, pr in enumerate(pairs)}
    codes = np.zeros(RR, np.int64)
    sid = np.repeat(np.arange(RR), np.diff(res.offsets))
    b = np.array([bit[(int(a), int(c))] for a, c in res.edges]) if len(res.edges) else np.zeros(0, np.int64)
    np.add.at(codes, sid, b)
    obs = np.bincount(codes, minlength=64)
    P = ubcm_p(x) if not ecm else ecm_p(x, y)[0]
    exp = np.ones(64)
    for code in range(64):
        for pr, bb in bit.items():
            exp[code] *= P[pr] if code & bb else 1 - P[pr]
    exp *= RR
    st = np.sum((obs - exp) ** 2 / exp)
    assert stats.chi2.sf(st, 63) > 1e-4, st


def test_erdos_renyi_special_case(O):
    """All x equal: p = q bitwise, so every landed candidate is accepted (proposals == edges),
    draws = edges + segments, and the edge count is Binomial(N(N-1)/2, p)."""
    n, RR = 200, 2000
    x = np.full(n, 0.05)
    pl = O.sort_plan(x, seg_target=8)
    res = O.sample(pl, seed=3, n_samples=RR, nthreads=O.ncores())
    assert res.landed == res.accepted
    assert res.draws == res.accepted + RR * pl.n_segments
    p = 0.05 * 0.05 / (1 + 0.05 * 0.05)
    m = n * (n - 1) // 2
    cnt = np.diff(res.offsets)
    assert abs(cnt.mean() - m * p) < 5 * math.sqrt(m * p * (1 - p) / RR)
    assert stats.chi2.sf(cnt.var(ddof=1) * (RR - 1) / (m * p * (1 - p)), RR - 1) > 1e-5


def test_homogeneous_ecm_acceptance_one(O):
    """Identical (x, y): T = t exactly, acceptance 1 (P:L265 'most efficient when beta homogeneous');
    weights ~ Geometric with mean 1/(1-t)."""
    n, RR = 300, 300
    x, y = np.full(n, 0.2), np.full(n, 0.6)
    pl = O.sort_plan(x, y, seg_target=8)
    res = O.sample(pl, seed=8, n_samples=RR, nthreads=O.ncores())
    assert res.landed == res.accepted
    t = 0.36
    w = res.weights.astype(np.float64)
    mean, sd = 1 / (1 - t), math.sqrt(t) / (1 - t)
    assert abs(w.mean() - mean) < 5 * sd / math.sqrt(len(w))


def test_complete_and_empty_graphs(O):
    n = 50
    pl = O.sort_plan(np.full(n, 1e10), seg_target=1 << 40)
    res = O.sample(pl, seed=1, n_samples=3)
    assert np.all(np.diff(res.offsets) == n * (n - 1) // 2)
    assert res.draws == 3 * (n * (n - 1) // 2 + (n - 1))          # every skip is 0, + 1 terminal per row
    e = np.sort(res.edges[: n * (n - 1) // 2].view(np.int64).ravel())
    iu = np.triu_indices(n, 1)
    want = np.sort(np.stack(iu, 1).astype(np.int32).view(np.int64).ravel())
    assert np.array_equal(e, want)
    pl0 = O.sort_plan(np.zeros(n))
    r0 = O.sample(pl0, seed=1, n_samples=5)
    assert len(r0.edges) == 0 and r0.draws == 5 * pl0.n_segments and r0.landed == 0
    # s = k limit: y -> 0 forces unit weights
    x = WL.random_fitness(2, 60, 2.5, 2.0)[0]
    y = np.full(60, 1e-12)
    r1 = O.sample(O.sort_plan(x / 1e-12, y), seed=2, n_samples=20)
    assert len(r1.weights) > 0 and np.all(r1.weights == 1)


def test_first_candidate_is_reached_by_a_skip(O):
    """Algorithm 1's literal j <- i+1 would include pair (i, i+1) with p/q (reading R3 fixes it):
    with a dominant first node the pair (0, 1) must still have frequency p, not 1."""
    x = np.array([50.0, 0.01, 0.01, 0.01, 0.01])
    pl = O.sort_plan(x)
    RR = 200_000
    res = O.sample(pl, seed=6, n_samples=RR)
    c = pair_counts(res.offsets, res.edges, 5)
    p = 0.5 / 1.5
    assert abs(c[0, 1] / RR - p) < 5 * math.sqrt(p * (1 - p) / RR)


@pytest.mark.parametrize("ecm", [False, True])
def test_closed_form_degrees_and_strengths(O, ecm):
    """Per-node mean degree (and strength) over R samples within 5 sigma of sum_j p_ij (BJ north_star)."""
    x, y = WL.random_fitness(21, 400, 2.5, 0.05 if not ecm else 0.12, ecm=ecm)
    RR = 3000
    pl = O.sort_plan(x, y, seg_target=16)
    res = O.sample(pl, seed=31, n_samples=RR, nthreads=O.ncores())
    k, kv, s, sv = O.expected(x, y)
    k1, k2, s1, s2 = degree_sums(res.offsets, res.edges, len(x), res.weights)
    z = (k1 / RR - k) / np.sqrt(np.maximum(kv, 1e-300) / RR)
    assert np.max(np.abs(z[kv > 0.5])) < 5.0
    # variance of the total edge count vs sum p(1-p)
    cnt = np.diff(res.offsets).astype(np.float64)
    var_exp = kv.sum() / 2
    assert abs(cnt.var(ddof=1) / var_exp - 1) < 5 * math.sqrt(2 / (RR - 1))
    if ecm:
        zs = (s1 / RR - s) / np.sqrt(sv / RR)
        assert np.max(np.abs(zs[sv > 0.5])) < 5.0


def test_determinism_batching_threads_rows(O):
    x, y = WL.random_fitness(4, 5000, 2.3, 0.01, ecm=True)
    for yy in (None, y):
        pl = O.sort_plan(x, yy, seg_target=64)
        a = O.sample(pl, seed=11, n_samples=4, first_sample=10, nthreads=1)
        b = O.sample(pl, seed=11, n_samples=4, first_sample=10, nthreads=7)
        assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.edges, b.edges)
        assert a.draws == b.draws and a.landed == b.landed
        for s in range(4):  # batch == singles (sample index keys the stream)
            c = O.sample(pl, seed=11, n_samples=1, first_sample=10 + s)
            assert np.array_equal(c.edges, a.sample(s)[0])
            if yy is not None:
                assert np.array_equal(c.weights, a.sample(s)[1])
        d = O.sample(pl, seed=12, n_samples=1, first_sample=10)
        assert not np.array_equal(d.edges, a.sample(0)[0])
        # rows subset == filter of the full sample
        rows = np.array([0, 1, 7, 100, 4998, 4999], np.int32)
        r = O.sample(pl, seed=11, n_samples=1, first_sample=10, rows=rows)
        rank = np.empty(len(x), np.int64)
        rank[pl.perm] = np.arange(len(x))
        e = a.sample(0)[0]
        row_of = np.minimum(rank[e[:, 0]], rank[e[:, 1]])
        sel = np.isin(row_of, rows)
        assert np.array_equal(r.edges, e[sel])


def test_permutation_equivariance(O):
    """Relabelling the nodes (no ties) relabels the output: keys use sorted rank, not id."""
    x = WL.random_fitness(8, 2000, 2.5, 0.03)[0]
    perm = np.random.default_rng(0).permutation(2000)
    a = O.sample(O.sort_plan(x), seed=5, n_samples=2)
    b = O.sample(O.sort_plan(x[perm]), seed=5, n_samples=2)
    inv = perm  # new id i holds old node perm[i]
    mapped = np.sort(inv[b.edges], axis=1)
    key = lambda e: np.sort(e[:, 0].astype(np.int64) * 2000 + e[:, 1])
    assert np.array_equal(key(a.edges), key(mapped))


def test_beta_refresh_invariants(O):
    """Per-candidate beta_min refresh (R17): with homogeneous y the bound never changes, so the
    samples are identical to the per-segment bound; with heterogeneous y it is tighter: fewer
    proposals per edge (1.67 -> 1.54 on config 3) and the same expected edge count."""
    n, RR = 400, 50
    x = WL.random_fitness(12, n, 2.5, 0.05)[0]
    pl = O.sort_plan(x, np.full(n, 0.4), seg_target=16)
    a = O.sample(pl, seed=3, n_samples=RR)
    b = O.sample(pl, seed=3, n_samples=RR, refresh=True)
    assert np.array_equal(a.offsets, b.offsets) and np.array_equal(a.edges, b.edges)
    assert np.array_equal(a.weights, b.weights) and a.draws == b.draws
    x, y = WL.random_fitness(12, 3000, 2.5, 0.02, ecm=True)
    pl = O.sort_plan(x, y, seg_target=256)
    a = O.sample(pl, seed=3, n_samples=40, nthreads=O.ncores())
    b = O.sample(pl, seed=3, n_samples=40, nthreads=O.ncores(), refresh=True)
    assert b.landed / b.accepted < 0.97 * a.landed / a.accepted
    ee = O.expected_edges(x, y) * 40
    for r in (a, b):
        assert abs(r.accepted - ee) < 5 * math.sqrt(ee)
