"""Pins of the oracle's rich-club functions (the top-alpha edge density of
P:L58-60): the count against a brute-force double loop, the expectation against closed
forms (homogeneous G(N,p); the total against the pinned expected_edges), and the oracle's own
samples against the expectation."""
import itertools

import numpy as np


def test_count_is_the_definition(O):
    rng = np.random.default_rng(3)
    n = 40
    order = rng.permutation(n).astype(np.int32)
    pairs = [(i, j) for i, j in itertools.combinations(range(n), 2) if rng.random() < 0.3]
    edges = np.array(pairs, dtype=np.int32)
    got = O.richclub_count(order, edges)
    top = lambda m: set(order[:m].tolist())  # noqa: E731
    want = [sum(1 for i, j in pairs if i in top(m) and j in top(m)) for m in range(n + 1)]
    assert got.tolist() == want
    assert got[-1] == len(pairs) and got[0] == 0 and got[1] == 0


def test_expectation_closed_forms(O):
    # homogeneous x: p = x^2/(1+x^2) for every pair -> E = p m(m-1)/2, Var = p(1-p) m(m-1)/2
    n, xv = 50, 0.7
    x = np.full(n, xv)
    order = np.arange(n, dtype=np.int32)
    mean, var = O.expected_richclub(x, None, order)
    p = xv * xv / (1 + xv * xv)
    m = np.arange(n + 1)
    np.testing.assert_allclose(mean, p * m * (m - 1) / 2, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(var, p * (1 - p) * m * (m - 1) / 2, rtol=1e-13, atol=1e-13)
    # heterogeneous, both models: the whole set is the expected edge count (pinned elsewhere)
    rng = np.random.default_rng(5)
    x = rng.uniform(0.05, 3.0, 300)
    y = rng.uniform(0.05, 0.85, 300)
    order = np.argsort(-x, kind="stable").astype(np.int32)
    for yy in (None, y):
        mean, _ = O.expected_richclub(x, yy, order)
        assert mean[-1] == np.float64(mean[-1])
        assert abs(mean[-1] - O.expected_edges(x, yy)) < 1e-9 * mean[-1]
        assert np.all(np.diff(mean) >= 0)


def test_oracle_samples_match_expectation(O):
    """The oracle's exact sampler (Alg. 1 chains) averaged over 4000 samples: e_top[m] within 5 sigma."""
    rng = np.random.default_rng(11)
    n, R = 60, 4000
    x = rng.pareto(1.5, n) * 0.1 + 0.02
    plan = O.sort_plan(x, seg_target=8)
    order = plan.perm
    res = O.sample(plan, seed=9, n_samples=R)
    acc = np.zeros(n + 1, dtype=np.int64)
    for s in range(R):
        e, _ = res.sample(s)
        acc += O.richclub_count(order, e)
    mean, var = O.expected_richclub(x, None, order)
    ms = [2, 5, 10, 20, 40, 60]
    z = [(acc[m] / R - mean[m]) / np.sqrt(var[m] / R) for m in ms]
    assert max(abs(v) for v in z) < 5, z
