"""Statistics helpers shared by oracle and GPU tests (no method arithmetic)."""
import numpy as np
from scipy import stats


def pair_counts(offsets, edges, n):
    """counts[i, j] (i < j) over all samples of an edge list."""
    idx = edges[:, 0].astype(np.int64) * n + edges[:, 1].astype(np.int64)
    c = np.bincount(idx, minlength=n * n).reshape(n, n)
    return c


def chi2_binomial(counts, R, p, min_var=5.0):
    """One-sample chi-square of per-pair counts vs Binomial(R, p) over pairs with R p (1-p) >= min_var.
    Returns (stat, dof, pvalue, max|z|)."""
    iu = np.triu_indices(p.shape[0], 1)
    c, pp = counts[iu].astype(np.float64), p[iu]
    var = R * pp * (1 - pp)
    m = var >= min_var
    z = (c[m] - R * pp[m]) / np.sqrt(var[m])
    stat = float(np.sum(z * z))
    dof = int(m.sum())
    return stat, dof, float(stats.chi2.sf(stat, dof)), float(np.max(np.abs(z))) if dof else 0.0


def two_sample_z(c1, c2, R1, R2, min_count=20):
    """Pooled two-proportion z over pairs; returns (chi2 stat, dof, pvalue)."""
    iu = np.triu_indices(c1.shape[0], 1)
    a, b = c1[iu].astype(np.float64), c2[iu].astype(np.float64)
    pp = (a + b) / (R1 + R2)
    m = ((a + b) >= min_count) & (pp < 1) & (pp > 0)
    z = (a[m] / R1 - b[m] / R2) / np.sqrt(pp[m] * (1 - pp[m]) * (1 / R1 + 1 / R2))
    stat = float(np.sum(z * z))
    return stat, int(m.sum()), float(stats.chi2.sf(stat, int(m.sum())))


def ubcm_p(x):
    X = np.outer(x, x)
    P = X / (1.0 + X)
    np.fill_diagonal(P, 0.0)
    return P


def ecm_p(x, y):
    t = np.outer(y, y)
    z = np.outer(x, x) * t
    P = z / (1.0 - t + z)
    np.fill_diagonal(P, 0.0)
    return P, t


def degrees(offsets, edges, n, weights=None):
    """per-sample degree (and strength) matrices [R, n]."""
    R = len(offsets) - 1
    k = np.zeros((R, n), np.int64)
    s = np.zeros((R, n), np.int64) if weights is not None else None
    for r in range(R):
        e = edges[offsets[r]:offsets[r + 1]]
        k[r] = np.bincount(e[:, 0], minlength=n) + np.bincount(e[:, 1], minlength=n)
        if weights is not None:
            w = weights[offsets[r]:offsets[r + 1]].astype(np.int64)
            s[r] = np.bincount(e[:, 0], weights=w, minlength=n) + np.bincount(e[:, 1], weights=w, minlength=n)
    return k, s


def degree_sums(offsets, edges, n, weights=None):
    """sum over samples of degree and degree^2 (and strength, strength^2), memory-light."""
    R = len(offsets) - 1
    k1 = np.zeros(n); k2 = np.zeros(n); s1 = np.zeros(n); s2 = np.zeros(n)
    for r in range(R):
        e = edges[offsets[r]:offsets[r + 1]]
        k = np.bincount(e[:, 0], minlength=n) + np.bincount(e[:, 1], minlength=n)
        k1 += k; k2 += k.astype(np.float64) ** 2
        if weights is not None:
            w = weights[offsets[r]:offsets[r + 1]].astype(np.float64)
            s = np.bincount(e[:, 0], weights=w, minlength=n) + np.bincount(e[:, 1], weights=w, minlength=n)
            s1 += s; s2 += s * s
    return k1, k2, s1, s2


def node_gate(D, k, kv, R, alpha=1e-3, sigma=5.0):
    """Per-node statistical gate on ensemble sums.

    D: per-node sum over R samples of the degree (or strength); the exact law has mean R k and
    variance R kv (independent pairs).  Nodes with R kv >= 25: z = (D - R k)/sqrt(R kv)
    must satisfy |z| < zc with zc = sigma for m <= 1000 tested nodes (the north star's 5 sigma;
    family-wise error ~6e-4) and the Bonferroni zc = Phi^-1(1 - alpha/(2m)) beyond (6.1 at m = 1e6).
    Nodes with 0 < R kv < 25 (non-normal): two-sided tail of Poisson(R k) -- heavier-tailed than
    the Poisson-binomial of the same mean -- must exceed alpha/(2m).  kv == 0: D == R k exactly.
    Aggregate: sum of z^2 over the normal nodes within 6 sqrt(2 m') of its mean m'.
    Returns a dict of diagnostics; raises AssertionError on failure."""
    D = np.asarray(D, np.float64)
    k = np.asarray(k, np.float64)
    kv = np.asarray(kv, np.float64)
    m = len(D)
    zc = sigma if m <= 1000 else max(sigma, float(stats.norm.isf(alpha / (2 * m))))
    big = R * kv >= 25
    z = (D[big] - R * k[big]) / np.sqrt(R * kv[big])
    zmax = float(np.max(np.abs(z))) if z.size else 0.0
    assert zmax < zc, f"max |z| = {zmax:.2f} >= {zc:.2f} over {int(big.sum())} nodes"
    small = (~big) & (kv > 0)
    if small.any():
        lam = R * k[small]
        lo = stats.poisson.cdf(D[small], lam)
        hi = stats.poisson.sf(D[small] - 1, lam)
        pmin = float(np.min(np.minimum(lo, hi)))
        assert pmin > alpha / (2 * m), f"low-variance node tail p = {pmin:.3g}"
    zero = kv == 0
    if zero.any():
        assert np.allclose(D[zero], R * k[zero], rtol=0, atol=1e-6), "deterministic nodes"
    mm = int(big.sum())
    agg = float(np.sum(z * z))
    if mm:
        assert abs(agg - mm) < 6 * np.sqrt(2 * mm), f"sum z^2 = {agg:.1f} for {mm} nodes"
    return {"nodes": m, "normal": mm, "zmax": zmax, "zc": zc, "sum_z2": agg}
