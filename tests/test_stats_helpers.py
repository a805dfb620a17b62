"""The statistical gate of the GPU tests (tests/_stats.py: node_gate) on synthetic data with a
known law: sums of independent Bernoulli variables pass, a one-sigma-per-node bias over many
nodes or a single 8-sigma node fails (CPU only)."""
import numpy as np
import pytest

from _stats import node_gate


def _sums(rng, p, R):
    # D_i = sum over R samples and over the node's pairs of Bernoulli(p_ij): Binomial(R, p_ij) per pair
    return rng.binomial(R, p).sum(axis=1).astype(np.float64)


def test_node_gate_accepts_the_exact_law_and_rejects_bias():
    rng = np.random.default_rng(0)
    m, pairs, R = 3000, 200, 64
    p = rng.uniform(0.0, 0.6, size=(m, pairs))
    p[:50] = rng.uniform(0, 0.002, size=(50, pairs))  # low-variance nodes (Poisson tail branch)
    k, kv = p.sum(axis=1), (p * (1 - p)).sum(axis=1)
    D = _sums(rng, p, R)
    info = node_gate(D, k, kv, R)
    assert info["normal"] > 2900
    with pytest.raises(AssertionError):
        node_gate(D + np.sqrt(R * kv), k, kv, R)   # every node one sigma high: the aggregate fails
    D2 = D.copy()
    D2[100] += 8 * np.sqrt(R * kv[100])
    with pytest.raises(AssertionError):
        node_gate(D2, k, kv, R)                    # one node far out: the per-node bound fails
