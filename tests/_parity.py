"""GPU-vs-oracle comparison helpers (sets per sample; GPU order is deterministic but not canonical, R14)."""
import numpy as np


def edge_keys(edges, n, weights=None):
    e = np.asarray(edges).astype(np.int64)
    k = e[:, 0] * n + e[:, 1]
    if weights is not None:
        k = k * (1 << 31) + np.asarray(weights).astype(np.int64)
    return np.sort(k)


def symdiff(a_keys, b_keys):
    return len(np.setxor1d(a_keys, b_keys, assume_unique=False))


def compare(gpu_off, gpu_edges, gpu_w, ref, n):
    """(mismatched elements of the symmetric difference, total oracle edges) over all samples."""
    bad = 0
    for s in range(len(gpu_off) - 1):
        g = gpu_edges[gpu_off[s]:gpu_off[s + 1]]
        gw = None if gpu_w is None else gpu_w[gpu_off[s]:gpu_off[s + 1]]
        o, ow = ref.sample(s)
        bad += symdiff(edge_keys(g, n, gw), edge_keys(o, n, ow))
    return bad, int(ref.offsets[-1])


def hygiene(edges, n, weights=None):
    e = np.asarray(edges)
    assert np.all(e[:, 0] < e[:, 1]), "src < dst, no self loops"
    assert e.min(initial=0) >= 0 and e.max(initial=0) < n
    if weights is not None:
        assert np.asarray(weights).min(initial=1) >= 1
