"""ECM per-candidate beta_min refresh (R17) on the GPU against the
oracle's refresh mode: exact canonical-order equality on small cases (undirected, bipartite,
directed), <= 1e-6 edge mismatch on full config 3, fewer proposals per edge than the per-segment
bound, and flag validation."""
import numpy as np
import pytest

from paper_2509_13230_b200 import workloads as WL
from _parity import compare, hygiene

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402

dev = lambda a: None if a is None else torch.from_numpy(a).cuda()  # noqa: E731


def _check(O, gplan, oplan, n, seed, R, first=0, exact=True, ordered=False):
    e = fm.sample_ecm(gplan, seed, n_samples=R, first_sample=first, refresh=True)
    E, W = e.edges.cpu().numpy(), e.weights.cpu().numpy()
    ref = O.sample(oplan, seed, n_samples=R, first_sample=first, nthreads=O.ncores(), refresh=True)
    if not ordered:
        hygiene(E, n, W)
    bad, tot = compare(e.offsets, E, W, ref, max(n, int(E.max(initial=0)) + 1))
    assert bad <= (0 if exact else int(1e-6 * tot)), (bad, tot)
    if bad == 0:
        assert (e.draws, e.landed, e.accepted) == (ref.draws, ref.landed, ref.accepted)
        assert np.array_equal(E, ref.edges) and np.array_equal(W, ref.weights)
    return e, ref


@pytest.mark.parametrize("n,S,R", [(2, 256, 50), (31, 8, 100), (1000, 8, 20), (4097, 256, 5), (20_011, 64, 3)])
def test_refresh_small_parity(O, n, S, R):
    x, y = WL.random_fitness(7 * n + 3, n, 2.5, 0.3 if n < 100 else 0.03, ecm=True)
    _check(O, fm.sort_plan(dev(x), dev(y), seg_target=S), O.sort_plan(x, y, seg_target=S), n, 500 + n, R, first=2)


@pytest.mark.parametrize("kind", ["bipartite", "directed"])
def test_refresh_bipartite_directed_parity(O, kind):
    n1 = 3000
    n2 = 2200 if kind == "bipartite" else n1
    x1, y1 = WL.random_fitness(41, n1, 2.4, 0.03, ecm=True)
    x2, y2 = WL.random_fitness(42, n2, 2.4, 0.03, ecm=True)
    g = fm.sort_plan_bipartite(dev(x1), dev(x2), dev(y1), dev(y2), kind=kind, seg_target=64)
    o = O.sort_plan(x1, y1, seg_target=64, kind=kind, x2=x2, y2=y2)
    _check(O, g, o, max(n1, n2), 77, 4, ordered=True)


def test_refresh_config3_full_and_fewer_proposals(O):
    w = WL.workload(3)
    x, y = WL.fitness(w)
    g = fm.sort_plan(dev(x), dev(y), seg_target=256)
    e, ref = _check(O, g, O.sort_plan(x, y, seg_target=256), w.n, w.seed, 4, exact=False)
    base = fm.sample_ecm(g, w.seed, n_samples=4)
    assert e.landed / e.accepted < 0.96 * base.landed / base.accepted  # 1.67 -> 1.54 draws/edge
    assert abs(e.accepted - base.accepted) < 5 * np.sqrt(base.accepted)


def test_refresh_flag_validation():
    x, y = WL.random_fitness(1, 100, 2.5, 0.1, ecm=True)
    g = fm.sort_plan(dev(x), dev(y))
    st = fm._Edges()
    rc = fm.lib.fm_sample_ecm_ex(g._h, 1, 0, 1, 0x80, None, fm.C.byref(st))
    assert rc == fm.FM_ERR_INVALID
