"""GPU parity of the bipartite and directed samplers (NEXT-1) against the oracle."""
import numpy as np
import pytest

from paper_2509_13230_b200 import workloads as WL
from _parity import compare

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402


def fitness(seed, n1, n2, c1, c2, ecm, directed):
    x1, y1 = WL.random_fitness(seed, n1, 2.4, c1, ecm=ecm)
    if directed:
        x2 = WL.random_fitness(seed + 1, n2, 2.4, c2)[0]
        y2 = y1 * 0.9 if ecm else None
    else:
        x2, y2 = WL.random_fitness(seed + 1, n2, 2.4, c2, ecm=ecm)
    return x1, y1, x2, y2


@pytest.mark.parametrize("ecm", [False, True])
@pytest.mark.parametrize("kind", ["bipartite", "directed"])
@pytest.mark.parametrize("n1,n2,S,R", [(1, 5, 8, 200), (7, 3, 8, 300), (500, 333, 8, 20), (4097, 2049, 256, 4),
                                       (30_000, 20_000, 64, 3)])
def test_parity(O, kind, ecm, n1, n2, S, R):
    directed = kind == "directed"
    if directed:
        n2 = n1
    c = 0.5 if n1 < 100 else 0.03
    x1, y1, x2, y2 = fitness(3 * n1 + n2, n1, n2, c, c, ecm, directed)
    dev = lambda a: None if a is None else torch.from_numpy(a).cuda()  # noqa: E731
    plan = fm.sort_plan_bipartite(dev(x1), dev(x2), dev(y1), dev(y2), kind=kind, seg_target=S)
    o = O.sort_plan(x1, y1, seg_target=S, kind=kind, x2=x2, y2=y2)
    gx, gc = plan.export(), plan.export_candidates()
    assert plan.n_segments == o.n_segments and plan.n_minus == o.nc
    assert np.array_equal(gx["perm"], o.perm) and np.array_equal(gc["cperm"], o.cperm)
    assert np.array_equal(gx["kappa_s"], o.kappa_s) and np.array_equal(gc["ckappa"], o.ckappa)
    assert np.array_equal(gc["excl"], o.excl)
    seg = gx["seg"]
    assert np.array_equal(seg[:, 0], o.seg_u) and np.array_equal(seg[:, 1], o.seg_a)
    assert np.array_equal(seg[:, 2], o.seg_b) and np.array_equal(seg[:, 3], o.seg_sigma)
    for k in ("seg_x0", "seg_d0", "seg_omT", "seg_iomT"):
        assert np.array_equal(gx[k], getattr(o, k)), k
    fn = fm.sample_ubcm if not ecm else fm.sample_ecm
    e = fn(plan, 1000 + n1, n_samples=R, first_sample=2)
    E = e.edges.cpu().numpy()
    W = None if e.weights is None else e.weights.cpu().numpy()
    ref = O.sample(o, 1000 + n1, n_samples=R, first_sample=2, nthreads=O.ncores())
    if len(E):
        assert E[:, 0].max() < n1 and E[:, 1].max() < n2
    if directed:
        assert not np.any(E[:, 0] == E[:, 1])  # no self loops
    bad, tot = compare(e.offsets, E, W, ref, max(n1, n2))
    assert bad == 0, f"{bad} of {tot}"
    assert (e.draws, e.landed, e.accepted) == (ref.draws, ref.landed, ref.accepted)
    assert np.array_equal(E, ref.edges)  # same canonical order (ordered pairs)
    if W is not None:
        assert np.array_equal(W, ref.weights)


def test_bipartite_status_codes():
    with pytest.raises(fm.FastMaxEntError) as ex:
        fm.sort_plan_bipartite(np.ones(3), np.ones(4), kind="directed")
    assert ex.value.status == fm.FM_ERR_INVALID
    with pytest.raises(fm.FastMaxEntError) as ex:
        fm.sort_plan_bipartite(np.ones(3), np.array([]), kind="bipartite")
    assert ex.value.status == fm.FM_ERR_INVALID
