"""fm_sample_richclub (the top-alpha density profile of P:L58-60): e_top[m]
summed over an ensemble without edge lists -- equal to the oracle's definition applied to the edge
lists of the same samples (GPU's own and the oracle's), and within 5 sigma of the closed form."""
import numpy as np
import pytest

from paper_2509_13230_b200 import workloads as WL

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402


@pytest.mark.parametrize("ecm", [False, True])
def test_richclub_equals_edge_list_counts(O, ecm):
    n, R = 3001, 12
    x, y = WL.random_fitness(17, n, 2.4, 0.02, ecm=ecm)
    dev = lambda a: None if a is None else torch.from_numpy(a).cuda()  # noqa: E731
    plan = fm.sort_plan(dev(x), dev(y), seg_target=32)
    order = plan.export()["perm"]
    e_top, cnt = fm.sample_richclub(plan, seed=77, n_samples=R, first_sample=5)
    edges = (fm.sample_ecm if ecm else fm.sample_ubcm)(plan, seed=77, n_samples=R, first_sample=5)
    want = np.zeros(n + 1, dtype=np.int64)
    for s in range(R):
        e, _ = edges.sample(s)
        want += O.richclub_count(order, e.cpu().numpy())
    assert np.array_equal(e_top.cpu().numpy(), want)
    assert cnt["accepted"] == edges.n_edges == want[-1]
    # the oracle's own samples (same plan contract, same seed): the same profile
    oplan = O.sort_plan(x, y, seg_target=32)
    assert np.array_equal(oplan.perm, order)
    res = O.sample(oplan, seed=77, n_samples=R, first_sample=5)
    ow = np.zeros(n + 1, dtype=np.int64)
    for s in range(R):
        e, _ = res.sample(s)
        ow += O.richclub_count(order, e)
    assert np.abs(ow - want).max() <= max(2, 1e-6 * want[-1]), np.abs(ow - want).max()


def test_richclub_accumulates_and_matches_expectation(O):
    n, R = 400, 20000
    x, _ = WL.random_fitness(23, n, 2.2, 0.03)
    plan = fm.sort_plan(torch.from_numpy(x).cuda(), seg_target=16)
    order = plan.export()["perm"]
    a, _ = fm.sample_richclub(plan, seed=3, n_samples=R // 2)
    b, _ = fm.sample_richclub(plan, seed=3, n_samples=R - R // 2, first_sample=R // 2)
    whole, _ = fm.sample_richclub(plan, seed=3, n_samples=R)
    assert torch.equal(a + b, whole)  # batches are exact slices of the ensemble
    mean, var = O.expected_richclub(x, None, order)
    got = whole.cpu().numpy() / R
    ms = np.array([2, 4, 8, 16, 32, 64, 128, 256, 400])
    z = (got[ms] - mean[ms]) / np.sqrt(var[ms] / R)
    assert np.abs(z).max() < 5, z


def test_richclub_rejects_bipartite():
    x = np.linspace(0.1, 1.0, 50)
    plan = fm.sort_plan_bipartite(torch.from_numpy(x).cuda(), torch.from_numpy(x[:40]).cuda())
    with pytest.raises(Exception):
        fm.sample_richclub(plan, seed=1, n_samples=2)
