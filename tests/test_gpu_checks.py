"""FM_DEBUG_CHECKS ("must abort, never silently clamp"): with the
check on, every landed candidate tests the contract p <= q (1 + 2^-50) (R13).  A plan
whose initial bounds are too small (the FM_DEBUG_BAD_BOUND test hook scales every segment's x0 by
1e-3) makes the call fail with FM_ERR_BOUND and leaves nothing allocated; valid plans never trip
the check (no false positives), UBCM and ECM, with and without the beta_min refresh."""
import os

import numpy as np
import pytest

from paper_2509_13230_b200 import workloads as WL

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)
from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402

FM_ERR_BOUND = -4


@pytest.fixture
def env():
    saved = {k: os.environ.get(k) for k in ("FM_DEBUG_CHECKS", "FM_DEBUG_BAD_BOUND")}
    yield os.environ
    for k, v in saved.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = v


def _case(ecm):
    x, y = WL.random_fitness(21, 20_000, 2.3, 0.02, ecm=ecm)
    return torch.from_numpy(x).cuda(), None if y is None else torch.from_numpy(y).cuda()


@pytest.mark.parametrize("ecm,refresh", [(False, False), (True, False), (True, True)])
def test_valid_plans_pass_the_check(env, ecm, refresh):
    env["FM_DEBUG_CHECKS"] = "1"
    x, y = _case(ecm)
    plan = fm.sort_plan(x, y, seg_target=32)
    e = fm.sample_ecm(plan, 3, n_samples=4, refresh=refresh) if ecm else fm.sample_ubcm(plan, 3, n_samples=4)
    assert e.n_edges > 0
    env.pop("FM_DEBUG_CHECKS")
    e2 = fm.sample_ecm(plan, 3, n_samples=4, refresh=refresh) if ecm else fm.sample_ubcm(plan, 3, n_samples=4)
    assert torch.equal(e.edges, e2.edges)  # the check changes nothing


@pytest.mark.parametrize("ecm", [False, True])
def test_bad_bound_fails_with_fm_err_bound(env, ecm):
    x, y = _case(ecm)
    env["FM_DEBUG_BAD_BOUND"] = "1"
    plan = fm.sort_plan(x, y, seg_target=32)
    env.pop("FM_DEBUG_BAD_BOUND")
    sample = (lambda **k: fm.sample_ecm(plan, 3, **k)) if ecm else (lambda **k: fm.sample_ubcm(plan, 3, **k))
    # without the check the bad plan is sampled silently (that is why the check exists)
    sample(n_samples=1).free()
    env["FM_DEBUG_CHECKS"] = "1"
    with pytest.raises(fm.FastMaxEntError) as ei:
        sample(n_samples=2)
    assert ei.value.status == FM_ERR_BOUND
    assert "p > q" in str(ei.value)
    # the statistics mode reports it too
    with pytest.raises(fm.FastMaxEntError) as ei2:
        fm.sample_degrees(plan, 3, n_samples=1)
    assert ei2.value.status == FM_ERR_BOUND
