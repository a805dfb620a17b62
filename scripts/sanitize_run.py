"""Small invocations of every product entry point, for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck): config 1 (UBCM, N = 1000), a small ECM case with forced segmentation and
the beta_min refresh, bipartite and directed ECM plans, the statistics modes, and a forced
scratch-overflow re-run.  Exits non-zero if a result differs from the oracle.

    compute-sanitizer --tool memcheck python scripts/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402
from paper_2509_13230_b200 import workloads as WL  # noqa: E402


def keys(e, n, w=None):
    k = e[:, 0].astype(np.int64) * n + e[:, 1]
    if w is not None:
        k = k * (1 << 31) + w
    return np.sort(k)


def main():
    O.build()
    torch.cuda.set_device(0)
    w = WL.workload(1)
    x, _ = WL.fitness(w)
    plan = fm.sort_plan(torch.from_numpy(x).cuda())
    e = fm.sample_ubcm(plan, w.seed, n_samples=2)
    ref = O.sample(O.sort_plan(x), w.seed, n_samples=2)
    for s in range(2):
        assert np.array_equal(keys(e.sample(s)[0].cpu().numpy(), w.n), keys(ref.sample(s)[0], w.n)), "cfg1"
    d = fm.sample_degrees(plan, w.seed, n_samples=2)
    rc = fm.sample_richclub(plan, w.seed, n_samples=2)
    e.free()

    x2, y2 = WL.random_fitness(7, 3000, 2.5, 0.02, ecm=True)
    p2 = fm.sort_plan(torch.from_numpy(x2).cuda(), torch.from_numpy(y2).cuda(), seg_target=16)
    for refresh in (False, True):
        e2 = fm.sample_ecm(p2, 5, n_samples=2, refresh=refresh)
        r2 = O.sample(O.sort_plan(x2, y2, seg_target=16), 5, n_samples=2, refresh=refresh)
        for s in range(2):
            g, gw = e2.sample(s)
            o, ow = r2.sample(s)
            assert np.array_equal(keys(g.cpu().numpy(), 3000, gw.cpu().numpy()), keys(o, 3000, ow)), "ecm"
        e2.free()

    xa, ya = WL.random_fitness(11, 1500, 2.3, 0.03, ecm=True)
    xb, yb = WL.random_fitness(12, 1200, 2.3, 0.03, ecm=True)
    for kind in ("bipartite", "directed"):
        xb_, yb_ = (xb, yb) if kind == "bipartite" else WL.random_fitness(13, 1500, 2.3, 0.03, ecm=True)
        p3 = fm.sort_plan_bipartite(torch.from_numpy(xa).cuda(), torch.from_numpy(xb_).cuda(),
                                    torch.from_numpy(ya).cuda(), torch.from_numpy(yb_).cuda(), kind=kind, seg_target=32)
        e3 = fm.sample_ecm(p3, 3, n_samples=1)
        r3 = O.sample(O.sort_plan(xa, ya, seg_target=32, kind=O.BIPARTITE if kind == "bipartite" else O.DIRECTED,
                                  x2=xb_, y2=yb_), 3, n_samples=1)
        nb = len(xb_)
        assert np.array_equal(keys(e3.edges.cpu().numpy(), nb, e3.weights.cpu().numpy()),
                              keys(r3.edges, nb, r3.weights)), kind
        fm.sample_degrees(p3, 3, n_samples=1)
        e3.free()
        p3.free()
    # round 2: pipelined sample groups (two streams, TMA-staged compaction) and the big lane-chunks
    xg, yg = WL.random_fitness(21, 6000, 2.4, 0.03, ecm=True)
    for yy in (None, yg):
        og = O.sample(O.sort_plan(xg, yy, seg_target=32), 8, n_samples=5)
        for env in ({"FM_SAMPLE_GROUPS": "2", "FM_COMPACT_SMALL": "2"},
                    {"FM_CHUNK_BIG_DRAWS": "300", "FM_TAIL_FACTOR_BIG": "0", "FM_TAIL_FACTOR": "0"}):
            os.environ.update(env)
            pg = fm.sort_plan(torch.from_numpy(xg).cuda(), None if yy is None else torch.from_numpy(yy).cuda(),
                              seg_target=32)
            eg = (fm.sample_ubcm if yy is None else fm.sample_ecm)(pg, 8, n_samples=5)
            for k in env:
                del os.environ[k]
            assert np.array_equal(eg.edges.cpu().numpy(), og.edges), "groups/chunks"
            if yy is not None:
                assert np.array_equal(eg.weights.cpu().numpy(), og.weights), "groups/chunks weights"
            eg.free()
            pg.free()
    torch.cuda.synchronize()
    print("sanitize_run ok", d[-1], int(rc[0][-1]))


if __name__ == "__main__":
    main()
