"""World-size-2 gloo test of the sample sharding, on CPU with the oracle:
the shards are disjoint, cover the ensemble, and their union equals a single-process run
(batch == concatenation of shards, because the sample index keys the RNG stream)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2509_13230_b200 import dist as D
from paper_2509_13230_b200 import workloads as WL


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle import oracle as O
    x, y = WL.random_fitness(3, 3000, 2.4, 0.02, ecm=True)
    plan = O.sort_plan(x, y, seg_target=32)
    first, n = D.shard_samples(rank, world, 3)
    res = O.sample(plan, seed=9, n_samples=n, first_sample=first)
    elapsed = D.reduce_max(0.5 + rank)
    tot = D.reduce_sum([res.accepted, res.draws])
    gathered = [None] * world
    dist.all_gather_object(gathered, (first, res.offsets.tolist(), res.edges.tolist(), res.weights.tolist()))
    if rank == 0:
        np.save(os.path.join(out_dir, "ok.npy"), np.array([elapsed, tot[0], tot[1]]))
        import pickle
        pickle.dump(gathered, open(os.path.join(out_dir, "g.pkl"), "wb"))
    dist.destroy_process_group()


def test_shard_samples_partition():
    seen = []
    for r in range(4):
        f, n = D.shard_samples(r, 4, 5, first=7)
        seen += list(range(f, f + n))
    assert seen == list(range(7, 27))
    with pytest.raises(ValueError):
        D.shard_samples(4, 4, 5)


def test_gloo_world2_shards_equal_single_run(tmp_path, O):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    import pickle
    ok = np.load(tmp_path / "ok.npy")
    assert ok[0] == 1.5  # max over ranks
    gathered = pickle.load(open(tmp_path / "g.pkl", "rb"))
    x, y = WL.random_fitness(3, 3000, 2.4, 0.02, ecm=True)
    ref = O.sample(O.sort_plan(x, y, seg_target=32), seed=9, n_samples=6, first_sample=0)
    assert ok[1] == ref.accepted and ok[2] == ref.draws
    for r, (first, off, e, w) in enumerate(gathered):
        assert first == 3 * r
        for s in range(3):
            a, b = off[s], off[s + 1]
            ra, rb = ref.offsets[3 * r + s], ref.offsets[3 * r + s + 1]
            assert np.array_equal(np.array(e[a:b]).reshape(-1, 2), ref.edges[ra:rb])
            assert np.array_equal(np.array(w[a:b]), ref.weights[ra:rb])


def test_bench_self_launches_n_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself with 2 ranks (here with the gloo
    self-test of its rank logic: shards, max over ranks, sums; no GPU)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--selftest-dist"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 only
    r = lines[0]
    R = WL.workload(5).n_samples
    assert r["n_gpus"] == 2 and r["samples_per_rank"] == R
    assert r["first_samples"] == [0, R] and r["t_max"] == 11.0 and r["edges_all"] == 3000
