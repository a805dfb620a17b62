"""Leak check: device memory free before / after many plan + sample + free cycles (pool trimmed)."""
import gc

gc.disable()  # reference counting alone must release everything
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402
from paper_2509_13230_b200 import workloads as WL  # noqa: E402


def free_mb(collect=False):
    torch.cuda.synchronize()
    if collect:
        gc.collect()
    torch.cuda.empty_cache()
    fm.pool_trim(0)
    return torch.cuda.mem_get_info()[0] / 2**20


x, y = WL.random_fitness(1, 30_000, 2.4, 0.02, ecm=True)
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
variants = [({}, None), ({"FM_SAMPLE_GROUPS": "3"}, None), ({}, yd), ({"FM_DEBUG_SCRATCH_CAP": "8"}, None),
            ({"FM_FUSE_WRITE": "1"}, None), ({"FM_SAMPLE_GROUPS": "2"}, yd)]
# warm every code path once (lazily created streams, tables, module data)
for env, yy in variants:
    os.environ.update(env)
    p = fm.sort_plan(xd, yy, seg_target=64)
    e = (fm.sample_ubcm if yy is None else fm.sample_ecm)(p, 1, n_samples=4)
    fm.sample_degrees(p, 1, n_samples=2)
    del e, p
    for k in env:
        del os.environ[k]
x2, y2 = WL.random_fitness(2, 11_000, 2.4, 0.02, ecm=True)
x2d, y2d = torch.from_numpy(x2).cuda(), torch.from_numpy(y2).cuda()
x3, y3 = WL.random_fitness(3, 30_000, 2.4, 0.02, ecm=True)
x3d, y3d = torch.from_numpy(x3).cuda(), torch.from_numpy(y3).cuda()


def make_plan(it, yy):
    kind = it % 4
    if kind == 1:
        return fm.sort_plan_bipartite(xd, x2d, yy, None if yy is None else y2d, kind="bipartite", seg_target=64)
    if kind == 2:
        return fm.sort_plan_bipartite(xd, x3d, yy, None if yy is None else y3d, kind="directed", seg_target=64)
    return fm.sort_plan(xd, yy, seg_target=64 if kind == 0 else 8)


for it in range(8):
    p = make_plan(it, yd if it >= 4 else None)
    e = (fm.sample_ubcm if it < 4 else fm.sample_ecm)(p, 1, n_samples=2)
    fm.sample_degrees(p, 1, n_samples=2)
    del e, p
HOST_E = torch.empty((4_000_000, 2), dtype=torch.int32).pin_memory()
HOST_W = torch.empty(4_000_000, dtype=torch.int32).pin_memory()
f0 = free_mb()
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 200):
    env, yy = variants[it % len(variants)]
    os.environ.update(env)
    p = make_plan(it // 2, yy)
    e = (fm.sample_ubcm if yy is None else fm.sample_ecm)(p, it, n_samples=4)
    if it % 3 == 0:
        fm.sample_degrees(p, it, n_samples=2)
    if it % 5 == 0 and yy is None and p.kind == 0:
        fm.sample_richclub(p, it, n_samples=2)
    if it % 7 == 0:
        e.to_host()
    if it % 6 == 1:  # the overlapped host path (forced groups)
        os.environ["FM_HOST_GROUPS"] = "3"
        eh = fm.sample_to_host(p, it, HOST_E, HOST_W if yy is not None else None, n_samples=4)
        del os.environ["FM_HOST_GROUPS"]
        del eh
    if it % 2 == 0:  # tensor views of the result (they once kept the result alive in an uncollectable cycle)
        v = e.edges[:10].clone()
        w = e.weights
    del e, p
    for k in env:
        del os.environ[k]
USED = (torch.cuda.mem_get_info()[1] - torch.cuda.mem_get_info()[0]) / 2**20
f1 = free_mb()
print(f"free before {f0:.1f} MiB, after {f1:.1f} MiB, delta {f0 - f1:.1f} MiB")
print("untrimmed used MiB during the loop:", USED)
assert f0 - f1 < 64, "device memory leak"
