"""Wall-clock breakdown of the host path on one config: fm_sort_plan(host x) and fm_sample_to_host."""
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402
from paper_2509_13230_b200 import workloads as WL  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = WL.workload(cfg)
x, y = WL.fitness(w)
xh = torch.from_numpy(x).pin_memory()
yh = None if y is None else torch.from_numpy(y).pin_memory()
plan = fm.sort_plan(xh, yh)
e = (fm.sample_ubcm if y is None else fm.sample_ecm)(plan, w.seed, n_samples=w.n_samples)
n = e.n_edges
e.free()
eh = torch.empty((int(1.1 * n), 2), dtype=torch.int32).pin_memory()
wh = torch.empty(int(1.1 * n), dtype=torch.int32).pin_memory() if y is not None else None
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = fm.sort_plan(xh, yh)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e = fm.sample_to_host(plan, w.seed, eh, wh, n_samples=w.n_samples)
    t2 = time.perf_counter()
    e.free()
    plan.free()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    e2 = (fm.sample_ubcm if y is None else fm.sample_ecm)(fm.sort_plan(xh, yh), w.seed, n_samples=w.n_samples)
    t4 = time.perf_counter()
    e2.to_host(eh, wh)
    t5 = time.perf_counter()
    print(f"plan {1e3 * (t1 - t0):.2f} ms, sample_to_host {1e3 * (t2 - t1):.2f} ms, free {1e3 * (t3 - t2):.2f} ms | "
          f"plan+sample {1e3 * (t4 - t3):.2f} ms, to_host {1e3 * (t5 - t4):.2f} ms; edges {n}")
    e2.free()
