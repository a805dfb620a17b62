import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2509_13230_b200 import fastmaxent as fm, workloads as WL
w = WL.workload(int(sys.argv[1]) if len(sys.argv) > 1 else 1)
x, y = WL.fitness(w)
plan = fm.sort_plan(torch.from_numpy(x).cuda(), None if y is None else torch.from_numpy(y).cuda())
print("plan ok", plan.info() if hasattr(plan, "info") else "", flush=True)
fn = fm.sample_ubcm if y is None else fm.sample_ecm
e = fn(plan, w.seed, n_samples=2)
torch.cuda.synchronize()
print("sample ok", e.n_edges, e.draws, flush=True)
