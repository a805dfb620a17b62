"""The README usage example (run from the repository root: PYTHONPATH=. python scripts/readme_example.py)."""
import torch
from paper_2509_13230_b200 import fastmaxent as fm
x = torch.rand(100_000, dtype=torch.float64, device="cuda") ** -0.8 * 1e-3
plan = fm.sort_plan(x)
e = fm.sample_ubcm(plan, seed=7, n_samples=16)
print(e.n_edges, e.offsets)
src_dst = e.edges
deg, *_ = fm.sample_degrees(plan, seed=7, n_samples=16)
host = torch.empty((int(1.1 * e.n_edges), 2), dtype=torch.int32).pin_memory()
eh = fm.sample_to_host(plan, 7, host, n_samples=16)
assert torch.equal(host[:eh.n_edges].cuda(), e.edges) and int(deg.sum()) == 2 * e.n_edges
print("readme example ok")
