"""Co-residency probe: the sampler (config 5) with a small-footprint copy kernel on a second stream."""
import ctypes as C
import os
import subprocess
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2509_13230_b200 import fastmaxent as fm  # noqa: E402
from paper_2509_13230_b200 import workloads as WL  # noqa: E402

so = "/tmp/libcoprobe.so"
subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                       "-o", so, os.path.join(ROOT, "scripts/probe/coprobe.cu")])
P = C.CDLL(so)
P.probe_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_long, C.c_int, C.c_int, C.c_void_p]
print("copy kernel registers:", P.probe_regs())

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
w = WL.workload(cfg)
x, _ = WL.fitness(w)
plan = fm.sort_plan(torch.from_numpy(x).cuda())
R = w.n_samples
nbytes = int(float(os.environ.get("PROBE_GB", "12.8")) * 1e9) // 16 * 16
src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dst = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
src.zero_()
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
fm.timing_enable(True)


def run_sampler():
    e = fm.sample_ubcm(plan, seed=w.seed, n_samples=R, stream=sa)
    n = e.n_edges
    e.free()
    return n


def copy(blocks, carve):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(sb)
    rc = P.probe_copy(dst.data_ptr(), src.data_ptr(), nbytes // 16, blocks, carve, sb.cuda_stream)
    assert rc == 0, rc
    ev1.record(sb)
    return ev0, ev1


for _ in range(2):
    run_sampler()
torch.cuda.synchronize()
fm.timing_get(reset=True)
run_sampler()
t = fm.timing_get(reset=True)
print(f"sampler alone: sample {t['sample_ms']:.3f} ms write {t['write_ms']:.3f} ms")
for blocks in (148, 148 * 16):
    for carve in (-1, 42):
        a, b = copy(blocks, carve)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        print(f"copy alone: blocks {blocks} carve {carve}: {ms:.3f} ms, {2 * nbytes / ms / 1e6:.0f} GB/s (read+write)")
for blocks in (148, 296, 148 * 16):
    for carve in (-1, 42, 50):
        a, b = copy(blocks, carve)
        run_sampler()
        torch.cuda.synchronize()
        t = fm.timing_get(reset=True)
        ms = a.elapsed_time(b)
        print(f"together: blocks {blocks} carve {carve}: copy {ms:.3f} ms ({2 * nbytes / ms / 1e6:.0f} GB/s), sample "
              f"{t['sample_ms']:.3f} ms write {t['write_ms']:.3f} ms")

# ---- reverse order: the sampler is resident first, the copy arrives 5 ms later (another host thread) ----
import threading
import time

P.probe_copy_short.argtypes = [C.c_void_p, C.c_void_p, C.c_long, C.c_long, C.c_void_p]
os.environ["FM_SAMPLE_GROUPS"] = "1"


def copy_short(per):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(sb)
    rc = P.probe_copy_short(dst.data_ptr(), src.data_ptr(), nbytes // 16, per, sb.cuda_stream)
    assert rc == 0, rc
    ev1.record(sb)
    return ev0, ev1


def late(fn, arg, out):
    time.sleep(0.005)
    out.append(time.perf_counter())
    out.extend(fn(*arg))


for name, fn, arg in (("persistent 148", copy, (148, -1)), ("persistent 2368", copy, (2368, -1)),
                      ("short 128KB", copy_short, (8192,)), ("short 1MB", copy_short, (65536,))):
    a, b = fn(*arg)
    torch.cuda.synchronize()
    solo = a.elapsed_time(b)
    evs = []
    th = threading.Thread(target=late, args=(fn, arg, evs))
    ref0, ref1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ref0.record(sa)
    t0 = time.perf_counter()
    th.start()
    run_sampler()
    t1 = time.perf_counter()
    ref1.record(sa)
    th.join()
    torch.cuda.synchronize()
    t = fm.timing_get(reset=True)
    print(f"sampler first, {name}: copy solo {solo:.3f} ms; late copy launched at host +{1e3 * (evs[0] - t0):.2f} ms, "
          f"device: copy starts {ref0.elapsed_time(evs[1]):.2f} ms ends {ref0.elapsed_time(evs[2]):.2f} ms after the call began; "
          f"sample {t['sample_ms']:.3f} ms write {t['write_ms']:.3f} ms, host call {1e3 * (t1 - t0):.2f} ms")
