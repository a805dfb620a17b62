#!/usr/bin/env python
"""Benchmark of the sampler hot path (BASELINE.json metric: accepted edges/s and proposals/s on
one B200, and % of the sampler roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl own|reference]

One STEP = one pass of the whole hot path over one batch:
fm_sort_plan(x) + fm_sample_ubcm/ecm(plan, seed, R samples) + release, inputs resident in HBM.
Default workload: BASELINE.json configs[4] (config 5: UBCM ensemble batch, N=1e6, gamma 2.3,
mean degree 50, R = 64 samples per call, ~1.6e9 edges = 12.8 GB of int32 pairs per step), the
largest configuration that fits one GPU's call; configs 1-4 via --config.  Each rank samples its
own R samples (sample indices rank*R ...): weak scaling, no data-path collective (the samples are
independent).  `--gpus N` without a torchrun environment re-launches itself
under torch.distributed.run with N ranks (one per GPU).

Timing: W untimed warm-up steps; then K steps, each bracketed by CUDA events on the launching
stream, with a 256 MiB L2 flush (a write larger than the 126 MB L2) between steps outside the
events; barrier + synchronize on both sides; max over ranks.  SM clocks and throttle reasons are
sampled with NVML during the timed region.

`--impl reference` times the CPU oracle (oracle/, the tier's reference arm) on a bounded sample
of the same workload on the host cores; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2509_13230_b200 import dist as D  # noqa: E402
from paper_2509_13230_b200 import workloads as WL  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
COSTS_PATH = os.path.join(ROOT, "profiles", "op_costs.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--seg-target", type=int, default=256)
    ap.add_argument("--impl", choices=["own", "reference"], default="own")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="oracle work budget for cpu_baseline")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-api", choices=["to_host", "two_calls"], default="to_host",
                    help="e2e leg: fm_sample_to_host (overlapped D2H) or fm_sample_* followed by fm_edges_to_host")
    ap.add_argument("--refresh", action="store_true",
                    help="ECM: per-candidate beta_min refresh (fm_sample_ecm_ex FM_SAMPLE_BETA_REFRESH, NEXT-4)")
    ap.add_argument("--selftest-dist", action="store_true",
                    help="CPU self-test of the rank logic (gloo, no GPU, no sampling): shards and reductions")
    return ap.parse_args()


def self_launch(args) -> bool:
    """`--gpus N` (N > 1) outside torchrun: re-run this command under torch.distributed.run with N
    ranks on this node (127.0.0.1 rendezvous).  Returns True if it did (the caller then exits)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return False
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    rc = subprocess.call(cmd)
    if rc != 0:
        raise SystemExit(rc)
    return True


def run_selftest_dist(args):
    """The multi-rank plumbing of the own arm without a GPU (gloo): each rank takes its sample shard
    and a synthetic per-rank time and count; rank 0 prints the reduced values as one JSON line."""
    import torch.distributed as dist
    rank, _, world = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    R = WL.workload(args.config).n_samples
    first, n = D.shard_samples(rank, world, R)
    t_max = D.reduce_max(10.0 + rank)
    shards = D.reduce_sum([first if r == rank else 0 for r in range(world)])
    edges = D.reduce_sum([1000 * (rank + 1)])[0]
    if rank == 0:
        print(json.dumps({"selftest": "dist", "n_gpus": world, "samples_per_rank": n, "first_samples": shards,
                          "t_max": t_max, "edges_all": edges}), flush=True)
    if world > 1:
        dist.destroy_process_group()


dist_env = D.env_rank_world


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period: float = 0.05):
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._th = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception as ex:  # pragma: no cover
            self._nv = None
            self.error = str(ex)
        self.period = period

    def _run(self):
        while not self._stop.is_set():
            try:
                c = self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM)
                r = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append(c)
                self.reasons |= int(r) & ~0x1  # idle is not a slowdown
            except Exception:  # pragma: no cover
                pass
            self._stop.wait(self.period)

    def start(self):
        if self._nv:
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()

    def stop(self):
        if self._th:
            self._stop.set()
            self._th.join()

    def summary(self):
        if not self._nv:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None, "sm_max_mhz": self.max_mhz,
                "reasons": [v for k, v in self.REASONS.items() if self.reasons & k], "n_samples": len(self.samples)}


# ------------------------------------------------------------------------------------------ roofline
def roofline(model: str, counters: dict, kernel_ms: float, launches: int, cfg: int = 2, refresh: bool = False,
             call_ms: float | None = None):
    """Roofline of the dominant kernel k_sample.

    Compute term: algorithmic warp-instructions of the chain (op list of DESIGN 7.1, per-op
    costs measured on the B200 by scripts/microbench_ops.cu, frozen in profiles/op_costs.json),
    against two resources: issue (4 warp-inst/clk/SM x SMs x max clock) and the FP64 pipe
    (measured DFMA rate).  Memory term: 8 B (UBCM) / 12 B (ECM) per accepted edge at the
    measured HBM copy bandwidth.  The binding resource is the one with the largest time."""
    peaks = json.load(open(PEAKS_PATH)) if os.path.exists(PEAKS_PATH) else {}
    hbm = peaks.get("hbm_gbs", 6650.0)
    hbm_src = "measured" if "hbm_gbs" in peaks else "fallback"
    if not os.path.exists(COSTS_PATH):
        return None
    C = json.load(open(COSTS_PATH))
    clk = C["clock_mhz"] * 1e6
    sms = C["sm_count"]
    issue_peak = C["issue_warp_inst_per_clk_per_sm"] * sms * clk            # warp-inst/s
    fp64_peak = C["fp64_warp_inst_per_clk_per_sm"] * sms * clk               # warp-inst/s
    per = {k: dict(v) for k, v in C["per_unit"][model].items()}
    if refresh:  # per landed: + Ymax[cur+1] gather (2), y_u * Ymax, 1 - T', RN(1/(1-T')) (a division)
        d = C["per_op_warp_inst"]["ddiv"]
        per["landed"] = {"inst": per["landed"]["inst"] + 4 + d["inst"], "fp64": per["landed"]["fp64"] + 2 + d["fp64"]}
    draws, landed, acc = counters["draws"], counters["landed"], counters["accepted"]
    units = {"draw": draws, "landed": landed, "accepted": acc}
    inst = sum(units[u] * per[u]["inst"] for u in units) / 32.0             # warp-instructions
    fp64 = sum(units[u] * per[u]["fp64"] for u in units) / 32.0
    t = kernel_ms * 1e-3 / max(1, launches)                                 # per launch
    inst_l, fp64_l = inst / launches, fp64 / launches
    bytes_l = acc * (8 if model == "ubcm" else 12) / launches
    t_issue, t_fp64, t_mem = inst_l / issue_peak, fp64_l / fp64_peak, bytes_l / (hbm * 1e9)
    bound = max(("issue", t_issue), ("fp64", t_fp64), ("hbm", t_mem), key=lambda kv: kv[1])[0]
    if bound == "hbm":
        ach, peak, unit = bytes_l / t / 1e9, hbm, "GB/s"
    elif bound == "fp64":
        ach, peak, unit = fp64_l / t / 1e9, fp64_peak / 1e9, "G fp64 warp-inst/s"
    else:
        ach, peak, unit = inst_l / t / 1e9, issue_peak / 1e9, "G warp-inst/s"
    traffic = traffic_compact = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    tag = f"{model}_cfg{cfg}" + ("_refresh" if refresh else "")
    if os.path.exists(tpath):
        tj = json.load(open(tpath))
        tr = tj.get("k_sample", {}).get(tag)
        if tr:
            traffic = tr["dram_read_bytes"] + tr["dram_write_bytes"]
        tc = tj.get("k_compact", {}).get(tag)
        if tc:
            traffic_compact = tc["dram_read_bytes"] + tc["dram_write_bytes"]
    t_roof = max(t_issue, t_fp64, t_mem)
    # the whole fm_sample_* call (sampler + count scan + offsets + compaction), SURVEY 8(d) timing
    call = None
    if call_ms is not None:
        tc_l = call_ms * 1e-3 / max(1, launches)
        call = {"ms_per_call": tc_l * 1e3, "frac": t_roof / tc_l,
                "note": "t_roof of the call's algorithmic work / (k_sample + write phase) device time per call"}
    return {"bound": "alu" if bound != "hbm" else "hbm", "resource": bound, "achieved": ach, "peak": peak,
            "unit": unit, "frac": ach / peak, "traffic": traffic, "traffic_compact": traffic_compact,
            "traffic_note": "dram read+write bytes per launch of k_sample (traffic) and k_compact (traffic_compact) "
                            "from ncu --set full captures (profiles/traffic.json)",
            "call": call,
            "kernel": "k_sample",
            "kernel_ms_per_launch": t * 1e3, "t_roof_ms": t_roof * 1e3,
            "terms_ms": {"issue": t_issue * 1e3, "fp64": t_fp64 * 1e3, "hbm": t_mem * 1e3},
            "alg_warp_inst_per_launch": inst_l, "alg_fp64_warp_inst_per_launch": fp64_l,
            "alg_bytes_per_launch": bytes_l, "peak_source": f"op_costs.json (measured) + hbm {hbm_src}",
            "clock_mhz_for_peak": C["clock_mhz"]}


# ------------------------------------------------------------------------------------------ oracle
def cpu_oracle_run(w, x, y, seg_target, budget_s, refresh=False):
    """Time the oracle as it stands on the host cores on a bounded sample of the workload."""
    from oracle import oracle as O
    O.build()
    nth = O.ncores()
    t0 = time.perf_counter()
    plan = O.sort_plan(x, y, seg_target=seg_target)
    t_plan = time.perf_counter() - t0
    # probe with one sample, then size the run to ~budget_s
    t0 = time.perf_counter()
    O.sample(plan, w.seed, n_samples=1, first_sample=0, nthreads=nth, refresh=refresh)
    t1 = time.perf_counter() - t0
    R = int(max(1, min(w.n_samples, budget_s / max(t1, 1e-6))))
    t0 = time.perf_counter()
    r = O.sample(plan, w.seed, n_samples=R, first_sample=0, nthreads=nth, refresh=refresh)
    dt = time.perf_counter() - t0
    # per-sample plan cost amortised like the GPU step: plan once per R samples of a step
    step_s = dt + t_plan * (R / w.n_samples)
    return {"value": r.accepted / step_s, "unit": "edges/s", "cores": nth, "kind": "oracle",
            "sample": f"{R} of the {w.n_samples} samples of {w.name} (+ plan time pro-rated), seed {w.seed}",
            "proposals_per_s": r.landed / step_s, "draws_per_s": r.draws / step_s, "seconds": dt + t_plan,
            "edges": r.accepted}


METRIC = "accepted edges/s (proposals/s alongside); % of sampler roofline"


def config_dict(w, args, R, world):
    """The workload of a bench line (both arms)."""
    return {"workload": w.name, "model": w.model, "n": w.n, "gamma": w.gamma, "kbar": w.kbar,
            "samples_per_step_per_gpu": R, "seg_target": args.seg_target, "seed": w.seed,
            "step": "fm_sort_plan + fm_sample_%s(%d samples) + free" % (w.model, R),
            "beta_refresh": bool(args.refresh and w.model == "ecm"),
            "l2": "256 MiB write between timed steps (outside events); output per step > L2",
            "parallelism": f"sample-parallel x{world} (no data-path collective)"}


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    w = WL.workload(args.config)
    x, y = WL.fitness(w)
    res = []
    for i in range(args.warmup + args.steps):
        c = cpu_oracle_run(w, x, y, args.seg_target, max(1.0, args.cpu_seconds / max(1, args.steps)),
                           refresh=args.refresh)
        if i >= args.warmup:
            res.append(c)
    v = statistics.median([c["value"] for c in res])
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "edges/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * statistics.median([c["seconds"] for c in res]), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(w, args, w.n_samples, 1),
            "cpu_baseline": {k: res[-1][k] for k in ("unit", "cores", "kind", "sample")} | {"value": v},
            "proposals_per_s": statistics.median([c["proposals_per_s"] for c in res]),
            "e2e": {"value": v, "unit": "edges/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------ own arm
def run_own(args):
    import torch
    import torch.distributed as dist

    rank, local_rank, world = dist_env()
    if world > 1:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()
    from paper_2509_13230_b200 import fastmaxent as fm

    w = WL.workload(args.config)
    x, y = WL.fitness(w)
    xd = torch.from_numpy(x).cuda()
    yd = None if y is None else torch.from_numpy(y).cuda()
    R = w.n_samples
    first, _ = D.shard_samples(rank, world, R)
    if w.model == "ubcm":
        sample = fm.sample_ubcm
    else:
        def sample(plan, seed, **kw):
            return fm.sample_ecm(plan, seed, refresh=args.refresh, **kw)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        plan = fm.sort_plan(xd, yd, seg_target=args.seg_target)
        e = sample(plan, w.seed, n_samples=R, first_sample=first)
        c = {"draws": e.draws, "landed": e.landed, "accepted": e.accepted, "n_edges": e.n_edges,
             "segments": e.segments, "chunks": e.chunks}
        e.free()
        plan.free()
        return c

    fm.timing_enable(True)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    fm.timing_get(reset=True)
    l0 = fm.timing_get()["launches"]

    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev)
    clocks.start()
    tot = {"draws": 0, "landed": 0, "accepted": 0, "n_edges": 0}
    ms = []
    for k in range(args.steps):
        flush.fill_(k & 0xFF)  # L2 flush, outside the timed events
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        c = step()
        b.record()
        b.synchronize()
        ms.append(a.elapsed_time(b))
        for kk in tot:
            tot[kk] += c[kk]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks.stop()
    tim = fm.timing_get(reset=True)
    launches = tim["launches"] - l0
    t_rank = sum(ms)
    t_max = D.reduce_max(t_rank, device="cuda")
    edges_all, landed_all, draws_all, launches_all = D.reduce_sum(
        [tot["n_edges"], tot["landed"], tot["draws"], launches], device="cuda")
    value = edges_all / (t_max * 1e-3)

    # ---------------- e2e through the C-ABI with host buffers (pinned), copies inside ----------
    e2e = None
    if not args.no_e2e:
        xh = torch.from_numpy(x).pin_memory()
        yh = None if y is None else torch.from_numpy(y).pin_memory()
        cap = int(1.3 * max(c["n_edges"], 1)) + 1024
        eh = torch.empty((cap, 2), dtype=torch.int32).pin_memory()
        wh = torch.empty(cap, dtype=torch.int32).pin_memory() if y is not None else None
        e_ms, e_edges, h2d, d2h = [], 0, 0, 0
        e_phase = {"plan_sample": 0.0, "d2h": 0.0}
        for k in range(args.e2e_steps + 1):
            flush.fill_(k & 0xFF)
            torch.cuda.synchronize()
            a, m, b = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            a.record()
            plan = fm.sort_plan(xh, yh, seg_target=args.seg_target)       # host pointers -> H2D inside
            if args.e2e_api == "to_host":
                # fm_sample_to_host: each group of samples is copied to the host while the next ones
                # are generated (the D2H of the list inside the call)
                e = fm.sample_to_host(plan, w.seed, eh, wh, n_samples=R, first_sample=first,
                                      refresh=args.refresh and y is not None)
                m.record()
                if e.flags & fm.FM_FLAG_HOST_TRUNCATED:  # (host buffers too small: plain copy of the device list)
                    eh = torch.empty((e.n_edges, 2), dtype=torch.int32).pin_memory()
                    wh = torch.empty(e.n_edges, dtype=torch.int32).pin_memory() if y is not None else None
                    e.to_host(eh, wh)
            else:
                e = sample(plan, w.seed, n_samples=R, first_sample=first)
                if e.n_edges > eh.shape[0]:
                    eh = torch.empty((e.n_edges, 2), dtype=torch.int32).pin_memory()
                    wh = torch.empty(e.n_edges, dtype=torch.int32).pin_memory() if y is not None else None
                m.record()
                e.to_host(eh, wh)                                             # D2H of the result
            b.record()
            b.synchronize()
            if k > 0:  # first iteration is a warm-up
                e_ms.append(a.elapsed_time(b))
                e_phase["plan_sample"] += a.elapsed_time(m) / args.e2e_steps
                e_phase["d2h"] += m.elapsed_time(b) / args.e2e_steps
                e_edges += e.n_edges
                h2d = x.nbytes + (0 if y is None else y.nbytes)
                d2h = e.n_edges * (8 if y is None else 12) + 8 * (R + 1)
            e.free()
            plan.free()
        e2e = {"value": e_edges / (sum(e_ms) * 1e-3), "unit": "edges/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": statistics.mean(e_ms), "steps": len(e_ms),
               "host_buffers": "pinned", "phase_ms": e_phase,
               "api": "fm_sort_plan(host x) + fm_sample_to_host (D2H of each sample group overlaps the next groups)"
               if args.e2e_api == "to_host" else "fm_sort_plan(host x) + fm_sample_* + fm_edges_to_host",
               "d2h_gbs": (d2h / (e_phase["d2h"] * 1e-3) / 1e9 if e_phase["d2h"] > 1e-3 else None) if args.e2e_api != "to_host"
               else d2h / (statistics.mean(e_ms) * 1e-3) / 1e9}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    refresh = args.refresh and w.model == "ecm"
    rf = roofline(w.model, tot, tim["sample_ms"], max(1, tim["sample_launches"]), cfg=args.config, refresh=refresh,
                  call_ms=tim["sample_ms"] + tim["write_ms"])
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        c = cpu_oracle_run(w, x, y, args.seg_target, args.cpu_seconds, refresh=refresh)
        cpu = {k: c[k] for k in ("value", "unit", "cores", "kind", "sample")}
        cpu["proposals_per_s"] = c["proposals_per_s"]
    line = {
        "metric": METRIC,
        "value": value, "unit": "edges/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_max / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": config_dict(w, args, R, world),
        "proposals_per_s": landed_all / (t_max * 1e-3), "draws_per_s": draws_all / (t_max * 1e-3),
        "edges_per_step": edges_all / args.steps / world,
        "phase_ms_per_step": {"plan": tim["plan_ms"] / args.steps, "sample_kernel": tim["sample_ms"] / args.steps,
                              "write": tim["write_ms"] / args.steps},
        "roofline": rf, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches_all),
        "clocks": clocks.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if self_launch(args):
        return
    if args.selftest_dist:
        run_selftest_dist(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_own(args)


if __name__ == "__main__":
    main()
