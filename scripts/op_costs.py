"""Freeze the per-op costs of the sampler roofline from the microbenchmark.

Input: an ncu CSV of scripts/microbench_ops (metrics sm__inst_executed.sum,
sm__inst_executed_pipe_fp64.sum, ... one row per kernel launch).  Output: profiles/op_costs.json
with warp-instructions (all pipes, and FP64 pipe) per warp-level call of each op, the FP64 pipe
rate per SM clock, and the per-unit algorithmic op lists of the chain.

    python scripts/op_costs.py gpurun_out/micro_ncu.csv [--impl stock|fm] > profiles/op_costs.json
"""
import collections
import csv
import json
import sys

M = 2048  # iterations per thread in microbench_ops.cu


def load(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    data = collections.OrderedDict()
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            # template args kept: "void k_log1p<(int)-30, 41>(double *, ...)" -> k_log1p<-30,41>
            name = d["Kernel Name"].replace("void ", "").replace("(int)", "").split("(")[0].replace(" ", "")
            data.setdefault(name, {})[d["Metric Name"]] = float(d["Metric Value"].replace(",", ""))
    return data


def main():
    path = sys.argv[1]
    impl = "stock"
    if "--impl" in sys.argv:
        impl = sys.argv[sys.argv.index("--impl") + 1]
    d = load(path)
    warps = None
    # warp-calls: threads / 32 * M ; threads from the DFMA kernel's fp64 count (8 chains x M per thread)
    fp64_dfma = d["k_dfma"]["sm__inst_executed_pipe_fp64.sum"]
    warp_calls = fp64_dfma / 8.0 / 1.0  # 8 DFMA per thread-iteration -> warp-calls * 8 (+ small epilogue)
    warp_calls = round(warp_calls / M) * M
    per_call = lambda k, base, key: (d[k][key] - d[base][key]) / warp_calls  # noqa: E731
    ops = {}
    # log1p: warp-uniform exponent e in [-30, 10] (each warp call takes one range path; round 2),
    # and per path: e in [-30, -2] (small X) and e in [0, 10] (large X)
    for op, k, base in (("philox", "k_philox", "k_base"), ("log", "k_log", "k_base_u01"),
                        ("log1p", "k_log1p<-30,41>", "k_base_log1p<-30,41>"), ("ddiv", "k_ddiv", "k_base_ddiv"),
                        ("u01", "k_base_u01", "k_base"),
                        ("log1p_small_path", "k_log1p<-30,29>", "k_base_log1p<-30,29>"),
                        ("log1p_large_path", "k_log1p<0,11>", "k_base_log1p<0,11>")):
        ops[op] = {"inst": per_call(k, base, "sm__inst_executed.sum"),
                   "fp64": per_call(k, base, "sm__inst_executed_pipe_fp64.sum")}
    ops["ddiv"]["inst"] += 1.0  # the base kernel has a DMUL in place of the division
    ops["ddiv"]["fp64"] += 1.0
    ops["u01"]["inst"] -= 1.0   # the base kernel accumulates with one DADD
    ops["u01"]["fp64"] -= 1.0
    cyc = d["k_dfma"]["sm__cycles_elapsed.avg"]
    fp64_rate = fp64_dfma / 148.0 / cyc  # fp64 warp-inst per SM clock (measured)
    o = {k: v for k, v in ops.items()}

    def unit(inst, fp64):
        return {"inst": round(inst, 2), "fp64": round(fp64, 2)}

    # algorithmic op lists; scalar ops: 1 warp-instruction each
    ph_u, ph_e = 0.5 * o["philox"]["inst"], o["philox"]["inst"]
    draw_u = unit(ph_u + o["u01"]["inst"] + o["log"]["inst"] + o["ddiv"]["inst"] + 4,
                  o["u01"]["fp64"] + o["log"]["fp64"] + o["ddiv"]["fp64"] + 2)
    draw_e = unit(ph_e + o["u01"]["inst"] + o["log"]["inst"] + o["ddiv"]["inst"] + 4,
                  o["u01"]["fp64"] + o["log"]["fp64"] + o["ddiv"]["fp64"] + 2)
    # landed (contract R10, division-free): F2I, 2 IADD, gather (LDG + address), X = DMUL, D = DADD,
    # accept: u01 + 3 DMUL + DSETP, log1p
    land_u = unit(1 + 2 + 2 + 1 + 1 + o["u01"]["inst"] + 3 + 1 + o["log1p"]["inst"],
                  1 + 1 + 1 + o["u01"]["fp64"] + 3 + 1 + o["log1p"]["fp64"])
    # ECM landed: + gathers y, log y; z, t, 1-t, Dp; accept 3 DMUL + DSETP; dq = DADD; z*iomT; log1p
    land_e = unit(1 + 2 + 6 + 4 + o["u01"]["inst"] + 3 + 1 + 1 + 1 + o["log1p"]["inst"],
                  1 + 4 + o["u01"]["fp64"] + 3 + 1 + 1 + 1 + o["log1p"]["fp64"])
    acc_u = unit(6, 0)
    # ECM accepted: log(u01) + DADD (log y_u + log y_v) + div + floor + F2I + saturation test + weight store
    acc_e = unit(6 + 2 + o["u01"]["inst"] + o["log"]["inst"] + 1 + o["ddiv"]["inst"] + 4,
                 o["u01"]["fp64"] + o["log"]["fp64"] + 1 + o["ddiv"]["fp64"] + 3)
    out = {
        "source": f"scripts/microbench_ops.cu under ncu ({path}); B200, CUDA 12.9",
        "impl": impl,
        "per_op_warp_inst": {k: {kk: round(vv, 2) for kk, vv in v.items()} for k, v in ops.items()},
        "fp64_warp_inst_per_clk_per_sm_measured": round(fp64_rate, 3),
        "fp64_warp_inst_per_clk_per_sm": 2.0,
        "issue_warp_inst_per_clk_per_sm": 4.0,
        "sm_count": 148,
        "clock_mhz": 1965.0,
        "per_unit": {"ubcm": {"draw": draw_u, "landed": land_u, "accepted": acc_u},
                     "ecm": {"draw": draw_e, "landed": land_e, "accepted": acc_e}},
        "notes": "inst/fp64 = warp-instructions per warp-level unit (32 lanes). Peaks: issue 4/clk/SM "
                 "(4 SMSPs x 1), FP64 pipe 2/clk/SM (64 lanes; measured DFMA rate alongside), "
                 "at the 1965 MHz max SM clock. log1p: warp-uniform input exponent in [-30, 10] (one range "
                 "path per warp call; divergence not counted as algorithmic work); per-path costs alongside.",
    }
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
