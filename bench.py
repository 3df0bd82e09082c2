#!/usr/bin/env python
"""bench.py -- factorizations/s of the hot path on B200 (BASELINE.json metric), vs the
INT32-ALU roofline (count) and the HBM roofline (store), with the CPU oracle beside it.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3count] [--impl fsgpu|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

A step = one full pass of the hot path over the workload instance: plan constants/DP tables
are resident in HBM, the persistent kernel enumerates every factorization of the rank's
block of the lex order (count consumer) and, for N > 1, one NCCL all_reduce combines the
partial counts.  Default workload: C3 = Z(4275, (13,14,20,22,23,24,35,39)),
|Z| = 100,032,405,189 (BASELINE.json configs[2]).  Strong scaling (fixed instance).
Extra keys: the store path (C2-XL materialise, 26 GB of u16 rows) with its HBM roofline and
the C4 length histogram, each measured in the same run.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2405_07989_b200 import workloads as W  # noqa: E402

METRIC = "factorizations/sec (count, store) at 1/2/4/8 B200 vs INT-ALU/HBM roofline"
UNIT = "factorizations/s"

# Algorithmic integer-op model per unit of the method, counting the
# minimal operations of the residue/quotient representation R_L = A g_{d-1} + rho:
#   node entry (advance to the next level-L prefix: transition load, residue, quotient;
#     first valid a* = A - k0(rho); run counter)                                   :  5
#   row (one valid factorization consumed, a_{d-1} -= s, compare, counter)           :  4
#   deeper node (ascend to a level-k prefix, k < L, greedy re-solve)                 : 12
OPS_NODE, OPS_ROW, OPS_DEEP = 5, 4, 12
INT_LANES_PER_CLK_PER_SM = 128  # 4 SMSPs x 32 lanes, one warp-instruction / clk each
NUM_SMS = 148


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS, "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def microbench():
    """Measured roofline denominators on this GPU (csrc/fs_micro.cu): INT32 lane-op rates of
    IADD3 / IMAD / 1:1 mix / LOP3 chains and coalesced 16 B streaming-store bandwidth."""
    import ctypes

    from paper_2405_07989_b200 import _lib as L

    out = {}
    for kind, name in [(0, "iadd"), (1, "imad"), (2, "mix"), (3, "lop3")]:
        r, a = ctypes.c_double(0), ctypes.c_double(0)
        L.check(L.lib().fsdbg_microbench(kind, 0, ctypes.byref(r), ctypes.byref(a)), "microbench")
        out[name] = {"ops_per_clk_per_sm": r.value, "tops": a.value}
    r, a = ctypes.c_double(0), ctypes.c_double(0)
    L.check(L.lib().fsdbg_microbench(4, 8 << 30, ctypes.byref(r), ctypes.byref(a)), "microbench")
    out["hbm_write_gbs"] = r.value
    return out


OPS_NODE_CLOSED = 8  # node entry (5) + closed-form row count floor(a*/s) + 1: max, mulhi, add (NEXT-1)
# Closed-tail count in STATE form (fs_kernels.cuh cq_group; info["state_block"] = K > 0): the
# level-L nodes of a run are walked K at a time through the (rho, A mod s) automaton table:
OPS_BLOCK_STATE = 3  # per K-block: quotient step, masked row-count add, block mask (the table
#                      load is an LSU op)
OPS_RUN_STATE = 12   # per run (level-(L-1) node): one-level ascend (prefix/residual update, a_L),
#                      budget/run-length min, entry rows add, state + quotient decode, run-length
#                      remainder adjust


OPS_NODE_HIST_CLOSED = 12  # closed-tail histogram: node entry (5) + rows (3) + first-row length (2) + two
#                            difference-array updates (2)
# Closed-tail histogram in STATE form (fs_kernels.cuh hq_group; info["state_block"] = 8 for a
# histogram plan): per level-L node two offset extracts, two base adds and the two
# difference-array updates; per 8-node block the two base steps and the link; per run the
# one-level ascend (12) plus the entered node's state and bases (one division, 10)
OPS_NODE_HIST_STATE = 6
OPS_RUN_HIST_STATE = 22
OPS_NODE_ANY_CLOSED = 14   # closed-tail any: node entry (5) + rows (3) + a_d of the first row (2) + the
#                            progression's extreme length (2) + compare/flag (2)


def ops_model(info, closed: bool = False, hist: bool = False, any_: bool = False) -> float:
    """algorithmic integer ops of the stream the kernel runs: per node
    entry, per row (per-row tail) or per node (closed tail), per deeper node."""
    nodes = info["nodes_per_level"]
    L = info["level"]
    deep = sum(nodes[1:L]) if L >= 2 else 0
    K = info.get("state_block", 0)
    if closed and K and not any_:
        runs = nodes[L - 1] if L >= 1 else 1
        deep2 = sum(nodes[1:L - 1]) if L >= 3 else 0
        if hist:
            return (OPS_NODE_HIST_STATE * nodes[L] + OPS_BLOCK_STATE * nodes[L] / K + OPS_RUN_HIST_STATE * runs
                    + OPS_DEEP * deep2)
        return OPS_BLOCK_STATE * nodes[L] / K + OPS_RUN_STATE * runs + OPS_DEEP * deep2
    if closed:
        per = OPS_NODE_HIST_CLOSED if hist else OPS_NODE_ANY_CLOSED if any_ else OPS_NODE_CLOSED
        return per * nodes[L] + OPS_DEEP * deep
    return OPS_NODE * nodes[L] + OPS_ROW * info["total_rows"] + OPS_DEEP * deep


OPS_CAND = 5  # one candidate of the paper's index-(d-1) loop: residue add, conditional subtract,
#              zero test, accumulate, loop (SURVEY 8(d) c_step)
OPS_MODEL_DOC = ("closed tail, state form (the headline): 3 int ops per block of K level-L nodes + 12 per run "
                 "(level-(L-1) node) + 12 per deeper node; closed tail, residue form: 8 per level-L node + 12 per "
                 "deeper node; histogram, state form: 6 per level-L node + 3 per 8-node block + 22 per run + 12 per "
                 "deeper node; per-row tail: 5 per node + 4 per row + 12 per deeper node; Skip ablations: "
                 "5 per candidate + 5 per node + 12 per deeper node (DESIGN.md section 6)")


def paper_candidates(inst, skip_paper: bool, gens=None) -> int:
    """Exact number of candidates the paper's stream (Alg. 3.1) visits on the
    instance, with or without its modulo skip: Skip=off visits
    sum_{k<d} #{prefixes of length k with phi < n}; with the skip, a level-(d-2)
    node of residual R > 0 visits c - j (s - 1) index-(d-1) candidates instead of
    c = ceil(R / g_{d-1}), where a* is its largest valid a_{d-1} and j = floor(a* / s) the jumps
    (none without a valid a*).  Reproduces SURVEY's 9,576 / 3,629 (C1)."""
    from math import gcd

    n = inst.n
    g = list(gens or inst.gens)
    d = len(g)
    if d < 2:
        return 1
    F = [0] * (n + 1)
    F[0] = 1
    tot = 1 if n > 0 else 0  # the empty prefix
    for k in range(d - 2):
        for r in range(g[k], n + 1):
            F[r] += F[r - g[k]]
        tot += sum(F[:n])  # prefixes of length k + 1 with phi < n
    gA, gB = g[d - 2], g[d - 1]
    s = gB // gcd(gA, gB)
    for phi in range(n):
        m = F[phi]
        if not m:
            continue
        R = n - phi
        c = -(-R // gA)
        cnt = c
        if skip_paper:
            a = R // gA
            while a >= 0 and (R - a * gA) % gB:
                a -= 1
            if a >= 0:
                cnt = c - (a // s) * (s - 1)
        tot += m * cnt
    return tot


# ------------------------------------------------------------------ CPU oracle (baseline arm)
def oracle_sample(inst, seconds: float, seed: int = 0):
    """Time the nested-loop oracle (as it stands, 1 thread) on a bounded sample of prefix boxes
    of the instance: prefixes (a_1..a_k), k = min(3, d-2), drawn with probability proportional
    to the oracle's work below them (innermost iterations, oracle.gf.work_tables), each run as
    one oracle box.  Ratio estimator of the whole-instance rate:
        rate = sum_i rows_i / w_i  /  sum_i secs_i / w_i.
    Returns (rate, rows, secs, boxes)."""
    import random

    import oracle
    from oracle import gf

    oracle.build()
    n, g = inst.n, inst.gens
    d = len(g)
    Wt = gf.work_tables(n, g)
    # deepest prefix length (<= 3, <= d-2) whose boxes average >= 1e6 innermost iterations
    depth = 0
    for k in range(1, max(0, min(3, d - 2)) + 1):
        nodes_k = sum(gf.count_table(n, g[:k]))
        if Wt[0][n] / nodes_k >= 1e6:
            depth = k
    rng = random.Random(seed)
    num = den = 0.0
    rows_tot, secs_tot, boxes = 0, 0.0, 0
    t_start = time.perf_counter()
    while time.perf_counter() - t_start < seconds:
        R, prefix = n, []
        for k in range(depth):
            top = R // g[k]
            cands = list(range(top + 1))
            w = [Wt[k + 1][R - x * g[k]] for x in cands]
            x = rng.choices(cands, weights=w, k=1)[0]
            prefix.append(x)
            R -= x * g[k]
        wi = Wt[depth][R] if depth < d else 1
        if depth == 0:
            box = None
        else:
            box = (tuple(prefix[:-1]), prefix[-1], prefix[-1])
        t0 = time.perf_counter()
        rows = oracle.run(n, g, box=box)["count"]
        dt = time.perf_counter() - t0
        num += rows / wi
        den += dt / wi
        rows_tot += rows
        secs_tot += dt
        boxes += 1
    return (num / den if den else 0.0), rows_tot, secs_tot, boxes


def cpu_info() -> dict:
    """Host CPU model and core count (the oracle baseline runs on one pinned core)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


class pinned_core:
    """Run the oracle on ONE host core (`taskset -c 0` equivalent); restores the
    previous affinity afterwards."""

    def __init__(self, core: int = 0):
        self.core = core
        self.prev = None

    def __enter__(self):
        try:
            self.prev = os.sched_getaffinity(0)
            core = self.core if self.core in self.prev else min(self.prev)
            os.sched_setaffinity(0, {core})
            self.core = core
        except (AttributeError, OSError):
            self.prev = None
        return self

    def __exit__(self, *exc):
        if self.prev is not None:
            os.sched_setaffinity(0, self.prev)


def base_config(inst, total: int, world: int) -> dict:
    """The workload keys both arms report (fsgpu and --impl reference), identical in both."""
    return {"workload": "%s: Z(%d, %s) count, |Z| = %d" % (inst.name, inst.n, list(inst.gens), total),
            "instance": inst.name, "n": inst.n, "gens": list(inst.gens), "consumer": "count",
            "parallelism": "lex-slice dp%d" % world,
            "l2": "flushed between steps (256 MB write)"}


def run_reference(args, inst):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    per_step = max(1.0, float(os.environ.get("FS_REF_STEP_SECONDS", "6")))
    vals = []
    tot_rows, tot_s = 0, 0.0
    with pinned_core(0) as pc:
        for _ in range(args.warmup):
            oracle_sample(inst, min(per_step, 2.0), seed=1)
        for k in range(args.steps):
            rate, rows, secs, boxes = oracle_sample(inst, per_step, seed=100 + k)
            vals.append(rate)
            tot_rows += rows
            tot_s += secs
    value = statistics.mean(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic", "config": base_config(inst, __import__("oracle").gf.count(inst.n, inst.gens), args.gpus),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "pinned_core": pc.core,
                         **cpu_info(),
                         "sample": "work-weighted prefix boxes of %s, seeds 100..%d, %.0f s per step, "
                                   "%d rows total, ratio estimator" % (inst.name, 99 + args.steps, per_step,
                                                                        tot_rows)},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fsgpu", choices=["fsgpu", "reference"])
    ap.add_argument("--workload", default="c3count", choices=["c3count", "c5count", "c2count"])
    ap.add_argument("--no-extra", action="store_true", help="skip the store/hist extra measurements")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    inst = {"c3count": W.C3, "c5count": W.C5, "c2count": W.C2}[args.workload]
    if args.impl == "reference":
        return run_reference(args, inst)

    import torch
    import torch.distributed as dist

    from paper_2405_07989_b200 import _lib as L
    from paper_2405_07989_b200 import api
    from paper_2405_07989_b200 import dist as fsdist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # one process per GPU; FS_DIST_BACKEND=gloo lets the multi-rank path run on a 1-GPU box
    # (ranks then share devices round-robin) for testing -- numbers from it are not scaling data
    backend = os.environ.get("FS_DIST_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            # the communicator's init line (rank / nranks) goes to stderr, so the rank count of
            # the run can be checked from the log
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        print("[bench] rank %d/%d backend=%s device=cuda:%d" % (rank, world, dist.get_backend(), local),
              file=sys.stderr, flush=True)
    stream = torch.cuda.current_stream()
    peaks, peaks_kind = load_peaks()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        fsdist.combine_max(t)
        return float(t.item())

    # ---- plan: constants + DP tables resident in HBM before the timed region
    # the configuration fs_count() runs: generators largest-first (NEXT-2) and the closed-form
    # tail (NEXT-1); the literal per-row stream over the given order is reported in extra
    headline = {"gen_order": L.FS_GENORDER_AUTO, "tail": L.FS_TAIL_CLOSED}
    plan = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_COUNT, device=local, stream=stream.cuda_stream,
                    rank=rank, world=world, **headline)
    info = plan.info
    out = torch.zeros(1, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    def step():
        plan.count_async(out)
        fsdist.combine_sum(out)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    assert int(out.item()) == info["total_rows"], ("count mismatch", int(out.item()), info["total_rows"])

    sampler = ClockSampler(local)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = L.lib().fsdbg_total_launches()
    barrier()
    sampler.start()
    time.sleep(0.3)
    for k in range(args.steps):
        flush.zero_()  # L2 flush between steps (outside the step events)
        ev[k][0].record(stream)
        kev[k][0].record(stream)
        plan.count_async(out)
        kev[k][1].record(stream)
        fsdist.combine_sum(out)  # NCCL all_reduce on the stream (gloo: staged through the host)
        ev[k][1].record(stream)
    barrier()
    clocks = sampler.stop()
    launches = L.lib().fsdbg_total_launches() - launches0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    kern_ms = [a.elapsed_time(b) for a, b in kev]
    ms_step = max_over_ranks(sum(step_ms) / len(step_ms))
    ms_kern = max_over_ranks(sum(kern_ms) / len(kern_ms))
    total = int(out.item())
    assert total == info["total_rows"]
    value = total / (ms_step / 1e3)

    # roofline of the dominant kernel (count): INT32 issue.  Denominator: the best measured
    # INT32 microbenchmark rate on this GPU (csrc/fs_micro.cu); the derived issue limit
    # (128 lane-ops/clk/SM x 148 x sm max clock) is reported beside it.
    sm_max = float((clocks or {}).get("sm_max_mhz") or peaks.get("sm_max_mhz", 1965.0))
    derived_tops = INT_LANES_PER_CLK_PER_SM * NUM_SMS * sm_max * 1e6 / 1e12
    mb = microbench() if rank == 0 or world > 1 else None
    measured_tops = max(v["tops"] for k, v in mb.items() if isinstance(v, dict)) if mb else None
    peak_tops = measured_tops or derived_tops
    share = (info["unit_end"] - info["unit_begin"]) / max(1, info["total_units"])
    ops = ops_model(info, closed=True) * share
    achieved = ops / (ms_kern / 1e3) / 1e12
    traffic = _traffic(args.workload)

    rank_units = [[info["unit_begin"], info["unit_end"]]]
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, rank_units[0])
        rank_units = allr
    cands = paper_candidates(inst, skip_paper=True)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": base_config(inst, total, world),
        "plan": {"method": "Alg. 3.1 stream over the generators largest-first (gen_order=auto, NEXT-2), "
                           "modulo skip at run entry, closed-form row count per node (tail=closed, NEXT-1)",
                 "nodes": info["nodes_per_level"][-1], "nodes_per_level": info["nodes_per_level"],
                 "dist_backend": (dist.get_backend() if world > 1 else None),
                 "slice_units": info["slice_units"], "num_slices": info["num_slices"],
                 "grid": plan.info["grid"], "block": info["block"], "rank_units": rank_units},
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_tops, "unit": "Tops/s (int32 lane-ops)",
                     "frac": achieved / peak_tops, "traffic": traffic,
                     "peak_source": ("measured: best INT32 microbenchmark (fs_micro.cu)" if measured_tops else
                                     "derived: 128 int lane-ops/clk/SM x 148 SMs x %.0f MHz" % sm_max),
                     "derived_issue_peak": derived_tops, "frac_of_derived": achieved / derived_tops,
                     "ops_per_launch": ops, "ops_model": OPS_MODEL_DOC, "kernel_ms": ms_kern,
                     # (the counters are for the whole one-GPU launch)
                     "executed": _executed(args.workload, ms_kern, peak_tops, derived_tops) if world == 1 else None},
        "gpu_launches": int(launches),
        "microbench": mb,
        "clocks": clocks,
        # the paper's own stream (Alg. 3.1 with its modulo skip) visits
        # `cands` candidates on this instance (exact DP count); the kernel skips most of them
        "cand_per_s": {"value": cands / (ms_step / 1e3), "candidates": cands,
                       "stream": "Alg. 3.1 with the paper's modulo skip (Skip=paper), exact DP count"},
    }

    # ---- e2e: through the public API with host buffers (DP + H2D + kernel + D2H per step)
    e2e_t = []
    for k in range(max(2, min(args.steps, 3))):
        barrier()
        t0 = time.perf_counter()
        if world > 1:
            c = fsdist.count(inst.n, inst.gens)
        else:
            c = api.fs_count(inst.n, inst.gens)
        torch.cuda.synchronize()
        e2e_t.append(max_over_ranks(time.perf_counter() - t0))
        assert c == total
    e2e_s = statistics.median(e2e_t)
    line["e2e"] = {"value": total / e2e_s, "unit": UNIT, "h2d_bytes_per_step": int(info["table_bytes"]),
                   "d2h_bytes_per_step": 8, "seconds": e2e_s}

    # ---- extras (same run): store (materialise C2-XL) and C4 length histogram; the rooflines
    # of the other consumers' kernels are nested in `roofline` (hist, any, store, store_any, ..)
    if not args.no_extra:
        ex = extras(args, world, rank, local, dev, stream, peaks, peaks_kind, barrier, max_over_ranks, mb)
        line["extra"] = ex
        for rk, ek in (("hist", "hist_auto_order_closed"), ("any", "c5_any_P_none_auto_order_closed"),
                       ("store", "store"), ("store_any", "store_any"), ("store_increasing", "store_increasing")):
            if ek in ex and isinstance(ex[ek], dict) and "roofline" in ex[ek]:
                line["roofline"][rk] = {**ex[ek]["roofline"], "ms": ex[ek].get("ms"),
                                        "workload": ex[ek].get("workload"), "extra_key": ek}

    # ---- CPU oracle beside it (rank 0, N = 1 only)
    if world == 1 and args.cpu_seconds > 0:
        with pinned_core(0) as pc:
            rate, rows, secs, boxes = oracle_sample(inst, args.cpu_seconds)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": 1, "kind": "oracle", "pinned_core": pc.core,
                                **cpu_info(),
                                "sample": "%d work-weighted prefix boxes of %s (seed 0): %d rows in %.1f s, "
                                          "1 thread pinned to one core, ratio estimator" % (boxes, inst.name, rows,
                                                                                          secs)}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _time_ms(fn, stream, reps, barrier, max_over_ranks):
    import torch

    ts = []
    barrier()
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return max_over_ranks(statistics.median(ts))


def _executed(key, ms, peak_tops, issue_tops):
    """Executed lane-instructions per launch of the same build (profiles/counters.json, from one
    `ncu --set full` capture: sm__sass_thread_inst_executed_op_integer_pred_on.sum and all
    sass thread instructions) over the kernel time measured here: the counter-based INT32 and
    issue fractions beside the algorithmic one."""
    prof = os.path.join(ROOT, "profiles", "counters.json")
    try:
        c = json.load(open(prof)).get(key)
    except Exception:
        c = None
    if not c or not ms:
        return None
    s = ms / 1e3
    return {"integer_lane_inst": c["integer_lane_inst"], "lane_inst": c["lane_inst"], "source": c["source"],
            "int_tops": c["integer_lane_inst"] / s / 1e12, "frac_int": c["integer_lane_inst"] / s / 1e12 / peak_tops,
            "frac_int_of_issue_peak": c["integer_lane_inst"] / s / 1e12 / issue_tops,
            "frac_all": c["lane_inst"] / s / 1e12 / peak_tops,
            "frac_all_of_issue_peak": c["lane_inst"] / s / 1e12 / issue_tops}


def _traffic(key):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the kernel, from one
    `ncu --set full` capture (profiles/traffic.json, written from the committed summaries)."""
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(prof)).get(key)
    except Exception:
        return None


def extras(args, world, rank, local, dev, stream, peaks, peaks_kind, barrier, max_over_ranks, mb):
    """Same-run measurements of the other hot-path consumers (each on its BASELINE config)."""
    import torch
    import torch.distributed as dist

    from paper_2405_07989_b200 import _lib as L
    from paper_2405_07989_b200 import api

    ex = {}
    kw = dict(device=local, stream=stream.cuda_stream, rank=rank, world=world)

    def allreduce(t, op=None):
        if world > 1:
            dist.all_reduce(t, op=op or dist.ReduceOp.SUM)

    # ---- store: C2-XL rows, u16; canonical layout (M1) and warp-compacted layout (M2)
    inst = W.C2XL
    store_out = None  # one output buffer, reused by the three layouts (as a caller would)
    # batch kernel (default, lockstep register batches) and the round-1 staged kernels
    for order, key, go, impl in ((L.FS_ORDER_CANONICAL, "store", 0, L.FS_ROWS_BATCH),
                                 (L.FS_ORDER_ANY, "store_any", 0, L.FS_ROWS_BATCH),
                                 (L.FS_ORDER_INCREASING, "store_increasing", 0, L.FS_ROWS_BATCH),
                                 (L.FS_ORDER_CANONICAL, "store_staged", 0, L.FS_ROWS_STAGED),
                                 (L.FS_ORDER_ANY, "store_any_staged_auto_order", L.FS_GENORDER_AUTO,
                                  L.FS_ROWS_STAGED)):
        p = api.Plan(inst.n, inst.gens, L.FS_CONSUMER_ROWS, order=order, gen_order=go, rows_impl=impl, **kw)
        info = p.info
        rows = info["row_end"] - info["row_begin"]
        if store_out is None or store_out.shape[0] < rows:
            store_out = None
            torch.cuda.empty_cache()
            store_out = torch.empty((rows, inst.d), dtype=torch.uint16, device=dev)
        out = store_out[:rows]
        p.enumerate_async(16, out, rows)
        p.rows_check()  # order = any: the M2 cursors met exactly (every row written once)
        ms = _time_ms(lambda: p.enumerate_async(16, out, rows), stream, 5, barrier, max_over_ranks)
        p.rows_check()
        total_rows = info["total_rows"]
        bytes_ = total_rows * inst.d * 2
        gbs_all = bytes_ / (ms / 1e3) / 1e9
        peak = peaks["hbm_gbs"] * world
        ex[key] = {"workload": "C2XL: Z(16000, (11,13,17,19,23)) materialise u16 rows, %s order%s"
                               % ({0: "canonical (exact offsets)", 1: "any (warp compaction)",
                                   2: "increasing lex (mirrored exact offsets)"}[order],
                                  ", NEXT-2 generator order" if go else ""),
                   "kernel": "batch (lockstep register batches)" if impl == L.FS_ROWS_BATCH
                   else "staged (round-1 per-step emission)",
                   "rows": total_rows, "bytes": bytes_, "ms": ms, "value": total_rows / (ms / 1e3), "unit": UNIT,
                   "roofline": {"bound": "hbm", "achieved": gbs_all, "peak": peak, "unit": "GB/s",
                                "frac": gbs_all / peak, "traffic": _traffic(key),
                                "peak_source": "MEASURED_PEAKS.json hbm_gbs x %d (%s, copy r+w)" % (world, peaks_kind),
                                "frac_of_write_microbench": (gbs_all / world / mb["hbm_write_gbs"]) if mb else None}}
        del out
    # common-divisor skip (NEXT-3): a non-coprime last pair; the batch kernel jumps over the
    # level-L nodes without factorizations, the staged kernel steps through them
    try:
        icd = W.C2CD
        for key, impl in (("store_cd", L.FS_ROWS_BATCH), ("store_cd_staged", L.FS_ROWS_STAGED)):
            p = api.Plan(icd.n, icd.gens, L.FS_CONSUMER_ROWS, rows_impl=impl, **kw)
            inf = p.info
            rows = inf["row_end"] - inf["row_begin"]
            out = store_out.view(-1)[: rows * icd.d].view(rows, icd.d)
            p.enumerate_async(16, out, rows)
            ms = _time_ms(lambda: p.enumerate_async(16, out, rows), stream, 3, barrier, max_over_ranks)
            gbs = inf["total_rows"] * icd.d * 2 / (ms / 1e3) / 1e9
            ex[key] = {"workload": "C2CD: Z(12000, (11,13,17,18,24)) materialise u16 rows, canonical order, %s kernel"
                                   % ("batch (dead-node skip)" if impl == L.FS_ROWS_BATCH else "staged"),
                       "rows": inf["total_rows"], "ms": ms, "value": inf["total_rows"] / (ms / 1e3), "unit": UNIT,
                       "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"] * world, "unit": "GB/s",
                                    "frac": gbs / (peaks["hbm_gbs"] * world)}}
    except Exception as e:
        ex["store_cd"] = {"error": repr(e)}
    # filtered materialise (NEXT-4): rows of one length class, two passes (count, write) through
    # the synchronous C-ABI call -- timed with CUDA events around the whole call (plan creation
    # on the host and both passes included)
    try:
        X = 1056  # a populated length class of C2-XL (lengths 688..1454)
        m_cnt, _ = api.fs_enumerate_filtered(inst.n, inst.gens, L.FS_PRED_LEN_EQ, X, B=16, cap=0, device=local,
                                             rank=rank, world=world)
        fout = store_out[:max(1, m_cnt)]
        def filt():
            api.fs_enumerate_filtered(inst.n, inst.gens, L.FS_PRED_LEN_EQ, X, B=16, cap=m_cnt, out=fout,
                                      device=local, rank=rank, world=world)
        ms = _time_ms(filt, stream, 3, barrier, max_over_ranks)
        ex["store_filtered"] = {"workload": "C2XL: rows of Z(16000, (11,13,17,19,23)) with a_1+..+a_5 = %d, u16, "
                                            "any order (count pass + write pass)" % X,
                                "matching_rows": m_cnt, "scanned_rows": info["total_rows"], "ms": ms,
                                "value": info["total_rows"] / (ms / 1e3), "unit": "scanned factorizations/s"}
    except Exception as e:  # an extra: report, do not fail the bench line
        ex["store_filtered"] = {"error": repr(e)}
    del store_out
    torch.cuda.empty_cache()

    # ---- count / hist / any on their configs; NEXT-1 (closed tail) and NEXT-2 (generator
    # order) variants of SURVEY 8(f) are labelled and reported beside the literal path
    c = torch.zeros(1, dtype=torch.int64, device=dev)
    f = torch.zeros(1, dtype=torch.int32, device=dev)
    w = torch.zeros(16, dtype=torch.int32, device=dev)
    AUTO = L.FS_GENORDER_AUTO
    runs = [
        ("count_literal", W.C3, L.FS_CONSUMER_COUNT, {}, "C3 count, given order, one step per row", 3),
        ("hist", W.C4, L.FS_CONSUMER_HIST, {}, "C4 length histogram (329 bins), given order", 2),
        ("hist_auto_order", W.C4, L.FS_CONSUMER_HIST, {"gen_order": AUTO}, "C4 histogram, NEXT-2 order", 2),
        ("hist_auto_order_closed", W.C4, L.FS_CONSUMER_HIST, {"gen_order": AUTO, "tail": 1},
         "C4 histogram, NEXT-1 + NEXT-2 (fs_length_set default)", 3),
        ("hist_auto_order_closed_residue", W.C4, L.FS_CONSUMER_HIST, {"gen_order": AUTO, "tail": 1, "walk": 1},
         "C4 histogram, NEXT-1 + NEXT-2, residue-form walk (ablation of the state form)", 2),
        ("count_auto_order_closed_residue", W.C3, L.FS_CONSUMER_COUNT, {"gen_order": AUTO, "tail": 1, "walk": 1},
         "C3 count, NEXT-1 + NEXT-2, residue-form walk (ablation of the state form)", 2),
        ("count_closed_tail", W.C3, L.FS_CONSUMER_COUNT, {"tail": 1}, "C3 count, NEXT-1 closed tail", 3),
        ("count_auto_order", W.C3, L.FS_CONSUMER_COUNT, {"gen_order": AUTO}, "C3 count, NEXT-2 order", 3),
        ("count_auto_order_closed", W.C3, L.FS_CONSUMER_COUNT, {"gen_order": AUTO, "tail": 1},
         "C3 count, NEXT-1 + NEXT-2", 3),
        ("c5_count", W.C5, L.FS_CONSUMER_COUNT, {}, "C5 count, given order", 1),
        ("c2cd_count_closed", W.C2CD, L.FS_CONSUMER_COUNT, {"tail": 1},
         "C2CD count, given order (gcd(18, 24) = 6: the closed tail walks live nodes only, NEXT-3)", 3),
        ("c2cd_count_rows", W.C2CD, L.FS_CONSUMER_COUNT, {},
         "C2CD count, given order, one step per row (no skip)", 3),
        ("c2cd_hist_closed", W.C2CD, L.FS_CONSUMER_HIST, {"tail": 1},
         "C2CD histogram, given order, closed tail over the live-node table (NEXT-3)", 3),
        ("c3cd_count_closed", W.C3CD, L.FS_CONSUMER_COUNT, {"tail": 1},
         "C3CD count (gcd(12, 18, 24) = 6), closed tail + dead-run skip in the ascend (NEXT-3, k = 3)", 3),
        ("c3cd_count_closed_noskip", W.C3CD, L.FS_CONSUMER_COUNT, {"tail": 1, "walk": 1},
         "C3CD count, closed tail, residue walk without the k >= 3 dead-subtree skip (ablation)", 3),
        ("c3cd_hist_closed", W.C3CD, L.FS_CONSUMER_HIST, {"tail": 1},
         "C3CD histogram, closed tail, live-node table + dead-run skip (NEXT-3)", 3),
        # E2 (Table 1 modulo on/off) re-run on B200: the index-(d-1) loop variants
        ("c2l_skip_off", W.C2L, L.FS_CONSUMER_COUNT, {"tail": 2}, "C2-L count, Skip=off (every candidate)", 2),
        ("c2l_skip_paper", W.C2L, L.FS_CONSUMER_COUNT, {"tail": 3}, "C2-L count, Skip=paper (P:170-176)", 2),
        ("c2l_skip_full", W.C2L, L.FS_CONSUMER_COUNT, {}, "C2-L count, Skip at run entry (rows)", 2),
        ("c2l_closed", W.C2L, L.FS_CONSUMER_COUNT, {"tail": 1}, "C2-L count, closed tail", 2),
        ("c5_count_auto_order", W.C5, L.FS_CONSUMER_COUNT, {"gen_order": AUTO}, "C5 count, NEXT-2 order", 3),
    ]
    for key, inst, cons, pk, label, reps in runs:
        p = api.Plan(inst.n, inst.gens, cons, **pk, **kw)
        if cons == L.FS_CONSUMER_HIST:
            h = torch.zeros(api.hist_len(inst.n, inst.gens), dtype=torch.int64, device=dev)

            def fn():
                p.hist_async(h)
                allreduce(h)
        else:
            def fn():
                p.count_async(c)
                allreduce(c)
        fn()
        ms = _time_ms(fn, stream, reps, barrier, max_over_ranks)
        total = int(h.sum().item()) if cons == L.FS_CONSUMER_HIST else int(c.item())
        assert total == p.info["total_rows"], (key, total)
        ex[key] = {"workload": "%s: Z(%d, %s)" % (label, inst.n, list(inst.gens)), "rows": total, "ms": ms,
                   "value": total / (ms / 1e3), "unit": UNIT,
                   "nodes": p.info["nodes_per_level"][-1]}
        pi = p.info
        sh = (pi["unit_end"] - pi["unit_begin"]) / max(1, pi["total_units"])
        tail = pk.get("tail", 0)
        if tail in (L.FS_TAIL_SKIP_OFF, L.FS_TAIL_SKIP_PAPER):  # the paper's candidate loop
            cands = paper_candidates(inst, tail == L.FS_TAIL_SKIP_PAPER)
            ex[key]["candidates"] = cands
            ex[key]["cand_per_s"] = cands * sh / (ms / 1e3)
        if mb and cons in (L.FS_CONSUMER_COUNT, L.FS_CONSUMER_HIST):
            if tail in (L.FS_TAIL_SKIP_OFF, L.FS_TAIL_SKIP_PAPER):
                ops = OPS_CAND * ex[key]["candidates"] + ops_model(pi, closed=True) - 3 * pi["nodes_per_level"][-1]
            elif cons == L.FS_CONSUMER_HIST:
                ops = ops_model(pi, closed=tail == 1, hist=True)
            else:
                ops = ops_model(pi, closed=tail == 1)
            ach = ops * sh / (ms / 1e3) / 1e12
            pk_tops = max(v["tops"] for v in mb.values() if isinstance(v, dict))
            ex[key]["roofline"] = {"bound": "alu", "achieved": ach, "peak": pk_tops, "unit": "Tops/s (int32 lane-ops)",
                                   "frac": ach / pk_tops, "ops_per_launch": ops * sh,
                                   "traffic": _traffic(key)}
    for order_name, pk in (("", {}), ("_auto_order", {"gen_order": AUTO}),
                           ("_auto_order_closed", {"gen_order": AUTO, "tail": L.FS_TAIL_CLOSED})):
        pa = api.Plan(W.C5.n, W.C5.gens, L.FS_CONSUMER_ANY, **pk, **kw)
        for name, pred, arg in (("P_late", L.FS_PRED_LEN_LE, 20), ("P_none", L.FS_PRED_LEN_LE, 19),
                                ("P_first", L.FS_PRED_LEN_GE, 19995)):
            def any_step():
                pa.any_async(pred, arg, f, w)
                allreduce(f, dist.ReduceOp.MAX if world > 1 else None)

            ms = _time_ms(any_step, stream, 3, barrier, max_over_ranks)
            ek = "c5_any_%s%s" % (name, order_name)
            ex[ek] = {"pred": [pred, arg], "found": bool(f.item()), "ms": ms}
            if name == "P_none" and pk.get("tail") == L.FS_TAIL_CLOSED and mb:
                # no witness: the whole stream is scanned, one closed-form test per node
                pi = pa.info
                sh = (pi["unit_end"] - pi["unit_begin"]) / max(1, pi["total_units"])
                ops = ops_model(pi, closed=True, any_=True) * sh
                pk_tops = max(v["tops"] for v in mb.values() if isinstance(v, dict))
                ach = ops / (ms / 1e3) / 1e12
                ex[ek]["workload"] = "C5 any-predicate sum(a) <= 19 (no witness: full scan), NEXT-1 + NEXT-2"
                ex[ek]["roofline"] = {"bound": "alu", "achieved": ach, "peak": pk_tops, "unit": "Tops/s (int32 lane-ops)",
                                      "frac": ach / pk_tops, "ops_per_launch": ops, "nodes": pi["nodes_per_level"][-1],
                                      "traffic": _traffic(ek)}
    return ex


if __name__ == "__main__":
    sys.exit(main())
