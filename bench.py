#!/usr/bin/env python3
"""Benchmark of the batched leaf expansion (BASELINE.json metric:
scenario-steps/s and ms per leaf-expansion batch, vs the CPU oracle).

One step = one despot_expand_batch over the config's leaves (update K1,
expansion + bounds + roll-outs + grouping K2, child order / CSR / outputs K3)
with the node arenas resident in HBM.  Default workload: BASELINE config 2
(multi-agent RockSample(15,15), 2 robots, K=500, 64 depth-1 leaves).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl despot|reference]

N > 1 (torchrun, one rank per GPU): the same workload scenario-sharded
(global id % N), with one NCCL all-reduce of the exact int64 partials per
batch (strong scaling).  Timing: CUDA events per step on the launching
stream, barrier + synchronize around the timed region, max over ranks; L2 is
flushed (a 256 MiB write) between timed steps, outside the events.  The
dominant kernel's live duration (roofline) comes from the library's own K2
events (DESPOT_X_TIMING_K2) in a second pass of the same steps, so the
throughput pass carries no per-call event overhead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1802_06215_b200 import inputs  # noqa: E402

# Algorithmic work per scenario-step (thread-instructions), SURVEY.md §8(d)
# "Algorithmic work per scenario-step": RockSample ~125, MARS ~175,
# navigation ~300, driving (20 pedestrians) ~1,300.  The roofline's
# `achieved` uses these fixed per-unit figures (not the kernel's own
# instruction count, which would credit overhead instructions); the measured
# count of the kernel as built is reported beside it (i_step_measured).
I_STEP_ALGO = {1: 125.0, 2: 175.0, 3: 300.0, 4: 1300.0, 5: 175.0}


def i_step(config):
    """(algorithmic thread-instructions per scenario-step, source)"""
    return I_STEP_ALGO[config], "SURVEY.md §8(d) per-unit figure"


def i_step_measured(config):
    """thread-instructions per scenario-step of K2 as built (ncu
    smsp__thread_inst_executed.sum / scenario-steps, scripts/measure_istep.py),
    newest round first; None if never measured"""
    for rnd in ("r02", "r01"):
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "i_step.json")) as f:
                return float(json.load(f)[str(config)]["i_step"]), f"profiles/{rnd}/i_step.json"
        except Exception:
            continue
    return None, None


def _profile_file(name):
    """newest committed profile file of that name (profiles/r02, else r01)"""
    for rnd in ("r02", "r01"):
        p = os.path.join(ROOT, "profiles", rnd, name)
        if os.path.exists(p):
            return p
    return os.path.join(ROOT, "profiles", "r01", name)


def ncu_traffic(config):
    """dram__bytes_read.sum + dram__bytes_write.sum of the dominant kernel,
    per launch, from the committed `ncu --set full` raw page of this config
    (profiles/r01/k2_config<C>_raw.csv); None if there is none."""
    import csv
    p = _profile_file(f"k2_config{config}_raw.csv")
    try:
        rows = list(csv.reader(open(p)))
        scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        tot = 0.0
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            i = rows[0].index(name)
            tot += float(rows[2][i].replace(",", "")) * scale[rows[1][i]]
        return {"bytes_per_launch": tot, "source": os.path.relpath(p, ROOT)}
    except Exception:
        return None


NCU_K2_METRICS = {
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "lanes_per_warp_instr": "smsp__thread_inst_executed_per_inst_executed.ratio",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
}


def ncu_k2_summary(config):
    """The per-pipe picture of the dominant kernel from the same committed
    `ncu --set full` raw page as `traffic` (SURVEY §8(d) metric list)."""
    import csv
    p = _profile_file(f"k2_config{config}_raw.csv")
    try:
        rows = list(csv.reader(open(p)))
        out = {}
        for k, name in NCU_K2_METRICS.items():
            out[k] = float(rows[2][rows[0].index(name)].replace(",", ""))
        out["source"] = os.path.relpath(p, ROOT)
        return out
    except Exception:
        return None


# Philox4x32-10 blocks drawn per scenario-step (DESIGN.md §3 model cards)
def philox_blocks_per_step(kind, peds):
    return {"tiger": 1, "rocksample": 1, "nav": 3}.get(kind, (peds + 1 + 3) // 4)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return json.load(f), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons, sampled every 20 ms from before
    the warm-up; summary() keeps the samples of the timed window (+-100 ms)."""

    def __init__(self, gpu_index=0):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.monotonic(), [x.strip() for x in line.split(",")]))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self, t0, t1):
        rows = [r for (t, r) in self.rows if t0 - 0.1 <= t <= t1 + 0.1]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        num = lambda v: v.replace(".", "").isdigit()  # noqa: E731
        sm = [float(r[0]) for r in rows if num(r[0])]
        mx = [float(r[1]) for r in rows if len(r) > 1 and num(r[1])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for i, n in enumerate(names):
                if len(r) > 4 + i and r[4 + i].lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(rows)}


def workload(cfg, K=None, peds=None):
    c = dict(inputs.CONFIGS[cfg])
    kind, params, st, w, seed, L = inputs.config_inputs(cfg, K=K, peds=peds)
    if peds is not None and kind == "car":
        c["name"] = f"car_{peds}peds_K{len(w)}_L{L}"
        c["peds"] = peds
    return c, kind, params, st, w, seed, L


def make_leaves(model, root, L, cfg_kind, extra_roots=None):
    """Depth-1 leaves from the root expansion (SURVEY §8(d) generator)."""
    R = model.expand([(root, -1, 0, 0)])
    lv = inputs.select_leaves(R["child_count"], R["child_begin"], model.A, L)
    return [(root, a, c, 1) for a, c in lv]


def host_cpu_info():
    """CPU model, sockets, physical cores and SMT of this host (/proc/cpuinfo),
    and the cores this process may use (the oracle's host)."""
    model, phys, cores_per, siblings = None, set(), None, None
    try:
        for line in open("/proc/cpuinfo"):
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k == "model name" and model is None:
                model = v
            elif k == "physical id":
                phys.add(v)
            elif k == "cpu cores" and cores_per is None:
                cores_per = int(v)
            elif k == "siblings" and siblings is None:
                siblings = int(v)
    except Exception:
        pass
    sockets = max(1, len(phys))
    smt = (siblings // cores_per) if (siblings and cores_per) else None
    return {"cpu_model": model, "sockets": sockets, "physical_cores": (cores_per * sockets) if cores_per else None,
            "threads_per_core": smt, "logical_cpus": os.cpu_count(), "usable_cpus": len(os.sched_getaffinity(0))}


def cpu_baseline(kind, params, st, w, seed, leaves_ac, budget_s=12.0, L=64, peds=20):
    """The oracle as it stands (single thread) on a bounded sample of the
    same workload: leaves expanded one at a time until ~budget_s of work."""
    import oracle

    om = oracle.Model(kind, params)
    if kind == "car":
        croots = inputs.car_roots(L, int(len(w)), peds=peds)
        items = [("root", j) for j in range(L)]
    else:
        root = om.belief_load(st, w, seed)
        om.expand([(root, -1, 0, 0)])
        items = leaves_ac
    steps = 0
    t0 = time.perf_counter()
    n = 0
    while True:  # the batch's leaves in order, cycling (small batches), until ~budget_s
        (a, c) = items[n % len(items)]
        if kind == "car":  # a self leaf: the root node itself is expanded
            r = om.belief_load(*croots[c])
            o = om.expand([(r, -1, 0, 0)])
            om.node_release(r)
        else:
            o = om.expand([(root, -1, 0, 0) if a < 0 else (root, a, c, 1)])
            if a >= 0:  # the new child node (long runs would otherwise hold every one)
                om.node_release(int(o["node"][0]))
        steps += o["scenario_steps"]
        n += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": steps / dt, "unit": "scenario-steps/s", "cores": 1, "kind": "oracle",
            "sample": f"{n} leaf expansions (all |A| actions each) over the batch's {len(items)} leaves "
                      f"({n / len(items):.2f} passes), {steps} scenario-steps in {dt:.1f} s",
            "host": host_cpu_info()}


def _oracle_share(job):
    """one process of the all-cores oracle baseline: expand its share of the
    leaves (every nproc-th) until the budget is spent"""
    kind, params, st, w, seed, leaves_ac, budget_s, L, peds, rank, nproc = job
    import oracle

    om = oracle.Model(kind, params)
    if kind == "car":
        croots = inputs.car_roots(L, int(len(w)), peds=peds)
        items = [("root", j) for j in range(L)][rank::nproc]
    else:
        root = om.belief_load(st, w, seed)
        om.expand([(root, -1, 0, 0)])
        items = leaves_ac[rank::nproc]
    steps, n = 0, 0
    t0 = time.perf_counter()
    while True:
        for (a, c) in items:
            if kind == "car":
                o = om.expand([(om.belief_load(*croots[c]), -1, 0, 0)])
            else:
                o = om.expand([(root, -1, 0, 0) if a < 0 else (root, a, c, 1)])
            steps += o["scenario_steps"]
            n += 1
            if time.perf_counter() - t0 > budget_s:
                return steps, time.perf_counter() - t0, n
        if not items:
            return 0, time.perf_counter() - t0, 0


def cpu_baseline_all_cores(kind, params, st, w, seed, leaves_ac, budget_s=8.0, L=64, peds=20):
    """The same oracle in one process per host core (independent leaves)."""
    import multiprocessing as mp

    nproc = len(os.sched_getaffinity(0))
    jobs = [(kind, params, st, w, seed, leaves_ac, budget_s, L, peds, r, nproc) for r in range(nproc)]
    with mp.get_context("fork").Pool(nproc) as pool:
        res = pool.map(_oracle_share, jobs)
    steps = sum(r[0] for r in res)
    secs = max(r[1] for r in res)
    return {"value": steps / secs, "unit": "scenario-steps/s", "cores": nproc, "kind": "oracle",
            "sample": f"{sum(r[2] for r in res)} leaf expansions in {nproc} processes, {steps} scenario-steps, "
                      f"{secs:.1f} s",
            "host": host_cpu_info()}


def run_plan(args):
    """--plan: tree size per planning time (the paper's speedup metric, P:566;
    SURVEY §8(f) NEXT-1/2) of the host tree driver (despot_plan) on the GPU
    backend vs the same driver on the CPU oracle backend with one worker (the
    serial DESPOT analog: this mode's cpu_baseline leg).  One JSON line per
    run, then the speedups.  Studies: "configs" (the BASELINE configs), "K"
    (navigation, K = 100 ... 5000), "A" (MARS |A| = 256/400/625,
    P:625-627)."""
    from paper_1802_06215_b200 import despot as D

    sys.path.insert(0, os.path.join(ROOT, "tests"))
    points = []
    if args.plan_study == "configs":
        for cfg in args.plan_configs:
            kind, params, st, w, seed, _ = inputs.config_inputs(cfg, K=args.K)
            points.append((f"config{cfg}", cfg, kind, params, st, w, seed))
    elif args.plan_study == "K":
        for K in args.plan_K:
            kind, params, st, w, seed, _ = inputs.config_inputs(3, K=K)
            points.append(("K_nav13", K, kind, params, st, w, seed))
    else:
        for n, m in ((11, 11), (15, 15), (20, 20)):  # |A| = (5 + m)^2 = 256, 400, 625
            params = inputs.rocksample_params(n, m, 2, D=20)
            K = args.K or 500
            points.append(("A_mars", f"MARS({n},{n}) |A|={(5 + m) ** 2}", "rocksample", params,
                           inputs.rocksample_belief(n, m, 2, K, 1002), inputs.weights(K), 1002))
    for study, point, kind, params, st, w, seed in points:
        rows = []
        gm = D.Model(kind, params)
        root = gm.belief_load(st, w, seed)
        for W in args.plan_workers:
            c = D.search_config(workers=W, max_inflight=8 if W > 1 else 1, max_batch=64, batch_wait_us=300,
                                time_budget_s=args.plan_budget, xi=0.95, c_a=0.3, c_o=0.1)
            r = gm.plan(root, c)
            r.update(study=study, point=point, backend="gpu", workers=W, K=len(w), A=gm.A,
                     nodes_per_s=r["nodes"] / r["seconds"], leaves_per_batch=r["expanded"] / max(1, r["batches"]))
            rows.append(r)
            print(json.dumps(r), flush=True)
        gm.close()
        if args.no_cpu_baseline:
            continue
        import oracle
        from test_search_cpu import OracleBackend
        om = oracle.Model(kind, params)
        orr = om.belief_load(st, w, seed)
        u0, l0 = om.rollout_bounds(orr)
        be = OracleBackend(om)
        c = D.search_config(workers=1, max_inflight=1, max_batch=1, time_budget_s=args.plan_budget, xi=0.95,
                            c_a=0.3, c_o=0.1)
        r, _ = D.search(be.problem(orr, u0, l0, K=len(w)), c)
        r.update(study=study, point=point, backend="oracle-serial", workers=1, K=len(w), A=om.A,
                 nodes_per_s=r["nodes"] / r["seconds"], cores=1)
        print(json.dumps(r), flush=True)
        for g in rows:
            print(json.dumps({"study": study, "point": point, "workers": g["workers"],
                              "speedup_tree_size_per_time": g["nodes_per_s"] / r["nodes_per_s"],
                              "gpu_max_depth": g["max_depth"], "oracle_max_depth": r["max_depth"]}), flush=True)
    return 0


_REF = {}


def _ref_init(kind, params, st, w, seed, L, root_cfg):
    """worker of the reference arm: the oracle model and the batch's leaves"""
    import oracle

    om = oracle.Model(kind, params)
    if kind == "car":
        rts = [om.belief_load(*cr) for cr in inputs.car_roots(L, int(len(w)))]
        lv = [(r, -1, 0, 0) for r in rts]
    else:
        root = om.belief_load(st, w, seed)
        R = om.expand([(root, -1, 0, 0)])
        lv = [(root, -1, 0, 0)] if root_cfg else [
            (root, a, cc, 1) for a, cc in inputs.select_leaves(R["child_count"], R["child_begin"], om.A, L)]
    _REF.update(om=om, lv=lv)


def _ref_leaf(i):
    om, lv = _REF["om"], _REF["lv"]
    leaf = lv[i % len(lv)]
    o = om.expand([leaf])
    if leaf[1] >= 0:
        om.node_release(int(o["node"][0]))
    return o["scenario_steps"]


def run_reference(args):
    """--impl reference: the CPU oracle as it stands, timed on this box's host
    cores.  One step = one leaf per host core (one process each, the leaves of
    the batch in order, cycling): a bounded sample of the batch, so that the
    run ends within minutes.  ms_per_step is the measured time of that
    sample step; the full batch's time is reported separately as an
    extrapolation at the measured rate."""
    import multiprocessing as mp

    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    c, kind, params, st, w, seed, L = workload(args.config)
    cores = len(os.sched_getaffinity(0))
    per_step = max(1, min(cores, args.ref_leaves)) if args.ref_leaves > 0 else cores
    ctx = mp.get_context("fork")
    with ctx.Pool(per_step, initializer=_ref_init, initargs=(kind, params, st, w, seed, L, bool(c.get("root")))) as pool:
        pool.map(_ref_leaf, range(per_step))  # every worker set up
        times, steps_all = [], []
        for it in range(args.warmup + args.steps):
            idx = [(it * per_step + j) % L for j in range(per_step)]
            t0 = time.perf_counter()
            st_ = pool.map(_ref_leaf, idx, chunksize=1)
            dt = time.perf_counter() - t0
            if it >= args.warmup:
                times.append(dt)
                steps_all.append(int(np.sum(st_)))
    import oracle

    om = oracle.Model(kind, params)
    value = float(np.sum(steps_all) / np.sum(times))
    full_steps = None
    if c.get("root"):
        full_steps = steps_all[0]
    line = {"impl": "reference", "metric": "scenario-steps/s", "value": value, "unit": "scenario-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * float(np.mean(times)), "higher_is_better": True,
            "step": f"{per_step} of the batch's {L} leaves per step (one per host process), measured",
            "ms_per_full_batch_extrapolated": (1e3 * float(np.mean(times)) * L / per_step) if L > per_step else None,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32+f64", "data": "synthetic",
            "config": {"workload": c["name"], "K": int(len(w)), "leaves": L, "actions": int(om.A),
                       "depth": int(om.D), "l2": "inputs < L2; host run"},
            "cpu_baseline": {"value": value, "unit": "scenario-steps/s", "cores": per_step, "kind": "oracle",
                             "sample": f"{args.steps} steps of {per_step} leaf expansions each (all |A| actions), "
                                       f"{int(np.sum(steps_all))} scenario-steps in {float(np.sum(times)):.1f} s",
                             "host": host_cpu_info()},
            "e2e": {"value": value, "unit": "scenario-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if full_steps is not None:
        line["config"]["scenario_steps_per_batch"] = int(full_steps)
    print(json.dumps(line))
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--K", type=int, default=None)
    ap.add_argument("--impl", default="despot", choices=["despot", "reference"])
    ap.add_argument("--ref-leaves", type=int, default=0,
                    help="reference arm: leaves per step (0 = one per host core)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    ap.add_argument("--all-cores-baseline", action="store_true", default=True,
                    help="also time the oracle in one process per host core")
    ap.add_argument("--no-all-cores-baseline", dest="all_cores_baseline", action="store_false")
    ap.add_argument("--peds", type=int, default=None, help="pedestrians of the driving config (NEXT-3 study)")
    ap.add_argument("--car-variant", default="auto", choices=["auto", "warp", "thread", "group", "pair"],
                    help="driving kernel: factored warp per scenario, thread per scenario, or per-batch choice")
    ap.add_argument("--plan", action="store_true",
                    help="tree size per planning time: despot_plan vs the serial oracle-backed driver (NEXT-1/2)")
    ap.add_argument("--plan-study", default="configs", choices=["configs", "K", "A"])
    ap.add_argument("--plan-configs", type=int, nargs="*", default=[1, 2, 3, 4])
    ap.add_argument("--plan-K", type=int, nargs="*", default=[100, 500, 1000, 2000, 5000])
    ap.add_argument("--plan-workers", type=int, nargs="*", default=[1, 8])
    ap.add_argument("--plan-budget", type=float, default=1.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.plan:
        return run_plan(args)

    import torch

    from paper_1802_06215_b200 import build as B
    from paper_1802_06215_b200.despot import Model

    B.build()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional test of the N > 1 path on a one-GPU box (never a measurement):
    # every rank on device 0, gloo collectives through host memory
    one_gpu_test = world > 1 and os.environ.get("DESPOT_BENCH_ONE_GPU_TEST") == "1"
    if one_gpu_test:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        if one_gpu_test:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    c, kind, params, st, w, seed, L = workload(args.config, args.K, args.peds)
    mflags = {"auto": 0, "thread": 1, "warp": 2, "group": 4, "pair": 16}[args.car_variant]
    comm = None
    if world > 1 and not one_gpu_test:
        # the library's own NCCL communicator (rank 0's unique id over the
        # process group): every batch runs its exchange inside the call
        from paper_1802_06215_b200.dist import init_comm
        comm = init_comm(device=local)
    model = Model(kind, params, device=local, rank=rank, world=world, flags=mflags, comm=comm)
    stream = torch.cuda.Stream(dev)  # a non-blocking stream of our own (not the legacy default stream)
    torch.cuda.set_stream(stream)
    if kind == "car":
        # config 4: L concurrent roots (inputs.car_roots)
        croots = inputs.car_roots(L, int(len(w)), peds=c.get("peds", 20))
        leaves = [(model.belief_load(s_, w_, sd_), -1, 0, 0) for s_, w_, sd_ in croots]
        lv_ac = None
    else:
        root = model.belief_load(st, w, seed)
        # root expansion (untimed): gives the depth-1 leaves
        if world > 1:
            from paper_1802_06215_b200.dist import expand_sharded
            R = expand_sharded(model, [(root, -1, 0, 0)])
        else:
            R = model.expand([(root, -1, 0, 0)])
        if c.get("root"):  # config 1: the root belief itself is the batch
            lv_ac = [(-1, 0)]
            leaves = [(root, -1, 0, 0)]
        else:
            lv_ac = inputs.select_leaves(R["child_count"], R["child_begin"], model.A, L)
            leaves = [(root, a, cc, 1) for a, cc in lv_ac]
    cap = model.child_capacity_bound(leaves)
    dev_out = model.alloc_outputs(leaves, device_outputs=True, child_capacity=cap)
    host_out = model.alloc_outputs(leaves, device_outputs=False, child_capacity=cap, pinned=True)

    preps = {}

    def one_step(outputs, device_outputs, timing=True, ev_end=None):
        if one_gpu_test:  # caller-driven exchange over gloo (functional test only)
            from paper_1802_06215_b200.dist import run_exchange
            b, ex = model.expand_begin(leaves, timing=timing)
            run_exchange(model, b, ex)  # one round of in-place collectives
            o = model.expand_end(b, leaves, device_outputs=device_outputs, timing=timing, outputs=outputs)
            nodes = o["node"]
        else:
            key = (device_outputs, timing)
            if key not in preps:
                # device outputs (inputs resident in HBM): DESPOT_X_RESIDENT where the batch
                # qualifies (self leaves, fused finalize: the graph is K2 alone); e2e:
                # page-locked host results and the per-step leaf-table copy
                preps[key] = model.prepare(leaves, device_outputs=device_outputs, child_capacity=cap, timing=timing,
                                           pinned=not device_outputs, resident=device_outputs)
            prep = preps[key]
            steps, launches, nodes = model.run_prepared(prep, stream=stream)
            if ev_end is not None:  # the call has returned (synchronous): the step ends here
                ev_end.record(stream)
            E = prep["E"]
            o = {"scenario_steps": steps, "launches": launches, "phase_ms": list(E.phase_ms),
                 "num_children": E.num_children, "h2d_bytes": int(E.h2d_bytes), "d2h_bytes": int(E.d2h_bytes),
                 "exchange_ms": float(E.exchange_ms), "exchange_rounds": int(E.exchange_rounds),
                 "exchange_bytes": int(E.exchange_bytes)}
        o["new_nodes"] = [n for (lf, n) in zip(leaves, nodes) if lf[1] >= 0]  # self leaves return their own node
        return o

    def release(o):
        if o["new_nodes"]:
            model.node_release_many(o["new_nodes"])

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize(dev)

    clk = ClockSampler(local).start()
    time.sleep(0.3)  # let nvidia-smi start streaming
    for _ in range(max(args.warmup, 3)):
        release(one_step(dev_out, True, timing=False))  # the timed steps' exact call (prepared batch)
        release(one_step(dev_out, True, timing="k2"))
    # K1 / K3 phases for the report (every phase's events, untimed steps)
    ph = [one_step(dev_out, True, timing=True) for _ in range(3)]
    for o in ph:
        release(o)
    k1_ph = float(np.mean([o["phase_ms"][0] for o in ph]))
    k3_ph = float(np.mean([o["phase_ms"][2] for o in ph]))
    k4_ph = float(np.mean([o.get("exchange_ms", 0.0) for o in ph]))  # the exchange (N > 1, library-owned)
    k4_bytes = int(ph[-1].get("exchange_bytes", 0))
    # ---- device-resident timed region 1: throughput (no library events) ----
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    steps_count, launches = [], 0
    barrier()
    tw0 = time.monotonic()
    for i in range(args.steps):
        flush.zero_()
        ev[i][0].record(stream)
        o = one_step(dev_out, True, timing=False, ev_end=ev[i][1])
        if one_gpu_test:
            ev[i][1].record(stream)
        release(o)  # host bookkeeping of the bench (the arenas a search would keep), outside the events
        steps_count.append(o["scenario_steps"])
        launches += o["launches"]
    barrier()
    # ---- timed region 2: the same steps with K2's two CUDA events (roofline) ----
    # (two library events cost ~10 us of host time per call, which the
    # throughput loop above does not pay)
    k2_ms = []
    for i in range(args.steps):
        flush.zero_()
        o = one_step(dev_out, True, timing="k2")
        release(o)
        k2_ms.append(o["phase_ms"][1])
    barrier()
    tw1 = time.monotonic()
    clk.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    if os.environ.get("BENCH_STEP_LOG"):
        print("step_ms", [round(x, 4) for x in step_ms], file=sys.stderr)
    t_local = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([t_local], device="cpu" if one_gpu_test else dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        t_total = float(t.item())
    else:
        t_total = t_local
    total_steps = float(np.sum(steps_count))  # global (exchanged) scenario-steps
    value = total_steps / (t_total / 1e3)
    # ---- end to end through the C ABI with host buffers ----
    for _ in range(max(args.warmup, 3)):  # warm-up of this call form (its prepared batch)
        release(one_step(host_out, False, timing=False))
    barrier()
    t0 = time.perf_counter()
    e2e_steps = 0
    e2e_n = max(3, args.steps // 2)
    ee = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ee[0].record(stream)
    for _ in range(e2e_n):
        o = one_step(host_out, False, timing=False)
        release(o)
        e2e_steps += o["scenario_steps"]
    ee[1].record(stream)
    barrier()
    e2e_ms = ee[0].elapsed_time(ee[1])
    e2e_wall = time.perf_counter() - t0
    # the library's own count of what one call copied (leaf table in; status and results out)
    h2d, d2h = o["h2d_bytes"], o["d2h_bytes"]
    A = model.A
    # ---- roofline of the dominant kernel (K2), live CUDA-event time ----
    peaks, peak_src = load_peaks()
    clocks = clk.summary(tw0, tw1)
    sm_clock = peaks.get("sm_max_mhz", 1965.0)
    num_sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_tinst = num_sms * 4 * 32 * sm_clock * 1e6 / 1e12  # issue slots, thread-instr/s (Tinst/s)
    k2_avg = float(np.mean(k2_ms))
    steps_local = total_steps / world
    istep, istep_src = i_step(args.config)
    achieved = istep * steps_local / (k2_avg / 1e3) / 1e12 / args.steps
    # K0: the measured Philox ceiling (RNG only, full occupancy) vs K2's own
    # Philox block rate (ceiling 2)
    k0_threads, k0_blocks = num_sms * 2048, 128
    k0_ms, _ = model.philox_ceiling(seed if kind != "car" else 1004, k0_threads, k0_blocks, reps=5, stream=stream)
    k0_rate = k0_threads * k0_blocks / (k0_ms / 1e3)
    bps = philox_blocks_per_step(kind, c.get("peds", 20))
    k2_blocks = bps * steps_local / args.steps / (k2_avg / 1e3)
    k2_share = float(np.sum(k2_ms) / np.sum(step_ms))
    traffic = ncu_traffic(args.config)
    if kind == "car":  # the variant rule of despot.cu (launch_k2_sparse) unless forced
        q_bound = A * sum(model.node_info(lf[0])[0] for lf in leaves)
        peds = c.get("peds", 20) if args.peds is None else args.peds
        big = q_bound >= num_sms * 256 or (peds <= 8 and q_bound >= num_sms * 4)
        tiny = q_bound < num_sms * 4
        k2_name = {"thread": "k2_car_thread", "warp": "k2_car_warp", "group": "k2_car_group", "pair": "k2_car_group<B>",
                   "auto": "k2_car_thread" if big else "k2_car_warp" if tiny else "k2_car_group"}[args.car_variant]
    else:
        k2_name = "k2_expand_dense"
    if rank == 0:
        line = {
            **({"note": "functional test of the N > 1 path on one GPU (DESPOT_BENCH_ONE_GPU_TEST): not a "
                        "measurement"} if one_gpu_test else {}),
            "metric": "scenario-steps/s",
            "value": value,
            "unit": "scenario-steps/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": max(args.warmup, 3),
            "ms_per_step": t_total / args.steps,
            "step_ms_percentiles": {"p10": float(np.percentile(step_ms, 10)), "p50": float(np.median(step_ms)),
                                    "p90": float(np.percentile(step_ms, 90)), "max": float(np.max(step_ms)),
                                    "rank": rank},
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "u32+f64",
            "data": "synthetic",
            "config": {"workload": c["name"], "K": int(len(w)), "leaves": L, "actions": int(A),
                       "depth": int(model.D), "parallelism": f"scenario-shard{world}",
                       "l2": "flushed between timed steps (256 MiB write, outside the events)",
                       "scenario_steps_per_batch": int(total_steps / args.steps)},
            "phases_ms": {"K1_update": k1_ph, "K2_expand_rollout": k2_avg, "K3_finalize": k3_ph,
                          "K4_exchange": k4_ph, "exchange_bytes_per_batch_per_rank": k4_bytes,
                          "K2_share_of_step": k2_share,
                          "note": "K2 from its CUDA events in timed region 2; K1/K3 from 3 untimed steps "
                                  "with every phase's events (8 events cost ~30 us of host time per call)"},
            "roofline": {"bound": "alu", "kernel": k2_name, "achieved": achieved,
                         "peak": peak_tinst, "unit": "Tinst/s", "frac": achieved / peak_tinst,
                         "traffic": traffic["bytes_per_launch"] if traffic else None,
                         "traffic_unit": "DRAM bytes per K2 launch",
                         "traffic_source": traffic["source"] if traffic else None,
                         "ncu_k2": ncu_k2_summary(args.config),
                         "k0_philox": {"ceiling_blocks_per_s": k0_rate, "k2_blocks_per_s": k2_blocks,
                                       "k2_over_k0": k2_blocks / k0_rate, "blocks_per_scenario_step": bps,
                                       "k0_ms": k0_ms, "k0_blocks_per_launch": k0_threads * k0_blocks},
                         "hbm_frac": (traffic["bytes_per_launch"] / (k2_avg / 1e3) / 1e9 / peaks.get("hbm_gbs", 6650.0))
                         if traffic else None,
                         "note": f"issue-slot peak {num_sms} SM x 4 SMSP x 32 lanes x {sm_clock} MHz "
                                 f"({peak_src} sm_max_mhz); achieved = {istep:.1f} thread-instr per "
                                 f"scenario-step ({istep_src}, DESIGN.md §7.1) x steps / live K2 event time",
                         "i_step_measured": {"thread_instr_per_step": i_step_measured(args.config)[0],
                                             "source": i_step_measured(args.config)[1]}},
            "e2e": {"value": e2e_steps / (e2e_ms / 1e3), "unit": "scenario-steps/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms / e2e_n,
                    "wall_ms_per_step": 1e3 * e2e_wall / e2e_n},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(kind, params, st, w, seed, lv_ac, args.cpu_budget, L,
                                                c.get("peds", 20))
            if args.all_cores_baseline:
                line["cpu_baseline_all_cores"] = cpu_baseline_all_cores(kind, params, st, w, seed, lv_ac,
                                                                        args.cpu_budget * 0.7, L, c.get("peds", 20))
        print(json.dumps(line))
    model.close()
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
