#!/usr/bin/env python
"""TRST-MI hot-path benchmark (BASELINE.json metric: TR iterations/sec & Gram
entries/sec, fp64 batched trials, % of roofline).

Workload (BASELINE.json configs[1], the headline config that fits one GPU):
complex lines in C^2, N = 100, 4096 independent seeded trials (trial i starts
from random_frame(SplitMix64(mix_seed(0, i)))), each a full anneal() with
TrustRegionConfig.max_outer = 500 (stage k capped at 500 + 50k, solver.hpp:187),
default delta schedule at eps_target 1e-7.  One step = the whole batch.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun: one rank per GPU, each rank anneals its own 4096
trials (trial ids offset by rank; weak scaling), then an NCCL allgather of
(best mu, trial id) and a broadcast of the winning frame (solver.hpp:256-267).
Rank 0 prints one JSON line.

--impl reference times the reference algorithm's CPU implementation on the
host cores: the CAS oracle (oracle/, an Eigen-free restatement of the
reference; the reference itself cannot be built here — DESIGN.md §5), all
host threads, each step a bounded sample of the same workload.
"""
import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2207_06374_b200 import abi  # noqa: E402

CONFIGS = {
    # name: field, d, N, trials per GPU, max_outer, workload
    #   "anneal": the reference's full anneal (every delta stage)
    #   "stage0": the anneal's first stage (delta = 0.1) with that max_outer —
    #             the fixed-work mode SURVEY.md §8d prescribes for configs 4-5,
    #             whose full anneals (CG up to 2*dim per iteration) cannot be timed
    "c1": (abi.REAL, 4, 10, 64, 200, "anneal"),
    "c2": (abi.COMPLEX, 2, 100, 4096, 500, "anneal"),
    "c3": (abi.COMPLEX, 6, 36, 1024, 1000, "anneal"),
    "c4": (abi.REAL, 64, 1024, 256, 300, "stage0"),
    "c5": (abi.COMPLEX, 128, 4096, 64, 100, "stage0"),
    # config 5's single frame, Gram row-blocks sharded over the ranks (NCCL)
    "c5frame": (abi.COMPLEX, 128, 4096, 1, 20, "stage0"),
}


def make_cfg(field, d, N, max_outer, workload):
    cfg = abi.default_cfg(field, d, N, max_outer)
    if workload == "stage0":
        from paper_2207_06374_b200 import api
        cfg.n_stages = 1
        cfg.schedule[0] = api.default_schedule(N)[0]
    return cfg
METRIC = "TR iterations/sec & Gram entries/sec (fp64, batched trials); % of roofline"


def flops_per_eval(field, d, N):
    """the two dense contractions eval_objective performs
    (smoothing.hpp:104,147): 16 d N^2 (complex), 4 d N^2 (real)."""
    return (16 if field == abi.COMPLEX else 4) * d * N * N


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu):
        self.gpu = gpu
        self.samples = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        sm = [float(s[0]) for s in self.samples if len(s) >= 7 and s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if len(s) >= 7 and s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for s in self.samples:
            if len(s) >= 7:
                for n, v in zip(names, s[3:7]):
                    if v.lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_sample(field, d, N, max_outer, trials, threads, first=0, workload="anneal"):
    """Oracle (port of the reference algorithm) over `trials` anneals on
    `threads` host threads; returns (seconds, outer iterations, evals)."""
    from tests import oracle_ffi as orc
    L = orc.lib()
    cfg = make_cfg(field, d, N, max_outer, workload)
    S = abi.lanes_for(field, d, N)
    params, st = orc.random_frames(field, d, N, 0, first, trials)
    outer = ctypes.c_int64()
    evals = ctypes.c_int64()
    sec = L.orc_time_solve_batch(ctypes.byref(cfg), S, trials, ctypes.c_void_p(params.ctypes.data),
                                 ctypes.c_void_p(st.ctypes.data), threads, ctypes.byref(outer), ctypes.byref(evals))
    return sec, outer.value, evals.value


def run_reference(args, rank, world):
    """--impl reference: the CPU implementation of the reference algorithm."""
    if rank != 0:
        return
    field, d, N, trials, max_outer, workload = CONFIGS[args.config]
    if workload == "stage0":
        max_outer = min(max_outer, args.cpu_outer or (1 if N > 2048 else 3))
    threads = os.cpu_count() or 1
    sample = args.cpu_trials or threads
    n = N * (N - 1) // 2
    for _ in range(args.warmup):
        cpu_sample(field, d, N, max_outer, min(sample, threads), threads, workload=workload)
    secs, outs, evs = [], [], []
    for _ in range(args.steps):
        s, o, e = cpu_sample(field, d, N, max_outer, sample, threads, workload=workload)
        secs.append(s)
        outs.append(o)
        evs.append(e)
    tot_s = sum(secs)
    v = sum(outs) / tot_s
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TR iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "gram_entries_per_s": sum(evs) * n / tot_s, "evals_per_s": sum(evs) / tot_s,
        "config": {"workload": "%s: %s d=%d N=%d, %d trials x anneal(max_outer=%d); CPU sample %d trials/step"
                   % (args.config, "complex" if field == abi.COMPLEX else "real", d, N, trials, max_outer, sample),
                   "trials": trials, "max_outer": max_outer, "seed": 0},
        "cpu_baseline": {"value": v, "unit": "TR iterations/s", "cores": min(sample, threads), "kind": "port",
                         "sample": "%d full anneals (trials 0..%d of the seed-0 batch) per step on %d threads; "
                                   "oracle/ CAS restatement (reference not buildable: no Eigen)"
                                   % (sample, sample - 1, threads)},
        "e2e": {"value": v, "unit": "TR iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--trials", type=int, default=0, help="override trials per rank (testing only)")
    ap.add_argument("--cpu-trials", type=int, default=0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-outer", type=int, default=0,
                    help="stage0 configs: outer iterations per CPU sample trial (default 3; 1 when N > 2048)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    from paper_2207_06374_b200 import api

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    field, d, N, trials, max_outer, workload = CONFIGS[args.config]
    if args.trials:
        trials = args.trials
    dim = abi.dim_of(field, d, N)
    n = N * (N - 1) // 2
    fpe = flops_per_eval(field, d, N)
    lib = api.load_library()
    lib.trstmi_launch_count.restype = ctypes.c_longlong
    lib.trstmi_measure_dfma_peak.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    ctx = api.Context(local_rank)
    cfg = make_cfg(field, d, N, max_outer, workload)
    ns = cfg.n_stages or api.default_schedule_len(N)
    first = rank * trials
    sharded = args.config == "c5frame"
    if sharded and world > 1:  # one frame, Gram row-blocks over the ranks
        obj = [api.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ctx.set_shard(world, rank, obj[0])
        first = 0

    # inputs: start frames + generator states (host, pinned for e2e)
    starts, rng0 = api.random_frames(field, d, N, 0, first, trials)
    stream = torch.cuda.current_stream()
    sptr = ctypes.c_void_p(stream.cuda_stream)
    d_start = torch.from_numpy(starts).cuda()
    d_params = torch.empty_like(d_start)
    d_frames = torch.empty_like(d_start)
    d_tout = torch.empty(trials * ctypes.sizeof(abi.TrialOut), dtype=torch.uint8, device="cuda")
    d_sout = torch.empty(trials * ns * ctypes.sizeof(abi.StageOut), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    h_tout = (abi.TrialOut * trials)()

    def device_step():
        rng = rng0.copy()
        d_params.copy_(d_start)
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rc = lib.trstmi_solve_batch_dev(ctx.h, ctypes.byref(cfg), trials, ctypes.c_void_p(d_params.data_ptr()),
                                        ctypes.c_void_p(rng.ctypes.data), ctypes.c_void_p(d_frames.data_ptr()),
                                        ctypes.c_void_p(d_tout.data_ptr()), ctypes.c_void_p(d_sout.data_ptr()),
                                        None, sptr)
        e1.record(stream)
        ctx.check(rc, "solve_batch_dev")
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / 1e3

    def reduce_best():
        """min over trials then over ranks, lowest trial id on ties (solver.hpp:256-263)."""
        host = d_tout.cpu().numpy()  # keep the host copy alive across the memmove
        ctypes.memmove(h_tout, host.ctypes.data, ctypes.sizeof(h_tout))
        best, bi = None, -1
        for t in range(trials):
            r = h_tout[t]
            if r.status == abi.TRIAL_OK and (best is None or r.coherence < best):
                best, bi = r.coherence, t
        outer = sum(h_tout[t].outer_iterations for t in range(trials))
        evals = sum(h_tout[t].evals for t in range(trials))
        return best, bi, outer, evals

    for _ in range(max(args.warmup, 0)):
        device_step()
    launches0 = lib.trstmi_launch_count()
    clocks = ClockSampler(local_rank)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times, outers, evals_l = [], [], []
    best_mu, best_trial = None, -1
    for _ in range(args.steps):
        times.append(device_step())
        best_mu, best_trial, o, e = reduce_best()
        outers.append(o)
        evals_l.append(e)
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = lib.trstmi_launch_count() - launches0
    t_local = sum(times)
    tot_outer = sum(outers)
    tot_evals = sum(evals_l)

    # cross-rank: max time, summed work, best mu + its frame (NCCL)
    best_frame = None
    if world > 1:
        t = torch.tensor([t_local], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_all = t.item()
        w = torch.tensor([tot_outer, tot_evals], dtype=torch.float64, device="cuda")
        dist.all_reduce(w)
        tot_outer_all, tot_evals_all = int(w[0].item()), int(w[1].item())
        if sharded:  # the ranks processed one frame together
            tot_outer_all, tot_evals_all = tot_outer, tot_evals
        cand = torch.tensor([best_mu if best_mu is not None else float("inf"), float(first + best_trial)],
                            dtype=torch.float64, device="cuda")
        allc = [torch.empty_like(cand) for _ in range(world)]
        dist.all_gather(allc, cand)
        allc = [tuple(x.tolist()) for x in allc]
        owner = min(range(world), key=lambda r: (allc[r][0], allc[r][1]))
        fr = d_frames[best_trial].clone() if best_trial >= 0 else torch.zeros(dim, dtype=torch.float64, device="cuda")
        dist.broadcast(fr, src=owner)
        best_mu, gbest = allc[owner]
        best_frame = fr
    else:
        t_all, tot_outer_all, tot_evals_all = t_local, tot_outer, tot_evals
        gbest = first + best_trial

    # end-to-end through the C ABI with host buffers (H2D + D2H in the timed region)
    e2e = None
    if rank == 0 or world > 1:
        h_params = starts.copy()
        h_frames = np.empty_like(starts)
        h_to = (abi.TrialOut * trials)()
        h_so = (abi.StageOut * (trials * ns))()
        e2e_times = []
        for _ in range(1 if args.steps > 0 else 0):
            h_params[:] = starts
            rng = rng0.copy()
            t0 = time.perf_counter()
            rc = lib.trstmi_solve_batch(ctx.h, ctypes.byref(cfg), trials, ctypes.c_void_p(h_params.ctypes.data),
                                        ctypes.c_void_p(rng.ctypes.data), ctypes.c_void_p(h_frames.ctypes.data),
                                        ctypes.cast(h_to, ctypes.c_void_p), ctypes.cast(h_so, ctypes.c_void_p), None)
            e2e_times.append(time.perf_counter() - t0)
            ctx.check(rc, "solve_batch")
        e2e_outer = sum(h_to[t].outer_iterations for t in range(trials))
        if e2e_times:
            e2e = {"value": e2e_outer / e2e_times[0] * (world if world > 1 else 1), "unit": "TR iterations/s",
                   "h2d_bytes_per_step": int(starts.nbytes + rng0.nbytes),
                   "d2h_bytes_per_step": int(2 * starts.nbytes + ctypes.sizeof(h_to) + ctypes.sizeof(h_so)
                                              + rng0.nbytes)}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # roofline: the anneal kernel is the only kernel of the step
    peak = ctypes.c_double()
    ctx.check(lib.trstmi_measure_dfma_peak(ctx.h, 20000, ctypes.byref(peak)), "dfma peak")
    achieved = tot_evals * fpe / t_local / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "anneal_traffic.json")
    if os.path.exists(prof):
        try:
            rec = json.load(open(prof)).get(args.config)
            if rec:  # ncu dram read+write bytes per trial, scaled to this launch's trials
                traffic = rec["bytes_per_trial"] * trials
        except Exception:
            traffic = None

    cpu = None
    if not args.no_cpu and world == 1:
        threads = os.cpu_count() or 1
        sample = args.cpu_trials or threads
        cpu_outer = max_outer if workload == "anneal" else min(max_outer, args.cpu_outer or (1 if N > 2048 else 3))
        s, o, e = cpu_sample(field, d, N, cpu_outer, sample, threads, workload=workload)
        cpu = {"value": o / s, "unit": "TR iterations/s", "cores": min(sample, threads), "kind": "port",
               "sample": "%d %s of this workload (trials 0..%d) on %d host threads, %.1f s; "
                         "oracle/ CAS restatement (reference not buildable: no Eigen)"
                         % (sample, "full anneals" if workload == "anneal" else
                            "stage-0 runs capped at %d outer iterations" % cpu_outer, sample - 1, threads, s),
               "gram_entries_per_s": e * n / s}

    value = tot_outer_all / t_all
    line = {
        "metric": METRIC, "value": value, "unit": "TR iterations/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_all / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "gram_entries_per_s": tot_evals_all * n / t_all, "evals_per_s": tot_evals_all / t_all,
        "config": {"workload": "%s: %s lines d=%d N=%d, %d trials/GPU x %s(max_outer=%d, eps 1e-7, %d stage%s)"
                   % (args.config, "complex" if field == abi.COMPLEX else "real", d, N, trials,
                      "anneal" if workload == "anneal" else "anneal stage 0", max_outer, ns, "s" if ns > 1 else ""),
                   "trials_per_gpu": trials, "max_outer": max_outer, "seed": 0,
                   "l2": "flushed (256 MB write) before every timed step; inputs 13 MB",
                   "parallelism": ("one frame, Gram row-blocks sharded over %d GPU(s) (NCCL)" % world) if sharded else
                                  ("trials sharded over %d GPU(s), NCCL allgather(best mu)+broadcast(frame)" % world)},
        "best_mu": best_mu, "best_trial": gbest,
        "welch_bound": api.welch_bound(d, N),
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
                     "frac": achieved / peak.value, "traffic": traffic, "traffic_unit": "bytes/launch",
                     "note": "achieved = evals x (16|4)dN^2 (dense contraction count, SURVEY 8d) / step device time; "
                             "peak = DFMA-loop throughput measured live on this GPU (MEASURED_PEAKS.json has no FP64)"},
        "e2e": e2e, "gpu_launches": int(launches), "clocks": clk, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
