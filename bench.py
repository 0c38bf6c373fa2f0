#!/usr/bin/env python
"""TRST-MI hot-path benchmark (BASELINE.json metric: TR iterations/sec & Gram
entries/sec, fp64 batched trials, % of roofline).

Workload (BASELINE.json configs[1], the headline config that fits one GPU):
complex lines in C^2, N = 100, 4096 independent seeded trials (trial i starts
from random_frame(SplitMix64(mix_seed(0, i)))), each a full anneal() with
TrustRegionConfig.max_outer = 500 (stage k capped at 500 + 50k, solver.hpp:187),
default delta schedule at eps_target 1e-7 (8 stages).

A step is the full anneal of one slice of the config's trials (default 2048
trials for config 2, so 2 consecutive steps cover the 4096 trials once; the
driver's 20 steps cover them 10 times; ~37 s per step, so the driver's
--steps 20 --warmup 5 run takes ~15 minutes with the CPU baseline).  A
wall-clock guard (--budget-s, default 1500 s) stops the timed loop early
rather than lose the line: "steps" then reports the steps actually timed and
"steps_requested" the K that was asked for.  Warm-up steps anneal one SM-wave of
trials (there is no JIT/autotune state to warm).  `e2e` repeats slice 0
through the host-pointer C ABI (trstmi_solve_batch: H2D of start frames and
generator states, D2H of parameters, frames and records inside the timed
region).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one rank per GPU.  Default --scaling strong: the
config's trials are split into contiguous blocks (trstmi_shard_range, trial i
on rank floor(i N / T)); each step anneals one slice of the rank's block; the
best-of exchange is the product's NCCL path (trstmi_best_of_ranks: allgather
of (mu, trial), broadcast of the winning frame).  --scaling weak gives every
rank its own T trials.

--impl reference times the reference's own CPU implementation on the host
cores: the reference headers compiled unchanged against an Eigen-API shim
(oracle/_ref), all host threads, each step one delta stage of a
group of trials (one trial per thread); the value is taken over whole anneal
cycles.  It loads nothing from the product library.
"""
import argparse
import ctypes
import json
import math
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2207_06374_b200 import abi  # noqa: E402  (pure ctypes layouts; loads no native code)

CONFIGS = {
    # name: field, d, N, trials (config), max_outer, workload, default slice
    #   "anneal": the reference's full anneal (every delta stage)
    #   "stage0": the anneal's first stage (delta = 0.1) with that max_outer —
    #             the fixed-work mode SURVEY.md §8d prescribes for configs 4-5
    "c1": (abi.REAL, 4, 10, 64, 200, "anneal", 64),
    "c2": (abi.COMPLEX, 2, 100, 4096, 500, "anneal", 2048),
    "c3": (abi.COMPLEX, 6, 36, 1024, 1000, "anneal", 1024),
    "c4": (abi.REAL, 64, 1024, 256, 300, "stage0", 256),
    "c5": (abi.COMPLEX, 128, 4096, 64, 100, "stage0", 64),
    # config 5's single frame, Gram row-blocks sharded over the ranks (NCCL)
    "c5frame": (abi.COMPLEX, 128, 4096, 1, 20, "stage0", 1),
}
METRIC = "TR iterations/sec & Gram entries/sec (fp64, batched trials); % of roofline"
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 148 SMs x 64 DFMA/clk x 2 flop x 1965 MHz


def default_schedule(N, eps=1e-7):
    """default_delta_schedule (solver.hpp:64-82), restated so the reference
    arm needs no native library for it."""
    terminal = eps / (2.0 * math.log(N))
    if terminal >= 1e-1:
        return [10.0 * terminal, terminal]
    out, delta = [], 1e-1
    while delta > terminal * (1.0 + 1e-12):
        out.append(delta)
        delta /= 10.0
    out.append(terminal)
    return out


def make_cfg(field, d, N, max_outer, workload):
    cfg = abi.default_cfg(field, d, N, max_outer)
    if workload == "stage0":
        cfg.n_stages = 1
        cfg.schedule[0] = default_schedule(N)[0]
    return cfg


def flops_per_eval(field, d, N):
    """the two dense contractions eval_objective performs
    (smoothing.hpp:104,147): 16 d N^2 (complex), 4 d N^2 (real)."""
    return (16 if field == abi.COMPLEX else 4) * d * N * N


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


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


# ---------------------------------------------------------------------------- CPU (reference) runs
def ref_cycle_sample(cfg, first, trials, threads, budget_s=None):
    """The reference's own code (oracle/_ref) annealing trials [first,
    first+trials) stage by stage on `threads` host threads.  Returns a list of
    per-stage (seconds, outer iterations, evaluator calls) and the kind."""
    from tests import ref_ffi
    starts = None
    if cfg.field == abi.REAL:  # real mode: start frames from the real random_frame (oracle restatement)
        from tests import oracle_ffi
        starts, _ = oracle_ffi.random_frames(cfg.field, cfg.d, cfg.N, 0, first, trials)
    b = ref_ffi.Batch(cfg, 0, first, trials, starts)
    out = []
    t0 = time.perf_counter()
    for k in range(b.ns):
        sec, o, e, _ = b.run(k, k + 1, threads)
        out.append((sec, o, e))
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            break
    b.close()
    return out, b.ns


def port_cycle_sample(cfg, first, trials, threads):
    """Fallback when oracle/_ref is absent (it is built where /root/reference
    exists and shipped prebuilt): the CAS oracle port, full anneals."""
    from tests import oracle_ffi as orc
    L = orc.lib()
    S = 32768 if cfg.d > 16 else 512
    params, st = orc.random_frames(cfg.field, cfg.d, cfg.N, 0, first, trials)
    outer, evals = ctypes.c_int64(), ctypes.c_int64()
    sec = L.orc_time_solve_batch(ctypes.byref(cfg), S, trials, ctypes.c_void_p(params.ctypes.data),
                                 ctypes.c_void_p(st.ctypes.data), threads, ctypes.byref(outer), ctypes.byref(evals))
    return [(sec, outer.value, evals.value)]


def ref_available():
    from tests import ref_ffi
    return ref_ffi.available()


def cpu_cfg(args, field, d, N, max_outer, workload):
    if workload == "stage0":  # CPU cost per eval at N >= 1024 is seconds: cap the stage
        max_outer = min(max_outer, args.cpu_outer or (1 if N > 2048 else 2))
    return make_cfg(field, d, N, max_outer, workload), max_outer


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation on all host threads."""
    if rank != 0:
        return
    field, d, N, trials, max_outer, workload, _ = CONFIGS[args.config]
    cfg, cpu_outer = cpu_cfg(args, field, d, N, max_outer, workload)
    threads = os.cpu_count() or 1
    group = args.cpu_trials or threads
    n = N * (N - 1) // 2
    use_ref = ref_available()
    ns = cfg.n_stages or len(default_schedule(N, cfg.eps_target))
    cycles = max(1, int(round(args.steps / ns))) if args.steps > 0 else 0
    if use_ref:
        if args.warmup > 0:  # nothing to warm on a CPU; one short stage keeps the W contract visible
            wc = make_cfg(field, d, N, 1, workload)
            ref_cycle_sample(wc, 10 ** 6, 1, 1, budget_s=0)
        secs, outs, evs = [], [], []
        for c in range(cycles):
            res, _ = ref_cycle_sample(cfg, c * group, group, threads)
            for s, o, e in res:
                secs.append(s)
                outs.append(o)
                evs.append(e)
        kind = "reference"
        sample = ("%d anneal cycle(s) of %d trials each (trials 0..%d of the seed-0 batch), one delta stage per step "
                  "(%d stage steps), %d host threads; the reference's own headers (proj/include/trstmi) compiled "
                  "unchanged against an Eigen-API shim (oracle/_ref, -O3 -DNDEBUG -std=c++20, naive loops for "
                  "Eigen's products); CPU %s" % (cycles, group, cycles * group - 1, len(secs), threads, cpu_model()))
    else:
        secs, outs, evs = [], [], []
        for c in range(cycles):
            for s, o, e in port_cycle_sample(cfg, c * group, group, threads):
                secs.append(s)
                outs.append(o)
                evs.append(e)
        kind = "port"
        sample = ("%d x %d full anneals on %d threads; CAS oracle port (oracle/_ref missing); CPU %s"
                  % (cycles, group, threads, cpu_model()))
    tot = sum(secs) or float("nan")
    v = sum(outs) / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "TR iterations/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / max(len(secs), 1),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "gram_entries_per_s": sum(evs) * n / tot, "evals_per_s": sum(evs) / tot,
        "config": {"workload": "%s: %s d=%d N=%d, trials x %s(max_outer=%d)"
                   % (args.config, "complex" if field == abi.COMPLEX else "real", d, N,
                      "anneal" if workload == "anneal" else "anneal stage 0", cpu_outer),
                   "trials": trials, "max_outer": cpu_outer, "seed": 0},
        "cpu_baseline": {"value": v, "unit": "TR iterations/s", "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": v, "unit": "TR iterations/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(args, field, d, N, workload):
    """cpu_baseline of the GPU line: one whole anneal cycle of one trial per
    host thread through the reference's code (oracle/_ref)."""
    threads = os.cpu_count() or 1
    group = args.cpu_trials or threads
    n = N * (N - 1) // 2
    cfg, cpu_outer = cpu_cfg(args, field, d, N, CONFIGS[args.config][4], workload)
    if ref_available():
        res, ns = ref_cycle_sample(cfg, 0, group, threads, budget_s=args.cpu_budget)
        kind = "reference"
        what = ("%d of %d delta stages of trials 0..%d (one trial per thread), the reference's own headers "
                "compiled against an Eigen-API shim (oracle/_ref, -O3 -DNDEBUG, no -march)"
                % (len(res), ns, group - 1))
    else:
        res = port_cycle_sample(cfg, 0, group, threads)
        kind = "port"
        what = "%d full anneals, CAS oracle port" % group
    s = sum(r[0] for r in res)
    o = sum(r[1] for r in res)
    e = sum(r[2] for r in res)
    return {"value": o / s, "unit": "TR iterations/s", "cores": threads, "kind": kind,
            "sample": "%s; %.1f s on %d threads; CPU %s" % (what, s, threads, cpu_model()),
            "gram_entries_per_s": e * n / s, "max_outer": cpu_outer}


# ---------------------------------------------------------------------------- GPU arm
def main():
    t_start = time.perf_counter()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--trials", type=int, default=0, help="override the config's trial count (testing only)")
    ap.add_argument("--slice", type=int, default=0, help="trials per step per rank (default: the config's)")
    ap.add_argument("--cpu-trials", type=int, default=0)
    ap.add_argument("--cpu-budget", type=float, default=150.0, help="seconds cap of the cpu_baseline cycle")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--budget-s", type=float, default=1500.0,
                    help="wall-clock guard: stop the timed loop (and skip the CPU baseline) rather than exceed this")
    ap.add_argument("--cpu-outer", type=int, default=0,
                    help="stage0 configs: outer iterations per CPU sample trial (default 2; 1 when N > 2048)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:  # the communicator's ranks / transport (NVLink, NVLS) are countable in the log
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")

    import torch
    import torch.distributed as dist
    from paper_2207_06374_b200 import api

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    field, d, N, T, max_outer, workload, slice_default = CONFIGS[args.config]
    if args.trials:
        T = args.trials
    dim = abi.dim_of(field, d, N)
    n = N * (N - 1) // 2
    fpe = flops_per_eval(field, d, N)
    lib = api.load_library()
    ctx = api.Context(local_rank)
    cfg = make_cfg(field, d, N, max_outer, workload)
    ns = cfg.n_stages or api.default_schedule_len(N)
    sharded_frame = args.config == "c5frame"

    def nccl_id():
        obj = [api.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return ctypes.create_string_buffer(bytes(obj[0]), 128)

    if world > 1:
        ctx.check(lib.trstmi_comm_init(ctx.h, world, rank, nccl_id()), "comm_init")
    if sharded_frame:  # one frame, Gram row-blocks over the ranks
        if world > 1:
            ctx.check(lib.trstmi_set_shard(ctx.h, world, rank, nccl_id()), "set_shard")
        first, count = 0, T
    elif args.scaling == "strong":  # the config's trials in contiguous blocks
        f, c = ctypes.c_int64(), ctypes.c_int64()
        ctx.check(lib.trstmi_shard_range(T, world, rank, ctypes.byref(f), ctypes.byref(c)), "shard_range")
        first, count = f.value, c.value
    else:
        first, count = rank * T, T
    slc = max(1, min(args.slice or slice_default, count))
    n_slices = (count + slc - 1) // slc

    # inputs: start frames + generator states of the rank's block (host), resident on the device
    starts, rng0 = api.random_frames(field, d, N, 0, first, count)
    stream = torch.cuda.current_stream()
    sptr = ctypes.c_void_p(stream.cuda_stream)
    d_start = torch.from_numpy(starts).cuda()
    d_params = torch.empty((slc, dim), dtype=torch.float64, device="cuda")
    d_frames = torch.empty_like(d_params)
    d_best = torch.zeros(dim, dtype=torch.float64, device="cuda")
    d_tout = torch.empty(slc * ctypes.sizeof(abi.TrialOut), dtype=torch.uint8, device="cuda")
    d_sout = torch.zeros(slc * ns * ctypes.sizeof(abi.StageOut), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2
    h_tout = (abi.TrialOut * slc)()
    best = {"mu": float("nan"), "trial": -1}

    def device_step(lo, cnt):
        rng = rng0[lo:lo + cnt].copy()
        d_params[:cnt].copy_(d_start[lo:lo + cnt])
        flush.fill_(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        rc = lib.trstmi_solve_batch_dev(ctx.h, ctypes.byref(cfg), cnt, ctypes.c_void_p(d_params.data_ptr()),
                                        ctypes.c_void_p(rng.ctypes.data), ctypes.c_void_p(d_frames.data_ptr()),
                                        ctypes.c_void_p(d_tout.data_ptr()), ctypes.c_void_p(d_sout.data_ptr()),
                                        None, sptr)
        e1.record(stream)
        ctx.check(rc, "solve_batch_dev")
        torch.cuda.synchronize()
        host = d_tout[:cnt * ctypes.sizeof(abi.TrialOut)].cpu().numpy()
        ctypes.memmove(h_tout, host.ctypes.data, host.nbytes)
        outer = evals = 0
        for t in range(cnt):  # best-of over the block (solver.hpp:256-263): strict <, ascending trial id
            r = h_tout[t]
            outer += r.outer_iterations
            evals += r.evals
            gid = first + lo + t
            if r.status == abi.TRIAL_OK and (best["trial"] < 0 or r.coherence < best["mu"] or
                                             (r.coherence == best["mu"] and gid < best["trial"])):
                best["mu"], best["trial"] = r.coherence, gid
                d_best.copy_(d_frames[t])
        return e0.elapsed_time(e1) / 1e3, outer, evals

    # warm-up: one SM wave of trials through the same entry point
    for _ in range(max(args.warmup, 0)):
        device_step(0, min(slc, 148))
    best.update(mu=float("nan"), trial=-1)
    launches0 = lib.trstmi_launch_count()
    clocks = ClockSampler(local_rank)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    times, outers, evals_l = [], [], []
    for i in range(args.steps):
        if times:  # wall-clock guard: this step, the e2e pass and the CPU baseline must still fit
            left = args.budget_s - (time.perf_counter() - t_start)
            need = 2.2 * max(times) + (0 if args.no_cpu or world > 1 else min(args.cpu_budget, 60.0))
            if world > 1:  # every rank must take the same decision
                f = torch.tensor([1.0 if left < need else 0.0], device="cuda")
                dist.all_reduce(f, op=dist.ReduceOp.MAX)
                stop = f.item() > 0
            else:
                stop = left < need
            if stop:
                break
        s = i % n_slices
        lo = s * slc
        t, o, e = device_step(lo, min(slc, count - lo))
        times.append(t)
        outers.append(o)
        evals_l.append(e)
    steps_done = len(times)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    launches = lib.trstmi_launch_count() - launches0
    t_local = sum(times)
    tot_outer, tot_evals = sum(outers), sum(evals_l)

    # cross-rank: max time, summed work (torch.distributed); best-of through the product (NCCL)
    if world > 1:
        t = torch.tensor([t_local], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_all = t.item()
        w = torch.tensor([tot_outer, tot_evals], dtype=torch.float64, device="cuda")
        dist.all_reduce(w)
        tot_outer_all, tot_evals_all = int(w[0].item()), int(w[1].item())
        if sharded_frame:  # the ranks processed one frame together
            tot_outer_all, tot_evals_all = tot_outer, tot_evals
    else:
        t_all, tot_outer_all, tot_evals_all = t_local, tot_outer, tot_evals
    bmu, bidx = ctypes.c_double(), ctypes.c_int64()
    d_win = torch.empty_like(d_best)
    ctx.check(lib.trstmi_best_of_ranks(ctx.h, dim, best["mu"], best["trial"], ctypes.c_void_p(d_best.data_ptr()),
                                       ctypes.c_void_p(d_win.data_ptr()), ctypes.byref(bmu), ctypes.byref(bidx), sptr),
              "best_of_ranks")

    # end-to-end through the host-pointer C ABI: slice 0 again, H2D + D2H inside the timed region
    cnt0 = min(slc, count)
    h_params = starts[:cnt0].copy()
    h_frames = np.empty_like(h_params)
    h_to = (abi.TrialOut * cnt0)()
    h_so = (abi.StageOut * (cnt0 * ns))()
    rng = rng0[:cnt0].copy()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    rc = lib.trstmi_solve_batch(ctx.h, ctypes.byref(cfg), cnt0, ctypes.c_void_p(h_params.ctypes.data),
                                ctypes.c_void_p(rng.ctypes.data), ctypes.c_void_p(h_frames.ctypes.data),
                                ctypes.cast(h_to, ctypes.c_void_p), ctypes.cast(h_so, ctypes.c_void_p), None)
    e2e_t = time.perf_counter() - t0
    ctx.check(rc, "solve_batch")
    e2e_outer = sum(h_to[t].outer_iterations for t in range(cnt0))
    if world > 1:
        w = torch.tensor([e2e_t, e2e_outer], dtype=torch.float64, device="cuda")
        mx = w.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(w)
        e2e_t_all, e2e_outer_all = mx[0].item(), (e2e_outer if sharded_frame else w[1].item())
    else:
        e2e_t_all, e2e_outer_all = e2e_t, e2e_outer
    e2e = {"value": e2e_outer_all / e2e_t_all, "unit": "TR iterations/s",
           "h2d_bytes_per_step": int(h_params.nbytes + rng.nbytes),
           "d2h_bytes_per_step": int(2 * h_params.nbytes + ctypes.sizeof(h_to) + ctypes.sizeof(h_so) + rng.nbytes),
           "what": "slice 0 (%d trials per rank) through trstmi_solve_batch with host buffers, wall clock" % cnt0}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # roofline: the anneal kernel is the only kernel of a step (profiles/)
    peak = ctypes.c_double()
    ctx.check(lib.trstmi_measure_dfma_peak(ctx.h, 20000, ctypes.byref(peak)), "dfma peak")
    achieved = tot_evals * fpe / t_local / 1e12
    traffic = None
    prof = os.path.join(ROOT, "profiles", "anneal_traffic.json")
    if os.path.exists(prof):
        try:
            rec = json.load(open(prof)).get(args.config)
            if rec:  # ncu dram read+write bytes per trial, scaled to one step's trials
                traffic = rec["bytes_per_trial"] * slc
        except Exception:
            traffic = None

    cpu = None
    if not args.no_cpu and world == 1:
        left = args.budget_s - (time.perf_counter() - t_start)
        if left > 30.0:
            args.cpu_budget = min(args.cpu_budget, max(left - 20.0, 10.0))
            cpu = cpu_baseline(args, field, d, N, workload)

    value = tot_outer_all / t_all
    line = {
        "metric": METRIC, "value": value, "unit": "TR iterations/s", "n_gpus": world, "steps": steps_done,
        "steps_requested": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_all / max(steps_done, 1), "higher_is_better": True,
        "scaling": "strong" if (sharded_frame or args.scaling == "strong") else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "gram_entries_per_s": tot_evals_all * n / t_all, "evals_per_s": tot_evals_all / t_all,
        "config": {"workload": "%s: %s lines d=%d N=%d, %d trials x %s(max_outer=%d, eps 1e-7, %d stage%s); "
                               "step = full anneal of a %d-trial slice per rank"
                   % (args.config, "complex" if field == abi.COMPLEX else "real", d, N, T,
                      "anneal" if workload == "anneal" else "anneal stage 0", max_outer, ns, "s" if ns > 1 else "",
                      slc),
                   "trials": T, "trials_per_rank": count, "slice": slc, "max_outer": max_outer, "seed": 0,
                   "l2": "flushed (256 MB write) before every timed step; trial state lives in shared memory",
                   "parallelism": ("one frame, Gram row-blocks sharded over %d GPU(s) (NCCL)" % world)
                   if sharded_frame else
                   ("%s: trials in contiguous blocks over %d GPU(s); best-of by NCCL allgather(mu, trial) + "
                    "broadcast(frame) (trstmi_best_of_ranks)" % (args.scaling, world))},
        "best_mu": bmu.value, "best_trial": bidx.value,
        "welch_bound": api.welch_bound(d, N),
        "roofline": {"bound": "fp64", "achieved": achieved, "peak": peak.value, "unit": "TFLOP/s",
                     "frac": achieved / peak.value, "traffic": traffic, "traffic_unit": "bytes/launch",
                     "peak_nominal": NOMINAL_FP64_TFLOPS, "frac_nominal": achieved / NOMINAL_FP64_TFLOPS,
                     "note": "achieved = evals x (16|4)dN^2 (dense contraction count, SURVEY 8d) / step device time; "
                             "peak = DFMA-loop throughput measured live on this GPU (MEASURED_PEAKS.json and "
                             "B200_PROFILING.md have no FP64 figure); peak_nominal = 148 SM x 64 DFMA/clk x 1965 MHz"},
        "e2e": e2e, "gpu_launches": int(launches), "clocks": clk, "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
