#!/usr/bin/env python
"""Benchmark of the B200 IDM hot path (arXiv 2412.16750) -- one JSON line on rank 0.

A "step" is one pass of the whole hot path over one batch: forward(K) -> Eq. 4 (L1) -> backward
-> Adam, on config C4 of BASELINE.json (2M vehicles in 20,000 lanes x 100, K = 300 steps of
dt = 0.1 s, per-vehicle parameters).  The headline path is the fused idm_fit_step (2 launches,
checkpoint interval k = 4, the library default); the 5-call API path, the forward alone, the
CUDA-graph loop, the end-to-end host path and the virtual-leader mode are reported beside it.
value = vehicle-steps/s over all ranks = (sum of the ranks' N) * K / max-over-ranks(step time).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--scaling strong|weak]
    torchrun --nproc-per-node N bench.py --gpus N ...

With --gpus N > 1 and no torchrun environment, bench.py launches the N ranks itself (torchrun,
127.0.0.1) -- or fails loudly if this host has fewer than N GPUs.  At N > 1 the headline is the
2M-vehicle strong split (BASELINE.json: "at 2M vehicles, 1/2/4/8 B200"); the weak-scaling
number (2M vehicles per rank) is a secondary field.

--impl reference times the fp64 CPU oracle (oracle/, the only other program of this method
here) on all host cores, on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2412_16750_b200 import parallel, synth  # noqa: E402

WORKLOAD = "C4"  # the headline configuration (BASELINE.json configs[3]); --config selects others
# Essential issue slots (thread-instructions) per vehicle-step:
# SURVEY.md 8(d)'s frozen scalar counts (the survey commit: 36 forward, 114 backward, 150 both)
# and the same essential math counted for THIS implementation, where two vehicles' FP32
# multiply-adds issue as one f32x2 instruction (SURVEY 8(d) addendum).  "bwd_fit": the
# optimizer-path backward with delta frozen at 4 (no dL/d delta, R#1).
ALG_INSTR = {"fwd": 36.0, "bwd": 114.0}
PACKED_INSTR = {"fwd": 20.5, "bwd": 41.0, "bwd_fit": 38.0}
ISSUE_PER_CLK = 148 * 4 * 32  # SMs x schedulers x lanes (thread-instr / clk)
N_SM = 148
# Essential operations per vehicle-step by execution pipe (DESIGN.md section 4 "ALU roofline"):
# the hand count of the step math (core + advance for the forward; core + jac_record +
# bwd_from_record + the gap rebuild for the backward), equal to the FP32 / MUFU / compare-select
# instructions in the kernels' SASS loops.  fp32 = FP32 lane operations (an FFMA2 is two);
# mufu = ex2 / lg2 / rcp; alu = max / select / setp / sign copies.  "bwd_fit": the optimizer-
# path backward with delta frozen (no dL/d delta, R#1).
ESSENTIAL = {
    "fwd": {"fp32": 22.0, "mufu": 5.0, "alu": 5.0},
    "bwd_fit": {"fp32": 48.0, "mufu": 5.0, "alu": 9.0},
}
# Pipe rates per SM per clock, nominal (sm_100: 4 SMSPs x 32 FP32 lanes; XU 16 lanes; ALU 64
# lanes for FMNMX / FSEL; 4 issue slots x 32 lanes) -- profiles/rNN_pipe_bench.txt holds the
# measured ones (profiles/pipe_bench.cu), which bench.py uses when present.
PIPE_NOMINAL = {"fp32": 128.0, "mufu": 16.0, "alu": 64.0, "issue": 128.0}


def pipe_rates():
    """Per-SM-per-clock lane-op rates measured by profiles/pipe_bench.cu on this B200."""
    path = os.path.join(ROOT, "profiles", "r02_pipe_bench.txt")
    rates, src = dict(PIPE_NOMINAL), "nominal"
    try:
        txt = open(path).read()

        def lane(name):
            for line in txt.splitlines():
                if line.startswith(name):
                    return float(line.split("warp-instr/clk/SM")[1].split()[0])
            return None
        r = {"fp32": lane("FFMA2 (packed f32x2)"), "mufu": lane("MUFU.EX2"),
             "alu": lane("FMNMX"), "issue": lane("FFMA (scalar)")}
        if all(v for v in r.values()):
            rates, src = r, "measured (profiles/r02_pipe_bench.txt)"
    except Exception:
        pass
    return rates, src


def alu_roofline(kind: str, units: float, seconds: float, clk_mhz: float) -> dict:
    """Pipe-by-pipe ceiling of a kernel from its essential op counts: the binding pipe is the
    one needing the most cycles per vehicle-step; achieved / peak are in that pipe's lane-ops."""
    ess = ESSENTIAL[kind]
    rates, src = pipe_rates()
    ops = dict(ess)
    ops["issue"] = ess["fp32"] / 2 + ess["mufu"] + ess["alu"]  # packed FP32: 2 per slot
    cyc = {p: ops[p] / rates[p] for p in ops}  # SM cycles per vehicle-step per pipe
    bind = max(cyc, key=cyc.get)
    hz = N_SM * clk_mhz * 1e6
    peak_vs = hz / cyc[bind]
    achieved_vs = units / seconds
    return {"binding_pipe": bind, "ops_per_vehicle_step": ops,
            "pipe_frac": {p: achieved_vs * cyc[p] / hz for p in cyc},
            "achieved": ops[bind] * achieved_vs / 1e12, "peak": rates[bind] * hz / 1e12,
            "frac": achieved_vs / peak_vs, "peak_vehicle_steps_per_s": peak_vs,
            "rates_per_sm_clk": rates, "rates_source": src}


# SURVEY.md 8(d) algorithmic HBM bytes per vehicle-step of the method's variants (k = 32 there):
# forward with the trajectory record 4.5; fwd+bwd through the API 21.0; with the loss inside the
# kernels (obs read twice) 9.0 -- the variant the fused idm_fit_step implements; single launch 4.2
SURVEY_BYTES = {"fwd": 4.5, "api": 21.0, "fused": 9.0, "single_launch": 4.2}


GAP_CK = 8  # the gap row of every 8th checkpoint is stored (csrc/idm_internal.h kGapCk)


def alg_bytes(K: int, k: int, path: str) -> dict:
    """HBM bytes per vehicle-step each kernel of this implementation moves by design
    (DESIGN.md section 4): the method's bytes plus the speed history the design stores."""
    if path == "vl":  # virtual leader, fused: the forward writes only speed + displacement
        # checkpoints; the backward derives Eq. 4 from obs; leaf Adam in the backward
        return {
            "fwd": 8.0 + 8.0 / k + (4 * 2 + 24) / K,  # dp, dv in; (v, D) checkpoints out
            # dp, dv, obs, 2x(m, v) in; 2x(x, m, v) out; checkpoints; params + Adam per vehicle
            "bwd": 8.0 + 4.0 + 16.0 + 24.0 + 8.0 / k + (4 + 24 + 24 + 8 + 120) / K,
        }
    if path == "vl_api":
        return {
            "fwd": 8.0 + 4.0 + 4.0 / k + (4 * 2 + 24) / K,
            "loss": 12.0,
            "bwd": 8.0 + 4.0 + 8.0 + 4.0 / k + (24 + 24 + 8) / K,
            "adam": 2 * 28.0 + 6 * 28.0 / K,
        }
    # lane mode: the forward stores the speed history (4 B), the gap of every GAP_CK-th
    # checkpoint (4 B / (GAP_CK k)) and the final gap (4 B / K), + displacement checkpoints
    # (4 B / k) on the fused L2 path; the backward reads them back instead of recomputing
    gk = GAP_CK * k
    if path == "api":
        return {
            "fwd": 8.0 + 4.0 / gk + (4 * 4 + 24 + 1 + 4) / K,   # P + speed rows, gap ckpt, loads
            "loss": 12.0,                                       # read P, obs; write dL/dP
            "bwd": 8.0 + 4.0 / gk + (24 + 24 + 8 + 1 + 4) / K,  # speed + dL/dP rows, ckpt, params
            "adam": 6 * 28.0 / K,                               # x, g, m, v in; x, m, v out
        }
    if path == "fwd_only":  # prediction rollout (IDM_FWD_NO_HISTORY): P rows only
        return {"fwd": 4.0 + (4 * 4 + 24 + 1) / K}
    if path == "fused_l2":  # the forward sums Eq. 4; the backward re-derives dL/dP from obs
        return {
            "fwd": 4.0 + 4.0 + 4.0 / k + 4.0 / gk + (4 * 4 + 24 + 1 + 4) / K,  # obs in; speeds,
            # gap + D out
            "bwd": 4.0 + 4.0 + 4.0 / k + 4.0 / gk + (24 + 1 + 4 + 4 + 24 + 8 + 6 * 20) / K,
        }
    # fused L1 (the headline): the forward sums Eq. 4 and records -sign(obs - P) as 2 bits
    return {
        "fwd": 4.0 + 4.0 + 4.0 / gk + 0.25 + (4 * 4 + 24 + 1 + 4) / K,  # obs in; speeds, gaps,
        # bits out; speed rows, sign bits, gaps; params, Adam (x, m, v in and out), grads out
        "bwd": 4.0 + 0.25 + 4.0 / gk + (24 + 1 + 4 + 24 + 8 + 6 * 20) / K,
    }


def _load_json(rel):
    try:
        with open(os.path.join(ROOT, rel)) as f:
            return json.load(f)
    except Exception:
        return {}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("sm_max_mhz", 1965.0)), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


# ---------------------------------------------------------------------------- clocks
REASONS = ["gpu_idle", "applications_clocks_setting", "sw_power_cap", "hw_slowdown",
           "sync_boost", "sw_thermal_slowdown", "hw_thermal_slowdown", "hw_power_brake_slowdown"]


class ClockSampler:
    """nvidia-smi sampled every 20 ms while the timed region runs."""

    def __init__(self, gpu_index: int):
        self.samples = []
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active")
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for line in self.p.stdout:
            parts = [x.strip() for x in line.split(",")]
            try:
                self.samples.append((time.time(), float(parts[0]), float(parts[1]),
                                     int(parts[2], 16)))
            except Exception:
                pass

    def wait_first(self, timeout=5.0):
        t0 = time.time()
        while self.p is not None and not self.samples and time.time() - t0 < timeout:
            time.sleep(0.02)

    def stop(self):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=2)
            except Exception:
                self.p.kill()

    def summary(self, t0, t1):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        inside = [s for s in self.samples if t0 <= s[0] <= t1] or \
            sorted(self.samples, key=lambda s: abs(s[0] - (t0 + t1) / 2))[:3]
        mask = 0
        for s in inside:
            mask |= s[3]
        reasons = [n for b, n in enumerate(REASONS) if mask >> b & 1 and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(s[1] for s in inside),
                "sm_max_mhz": max(s[2] for s in inside), "reasons": reasons,
                "samples": len(inside)}


# ---------------------------------------------------------------------------- workload
def make_rank_workload(rank: int, world: int, scaling: str, shard=None):
    """strong: the 2M-vehicle C4 workload split in contiguous whole-lane shards;
    weak: every rank its own C4-sized workload (seed per rank).  shard = (r, n): one process
    runs shard r of an n-way strong split (an estimate of the per-GPU work at n GPUs)."""
    if shard is not None:
        full = synth.make_workload(WORKLOAD)
        l0, l1 = parallel.shard_lanes(full.n_lanes, shard[1], shard[0])
        return synth.lane_subset(full, np.arange(l0, l1))
    if scaling == "weak" or world == 1:
        return synth.make_workload(WORKLOAD, seed=synth.CONFIGS[WORKLOAD]["seed"] + 1000 * rank)
    full = synth.make_workload(WORKLOAD)
    l0, l1 = parallel.shard_lanes(full.n_lanes, world, rank)
    return synth.lane_subset(full, np.arange(l0, l1))


# ------------------------------------------------------------------ oracle on the host cores
def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _oracle_inputs(full, lanes, K):
    from oracle import oracle as O
    w = synth.lane_subset(full, lanes)
    w.K = K
    obs = synth.kinematic_obs(w).astype(np.float64)
    st = dict(leader=O.leader_from_lanes(w.lane_offsets), length=w.length, p0=w.p0, v0=w.v0,
              params=synth.init_params(w.n).astype(np.float64), m1=np.zeros((6, w.n)),
              m2=np.zeros((6, w.n)))
    return w.n * K, st, obs


_FULL_WORKLOADS = {}


def _full_workload():
    """The configuration's synthetic workload, drawn once per process (2M vehicles at C4)."""
    key = (WORKLOAD, synth.CONFIGS[WORKLOAD]["seed"])
    if key not in _FULL_WORKLOADS:
        _FULL_WORKLOADS[key] = synth.make_workload(WORKLOAD, seed=key[1])
    return _FULL_WORKLOADS[key]


def oracle_prepare(lanes: int, K: int, threads: int, lane0: int = 0):
    """Inputs of the oracle's fit on `lanes` consecutive lanes of the workload from lane `lane0`,
    split into whole-lane tasks for `threads` host threads (the adjoint scatters into leaders,
    so lanes are the unit of parallelism)."""
    full = _full_workload()
    lanes = min(lanes, full.n_lanes)
    lane0 = lane0 % (full.n_lanes - lanes + 1)
    idx = np.arange(lane0, lane0 + lanes)
    chunks = [c for c in np.array_split(idx, max(1, 4 * threads)) if len(c)]
    return [_oracle_inputs(full, c, K) for c in chunks]


def oracle_run(work, threads: int, it: int = 0):
    """One step of the fp64 oracle as it stands (oracle.fit_iteration: rollout, Eq. 4 L1,
    adjoint, Adam iteration `it`) over prepared inputs on `threads` host threads (the C oracle
    releases the GIL).  Returns (vehicle-steps, seconds)."""
    from oracle import oracle as O
    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        list(ex.map(lambda x: O.fit_iteration(x[1], x[2], it), work))
    dt = time.perf_counter() - t0
    return sum(x[0] for x in work), dt


def oracle_step(lanes: int, K: int, threads: int, lane0: int = 0):
    """oracle_prepare + one oracle_run (inputs prepared before the timed region)."""
    return oracle_run(oracle_prepare(lanes, K, threads, lane0), threads)


def oracle_c1_fit_seconds() -> float:
    """The paper's whole 500-iteration fit of C1 by the oracle."""
    from oracle import oracle as O
    w = synth.make_workload("C1")
    obs = synth.kinematic_obs(w).astype(np.float64)
    st = dict(leader=O.leader_from_lanes(w.lane_offsets), length=w.length, p0=w.p0, v0=w.v0,
              params=synth.init_params(w.n).astype(np.float64), m1=np.zeros((6, w.n)),
              m2=np.zeros((6, w.n)))
    t0 = time.perf_counter()
    for it in range(500):
        O.fit_iteration(st, obs, it)
    return time.perf_counter() - t0


def sample_lanes(K: int, cpu_seconds: float) -> int:
    """Lanes of the workload that take about `cpu_seconds` of single-core oracle work."""
    vs, t = oracle_step(8, K, 1)
    per_lane = t / 8
    return int(max(1, min(synth.CONFIGS[WORKLOAD].get("lanes", 10 ** 9), cpu_seconds / per_lane)))


def cpu_baseline(K: int, cpu_seconds: float) -> dict:
    cores = host_cores()
    lanes = sample_lanes(K, cpu_seconds)
    vs, t = oracle_step(lanes, K, cores)
    out = {"value": vs / t, "unit": "vehicle-steps/s", "cores": cores, "kind": "oracle",
           "cpu_model": cpu_model(),
           "sample": f"first {lanes} lanes x {K} steps of {WORKLOAD} ({vs:.3g} vehicle-steps), "
                     f"one full step (fp64 rollout + Eq.4 L1 + adjoint + Adam), whole lanes over "
                     f"{cores} threads, {t:.2f} s wall"}
    if cores >= 16:  # the paper's CPU setting: 16 threads (Xeon W-2255)
        vs16, t16 = oracle_step(lanes, K, 16)
        out["threads_16"] = {"value": vs16 / t16, "seconds": t16}
    else:
        out["threads_16"] = f"not run: the host has {cores} cores"
    vs1, t1 = oracle_step(max(1, lanes // max(1, cores)), K, 1)
    out["threads_1"] = {"value": vs1 / t1, "seconds": t1}
    out["c1_full_fit_s"] = oracle_c1_fit_seconds()
    return out


def run_reference(args, rank, world):
    """--impl reference: the oracle timed on the host cores (rank 0 only)."""
    if rank != 0:
        return
    K = synth.CONFIGS[WORKLOAD]["K"]
    cores = host_cores()
    # each step a bounded sample sized so the whole --warmup + --steps run ends in ~ref_budget s
    vs, t = oracle_step(8, K, 1)
    per_lane_core = t / 8
    per_step = args.ref_budget / max(1, args.steps + args.warmup)
    lanes = int(max(1, min(synth.CONFIGS[WORKLOAD].get("lanes", 10 ** 9),
                           per_step * 0.8 * cores / per_lane_core)))
    # the sample's inputs once; each step is one more iteration of its fit (as the GPU arm
    # iterates on resident inputs)
    work = oracle_prepare(lanes, K, cores)
    for it in range(args.warmup):
        oracle_run(work, cores, it)
    tot_vs, tot_t = 0, 0.0
    for i in range(args.steps):
        vs, t = oracle_run(work, cores, args.warmup + i)
        tot_vs += vs
        tot_t += t
    value = tot_vs / tot_t
    sample = (f"first {lanes} lanes x {K} steps of {WORKLOAD}, one fit iteration per step "
              f"(rollout + Eq.4 L1 + adjoint + Adam, fp64), whole lanes over {cores} host "
              f"threads ({cpu_model()})")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "vehicle-steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / max(1, args.steps), "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC, "sample": sample},
        "cpu_baseline": {"value": value, "unit": "vehicle-steps/s", "cores": cores,
                         "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "vehicle-steps/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "vehicle-steps/s, forward+loss+backward+Adam (C4: 2M vehicles, K=300)"
WORKLOAD_DESC = ("C4: 20,000 lanes x 100 vehicles = 2M, K=300 steps, dt=0.1 s, Eq.4 L1 loss "
                 "on dense noisy observations, per-vehicle IDM params, Adam")
CONFIG_DESC = {
    "C1": "C1: 1 lane x 10 vehicles, K=100, dt=0.1 s (latency-bound: one CTA)",
    "C2": "C2: 1,000 lanes x 100 vehicles = 1e5, K=300, dt=0.1 s, filtering",
    "C3": "C3: NGSIM-shaped, 6 lanes x 333 vehicles, K=27,000 (45 min at 0.1 s; latency-bound: "
          "6 CTAs)",
    "C4": WORKLOAD_DESC,
    "C5": "C5: Waymo-shaped, 100k scenes x 4-12 lanes x 1+Bin(7,0.2) vehicles (~1.9M), K=10 "
          "history fit",
    "C4L": "C4L (not a BASELINE config): 2,000 lanes x 1,000 vehicles = 2M, K=300 -- lanes "
           "longer than a tile, each over a 2-CTA thread-block cluster",
}


def set_config(name: str):
    global WORKLOAD, METRIC, WORKLOAD_DESC
    WORKLOAD = name
    WORKLOAD_DESC = CONFIG_DESC[name]
    if name != "C4":
        METRIC = "vehicle-steps/s, forward+loss+backward+Adam (" + name + ")"


# ------------------------------------------------------------------------------- our arm
def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2412_16750_b200 import idm

    dev = torch.device("cuda", local_rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    scaling = args.scaling or ("strong" if world > 1 else "weak")
    shard = tuple(int(x) for x in args.shard.split("/")) if args.shard else None
    w = make_rank_workload(rank, world, scaling, shard)
    vl = args.leader == "virtual"
    K, k = w.K, (4 if vl else (args.ckpt or idm.DEFAULT_CKPT))
    n_total = parallel.sum_over_ranks(w.n)
    vsteps = float(n_total) * K  # whole job, per step
    clocks = ClockSampler(local_rank)
    clocks.wait_first()

    def build(wl, virtual):
        """A handle on workload wl with synthetic observations: the truth rollout with
        theta_true (our forward) + N(0, 0.3^2)."""
        stage = 2 if args.e2e > 0 and not virtual else 0
        s = idm.from_workload(wl, wl.theta_true, max_steps=wl.K, ckpt_every=k, stage_obs=stage)
        s.forward(wl.K)
        gen = torch.Generator(device=dev).manual_seed(1234 + rank)
        o = s.traj.clone()
        o[1:].add_(torch.randn(o[1:].shape, device=dev, generator=gen), alpha=0.3)
        if virtual:  # the paper's per-trajectory fit: free leader terms
            s.close()
            del s
            torch.cuda.empty_cache()
            s = idm.from_workload(wl, None, max_steps=wl.K, ckpt_every=4, virtual_leader=True)
        return s, o

    def reset(s):
        s.params.copy_(torch.as_tensor(synth.init_params(s.n), device=dev))
        s.adam_m.zero_()
        s.adam_v.zero_()
        if s.virtual_leader:
            s.vl_dp.fill_(idm.VL_INIT[0])
            s.vl_dv.fill_(idm.VL_INIT[1])
            s.vl_adam_m.zero_()
            s.vl_adam_v.zero_()

    def run_path(s, step_fn, n_vs, per_kernel=True):
        reset(s)
        for i in range(args.warmup):
            step_fn(i)
        torch.cuda.synchronize()
        parallel.barrier()
        start, stop = _events(torch)
        n0 = s.launch_count
        tw0 = time.time()
        start.record(s.stream)
        for i in range(args.steps):
            step_fn(args.warmup + i)
        stop.record(s.stream)
        torch.cuda.synchronize()
        tw1 = time.time()
        launches = s.launch_count - n0
        ms = parallel.max_over_ranks(start.elapsed_time(stop), dev) / args.steps
        kms = {}
        if per_kernel:  # the same steps again with per-launch events in the library
            s.timing(True)
            s.timing_read()
            for i in range(args.steps):
                step_fn(args.warmup + args.steps + i)
            kt = s.timing_read()
            s.timing(False)
            kms = {kk: parallel.max_over_ranks(v[0], dev) / args.steps for kk, v in kt.items()
                   if v[1] > 0}
        return {"ms_per_step": ms, "value": n_vs / (ms * 1e-3), "kernel_ms": kms,
                "launches_per_step": launches / args.steps, "window": (tw0, tw1)}

    sim, obs = build(w, vl)

    def step_api(it):
        sim.forward(K)
        sim.loss_grad(obs, kind=args.loss, sync=False)
        parallel.reduce_loss(sim.loss_dev)  # total loss: one 8-byte NCCL all-reduce
        sim.backward()
        sim.adam_step(it % 500, 500, 0.1, 0.01)

    def step_fused(it):
        sim.fit_step(obs, kind=args.loss, iteration=it % 500, total=500, lr0=0.1, lr1=0.01)
        parallel.reduce_loss(sim.loss_dev)

    api = run_path(sim, step_api, vsteps)
    fused = run_path(sim, step_fused, vsteps)
    # the forward alone (BASELINE.json's fwd metric): the prediction rollout, P rows only
    fwd_only = None
    if not vl:
        fwd_only = run_path(sim, lambda it: sim.forward(K, history=False), vsteps)
    # the same iterations as ONE CUDA graph (idm_fit_steps): capture + instantiate + launch, all
    # inside the timed region (the host capture is part of what a user pays)
    reset(sim)
    sim.fit_steps(obs, iters=2, total=max(args.steps, 2) + 2)
    torch.cuda.synchronize()
    reset(sim)
    g0, g1 = _events(torch)
    g0.record(sim.stream)
    sim.fit_steps(obs, iters=args.steps, total=args.steps)
    g1.record(sim.stream)
    torch.cuda.synchronize()
    t_g = parallel.max_over_ranks(g0.elapsed_time(g1), dev)
    graph = {"iters": args.steps, "ms_per_step": t_g / args.steps,
             "value": vsteps * args.steps / (t_g * 1e-3), "unit": "vehicle-steps/s",
             "path": "idm_fit_steps: the iteration loop captured as one CUDA graph (capture and "
                     "instantiation inside the timed region)"}
    whole = None
    if not vl and k == 4 and args.whole_iters > 0:
        # every iteration of a fit in ONE launch (idm_fit: on chip for <= 12-step horizons, else
        # each CTA its tile's whole fit with the history through memory -- NEXT-4)
        on_chip = K <= idm.load_library().idm_fit_max_steps()
        n_it = 500 if on_chip else args.whole_iters
        reset(sim)
        sim.fit(obs, iters=min(10, n_it), kind=args.loss, total=500)
        torch.cuda.synchronize()
        reset(sim)
        e0, e1 = _events(torch)
        e0.record(sim.stream)
        sim.fit(obs, iters=n_it, kind=args.loss, total=500)
        e1.record(sim.stream)
        torch.cuda.synchronize()
        t_fit = parallel.max_over_ranks(e0.elapsed_time(e1), dev)
        whole = {"iters": n_it, "ms_total": t_fit, "ms_per_iteration": t_fit / n_it,
                 "value": vsteps * n_it / (t_fit * 1e-3), "unit": "vehicle-steps/s",
                 "launches": 1 + (args.loss == "l2" or on_chip),
                 "path": "idm_fit: (fwd+Eq.4+bwd+Adam) x iters in one launch, " +
                         ("state on chip" if on_chip else
                          "each CTA its tile's whole fit, history through memory")}
    clocks_main = clocks.summary(*fused["window"])

    # ---- end to end through the C-ABI with HOST buffers (idm_step_host)
    e2e = None
    if args.e2e > 0 and not vl:
        obs_h = obs.cpu().pin_memory()
        p0_h = sim.pos0.cpu().pin_memory()
        v0_h = sim.vel0.cpu().pin_memory()
        sim.step_host(K, obs_h, p0_h, v0_h, iteration=0)
        torch.cuda.synchronize()
        parallel.barrier()
        t0 = time.perf_counter()
        # pipelined: step i+1's upload overlaps step i's backward and Adam; every step's loss is
        # read back to the host (step_host_wait) inside the timed region
        for i in range(args.e2e):
            sim.step_host_async(K, obs_h, p0_h, v0_h, iteration=1 + i)
            if i > 0:
                sim.step_host_wait()
        sim.step_host_wait()
        te = parallel.max_over_ranks(time.perf_counter() - t0, dev)
        h2d = int(obs_h.numel() * 4 + 8 * w.n)
        # the ceiling: a plain pinned host -> device copy of the same observation bytes
        scratch = torch.empty_like(obs)
        scratch.copy_(obs_h, non_blocking=True)
        torch.cuda.synchronize()
        c0, c1 = _events(torch)
        c0.record()
        for _ in range(2):
            scratch.copy_(obs_h, non_blocking=True)
        c1.record()
        torch.cuda.synchronize()
        copy_gbps = 2 * obs_h.numel() * 4 / (c0.elapsed_time(c1) * 1e-3) / 1e9
        del scratch, obs_h
        e2e = {"value": vsteps * args.e2e / te, "unit": "vehicle-steps/s",
               "h2d_bytes_per_step": h2d,
               "h2d_GBps": h2d * args.e2e / te / 1e9,
               "h2d_copy_ceiling_GBps": copy_gbps,
               "bound": "host-to-device copy of the step's observations (PCIe); "
                        "h2d_copy_ceiling_GBps = plain pinned cudaMemcpyAsync of the same bytes",
               "d2h_bytes_per_step": 8, "steps": args.e2e,
               "path": "idm_step_host_async / idm_step_host_wait: pinned host pos0/vel0/obs "
                       "-> device (obs upload overlapping the forward and the previous step's "
                       "backward), fwd, loss, bwd, adam, loss -> host every step; wall clock, "
                       "max over ranks"}

    # ---- secondary measurements of the same metric: weak scaling (N > 1), virtual leader (N = 1)
    weak = None
    vl_line = None
    if world > 1 and scaling == "strong" and args.weak_also:
        sim.close()
        del sim, obs
        torch.cuda.empty_cache()
        ww = make_rank_workload(rank, world, "weak")
        sim, obs = build(ww, False)
        wr = run_path(sim, step_fused, float(parallel.sum_over_ranks(ww.n)) * K, per_kernel=False)
        weak = {"value": wr["value"], "ms_per_step": wr["ms_per_step"], "scaling": "weak",
                "vehicles_per_rank": ww.n, "path": "idm_fit_step"}
    if world == 1 and not vl and args.vl_also:
        sim.close()
        del sim, obs
        torch.cuda.empty_cache()
        sim, obs = build(w, True)
        vr = run_path(sim, step_fused, vsteps)
        vl_line = {"ms_per_step": vr["ms_per_step"], "value": vr["value"],
                   "kernel_ms": vr["kernel_ms"], "clocks": clocks.summary(*vr["window"]),
                   "what": "virtual-leader fit step (PAPER.md:208): every vehicle fitted alone "
                           "with free per-step (dp, dv) leaves updated by Adam"}
    clocks.stop()

    if rank != 0:
        return
    hbm_gbs, sm_mhz_max, peak_src = load_peaks()
    n_veh_steps = float(w.n) * K  # per rank per launch
    head = fused
    kms = head["kernel_ms"]
    dom = max(kms, key=kms.get)
    ncu = _load_json("profiles/ncu_metrics.json")
    if vl:  # HBM-bound mode: roofline against the measured copy bandwidth
        ab = alg_bytes(K, k, "vl")
        achieved = ab[dom] * n_veh_steps / (kms[dom] * 1e-3) / 1e9
        roofline = {"bound": "hbm", "kernel": f"vl_{dom}_kernel (fused path)",
                    "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s",
                    "frac": achieved / hbm_gbs,
                    "traffic": ncu.get(f"vl_{dom}_kernel", {}).get("dram_bytes"),
                    "basis": f"{ab[dom]:.2f} algorithmic bytes per vehicle-step x "
                             f"{n_veh_steps:.3g} per launch / CUDA-event launch time; peak = "
                             f"MEASURED_PEAKS hbm_gbs ({peak_src})"}
    else:
        issue_peak = ISSUE_PER_CLK * sm_mhz_max * 1e6 / 1e12  # Tinstr/s
        kk = "bwd" if dom == "bwd" else "fwd"
        kp = "bwd_fit" if kk == "bwd" else kk  # the headline path is idm_fit_step, delta frozen
        t_dom = kms[dom] * 1e-3
        alu = alu_roofline(kp, n_veh_steps, t_dom, sm_mhz_max)
        frozen = ALG_INSTR[kk] * n_veh_steps / t_dom / 1e12
        packed = PACKED_INSTR[kp] * n_veh_steps / t_dom / 1e12
        nm = ncu.get(f"{dom}_kernel", {})
        roofline = {"bound": "alu", "kernel": f"{dom}_kernel (fused path)",
                    "achieved": alu["achieved"], "peak": alu["peak"],
                    "unit": f"T {alu['binding_pipe']} lane-ops/s", "frac": alu["frac"],
                    "traffic": nm.get("dram_bytes"),
                    "binding_pipe": alu["binding_pipe"], "pipe_frac": alu["pipe_frac"],
                    "ops_per_vehicle_step": alu["ops_per_vehicle_step"],
                    "rates_per_sm_clk": alu["rates_per_sm_clk"],
                    "rates_source": alu["rates_source"],
                    "frac_issue_packed": packed / issue_peak,
                    "frac_survey": frozen / issue_peak,
                    "ncu": {key: nm.get(key) for key in (
                        "issue_active_pct", "fma_pipe_pct", "xu_pipe_pct", "alu_pipe_pct",
                        "warp_instr_per_unit", "dram_bytes_per_unit", "registers", "source")}
                    if nm else None,
                    "basis": f"essential ops per vehicle-step by pipe (DESIGN.md section 4: "
                             f"{alu['ops_per_vehicle_step']}) x {n_veh_steps:.3g} vehicle-steps "
                             f"per launch / CUDA-event launch time; peak = the binding pipe's "
                             f"lane-op rate per SM per clock ({alu['rates_source']}) x 148 SMs x "
                             f"{sm_mhz_max:.0f} MHz (MEASURED_PEAKS sm_max, {peak_src}); "
                             f"frac_issue_packed: {PACKED_INSTR[kp]} packed issue slots per "
                             f"vehicle-step against 4 issue/clk/SM (round 1's figure); "
                             f"frac_survey: SURVEY 8(d)'s frozen scalar count "
                             f"{ALG_INSTR[kk]:.0f} against the issue peak (a packed kernel can "
                             f"exceed 1); ncu = the kernel's measured pipe utilisation "
                             f"(profiles/ncu_metrics.json); traffic = its ncu dram bytes per "
                             f"launch"}

    def hbm_of(p, path, survey_key=None):
        ab = alg_bytes(K, k, path)
        tot = sum(ab.values()) * n_veh_steps
        r = {"bytes_per_vehicle_step": round(sum(ab.values()), 3),
             "achieved_GBps": tot / (p["ms_per_step"] * 1e-3) / 1e9, "peak_GBps": hbm_gbs,
             "frac": tot / (p["ms_per_step"] * 1e-3) / 1e9 / hbm_gbs,
             "per_kernel_frac": {kk: ab[kk] * n_veh_steps / (p["kernel_ms"][kk] * 1e-3) / 1e9
                                 / hbm_gbs for kk in ab if kk in p["kernel_ms"]}}
        if survey_key:  # the same time on the METHOD's algorithmic bytes
            b = SURVEY_BYTES[survey_key]
            r["survey_bytes_per_vehicle_step"] = b
            r["frac_survey_bytes"] = b * n_veh_steps / (p["ms_per_step"] * 1e-3) / 1e9 / hbm_gbs
        return r

    cpu = None
    if world == 1 and args.cpu_seconds > 0:
        cpu = cpu_baseline(K, args.cpu_seconds)
    fwd_line = None
    if fwd_only is not None:
        fwd_line = {"value": fwd_only["value"], "unit": "vehicle-steps/s",
                    "ms": fwd_only["ms_per_step"],
                    "what": "idm_forward_ex(IDM_FWD_NO_HISTORY): the K-step rollout writing P "
                            "(the prediction path)",
                    "hbm": hbm_of(fwd_only, "fwd_only", "fwd"),
                    "roofline": alu_roofline("fwd", n_veh_steps, fwd_only["ms_per_step"] * 1e-3,
                                             sm_mhz_max),
                    "with_history": {"value": vsteps / (api["kernel_ms"]["fwd"] * 1e-3),
                                     "ms": api["kernel_ms"]["fwd"],
                                     "what": "idm_forward (P + the state history a backward "
                                             "reads)"}}
    line = {
        "metric": METRIC, "value": head["value"], "unit": "vehicle-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": scaling if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC + ("; virtual-leader mode (PAPER.md:208): every "
                                                "vehicle fitted alone with free per-step "
                                                "(dp, dv) leaves" if vl else ""),
                   "vehicles_total": n_total, "vehicles_rank0": w.n, "K": K,
                   "shard": args.shard,
                   "ckpt_every": k, "loss": args.loss,
                   "path": "idm_fit_step (fused fwd+Eq.4 / bwd+Adam)",
                   "parallelism": f"lane-sharded x{world} ({scaling})",
                   "l2": "no flush: inputs larger than L2 (2.4 GB obs read by both kernels + "
                         "2.4 GB speed history per rank per step vs 126 MB L2)"},
        "fwd": fwd_line,
        "fused_path": {kk: head[kk] for kk in ("ms_per_step", "value", "kernel_ms",
                                               "launches_per_step")},
        "api_path": {kk: api[kk] for kk in ("ms_per_step", "value", "kernel_ms",
                                            "launches_per_step")},
        "whole_fit_path": whole,
        "graph_path": graph,
        "weak_scaling": weak,
        "virtual_leader": vl_line,
        "roofline": roofline,
        "hbm": {"fused": hbm_of(fused, "vl" if vl else ("fused_l2" if args.loss == "l2" else
                                                        "fused"),
                                None if vl else "fused"),
                "api": hbm_of(api, "vl_api" if vl else "api", None if vl else "api"),
                "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(round(head["launches_per_step"] * args.steps)),
        "clocks": clocks_main,
        "paper_context": "< 30 ms per timestep per pass at 2M vehicles on 16-thread Xeon "
                         "W-2255 or one RTX A5000 (PAPER.md:36, :253) = > 6.7e7 vehicle-steps/s "
                         "per pass",
    }
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="collective backend for N > 1 (gloo only to exercise the multi-rank "
                         "host path on fewer GPUs than ranks)")
    ap.add_argument("--ref-budget", type=float, default=150.0,
                    help="seconds of oracle work for --impl reference")
    ap.add_argument("--leader", choices=["lane", "virtual"], default="lane",
                    help="lane leader (default) or the paper's virtual-leader fit (PAPER.md:208)")
    ap.add_argument("--config", choices=["C1", "C2", "C3", "C4", "C5", "C4L"], default="C4",
                    help="BASELINE.json configuration (C4 = the headline)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default=None,
                    help="N > 1: strong (default; the 2M vehicles split over the ranks) or weak")
    ap.add_argument("--weak-also", type=int, default=1,
                    help="N > 1 strong: also measure weak scaling (secondary field)")
    ap.add_argument("--vl-also", type=int, default=1,
                    help="N = 1: also measure the virtual-leader fit step (secondary field)")
    ap.add_argument("--ckpt", type=int, default=None, help="checkpoint interval k")
    ap.add_argument("--shard", default=None,
                    help="r/n: run only shard r of an n-way strong split on this one GPU (the "
                         "per-GPU work at n GPUs; an estimate, not a multi-GPU measurement)")
    ap.add_argument("--loss", choices=["l1", "l2"], default="l1",
                    help="Eq. 4 as the paper's L1 (headline) or the smooth L2 variant")
    ap.add_argument("--e2e", type=int, default=8, help="end-to-end steps (0 = skip)")
    ap.add_argument("--whole-iters", type=int, default=100,
                    help="iterations of the one-launch whole fit beyond the on-chip horizon "
                         "(0 = skip)")
    ap.add_argument("--cpu-seconds", type=float, default=20.0,
                    help="core-seconds of oracle work in the cpu_baseline sample (0 = skip)")
    args = ap.parse_args()
    set_config(args.config)
    if args.leader == "virtual":
        global METRIC
        METRIC = METRIC.replace("forward+loss+backward+Adam", "virtual-leader fit step")
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launch the N ranks here (one process per GPU, NCCL) -- or fail loudly
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus and args.backend == "nccl":
            sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this host has {have}")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
               f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and args.impl == "ours":
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        dev = torch.device("cuda", local_rank % torch.cuda.device_count())
        torch.cuda.set_device(dev)
        if args.backend == "nccl":
            # communicator set-up logged to stderr (which transport, NVLS or not)
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
        else:  # host-logic check of the multi-rank path on fewer GPUs than ranks
            dist.init_process_group("gloo")
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
