#!/usr/bin/env python
"""Benchmark of the B200 IDM hot path (arXiv 2412.16750) -- one JSON line on rank 0.

A "step" is one pass of the whole hot path over one batch: idm_forward(K) -> idm_loss_grad
(Eq. 4, L1) -> idm_backward -> idm_adam_step, on config C4 of BASELINE.json (2M vehicles in
20,000 lanes x 100, K = 300 steps of dt = 0.1 s, per-vehicle parameters, checkpoint k = 16).
value = vehicle-steps/s over all ranks = ranks * N * K / max-over-ranks(step time).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--scaling weak|strong]
    torchrun --nproc-per-node N bench.py --gpus N ...

--impl reference times the fp64 CPU oracle (oracle/, the only other program of this method
here) on the host cores, on a bounded sample of the same workload.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2412_16750_b200 import parallel, synth  # noqa: E402

LANE_VEH = 100
WORKLOAD = "C4"  # the headline configuration (BASELINE.json configs[3]); --config selects others
# Frozen algorithmic counts: thread-instructions (issue slots) per
# vehicle-step that any implementation of the kernel's math must issue, and HBM bytes per
# vehicle-step the method must move at k = 16, K = 300.
ALG_INSTR = {"fwd": 36.0, "bwd": 114.0}  # SURVEY.md 8(d) frozen essential-op counts
# The same essential math counted in issue slots of THIS implementation, where two vehicles'
# FP32 multiply-adds issue as one f32x2 instruction: the frozen scalar
# counts over-credit a packed kernel, so both fractions are reported.
# "bwd_fit": the optimizer-path backward with delta frozen at 4 (the paper's five parameters,
# PAPER.md:208), which does not compute dL/d delta (one log2, one max, one multiply, one FMA per
# vehicle-step fewer: 3 slots per vehicle-step; R#1).  The counts are after the
# constant folding of DESIGN.md "Adjoint scaling" (lane heads at gap +inf: -0.5 slot per
# vehicle-step forward and backward; dt and ln2 in per-vehicle constants: -1 backward).
PACKED_INSTR = {"fwd": 20.5, "bwd": 44.0, "bwd_fit": 41.0}
ISSUE_PER_CLK = 148 * 4 * 32  # SMs x schedulers x lanes (thread-instr / clk)


def alg_bytes(K: int, k: int, path: str) -> dict:
    """Algorithmic HBM bytes per vehicle-step of each kernel."""
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
    # lane mode: the forward stores the speed history (4 B) and the gap checkpoint (4 B / k;
    # + displacement on the fused path); the backward reads them back instead of recomputing
    if path == "api":
        return {
            "fwd": 8.0 + 4.0 / k + (4 * 4 + 24 + 1) / K,        # P + speed rows, gap ckpt, loads
            "loss": 12.0,                                       # read P, obs; write dL/dP
            "bwd": 8.0 + 4.0 / k + (24 + 24 + 8 + 1) / K,       # speed + dL/dP rows, ckpt, params
            "adam": 6 * 28.0 / K,                               # x, g, m, v in; x, m, v out
        }
    if path == "fused_l2":  # the forward sums Eq. 4; the backward re-derives dL/dP from obs
        return {
            "fwd": 4.0 + 4.0 + 8.0 / k + (4 * 4 + 24 + 1) / K,  # obs in; speeds, gap + D out
            "bwd": 4.0 + 4.0 + 8.0 / k + (24 + 1 + 4 + 24 + 8 + 6 * 20) / K,  # + obs, p0
        }
    # fused L1 (the headline): the forward sums Eq. 4 and records -sign(obs - P) as 2 bits
    return {
        "fwd": 4.0 + 4.0 + 4.0 / k + 0.25 + (4 * 4 + 24 + 1) / K,  # obs in; speeds, gap, bits out
        # speed rows, sign bits, gap checkpoint; params, Adam (x, m, v in and out), grads out
        "bwd": 4.0 + 0.25 + 4.0 / k + (24 + 1 + 24 + 8 + 6 * 20) / K,
    }


def load_traffic():
    """ncu dram bytes per launch of the dominant kernel, from the committed capture summary."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
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
        self.window = None
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
def make_rank_workload(rank: int, world: int, scaling: str):
    if scaling == "weak" or world == 1:
        w = synth.make_workload(WORKLOAD, seed=synth.CONFIGS[WORKLOAD]["seed"] + 1000 * rank)
    else:
        full = synth.make_workload(WORKLOAD)
        l0, l1 = parallel.shard_lanes(full.n_lanes, world, rank)
        w = synth.lane_subset(full, np.arange(l0, l1))
    return w


def cpu_baseline(lanes: int, K: int, seed: int = 99):
    """The fp64 oracle as it stands, single-threaded, one full step (rollout, Eq. 4 L1 loss,
    adjoint, Adam) on the first `lanes` lanes of the configured workload."""
    from oracle import oracle as O
    full = synth.make_workload(WORKLOAD, seed=seed)
    w = synth.lane_subset(full, np.arange(min(lanes, full.n_lanes)))
    w.K = K
    obs = synth.kinematic_obs(w).astype(np.float64)
    st = dict(leader=O.leader_from_lanes(w.lane_offsets), length=w.length, p0=w.p0, v0=w.v0,
              params=synth.init_params(w.n).astype(np.float64), m1=np.zeros((6, w.n)),
              m2=np.zeros((6, w.n)))
    t0 = time.perf_counter()
    O.fit_iteration(st, obs, 0)
    dt = time.perf_counter() - t0
    return w.n * K, dt


def run_reference(args, rank, world):
    """--impl reference: the oracle timed on the host cores (rank 0 only)."""
    if rank != 0:
        return
    K = synth.CONFIGS[WORKLOAD]["K"]
    vs, t = cpu_baseline(4, K)
    per_lane = t / min(4, synth.make_workload(WORKLOAD).n_lanes)
    budget = args.ref_budget  # seconds for the whole --warmup + --steps run
    lanes = int(max(1, min(20000, budget / max(1, args.steps + args.warmup) / per_lane)))
    for _ in range(args.warmup):
        cpu_baseline(lanes, K)
    tot_vs, tot_t = 0, 0.0
    for i in range(args.steps):
        vs, t = cpu_baseline(lanes, K, seed=100 + i)
        tot_vs += vs
        tot_t += t
    value = tot_vs / tot_t
    sample = (f"first {lanes} lanes x {K} steps of {WORKLOAD} per step "
              f"(rollout + Eq.4 L1 + adjoint + Adam, fp64, single thread)")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "vehicle-steps/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC, "sample": sample},
        "cpu_baseline": {"value": value, "unit": "vehicle-steps/s", "cores": 1,
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
}


def set_config(name: str):
    global WORKLOAD, METRIC, WORKLOAD_DESC
    WORKLOAD = name
    WORKLOAD_DESC = CONFIG_DESC[name]
    if name != "C4":
        METRIC = "vehicle-steps/s, forward+loss+backward+Adam (" + name + ")"


def run_ours(args, rank, world, local_rank):
    import torch

    from paper_2412_16750_b200 import idm

    dev = torch.device("cuda", local_rank % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    w = make_rank_workload(rank, world, args.scaling)
    vl = args.leader == "virtual"
    K, k = w.K, (4 if vl else (args.ckpt or idm.DEFAULT_CKPT))
    # synthetic observations: truth rollout with theta_true (our forward) + N(0, 0.3^2)
    stage = 2 if args.e2e > 0 else 0  # e2e: two alternating observation staging buffers
    sim = idm.from_workload(w, w.theta_true, max_steps=K, ckpt_every=k, stage_obs=stage)
    sim.forward(K)
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    obs = sim.traj.clone()
    obs[1:].add_(torch.randn(obs[1:].shape, device=dev, generator=gen), alpha=0.3)
    if vl:  # the paper's per-trajectory fit: free leader terms
        sim.close()
        del sim
        torch.cuda.empty_cache()
        sim = idm.from_workload(w, None, max_steps=K, ckpt_every=k, stage_obs=stage,
                                virtual_leader=True)
    init = torch.as_tensor(synth.init_params(w.n), device=dev)
    stream = sim.stream
    vsteps = float(w.n) * K * world

    def reset():
        sim.params.copy_(init)
        sim.adam_m.zero_()
        sim.adam_v.zero_()
        if vl:
            sim.vl_dp.fill_(idm.VL_INIT[0])
            sim.vl_dv.fill_(idm.VL_INIT[1])
            sim.vl_adam_m.zero_()
            sim.vl_adam_v.zero_()

    def step_api(it):
        sim.forward(K)
        sim.loss_grad(obs, kind=args.loss, sync=False)
        parallel.reduce_step(sim.loss_dev)  # total loss: one 8-byte NCCL all-reduce
        sim.backward()
        sim.adam_step(it % 500, 500, 0.1, 0.01)

    def step_fused(it):
        sim.fit_step(obs, kind=args.loss, iteration=it % 500, total=500, lr0=0.1, lr1=0.01)
        parallel.reduce_step(sim.loss_dev)

    clocks = ClockSampler(local_rank)
    clocks.wait_first()

    def run_path(step_fn):
        reset()
        for i in range(args.warmup):
            step_fn(i)
        torch.cuda.synchronize()
        parallel.barrier()
        start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n0 = sim.launch_count
        tw0 = time.time()
        start.record(stream)
        for i in range(args.steps):
            step_fn(args.warmup + i)
        stop.record(stream)
        torch.cuda.synchronize()
        tw1 = time.time()
        launches = sim.launch_count - n0
        ms = parallel.max_over_ranks(start.elapsed_time(stop), dev) / args.steps
        # per-kernel device time: the same steps again with per-launch events in the library
        sim.timing(True)
        sim.timing_read()
        for i in range(args.steps):
            step_fn(args.warmup + args.steps + i)
        kt = sim.timing_read()
        sim.timing(False)
        kms = {kk: parallel.max_over_ranks(v[0], dev) / args.steps for kk, v in kt.items()
               if v[1] > 0}
        return {"ms_per_step": ms, "value": vsteps / (ms * 1e-3), "kernel_ms": kms,
                "launches_per_step": launches / args.steps, "window": (tw0, tw1)}

    api = run_path(step_api)
    fused = run_path(step_fused)
    # the same iterations as ONE CUDA graph (idm_fit_steps): capture + instantiate + launch, all
    # inside the timed region (the host capture is part of what a user pays)
    reset()
    sim.fit_steps(obs, iters=2, total=max(args.steps, 2) + 2)
    torch.cuda.synchronize()
    reset()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    sim.fit_steps(obs, iters=args.steps, total=args.steps)
    g1.record(stream)
    torch.cuda.synchronize()
    t_g = parallel.max_over_ranks(g0.elapsed_time(g1), dev)
    graph = {"iters": args.steps, "ms_per_step": t_g / args.steps,
             "value": vsteps * args.steps / (t_g * 1e-3), "unit": "vehicle-steps/s",
             "path": "idm_fit_steps: the iteration loop captured as one CUDA graph (capture and "
                     "instantiation inside the timed region)"}
    whole = None
    if not vl and K <= idm.load_library().idm_fit_max_steps():
        # short horizons (C1-like, C5): every iteration of a 500-iteration fit in ONE launch
        reset()
        sim.fit(obs, iters=10, total=500)
        torch.cuda.synchronize()
        reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        sim.fit(obs, iters=500, total=500)
        e1.record(stream)
        torch.cuda.synchronize()
        t_fit = parallel.max_over_ranks(e0.elapsed_time(e1), dev)
        whole = {"iters": 500, "ms_total": t_fit, "ms_per_iteration": t_fit / 500,
                 "value": vsteps * 500 / (t_fit * 1e-3), "unit": "vehicle-steps/s",
                 "launches": 2, "path": "idm_fit (fwd+Eq.4+bwd+Adam x 500 on chip)"}
    clocks.stop()

    # ---- end to end through the C-ABI with HOST buffers (idm_step_host)
    e2e = None
    if args.e2e > 0:
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
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(2):
            scratch.copy_(obs_h, non_blocking=True)
        c1.record()
        torch.cuda.synchronize()
        copy_gbps = 2 * obs_h.numel() * 4 / (c0.elapsed_time(c1) * 1e-3) / 1e9
        del scratch
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

    if rank != 0:
        return
    hbm_gbs, sm_mhz_max, peak_src = load_peaks()
    n_veh_steps = float(w.n) * K  # per rank per launch
    head = fused
    kms = head["kernel_ms"]
    dom = max(kms, key=kms.get)
    if vl:  # HBM-bound mode: roofline against the measured copy bandwidth
        ab = alg_bytes(K, k, "vl")
        achieved = ab[dom] * n_veh_steps / (kms[dom] * 1e-3) / 1e9
        traffic = load_traffic().get(f"vl_{dom}_kernel")
        roofline = {"bound": "hbm", "kernel": f"vl_{dom}_kernel (fused path)",
                    "achieved": achieved, "peak": hbm_gbs, "unit": "GB/s",
                    "frac": achieved / hbm_gbs, "traffic": traffic,
                    "basis": f"{ab[dom]:.2f} algorithmic bytes per vehicle-step x "
                             f"{n_veh_steps:.3g} per launch / CUDA-event launch time; peak = "
                             f"MEASURED_PEAKS hbm_gbs ({peak_src})"}
    else:
        issue_peak = ISSUE_PER_CLK * sm_mhz_max * 1e6 / 1e12  # Tinstr/s
        kk = "bwd" if dom == "bwd" else "fwd"
        kp = "bwd_fit" if kk == "bwd" else kk  # the headline path is idm_fit_step, delta frozen
        # essential issue slots of THIS (f32x2-packed) implementation: SURVEY 8(d) addendum
        achieved = PACKED_INSTR[kp] * n_veh_steps / (kms[dom] * 1e-3) / 1e12
        frozen = ALG_INSTR[kk] * n_veh_steps / (kms[dom] * 1e-3) / 1e12
        traffic = load_traffic().get(f"{dom}_kernel")
        roofline = {"bound": "alu", "kernel": f"{dom}_kernel (fused path)", "achieved": achieved,
                    "peak": issue_peak, "unit": "Tinstr/s", "frac": achieved / issue_peak,
                    "traffic": traffic,
                    "frac_frozen_scalar_count": frozen / issue_peak,
                    "basis": f"{PACKED_INSTR[kp]} essential issue slots per vehicle-step (packed "
                             f"f32x2 implementation; SURVEY 8(d) addendum) x {n_veh_steps:.3g} "
                             f"vehicle-steps per launch / CUDA-event launch time; peak = 148 SM "
                             f"x 4 issue/clk x 32 lanes x {sm_mhz_max:.0f} MHz (MEASURED_PEAKS "
                             f"sm_max, {peak_src}); frac_frozen_scalar_count uses the round-1 "
                             f"scalar count {ALG_INSTR[kk]:.0f}, which a packed kernel can exceed; "
                             f"traffic = ncu dram bytes/launch (profiles/traffic.json)"}

    def hbm_of(p, path):
        ab = alg_bytes(K, k, path)
        tot = sum(ab.values()) * n_veh_steps
        return {"bytes_per_vehicle_step": round(sum(ab.values()), 3),
                "achieved_GBps": tot / (p["ms_per_step"] * 1e-3) / 1e9, "peak_GBps": hbm_gbs,
                "frac": tot / (p["ms_per_step"] * 1e-3) / 1e9 / hbm_gbs,
                "per_kernel_frac": {kk: ab[kk] * n_veh_steps / (p["kernel_ms"][kk] * 1e-3) / 1e9
                                    / hbm_gbs for kk in ab if kk in p["kernel_ms"]}}

    cpu = None
    if world == 1 and args.cpu_lanes > 0:
        vs_c, t_c = cpu_baseline(args.cpu_lanes, K)
        cpu = {"value": vs_c / t_c, "unit": "vehicle-steps/s", "cores": 1, "kind": "oracle",
               "sample": f"first {args.cpu_lanes} lanes x {K} steps of {WORKLOAD}, one "
                         f"full step (fp64 rollout + Eq.4 L1 + adjoint + Adam), 1 thread, "
                         f"{t_c:.1f} s"}
    line = {
        "metric": METRIC, "value": head["value"], "unit": "vehicle-steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": head["ms_per_step"],
        "higher_is_better": True, "scaling": args.scaling if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": WORKLOAD_DESC + ("; virtual-leader mode (PAPER.md:208): every "
                                                "vehicle fitted alone with free per-step "
                                                "(dp, dv) leaves" if vl else ""),
                   "vehicles_per_rank": w.n, "K": K,
                   "ckpt_every": k, "loss": args.loss,
                   "path": "idm_fit_step (fused fwd+Eq.4 / bwd+Adam)",
                   "parallelism": f"lane-sharded x{world}",
                   "l2": "no flush: inputs larger than L2 (2.4 GB obs read by both kernels + "
                         "2.4 GB speed history per rank per step vs 126 MB L2)"},
        "fwd": {"value": vsteps / (api["kernel_ms"]["fwd"] * 1e-3), "unit": "vehicle-steps/s",
                "ms": api["kernel_ms"]["fwd"], "what": "idm_forward, trajectory record on"},
        "fused_path": {kk: head[kk] for kk in ("ms_per_step", "value", "kernel_ms",
                                               "launches_per_step")},
        "api_path": {kk: api[kk] for kk in ("ms_per_step", "value", "kernel_ms",
                                            "launches_per_step")},
        "whole_fit_path": whole,
        "graph_path": graph,
        "roofline": roofline,
        "hbm": {"fused": hbm_of(fused, "vl" if vl else ("fused_l2" if args.loss == "l2" else
                                                        "fused")),
                "api": hbm_of(api, "vl_api" if vl else "api"), "peak_source": peak_src},
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(round(head["launches_per_step"] * args.steps)),
        "clocks": clocks.summary(*head["window"]),
        "paper_context": "< 30 ms per timestep per pass at 2M vehicles on 16-thread Xeon "
                         "W-2255 or one RTX A5000 (PAPER.md:36, :253) = > 6.7e7 vehicle-steps/s "
                         "per pass",
    }
    print(json.dumps(line), flush=True)


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
    ap.add_argument("--config", choices=["C1", "C2", "C3", "C4", "C5"], default="C4",
                    help="BASELINE.json configuration (C4 = the headline)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak")
    ap.add_argument("--ckpt", type=int, default=None, help="checkpoint interval k")
    ap.add_argument("--loss", choices=["l1", "l2"], default="l1",
                    help="Eq. 4 as the paper's L1 (headline) or the smooth L2 variant")
    ap.add_argument("--e2e", type=int, default=8, help="end-to-end steps (0 = skip)")
    ap.add_argument("--cpu-lanes", type=int, default=2000,
                    help="C4 lanes in the oracle cpu_baseline sample (0 = skip)")
    ap.add_argument("--traffic", type=float, default=None,
                    help="ncu dram bytes per launch of the dominant kernel (from profiles/)")
    args = ap.parse_args()
    set_config(args.config)
    if args.leader == "virtual":
        global METRIC
        METRIC = METRIC.replace("forward+loss+backward+Adam", "virtual-leader fit step")
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
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
