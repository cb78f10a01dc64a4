"""Profiling driver: the headline fused iteration (idm_fit_step, C4, L1) in the bench.py launch
configuration, `warmup` iterations then `iters` more, nothing else.  Used under ncu so that the
capture holds only the fused kernels:

    python profiles/prof_fused.py                                  # runs cleanly first
    ncu --set full --clock-control none --import-source on \
        -k regex:"fwd_kernel|bwd_kernel" --launch-skip 4 --launch-count 2 \
        -o gpurun_out/prof python profiles/prof_fused.py [--leader virtual]
    python profiles/summarize.py gpurun_out/prof.ncu-rep > profiles/rNN_fused_fwd_bwd_summary.txt
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2412_16750_b200 import idm, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--iters", type=int, default=1)
    ap.add_argument("--leader", choices=["lane", "virtual"], default="lane")
    ap.add_argument("--fwd-only", action="store_true",
                    help="the prediction rollout idm_forward_ex(IDM_FWD_NO_HISTORY) instead")
    args = ap.parse_args()
    w = synth.make_workload(args.config, seed=synth.CONFIGS[args.config]["seed"])
    sim = idm.from_workload(w, w.theta_true, max_steps=w.K, ckpt_every=idm.DEFAULT_CKPT)
    sim.forward(w.K)
    gen = torch.Generator(device="cuda").manual_seed(1234)
    obs = sim.traj.clone()
    obs[1:].add_(torch.randn(obs[1:].shape, device="cuda", generator=gen), alpha=0.3)
    if args.leader == "virtual":  # bench.py --leader virtual: the paper's per-trajectory fit
        sim.close()
        del sim
        torch.cuda.empty_cache()
        sim = idm.from_workload(w, None, max_steps=w.K, ckpt_every=4, virtual_leader=True)
    sim.params.copy_(torch.as_tensor(synth.init_params(w.n), device="cuda"))
    for it in range(args.warmup + args.iters):
        if args.fwd_only:
            sim.forward(w.K, history=False)
        else:
            sim.fit_step(obs, kind="l1", iteration=it, total=500)
    torch.cuda.synchronize()
    print(f"ok: {args.config} {w.n} vehicles x {w.K} steps, {args.warmup + args.iters} fused iterations")


if __name__ == "__main__":
    main()
