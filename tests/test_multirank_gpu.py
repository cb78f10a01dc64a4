"""The CUDA path (libidm.so) under several ranks: 2 processes on cuda:0 with the gloo backend,
each running its whole-lane shard (lanes are independent blocks, so no state
crosses ranks).  The ranks' kernels never wait on one another -- the only exchanges are the
host-side collectives -- so running both on one GPU is safe.

  * per-vehicle parameters: every rank's parameters, gradients, dL/dp0, dL/dv0 and Adam moments
    equal the one-rank run's bit for bit (fused idm_fit_step and the separate calls);
  * shared parameters: the per-lane rows gathered exactly and summed in the global lane order
    (parallel.reduce_shared_step -> idm_reduce_shared) give the one-rank gradient bit for bit
    (shard-count invariance) and match the fp64 oracle."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU hosts
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from paper_2412_16750_b200 import synth  # noqa: E402
from tests.parity_helpers import grad_check, oracle_truth_obs  # noqa: E402

LANES = [100] * 30 + [0, 7, 1, 512, 3, 60, 61]
K = 60
SHARED = np.array([8.0, 1.7, 3.0, 1.4, 33.0, 4.0], np.float32)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _workload():
    return synth.make_workload("C2", lane_sizes=LANES, K=K, seed=23)


def _run(sub, obs, shared, lane0=0, total=None):
    """Two optimizer iterations on a shard: per-vehicle -- fused idm_fit_step then the separate
    calls; shared -- the separate calls with the cross-rank gradient reduction."""
    from paper_2412_16750_b200 import idm, parallel
    o = torch.as_tensor(obs, device="cuda").contiguous()
    out = {}
    if not shared:
        a = idm.from_workload(sub, None, max_steps=K)
        for it in range(2):
            a.fit_step(o, kind="l1", iteration=it)
        b = idm.from_workload(sub, None, max_steps=K)
        for it in range(2):
            b.forward(K)
            b.loss_grad(o, kind="l1", sync=False)
            parallel.reduce_loss(b.loss_dev)
            b.backward()
            b.adam_step(it)
        torch.cuda.synchronize()
        for name, s in (("fused", a), ("api", b)):
            for f in ("params", "grad_params", "grad_state0", "adam_m", "adam_v"):
                out[f"{name}_{f}"] = getattr(s, f).cpu().numpy()
        out["loss"] = b.loss_dev.cpu().numpy()
    else:
        total = sub.n_lanes if total is None else total
        s = idm.from_workload(sub, SHARED, max_steps=K, shared_params=True)
        for it in range(2):
            s.forward(K)
            s.loss_grad(o, kind="l2", sync=False)
            s.backward()
            parallel.reduce_shared_step(s, lane0, total)
            torch.cuda.synchronize()
            out[f"grad_{it}"] = s.grad_params.cpu().numpy()
            s.adam_step(it)
        torch.cuda.synchronize()
        out["params"] = s.params.cpu().numpy()
        out["loss"] = s.loss_dev.cpu().numpy()
    return out


def _rank_main(rank, world, port, shared, outdir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2412_16750_b200 import parallel
        w = _workload()
        obs = np.load(os.path.join(outdir, "obs.npy"))
        l0, l1 = parallel.shard_lanes(w.n_lanes, world, rank)
        sub = synth.lane_subset(w, np.arange(l0, l1))
        lane0, total = parallel.lane_offset(l1 - l0)
        out = _run(sub, obs[:, sub.meta["vehicle_index"]], shared, lane0, total)
        np.savez(os.path.join(outdir, f"rank{rank}.npz"), vi=sub.meta["vehicle_index"], **out)
    finally:
        dist.destroy_process_group()


def _spawn(world, shared, outdir):
    import torch.multiprocessing as mp
    port = _free_port()
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, shared, str(outdir)))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=600)
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    return [dict(np.load(os.path.join(outdir, f"rank{r}.npz"))) for r in range(world)]


@pytest.mark.parametrize("shared", [False, True])
def test_two_ranks_equal_one_rank(oracle, tmp_path, shared):
    w = _workload()
    obs = oracle_truth_obs(oracle, w)
    np.save(tmp_path / "obs.npy", obs)
    ref = _run(w, obs, shared)
    ranks = _spawn(2, shared, tmp_path)
    if not shared:
        for r in ranks:
            vi = r["vi"]
            for key, val in ref.items():
                if key == "loss":
                    continue
                assert np.array_equal(r[key], val[..., vi]), key
        total = sum(float(r["loss"][0]) for r in ranks) / len(ranks)  # each holds the sum
        assert abs(float(ranks[0]["loss"][0]) - float(ref["loss"][0])) <= 1e-12 * abs(total)
        return
    for r in ranks:
        # shard-count invariance: the gathered per-lane rows summed in the global lane order
        for it in range(2):
            assert np.array_equal(r[f"grad_{it}"], ref[f"grad_{it}"]), it
        assert np.array_equal(r["params"], ref["params"])
        assert abs(float(r["loss"][0]) - float(ref["loss"][0])) <= 1e-12 * float(ref["loss"][0])
    # ... and the shared gradient of iteration 0 against the fp64 oracle's shared mode
    h = oracle.leader_from_lanes(w.lane_offsets)
    P, V = oracle.rollout(h, w.length, w.p0, w.v0, SHARED.astype(np.float64), K)
    _, gP = oracle.loss(P, obs, "l2")
    g = oracle.backward(h, w.length, SHARED.astype(np.float64), P, V, gP)
    worst, _ = grad_check(ref["grad_0"][:, 0], g["g_params"][:, 0], g["g_abs"][:, 0])
    assert worst <= 1.0
