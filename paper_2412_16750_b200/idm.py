"""Thin ctypes binding of the C-ABI library libidm.so (include/idm.h).

Argument marshalling only: every step of the hot path runs in the library's sm_100a kernels.
PyTorch provides the device memory (the arrays idm_desc points to, and the workspace) and the
CUDA stream.  There is no CPU fallback: if libidm.so is missing or no sm_100a GPU is present
the calls raise.

Function names mirror the C-ABI (idm_init, idm_forward, idm_loss_grad, idm_backward,
idm_adam_step); :class:`IdmSim` bundles a handle with its tensors.
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libidm.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "idm.h")

IDM_OK, IDM_EINVAL, IDM_ENUMERIC, IDM_ECUDA, IDM_ESTATE = range(5)
STATUS_NAMES = {0: "IDM_OK", 1: "IDM_EINVAL", 2: "IDM_ENUMERIC", 3: "IDM_ECUDA", 4: "IDM_ESTATE"}
PARAMS_PER_VEHICLE, PARAMS_SHARED = 0, 1
LEADER_LANE, LEADER_VIRTUAL = 0, 1
VL_INIT = (10.0, 0.0)  # initial (Delta p_k, Delta v_k)
LOSS_KINDS = {"l1": 0, "l2": 1}
FWD_NO_HISTORY = 1  # idm_forward_ex flag: prediction rollout, no state history
PAPER_OPT_MASK = 0x1F  # the paper optimizes five parameters; delta frozen
DEFAULT_CKPT = 4  # backward checkpoint interval k (tuned on B200)


class IdmDesc(C.Structure):
    """Mirror of idm_desc (include/idm.h)."""
    _fields_ = [
        ("n_vehicles", C.c_int64),
        ("n_lanes", C.c_int32),
        ("lane_offsets", C.c_void_p),
        ("pos0", C.c_void_p),
        ("vel0", C.c_void_p),
        ("length", C.c_void_p),
        ("params", C.c_void_p),
        ("grad_params", C.c_void_p),
        ("adam_m", C.c_void_p),
        ("adam_v", C.c_void_p),
        ("grad_state0", C.c_void_p),
        ("traj", C.c_void_p),
        ("vel_traj", C.c_void_p),
        ("grad_traj", C.c_void_p),
        ("state_out", C.c_void_p),
        ("obs_stage", C.c_void_p),
        ("mask_stage", C.c_void_p),
        ("max_steps", C.c_int32),
        ("ckpt_every", C.c_int32),
        ("dt", C.c_float),
        ("a_min", C.c_float),
        ("eps_gap", C.c_float),
        ("param_mode", C.c_int32),
        ("opt_mask", C.c_uint32),
        ("stream", C.c_void_p),
        ("workspace", C.c_void_p),
        ("workspace_bytes", C.c_size_t),
        ("leader_mode", C.c_int32),
        ("vl_dp", C.c_void_p),
        ("vl_dv", C.c_void_p),
        ("vl_grad", C.c_void_p),
        ("vl_adam_m", C.c_void_p),
        ("vl_adam_v", C.c_void_p),
        ("obs_stage2", C.c_void_p),
        ("lane_grads", C.c_void_p),
    ]


class IdmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(code, code)}: {msg}")
        self.code = code


_lib = None


def header_symbols() -> list[str]:
    """Function names declared in include/idm.h."""
    txt = open(HEADER_PATH).read()
    return sorted(set(re.findall(r"^\s*[a-z_0-9 ]+[ \*]+(idm_[a-z_0-9]+)\s*\(", txt, re.M)))


def load_library(path: str | None = None):
    """Load libidm.so (raises if it has not been built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("IDM_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with `python -m paper_2412_16750_b200.build`"
                          " (there is no CPU fallback)")
    L = C.CDLL(path)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    L.idm_workspace_bytes.restype = C.c_size_t
    L.idm_workspace_bytes.argtypes = [C.POINTER(IdmDesc)]
    L.idm_init.restype = C.c_int
    L.idm_init.argtypes = [C.POINTER(vp), C.POINTER(IdmDesc)]
    L.idm_forward.restype = C.c_int
    L.idm_forward.argtypes = [vp, i32]
    L.idm_forward_ex.restype = C.c_int
    L.idm_forward_ex.argtypes = [vp, i32, C.c_uint32]
    L.idm_state_from_obs.restype = C.c_int
    L.idm_state_from_obs.argtypes = [vp, i64, i32, C.c_float, vp, vp, vp]
    L.idm_reduce_shared.restype = C.c_int
    L.idm_reduce_shared.argtypes = [vp, vp, i64]
    L.idm_loss_grad.restype = C.c_int
    L.idm_loss_grad.argtypes = [vp, vp, vp, i32, vp, C.POINTER(C.c_double)]
    L.idm_backward.restype = C.c_int
    L.idm_backward.argtypes = [vp]
    L.idm_adam_step.restype = C.c_int
    L.idm_adam_step.argtypes = [vp, i32, i32, C.c_float, C.c_float]
    L.idm_fit_step.restype = C.c_int
    L.idm_fit_step.argtypes = [vp, i32, vp, vp, i32, i32, i32, C.c_float, C.c_float, vp,
                               C.POINTER(C.c_double)]
    L.idm_fit.restype = C.c_int
    L.idm_fit.argtypes = [vp, i32, vp, i32, i32, i32, i32, C.c_float, C.c_float, vp,
                          C.POINTER(C.c_double)]
    L.idm_fit_steps.restype = C.c_int
    L.idm_fit_steps.argtypes = [vp, i32, vp, i32, i32, i32, i32, C.c_float, C.c_float, vp,
                                C.POINTER(C.c_double)]
    L.idm_plan_tiles.restype = C.c_int64
    L.idm_plan_tiles.argtypes = [vp, i32, C.c_int64, vp]
    L.idm_fit_max_steps.restype = i32
    L.idm_fit_max_steps.argtypes = []
    L.idm_step_host_async.restype = C.c_int
    L.idm_step_host_async.argtypes = [vp, i32, vp, vp, vp, vp, i32, i32, i32, C.c_float,
                                      C.c_float]
    L.idm_step_host_wait.restype = C.c_int
    L.idm_step_host_wait.argtypes = [vp, C.POINTER(C.c_double)]
    L.idm_step_host.restype = C.c_int
    L.idm_step_host.argtypes = [vp, i32, vp, vp, vp, vp, i32, i32, i32, C.c_float, C.c_float,
                                C.POINTER(C.c_double)]
    L.idm_timing_enable.restype = C.c_int
    L.idm_timing_enable.argtypes = [vp, C.c_int]
    L.idm_timing_read.restype = C.c_int
    L.idm_timing_read.argtypes = [vp, vp, vp]
    L.idm_check.restype = C.c_int
    L.idm_check.argtypes = [vp]
    L.idm_launch_count.restype = i64
    L.idm_launch_count.argtypes = [vp]
    L.idm_max_lane_vehicles.restype = i32
    L.idm_max_lane_vehicles.argtypes = []
    L.idm_max_lane_length.restype = i32
    L.idm_max_lane_length.argtypes = []
    L.idm_last_error.restype = C.c_char_p
    L.idm_last_error.argtypes = [vp]
    L.idm_destroy.restype = None
    L.idm_destroy.argtypes = [vp]
    _lib = L
    return L


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def _dev(x, dtype, device):
    if isinstance(x, torch.Tensor):
        return x.detach().to(device=device, dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device=device)


class IdmSim:
    """A handle plus the device tensors its descriptor points to.

    Inputs are copied to fp32 device tensors; ``params`` defaults to the paper's
    initialisation.  Shapes: lane_offsets [L+1], pos0/vel0/length [N],
    params [6, N] (per-vehicle) or [6] (shared)."""

    def __init__(self, lane_offsets, pos0, vel0, length, params=None, *, max_steps: int,
                 ckpt_every: int = DEFAULT_CKPT, dt: float = 0.1, a_min: float = -10.0,
                 eps_gap: float = 0.1, shared_params: bool = False,
                 opt_mask: int = PAPER_OPT_MASK, record_velocity: bool = False,
                 stage_obs: int = 0, stage_mask: bool = False, state_out: bool = True,
                 virtual_leader: bool = False, vl_dp=None, vl_dv=None,
                 device=None, stream: torch.cuda.Stream | None = None):
        L = load_library()
        if not torch.cuda.is_available():
            raise IdmError(IDM_ECUDA, "no CUDA device (there is no CPU fallback)")
        self.device = torch.device(device) if device is not None else \
            torch.device("cuda", torch.cuda.current_device())
        dev = self.device
        self.stream = stream or torch.cuda.current_stream(dev)
        f32 = torch.float32
        self.lane_offsets = _dev(lane_offsets, torch.int32, dev)
        self.n = n = int(self.lane_offsets[-1].item())
        self.n_lanes = int(self.lane_offsets.numel() - 1)
        self.pos0 = _dev(pos0, f32, dev).reshape(-1)
        self.vel0 = _dev(vel0, f32, dev).reshape(-1)
        self.length = _dev(length, f32, dev).reshape(-1)
        for name, t in (("pos0", self.pos0), ("vel0", self.vel0), ("length", self.length)):
            if t.numel() != n:
                raise IdmError(IDM_EINVAL, f"{name} has {t.numel()} entries; lane_offsets "
                                           f"describe {n} vehicles")
        n_par = 1 if shared_params else n
        self.shared_params = bool(shared_params)
        # shared mode: per-lane gradient sums [n_lanes, 6] fp64, the unit of the shard-count
        # invariant cross-rank reduction (parallel.reduce_step -> idm_reduce_shared)
        self.lane_grads = torch.zeros(self.n_lanes, 6, dtype=torch.float64, device=dev) \
            if shared_params else None
        if params is None:
            from .synth import init_params
            params = init_params(n_par)
        self.params = _dev(params, f32, dev).reshape(6, n_par).contiguous()
        self.grad_params = torch.zeros_like(self.params)
        self.adam_m = torch.zeros_like(self.params)
        self.adam_v = torch.zeros_like(self.params)
        self.grad_state0 = torch.zeros(2, n, dtype=f32, device=dev)
        self.traj = torch.empty(max_steps + 1, n, dtype=f32, device=dev)
        self.vel_traj = torch.empty(max_steps + 1, n, dtype=f32, device=dev) \
            if record_velocity else None
        self.grad_traj = torch.empty(max_steps + 1, n, dtype=f32, device=dev)
        self.state_out = torch.empty(2, n, dtype=f32, device=dev) if state_out else None
        # stage_obs: 0 none, 1 (or True) one staging buffer for step_host, 2 two (alternating)
        self.obs_stage = torch.empty(max_steps + 1, n, dtype=f32, device=dev) \
            if stage_obs else None
        self.obs_stage2 = torch.empty(max_steps + 1, n, dtype=f32, device=dev) \
            if int(stage_obs) >= 2 else None
        self.mask_stage = torch.empty(max_steps + 1, n, dtype=torch.uint8, device=dev) \
            if stage_mask else None
        self.loss_dev = torch.zeros(1, dtype=torch.float64, device=dev)
        self.max_steps = max_steps
        self.virtual_leader = virtual_leader
        if virtual_leader:
            # free per-step leader terms, paper init (10, 0) unless given
            self.vl_dp = _dev(vl_dp, f32, dev).reshape(max_steps, n).contiguous() \
                if vl_dp is not None else torch.full((max_steps, n), VL_INIT[0], dtype=f32,
                                                     device=dev)
            self.vl_dv = _dev(vl_dv, f32, dev).reshape(max_steps, n).contiguous() \
                if vl_dv is not None else torch.full((max_steps, n), VL_INIT[1], dtype=f32,
                                                     device=dev)
            self.vl_grad = torch.zeros(2, max_steps, n, dtype=f32, device=dev)
            self.vl_adam_m = torch.zeros(2, max_steps, n, dtype=f32, device=dev)
            self.vl_adam_v = torch.zeros(2, max_steps, n, dtype=f32, device=dev)
        d = IdmDesc()
        d.n_vehicles = n
        d.n_lanes = self.n_lanes
        d.lane_offsets = self.lane_offsets.data_ptr()
        d.pos0 = self.pos0.data_ptr()
        d.vel0 = self.vel0.data_ptr()
        d.length = self.length.data_ptr()
        d.params = self.params.data_ptr()
        d.grad_params = self.grad_params.data_ptr()
        d.adam_m = self.adam_m.data_ptr()
        d.adam_v = self.adam_v.data_ptr()
        d.grad_state0 = self.grad_state0.data_ptr()
        d.traj = self.traj.data_ptr()
        d.vel_traj = self.vel_traj.data_ptr() if self.vel_traj is not None else None
        d.grad_traj = self.grad_traj.data_ptr()
        d.state_out = self.state_out.data_ptr() if self.state_out is not None else None
        d.obs_stage = self.obs_stage.data_ptr() if self.obs_stage is not None else None
        d.obs_stage2 = self.obs_stage2.data_ptr() if self.obs_stage2 is not None else None
        d.mask_stage = self.mask_stage.data_ptr() if self.mask_stage is not None else None
        d.max_steps = max_steps
        d.ckpt_every = ckpt_every
        d.dt = dt
        d.a_min = a_min
        d.eps_gap = eps_gap
        d.param_mode = PARAMS_SHARED if shared_params else PARAMS_PER_VEHICLE
        d.lane_grads = self.lane_grads.data_ptr() if self.lane_grads is not None else None
        d.opt_mask = opt_mask
        d.stream = self.stream.cuda_stream
        if virtual_leader:
            d.leader_mode = LEADER_VIRTUAL
            d.vl_dp = self.vl_dp.data_ptr()
            d.vl_dv = self.vl_dv.data_ptr()
            d.vl_grad = self.vl_grad.data_ptr()
            d.vl_adam_m = self.vl_adam_m.data_ptr()
            d.vl_adam_v = self.vl_adam_v.data_ptr()
        nbytes = L.idm_workspace_bytes(C.byref(d))
        if nbytes == 0:
            raise IdmError(IDM_EINVAL, "malformed descriptor")
        self.workspace = torch.empty(nbytes + 256, dtype=torch.uint8, device=dev)
        base = self.workspace.data_ptr()
        d.workspace = (base + 255) & ~255
        d.workspace_bytes = nbytes
        self.desc = d
        h = C.c_void_p()
        with torch.cuda.device(dev):  # the handle belongs to the device current at idm_init
            rc = L.idm_init(C.byref(h), C.byref(d))
        if rc != IDM_OK:
            raise IdmError(rc, "idm_init failed (message on stderr)")
        self.handle = h
        self._lib = L
        self.steps = 0

    # -- C-ABI calls --------------------------------------------------------------------
    def _check(self, rc):
        if rc != IDM_OK:
            raise IdmError(rc, self._lib.idm_last_error(self.handle).decode())

    def forward(self, steps: int, history: bool = True):
        """idm_forward (history=False: idm_forward_ex IDM_FWD_NO_HISTORY, a prediction rollout
        that writes only traj / vel_traj / state_out; no backward may follow)."""
        if history:
            self._check(self._lib.idm_forward(self.handle, int(steps)))
        else:
            self._check(self._lib.idm_forward_ex(self.handle, int(steps), FWD_NO_HISTORY))
        self.steps = int(steps)

    def reduce_shared(self, lane_grads: torch.Tensor):
        """idm_reduce_shared: grad_params = the fixed-order sum of the GLOBAL per-lane rows
        (all ranks' lanes, [n_lanes_total, 6] fp64 on this device)."""
        assert lane_grads.dtype == torch.float64 and lane_grads.is_contiguous()
        assert lane_grads.device == self.device and lane_grads.dim() == 2
        self._check(self._lib.idm_reduce_shared(self.handle, _ptr(lane_grads),
                                                lane_grads.shape[0]))

    def loss_grad(self, obs: torch.Tensor, mask: torch.Tensor | None = None, kind: str = "l1",
                  sync: bool = True):
        assert obs.dtype == torch.float32 and obs.is_contiguous() and obs.device == self.device
        assert obs.numel() >= (self.steps + 1) * self.n
        if mask is not None:
            assert mask.dtype == torch.uint8 and mask.is_contiguous()
        out = C.c_double(0.0)
        self._check(self._lib.idm_loss_grad(self.handle, _ptr(obs), _ptr(mask), LOSS_KINDS[kind],
                                            _ptr(self.loss_dev), C.byref(out) if sync else None))
        return out.value if sync else None

    def backward(self):
        self._check(self._lib.idm_backward(self.handle))

    def adam_step(self, iteration: int, total: int = 500, lr0: float = 0.1, lr1: float = 0.01):
        self._check(self._lib.idm_adam_step(self.handle, iteration, total, lr0, lr1))

    def _no_sharded_shared(self, what: str):
        """The fused optimizer calls apply Adam inside the library, on this process's gradient
        sum: with shared parameters over several ranks that would skip the all-reduce."""
        import torch.distributed as dist
        if self.shared_params and dist.is_available() and dist.is_initialized() and \
                dist.get_world_size() > 1:
            raise IdmError(IDM_EINVAL, f"{what}: shared parameters over {dist.get_world_size()} "
                           "ranks need the gradient all-reduce between backward and adam_step "
                           "(parallel.reduce_step); use the separate calls")

    def fit_step(self, obs: torch.Tensor, kind: str = "l1", iteration: int = 0,
                 total: int = 500, lr0: float = 0.1, lr1: float = 0.01, steps: int | None = None,
                 sync: bool = False):
        """One fused iteration (idm_fit_step): forward + Eq. 4 + backward + Adam in two
        launches.  Missing observations are NaN.  Returns the loss if sync, else None (the
        loss is in self.loss_dev).  Shared parameters across several ranks need the gradient
        all-reduce between backward and Adam: use the separate calls there."""
        self._no_sharded_shared("fit_step")
        steps = self.max_steps if steps is None else int(steps)
        assert obs.dtype == torch.float32 and obs.is_contiguous() and obs.device == self.device
        assert obs.numel() >= (steps + 1) * self.n
        out = C.c_double(0.0)
        self._check(self._lib.idm_fit_step(self.handle, steps, _ptr(obs), None, LOSS_KINDS[kind],
                                           iteration, total, lr0, lr1, _ptr(self.loss_dev),
                                           C.byref(out) if sync else None))
        self.steps = steps
        return out.value if sync else None

    def fit(self, obs: torch.Tensor, iters: int, kind: str = "l1", iter0: int = 0,
            total: int = 500, lr0: float = 0.1, lr1: float = 0.01, steps: int | None = None,
            sync: bool = False):
        """`iters` fused iterations in ONE launch (idm_fit: on chip for horizons <=
        idm_fit_max_steps(), else each CTA runs its lane tile's whole fit with the history
        through memory): bit-identical to calling fit_step for iterations iter0 .. iter0+iters-1."""
        self._no_sharded_shared("fit")
        steps = self.max_steps if steps is None else int(steps)
        assert obs.dtype == torch.float32 and obs.is_contiguous() and obs.device == self.device
        assert obs.numel() >= (steps + 1) * self.n
        out = C.c_double(0.0)
        self._check(self._lib.idm_fit(self.handle, steps, _ptr(obs), LOSS_KINDS[kind], iter0,
                                      iters, total, lr0, lr1, _ptr(self.loss_dev),
                                      C.byref(out) if sync else None))
        self.steps = steps
        return out.value if sync else None

    def fit_steps(self, obs: torch.Tensor, iters: int, kind: str = "l1", iter0: int = 0,
                  total: int = 500, lr0: float = 0.1, lr1: float = 0.01,
                  steps: int | None = None, sync: bool = False):
        """`iters` fused iterations (any horizon) launched as ONE CUDA graph (idm_fit_steps):
        bit-identical to calling fit_step for iterations iter0 .. iter0+iters-1."""
        self._no_sharded_shared("fit_steps")
        steps = self.max_steps if steps is None else int(steps)
        assert obs.dtype == torch.float32 and obs.is_contiguous() and obs.device == self.device
        assert obs.numel() >= (steps + 1) * self.n
        out = C.c_double(0.0)
        self._check(self._lib.idm_fit_steps(self.handle, steps, _ptr(obs), LOSS_KINDS[kind],
                                            iter0, iters, total, lr0, lr1, _ptr(self.loss_dev),
                                            C.byref(out) if sync else None))
        self.steps = steps
        return out.value if sync else None

    def step_host(self, steps, obs_host: torch.Tensor, pos0_host=None, vel0_host=None,
                  mask_host=None, kind="l1", iteration=0, total=500, lr0=0.1, lr1=0.01):
        """One full iteration from HOST tensors (pinned for overlap); returns the loss."""
        for t in (obs_host, pos0_host, vel0_host, mask_host):
            assert t is None or (t.device.type == "cpu" and t.is_contiguous())
        out = C.c_double(0.0)
        self._check(self._lib.idm_step_host(
            self.handle, int(steps), _ptr(pos0_host), _ptr(vel0_host), _ptr(obs_host),
            _ptr(mask_host), LOSS_KINDS[kind], iteration, total, lr0, lr1, C.byref(out)))
        self.steps = int(steps)
        return out.value

    def step_host_async(self, steps, obs_host: torch.Tensor, pos0_host=None, vel0_host=None,
                        mask_host=None, kind="l1", iteration=0, total=500, lr0=0.1, lr1=0.01):
        """idm_step_host without the final synchronization (at most two in flight); the host
        tensors must stay alive and unchanged until the matching step_host_wait."""
        for t in (obs_host, pos0_host, vel0_host, mask_host):
            assert t is None or (t.device.type == "cpu" and t.is_contiguous())
        self._check(self._lib.idm_step_host_async(
            self.handle, int(steps), _ptr(pos0_host), _ptr(vel0_host), _ptr(obs_host),
            _ptr(mask_host), LOSS_KINDS[kind], iteration, total, lr0, lr1))
        self.steps = int(steps)

    def step_host_wait(self) -> float:
        """Retire the oldest step_host_async step; returns its loss."""
        out = C.c_double(0.0)
        self._check(self._lib.idm_step_host_wait(self.handle, C.byref(out)))
        return out.value

    def timing(self, enable: bool = True):
        """Bracket every launch with CUDA events on the handle's stream (benchmarks)."""
        self._check(self._lib.idm_timing_enable(self.handle, int(enable)))

    def timing_read(self) -> dict:
        """Summed device ms and launch counts per kernel class since the last read."""
        ms = (C.c_double * 6)()
        n = (C.c_int64 * 6)()
        self._check(self._lib.idm_timing_read(self.handle, ms, n))
        names = ("fwd", "loss", "reduce", "bwd", "adam", "other")
        return {k: (ms[i], n[i]) for i, k in enumerate(names)}

    def check(self):
        self._check(self._lib.idm_check(self.handle))

    @property
    def launch_count(self) -> int:
        return int(self._lib.idm_launch_count(self.handle))

    def close(self):
        if getattr(self, "handle", None):
            self._lib.idm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# C-ABI-named entry points -------------------------------------------------------------
def idm_init(lane_offsets, pos0, vel0, length, params=None, **kw) -> IdmSim:
    return IdmSim(lane_offsets, pos0, vel0, length, params, **kw)


def idm_forward(sim: IdmSim, steps: int):
    sim.forward(steps)


def idm_loss_grad(sim: IdmSim, obs, mask=None, kind="l1", sync=True):
    return sim.loss_grad(obs, mask, kind, sync)


def idm_backward(sim: IdmSim):
    sim.backward()


def idm_adam_step(sim: IdmSim, iteration: int, total: int = 500, lr0=0.1, lr1=0.01):
    sim.adam_step(iteration, total, lr0, lr1)


def idm_fit_step(sim: IdmSim, obs, kind="l1", iteration=0, total=500, lr0=0.1, lr1=0.01,
                 sync=False):
    return sim.fit_step(obs, kind, iteration, total, lr0, lr1, sync=sync)


def idm_state_from_obs(obs: torch.Tensor, dt: float = 0.1, steps: int | None = None,
                       stream: torch.cuda.Stream | None = None):
    """(pos0, vel0) device tensors [N] from step-major observations [(K+1), N] (NaN = missing):
    the paper's initialisation from the first two data points (include/idm.h)."""
    assert obs.dtype == torch.float32 and obs.is_contiguous() and obs.is_cuda and obs.dim() == 2
    L = load_library()
    steps = obs.shape[0] - 1 if steps is None else int(steps)
    n = obs.shape[1]
    pos0 = torch.empty(n, dtype=torch.float32, device=obs.device)
    vel0 = torch.empty(n, dtype=torch.float32, device=obs.device)
    st = stream or torch.cuda.current_stream(obs.device)
    with torch.cuda.device(obs.device):
        rc = L.idm_state_from_obs(_ptr(obs), n, steps, float(dt), _ptr(pos0), _ptr(vel0),
                                  C.c_void_p(st.cuda_stream))
    if rc != IDM_OK:
        raise IdmError(rc, "idm_state_from_obs failed")
    return pos0, vel0


def idm_plan_tiles(lane_offsets) -> "np.ndarray":
    """The lane -> CTA tile plan (host only): tile start vehicle indices, [n_tiles + 1]."""
    import numpy as np
    off = np.ascontiguousarray(np.asarray(lane_offsets, np.int32))
    lib = load_library()
    n_lanes, n = len(off) - 1, int(off[-1])
    nt = lib.idm_plan_tiles(off.ctypes.data, n_lanes, n, None)
    if nt < 0:
        raise IdmError(IDM_EINVAL, "malformed lane offsets or a lane longer than "
                                   "idm_max_lane_length()")
    out = np.zeros(nt + 1, np.int64)
    lib.idm_plan_tiles(off.ctypes.data, n_lanes, n, out.ctypes.data)
    return out


def from_workload(w, params=None, **kw) -> IdmSim:
    """IdmSim for a synth.Workload."""
    kw.setdefault("max_steps", w.K)
    kw.setdefault("dt", w.dt)
    return IdmSim(w.lane_offsets, w.p0, w.v0, w.length, params, **kw)
