"""CPU-side checks of the C-ABI boundary: libidm.so builds for sm_100a, loads, exports every
function include/idm.h declares, and refuses to run without a GPU (no CPU fallback)."""
import ctypes as C
import subprocess

import pytest

from paper_2412_16750_b200 import build as B


@pytest.fixture(scope="module")
def lib():
    B.build()
    from paper_2412_16750_b200 import idm
    return idm.load_library()


def test_header_declares_the_five_calls():
    from paper_2412_16750_b200 import idm
    syms = idm.header_symbols()
    for name in ("idm_init", "idm_forward", "idm_loss_grad", "idm_backward", "idm_adam_step"):
        assert name in syms
    assert len(syms) >= 12


def test_library_exports_every_header_symbol(lib):
    from paper_2412_16750_b200 import idm
    out = subprocess.run(["nm", "-D", "--defined-only", B.LIB], capture_output=True,
                         text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    missing = [s for s in idm.header_symbols() if s not in exported]
    assert not missing, missing
    for s in idm.header_symbols():
        assert hasattr(lib, s)


def test_library_is_sm100a_sass(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", B.LIB],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_workspace_bytes_and_descriptor_checks(lib):
    from paper_2412_16750_b200 import idm
    d = idm.IdmDesc()
    d.n_vehicles = 1000
    d.n_lanes = 10
    d.max_steps = 300
    d.ckpt_every = 4
    ws = lib.idm_workspace_bytes(C.byref(d))
    # the speed history dominates: every vehicle slot at every step, fp32 (tile-local; with
    # lane_offsets unreadable the size is for the worst-case tile count)
    assert ws >= 301 * 4 * 1000
    assert ws % 256 == 0
    for bad in (0, 1, 3, 5, 16):
        d.ckpt_every = bad
        assert lib.idm_workspace_bytes(C.byref(d)) == 0
    d.ckpt_every = 4
    d.n_vehicles = 0
    assert lib.idm_workspace_bytes(C.byref(d)) == 0
    assert lib.idm_max_lane_vehicles() >= 333  # NGSIM-shaped lanes (C3) fit one tile


def test_init_without_gpu_fails_loudly(lib):
    """No CPU fallback: with no usable device idm_init returns IDM_ECUDA (or EINVAL for a
    malformed descriptor), never a handle."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2412_16750_b200 import idm
    import numpy as np
    keep = [np.zeros(16, np.float32) for _ in range(12)]
    d = idm.IdmDesc()
    d.n_vehicles, d.n_lanes, d.max_steps, d.ckpt_every = 4, 1, 10, 4
    d.dt, d.a_min, d.eps_gap = 0.1, -10.0, 0.1
    ptrs = [k.ctypes.data for k in keep]
    (d.lane_offsets, d.pos0, d.vel0, d.length, d.params, d.grad_params, d.adam_m, d.adam_v,
     d.traj, d.grad_traj, d.grad_state0, d.state_out) = ptrs
    ws = np.zeros(lib.idm_workspace_bytes(C.byref(d)) + 512, np.uint8)
    d.workspace = (ws.ctypes.data + 255) & ~255
    d.workspace_bytes = lib.idm_workspace_bytes(C.byref(d))
    h = C.c_void_p()
    rc = lib.idm_init(C.byref(h), C.byref(d))
    assert rc == idm.IDM_ECUDA and not h.value
    with pytest.raises(idm.IdmError):
        idm.IdmSim([0, 4], np.zeros(4), np.ones(4), np.full(4, 4.0), max_steps=10)


def test_tile_plan_properties(lib):
    """The host tile planner (idm_plan_tiles, what idm_init uploads and idm_workspace_bytes
    sizes for): whole lanes per tile, at most the tile capacity per tile, greedy (consecutive
    tiles hold more than a tile's capacity), within the 2N/cap + 1 bound, and equal to a plain
    greedy packing written here; malformed offsets and over-long lanes are rejected."""
    import numpy as np
    from paper_2412_16750_b200 import idm
    cap = lib.idm_max_lane_vehicles()
    rng = np.random.default_rng(0)
    cases = [[100] * 2000, [1, 7, cap, 3, cap, 1], list(rng.integers(1, cap + 1, 3000)),
             [cap] * 5, [1] * 9000]
    for sizes in cases:
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
        tiles = idm.idm_plan_tiles(off)
        n = int(off[-1])
        assert tiles[0] == 0 and tiles[-1] == n
        lens = np.diff(tiles)
        assert np.all(lens > 0) and np.all(lens <= cap)
        assert set(tiles).issubset(set(off.tolist()))          # whole lanes only
        assert np.all(lens[:-1] + lens[1:] > cap)               # greedy
        assert len(lens) <= 2 * ((n + cap - 1) // cap) + 1
        expect, cur = [0], 0                                    # plain greedy packing
        for a, b in zip(off[:-1], off[1:]):
            if cur + (b - a) > cap:
                expect.append(int(a))
                cur = 0
            cur += int(b - a)
        expect.append(n)
        assert tiles.tolist() == expect
    mx = lib.idm_max_lane_length()
    assert mx == 8 * cap
    with pytest.raises(idm.IdmError):
        idm.idm_plan_tiles([0, mx + 1])
    with pytest.raises(idm.IdmError):
        idm.idm_plan_tiles([0, 5, 3])


def test_tile_plan_long_lanes(lib):
    """Lanes longer than a tile (up to idm_max_lane_length()) run over thread-block clusters of
    cs = ceil(longest / cap) consecutive tiles: every such lane starts at a tile index that is a
    multiple of cs and fills full tiles of cap vehicles (the last one the remainder, then empty
    padding tiles); short lanes still pack greedily into whole-lane tiles; the tile count is a
    multiple of cs; every vehicle is in exactly one tile."""
    import numpy as np
    from paper_2412_16750_b200 import idm
    cap = lib.idm_max_lane_vehicles()
    for sizes in ([cap + 1], [3, 2 * cap + 5, 7, 0, 100, 3 * cap, 1, cap, 40],
                  [5] * 300 + [8 * cap] + [5] * 300, [cap + 1, cap + 1, 1]):
        off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int32)
        tiles = idm.idm_plan_tiles(off)
        n = int(off[-1])
        lens = np.diff(tiles)
        cs = max(1, -(-max(sizes) // cap))
        assert tiles[0] == 0 and tiles[-1] == n and np.all(lens >= 0) and np.all(lens <= cap)
        assert len(lens) % cs == 0
        for a, b in zip(off[:-1], off[1:]):
            a, b = int(a), int(b)
            if b - a <= cap:
                if b > a:  # whole lane inside one tile
                    t = np.searchsorted(tiles, a, side="right") - 1
                    assert tiles[t] <= a and b <= tiles[t + 1]
                continue
            t = int(np.where(tiles[:-1] == a)[0][-1])  # the first tile of the lane (after pads)
            assert t % cs == 0
            nfull = (b - a) // cap
            for c in range(cs):
                lo, hi = tiles[t + c], tiles[t + c + 1]
                if c < nfull:
                    assert (lo, hi) == (a + c * cap, a + (c + 1) * cap)
                elif c == nfull:
                    assert (lo, hi) == (a + c * cap, b)
                else:
                    assert lo == hi == b
