"""CPU tests of the C ABI and the host-side mirror (no GPU needed).

* the shared library loads and exports every symbol include/flocksim_b200.h
  declares, and the ctypes table covers them;
* argument errors are detected before any launch and map to the reference's
  exception types and messages ("dt", "length", ...: dynamics.py:257-260,
  control.py:362-363);
* host-side parameter validation mirrors RobotParams / ControlGains /
  ControlLimits (test_dynamics.py:37-62, test_control.py:40-59).
"""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2305_16510_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flocksim_b200.h")


def header_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(fs_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2305_16510_b200 import build
    build.build()
    return N.load()


def test_library_exports_every_declared_symbol(lib):
    names = header_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), f"{name} declared in the header but not exported"
    assert set(names) == set(N.EXPORTED_SYMBOLS)


def test_abi_version(lib):
    assert lib.fs_abi_version() == N.FS_ABI_VERSION


def test_ctypes_struct_sizes_match_header_layout():
    # float64 parameter blocks: 2 + 9 + 9 + 1 + 3 + 2 + 1 doubles
    assert C.sizeof(N.fs_robot) == 27 * 8
    assert C.sizeof(N.fs_gains) == 12 * 8
    assert C.sizeof(N.fs_limits) == 3 * 8
    assert C.sizeof(N.fs_airframe) == 8 + 4 * 48


def _desc(**kw):
    d = N.fs_step_desc()
    d.n = 8
    d.state_in = d.state_out = C.c_void_p(0x1000)
    d.state_in_stride = d.state_out_stride = 8
    d.cmd = C.c_void_p(0x2000)
    d.cmd_stride = 8
    d.mode = N.FS_MODE_VELOCITY
    d.integrate = 1
    d.dt = 0.01
    for k, v in kw.items():
        setattr(d, k, v)
    return d


def _params():
    from paper_2305_16510_b200.control import ControlGains, ControlLimits
    from paper_2305_16510_b200.dynamics import RobotParams
    return RobotParams().native(), ControlGains().native(), ControlLimits().native()


@pytest.mark.parametrize("field,value,msg", [
    ("dt", 0.2, "dt"), ("dt", 0.0, "dt"), ("dt", -0.01, "dt"),
    ("mode", 9, "mode"), ("state_in_stride", 4, "stride"),
    ("stats_nslots", 3, "power of two"), ("reset_prob", 1.5, "reset_prob"),
])
def test_step_rejects_bad_arguments_before_launch(lib, field, value, msg):
    d = _desc(**{field: value})
    if field == "stats_nslots":
        d.stats_slots = C.c_void_p(0x3000)
    r, g, l = _params()
    rc = lib.fs_step(C.byref(d), r, g, l, None, None)
    assert rc == N.FS_EINVAL
    assert msg in lib.fs_last_error().decode()


def test_mixed_mode_requires_mode_plane(lib):
    d = _desc(mode=N.FS_MODE_MIXED)
    r, g, l = _params()
    assert lib.fs_step(C.byref(d), r, g, l, None, None) == N.FS_EINVAL
    assert "mode_per_vehicle" in lib.fs_last_error().decode()


def test_rollout_and_integrate_validation(lib):
    r, g, l = _params()
    d = _desc()
    assert lib.fs_rollout(C.byref(d), r, g, l, None, 0, None) == N.FS_EINVAL
    assert lib.fs_integrate(4, C.c_void_p(0x1000), 4, C.c_void_p(0x2000), 4, r, 0.5,
                            C.c_void_p(0x3000), 4, None, None) == N.FS_EINVAL
    assert "dt" in lib.fs_last_error().decode()
    # n == 0 is a no-op, not an error
    d0 = _desc(n=0)
    assert lib.fs_step(C.byref(d0), r, g, l, None, None) == N.FS_OK


def test_chained_step_validation(lib):
    """tile_sync (chained steps): counter count per FS_SYNC_GRANULE vehicles;
    only integrating fs_step calls take it (validated before any launch)."""
    assert lib.fs_tile_sync_len(0) == 0
    assert lib.fs_tile_sync_len(1) == 1
    assert lib.fs_tile_sync_len(N.FS_SYNC_GRANULE) == 1
    assert lib.fs_tile_sync_len(N.FS_SYNC_GRANULE + 1) == 2
    assert lib.fs_tile_sync_len(1 << 24) == (1 << 24) // N.FS_SYNC_GRANULE
    r, g, l = _params()
    d = _desc(integrate=0, tile_sync=C.c_void_p(0x4000), sync_wait=1, sync_post=2)
    assert lib.fs_step(C.byref(d), r, g, l, None, None) == N.FS_EINVAL
    assert "integrate" in lib.fs_last_error().decode()
    d = _desc(tile_sync=C.c_void_p(0x4000))
    assert lib.fs_rollout(C.byref(d), r, g, l, None, 4, None) == N.FS_EINVAL
    assert "tile_sync" in lib.fs_last_error().decode()


def test_check_maps_status_to_reference_exceptions(lib):
    r, g, l = _params()
    d = _desc(dt=0.5)
    rc = lib.fs_step(C.byref(d), r, g, l, None, None)
    with pytest.raises(ValueError, match="dt"):
        N.check(rc, "fs_step")


def test_tuning_keys(lib):
    assert lib.fs_set_tuning(99, 1) == N.FS_EINVAL
    assert lib.fs_set_tuning(N.FS_TUNE_KERNEL, 0) == N.FS_OK
    assert lib.fs_set_tuning(N.FS_TUNE_NCW, 5) == N.FS_EINVAL
    assert lib.fs_set_tuning(N.FS_TUNE_NCW, 20) == N.FS_OK
    assert lib.fs_set_tuning(N.FS_TUNE_NCW, 0) == N.FS_OK


# --- host-side validation mirrors the reference ------------------------------

def test_robot_params_validation():
    from paper_2305_16510_b200.dynamics import RobotParams
    assert RobotParams().hover_thrust == pytest.approx(9.81)
    with pytest.raises(ValueError, match="mass"):
        RobotParams(mass=-1.0)
    j = np.diag([0.01, 0.01, 0.02])
    j[0, 1] = 1e-3
    with pytest.raises(ValueError, match="symmetric"):
        RobotParams(inertia=j)
    with pytest.raises(ValueError, match="positive definite"):
        RobotParams(inertia=np.diag([0.01, -0.01, 0.02]))
    with pytest.raises(ValueError, match="thrust_max"):
        RobotParams(thrust_max=5.0)
    with pytest.raises(ValueError, match="moment_max"):
        RobotParams(moment_max=[1.0, 0.0, 1.0])


def test_robot_params_native_struct():
    from paper_2305_16510_b200.dynamics import RobotParams
    r = RobotParams(inertia=[[0.02, 0.001, 0], [0.001, 0.02, 0], [0, 0, 0.03]]).native()
    inv = np.linalg.inv(np.array([[0.02, 0.001, 0], [0.001, 0.02, 0], [0, 0, 0.03]]))
    np.testing.assert_allclose(np.array(r.inertia_inv[:]).reshape(3, 3), inv, rtol=1e-6)
    assert r.gimbal_cos == np.cos(1e-6)


def test_gains_and_limits_validation():
    from paper_2305_16510_b200.control import ControlGains, ControlLimits
    with pytest.raises(ValueError):
        ControlGains(attitude=[8.0, 0.0, 2.0])
    with pytest.raises(ValueError):
        ControlLimits(max_tilt=2.0)
    with pytest.raises(ValueError):
        ControlLimits(max_speed_cmd=0.0)


def test_step_batch_validation_precedes_device_work():
    from paper_2305_16510_b200.dynamics import RobotParams, step_batch

    class Stub:
        def __init__(self, n):
            self.n = n

    with pytest.raises(ValueError, match="dt"):
        step_batch(Stub(2), RobotParams(), Stub(2), 0.2)
    with pytest.raises(ValueError, match="length"):
        step_batch(Stub(2), RobotParams(), Stub(3), 0.01)


def test_control_batch_length_validation_precedes_device_work():
    from paper_2305_16510_b200.control import ControlGains, control_batch
    from paper_2305_16510_b200.dynamics import RobotParams

    class Stub:
        def __init__(self, n):
            self.n = n

    with pytest.raises(ValueError, match="command batch length"):
        control_batch(Stub(2), Stub(3), ControlGains(), RobotParams())


def test_airframe_native_layout():
    from paper_2305_16510_b200.allocation import HEXAROTOR, QUAD_X
    for frame in (QUAD_X, HEXAROTOR):
        f = frame.native()
        assert f.n_rotors == frame.n_rotors
        pinv = np.array(f.pinv[:]).reshape(N.FS_MAX_ROTORS, 4)[:frame.n_rotors]
        alloc = np.array(f.alloc[:]).reshape(4, N.FS_MAX_ROTORS)[:, :frame.n_rotors]
        np.testing.assert_allclose(alloc @ pinv, np.eye(4), atol=1e-5)


def test_obstacle_poses_validation(lib):
    """fs_obstacles_poses (World.instances on demand) checks its tables,
    planes, counters and bounds before any launch."""
    ob = N.fs_obstacles()
    bounds = (C.c_double * 3)(12.0, 12.0, 6.0)
    assert lib.fs_obstacles_poses(None, 4, 0, 1, None, bounds, None) == N.FS_EINVAL
    assert lib.fs_obstacles_poses(C.byref(ob), -1, 0, 1, None, bounds, None) == N.FS_EINVAL
    assert lib.fs_obstacles_poses(C.byref(ob), 0, 0, 1, None, bounds, None) == N.FS_OK
    ob.instances_per_env = 2
    assert lib.fs_obstacles_poses(C.byref(ob), 4, 0, 1, None, bounds, None) == N.FS_EINVAL
    assert "pose planes" in lib.fs_last_error().decode()
    ob.inst_pose = ob.inst_proto = ob.classes = C.c_void_p(0x3000).value
    ob.plane_stride = 2
    assert lib.fs_obstacles_poses(C.byref(ob), 4, 0, 1, C.c_void_p(0x4000), bounds,
                                  None) == N.FS_EINVAL
    assert "stride" in lib.fs_last_error().decode()


@pytest.mark.parametrize("n,w,threads", [(0, 3, 0), (1, 4, 1), (1000, 3, 2), (300001, 4, 0),
                                         (200003, 1, 7)])
def test_host_pack_unpack_f64(lib, n, w, threads):
    """fs_host_pack_f64 / fs_host_unpack_f64 (host only, no GPU): float64
    (n, w) rows <-> fp32 planes with a plane stride, rounded to nearest like
    numpy's astype, over any thread count."""
    rng = np.random.default_rng(n + w)
    src = rng.normal(size=(n, w)) * 10.0 ** rng.integers(-3, 4, size=(n, w))
    stride = n + 5
    planes = np.full((w, stride), np.nan, np.float32)
    assert lib.fs_host_pack_f64(src.ctypes.data, n, w, w, planes.ctypes.data, stride,
                                threads) == 0
    assert np.array_equal(planes[:, :n], src.astype(np.float32).T)
    assert np.isnan(planes[:, n:]).all()                # nothing past n
    back = np.empty((n, w), np.float64)
    assert lib.fs_host_unpack_f64(planes.ctypes.data, stride, n, w, back.ctypes.data, w,
                                  threads) == 0
    assert np.array_equal(back, src.astype(np.float32).astype(np.float64))
    assert lib.fs_host_pack_f64(src.ctypes.data, n, w, w - 1, planes.ctypes.data, stride,
                                threads) == 22          # ld < w
    if n > 0:                                           # plane stride < n
        assert lib.fs_host_unpack_f64(planes.ctypes.data, n - 1, n, w, back.ctypes.data, w,
                                      threads) == 22
