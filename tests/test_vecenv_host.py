"""CPU tests of the RL bindings' host side (no GPU).

* the config loader mirrors flocksim.config.load_config / from_dict
  (config.py:100-203): defaults, unknown keys with their location, version
  pin, per-section construction errors as ConfigError, 1-D inertia -> diag;
  content the GPU World does not model is rejected, not dropped;
* VecEnvHandle's error behaviour (pkg/bindings/tests/test_bindings.py):
  shape mismatch, closed handle, concurrent step, schema pin, disabled
  camera -- checked on a stub world, before any device work;
* fs_vecenv_step rejects bad arguments before any launch.
"""

import ctypes as C
import threading

import numpy as np
import pytest

from paper_2305_16510_b200 import _native as N
from paper_2305_16510_b200 import config as cfgmod
from paper_2305_16510_b200 import rl
from paper_2305_16510_b200.world import ConfigError

BASE_YAML = """
version: 1
env:
  num_envs: {n}
  seed: {seed}
  control_mode: {mode}
  bounds: [10.0, 10.0, 5.0]
  episode_max_steps: 120
  wall_enabled: true
"""


def write(tmp_path, text, name="sim.yaml"):
    p = tmp_path / name
    p.write_text(text)
    return p


# ---------------------------------------------------------------- config loader

def test_load_config_defaults_and_values(tmp_path):
    cfg = cfgmod.load_config(write(tmp_path, BASE_YAML.format(n=4, seed=3, mode="attitude")))
    assert cfg.env.num_envs == 4 and cfg.env.seed == 3 and cfg.env.control_mode == "attitude"
    assert cfg.env.wall_enabled and cfg.env.episode_max_steps == 120
    assert cfg.robot.mass == 1.0 and cfg.limits.max_tilt == 0.6
    np.testing.assert_array_equal(cfg.gains.velocity, [3.0, 3.0, 3.0])
    assert cfg.reward.c_success == 10.0


def test_empty_file_is_all_defaults(tmp_path):
    cfg = cfgmod.load_config(write(tmp_path, ""))
    assert cfg.env.num_envs == 16 and cfg.env.control_mode == "velocity"


def test_inertia_vector_becomes_diagonal(tmp_path):
    cfg = cfgmod.load_config(write(tmp_path, "robot: {inertia: [0.02, 0.03, 0.04]}\n"))
    np.testing.assert_array_equal(cfg.robot.inertia, np.diag([0.02, 0.03, 0.04]))


@pytest.mark.parametrize("text,match", [
    ("bogus: 1\n", "config root"),
    ("env: {num_envs: 2, colour: red}\n", r"in env"),
    ("robot: {mass: -1.0}\n", "robot"),
    ("gains: {attitude: [1, 0, 1]}\n", "gains"),
    ("limits: {max_tilt: 2.0}\n", "limits"),
    ("env: {dt: 0.5}\n", "dt"),
    ("env: {control_mode: position}\n", "control_mode"),
    ("version: 2\n", "version"),
    ("- 1\n- 2\n", "mapping"),
    ("env: [1, 2\n", "YAML"),
    ("asset_classes: [{name: x, oops: 1}]\n", "asset_classes"),
    ("asset_classes: [{count_per_env: 1}]\n", "missing class name"),
    ("asset_classes: [{name: x, count_per_env: -1}]\n", r"asset_classes\[0\]"),
    ("camera: {lens: 3}\n", "camera"),
    ("camera: {width: 0}\n", "camera"),
])
def test_config_errors(tmp_path, text, match):
    with pytest.raises(ConfigError, match=match):
        cfgmod.load_config(write(tmp_path, text))


def test_camera_and_asset_classes_parse(tmp_path):
    """config.py:166-180 (the reference's test_config.py:41-63)."""
    cfg = cfgmod.load_config(write(tmp_path, """
asset_classes:
  - name: trees
    count_per_env: 3
    position_min: [0.1, 0.1, 0.0]
    position_max: [0.9, 0.9, 0.0]
    frozen: [null, null, 0.0]
    segmentation_id: 4
camera: {width: 64, height: 48, randomize_euler: [0.01, 0.0, 0.0]}
"""))
    c = cfg.asset_classes[0]
    assert c.name == "trees" and c.count_per_env == 3 and c.segmentation_id == 4
    assert c.frozen == (None, None, 0.0)
    np.testing.assert_array_equal(c.position_max, [0.9, 0.9, 0.0])
    assert (cfg.camera.width, cfg.camera.height) == (64, 48)
    assert cfg.camera.randomize_euler[0] == 0.01


def test_disabled_camera_section_is_accepted(tmp_path):
    cfg = cfgmod.load_config(write(tmp_path, "camera: {enabled: false, width: 8}\n"))
    assert cfg.camera is None


def test_missing_file_is_config_error(tmp_path):
    with pytest.raises(ConfigError):
        rl.make(tmp_path / "missing.yaml")


def test_shipped_demo_schema(tmp_path):
    """The reference's pkg/configs/demo.yaml schema (every section, every key)."""
    text = """
version: 1
robot: {mass: 1.0, inertia: [0.01, 0.01, 0.02], collision_radius: 0.2, thrust_max: 25.0,
        moment_max: [2.0, 2.0, 1.0], gravity: 9.81}
gains: {attitude: [8.0, 8.0, 2.0], rate: [1.2, 1.2, 0.6], velocity: [3.0, 3.0, 3.0]}
limits: {max_tilt: 0.6, max_speed_cmd: 5.0, max_yaw_rate: 3.0}
env: {num_envs: 16, bounds: [10.0, 10.0, 5.0], episode_max_steps: 1000, dt: 0.01,
      control_mode: velocity, seed: 0, wall_enabled: false, goal_min: [0.1, 0.1, 0.2],
      goal_max: [0.9, 0.9, 0.8], spawn_min: [0.1, 0.1, 0.2], spawn_max: [0.9, 0.9, 0.8]}
reward: {c_dist: 0.1, c_vel: 0.01, c_step: 0.01, c_success: 10.0, c_crash: 10.0,
         success_radius: 0.2}
"""
    cfg = cfgmod.load_config(write(tmp_path, text))
    assert cfg.env.num_envs == 16 and cfg.robot.thrust_max == 25.0


# ---------------------------------------------------------------- handle logic

class StubWorld:
    """Enough of World for the handle's host-side checks (no device)."""

    def __init__(self, n=4, mode="velocity"):
        from paper_2305_16510_b200.world import EnvConfig
        self.num_envs = n
        self.env = EnvConfig(num_envs=n, control_mode=mode)
        self.device = "cpu"
        self.camera = None
        self.stepped = []

    def step_actions(self, actions):
        self.stepped.append(actions)
        raise AssertionError("reached device work")

    def observations(self):
        return np.zeros((self.num_envs, 16))


def test_spaces():
    h = rl.VecEnvHandle(StubWorld(n=4))
    assert h.observation_space.shape == (4, 16)
    assert h.action_space.shape == (4, rl.ACTION_DIM) == (4, 4)
    assert h.action_space.low == -1.0 and h.action_space.high == 1.0
    assert h.num_envs == 4 and h.control_mode == "velocity"


@pytest.mark.parametrize("shape", [(3, 4), (4, 3), (4,), (4, 4, 1)])
def test_shape_mismatch_before_device_work(shape):
    w = StubWorld(n=4)
    h = rl.VecEnvHandle(w)
    with pytest.raises(rl.ShapeMismatchError):
        h.step(np.zeros(shape))
    assert not w.stepped


def test_nan_actions_are_invalid_commands():
    from paper_2305_16510_b200.control import InvalidCommandError
    w = StubWorld(n=4)
    h = rl.VecEnvHandle(w)
    a = np.zeros((4, 4))
    a[2, 1] = np.nan
    with pytest.raises(InvalidCommandError):
        h.step(a)
    assert not w.stepped


def test_closed_handle():
    with rl.VecEnvHandle(StubWorld()) as h:
        h.observations()
    for call in (h.observations, h.reset, h.render_depth, lambda: h.step(np.zeros((4, 4)))):
        with pytest.raises(rl.ClosedHandleError):
            call()


def test_step_in_flight_enforced():
    h = rl.VecEnvHandle(StubWorld())
    assert h._step_lock.acquire(blocking=False)
    try:
        with pytest.raises(rl.ConcurrentStepError):
            h.step(np.zeros((4, 4)))
    finally:
        h._step_lock.release()


def test_concurrent_steps_from_threads_one_wins():
    """Two threads stepping at once: one proceeds, the other gets
    ConcurrentStepError (vec_env.py:117-118)."""
    gate, release = threading.Event(), threading.Event()

    class Slow(StubWorld):
        def step_actions(self, actions):
            gate.set()
            release.wait(5)
            from paper_2305_16510_b200.world import StepResult
            return StepResult(None, None, None, None, {})

    h = rl.VecEnvHandle(Slow())
    t = threading.Thread(target=h.step, args=(np.zeros((4, 4)),))
    t.start()
    assert gate.wait(5)
    with pytest.raises(rl.ConcurrentStepError):
        h.step(np.zeros((4, 4)))
    release.set()
    t.join()


def test_schema_version_checked(monkeypatch):
    monkeypatch.setattr(cfgmod, "CONFIG_VERSION", 2)
    with pytest.raises(RuntimeError, match="schema"):
        rl.VecEnvHandle(StubWorld())


def test_render_depth_camera_disabled():
    with pytest.raises(rl.CameraDisabledError):
        rl.VecEnvHandle(StubWorld()).render_depth()


# ---------------------------------------------------------------- C ABI

@pytest.fixture(scope="module")
def lib():
    from paper_2305_16510_b200 import build
    build.build()
    return N.load()


def _wdesc(mode=N.FS_MODE_VELOCITY, n=8):
    w = N.fs_world_desc()
    d = w.step
    d.n = n
    d.state_in = d.state_out = C.c_void_p(0x1000)
    d.state_in_stride = d.state_out_stride = n
    d.mode = mode
    d.integrate = 1
    d.dt = 0.01
    w.goal = C.c_void_p(0x2000)
    w.goal_stride = n
    w.steps_in_episode = C.c_void_p(0x3000)
    w.reset_counter = C.c_void_p(0x4000)
    w.pending_reset = C.c_void_p(0x5000)
    w.obs = C.c_void_p(0x6000)
    w.obs_stride = n
    w.reward = C.c_void_p(0x7000)
    w.info = C.c_void_p(0x8000)
    return w


@pytest.mark.parametrize("mode,dtype,stride,addr,msg", [
    (N.FS_MODE_POSITION, N.FS_DTYPE_F32, 4, 0x9000, "attitude or velocity"),
    (N.FS_MODE_MIXED, N.FS_DTYPE_F32, 4, 0x9000, "attitude or velocity"),
    (N.FS_MODE_VELOCITY, 7, 4, 0x9000, "dtype"),
    (N.FS_MODE_VELOCITY, N.FS_DTYPE_F32, 3, 0x9000, "stride"),
    (N.FS_MODE_VELOCITY, N.FS_DTYPE_F64, 6, 0x9000, "stride"),
    (N.FS_MODE_ATTITUDE, N.FS_DTYPE_F32, 4, 0x9004, "aligned"),
    (N.FS_MODE_ATTITUDE, N.FS_DTYPE_F32, 4, 0, "aligned"),
])
def test_vecenv_step_rejects_bad_arguments_before_launch(lib, mode, dtype, stride, addr, msg):
    from paper_2305_16510_b200.control import ControlGains, ControlLimits
    from paper_2305_16510_b200.dynamics import RobotParams
    w = _wdesc(mode)
    cfg = N.fs_world_cfg()
    cfg.episode_max_steps = 10
    rc = lib.fs_vecenv_step(C.byref(w), C.byref(cfg), RobotParams().native(),
                            ControlGains().native(), ControlLimits().native(),
                            C.c_void_p(addr), dtype, stride, None)
    assert rc == N.FS_EINVAL
    assert msg in lib.fs_last_error().decode()


def test_vecenv_step_empty_world_is_noop(lib):
    from paper_2305_16510_b200.control import ControlGains, ControlLimits
    from paper_2305_16510_b200.dynamics import RobotParams
    w = _wdesc(n=0)
    cfg = N.fs_world_cfg()
    cfg.episode_max_steps = 10
    assert lib.fs_vecenv_step(C.byref(w), C.byref(cfg), RobotParams().native(),
                              ControlGains().native(), ControlLimits().native(), None,
                              N.FS_DTYPE_F32, 4, None) == N.FS_OK
