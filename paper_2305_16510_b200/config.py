"""Simulator config files -- drop-in for ``flocksim.config.load_config``.

Mirrors /root/reference/pkg/src/flocksim/config.py:100-203: a YAML mapping
with sections {robot, gains, limits, env, asset_classes, camera, reward},
shipped defaults for every key, unknown keys rejected with their location,
``version`` pinned to CONFIG_VERSION, and every construction error surfaced
as ConfigError with its section.  Asset classes build
assets.AssetClassConfig and an enabled camera camera.CameraConfig, as in the
reference (config.py:166-180).
"""

from __future__ import annotations

from pathlib import Path

import numpy as np
import yaml

from .assets import AssetClassConfig
from .camera import CameraConfig
from .control import ControlGains, ControlLimits
from .dynamics import RobotParams
from .world import ConfigError, EnvConfig, RewardConfig, SimConfig

CONFIG_VERSION = 1             # flocksim/__init__.py:19

_ROBOT_KEYS = ("mass", "inertia", "collision_radius", "thrust_max",
               "moment_max", "gravity", "v_limit", "omega_limit")
# "position" is the EXTENSION position-loop gain
_GAINS_KEYS = ("attitude", "rate", "velocity", "position")
_LIMITS_KEYS = ("max_tilt", "max_speed_cmd", "max_yaw_rate")
_ENV_KEYS = ("num_envs", "bounds", "episode_max_steps", "dt", "control_mode",
             "seed", "wall_enabled", "wall_thickness", "wall_segmentation_id",
             "goal_min", "goal_max", "spawn_min", "spawn_max")
_CLASS_KEYS = ("name", "count_per_env", "position_min", "position_max",
               "euler_min", "euler_max", "frozen", "segmentation_id",
               "collision_enabled")
_CAMERA_KEYS = ("enabled", "width", "height", "hfov", "max_range",
                "mount_position", "mount_euler", "randomize_position",
                "randomize_euler")
_REWARD_KEYS = ("c_dist", "c_vel", "c_step", "c_success", "c_crash",
                "success_radius")
_ROOT_KEYS = ("version", "robot", "gains", "limits", "env", "asset_classes",
              "camera", "reward")


def _check_keys(section: dict, allowed, where: str) -> None:
    unknown = sorted(set(section) - set(allowed))
    if unknown:
        raise ConfigError(f"unknown key(s) {unknown} in {where}; allowed: {sorted(allowed)}")


def _section(data: dict, name: str, allowed) -> dict:
    sec = data.get(name) or {}
    if not isinstance(sec, dict):
        raise ConfigError(f"section {name} must be a mapping")
    sec = dict(sec)
    _check_keys(sec, allowed, name)
    return sec


def _build(cls, section: dict, where: str):
    try:
        return cls(**section)
    except (ValueError, TypeError) as exc:
        if isinstance(exc, ConfigError):
            raise
        raise ConfigError(f"{where}: {exc}") from exc


def from_dict(data) -> SimConfig:
    """Build a SimConfig from parsed YAML content (config.py:131-189)."""
    if data is None:
        data = {}
    if not isinstance(data, dict):
        raise ConfigError("config root must be a mapping")
    _check_keys(data, _ROOT_KEYS, "config root")
    version = data.get("version", CONFIG_VERSION)
    if version != CONFIG_VERSION:
        raise ConfigError(f"config version {version} not supported (expected {CONFIG_VERSION})")

    robot_sec = _section(data, "robot", _ROBOT_KEYS)
    if "inertia" in robot_sec:
        inertia = np.asarray(robot_sec["inertia"], dtype=np.float64)
        robot_sec["inertia"] = np.diag(inertia) if inertia.ndim == 1 else inertia
    robot = _build(RobotParams, robot_sec, "robot")
    gains = _build(ControlGains, _section(data, "gains", _GAINS_KEYS), "gains")
    limits = _build(ControlLimits, _section(data, "limits", _LIMITS_KEYS), "limits")
    env = _build(EnvConfig, _section(data, "env", _ENV_KEYS), "env")

    classes = []
    for i, sec in enumerate(data.get("asset_classes") or []):
        where = f"asset_classes[{i}]"
        if not isinstance(sec, dict):
            raise ConfigError(f"{where} must be a mapping")
        sec = dict(sec)
        _check_keys(sec, _CLASS_KEYS, where)
        if "name" not in sec:
            raise ConfigError(f"{where}: missing class name")
        classes.append(_build(AssetClassConfig, sec, where))
    camera = None
    cam = data.get("camera")
    if cam is not None:
        if not isinstance(cam, dict):
            raise ConfigError("section camera must be a mapping")
        cam = dict(cam)
        _check_keys(cam, _CAMERA_KEYS, "camera")
        if cam.pop("enabled", True):
            camera = _build(CameraConfig, cam, "camera")
    reward = _build(RewardConfig, _section(data, "reward", _REWARD_KEYS), "reward")
    return SimConfig(robot=robot, gains=gains, limits=limits, env=env,
                     asset_classes=classes, camera=camera, reward=reward)


def load_config(path) -> SimConfig:
    """Load and validate a simulator config file (config.py:192-203)."""
    path = Path(path)
    try:
        text = path.read_text()
    except OSError as exc:
        raise ConfigError(f"cannot read config {path}: {exc}") from exc
    try:
        data = yaml.safe_load(text)
    except yaml.YAMLError as exc:
        raise ConfigError(f"{path}: YAML parse error: {exc}") from exc
    return from_dict(data)


__all__ = ["CONFIG_VERSION", "ConfigError", "from_dict", "load_config"]
