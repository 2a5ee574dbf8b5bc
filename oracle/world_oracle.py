"""CPU oracle of the free-space World.step epilogue -- TEST INFRASTRUCTURE.

Restates, in float64 NumPy over the planar (13, E) state layout, the
reference's environment step for a world without obstacles or camera:

  World.step            world.py:277-326  (auto-reset-then-void ordering,
                                           bookkeeping, terminated/truncated)
  check_collisions      world.py:95-106   (sphere vs. env bounds; no primitives)
  reward_goal_reaching  world.py:109-116
  World.observations    world.py:331-342  (16 values, goal in the vehicle frame)
  World._place_robot_and_goal  world.py:213-227  (robot at rest at the spawn)
  VecEnvHandle._commands_from_actions
                        pkg/bindings/src/flocksim_rl/vec_env.py:85-104
                        (clip to [-1, 1], denormalize against the limits)

The reference draws re-spawn points from NumPy Philox streams per (seed,
env, reset) (assets.py:310-315), which the device cannot reproduce; the
oracle therefore takes the re-spawn points as an input (`spawn_fn`).  Pinned
against the reference World (tests/golden/world.npz, make_golden_world.py).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import flocksim_oracle as O


@dataclass
class EnvCfg:
    """EnvConfig subset (config.py:29-60)."""

    bounds: np.ndarray = field(default_factory=lambda: np.array([10.0, 10.0, 5.0]))
    episode_max_steps: int = 1000
    dt: float = 0.01
    goal_min: np.ndarray = field(default_factory=lambda: np.array([0.1, 0.1, 0.2]))
    goal_max: np.ndarray = field(default_factory=lambda: np.array([0.9, 0.9, 0.8]))
    spawn_min: np.ndarray = field(default_factory=lambda: np.array([0.1, 0.1, 0.2]))
    spawn_max: np.ndarray = field(default_factory=lambda: np.array([0.9, 0.9, 0.8]))
    collision_radius: float = 0.2      # RobotParams.collision_radius (dynamics.py:57)


@dataclass
class RewardCfg:
    """RewardConfig (config.py:82-90)."""

    c_dist: float = 0.1
    c_vel: float = 0.01
    c_step: float = 0.01
    c_success: float = 10.0
    c_crash: float = 10.0
    success_radius: float = 0.2


def reward_goal_reaching(p, v, goal, collided, cfg: RewardCfg):
    """world.py:109-116 on planar (3, E) arrays."""
    d = np.linalg.norm(goal - p, axis=0)
    speed = np.linalg.norm(v, axis=0)
    return (-d * cfg.c_dist - speed * cfg.c_vel - cfg.c_step
            + cfg.c_success * (d < cfg.success_radius)
            - cfg.c_crash * np.asarray(collided, dtype=np.float64))


def out_of_bounds(p, bounds, r):
    """world.py:103-106 (p within r of any bounding plane)."""
    b = np.asarray(bounds, dtype=np.float64)[:, None]
    return ((p < r) | (p > b - r)).any(axis=0)


def observations(s, goals):
    """world.py:331-342: (16, E) = p, q, v, w, goal - p in the vehicle frame."""
    yaw, _ = O.yaw_of(tuple(s[3:7]))
    c, sn = np.cos(yaw), np.sin(yaw)
    gx, gy, gz = goals[0] - s[0], goals[1] - s[1], goals[2] - s[2]
    return np.concatenate([s, np.stack([c * gx + sn * gy, -sn * gx + c * gy, gz])])


def commands_from_actions(actions, control_mode: str, robot: O.Robot, limits: O.Limits):
    """vec_env.py:85-104 on (E, 4) actions: clip to [-1, 1] (NaN passes, like
    np.clip), then attitude: (a0, a1) max_tilt, a2 max_yaw_rate,
    (a3 + 1) / 2 thrust_max; velocity: a0..a2 max_speed_cmd, a3 max_yaw_rate.
    Returns world_step's (mode, att (4, E), vel (4, E))."""
    a = np.clip(np.asarray(actions, dtype=np.float64), -1.0, 1.0)
    E = a.shape[0]
    zeros = np.zeros((4, E))
    if control_mode == "attitude":
        att = np.stack([a[:, 0] * limits.max_tilt, a[:, 1] * limits.max_tilt,
                        a[:, 2] * limits.max_yaw_rate,
                        (a[:, 3] + 1.0) / 2.0 * robot.thrust_max])
        return np.zeros(E, np.uint8), att, zeros
    vel = np.concatenate([(a[:, 0:3] * limits.max_speed_cmd).T,
                          (a[:, 3] * limits.max_yaw_rate)[None]])
    return np.ones(E, np.uint8), zeros, vel


def world_step(s, goals, pending, steps, mode, att, vel, robot: O.Robot, gains: O.Gains,
               limits: O.Limits, env: EnvCfg, rcfg: RewardCfg, spawn_fn, hit_fn=None):
    """One World.step.  spawn_fn(idx) -> (spawn p (3,k), goal (3,k)) for the
    envs that auto-reset now.  hit_fn(p (E, 3)) -> bool (E,): the primitive
    part of check_collisions (world.py:100, min_distance < r; scene_oracle),
    None in free space.  Returns a dict of post-step arrays."""
    s = np.array(s, dtype=np.float64)
    goals = np.array(goals, dtype=np.float64)
    steps = np.array(steps, dtype=np.int64)
    resetting = np.asarray(pending, dtype=bool).copy()
    if resetting.any():                                       # world.py:287-289
        idx = np.nonzero(resetting)[0]
        sp, gl = spawn_fn(idx)
        s[:, idx] = 0.0
        s[0:3, idx] = sp
        s[3, idx] = 1.0                                       # world.py:219-222
        goals[:, idx] = gl
        steps[idx] = 0
    with np.errstate(invalid="ignore", over="ignore"):
        new, info = O.step(s, mode, att, vel, gains, robot, env.dt, limits)   # :291
    nonfinite = info["nonfinite"]
    if resetting.any():                                       # world.py:293-299
        new[:, resetting] = s[:, resetting]
        nonfinite = nonfinite & ~resetting
    oob = out_of_bounds(new[0:3], env.bounds, env.collision_radius)   # :302-306
    collided = oob.copy()                 # free space: min_distance = +inf
    if hit_fn is not None:
        collided |= np.asarray(hit_fn(new[0:3].T), dtype=bool)
    collided &= ~resetting
    oob &= ~resetting
    active = ~resetting
    steps[active] += 1                                        # :308
    terminated = (collided | nonfinite) & active              # :309
    truncated = (steps >= env.episode_max_steps) & active & ~terminated
    reward = reward_goal_reaching(new[0:3], new[7:10], goals, collided, rcfg)
    reward = np.where(resetting, 0.0, reward)                 # :314-315
    return dict(state=new, goal=goals, steps=steps, pending=terminated | truncated,
                obs=observations(new, goals), reward=reward, terminated=terminated,
                truncated=truncated, collision=collided, oob=oob, nonfinite=nonfinite,
                autoreset=resetting)
