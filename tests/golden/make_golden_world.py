"""Golden vectors for the World.step epilogue, from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_world.py

A free-space flocksim World (no obstacles, no camera) is driven for STEPS
steps by seeded random velocity commands large enough to fly vehicles out of
the box (out-of-bounds -> collision -> terminated) with a short episode limit
(-> truncated), so every branch of World.step (world.py:277-326) occurs:
auto-reset-then-void, collision, truncation, reward, observation.  Recorded
per step: the commands and the outputs; state/goal/pending/steps are stored
as sequences of length STEPS+1 (entry k = before step k).  The reference's own re-spawn draws (NumPy Philox per env
and reset, assets.py:310-315) appear in the post-step arrays of the envs
that reset; tests feed them to the oracle instead of drawing them.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
E, STEPS = 24, 240


def planar(st):
    return np.concatenate([st.p.T, st.q.T, st.v.T, st.omega.T], axis=0)


def main():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from flocksim.config import EnvConfig, SimConfig
    from flocksim.control import CommandBatch, VelocityCommands
    from flocksim.world import World

    cfg = SimConfig(env=EnvConfig(num_envs=E, seed=5, episode_max_steps=150))
    world = World.create(cfg)
    rng = np.random.default_rng(77)
    rec = {k: [] for k in ("state", "goal", "pending", "steps", "vel_cmd",
                           "obs", "reward", "terminated", "truncated", "collision", "oob",
                           "nonfinite", "autoreset")}
    # per-env constant direction (fly into a wall within ~1 s) + jitter
    heading = rng.normal(size=(E, 3))
    heading /= np.linalg.norm(heading, axis=1, keepdims=True)
    rec["state"].append(planar(world.states))
    rec["goal"].append(world.goals.T.copy())
    rec["pending"].append(world.pending_reset.copy())
    rec["steps"].append(world.steps_in_episode.copy())
    for _ in range(STEPS):
        v = 5.0 * heading + rng.uniform(-1.0, 1.0, (E, 3))
        v = np.asarray(v, dtype=np.float32).astype(np.float64)
        yr = np.asarray(rng.uniform(-1.0, 1.0, E), dtype=np.float32).astype(np.float64)
        rec["vel_cmd"].append(np.concatenate([v.T, yr[None]]))
        res = world.step(CommandBatch.all_velocity(VelocityCommands(v=v, yaw_rate=yr)))
        rec["obs"].append(res.observations.T.copy())
        rec["reward"].append(res.reward.copy())
        rec["terminated"].append(res.terminated.copy())
        rec["truncated"].append(res.truncated.copy())
        for k in ("collision", "nonfinite", "autoreset"):
            rec[k].append(np.asarray(res.info[k]).copy())
        rec["oob"].append(np.asarray(res.info["out_of_bounds"]).copy())
        rec["state"].append(planar(world.states))
        rec["goal"].append(world.goals.T.copy())
        rec["steps"].append(world.steps_in_episode.copy())
        rec["pending"].append(world.pending_reset.copy())
    arrays = {k: np.stack(v) for k, v in rec.items()}
    arrays["bounds"] = np.asarray(cfg.env.bounds)
    arrays["episode_max_steps"] = np.int64(cfg.env.episode_max_steps)
    arrays["dt"] = np.float64(cfg.env.dt)
    path = os.path.join(HERE, "world.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes); resets={int(arrays['autoreset'].sum())}"
          f" terminated={int(arrays['terminated'].sum())} truncated={int(arrays['truncated'].sum())}")


if __name__ == "__main__":
    main()
