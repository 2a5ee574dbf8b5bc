"""Golden vectors for the RL bindings' step, from the UNMODIFIED reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_vecenv.py

For each control mode a flocksim_rl handle (pkg/bindings/src/flocksim_rl/
vec_env.py) built from a YAML config (the one pkg/bindings/tests/
test_bindings.py:19-27 writes, plus a shorter episode) is stepped STEPS
times with seeded actions in [-1.3, 1.3] (so the clip to [-1, 1] is hit)
with a few +-inf entries (clipped to +-1).  Actions are rounded to fp32 so
the same values can be fed as float32 or float64.  Recorded per step: the
actions, the reference's denormalized commands (the handle's own
_commands_from_actions), the outputs, and the world arrays before each step
(entry k = before step k, length STEPS+1).
"""

from __future__ import annotations

import os
import sys
import tempfile

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_BIND = "/root/reference/pkg/bindings/src"
HERE = os.path.dirname(os.path.abspath(__file__))
E, STEPS = 8, 200

CFG = """
version: 1
env:
  num_envs: {n}
  seed: {seed}
  control_mode: {mode}
  bounds: [10.0, 10.0, 5.0]
  episode_max_steps: 120
  wall_enabled: true
"""


def planar(st):
    return np.concatenate([st.p.T, st.q.T, st.v.T, st.omega.T], axis=0)


def record(mode, seed):
    from flocksim_rl import make

    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "sim.yaml")
        with open(path, "w") as f:
            f.write(CFG.format(n=E, seed=seed, mode=mode))
        handle = make(path)
    world = handle._world
    rng = np.random.default_rng(1000 + seed)
    rec = {k: [] for k in ("state", "goal", "pending", "steps", "actions", "cmd", "obs",
                           "reward", "terminated", "truncated", "collision", "oob",
                           "nonfinite", "autoreset")}

    def snap():
        rec["state"].append(planar(world.states))
        rec["goal"].append(world.goals.T.copy())
        rec["pending"].append(world.pending_reset.copy())
        rec["steps"].append(world.steps_in_episode.copy())

    snap()
    for k in range(STEPS):
        a = rng.uniform(-1.3, 1.3, (E, 4))
        if k % 50 == 7:
            a[k % E, k % 4] = np.inf if k % 100 == 7 else -np.inf
        a = np.asarray(a, dtype=np.float32).astype(np.float64)
        cmds = handle._commands_from_actions(a)
        if mode == "attitude":
            c = cmds.attitude
            cmd = np.stack([c.roll, c.pitch, c.yaw_rate, c.thrust])
        else:
            c = cmds.velocity
            cmd = np.concatenate([c.v.T, c.yaw_rate[None]])
        obs, rew, term, trunc, info = handle.step(a)
        rec["actions"].append(a)
        rec["cmd"].append(cmd)
        rec["obs"].append(np.asarray(obs).T.copy())
        rec["reward"].append(np.asarray(rew).copy())
        rec["terminated"].append(np.asarray(term).copy())
        rec["truncated"].append(np.asarray(trunc).copy())
        for key in ("collision", "nonfinite", "autoreset"):
            rec[key].append(np.asarray(info[key]).copy())
        rec["oob"].append(np.asarray(info["out_of_bounds"]).copy())
        snap()
    arrays = {k: np.stack(v) for k, v in rec.items()}
    arrays["bounds"] = np.asarray(world.bounds)
    arrays["episode_max_steps"] = np.int64(world.env.episode_max_steps)
    arrays["seed"] = np.int64(seed)
    return arrays


def main():
    for p in (REF_SRC, REF_BIND):
        if p not in sys.path:
            sys.path.insert(0, p)
    for mode, seed in (("velocity", 17), ("attitude", 19)):
        arrays = record(mode, seed)
        path = os.path.join(HERE, f"vecenv_{mode}.npz")
        np.savez_compressed(path, **arrays)
        print(f"wrote {path} ({os.path.getsize(path)} bytes); "
              f"resets={int(arrays['autoreset'].sum())} "
              f"terminated={int(arrays['terminated'].sum())} "
              f"truncated={int(arrays['truncated'].sum())} "
              f"clipped={int((np.abs(arrays['actions']) > 1).sum())}")


if __name__ == "__main__":
    main()
