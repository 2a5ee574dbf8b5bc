"""Golden vectors for the obstacle scene and depth camera, from the UNMODIFIED
reference.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_scene.py

Writes tests/golden/scene.npz with:
  sdf_*     a seeded random primitive soup (boxes, z-cylinders, spheres in
            random local and instance poses, one instance per env) and one
            query point per env near it: flocksim.scene.signed_distances and
            min_distance (collision_only True / False);
  ray_*     seeded rays (random and axis-parallel directions) cast against
            three of those envs: flocksim.camera.cast_rays;
  ren_*     a forest World (generated trees + walls + a randomized camera)
            with perturbed robot poses, rendered by flocksim.camera.render;
  tree_*    URDF text of assets.generate_tree for a few configs;
  trj_*     that forest World stepped STEPS times by seeded velocity
            commands (fp32-representable), with the pre-step state, goals,
            pending flags, counters and -- whenever it changed -- the
            primitive set, plus every step's outputs.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
STEPS = 400


def planar(st):
    return np.concatenate([st.p.T, st.q.T, st.v.T, st.omega.T], axis=0)


def pset_arrays(ps, prefix):
    return {f"{prefix}{k}": np.array(getattr(ps, k)) for k in
            ("kind", "dims", "position", "rot", "seg_id", "collision", "aabb_min", "aabb_max")}


def random_soup(rng, assets, se3, n_env):
    kinds = ["box", "cylinder", "sphere"]
    envs = []
    for e in range(n_env):
        prims = []
        for _ in range(3):
            kind = kinds[rng.integers(0, 3)]
            dims = {"box": tuple(rng.uniform(0.2, 1.5, 3)),
                    "cylinder": (rng.uniform(0.1, 0.6), rng.uniform(0.5, 2.0), 0.0),
                    "sphere": (rng.uniform(0.2, 1.0), 0.0, 0.0)}[kind]
            prims.append(assets.Primitive(kind=kind, dims=dims,
                                          position=rng.uniform(-1.0, 1.0, 3),
                                          rotation=se3.rot_zyx(*rng.uniform(-2, 2, 3))))
        proto = assets.AssetPrototype(source="soup", class_name="soup", primitives=prims)
        envs.append([assets.AssetInstance(
            prototype=proto, position=rng.uniform(2.0, 8.0, 3),
            rotation=se3.rot_zyx(*rng.uniform(-3, 3, 3)), segmentation_id=int(rng.integers(1, 9)),
            env_index=e, class_name="soup", collision_enabled=bool(rng.random() < 0.85))])
    return envs


def forest_world(World, SimConfig, EnvConfig, AssetClassConfig, CameraConfig, assets, n_env):
    pools = {"trees": [assets.generate_tree(assets.TreeConfig(seed=s, depth=3))[0]
                       for s in range(4)]}
    cfg = SimConfig(
        env=EnvConfig(num_envs=n_env, seed=7, bounds=np.array([12.0, 12.0, 6.0]),
                      episode_max_steps=150, wall_enabled=True,
                      goal_min=np.array([0.15, 0.15, 0.25]), goal_max=np.array([0.85, 0.85, 0.6]),
                      spawn_min=np.array([0.15, 0.15, 0.25]),
                      spawn_max=np.array([0.85, 0.85, 0.6])),
        asset_classes=[AssetClassConfig(name="trees", count_per_env=10,
                                        position_min=[0.05, 0.05, 0.0],
                                        position_max=[0.95, 0.95, 0.0],
                                        frozen=(None, None, 0.0),
                                        euler_min=[0.0, 0.0, -3.14159],
                                        euler_max=[0.0, 0.0, 3.14159], segmentation_id=2)],
        camera=CameraConfig(width=64, height=40, hfov=1.57, max_range=10.0,
                            mount_position=[0.1, 0.0, 0.0],
                            randomize_position=[0.01, 0.01, 0.01],
                            randomize_euler=[0.02, 0.02, 0.02]))
    return World.create(cfg, pools=pools)


def main():
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    from flocksim import assets, se3
    from flocksim.assets import AssetClassConfig
    from flocksim.camera import CameraConfig, cast_rays, render
    from flocksim.config import EnvConfig, SimConfig
    from flocksim.control import CommandBatch, VelocityCommands
    from flocksim.scene import compile_instances, min_distance, signed_distances
    from flocksim.world import World

    out = {}
    rng = np.random.default_rng(2305)
    # -- signed distances ------------------------------------------------------
    n_env = 256
    ps = compile_instances(random_soup(rng, assets, se3, n_env))
    pts = ps.position[:, 0, :] + rng.normal(0.0, 0.8, (n_env, 3))
    out.update(pset_arrays(ps, "sdf_"))
    out["sdf_points"] = pts
    out["sdf_dist"] = signed_distances(ps, pts)
    out["sdf_min_coll"] = min_distance(ps, pts, collision_only=True)
    out["sdf_min_all"] = min_distance(ps, pts, collision_only=False)
    # -- ray casts ---------------------------------------------------------------
    m = 3000
    origins, dirs, depth, seg = [], [], [], []
    for e in (0, 1, 2):
        o = ps.position[e, 0] + rng.normal(0.0, 2.5, 3)
        d = rng.normal(size=(m, 3))
        d[:300] = 0.0
        d[np.arange(300), rng.integers(0, 3, 300)] = rng.choice([-1.0, 1.0], 300)
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        t, s = cast_rays(o, d, ps, e, 12.0)
        origins.append(o)
        dirs.append(d)
        depth.append(t)
        seg.append(s)
    out["ray_env"] = np.array([0, 1, 2])
    out["ray_origin"] = np.array(origins)
    out["ray_dirs"] = np.array(dirs)
    out["ray_depth"] = np.array(depth)
    out["ray_seg"] = np.array(seg)
    out["ray_max_range"] = 12.0
    # -- render of a forest world -----------------------------------------------
    world = forest_world(World, SimConfig, EnvConfig, AssetClassConfig, CameraConfig, assets, 4)
    world.states.q[:] = se3.exp_so3(rng.uniform(-0.4, 0.4, (4, 3)))
    world.states.p[:] += rng.uniform(-0.3, 0.3, (4, 3))
    img = render(world, world.camera)
    mp, mq = world.camera_mounts(world.camera)
    out.update(pset_arrays(world.pset, "ren_"))
    out["ren_p"] = world.states.p.copy()
    out["ren_q"] = world.states.q.copy()
    out["ren_mount_p"] = np.array(mp)
    out["ren_mount_q"] = np.array(mq)
    out["ren_depth"] = img.depth
    out["ren_seg"] = img.segmentation
    cam = world.camera
    out["ren_cam"] = np.array([cam.width, cam.height, cam.hfov, cam.max_range])
    # -- trajectory of a forest world ------------------------------------------------
    n_env = 8
    world = forest_world(World, SimConfig, EnvConfig, AssetClassConfig, CameraConfig, assets, n_env)
    heading = rng.normal(size=(n_env, 3))
    heading[:, 2] *= 0.2
    heading /= np.linalg.norm(heading, axis=1, keepdims=True)
    rec = {k: [] for k in ("state", "goal", "pending", "steps", "vel_cmd", "obs", "reward",
                           "terminated", "truncated", "collision", "oob", "nonfinite",
                           "autoreset", "mount_p", "mount_q")}
    snaps, snap_steps = [], []
    prev_pos = None
    for k in range(STEPS):
        if prev_pos is None or not np.array_equal(prev_pos, world.pset.position):
            snap_steps.append(k)
            snaps.append(pset_arrays(world.pset, ""))
            prev_pos = world.pset.position.copy()
        rec["state"].append(planar(world.states))
        rec["goal"].append(world.goals.T.copy())
        rec["pending"].append(world.pending_reset.copy())
        rec["steps"].append(world.steps_in_episode.copy())
        mp, mq = world.camera_mounts(world.camera)
        rec["mount_p"].append(np.array(mp))
        rec["mount_q"].append(np.array(mq))
        v = 5.0 * heading + rng.uniform(-0.5, 0.5, (n_env, 3))
        v = np.asarray(v, np.float32).astype(np.float64)
        yr = np.asarray(rng.uniform(-0.5, 0.5, n_env), np.float32).astype(np.float64)
        rec["vel_cmd"].append(np.concatenate([v.T, yr[None]]))
        res = world.step(CommandBatch.all_velocity(VelocityCommands(v=v, yaw_rate=yr)))
        rec["obs"].append(res.observations.T.copy())
        rec["reward"].append(res.reward.copy())
        rec["terminated"].append(res.terminated.copy())
        rec["truncated"].append(res.truncated.copy())
        rec["collision"].append(res.info["collision"].copy())
        rec["oob"].append(res.info["out_of_bounds"].copy())
        rec["nonfinite"].append(res.info["nonfinite"].copy())
        rec["autoreset"].append(res.info["autoreset"].copy())
    for key, vals in rec.items():
        out[f"trj_{key}"] = np.array(vals)
    out["trj_snap_steps"] = np.array(snap_steps)
    for key in snaps[0]:
        out[f"trj_pset_{key}"] = np.stack([s[key] for s in snaps])
    # -- procedural trees (assets.generate_tree): URDF text of a few configs ------
    for seed, depth, bf in ((0, 3, 2), (3, 3, 2), (5, 4, 3), (9, 2, 1)):
        _, text = assets.generate_tree(assets.TreeConfig(seed=seed, depth=depth, branch_factor=bf))
        out[f"tree_{seed}_{depth}_{bf}"] = np.frombuffer(text.encode(), dtype=np.uint8)
    out["trj_bounds"] = world.bounds
    out["trj_episode_max_steps"] = world.env.episode_max_steps
    out["trj_collision_radius"] = world.robot.collision_radius
    print("trajectory: resets", int(out["trj_autoreset"].sum()),
          "collisions", int(out["trj_collision"].sum()),
          "oob", int(out["trj_oob"].sum()), "truncations", int(out["trj_truncated"].sum()),
          "pset snapshots", len(snap_steps))
    path = os.path.join(HERE, "scene.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
