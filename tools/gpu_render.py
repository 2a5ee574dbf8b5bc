"""Render throughput probe (diagnostics, not the bench contract).

python tools/gpu_render.py [--envs 1024] [--width 480] [--height 270] [--iters 20]

A forest World (10 depth-3 trees + walls per env, forest.yaml's layout) with a
forward camera; times camera.render over `iters` calls with CUDA events and
prints frames/s, rays/s and output GB/s.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--envs", type=int, default=1024)
    ap.add_argument("--width", type=int, default=480)
    ap.add_argument("--height", type=int, default=270)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--depth", type=int, default=3)
    a = ap.parse_args()
    from paper_2305_16510_b200 import assets
    from paper_2305_16510_b200 import world as W
    from paper_2305_16510_b200.assets import AssetClassConfig
    from paper_2305_16510_b200.camera import CameraConfig, render

    env = W.EnvConfig(num_envs=a.envs, seed=7, bounds=[12.0, 12.0, 6.0], wall_enabled=True,
                      goal_min=[0.15, 0.15, 0.25], goal_max=[0.85, 0.85, 0.6],
                      spawn_min=[0.15, 0.15, 0.25], spawn_max=[0.85, 0.85, 0.6])
    trees = AssetClassConfig(name="trees", count_per_env=10, position_min=[0.05, 0.05, 0.0],
                             position_max=[0.95, 0.95, 0.0], frozen=(None, None, 0.0),
                             euler_min=[0.0, 0.0, -3.14159], euler_max=[0.0, 0.0, 3.14159],
                             segmentation_id=2)
    cam = CameraConfig(width=a.width, height=a.height, mount_position=[0.1, 0.0, 0.0],
                       randomize_position=[0.01] * 3, randomize_euler=[0.02] * 3)
    pools = {"trees": [assets.generate_tree(assets.TreeConfig(seed=s, depth=a.depth))[0]
                       for s in range(4)]}
    world = W.World.create(W.SimConfig(env=env, asset_classes=[trees], camera=cam), pools=pools)
    out = render(world, cam)
    for _ in range(3):
        render(world, cam, out=out)
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(a.iters):
        render(world, cam, out=out)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / a.iters
    frames = a.envs / (ms * 1e-3)
    rays = frames * a.width * a.height
    gbs = a.envs * a.width * a.height * 8 / (ms * 1e-3) / 1e9
    print(json.dumps({"envs": a.envs, "width": a.width, "height": a.height,
                      "prims_per_env": world.pset.width, "ms_per_render": ms,
                      "frames_per_s": frames, "rays_per_s": rays, "output_gbs": gbs}))


if __name__ == "__main__":
    main()
