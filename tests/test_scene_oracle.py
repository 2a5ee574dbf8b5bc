"""Pin the scene / camera oracle (oracle/scene_oracle.py) to the reference.

CPU only.  tests/golden/scene.npz was recorded from the unmodified flocksim
(tests/golden/make_golden_scene.py): signed distances and min_distance on a
random primitive soup (scene.py:127-181), cast_rays with random and
axis-parallel rays (camera.py:230-282), a rendered forest World
(camera.py:306-335), procedural tree URDF text (assets.py:435-459) and a
forest World trajectory with tree collisions, wall hits, truncations and
auto-resets (world.py:277-326 with check_collisions' primitive part).
"""

import numpy as np
import pytest

from oracle import flocksim_oracle as O
from oracle import scene_oracle as S
from oracle import world_oracle as WO

PSET_KEYS = ("kind", "dims", "position", "rot", "seg_id", "collision", "aabb_min", "aabb_max")


def pset(g, prefix, idx=None):
    out = {k: g[f"{prefix}{k}"] for k in PSET_KEYS}
    if idx is not None:
        out = {k: v[idx] for k, v in out.items()}
    return out


@pytest.fixture(scope="module")
def g():
    from conftest import load_golden
    return load_golden("scene")


def test_signed_distances_match_reference(g):
    ps = pset(g, "sdf_")
    d = S.signed_distances(ps, g["sdf_points"])
    np.testing.assert_allclose(d, g["sdf_dist"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(S.min_distance(ps, g["sdf_points"], True), g["sdf_min_coll"],
                               rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(S.min_distance(ps, g["sdf_points"], False), g["sdf_min_all"],
                               rtol=1e-12, atol=1e-12)
    # every kind and both signs occur
    assert set(np.unique(ps["kind"])) == {0, 1, 2}
    assert (g["sdf_dist"] < 0).any() and (g["sdf_dist"] > 0).any()


def test_aabb_matches_reference(g):
    ps = pset(g, "sdf_")
    lo, hi = S.aabb(ps["kind"], ps["dims"], ps["position"], ps["rot"])
    np.testing.assert_allclose(lo, ps["aabb_min"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(hi, ps["aabb_max"], rtol=1e-12, atol=1e-12)


def test_cast_rays_match_reference(g):
    ps = pset(g, "sdf_")
    for i, e in enumerate(g["ray_env"]):
        t, s = S.cast_rays(g["ray_origin"][i], g["ray_dirs"][i], ps, int(e),
                           float(g["ray_max_range"]))
        np.testing.assert_allclose(t, g["ray_depth"][i], rtol=1e-12, atol=1e-12)
        np.testing.assert_array_equal(s, g["ray_seg"][i])
    assert (g["ray_seg"] != 0).any() and (g["ray_seg"] == 0).any()


def test_render_matches_reference(g):
    ps = pset(g, "ren_")
    w, h, hfov, rmax = g["ren_cam"]
    depth, seg = S.render(g["ren_p"], g["ren_q"], g["ren_mount_p"], g["ren_mount_q"], ps,
                          int(w), int(h), float(hfov), float(rmax))
    np.testing.assert_array_equal(seg, g["ren_seg"])
    np.testing.assert_allclose(depth, g["ren_depth"], rtol=2e-7, atol=0)
    assert {1, 2} <= set(np.unique(seg))       # walls and trees in view


def test_tree_urdf_text_matches_reference(g):
    from paper_2305_16510_b200 import assets
    for key in [k for k in g if k.startswith("tree_")]:
        _, seed, depth, bf = key.split("_")
        _, text = assets.generate_tree(assets.TreeConfig(seed=int(seed), depth=int(depth),
                                                         branch_factor=int(bf)))
        assert text == bytes(g[key]).decode(), key


def test_world_step_with_obstacles_matches_reference(g):
    """The oracle world step + primitive collisions reproduces the reference's
    forest trajectory; the reference's own re-spawn draws are fed in."""
    E = g["trj_state"].shape[2]
    env = WO.EnvCfg(bounds=g["trj_bounds"], episode_max_steps=int(g["trj_episode_max_steps"]),
                    collision_radius=float(g["trj_collision_radius"]))
    ones, zeros4 = np.ones(E, np.uint8), np.zeros((4, E))
    snaps = list(g["trj_snap_steps"])
    steps_total = g["trj_vel_cmd"].shape[0]
    hits = 0
    for k in range(steps_total):
        si = max(i for i, s in enumerate(snaps) if s <= k)
        ps = pset(g, "trj_pset_", si)
        nxt_state = g["trj_state"][k + 1] if k + 1 < steps_total else None
        nxt_goal = g["trj_goal"][k + 1] if k + 1 < steps_total else None

        def spawn(idx, nxt_state=nxt_state, nxt_goal=nxt_goal):
            return nxt_state[0:3][:, idx], nxt_goal[:, idx]

        def hit(p, ps=ps):
            return S.min_distance(ps, p) < env.collision_radius

        ref = WO.world_step(g["trj_state"][k], g["trj_goal"][k], g["trj_pending"][k],
                            g["trj_steps"][k], ones, zeros4, g["trj_vel_cmd"][k], O.Robot(),
                            O.Gains(), O.Limits(), env, WO.RewardCfg(),
                            spawn if g["trj_pending"][k].any() else None, hit_fn=hit)
        for key in ("terminated", "truncated", "collision", "oob", "nonfinite", "autoreset"):
            np.testing.assert_array_equal(ref[key], g[f"trj_{key}"][k], err_msg=f"{key} {k}")
        np.testing.assert_allclose(ref["reward"], g["trj_reward"][k], rtol=1e-9, atol=1e-9)
        np.testing.assert_allclose(ref["obs"], g["trj_obs"][k], rtol=1e-9, atol=1e-9)
        hits += int((ref["collision"] & ~ref["oob"]).sum())
    assert hits > 0, "no primitive (tree) collision in the recorded trajectory"
