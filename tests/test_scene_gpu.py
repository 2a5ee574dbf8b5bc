"""GPU tests of the obstacle scene, collisions and the depth camera
(SURVEY.md 8(f) rank 4).

The device results are compared with the pinned float64 scene oracle
(oracle/scene_oracle.py, pinned to the reference in
tests/test_scene_oracle.py) on IDENTICAL inputs: the fp32 primitive rows
and fp32 robot states the device holds are read back and given to the
oracle.  Bars:
  * distances / ray parameters: float64 on both sides from the same fp32
    values -> rtol 1e-10;
  * depth images: float32 equal to the oracle's float32 rounding except at
    most 1e-4 of the pixels, which may differ by 1 ulp;
  * segmentation: equal except on ill-conditioned pixels (the oracle's own
    segmentation flips under a 1e-6 rad ray jitter: silhouettes, grazes);
  * world step with obstacles: the reference's forest trajectory replayed
    step by step at 1e-5 rel / 1e-6 abs, flags exact.
Against the reference's own float64 primitive rows (before fp32 rounding),
the images must agree except on pixels ill-conditioned at 1e-5 rad.
"""

import math

import numpy as np
import pytest
import torch

from fs_parity import assert_parity
from oracle import flocksim_oracle as O
from oracle import scene_oracle as S
from oracle import world_oracle as WO

pytestmark = pytest.mark.gpu

PSET_KEYS = ("kind", "dims", "position", "rot", "seg_id", "collision", "aabb_min", "aabb_max")


@pytest.fixture(scope="module")
def fs():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2305_16510_b200 as fs
    fs._native.load()
    return fs


@pytest.fixture(scope="module")
def g():
    from conftest import load_golden
    return load_golden("scene")


def ref_pset(g, prefix, idx=None):
    out = {k: g[f"{prefix}{k}"] for k in PSET_KEYS}
    if idx is not None:
        out = {k: v[idx] for k, v in out.items()}
    return out


def device_pset(fs, arrays):
    from paper_2305_16510_b200.scene import PrimitiveSet
    e, k = arrays["kind"].shape
    return PrimitiveSet(e, k).load_arrays(*(arrays[key] for key in PSET_KEYS))


class Stub:
    """The world surface camera.render needs (camera.py:306-335)."""

    def __init__(self, fs, p, q, pset, camera=None, mounts=None):
        n = len(p)
        self.states = fs.RigidStateBatch(p=np.asarray(p), q=np.asarray(q), v=np.zeros((n, 3)),
                                         omega=np.zeros((n, 3)))
        self.pset = pset
        self.camera = camera
        self._mounts = mounts

    def camera_mounts(self, cfg):
        n = self.states.n
        if self._mounts is not None:
            return self._mounts
        return (np.broadcast_to(cfg.mount_position, (n, 3)),
                np.broadcast_to(cfg.mount_rotation, (n, 4)))


def _f32(x):
    return np.asarray(x, dtype=np.float32).astype(np.float64)


# ---- distances ----------------------------------------------------------------------

def test_signed_distances_match_oracle(fs, g):
    from paper_2305_16510_b200 import scene
    ps = device_pset(fs, ref_pset(g, "sdf_"))
    host = ps.to_numpy()
    pts = _f32(g["sdf_points"])
    d = scene.signed_distances(ps, pts).cpu().numpy()
    np.testing.assert_allclose(d, S.signed_distances(host, pts), rtol=1e-10, atol=1e-12)
    for coll in (True, False):
        m = scene.min_distance(ps, pts, collision_only=coll).cpu().numpy()
        np.testing.assert_allclose(m, S.min_distance(host, pts, coll), rtol=1e-10, atol=1e-12)
    # and against the reference's float64 rows: fp32 storage of the geometry only
    np.testing.assert_allclose(d, g["sdf_dist"], rtol=1e-5, atol=2e-5)


def test_stored_rows_and_outward_aabb(fs, g):
    ref = ref_pset(g, "sdf_")
    host = device_pset(fs, ref).to_numpy()
    for key in ("dims", "position", "rot"):
        np.testing.assert_array_equal(host[key], ref[key].astype(np.float32))
    assert (host["aabb_min"] <= ref["aabb_min"]).all()
    assert (host["aabb_max"] >= ref["aabb_max"]).all()
    np.testing.assert_allclose(host["aabb_min"], ref["aabb_min"], rtol=1e-6, atol=1e-6)
    np.testing.assert_array_equal(host["kind"], ref["kind"])
    np.testing.assert_array_equal(host["seg_id"], ref["seg_id"])
    np.testing.assert_array_equal(host["collision"], ref["collision"])


# ---- rays ---------------------------------------------------------------------------------

def test_cast_rays_match_oracle(fs, g):
    from paper_2305_16510_b200 import camera
    ps = device_pset(fs, ref_pset(g, "sdf_"))
    host = ps.to_numpy()
    rmax = float(g["ray_max_range"])
    for i, e in enumerate(g["ray_env"]):
        o, d = g["ray_origin"][i], g["ray_dirs"][i]
        t, s = camera.cast_rays(o, d, ps, int(e), rmax)
        rt, rs = S.cast_rays(o, d, host, int(e), rmax)
        np.testing.assert_allclose(t.cpu().numpy(), rt, rtol=1e-10, atol=1e-12)
        np.testing.assert_array_equal(s.cpu().numpy(), rs)


def _prim(fs, kind, dims, position=(0, 0, 0), euler=(0, 0, 0)):
    from paper_2305_16510_b200 import _se3
    from paper_2305_16510_b200.assets import Primitive
    return Primitive(kind=kind, dims=dims, position=np.asarray(position, float),
                     rotation=_se3.rot_zyx(*euler))


def test_ray_primitive_known_answers(fs):
    """camera.py:285-303; the reference's test_camera.py TestRayPrimitive cases."""
    from paper_2305_16510_b200.camera import ray_primitive
    t, seg = ray_primitive([-5.0, 0, 0], [1.0, 0, 0], _prim(fs, "sphere", (1.0, 0, 0)), seg_id=7)
    assert t == pytest.approx(4.0, abs=1e-12) and seg == 7
    assert ray_primitive([-5.0, 0, 0], [1.0, 0, 0],
                         _prim(fs, "box", (1.0, 1.0, 1.0)))[0] == pytest.approx(4.5, abs=1e-12)
    hit = ray_primitive([-5.0, 1.0, 0], [1.0, 0, 0], _prim(fs, "sphere", (1.0, 0, 0)))
    assert hit is not None and hit[0] == pytest.approx(5.0, abs=1e-6)      # tangent graze
    assert ray_primitive([-5.0, 1.5, 0], [1.0, 0, 0], _prim(fs, "sphere", (1.0, 0, 0))) is None
    cyl = _prim(fs, "cylinder", (0.5, 2.0, 0))
    assert ray_primitive([-4.0, 0, 0], [1.0, 0, 0], cyl)[0] == pytest.approx(3.5, abs=1e-12)
    assert ray_primitive([0.0, 0, 5.0], [0.0, 0, -1.0], cyl)[0] == pytest.approx(4.0, abs=1e-12)
    assert ray_primitive([-4.0, 0, 1.5], [1.0, 0, 0], cyl) is None
    assert ray_primitive([0.0, 0, 0], [1.0, 0, 0],
                         _prim(fs, "sphere", (2.0, 0, 0)))[0] == pytest.approx(2.0, abs=1e-12)
    assert ray_primitive([5.0, 0, 0], [1.0, 0, 0], _prim(fs, "sphere", (1.0, 0, 0))) is None
    assert ray_primitive([-5.0, 0, 0], [1.0, 0, 0], _prim(fs, "sphere", (1.0, 0, 0)),
                         max_range=3.0) is None
    box45 = _prim(fs, "box", (1.0, 1.0, 1.0), euler=(0, 0, math.pi / 4))
    assert ray_primitive([-5.0, 0, 0], [1.0, 0, 0], box45)[0] == pytest.approx(
        5.0 - math.sqrt(2.0) / 2.0, abs=1e-6)
    with pytest.raises(ValueError, match="unit"):
        ray_primitive([0, 0, 0], [2.0, 0, 0], _prim(fs, "sphere", (1.0, 0, 0)))


# ---- rendering ------------------------------------------------------------------------------

def _check_images(depth, seg, ref_depth, ref_seg, bad, what, ulp_frac=1e-4):
    mism = seg != ref_seg
    assert not (mism & ~bad).any(), f"{what}: {int((mism & ~bad).sum())} well-conditioned " \
                                    f"segmentation mismatches"
    same = ~mism
    dd = depth[same] != ref_depth[same]
    assert dd.mean() <= ulp_frac, f"{what}: {int(dd.sum())} depth mismatches"
    if dd.any():
        a, b = depth[same][dd], ref_depth[same][dd]
        assert (np.abs(a - b) <= np.spacing(np.abs(b).astype(np.float32)) * 1.01).all(), what


def test_render_forest_matches_oracle(fs, g):
    from paper_2305_16510_b200.camera import CameraConfig, render
    ref = ref_pset(g, "ren_")
    ps = device_pset(fs, ref)
    host = ps.to_numpy()
    w, h, hfov, rmax = g["ren_cam"]
    cam = CameraConfig(width=int(w), height=int(h), hfov=float(hfov), max_range=float(rmax))
    mounts = (g["ren_mount_p"], g["ren_mount_q"])
    world = Stub(fs, g["ren_p"], g["ren_q"], ps, cam, mounts)
    img = render(world, cam)
    depth, seg = img.depth.cpu().numpy(), img.segmentation.cpu().numpy()
    p32, q32 = _f32(g["ren_p"]), _f32(g["ren_q"])
    rd, rs = S.render(p32, q32, g["ren_mount_p"], g["ren_mount_q"], host, int(w), int(h),
                      float(hfov), float(rmax))
    bad = S.ill_conditioned_pixels(p32, q32, g["ren_mount_p"], g["ren_mount_q"], host, int(w),
                                   int(h), float(hfov), float(rmax))
    _check_images(depth, seg, rd, rs, bad, "oracle")
    # against the reference's own image (float64 rows and states): geometry
    # rounding to fp32 moves silhouettes by ~1e-6 m
    bad5 = S.ill_conditioned_pixels(g["ren_p"], g["ren_q"], g["ren_mount_p"], g["ren_mount_q"],
                                    ref, int(w), int(h), float(hfov), float(rmax), eps=1e-5)
    assert not ((seg != g["ren_seg"]) & ~bad5).any()
    same = seg == g["ren_seg"]
    np.testing.assert_allclose(depth[same], g["ren_depth"][same], rtol=1e-5, atol=1e-6)


def _forward(fs, scenes, seg=3):
    """One sphere/box/cylinder soup per env, robots at rest at the origin."""
    from paper_2305_16510_b200 import _se3
    from paper_2305_16510_b200.scene import KIND_CODES, compile_instances  # noqa: F401
    from paper_2305_16510_b200.assets import AssetInstance, AssetPrototype
    inst = []
    for e, prims in enumerate(scenes):
        if prims:
            proto = AssetPrototype(source="t", class_name="x", primitives=list(prims))
            inst.append([AssetInstance(prototype=proto, position=np.zeros(3),
                                       rotation=[1.0, 0, 0, 0], segmentation_id=seg,
                                       env_index=e, class_name="x")])
        else:
            inst.append([])
    n = len(scenes)
    ps = compile_instances(inst)
    return Stub(fs, np.zeros((n, 3)), np.tile([1.0, 0, 0, 0], (n, 1)), ps)


def test_render_reference_scenes(fs):
    """The reference's test_camera.py TestRender cases on the GPU."""
    from paper_2305_16510_b200.camera import CameraConfig, _pixel_rays, render
    cfg = CameraConfig(width=65, height=37, hfov=1.2, max_range=10.0)
    img = render(_forward(fs, [[]]), cfg)
    assert (img.depth == 10.0).all() and (img.segmentation == 0).all()
    img = render(_forward(fs, [[_prim(fs, "sphere", (1.0, 0, 0), (5.0, 0, 0))]]), cfg)
    assert float(img.depth[0, 18, 32]) == pytest.approx(4.0, abs=1e-6)
    assert int(img.segmentation[0, 18, 32]) == 3
    img = render(_forward(fs, [[_prim(fs, "box", (0.01, 40.0, 40.0), (5.005, 0, 0))]]), cfg)
    cos = _pixel_rays(65, 37, 1.2)[:, 2].reshape(37, 65)
    np.testing.assert_allclose(img.depth[0].cpu().numpy(), 5.0 / cos, atol=1e-5)
    img = render(_forward(fs, [[_prim(fs, "sphere", (1.0, 0, 0), (-5.0, 0, 0))]]), cfg)
    assert (img.depth == 10.0).all()


def test_render_occlusion_monotonicity(fs):
    """Adding an obstacle never increases any depth (test_camera.py occlusion test)."""
    from paper_2305_16510_b200.camera import CameraConfig, render
    rng = np.random.default_rng(31)
    cfg = CameraConfig(width=24, height=16, hfov=1.3, max_range=15.0)
    kinds = ["sphere", "box", "cylinder"]
    base_scenes, more_scenes = [], []
    for _ in range(100):
        prims = []
        for _ in range(5):
            kind = kinds[rng.integers(0, 3)]
            dims = {"sphere": (rng.uniform(0.2, 1.0), 0, 0),
                    "box": tuple(rng.uniform(0.2, 1.5, 3)),
                    "cylinder": (rng.uniform(0.1, 0.6), rng.uniform(0.5, 2.0), 0)}[kind]
            prims.append(_prim(fs, kind, dims, rng.uniform([1, -3, -3], [9, 3, 3]),
                               rng.uniform(-2, 2, 3)))
        extra = _prim(fs, kinds[rng.integers(0, 3)], (0.8, 0.8, 0.8),
                      rng.uniform([1, -2, -2], [7, 2, 2]), rng.uniform(-2, 2, 3))
        base_scenes.append(prims)
        more_scenes.append(prims + [extra])
    base = render(_forward(fs, base_scenes), cfg).depth
    more = render(_forward(fs, more_scenes), cfg).depth
    assert (more <= base).all()


def test_render_batch_equals_single_and_is_deterministic(fs):
    from paper_2305_16510_b200.camera import CameraConfig, render
    rng = np.random.default_rng(8)
    scenes = [[_prim(fs, "box", tuple(rng.uniform(0.5, 2, 3)), rng.uniform([2, -2, -2], [8, 2, 2]),
                     rng.uniform(-1, 1, 3))] for _ in range(5)]
    cfg = CameraConfig(width=32, height=20, hfov=1.4)
    world = _forward(fs, scenes)
    world.states.buf[0:3, :5] = torch.as_tensor(rng.uniform(-1, 1, (3, 5)), dtype=torch.float32)
    a = render(world, cfg)
    b = render(world, cfg)
    assert torch.equal(a.depth, b.depth) and torch.equal(a.segmentation, b.segmentation)
    for i in range(5):
        single = Stub(fs, world.states.p[i:i + 1].cpu().numpy(), world.states.q[i:i + 1].cpu().numpy(),
                      world.pset.env_view(i))
        s = render(single, cfg)
        assert torch.equal(s.depth[0], a.depth[i]) and torch.equal(s.segmentation[0],
                                                                   a.segmentation[i])


def test_large_primitive_count_chunks(fs):
    """More primitives than one shared-memory chunk (256): same image as the oracle."""
    from paper_2305_16510_b200.camera import CameraConfig, render
    rng = np.random.default_rng(4)
    prims = [_prim(fs, "sphere", (rng.uniform(0.05, 0.3), 0, 0),
                   rng.uniform([2, -4, -3], [9, 4, 3])) for _ in range(600)]
    world = _forward(fs, [prims, prims[:100]])
    cfg = CameraConfig(width=40, height=24, hfov=1.4, max_range=12.0)
    img = render(world, cfg)
    host = world.pset.to_numpy()
    p = np.zeros((2, 3))
    q = np.tile([1.0, 0, 0, 0], (2, 1))
    mp = np.broadcast_to(cfg.mount_position, (2, 3))
    mq = np.broadcast_to(cfg.mount_rotation, (2, 4))
    rd, rs = S.render(p, q, mp, mq, host, 40, 24, 1.4, 12.0)
    bad = S.ill_conditioned_pixels(p, q, mp, mq, host, 40, 24, 1.4, 12.0)
    _check_images(img.depth.cpu().numpy(), img.segmentation.cpu().numpy(), rd, rs, bad, "chunks")


def test_depth_dump_roundtrip(fs, tmp_path):
    from paper_2305_16510_b200.camera import CameraConfig, DepthImageBatch, render
    img = render(_forward(fs, [[_prim(fs, "sphere", (1.0, 0, 0), (4.0, 0, 0))],
                               [_prim(fs, "box", (1.0, 1.0, 1.0), (3.0, 0, 0))]]),
                 CameraConfig(width=16, height=12, hfov=1.2))
    path = tmp_path / "frames.bin"
    img.write_binary(path)
    back = DepthImageBatch.read_binary(path, max_range=img.max_range)
    assert torch.equal(back.depth, img.depth.cpu())
    assert torch.equal(back.segmentation, img.segmentation.cpu())
    img.write_png(0, tmp_path / "f.png")


# ---- worlds with obstacles --------------------------------------------------------------

def forest_cfg(W, n, seed=7, camera=True):
    from paper_2305_16510_b200.assets import AssetClassConfig
    from paper_2305_16510_b200.camera import CameraConfig
    env = W.EnvConfig(num_envs=n, seed=seed, bounds=[12.0, 12.0, 6.0], episode_max_steps=150,
                      wall_enabled=True, goal_min=[0.15, 0.15, 0.25], goal_max=[0.85, 0.85, 0.6],
                      spawn_min=[0.15, 0.15, 0.25], spawn_max=[0.85, 0.85, 0.6])
    trees = AssetClassConfig(name="trees", count_per_env=10, position_min=[0.05, 0.05, 0.0],
                             position_max=[0.95, 0.95, 0.0], frozen=(None, None, 0.0),
                             euler_min=[0.0, 0.0, -3.14159], euler_max=[0.0, 0.0, 3.14159],
                             segmentation_id=2)
    cam = CameraConfig(width=64, height=40, mount_position=[0.1, 0.0, 0.0],
                       randomize_position=[0.01, 0.01, 0.01],
                       randomize_euler=[0.02, 0.02, 0.02]) if camera else None
    return W.SimConfig(env=env, asset_classes=[trees], camera=cam)


def tree_pools():
    from paper_2305_16510_b200 import assets
    return {"trees": [assets.generate_tree(assets.TreeConfig(seed=s, depth=3))[0]
                      for s in range(4)]}


def test_forest_world_creation_invariants(fs):
    from paper_2305_16510_b200 import scene
    from paper_2305_16510_b200 import world as W
    n = 512
    world = W.World.create(forest_cfg(W, n), pools=tree_pools())
    assert world.pset.width == 10 * 7 + 6
    inst = world.instances
    for e in (0, 17, n - 1):
        trees = [i for i in inst[e] if i.class_name == "trees"]
        assert len(trees) == 10 and all(i.position[2] == 0.0 for i in trees)
        assert inst[e][-1].class_name == W.WALL_CLASS
    d = scene.min_distance(world.pset, world.states.p).cpu().numpy()
    assert (d >= 0.2).all()
    gd = scene.min_distance(world.pset, world.goals).cpu().numpy()
    assert (gd >= 0.2).all()
    info = world.privileged_info()
    assert len(info.per_env) == n and all(a.segmentation_id in (1, 2) for a in info.per_env[3])
    # seeded determinism
    again = W.World.create(forest_cfg(W, n), pools=tree_pools())
    assert torch.equal(again.pset.position, world.pset.position)
    assert torch.equal(again.states.buf, world.states.buf)


def test_forest_world_reset_draws_match_twin(fs):
    """Device picks, instance poses and camera mounts equal the CPU twin of
    the library's draw layout (oracle/scene_oracle.py twin_*)."""
    from paper_2305_16510_b200 import world as W
    n = 64
    cfg = forest_cfg(W, n, seed=19)
    world = W.World.create(cfg, pools=tree_pools())
    world.reset_env(5)
    c = cfg.asset_classes[0]
    cls = [(c.position_min, c.position_max, c.euler_min, c.euler_max, c.frozen)] * 10
    cam = cfg.camera
    picks_dev = world._inst_proto[:10, :n].cpu().numpy()
    world.instances         # fills the pose planes on demand (fs_obstacles_poses)
    pose_dev = world._inst_pose[:70, :n].cpu().numpy().reshape(10, 7, n)
    mount_dev = world._mount[:, :n].cpu().numpy()
    for e in (0, 5, 63):
        counter = 1 if e == 5 else 0
        assert list(picks_dev[:, e]) == S.twin_picks(19, e, [(10, 0, 4)])
        pos, quat = S.twin_poses(19, e, counter, cls, cfg.env.bounds)
        np.testing.assert_allclose(pose_dev[:, 0:3, e], pos, rtol=1e-14, atol=1e-14)
        np.testing.assert_allclose(pose_dev[:, 3:7, e], quat, rtol=1e-13, atol=1e-14)
        mp, mq = S.twin_mount(19, e, counter, cam.mount_position, cam.mount_euler,
                              cam.randomize_position, cam.randomize_euler)
        np.testing.assert_allclose(mount_dev[0:3, e], mp, rtol=1e-14, atol=1e-15)
        np.testing.assert_allclose(mount_dev[3:7, e], mq, rtol=1e-13, atol=1e-14)
    # the compiled rows are compile_instances of the device instances
    host = world.pset.to_numpy()
    rows = [[(S.BOX if p.kind == "box" else S.CYL if p.kind == "cylinder" else S.SPH, p.dims,
              p.position, p.rotation, i.position, i.rotation, i.segmentation_id,
              i.collision_enabled) for i in world.instances[e] for p in i.prototype.primitives]
            for e in (0, 5)]
    ref = S.compile_rows(rows, width=world.pset.width)
    for k, e in enumerate((0, 5)):
        np.testing.assert_allclose(host["position"][e], ref["position"][k], rtol=1e-6, atol=1e-6)
        np.testing.assert_allclose(host["rot"][e], ref["rot"][k], rtol=1e-6, atol=1e-6)
        assert (host["aabb_min"][e] <= ref["aabb_min"][k] + 1e-12).all()
        assert (host["aabb_max"][e] >= ref["aabb_max"][k] - 1e-12).all()
    # after World.step's auto-resets (which leave the pose planes alone) the
    # on-demand poses still describe the rows and the twin's draws
    g = torch.Generator(device="cpu").manual_seed(3)
    v = (torch.randn(n, 3, generator=g) * 4.0).cuda()
    cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(v=v, yaw_rate=torch.zeros(n).cuda(),
                                                            validate=False))
    for _ in range(80):
        world.step(cmds)
    counters = world.reset_counter.cpu().numpy()
    moved = [int(e) for e in np.nonzero(counters > (np.arange(n) == 5))[0][:3]]
    assert moved, counters
    inst = world.instances
    host = world.pset.to_numpy()
    for e in moved:
        pos, quat = S.twin_poses(19, e, int(counters[e]), cls, cfg.env.bounds)
        got = np.array([i.position for i in inst[e][:10]])
        np.testing.assert_allclose(got, pos, rtol=1e-14, atol=1e-14)
        rows = [[(S.BOX if p.kind == "box" else S.CYL if p.kind == "cylinder" else S.SPH, p.dims,
                  p.position, p.rotation, i.position, i.rotation, i.segmentation_id,
                  i.collision_enabled) for i in inst[e] for p in i.prototype.primitives]]
        ref = S.compile_rows(rows, width=world.pset.width)
        np.testing.assert_allclose(host["position"][e], ref["position"][0], rtol=1e-6, atol=1e-6)


def test_reset_env_isolation(fs):
    from paper_2305_16510_b200 import world as W
    world = W.World.create(forest_cfg(W, 6, seed=21), pools=tree_pools())
    before = world.pset.position.clone()
    inst_before = [[i.position.copy() for i in env] for env in world.instances]
    world.reset_env(1)
    after = world.pset.position
    for e in (0, 2, 3, 4, 5):
        assert torch.equal(before[e], after[e])
    assert not torch.equal(before[1], after[1])
    inst_after = world.instances
    assert any(not np.array_equal(a, b.position) for a, b in zip(inst_before[1], inst_after[1]))
    assert world.reset_counter.cpu().tolist() == [0, 1, 0, 0, 0, 0]


def test_placement_failure(fs):
    """No free spawn (world.py:203-211): an obstacle filling the box."""
    from paper_2305_16510_b200 import assets
    from paper_2305_16510_b200 import world as W
    big = assets.parse_urdf_subset('<robot name="b"><link name="l"><collision><geometry>'
                                   '<box size="40 40 40"/></geometry></collision></link></robot>')
    cfg = W.SimConfig(env=W.EnvConfig(num_envs=3, seed=1),
                      asset_classes=[assets.AssetClassConfig(name="big", count_per_env=1)])
    with pytest.raises(W.PlacementFailureError):
        W.World.create(cfg, pools={"big": [big]})


def test_autoreset_placement_failure_raises(fs):
    """An auto-reset inside World.step that finds no free pose raises
    PlacementFailureError like the reference's step -> reset_env ->
    _find_free_point (world.py:200-211, 287-289); step_async does not check
    and leaves the bit readable in info['placement_failed']."""
    from paper_2305_16510_b200 import world as W
    from paper_2305_16510_b200.control import CommandBatch, VelocityCommands
    n = 4
    world = W.World.create(forest_cfg(W, n, camera=False), pools=tree_pools())
    cmds = CommandBatch.all_velocity(VelocityCommands(v=torch.zeros(n, 3, device="cuda"),
                                                      yaw_rate=torch.zeros(n, device="cuda")))
    world.step(cmds)           # nothing pending: no reset, no failure
    # a collision radius larger than half the env box: no in-bounds point clears it
    world._wcfg.collision_radius = 100.0
    pend = torch.zeros(n, dtype=torch.uint8)
    pend[2] = 1
    world.load(pending=pend)
    with pytest.raises(W.PlacementFailureError, match="env 2"):
        world.step(cmds)
    world.load(pending=pend)
    world.step_async(cmds)
    torch.cuda.synchronize()
    info = world._info[:n]
    assert ((info & fs._native.FS_INFO_PLACEMENT_FAILED) != 0).cpu().tolist() == \
        [False, False, True, False]


def test_forest_trajectory_replay_matches_oracle(fs, g):
    """The reference's forest trajectory replayed on the device step by step:
    the reference's primitive rows, state, goals, counters and commands in;
    state, observation, reward and every flag out, against the oracle on the
    same fp32 inputs (device re-spawn draws fed to the oracle)."""
    from paper_2305_16510_b200 import world as W
    E = g["trj_state"].shape[2]
    cfg = forest_cfg(W, E)
    cfg.env.episode_max_steps = int(g["trj_episode_max_steps"])
    world = W.World.create(cfg, pools=tree_pools())
    env = WO.EnvCfg(bounds=g["trj_bounds"], episode_max_steps=int(g["trj_episode_max_steps"]),
                    collision_radius=float(g["trj_collision_radius"]))
    ones, zeros4 = np.ones(E, np.uint8), np.zeros((4, E))
    snaps = list(g["trj_snap_steps"])
    hits = resets = 0
    for k in range(g["trj_vel_cmd"].shape[0]):
        si = max(i for i, s in enumerate(snaps) if s <= k)
        world.load(scene=ref_pset(g, "trj_pset_", si))
        host = world.pset.to_numpy()
        s_in, goal_in = _f32(g["trj_state"][k]), _f32(g["trj_goal"][k])
        world.load(state=s_in, goals=goal_in, pending=g["trj_pending"][k],
                   steps=g["trj_steps"][k])
        vel = _f32(g["trj_vel_cmd"][k])
        cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(v=vel[0:3].T, yaw_rate=vel[3],
                                                                validate=False))
        res = world.step(cmds)
        got_state = world.states.numpy()
        got_goal = world.goals.T.double().cpu().numpy()
        spawn = lambda idx: (got_state[0:3][:, idx], got_goal[:, idx])
        hit = lambda p: S.min_distance(host, p) < env.collision_radius
        ref = WO.world_step(s_in, goal_in, g["trj_pending"][k], g["trj_steps"][k], ones, zeros4,
                            vel, O.Robot(), O.Gains(), O.Limits(), env, WO.RewardCfg(), spawn,
                            hit_fn=hit)
        assert_parity(got_state, ref["state"], s_in, f"forest state step {k}")
        assert_parity(res.observations.T.double().cpu().numpy(), ref["obs"], s_in,
                      f"forest obs step {k}")
        assert_parity(res.reward.double().cpu().numpy(), ref["reward"], s_in,
                      f"forest reward step {k}")
        for key, got in (("terminated", res.terminated), ("truncated", res.truncated),
                         ("collision", res.info["collision"]), ("oob", res.info["out_of_bounds"]),
                         ("nonfinite", res.info["nonfinite"]),
                         ("autoreset", res.info["autoreset"])):
            np.testing.assert_array_equal(got.cpu().numpy(), ref[key], err_msg=f"{key} {k}")
            # and the reference's own flags
            np.testing.assert_array_equal(got.cpu().numpy(), g[f"trj_{key}"][k],
                                          err_msg=f"reference {key} {k}")
        hits += int((ref["collision"] & ~ref["oob"]).sum())
        resets += int(ref["autoreset"].sum())
        if ref["autoreset"].any():
            # a device re-spawn is collision-free against its fresh rows
            idx = np.nonzero(ref["autoreset"])[0]
            fresh = world.pset.to_numpy()
            d = S.min_distance(fresh, got_state[0:3].T)
            assert (d[idx] >= env.collision_radius).all()
    assert hits > 0 and resets > 0


def test_forest_world_render_matches_oracle(fs):
    from paper_2305_16510_b200 import world as W
    from paper_2305_16510_b200.camera import render
    world = W.World.create(forest_cfg(W, 16, seed=3), pools=tree_pools())
    img = render(world, world.camera)
    host = world.pset.to_numpy()
    st = world.states.numpy()
    mp, mq = (t.cpu().numpy() for t in world.camera_mounts(world.camera))
    cam = world.camera
    rd, rs = S.render(st[0:3].T, st[3:7].T, mp, mq, host, cam.width, cam.height, cam.hfov,
                      cam.max_range)
    bad = S.ill_conditioned_pixels(st[0:3].T, st[3:7].T, mp, mq, host, cam.width, cam.height,
                                   cam.hfov, cam.max_range)
    _check_images(img.depth.cpu().numpy(), img.segmentation.cpu().numpy(), rd, rs, bad, "world")
    assert {1, 2} <= set(np.unique(img.segmentation.cpu().numpy()))


def test_vecenv_render_depth(fs, tmp_path):
    from paper_2305_16510_b200 import rl
    path = tmp_path / "cam.yaml"
    path.write_text("env: {num_envs: 3, wall_enabled: true}\n"
                    "camera: {width: 32, height: 24}\n")
    with rl.make(path) as h:
        h.reset()
        img = h.render_depth()
        assert img.depth.shape == (3, 24, 32)
        assert set(np.unique(img.segmentation.cpu().numpy())) <= {0, 1}
        h.step(torch.zeros((3, 4), device="cuda"))


def test_obstacle_world_shard_invariance(fs):
    """Every draw is keyed by (seed, global env id, reset counter): two
    half-worlds (first_env 0 and n/2) reproduce the whole world bitwise --
    obstacle rows, spawns, goals, mounts -- and stay identical under steps
    with auto-resets (the multi-GPU sharding)."""
    from paper_2305_16510_b200 import world as W
    n = 64
    cfg = forest_cfg(W, n, seed=13)
    cfg.env.episode_max_steps = 25
    whole = W.World(cfg, pools=tree_pools())
    halves = []
    for first in (0, n // 2):
        c = forest_cfg(W, n // 2, seed=13)
        c.env.episode_max_steps = 25
        halves.append(W.World(c, pools=tree_pools(), first_env=first))
    rng = np.random.default_rng(5)
    for k in range(60):
        v = np.asarray(rng.normal(0.0, 2.0, (n, 3)), np.float32)
        cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(v=v, yaw_rate=np.zeros(n),
                                                                validate=False))
        whole.step(cmds)
        for h, (a, b) in zip(halves, ((0, n // 2), (n // 2, n))):
            hc = fs.CommandBatch.all_velocity(fs.VelocityCommands(
                v=v[a:b], yaw_rate=np.zeros(b - a), validate=False))
            h.step(hc)
    for h, (a, b) in zip(halves, ((0, n // 2), (n // 2, n))):
        assert torch.equal(h.pset._rec[:b - a], whole.pset._rec[a:b])
        assert torch.equal(h.states.buf[:, :b - a], whole.states.buf[:, a:b])
        assert torch.equal(h.goals, whole.goals[a:b])
        assert torch.equal(h.reset_counter, whole.reset_counter[a:b])
        assert torch.equal(h._mount[:, :b - a], whole._mount[:, a:b])
    assert int(whole.reset_counter.sum()) > 0


def _bench_forest(n, seed, camera):
    """bench.py's forest.yaml world (the render / forest bench workloads)."""
    import bench
    return bench.forest_sim_config(n, seed, camera=camera)


def test_full_size_render_sampled_envs_match_oracle(fs):
    """The render bench workload itself -- 1024 robots, 480x270, forest scene
    with randomized mounts -- checked against the oracle on sampled envs
    (every image is independent, so a sample is exact)."""
    from paper_2305_16510_b200 import world as W
    from paper_2305_16510_b200.camera import render
    cfg, pools = _bench_forest(1024, 7, camera=True)
    world = W.World(cfg, pools=pools)
    img = render(world, world.camera)
    torch.cuda.synchronize()
    host = world.pset.to_numpy()
    st = world.states.numpy()
    mp, mq = (t.cpu().numpy() for t in world.camera_mounts(world.camera))
    cam = world.camera
    for e in (0, 511, 1023):
        rd, rs = S.render(st[0:3].T, st[3:7].T, mp, mq, host, cam.width, cam.height, cam.hfov,
                          cam.max_range, envs=[e])
        bad = S.ill_conditioned_pixels(st[0:3].T, st[3:7].T, mp, mq, host, cam.width,
                                       cam.height, cam.hfov, cam.max_range, envs=[e])
        _check_images(img.depth[e:e + 1].cpu().numpy(), img.segmentation[e:e + 1].cpu().numpy(),
                      rd, rs, bad, f"env {e}")


def test_full_size_forest_collision_flags(fs):
    """The forest bench workload (2^21 envs): after steps with crashes and
    auto-resets, the collision flag of sampled envs equals the oracle's
    check_collisions on the device's own rows and positions."""
    from paper_2305_16510_b200 import world as W
    n = 1 << 21
    cfg, pools = _bench_forest(n, 3, camera=False)
    world = W.World(cfg, pools=pools)
    g = torch.Generator(device="cpu").manual_seed(3)
    v = (torch.randn(n, 3, generator=g) * 3.0).cuda()
    cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(v=v, yaw_rate=torch.zeros(n).cuda(),
                                                            validate=False))
    for _ in range(60):
        res = world.step(cmds)
    rng = np.random.default_rng(0)
    idx = np.sort(rng.choice(n, 512, replace=False))
    coll = res.info["collision"].cpu().numpy()[idx]
    auto = res.info["autoreset"].cpu().numpy()[idx]
    p = world.states.numpy()[0:3][:, idx].T
    full = world.pset.to_numpy()
    sub = {k: v[idx] for k, v in full.items()}
    want, oob = S.check_collisions(p, 0.2, sub, cfg.env.bounds)
    live = ~auto
    np.testing.assert_array_equal(coll[live], want[live])
    assert want[live].any() and (~want[live]).any()
    np.testing.assert_array_equal(res.info["out_of_bounds"].cpu().numpy()[idx][live], oob[live])


@pytest.mark.parametrize("n", [4096, (1 << 15) + 4096])
def test_clearance_cache_is_bitwise_transparent(fs, n):
    """The collision clearance cache (fs_obstacles.clear) only skips tests
    that cannot hit: a forest world stepped with the cache and the same world
    with it disabled agree bitwise on every output over 300 steps with
    crashes, truncations and auto-resets (which invalidate the cache), and
    the cache ends up valid for most envs (the skip path ran).  n = 4096 runs
    the thread-per-env step kernel; n = 2^15 + 4096 the streaming one, which
    also defers the auto-resets through the skipped-env list
    (fs_obstacles.reset_list) to after the step kernel; the obstacle rows and
    instance boxes agree bitwise as well."""
    from paper_2305_16510_b200 import world as W
    cfgs = [_bench_forest(n, 11, camera=False) for _ in range(3)]
    for c, _ in cfgs:
        c.env.episode_max_steps = 120
    a = W.World(cfgs[0][0], pools=cfgs[0][1])
    b = W.World(cfgs[1][0], pools=cfgs[1][1])
    c3 = W.World(cfgs[2][0], pools=cfgs[2][1])
    assert a._clear is not None and a._ob.worklist     # a: cache + deferred worklist test
    b._ob.clear = None                       # b: the full test every step, inline
    c3._ob.worklist = None                   # c3: cache, inline test
    worlds = (a, c3)
    g = torch.Generator(device="cpu").manual_seed(11)
    v = (torch.randn(n, 3, generator=g) * 1.5).cuda()
    cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(v=v, yaw_rate=torch.zeros(n).cuda(),
                                                            validate=False))
    crashes = 0
    for k in range(300):
        rb = b.step(cmds)
        for w in worlds:
            r = w.step(cmds)
            if w is a:
                ra = r
            assert torch.equal(w.states.buf[:, :n], b.states.buf[:, :n]), k
            assert torch.equal(r.reward, rb.reward), k
            assert torch.equal(w._info[:n], b._info[:n]), k
            assert torch.equal(w._pending[:n], b._pending[:n]), k
            assert torch.equal(r.observations, rb.observations), k
        crashes += int(ra.info["collision"].sum())
    for w in worlds:
        assert torch.equal(w.pset._rec[:n], b.pset._rec[:n])
        assert torch.equal(w._inst_box[:, :n], b._inst_box[:, :n])
    assert int(a._worklist[0]) == 0              # emptied by the last block
    if n >= (1 << 15):
        assert int(a._reset_list[0]) == 0        # the skipped envs were reset and the list emptied
    assert crashes > 0
    valid = (a._clear[3, :n] > 0).float().mean().item()
    assert valid > 0.5, valid


def test_deferred_resets_with_host_written_pending_flags(fs):
    """The streaming path defers the auto-resets (fs_obstacles.reset_list):
    it skips the envs pending at the step's start and resets them after the
    step kernel.  Against the same world resetting first (no list), over 150
    steps with crashes, truncations and pending flags written from the host
    every 25 steps: every output, the obstacle rows and instance boxes agree
    bitwise, and the list is empty after every step."""
    from paper_2305_16510_b200 import world as W
    n = (1 << 15) + 4096
    cfgs = [_bench_forest(n, 17, camera=False) for _ in range(2)]
    for c, _ in cfgs:
        c.env.episode_max_steps = 90
    a = W.World(cfgs[0][0], pools=cfgs[0][1])
    b = W.World(cfgs[1][0], pools=cfgs[1][1])
    assert a._ob.reset_list
    b._ob.reset_list = None                  # b: auto-resets first, every pending flag scanned
    g = torch.Generator(device="cpu").manual_seed(17)
    v = (torch.randn(n, 3, generator=g) * 1.5).cuda()
    cmds = fs.CommandBatch.all_velocity(fs.VelocityCommands(v=v, yaw_rate=torch.zeros(n).cuda(),
                                                            validate=False))
    resets = 0
    for k in range(150):
        if k % 25 == 24:
            pend = (torch.rand(n, generator=g) < 0.05).to(torch.uint8)
            pend |= a._pending[:n].cpu()
            for w in (a, b):
                w.load(pending=pend)
        ra = a.step(cmds)
        rb = b.step(cmds)
        assert torch.equal(a.states.buf[:, :n], b.states.buf[:, :n]), k
        assert torch.equal(ra.reward, rb.reward), k
        assert torch.equal(a._info[:n], b._info[:n]), k
        assert torch.equal(a._pending[:n], b._pending[:n]), k
        assert torch.equal(ra.observations, rb.observations), k
        assert torch.equal(a._goal[:, :n], b._goal[:, :n]), k
        assert int(a._reset_list[0]) == 0, k
        resets += int(((a._info[:n] & fs._native.FS_INFO_AUTORESET) != 0).sum())
    assert torch.equal(a.pset._rec[:n], b.pset._rec[:n])
    assert torch.equal(a._inst_box[:, :n], b._inst_box[:, :n])
    assert resets > 1000, resets
