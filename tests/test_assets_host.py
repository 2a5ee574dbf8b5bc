"""CPU tests of the host-side asset / scene-construction mirror
(paper_2305_16510_b200.assets, assets.py in the reference) and the camera
config: URDF subset parsing and its errors, class-directory pools, sampling
and pose randomization, procedural trees, and the camera mount -- the
behaviours the reference's tests/test_assets.py and test_camera.py check."""

import math

import numpy as np
import pytest

from paper_2305_16510_b200 import _se3
from paper_2305_16510_b200 import assets as A
from paper_2305_16510_b200.camera import CameraConfig, _pixel_rays, randomize_mount


def urdf(body: str) -> str:
    return f'<robot name="t">{body}</robot>'


BOX_LINK = ('<link name="base"><collision><origin xyz="1 2 3" rpy="0 0 0"/><geometry>'
            '<box size="1 2 3"/></geometry></collision></link>')


class TestParser:
    def test_box_with_origin(self):
        p = A.parse_urdf_subset(urdf(BOX_LINK), class_name="c")
        assert p.class_name == "c" and len(p.primitives) == 1
        prim = p.primitives[0]
        assert prim.kind == A.BOX and prim.dims == (1.0, 2.0, 3.0)
        np.testing.assert_array_equal(prim.position, [1.0, 2.0, 3.0])
        np.testing.assert_allclose(prim.rotation, [1, 0, 0, 0], atol=0)

    def test_joint_chain_composes_poses(self):
        # child link 1 m along the parent's x, parent yawed by 90 degrees:
        # the child's sphere lands at (0, 1, 0) in the asset frame
        text = urdf('<link name="a"><collision><geometry><sphere radius="0.1"/></geometry>'
                    '</collision></link>'
                    '<link name="b"><collision><geometry><sphere radius="0.2"/></geometry>'
                    '</collision></link>'
                    '<joint name="j" type="fixed"><parent link="a"/><child link="b"/>'
                    f'<origin xyz="0 0 0" rpy="0 0 {math.pi / 2!r}"/></joint>'
                    '<link name="c"><collision><geometry><cylinder radius="0.1" length="1"/>'
                    '</geometry></collision></link>'
                    '<joint name="k" type="fixed"><parent link="b"/><child link="c"/>'
                    '<origin xyz="1 0 0"/></joint>')
        p = A.parse_urdf_subset(text)
        assert [q.kind for q in p.primitives] == [A.SPHERE, A.SPHERE, A.CYLINDER]
        np.testing.assert_allclose(p.primitives[2].position, [0.0, 1.0, 0.0], atol=1e-12)
        # the cylinder inherits the 90-degree yaw
        np.testing.assert_allclose(_se3.quat_rotate(p.primitives[2].rotation, [1, 0, 0]),
                                   [0, 1, 0], atol=1e-12)

    @pytest.mark.parametrize("geom,err", [
        ('<mesh filename="x.stl"/>', A.UnsupportedGeometryError),
        ('<cylinder radius="0" length="1"/>', A.InvalidGeometryError),
        ('<box size="1 2"/>', A.InvalidGeometryError),
        ('<box size="1 -2 3"/>', A.InvalidGeometryError),
        ('<sphere radius="-1"/>', A.InvalidGeometryError),
    ])
    def test_bad_geometry(self, geom, err):
        with pytest.raises(err):
            A.parse_urdf_subset(urdf(f'<link name="l"><collision><geometry>{geom}</geometry>'
                                     '</collision></link>'))

    def test_malformed_xml_reports_position(self):
        with pytest.raises(A.MalformedXmlError, match="line"):
            A.parse_urdf_subset("<robot><link></robot>")

    def test_wrong_root(self):
        with pytest.raises(A.MalformedXmlError, match="robot"):
            A.parse_urdf_subset("<model/>")

    def test_revolute_joint_rejected(self):
        text = urdf(BOX_LINK + '<link name="b"/>'
                    '<joint name="j" type="revolute"><parent link="base"/><child link="b"/></joint>')
        with pytest.raises(A.UnsupportedGeometryError, match="fixed"):
            A.parse_urdf_subset(text)

    def test_two_roots_and_unknown_links(self):
        with pytest.raises(A.InvalidGeometryError, match="root"):
            A.parse_urdf_subset(urdf(BOX_LINK + '<link name="other"><collision><geometry>'
                                     '<sphere radius="1"/></geometry></collision></link>'))
        with pytest.raises(A.InvalidGeometryError, match="unknown link"):
            A.parse_urdf_subset(urdf(BOX_LINK + '<joint name="j" type="fixed">'
                                     '<parent link="base"/><child link="nope"/></joint>'))

    def test_visual_only_asset_is_empty(self):
        with pytest.raises(A.InvalidGeometryError, match="no primitives"):
            A.parse_urdf_subset(urdf('<link name="l"><visual><geometry><box size="1 1 1"/>'
                                     '</geometry></visual></link>'))


class TestPools:
    def test_census_sorted(self, tmp_path):
        for cls, names in (("rocks", ["b", "a"]), ("poles", ["x"])):
            d = tmp_path / cls
            d.mkdir()
            for n in names:
                (d / f"{n}.urdf").write_text(urdf(BOX_LINK))
        pools = A.load_asset_dir(tmp_path)
        assert list(pools) == ["poles", "rocks"]
        assert [p.source.split("/")[-1] for p in pools["rocks"]] == ["a.urdf", "b.urdf"]
        assert all(p.class_name == "rocks" for p in pools["rocks"])

    def test_empty_class_dir(self, tmp_path):
        (tmp_path / "empty").mkdir()
        with pytest.raises(A.EmptyClassDirError):
            A.load_asset_dir(tmp_path)

    def test_parse_error_carries_file(self, tmp_path):
        (tmp_path / "bad").mkdir()
        (tmp_path / "bad" / "dud.urdf").write_text("<robot><link></robot>")
        with pytest.raises(A.AssetParseError, match="dud.urdf") as exc:
            A.load_asset_dir(tmp_path)
        assert exc.value.path.endswith("dud.urdf")

    def test_missing_root(self, tmp_path):
        with pytest.raises(FileNotFoundError):
            A.load_asset_dir(tmp_path / "nope")


def pools3():
    return {"trees": [A.generate_tree(A.TreeConfig(seed=s, depth=2))[0] for s in range(3)]}


class TestSampling:
    def test_counts_and_fields(self):
        cfg = A.AssetClassConfig(name="trees", count_per_env=7, segmentation_id=4,
                                 collision_enabled=False)
        inst = A.sample_env_assets(pools3(), [cfg], A.env_stream(1, 2, 0), env_index=2)
        assert len(inst) == 7
        assert all(i.segmentation_id == 4 and i.env_index == 2 and not i.collision_enabled
                   for i in inst)
        assert A.sample_env_assets(pools3(), [A.AssetClassConfig(name="trees")],
                                   A.env_stream(1, 2, 0)) == []

    def test_streams_are_counter_based(self):
        a = A.env_stream(5, 3, 1).uniform(size=4)
        b = A.env_stream(5, 3, 1).uniform(size=4)
        c = A.env_stream(5, 3, 2).uniform(size=4)
        d = A.env_stream(5, 4, 1).uniform(size=4)
        assert np.array_equal(a, b) and not np.array_equal(a, c) and not np.array_equal(a, d)

    def test_unknown_class(self):
        with pytest.raises(A.UnknownClassError):
            A.sample_env_assets(pools3(), [A.AssetClassConfig(name="rocks", count_per_env=1)],
                                A.env_stream(0, 0, 0))

    def test_frozen_component_and_bounds(self):
        cfg = A.AssetClassConfig(name="trees", count_per_env=1, position_min=[0.2, 0.1, 0.5],
                                 position_max=[0.4, 0.9, 0.5], frozen=(None, None, 0.0),
                                 euler_min=[0, 0, -1.0], euler_max=[0, 0, 1.0])
        bounds = np.array([10.0, 20.0, 4.0])
        rng = A.env_stream(9, 0, 0)
        base = A.sample_env_assets(pools3(), [cfg], rng)[0]
        for _ in range(200):
            inst = A.randomize_pose(base, cfg, bounds, rng)
            assert inst.position[2] == 0.0
            assert 2.0 <= inst.position[0] <= 4.0 and 2.0 <= inst.position[1] <= 18.0
            # yaw only, within +-1 rad: R e3 = e3 and |yaw| <= 1
            q = inst.rotation
            np.testing.assert_allclose(_se3.quat_rotate(q, [0, 0, 1]), [0, 0, 1], atol=1e-12)
            assert abs(2.0 * math.atan2(q[3], q[0])) <= 1.0 + 1e-12

    def test_config_validation(self):
        for kw in (dict(count_per_env=-1), dict(position_min=[0.6, 0, 0], position_max=[0.5, 1, 1]),
                   dict(euler_min=[1, 0, 0]), dict(segmentation_id=0), dict(frozen=(None, None))):
            with pytest.raises(ValueError):
                A.AssetClassConfig(name="x", **kw)


class TestTrees:
    def test_counts(self):
        assert A.TreeConfig(depth=1).primitive_count == 1
        assert A.TreeConfig(depth=4, branch_factor=3).primitive_count == 1 + 3 + 9 + 27
        assert A.TreeConfig(depth=5, branch_factor=1).primitive_count == 5
        proto, _ = A.generate_tree(A.TreeConfig(depth=3, seed=4))
        assert len(proto.primitives) == 7 and all(p.kind == A.CYLINDER for p in proto.primitives)

    def test_deterministic_and_reparses(self):
        p1, t1 = A.generate_tree(A.TreeConfig(seed=11))
        p2, t2 = A.generate_tree(A.TreeConfig(seed=11))
        assert t1 == t2
        again = A.parse_urdf_subset(t1)
        for a, b in zip(p1.primitives, again.primitives):
            assert a.dims == b.dims
            np.testing.assert_array_equal(a.position, b.position)
            np.testing.assert_array_equal(a.rotation, b.rotation)

    def test_decay_and_trunk(self):
        cfg = A.TreeConfig(depth=3, trunk_length=2.0, trunk_radius=0.1, length_decay=0.5,
                           radius_decay=0.5)
        proto, _ = A.generate_tree(cfg)
        radii = sorted({p.dims[0] for p in proto.primitives}, reverse=True)
        lengths = sorted({p.dims[1] for p in proto.primitives}, reverse=True)
        np.testing.assert_allclose(radii, [0.1, 0.05, 0.025])
        np.testing.assert_allclose(lengths, [2.0, 1.0, 0.5])
        np.testing.assert_allclose(proto.primitives[0].position, [0, 0, 1.0])

    def test_limits_and_validation(self):
        with pytest.raises(A.TooManyPrimitivesError):
            A.generate_tree(A.TreeConfig(depth=20, branch_factor=2))
        for kw in (dict(depth=0), dict(length_decay=1.5), dict(branch_factor=-1),
                   dict(trunk_radius=0.0)):
            with pytest.raises(ValueError):
                A.TreeConfig(**kw)


class TestCameraConfig:
    def test_defaults_and_validation(self):
        c = CameraConfig()
        assert (c.width, c.height, c.max_range) == (480, 270, 10.0)
        for kw in (dict(width=0), dict(hfov=4.0), dict(max_range=0.0)):
            with pytest.raises(ValueError):
                CameraConfig(**kw)

    def test_forward_mount(self):
        m = CameraConfig().mount_rotation
        np.testing.assert_allclose(_se3.quat_rotate(m, [0, 0, 1]), [1, 0, 0], atol=1e-12)
        np.testing.assert_allclose(_se3.quat_rotate(m, [1, 0, 0]), [0, -1, 0], atol=1e-12)
        np.testing.assert_allclose(_se3.quat_rotate(m, [0, 1, 0]), [0, 0, -1], atol=1e-12)

    def test_pixel_rays_unit_and_centered(self):
        d = _pixel_rays(8, 6, 1.2)
        np.testing.assert_allclose(np.linalg.norm(d, axis=1), 1.0, atol=1e-15)
        np.testing.assert_allclose(d[:, 0].reshape(6, 8).sum(axis=1), 0.0, atol=1e-12)

    def test_randomize_mount(self):
        cfg = CameraConfig(randomize_position=[0.01, 0.02, 0.0],
                           randomize_euler=[0.05, 0.0, 0.0])
        rng = np.random.default_rng(1)
        for _ in range(100):
            p, q = randomize_mount(cfg, rng)
            assert (np.abs(p - cfg.mount_position) <= [0.01, 0.02, 0.0]).all()
            np.testing.assert_allclose(np.linalg.norm(q), 1.0, atol=1e-12)
        p, q = randomize_mount(CameraConfig(), np.random.default_rng(0))
        np.testing.assert_array_equal(p, CameraConfig().mount_position)
        np.testing.assert_array_equal(q, CameraConfig().mount_rotation)
