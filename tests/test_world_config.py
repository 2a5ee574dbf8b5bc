"""CPU tests of the World config mirror (config.py:29-90 validation)."""

import pytest

from paper_2305_16510_b200 import world as W


@pytest.mark.parametrize("kw", [dict(num_envs=0), dict(bounds=[1, -1, 1]), dict(dt=0.2),
                                dict(episode_max_steps=0), dict(control_mode="position"),
                                dict(goal_min=[0.5, 0.5, 0.5], goal_max=[0.4, 0.9, 0.9]),
                                dict(spawn_max=[1.2, 0.5, 0.5]), dict(wall_thickness=0.0)])
def test_env_config_validation(kw):
    with pytest.raises(W.ConfigError):
        W.EnvConfig(**kw)


def test_defaults_match_reference():
    e, r = W.EnvConfig(), W.RewardConfig()
    assert list(e.bounds) == [10.0, 10.0, 5.0] and e.episode_max_steps == 1000 and e.dt == 0.01
    assert (r.c_dist, r.c_vel, r.c_step, r.c_success, r.c_crash, r.success_radius) == \
        (0.1, 0.01, 0.01, 10.0, 10.0, 0.2)
    assert W.OBS_DIM == 16 and W.PLACEMENT_ATTEMPTS == 100


def test_wall_prototype_geometry():
    """world.py:74-91: six slabs just outside the bounding planes (the
    reference's test_world.py:221-232 check, restated)."""
    proto = W.make_wall_prototype([10.0, 8.0, 4.0], 0.2)
    assert len(proto.primitives) == 6 and proto.class_name == W.WALL_CLASS
    lo_x, hi_x = proto.primitives[0], proto.primitives[1]
    assert lo_x.position[0] == -0.1 and abs(hi_x.position[0] - 10.1) < 1e-12
    assert tuple(lo_x.dims) == (0.2, 8.4, 4.4)
    floor = proto.primitives[4]
    assert floor.position[2] == -0.1 and tuple(floor.dims) == (10.4, 8.4, 0.2)
