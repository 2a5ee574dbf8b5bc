"""ctypes binding of the C ABI in include/flocksim_b200.h.

The product path has no CPU fallback: if the shared library is missing or
fails to load, every entry point raises ``NativeLibraryError``.  Build it
with ``python -m paper_2305_16510_b200.build`` (or ``__graft_entry__.build()``).
"""

from __future__ import annotations

import ctypes as C
import os

LIB_NAME = "libflocksim_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", LIB_NAME)

FS_ABI_VERSION = 8
FS_SYNC_GRANULE = 128
FS_OK = 0
FS_EINVAL = 22
FS_ELAUNCH = 1001

FS_MODE_ATTITUDE = 0
FS_MODE_VELOCITY = 1
FS_MODE_MIXED = 2
FS_MODE_POSITION = 3

FS_FLAG_CLAMPED = 1
FS_FLAG_NONFINITE = 2
FS_FLAG_GIMBAL = 4
FS_FLAG_DEGENERATE = 8
FS_FLAG_RESET = 16

FS_MAX_ROTORS = 6

FS_TUNE_KERNEL = 1
FS_TUNE_PREC = 2
FS_TUNE_CTAS_PER_SM = 3
FS_TUNE_NCW = 4
FS_TUNE_VPT = 5
FS_TUNE_WORLD_KERNEL = 6
FS_TUNE_CHAIN_RELEASE = 7
FS_TUNE_L2_KEEP_MB = 8
FS_TUNE_SYNC_TIMEOUT_MS = 9
FS_TUNE_CHAIN_ACQUIRE = 10
FS_TUNE_SPAWN_WAIT_NS = 11
FS_TUNE_CONS_WAIT_NS = 12
FS_TUNE_CLEAR_WALK_CM = 13
FS_TUNE_CLEAR_EXACT = 14


class NativeLibraryError(RuntimeError):
    """The CUDA extension is missing or unusable (there is no fallback)."""


class fs_robot(C.Structure):
    _fields_ = [
        ("mass", C.c_double),
        ("gravity", C.c_double),
        ("inertia", C.c_double * 9),
        ("inertia_inv", C.c_double * 9),
        ("thrust_max", C.c_double),
        ("moment_max", C.c_double * 3),
        ("v_limit", C.c_double),
        ("omega_limit", C.c_double),
        ("gimbal_cos", C.c_double),
    ]


class fs_gains(C.Structure):
    _fields_ = [
        ("attitude", C.c_double * 3),
        ("rate", C.c_double * 3),
        ("velocity", C.c_double * 3),
        ("position", C.c_double * 3),
    ]


class fs_limits(C.Structure):
    _fields_ = [
        ("max_tilt", C.c_double),
        ("max_speed_cmd", C.c_double),
        ("max_yaw_rate", C.c_double),
    ]


class fs_airframe(C.Structure):
    _fields_ = [
        ("n_rotors", C.c_int32),
        ("rotor_max", C.c_float),
        ("pinv", C.c_float * (FS_MAX_ROTORS * 4)),
        ("alloc", C.c_float * (4 * FS_MAX_ROTORS)),
    ]


class fs_step_desc(C.Structure):
    _fields_ = [
        ("n", C.c_int64),
        ("first_id", C.c_int64),
        ("state_in", C.c_void_p),
        ("state_in_stride", C.c_int64),
        ("state_out", C.c_void_p),
        ("state_out_stride", C.c_int64),
        ("mode", C.c_int32),
        ("integrate", C.c_int32),
        ("mode_per_vehicle", C.c_void_p),
        ("cmd", C.c_void_p),
        ("cmd_stride", C.c_int64),
        ("vparams", C.c_void_p),
        ("vparams_stride", C.c_int64),
        ("airframe_split", C.c_int64),
        ("wrench_out", C.c_void_p),
        ("wrench_stride", C.c_int64),
        ("rotor_out", C.c_void_p),
        ("rotor_stride", C.c_int64),
        ("flags_out", C.c_void_p),
        ("rotor_dynamics", C.c_int32),
        ("dt", C.c_float),
        ("reset_prob", C.c_float),
        ("seed", C.c_uint64),
        ("step_index", C.c_uint64),
        ("stats_slots", C.c_void_p),
        ("stats_nslots", C.c_int32),
        ("tile_sync", C.c_void_p),
        ("sync_wait", C.c_uint32),
        ("sync_post", C.c_uint32),
    ]


class fs_host_ws(C.Structure):
    _fields_ = [
        ("dev_state", C.c_void_p),
        ("dev_cmd", C.c_void_p),
        ("dev_mode", C.c_void_p),
        ("dev_wrench", C.c_void_p),
        ("dev_flags", C.c_void_p),
        ("dev_stride", C.c_int64),
        ("chunks", C.c_int32),
        ("nstreams", C.c_int32),
        ("streams", C.POINTER(C.c_void_p)),
    ]


class fs_world_cfg(C.Structure):
    _fields_ = [
        ("bounds", C.c_double * 3),
        ("spawn_lo", C.c_double * 3), ("spawn_hi", C.c_double * 3),
        ("goal_lo", C.c_double * 3), ("goal_hi", C.c_double * 3),
        ("collision_radius", C.c_double),
        ("episode_max_steps", C.c_int32),
        ("placement_attempts", C.c_int32),
        ("c_dist", C.c_double), ("c_vel", C.c_double), ("c_step", C.c_double),
        ("c_success", C.c_double), ("c_crash", C.c_double), ("success_radius", C.c_double),
    ]


FS_PRIM_PAD = -1
FS_PRIM_BOX = 0
FS_PRIM_CYLINDER = 1
FS_PRIM_SPHERE = 2
FS_PRIM_FIELDS = 24
FS_COLL_WALL = 2


class fs_scene(C.Structure):
    _fields_ = [
        ("num_envs", C.c_int64),
        ("width", C.c_int32),
        ("reserved_", C.c_int32),
        ("rec", C.c_void_p),
    ]


class fs_proto_prim(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("reserved_", C.c_int32),
        ("dims", C.c_double * 3),
        ("position", C.c_double * 3),
        ("rotation", C.c_double * 4),
    ]


class fs_asset_class(C.Structure):
    _fields_ = [
        ("position_min", C.c_double * 3), ("position_max", C.c_double * 3),
        ("euler_min", C.c_double * 3), ("euler_max", C.c_double * 3),
        ("frozen_value", C.c_double * 3),
        ("frozen_mask", C.c_int32),
        ("segmentation_id", C.c_int32),
        ("collision_enabled", C.c_int32),
        ("count_per_env", C.c_int32),
        ("pool_first", C.c_int32),
        ("pool_size", C.c_int32),
    ]


class fs_obstacles(C.Structure):
    _fields_ = [
        ("scene", fs_scene),
        ("num_classes", C.c_int32),
        ("instances_per_env", C.c_int32),
        ("classes", C.c_void_p),
        ("proto_offset", C.c_void_p),
        ("proto_prims", C.c_void_p),
        ("plane_stride", C.c_int64),
        ("inst_proto", C.c_void_p),
        ("inst_pose", C.c_void_p),
        ("wall_proto", C.c_int32),
        ("wall_seg", C.c_int32),
        ("mount", C.c_void_p),
        ("mount_stride", C.c_int64),
        ("mount_position", C.c_double * 3), ("mount_euler", C.c_double * 3),
        ("randomize_position", C.c_double * 3), ("randomize_euler", C.c_double * 3),
        ("inst_box", C.c_void_p),
        ("clear", C.c_void_p),
        ("worklist", C.c_void_p),
        ("reset_list", C.c_void_p),
        ("walk_slots", C.c_void_p),
    ]


class fs_camera(C.Structure):
    _fields_ = [
        ("width", C.c_int32),
        ("height", C.c_int32),
        ("pixel_scale", C.c_double),
        ("max_range", C.c_double),
        ("mount_position", C.c_double * 3),
        ("mount_rotation", C.c_double * 4),
    ]


class fs_world_desc(C.Structure):
    _fields_ = [
        ("step", fs_step_desc),
        ("goal", C.c_void_p),
        ("goal_stride", C.c_int64),
        ("steps_in_episode", C.c_void_p),
        ("reset_counter", C.c_void_p),
        ("pending_reset", C.c_void_p),
        ("obs", C.c_void_p),
        ("obs_stride", C.c_int64),
        ("reward", C.c_void_p),
        ("info", C.c_void_p),
        ("obstacles", C.POINTER(fs_obstacles)),
    ]


FS_INFO_TERMINATED = 1
FS_INFO_TRUNCATED = 2
FS_INFO_COLLISION = 4
FS_INFO_OUT_OF_BOUNDS = 8
FS_INFO_NONFINITE = 16
FS_INFO_AUTORESET = 32
FS_INFO_PLACEMENT_FAILED = 64

FS_SE3_OPS = ("QUAT_NORMALIZE", "QUAT_MULTIPLY", "QUAT_CONJUGATE", "QUAT_ROTATE",
              "QUAT_ROTATE_INVERSE", "QUAT_TO_MATRIX", "QUAT_FROM_MATRIX", "ROT_ZYX", "ROT_Z",
              "YAW_OF", "EXP_SO3", "HAT", "VEE")
FS_SE3 = {name: code for code, name in enumerate(FS_SE3_OPS)}

FS_DTYPE_F32 = 0
FS_DTYPE_F64 = 1

_P = C.c_void_p
_I64 = C.c_int64
_SIGS = {
    "fs_abi_version": (C.c_int, []),
    "fs_set_tuning": (C.c_int, [C.c_int32, C.c_int32]),
    "fs_last_error": (C.c_char_p, []),
    "fs_device_sm_count": (C.c_int, []),
    "fs_tile_sync_len": (C.c_int64, [_I64]),
    "fs_step": (C.c_int, [C.POINTER(fs_step_desc), C.POINTER(fs_robot), C.POINTER(fs_gains),
                          C.POINTER(fs_limits), C.POINTER(fs_airframe), _P]),
    "fs_step_host_ex": (C.c_int, [C.POINTER(fs_step_desc), C.POINTER(fs_robot),
                                  C.POINTER(fs_gains), C.POINTER(fs_limits),
                                  C.POINTER(fs_airframe), C.POINTER(fs_host_ws)]),
    "fs_step_host": (C.c_int, [C.POINTER(fs_step_desc), C.POINTER(fs_robot), C.POINTER(fs_gains),
                               C.POINTER(fs_limits), C.POINTER(fs_airframe), _P, _P, _I64,
                               C.c_int32, C.POINTER(C.c_void_p), C.c_int32]),
    "fs_step_many": (C.c_int, [C.POINTER(fs_step_desc), C.POINTER(fs_robot), C.POINTER(fs_gains),
                               C.POINTER(fs_limits), C.POINTER(fs_airframe), C.c_int32, _P]),
    "fs_host_pack_f64": (C.c_int, [_P, _I64, C.c_int32, _I64, _P, _I64, C.c_int32]),
    "fs_host_unpack_f64": (C.c_int, [_P, _I64, _I64, C.c_int32, _P, _I64, C.c_int32]),
    "fs_rollout": (C.c_int, [C.POINTER(fs_step_desc), C.POINTER(fs_robot), C.POINTER(fs_gains),
                             C.POINTER(fs_limits), C.POINTER(fs_airframe), C.c_int32, _P]),
    "fs_integrate": (C.c_int, [_I64, _P, _I64, _P, _I64, C.POINTER(fs_robot), C.c_float, _P,
                               _I64, _P, _P]),
    "fs_saturate": (C.c_int, [_I64, _P, _I64, C.POINTER(fs_robot), _P, _I64, _P]),
    "fs_velocity_control": (C.c_int, [_I64, _P, _I64, _P, _I64, C.POINTER(fs_robot),
                                      C.POINTER(fs_gains), C.POINTER(fs_limits), _P, _I64, _P,
                                      _P]),
    "fs_attitude_control": (C.c_int, [_I64, _P, _I64, _P, _I64, C.POINTER(fs_robot),
                                      C.POINTER(fs_gains), _P, _I64, _P]),
    "fs_yaw_of": (C.c_int, [_I64, _P, _I64, C.c_double, _P, _P, _P]),
    "fs_desired_attitude": (C.c_int, [_I64, _P, _P, _I64, _P, _I64, _P, _I64, _P]),
    "fs_attitude_errors": (C.c_int, [_I64, _P, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _P,
                                     _I64, _P]),
    "fs_init_fleet": (C.c_int, [_I64, _I64, C.c_uint64, C.c_int32, _P, _I64, _P, _I64, _P,
                                _I64, C.POINTER(fs_robot), _P]),
    "fs_stats_reduce": (C.c_int, [_P, C.c_int32, _P, _P]),
    "fs_world_step": (C.c_int, [C.POINTER(fs_world_desc), C.POINTER(fs_world_cfg),
                                C.POINTER(fs_robot), C.POINTER(fs_gains), C.POINTER(fs_limits),
                                _P]),
    "fs_world_reset": (C.c_int, [C.POINTER(fs_world_desc), C.POINTER(fs_world_cfg), _P,
                                 C.c_int32, _P]),
    "fs_vecenv_step": (C.c_int, [C.POINTER(fs_world_desc), C.POINTER(fs_world_cfg),
                                 C.POINTER(fs_robot), C.POINTER(fs_gains), C.POINTER(fs_limits),
                                 _P, C.c_int32, _I64, _P]),
    "fs_scene_distances": (C.c_int, [C.POINTER(fs_scene), _P, _I64, C.c_int32, _P, _I64, _P,
                                     _P]),
    "fs_cast_rays": (C.c_int, [C.POINTER(fs_scene), _I64, C.c_double, C.c_double, C.c_double,
                               _P, _I64, C.c_double, _P, _P, _P]),
    "fs_render": (C.c_int, [C.POINTER(fs_scene), C.POINTER(fs_camera), _P, _I64, _P, _I64,
                            _I64, _I64, _P, _P, _P]),
    "fs_obstacles_pick": (C.c_int, [C.POINTER(fs_obstacles), _I64, _I64, C.c_uint64, _P, _P]),
    "fs_obstacles_poses": (C.c_int, [C.POINTER(fs_obstacles), _I64, _I64, C.c_uint64, _P,
                                     C.POINTER(C.c_double), _P]),
    "fs_se3": (C.c_int, [C.c_int32, _I64, _P, _P, _P, _P, _P, _P]),
}

EXPORTED_SYMBOLS = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load (once) and return the native library; raises if unavailable."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NativeLibraryError(
            f"{path} not found: build it with `python -m paper_2305_16510_b200.build` "
            "(there is no CPU fallback)")
    try:
        lib = C.CDLL(path)
    except OSError as exc:
        raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.fs_abi_version() != FS_ABI_VERSION:
        raise NativeLibraryError("ABI version mismatch between header and library")
    _lib = lib
    return lib


def set_tuning(key: int, value: int) -> None:
    """Process-wide kernel selection (benchmarks/diagnostics only)."""
    check(load().fs_set_tuning(key, value), "fs_set_tuning")


def check(rc: int, what: str) -> None:
    """Map a status code to the reference's exception types."""
    if rc == FS_OK:
        return
    msg = load().fs_last_error().decode(errors="replace")
    if rc == FS_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed ({rc}): {msg}")
