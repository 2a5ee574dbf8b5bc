"""CPU oracle for the batched multirotor control step.

TEST INFRASTRUCTURE ONLY.  This module is the checker, never the product:
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
``--impl reference`` legs may import it.  The product path
(``paper_2305_16510_b200``) never imports it and has no CPU fallback.

What it is
----------
A float64 NumPy restatement of the reference's hot path
(``flocksim.control.control_batch`` followed by ``flocksim.dynamics.step_batch``)
over the same *planar* structure-of-arrays layout the CUDA kernels use:
a state is a ``(13, N)`` float64 array whose rows are
``px py pz | qw qx qy qz | vx vy vz | wx wy wz``.  Every function cites the
reference ``file:line`` (relative to ``/root/reference/pkg/src/flocksim``) whose
arithmetic it restates.  Operation order follows the reference expression by
expression so that, on identical float64 inputs, results agree with the
reference to the last bit in practice (the golden-vector tests pin this at
1e-12 relative, see ``tests/test_oracle_golden.py``).

Pinning
-------
* attitude / velocity / mixed control and the integrator: pinned against
  golden vectors produced by running the reference itself in the build
  container (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``) and
  against the reference's own known-answer cases.
* position controller, wrench->rotor allocation, per-vehicle parameters,
  reset RNG and episode statistics are EXTENSIONS that do not exist in the
  reference.  They are builder-defined here and in
  DESIGN.md section 5; their parity is **unpinned** by the reference and is
  established only by property tests (hover fixed point, A*A+ = I,
  convergence, yaw tracking).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# --- constants (reference: se3.py:19-25, control.py:33, dynamics.py:31) ------
EXP_TAYLOR_ANGLE = 1e-8          # se3.py:19
GIMBAL_TOL = 1e-6                # se3.py:25
DEGENERATE_ACCEL = 1e-6          # control.py:33
DEFAULT_GRAVITY = 9.81           # dynamics.py:31

MODE_ATTITUDE = 0                # control.py:29
MODE_VELOCITY = 1                # control.py:30

# planar state rows
PX, PY, PZ, QW, QX, QY, QZ, VX, VY, VZ, WX, WY, WZ = range(13)
NSTATE = 13


@dataclass
class Robot:
    """Shared physical parameters; defaults from dynamics.py:54-63."""

    mass: float = 1.0
    inertia: np.ndarray = field(default_factory=lambda: np.diag([0.01, 0.01, 0.02]))
    thrust_max: float = 25.0
    moment_max: np.ndarray = field(default_factory=lambda: np.array([2.0, 2.0, 1.0]))
    gravity: float = DEFAULT_GRAVITY
    v_limit: float = 50.0
    omega_limit: float = 100.0

    def __post_init__(self):
        self.inertia = np.asarray(self.inertia, dtype=np.float64)
        self.moment_max = np.asarray(self.moment_max, dtype=np.float64)
        self.inertia_inv = np.linalg.inv(self.inertia)   # dynamics.py:82

    @property
    def hover_thrust(self) -> float:                      # dynamics.py:89-90
        return self.mass * self.gravity


@dataclass
class Gains:
    """Diagonal gains; defaults from control.py:48-50 (+ position: extension)."""

    attitude: np.ndarray = field(default_factory=lambda: np.array([8.0, 8.0, 2.0]))
    rate: np.ndarray = field(default_factory=lambda: np.array([1.2, 1.2, 0.6]))
    velocity: np.ndarray = field(default_factory=lambda: np.array([3.0, 3.0, 3.0]))
    position: np.ndarray = field(default_factory=lambda: np.array([2.0, 2.0, 2.0]))


@dataclass
class Limits:
    """Command envelope; defaults from control.py:66-68."""

    max_tilt: float = 0.6
    max_speed_cmd: float = 5.0
    max_yaw_rate: float = 3.0


# =============================================================================
# rotation primitives (se3.py)
# =============================================================================

def quat_normalize(w, x, y, z):
    """se3.py:70-75 -- divide by the Euclidean norm."""
    n = np.sqrt(w * w + x * x + y * y + z * z)
    return w / n, x / n, y / n, z / n


def quat_mul(a, b):
    """Hamilton product, renormalized (se3.py:78-97)."""
    aw, ax, ay, az = a
    bw, bx, by, bz = b
    return quat_normalize(
        aw * bw - ax * bx - ay * by - az * bz,
        aw * bx + ax * bw + ay * bz - az * by,
        aw * by - ax * bz + ay * bw + az * bx,
        aw * bz + ax * by - ay * bx + az * bw,
    )


def quat_rotate(q, u):
    """R(q) u via t = 2 q_v x u; u + w t + q_v x t (se3.py:106-130)."""
    w, x, y, z = q
    ux, uy, uz = u
    tx = 2.0 * (y * uz - z * uy)
    ty = 2.0 * (z * ux - x * uz)
    tz = 2.0 * (x * uy - y * ux)
    return (ux + w * tx + (y * tz - z * ty),
            uy + w * ty + (z * tx - x * tz),
            uz + w * tz + (x * ty - y * tx))


def rotmat(q):
    """Nine entries r[i][j] of R(q) (se3.py:138-153)."""
    w, x, y, z = q
    return (
        (1.0 - 2.0 * (y * y + z * z), 2.0 * (x * y - w * z), 2.0 * (x * z + w * y)),
        (2.0 * (x * y + w * z), 1.0 - 2.0 * (x * x + z * z), 2.0 * (y * z - w * x)),
        (2.0 * (x * z - w * y), 2.0 * (y * z + w * x), 1.0 - 2.0 * (x * x + y * y)),
    )


def rot_zyx(roll, pitch, yaw):
    """R_z(yaw) R_y(pitch) R_x(roll) as a quaternion (se3.py:200-215)."""
    hr, hp, hy = roll / 2.0, pitch / 2.0, yaw / 2.0
    zero = np.zeros_like(np.asarray(hr, dtype=np.float64))
    qx = (np.cos(hr), np.sin(hr), zero, zero)
    qy = (np.cos(hp), zero, np.sin(hp), zero)
    qz = (np.cos(hy), zero, zero, np.sin(hy))
    return quat_mul(qz, quat_mul(qy, qx))


def yaw_of(q):
    """psi = atan2(r10, r00) and the gimbal flag (se3.py:226-243)."""
    w, x, y, z = q
    r10 = 2.0 * (x * y + w * z)
    r00 = 1.0 - 2.0 * (y * y + z * z)
    r20 = 2.0 * (x * z - w * y)
    return np.arctan2(r10, r00), np.abs(r20) >= np.cos(GIMBAL_TOL)


def exp_so3(wx, wy, wz):
    """Rodrigues as a unit quaternion with a series branch (se3.py:246-266)."""
    theta = np.sqrt(wx * wx + wy * wy + wz * wz)
    small = theta < EXP_TAYLOR_ANGLE
    safe = np.where(small, 1.0, theta)
    k = np.where(small, 0.5 - theta * theta / 48.0, np.sin(safe / 2.0) / safe)
    return quat_normalize(np.cos(theta / 2.0), k * wx, k * wy, k * wz)


# =============================================================================
# controller (control.py)
# =============================================================================

def desired_attitude(yaw, roll, pitch, yaw_rate):
    """q_d = rot_zyx(roll, pitch, yaw); omega_d via the Euler-rate map
    (control.py:190-218, Eq. 2)."""
    q_d = rot_zyx(roll, pitch, yaw)
    sp, cp = np.sin(pitch), np.cos(pitch)
    sr, cr = np.sin(roll), np.cos(roll)
    return q_d, (-sp * yaw_rate, sr * cp * yaw_rate, cr * cp * yaw_rate)


def _rdt_r(rd, r):
    """a[i][j] = sum_k rd[k][i] r[k][j] evaluated as control.py:234-239."""
    return [[rd[0][i] * r[0][j] + rd[1][i] * r[1][j] + rd[2][i] * r[2][j]
             for j in range(3)] for i in range(3)]


def attitude_errors_mat(r, omega, rd, omega_d):
    """e_R, e_W from rotation-matrix entries (control.py:221-258, Eqs. 3-4)."""
    a = _rdt_r(rd, r)
    e_rot = (0.5 * (a[2][1] - a[1][2]),
             0.5 * (a[0][2] - a[2][0]),
             0.5 * (a[1][0] - a[0][1]))
    wd = omega_d
    wd_body = (a[0][0] * wd[0] + a[1][0] * wd[1] + a[2][0] * wd[2],
               a[0][1] * wd[0] + a[1][1] * wd[1] + a[2][1] * wd[2],
               a[0][2] * wd[0] + a[1][2] * wd[1] + a[2][2] * wd[2])
    return e_rot, tuple(omega[i] - wd_body[i] for i in range(3))


def attitude_errors(q, omega, q_d, omega_d):
    """control.py:221-258 on quaternions."""
    return attitude_errors_mat(rotmat(q), omega, rotmat(q_d), omega_d)


def gyro_term(omega, inertia):
    """omega x (J omega) with J's entries as scalars (control.py:271-277)."""
    wx, wy, wz = omega
    j = inertia
    jwx = j[0, 0] * wx + j[0, 1] * wy + j[0, 2] * wz
    jwy = j[1, 0] * wx + j[1, 1] * wy + j[1, 2] * wz
    jwz = j[2, 0] * wx + j[2, 1] * wy + j[2, 2] * wz
    return (wy * jwz - wz * jwy, wz * jwx - wx * jwz, wx * jwy - wy * jwx)


def saturate(thrust, moment, robot: Robot):
    """Clamp thrust to [0, f_max] and each moment to +-M_max (dynamics.py:214-218)."""
    f = np.clip(thrust, 0.0, robot.thrust_max)
    m = tuple(np.clip(moment[i], -robot.moment_max[i], robot.moment_max[i])
              for i in range(3))
    return f, m


def moment_law(e_rot, e_rate, omega, gains: Gains, inertia):
    """M = -k_R e_R - k_W e_W + omega x J omega (control.py:279, Eq. 5)."""
    g = gyro_term(omega, inertia)
    return tuple(-gains.attitude[i] * e_rot[i] - gains.rate[i] * e_rate[i] + g[i]
                 for i in range(3))


def attitude_control(s, roll, pitch, yaw_rate, thrust, gains: Gains, robot: Robot):
    """Attitude-mode law -> saturated (thrust, moment) (control.py:261-280)."""
    q = (s[QW], s[QX], s[QY], s[QZ])
    omega = (s[WX], s[WY], s[WZ])
    yaw, _ = yaw_of(q)
    q_d, omega_d = desired_attitude(yaw, roll, pitch, yaw_rate)
    e_rot, e_rate = attitude_errors(q, omega, q_d, omega_d)
    moment = moment_law(e_rot, e_rate, omega, gains, robot.inertia)
    return saturate(np.asarray(thrust, dtype=np.float64), moment, robot)


def velocity_control(s, vcmd, yaw_rate, gains: Gains, robot: Robot, limits: Limits):
    """Velocity outer loop -> (roll, pitch, yaw_rate, thrust, degenerate)
    (control.py:283-349, Eqs. 6-9)."""
    q = (s[QW], s[QX], s[QY], s[QZ])
    yaw, _ = yaw_of(q)
    cy, sy = np.cos(yaw), np.sin(yaw)

    cx, cyv, cz = vcmd                                     # control.py:312-316
    vnorm = np.sqrt(cx * cx + cyv * cyv + cz * cz)
    scale = np.where(vnorm > limits.max_speed_cmd,
                     limits.max_speed_cmd / np.where(vnorm == 0.0, 1.0, vnorm), 1.0)
    cx, cyv, cz = cx * scale, cyv * scale, cz * scale

    vx = cy * s[VX] + sy * s[VY]                           # control.py:319-321
    vy = -sy * s[VX] + cy * s[VY]
    vz = s[VZ]

    ax = gains.velocity[0] * (cx - vx)                     # control.py:323-325
    ay = gains.velocity[1] * (cyv - vy)
    az = gains.velocity[2] * (cz - vz) + robot.gravity

    w, x, y, z = q                                         # control.py:328-333
    b3x = 2.0 * (x * z + w * y)
    b3y = 2.0 * (y * z - w * x)
    b3z = 1.0 - 2.0 * (x * x + y * y)
    vb3x = cy * b3x + sy * b3y
    vb3y = -sy * b3x + cy * b3y

    thrust = robot.mass * (ax * vb3x + ay * vb3y + az * b3z)   # control.py:335-339
    roll = np.clip(np.arctan2(-ay, np.sqrt(ax * ax + az * az)), -limits.max_tilt, limits.max_tilt)
    pitch = np.clip(np.arctan2(ax, az), -limits.max_tilt, limits.max_tilt)

    degenerate = np.sqrt(ax * ax + ay * ay + az * az) < DEGENERATE_ACCEL  # 341-345
    roll = np.where(degenerate, 0.0, roll)
    pitch = np.where(degenerate, 0.0, pitch)
    thrust = np.where(degenerate, robot.hover_thrust, thrust)
    yaw_rate = np.asarray(yaw_rate, dtype=np.float64) + np.zeros_like(roll)
    return roll, pitch, yaw_rate, thrust, degenerate


def control(s, mode, att_cmd, vel_cmd, gains: Gains, robot: Robot,
            limits: Limits | None = None):
    """Mixed-mode router (control.py:352-386).

    att_cmd: (4, N) rows roll, pitch, yaw_rate, thrust.
    vel_cmd: (4, N) rows vx, vy, vz, yaw_rate (vehicle frame).
    Returns (thrust, moment(3), gimbal, degenerate).
    """
    limits = limits or Limits()
    q = (s[QW], s[QX], s[QY], s[QZ])
    _, gimbal = yaw_of(q)
    mode = np.asarray(mode)
    is_vel = mode == MODE_VELOCITY
    degenerate = np.zeros(s.shape[1], dtype=bool)
    roll, pitch, yr, thr = att_cmd
    if is_vel.any():
        vr, vp, vy, vf, dg = velocity_control(s, vel_cmd[0:3], vel_cmd[3], gains,
                                              robot, limits)
        roll = np.where(is_vel, vr, roll)
        pitch = np.where(is_vel, vp, pitch)
        yr = np.where(is_vel, vy, yr)
        thr = np.where(is_vel, vf, thr)
        degenerate = dg & is_vel
    thrust, moment = attitude_control(s, roll, pitch, yr, thr, gains, robot)
    return thrust, moment, gimbal, degenerate


# =============================================================================
# integrator (dynamics.py)
# =============================================================================

def clamp_norm(x, y, z, limit):
    """Rescale vectors whose norm exceeds limit (dynamics.py:229-235)."""
    n = np.sqrt(x * x + y * y + z * z)
    over = n > limit
    sc = np.where(over, limit / np.where(n == 0.0, 1.0, n), 1.0)
    return x * sc, y * sc, z * sc, over


def integrate(s, thrust, moment, robot: Robot, dt: float,
              mass=None, inertia_diag=None):
    """Semi-implicit Euler with the momentum-rotation gyroscopic update
    (dynamics.py:286-341).  Returns (new_state (13,N), clamped, nonfinite).

    ``mass`` (N,) and ``inertia_diag`` (3, N) override the shared parameters
    with per-vehicle values (heterogeneous-fleet EXTENSION); when omitted the
    reference arithmetic is used unchanged.
    """
    if not 0.0 < dt <= 0.1:
        raise ValueError(f"dt must be in (0, 0.1], got {dt}")
    if inertia_diag is None:
        j, ji = robot.inertia, robot.inertia_inv
    else:
        zero = np.zeros_like(inertia_diag[0])
        d, di = inertia_diag, 1.0 / inertia_diag
        j = np.array([[d[0], zero, zero], [zero, d[1], zero], [zero, zero, d[2]]])
        ji = np.array([[di[0], zero, zero], [zero, di[1], zero], [zero, zero, di[2]]])
    w, x, y, z = s[QW], s[QX], s[QY], s[QZ]
    b3x = 2.0 * (x * z + w * y)                            # dynamics.py:295-297
    b3y = 2.0 * (y * z - w * x)
    b3z = 1.0 - 2.0 * (x * x + y * y)

    a = thrust / (robot.mass if mass is None else mass)    # dynamics.py:299
    vx = s[VX] + dt * (a * b3x)                            # dynamics.py:300-307
    vy = s[VY] + dt * (a * b3y)
    vz = s[VZ] + dt * (a * b3z - robot.gravity)
    vx, vy, vz, v_over = clamp_norm(vx, vy, vz, robot.v_limit)   # :308
    px = s[PX] + dt * vx                                   # :309
    py = s[PY] + dt * vy
    pz = s[PZ] + dt * vz

    ox, oy, oz = s[WX], s[WY], s[WZ]                       # dynamics.py:311-315
    lx = j[0, 0] * ox + j[0, 1] * oy + j[0, 2] * oz
    ly = j[1, 0] * ox + j[1, 1] * oy + j[1, 2] * oz
    lz = j[2, 0] * ox + j[2, 1] * oy + j[2, 2] * oz
    lr = quat_rotate(exp_so3(-dt * ox, -dt * oy, -dt * oz), (lx, ly, lz))   # :317-318
    tx = lr[0] + dt * moment[0]                            # :319-321
    ty = lr[1] + dt * moment[1]
    tz = lr[2] + dt * moment[2]
    nx = ji[0, 0] * tx + ji[0, 1] * ty + ji[0, 2] * tz     # :322-329
    ny = ji[1, 0] * tx + ji[1, 1] * ty + ji[1, 2] * tz
    nz = ji[2, 0] * tx + ji[2, 1] * ty + ji[2, 2] * tz
    nx, ny, nz, w_over = clamp_norm(nx, ny, nz, robot.omega_limit)   # :330

    qn = quat_mul((w, x, y, z), exp_so3(dt * nx, dt * ny, dt * nz))  # :332
    out = np.stack([px, py, pz, *qn, vx, vy, vz, nx, ny, nz])
    nonfinite = ~np.isfinite(out).all(axis=0)              # :334-339
    return out, v_over | w_over, nonfinite


def step(s, mode, att_cmd, vel_cmd, gains: Gains, robot: Robot, dt: float,
         limits: Limits | None = None):
    """control() then integrate(): the reference pipeline step (bench.py:146-149)."""
    thrust, moment, gimbal, degen = control(s, mode, att_cmd, vel_cmd, gains, robot, limits)
    out, clamped, nonfinite = integrate(s, thrust, moment, robot, dt)
    return out, dict(thrust=thrust, moment=moment, gimbal=gimbal, degenerate=degen,
                     clamped=clamped, nonfinite=nonfinite)


# =============================================================================
# EXTENSIONS (not in the reference; builder-defined, parity unpinned)
# =============================================================================

# Lower bound on the commanded vertical acceleration of the position loop
# (m/s^2).  Keeps b3d in the upper hemisphere so the tilt limit is defined.
POS_MIN_UP_ACCEL = 0.5


def position_control(s, pd, yaw_d, gains: Gains, robot: Robot, limits: Limits,
                     mass=None, inertia_diag=None):
    """Lee geometric position controller, z-up, thrust along +b3
    (EXTENSION).

        a   = -k_p (p - p_d) - k_v v + g e3
        a_z = max(a_z, POS_MIN_UP_ACCEL);  |a_xy| <= a_z tan(max_tilt)
        f   = m a . b3
        b3d = a/|a|, b1c = (cos yaw_d, sin yaw_d, 0)
        b2d = (b3d x b1c)/|.|, b1d = b2d x b3d, R_d = [b1d b2d b3d], omega_d = 0
        M   = -k_R e_R - k_W omega + omega x J omega, then saturation.
    Returns (thrust, moment(3), degenerate).
    """
    m = robot.mass if mass is None else mass
    kp, kv = gains.position, gains.velocity
    ax = -kp[0] * (s[PX] - pd[0]) - kv[0] * s[VX]
    ay = -kp[1] * (s[PY] - pd[1]) - kv[1] * s[VY]
    az = -kp[2] * (s[PZ] - pd[2]) - kv[2] * s[VZ] + robot.gravity
    az = np.maximum(az, POS_MIN_UP_ACCEL)
    h = np.sqrt(ax * ax + ay * ay)
    hmax = az * np.tan(limits.max_tilt)
    sc = np.where(h > hmax, hmax / np.where(h == 0.0, 1.0, h), 1.0)
    ax, ay = ax * sc, ay * sc

    q = (s[QW], s[QX], s[QY], s[QZ])
    r = rotmat(q)
    thrust = m * (ax * r[0][2] + ay * r[1][2] + az * r[2][2])
    an = np.sqrt(ax * ax + ay * ay + az * az)
    degenerate = an < DEGENERATE_ACCEL
    b3 = (ax / an, ay / an, az / an)
    c, sn = np.cos(yaw_d), np.sin(yaw_d)
    # b3d x b1c with b1c = (c, sn, 0)
    cx = -b3[2] * sn
    cy = b3[2] * c
    cz = b3[0] * sn - b3[1] * c
    cn = np.sqrt(cx * cx + cy * cy + cz * cz)
    b2 = (cx / cn, cy / cn, cz / cn)
    b1 = (b2[1] * b3[2] - b2[2] * b3[1],
          b2[2] * b3[0] - b2[0] * b3[2],
          b2[0] * b3[1] - b2[1] * b3[0])
    rd = ((b1[0], b2[0], b3[0]), (b1[1], b2[1], b3[1]), (b1[2], b2[2], b3[2]))
    omega = (s[WX], s[WY], s[WZ])
    zero = np.zeros_like(s[WX])
    e_rot, e_rate = attitude_errors_mat(r, omega, rd, (zero, zero, zero))
    if inertia_diag is None:
        moment = moment_law(e_rot, e_rate, omega, gains, robot.inertia)
    else:   # per-vehicle diagonal inertia (3, N)
        j = inertia_diag
        wx, wy, wz = omega
        jx, jy, jz = j[0] * wx, j[1] * wy, j[2] * wz
        gy = (wy * jz - wz * jy, wz * jx - wx * jz, wx * jy - wy * jx)
        moment = tuple(-gains.attitude[i] * e_rot[i] - gains.rate[i] * e_rate[i] + gy[i]
                       for i in range(3))
    thrust = np.where(degenerate, m * robot.gravity, thrust)
    f, mo = saturate(thrust, moment, robot)
    return f, mo, degenerate


@dataclass
class Airframe:
    """Rotor geometry for allocation (EXTENSION).

    Rotor i sits at arm_length * (cos a_i, sin a_i, 0) in the body frame with
    spin s_i = +-1; its thrust T_i >= 0 acts along +b3 and its drag torque is
    s_i * kappa * T_i about +b3.  Wrench = A T with column i
    (1, y_i, -x_i, s_i kappa).
    """

    angles_deg: tuple
    spins: tuple
    arm_length: float = 0.2
    kappa: float = 0.05
    rotor_max: float = 10.0

    def matrix(self) -> np.ndarray:
        a = np.deg2rad(np.asarray(self.angles_deg, dtype=np.float64))
        x, y = self.arm_length * np.cos(a), self.arm_length * np.sin(a)
        s = np.asarray(self.spins, dtype=np.float64)
        return np.stack([np.ones_like(x), y, -x, s * self.kappa])

    def pinv(self) -> np.ndarray:
        a = self.matrix()
        return a.T @ np.linalg.inv(a @ a.T)


QUAD_X = Airframe(angles_deg=(45.0, 135.0, 225.0, 315.0), spins=(1, -1, 1, -1),
                  arm_length=0.2, kappa=0.05, rotor_max=10.0)
HEX = Airframe(angles_deg=(0.0, 60.0, 120.0, 180.0, 240.0, 300.0),
               spins=(1, -1, 1, -1, 1, -1), arm_length=0.2, kappa=0.05, rotor_max=7.0)


def allocate(thrust, moment, frame: Airframe):
    """T = clip(A+ [f, M], 0, T_max) per rotor (EXTENSION, Appendix A.6).
    Returns (rotors (n_rotor, N), realized thrust, realized moment(3))."""
    pinv = frame.pinv()
    w = np.stack([thrust, moment[0], moment[1], moment[2]])
    t = np.clip(pinv @ w, 0.0, frame.rotor_max)
    real = frame.matrix() @ t
    return t, real[0], (real[1], real[2], real[3])
