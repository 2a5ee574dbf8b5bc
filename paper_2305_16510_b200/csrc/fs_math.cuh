// fs_math.cuh -- per-vehicle math of the fused control step (device side).
//
// One vehicle = one register-resident record; no shared memory, no
// cross-vehicle coupling (dynamics.py:18-19).  The arithmetic
// restates, in fp32 and with the transcendental budget trimmed, the
// reference's
//   se3.yaw_of            se3.py:226-243
//   desired_attitude      control.py:190-218
//   attitude_errors       control.py:221-258
//   attitude_control      control.py:261-280
//   velocity_control      control.py:283-349
//   control_batch         control.py:352-386
//   saturate_batch        dynamics.py:214-218
//   _step_kernel          dynamics.py:286-341
// Identities used (exact in real arithmetic, differ from the reference only
// by fp32 rounding):
//   * (cos psi, sin psi) = (r00, r10)/hypot(r00, r10)  instead of atan2 + sincos
//   * R_d = R_z(psi) R_y(theta) R_x(phi) built from the three (cos, sin) pairs
//     instead of half-angle quaternion products
//   * R^T R_d omega_d = yaw_rate * R^T e3 = yaw_rate * (r20, r21, r22), since
//     omega_d = yaw_rate * R_d^T e3 (Eq. 2)
//   * velocity mode: (cos, sin) of the commanded tilt as ratios of the
//     acceleration demand; the +-max_tilt clip becomes cos < cos(max_tilt)
//   * exp_so3 via a polynomial in (theta/2)^2 (no sqrt, no MUFU) for
//     theta/2 <= pi/4, sincosf beyond; the final quaternion is renormalized.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "flocksim_b200.h"

namespace fs {

// ---------------------------------------------------------------------------
// launch-constant parameters (passed by value, __grid_constant__)
// ---------------------------------------------------------------------------
struct KParams {
    fs_step_desc d;
    fs_robot r;
    fs_gains g;
    fs_limits l;
    fs_airframe frame[2];
    int32_t n_frames;      // 0, 1 or 2
    int32_t jdiag;         // shared inertia is diagonal
    int32_t want_flags;    // flags_out or stats requested
    int32_t steps;         // rollout length (fs_rollout)
    float cos_tilt, sin_tilt, tan_tilt;
    float max_speed2;
    float v_lim2, w_lim2;
    float inv_mass;
    uint32_t reset_thresh;
};

struct VState {
    float p[3];
    float q[4];
    float v[3];
    float w[3];
};

struct StepOut {
    float f, m[3];
    float rotor[FS_MAX_ROTORS];
    uint32_t flags;
};

constexpr float kPi = 3.14159265358979323846f;
constexpr float kQuarterPiSq = 0.61685027506808491f;   // (pi/4)^2
constexpr float kHalfPi = 1.57079632679489662f;

// ---------------------------------------------------------------------------
// small-angle trigonometry
// ---------------------------------------------------------------------------

// sin(x)/x and cos(x) from x2 = x^2, |x| <= pi/4 (Taylor to x^8 / x^10; the
// truncation error is < 3e-9 relative, below fp32 rounding).
__device__ __forceinline__ void sinc_cos_sq(float x2, float& sinc, float& c) {
    sinc = fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, 2.75573192e-6f, -1.98412698e-4f),
                                   8.33333333e-3f), -1.66666667e-1f), 1.0f);
    c = fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, -2.75573192e-7f, 2.48015873e-5f),
                                        -1.38888889e-3f), 4.16666667e-2f), -0.5f), 1.0f);
}

// sin and cos of |x| <= pi/2 (commanded tilt angles; control.py:94 rejects
// |angle| >= pi/2).  Taylor to x^13 / x^14: truncation < 7e-10.
__device__ __forceinline__ void sincos_tilt(float x, float& s, float& c) {
    if (fabsf(x) <= kHalfPi) {
        const float x2 = x * x;
        const float ps = fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2,
                         -1.60590438e-10f, 2.50521084e-8f), -2.75573192e-6f), 1.98412698e-4f),
                         -8.33333333e-3f), 1.66666667e-1f), -1.0f);
        s = -x * ps;   // x * (1 - x^2/6 + ...)
        c = fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2,
                 -1.14707456e-11f, 2.08767570e-9f), -2.75573192e-7f), 2.48015873e-5f),
                 -1.38888889e-3f), 4.16666667e-2f), -0.5f), 1.0f);
    } else {
        sincosf(x, &s, &c);
    }
}

// Full-range sin/cos (yaw setpoints): Cody-Waite reduction by pi/2 then the
// quarter-range polynomial; sincosf for |x| > 1e5.
__device__ __forceinline__ void sincos_full(float x, float& s, float& c) {
    if (fabsf(x) > 1.0e5f) { sincosf(x, &s, &c); return; }
    const float k = rintf(x * 6.366197467e-01f);
    // pi/2 = C1 + C2 + C3 (float32 head and tails)
    float r = fmaf(k, -1.570796371e+00f, x);
    r = fmaf(k, 4.371138829e-08f, r);
    r = fmaf(k, 1.776356839e-15f, r);
    float sinc, cr;
    sinc_cos_sq(r * r, sinc, cr);
    const float sr = r * sinc;
    const int q = static_cast<int>(k) & 3;
    const float ss = (q & 1) ? cr : sr;
    const float cc = (q & 1) ? sr : cr;
    s = (q & 2) ? -ss : ss;
    c = ((q + 1) & 2) ? -cc : cc;
}

// exp_so3(w) as an (unnormalized to fp32 rounding) quaternion: se3.py:246-266.
// theta = |w|; (cos(theta/2), sin(theta/2)/theta * w).  w = 0 gives exactly
// (1, 0, 0, 0) like the reference's series branch.
__device__ __forceinline__ void exp_quat(float wx, float wy, float wz, float& ew, float& ex,
                                         float& ey, float& ez) {
    const float t2 = fmaf(wx, wx, fmaf(wy, wy, wz * wz));
    const float x2 = 0.25f * t2;
    float k, c;
    if (x2 <= kQuarterPiSq) {
        float sinc;
        sinc_cos_sq(x2, sinc, c);
        k = 0.5f * sinc;
    } else {
        const float t = sqrtf(t2);
        float s;
        sincosf(0.5f * t, &s, &c);
        k = s / t;
    }
    ew = c;
    ex = k * wx;
    ey = k * wy;
    ez = k * wz;
}

// R(q) u with t = 2 q_v x u; u + w t + q_v x t (se3.py:106-130).
__device__ __forceinline__ void quat_rotate(float w, float x, float y, float z, float& ux,
                                            float& uy, float& uz) {
    const float tx = 2.0f * (y * uz - z * uy);
    const float ty = 2.0f * (z * ux - x * uz);
    const float tz = 2.0f * (x * uy - y * ux);
    const float ox = ux + w * tx + (y * tz - z * ty);
    const float oy = uy + w * ty + (z * tx - x * tz);
    const float oz = uz + w * tz + (x * ty - y * tx);
    ux = ox;
    uy = oy;
    uz = oz;
}

__device__ __forceinline__ float clampf(float x, float lo, float hi) {
    return fminf(fmaxf(x, lo), hi);
}

// Rescale (x, y, z) to norm `lim` when its squared norm exceeds lim^2
// (dynamics.py:229-235).  Returns the "over" flag.
__device__ __forceinline__ bool clamp_norm(float& x, float& y, float& z, float lim,
                                           float lim2) {
    const float n2 = fmaf(x, x, fmaf(y, y, z * z));
    if (n2 > lim2) {
        const float sc = lim * rsqrtf(n2);
        x *= sc;
        y *= sc;
        z *= sc;
        return true;
    }
    return false;
}

// fp64 gimbal test, bit-identical to the reference on fp32 inputs: the
// products of two fp32 values are exact in fp64 (se3.py:240-242).
__device__ __forceinline__ bool gimbal_flag(float qw, float qx, float qy, float qz,
                                            double gimbal_cos) {
    const double r20 = 2.0 * ((double)qx * (double)qz - (double)qw * (double)qy);
    return fabs(r20) >= gimbal_cos;
}

// ---------------------------------------------------------------------------
// the fused per-vehicle step
// ---------------------------------------------------------------------------
//
// MODE:  FS_MODE_ATTITUDE / VELOCITY / MIXED / POSITION
// HETERO: per-vehicle mass and diagonal inertia (vp[0..3]) and two airframes
// cmd:   the vehicle's command values (4, or 8 for MIXED)
// vmode: the vehicle's mode byte (MIXED only)
// Returns the control output in `o`; if `integrate`, advances `s` in place.
template <int MODE, bool HETERO>
__device__ __forceinline__ void vehicle_step(VState& s, const float* cmd, uint32_t vmode,
                                             const float* vp, int frame_id,
                                             const KParams& P, bool integrate, StepOut& o) {
    const float qw = s.q[0], qx = s.q[1], qy = s.q[2], qz = s.q[3];
    const float wx = s.w[0], wy = s.w[1], wz = s.w[2];
    const float g = P.r.gravity;
    const float mass = HETERO ? vp[0] : P.r.mass;
    uint32_t flags = 0;

    // --- R(q), se3.py:148-152 ---------------------------------------------
    const float xx = qx * qx, yy = qy * qy, zz = qz * qz;
    const float xy = qx * qy, xz = qx * qz, yz = qy * qz;
    const float qwx = qw * qx, qwy = qw * qy, qwz = qw * qz;
    const float R00 = 1.0f - 2.0f * (yy + zz), R01 = 2.0f * (xy - qwz), R02 = 2.0f * (xz + qwy);
    const float R10 = 2.0f * (xy + qwz), R11 = 1.0f - 2.0f * (xx + zz), R12 = 2.0f * (yz - qwx);
    const float R20 = 2.0f * (xz - qwy), R21 = 2.0f * (yz + qwx), R22 = 1.0f - 2.0f * (xx + yy);

    float eR0, eR1, eR2, eW0, eW1, eW2, thrust;

    if constexpr (MODE == FS_MODE_POSITION) {
        // --- Lee position controller (EXTENSION) -------------
        const float kp0 = P.g.position[0], kp1 = P.g.position[1], kp2 = P.g.position[2];
        const float kv0 = P.g.velocity[0], kv1 = P.g.velocity[1], kv2 = P.g.velocity[2];
        float ax = -kp0 * (s.p[0] - cmd[0]) - kv0 * s.v[0];
        float ay = -kp1 * (s.p[1] - cmd[1]) - kv1 * s.v[1];
        float az = -kp2 * (s.p[2] - cmd[2]) - kv2 * s.v[2] + g;
        az = fmaxf(az, 0.5f);                                  // POS_MIN_UP_ACCEL
        const float h2 = fmaf(ax, ax, ay * ay);
        const float hmax = az * P.tan_tilt;
        if (h2 > hmax * hmax) {
            const float sc = hmax * rsqrtf(h2);
            ax *= sc;
            ay *= sc;
        }
        thrust = mass * (ax * R02 + ay * R12 + az * R22);
        const float an2 = fmaf(ax, ax, fmaf(ay, ay, az * az));
        const float ia = rsqrtf(an2);
        const float b3x = ax * ia, b3y = ay * ia, b3z = az * ia;
        float sy, cy;
        sincos_full(cmd[3], sy, cy);
        // b2d = normalize(b3d x b1c), b1c = (cy, sy, 0)
        float cx_ = -b3z * sy, cy_ = b3z * cy, cz_ = b3x * sy - b3y * cy;
        const float icn = rsqrtf(fmaf(cx_, cx_, fmaf(cy_, cy_, cz_ * cz_)));
        const float b2x = cx_ * icn, b2y = cy_ * icn, b2z = cz_ * icn;
        const float b1x = b2y * b3z - b2z * b3y;
        const float b1y = b2z * b3x - b2x * b3z;
        const float b1z = b2x * b3y - b2y * b3x;
        // A = R_d^T R, A_ij = (column i of R_d) . (column j of R)
        const float A21 = b3x * R01 + b3y * R11 + b3z * R21;
        const float A12 = b2x * R02 + b2y * R12 + b2z * R22;
        const float A02 = b1x * R02 + b1y * R12 + b1z * R22;
        const float A20 = b3x * R00 + b3y * R10 + b3z * R20;
        const float A10 = b2x * R00 + b2y * R10 + b2z * R20;
        const float A01 = b1x * R01 + b1y * R11 + b1z * R21;
        eR0 = 0.5f * (A21 - A12);
        eR1 = 0.5f * (A02 - A20);
        eR2 = 0.5f * (A10 - A01);
        eW0 = wx;
        eW1 = wy;
        eW2 = wz;
        if (P.want_flags && !(an2 >= 1e-12f) && an2 == an2) flags |= FS_FLAG_DEGENERATE;
    } else {
        // --- yaw of the current attitude as (cos, sin): se3.py:237-241 --------
        const float rho2 = fmaf(R00, R00, R10 * R10);
        float cy = 1.0f, sy = 0.0f;
        if (rho2 > 0.0f) {
            const float ir = rsqrtf(rho2);
            cy = R00 * ir;
            sy = R10 * ir;
        }
        float cr, sr, ct, st, yr;
        bool vel = (MODE == FS_MODE_VELOCITY);
        if constexpr (MODE == FS_MODE_MIXED) vel = (vmode == FS_MODE_VELOCITY);
        if (vel) {
            // --- velocity outer loop: control.py:306-349 ----------------------
            const float* vc = (MODE == FS_MODE_MIXED) ? cmd + 4 : cmd;
            float vcx = vc[0], vcy = vc[1], vcz = vc[2];
            const float vn2 = fmaf(vcx, vcx, fmaf(vcy, vcy, vcz * vcz));
            if (vn2 > P.max_speed2) {
                const float sc = P.l.max_speed_cmd * rsqrtf(vn2);
                vcx *= sc;
                vcy *= sc;
                vcz *= sc;
            }
            const float vvx = cy * s.v[0] + sy * s.v[1];
            const float vvy = -sy * s.v[0] + cy * s.v[1];
            const float ax = P.g.velocity[0] * (vcx - vvx);
            const float ay = P.g.velocity[1] * (vcy - vvy);
            const float az = P.g.velocity[2] * (vcz - s.v[2]) + g;
            const float vb3x = cy * R02 + sy * R12;
            const float vb3y = -sy * R02 + cy * R12;
            thrust = mass * (ax * vb3x + ay * vb3y + az * R22);
            const float hxz2 = fmaf(ax, ax, az * az);
            const float a2 = fmaf(ay, ay, hxz2);
            // pitch = atan2(ax, az) -> (cos, sin) = (az, ax)/|(ax, az)|
            const float ih = rsqrtf(hxz2);
            ct = az * ih;
            st = ax * ih;
            float hxz = hxz2 * ih;
            if (hxz2 == 0.0f) { ct = 1.0f; st = 0.0f; hxz = 0.0f; }
            if (ct < P.cos_tilt) { ct = P.cos_tilt; st = copysignf(P.sin_tilt, ax); }
            // roll = atan2(-ay, |(ax, az)|) -> (cos, sin) = (|(ax,az)|, -ay)/|a|
            const float ia = rsqrtf(a2);
            cr = hxz * ia;
            sr = -ay * ia;
            if (cr < P.cos_tilt) { cr = P.cos_tilt; sr = copysignf(P.sin_tilt, -ay); }
            if (a2 < 1e-12f) {                                   // DEGENERATE_ACCEL^2
                cr = 1.0f; sr = 0.0f; ct = 1.0f; st = 0.0f;
                thrust = mass * g;
                flags |= FS_FLAG_DEGENERATE;
            }
            yr = vc[3];
        } else {
            sincos_tilt(cmd[0], sr, cr);
            sincos_tilt(cmd[1], st, ct);
            yr = cmd[2];
            thrust = cmd[3];
        }
        // --- attitude errors, Eqs. 3-4 (control.py:221-258) --------------------
        // P = R_z(psi)^T R (rows 0, 1; row 2 = R row 2)
        const float P00 = cy * R00 + sy * R10, P01 = cy * R01 + sy * R11, P02 = cy * R02 + sy * R12;
        const float P10 = cy * R10 - sy * R00, P11 = cy * R11 - sy * R01, P12 = cy * R12 - sy * R02;
        // M = R_y(theta) R_x(phi); A = M^T P
        const float stsr = st * sr, stcr = st * cr, ctsr = ct * sr, ctcr = ct * cr;
        const float A21 = stcr * P01 - sr * P11 + ctcr * R21;
        const float A12 = stsr * P02 + cr * P12 + ctsr * R22;
        const float A02 = ct * P02 - st * R22;
        const float A20 = stcr * P00 - sr * P10 + ctcr * R20;
        const float A10 = stsr * P00 + cr * P10 + ctsr * R20;
        const float A01 = ct * P01 - st * R21;
        eR0 = 0.5f * (A21 - A12);
        eR1 = 0.5f * (A02 - A20);
        eR2 = 0.5f * (A10 - A01);
        eW0 = wx - yr * R20;
        eW1 = wy - yr * R21;
        eW2 = wz - yr * R22;
    }

    // --- moment law, Eq. 5 (control.py:271-279) --------------------------------
    float jwx, jwy, jwz;
    if (HETERO) {
        jwx = vp[1] * wx;
        jwy = vp[2] * wy;
        jwz = vp[3] * wz;
    } else if (P.jdiag) {
        jwx = P.r.inertia[0] * wx;
        jwy = P.r.inertia[4] * wy;
        jwz = P.r.inertia[8] * wz;
    } else {
        const float* J = P.r.inertia;
        jwx = J[0] * wx + J[1] * wy + J[2] * wz;
        jwy = J[3] * wx + J[4] * wy + J[5] * wz;
        jwz = J[6] * wx + J[7] * wy + J[8] * wz;
    }
    float m0 = -P.g.attitude[0] * eR0 - P.g.rate[0] * eW0 + (wy * jwz - wz * jwy);
    float m1 = -P.g.attitude[1] * eR1 - P.g.rate[1] * eW1 + (wz * jwx - wx * jwz);
    float m2 = -P.g.attitude[2] * eR2 - P.g.rate[2] * eW2 + (wx * jwy - wy * jwx);

    // --- saturation: dynamics.py:214-218 ----------------------------------------
    float f = clampf(thrust, 0.0f, P.r.thrust_max);
    m0 = clampf(m0, -P.r.moment_max[0], P.r.moment_max[0]);
    m1 = clampf(m1, -P.r.moment_max[1], P.r.moment_max[1]);
    m2 = clampf(m2, -P.r.moment_max[2], P.r.moment_max[2]);
    o.f = f;
    o.m[0] = m0;
    o.m[1] = m1;
    o.m[2] = m2;

    // --- allocation T = clip(A^+ w) (EXTENSION) ------------------
    if (P.n_frames > 0) {
        const fs_airframe& fr = P.frame[frame_id];
        float rf = 0.0f, rm0 = 0.0f, rm1 = 0.0f, rm2 = 0.0f;
#pragma unroll
        for (int i = 0; i < FS_MAX_ROTORS; ++i) {
            float t = 0.0f;
            if (i < fr.n_rotors) {
                const float* row = fr.pinv + 4 * i;
                t = clampf(row[0] * f + row[1] * m0 + row[2] * m1 + row[3] * m2, 0.0f,
                           fr.rotor_max);
                rf += fr.alloc[0 * FS_MAX_ROTORS + i] * t;
                rm0 += fr.alloc[1 * FS_MAX_ROTORS + i] * t;
                rm1 += fr.alloc[2 * FS_MAX_ROTORS + i] * t;
                rm2 += fr.alloc[3 * FS_MAX_ROTORS + i] * t;
            }
            o.rotor[i] = t;
        }
        if (P.d.rotor_dynamics) {
            f = rf;
            m0 = rm0;
            m1 = rm1;
            m2 = rm2;
        }
    }

    if (P.want_flags && gimbal_flag(qw, qx, qy, qz, P.r.gimbal_cos) && MODE != FS_MODE_POSITION)
        flags |= FS_FLAG_GIMBAL;

    if (integrate) {
        // --- semi-implicit Euler: dynamics.py:286-341 ----------------------------
        const float dt = P.d.dt;
        const float a = HETERO ? f / mass : f * P.inv_mass;      // dynamics.py:299
        float vx = s.v[0] + dt * (a * R02);
        float vy = s.v[1] + dt * (a * R12);
        float vz = s.v[2] + dt * (a * R22 - g);
        bool over = clamp_norm(vx, vy, vz, P.r.v_limit, P.v_lim2);
        s.p[0] += dt * vx;
        s.p[1] += dt * vy;
        s.p[2] += dt * vz;
        s.v[0] = vx;
        s.v[1] = vy;
        s.v[2] = vz;

        // body angular momentum L = J w, rotated by exp(-dt w), plus dt M
        float lx = jwx, ly = jwy, lz = jwz;
        float ew, ex, ey, ez;
        exp_quat(-dt * wx, -dt * wy, -dt * wz, ew, ex, ey, ez);
        quat_rotate(ew, ex, ey, ez, lx, ly, lz);
        const float tx = lx + dt * m0, ty = ly + dt * m1, tz = lz + dt * m2;
        float nx, ny, nz;
        if (HETERO) {
            nx = tx / vp[1];
            ny = ty / vp[2];
            nz = tz / vp[3];
        } else if (P.jdiag) {
            nx = P.r.inertia_inv[0] * tx;
            ny = P.r.inertia_inv[4] * ty;
            nz = P.r.inertia_inv[8] * tz;
        } else {
            const float* Ji = P.r.inertia_inv;
            nx = Ji[0] * tx + Ji[1] * ty + Ji[2] * tz;
            ny = Ji[3] * tx + Ji[4] * ty + Ji[5] * tz;
            nz = Ji[6] * tx + Ji[7] * ty + Ji[8] * tz;
        }
        over |= clamp_norm(nx, ny, nz, P.r.omega_limit, P.w_lim2);
        s.w[0] = nx;
        s.w[1] = ny;
        s.w[2] = nz;

        // q+ = normalize(q (x) exp(dt w+)): se3.py:78-97
        exp_quat(dt * nx, dt * ny, dt * nz, ew, ex, ey, ez);
        float pw = qw * ew - qx * ex - qy * ey - qz * ez;
        float px = qw * ex + qx * ew + qy * ez - qz * ey;
        float py = qw * ey - qx * ez + qy * ew + qz * ex;
        float pz = qw * ez + qx * ey - qy * ex + qz * ew;
        const float iq = rsqrtf(fmaf(pw, pw, fmaf(px, px, fmaf(py, py, pz * pz))));
        s.q[0] = pw * iq;
        s.q[1] = px * iq;
        s.q[2] = py * iq;
        s.q[3] = pz * iq;
        if (over) flags |= FS_FLAG_CLAMPED;
        if (P.want_flags) {
            // any non-finite component (dynamics.py:334-339): x*0 is NaN iff x is
            float z = 0.0f;
#pragma unroll
            for (int k = 0; k < 3; ++k) z = fmaf(s.p[k], 0.0f, z);
#pragma unroll
            for (int k = 0; k < 4; ++k) z = fmaf(s.q[k], 0.0f, z);
#pragma unroll
            for (int k = 0; k < 3; ++k) z = fmaf(s.v[k], 0.0f, fmaf(s.w[k], 0.0f, z));
            if (z != z) flags |= FS_FLAG_NONFINITE;
        }
    }
    o.flags = flags;
}

}  // namespace fs
