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

#include <type_traits>

#include "flocksim_b200.h"

namespace fs {

// ---------------------------------------------------------------------------
// launch-constant parameters (passed by value, __grid_constant__)
// ---------------------------------------------------------------------------
// Parameters in one precision T: the fp32 copy feeds the fp32 paths, the
// float64 copy (the reference's own values, dynamics.py:54-63,
// control.py:48-68) feeds the float64 controller.
template <typename T>
struct TP {
    T mass, inv_mass, gravity, thrust_max, moment_max[3];
    T v_limit, omega_limit, v_lim2, w_lim2;
    T inertia[9], inertia_inv[9];
    T g_att[3], g_rate[3], g_vel[3], g_pos[3];
    T max_tilt, cos_tilt, sin_tilt, tan_tilt, max_speed, max_speed2;
};

struct KParams {
    fs_step_desc d;
    TP<float> pf;
    TP<double> pd;
    double gimbal_cos;
    fs_airframe frame[2];
    int32_t n_frames;      // 0, 1 or 2
    int32_t jdiag;         // shared inertia is diagonal
    int32_t want_flags;    // flags_out or stats requested
    int32_t steps;         // rollout length (fs_rollout)
    uint32_t reset_thresh;
    uint32_t rs_key;       // step_key(seed, step_index), host-computed (fs_rng.cuh)
    int32_t chain_release; // chained steps: gpu-scope fence before publishing (tuning)
    uint64_t sync_timeout_ns; // chained steps: trap after waiting this long (0 = never)
    int32_t chain_acquire; // chained steps: acquire counter loads + proxy fence (tuning)
    uint32_t spawn_wait_ns;   // streaming kernel: spawn warps' wait back-off start (0 = try_wait)
    uint32_t cons_wait_ns;    // streaming kernel: consumers' wait back-off start (0 = try_wait)
    int32_t l2_keep_tiles; // streaming kernel: tiles t < this keep an L2 evict_last policy
    int32_t exp2_poly;     // dt * omega_limit / 2 <= pi/4: exp(dt w+) needs no fallback
    float* out_plane[13];  // state_out + k * state_out_stride (host-computed bases)
};

template <typename T>
__device__ __forceinline__ const TP<T>& tp(const KParams& P);
template <>
__device__ __forceinline__ const TP<float>& tp<float>(const KParams& P) { return P.pf; }
template <>
__device__ __forceinline__ const TP<double>& tp<double>(const KParams& P) { return P.pd; }

struct VState {
    float p[3];
    float q[4];
    float v[3];
    float w[3];
};

// Optional-feature bits of the fused kernels (template parameter FEAT).
constexpr int kFeatStats = 1;   // episode statistics (+ the non-finite test they need)
constexpr int kFeatReset = 2;   // per-step Bernoulli re-spawns
constexpr int kFeatOut = 4;     // flags / wrench / rotor outputs, allocation, gimbal flag
constexpr int kFeatAll = 7;

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

// exp_quat without the large-angle fallback: valid when (theta/2)^2 <= (pi/4)^2,
// which the host proves for exp(dt w+) from dt * omega_limit (KParams.exp2_poly).
__device__ __forceinline__ void exp_quat_small(float wx, float wy, float wz, float& ew,
                                               float& ex, float& ey, float& ez) {
    const float x2 = 0.25f * fmaf(wx, wx, fmaf(wy, wy, wz * wz));
    float sinc;
    sinc_cos_sq(x2, sinc, ew);
    const float k = 0.5f * sinc;
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
// (dynamics.py:229-235); branch-free (the scale is exactly 1 otherwise).
// Returns the "over" flag.
__device__ __forceinline__ bool clamp_norm(float& x, float& y, float& z, float lim,
                                           float lim2) {
    const float n2 = fmaf(x, x, fmaf(y, y, z * z));
    const bool over = n2 > lim2;
    const float sc = over ? lim * rsqrtf(n2) : 1.0f;
    x *= sc;
    y *= sc;
    z *= sc;
    return over;
}

__device__ __forceinline__ float copysign_t(float a, float b) { return copysignf(a, b); }
__device__ __forceinline__ double copysign_t(double a, double b) { return copysign(a, b); }

// 1/sqrt(x) in float64: hardware seed (MUFU.RSQ64H, ~2^-22 rel.) + one
// Newton step (rel. err ~1e-13).
__device__ __forceinline__ double rsqrt_d(double x) {
    double r;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    return r * fma(-0.5 * x * r, r, 1.5);
}

// fp32 <-> fp64 conversions without the denormal-flush multiply -ftz adds
__device__ __forceinline__ double f2d(float x) {
    double r;
    asm("cvt.f64.f32 %0, %1;" : "=d"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ float d2f(double x) {
    float r;
    asm("cvt.rn.f32.f64 %0, %1;" : "=f"(r) : "d"(x));
    return r;
}
template <typename T>
__device__ __forceinline__ T up(float x);
template <>
__device__ __forceinline__ float up<float>(float x) { return x; }
template <>
__device__ __forceinline__ double up<double>(float x) { return f2d(x); }
// float64 command values (the fused action denormalization, fs_world.cu)
template <typename T>
__device__ __forceinline__ T up(double x);
template <>
__device__ __forceinline__ float up<float>(double x) { return d2f(x); }
template <>
__device__ __forceinline__ double up<double>(double x) { return x; }
__device__ __forceinline__ float down(float x) { return x; }
__device__ __forceinline__ float down(double x) { return d2f(x); }

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
// Precision (template PREC):
//   0  fp32 everywhere;
//   1  fp64 velocity front end (yaw extraction + acceleration demand);
//   2  fp64 controller: rotation matrix, yaw, tilt, attitude errors and the
//      moment law in float64 from the fp32 inputs (exact products), the
//      saturated wrench rounded once to fp32; the integrator stays fp32.
// The reference is float64 throughout; PREC 2 is what meets 1e-5 rel /
// 1e-6 abs on every vehicle outside the gimbal band (fp32 sums of O(10)
// moment terms cannot: k_R = 8 amplifies a 1-ulp attitude error to ~1e-6).

__device__ __forceinline__ float rsqrt_t(float x) { return rsqrtf(x); }
__device__ __forceinline__ double rsqrt_t(double x) { return rsqrt_d(x); }

template <typename T>
struct Rot {
    T r00, r01, r02, r10, r11, r12, r20, r21, r22;
};

// R(q), se3.py:148-152, evaluated in T from the fp32 quaternion.  The 2x is
// folded into the factors (exact), e.g. r01 = x (2y) - w (2z).
template <typename T>
__device__ __forceinline__ Rot<T> rotmat(float qw, float qx, float qy, float qz) {
    const T w = up<T>(qw), x = up<T>(qx), y = up<T>(qy), z = up<T>(qz);
    const T x2 = x + x, y2 = y + y, z2 = z + z;
    const T xx = x * x2, yy = y * y2, zz = z * z2;
    const T xy = x * y2, xz = x * z2, yz = y * z2;
    const T wx = w * x2, wy = w * y2, wz = w * z2;
    Rot<T> R;
    R.r00 = T(1) - (yy + zz); R.r01 = xy - wz; R.r02 = xz + wy;
    R.r10 = xy + wz; R.r11 = T(1) - (xx + zz); R.r12 = yz - wx;
    R.r20 = xz - wy; R.r21 = yz + wx; R.r22 = T(1) - (xx + yy);
    return R;
}

// Desired tilt and current yaw as (cos, sin) pairs, yaw rate, thrust.
template <typename T>
struct Tilt {
    T cy, sy, cr, sr, ct, st, yr, thrust;
};

// (cos psi, sin psi) = (r00, r10)/hypot: se3.py:237-241 (atan2(0,0) = 0)
template <typename T>
__device__ __forceinline__ void yaw_cs(const Rot<T>& R, T& cy, T& sy) {
    const T rho2 = R.r00 * R.r00 + R.r10 * R.r10;
    const T ir = rsqrt_t(rho2);
    const bool ok = rho2 > T(0);
    cy = ok ? R.r00 * ir : T(1);
    sy = ok ? R.r10 * ir : T(0);
}

// sin/cos of |x| <= pi/2 in float64 (Taylor to x^15 / x^16: < 7e-10 rel.)
__device__ __forceinline__ void sincos_tilt_d(double x, double& s, double& c) {
    if (fabs(x) <= 1.5707963267948966) {
        const double x2 = x * x;
        s = x * fma(x2, fma(x2, fma(x2, fma(x2, fma(x2, fma(x2, fma(x2,
                 -7.6471637318198164e-13, 1.6059043836821613e-10), -2.5052108385441720e-8),
                 2.7557319223985888e-6), -1.9841269841269841e-4), 8.3333333333333333e-3),
                 -1.6666666666666667e-1), 1.0);
        c = fma(x2, fma(x2, fma(x2, fma(x2, fma(x2, fma(x2, fma(x2, fma(x2,
                 4.7794773323873853e-14, -1.1470745597729725e-11), 2.0876756987868099e-9),
                 -2.7557319223985891e-7), 2.4801587301587302e-5), -1.3888888888888889e-3),
                 4.1666666666666667e-2), -0.5), 1.0);
    } else {
        sincos(x, &s, &c);
    }
}

__device__ __forceinline__ void sincos_tilt_t(float x, float& s, float& c) { sincos_tilt(x, s, c); }
__device__ __forceinline__ void sincos_tilt_t(float x, double& s, double& c) {
    sincos_tilt_d((double)x, s, c);
}
__device__ __forceinline__ void sincos_tilt_t(double x, double& s, double& c) {
    sincos_tilt_d(x, s, c);
}
__device__ __forceinline__ void sincos_tilt_t(double x, float& s, float& c) {
    sincos_tilt(d2f(x), s, c);
}

// Velocity outer loop, control.py:306-349, with (cos, sin) pairs in place of
// atan2 / clip / sin / cos.
template <typename T, typename CT>
__device__ __forceinline__ void velocity_tilt(const Rot<T>& R, const float* v, const CT* vc,
                                              T mass, const KParams& P, Tilt<T>& c,
                                              uint32_t& flags) {
    const TP<T>& Q = tp<T>(P);
    yaw_cs(R, c.cy, c.sy);
    const T cy = c.cy, sy = c.sy;
    T vcx = up<T>(vc[0]), vcy = up<T>(vc[1]), vcz = up<T>(vc[2]);
    const T vn2 = vcx * vcx + vcy * vcy + vcz * vcz;
    if (vn2 > Q.max_speed2) {
        const T sc = Q.max_speed * rsqrt_t(vn2);
        vcx *= sc;
        vcy *= sc;
        vcz *= sc;
    }
    const T vx = up<T>(v[0]), vy = up<T>(v[1]), vz = up<T>(v[2]);
    const T vvx = cy * vx + sy * vy;
    const T vvy = -sy * vx + cy * vy;
    const T ax = Q.g_vel[0] * (vcx - vvx);
    const T ay = Q.g_vel[1] * (vcy - vvy);
    const T az = Q.g_vel[2] * (vcz - vz) + Q.gravity;
    const T vb3x = cy * R.r02 + sy * R.r12;
    const T vb3y = -sy * R.r02 + cy * R.r12;
    T thrust = mass * (ax * vb3x + ay * vb3y + az * R.r22);
    const T hxz2 = ax * ax + az * az;
    const T a2 = ay * ay + hxz2;
    const bool hz = hxz2 > T(0);                   // atan2(0, 0) = 0 -> (cos, sin) = (1, 0)
    const T ih = rsqrt_t(hxz2);
    const T cmax = Q.cos_tilt, smax = Q.sin_tilt;
    T ct = hz ? az * ih : T(1);
    T st = hz ? ax * ih : T(0);
    const T hxz = hz ? hxz2 * ih : T(0);
    const bool clip_p = ct < cmax;
    st = clip_p ? copysign_t(smax, ax) : st;
    ct = clip_p ? cmax : ct;
    const T ia = rsqrt_t(a2);
    T cr = hxz * ia, sr = -ay * ia;
    const bool clip_r = cr < cmax;
    sr = clip_r ? copysign_t(smax, -ay) : sr;
    cr = clip_r ? cmax : cr;
    const bool degen = a2 < T(1e-12);                   // DEGENERATE_ACCEL^2
    cr = degen ? T(1) : cr;
    sr = degen ? T(0) : sr;
    ct = degen ? T(1) : ct;
    st = degen ? T(0) : st;
    thrust = degen ? mass * Q.gravity : thrust;
    flags |= degen ? FS_FLAG_DEGENERATE : 0u;
    c.cr = cr; c.sr = sr; c.ct = ct; c.st = st;
    c.yr = up<T>(vc[3]);
    c.thrust = thrust;
}

template <typename T, typename CT>
__device__ __forceinline__ void attitude_tilt(const Rot<T>& R, const CT* cmd, Tilt<T>& c) {
    yaw_cs(R, c.cy, c.sy);
    sincos_tilt_t(cmd[0], c.sr, c.cr);
    sincos_tilt_t(cmd[1], c.st, c.ct);
    c.yr = up<T>(cmd[2]);
    c.thrust = up<T>(cmd[3]);
}

// Attitude errors, Eqs. 3-4 (control.py:221-258):
// P = R_z(psi)^T R (rows 0, 1; row 2 = R row 2); M = R_y(theta) R_x(phi);
// A = M^T P; e_R = vee(A - A^T)/2; R^T R_d omega_d = yaw_rate R^T e3.
template <typename T>
__device__ __forceinline__ void attitude_errors(const Rot<T>& R, const Tilt<T>& c, T wx, T wy,
                                                T wz, T (&eR)[3], T (&eW)[3]) {
    const T cy = c.cy, sy = c.sy, cr = c.cr, sr = c.sr, ct = c.ct, st = c.st;
    const T P00 = cy * R.r00 + sy * R.r10, P01 = cy * R.r01 + sy * R.r11, P02 = cy * R.r02 + sy * R.r12;
    const T P10 = cy * R.r10 - sy * R.r00, P11 = cy * R.r11 - sy * R.r01, P12 = cy * R.r12 - sy * R.r02;
    const T stsr = st * sr, stcr = st * cr, ctsr = ct * sr, ctcr = ct * cr;
    const T A21 = stcr * P01 - sr * P11 + ctcr * R.r21;
    const T A12 = stsr * P02 + cr * P12 + ctsr * R.r22;
    const T A02 = ct * P02 - st * R.r22;
    const T A20 = stcr * P00 - sr * P10 + ctcr * R.r20;
    const T A10 = stsr * P00 + cr * P10 + ctsr * R.r20;
    const T A01 = ct * P01 - st * R.r21;
    eR[0] = T(0.5) * (A21 - A12);
    eR[1] = T(0.5) * (A02 - A20);
    eR[2] = T(0.5) * (A10 - A01);
    eW[0] = wx - c.yr * R.r20;
    eW[1] = wy - c.yr * R.r21;
    eW[2] = wz - c.yr * R.r22;
}

// M = -k_R e_R - k_W e_W + w x J w (control.py:271-279, Eq. 5), saturated
// (dynamics.py:214-218).  jw = J w.
template <typename T>
__device__ __forceinline__ void moment_law(const T (&eR)[3], const T (&eW)[3], T wx, T wy, T wz,
                                           T jwx, T jwy, T jwz, const KParams& P, float (&m)[3]) {
    const TP<T>& Q = tp<T>(P);
    const T g0 = wy * jwz - wz * jwy, g1 = wz * jwx - wx * jwz, g2 = wx * jwy - wy * jwx;
    const T m0 = -Q.g_att[0] * eR[0] - Q.g_rate[0] * eW[0] + g0;
    const T m1 = -Q.g_att[1] * eR[1] - Q.g_rate[1] * eW[1] + g1;
    const T m2 = -Q.g_att[2] * eR[2] - Q.g_rate[2] * eW[2] + g2;
    // round once, then clamp with the rounded bounds: identical to rounding
    // the T-precision clamp, because rounding is monotonic
    const TP<float>& F = P.pf;
    m[0] = clampf(down(m0), -F.moment_max[0], F.moment_max[0]);
    m[1] = clampf(down(m1), -F.moment_max[1], F.moment_max[1]);
    m[2] = clampf(down(m2), -F.moment_max[2], F.moment_max[2]);
}

// Full-range sin/cos (yaw setpoints) in T (float: sincos_full).
__device__ __forceinline__ void sincos_full_t(float x, float& s, float& c) { sincos_full(x, s, c); }
// Full-range float64 sin/cos of a float32 angle (the position controller's
// yaw setpoint): k = rint(x 32/pi), r = x - k pi/32 (two-constant Cody-Waite,
// |r| <= pi/64), (cos, sin)(k pi/32) from a 64-entry table (correctly
// rounded, generated with mpmath), short Taylor polynomials for r (terms
// below 1e-20), and the angle-sum formulas.  ~25 instructions.
__device__ const double2 kSinCos64[64] = {
    {1.0, 0.0},
    {0.9951847266721969, 0.0980171403295606},
    {0.9807852804032304, 0.19509032201612828},
    {0.9569403357322088, 0.2902846772544624},
    {0.9238795325112867, 0.3826834323650898},
    {0.881921264348355, 0.47139673682599764},
    {0.8314696123025452, 0.5555702330196022},
    {0.773010453362737, 0.6343932841636455},
    {0.7071067811865476, 0.7071067811865476},
    {0.6343932841636455, 0.773010453362737},
    {0.5555702330196022, 0.8314696123025452},
    {0.47139673682599764, 0.881921264348355},
    {0.3826834323650898, 0.9238795325112867},
    {0.2902846772544624, 0.9569403357322088},
    {0.19509032201612828, 0.9807852804032304},
    {0.0980171403295606, 0.9951847266721969},
    {5.709968497124349e-62, 1.0},
    {-0.0980171403295606, 0.9951847266721969},
    {-0.19509032201612828, 0.9807852804032304},
    {-0.2902846772544624, 0.9569403357322088},
    {-0.3826834323650898, 0.9238795325112867},
    {-0.47139673682599764, 0.881921264348355},
    {-0.5555702330196022, 0.8314696123025452},
    {-0.6343932841636455, 0.773010453362737},
    {-0.7071067811865476, 0.7071067811865476},
    {-0.773010453362737, 0.6343932841636455},
    {-0.8314696123025452, 0.5555702330196022},
    {-0.881921264348355, 0.47139673682599764},
    {-0.9238795325112867, 0.3826834323650898},
    {-0.9569403357322088, 0.2902846772544624},
    {-0.9807852804032304, 0.19509032201612828},
    {-0.9951847266721969, 0.0980171403295606},
    {-1.0, 1.1419936994248699e-61},
    {-0.9951847266721969, -0.0980171403295606},
    {-0.9807852804032304, -0.19509032201612828},
    {-0.9569403357322088, -0.2902846772544624},
    {-0.9238795325112867, -0.3826834323650898},
    {-0.881921264348355, -0.47139673682599764},
    {-0.8314696123025452, -0.5555702330196022},
    {-0.773010453362737, -0.6343932841636455},
    {-0.7071067811865476, -0.7071067811865476},
    {-0.6343932841636455, -0.773010453362737},
    {-0.5555702330196022, -0.8314696123025452},
    {-0.47139673682599764, -0.881921264348355},
    {-0.3826834323650898, -0.9238795325112867},
    {-0.2902846772544624, -0.9569403357322088},
    {-0.19509032201612828, -0.9807852804032304},
    {-0.0980171403295606, -0.9951847266721969},
    {2.3179070562307263e-60, -1.0},
    {0.0980171403295606, -0.9951847266721969},
    {0.19509032201612828, -0.9807852804032304},
    {0.2902846772544624, -0.9569403357322088},
    {0.3826834323650898, -0.9238795325112867},
    {0.47139673682599764, -0.881921264348355},
    {0.5555702330196022, -0.8314696123025452},
    {0.6343932841636455, -0.773010453362737},
    {0.7071067811865476, -0.7071067811865476},
    {0.773010453362737, -0.6343932841636455},
    {0.8314696123025452, -0.5555702330196022},
    {0.881921264348355, -0.47139673682599764},
    {0.9238795325112867, -0.3826834323650898},
    {0.9569403357322088, -0.2902846772544624},
    {0.9807852804032304, -0.19509032201612828},
    {0.9951847266721969, -0.0980171403295606},
};

__device__ __forceinline__ void sincos_full_t(float xf, double& s, double& c) {
    const double x = xf;
    const double k = rint(x * 10.185916357881302);
    double r = fma(k, -0.09817477042468103, x);
    r = fma(k, -3.827021247335479e-18, r);
    const double2 t = __ldg(&kSinCos64[(int)(long long)k & 63]);   // (cos, sin)
    const double r2 = r * r;
    const double sr = fma(r * r2, fma(r2, fma(r2, fma(r2, 2.7557319223985891e-6,
                          -1.9841269841269841e-4), 8.3333333333333333e-3),
                          -1.6666666666666667e-1), r);
    const double cr = fma(r2, fma(r2, fma(r2, fma(r2, 2.4801587301587302e-5,
                          -1.3888888888888889e-3), 4.1666666666666667e-2), -0.5), 1.0);
    c = fma(t.x, cr, -t.y * sr);
    s = fma(t.y, cr, t.x * sr);
}

// Desired rotation of the position controller as columns (d1, d2, d3) and
// the collective thrust.
template <typename T>
struct DesRot {
    T thrust, d1[3], d2[3], d3[3];
};

// Lee position controller, z-up, thrust along +b3 (EXTENSION; SURVEY.md
// Appendix A.5):
//   a = -k_p (p - p_d) - k_v v + g e3;  a_z >= POS_MIN_UP_ACCEL;
//   |a_xy| <= a_z tan(max_tilt);  f = m a . b3;  d3 = a/|a|;
//   d2 = normalize(d3 x (cos yaw_d, sin yaw_d, 0));  d1 = d2 x d3.
template <typename T>
__device__ __forceinline__ void position_ref(const Rot<T>& R, const float* p, const float* v,
                                             const float* cmd, T mass, const KParams& P,
                                             DesRot<T>& o) {
    const TP<T>& Q = tp<T>(P);
    T ax = -Q.g_pos[0] * (up<T>(p[0]) - up<T>(cmd[0])) - Q.g_vel[0] * up<T>(v[0]);
    T ay = -Q.g_pos[1] * (up<T>(p[1]) - up<T>(cmd[1])) - Q.g_vel[1] * up<T>(v[1]);
    T az = -Q.g_pos[2] * (up<T>(p[2]) - up<T>(cmd[2])) - Q.g_vel[2] * up<T>(v[2]) + Q.gravity;
    az = az > T(0.5) ? az : T(0.5);                               // POS_MIN_UP_ACCEL
    const T h2 = ax * ax + ay * ay;
    const T hmax = az * Q.tan_tilt;
    if (h2 > hmax * hmax) {
        const T hs = hmax * rsqrt_t(h2);
        ax *= hs;
        ay *= hs;
    }
    o.thrust = mass * (ax * R.r02 + ay * R.r12 + az * R.r22);
    const T ia = rsqrt_t(ax * ax + ay * ay + az * az);
    o.d3[0] = ax * ia;
    o.d3[1] = ay * ia;
    o.d3[2] = az * ia;
    T sy, cy;
    sincos_full_t(cmd[3], sy, cy);
    const T cx_ = -o.d3[2] * sy, cy_ = o.d3[2] * cy, cz_ = o.d3[0] * sy - o.d3[1] * cy;
    const T icn = rsqrt_t(cx_ * cx_ + cy_ * cy_ + cz_ * cz_);      // >= d3_z > 0
    o.d2[0] = cx_ * icn;
    o.d2[1] = cy_ * icn;
    o.d2[2] = cz_ * icn;
    o.d1[0] = o.d2[1] * o.d3[2] - o.d2[2] * o.d3[1];
    o.d1[1] = o.d2[2] * o.d3[0] - o.d2[0] * o.d3[2];
    o.d1[2] = o.d2[0] * o.d3[1] - o.d2[1] * o.d3[0];
}

// e_R = vee(A - A^T)/2 with A = R_d^T R, A_ij = (column i of R_d).(column j of R)
template <typename T>
__device__ __forceinline__ void rotation_error(const Rot<T>& R, const DesRot<T>& d, T (&eR)[3]) {
    const T A21 = d.d3[0] * R.r01 + d.d3[1] * R.r11 + d.d3[2] * R.r21;
    const T A12 = d.d2[0] * R.r02 + d.d2[1] * R.r12 + d.d2[2] * R.r22;
    const T A02 = d.d1[0] * R.r02 + d.d1[1] * R.r12 + d.d1[2] * R.r22;
    const T A20 = d.d3[0] * R.r00 + d.d3[1] * R.r10 + d.d3[2] * R.r20;
    const T A10 = d.d2[0] * R.r00 + d.d2[1] * R.r10 + d.d2[2] * R.r20;
    const T A01 = d.d1[0] * R.r01 + d.d1[1] * R.r11 + d.d1[2] * R.r21;
    eR[0] = T(0.5) * (A21 - A12);
    eR[1] = T(0.5) * (A02 - A20);
    eR[2] = T(0.5) * (A10 - A01);
}

// T_i = clip(A^+_i . w, 0, T_max) and the realized wrench A T over the first
// NR rotors of an airframe (the sums in rotor order, as the generic loop)
template <int NR>
__device__ __forceinline__ void allocate_rotors(const fs_airframe& fr, float f, float m0,
                                                float m1, float m2, StepOut& o, float& rf,
                                                float& rm0, float& rm1, float& rm2) {
#pragma unroll
    for (int i = 0; i < FS_MAX_ROTORS; ++i) {
        float t = 0.0f;
        if (i < NR) {
            const float* row = fr.pinv + 4 * i;
            t = clampf(row[0] * f + row[1] * m0 + row[2] * m1 + row[3] * m2, 0.0f, fr.rotor_max);
            rf += fr.alloc[0 * FS_MAX_ROTORS + i] * t;
            rm0 += fr.alloc[1 * FS_MAX_ROTORS + i] * t;
            rm1 += fr.alloc[2 * FS_MAX_ROTORS + i] * t;
            rm2 += fr.alloc[3 * FS_MAX_ROTORS + i] * t;
        }
        o.rotor[i] = t;
    }
}

template <int FR>
__device__ __forceinline__ void allocate_frame(const KParams& P, float f, float m0, float m1,
                                               float m2, StepOut& o, float& rf, float& rm0,
                                               float& rm1, float& rm2) {
    const fs_airframe& fr = P.frame[FR];
    switch (fr.n_rotors) {
        case 4: allocate_rotors<4>(fr, f, m0, m1, m2, o, rf, rm0, rm1, rm2); break;
        case 6: allocate_rotors<6>(fr, f, m0, m1, m2, o, rf, rm0, rm1, rm2); break;
        default: {
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
        }
    }
}

// MODE:  FS_MODE_ATTITUDE / VELOCITY / MIXED / POSITION
// HETERO: per-vehicle mass and diagonal inertia (vp[0..3]) and two airframes
// PREC:  0 / 1 / 2 (see above)
// cmd:   the vehicle's command values (4, or 8 for MIXED)
// vmode: the vehicle's mode byte (MIXED only)
// CT:    command element type: float (command planes) or double (commands
//        denormalized in float64 from RL actions, fs_world.cu)
// Returns the control output in `o`; if `integrate`, advances `s` in place.
template <int MODE, bool HETERO, int PREC, int FEAT = kFeatAll, typename CT = float>
__device__ __forceinline__ void vehicle_step(VState& s, const CT* cmd, uint32_t vmode,
                                             const float* vp, int frame_id,
                                             const KParams& P, bool integrate, StepOut& o) {
    using TF = typename std::conditional<(PREC >= 1), double, float>::type;   // front end
    using TC = typename std::conditional<(PREC >= 2), double, float>::type;   // core
    const float qw = s.q[0], qx = s.q[1], qy = s.q[2], qz = s.q[3];
    const float wx = s.w[0], wy = s.w[1], wz = s.w[2];
    const TP<float>& F = P.pf;
    const float g = F.gravity;
    const float mass = HETERO ? vp[0] : F.mass;
    uint32_t flags = 0;

    // J w (body angular momentum), used by the moment law and the integrator
    float jwx, jwy, jwz;
    if (HETERO) {
        jwx = vp[1] * wx;
        jwy = vp[2] * wy;
        jwz = vp[3] * wz;
    } else if (P.jdiag) {
        jwx = F.inertia[0] * wx;
        jwy = F.inertia[4] * wy;
        jwz = F.inertia[8] * wz;
    } else {
        const float* J = F.inertia;
        jwx = J[0] * wx + J[1] * wy + J[2] * wz;
        jwy = J[3] * wx + J[4] * wy + J[5] * wz;
        jwz = J[6] * wx + J[7] * wy + J[8] * wz;
    }

    float b3x, b3y, b3z;       // body z axis (third column of R), fp32
    float f, m[3];             // saturated wrench

    if constexpr (MODE == FS_MODE_POSITION) {
        // --- Lee position controller (EXTENSION) ----------------
        const Rot<TF> RF = rotmat<TF>(qw, qx, qy, qz);
        const TF massT = HETERO ? up<TF>(vp[0]) : tp<TF>(P).mass;
        DesRot<TF> df;
        position_ref<TF>(RF, s.p, s.v, cmd, massT, P, df);
        Rot<TC> RC;
        DesRot<TC> dc;
        if constexpr (std::is_same<TF, TC>::value) {
            RC = RF;
            dc = df;
        } else {
            RC = rotmat<TC>(qw, qx, qy, qz);
            dc = DesRot<TC>{(TC)df.thrust, {(TC)df.d1[0], (TC)df.d1[1], (TC)df.d1[2]},
                            {(TC)df.d2[0], (TC)df.d2[1], (TC)df.d2[2]},
                            {(TC)df.d3[0], (TC)df.d3[1], (TC)df.d3[2]}};
        }
        TC eR[3];
        rotation_error<TC>(RC, dc, eR);
        const TC eW[3] = {up<TC>(wx), up<TC>(wy), up<TC>(wz)};     // omega_d = 0
        moment_law<TC>(eR, eW, eW[0], eW[1], eW[2], up<TC>(jwx), up<TC>(jwy), up<TC>(jwz), P, m);
        f = clampf(down(df.thrust), 0.0f, F.thrust_max);
        b3x = down(RF.r02);
        b3y = down(RF.r12);
        b3z = down(RF.r22);
    } else {
        bool vel = (MODE == FS_MODE_VELOCITY);
        if constexpr (MODE == FS_MODE_MIXED) vel = (vmode == FS_MODE_VELOCITY);
        const CT* vc = (MODE == FS_MODE_MIXED) ? cmd + 4 : cmd;
        const Rot<TF> RF = rotmat<TF>(qw, qx, qy, qz);
        Tilt<TF> cf;
        const TF massT = HETERO ? up<TF>(vp[0]) : tp<TF>(P).mass;
        if (vel)
            velocity_tilt<TF, CT>(RF, s.v, vc, massT, P, cf, flags);
        else
            attitude_tilt<TF, CT>(RF, cmd, cf);
        Rot<TC> RC;
        Tilt<TC> cc;
        if constexpr (std::is_same<TF, TC>::value) {
            RC = RF;
            cc = cf;
        } else {
            RC = rotmat<TC>(qw, qx, qy, qz);
            cc = Tilt<TC>{(TC)cf.cy, (TC)cf.sy, (TC)cf.cr, (TC)cf.sr,
                          (TC)cf.ct, (TC)cf.st, (TC)cf.yr, (TC)cf.thrust};
        }
        TC eR[3], eW[3];
        const TC wxc = up<TC>(wx), wyc = up<TC>(wy), wzc = up<TC>(wz);
        attitude_errors<TC>(RC, cc, wxc, wyc, wzc, eR, eW);
        moment_law<TC>(eR, eW, wxc, wyc, wzc, up<TC>(jwx), up<TC>(jwy), up<TC>(jwz), P, m);
        f = clampf(down(cf.thrust), 0.0f, F.thrust_max);
        b3x = down(RF.r02);
        b3y = down(RF.r12);
        b3z = down(RF.r22);
    }
    o.f = f;
    o.m[0] = m[0];
    o.m[1] = m[1];
    o.m[2] = m[2];
    float m0 = m[0], m1 = m[1], m2 = m[2];

    // --- allocation T = clip(A^+ w) (EXTENSION) ------------------
    if ((FEAT & kFeatOut) && P.n_frames > 0) {
        // airframe index and rotor count as compile-time constants wherever
        // they are warp-uniform (every warp but the one straddling the split):
        // the A^+ rows and A columns become constant-bank operands
        float rf = 0.0f, rm0 = 0.0f, rm1 = 0.0f, rm2 = 0.0f;
        if (!HETERO || frame_id == 0)
            allocate_frame<0>(P, f, m0, m1, m2, o, rf, rm0, rm1, rm2);
        else
            allocate_frame<1>(P, f, m0, m1, m2, o, rf, rm0, rm1, rm2);
        if (P.d.rotor_dynamics) {
            f = rf;
            m0 = rm0;
            m1 = rm1;
            m2 = rm2;
        }
    }

    if ((FEAT & kFeatOut) && P.want_flags && MODE != FS_MODE_POSITION &&
        gimbal_flag(qw, qx, qy, qz, P.gimbal_cos))
        flags |= FS_FLAG_GIMBAL;

    if (integrate) {
        // --- semi-implicit Euler: dynamics.py:286-341 ----------------------------
        const float dt = P.d.dt;
        const float a = HETERO ? f / mass : f * F.inv_mass;      // dynamics.py:299
        float vx = s.v[0] + dt * (a * b3x);
        float vy = s.v[1] + dt * (a * b3y);
        float vz = s.v[2] + dt * (a * b3z - g);
        bool over = clamp_norm(vx, vy, vz, F.v_limit, F.v_lim2);
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
            nx = F.inertia_inv[0] * tx;
            ny = F.inertia_inv[4] * ty;
            nz = F.inertia_inv[8] * tz;
        } else {
            const float* Ji = F.inertia_inv;
            nx = Ji[0] * tx + Ji[1] * ty + Ji[2] * tz;
            ny = Ji[3] * tx + Ji[4] * ty + Ji[5] * tz;
            nz = Ji[6] * tx + Ji[7] * ty + Ji[8] * tz;
        }
        over |= clamp_norm(nx, ny, nz, F.omega_limit, F.w_lim2);
        s.w[0] = nx;
        s.w[1] = ny;
        s.w[2] = nz;

        // q+ = normalize(q (x) exp(dt w+)): se3.py:78-97
        if (P.exp2_poly)
            exp_quat_small(dt * nx, dt * ny, dt * nz, ew, ex, ey, ez);
        else
            exp_quat(dt * nx, dt * ny, dt * nz, ew, ex, ey, ez);
        const float pw = qw * ew - qx * ex - qy * ey - qz * ez;
        const float px = qw * ex + qx * ew + qy * ez - qz * ey;
        const float py = qw * ey - qx * ez + qy * ew + qz * ex;
        const float pz = qw * ez + qx * ey - qy * ex + qz * ew;
        const float iq = rsqrtf(fmaf(pw, pw, fmaf(px, px, fmaf(py, py, pz * pz))));
        s.q[0] = pw * iq;
        s.q[1] = px * iq;
        s.q[2] = py * iq;
        s.q[3] = pz * iq;
        if (over) flags |= FS_FLAG_CLAMPED;
        if ((FEAT & (kFeatOut | kFeatStats)) && P.want_flags) {
            // any non-finite component (dynamics.py:334-339): x*0 is NaN iff x
            // is.  p and q cover v and w: a non-finite v makes p = p + dt v
            // non-finite (the norm clamp turns an infinite v into NaN), and a
            // non-finite w makes exp(dt w), hence the renormalized q, NaN
            float zr = 0.0f;
#pragma unroll
            for (int k = 0; k < 3; ++k) zr = fmaf(s.p[k], 0.0f, zr);
#pragma unroll
            for (int k = 0; k < 4; ++k) zr = fmaf(s.q[k], 0.0f, zr);
            if (zr != zr) flags |= FS_FLAG_NONFINITE;
        }
    }
    o.flags = flags;
}

}  // namespace fs
