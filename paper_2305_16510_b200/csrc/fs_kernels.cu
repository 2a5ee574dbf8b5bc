// fs_kernels.cu -- sm_100a kernels and the extern "C" boundary
// (include/flocksim_b200.h).
//
// Hot kernel: step_kernel<MODE, HETERO, VPT, ROLLOUT>.  One thread owns VPT
// consecutive vehicles; every state/command plane is read with one
// VPT-wide vector load (float4 for VPT = 4) and written with one vector
// store, so a warp moves 32 * VPT * 4 contiguous bytes per plane: fully
// coalesced 128-B lines on all 13 + 4 (+ 4) planes.  No shared memory, no
// block barrier except the optional statistics reduction.  Grid = ceil(n /
// (VPT * 256)) CTAs of 256 threads; at the bench sizes that is >= 4 waves of
// the 148 SMs.  ROLLOUT keeps the vehicle in registers for P.steps steps
// (fs_rollout).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <thread>
#include <vector>
#include <atomic>
#include <cmath>

#include "flocksim_b200.h"
#include "fs_host.h"
#include "fs_math.cuh"
#include "fs_rng.cuh"
#include "fs_step.cuh"

namespace fs {

// ---------------------------------------------------------------------------
// unfused drop-in kernels (one vehicle per thread; not on the bench path).
// The controller pieces evaluate in float64 from the fp32 inputs, like the
// fused kernel's PREC 2 controller; the integrator is fp32 like the fused one.
// ---------------------------------------------------------------------------
__global__ void integrate_kernel(const __grid_constant__ KParams P, const float* __restrict__ wr,
                                 int64_t wstride) {
    const fs_step_desc& d = P.d;
    const TP<float>& F = P.pf;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d.n) return;
    const float* S = d.state_in;
    const int64_t ss = d.state_in_stride;
    VState s;
    for (int k = 0; k < 3; ++k) {
        s.p[k] = S[k * ss + i];
        s.v[k] = S[(7 + k) * ss + i];
        s.w[k] = S[(10 + k) * ss + i];
    }
    for (int k = 0; k < 4; ++k) s.q[k] = S[(3 + k) * ss + i];
    const float f = wr[i], m0 = wr[wstride + i], m1 = wr[2 * wstride + i], m2 = wr[3 * wstride + i];
    // dynamics.py:286-341 (same arithmetic as the fused kernel's integrator)
    const float qw = s.q[0], qx = s.q[1], qy = s.q[2], qz = s.q[3];
    const Rot<float> R = rotmat<float>(qw, qx, qy, qz);
    const float dt = d.dt;
    const float a = f * F.inv_mass;
    float vx = s.v[0] + dt * (a * R.r02);
    float vy = s.v[1] + dt * (a * R.r12);
    float vz = s.v[2] + dt * (a * R.r22 - F.gravity);
    bool over = clamp_norm(vx, vy, vz, F.v_limit, F.v_lim2);
    const float* J = F.inertia;
    const float* Ji = F.inertia_inv;
    const float wx = s.w[0], wy = s.w[1], wz = s.w[2];
    float lx = J[0] * wx + J[1] * wy + J[2] * wz;
    float ly = J[3] * wx + J[4] * wy + J[5] * wz;
    float lz = J[6] * wx + J[7] * wy + J[8] * wz;
    float ew, ex, ey, ez;
    exp_quat(-dt * wx, -dt * wy, -dt * wz, ew, ex, ey, ez);
    quat_rotate(ew, ex, ey, ez, lx, ly, lz);
    const float tx = lx + dt * m0, ty = ly + dt * m1, tz = lz + dt * m2;
    float nx = Ji[0] * tx + Ji[1] * ty + Ji[2] * tz;
    float ny = Ji[3] * tx + Ji[4] * ty + Ji[5] * tz;
    float nz = Ji[6] * tx + Ji[7] * ty + Ji[8] * tz;
    over |= clamp_norm(nx, ny, nz, F.omega_limit, F.w_lim2);
    exp_quat(dt * nx, dt * ny, dt * nz, ew, ex, ey, ez);
    float pw = qw * ew - qx * ex - qy * ey - qz * ez;
    float px = qw * ex + qx * ew + qy * ez - qz * ey;
    float py = qw * ey - qx * ez + qy * ew + qz * ex;
    float pz = qw * ez + qx * ey - qy * ex + qz * ew;
    const float iq = rsqrtf(fmaf(pw, pw, fmaf(px, px, fmaf(py, py, pz * pz))));
    float out[13] = {s.p[0] + dt * vx, s.p[1] + dt * vy, s.p[2] + dt * vz,
                     pw * iq, px * iq, py * iq, pz * iq, vx, vy, vz, nx, ny, nz};
    float* O = d.state_out;
    const int64_t os = d.state_out_stride;
    float z = 0.0f;
    for (int k = 0; k < 13; ++k) {
        O[k * os + i] = out[k];
        z = fmaf(out[k], 0.0f, z);
    }
    if (d.flags_out)
        d.flags_out[i] = (uint8_t)((over ? FS_FLAG_CLAMPED : 0) | ((z != z) ? FS_FLAG_NONFINITE : 0));
}

// saturate_batch, dynamics.py:214-218 (bounds in float64, one rounding)
__global__ void saturate_kernel(const __grid_constant__ KParams P, const float* __restrict__ in,
                                int64_t is, float* __restrict__ out, int64_t os) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= P.d.n) return;
    const TP<double>& D = P.pd;
    out[i] = (float)fmin(fmax((double)in[i], 0.0), D.thrust_max);
    for (int k = 0; k < 3; ++k)
        out[(k + 1) * os + i] =
            (float)fmin(fmax((double)in[(k + 1) * is + i], -D.moment_max[k]), D.moment_max[k]);
}

// velocity_control (control.py:283-349): attitude-command planes (roll,
// pitch, yaw_rate, thrust), returned as angles like the reference, float64.
__global__ void velocity_control_kernel(const __grid_constant__ KParams P,
                                        float* __restrict__ att, int64_t as,
                                        uint8_t* __restrict__ degen) {
    const fs_step_desc& d = P.d;
    const TP<double>& D = P.pd;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d.n) return;
    const float* S = d.state_in;
    const int64_t ss = d.state_in_stride;
    const Rot<double> R = rotmat<double>(S[3 * ss + i], S[4 * ss + i], S[5 * ss + i], S[6 * ss + i]);
    const double yaw = atan2(R.r10, R.r00);
    double sy, cy;
    sincos(yaw, &sy, &cy);
    const float* vc = d.cmd;
    const int64_t cs = d.cmd_stride;
    double vcx = vc[i], vcy = vc[cs + i], vcz = vc[2 * cs + i];
    const double vn = sqrt(vcx * vcx + vcy * vcy + vcz * vcz);
    if (vn > D.max_speed) {
        const double sc = D.max_speed / vn;
        vcx *= sc; vcy *= sc; vcz *= sc;
    }
    const double vx = S[7 * ss + i], vy = S[8 * ss + i], vz = S[9 * ss + i];
    const double vvx = cy * vx + sy * vy, vvy = -sy * vx + cy * vy;
    const double ax = D.g_vel[0] * (vcx - vvx);
    const double ay = D.g_vel[1] * (vcy - vvy);
    const double az = D.g_vel[2] * (vcz - vz) + D.gravity;
    double thrust = D.mass * (ax * (cy * R.r02 + sy * R.r12) + ay * (-sy * R.r02 + cy * R.r12) +
                              az * R.r22);
    double roll = fmin(fmax(atan2(-ay, sqrt(ax * ax + az * az)), -D.max_tilt), D.max_tilt);
    double pitch = fmin(fmax(atan2(ax, az), -D.max_tilt), D.max_tilt);
    const bool dg = sqrt(ax * ax + ay * ay + az * az) < 1e-6;
    if (dg) { roll = 0.0; pitch = 0.0; thrust = D.mass * D.gravity; }
    att[i] = (float)roll;
    att[as + i] = (float)pitch;
    att[2 * as + i] = vc[3 * cs + i];
    att[3 * as + i] = (float)thrust;
    if (degen) degen[i] = dg ? 1 : 0;
}

// se3.yaw_of, se3.py:226-243 (float64; the gimbal test is bit-exact)
__global__ void yaw_kernel(int64_t n, const float* __restrict__ q, int64_t qs, double gcos,
                           float* __restrict__ yaw, uint8_t* __restrict__ gimbal) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float w = q[i], x = q[qs + i], y = q[2 * qs + i], z = q[3 * qs + i];
    const Rot<double> R = rotmat<double>(w, x, y, z);
    if (yaw) yaw[i] = (float)atan2(R.r10, R.r00);
    if (gimbal) gimbal[i] = gimbal_flag(w, x, y, z, gcos) ? 1 : 0;
}

// desired_attitude, control.py:190-218: q_d = rot_zyx(roll, pitch, yaw)
// (half-angle products, se3.py:200-215), omega_d via the Euler-rate map.
__global__ void desired_kernel(int64_t n, const float* __restrict__ yaw,
                               const float* __restrict__ a, int64_t as, float* __restrict__ qd,
                               int64_t qs, float* __restrict__ wd, int64_t ws) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double roll = a[i], pitch = a[as + i], yr = a[2 * as + i], ya = yaw[i];
    double sr2, cr2, sp2, cp2, sy2, cy2;
    sincos(0.5 * roll, &sr2, &cr2);
    sincos(0.5 * pitch, &sp2, &cp2);
    sincos(0.5 * ya, &sy2, &cy2);
    const double w = cy2 * cp2 * cr2 + sy2 * sp2 * sr2;
    const double x = cy2 * cp2 * sr2 - sy2 * sp2 * cr2;
    const double y = cy2 * sp2 * cr2 + sy2 * cp2 * sr2;
    const double z = sy2 * cp2 * cr2 - cy2 * sp2 * sr2;
    const double iq = 1.0 / sqrt(w * w + x * x + y * y + z * z);
    qd[i] = (float)(w * iq);
    qd[qs + i] = (float)(x * iq);
    qd[2 * qs + i] = (float)(y * iq);
    qd[3 * qs + i] = (float)(z * iq);
    double sr, cr, sp, cp;
    sincos(roll, &sr, &cr);
    sincos(pitch, &sp, &cp);
    wd[i] = (float)(-sp * yr);
    wd[ws + i] = (float)(sr * cp * yr);
    wd[2 * ws + i] = (float)(cr * cp * yr);
}

// attitude_errors, control.py:221-258: e_R = 0.5 vee(Rd^T R - R^T Rd),
// e_W = w - (Rd^T R)^T wd (float64)
__global__ void errors_kernel(int64_t n, const float* __restrict__ q, int64_t qs,
                              const float* __restrict__ om, int64_t os,
                              const float* __restrict__ qd, int64_t qds,
                              const float* __restrict__ wd, int64_t wds, float* __restrict__ er,
                              float* __restrict__ ew, int64_t es) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Rot<double> R = rotmat<double>(q[i], q[qs + i], q[2 * qs + i], q[3 * qs + i]);
    const Rot<double> D = rotmat<double>(qd[i], qd[qds + i], qd[2 * qds + i], qd[3 * qds + i]);
    const double r[3][3] = {{R.r00, R.r01, R.r02}, {R.r10, R.r11, R.r12}, {R.r20, R.r21, R.r22}};
    const double dm[3][3] = {{D.r00, D.r01, D.r02}, {D.r10, D.r11, D.r12}, {D.r20, D.r21, D.r22}};
    double A[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) A[a][b] = dm[0][a] * r[0][b] + dm[1][a] * r[1][b] + dm[2][a] * r[2][b];
    er[i] = (float)(0.5 * (A[2][1] - A[1][2]));
    er[es + i] = (float)(0.5 * (A[0][2] - A[2][0]));
    er[2 * es + i] = (float)(0.5 * (A[1][0] - A[0][1]));
    const double w0 = wd[i], w1 = wd[wds + i], w2 = wd[2 * wds + i];
    for (int b = 0; b < 3; ++b)
        ew[b * es + i] = (float)((double)om[b * os + i] - (A[0][b] * w0 + A[1][b] * w1 + A[2][b] * w2));
}

__global__ void init_fleet_kernel(int64_t n, int64_t first_id, uint64_t seed, int mode,
                                  float* __restrict__ st, int64_t ss, float* __restrict__ cmd,
                                  int64_t cs, float* __restrict__ vpar, int64_t vs, float mass,
                                  float gravity, float jxx, float jyy, float jzz) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int64_t gid = first_id + i;
    float vp[4] = {mass, jxx, jyy, jzz};
    if (vpar) {
        spawn_vparams(seed, gid, mass, jxx, jyy, jzz, vp);
        for (int k = 0; k < 4; ++k) vpar[k * vs + i] = vp[k];
    }
    float s[13], c[8];
    spawn(seed, gid, kInitStep, mode, vp[0], gravity, s, c);
    if (st)
        for (int k = 0; k < 13; ++k) st[k * ss + i] = s[k];
    if (cmd) {
        const int nc = (mode == FS_MODE_MIXED) ? 8 : 4;
        for (int k = 0; k < nc; ++k) cmd[k * cs + i] = c[k];
    }
}

__global__ void stats_reduce_kernel(const int64_t* __restrict__ slots, int nslots,
                                    int64_t* __restrict__ out) {
    __shared__ long long red[3][kThreads];
    long long a = 0, b = 0, c = 0;
    for (int s = threadIdx.x; s < nslots; s += blockDim.x) {
        a += slots[3 * s];
        b += slots[3 * s + 1];
        c += slots[3 * s + 2];
    }
    red[0][threadIdx.x] = a;
    red[1][threadIdx.x] = b;
    red[2][threadIdx.x] = c;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o)
            for (int k = 0; k < 3; ++k) red[k][threadIdx.x] += red[k][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0)
        for (int k = 0; k < 3; ++k) out[k] = red[k][0];
}

}  // namespace fs

// ===========================================================================
// host side: validation + dispatch
// ===========================================================================
namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

}  // namespace

namespace fs {
int g_world_kernel = 0;     // free-space World.step kernel (fs_world.cu)
int g_clear_walk_cm = 60;   // obstacle worlds: clearance-cache slot-walk radius, cm (40-150 swept)
int g_clear_exact = 1;      // obstacle worlds: walked slots bound the clearance by their SDF
int g_kernel = 0;
int g_prec = -1;
int g_ctas_per_sm = 0;
int g_ncw = 0;
int g_vpt = 0;
int g_chain_release = 0;   // chained steps: gpu-scope fence before publishing a tile
int g_l2_keep_mb = 0;      // streaming kernel: MiB of tiles kept L2-resident across steps
int g_sync_timeout_ms = 10000;  // chained steps: trap after a tile wait this long (0 = never)
// chained steps, the load warp's side of a tile handoff: bit 0 gpu-scope
// acquire counter loads (LDG.STRONG.GPU + CCTL.IVALL), bit 1 fence.proxy.async
// before the tile's TMA loads, bit 2 fence.acq_rel.gpu after relaxed loads.
// Measured on cfg2 (500 steps, 2^22): 0 -> 76.8 us, 2 -> 77.3-77.7, 3 -> 81.6-82.2
// (the per-tile L1 invalidation stalls the TMA issue), 6 -> 106.9 us.
int g_chain_acquire = 2;
int g_spawn_wait_ns = 0;   // spawn warps: try_wait (0) or a nanosleep back-off start in ns (64: +0.3 us on cfg3)
int g_cons_wait_ns = 0;    // consumers: try_wait (0) or a back-off start in ns

// SM count of the CURRENT device, cached per device (thread-safe: a race
// only recomputes the same value)
int device_sm_count() {
    static std::atomic<int> cached[kMaxDevices];
    const int dev = current_device();
    if (dev < 0) return -1;
    if (dev < kMaxDevices) {
        const int c = cached[dev].load(std::memory_order_relaxed);
        if (c > 0) return c;
    }
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    if (dev < kMaxDevices) cached[dev].store(sms, std::memory_order_relaxed);
    return sms;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
        return FS_ELAUNCH;
    }
    return FS_OK;
}

int chain_unsupported() {
    snprintf(g_err, sizeof(g_err),
             "tile_sync (chained steps) needs the streaming kernel: 16-byte aligned planes "
             "with strides a multiple of 4 and n >= 2^15");
    return FS_EINVAL;
}
}  // namespace fs

namespace {
using fs::check_launch;

template <typename T>
void fill_tp(fs::TP<T>& t, const fs_robot* r, const fs_gains* g, const fs_limits* l) {
    if (r) {
        t.mass = (T)r->mass;
        t.inv_mass = (T)(1.0 / r->mass);
        t.gravity = (T)r->gravity;
        t.thrust_max = (T)r->thrust_max;
        for (int k = 0; k < 3; ++k) t.moment_max[k] = (T)r->moment_max[k];
        t.v_limit = (T)r->v_limit;
        t.omega_limit = (T)r->omega_limit;
        t.v_lim2 = (T)(r->v_limit * r->v_limit);
        t.w_lim2 = (T)(r->omega_limit * r->omega_limit);
        for (int k = 0; k < 9; ++k) {
            t.inertia[k] = (T)r->inertia[k];
            t.inertia_inv[k] = (T)r->inertia_inv[k];
        }
    }
    if (g) {
        for (int k = 0; k < 3; ++k) {
            t.g_att[k] = (T)g->attitude[k];
            t.g_rate[k] = (T)g->rate[k];
            t.g_vel[k] = (T)g->velocity[k];
            t.g_pos[k] = (T)g->position[k];
        }
    }
    if (l) {
        t.max_tilt = (T)l->max_tilt;
        t.cos_tilt = (T)std::cos(l->max_tilt);
        t.sin_tilt = (T)std::sin(l->max_tilt);
        t.tan_tilt = (T)std::tan(l->max_tilt);
        t.max_speed = (T)l->max_speed_cmd;
        t.max_speed2 = (T)(l->max_speed_cmd * l->max_speed_cmd);
    }
}

int fill_params(fs::KParams& P, const fs_step_desc* d, const fs_robot* r, const fs_gains* g,
                const fs_limits* l, const fs_airframe* frames) {
    memset(&P, 0, sizeof(P));
    P.chain_release = fs::g_chain_release;
    P.chain_acquire = fs::g_chain_acquire;
    P.spawn_wait_ns = (uint32_t)fs::g_spawn_wait_ns;
    P.cons_wait_ns = (uint32_t)fs::g_cons_wait_ns;
    P.sync_timeout_ns = (uint64_t)(fs::g_sync_timeout_ms > 0 ? fs::g_sync_timeout_ms : 0) * 1000000ull;
    if (d) {
        P.d = *d;
        if (d->state_out)
            for (int k = 0; k < 13; ++k) P.out_plane[k] = d->state_out + k * d->state_out_stride;
    }
    fill_tp(P.pf, r, g, l);
    fill_tp(P.pd, r, g, l);
    if (r) {
        P.gimbal_cos = r->gimbal_cos;
        P.jdiag = (r->inertia[1] == 0.0 && r->inertia[2] == 0.0 && r->inertia[3] == 0.0 &&
                   r->inertia[5] == 0.0 && r->inertia[6] == 0.0 && r->inertia[7] == 0.0 &&
                   r->inertia_inv[1] == 0.0 && r->inertia_inv[2] == 0.0 &&
                   r->inertia_inv[3] == 0.0 && r->inertia_inv[5] == 0.0 &&
                   r->inertia_inv[6] == 0.0 && r->inertia_inv[7] == 0.0);
    }
    if (d && r) P.exp2_poly = (0.5 * (double)d->dt * r->omega_limit) <= 0.78;
    if (frames) {
        P.frame[0] = frames[0];
        P.frame[1] = frames[1];
        P.n_frames = frames[0].n_rotors > 0 ? 2 : 0;
        for (int k = 0; k < 2; ++k)
            if (frames[k].n_rotors < 0 || frames[k].n_rotors > FS_MAX_ROTORS)
                return fail(FS_EINVAL, "airframe n_rotors must be in [0, 6]");
    }
    return FS_OK;
}

int validate_step(const fs_step_desc* d, const fs_robot* r, const fs_gains* g,
                  const fs_limits* l) {
    if (!d || !r || !g || !l) return fail(FS_EINVAL, "null descriptor/params");
    if (d->n < 0) return fail(FS_EINVAL, "length must be >= 0");
    if (d->mode < FS_MODE_ATTITUDE || d->mode > FS_MODE_POSITION)
        return fail(FS_EINVAL, "mode must be one of FS_MODE_*");
    if (d->n == 0) return FS_OK;
    if (!d->state_in || !d->cmd) return fail(FS_EINVAL, "state_in and cmd are required");
    if (d->state_in_stride < d->n || d->cmd_stride < d->n)
        return fail(FS_EINVAL, "plane stride shorter than length");
    if (d->integrate) {
        if (!(d->dt > 0.0f && d->dt <= 0.1f)) return fail(FS_EINVAL, "dt must be in (0, 0.1]");
        if (!d->state_out || d->state_out_stride < d->n)
            return fail(FS_EINVAL, "state_out missing or stride shorter than length");
    }
    if (d->mode == FS_MODE_MIXED && !d->mode_per_vehicle)
        return fail(FS_EINVAL, "FS_MODE_MIXED needs mode_per_vehicle");
    if (d->vparams && d->vparams_stride < d->n)
        return fail(FS_EINVAL, "vparams stride shorter than length");
    if (d->wrench_out && d->wrench_stride < d->n)
        return fail(FS_EINVAL, "wrench stride shorter than length");
    if (d->rotor_out && d->rotor_stride < d->n)
        return fail(FS_EINVAL, "rotor stride shorter than length");
    if (d->stats_slots && (d->stats_nslots <= 0 || (d->stats_nslots & (d->stats_nslots - 1))))
        return fail(FS_EINVAL, "stats_nslots must be a power of two");
    if (d->reset_prob < 0.0f || d->reset_prob > 1.0f)
        return fail(FS_EINVAL, "reset_prob must be in [0, 1]");
    if (d->reset_prob > 0.0f && d->n > INT32_MAX)
        return fail(FS_EINVAL, "re-spawning shards must hold fewer than 2^31 vehicles");
    if (d->tile_sync && !d->integrate)
        return fail(FS_EINVAL, "tile_sync (chained steps) needs integrate = 1");
    return FS_OK;
}

template <bool ROLLOUT>
int launch_step(const fs::KParams& P, cudaStream_t s) {
    switch (P.d.mode) {
        case FS_MODE_ATTITUDE: return fs::launch_attitude(P, s, ROLLOUT);
        case FS_MODE_VELOCITY: return fs::launch_velocity(P, s, ROLLOUT);
        case FS_MODE_MIXED: return fs::launch_mixed(P, s, ROLLOUT);
        default: return fs::launch_position(P, s, ROLLOUT);
    }
}

// reset iff the mask word < floor(p * 2^32)  (CPU twin: oracle/rng_twin.py)
uint32_t reset_threshold(float p) {
    const double t = std::floor((double)p * 4294967296.0);
    return t >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)t;
}

unsigned grid1(int64_t n) { return (unsigned)((n + fs::kThreads - 1) / fs::kThreads); }

}  // namespace

// hooks for fs_world.cu (same library)
int fs_fill_params_for_world(fs::KParams& P, const fs_step_desc* d, const fs_robot* r,
                             const fs_gains* g, const fs_limits* l) {
    const int rc = fill_params(P, d, r, g, l, nullptr);
    P.steps = 1;
    return rc;
}
int fs_fail_einval(const char* msg) { return fail(FS_EINVAL, msg); }

extern "C" {

int fs_abi_version(void) { return FS_ABI_VERSION; }

int fs_set_tuning(int32_t key, int32_t value) {
    switch (key) {
        case FS_TUNE_KERNEL: fs::g_kernel = value; return FS_OK;
        case FS_TUNE_PREC: fs::g_prec = value; return FS_OK;
        case FS_TUNE_CTAS_PER_SM: fs::g_ctas_per_sm = value; return FS_OK;
        case FS_TUNE_VPT:
            if (value != 0 && value != 1 && value != 2) return fail(FS_EINVAL, "VPT must be 0, 1 or 2");
            fs::g_vpt = value;
            return FS_OK;
        case FS_TUNE_WORLD_KERNEL:
            if (value < 0 || value > 2) return fail(FS_EINVAL, "world kernel must be 0, 1 or 2");
            fs::g_world_kernel = value;
            return FS_OK;
        case FS_TUNE_L2_KEEP_MB:
            if (value < 0 || value > 1024) return fail(FS_EINVAL, "L2 keep must be 0..1024 MiB");
            fs::g_l2_keep_mb = value;
            return FS_OK;
        case FS_TUNE_CHAIN_RELEASE:
            if (value != 0 && value != 1) return fail(FS_EINVAL, "chain release must be 0 or 1");
            fs::g_chain_release = value;
            return FS_OK;
        case FS_TUNE_CLEAR_EXACT:
            if (value != 0 && value != 1) return fail(FS_EINVAL, "clear exact must be 0 or 1");
            fs::g_clear_exact = value;
            return FS_OK;
        case FS_TUNE_CLEAR_WALK_CM:
            if (value < 0 || value > 10000) return fail(FS_EINVAL, "walk radius must be 0..10000 cm");
            fs::g_clear_walk_cm = value;
            return FS_OK;
        case FS_TUNE_SPAWN_WAIT_NS:
            if (value < 0 || value > 100000) return fail(FS_EINVAL, "wait must be 0..100000 ns");
            fs::g_spawn_wait_ns = value;
            return FS_OK;
        case FS_TUNE_CONS_WAIT_NS:
            if (value < 0 || value > 100000) return fail(FS_EINVAL, "wait must be 0..100000 ns");
            fs::g_cons_wait_ns = value;
            return FS_OK;
        case FS_TUNE_CHAIN_ACQUIRE:
            if (value < 0 || value > 7) return fail(FS_EINVAL, "chain acquire must be 0..7");
            fs::g_chain_acquire = value;
            return FS_OK;
        case FS_TUNE_SYNC_TIMEOUT_MS:
            if (value < 0) return fail(FS_EINVAL, "sync timeout must be >= 0 ms");
            fs::g_sync_timeout_ms = value;
            return FS_OK;
        case FS_TUNE_NCW:
            if (value != 0 && value != 12 && value != 16 && value != 20)
                return fail(FS_EINVAL, "NCW must be 0, 12, 16 or 20");
            fs::g_ncw = value;
            return FS_OK;
        default: return fail(FS_EINVAL, "unknown tuning key");
    }
}

const char* fs_last_error(void) { return g_err; }

int fs_device_sm_count(void) { return fs::device_sm_count(); }

int64_t fs_tile_sync_len(int64_t n) {
    return n <= 0 ? 0 : (n + FS_SYNC_GRANULE - 1) / FS_SYNC_GRANULE;
}

int fs_step(const fs_step_desc* d, const fs_robot* robot, const fs_gains* gains,
            const fs_limits* limits, const fs_airframe* frames, void* stream) {
    int rc = validate_step(d, robot, gains, limits);
    if (rc != FS_OK || d->n == 0) return rc;
    fs::KParams P;
    if ((rc = fill_params(P, d, robot, gains, limits, frames)) != FS_OK) return rc;
    P.want_flags = (d->flags_out != nullptr) || (d->stats_slots != nullptr);
    P.steps = 1;
    P.reset_thresh = reset_threshold(d->reset_prob);
    P.rs_key = fs::step_key(d->seed, (uint32_t)d->step_index);
    return launch_step<false>(P, (cudaStream_t)stream);
}

int fs_step_many(const fs_step_desc* d, const fs_robot* robot, const fs_gains* gains,
                 const fs_limits* limits, const fs_airframe* frames, int32_t steps,
                 void* stream) {
    if (steps < 1) return fail(FS_EINVAL, "steps must be >= 1");
    if (d && !d->integrate) return fail(FS_EINVAL, "fs_step_many integrates: set d->integrate");
    if (d && steps > 1 && !d->tile_sync)
        return fail(FS_EINVAL, "fs_step_many: steps > 1 needs tile_sync (fs_tile_sync_len(n))");
    if (d && d->tile_sync && d->sync_post != d->sync_wait + 1u)
        return fail(FS_EINVAL, "fs_step_many: sync_post must be sync_wait + 1");
    int rc = validate_step(d, robot, gains, limits);
    if (rc != FS_OK || d->n == 0) return rc;
    fs::KParams P;
    if ((rc = fill_params(P, d, robot, gains, limits, frames)) != FS_OK) return rc;
    P.want_flags = (d->flags_out != nullptr) || (d->stats_slots != nullptr);
    P.steps = steps;
    P.reset_thresh = reset_threshold(d->reset_prob);
    P.rs_key = fs::step_key(d->seed, (uint32_t)d->step_index);
    return launch_step<false>(P, (cudaStream_t)stream);
}

int fs_step_host_ex(const fs_step_desc* d, const fs_robot* robot, const fs_gains* gains,
                    const fs_limits* limits, const fs_airframe* frames, const fs_host_ws* ws) {
    int rc = validate_step(d, robot, gains, limits);
    if (rc != FS_OK || d->n == 0) return rc;
    if (!ws) return fail(FS_EINVAL, "null workspace");
    const bool mixed = d->mode == FS_MODE_MIXED;
    if (!ws->dev_state || !ws->dev_cmd || ws->dev_stride < d->n || (ws->dev_stride & 3))
        return fail(FS_EINVAL, "device workspace missing or dev_stride < n / not a multiple of 4");
    if (mixed && !ws->dev_mode) return fail(FS_EINVAL, "FS_MODE_MIXED needs dev_mode");
    if (d->wrench_out && !ws->dev_wrench) return fail(FS_EINVAL, "wrench_out needs dev_wrench");
    if (d->flags_out && !ws->dev_flags) return fail(FS_EINVAL, "flags_out needs dev_flags");
    if (ws->chunks < 1 || ws->nstreams < 1 || !ws->streams)
        return fail(FS_EINVAL, "chunks/streams must be >= 1");
    if (d->vparams || d->rotor_out || d->stats_slots || d->reset_prob > 0.0f || d->tile_sync)
        return fail(FS_EINVAL, "fs_step_host: optional device outputs/extensions not supported");
    const int nc = mixed ? 8 : 4;
    const int64_t n = d->n, ds = ws->dev_stride;
    const int chunks = ws->chunks;
    auto copy2d = [](void* dst, int64_t dpitch, const void* src, int64_t spitch, size_t w,
                     int rows, cudaMemcpyKind k, cudaStream_t s) {
        return cudaMemcpy2DAsync(dst, (size_t)dpitch, src, (size_t)spitch, w, (size_t)rows, k, s);
    };
    for (int c = 0; c < chunks; ++c) {
        // chunk bounds: multiples of 512 vehicles (TMA tile) except the last
        const int64_t a = ((n * c) / chunks) / 512 * 512;
        const int64_t b = (c == chunks - 1) ? n : ((n * (c + 1)) / chunks) / 512 * 512;
        if (b <= a) continue;
        cudaStream_t s = (cudaStream_t)ws->streams[c % ws->nstreams];
        const size_t w = (size_t)(b - a) * sizeof(float);
        const int64_t fp = ds * (int64_t)sizeof(float);
        cudaError_t e = copy2d(ws->dev_state + a, fp, d->state_in + a,
                               d->state_in_stride * (int64_t)sizeof(float), w, 13,
                               cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess)
            e = copy2d(ws->dev_cmd + a, fp, d->cmd + a, d->cmd_stride * (int64_t)sizeof(float), w,
                       nc, cudaMemcpyHostToDevice, s);
        if (e == cudaSuccess && mixed)
            e = cudaMemcpyAsync(ws->dev_mode + a, d->mode_per_vehicle + a, (size_t)(b - a),
                                cudaMemcpyHostToDevice, s);
        if (e != cudaSuccess) return fail(FS_ELAUNCH, cudaGetErrorString(e));
        fs_step_desc dc = *d;
        dc.n = b - a;
        dc.first_id = d->first_id + a;
        dc.state_in = ws->dev_state + a;
        dc.state_out = ws->dev_state + a;
        dc.state_in_stride = dc.state_out_stride = ds;
        dc.cmd = ws->dev_cmd + a;
        dc.cmd_stride = ds;
        dc.mode_per_vehicle = mixed ? ws->dev_mode + a : nullptr;
        dc.wrench_out = d->wrench_out ? ws->dev_wrench + a : nullptr;
        dc.wrench_stride = ds;
        dc.flags_out = d->flags_out ? ws->dev_flags + a : nullptr;
        if ((rc = fs_step(&dc, robot, gains, limits, frames, s)) != FS_OK) return rc;
        if (d->integrate)
            e = copy2d(d->state_out + a, d->state_out_stride * (int64_t)sizeof(float),
                       ws->dev_state + a, fp, w, 13, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && d->wrench_out)
            e = copy2d(d->wrench_out + a, d->wrench_stride * (int64_t)sizeof(float),
                       ws->dev_wrench + a, fp, w, 4, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess && d->flags_out)
            e = cudaMemcpyAsync(d->flags_out + a, ws->dev_flags + a, (size_t)(b - a),
                                cudaMemcpyDeviceToHost, s);
        if (e != cudaSuccess) return fail(FS_ELAUNCH, cudaGetErrorString(e));
    }
    return FS_OK;
}

int fs_step_host(const fs_step_desc* d, const fs_robot* robot, const fs_gains* gains,
                 const fs_limits* limits, const fs_airframe* frames, float* dev_state,
                 float* dev_cmd, int64_t dev_stride, int32_t chunks, void* const* streams,
                 int32_t nstreams) {
    if (d && d->mode == FS_MODE_MIXED)
        return fail(FS_EINVAL, "fs_step_host: mixed mode not supported (use fs_step_host_ex)");
    if (d && (d->wrench_out || d->flags_out))
        return fail(FS_EINVAL, "fs_step_host: optional device outputs/extensions not supported");
    fs_host_ws ws;
    memset(&ws, 0, sizeof(ws));
    ws.dev_state = dev_state;
    ws.dev_cmd = dev_cmd;
    ws.dev_stride = dev_stride;
    ws.chunks = chunks;
    ws.nstreams = nstreams;
    ws.streams = streams;
    return fs_step_host_ex(d, robot, gains, limits, frames, &ws);
}

int fs_rollout(const fs_step_desc* d, const fs_robot* robot, const fs_gains* gains,
               const fs_limits* limits, const fs_airframe* frames, int32_t steps,
               void* stream) {
    if (steps < 1) return fail(FS_EINVAL, "steps must be >= 1");
    if (d && !d->integrate) return fail(FS_EINVAL, "fs_rollout integrates: set d->integrate");
    if (d && d->tile_sync) return fail(FS_EINVAL, "fs_rollout takes no tile_sync (one launch)");
    int rc = validate_step(d, robot, gains, limits);
    if (rc != FS_OK || d->n == 0) return rc;
    fs::KParams P;
    if ((rc = fill_params(P, d, robot, gains, limits, frames)) != FS_OK) return rc;
    P.want_flags = (d->flags_out != nullptr) || (d->stats_slots != nullptr);
    P.steps = steps;
    P.reset_thresh = reset_threshold(d->reset_prob);
    return launch_step<true>(P, (cudaStream_t)stream);
}

int fs_integrate(int64_t n, const float* state_in, int64_t state_in_stride, const float* wrench,
                 int64_t wrench_stride, const fs_robot* robot, float dt, float* state_out,
                 int64_t state_out_stride, uint8_t* flags_out, void* stream) {
    if (!robot) return fail(FS_EINVAL, "null robot");
    if (!(dt > 0.0f && dt <= 0.1f)) return fail(FS_EINVAL, "dt must be in (0, 0.1]");
    if (n < 0) return fail(FS_EINVAL, "length must be >= 0");
    if (n == 0) return FS_OK;
    if (!state_in || !wrench || !state_out) return fail(FS_EINVAL, "null pointer");
    if (state_in_stride < n || wrench_stride < n || state_out_stride < n)
        return fail(FS_EINVAL, "plane stride shorter than length");
    fs_step_desc d;
    memset(&d, 0, sizeof(d));
    d.n = n;
    d.state_in = state_in;
    d.state_in_stride = state_in_stride;
    d.state_out = state_out;
    d.state_out_stride = state_out_stride;
    d.flags_out = flags_out;
    d.dt = dt;
    d.integrate = 1;
    fs::KParams P;
    fill_params(P, &d, robot, nullptr, nullptr, nullptr);
    fs::integrate_kernel<<<grid1(n), fs::kThreads, 0, (cudaStream_t)stream>>>(P, wrench,
                                                                             wrench_stride);
    return check_launch("integrate_kernel");
}

int fs_saturate(int64_t n, const float* wrench_in, int64_t in_stride, const fs_robot* robot,
                float* wrench_out, int64_t out_stride, void* stream) {
    if (!robot || n < 0) return fail(FS_EINVAL, "bad arguments");
    if (n == 0) return FS_OK;
    if (!wrench_in || !wrench_out || in_stride < n || out_stride < n)
        return fail(FS_EINVAL, "bad wrench buffers");
    fs_step_desc d;
    memset(&d, 0, sizeof(d));
    d.n = n;
    fs::KParams P;
    fill_params(P, &d, robot, nullptr, nullptr, nullptr);
    fs::saturate_kernel<<<grid1(n), fs::kThreads, 0, (cudaStream_t)stream>>>(
        P, wrench_in, in_stride, wrench_out, out_stride);
    return check_launch("saturate_kernel");
}

int fs_velocity_control(int64_t n, const float* state, int64_t state_stride, const float* vcmd,
                        int64_t vcmd_stride, const fs_robot* robot, const fs_gains* gains,
                        const fs_limits* limits, float* att_out, int64_t att_stride,
                        uint8_t* degenerate_out, void* stream) {
    if (!robot || !gains || !limits || n < 0) return fail(FS_EINVAL, "bad arguments");
    if (n == 0) return FS_OK;
    if (!state || !vcmd || !att_out || state_stride < n || vcmd_stride < n || att_stride < n)
        return fail(FS_EINVAL, "bad buffers");
    fs_step_desc d;
    memset(&d, 0, sizeof(d));
    d.n = n;
    d.state_in = state;
    d.state_in_stride = state_stride;
    d.cmd = const_cast<float*>(vcmd);
    d.cmd_stride = vcmd_stride;
    fs::KParams P;
    fill_params(P, &d, robot, gains, limits, nullptr);
    fs::velocity_control_kernel<<<grid1(n), fs::kThreads, 0, (cudaStream_t)stream>>>(
        P, att_out, att_stride, degenerate_out);
    return check_launch("velocity_control_kernel");
}

int fs_attitude_control(int64_t n, const float* state, int64_t state_stride, const float* acmd,
                        int64_t acmd_stride, const fs_robot* robot, const fs_gains* gains,
                        float* wrench_out, int64_t wrench_stride, void* stream) {
    fs_limits l = {0.6, 5.0, 3.0};
    fs_step_desc d;
    memset(&d, 0, sizeof(d));
    d.n = n;
    d.state_in = state;
    d.state_in_stride = state_stride;
    d.cmd = const_cast<float*>(acmd);
    d.cmd_stride = acmd_stride;
    d.mode = FS_MODE_ATTITUDE;
    d.integrate = 0;
    d.wrench_out = wrench_out;
    d.wrench_stride = wrench_stride;
    if (!wrench_out && n > 0) return fail(FS_EINVAL, "wrench_out required");
    return fs_step(&d, robot, gains, &l, nullptr, stream);
}

int fs_yaw_of(int64_t n, const float* q, int64_t q_stride, double gimbal_cos, float* yaw_out,
              uint8_t* gimbal_out, void* stream) {
    if (n < 0) return fail(FS_EINVAL, "length must be >= 0");
    if (n == 0) return FS_OK;
    if (!q || q_stride < n) return fail(FS_EINVAL, "bad quaternion buffer");
    fs::yaw_kernel<<<grid1(n), fs::kThreads, 0, (cudaStream_t)stream>>>(n, q, q_stride, gimbal_cos,
                                                                       yaw_out, gimbal_out);
    return check_launch("yaw_kernel");
}

int fs_desired_attitude(int64_t n, const float* yaw, const float* acmd, int64_t acmd_stride,
                        float* qd_out, int64_t qd_stride, float* wd_out, int64_t wd_stride,
                        void* stream) {
    if (n < 0) return fail(FS_EINVAL, "length must be >= 0");
    if (n == 0) return FS_OK;
    if (!yaw || !acmd || !qd_out || !wd_out || acmd_stride < n || qd_stride < n || wd_stride < n)
        return fail(FS_EINVAL, "bad buffers");
    fs::desired_kernel<<<grid1(n), fs::kThreads, 0, (cudaStream_t)stream>>>(
        n, yaw, acmd, acmd_stride, qd_out, qd_stride, wd_out, wd_stride);
    return check_launch("desired_kernel");
}

int fs_attitude_errors(int64_t n, const float* q, int64_t q_stride, const float* omega,
                       int64_t omega_stride, const float* qd, int64_t qd_stride, const float* wd,
                       int64_t wd_stride, float* erot_out, float* erate_out, int64_t err_stride,
                       void* stream) {
    if (n < 0) return fail(FS_EINVAL, "length must be >= 0");
    if (n == 0) return FS_OK;
    if (!q || !omega || !qd || !wd || !erot_out || !erate_out || q_stride < n ||
        omega_stride < n || qd_stride < n || wd_stride < n || err_stride < n)
        return fail(FS_EINVAL, "bad buffers");
    fs::errors_kernel<<<grid1(n), fs::kThreads, 0, (cudaStream_t)stream>>>(
        n, q, q_stride, omega, omega_stride, qd, qd_stride, wd, wd_stride, erot_out, erate_out,
        err_stride);
    return check_launch("errors_kernel");
}

int fs_init_fleet(int64_t n, int64_t first_id, uint64_t seed, int32_t mode, float* state,
                  int64_t state_stride, float* cmd, int64_t cmd_stride, float* vparams,
                  int64_t vparams_stride, const fs_robot* robot, void* stream) {
    if (!robot || n < 0) return fail(FS_EINVAL, "bad arguments");
    if (mode < FS_MODE_ATTITUDE || mode > FS_MODE_POSITION) return fail(FS_EINVAL, "bad mode");
    if (n == 0) return FS_OK;
    if ((state && state_stride < n) || (cmd && cmd_stride < n) || (vparams && vparams_stride < n))
        return fail(FS_EINVAL, "plane stride shorter than length");
    fs::init_fleet_kernel<<<grid1(n), fs::kThreads, 0, (cudaStream_t)stream>>>(
        n, first_id, seed, mode, state, state_stride, cmd, cmd_stride, vparams, vparams_stride,
        (float)robot->mass, (float)robot->gravity, (float)robot->inertia[0],
        (float)robot->inertia[4], (float)robot->inertia[8]);
    return check_launch("init_fleet_kernel");
}

int fs_stats_reduce(const int64_t* slots, int32_t nslots, int64_t* out, void* stream) {
    if (!slots || !out || nslots <= 0) return fail(FS_EINVAL, "bad arguments");
    fs::stats_reduce_kernel<<<1, fs::kThreads, 0, (cudaStream_t)stream>>>(slots, nslots, out);
    return check_launch("stats_reduce_kernel");
}

}  // extern "C"

// ---- host-side layout conversion (fs_host_pack_f64 / fs_host_unpack_f64) ----
namespace {
template <class F>
void host_parallel(int64_t n, int32_t nthreads, F&& body) {
    int t = nthreads > 0 ? nthreads : (int)std::thread::hardware_concurrency();
    if (t < 1) t = 1;
    // at least 64K elements per thread: below that the spawn costs more
    const int64_t per_min = 1 << 16;
    if ((int64_t)t * per_min > n) t = (int)std::max<int64_t>(1, n / per_min);
    if (t == 1) {
        body(0, n);
        return;
    }
    std::vector<std::thread> th;
    th.reserve(t);
    int64_t done = 0;           // [0, done) is covered by started threads
    try {
        for (int k = 0; k < t; ++k) {
            const int64_t a = n * k / t, b = n * (k + 1) / t;
            th.emplace_back([=, &body] { body(a, b); });
            done = b;
        }
    } catch (...) {
        // (no more threads available: the caller's thread does the rest)
    }
    if (done < n) body(done, n);
    for (auto& x : th) x.join();
}
}  // namespace

extern "C" int fs_host_pack_f64(const double* src, int64_t n, int32_t w, int64_t ld, float* dst,
                                int64_t plane_stride, int32_t nthreads) {
    if (n < 0 || w < 1 || ld < w || plane_stride < n || (n > 0 && (!src || !dst)))
        return fail(FS_EINVAL, "fs_host_pack_f64: bad sizes or null pointers");
    host_parallel(n, nthreads, [&](int64_t a, int64_t b) {
        for (int k = 0; k < w; ++k) {
            float* o = dst + k * plane_stride;
            const double* s = src + k;
            for (int64_t i = a; i < b; ++i) o[i] = (float)s[i * ld];
        }
    });
    return FS_OK;
}

extern "C" int fs_host_unpack_f64(const float* src, int64_t plane_stride, int64_t n, int32_t w,
                                  double* dst, int64_t ld, int32_t nthreads) {
    if (n < 0 || w < 1 || ld < w || plane_stride < n || (n > 0 && (!src || !dst)))
        return fail(FS_EINVAL, "fs_host_unpack_f64: bad sizes or null pointers");
    host_parallel(n, nthreads, [&](int64_t a, int64_t b) {
        for (int64_t i = a; i < b; ++i) {
            double* o = dst + i * ld;
            for (int k = 0; k < w; ++k) o[k] = (double)src[k * plane_stride + i];
        }
    });
    return FS_OK;
}

