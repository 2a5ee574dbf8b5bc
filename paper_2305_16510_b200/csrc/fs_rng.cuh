// fs_rng.cuh -- counter-based Philox4x32-10 and the fleet "spawn" draw.
//
// EXTENSION (no reference counterpart): the reference draws obstacles and
// spawns from per-(seed, env, reset) NumPy Philox streams
// (assets.py:310-315, world.py:229-243).  Here one spawn is a pure function
// of (seed, global vehicle id, step counter), so 1/2/4/8-GPU shardings of a
// fleet produce bitwise-identical vehicles, and the CPU twin
// (oracle/rng_twin.py) regenerates any vehicle exactly.
//
// Counter layout: (gid_lo, gid_hi, step, block).  step = 0xFFFFFFFF is the
// initial spawn; step = k is the re-spawn at control step k (BASELINE
// config 3).  The per-step re-spawn decision itself uses a cheaper
// counter-based hash evaluated for every vehicle every step (reset_word: a
// per-step 32-bit key -- splitmix64 of seed and step, loop-invariant, so the
// compiler hoists it out of the vehicle loop -- xor the global id, through
// one lowbias32 round: ~7 instructions per vehicle).
//
// Blocks: 0 = (mask, px, py, pz); 1 = (q u1, u2, u3, cmd a); 2 = (cmd b, c, d,
// -); 3, 4 = Box-Muller pairs for v, w and velocity-command x, y; 5 = vehicle
// parameters; 6 = Box-Muller pair for the velocity-command z.
//
// Word -> float: u = (w >> 8) * 2^-24, exact in fp32.  Affine maps use
// explicitly rounded fp32 ops (__fmul_rn/__fadd_rn) so that the CPU twin in
// numpy float32 is bit-exact.  Normals (Box-Muller) and the Shoemake
// quaternion use libm-class functions and agree with the twin to ~1 ulp.
#pragma once

#include <stdint.h>

namespace fs {

constexpr uint32_t kInitStep = 0xFFFFFFFFu;

__host__ __device__ __forceinline__ uint32_t mulhi32(uint32_t a, uint32_t b) {
#ifdef __CUDA_ARCH__
    return __umulhi(a, b);
#else
    return (uint32_t)(((uint64_t)a * (uint64_t)b) >> 32);
#endif
}

struct U4 {
    uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = mulhi32(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = mulhi32(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// Bernoulli(p) re-spawn word of vehicle gid at step: re-spawn iff word <
// floor(p * 2^32).
__host__ __device__ __forceinline__ uint32_t step_key(uint64_t seed, uint32_t step) {
    uint64_t x = seed ^ ((uint64_t)step * 0xD1B54A32D192ED03ull);
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    return (uint32_t)(x >> 32);
}

// lowbias32 (a 32-bit xorshift-multiply finalizer)
__host__ __device__ __forceinline__ uint32_t lowbias32(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7FEB352Du;
    x ^= x >> 15;
    x *= 0x846CA68Bu;
    x ^= x >> 16;
    return x;
}

// the word from a precomputed step key (hoist step_key out of vehicle loops)
__host__ __device__ __forceinline__ uint32_t reset_word_k(uint32_t key, int64_t gid) {
    const uint64_t g = (uint64_t)gid;
    return lowbias32((uint32_t)g ^ key ^ ((uint32_t)(g >> 32) * 0x85EBCA6Bu));
}

__host__ __device__ __forceinline__ uint32_t reset_word(uint64_t seed, int64_t gid,
                                                        uint32_t step) {
    return reset_word_k(step_key(seed, step), gid);
}

__device__ __forceinline__ U4 draw_block(uint64_t seed, int64_t gid, uint32_t step,
                                         uint32_t block) {
    return philox4x32_10(U4{(uint32_t)gid, (uint32_t)((uint64_t)gid >> 32), step, block},
                         (uint32_t)seed, (uint32_t)(seed >> 32));
}

__device__ __forceinline__ float u01(uint32_t w) {
    return (float)(w >> 8) * 5.9604644775390625e-8f;   // 2^-24
}

// lo + (hi - lo) * u with explicit rounding (bit-exact twin in float32)
__device__ __forceinline__ float uaff(uint32_t w, float lo, float span) {
    return __fadd_rn(lo, __fmul_rn(span, u01(w)));
}

__device__ __forceinline__ void box_muller(uint32_t w1, uint32_t w2, float& n0, float& n1) {
    const float u1 = (float)((w1 >> 8) + 1u) * 5.9604644775390625e-8f;   // (0, 1]
    const float u2 = u01(w2);
    const float r = sqrtf(-2.0f * logf(u1));
    float s, c;
    sincospif(2.0f * u2, &s, &c);
    n0 = r * c;
    n1 = r * s;
}

// The spawn of one vehicle: BASELINE.json config-0 state distributions
// (p ~ U[-5,5]^3, q uniform on S^3, v ~ N(0,1)^3, w ~ N(0, 0.5^2)^3) and the
// command distribution of `mode` (configs 1-4).
// cmd receives 4 planes (8 for MIXED: attitude then velocity).
__device__ __forceinline__ void spawn(uint64_t seed, int64_t gid, uint32_t step, int mode,
                                      float mass, float gravity, float* st, float* cmd) {
    const U4 b0 = draw_block(seed, gid, step, 0);
    const U4 b1 = draw_block(seed, gid, step, 1);
    const U4 b2 = draw_block(seed, gid, step, 2);
    const U4 b3 = draw_block(seed, gid, step, 3);
    const U4 b4 = draw_block(seed, gid, step, 4);
    st[0] = uaff(b0.y, -5.0f, 10.0f);
    st[1] = uaff(b0.z, -5.0f, 10.0f);
    st[2] = uaff(b0.w, -5.0f, 10.0f);
    // Shoemake: q = (b cos t2, a sin t1, a cos t1, b sin t2)
    {
        const float u1 = u01(b1.x);
        const float a = sqrtf(1.0f - u1), b = sqrtf(u1);
        float s1, c1, s2, c2;
        sincospif(2.0f * u01(b1.y), &s1, &c1);
        sincospif(2.0f * u01(b1.z), &s2, &c2);
        float qw = b * c2, qx = a * s1, qy = a * c1, qz = b * s2;
        const float iq = rsqrtf(qw * qw + qx * qx + qy * qy + qz * qz);
        st[3] = qw * iq;
        st[4] = qx * iq;
        st[5] = qy * iq;
        st[6] = qz * iq;
    }
    float n[8];
    box_muller(b3.x, b3.y, n[0], n[1]);
    box_muller(b3.z, b3.w, n[2], n[3]);
    box_muller(b4.x, b4.y, n[4], n[5]);
    box_muller(b4.z, b4.w, n[6], n[7]);
    st[7] = n[0];
    st[8] = n[1];
    st[9] = n[2];
    st[10] = 0.5f * n[3];
    st[11] = 0.5f * n[4];
    st[12] = 0.5f * n[5];
    if (mode == FS_MODE_ATTITUDE || mode == FS_MODE_MIXED) {
        cmd[0] = uaff(b1.w, -0.5f, 1.0f);                          // roll
        cmd[1] = uaff(b2.x, -0.5f, 1.0f);                          // pitch
        cmd[2] = uaff(b2.y, -1.0f, 2.0f);                          // yaw rate
        cmd[3] = __fmul_rn(uaff(b2.z, 0.5f, 1.0f), __fmul_rn(mass, gravity));  // thrust
    }
    if (mode == FS_MODE_VELOCITY || mode == FS_MODE_MIXED) {
        float* vc = (mode == FS_MODE_MIXED) ? cmd + 4 : cmd;
        vc[0] = n[6];
        vc[1] = n[7];
        const U4 b6 = draw_block(seed, gid, step, 6);
        float n8, n9;
        box_muller(b6.x, b6.y, n8, n9);
        vc[2] = n8;
        vc[3] = uaff(b2.y, -1.0f, 2.0f);                           // yaw rate
    }
    if (mode == FS_MODE_POSITION) {
        cmd[0] = uaff(b1.w, -5.0f, 10.0f);
        cmd[1] = uaff(b2.x, -5.0f, 10.0f);
        cmd[2] = uaff(b2.z, -5.0f, 10.0f);
        cmd[3] = uaff(b2.y, -3.14159274f, 6.28318548f);            // yaw setpoint
    }
}

// Per-vehicle parameter scaling for the heterogeneous fleet (config 4):
// mass and each diagonal inertia entry scaled by independent U[0.8, 1.2].
__device__ __forceinline__ void spawn_vparams(uint64_t seed, int64_t gid, float mass,
                                              float jxx, float jyy, float jzz, float* vp) {
    const U4 b = draw_block(seed, gid, kInitStep, 5);
    vp[0] = __fmul_rn(mass, uaff(b.x, 0.8f, 0.4f));
    vp[1] = __fmul_rn(jxx, uaff(b.y, 0.8f, 0.4f));
    vp[2] = __fmul_rn(jyy, uaff(b.z, 0.8f, 0.4f));
    vp[3] = __fmul_rn(jzz, uaff(b.w, 0.8f, 0.4f));
}

}  // namespace fs
