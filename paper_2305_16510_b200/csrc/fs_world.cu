// fs_world.cu -- free-space World.step on the GPU.
//
// One thread per environment (planar, coalesced loads/stores):
//   pending -> auto-reset: counter++, re-spawn at rest + new goal, step voided
//              (world.py:287-299), reward 0, info AUTORESET;
//   else    -> the fused control step (fs_math.cuh vehicle_step), collision
//              against the env box (world.py:95-106: no primitives in free
//              space), steps++, terminated = collided | nonfinite, truncated
//              = steps >= max & !terminated (world.py:308-312), reward
//              (world.py:109-116), pending = terminated | truncated;
//   always  -> 16-value observation (world.py:331-342).
// fs_vecenv_step feeds the same kernel from RL
// actions instead of command planes: flocksim_rl VecEnvHandle.step's clip to
// [-1, 1] and denormalization (vec_env.py:85-104) run in float64 on the
// loaded action row and the float64 commands go straight into the controller.
// Reward, collision test and observation frame rotation evaluate in float64
// from the fp32 state (exact products), rounded once.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>

#include "flocksim_b200.h"
#include "fs_math.cuh"
#include "fs_rng.cuh"
#include "fs_scene.cuh"
#include "fs_step.cuh"

namespace fs {

extern int g_world_kernel;   // FS_TUNE_WORLD_KERNEL (fs_kernels.cu)
extern int g_clear_walk_cm;  // FS_TUNE_CLEAR_WALK_CM
extern int g_clear_exact;    // FS_TUNE_CLEAR_EXACT

struct WorldParams {
    fs_world_desc w;
    float bounds[3];
    float lo_spawn[3], span_spawn[3], lo_goal[3], span_goal[3];
    float r;                       // collision radius (fp32 placement test)
    double bounds_d[3], r_d;
    int32_t max_steps, attempts;
    double c_dist, c_vel, c_step, c_success, c_crash, success_radius;
    const uint8_t* mask;
    int32_t increment;
    // fs_vecenv_step: (E, 4) action rows, row stride in elements (NULL: the
    // command planes); act_f64: float64 rows
    const void* actions;
    int64_t action_stride;
    int32_t act_f64;
    double act_scale[4];           // per-component denormalization scale
    // obstacle scene; has_ob == 0 in free space
    fs_obstacles ob;
    int32_t has_ob;
    float clear_walk;              // clearance-cache slot-walk radius, m
    int32_t clear_exact;           // walked slots bound the clearance by their exact SDF
    // host-computed plane bases of the state and observation outputs: a store
    // is base + i (no per-plane 64-bit stride arithmetic in the kernels)
    float* state_plane[13];
    float* obs_plane[16];
};

// Action element loads: one 16-B vector (f32) or two (f64) per env.
__device__ __forceinline__ void load_action(const float* a, double (&x)[4]) {
    const float4 v = __ldg(reinterpret_cast<const float4*>(a));
    x[0] = f2d(v.x);
    x[1] = f2d(v.y);
    x[2] = f2d(v.z);
    x[3] = f2d(v.w);
}
__device__ __forceinline__ void load_action(const double* a, double (&x)[4]) {
    const double2 u = __ldg(reinterpret_cast<const double2*>(a));
    const double2 v = __ldg(reinterpret_cast<const double2*>(a) + 1);
    x[0] = u.x;
    x[1] = u.y;
    x[2] = v.x;
    x[3] = v.y;
}

// vec_env.py:91-104: a = clip(actions, -1, 1) (NaN passes through, like
// np.clip); attitude: (a0 max_tilt, a1 max_tilt, a2 max_yaw_rate,
// (a3 + 1) / 2 thrust_max); velocity: (a0..a2 max_speed_cmd, a3 max_yaw_rate).
// Same float64 operations in the same order as the reference.
template <int MODE>
__device__ __forceinline__ void denorm_actions(const WorldParams& W, const double (&a)[4],
                                               double (&cmd)[4]) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const double x = a[k] < -1.0 ? -1.0 : (a[k] > 1.0 ? 1.0 : a[k]);
        cmd[k] = x * W.act_scale[k];
    }
    if (MODE == FS_MODE_ATTITUDE) {
        const double x = a[3] < -1.0 ? -1.0 : (a[3] > 1.0 ? 1.0 : a[3]);
        cmd[3] = (x + 1.0) / 2.0 * W.act_scale[3];
    }
}

template <int MODE, typename AT>
__device__ __forceinline__ void action_commands(const WorldParams& W, int64_t i,
                                                double (&cmd)[4]) {
    double a[4];
    load_action(static_cast<const AT*>(W.actions) + i * W.action_stride, a);
    denorm_actions<MODE>(W, a, cmd);
}

constexpr uint32_t kPlaceBlock = 0x100;   // Philox block ids of the placement draws

// One placement (world.py:196-211): p = (lo + u (hi - lo)) * bounds, accepted
// when r <= p <= bounds - r and (with obstacles) every collision-enabled
// primitive of env i is at least r away; up to `attempts` draws, block
// kPlaceBlock + 2a (+1 for the goal).  fp32 with explicit rounding: bit-exact
// CPU twin.
__device__ __forceinline__ bool place(const WorldParams& W, int64_t i, uint64_t seed, int64_t gid,
                                      uint32_t counter, bool goal, float* p) {
    const float* lo = goal ? W.lo_goal : W.lo_spawn;
    const float* span = goal ? W.span_goal : W.span_spawn;
    for (int a = 0; a < W.attempts; ++a) {
        const U4 b = draw_block(seed, gid, counter, kPlaceBlock + 2 * a + (goal ? 1 : 0));
        const uint32_t wv[3] = {b.x, b.y, b.z};
        bool ok = true;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            p[k] = __fmul_rn(__fadd_rn(lo[k], __fmul_rn(u01(wv[k]), span[k])), W.bounds[k]);
            ok &= (p[k] >= W.r) && (p[k] <= __fsub_rn(W.bounds[k], W.r));
        }
        if (ok && W.has_ob)
            ok = !scene_hit(W.ob.scene, i, f2d(p[0]), f2d(p[1]), f2d(p[2]), W.r_d);
        if (ok) return true;
    }
    return false;
}

// the observation's goal part: R_z(yaw)^T (goal - p) in float64, rounded once
__device__ __forceinline__ void obs_goal(const VState& s, const float* goal, float (&gb)[3]) {
    const Rot<double> R = rotmat<double>(s.q[0], s.q[1], s.q[2], s.q[3]);
    double cy, sy;
    yaw_cs(R, cy, sy);
    const double gx = f2d(goal[0]) - f2d(s.p[0]), gy = f2d(goal[1]) - f2d(s.p[1]);
    const double gz = f2d(goal[2]) - f2d(s.p[2]);
    gb[0] = d2f(cy * gx + sy * gy);
    gb[1] = d2f(-sy * gx + cy * gy);
    gb[2] = d2f(gz);
}

// observation: p, q, v, w, R_z(yaw)^T (goal - p)  (world.py:331-342)
__device__ __forceinline__ void write_obs(const WorldParams& W, int64_t i, const VState& s,
                                          const float* goal) {
    float* const* o = W.obs_plane;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        o[k][i] = s.p[k];
        o[7 + k][i] = s.v[k];
        o[10 + k][i] = s.w[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) o[3 + k][i] = s.q[k];
    float gb[3];
    obs_goal(s, goal, gb);
    o[13][i] = gb[0];
    o[14][i] = gb[1];
    o[15][i] = gb[2];
}

__device__ __forceinline__ void load_state(const fs_step_desc& d, int64_t i, VState& s) {
    const float* S = d.state_in + i;
    const int64_t ss = d.state_in_stride;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        s.p[k] = S[k * ss];
        s.v[k] = S[(7 + k) * ss];
        s.w[k] = S[(10 + k) * ss];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) s.q[k] = S[(3 + k) * ss];
}

__device__ __forceinline__ void store_state(const WorldParams& W, int64_t i, const VState& s) {
    float* const* S = W.state_plane;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        S[k][i] = s.p[k];
        S[7 + k][i] = s.v[k];
        S[10 + k][i] = s.w[k];
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) S[3 + k][i] = s.q[k];
}

// re-spawn env i at counter c (world.py:229-243): fresh obstacle poses when
// the world has obstacles, then the robot at rest at the spawn, the goal
// (world.py:213-227), and the camera mount
__device__ __forceinline__ uint32_t respawn_env(const WorldParams& W, int64_t i, uint32_t c,
                                                VState& s, float* goal) {
    const fs_step_desc& d = W.w.step;
    const int64_t gid = d.first_id + i;
    if (W.has_ob) rebuild_env(W.ob, i, d.seed, gid, c, W.bounds_d);
    float sp[3];
    const bool ok1 = place(W, i, d.seed, gid, c, false, sp);
    const bool ok2 = place(W, i, d.seed, gid, c, true, goal);
    if (W.has_ob && W.ob.mount) randomize_mount_d(W.ob, i, d.seed, gid, c);
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        s.p[k] = sp[k];
        s.v[k] = 0.0f;
        s.w[k] = 0.0f;
    }
    s.q[0] = 1.0f;
    s.q[1] = s.q[2] = s.q[3] = 0.0f;
    return (ok1 && ok2) ? 0u : (uint32_t)FS_INFO_PLACEMENT_FAILED;
}

// reward_goal_reaching (world.py:109-116) in float64 from the fp32 state, rounded once
__device__ __forceinline__ float world_reward(const WorldParams& W, const VState& s,
                                              const float* goal, bool collided) {
    const double gx = f2d(goal[0]) - f2d(s.p[0]), gy = f2d(goal[1]) - f2d(s.p[1]);
    const double gz = f2d(goal[2]) - f2d(s.p[2]);
    const double dist = sqrt(gx * gx + gy * gy + gz * gz);
    const double vx = f2d(s.v[0]), vy = f2d(s.v[1]), vz = f2d(s.v[2]);
    const double speed = sqrt(vx * vx + vy * vy + vz * vz);
    const double r = -dist * W.c_dist - speed * W.c_vel - W.c_step +
                     (dist < W.success_radius ? W.c_success : 0.0) -
                     (collided ? W.c_crash : 0.0);
    return d2f(r);
}

// the clearance-cache test (fs_obstacles.clear): true when the robot at p
// moved less than c - r from the point of the last broad phase, so it is
// farther than r from every collision-enabled instance box (fp32 margins:
// |dp| and c carry < 1e-6 relative rounding)
// (clr: the env's 4 cache values already loaded, else read from global memory)
__device__ __forceinline__ bool clear_cached(const WorldParams& W, int64_t i, const float* p,
                                             const float* clr = nullptr) {
    float cx, cy, cz, cc;
    if (clr) {
        cx = clr[0], cy = clr[1], cz = clr[2], cc = clr[3];
    } else {
        const int64_t ps = W.ob.plane_stride;
        const float* cl = W.ob.clear + i;
        cx = cl[0], cy = cl[ps], cz = cl[2 * ps], cc = cl[3 * ps];
    }
    const float dx = p[0] - cx, dy = p[1] - cy, dz = p[2] - cz;
    const float dpp = sqrtf(dx * dx + dy * dy + dz * dz);
    const float rr = W.r * 1.0001f + 1e-5f;
    return dpp + rr < cc * 0.99999f - 1e-6f;
}

// instances within W.clear_walk metres (FS_TUNE_CLEAR_WALK_CM, default 1 m)
// are walked slot by slot when the cache is refreshed: their primitives'
// boxes bound the clearance, not the instance box

// the full primitive test at p with the cache refreshed
__device__ __forceinline__ bool scene_test_refresh(const WorldParams& W, int64_t i,
                                                   const float* p) {
    float cmin = -1.0f;
    const bool hit = scene_hit_inst<true>(W.ob, i, f2d(p[0]), f2d(p[1]), f2d(p[2]), W.r_d, &cmin,
                                          W.clear_walk);
    const int64_t ps = W.ob.plane_stride;
    float* cl = W.ob.clear + i;
    cl[0] = p[0];
    cl[ps] = p[1];
    cl[2 * ps] = p[2];
    cl[3 * ps] = hit ? -1.0f : cmin;
    return hit;
}

// append env i to the deferred-collision worklist (warp-aggregated atomic)
__device__ __forceinline__ void worklist_push(int32_t* wl, int64_t i) {
    const unsigned m = __activemask();
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    const int rank = __popc(m & ((1u << lane) - 1u));
    int base = 0;
    if (lane == leader) base = atomicAdd(wl, __popc(m));
    base = __shfl_sync(m, base, leader);
    wl[3 + base + rank] = (int32_t)i;
}

// One env's World.step (world.py:277-342) on its loaded inputs: state s,
// goal, episode counter `steps`, `pending` (in: auto-reset due; out: the
// next step's) and the float64 commands (from the command planes or RL
// action rows; unused when the env resets).  Writes only the reset path's
// goal and counter to global memory; the caller stores the outputs.
// SCENE: the world has obstacles (primitive collision test; the auto-reset
// already ran in world_reset_warp_kernel<true>); 1: the test inline, with the
// clearance cache when the world has one; 2: deferred -- envs the cache does
// not clear go to the worklist and scene_fix_kernel finishes them.
template <int MODE, int PREC, int SCENE>
__device__ __forceinline__ void world_env_step(const KParams& P, const WorldParams& W, int64_t i,
                                               VState& s, float* goal, int32_t& steps,
                                               bool& pending, uint32_t vmode,
                                               const double (&cmd)[cmd_planes<MODE>()],
                                               float& reward, uint32_t& info,
                                               const float* clr = nullptr,
                                               bool* need_test = nullptr) {
    constexpr int NC = cmd_planes<MODE>();
    if (pending) {
        // world.py:287-289 + 293-299: reset first, the step is voided
        if constexpr (SCENE) {
            // world_reset_warp_kernel<true> ran just before on this stream:
            // fresh obstacles, spawn, goal, counter and the info bits
            info = W.w.info[i];
        } else {
            const uint32_t c = (uint32_t)(W.w.reset_counter[i] + 1);
            W.w.reset_counter[i] = (int32_t)c;
            info = FS_INFO_AUTORESET | respawn_env(W, i, c, s, goal);
#pragma unroll
            for (int k = 0; k < 3; ++k) W.w.goal[k * W.w.goal_stride + i] = goal[k];
        }
        steps = 0;
        reward = 0.0f;
        pending = false;
        return;
    }
    const float vp[4] = {0.f, 0.f, 0.f, 0.f};
    StepOut o;
    vehicle_step<MODE, false, PREC, kFeatStats, double>(s, cmd, vmode, vp, 0, P, true, o);
    // collision with the env box (world.py:103-106), float64 bounds
    bool oob = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double pk = f2d(s.p[k]);
        oob |= (pk < W.r_d) || (pk > W.bounds_d[k] - W.r_d);
    }
    // ... and with the primitives (world.py:100: min_distance < r)
    bool hit = false;
    if constexpr (SCENE == 2) {
        // out of bounds already collides; otherwise the cache or the worklist
        // (need_test: the caller collects the misses itself)
        const bool miss = !oob && !clear_cached(W, i, s.p, clr);
        if (need_test)
            *need_test = miss;
        else if (miss)
            worklist_push(W.ob.worklist, i);
    } else if constexpr (SCENE == 1) {
        if (W.ob.clear && W.ob.inst_box) {
            if (!clear_cached(W, i, s.p)) hit = scene_test_refresh(W, i, s.p);
        } else {
            hit = scene_hit_inst(W.ob, i, f2d(s.p[0]), f2d(s.p[1]), f2d(s.p[2]), W.r_d);
        }
    }
    const bool collided = hit || oob;
    const bool nonfinite = (o.flags & FS_FLAG_NONFINITE) != 0;
    steps += 1;
    const bool term = collided || nonfinite;
    const bool trunc = (steps >= W.max_steps) && !term;
    reward = world_reward(W, s, goal, collided);     // (world.py:109-116)
    pending = term || trunc;
    info = (term ? FS_INFO_TERMINATED : 0u) | (trunc ? FS_INFO_TRUNCATED : 0u) |
           (collided ? FS_INFO_COLLISION : 0u) | (oob ? FS_INFO_OUT_OF_BOUNDS : 0u) |
           (nonfinite ? FS_INFO_NONFINITE : 0u);
}

__device__ __forceinline__ void store_world_outputs(const WorldParams& W, int64_t i,
                                                    const VState& s, const float* goal,
                                                    int32_t steps, bool pending, float reward,
                                                    uint32_t info) {
    store_state(W, i, s);
    W.w.steps_in_episode[i] = steps;
    W.w.pending_reset[i] = pending ? 1 : 0;
    W.w.reward[i] = reward;
    W.w.info[i] = (uint8_t)info;
    write_obs(W, i, s, goal);
}

// Thread-per-env World.step (obstacle worlds; unaligned or small batches).
// Commands come from the command planes or, for fs_vecenv_step, from the
// action rows (W.actions, float32 or float64): World.step and
// VecEnvHandle.step take the same kernel path on identical float64 command
// values (the transparency property of test_bindings.py:108-127 holds by
// construction).
template <int MODE, int PREC, int SCENE = 0>
__global__ void __launch_bounds__(256, SCENE == 1 ? 2 : 3) world_step_kernel(const __grid_constant__ KParams P,
                                                         const __grid_constant__ WorldParams W) {
    constexpr int NC = cmd_planes<MODE>();
    const fs_step_desc& d = W.w.step;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d.n) return;
    VState s;
    load_state(d, i, s);
    float goal[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) goal[k] = W.w.goal[k * W.w.goal_stride + i];
    int32_t steps = W.w.steps_in_episode[i];
    bool pending = W.w.pending_reset[i] != 0;
    const uint32_t vmode = (MODE == FS_MODE_MIXED && !pending) ? d.mode_per_vehicle[i] : 0u;
    double cmd[NC];
    bool planes = true;
    if constexpr (MODE != FS_MODE_MIXED) {
        if (W.actions) {
            planes = false;
            if (W.act_f64)
                action_commands<MODE, double>(W, i, cmd);
            else
                action_commands<MODE, float>(W, i, cmd);
        }
    }
    if (planes) {
#pragma unroll
        for (int k = 0; k < NC; ++k) cmd[k] = f2d(d.cmd[k * d.cmd_stride + i]);
    }
    float reward;
    uint32_t info;
    world_env_step<MODE, PREC, SCENE>(P, W, i, s, goal, steps, pending, vmode, cmd, reward, info);
    store_world_outputs(W, i, s, goal, steps, pending, reward, info);
}

// ---------------------------------------------------------------------------
// Streaming free-space World.step: the fs_step stream kernel's architecture
// (persistent, one CTA per SM, warp-specialized) for the World.  The load
// warp keeps STAGES tiles of every input in flight with 1-D TMA bulk copies
// (13 state planes, 3 goal planes, the command planes or the tile's action
// rows, the episode counters, the pending and mode bytes) into a shared ring;
// each consumer thread takes one env per tile from the ring, runs
// world_env_step and writes its outputs (state, observation, reward,
// counter, pending and info bytes) into a shared output tile; the store
// warp writes each output tile back with one TMA bulk store per plane (the
// 0..15 entries past the last 16-byte multiple of the final tile as plain
// stores).  Counters / flag bytes past the last 16-byte multiple of the
// final tile are read from global memory directly, so no buffer is read or
// written beyond n.
// ---------------------------------------------------------------------------
#ifndef FS_WORLD_NCW
#define FS_WORLD_NCW 14   // 16 warps: up to 128 registers, no spills (16 consumer warps spill: 181 vs 163 us)
#endif
constexpr int kWorldNCW = FS_WORLD_NCW;   // consumer warps (+ load + store warps)
constexpr int kWorldOutPlanes = 31;   // 13 state + 16 obs + reward + counter (4-byte planes)

template <int MODE>
__host__ __device__ constexpr int world_stage_bytes(int T) {
    // state + goal planes, commands (planes or rows: up to 32 B / env), steps,
    // pending, mode (reserved), the 4 clearance-cache planes (obstacle worlds)
    return (16 * 4 + 32 + 4 + 1 + 1 + 16) * T;
}

__host__ __device__ constexpr int world_out_bytes(int T) {
    return kWorldOutPlanes * 4 * T + 2 * T;   // + pending, info bytes
}

// SC: 0 free space; 2 an obstacle world with the deferred collision test
// (the clearance cache per env, misses to the worklist; world_env_step).
// The skipped-env list (fs_obstacles.reset_list, n + 4 int32): [0] count,
// [3] next entry to take, [4..] env ids.  With it the streaming step DEFERS
// the auto-resets: it skips every env that is pending when the step starts
// (its step is voided) and lists it, and world_post_kernel resets the listed
// envs after the step, writing every output of the reset.  The list is
// filled and emptied within one step.

template <int MODE, int PREC, int STAGES, int OSTAGES, int SC = 0>
__global__ void __launch_bounds__((kWorldNCW + 2) * 32, 1)
    world_stream_kernel(const __grid_constant__ KParams P, const __grid_constant__ WorldParams W) {
    constexpr int NCW = kWorldNCW;
    constexpr int T = 32 * NCW;
    constexpr int NC = cmd_planes<MODE>();
    constexpr bool MIX = MODE == FS_MODE_MIXED;
    constexpr int SB = world_stage_bytes<MODE>(T);
    constexpr int OB = world_out_bytes(T);
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);     // [STAGES]
    uint64_t* empty = full + STAGES;                         // [STAGES]
    uint64_t* ofull = empty + STAGES;                        // [OSTAGES]
    uint64_t* oempty = ofull + OSTAGES;                      // [OSTAGES]
    static_assert((2 * STAGES + 2 * OSTAGES) * 8 + 8 * OSTAGES <= 128, "mbarrier region");
    // SC == 2: per output stage, the count and the env ids of the tile's
    // collision-test misses; the store lane appends them to the global
    // worklist with ONE atomic per tile
    int* pcount = reinterpret_cast<int*>(smem + (2 * STAGES + 2 * OSTAGES) * 8);  // [OSTAGES]
    int* rcount = pcount + OSTAGES;     // [OSTAGES] the tile's envs left pending (reset list)
    unsigned char* ring = smem + 128;
    unsigned char* otiles = ring + (size_t)STAGES * SB;     // [OSTAGES][OB]
    int* plist = reinterpret_cast<int*>(otiles + (size_t)OSTAGES * OB);   // [OSTAGES][T] (SC == 2)
    int* rlist = plist + (size_t)OSTAGES * T;                              // [OSTAGES][T] (SC == 2)
    // deferred auto-resets (SC == 2 with the list): pending envs are skipped
    // -- their step is voided and world_post_kernel writes every output of
    // their reset after this kernel -- and listed for it
    const bool rl = SC == 2 && W.ob.reset_list != nullptr;
    const fs_step_desc& d = W.w.step;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const bool rows = W.actions != nullptr;
    const int row_bytes = W.act_f64 ? 32 : 16;
    // stage layout (byte offsets)
    constexpr int O_CMD = 16 * T * 4;
    constexpr int O_STEPS = O_CMD + 32 * T, O_PEND = O_STEPS + 4 * T, O_MODE = O_PEND + T;
    constexpr int O_CLR = O_MODE + T;      // 4 fp32 planes (SC == 2)
    static_assert(O_CLR % 16 == 0, "16-byte aligned TMA destinations");
    // output tile layout: 31 four-byte planes, then the pending and info bytes
    constexpr int P_REWARD = 29, P_STEPS = 30, OB_PEND = kWorldOutPlanes * 4 * T;

    if (threadIdx.x == 0) {
        for (int st = 0; st < STAGES; ++st) {
            mbar_init(&full[st], 1);
            mbar_init(&empty[st], NCW);
        }
        for (int os = 0; os < OSTAGES; ++os) {
            mbar_init(&ofull[os], NCW);
            mbar_init(&oempty[os], 1);
            pcount[os] = 0;
            rcount[os] = 0;
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NCW) {
        // ------------------------------ load warp ----------------------------
        if (lane == 0) {
            const uint64_t pol = evict_first_policy();
            int it = 0;
            for (VTiles V(d.n, T, 1); V.valid(); V.next(), ++it) {
                const int64_t i0 = V.i0();
                const int cnt = V.cnt();
                const int st = it % STAGES;
                mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1);
                const uint32_t fb = (uint32_t)((cnt * 4 + 15) & ~15);   // float planes
                const uint32_t ib = (uint32_t)((cnt & ~3) * 4);         // int32 counters
                const uint32_t bb = (uint32_t)(cnt & ~15);              // byte flags
                const uint32_t cb = rows ? (uint32_t)(cnt * row_bytes) : NC * fb;
                mbar_expect_tx(&full[st],
                               (16 + (SC == 2 ? 4 : 0)) * fb + cb + ib + bb + (MIX ? bb : 0u));
                unsigned char* sl = ring + (size_t)st * SB;
                float* sf = reinterpret_cast<float*>(sl);
#pragma unroll
                for (int k = 0; k < kStatePlanes; ++k)
                    bulk_g2s(sf + k * T, d.state_in + k * d.state_in_stride + i0, fb, &full[st],
                             pol);
#pragma unroll
                for (int k = 0; k < 3; ++k)
                    bulk_g2s(sf + (13 + k) * T, W.w.goal + k * W.w.goal_stride + i0, fb,
                             &full[st], pol);
                if (rows) {
                    bulk_g2s(sl + O_CMD,
                             static_cast<const unsigned char*>(W.actions) + i0 * row_bytes, cb,
                             &full[st], pol);
                } else {
#pragma unroll
                    for (int k = 0; k < NC; ++k)
                        bulk_g2s(sl + O_CMD + k * T * 4, d.cmd + k * d.cmd_stride + i0, fb,
                                 &full[st], pol);
                }
                if (ib) bulk_g2s(sl + O_STEPS, W.w.steps_in_episode + i0, ib, &full[st], pol);
                if (bb) bulk_g2s(sl + O_PEND, W.w.pending_reset + i0, bb, &full[st], pol);
                if (MIX && bb) bulk_g2s(sl + O_MODE, d.mode_per_vehicle + i0, bb, &full[st], pol);
                if constexpr (SC == 2) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        bulk_g2s(sl + O_CLR + k * T * 4, W.ob.clear + k * W.ob.plane_stride + i0,
                                 fb, &full[st], pol);
                }
            }
        }
        return;
    }
    if (warp == NCW + 1) {
        // ------------------------------ store warp ---------------------------
        if (lane == 0) {
            const uint64_t pol = evict_first_policy();
            int it = 0;
            for (VTiles V(d.n, T, 1); V.valid(); V.next(), ++it) {
                const int64_t i0 = V.i0();
                const int cnt = V.cnt();
                const int os = it % OSTAGES;
                mbar_wait(&ofull[os], (it / OSTAGES) & 1);
                const unsigned char* ot = otiles + (size_t)os * OB;
                const float* of = reinterpret_cast<const float*>(ot);
                const int c4 = cnt & ~3, c16 = cnt & ~15;
                if (c4 > 0) {
                    const uint32_t fb = (uint32_t)c4 * 4u;
#pragma unroll
                    for (int k = 0; k < kStatePlanes; ++k)
                        bulk_s2g(W.state_plane[k] + i0, of + k * T, fb, pol);
#pragma unroll
                    for (int k = 0; k < 16; ++k)
                        bulk_s2g(W.obs_plane[k] + i0, of + (13 + k) * T, fb, pol);
                    bulk_s2g(W.w.reward + i0, of + P_REWARD * T, fb, pol);
                    bulk_s2g(W.w.steps_in_episode + i0, of + P_STEPS * T, fb, pol);
                }
                if (c16 > 0) {
                    bulk_s2g(W.w.pending_reset + i0, ot + OB_PEND, (uint32_t)c16, pol);
                    bulk_s2g(W.w.info + i0, ot + OB_PEND + T, (uint32_t)c16, pol);
                }
                // the final tile's tail: plain stores, nothing beyond n
                for (int c = c4; c < cnt; ++c) {
#pragma unroll 1
                    for (int k = 0; k < kStatePlanes; ++k) W.state_plane[k][i0 + c] = of[k * T + c];
#pragma unroll 1
                    for (int k = 0; k < 16; ++k) W.obs_plane[k][i0 + c] = of[(13 + k) * T + c];
                    W.w.reward[i0 + c] = of[P_REWARD * T + c];
                    W.w.steps_in_episode[i0 + c] =
                        reinterpret_cast<const int32_t*>(of)[P_STEPS * T + c];
                }
                for (int c = c16; c < cnt; ++c) {
                    W.w.pending_reset[i0 + c] = ot[OB_PEND + c];
                    W.w.info[i0 + c] = ot[OB_PEND + T + c];
                }
                if constexpr (SC == 2) {
                    const int np = pcount[os];
                    if (np > 0) {
                        int32_t* wl = W.ob.worklist;
                        const int base = atomicAdd(wl, np);
                        const int* pl = plist + (size_t)os * T;
                        for (int k = 0; k < np; ++k) wl[3 + base + k] = pl[k];
                        pcount[os] = 0;
                    }
                    const int nr = rcount[os];
                    if (rl && nr > 0) {
                        int32_t* rs = W.ob.reset_list;
                        const int base = atomicAdd(rs, nr);
                        const int* pl = rlist + (size_t)os * T;
                        for (int k = 0; k < nr; ++k) rs[4 + base + k] = pl[k];
                        rcount[os] = 0;
                    }
                }
                bulk_commit();
                bulk_wait_read_all();        // the output tile may be rewritten now
                mbar_arrive(&oempty[os]);
            }
            bulk_wait_all();                  // writes complete before the CTA retires
        }
        return;
    }

    // ------------------------------- consumers -------------------------------
    // (32-bit tile bookkeeping, incremental ring stage / phase, barriers as
    // shared-window addresses: one env per thread per tile, so per-tile
    // overhead is per-env overhead)
    const int c = threadIdx.x;
    const uint32_t bars = smem_u32(smem);
    int st = 0, os = 0;
    uint32_t ph = 0, oph = 0;
    for (VTiles V(d.n, T, 1); V.valid(); V.next()) {
        const int cnt = V.cnt();
        const int64_t i = V.i0() + c;
        mbar_wait_u32(bars + 8u * st, ph);                                 // full[st]
        const unsigned char* sl = ring + (size_t)st * SB;
        const float* sf = reinterpret_cast<const float*>(sl);
        VState s;
        float goal[3];
        int32_t steps = 0;
        bool pending = false;
        uint32_t vmode = 0;
        double cmd[NC];
        float clr[4] = {0.0f, 0.0f, 0.0f, -1.0f};
        bool miss = false;
        const bool live = c < cnt;
        if (live) {
            if constexpr (SC == 2) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    clr[k] = reinterpret_cast<const float*>(sl + O_CLR)[k * T + c];
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                s.p[k] = sf[k * T + c];
                s.v[k] = sf[(7 + k) * T + c];
                s.w[k] = sf[(10 + k) * T + c];
                goal[k] = sf[(13 + k) * T + c];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) s.q[k] = sf[(3 + k) * T + c];
            // the final tile's tail counters / flags: straight from global memory
            steps = c < (cnt & ~3) ? reinterpret_cast<const int32_t*>(sl + O_STEPS)[c]
                                   : W.w.steps_in_episode[i];
            pending = (c < (cnt & ~15) ? sl[O_PEND + c] : W.w.pending_reset[i]) != 0;
            if (MIX) vmode = c < (cnt & ~15) ? sl[O_MODE + c] : d.mode_per_vehicle[i];
            if constexpr (MODE != FS_MODE_MIXED) {
                if (rows) {
                    double a[4];
                    if (W.act_f64) {
                        const double2* r = reinterpret_cast<const double2*>(sl + O_CMD) + 2 * c;
                        const double2 u = r[0], v = r[1];
                        a[0] = u.x; a[1] = u.y; a[2] = v.x; a[3] = v.y;
                    } else {
                        const float4 v = reinterpret_cast<const float4*>(sl + O_CMD)[c];
                        a[0] = f2d(v.x); a[1] = f2d(v.y); a[2] = f2d(v.z); a[3] = f2d(v.w);
                    }
                    denorm_actions<MODE>(W, a, cmd);
                } else {
#pragma unroll
                    for (int k = 0; k < NC; ++k)
                        cmd[k] = f2d(reinterpret_cast<const float*>(sl + O_CMD)[k * T + c]);
                }
            } else {
#pragma unroll
                for (int k = 0; k < NC; ++k)
                    cmd[k] = f2d(reinterpret_cast<const float*>(sl + O_CMD)[k * T + c]);
            }
        }
        // every read of this slot is done: release it
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(bars + 8u * (STAGES + st));      // empty[st]
        float reward = 0.0f;
        uint32_t info = 0;
        const bool skip = rl && live && pending;
        if (live && !skip)
            world_env_step<MODE, PREC, SC>(P, W, i, s, goal, steps, pending, vmode, cmd,
                                           reward, info, SC == 2 ? clr : nullptr,
                                           SC == 2 ? &miss : nullptr);
        // outputs into the shared output tile (its previous tile has been read
        // by the store warp's bulk stores)
        mbar_wait_u32(bars + 8u * (2 * STAGES + OSTAGES + os), oph ^ 1u);   // oempty[os]
        if constexpr (SC == 2) {
            const unsigned m = __ballot_sync(0xffffffffu, miss);
            if (m) {
                int base = 0;
                if (lane == 0) base = atomicAdd(&pcount[os], __popc(m));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (miss) plist[(size_t)os * T + base + __popc(m & ((1u << lane) - 1u))] = (int)i;
            }
            const bool pend = skip;
            const unsigned pm = rl ? __ballot_sync(0xffffffffu, pend) : 0u;
            if (pm) {
                int base = 0;
                if (lane == 0) base = atomicAdd(&rcount[os], __popc(pm));
                base = __shfl_sync(0xffffffffu, base, 0);
                if (pend) rlist[(size_t)os * T + base + __popc(pm & ((1u << lane) - 1u))] = (int)i;
            }
        }
        if (live) {
            unsigned char* ot = otiles + (size_t)os * OB;
            float* of = reinterpret_cast<float*>(ot);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                of[k * T + c] = s.p[k];
                of[(7 + k) * T + c] = s.v[k];
                of[(10 + k) * T + c] = s.w[k];
                of[(13 + k) * T + c] = s.p[k];
                of[(20 + k) * T + c] = s.v[k];
                of[(23 + k) * T + c] = s.w[k];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                of[(3 + k) * T + c] = s.q[k];
                of[(16 + k) * T + c] = s.q[k];
            }
            float gb[3];
            obs_goal(s, goal, gb);
#pragma unroll
            for (int k = 0; k < 3; ++k) of[(26 + k) * T + c] = gb[k];
            of[P_REWARD * T + c] = reward;
            reinterpret_cast<int32_t*>(of)[P_STEPS * T + c] = steps;
            ot[OB_PEND + c] = pending ? 1 : 0;
            ot[OB_PEND + T + c] = (uint8_t)info;
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive_u32(bars + 8u * (2 * STAGES + os));    // ofull[os]
        if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
        }
        if (++os == OSTAGES) {
            os = 0;
            oph ^= 1u;
        }
    }
}

__global__ void __launch_bounds__(256) world_reset_kernel(const __grid_constant__ WorldParams W) {
    const fs_step_desc& d = W.w.step;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= d.n) return;
    if (W.mask && !W.mask[i]) return;
    const uint32_t c = (uint32_t)(W.w.reset_counter[i] + W.increment);
    W.w.reset_counter[i] = (int32_t)c;
    VState s;
    float goal[3];
    const uint32_t info = respawn_env(W, i, c, s, goal);
    store_state(W, i, s);
#pragma unroll
    for (int k = 0; k < 3; ++k) W.w.goal[k * W.w.goal_stride + i] = goal[k];
    W.w.steps_in_episode[i] = 0;
    W.w.pending_reset[i] = 0;
    if (W.w.reward) W.w.reward[i] = 0.0f;
    if (W.w.info) W.w.info[i] = (uint8_t)info;
    write_obs(W, i, s, goal);
}

// Obstacle-world resets (world.py:160-252, 287-289): each warp owns 32
// consecutive envs, ballots which of them reset, and resets those one after
// another with the whole warp (warp_rebuild_env + lane-split SDF placement).
// AUTO: envs with pending_reset (World.step's auto-reset; the step kernel
// then voids their step); else envs with mask[e] != 0 (all when mask is
// NULL) and counter += increment (reset_env / reset_all / creation),
// finishing the env's outputs here.
// the env's robot / goal placement and its outputs after the obstacle rows
// are rebuilt (`sm`: the instance records with their boxes when nI <=
// kMaxInstWarp)
// POST (with AUTO): the auto-reset runs after the step kernel, which skipped
// the env (deferred resets, fs_obstacles.reset_list): it writes every output
// the step kernel would have written for a reset env (state at rest, obs,
// reward 0, steps 0, pending 0, info AUTORESET)
template <bool AUTO, bool POST = false>
__device__ __forceinline__ void finish_reset(const WorldParams& W, int64_t i, uint32_t c,
                                             const InstS* sm, int lane) {
    const fs_step_desc& d = W.w.step;
    const fs_obstacles& ob = W.ob;
    const int64_t gid = d.first_id + i;
    const int nI = ob.instances_per_env + (ob.wall_proto >= 0 ? 1 : 0);
    // placement (world.py:196-227): every lane evaluates the same draws, the
    // SDF clearance is split over the lanes
    float pt[2][3];
    bool ok[2];
#pragma unroll
    for (int which = 0; which < 2; ++which) {
        const bool goal = which == 1;
        const float* lo = goal ? W.lo_goal : W.lo_spawn;
        const float* span = goal ? W.span_goal : W.span_spawn;
        ok[which] = false;
        for (int a = 0; a < W.attempts && !ok[which]; ++a) {
            const U4 b = draw_block(d.seed, gid, c, kPlaceBlock + 2 * a + (goal ? 1 : 0));
            const uint32_t wv[3] = {b.x, b.y, b.z};
            bool in = true;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                pt[which][k] = __fmul_rn(__fadd_rn(lo[k], __fmul_rn(u01(wv[k]), span[k])),
                                         W.bounds[k]);
                in &= (pt[which][k] >= W.r) && (pt[which][k] <= __fsub_rn(W.bounds[k], W.r));
            }
            if (in)     // warp-uniform: every lane drew the same point
                ok[which] = (nI <= kMaxInstWarp &&
                             warp_far_from_instances(ob, sm, pt[which], W.r * 1.0001f + 1e-5f,
                                                     lane)) ||
                            !warp_scene_hit(ob.scene, i, f2d(pt[which][0]), f2d(pt[which][1]),
                                            f2d(pt[which][2]), W.r_d, lane);
        }
    }
    const uint32_t failed = (ok[0] && ok[1]) ? 0u : (uint32_t)FS_INFO_PLACEMENT_FAILED;
    if (AUTO && !POST) {
        // the env's stores, one per lane: state planes 0-12 (at rest at the
        // spawn), goal 13-15, counter / cache / info 16, camera mount 17
        if (lane < 13) {
            const float v = lane < 3 ? (lane == 0 ? pt[0][0] : lane == 1 ? pt[0][1] : pt[0][2])
                                     : (lane == 3 ? 1.0f : 0.0f);
            W.state_plane[lane][i] = v;
        } else if (lane < 16) {
            const int k = lane - 13;
            W.w.goal[k * W.w.goal_stride + i] = k == 0 ? pt[1][0] : k == 1 ? pt[1][1] : pt[1][2];
        } else if (lane == 16) {
            W.w.reset_counter[i] = (int32_t)c;
            // fresh obstacles and robot: the clearance cache is stale
            if (ob.clear) ob.clear[3 * ob.plane_stride + i] = -1.0f;
            W.w.info[i] = (uint8_t)(FS_INFO_AUTORESET | failed);
        } else if (lane == 17 && ob.mount) {
            randomize_mount_d(ob, i, d.seed, gid, c);
        }
    } else if (lane == 0) {
        W.w.reset_counter[i] = (int32_t)c;
        if (ob.mount) randomize_mount_d(ob, i, d.seed, gid, c);
        VState s;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            s.p[k] = pt[0][k];
            s.v[k] = 0.0f;
            s.w[k] = 0.0f;
            W.w.goal[k * W.w.goal_stride + i] = pt[1][k];
        }
        s.q[0] = 1.0f;
        s.q[1] = s.q[2] = s.q[3] = 0.0f;
        store_state(W, i, s);
        if (ob.clear) ob.clear[3 * ob.plane_stride + i] = -1.0f;
        W.w.steps_in_episode[i] = 0;
        W.w.pending_reset[i] = 0;
        if (W.w.reward) W.w.reward[i] = 0.0f;
        if (W.w.info) W.w.info[i] = (uint8_t)(failed | (POST ? FS_INFO_AUTORESET : 0u));
        write_obs(W, i, s, pt[1]);
    }
    __syncwarp();
}

template <bool AUTO, bool POST = false>
__device__ __forceinline__ void reset_one_env(const WorldParams& W, int64_t i, InstS* sm,
                                              uint8_t* s2i, uint16_t* s2p, int lane) {
    const fs_step_desc& d = W.w.step;
    const uint32_t c = (uint32_t)(W.w.reset_counter[i] + (AUTO ? 1 : W.increment));
    const fs_obstacles& ob = W.ob;
    const int nI = ob.instances_per_env + (ob.wall_proto >= 0 ? 1 : 0);
    if (nI <= kMaxInstWarp) {
        warp_rebuild_env(ob, i, d.seed, d.first_id + i, c, W.bounds_d, sm, lane, s2i, s2p);
    } else {
        if (lane == 0) rebuild_env(ob, i, d.seed, d.first_id + i, c, W.bounds_d);
        __syncwarp();
    }
    finish_reset<AUTO, POST>(W, i, c, sm, lane);
}


// Each warp scans kResetSpan envs per round -- 16 flag bytes per lane, one
// 16-byte load where aligned -- and resets the flagged ones one after another
// with the whole warp; a grid-stride loop covers the batch.  (One env per
// lane, one warp per 32 envs, spent ~40 us per step at 2^21 envs just
// retiring 65K warps that each waited on one 32-byte load.)
// (The streaming path with a skipped-env list does not run it: its
// auto-resets run after the step, in world_post_kernel.)
constexpr int kResetSpan = 512;
constexpr int kResetWarps = 4;      // warps per block (their InstS tables: 4 x 64 x 96 B)

#ifndef FS_RESET_MINB
#define FS_RESET_MINB 6     // <= 80 registers: 6 blocks per SM (was 124 registers, 4)
#endif
template <bool AUTO>
__global__ void __launch_bounds__(32 * kResetWarps, FS_RESET_MINB) world_reset_warp_kernel(const __grid_constant__ WorldParams W) {
    __shared__ InstS inst_sm[kResetWarps][kMaxInstWarp];
    __shared__ uint8_t s2i_sm[kResetWarps][kSlotTable];
    __shared__ uint16_t s2p_sm[kResetWarps][kSlotTable];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const fs_step_desc& d = W.w.step;
    const uint8_t* flags = AUTO ? W.w.pending_reset : W.mask;
    for (int64_t base = ((int64_t)blockIdx.x * kResetWarps + wib) * kResetSpan; base < d.n;
         base += (int64_t)gridDim.x * kResetWarps * kResetSpan) {
        const int64_t e0 = base + 16 * lane;
        uint32_t m16 = 0;       // bit b: env e0 + b resets
        if (!AUTO && !flags) {
            for (int b = 0; b < 16 && e0 + b < d.n; ++b) m16 |= 1u << b;
        } else if (e0 + 16 <= d.n && (reinterpret_cast<uintptr_t>(flags + e0) & 15u) == 0) {
            const uint4 v = *reinterpret_cast<const uint4*>(flags + e0);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int b = 0; b < 4; ++b)
                    if ((w[q] >> (8 * b)) & 0xFFu) m16 |= 1u << (4 * q + b);
        } else {
            for (int b = 0; b < 16 && e0 + b < d.n; ++b)
                if (flags[e0 + b]) m16 |= 1u << b;
        }
        unsigned todo = __ballot_sync(0xffffffffu, m16 != 0);
        while (todo) {
            const int u = __ffs(todo) - 1;
            todo &= todo - 1;
            for (uint32_t m = __shfl_sync(0xffffffffu, m16, u); m; m &= m - 1)
                reset_one_env<AUTO>(W, base + 16 * u + (__ffs(m) - 1), inst_sm[wib], s2i_sm[wib],
                                    s2p_sm[wib], lane);
        }
    }

}

// The deferred collision test (fs_obstacles.worklist): the envs the streaming
// step kernel could not clear with the clearance cache, as one compact list,
// a warp or quarter warp per env.  Each gets the full test at its new position and the
// cache refreshed; a hit turns the provisional no-collision outcome into the
// collision one: COLLISION | TERMINATED (never TRUNCATED), pending reset, and
// the reward with the crash term, from the same stored state and goal
// (world.py:95-116, 300-316).  The last block to finish empties the list.
//
// group_scene_test_refresh<G>: the full test of env i at p by a group of G
// lanes (a warp, or a quarter warp when the env has at most 16 instances, so
// one warp keeps four envs' scattered reads in flight); group-uniform result.
// Lane j takes instance j's broad-phase record; the instances within
// clear_walk are walked slot by slot, G slots at a time; the new clearance is
// the group minimum of the walked slots' exact SDFs (clear_exact; else their
// box distances) and the other instances' box distances.
template <int G>
__device__ __forceinline__ bool group_scene_test_refresh(const WorldParams& W, int64_t i,
                                                         const float* p, int sub, unsigned gmask,
                                                         int gshift, int& walked) {
    const fs_obstacles& ob = W.ob;
    const int J = ob.instances_per_env;
    const int64_t ps = ob.plane_stride;
    const float4* rec = reinterpret_cast<const float4*>(ob.inst_box) + i;
    const double px = f2d(p[0]), py = f2d(p[1]), pz = f2d(p[2]), r = W.r_d;
    const float rr = W.r * 1.0001f + 1e-5f;
    const float rv = fmaxf(rr, W.clear_walk);
    float c2 = 3.0e38f;
    bool hit = false;
    // the first two rounds' instance records are requested together (one
    // latency for both, e.g. 16 instances on a quarter warp)
    float4 lo_a = make_float4(0.f, 0.f, 0.f, 0.f), hi_a = lo_a, lo_b = lo_a, hi_b = lo_a;
#ifndef FS_FIX_NOPREFETCH
    if (sub < J) {
        lo_a = __ldg(rec + (int64_t)(2 * sub) * ps);
        hi_a = __ldg(rec + (int64_t)(2 * sub + 1) * ps);
    }
    if (G + sub < J) {
        lo_b = __ldg(rec + (int64_t)(2 * (G + sub)) * ps);
        hi_b = __ldg(rec + (int64_t)(2 * (G + sub) + 1) * ps);
    }
#endif
    for (int j0 = 0; j0 < J && !hit; j0 += G) {
        const int j = j0 + sub;
        bool walk = false;
        int32_t span = 0;
        if (j < J) {
#ifndef FS_FIX_NOPREFETCH
            const float4 lo = j0 == 0 ? lo_a : j0 == G ? lo_b : __ldg(rec + (int64_t)(2 * j) * ps);
            const float4 hi =
                j0 == 0 ? hi_a : j0 == G ? hi_b : __ldg(rec + (int64_t)(2 * j + 1) * ps);
#else
            const float4 lo = __ldg(rec + (int64_t)(2 * j) * ps);
            const float4 hi = __ldg(rec + (int64_t)(2 * j + 1) * ps);
#endif
            const float dx = fmaxf(fmaxf(lo.x - p[0], p[0] - hi.x), 0.0f);
            const float dy = fmaxf(fmaxf(lo.y - p[1], p[1] - hi.y), 0.0f);
            const float dz = fmaxf(fmaxf(lo.z - p[2], p[2] - hi.z), 0.0f);
            const float b2 = dx * dx + dy * dy + dz * dz;
            if (hi.w != 0.0f) {
                walk = b2 < rv * rv;
                if (!walk) c2 = fminf(c2, b2);
            }
            span = __float_as_int(lo.w);
        }
        unsigned wm = __ballot_sync(gmask, walk) >> gshift;
        while (wm && !hit) {
            const int u = __ffs(wm) - 1;
            wm &= wm - 1;
            const int32_t sp = __shfl_sync(gmask, span, u, G);
            const int first = sp & 0xffff, end = first + ((sp >> 16) & 0xffff);
            bool h = false;
            if (sub == 0) walked += end - first;      // (measurement: slots read)
            for (int k = first + sub; k < end; k += G) {
                SlotBox b;
                load_box(ob.scene, k, i, b);
                const double bd2 = box_dist2(b, px, py, pz);
                if (bd2 < r * r || W.clear_exact) {
                    // the primitive's exact distance: the hit test, and (with
                    // clear_exact) a much tighter clearance than its box for
                    // slanted branches -- an exact SDF is 1-Lipschitz
                    PrimD pr;
                    load_prim(ob.scene, k, i, pr);
                    const double sd = sdf(pr, px, py, pz);
                    h |= bd2 < r * r && sd < r;
                    const double e = fmax(sd, 0.0);
                    c2 = fminf(c2, W.clear_exact ? (float)(e * e) : (float)bd2);
                } else {
                    c2 = fminf(c2, (float)bd2);
                }
            }
            hit = __any_sync(gmask, h);
        }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) c2 = fminf(c2, __shfl_xor_sync(gmask, c2, o, G));
    if (sub == 0) {
        float* cl = ob.clear + i;
        cl[0] = p[0];
        cl[ps] = p[1];
        cl[2 * ps] = p[2];
        cl[3 * ps] = hit ? -1.0f : sqrtf(c2);
    }
    return hit;
}

// worklist entry k by a group of G lanes
template <int G>
__device__ __forceinline__ void scene_fix_one(const WorldParams& W, int k, int sub, unsigned gmask,
                                              int gshift, int& walked) {
    const int64_t i = W.ob.worklist[3 + k];
    VState s;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        s.p[c] = W.state_plane[c][i];
        s.v[c] = W.state_plane[7 + c][i];
    }
    const bool hit = group_scene_test_refresh<G>(W, i, s.p, sub, gmask, gshift, walked);
    if (hit && sub == 0) {
        float goal[3];
#pragma unroll
        for (int c = 0; c < 3; ++c) goal[c] = W.w.goal[c * W.w.goal_stride + i];
        const uint32_t nonfinite = W.w.info[i] & FS_INFO_NONFINITE;
        W.w.info[i] = (uint8_t)(FS_INFO_TERMINATED | FS_INFO_COLLISION | nonfinite);
        W.w.pending_reset[i] = 1;
        W.w.reward[i] = world_reward(W, s, goal, true);
    }
}

// one list entry per group of G lanes
template <int G>
__device__ __forceinline__ void scene_fix_entries(const WorldParams& W, int count, int& walked) {
    const int lane = threadIdx.x & 31;
    const int sub = lane % G, grp = lane / G;
    const int gshift = grp * G;
    const unsigned gmask = G == 32 ? 0xffffffffu : (((1u << G) - 1u) << gshift);
    constexpr int per_warp = 32 / G;
    const int nwarps = gridDim.x * (blockDim.x / 32);
    const int gw = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    for (int k = gw * per_warp + grp; k < count; k += nwarps * per_warp)
        scene_fix_one<G>(W, k, sub, gmask, gshift, walked);
}

// the block's walked-slot count onto fs_obstacles.walk_slots (one atomic per block)
__device__ __forceinline__ void flush_walked(const WorldParams& W, int walked) {
    walked = __reduce_add_sync(0xffffffffu, walked);
    if (W.ob.walk_slots && (threadIdx.x & 31) == 0 && walked)
        atomicAdd(reinterpret_cast<unsigned long long*>(W.ob.walk_slots),
                  (unsigned long long)walked);
}

// worklist bookkeeping by the last block of a pass over it
__device__ __forceinline__ void worklist_done(int32_t* wl, int count) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&wl[1], 1) == (int)gridDim.x - 1) {
            wl[2] += count;     // running total (diagnostics: how many envs were tested)
            wl[0] = 0;          // every block has read the count: empty the list
            wl[1] = 0;
            __threadfence();
        }
    }
}

#ifndef FS_FIX_MINB
#define FS_FIX_MINB 8      // <= 64 registers, no spills
#endif
__global__ void __launch_bounds__(128, FS_FIX_MINB) scene_fix_kernel(const __grid_constant__ WorldParams W) {
    int32_t* wl = W.ob.worklist;
    const int count = wl[0];
    // a quarter warp per env when it has at most 16 instances (each lane
    // takes two instance records: four envs' scattered reads in flight per
    // warp; forest fix kernel 51.3 -> 48.6 us at 2^21 envs), else a warp
    int walked = 0;
    if (W.ob.instances_per_env <= 16)
        scene_fix_entries<8>(W, count, walked);
    else
        scene_fix_entries<32>(W, count, walked);
    flush_walked(W, walked);
    worklist_done(wl, count);
}

// After the streaming step with deferred resets (reset lists valid): the
// auto-resets of the envs the previous step left pending (the step kernel
// skipped them) and the deferred collision test of this step's cache
// misses, as ONE pool of tasks that warps take from a counter -- first the
// resets (a warp per env, long latency chains), then the tests (a quarter
// warp per env, four per task).  The two sets are disjoint envs: a skipped
// env is never tested.  Both kinds of latency-bound work share the SMs
// instead of running one after the other, each with its own tail.
#ifndef FS_POST_MINB
#define FS_POST_MINB 5      // 96 registers (64 B stack): 84.1 -> 83.0 us at step 110 (4, 6, 8, 10 measured)
#endif
__global__ void __launch_bounds__(32 * kResetWarps, FS_POST_MINB)
    world_post_kernel(const __grid_constant__ WorldParams W) {
    __shared__ InstS inst_sm[kResetWarps][kMaxInstWarp];
    __shared__ uint8_t s2i_sm[kResetWarps][kSlotTable];
    __shared__ uint16_t s2p_sm[kResetWarps][kSlotTable];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    int32_t* rs = W.ob.reset_list;
    int32_t* wl = W.ob.worklist;
    int32_t* cur = rs;
    const int nres = rs[0];
    const int nfix = wl[0];
    const bool quarter = W.ob.instances_per_env <= 16;
    const int per_task = quarter ? 4 : 1;
    const int ntask = nres + (nfix + per_task - 1) / per_task;
    const int sub8 = lane & 7, grp = lane >> 3;
    int walked = 0;
    for (;;) {
        int k = 0;
        if (lane == 0) k = atomicAdd(&cur[3], 1);
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k >= ntask) break;
        if (k < nres) {
            const int64_t e = cur[4 + k];
            if (W.w.pending_reset[e])
                reset_one_env<true, true>(W, e, inst_sm[wib], s2i_sm[wib], s2p_sm[wib], lane);
        } else if (quarter) {
            const int f = (k - nres) * 4 + grp;
            if (f < nfix) scene_fix_one<8>(W, f, sub8, 0xffu << (8 * grp), 8 * grp, walked);
        } else {
            scene_fix_one<32>(W, k - nres, lane, 0xffffffffu, 0, walked);
        }
    }
    flush_walked(W, walked);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(&wl[1], 1) == (int)gridDim.x - 1) {
            wl[2] += nfix;
            wl[0] = 0;
            wl[1] = 0;
            cur[0] = 0;
            cur[3] = 0;
            __threadfence();
        }
    }
}

}  // namespace fs

namespace {

int fill_world(fs::WorldParams& W, const fs_world_desc* w, const fs_world_cfg* c) {
    memset(&W, 0, sizeof(W));
    W.w = *w;
    for (int k = 0; k < 13; ++k)
        W.state_plane[k] = w->step.state_out ? w->step.state_out + k * w->step.state_out_stride
                                             : nullptr;
    for (int k = 0; k < 16; ++k)
        W.obs_plane[k] = w->obs ? w->obs + k * w->obs_stride : nullptr;
    for (int k = 0; k < 3; ++k) {
        W.bounds[k] = (float)c->bounds[k];
        W.bounds_d[k] = c->bounds[k];
        W.lo_spawn[k] = (float)c->spawn_lo[k];
        W.span_spawn[k] = (float)(c->spawn_hi[k] - c->spawn_lo[k]);
        W.lo_goal[k] = (float)c->goal_lo[k];
        W.span_goal[k] = (float)(c->goal_hi[k] - c->goal_lo[k]);
    }
    W.r = (float)c->collision_radius;
    W.r_d = c->collision_radius;
    W.max_steps = c->episode_max_steps;
    W.attempts = c->placement_attempts > 0 ? c->placement_attempts : 100;
    W.c_dist = c->c_dist;
    W.c_vel = c->c_vel;
    W.c_step = c->c_step;
    W.c_success = c->c_success;
    W.c_crash = c->c_crash;
    W.success_radius = c->success_radius;
    if (w->obstacles) {
        const fs_obstacles& ob = *w->obstacles;
        const fs_scene& sc = ob.scene;
        if (sc.num_envs != w->step.n || sc.width < 0 ||
            (sc.width > 0 && (!sc.rec || (reinterpret_cast<uintptr_t>(sc.rec) & 15) != 0)) ||
            ob.plane_stride < w->step.n || !ob.proto_offset ||
            (ob.instances_per_env > 0 && (!ob.classes || !ob.inst_proto || ob.num_classes < 1)) ||
            (ob.mount && ob.mount_stride < w->step.n))
            return FS_EINVAL;
        W.ob = ob;
        W.has_ob = 1;
        W.clear_walk = (float)fs::g_clear_walk_cm * 0.01f;
        W.clear_exact = fs::g_clear_exact;
    }
    return 0;
}

bool a16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// the streaming kernel's layout contract: state updated in place, every base
// 16-byte aligned, plane strides multiples of 4, action rows contiguous
bool world_deferred_scene(const fs::WorldParams& W) {
    return W.has_ob && W.ob.worklist && W.ob.clear && W.ob.inst_box;
}

bool world_stream_layout_ok(const fs::WorldParams& W) {
    const fs_step_desc& d = W.w.step;
    // obstacle worlds stream only with the deferred collision test
    if ((W.has_ob && !world_deferred_scene(W)) || d.state_in != d.state_out) return false;
    if (!a16(d.state_in) || d.state_in_stride % 4 || !a16(W.w.goal) || W.w.goal_stride % 4 ||
        !a16(W.w.steps_in_episode) || !a16(W.w.pending_reset) || !a16(W.w.obs) ||
        W.w.obs_stride % 4 || !a16(W.w.reward) || !a16(W.w.info))
        return false;
    if (W.has_ob && (!a16(W.ob.clear) || W.ob.plane_stride % 4)) return false;
    if (W.actions) return a16(W.actions) && W.action_stride == 4;
    if (!a16(d.cmd) || d.cmd_stride % 4) return false;
    return d.mode != FS_MODE_MIXED || a16(d.mode_per_vehicle);
}

// ... and big enough to stream (small batches: the thread-per-env kernel)
bool world_stream_ok(const fs::WorldParams& W) {
    return W.w.step.n >= (1 << 15) && world_stream_layout_ok(W);
}


// blocks of the reset scan: one round of kResetSpan envs per warp, at most
// 8 blocks of kResetWarps warps per SM (grid-stride beyond)
unsigned reset_blocks(int64_t n) {
    int sms = fs_device_sm_count();
    if (sms <= 0) sms = 148;
    const int64_t per = (int64_t)fs::kResetWarps * fs::kResetSpan;
    const int64_t need = (n + per - 1) / per;
    const int64_t cap = 8 * (int64_t)sms;
    return (unsigned)(need < 1 ? 1 : (need < cap ? need : cap));
}

template <int MODE>
void launch_world_step(const fs::KParams& P, const fs::WorldParams& W, unsigned blocks,
                       cudaStream_t s) {
    const bool deferred = world_deferred_scene(W);
    int sms = fs_device_sm_count();
    if (sms <= 0) sms = 148;
    const bool stream = fs::g_world_kernel != 1 &&
                        (world_stream_ok(W) || (fs::g_world_kernel == 2 && world_stream_layout_ok(W)));
    // the streaming deferred path with a skipped-env list defers the
    // auto-resets to after the step (world_post_kernel); every other path
    // resets first
    const bool keep_list = deferred && stream && W.ob.reset_list;
    fs::WorldParams Wn = W;
    if (!keep_list) Wn.ob.reset_list = nullptr;
    if (W.has_ob && !keep_list) {
        // auto-resets first (warp per env), then the step
        fs::world_reset_warp_kernel<true>
            <<<reset_blocks(W.w.step.n), 32 * fs::kResetWarps, 0, s>>>(Wn);
        if (!deferred) {
            fs::world_step_kernel<MODE, 2, 1><<<blocks, 256, 0, s>>>(P, Wn);
            return;
        }
    }
    if (deferred && !stream) {
        // the step with the collision test deferred, then the test over the
        // compact worklist of the envs the clearance cache did not clear
        fs::world_step_kernel<MODE, 2, 2><<<blocks, 256, 0, s>>>(P, Wn);
        fs::scene_fix_kernel<<<(unsigned)(16 * sms), 128, 0, s>>>(Wn);
        return;
    }
    if (stream) {
        constexpr int T = 32 * fs::kWorldNCW;
        constexpr int SB = fs::world_stage_bytes<MODE>(T);
        constexpr int OB = fs::world_out_bytes(T);
#ifndef FS_WORLD_OST
#define FS_WORLD_OST 2   // double-buffered output tile, two input stages (162.8 -> 159.0 us)
#endif
        constexpr int OS = FS_WORLD_OST;
        constexpr int S0 = (225 * 1024 - 128 - OS * OB - 2 * OS * T * 4) / SB;
        constexpr int S = S0 > 4 ? 4 : S0;
        static_assert(S >= 2, "world ring too shallow");
        auto kern = deferred ? fs::world_stream_kernel<MODE, 2, S, OS, 2>
                             : fs::world_stream_kernel<MODE, 2, S, OS, 0>;
        const size_t smem = 128 + (size_t)S * SB + (size_t)OS * OB + (size_t)2 * OS * T * 4;
        static fs::PerDeviceOnce once;
        once([&](int) {
            cudaFuncSetAttribute(fs::world_stream_kernel<MODE, 2, S, OS, 0>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cudaFuncSetAttribute(fs::world_stream_kernel<MODE, 2, S, OS, 2>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        });
        const int64_t ntiles = (W.w.step.n + T - 1) / T;
        const unsigned grid = (unsigned)(ntiles < sms ? ntiles : sms);
        kern<<<grid, (fs::kWorldNCW + 2) * 32, smem, s>>>(P, Wn);
        if (deferred && keep_list)
            // the deferred auto-resets and collision tests, one task pool
            fs::world_post_kernel<<<(unsigned)(FS_POST_MINB * sms), 32 * fs::kResetWarps, 0, s>>>(Wn);
        else if (deferred)
            fs::scene_fix_kernel<<<(unsigned)(16 * sms), 128, 0, s>>>(Wn);
        return;
    }
    fs::world_step_kernel<MODE, 2, false><<<blocks, 256, 0, s>>>(P, W);
}

bool world_buffers_ok(const fs_world_desc* w) {
    const fs_step_desc& d = w->step;
    return d.state_in && d.state_out && w->goal && w->steps_in_episode && w->reset_counter &&
           w->pending_reset && w->obs && d.state_in_stride >= d.n && d.state_out_stride >= d.n &&
           w->goal_stride >= d.n && w->obs_stride >= d.n;
}

}  // namespace

// defined in fs_kernels.cu
int fs_fill_params_for_world(fs::KParams& P, const fs_step_desc* d, const fs_robot* r,
                             const fs_gains* g, const fs_limits* l);
int fs_fail_einval(const char* msg);

namespace {

int world_step_checks(const fs_world_desc* w, const fs_world_cfg* cfg, const fs_robot* robot,
                      const fs_gains* gains, const fs_limits* limits) {
    if (!w || !cfg || !robot || !gains || !limits) return fs_fail_einval("null descriptor/params");
    const fs_step_desc& d = w->step;
    if (d.n < 0) return fs_fail_einval("length must be >= 0");
    if (!(d.dt > 0.0f && d.dt <= 0.1f)) return fs_fail_einval("dt must be in (0, 0.1]");
    if (cfg->episode_max_steps < 1) return fs_fail_einval("episode_max_steps must be >= 1");
    if (d.n > 0 && (!world_buffers_ok(w) || !w->reward || !w->info))
        return fs_fail_einval("world buffers missing or strides shorter than length");
    return FS_OK;
}

}  // namespace

extern "C" int fs_world_step(const fs_world_desc* w, const fs_world_cfg* cfg, const fs_robot* robot,
                             const fs_gains* gains, const fs_limits* limits, void* stream) {
    int rc = world_step_checks(w, cfg, robot, gains, limits);
    if (rc != FS_OK) return rc;
    const fs_step_desc& d = w->step;
    if (d.n == 0) return FS_OK;
    if (!d.cmd || d.cmd_stride < d.n)
        return fs_fail_einval("command planes missing or stride shorter than length");
    if (d.mode != FS_MODE_ATTITUDE && d.mode != FS_MODE_VELOCITY && d.mode != FS_MODE_MIXED)
        return fs_fail_einval("world control_mode must be attitude, velocity or mixed");
    if (d.mode == FS_MODE_MIXED && !d.mode_per_vehicle)
        return fs_fail_einval("FS_MODE_MIXED needs mode_per_vehicle");
    fs::KParams P;
    rc = fs_fill_params_for_world(P, &d, robot, gains, limits);
    if (rc != FS_OK) return rc;
    P.want_flags = 1;
    fs::WorldParams W;
    if (fill_world(W, w, cfg) != 0) return fs_fail_einval("invalid obstacle descriptor");
    const unsigned blocks = (unsigned)((d.n + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    switch (d.mode) {
        case FS_MODE_ATTITUDE:
            launch_world_step<FS_MODE_ATTITUDE>(P, W, blocks, s);
            break;
        case FS_MODE_VELOCITY:
            launch_world_step<FS_MODE_VELOCITY>(P, W, blocks, s);
            break;
        default:
            launch_world_step<FS_MODE_MIXED>(P, W, blocks, s);
    }
    return fs::check_launch("world_step_kernel");
}

extern "C" int fs_vecenv_step(const fs_world_desc* w, const fs_world_cfg* cfg,
                              const fs_robot* robot, const fs_gains* gains,
                              const fs_limits* limits, const void* actions, int32_t action_dtype,
                              int64_t action_stride, void* stream) {
    int rc = world_step_checks(w, cfg, robot, gains, limits);
    if (rc != FS_OK) return rc;
    const fs_step_desc& d = w->step;
    if (d.mode != FS_MODE_ATTITUDE && d.mode != FS_MODE_VELOCITY)
        return fs_fail_einval("vecenv control_mode must be attitude or velocity");
    if (action_dtype != FS_DTYPE_F32 && action_dtype != FS_DTYPE_F64)
        return fs_fail_einval("action dtype must be FS_DTYPE_F32 or FS_DTYPE_F64");
    if (action_stride < 4 || (action_stride & 3) != 0)
        return fs_fail_einval("action row stride must be a multiple of 4 elements");
    if (d.n == 0) return FS_OK;
    if (!actions || (reinterpret_cast<uintptr_t>(actions) & 15) != 0)
        return fs_fail_einval("actions must be a 16-byte aligned device pointer");
    fs::KParams P;
    rc = fs_fill_params_for_world(P, &d, robot, gains, limits);
    if (rc != FS_OK) return rc;
    P.want_flags = 1;
    fs::WorldParams W;
    if (fill_world(W, w, cfg) != 0) return fs_fail_einval("invalid obstacle descriptor");
    W.actions = actions;
    W.action_stride = action_stride;
    if (d.mode == FS_MODE_ATTITUDE) {
        W.act_scale[0] = W.act_scale[1] = limits->max_tilt;
        W.act_scale[2] = limits->max_yaw_rate;
        W.act_scale[3] = robot->thrust_max;
    } else {
        W.act_scale[0] = W.act_scale[1] = W.act_scale[2] = limits->max_speed_cmd;
        W.act_scale[3] = limits->max_yaw_rate;
    }
    const unsigned blocks = (unsigned)((d.n + 255) / 256);
    cudaStream_t s = (cudaStream_t)stream;
    W.act_f64 = action_dtype == FS_DTYPE_F64;
    if (d.mode == FS_MODE_ATTITUDE)
        launch_world_step<FS_MODE_ATTITUDE>(P, W, blocks, s);
    else
        launch_world_step<FS_MODE_VELOCITY>(P, W, blocks, s);
    return fs::check_launch("world_step_kernel");
}

extern "C" int fs_world_reset(const fs_world_desc* w, const fs_world_cfg* cfg, const uint8_t* mask,
                              int32_t increment, void* stream) {
    if (!w || !cfg) return fs_fail_einval("null descriptor/config");
    const fs_step_desc& d = w->step;
    if (d.n < 0) return fs_fail_einval("length must be >= 0");
    if (d.n == 0) return FS_OK;
    if (!world_buffers_ok(w)) return fs_fail_einval("world buffers missing or strides too short");
    fs::WorldParams W;
    if (fill_world(W, w, cfg) != 0) return fs_fail_einval("invalid obstacle descriptor");
    W.mask = mask;
    W.increment = increment;
    if (W.has_ob) {
        fs::world_reset_warp_kernel<false>
            <<<reset_blocks(d.n), 32 * fs::kResetWarps, 0, (cudaStream_t)stream>>>(W);
        return fs::check_launch("world_reset_warp_kernel");
    }
    const unsigned blocks = (unsigned)((d.n + 255) / 256);
    fs::world_reset_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(W);
    return fs::check_launch("world_reset_kernel");
}
