// fs_step.cuh -- the fused step kernels (templates), shared by the per-mode
// translation units fs_step_{att,vel,mix,pos}.cu.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "flocksim_b200.h"
#include "fs_host.h"
#include "fs_math.cuh"
#include "fs_rng.cuh"

namespace fs {

constexpr int kThreads = 256;

// ---------------------------------------------------------------------------
// vector plane access
// ---------------------------------------------------------------------------
template <int VPT>
struct Vec;
template <>
struct Vec<1> {
    using T = float;
};
template <>
struct Vec<2> {
    using T = float2;
};
template <>
struct Vec<4> {
    using T = float4;
};

template <int VPT>
__device__ __forceinline__ void load_plane(const float* __restrict__ base, int64_t i0, int cnt,
                                           float (&out)[VPT]) {
    if (cnt == VPT) {
        if constexpr (VPT == 4) {
            const float4 t = *reinterpret_cast<const float4*>(base + i0);
            out[0] = t.x; out[1] = t.y; out[2] = t.z; out[3] = t.w;
        } else if constexpr (VPT == 2) {
            const float2 t = *reinterpret_cast<const float2*>(base + i0);
            out[0] = t.x; out[1] = t.y;
        } else {
            out[0] = base[i0];
        }
    } else {
#pragma unroll
        for (int j = 0; j < VPT; ++j) out[j] = (j < cnt) ? base[i0 + j] : 0.0f;
    }
}

template <int VPT>
__device__ __forceinline__ void store_plane(float* __restrict__ base, int64_t i0, int cnt,
                                            const float (&v)[VPT]) {
    if (cnt == VPT) {
        if constexpr (VPT == 4) {
            *reinterpret_cast<float4*>(base + i0) = make_float4(v[0], v[1], v[2], v[3]);
        } else if constexpr (VPT == 2) {
            *reinterpret_cast<float2*>(base + i0) = make_float2(v[0], v[1]);
        } else {
            base[i0] = v[0];
        }
    } else {
#pragma unroll
        for (int j = 0; j < VPT; ++j)
            if (j < cnt) base[i0 + j] = v[j];
    }
}

// int64 block reduction of three counters, one atomicAdd per CTA into a slot
__device__ __forceinline__ void block_stats(long long a, long long b, long long c,
                                            int64_t* slots, int nslots) {
    __shared__ long long red[3][kThreads / 32];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        c += __shfl_xor_sync(0xffffffffu, c, o);
    }
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        red[0][warp] = a;
        red[1][warp] = b;
        red[2][warp] = c;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long sa = 0, sb = 0, sc = 0;
#pragma unroll
        for (int w = 0; w < kThreads / 32; ++w) {
            sa += red[0][w];
            sb += red[1][w];
            sc += red[2][w];
        }
        unsigned long long* s =
            reinterpret_cast<unsigned long long*>(slots + 3 * (blockIdx.x & (nslots - 1)));
        atomicAdd(s + 0, (unsigned long long)sa);
        atomicAdd(s + 1, (unsigned long long)sb);
        atomicAdd(s + 2, (unsigned long long)sc);
    }
}

constexpr int kStatePlanes = 13;

template <int MODE>
__host__ __device__ constexpr int cmd_planes() {
    return MODE == FS_MODE_MIXED ? 8 : 4;
}

// ---------------------------------------------------------------------------
// per-vehicle driver shared by both fused kernels: optional Bernoulli
// re-spawn (EXTENSION, config 3), the fused step, statistics
// ---------------------------------------------------------------------------
struct StatAcc {
    long long err = 0;          // sum |p - p_d| in 2^-20 m
    int crash = 0, count = 0;   // per thread and launch: far below 2^31
};

// defer: re-spawns are not drawn inline but reported through `respawned`
// (the stream kernel's spawn warps draw them); known_reset >= 0: the
// caller already evaluated the Bernoulli word (1 = re-spawn).
template <int MODE, bool HETERO, int PREC, int NC, int FEAT = kFeatAll>
__device__ __forceinline__ void drive_vehicle(VState& s, float (&cmd)[NC], uint32_t vmode,
                                              const float* vp, int64_t gid, const KParams& P,
                                              bool integrate, int nsteps, StepOut& o,
                                              uint32_t& flags_all, bool& cmd_dirty,
                                              StatAcc& acc, bool defer = false,
                                              bool* respawned = nullptr, int known_reset = -1) {
    const fs_step_desc& d = P.d;
    const int frame_id = (HETERO && gid >= d.airframe_split) ? 1 : 0;
    for (int t = 0; t < nsteps; ++t) {
        bool reset = false;
        if ((FEAT & kFeatReset) && d.reset_prob > 0.0f) {
            const uint32_t stp = (uint32_t)(d.step_index + t);
            const bool fire = known_reset >= 0 ? known_reset != 0
                                               : reset_word(d.seed, gid, stp) < P.reset_thresh;
            if (fire) {
              reset = true;
              if (defer) {
                *respawned = true;
              } else {
                float st[13];
                spawn(d.seed, gid, stp, MODE, HETERO ? vp[0] : P.pf.mass, P.pf.gravity, st, cmd);
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    s.p[k] = st[k];
                    s.v[k] = st[7 + k];
                    s.w[k] = st[10 + k];
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) s.q[k] = st[3 + k];
                cmd_dirty = true;
              }
            }
        }
        if (!reset) {
            vehicle_step<MODE, HETERO, PREC, FEAT>(s, cmd, vmode, vp, frame_id, P, integrate, o);
            if ((FEAT & kFeatStats) && d.stats_slots) {
                float err = 0.0f;
                if (MODE == FS_MODE_POSITION) {
                    const float ex = s.p[0] - cmd[0], ey = s.p[1] - cmd[1], ez = s.p[2] - cmd[2];
                    // one MUFU op (rel. error ~2^-22; the statistic's bar is 1e-6)
                    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(err) : "f"(ex * ex + ey * ey + ez * ez));
                }
                // !(err <= 1e9) is err > 1e9 or NaN (one compare)
                const bool crash = (o.flags & (FS_FLAG_CLAMPED | FS_FLAG_NONFINITE)) != 0 ||
                                   !(err <= 1.0e9f);
                // (the select on the float: one FSEL instead of two 64-bit selects)
                acc.err += __float2ll_rn(crash ? 0.0f : err * 1048576.0f);
                acc.crash += crash ? 1 : 0;
                acc.count += 1;
            }
        } else {
            o.f = 0.f;
            o.m[0] = o.m[1] = o.m[2] = 0.f;
#pragma unroll
            for (int r = 0; r < FS_MAX_ROTORS; ++r) o.rotor[r] = 0.f;
            o.flags = FS_FLAG_RESET;
        }
        flags_all |= o.flags;
    }
}

// ---------------------------------------------------------------------------
// simple kernel: VPT vehicles per thread, vector loads straight to registers
// (fallback for unaligned buffers, small n, and the register-resident
// K-step rollout)
// ---------------------------------------------------------------------------
template <int MODE, bool HETERO, int PREC, int VPT, bool ROLLOUT>
__global__ void __launch_bounds__(kThreads)
    step_kernel(const __grid_constant__ KParams P) {
    constexpr int NC = cmd_planes<MODE>();
    const fs_step_desc& d = P.d;
    const int64_t i0 = ((int64_t)blockIdx.x * kThreads + threadIdx.x) * VPT;
    const int cnt = (i0 < d.n) ? (int)min((int64_t)VPT, d.n - i0) : 0;
    StatAcc acc;

    if (cnt > 0) {
        float S[kStatePlanes][VPT];
        float C[NC][VPT];
        float VP[4][VPT];
        uint32_t vmode[VPT];
#pragma unroll
        for (int k = 0; k < kStatePlanes; ++k)
            load_plane<VPT>(d.state_in + k * d.state_in_stride, i0, cnt, S[k]);
#pragma unroll
        for (int k = 0; k < NC; ++k) load_plane<VPT>(d.cmd + k * d.cmd_stride, i0, cnt, C[k]);
        if constexpr (HETERO) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                load_plane<VPT>(d.vparams + k * d.vparams_stride, i0, cnt, VP[k]);
        }
#pragma unroll
        for (int j = 0; j < VPT; ++j)
            vmode[j] = (MODE == FS_MODE_MIXED && j < cnt) ? d.mode_per_vehicle[i0 + j] : 0u;

        float WR[4][VPT];
        float RT[FS_MAX_ROTORS][VPT];
        uint32_t FL[VPT];
        const int nsteps = ROLLOUT ? P.steps : 1;
        const bool integrate = ROLLOUT || d.integrate;
        bool cmd_dirty = false;

#pragma unroll
        for (int j = 0; j < VPT; ++j) {
            VState s;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                s.p[k] = S[k][j];
                s.v[k] = S[7 + k][j];
                s.w[k] = S[10 + k][j];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) s.q[k] = S[3 + k][j];
            float cmd[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) cmd[k] = C[k][j];
            float vp[4] = {0.f, 0.f, 0.f, 0.f};
            if constexpr (HETERO) {
#pragma unroll
                for (int k = 0; k < 4; ++k) vp[k] = VP[k][j];
            }
            StepOut o;
            uint32_t flags_all = 0;
            drive_vehicle<MODE, HETERO, PREC, NC>(s, cmd, vmode[j], vp, d.first_id + i0 + j, P,
                                                  integrate, nsteps, o, flags_all, cmd_dirty,
                                                  acc);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                S[k][j] = s.p[k];
                S[7 + k][j] = s.v[k];
                S[10 + k][j] = s.w[k];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) S[3 + k][j] = s.q[k];
#pragma unroll
            for (int k = 0; k < NC; ++k) C[k][j] = cmd[k];
            WR[0][j] = o.f;
            WR[1][j] = o.m[0];
            WR[2][j] = o.m[1];
            WR[3][j] = o.m[2];
#pragma unroll
            for (int r = 0; r < FS_MAX_ROTORS; ++r) RT[r][j] = (P.n_frames > 0) ? o.rotor[r] : 0.f;
            FL[j] = ROLLOUT ? flags_all : o.flags;
        }

        if (integrate) {
#pragma unroll
            for (int k = 0; k < kStatePlanes; ++k)
                store_plane<VPT>(d.state_out + k * d.state_out_stride, i0, cnt, S[k]);
        }
        if (d.reset_prob > 0.0f) {
#pragma unroll
            for (int k = 0; k < NC; ++k) store_plane<VPT>(d.cmd + k * d.cmd_stride, i0, cnt, C[k]);
        }
        if (d.wrench_out) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                store_plane<VPT>(d.wrench_out + k * d.wrench_stride, i0, cnt, WR[k]);
        }
        if (d.rotor_out && P.n_frames > 0) {
#pragma unroll
            for (int k = 0; k < FS_MAX_ROTORS; ++k)
                store_plane<VPT>(d.rotor_out + k * d.rotor_stride, i0, cnt, RT[k]);
        }
        if (d.flags_out) {
#pragma unroll
            for (int j = 0; j < VPT; ++j)
                if (j < cnt) d.flags_out[i0 + j] = (uint8_t)FL[j];
        }
    }
    if (d.stats_slots) block_stats(acc.err, acc.crash, acc.count, d.stats_slots, d.stats_nslots);
}

// ---------------------------------------------------------------------------
// streaming kernel: persistent CTAs, warp-specialized TMA pipeline
// ---------------------------------------------------------------------------
//
// One producer warp streams tiles of T = 32 * NCW vehicles from HBM into a
// STAGES-deep shared-memory ring with 1-D bulk copies (cp.async.bulk, one per
// plane, completion on an mbarrier with expected-transaction bytes).  NCW
// consumer warps take one vehicle per thread from the ring, release the slot
// (mbarrier arrive), run the fused step in registers and store the results
// with coalesced 128-B-per-warp stores.  Memory-level parallelism is set by
// STAGES * tile bytes, not by registers, so HBM stays busy while the
// consumers compute.  Tiles are dealt round-robin (VTiles).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// try_wait with a suspend-time hint: a waiting warp is parked by the
// hardware until the phase flips (or the hint expires) instead of spinning,
// so waiting consumers do not take issue slots from computing ones
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(0x989680)
        : "memory");
}

// the same on precomputed shared-window addresses (the consumers' hot loop:
// no generic-to-shared conversion per tile)
__device__ __forceinline__ void mbar_arrive_u32(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
        "@!P1 bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity), "r"(0x989680)
        : "memory");
}

// non-blocking phase test
__device__ __forceinline__ bool mbar_test_u32(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
    return ok != 0;
}

// wait with an exponential nanosleep back-off (ns0 .. nsmax): a warp that
// expects to wait for a while (a spawn warp holding its draws until the
// output stage frees) parks instead of re-polling, so it does not take issue
// slots from the computing warps; ns0 == 0 falls back to try_wait
__device__ __forceinline__ void mbar_wait_backoff(uint32_t bar, uint32_t parity, uint32_t ns0,
                                                  uint32_t nsmax) {
    if (ns0 == 0) {
        mbar_wait_u32(bar, parity);
        return;
    }
    uint32_t ns = ns0;
    while (!mbar_test_u32(bar, parity)) {
        __nanosleep(ns);
        ns = ns * 2 < nsmax ? ns * 2 : nsmax;
    }
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

__device__ __forceinline__ uint64_t evict_last_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

__device__ __forceinline__ uint64_t evict_first_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

template <int MODE, bool HETERO>
__host__ __device__ constexpr int stream_float_planes() {
    return kStatePlanes + cmd_planes<MODE>() + (HETERO ? 4 : 0);
}

// Draw vehicle i's re-spawn at this step (fs_rng.cuh) and write its state
// (when integrating) and command planes straight to global memory.
template <int MODE, bool HETERO>
__device__ __forceinline__ void spawn_write(const KParams& P, int64_t i, bool integrate) {
    const fs_step_desc& d = P.d;
    constexpr int NC = cmd_planes<MODE>();
    const float mass = HETERO ? d.vparams[i] : P.pf.mass;
    float st[13], cmd[8];
    spawn(d.seed, d.first_id + i, (uint32_t)d.step_index, MODE, mass, P.pf.gravity, st, cmd);
    if (integrate) {
#pragma unroll
        for (int k = 0; k < 13; ++k) d.state_out[k * d.state_out_stride + i] = st[k];
    }
#pragma unroll
    for (int k = 0; k < NC; ++k) d.cmd[k * d.cmd_stride + i] = cmd[k];
}

// shared memory: mbarriers (offset 0), input ring [STAGES][NF][T], mode bytes
// [STAGES][T], output tiles [OST][13][T], and with kFeatReset the spawn
// warp's per-tile re-spawn list [T]
// double-buffered output tiles; the re-spawning variants take a third
// (FS_OUT_STAGES_RS = 3) when the shared-memory budget still leaves a
// two-stage input ring, so a store that waits for a spawn warp does not
// stall the consumers
#ifndef FS_OUT_STAGES_RS
#define FS_OUT_STAGES_RS 2
#endif
static_assert(FS_OUT_STAGES_RS >= 2 && FS_OUT_STAGES_RS <= 3, "output stages: 2 or 3 (kMaskSlots)");

constexpr int kBarBytes = 256;      // mbarrier region at the start of shared memory

// re-spawn ballot slots: consumers publish a tile's ballot words BEFORE they
// wait for its output stage (they wait for it only to write their outputs),
// so the words of tile it live in slot it % 4 (the spawn warp of tile
// it - 4 >= it - 1 - OST is done with that slot by then).  (Publishing them
// a tile EARLIER, so the draws start sooner, measured slower: 48.8 -> 60 us
// on cfg3 at 2^21, since the spawn warp must then also wait for the tile's
// commands to be loaded before it may overwrite them.)
constexpr int kMaskSlots = 4;

// In-place streaming (FS_INPLACE_RS for the re-spawning variants,
// FS_INPLACE_ALL for every variant): consumers write a tile's new state back
// into its input ring slot and the store lane stores it from there, then
// frees the slot, so the ring's slots serve as input and output stages at
// once (5 slots instead of 3 input + 2 output tiles): a consumer warp never
// waits for an output stage, and may run up to a whole ring ahead of the
// tile's slowest warp or its spawn warp.  The ballot slots then cover the
// ring (8).  Measured: cfg2 at 2^22 81.4 -> 79.5 us, cfg3 at 2^21 49.05 ->
// 48.4 us.
#ifndef FS_INPLACE_RS
#define FS_INPLACE_RS 1
#endif
#ifndef FS_INPLACE_ALL
#define FS_INPLACE_ALL 1
#endif
#ifndef FS_IP_SPAWN_WARPS
#define FS_IP_SPAWN_WARPS 2     // spawn warps of the in-place re-spawning variants
#endif
__host__ __device__ constexpr bool inplace_feat(int feat) {
    return FS_INPLACE_RS != 0 && ((feat & kFeatReset) != 0 || FS_INPLACE_ALL != 0);
}
__host__ __device__ constexpr int mask_slots(int feat) { return inplace_feat(feat) ? 8 : kMaskSlots; }

__host__ __device__ constexpr size_t respawn_smem_bytes(int feat, int T, int ost) {
    // ballot words [mask slots][T/32] + each spawn warp's compacted list [T]
    return (feat & kFeatReset) ? (size_t)mask_slots(feat) * (T / 32) * 4 + (size_t)ost * T * 4 : 0;
}

// output stages of a variant (spawn warp w owns output stage w); the
// in-place variants have two spawn warps and no output tiles
template <int MODE, bool HETERO, int NCW, int FEAT>
__host__ __device__ constexpr int out_stages() {
    return inplace_feat(FEAT) ? FS_IP_SPAWN_WARPS : (((FEAT & kFeatReset) && FS_OUT_STAGES_RS == 3 &&
            225 * 1024 - (kBarBytes + 3 * kStatePlanes * (32 * NCW) * 4 +
                          (int)respawn_smem_bytes(FEAT, 32 * NCW, 3)) >=
                2 * (stream_float_planes<MODE, HETERO>() * (32 * NCW) * 4 +
                     (MODE == FS_MODE_MIXED ? 32 * NCW : 0)))
               ? 3
               : 2);
}

// output tiles in shared memory (none in place)
template <int MODE, bool HETERO, int NCW, int FEAT>
__host__ __device__ constexpr int out_tiles() {
    return inplace_feat(FEAT) ? 0 : out_stages<MODE, HETERO, NCW, FEAT>();
}

// threads per CTA: NCW consumer warps, the load warp, the store warp, and
// with kFeatReset the spawn warps
template <int MODE, bool HETERO, int NCW, int FEAT>
__host__ __device__ constexpr int stream_threads() {
    return (NCW + 2 + ((FEAT & kFeatReset) ? out_stages<MODE, HETERO, NCW, FEAT>() : 0)) * 32;
}

template <int MODE, bool HETERO, int NCW, int VPT, int STAGES, int FEAT>
__host__ __device__ constexpr size_t stream_smem_bytes() {
    return kBarBytes + (size_t)STAGES * stream_float_planes<MODE, HETERO>() * (32 * NCW * VPT) * 4 +
           (MODE == FS_MODE_MIXED ? (size_t)STAGES * 32 * NCW * VPT : 0) +
           (size_t)out_tiles<MODE, HETERO, NCW, FEAT>() * kStatePlanes * (32 * NCW * VPT) * 4 +
           respawn_smem_bytes(FEAT, 32 * NCW * VPT, out_stages<MODE, HETERO, NCW, FEAT>());
}

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes,
                                         uint64_t policy) {
    asm volatile(
        "cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
        "r"(smem_u32(src)), "r"(bytes), "l"(policy)
        : "memory");
}

__device__ __forceinline__ void bulk_commit() {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_read_all() {
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void bulk_wait_all() {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void consumer_bar(int nthreads) {
    asm volatile("bar.sync 1, %0;" ::"r"(nthreads) : "memory");
}

// named barrier 2: the store warp arrives once its bulk stores are complete,
// the consumers wait before writing re-spawned vehicles to global memory
__device__ __forceinline__ void drained_arrive(int nthreads) {
    asm volatile("bar.arrive 2, %0;" ::"r"(nthreads) : "memory");
}
__device__ __forceinline__ void drained_wait(int nthreads) {
    asm volatile("bar.sync 2, %0;" ::"r"(nthreads) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---- chained steps (fs_step_desc.tile_sync) ---------------------------------
// A step publishes, per FS_SYNC_GRANULE vehicles, the counter value
// sync_post once the tile's state is in global memory; the next step of the
// chain (a programmatic dependent launch) loads a tile only after its
// counters have reached sync_wait.  Consecutive steps then overlap: CTAs of
// step k+1 start on the SMs that step k has left and stream the tiles step
// k finished long ago, instead of the whole GPU draining and refilling the
// pipeline at every launch boundary.
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// The protocol leans on where the bytes live: every write a step makes to a
// tile (TMA bulk stores of the state, plain stores of re-spawned commands) is
// COMPLETE -- performed at L2, the GPU's point of coherence -- before the
// tile's counters are stored (bulk wait_group / MEMBAR by the writer), and
// the next step reads counters with strong L2 loads and the tile with TMA
// loads, which also read L2.  So no fence is needed on either side of the
// counter itself; a gpu-scope MEMBAR there would also wait for the bulk
// copies the thread has in flight and serialize its stream (measured:
// FS_TUNE_CHAIN_RELEASE = 1 adds one to the publishing side).

// lane g of the load warp: strong L2 load of the tile's counter g (issued one
// tile ahead, so its latency hides behind the ring-slot wait)
__device__ __forceinline__ uint32_t counter_load(const uint32_t* p, bool acquire) {
    uint32_t v;
    if (acquire)
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    else
        asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ uint32_t tile_sync_load(const uint32_t* sync, int64_t i0, int cnt,
                                                   int lane, bool acquire) {
    uint32_t v = 0xffffffffu;
    if (lane < (cnt + FS_SYNC_GRANULE - 1) / FS_SYNC_GRANULE)
        v = counter_load(sync + i0 / FS_SYNC_GRANULE + lane, acquire);
    return v;
}

// warp-collective: each lane checks its prefetched counter and, only if the
// tile is not published yet, spins on it.  Every counter load is an
// acquire at gpu scope; __syncwarp carries that ordering to lane 0, which
// then orders the generic-proxy acquire before its async-proxy (TMA) reads
// of the tile with fence.proxy.async.global (the caller does that).  A
// wait longer than timeout_ns (FS_TUNE_SYNC_TIMEOUT_MS; 0 = wait forever)
// traps, so a broken chain is a kernel error instead of a hung GPU.  The
// launch is cooperative (all CTAs resident), so a legitimate wait is
// bounded by one step's streaming time; the default limit (10 s) only fires
// on a broken chain or a GPU time-sliced away for that long.
__device__ __forceinline__ void tile_sync_check(const uint32_t* sync, int64_t i0, int cnt,
                                                uint32_t v, uint32_t want, int lane,
                                                uint64_t timeout_ns, bool acquire) {
    if (lane < (cnt + FS_SYNC_GRANULE - 1) / FS_SYNC_GRANULE && (int32_t)(v - want) < 0) {
        const uint32_t* p = sync + i0 / FS_SYNC_GRANULE + lane;
        const uint64_t t0 = global_ns();
        do {
            __nanosleep(64);
            v = counter_load(p, acquire);
            if (timeout_ns != 0 && global_ns() - t0 > timeout_ns) __trap();
        } while ((int32_t)(v - want) < 0);
    }
    __syncwarp();
}

// store lane, once the tile's bulk stores have completed: publish its counters
// (release = 1: proxy + gpu-scope fences first, FS_TUNE_CHAIN_RELEASE)
__device__ __forceinline__ void tile_sync_post(uint32_t* sync, int64_t i0, int cnt,
                                               uint32_t post, bool release) {
    if (release) asm volatile("fence.proxy.async.global;\n\tfence.acq_rel.gpu;" ::: "memory");
    const int ng = (cnt + FS_SYNC_GRANULE - 1) / FS_SYNC_GRANULE;
    for (int g = 0; g < ng; ++g)
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(sync + i0 / FS_SYNC_GRANULE + g),
                     "r"(post)
                     : "memory");
}

// store lane: wait until the spawn warp of tile `it`'s stage has fenced that
// tile's commands (its counter has reached it; tiles of a stage increase)
__device__ __forceinline__ void wait_cfenced(const uint32_t* c, uint32_t it) {
    uint32_t v;
    for (;;) {
        asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(c)) : "memory");
        if (v != 0xffffffffu && v >= it) break;
        __nanosleep(32);
    }
}

template <int N>
__device__ __forceinline__ void bulk_wait_pending() {
    asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

// Tile schedule of a persistent streaming kernel: tiles of T dealt
// round-robin (tile it * G + b at iteration it), so at any moment the CTAs
// stream neighbouring regions, which DRAM likes.  (Two alternatives measured
// no better: contiguous per-CTA ranges cost DRAM locality, 84 -> 90 us on
// cfg2; balancing the last round's remainder into equal chunks gained
// nothing, because a partial tile costs nearly a full tile's latency.)
// Tile starts are multiples of T (a multiple of 16): 16-byte aligned for TMA
// even on byte planes.  All warp roles walk the same sequence.
//
// Over K consecutive steps (fs_step_many; K = 1 for fs_step) the virtual tile
// v = s * ntiles + t (step s, tile t) is dealt round-robin, v = b, b + G, ...
// Step by step this is the sequence above, continued across steps without
// a launch boundary, so the ring never drains
// between steps.  Tile t of step s + 1 depends only on tile t of step s
// (elementwise state), which another CTA stored ntiles / G rounds earlier:
// the tile_sync counters carry that dependency.
struct VTiles {
    // 32-bit tile indices (n < 2^31 * T): the per-tile bookkeeping is one add,
    // one compare and a select, and the tile start is only widened where used.
    // The grid never exceeds the tile count (launch_stream), so a step
    // boundary is crossed at most once per advance.
    int t, nt, G, K, s, T, last;
    __device__ __forceinline__ VTiles(int64_t n, int T_, int K_)
        : t((int)blockIdx.x), nt((int)((n + T_ - 1) / T_)), G((int)gridDim.x), K(K_), s(0), T(T_),
          last((int)(n - (int64_t)(((n + T_ - 1) / T_) - 1) * T_)) {
        if (t >= nt) s = K;                       // (no tile for this CTA)
    }
    __device__ __forceinline__ bool valid() const { return s < K; }
    __device__ __forceinline__ int64_t i0() const { return (int64_t)t * T; }
    __device__ __forceinline__ int cnt() const { return t == nt - 1 ? last : T; }
    __device__ __forceinline__ void next() {
        t += G;
        if (t >= nt) {
            t -= nt;
            ++s;
        }
    }
};

// Persistent, warp-specialized streaming kernel (one CTA per SM):
//  * load warp (warp NCW, one lane): streams the CTA's tiles of T = 32*NCW*VPT vehicles
//    from HBM into a STAGES-deep shared ring, one 1-D TMA bulk copy per
//    plane, completion counted on the slot's `full` mbarrier (expect-tx);
//  * NCW consumer warps: each thread takes VPT vehicles per tile (vehicle
//    tid + j*32*NCW), loads each just in time from the ring (immediate
//    offsets), releases the slot (`empty`), runs the fused step in registers
//    and writes the 13 new planes into a double-buffered shared output tile
//    (immediate offsets), then signals `ofull`;
//  * store warp (warp NCW+1, one lane): waits for `ofull`, writes the tile
//    back with one TMA bulk store per plane, waits for the shared-memory
//    reads to finish and releases the output tile (`oempty`).
//  * spawn warp (warp NCW+2, kFeatReset only): for each tile it evaluates the
//    Bernoulli re-spawn word of every vehicle itself (a pure function of
//    seed, global id and step), draws the tile's spawns lane-parallel, writes
//    their states into the output tile and their commands to global memory,
//    and signals `ofull` with the consumers; the consumers skip those
//    vehicles (their step is voided, world.py:287-299 semantics).  The draws
//    overlap the streaming: no tail, no divergent spawns in consumer warps.
// Consumers never touch a global address on the pure path and never wait on
// a CTA-wide barrier.  FEAT selects the optional features compiled in
// (kFeatStats / kFeatReset / kFeatOut); FEAT = 0 is the pure step, the bench
// hot path.  Optional outputs (kFeatOut) are plain coalesced stores.
template <int MODE, bool HETERO, int PREC, int NCW, int VPT, int STAGES, int FEAT>
__global__ void __launch_bounds__(stream_threads<MODE, HETERO, NCW, FEAT>(), 1)
    stream_kernel(const __grid_constant__ KParams P) {
    constexpr int TW = 32 * NCW;          // vehicles per "row" (one per consumer thread)
    constexpr int T = TW * VPT;           // vehicles per tile
    constexpr int NC = cmd_planes<MODE>();
    constexpr int NF = stream_float_planes<MODE, HETERO>();
    constexpr bool MIX = MODE == FS_MODE_MIXED;
    // IP (in-place re-spawning variants): the output stages ARE the ring slots
    constexpr bool IP = inplace_feat(FEAT);
    constexpr int kOutStages = IP ? STAGES : out_stages<MODE, HETERO, NCW, FEAT>();
    constexpr int kSpawnWarps = out_stages<MODE, HETERO, NCW, FEAT>();
    constexpr int kOutTiles = out_tiles<MODE, HETERO, NCW, FEAT>();
    constexpr int kMS = mask_slots(FEAT);
    extern __shared__ __align__(128) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem);                         // [STAGES]
    uint64_t* empty = full + STAGES;                                             // [STAGES]
    uint64_t* ofull = empty + STAGES;                                            // [kOutStages]
    uint64_t* oempty = ofull + kOutStages;                                       // [kOutStages]
    // [kMS] re-spawn ballots complete (arrived after the consumers read the
    // tile's inputs)
    uint64_t* lfull = oempty + kOutStages;
    // [kSpawnWarps] chained: newest tile of the spawn warp whose spawned commands are at L2
    uint32_t* cfenced = reinterpret_cast<uint32_t*>(lfull + kMS);
    float* ring = reinterpret_cast<float*>(smem + kBarBytes);                   // [STAGES][NF][T]
    uint8_t* mring = smem + kBarBytes + (size_t)STAGES * NF * T * 4;            // [STAGES][T]
    float* otile = reinterpret_cast<float*>(mring + (MIX ? (size_t)STAGES * T : 0));  // [OT][13][T]
    // per ballot slot, one re-spawn ballot word per 32 vehicles of the tile
    uint32_t* rs_mask = reinterpret_cast<uint32_t*>(otile + (size_t)kOutTiles * kStatePlanes * T);
    int* rs_list = reinterpret_cast<int*>(rs_mask + (size_t)kMS * (T / 32));  // [SW][T]
    constexpr bool RS = (FEAT & kFeatReset) != 0;
    static_assert(IP || !RS || kSpawnWarps == kOutStages, "spawn warp w owns output stage w");
    static_assert((2 * STAGES + 2 * kOutStages + kMS) * 8 + 4 * kSpawnWarps <= kBarBytes,
                  "mbarrier region");
    // the output tile of ring stage / output stage `os`
    auto out_of = [&](int os) -> float* {
        return IP ? ring + (size_t)os * NF * T : otile + (size_t)os * kStatePlanes * T;
    };

    const fs_step_desc& d = P.d;
    const int K = P.steps;      // consecutive steps streamed by this launch (VTiles)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // FEAT = 0 (no outputs, statistics or re-spawns) only exists for the
    // integrating step (launch_variant skips a control-only call with nothing
    // to write), so there the flag is a compile-time constant
    const bool integrate = FEAT == 0 ? true : d.integrate != 0;
    static_assert(T % FS_SYNC_GRANULE == 0, "tiles are whole sync granules");
    const bool chained = d.tile_sync != nullptr;
    // the next step of a chain may be scheduled now (its CTAs take the SMs
    // this grid leaves; its tiles wait on tile_sync, not on grid completion)
    if (chained) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            // (in place the store lane frees a slot, once it has stored it)
            mbar_init(&empty[s], IP ? 1 : NCW);
        }
        for (int s = 0; s < kOutStages; ++s) {
            mbar_init(&ofull[s], NCW + (RS ? 1 : 0));
            mbar_init(&oempty[s], 1);
        }
        for (int s = 0; s < kSpawnWarps; ++s) cfenced[s] = 0xffffffffu;
        for (int s = 0; s < kMS; ++s) mbar_init(&lfull[s], NCW);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    if (warp == NCW) {
        // ------------------------------ load warp ----------------------------
        // L2 residency: the first l2_keep_tiles tiles (of every step) load and
        // store with evict_last, so they stay in L2 from one step to the next;
        // the rest stream with evict_first
        const uint64_t pol_first = evict_first_policy(), pol_last = evict_last_policy();
        // step 0 reads state_in; steps s >= 1 of an fs_step_many launch read
        // the previous step's state_out (out-of-place K-step launches)
        auto issue = [&](int it, int64_t i0, int cnt, int s) {
            const uint64_t pol = (i0 < (int64_t)P.l2_keep_tiles * T) ? pol_last : pol_first;
            const float* sin = s == 0 ? d.state_in : d.state_out;
            const int64_t sst = s == 0 ? d.state_in_stride : d.state_out_stride;
            const int st = it % STAGES;
            mbar_wait(&empty[st], ((it / STAGES) & 1) ^ 1);
            const uint32_t fb = (uint32_t)((cnt * 4 + 15) & ~15);
            const uint32_t mb = MIX ? (uint32_t)((cnt + 15) & ~15) : 0u;
            mbar_expect_tx(&full[st], NF * fb + mb);
            float* slot = ring + (size_t)st * NF * T;
#pragma unroll
            for (int k = 0; k < kStatePlanes; ++k)
                bulk_g2s(slot + k * T, sin + k * sst + i0, fb, &full[st], pol);
#pragma unroll
            for (int k = 0; k < NC; ++k)
                bulk_g2s(slot + (kStatePlanes + k) * T, d.cmd + k * d.cmd_stride + i0, fb, &full[st],
                         pol);
            if constexpr (HETERO) {
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    bulk_g2s(slot + (kStatePlanes + NC + k) * T, d.vparams + k * d.vparams_stride + i0,
                             fb, &full[st], pol);
            }
            if constexpr (MIX) bulk_g2s(mring + st * T, d.mode_per_vehicle + i0, mb, &full[st], pol);
        };
        if (!chained) {
            if (lane == 0) {
                int it = 0;
                for (VTiles V(d.n, T, K); V.valid(); V.next(), ++it) issue(it, V.i0(), V.cnt(), V.s);
            }
            return;
        }
        // counters: lanes prefetch the next tile's, check them when the tile
        // comes up (step s waits for sync_wait + s; the first step of an
        // unchained launch, sync_wait == 0, waits for nothing), lane 0 streams
        const bool acq = (P.chain_acquire & 1) != 0;      // gpu-scope acquire counter loads
        const bool pfence = (P.chain_acquire & 2) != 0;   // proxy fence before the TMA loads
        const bool mfence = (P.chain_acquire & 4) != 0;   // relaxed loads + fence.acq_rel.gpu
        VTiles V(d.n, T, K);
        uint32_t v = V.valid() ? tile_sync_load(d.tile_sync, V.i0(), V.cnt(), lane, acq) : 0u;
        for (int it = 0; V.valid(); ++it) {
            const bool waited = V.s > 0 || d.sync_wait != 0;
            if (waited)
                tile_sync_check(d.tile_sync, V.i0(), V.cnt(), v, d.sync_wait + (uint32_t)V.s, lane,
                                P.sync_timeout_ns, acq);
            if (waited && mfence) asm volatile("fence.acq_rel.gpu;" ::: "memory");
            VTiles X = V;
            X.next();
            if (X.valid()) v = tile_sync_load(d.tile_sync, X.i0(), X.cnt(), lane, acq);
            if (lane == 0) {
                // acquire -> TMA reads of the tile
                if (waited && pfence) fence_proxy_async_global();
                issue(it, V.i0(), V.cnt(), V.s);
            }
            __syncwarp();
            V = X;
        }
        return;
    }
    if (warp == NCW + 1) {
        // ------------------------------ store warp ---------------------------
        // (in place the store lane also frees the slots of a control-only
        // call, which stores nothing)
        if (lane == 0 && (integrate || RS || IP)) {
            const uint64_t pol_first = evict_first_policy(), pol_last = evict_last_policy();
            // chained: a tile is published once its stores have completed, up
            // to `lag` tiles later (its newest groups may still be in flight,
            // so the wait rarely blocks); tile j waits in slot j & 1.  Within
            // one launch (K > 1) a tile may be published only before this CTA
            // needs a tile that depends on it: lag * G < ntiles.
            const int64_t nt = (d.n + T - 1) / T;
            const int G = (int)gridDim.x;
            const int lag = K == 1 ? 2 : (2 * (int64_t)G < nt ? 2 : ((int64_t)G < nt ? 1 : 0));
            // (two named slots, no local arrays: nvcc 12.9 mis-addressed
            // lambda-captured local arrays here, storing a count as the value)
            int64_t pi0 = 0, pi1 = 0;
            int pc0 = 0, pc1 = 0;
            uint32_t pv0 = 0u, pv1 = 0u;
            auto publish = [&](int j) {
#ifndef FS_DIAG_NO_CFENCE
                if (RS) wait_cfenced(&cfenced[j % kSpawnWarps], (uint32_t)j);
#endif
                const bool odd = (j & 1) != 0;
                const int pc = odd ? pc1 : pc0;
                if (pc & 3) __threadfence();    // ragged tile: its plain stores too
                tile_sync_post(d.tile_sync, odd ? pi1 : pi0, pc, odd ? pv1 : pv0, P.chain_release);
            };
            int it = 0;
            for (VTiles V(d.n, T, K); V.valid(); V.next(), ++it) {
                const int os = it % kOutStages;
                const int64_t i0 = V.i0();
                const int cnt = V.cnt();
                mbar_wait(&ofull[os], (it / kOutStages) & 1);
                if (!integrate) {           // control only: the re-spawn handshake alone
                    mbar_arrive(IP ? &empty[os] : &oempty[os]);
                    continue;
                }
                // bulk-store the 16-byte multiple; the 0..3 vehicles past it (only in
                // the last tile) are plain stores, so nothing beyond n is written
                const uint64_t pol = (V.t < P.l2_keep_tiles) ? pol_last : pol_first;
                const int cbulk = cnt & ~3;
                const float* src = out_of(os);
                if (cbulk > 0) {
#pragma unroll
                    for (int k = 0; k < kStatePlanes; ++k)
                        bulk_s2g(d.state_out + k * d.state_out_stride + i0, src + k * T,
                                 (uint32_t)cbulk * 4u, pol);
                }
                for (int c = cbulk; c < cnt; ++c)
                    for (int k = 0; k < kStatePlanes; ++k)
                        d.state_out[k * d.state_out_stride + i0 + c] = src[k * T + c];
                bulk_commit();
                bulk_wait_read_all();            // the output tile may be rewritten now
                mbar_arrive(IP ? &empty[os] : &oempty[os]);
                if (chained) {
                    const int q = it & 1;
                    if (lag == 2) {
                        if (it >= 2) {
                            bulk_wait_pending<2>();
                            publish(it - 2);
                        }
                    } else if (lag == 1) {
                        if (it >= 1) {
                            bulk_wait_pending<1>();
                            publish(it - 1);
                        }
                    }
                    if (q) {
                        pi1 = i0;
                        pc1 = cnt;
                        pv1 = d.sync_post + (uint32_t)V.s;
                    } else {
                        pi0 = i0;
                        pc0 = cnt;
                        pv0 = d.sync_post + (uint32_t)V.s;
                    }
                    if (lag == 0) {
                        bulk_wait_pending<0>();
                        publish(it);
                    }
                }
            }
            bulk_wait_all();                      // writes complete before the CTA retires
            if (chained && integrate && lag > 0)
                for (int j = it >= lag ? it - lag : 0; j < it; ++j) publish(j);
        }
        return;
    }
    if (RS && warp >= NCW + 2) {
        // ------------------------------ spawn warps --------------------------
        // spawn warp w takes the tiles of output stage w: it waits for the
        // consumers' re-spawn list of the tile, draws those spawns
        // lane-parallel into the output tile (+ their commands to global
        // memory) while the consumers step the rest, and signals `ofull`
        const int sw = warp - (NCW + 2);
        int it = 0;
        for (VTiles V(d.n, T, K); V.valid(); V.next(), ++it) {
            if (it % kSpawnWarps != sw) continue;
            const int os = it % kOutStages;
            const int64_t i0 = V.i0();
            const uint32_t stp = (uint32_t)(d.step_index + (uint64_t)V.s);
            const int ms = it % kMS;
            mbar_wait_backoff(smem_u32(&lfull[ms]), (it / kMS) & 1, P.spawn_wait_ns,
                              4 * P.spawn_wait_ns);
            const uint32_t* msk = rs_mask + (size_t)ms * (T / 32);
            float* out = out_of(os);
            // compact the ballot words into this warp's list (warp scan of the
            // per-word counts), then draw the spawns lane-parallel
            int* lst = rs_list + (size_t)sw * T;
            int total = 0;
            for (int w0 = 0; w0 < T / 32; w0 += 32) {
                const int w = w0 + lane;
                const uint32_t m = w < T / 32 ? msk[w] : 0u;
                const int cntw = __popc(m);
                int incl = cntw;
#pragma unroll
                for (int off = 1; off < 32; off <<= 1) {
                    const int v = __shfl_up_sync(0xffffffffu, incl, off);
                    if (lane >= off) incl += v;
                }
                int pos = total + incl - cntw;
                for (uint32_t mm = m; mm; mm &= mm - 1) lst[pos++] = w * 32 + __ffs(mm) - 1;
                total += __shfl_sync(0xffffffffu, incl, 31);
            }
            __syncwarp();
            // the first 32 spawns are drawn into registers BEFORE the output
            // stage is free (the consumers now wait for it only when they
            // write, after their compute), then written once it is
            auto draw = [&](int q, float (&st)[13], float (&ncmd)[8]) {
                const int64_t i = i0 + lst[q];
                spawn(d.seed, d.first_id + i, stp, MODE, HETERO ? d.vparams[i] : P.pf.mass,
                      P.pf.gravity, st, ncmd);
            };
            auto put = [&](int q, const float (&st)[13], const float (&ncmd)[8]) {
                const int c = lst[q];
                const int64_t i = i0 + c;
                if (integrate) {
#pragma unroll
                    for (int k = 0; k < kStatePlanes; ++k) out[k * T + c] = st[k];
                }
#pragma unroll
                for (int k = 0; k < NC; ++k) d.cmd[k * d.cmd_stride + i] = ncmd[k];
            };
            {
                float st[13], ncmd[8];
                if (lane < total) draw(lane, st, ncmd);
                if (integrate && !IP)
                    mbar_wait_backoff(smem_u32(&oempty[os]), ((it / kOutStages) & 1) ^ 1,
                                      P.spawn_wait_ns, 4 * P.spawn_wait_ns);
                if (lane < total) put(lane, st, ncmd);
            }
            for (int q = lane + 32; q < total; q += 32) {     // (more than 32 in a tile)
                float st[13], ncmd[8];
                draw(q, st, ncmd);
                put(q, st, ncmd);
            }
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&ofull[os]);
            if (chained && integrate) {
                // the commands must be at L2 before the store lane publishes
                // this tile (tile_sync_post): MEMBAR after `ofull`, off the
                // store path, then tell the store lane the newest such tile
                // (a counter, not an mbarrier phase: this warp may run two
                // tiles of its stage ahead of the store lane's check)
#ifndef FS_DIAG_NO_CFENCE
                if (total > 0) __threadfence();
#endif
                __syncwarp();
                if (lane == 0)
                    asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"(smem_u32(&cfenced[sw])),
                                 "r"((uint32_t)it)
                                 : "memory");
            }
        }
        return;
    }

    // ------------------------------- consumers -------------------------------
    const int tid = threadIdx.x;   // 0 .. TW-1
    StatAcc acc;
    // the VTiles sequence with the ring stage and output stage (and their
    // phases) advanced incrementally, and the barriers as shared-window
    // addresses: the per-tile bookkeeping is a few integer ops
    const uint32_t bars = smem_u32(smem);
    int st = 0, os = 0, ms = 0;
    uint32_t ph = 0, oph = 0;
    int key_step = 0;                 // re-spawn key of step key_step (host key for step 0)
    uint32_t rs_key = P.rs_key;
    for (VTiles V(d.n, T, K); V.valid(); V.next()) {
        const int64_t i0 = V.i0();
        const int cnt = V.cnt();
        if (RS && V.s != key_step) {
            key_step = V.s;
            rs_key = step_key(d.seed, (uint32_t)(d.step_index + (uint64_t)key_step));
        }
        mbar_wait_backoff(bars + 8u * st, ph, P.cons_wait_ns, 4 * P.cons_wait_ns);   // full[st]
        const float* slot = ring + (size_t)st * NF * T;
        float* out = IP ? ring + (size_t)st * NF * T : otile + (size_t)os * kStatePlanes * T;
#pragma unroll 1
        for (int j = 0; j < VPT; ++j) {
            // just-in-time loads from the ring: one vehicle's registers at a time
            const int c = tid + j * TW;
            const int64_t i = i0 + c;
            VState sv;
            float cmd[NC];
            float vp[4];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                sv.p[k] = slot[k * T + c];
                sv.v[k] = slot[(7 + k) * T + c];
                sv.w[k] = slot[(10 + k) * T + c];
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) sv.q[k] = slot[(3 + k) * T + c];
#pragma unroll
            for (int k = 0; k < NC; ++k) cmd[k] = slot[(kStatePlanes + k) * T + c];
#pragma unroll
            for (int k = 0; k < 4; ++k) vp[k] = HETERO ? slot[(kStatePlanes + NC + k) * T + c] : 0.0f;
            const uint32_t vmode = MIX ? (uint32_t)mring[st * T + c] : 0u;
            if (!IP && j == VPT - 1) {
                // the slot's last reads by this warp are done: release it
                // (in place the store lane does, once the slot is stored)
                __syncwarp();
                if (lane == 0) mbar_arrive_u32(bars + 8u * (STAGES + st));     // empty[st]
            }
            bool respawn = false;
            if constexpr (RS) {
                // Bernoulli re-spawn: publish the warp's ballot for this tile's
                // spawn warp (after the inputs are read: lfull also tells it
                // that the tile's command planes have been loaded, so its
                // re-spawned commands may overwrite them in global memory)
                respawn = c < cnt && reset_word_k(rs_key, d.first_id + i) < P.reset_thresh;
                const unsigned b = __ballot_sync(0xffffffffu, respawn);
                if (lane == 0) rs_mask[(size_t)ms * (T / 32) + (c >> 5)] = b;
                if (j == VPT - 1) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive_u32(bars + 8u * (2 * STAGES + 2 * kOutStages + ms));
                }
            }
            if (c < cnt) {
                StepOut o;
                uint32_t flags_all = 0;
                bool cmd_dirty = false;
                bool dummy = false;
                drive_vehicle<MODE, HETERO, PREC, NC, FEAT>(sv, cmd, vmode, vp, d.first_id + i, P,
                                                            integrate, 1, o, flags_all, cmd_dirty,
                                                            acc, RS, &dummy, RS ? (int)respawn : -1);
                if constexpr ((FEAT & kFeatOut) != 0) {
                    if (cmd_dirty) {
#pragma unroll
                        for (int k = 0; k < NC; ++k) d.cmd[k * d.cmd_stride + i] = cmd[k];
                    }
                    // outputs hold the LAST step's values: a K-step launch
                    // writes them in its last step only
                    if (d.wrench_out && V.s == K - 1) {
                        float* w = d.wrench_out + i;
                        w[0] = o.f;
                        w[d.wrench_stride] = o.m[0];
                        w[2 * d.wrench_stride] = o.m[1];
                        w[3 * d.wrench_stride] = o.m[2];
                    }
                    if (d.rotor_out && P.n_frames > 0 && V.s == K - 1) {
#pragma unroll
                        for (int r = 0; r < FS_MAX_ROTORS; ++r)
                            d.rotor_out[r * d.rotor_stride + i] = o.rotor[r];
                    }
                    if (d.flags_out && V.s == K - 1) d.flags_out[i] = (uint8_t)o.flags;
                }
            }
            // the output stage: waited for only now, after the compute, so the
            // consumers overlap their work with the store of the tile that
            // used this stage before
            if (!IP && (integrate || RS) && j == 0)
                mbar_wait_backoff(bars + 8u * (2 * STAGES + kOutStages + os), oph ^ 1u,
                                  P.cons_wait_ns, 4 * P.cons_wait_ns);
            if (integrate && !(RS && respawn)) {
                // (a re-spawned vehicle's slot is the spawn warp's)
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    out[k * T + c] = sv.p[k];
                    out[(7 + k) * T + c] = sv.v[k];
                    out[(10 + k) * T + c] = sv.w[k];
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) out[(3 + k) * T + c] = sv.q[k];
            }
        }
        if constexpr ((FEAT & kFeatOut) != 0) {
            // chained: the plain stores of the optional outputs are performed
            // at gpu scope before the tile can be published, so a later
            // launch's stores to the same addresses land after them (no
            // write-after-write race).  Within a K-step launch only the last
            // step writes them, so only its tiles pay the fence.
            if (chained && V.s == K - 1) __threadfence();
        }
        if (integrate || RS || IP) {
            // make this warp's generic-proxy writes visible to the TMA store
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive_u32(bars + 8u * (2 * STAGES + (IP ? st : os)));  // ofull
        }
        if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
        }
        if (++os == kOutStages) {
            os = 0;
            oph ^= 1u;
        }
        if (++ms == kMS) ms = 0;
    }
    if ((FEAT & kFeatStats) && d.stats_slots) {
        // consumers only (the load/store warps have left): named barrier 1
        __shared__ long long red[3][NCW];
        long long a = acc.err, b = acc.crash, c = acc.count;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            a += __shfl_xor_sync(0xffffffffu, a, o);
            b += __shfl_xor_sync(0xffffffffu, b, o);
            c += __shfl_xor_sync(0xffffffffu, c, o);
        }
        if (lane == 0) {
            red[0][warp] = a;
            red[1][warp] = b;
            red[2][warp] = c;
        }
        consumer_bar(TW);
        if (tid == 0) {
            long long sa = 0, sb = 0, sc = 0;
            for (int w = 0; w < NCW; ++w) {
                sa += red[0][w];
                sb += red[1][w];
                sc += red[2][w];
            }
            unsigned long long* sl = reinterpret_cast<unsigned long long*>(
                d.stats_slots + 3 * (blockIdx.x & (d.stats_nslots - 1)));
            atomicAdd(sl + 0, (unsigned long long)sa);
            atomicAdd(sl + 1, (unsigned long long)sb);
            atomicAdd(sl + 2, (unsigned long long)sc);
        }
    }
    // a chained step completes only after the step before it, so work
    // ordered after the chain in the stream sees every step finished (the
    // previous grid is long done by now: this step read all of its tiles)
    if (chained && d.sync_wait != 0) asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace fs

// ---- process-wide tuning (defined in fs_kernels.cu, set by fs_set_tuning) ----
namespace fs {
extern int g_kernel;        // 0 auto, 1 simple, 2 stream
extern int g_prec;          // -1 auto, 0 / 1 / 2
extern int g_ctas_per_sm;   // 0 = occupancy maximum
extern int g_ncw;           // stream consumer warps: 0 auto, 8 or 16
extern int g_vpt;           // stream vehicles per consumer thread: 0 auto, 1 or 2
extern int g_chain_release; // chained steps: fence.acq_rel.gpu before publishing
extern int g_chain_acquire; // chained steps: acquire counter loads + proxy fence
extern int g_spawn_wait_ns; // spawn warps' wait back-off (ns)
extern int g_cons_wait_ns;  // consumers' wait back-off (ns, 0 = try_wait)
extern int g_l2_keep_mb;     // streaming kernel: MiB of tiles kept L2-resident (evict_last)
int check_launch(const char* what);
int chain_unsupported();   // FS_EINVAL: tile_sync needs the streaming kernel
int device_sm_count();
bool aligned16(const void* p);

template <int MODE, bool HETERO, int PREC, int NCW, int VPT, int STAGES, int FEAT>
int launch_stream(const KParams& P, cudaStream_t s) {
    auto kern = stream_kernel<MODE, HETERO, PREC, NCW, VPT, STAGES, FEAT>;
    const size_t smem = stream_smem_bytes<MODE, HETERO, NCW, VPT, STAGES, FEAT>();
    // per-device setup: the opt-in shared-memory size and the occupancy limit
    static PerDeviceOnce once;
    static int per_dev[kMaxDevices];
    const int dev = once([&](int dv) {
        int m = 1;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, kern, stream_threads<MODE, HETERO, NCW, FEAT>(), smem);
        if (dv < kMaxDevices) per_dev[dv] = m < 1 ? 1 : m;
    });
    const int max_per_sm = dev < kMaxDevices && per_dev[dev] > 0 ? per_dev[dev] : 1;
    int sms = device_sm_count();
    if (sms <= 0) sms = 148;
    const int per_sm = g_ctas_per_sm > 0 ? std::min(g_ctas_per_sm, max_per_sm) : max_per_sm;
    const int64_t ntiles = (P.d.n + 32 * NCW * VPT - 1) / (32 * NCW * VPT);
    const unsigned grid =
        (unsigned)std::max<int64_t>(1, std::min<int64_t>(ntiles, (int64_t)sms * per_sm));
    KParams Q = P;   // (per-launch copy: the kernel parameter block)
    if (g_l2_keep_mb > 0) {
        // L2-resident tiles: their input planes (state, commands, params) fit
        // in g_l2_keep_mb MiB
        const int64_t tile_bytes =
            (int64_t)stream_float_planes<MODE, HETERO>() * 4 * (32 * NCW * VPT);
        const int64_t keep = ((int64_t)g_l2_keep_mb << 20) / tile_bytes;
        Q.l2_keep_tiles = (int32_t)std::min<int64_t>(keep, ntiles);
    }
    const bool pdl = Q.d.tile_sync != nullptr && Q.d.sync_wait != 0;
    const bool coop = Q.steps > 1;
    if (pdl || coop) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(stream_threads<MODE, HETERO, NCW, FEAT>());
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[2];
        int na = 0;
        if (pdl) {
            // a chained step: programmatic dependent of the previous step
            at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[na].val.programmaticStreamSerializationAllowed = 1;
            ++na;
        }
        if (coop) {
            // fs_step_many: CTAs wait on tiles other CTAs publish, so all of
            // them must be resident at once -- a cooperative launch
            // guarantees it (the grid is at most SMs x occupancy)
            at[na].id = cudaLaunchAttributeCooperative;
            at[na].val.cooperative = 1;
            ++na;
        }
        cfg.attrs = at;
        cfg.numAttrs = na;
        cudaLaunchKernelEx(&cfg, kern, Q);
    } else {
        kern<<<grid, stream_threads<MODE, HETERO, NCW, FEAT>(), smem, s>>>(Q);
    }
    return check_launch("stream_kernel");
}

// ring depth from the shared-memory budget (227 KB per CTA: two output tiles,
// the rest input ring)
template <int MODE, bool HETERO, int PREC, int NCW, int FEAT>
int launch_stream_w(const KParams& P, cudaStream_t s) {
    constexpr int T = 32 * NCW;
    constexpr int NF = stream_float_planes<MODE, HETERO>();
    constexpr int OST = out_stages<MODE, HETERO, NCW, FEAT>();
    constexpr int OT = out_tiles<MODE, HETERO, NCW, FEAT>();
    constexpr int S = std::min(inplace_feat(FEAT) ? 5 : 6,
                               (int)((225 * 1024 - kBarBytes - OT * 13 * T * 4 -
                                      (int)respawn_smem_bytes(FEAT, T, OST)) /
                                     (NF * T * 4 + T)));
    static_assert(S >= 2, "ring too shallow");
    static_assert(stream_smem_bytes<MODE, HETERO, NCW, 1, S, FEAT>() <= 232448, "smem budget");
    return launch_stream<MODE, HETERO, PREC, NCW, 1, S, FEAT>(P, s);
}

template <int MODE, bool HETERO, int PREC>
int launch_variant(const KParams& P, cudaStream_t s, bool rollout) {
    const fs_step_desc& d = P.d;
    const bool vec4 =
        aligned16(d.state_in) && (d.state_in_stride % 4 == 0) &&
        (!d.integrate || (aligned16(d.state_out) && d.state_out_stride % 4 == 0)) &&
        aligned16(d.cmd) && (d.cmd_stride % 4 == 0) &&
        (!d.vparams || (aligned16(d.vparams) && d.vparams_stride % 4 == 0)) &&
        (MODE != FS_MODE_MIXED || aligned16(d.mode_per_vehicle));
    const unsigned blocks = (unsigned)((d.n + kThreads - 1) / kThreads);
    if (rollout) {
        step_kernel<MODE, HETERO, PREC, 1, true><<<blocks, kThreads, 0, s>>>(P);
        return check_launch("rollout_kernel");
    }
    if (vec4 && g_kernel != 1 && (g_kernel == 2 || d.n >= (1 << 15))) {
        const bool outs = d.flags_out || d.wrench_out || d.rotor_out || P.n_frames > 0;
        const bool extra = d.stats_slots || d.reset_prob > 0.0f;
        if (!d.integrate && !outs && !extra) return FS_OK;   // control only, nothing requested
        if (outs) {
            // optional outputs / allocation: only the features the call uses
            // (re-spawn machinery and statistics cost ~60 instructions per
            // vehicle even when idle)
            if (d.reset_prob > 0.0f) return launch_stream_w<MODE, HETERO, PREC, 16, kFeatAll>(P, s);
            if (d.stats_slots)
                return launch_stream_w<MODE, HETERO, PREC, 16, kFeatOut | kFeatStats>(P, s);
            // 20 consumer warps at 80 registers, no spills (cfg4: 263 -> 249 us)
            if (g_ncw == 16) return launch_stream_w<MODE, HETERO, PREC, 16, kFeatOut>(P, s);
            return launch_stream_w<MODE, HETERO, PREC, 20, kFeatOut>(P, s);
        }
        if (extra && d.reset_prob > 0.0f) {
            constexpr int F = kFeatStats | kFeatReset;
            if (g_ncw == 12) return launch_stream_w<MODE, HETERO, PREC, 12, F>(P, s);
            if (g_ncw == 16) return launch_stream_w<MODE, HETERO, PREC, 16, F>(P, s);
            return launch_stream_w<MODE, HETERO, PREC, 20, F>(P, s);
        }
        if (extra)      // statistics only: no spawn warps
            return launch_stream_w<MODE, HETERO, PREC, 20, kFeatStats>(P, s);
        if (g_ncw == 12)
            return launch_stream_w<MODE, HETERO, PREC, 12, 0>(P, s);
        else if (g_ncw == 16)
            return launch_stream_w<MODE, HETERO, PREC, 16, 0>(P, s);
        else   // default: 20 consumer warps (measured best)
            return launch_stream_w<MODE, HETERO, PREC, 20, 0>(P, s);
    }
    if (d.tile_sync != nullptr || P.steps > 1) return chain_unsupported();
    step_kernel<MODE, HETERO, PREC, 1, false><<<blocks, kThreads, 0, s>>>(P);
    return check_launch("step_kernel");
}

// default controller precision (fs_set_tuning(FS_TUNE_PREC, -1)); DESIGN.md 4.2
constexpr int kDefaultPrec = 2;

// per-mode entry points (one translation unit each)
int launch_attitude(const KParams& P, cudaStream_t s, bool rollout);
int launch_velocity(const KParams& P, cudaStream_t s, bool rollout);
int launch_mixed(const KParams& P, cudaStream_t s, bool rollout);
int launch_position(const KParams& P, cudaStream_t s, bool rollout);

template <int MODE>
int launch_mode_prec(const KParams& P, cudaStream_t s, bool rollout) {
    const bool het = P.d.vparams != nullptr;
    {
        const int prec = g_prec < 0 ? kDefaultPrec : g_prec;
        if (prec == 0)
            return het ? launch_variant<MODE, true, 0>(P, s, rollout)
                       : launch_variant<MODE, false, 0>(P, s, rollout);
        if (prec == 1)
            return het ? launch_variant<MODE, true, 1>(P, s, rollout)
                       : launch_variant<MODE, false, 1>(P, s, rollout);
        return het ? launch_variant<MODE, true, 2>(P, s, rollout)
                   : launch_variant<MODE, false, 2>(P, s, rollout);
    }
}

}  // namespace fs
