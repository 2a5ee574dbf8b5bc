/*
 * flocksim_b200.h -- C ABI of the B200-native batched multirotor control step.
 *
 * This is the drop-in boundary for the reference's hot path
 * (flocksim.control.control_batch -> flocksim.dynamics.step_batch, see
 * SURVEY.md section 8(b)).  The reference exposes that path as module-level
 * pure Python functions over NumPy dataclasses; every entry point below
 * replaces one of them and names the reference interface it replaces
 * (paths relative to /root/reference/pkg/src/flocksim).
 *
 * Conventions (all entry points):
 *   - caller-owned DEVICE pointers; the library never allocates, never
 *     synchronises, and launches asynchronously on the caller's stream
 *     (a cudaStream_t passed as void*, NULL = legacy default stream);
 *   - structure-of-arrays fp32 "planes": component k of vehicle i lives at
 *     base[k * stride + i].  A state has 13 planes
 *       px py pz | qw qx qy qz | vx vy vz | wx wy wz
 *     (world position m, body->world unit quaternion scalar-first, world
 *     velocity m/s, body rate rad/s -- dynamics.py:93-131);
 *   - 16-byte aligned bases with stride % 4 == 0 select the float4 path;
 *     anything else runs the scalar path (same results);
 *   - return value: FS_OK or an FS_E* status.  Argument errors are detected
 *     before any launch.  Per-vehicle numerical failures are NOT errors:
 *     they are reported in the per-vehicle flag byte (dynamics.py:203-211,
 *     control.py:182-187), as the reference does.
 */
#ifndef FLOCKSIM_B200_H
#define FLOCKSIM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FS_ABI_VERSION 8

/* status codes */
#define FS_OK 0
#define FS_EINVAL 22       /* bad argument (length, dt, null, mode ...) */
#define FS_ELAUNCH 1001    /* CUDA launch failed (see fs_last_error) */

/* command modes (control.py:29-30 for 0/1; 2 = per-vehicle tagged union,
 * CommandBatch control.py:140-171; 3 = position: EXTENSION) */
#define FS_MODE_ATTITUDE 0
#define FS_MODE_VELOCITY 1
#define FS_MODE_MIXED 2
#define FS_MODE_POSITION 3

/* element types of caller-supplied action rows (fs_vecenv_step) */
#define FS_DTYPE_F32 0
#define FS_DTYPE_F64 1

/* per-vehicle flag bits (one uint8 per vehicle) */
#define FS_FLAG_CLAMPED 1     /* StepFlags.clamped      dynamics.py:207 */
#define FS_FLAG_NONFINITE 2   /* StepFlags.nonfinite    dynamics.py:208 */
#define FS_FLAG_GIMBAL 4      /* ControlFlags.gimbal_degenerate   control.py:186 */
#define FS_FLAG_DEGENERATE 8  /* ControlFlags.degenerate_acceleration control.py:187 */
#define FS_FLAG_RESET 16      /* vehicle was re-spawned this step (EXTENSION) */

/* RobotParams (dynamics.py:38-90), float64 like the reference: the float64
 * controller uses these values as given, the fp32 paths round them once.
 * inertia_inv is computed by the caller in float64 (dynamics.py:82). */
typedef struct fs_robot {
    double mass;
    double gravity;
    double inertia[9];       /* row-major J, kg m^2 */
    double inertia_inv[9];   /* row-major J^-1 */
    double thrust_max;
    double moment_max[3];
    double v_limit;
    double omega_limit;
    double gimbal_cos;       /* cos(GIMBAL_TOL) (se3.py:25,242) */
} fs_robot;

/* ControlGains (control.py:40-59) + position gain k_p (EXTENSION). */
typedef struct fs_gains {
    double attitude[3];
    double rate[3];
    double velocity[3];
    double position[3];
} fs_gains;

/* ControlLimits (control.py:62-74). */
typedef struct fs_limits {
    double max_tilt;
    double max_speed_cmd;
    double max_yaw_rate;
} fs_limits;

/* Rotor geometry for wrench -> rotor-thrust allocation (EXTENSION, no
 * reference counterpart).  pinv is A^+ (n_rotors x 4,
 * row-major), alloc is A (4 x n_rotors, row-major). */
#define FS_MAX_ROTORS 6
typedef struct fs_airframe {
    int32_t n_rotors;                    /* 0 = no allocation, 4 or 6 */
    float rotor_max;                     /* per-rotor thrust limit, N */
    float pinv[FS_MAX_ROTORS * 4];
    float alloc[4 * FS_MAX_ROTORS];
} fs_airframe;

/* One fused control (+ optional integration) step over n vehicles.
 * Replaces control_batch (control.py:352-386) followed by step_batch
 * (dynamics.py:238-264), i.e. bench._pipeline_step (bench.py:146-149) and
 * World._pipeline (world.py:254-257).
 *
 * Command planes by mode (cmd + k*cmd_stride):
 *   ATTITUDE: roll, pitch, yaw_rate, thrust        (AttitudeCommands, control.py:77-95)
 *   VELOCITY: vx, vy, vz (vehicle frame), yaw_rate (VelocityCommands, control.py:115-126)
 *   MIXED:    the 4 attitude planes then the 4 velocity planes, plus
 *             mode_per_vehicle[i] in {0, 1}        (CommandBatch, control.py:140-171)
 *   POSITION: px_d, py_d, pz_d, yaw_d              (EXTENSION)
 */
typedef struct fs_step_desc {
    int64_t n;                  /* vehicles in this call (shard) */
    int64_t first_id;           /* global id of vehicle 0 (RNG keying, airframe split) */
    const float* state_in;      /* 13 planes */
    int64_t state_in_stride;
    float* state_out;           /* 13 planes; may alias state_in (in-place) */
    int64_t state_out_stride;
    int32_t mode;               /* FS_MODE_* */
    int32_t integrate;          /* 0: control only (control_batch); 1: fused step */
    const uint8_t* mode_per_vehicle;   /* FS_MODE_MIXED only */
    float* cmd;                 /* command planes (written only by resets) */
    int64_t cmd_stride;
    const float* vparams;       /* NULL, or 4 planes: mass, Jxx, Jyy, Jzz (EXTENSION) */
    int64_t vparams_stride;
    int64_t airframe_split;     /* global ids < split use airframe[0], others airframe[1] */
    float* wrench_out;          /* NULL, or 4 planes: thrust, Mx, My, Mz (saturated) */
    int64_t wrench_stride;
    float* rotor_out;           /* NULL, or FS_MAX_ROTORS planes of rotor thrust */
    int64_t rotor_stride;
    uint8_t* flags_out;         /* NULL, or one FS_FLAG_* byte per vehicle */
    int32_t rotor_dynamics;     /* 1: integrate the realized wrench A*clip(A^+ w) */
    float dt;                   /* (0, 0.1] (dynamics.py:257-258) */
    float reset_prob;           /* per-step Bernoulli re-spawn probability (EXTENSION) */
    uint64_t seed;
    uint64_t step_index;        /* counter of this step (RNG stream) */
    int64_t* stats_slots;       /* NULL, or nslots x 3 int64: sum|p-p_d|*2^20, crashes, samples */
    int32_t stats_nslots;       /* power of two */
    /* Chained in-place steps (EXTENSION; no reference counterpart).  NULL, or
     * fs_tile_sync_len(n) uint32 counters, one per FS_SYNC_GRANULE vehicles:
     * once a step's stores of a tile have completed it publishes sync_post on
     * the tile's counters (strong gpu-scope stores after the bulk-store
     * completion wait).  With sync_wait != 0 the step
     * loads a tile only once its counters have reached sync_wait (strong
     * loads; wrap-safe comparison) and is launched as a programmatic dependent of
     * the previous kernel in the stream, so consecutive steps overlap
     * (a step's first tiles start while the previous step drains).  Only the
     * streaming kernel takes part (16-byte aligned planes, n >= 2^15);
     * otherwise fs_step fails with FS_EINVAL.  The caller zeroes the counters
     * before a chain and posts 1, 2, ... (wait 0, 1, ...).  The counter
     * check is fenced against the tile's TMA reads (fence.proxy.async;
     * FS_TUNE_CHAIN_ACQUIRE adds gpu-scope acquires).  A wait
     * not satisfied within FS_TUNE_SYNC_TIMEOUT_MS (default 10 s; 0 = never)
     * traps (a kernel error, not a hang).
     * fs_step_many uses the same counters between the steps of one launch:
     * its step s waits for sync_wait + s and publishes sync_post + s. */
    uint32_t* tile_sync;
    uint32_t sync_wait;
    uint32_t sync_post;
} fs_step_desc;

#define FS_SYNC_GRANULE 128
/* counters a chained fs_step over n vehicles needs: ceil(n / FS_SYNC_GRANULE) */
int64_t fs_tile_sync_len(int64_t n);

/* ---- library ------------------------------------------------------------ */
int fs_abi_version(void);

/* Process-wide kernel selection (benchmarking / diagnostics; defaults are
 * the production choice).  No reference counterpart. */
#define FS_TUNE_KERNEL 1        /* 0 auto, 1 simple (registers), 2 stream (TMA ring) */
#define FS_TUNE_PREC 2          /* -1 auto (2), 0 fp32, 1 fp64 velocity front end, 2 fp64 controller */
#define FS_TUNE_CTAS_PER_SM 3   /* stream kernel CTAs per SM, 0 = occupancy max */
#define FS_TUNE_NCW 4           /* stream kernel consumer warps: 0 auto (16), 12, 16 or 20 */
#define FS_TUNE_VPT 5           /* register kernel only: reserved */
#define FS_TUNE_WORLD_KERNEL 6  /* free-space World.step: 0 auto, 1 thread per env, 2 streaming */
#define FS_TUNE_CHAIN_RELEASE 7 /* chained steps: 0 publish after bulk-store completion, 1 + gpu-scope fence */
#define FS_TUNE_L2_KEEP_MB 8    /* streaming kernel: MiB of tiles kept L2-resident across steps (evict_last), 0 = off */
#define FS_TUNE_SYNC_TIMEOUT_MS 9 /* chained steps: a tile wait longer than this traps (default 10000; 0 = wait forever) */
#define FS_TUNE_SPAWN_WAIT_NS 11  /* streaming kernel: spawn warps' nanosleep back-off start, ns (default 0 = try_wait) */
#define FS_TUNE_CONS_WAIT_NS 12   /* streaming kernel: consumers' back-off start, ns (default 0 = try_wait) */
#define FS_TUNE_CLEAR_WALK_CM 13  /* obstacle worlds: instances within this many cm are walked slot by slot when the clearance cache is refreshed (default 60) */
#define FS_TUNE_CLEAR_EXACT 14    /* obstacle worlds: 1 (default) walked slots bound the clearance by their exact SDF, 0 by their AABB */
#define FS_TUNE_CHAIN_ACQUIRE 10  /* chained steps, load side: bit 0 gpu-scope acquire counter loads, bit 1 fence.proxy.async before the tile's TMA loads (default 2), bit 2 fence.acq_rel.gpu after the counter loads */
int fs_set_tuning(int32_t key, int32_t value);
const char* fs_last_error(void);
int fs_device_sm_count(void);

/* ---- the hot path ------------------------------------------------------- */

/* control_batch (+ step_batch when d->integrate) -- control.py:352-386,
 * dynamics.py:238-264.  Pure when state_out != state_in. */
int fs_step(const fs_step_desc* d, const fs_robot* robot, const fs_gains* gains,
            const fs_limits* limits, const fs_airframe* frames /* [2] or NULL */,
            void* stream);

/* `steps` consecutive fused steps (control + integration, in place or
 * state_in -> state_out) in ONE persistent launch of the streaming kernel:
 * step s uses step_index + s (RNG keys) and, like fs_step, reads state and
 * commands from and writes state to global memory -- the same bytes and the
 * same results (bitwise) as `steps` fs_step calls -- but the tile pipeline
 * runs on from one step into the next instead of draining at a launch
 * boundary.  Tile t of step s + 1 waits for tile t of step s through
 * tile_sync (required when steps > 1; step s waits for sync_wait + s and
 * publishes sync_post + s, sync_post == sync_wait + 1; zeroed counters and
 * sync_wait 0 start a chain).  Optional outputs (wrench, rotor thrusts,
 * flags) hold the last step's values and are written in the last step only;
 * statistics accumulate over all steps.  EXTENSION (no reference
 * counterpart; the reference loop is bench._pipeline_step, bench.py:146-149). */
int fs_step_many(const fs_step_desc* d, const fs_robot* robot, const fs_gains* gains,
                 const fs_limits* limits, const fs_airframe* frames /* [2] or NULL */,
                 int32_t steps, void* stream);

/* fs_step on HOST-resident data (the call a NumPy-side caller makes):
 * d->state_in, d->state_out and d->cmd (and d->mode_per_vehicle) are host
 * pointers (pinned for full PCIe speed) with the usual plane strides;
 * dev_state (13 planes) and dev_cmd (command planes) are caller-owned device
 * workspaces with plane stride dev_stride >= n.  The batch is cut into
 * `chunks` slices; slice c runs on streams[c % nstreams]: one
 * cudaMemcpy2DAsync per array host->device, fs_step, one cudaMemcpy2DAsync
 * device->host.  Asynchronous: synchronise the streams before reading
 * d->state_out. */
int fs_step_host(const fs_step_desc* d, const fs_robot* robot, const fs_gains* gains,
                 const fs_limits* limits, const fs_airframe* frames, float* dev_state,
                 float* dev_cmd, int64_t dev_stride, int32_t chunks, void* const* streams,
                 int32_t nstreams);

/* Device workspace and streams of fs_step_host_ex.  Every array is caller
 * owned with plane stride dev_stride (>= n, a multiple of 4). */
typedef struct fs_host_ws {
    float* dev_state;           /* 13 planes */
    float* dev_cmd;             /* command planes: 8 for FS_MODE_MIXED, else 4 */
    uint8_t* dev_mode;          /* n bytes; FS_MODE_MIXED only */
    float* dev_wrench;          /* 4 planes; only when d->wrench_out is set */
    uint8_t* dev_flags;         /* n bytes; only when d->flags_out is set */
    int64_t dev_stride;
    int32_t chunks;             /* the batch is cut into this many slices */
    int32_t nstreams;           /* slice c runs on streams[c % nstreams] */
    void* const* streams;
} fs_host_ws;

/* fs_step_host for every caller-visible output of the reference's pair
 * control_batch (control.py:352-386) -> step_batch (dynamics.py:238-264)
 * on HOST buffers -- the call a NumPy-side caller (flocksim's World._pipeline,
 * world.py:254-257, or bench._pipeline_step, bench.py:146-149) makes:
 * d->state_in / state_out, d->cmd, d->mode_per_vehicle (FS_MODE_MIXED),
 * d->wrench_out (NULL or 4 host planes: the saturated wrench) and
 * d->flags_out (NULL or n host bytes of FS_FLAG_*) are host pointers
 * (pinned for full PCIe speed).  Per slice: H2D copies of state, commands
 * and modes, fs_step, D2H copies of the new state (when integrating), the
 * wrench and the flags.  Asynchronous on the workspace streams.
 * Rotor outputs, per-vehicle parameters, statistics, re-spawns and chaining
 * are device-side features (FS_EINVAL here). */
int fs_step_host_ex(const fs_step_desc* d, const fs_robot* robot, const fs_gains* gains,
                    const fs_limits* limits, const fs_airframe* frames /* [2] or NULL */,
                    const fs_host_ws* ws);

/* Host-side layout conversion for NumPy callers of fs_step_host(_ex) (the
 * reference's float64 (n, w) row arrays, e.g. RigidStateBatch.p, against the
 * library's fp32 planes), split over `nthreads` host threads (<= 0: all
 * hardware threads).  pack: dst[k * plane_stride + i] = (float)src[i * ld + k]
 * (round to nearest); unpack: dst[i * ld + k] = src[k * plane_stride + i].
 * No reference counterpart (compat.py uses them around fs_step_host_ex). */
int fs_host_pack_f64(const double* src, int64_t n, int32_t w, int64_t ld, float* dst,
                     int64_t plane_stride, int32_t nthreads);
int fs_host_unpack_f64(const float* src, int64_t plane_stride, int64_t n, int32_t w,
                       double* dst, int64_t ld, int32_t nthreads);

/* `steps` consecutive fused steps with the vehicle state held in registers
 * (commands constant over the rollout, as in bench_dynamics, bench.py:161-167).
 * Step t uses RNG counter d->step_index + t.  Result equals `steps` calls of
 * fs_step on the same descriptor. */
int fs_rollout(const fs_step_desc* d, const fs_robot* robot, const fs_gains* gains,
               const fs_limits* limits, const fs_airframe* frames, int32_t steps,
               void* stream);

/* step_batch on given wrenches -- dynamics.py:238-264 / _step_kernel 286-341.
 * wrench: 4 planes thrust, Mx, My, Mz (already saturated by the caller, as
 * the reference expects).  flags_out: CLAMPED | NONFINITE. */
int fs_integrate(int64_t n, const float* state_in, int64_t state_in_stride,
                 const float* wrench, int64_t wrench_stride, const fs_robot* robot,
                 float dt, float* state_out, int64_t state_out_stride,
                 uint8_t* flags_out, void* stream);

/* saturate_batch -- dynamics.py:214-218 (in 4 planes -> out 4 planes). */
int fs_saturate(int64_t n, const float* wrench_in, int64_t in_stride,
                const fs_robot* robot, float* wrench_out, int64_t out_stride, void* stream);

/* velocity_control -- control.py:283-349.  Outputs 4 planes roll, pitch,
 * yaw_rate, thrust and one degenerate byte (0/1) per vehicle. */
int fs_velocity_control(int64_t n, const float* state, int64_t state_stride,
                        const float* vcmd, int64_t vcmd_stride, const fs_robot* robot,
                        const fs_gains* gains, const fs_limits* limits,
                        float* att_out, int64_t att_stride, uint8_t* degenerate_out,
                        void* stream);

/* attitude_control -- control.py:261-280 (saturated wrench, 4 planes). */
int fs_attitude_control(int64_t n, const float* state, int64_t state_stride,
                        const float* acmd, int64_t acmd_stride, const fs_robot* robot,
                        const fs_gains* gains, float* wrench_out, int64_t wrench_stride,
                        void* stream);

/* se3.yaw_of -- se3.py:226-243: yaw (1 plane) and gimbal byte per vehicle. */
int fs_yaw_of(int64_t n, const float* q, int64_t q_stride, double gimbal_cos,
              float* yaw_out, uint8_t* gimbal_out, void* stream);

/* desired_attitude -- control.py:190-218.  yaw (1 plane), attitude command
 * planes (roll, pitch, yaw_rate, ...) -> q_d (4 planes), omega_d (3 planes). */
int fs_desired_attitude(int64_t n, const float* yaw, const float* acmd, int64_t acmd_stride,
                        float* qd_out, int64_t qd_stride, float* wd_out, int64_t wd_stride,
                        void* stream);

/* attitude_errors -- control.py:221-258.  q (4), omega (3), q_d (4),
 * omega_d (3) planes -> e_R (3), e_W (3) planes. */
int fs_attitude_errors(int64_t n, const float* q, int64_t q_stride, const float* omega,
                       int64_t omega_stride, const float* qd, int64_t qd_stride,
                       const float* wd, int64_t wd_stride, float* erot_out,
                       float* erate_out, int64_t err_stride, void* stream);

/* ---- obstacle scenes -------------------------------
 * The per-environment primitive soup of scene.py:PrimitiveSet (scene.py:24-59),
 * padded to a common width K, stored on the device as one 96-byte record per
 * (env, slot): record k of env e at rec[(e * width + k) * FS_PRIM_FIELDS],
 * six 16-byte groups
 *   [aabb_min xyz, kind] [aabb_max xyz, collision] [dims xyz, seg_id]
 *   [position xyz, R22] [R00 R01 R02 R10] [R11 R12 R20 R21]
 * (R row-major, local -> env; kind / collision / seg_id as int32 bit
 * patterns; AABB rounded outward to fp32).  A thread reads a slot with two
 * (bounds test) or six (full primitive) vector loads.
 * Kinds follow scene.py:20-21 (0 box, 1 cylinder, 2 sphere, -1 pad).
 * collision: 0 disabled, 1 enabled, FS_COLL_WALL for the World's wall slabs
 * (enabled; the World's collision and placement tests skip them because a
 * wall contact is exactly the env-bounds test, world.py:74-106). */
#define FS_PRIM_PAD (-1)
#define FS_PRIM_BOX 0
#define FS_PRIM_CYLINDER 1
#define FS_PRIM_SPHERE 2
#define FS_PRIM_FIELDS 24
#define FS_COLL_WALL 2

typedef struct fs_scene {
    int64_t num_envs;
    int32_t width;              /* K slots per env */
    int32_t reserved_;
    float* rec;                 /* num_envs * width records, 16-byte aligned */
} fs_scene;

/* One primitive of an asset prototype, asset-local (assets.py:70-90). */
typedef struct fs_proto_prim {
    int32_t kind;
    int32_t reserved_;
    double dims[3];
    double position[3];
    double rotation[4];         /* scalar-first quaternion */
} fs_proto_prim;

/* AssetClassConfig (assets.py:125-166) plus its prototype pool range. */
typedef struct fs_asset_class {
    double position_min[3], position_max[3];  /* fractions of the env bounds */
    double euler_min[3], euler_max[3];        /* ZYX euler, rad */
    double frozen_value[3];                   /* used where frozen_mask bit i is set */
    int32_t frozen_mask;
    int32_t segmentation_id;
    int32_t collision_enabled;
    int32_t count_per_env;
    int32_t pool_first;         /* prototypes [pool_first, pool_first + pool_size) */
    int32_t pool_size;
} fs_asset_class;

/* Everything World.reset_env needs to re-randomize obstacles on the device
 * (world.py:229-243): class table, prototype table, per-env instance picks
 * and poses, the wall prototype, and the camera mounts (camera.py:238-244).
 * All pointers are device memory. */
typedef struct fs_obstacles {
    fs_scene scene;
    int32_t num_classes;
    int32_t instances_per_env;  /* J = sum of count_per_env */
    const fs_asset_class* classes;
    const int32_t* proto_offset;     /* num_protos + 1 primitive ranges */
    const fs_proto_prim* proto_prims;
    int64_t plane_stride;       /* stride of the per-env planes below (>= num envs) */
    int32_t* inst_proto;        /* J planes: prototype id of instance j */
    double* inst_pose;          /* NULL or 7 J planes: position(3), quaternion(4) */
    int32_t wall_proto;         /* prototype id of the walls (make_wall_prototype), -1 none */
    int32_t wall_seg;
    double* mount;              /* NULL (no camera) or 7 planes: mount p(3), q(4) */
    int64_t mount_stride;
    double mount_position[3], mount_euler[3];
    double randomize_position[3], randomize_euler[3];
    float* inst_box;            /* NULL, or the collision broad phase (written by the
                                   resets): per env J records of two float4, instance-major:
                                   half h of record j of env e at
                                   inst_box[((2 j + h) * plane_stride + e) * 4]; h = 0:
                                   AABB lo xyz, slot span (int bits: first | count << 16);
                                   h = 1: AABB hi xyz, collision flag (1.0 / 0.0);
                                   16-byte aligned */
    float* clear;               /* NULL, or (with inst_box) the collision clearance cache:
                                   4 planes of plane_stride floats per env, (x, y, z) of the
                                   point where the broad phase last ran and c = a lower bound
                                   of the distance from it to every collision-enabled
                                   instance box (c < 0: invalid).  A step whose robot moved
                                   less than c - collision_radius from that point cannot
                                   touch a primitive and skips the test (same result).
                                   Written by fs_world_step, invalidated by every reset;
                                   the caller invalidates it when it rewrites states or
                                   scene rows. */
    int32_t* worklist;          /* NULL, or (with clear) n + 3 int32, zeroed once by the
                                   caller: fs_world_step then defers the collision test of
                                   the envs the cache does not clear to a second kernel
                                   over this compact list ([0] count, [1] blocks done,
                                   [2] running total of tested envs, [3..] env ids), which
                                   patches their collision bits,
                                   termination, pending flag and reward; it leaves the list
                                   empty again.  Same results as the inline test. */
    int32_t* reset_list;        /* NULL, or (with worklist) n + 4 int32, zeroed once by the
                                   caller: the streaming step then DEFERS the auto-resets.
                                   It skips every env pending when the step starts (its
                                   step is voided) and lists it ([0] count, [3] next entry
                                   to take, [4..] env ids); a second kernel resets the
                                   listed envs after the step -- every output of the reset
                                   -- in one task pool with the deferred collision test,
                                   and empties the list.  Same results as resetting first
                                   (world.py:287-299).  Words [1] and [2] are unused. */
    int64_t* walk_slots;        /* NULL, or one int64 zeroed once by the caller: running
                                   total of the slot records (96 B each) the deferred
                                   collision test read (measurement: the test's
                                   data-dependent bytes) */
} fs_obstacles;

/* ---- free-space World.step on the GPU -------------
 * The reference's environment step (world.py:277-342) for a world without
 * obstacles or camera: pending auto-resets first (re-spawn at rest + new goal,
 * step voided), then the fused control step for everyone else, collision
 * against the env box (world.py:95-106), episode counters,
 * terminated/truncated, the goal-reaching reward (world.py:109-116) and the
 * 16-value observation (world.py:331-342).  Per-env re-spawn draws use the
 * library's Philox4x32-10 keyed by (seed, env id, reset counter) instead of
 * NumPy's Philox-4x64 (assets.py:310-315). */
#define FS_INFO_TERMINATED 1
#define FS_INFO_TRUNCATED 2
#define FS_INFO_COLLISION 4
#define FS_INFO_OUT_OF_BOUNDS 8
#define FS_INFO_NONFINITE 16
#define FS_INFO_AUTORESET 32
#define FS_INFO_PLACEMENT_FAILED 64  /* no free in-bounds point in placement_attempts draws */

typedef struct fs_world_cfg {
    double bounds[3];              /* EnvConfig.bounds (config.py:41) */
    double spawn_lo[3], spawn_hi[3];  /* EnvConfig.spawn_min/max, fractions of bounds */
    double goal_lo[3], goal_hi[3];    /* EnvConfig.goal_min/max */
    double collision_radius;       /* RobotParams.collision_radius */
    int32_t episode_max_steps;
    int32_t placement_attempts;    /* world.py:38 PLACEMENT_ATTEMPTS = 100 */
    double c_dist, c_vel, c_step, c_success, c_crash, success_radius;  /* RewardConfig */
} fs_world_cfg;

typedef struct fs_world_desc {
    fs_step_desc step;             /* state (updated in place), commands, mode, dt, seed,
                                      first_id (global env id of env 0) */
    float* goal;                   /* 3 planes */
    int64_t goal_stride;
    int32_t* steps_in_episode;
    int32_t* reset_counter;
    uint8_t* pending_reset;
    float* obs;                    /* 16 planes: p, q, v, w, goal - p in the vehicle frame */
    int64_t obs_stride;
    float* reward;
    uint8_t* info;                 /* FS_INFO_* bits */
    const fs_obstacles* obstacles; /* NULL: free space; else the obstacle scene
                                      (collisions world.py:95-106, resets 229-243) */
} fs_world_desc;

/* World.step: returns observations, reward, terminated/truncated and info
 * through the descriptor's planes.  With w->obstacles the collision test
 * adds the primitives (min signed distance < collision_radius, world.py:100)
 * and auto-resets re-randomize the env's obstacles as fs_world_reset does. */
int fs_world_step(const fs_world_desc* w, const fs_world_cfg* cfg, const fs_robot* robot,
                  const fs_gains* gains, const fs_limits* limits, void* stream);

/* World.reset_env / reset_all (world.py:229-252): for envs with mask[e] != 0
 * (mask NULL = all), reset_counter += increment, draw spawn + goal, robot at
 * rest, steps = 0, pending = 0, observation written.  increment = 0 is the
 * creation-time placement (counter 0, world.py:160-176).  With w->obstacles
 * the env's obstacles get fresh poses first (prototypes kept, walls
 * unchanged, rows recompiled and padded), spawn and goal must also clear
 * every collision-enabled primitive by collision_radius (world.py:196-211),
 * and the camera mount is re-drawn when ob->mount is set. */
int fs_world_reset(const fs_world_desc* w, const fs_world_cfg* cfg, const uint8_t* mask,
                   int32_t increment, void* stream);

/* flocksim_rl VecEnvHandle.step (pkg/bindings/src/flocksim_rl/vec_env.py:85-126)
 * fused into World.step's command load.  `actions`
 * are E rows of ACTION_DIM = 4 values (row stride `action_stride` elements,
 * a multiple of 4; 16-byte aligned device memory; FS_DTYPE_F32 or _F64).
 * Each row is clipped to [-1, 1] and denormalized in float64 exactly as
 * vec_env.py:91-104 does:
 *   attitude: (a0 max_tilt, a1 max_tilt, a2 max_yaw_rate, (a3 + 1) / 2 thrust_max)
 *   velocity: (a0 max_speed_cmd, a1 max_speed_cmd, a2 max_speed_cmd, a3 max_yaw_rate)
 * and drives one World.step (w->step.mode: attitude or velocity;
 * w->step.cmd is not read).  Non-finite actions are the caller's check
 * (the reference raises InvalidCommandError building the CommandBatch). */
int fs_vecenv_step(const fs_world_desc* w, const fs_world_cfg* cfg, const fs_robot* robot,
                   const fs_gains* gains, const fs_limits* limits, const void* actions,
                   int32_t action_dtype, int64_t action_stride, void* stream);

/* ---- scene queries and the depth camera ------------ */

/* scene.signed_distances / min_distance (scene.py:127-181): one fp32 query
 * point per env (3 planes).  dist_out (NULL or width planes, float64): the
 * signed distance to every slot, +inf on pads.  min_out (NULL or E float64):
 * the smallest over collision-enabled slots (all non-pad slots when
 * collision_only == 0), +inf when there is none. */
int fs_scene_distances(const fs_scene* s, const float* points, int64_t point_stride,
                       int32_t collision_only, double* dist_out, int64_t dist_stride,
                       double* min_out, void* stream);

/* camera.cast_rays (camera.py:230-282): m rays from a common origin (env
 * frame) with unit directions dirs (m x 3 row-major float64, device) against
 * env `env`'s collision-enabled primitives.  depth_out (m float64): nearest
 * hit, max_range where none within max_range; seg_out (m int32): its
 * segmentation id, 0 on a miss. */
int fs_cast_rays(const fs_scene* s, int64_t env, double ox, double oy, double oz,
                 const double* dirs, int64_t m, double max_range, double* depth_out,
                 int32_t* seg_out, void* stream);

/* CameraConfig (camera.py:39-69) reduced to what a render needs. */
typedef struct fs_camera {
    int32_t width, height;
    double pixel_scale;         /* 2 tan(hfov / 2) / width (camera.py:123-130) */
    double max_range;
    double mount_position[3];   /* used when the mount planes are NULL */
    double mount_rotation[4];
} fs_camera;

/* camera.render (camera.py:247-282) for envs [first_env, first_env + n):
 * camera at p + R(q) mount_p, orientation q (x) mount_q, per-pixel rays of a
 * pinhole with square pixels, nearest collision-enabled primitive.  state: 13
 * fp32 planes (indexed by env); mount: NULL or 7 float64 planes p(3), q(4).
 * depth_out: n x height x width float32 (Euclidean range, max_range on a
 * miss); seg_out: n x height x width int32 (0 on a miss). */
int fs_render(const fs_scene* s, const fs_camera* cam, const float* state, int64_t state_stride,
              const double* mount, int64_t mount_stride, int64_t first_env, int64_t n,
              float* depth_out, int32_t* seg_out, void* stream);

/* World creation's prototype picks (assets.py:335-356, counter 0 of each
 * env's stream): fills ob->inst_proto for envs [0, n) and writes each env's
 * primitive count (walls included) to count_out, from which the caller
 * sizes the scene width (max over envs, scene.py:92). */
int fs_obstacles_pick(const fs_obstacles* ob, int64_t n, int64_t first_id, uint64_t seed,
                      int32_t* count_out, void* stream);

/* The instance poses of envs [0, n) at their reset counters (device
 * reset_counter[e]; host bounds[3] = EnvConfig.bounds) into ob->inst_pose:
 * World.instances' positions and rotations (world.py:165-176, 233-240) on
 * demand.  World.step's resets do not write the pose planes (pass
 * inst_pose = NULL there); the poses are a pure function of (seed, env id,
 * counter), so this reproduces what they would have written. */
int fs_obstacles_poses(const fs_obstacles* ob, int64_t n, int64_t first_id, uint64_t seed,
                       const int32_t* reset_counter, const double* bounds, void* stream);

/* ---- se3: rotation-group primitives (se3.py:32-266) -------------------------
 * Batched float64 rows, contiguous (the reference's trailing (..., k) layout).
 * fs_se3(op, n, a, b, c, out, out2): per op,
 *   QUAT_NORMALIZE      a q(n,4)              -> out (n,4)          se3.py:70-75
 *   QUAT_MULTIPLY       a q1(n,4), b q2(n,4)  -> out (n,4)          se3.py:78-97
 *   QUAT_CONJUGATE      a q(n,4)              -> out (n,4)          se3.py:100-103
 *   QUAT_ROTATE         a q(n,4), b v(n,3)    -> out (n,3)          se3.py:106-130
 *   QUAT_ROTATE_INVERSE a q(n,4), b v(n,3)    -> out (n,3)          se3.py:133-135
 *   QUAT_TO_MATRIX      a q(n,4)              -> out (n,9) row-major se3.py:138-153
 *   QUAT_FROM_MATRIX    a R(n,9)              -> out (n,4)          se3.py:156-197
 *   ROT_ZYX             a roll, b pitch, c yaw (n each) -> out (n,4) se3.py:200-215
 *   ROT_Z               a yaw (n)             -> out (n,4)          se3.py:218-223
 *   YAW_OF              a q(n,4) -> out psi (n), out2 gimbal flag 0/1 (n)  se3.py:226-243
 *   EXP_SO3             a w(n,3)              -> out (n,4)          se3.py:246-266
 *   HAT                 a w(n,3)              -> out (n,9)          se3.py:32-48
 *   VEE                 a S(n,9) -> out (n,3), out2 per-row max |S + S^T| (the
 *                       caller raises NotSkewSymmetricError above SKEW_TOL)  se3.py:51-67 */
#define FS_SE3_QUAT_NORMALIZE 0
#define FS_SE3_QUAT_MULTIPLY 1
#define FS_SE3_QUAT_CONJUGATE 2
#define FS_SE3_QUAT_ROTATE 3
#define FS_SE3_QUAT_ROTATE_INVERSE 4
#define FS_SE3_QUAT_TO_MATRIX 5
#define FS_SE3_QUAT_FROM_MATRIX 6
#define FS_SE3_ROT_ZYX 7
#define FS_SE3_ROT_Z 8
#define FS_SE3_YAW_OF 9
#define FS_SE3_EXP_SO3 10
#define FS_SE3_HAT 11
#define FS_SE3_VEE 12
int fs_se3(int32_t op, int64_t n, const double* a, const double* b, const double* c,
           double* out, double* out2, void* stream);

/* ---- workload generation / statistics (EXTENSIONS) ----------------------- */

/* Seeded counter-based (Philox4x32-10) generator of the BASELINE.json
 * config distributions, keyed by (seed, global id): state (13 planes), the
 * command planes of `mode`, and optionally per-vehicle parameter planes. */
int fs_init_fleet(int64_t n, int64_t first_id, uint64_t seed, int32_t mode,
                  float* state, int64_t state_stride, float* cmd, int64_t cmd_stride,
                  float* vparams, int64_t vparams_stride, const fs_robot* robot,
                  void* stream);

/* Sum the nslots x 3 int64 statistic slots into out[3]. */
int fs_stats_reduce(const int64_t* slots, int32_t nslots, int64_t* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FLOCKSIM_B200_H */
