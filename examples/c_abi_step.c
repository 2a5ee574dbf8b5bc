/*
 * c_abi_step.c -- the drop-in boundary used from plain C (no Python, no torch).
 *
 * A maintainer binding flocksim's hot path (control_batch + step_batch,
 * pkg/src/flocksim/control.py:352-386, dynamics.py:238-264) from another
 * host language links libflocksim_b200.so and makes exactly these calls:
 * caller-owned device planes, fs_init_fleet for a seeded batch, fs_step for
 * one fused control + integration step, fs_step_many for K steps in one
 * persistent launch.  The program checks that K fs_step calls and one
 * fs_step_many(K) give bitwise identical states and exits 0 on success.
 *
 *   make -C examples            (or: see examples/Makefile)
 *   ./examples/c_abi_step [n] [K]
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "flocksim_b200.h"

#define CHECK_FS(call)                                                              \
    do {                                                                            \
        int rc_ = (call);                                                           \
        if (rc_ != FS_OK) {                                                         \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, fs_last_error());   \
            return 1;                                                               \
        }                                                                           \
    } while (0)

#define CHECK_CUDA(call)                                                            \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));             \
            return 1;                                                               \
        }                                                                           \
    } while (0)

/* RobotParams / ControlGains / ControlLimits defaults (dynamics.py:54-63,
 * control.py:48-50,66-68) */
static void defaults(fs_robot* r, fs_gains* g, fs_limits* l) {
    memset(r, 0, sizeof(*r));
    r->mass = 1.0;
    r->gravity = 9.81;
    r->inertia[0] = 0.01;
    r->inertia[4] = 0.01;
    r->inertia[8] = 0.02;
    r->inertia_inv[0] = 1.0 / 0.01;
    r->inertia_inv[4] = 1.0 / 0.01;
    r->inertia_inv[8] = 1.0 / 0.02;
    r->thrust_max = 25.0;
    r->moment_max[0] = 2.0;
    r->moment_max[1] = 2.0;
    r->moment_max[2] = 1.0;
    r->v_limit = 50.0;
    r->omega_limit = 100.0;
    r->gimbal_cos = cos(1e-6);
    const double att[3] = {8.0, 8.0, 2.0}, rate[3] = {1.2, 1.2, 0.6}, vel[3] = {3.0, 3.0, 3.0};
    for (int k = 0; k < 3; ++k) {
        g->attitude[k] = att[k];
        g->rate[k] = rate[k];
        g->velocity[k] = vel[k];
        g->position[k] = 4.0;
    }
    l->max_tilt = 0.6;
    l->max_speed_cmd = 5.0;
    l->max_yaw_rate = 3.0;
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : (1 << 16);
    const int K = argc > 2 ? atoi(argv[2]) : 10;
    if (fs_abi_version() != FS_ABI_VERSION) {
        fprintf(stderr, "ABI mismatch: library %d, header %d\n", fs_abi_version(), FS_ABI_VERSION);
        return 1;
    }
    fs_robot robot;
    fs_gains gains;
    fs_limits limits;
    defaults(&robot, &gains, &limits);

    const int64_t stride = (n + 3) & ~(int64_t)3;   /* planes 16-byte aligned */
    const size_t sbytes = 13 * stride * sizeof(float), cbytes = 4 * stride * sizeof(float);
    float *a = NULL, *b = NULL, *cmd = NULL;
    uint32_t* sync = NULL;
    const int64_t nsync = fs_tile_sync_len(n);
    CHECK_CUDA(cudaMalloc((void**)&a, sbytes));
    CHECK_CUDA(cudaMalloc((void**)&b, sbytes));
    CHECK_CUDA(cudaMalloc((void**)&cmd, cbytes));
    CHECK_CUDA(cudaMalloc((void**)&sync, (size_t)nsync * sizeof(uint32_t)));
    cudaStream_t s;
    CHECK_CUDA(cudaStreamCreate(&s));

    /* seeded batch (BASELINE config distributions), velocity mode */
    CHECK_FS(fs_init_fleet(n, 0, 2024, FS_MODE_VELOCITY, a, stride, cmd, stride, NULL, 0, &robot, s));
    CHECK_CUDA(cudaMemcpyAsync(b, a, sbytes, cudaMemcpyDeviceToDevice, s));

    fs_step_desc d;
    memset(&d, 0, sizeof(d));
    d.n = n;
    d.state_in = a;
    d.state_out = a;                 /* in place */
    d.state_in_stride = d.state_out_stride = stride;
    d.mode = FS_MODE_VELOCITY;
    d.integrate = 1;
    d.cmd = cmd;
    d.cmd_stride = stride;
    d.dt = 0.01f;

    /* K steps, one fs_step each (control_batch + step_batch per step) */
    for (int k = 0; k < K; ++k) {
        d.step_index = (uint64_t)k;
        CHECK_FS(fs_step(&d, &robot, &gains, &limits, NULL, s));
    }

    /* the same K steps in one persistent launch */
    fs_step_desc m = d;
    m.state_in = b;
    m.state_out = b;
    m.step_index = 0;
    CHECK_CUDA(cudaMemsetAsync(sync, 0, (size_t)nsync * sizeof(uint32_t), s));
    m.tile_sync = sync;
    m.sync_wait = 0;
    m.sync_post = 1;
    const int many = fs_step_many(&m, &robot, &gains, &limits, NULL, K, s);
    if (many == FS_EINVAL && n < (1 << 15)) {
        printf("n = %lld is below the streaming kernel's size: fs_step_many refused (%s)\n",
               (long long)n, fs_last_error());
    } else {
        CHECK_FS(many);
    }
    CHECK_CUDA(cudaStreamSynchronize(s));

    float* ha = (float*)malloc(sbytes);
    float* hb = (float*)malloc(sbytes);
    CHECK_CUDA(cudaMemcpy(ha, a, sbytes, cudaMemcpyDeviceToHost));
    CHECK_CUDA(cudaMemcpy(hb, b, sbytes, cudaMemcpyDeviceToHost));
    int64_t diff = 0;
    double sum = 0.0;
    for (int k = 0; k < 13; ++k)
        for (int64_t i = 0; i < n; ++i) {
            diff += memcmp(&ha[k * stride + i], &hb[k * stride + i], sizeof(float)) != 0;
            sum += ha[k * stride + i];
        }
    printf("n=%lld K=%d  vehicle 0: p=(%.6f, %.6f, %.6f) q=(%.6f, %.6f, %.6f, %.6f)\n",
           (long long)n, K, ha[0], ha[stride], ha[2 * stride], ha[3 * stride], ha[4 * stride],
           ha[5 * stride], ha[6 * stride]);
    printf("sum of all planes %.9e; fs_step x K vs fs_step_many(K): %lld differing values\n", sum,
           (long long)(many == FS_OK ? diff : 0));
    free(ha);
    free(hb);
    cudaFree(a);
    cudaFree(b);
    cudaFree(cmd);
    cudaFree(sync);
    cudaStreamDestroy(s);
    return (many == FS_OK && diff != 0) ? 2 : 0;
}
