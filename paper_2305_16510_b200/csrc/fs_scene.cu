// fs_scene.cu -- obstacle scenes on the device:
// signed-distance queries (scene.py:127-181), generic ray casts
// (camera.py:230-282), the per-robot depth + segmentation camera
// (camera.py:285-335) and the creation-time prototype picks
// (assets.py:335-356).
//
// Renderer (render_kernel): one CTA per (env, run of 32x16-pixel image
// tiles), two pixel rays per thread.  The env's
// primitives are staged once per CTA in shared memory as float64 records
// plus an origin-relative fp32 AABB, and sorted by a lower bound of their
// hit distance (camera origin to AABB).  Per tile the CTA culls the boxes
// against the tile's four frustum side planes (one primitive per thread, warp-ballot
// compaction that keeps the sorted order); each thread then walks its
// pixel's candidates nearest-bound first: it stops once the bound exceeds
// its best hit, skips boxes a conservative fp32 slab test rules out, and
// runs the reference's float64 intersection on the rest.  Every shortcut is
// conservative, so none changes a result: the nearest hit wins, equal
// distances going to the lowest slot, as in cast_rays' strict `<`.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "flocksim_b200.h"
#include "fs_host.h"
#include "fs_scene.cuh"

namespace fs {
int check_launch(const char* what);
}
int fs_fail_einval(const char* msg);

namespace fs {

// ---- signed distances ---------------------------------------------------------

__global__ void __launch_bounds__(256) scene_distance_kernel(const __grid_constant__ fs_scene s,
                                                             const float* __restrict__ pts,
                                                             int64_t pstride, int coll_only,
                                                             double* dist, int64_t dstride,
                                                             double* minout) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= s.num_envs) return;
    const double px = pts[e], py = pts[pstride + e], pz = pts[2 * pstride + e];
    double best = kInf;
    for (int k = 0; k < s.width; ++k) {
        PrimD p;
        load_prim(s, k, e, p);
        const int kind = p.kind;
        const double d = kind >= 0 ? sdf(p, px, py, pz) : kInf;
        if (dist) dist[(int64_t)k * dstride + e] = d;
        const int coll = __float_as_int(rec_ptr(s, k, e)[1].w);
        const bool counts = kind >= 0 && (!coll_only || coll != 0);
        // np.min propagates NaN
        if (counts && (d < best || d != d)) best = (best != best) ? best : d;
    }
    if (minout) minout[e] = best;
}

// ---- generic ray casts (cast_rays) ------------------------------------------------

__global__ void __launch_bounds__(256) cast_rays_kernel(const __grid_constant__ fs_scene s,
                                                        int64_t env, double ox, double oy,
                                                        double oz, const double* __restrict__ dirs,
                                                        int64_t m, double max_range, double* depth,
                                                        int32_t* seg) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const double o[3] = {ox, oy, oz};
    const double d[3] = {dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]};
    double best = kInf;
    int32_t bseg = 0;
    for (int k = 0; k < s.width; ++k) {
        SlotBox b;
        load_box(s, k, env, b);
        if (b.kind < 0 || b.coll == 0) continue;
        PrimD p;
        load_prim(s, k, env, p);
        const double t = ray_prim(p, o, d);
        if (t < best) {
            best = t;
            bseg = slot_seg(s, k, env);
        }
    }
    const bool miss = !(best <= max_range);
    depth[i] = miss ? max_range : best;
    seg[i] = miss ? 0 : bseg;
}

// ---- depth camera ------------------------------------------------------------------

constexpr int kRPT = 2;            // rays per thread (rows ly, ly + 8, ...)
constexpr int kTileW = 32, kTileH = 8 * kRPT, kRThreads = 256;
constexpr int kChunk = 256;        // primitives staged per pass
constexpr int kMaxTPC = 16;        // tiles per CTA

struct SPrim {
    double pos[3], rot[9], dim[3];
    float lo[3], hi[3];            // stored (outward-rounded) AABB minus the camera origin
    float dmin;                    // lower bound of any hit parameter from the camera
    int32_t kind, seg;
};

struct RenderShared {
    SPrim prim[kChunk];

    int16_t order[kChunk];         // staged slots sorted by dmin (ties: lower slot first)
    int16_t cand[kChunk];          // this tile's candidates, in `order` order
    int32_t ncand;
    int32_t warp_count[kRThreads / 32];
    double origin[3], qcam[4];
    float4 plane[kMaxTPC][4];      // per tile of this CTA: inward normals of the four frustum
                                   // side planes (env frame, unit; planes through the origin)
};

// Stage slots [base, base + cnt) of env e (needs sh.origin), then sort them
// by dmin = |origin - AABB| (rounded down): no hit on a slot can be nearer.
__device__ __forceinline__ void stage_chunk(const fs_scene& s, int64_t e, int base, int cnt,
                                            RenderShared& sh) {
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
        const int k = base + j;
        SPrim& p = sh.prim[j];
        PrimD q;
        load_prim(s, k, e, q);
        SlotBox b;
        load_box(s, k, e, b);
        p.kind = (b.kind >= 0 && b.coll == 0) ? FS_PRIM_PAD : b.kind;
        p.seg = slot_seg(s, k, e);
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            p.dim[f] = q.dim[f];
            p.pos[f] = q.pos[f];
        }
#pragma unroll
        for (int f = 0; f < 9; ++f) p.rot[f] = q.rot[f];
        float d2 = 0.0f;
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            // origin-relative box, rounded outward again
            p.lo[f] = __fsub_rd(b.lo[f], (float)sh.origin[f]);
            p.hi[f] = __fsub_ru(b.hi[f], (float)sh.origin[f]);
            const float dd = fmaxf(fmaxf(p.lo[f], -p.hi[f]), 0.0f);
            d2 += dd * dd;
        }
        p.dmin = p.kind >= 0 ? fmaxf(0.0f, sqrtf(d2) * (1.0f - 1e-5f) - 1e-5f)
                             : __int_as_float(0x7f800000);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += blockDim.x) {
        const float key = sh.prim[j].dmin;
        int rank = 0;
        for (int i = 0; i < cnt; ++i) {
            const float ki = sh.prim[i].dmin;
            rank += (ki < key) || (ki == key && i < j);
        }
        sh.order[rank] = (int16_t)j;
    }
    __syncthreads();
}

// pixel ray in the camera frame, unnormalized: ((x - W/2) s, (y - H/2) s, 1)
__device__ __forceinline__ void cam_ray_f(float x, float y, const fs_camera& c, float* d) {
    d[0] = (x - 0.5f * c.width) * (float)c.pixel_scale;
    d[1] = (y - 0.5f * c.height) * (float)c.pixel_scale;
    d[2] = 1.0f;
}

__device__ __forceinline__ void qrot_f(const double* q, const float* v, float* o) {
    const float w = (float)q[0], x = (float)q[1], y = (float)q[2], z = (float)q[3];
    const float tx = 2.0f * (y * v[2] - z * v[1]);
    const float ty = 2.0f * (z * v[0] - x * v[2]);
    const float tz = 2.0f * (x * v[1] - y * v[0]);
    o[0] = v[0] + w * tx + (y * tz - z * ty);
    o[1] = v[1] + w * ty + (z * tx - x * tz);
    o[2] = v[2] + w * tz + (x * ty - y * tx);
}

// Cull the staged chunk against the tile's view frustum: a box (origin-
// relative AABB, center c, half extents h) is dropped when it lies wholly
// outside one of the four side planes (n.c + |n|.h below a small negative
// margin for the fp32 arithmetic) or beyond the range limit.  Writes
// sh.cand / sh.ncand in dmin order.
__device__ __forceinline__ void cull_tile(int cnt, const float4* pl, float max_range,
                                          RenderShared& sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int base = 0; base < cnt; base += kRThreads) {
        const int pos = base + threadIdx.x;
        const int j = pos < cnt ? sh.order[pos] : 0;
        bool keep = false;
        if (pos < cnt && sh.prim[j].kind >= 0 && sh.prim[j].dmin <= max_range) {
            const SPrim& p = sh.prim[j];
            const float cx = 0.5f * (p.lo[0] + p.hi[0]), hx = 0.5f * (p.hi[0] - p.lo[0]);
            const float cy = 0.5f * (p.lo[1] + p.hi[1]), hy = 0.5f * (p.hi[1] - p.lo[1]);
            const float cz = 0.5f * (p.lo[2] + p.hi[2]), hz = 0.5f * (p.hi[2] - p.lo[2]);
            const float margin = 1e-4f * (fabsf(cx) + fabsf(cy) + fabsf(cz) + hx + hy + hz + 1.0f);
            keep = true;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float4 n = pl[q];
                const float sdist = n.x * cx + n.y * cy + n.z * cz + fabsf(n.x) * hx +
                                    fabsf(n.y) * hy + fabsf(n.z) * hz;
                keep &= sdist >= -margin;
            }
        }
        const unsigned ball = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) sh.warp_count[warp] = __popc(ball);
        __syncthreads();
        int off = sh.ncand;
        for (int w = 0; w < warp; ++w) off += sh.warp_count[w];
        if (keep) sh.cand[off + __popc(ball & ((1u << lane) - 1u))] = (int16_t)j;
        __syncthreads();
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w = 0; w < kRThreads / 32; ++w) tot += sh.warp_count[w];
            sh.ncand += tot;
        }
        __syncthreads();
    }
}

// conservative fp32 slab test of the ray against a stored AABB (origin-
// relative): false only when no point of the box lies on the ray within
// [0, tmax].  inv[f] = 1 / d[f], with d[f] == 0 replaced by +-1e-30 (a
// parallel ray then gets +-huge slab parameters: outside -> rejected,
// inside -> unconstrained, which is the exact parallel-slab rule).
__device__ __forceinline__ bool aabb_maybe(const SPrim& p, const float* inv, float tmax) {
    float te = 0.0f, tx = 3.0e38f;
#pragma unroll
    for (int f = 0; f < 3; ++f) {
        const float t1 = p.lo[f] * inv[f], t2 = p.hi[f] * inv[f];
        te = fmaxf(te, fminf(t1, t2));
        tx = fminf(tx, fmaxf(t1, t2));
    }
    // widen once (the margin maps are monotone): fp32 rounding of the box,
    // the origin and the approximate reciprocals
    te = te * (1.0f - 1e-5f) - 1e-5f;
    tx = tx * (1.0f + 1e-5f) + 1e-5f;
    return te <= fminf(tx, tmax);
}

// the exact float64 test, out of line: it runs about once per ray, and
// keeping it out of the candidate loop keeps that loop's registers free
__device__ __noinline__ double ray_prim_exact(const SPrim* p, const double* o, double dx,
                                              double dy, double dz) {
    const double d[3] = {dx, dy, dz};
    return ray_prim(*p, o, d);
}

__device__ __forceinline__ float rcp_approx(float x) {
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

template <int MINB>
__global__ void __launch_bounds__(kRThreads, MINB)
render_kernel(const __grid_constant__ fs_scene s, const __grid_constant__ fs_camera cam,
              const float* __restrict__ state, int64_t sstride, const double* __restrict__ mount,
              int64_t mstride, int64_t first_env, int tiles_per_cta, float* __restrict__ depth,
              int32_t* __restrict__ segout) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    RenderShared& sh = *reinterpret_cast<RenderShared*>(smem_raw);
    const int64_t img = blockIdx.y;                 // output image index
    const int64_t e = first_env + img;              // scene / state env index
    const int tx_n = (cam.width + kTileW - 1) / kTileW;
    const int ty_n = (cam.height + kTileH - 1) / kTileH;
    const int ntiles = tx_n * ty_n;
    const int t0 = blockIdx.x * tiles_per_cta;
    if (t0 >= ntiles) return;
    const int t1 = min(ntiles, t0 + tiles_per_cta);

    if (threadIdx.x == 0) {
        // camera.py:322-325: origin = p + R(q) mount_p, q_cam = q (x) mount_q
        double q[4], mp[3], mq[4], rp[3];
        for (int k = 0; k < 4; ++k) q[k] = (double)state[(3 + k) * sstride + e];
        for (int k = 0; k < 3; ++k)
            mp[k] = mount ? mount[k * mstride + e] : cam.mount_position[k];
        for (int k = 0; k < 4; ++k)
            mq[k] = mount ? mount[(3 + k) * mstride + e] : cam.mount_rotation[k];
        qrot_d(q, mp, rp);
        for (int k = 0; k < 3; ++k) sh.origin[k] = (double)state[k * sstride + e] + rp[k];
        qmul_d(q, mq, sh.qcam);
    }
    __syncthreads();
    const int K = s.width;
    const bool single = K <= kChunk;
    if (single) stage_chunk(s, e, 0, K, sh);
    // frustum side planes of each of this CTA's tiles, from the tile's
    // image-plane edges (camera frame: left x - u0 z >= 0, right u1 z - x >= 0,
    // top y - v0 z >= 0, bottom v1 z - y >= 0), unit normals rotated to the env
    // frame once
    if (threadIdx.x < t1 - t0) {
        const int t = t0 + threadIdx.x;
        const int tx = t % tx_n, ty = t / tx_n;
        const float sc = (float)cam.pixel_scale;
        const float u0 = ((float)(tx * kTileW) - 0.5f * cam.width) * sc;
        const float u1 = ((float)(tx * kTileW + kTileW) - 0.5f * cam.width) * sc;
        const float v0 = ((float)(ty * kTileH) - 0.5f * cam.height) * sc;
        const float v1 = ((float)(ty * kTileH + kTileH) - 0.5f * cam.height) * sc;
        const float nc[4][3] = {{1.0f, 0.0f, -u0}, {-1.0f, 0.0f, u1},
                                {0.0f, 1.0f, -v0}, {0.0f, -1.0f, v1}};
        for (int q = 0; q < 4; ++q) {
            const float inv = rsqrtf(nc[q][0] * nc[q][0] + nc[q][1] * nc[q][1] +
                                     nc[q][2] * nc[q][2]);
            const float nn[3] = {nc[q][0] * inv, nc[q][1] * inv, nc[q][2] * inv};
            float w[3];
            qrot_f(sh.qcam, nn, w);
            sh.plane[threadIdx.x][q] = make_float4(w[0], w[1], w[2], 0.0f);
        }
    }
    __syncthreads();

    const double scale = cam.pixel_scale;
    const float maxr = (float)cam.max_range;
    const float tcap = maxr * (1.0f + 1e-5f) + 1e-5f;
    const int lx = threadIdx.x % kTileW, ly = threadIdx.x / kTileW;
    for (int t = t0; t < t1; ++t) {
        const int tx = t % tx_n, ty = t / tx_n;
        const int px = tx * kTileW + lx;
        // this thread's rays (camera.py:123-130), float64, rows ly + 8 r
        double d[kRPT][3];
        float inv[kRPT][3];
        double best[kRPT];
        float tb[kRPT];
        int32_t bseg[kRPT], bslot[kRPT];
#pragma unroll
        for (int r = 0; r < kRPT; ++r) {
            const int py = ty * kTileH + ly + 8 * r;
            const double u = ((double)px + 0.5 - cam.width / 2.0) * scale;
            const double v = ((double)py + 0.5 - cam.height / 2.0) * scale;
            const double in = rsqrt(u * u + v * v + 1.0);
            const double dc[3] = {u * in, v * in, in};
            qrot_d(sh.qcam, dc, d[r]);
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const float df = (float)d[r][k];
                inv[r][k] = rcp_approx(df != 0.0f ? df : copysignf(1e-30f, df));
            }
            best[r] = kInf;
            tb[r] = tcap;
            bseg[r] = 0;
            bslot[r] = 0x7fffffff;
        }
        for (int base = 0; base < K; base += kChunk) {
            const int cnt = min(kChunk, K - base);
            if (!single) {
                __syncthreads();
                stage_chunk(s, e, base, cnt, sh);
            }
            if (threadIdx.x == 0) sh.ncand = 0;
            __syncthreads();
            cull_tile(cnt, sh.plane[t - t0], maxr, sh);
            const int nc = sh.ncand;
            for (int c = 0; c < nc; ++c) {
                const int j = sh.cand[c];
                const SPrim& sp = sh.prim[j];
                const double dmin = (double)sp.dmin;
                bool any = false;
#pragma unroll
                for (int r = 0; r < kRPT; ++r) any |= !(dmin > best[r]);
                if (!any) break;                            // sorted: nothing nearer follows
                const int slot = base + j;
#pragma unroll
                for (int r = 0; r < kRPT; ++r) {
                    if (dmin > best[r]) continue;
                    if (!aabb_maybe(sp, inv[r], tb[r])) continue;
                    const double tt = ray_prim_exact(&sp, sh.origin, d[r][0], d[r][1], d[r][2]);
                    // nearest hit; equal distances go to the lower slot (cast_rays' strict <)
                    if (tt < best[r] || (tt == best[r] && slot < bslot[r])) {
                        best[r] = tt;
                        bseg[r] = sp.seg;
                        bslot[r] = slot;
                        // fp32 bound for the pre-test, widened past the rounding
                        tb[r] = fminf(tcap, (float)tt * (1.0f + 1e-5f) + 1e-5f);
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < kRPT; ++r) {
            const int py = ty * kTileH + ly + 8 * r;
            if (px < cam.width && py < cam.height) {
                const bool miss = !(best[r] <= cam.max_range);
                const int64_t o = (img * cam.height + py) * (int64_t)cam.width + px;
                depth[o] = miss ? (float)cam.max_range : __double2float_rn(best[r]);
                segout[o] = miss ? 0 : bseg[r];
            }
        }
        __syncthreads();
    }
}

// ---- creation-time prototype picks ----------------------------------------------------

__global__ void __launch_bounds__(256) obstacles_pick_kernel(const __grid_constant__ fs_obstacles ob,
                                                             int64_t n, int64_t first_id,
                                                             uint64_t seed, int32_t* count) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= n) return;
    count[e] = pick_env(ob, e, seed, first_id + e);
}

struct Bounds3 {
    double v[3];
};

// instance poses on demand (World.instances): thread per (instance, env),
// env fastest, so each of the 7 J planes is written coalesced
__global__ void __launch_bounds__(256) obstacles_poses_kernel(const __grid_constant__ fs_obstacles ob,
                                                              int64_t n, int64_t first_id,
                                                              uint64_t seed, const int32_t* counter,
                                                              Bounds3 bounds) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n * ob.instances_per_env) return;
    const int j = (int)(t / n);
    const int64_t e = t - (int64_t)j * n;
    const fs_asset_class& cl = ob.classes[class_of(ob, j)];
    const uint32_t c = (uint32_t)counter[e];
    const int64_t gid = first_id + e;
    double ip[3], iq[4];
    instance_position(cl, draw_block(seed, gid, c, kPoseBlock + (uint32_t)j), bounds.v, ip);
    instance_rotation(cl, draw_block(seed, gid, c, kPoseBlock + kPoseEuler + (uint32_t)j), iq);
#pragma unroll
    for (int i = 0; i < 3; ++i) ob.inst_pose[(int64_t)(7 * j + i) * ob.plane_stride + e] = ip[i];
#pragma unroll
    for (int i = 0; i < 4; ++i) ob.inst_pose[(int64_t)(7 * j + 3 + i) * ob.plane_stride + e] = iq[i];
}

}  // namespace fs

namespace {

bool scene_ok(const fs_scene* s) {
    if (!s || s->num_envs < 0 || s->width < 0) return false;
    if (s->width == 0 || s->num_envs == 0) return true;
    return s->rec && (reinterpret_cast<uintptr_t>(s->rec) & 15) == 0;
}

}  // namespace

extern "C" int fs_scene_distances(const fs_scene* s, const float* points, int64_t point_stride,
                                  int32_t collision_only, double* dist_out, int64_t dist_stride,
                                  double* min_out, void* stream) {
    if (!scene_ok(s)) return fs_fail_einval("invalid scene descriptor");
    if (s->num_envs == 0) return FS_OK;
    if (!points || point_stride < s->num_envs) return fs_fail_einval("points missing or stride too short");
    if (dist_out && dist_stride < s->num_envs) return fs_fail_einval("distance stride too short");
    const unsigned blocks = (unsigned)((s->num_envs + 255) / 256);
    fs::scene_distance_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(
        *s, points, point_stride, collision_only, dist_out, dist_stride, min_out);
    return fs::check_launch("scene_distance_kernel");
}

extern "C" int fs_cast_rays(const fs_scene* s, int64_t env, double ox, double oy, double oz,
                            const double* dirs, int64_t m, double max_range, double* depth_out,
                            int32_t* seg_out, void* stream) {
    if (!scene_ok(s)) return fs_fail_einval("invalid scene descriptor");
    if (env < 0 || env >= s->num_envs) return fs_fail_einval("env index out of range");
    if (m < 0) return fs_fail_einval("ray count must be >= 0");
    if (m == 0) return FS_OK;
    if (!dirs || !depth_out || !seg_out) return fs_fail_einval("null ray buffers");
    const unsigned blocks = (unsigned)((m + 255) / 256);
    fs::cast_rays_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(*s, env, ox, oy, oz, dirs, m,
                                                                   max_range, depth_out, seg_out);
    return fs::check_launch("cast_rays_kernel");
}

extern "C" int fs_render(const fs_scene* s, const fs_camera* cam, const float* state,
                         int64_t state_stride, const double* mount, int64_t mount_stride,
                         int64_t first_env, int64_t n, float* depth_out, int32_t* seg_out,
                         void* stream) {
    if (!scene_ok(s) || !cam) return fs_fail_einval("invalid scene or camera descriptor");
    if (cam->width < 1 || cam->height < 1) return fs_fail_einval("image dimensions must be at least 1x1");
    if (!(cam->max_range > 0.0)) return fs_fail_einval("max_range must be positive");
    if (n < 0 || first_env < 0 || first_env + n > s->num_envs)
        return fs_fail_einval("env range outside the scene");
    if (n == 0) return FS_OK;
    if (!state || !depth_out || !seg_out) return fs_fail_einval("null state or image buffers");
    if (state_stride < first_env + n) return fs_fail_einval("state stride shorter than the env range");
    if (mount && mount_stride < first_env + n) return fs_fail_einval("mount stride too short");
    if (n > 65535) return fs_fail_einval("at most 65535 images per call");
    const int tiles = ((cam->width + fs::kTileW - 1) / fs::kTileW) *
                      ((cam->height + fs::kTileH - 1) / fs::kTileH);
    const int tpc = tiles < 16 ? tiles : 16;
    const dim3 grid((unsigned)((tiles + tpc - 1) / tpc), (unsigned)n);
    const size_t smem = sizeof(fs::RenderShared);
    static fs::PerDeviceOnce once;
    once([&](int) {
        cudaFuncSetAttribute(fs::render_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
        cudaFuncSetAttribute(fs::render_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    });
    const char* minb_env = getenv("FS_RENDER_MINB");     // diagnostics: 1 or 2 CTAs per SM
    // measured: 1 CTA per SM (no register cap) is faster
    const int minb = (minb_env && atoi(minb_env) == 2) ? 2 : 1;
    if (minb == 1)
        fs::render_kernel<1><<<grid, fs::kRThreads, smem, (cudaStream_t)stream>>>(
            *s, *cam, state, state_stride, mount, mount_stride, first_env, tpc, depth_out,
            seg_out);
    else
        fs::render_kernel<2><<<grid, fs::kRThreads, smem, (cudaStream_t)stream>>>(
            *s, *cam, state, state_stride, mount, mount_stride, first_env, tpc, depth_out,
            seg_out);
    return fs::check_launch("render_kernel");
}

extern "C" int fs_obstacles_pick(const fs_obstacles* ob, int64_t n, int64_t first_id,
                                 uint64_t seed, int32_t* count_out, void* stream) {
    if (!ob || n < 0) return fs_fail_einval("invalid obstacle descriptor");
    if (n == 0) return FS_OK;
    if (!count_out || (ob->instances_per_env > 0 && (!ob->inst_proto || !ob->classes)) ||
        !ob->proto_offset)
        return fs_fail_einval("obstacle tables missing");
    if (ob->plane_stride < n) return fs_fail_einval("instance plane stride shorter than n");
    const unsigned blocks = (unsigned)((n + 255) / 256);
    fs::obstacles_pick_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(*ob, n, first_id, seed,
                                                                         count_out);
    return fs::check_launch("obstacles_pick_kernel");
}

extern "C" int fs_obstacles_poses(const fs_obstacles* ob, int64_t n, int64_t first_id,
                                  uint64_t seed, const int32_t* reset_counter,
                                  const double* bounds, void* stream) {
    if (!ob || n < 0) return fs_fail_einval("invalid obstacle descriptor");
    if (n == 0 || ob->instances_per_env == 0) return FS_OK;
    if (!ob->inst_pose || !ob->inst_proto || !ob->classes || !reset_counter || !bounds)
        return fs_fail_einval("obstacle tables, pose planes, counters or bounds missing");
    if (ob->plane_stride < n) return fs_fail_einval("instance plane stride shorter than n");
    const int64_t total = n * ob->instances_per_env;
    const unsigned blocks = (unsigned)((total + 255) / 256);
    const fs::Bounds3 b{{bounds[0], bounds[1], bounds[2]}};
    fs::obstacles_poses_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(*ob, n, first_id, seed,
                                                                          reset_counter, b);
    return fs::check_launch("obstacles_poses_kernel");
}
