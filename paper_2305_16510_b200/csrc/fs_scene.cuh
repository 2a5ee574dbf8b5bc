// fs_scene.cuh -- obstacle primitive soup on the device.
//
// Layout: one 96-byte record per (env, slot), record k of env e at
// rec[(e * K + k) * 24] (include/flocksim_b200.h fs_scene), six float4 groups
//   [lo xyz, kind] [hi xyz, coll] [dims xyz, seg] [pos xyz, R22]
//   [R00 R01 R02 R10] [R11 R12 R20 R21]
// so a bounds test is two vector loads and a full primitive six; a reset
// writes a slot with six vector stores.
//
// All geometry evaluates in float64 from the stored fp32 values, restating
// scene.py:signed_distances (127-165) and camera.py:_cast_one_primitive
// (170-227) operation for operation; the AABB is rounded outward so it stays
// conservative after the fp32 store.
#pragma once

#include <math.h>
#include <stdint.h>

#include "flocksim_b200.h"
#include "fs_rng.cuh"

namespace fs {

__device__ __forceinline__ float4* rec_ptr(const fs_scene& s, int k, int64_t e) {
    return reinterpret_cast<float4*>(s.rec + (e * s.width + k) * (int64_t)FS_PRIM_FIELDS);
}

struct PrimD {
    int kind;
    double dim[3], pos[3], rot[9];
};

struct SlotBox {
    float lo[3], hi[3];
    int kind, coll;
};

__device__ __forceinline__ void load_box(const fs_scene& s, int k, int64_t e, SlotBox& b) {
    const float4* r = rec_ptr(s, k, e);
    const float4 a = r[0], c = r[1];
    b.lo[0] = a.x;
    b.lo[1] = a.y;
    b.lo[2] = a.z;
    b.kind = __float_as_int(a.w);
    b.hi[0] = c.x;
    b.hi[1] = c.y;
    b.hi[2] = c.z;
    b.coll = __float_as_int(c.w);
}

__device__ __forceinline__ int slot_seg(const fs_scene& s, int k, int64_t e) {
    return __float_as_int(rec_ptr(s, k, e)[2].w);
}

__device__ __forceinline__ void load_prim(const fs_scene& s, int k, int64_t e, PrimD& p) {
    const float4* r = rec_ptr(s, k, e);
    const float4 g0 = r[0], g2 = r[2], g3 = r[3], g4 = r[4], g5 = r[5];
    p.kind = __float_as_int(g0.w);
    p.dim[0] = g2.x;
    p.dim[1] = g2.y;
    p.dim[2] = g2.z;
    p.pos[0] = g3.x;
    p.pos[1] = g3.y;
    p.pos[2] = g3.z;
    p.rot[8] = g3.w;
    p.rot[0] = g4.x;
    p.rot[1] = g4.y;
    p.rot[2] = g4.z;
    p.rot[3] = g4.w;
    p.rot[4] = g5.x;
    p.rot[5] = g5.y;
    p.rot[6] = g5.z;
    p.rot[7] = g5.w;
}

__device__ __forceinline__ void store_slot(const fs_scene& s, int k, int64_t e, const float* lo,
                                           const float* hi, const float* dim, const float* pos,
                                           const float* r, int kind, int seg, int coll) {
    float4* q = rec_ptr(s, k, e);
    q[0] = make_float4(lo[0], lo[1], lo[2], __int_as_float(kind));
    q[1] = make_float4(hi[0], hi[1], hi[2], __int_as_float(coll));
    q[2] = make_float4(dim[0], dim[1], dim[2], __int_as_float(seg));
    q[3] = make_float4(pos[0], pos[1], pos[2], r[8]);
    q[4] = make_float4(r[0], r[1], r[2], r[3]);
    q[5] = make_float4(r[4], r[5], r[6], r[7]);
}

// ---- float64 SE(3) helpers (se3.py) -----------------------------------------

// quat_multiply (se3.py:78-97): Hamilton product, renormalized
__device__ __forceinline__ void qmul_d(const double* a, const double* b, double* o) {
    const double w = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    const double x = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
    const double y = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
    const double z = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
    const double n = sqrt(w * w + x * x + y * y + z * z);
    o[0] = w / n;
    o[1] = x / n;
    o[2] = y / n;
    o[3] = z / n;
}

// qmul_d with one division (the reciprocal of the norm) instead of four: the
// obstacle-row rebuild, whose results are rounded to fp32 records anyway
__device__ __forceinline__ void qmul_d_fast(const double* a, const double* b, double* o) {
    const double w = a[0] * b[0] - a[1] * b[1] - a[2] * b[2] - a[3] * b[3];
    const double x = a[0] * b[1] + a[1] * b[0] + a[2] * b[3] - a[3] * b[2];
    const double y = a[0] * b[2] - a[1] * b[3] + a[2] * b[0] + a[3] * b[1];
    const double z = a[0] * b[3] + a[1] * b[2] - a[2] * b[1] + a[3] * b[0];
    const double inv = 1.0 / sqrt(w * w + x * x + y * y + z * z);
    o[0] = w * inv;
    o[1] = x * inv;
    o[2] = y * inv;
    o[3] = z * inv;
}

// quat_rotate (se3.py:106-130): v + w t + u x t, t = 2 u x v
__device__ __forceinline__ void qrot_d(const double* q, const double* v, double* o) {
    const double tx = 2.0 * (q[2] * v[2] - q[3] * v[1]);
    const double ty = 2.0 * (q[3] * v[0] - q[1] * v[2]);
    const double tz = 2.0 * (q[1] * v[1] - q[2] * v[0]);
    o[0] = v[0] + q[0] * tx + (q[2] * tz - q[3] * ty);
    o[1] = v[1] + q[0] * ty + (q[3] * tx - q[1] * tz);
    o[2] = v[2] + q[0] * tz + (q[1] * ty - q[2] * tx);
}

// quat_to_matrix (se3.py:138-153), row-major
__device__ __forceinline__ void qmat_d(const double* q, double* r) {
    const double w = q[0], x = q[1], y = q[2], z = q[3];
    r[0] = 1.0 - 2.0 * (y * y + z * z);
    r[1] = 2.0 * (x * y - w * z);
    r[2] = 2.0 * (x * z + w * y);
    r[3] = 2.0 * (x * y + w * z);
    r[4] = 1.0 - 2.0 * (x * x + z * z);
    r[5] = 2.0 * (y * z - w * x);
    r[6] = 2.0 * (x * z - w * y);
    r[7] = 2.0 * (y * z + w * x);
    r[8] = 1.0 - 2.0 * (x * x + y * y);
}

// rot_zyx (se3.py:200-215): q_z(yaw) (x) (q_y(pitch) (x) q_x(roll)) from
// half-angle axis quaternions, both products renormalized
__device__ __forceinline__ void rot_zyx_d(double roll, double pitch, double yaw, double* q) {
    double sr, cr, sp, cp, sy, cy;
    sincos(roll / 2.0, &sr, &cr);
    sincos(pitch / 2.0, &sp, &cp);
    sincos(yaw / 2.0, &sy, &cy);
    const double qx[4] = {cr, sr, 0.0, 0.0};
    const double qy[4] = {cp, 0.0, sp, 0.0};
    const double qz[4] = {cy, 0.0, 0.0, sy};
    double t[4];
    qmul_d(qy, qx, t);
    qmul_d(qz, t, q);
}

// scene.py:_primitive_aabb (62-73): conservative half extents
__device__ __forceinline__ void prim_half_extent(int kind, const double* dim, const double* r,
                                                 double* half) {
    if (kind == FS_PRIM_BOX) {
#pragma unroll
        for (int i = 0; i < 3; ++i)
            half[i] = fabs(r[3 * i]) * (dim[0] / 2.0) + fabs(r[3 * i + 1]) * (dim[1] / 2.0) +
                      fabs(r[3 * i + 2]) * (dim[2] / 2.0);
    } else if (kind == FS_PRIM_CYLINDER) {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            const double a = r[3 * i + 2];   // local z axis = column 2
            half[i] = fabs(a) * (dim[1] / 2.0) + dim[0] * sqrt(fmax(0.0, 1.0 - a * a));
        }
    } else {
        half[0] = half[1] = half[2] = dim[0];
    }
}

// ---- signed distance (scene.py:127-165) ---------------------------------------

// R^T (p - c): lx = r00 dx + r10 dy + r20 dz, ...
__device__ __forceinline__ void to_local(const PrimD& p, double px, double py, double pz,
                                         double& lx, double& ly, double& lz) {
    const double dx = px - p.pos[0], dy = py - p.pos[1], dz = pz - p.pos[2];
    lx = p.rot[0] * dx + p.rot[3] * dy + p.rot[6] * dz;
    ly = p.rot[1] * dx + p.rot[4] * dy + p.rot[7] * dz;
    lz = p.rot[2] * dx + p.rot[5] * dy + p.rot[8] * dz;
}

__device__ __forceinline__ double sdf(const PrimD& p, double px, double py, double pz) {
    double lx, ly, lz;
    to_local(p, px, py, pz, lx, ly, lz);
    if (p.kind == FS_PRIM_BOX) {
        const double qx = fabs(lx) - p.dim[0] / 2.0;
        const double qy = fabs(ly) - p.dim[1] / 2.0;
        const double qz = fabs(lz) - p.dim[2] / 2.0;
        const double mx = fmax(qx, 0.0), my = fmax(qy, 0.0), mz = fmax(qz, 0.0);
        const double outside = sqrt(mx * mx + my * my + mz * mz);
        const double inside = fmin(fmax(qx, fmax(qy, qz)), 0.0);
        return outside + inside;
    }
    if (p.kind == FS_PRIM_CYLINDER) {
        const double rho = sqrt(lx * lx + ly * ly) - p.dim[0];
        const double ax = fabs(lz) - p.dim[1] / 2.0;
        const double mr = fmax(rho, 0.0), ma = fmax(ax, 0.0);
        return sqrt(mr * mr + ma * ma) + fmin(fmax(rho, ax), 0.0);
    }
    return sqrt(lx * lx + ly * ly + lz * lz) - p.dim[0];
}

// squared distance from a point to a (stored, outward-rounded) AABB; 0 inside
__device__ __forceinline__ double box_dist2(const SlotBox& b, double px, double py, double pz) {
    const double p[3] = {px, py, pz};
    double d2 = 0.0;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        const double d = fmax(fmax((double)b.lo[j] - p[j], p[j] - (double)b.hi[j]), 0.0);
        d2 += d * d;
    }
    return d2;
}

// One slot of check_collisions' primitive part (world.py:100-101,
// min_distance with collision_only): collision-enabled, not a wall slab (a
// wall contact is exactly the caller's bounds test), and closer than r.  The
// AABB test skips a slot only when its box is at least r away, which the
// primitive (inside the box) then is too.
__device__ __forceinline__ bool slot_hit(const fs_scene& s, int k, int64_t e, double px,
                                         double py, double pz, double r) {
    SlotBox b;
    load_box(s, k, e, b);
    if (b.kind < 0 || b.coll == 0 || b.coll == FS_COLL_WALL) return false;
    if (box_dist2(b, px, py, pz) >= r * r) return false;
    PrimD p;
    load_prim(s, k, e, p);
    return sdf(p, px, py, pz) < r;
}

// is any collision-enabled primitive of env e closer than r to the point?
// (the caller also applies the env-bounds test)
__device__ __forceinline__ bool scene_hit(const fs_scene& s, int64_t e, double px, double py,
                                          double pz, double r) {
    for (int k = 0; k < s.width; ++k)
        if (slot_hit(s, k, e, px, py, pz, r)) return true;
    return false;
}

// ---- ray casting (camera.py:132-227) ---------------------------------------------

constexpr double kInf = __builtin_huge_val();

__device__ __forceinline__ double dmin2(double a, double b) { return a < b ? a : b; }
__device__ __forceinline__ double dmax2(double a, double b) { return a > b ? a : b; }

// one slab of _ray_box / the cylinder cap test (one reciprocal instead of
// the reference's two divisions: the parameters agree to an ulp of float64;
// compare-selects instead of fmin/fmax, whose NaN handling costs ~3x and
// only matters for NaN inputs)
__device__ __forceinline__ void slab(double o, double d, double h, double& lo, double& hi) {
    if (d == 0.0) {
        const bool in = fabs(o) <= h;
        lo = dmax2(lo, in ? -kInf : kInf);
        hi = dmin2(hi, in ? kInf : -kInf);
    } else {
        const double inv = 1.0 / d;
        const double t1 = (-h - o) * inv, t2 = (h - o) * inv;
        lo = dmax2(lo, dmin2(t1, t2));
        hi = dmin2(hi, dmax2(t1, t2));
    }
}

// _ray_interval_to_t (camera.py:163-167)
__device__ __forceinline__ double interval_t(double lo, double hi) {
    const double t = lo > 0.0 ? lo : hi;
    return (hi >= lo && t > 0.0) ? t : kInf;
}

// _cast_one_primitive: smallest positive ray parameter, +inf on a miss.
// o, d in the env frame; d a unit vector.  P: any record with kind, dim[3],
// pos[3], rot[9] (registers or shared memory).
template <typename P>
__device__ __forceinline__ double ray_prim(const P& p, const double* o, const double* d) {
    const double rx = o[0] - p.pos[0], ry = o[1] - p.pos[1], rz = o[2] - p.pos[2];
    const double ox = rx * p.rot[0] + ry * p.rot[3] + rz * p.rot[6];
    const double oy = rx * p.rot[1] + ry * p.rot[4] + rz * p.rot[7];
    const double oz = rx * p.rot[2] + ry * p.rot[5] + rz * p.rot[8];
    const double dx = d[0] * p.rot[0] + d[1] * p.rot[3] + d[2] * p.rot[6];
    const double dy = d[0] * p.rot[1] + d[1] * p.rot[4] + d[2] * p.rot[7];
    const double dz = d[0] * p.rot[2] + d[1] * p.rot[5] + d[2] * p.rot[8];
    if (p.kind == FS_PRIM_BOX) {
        double lo = -kInf, hi = kInf;
        slab(ox, dx, p.dim[0] / 2.0, lo, hi);
        slab(oy, dy, p.dim[1] / 2.0, lo, hi);
        slab(oz, dz, p.dim[2] / 2.0, lo, hi);
        return interval_t(lo, hi);
    }
    if (p.kind == FS_PRIM_SPHERE) {
        const double r = p.dim[0];
        const double b = ox * dx + oy * dy + oz * dz;
        const double c = ox * ox + oy * oy + oz * oz - r * r;
        const double disc = b * b - c;
        const double root = sqrt(fmax(disc, 0.0));
        const double t1 = -b - root, t2 = -b + root;
        const double t = t1 > 0.0 ? t1 : t2;
        return (disc >= 0.0 && t > 0.0) ? t : kInf;
    }
    // finite cylinder along local z: lateral quadratic + cap slab
    const double r = p.dim[0];
    const double a = dx * dx + dy * dy;
    const double b = ox * dx + oy * dy;
    const double c = ox * ox + oy * oy - r * r;
    double qlo, qhi;
    if (a == 0.0) {
        const bool in = c <= 0.0;
        qlo = in ? -kInf : kInf;
        qhi = in ? kInf : -kInf;
    } else {
        const double disc = b * b - a * c;
        if (disc < 0.0) {
            qlo = kInf;
            qhi = -kInf;
        } else {
            const double root = sqrt(disc), ia = 1.0 / a;
            qlo = (-b - root) * ia;
            qhi = (-b + root) * ia;
        }
    }
    slab(oz, dz, p.dim[1] / 2.0, qlo, qhi);
    return interval_t(qlo, qhi);
}


// ---- obstacle re-randomization (world.py:229-243, assets.py:372-403) -------------
//
// Draw layout per (seed, env gid, reset counter c) -- the library's Philox
// stream (documented deviation from NumPy's Philox-4x64, assets.py:310-315):
//   prototype picks (creation only, c = 0): block kPickBlock + j/4, word j%4,
//       proto = pool_first + mulhi(word, pool_size)   (assets.py:344-346)
//   instance j pose: block kPoseBlock + j, words x, y, z -> position
//       uniforms; block kPoseBlock + kPoseEuler + j -> euler uniforms
//       (randomize_pose draws 3 position then 3 euler uniforms, 392-401)
//   robot / goal placement: fs_world.cu kPlaceBlock (world.py:196-211)
//   camera mount: block kMountBlock (position), kMountBlock + 1 (euler)
//       (camera.py:238-244)
// u = (word >> 8) 2^-24 is exact in float64; every affine map and rotation
// after it is the reference's float64 arithmetic.
constexpr uint32_t kPoseBlock = 0x10000;
constexpr uint32_t kPoseEuler = 0x8000;
constexpr uint32_t kPickBlock = 0x20000;
constexpr uint32_t kMountBlock = 0x30000;

__device__ __forceinline__ double u01d(uint32_t w) {
    return (double)(w >> 8) * 5.9604644775390625e-8;   // 2^-24
}

__device__ __forceinline__ uint32_t word_of(const U4& b, int i) {
    return i == 0 ? b.x : (i == 1 ? b.y : (i == 2 ? b.z : b.w));
}

// class of instance j (instances are laid out class by class, assets.py:340-356)
__device__ __forceinline__ int class_of(const fs_obstacles& ob, int j) {
    int c = 0, acc = ob.classes[0].count_per_env;
    while (j >= acc && c + 1 < ob.num_classes) acc += ob.classes[++c].count_per_env;
    return c;
}

__device__ __forceinline__ int32_t& inst_proto(const fs_obstacles& ob, int j, int64_t e) {
    return ob.inst_proto[(int64_t)j * ob.plane_stride + e];
}

// prototype picks at creation; returns the env's primitive count (walls included)
__device__ __forceinline__ int32_t pick_env(const fs_obstacles& ob, int64_t e, uint64_t seed,
                                            int64_t gid) {
    int32_t count = 0;
    for (int j = 0; j < ob.instances_per_env; ++j) {
        const fs_asset_class& cl = ob.classes[class_of(ob, j)];
        const U4 b = draw_block(seed, gid, 0u, kPickBlock + (uint32_t)(j >> 2));
        const int32_t p = cl.pool_first + (int32_t)mulhi32(word_of(b, j & 3), (uint32_t)cl.pool_size);
        inst_proto(ob, j, e) = p;
        count += ob.proto_offset[p + 1] - ob.proto_offset[p];
    }
    if (ob.wall_proto >= 0) count += ob.proto_offset[ob.wall_proto + 1] - ob.proto_offset[ob.wall_proto];
    return count;
}

// float -> float rounded toward -inf / +inf (conservative AABB after the store)
__device__ __forceinline__ float f_down(double x) { return __double2float_rd(x); }
__device__ __forceinline__ float f_up(double x) { return __double2float_ru(x); }

// scene_hit with the instance broad phase: the env's instance records (two
// 16-B loads each, 8 instances in flight at a time) first, then only the
// slots of collision-enabled instances whose box is within r.  A box is
// skipped only when it is at least r away (float32 distance, widened), so
// the result is scene_hit's.
// CLR: also return in *cmin a lower bound of the distance from the point to
// every collision-enabled primitive (meaningful only when the result is
// false): instances whose box is within rvis are walked slot by slot and
// contribute their slot boxes' distances, the others their instance box's
// -- the clearance cache (the tighter slot boxes matter: a robot is often
// inside a tree's box but far from its trunk and branches).
template <bool CLR = false>
__device__ __forceinline__ bool scene_hit_inst(const fs_obstacles& ob, int64_t e, double px,
                                               double py, double pz, double r,
                                               float* cmin = nullptr, float rvis = 0.0f) {
    if (!ob.inst_box) return scene_hit(ob.scene, e, px, py, pz, r);
    float c2 = 3.0e38f;
    const int J = ob.instances_per_env;
    const int64_t ps = ob.plane_stride;
    const float4* rec = reinterpret_cast<const float4*>(ob.inst_box) + e;   // + (2j + h) ps
    const float p[3] = {(float)px, (float)py, (float)pz};
    const float rr = (float)r * 1.0001f + 1e-5f;
    const float rv = CLR ? fmaxf(rr, rvis) : rr;      // slot-walk radius
    constexpr int G = 8;
    for (int j0 = 0; j0 < J; j0 += G) {
        float4 lo[G], hi[G];
#pragma unroll
        for (int u = 0; u < G; ++u) {
            if (j0 + u < J) {
                lo[u] = __ldg(rec + (int64_t)(2 * (j0 + u)) * ps);
                hi[u] = __ldg(rec + (int64_t)(2 * (j0 + u) + 1) * ps);
            }
        }
        unsigned near = 0;
#pragma unroll
        for (int u = 0; u < G; ++u) {
            if (j0 + u < J) {
                const float dx = fmaxf(fmaxf(lo[u].x - p[0], p[0] - hi[u].x), 0.0f);
                const float dy = fmaxf(fmaxf(lo[u].y - p[1], p[1] - hi[u].y), 0.0f);
                const float dz = fmaxf(fmaxf(lo[u].z - p[2], p[2] - hi[u].z), 0.0f);
                const float b2 = dx * dx + dy * dy + dz * dz;
                const bool on = hi[u].w != 0.0f && b2 < rv * rv;
                if (CLR && hi[u].w != 0.0f && !on) c2 = fminf(c2, b2);
                near |= (on ? 1u : 0u) << u;
            }
        }
        while (near) {
            const int u = __ffs(near) - 1;
            near &= near - 1;
            const int32_t span = __float_as_int(lo[u].w);
            const int first = span & 0xffff, end = first + ((span >> 16) & 0xffff);
            // the instance's slot boxes, B at a time (2B vector loads in flight)
            constexpr int B = 2;
            for (int k0 = first; k0 < end; k0 += B) {
                SlotBox b[B];
#pragma unroll
                for (int v = 0; v < B; ++v)
                    if (k0 + v < end) load_box(ob.scene, k0 + v, e, b[v]);
                unsigned m = 0;
#pragma unroll
                for (int v = 0; v < B; ++v) {
                    if (k0 + v < end) {
                        const double bd2 = box_dist2(b[v], px, py, pz);
                        if (bd2 < r * r) m |= 1u << v;
                        if (CLR) c2 = fminf(c2, (float)bd2);
                    }
                }
                while (m) {
                    const int v = __ffs(m) - 1;
                    m &= m - 1;
                    PrimD pr;
                    load_prim(ob.scene, k0 + v, e, pr);
                    if (sdf(pr, px, py, pz) < r) return true;
                }
            }
        }
    }
    if (CLR) *cmin = sqrtf(c2);
    return false;
}

// write slot k of env e: compile_instances' per-primitive body (scene.py:100-124)
__device__ __forceinline__ void write_slot(const fs_obstacles& ob, int k, int64_t e,
                                          const fs_proto_prim& pp, const double* ip,
                                          const double* iq, int32_t seg, int32_t coll,
                                          float* lo_out = nullptr, float* hi_out = nullptr) {
    double pos[3], q[4], r[9], half[3];
    qrot_d(iq, pp.position, pos);
#pragma unroll
    for (int j = 0; j < 3; ++j) pos[j] += ip[j];
    qmul_d_fast(iq, pp.rotation, q);
    qmat_d(q, r);
    prim_half_extent(pp.kind, pp.dims, r, half);
    float lo[3], hi[3], dim[3], pf[3], rf[9];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        dim[j] = (float)pp.dims[j];
        pf[j] = (float)pos[j];
        lo[j] = f_down(pos[j] - half[j]);
        hi[j] = f_up(pos[j] + half[j]);
    }
#pragma unroll
    for (int j = 0; j < 9; ++j) rf[j] = (float)r[j];
    store_slot(ob.scene, k, e, lo, hi, dim, pf, rf, pp.kind, seg, coll);   // coll: 0, 1, FS_COLL_WALL
    if (lo_out) {
#pragma unroll
        for (int j = 0; j < 3; ++j) {
            lo_out[j] = lo[j];
            hi_out[j] = hi[j];
        }
    }
}

__device__ __forceinline__ void pad_slot(const fs_scene& s, int k, int64_t e) {
    const float z[3] = {0.0f, 0.0f, 0.0f};
    const float id[9] = {1.0f, 0.0f, 0.0f, 0.0f, 1.0f, 0.0f, 0.0f, 0.0f, 1.0f};
    store_slot(s, k, e, z, z, z, z, id, FS_PRIM_PAD, 0, 0);
}

// instance j's pose at reset counter c (world.py:233-240, assets.py:
// place_instances): position from Philox block kPoseBlock + j, orientation
// (ZYX Euler -> quaternion) from block kPoseBlock + kPoseEuler + j
__device__ __forceinline__ void instance_position(const fs_asset_class& cl, const U4& bp,
                                                  const double* bounds, double* ip) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double frac = cl.position_min[i] + u01d(word_of(bp, i)) *
                                                     (cl.position_max[i] - cl.position_min[i]);
        ip[i] = (cl.frozen_mask >> i & 1) ? cl.frozen_value[i] : frac * bounds[i];
    }
}

__device__ __forceinline__ void instance_rotation(const fs_asset_class& cl, const U4& be,
                                                  double* iq) {
    double eul[3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
        eul[i] = cl.euler_min[i] + u01d(word_of(be, i)) * (cl.euler_max[i] - cl.euler_min[i]);
    rot_zyx_d(eul[0], eul[1], eul[2], iq);
}

// reset_env's obstacle half (world.py:233-240): fresh poses for every
// randomizable instance, walls appended unchanged, rows recompiled, the rest
// padded.  bounds: EnvConfig.bounds.
__device__ __forceinline__ void rebuild_env(const fs_obstacles& ob, int64_t e, uint64_t seed,
                                            int64_t gid, uint32_t c, const double* bounds) {
    int k = 0;
    for (int j = 0; j < ob.instances_per_env; ++j) {
        const fs_asset_class& cl = ob.classes[class_of(ob, j)];
        double ip[3], iq[4];
        instance_position(cl, draw_block(seed, gid, c, kPoseBlock + (uint32_t)j), bounds, ip);
        instance_rotation(cl, draw_block(seed, gid, c, kPoseBlock + kPoseEuler + (uint32_t)j), iq);
        if (ob.inst_pose) {
#pragma unroll
            for (int i = 0; i < 3; ++i) ob.inst_pose[(int64_t)(7 * j + i) * ob.plane_stride + e] = ip[i];
#pragma unroll
            for (int i = 0; i < 4; ++i)
                ob.inst_pose[(int64_t)(7 * j + 3 + i) * ob.plane_stride + e] = iq[i];
        }
        const int32_t p = inst_proto(ob, j, e);
        for (int q = ob.proto_offset[p]; q < ob.proto_offset[p + 1]; ++q)
            write_slot(ob, k++, e, ob.proto_prims[q], ip, iq, cl.segmentation_id,
                       cl.collision_enabled);
    }
    if (ob.wall_proto >= 0) {
        const double zp[3] = {0.0, 0.0, 0.0}, id[4] = {1.0, 0.0, 0.0, 0.0};
        for (int q = ob.proto_offset[ob.wall_proto]; q < ob.proto_offset[ob.wall_proto + 1]; ++q)
            write_slot(ob, k++, e, ob.proto_prims[q], zp, id, ob.wall_seg, FS_COLL_WALL);
    }
    for (; k < ob.scene.width; ++k) pad_slot(ob.scene, k, e);
}

// randomize_mount (camera.py:238-244): U(-1, 1) bounds around the nominal mount
__device__ __forceinline__ void randomize_mount_d(const fs_obstacles& ob, int64_t e,
                                                  uint64_t seed, int64_t gid, uint32_t c) {
    const U4 bp = draw_block(seed, gid, c, kMountBlock);
    const U4 be = draw_block(seed, gid, c, kMountBlock + 1);
    double eul[3], q[4];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        const double dp = (-1.0 + 2.0 * u01d(word_of(bp, i))) * ob.randomize_position[i];
        const double de = (-1.0 + 2.0 * u01d(word_of(be, i))) * ob.randomize_euler[i];
        ob.mount[(int64_t)i * ob.mount_stride + e] = ob.mount_position[i] + dp;
        eul[i] = ob.mount_euler[i] + de;
    }
    rot_zyx_d(eul[0], eul[1], eul[2], q);
#pragma unroll
    for (int i = 0; i < 4; ++i) ob.mount[(int64_t)(3 + i) * ob.mount_stride + e] = q[i];
}

// ---- warp-cooperative obstacle reset (one warp per env) ---------------------------
//
// Same draws and arithmetic as rebuild_env; the lanes share the work: lane
// j computes instance j's pose and slot count, a warp prefix sum places the
// instances' slot runs, then the lanes write the slots (and pads) round-robin
// and finally the per-instance broad-phase boxes.  `sm` holds up to
// kMaxInstWarp instance records (walls included) of this warp.
constexpr int kMaxInstWarp = 64;

struct InstS {
    double p[3], q[4];
    int32_t first, count, proto, cls;     // cls -1: the walls
    // the instance's AABB over its slots' (outward-rounded) boxes, as
    // order-preserving int keys of the fp32 bounds (shared-memory atomics)
    int32_t lo[3], hi[3];
};

// order-preserving float <-> int32 keys (atomicMin / atomicMax on floats)
__device__ __forceinline__ int32_t fkey(float f) {
    const int32_t i = __float_as_int(f);
    return i >= 0 ? i : i ^ 0x7FFFFFFF;
}
__device__ __forceinline__ float funkey(int32_t k) {
    return __int_as_float(k >= 0 ? k : k ^ 0x7FFFFFFF);
}

// s2i / s2p (nullptr or kSlotTable entries): slot -> instance and slot ->
// prototype primitive tables for the slot writes (else a linear search over
// the instances' first slots)
constexpr int kSlotTable = 256;

// the instances' poses, prototypes and slot ranges of env e (one warp;
// `recs` in shared or global memory, nI records); returns the used slots
__device__ __forceinline__ int warp_rebuild_poses(const fs_obstacles& ob, int64_t e, uint64_t seed,
                                                  int64_t gid, uint32_t c, const double* bounds,
                                                  InstS* recs, int lane) {
    const int J = ob.instances_per_env;
    const int nI = J + (ob.wall_proto >= 0 ? 1 : 0);
    // up to 16 instances: lane j draws instance j's position, lane 16 + j its
    // orientation (the two Philox blocks and the Euler -> quaternion in
    // parallel); else lane j does both for instance j0 + j
    const bool split = nI <= 16;
    const bool pos_lane = !split || lane < 16;
    const bool rot_lane = !split || lane >= 16;
    int carry = 0;
    for (int j0 = 0; j0 < nI; j0 += 32) {
        const int j = j0 + (split ? (lane & 15) : lane);
        int cnt = 0;
        if (j < J) {
            const int cl_i = class_of(ob, j);
            const fs_asset_class& cl = ob.classes[cl_i];
            InstS& r = recs[j];
            if (pos_lane) {
                instance_position(cl, draw_block(seed, gid, c, kPoseBlock + (uint32_t)j), bounds,
                                  r.p);
                r.proto = inst_proto(ob, j, e);
                r.cls = cl_i;
                cnt = ob.proto_offset[r.proto + 1] - ob.proto_offset[r.proto];
                if (ob.inst_pose) {
#pragma unroll
                    for (int i = 0; i < 3; ++i)
                        ob.inst_pose[(int64_t)(7 * j + i) * ob.plane_stride + e] = r.p[i];
                }
            }
            if (rot_lane) {
                instance_rotation(cl, draw_block(seed, gid, c, kPoseBlock + kPoseEuler + (uint32_t)j),
                                  r.q);
                if (ob.inst_pose) {
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        ob.inst_pose[(int64_t)(7 * j + 3 + i) * ob.plane_stride + e] = r.q[i];
                }
            }
        } else if (j == J && j < nI) {
            InstS& r = recs[j];
            if (pos_lane) {
                r.p[0] = r.p[1] = r.p[2] = 0.0;
                r.proto = ob.wall_proto;
                r.cls = -1;
                cnt = ob.proto_offset[r.proto + 1] - ob.proto_offset[r.proto];
            }
            if (rot_lane) {
                r.q[0] = 1.0;
                r.q[1] = r.q[2] = r.q[3] = 0.0;
            }
        }
        // inclusive warp scan of the slot counts (0 on the orientation lanes)
        int incl = cnt;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, incl, off);
            if (lane >= off) incl += v;
        }
        if (pos_lane && j < nI) {
            recs[j].first = carry + incl - cnt;
            recs[j].count = cnt;
#pragma unroll
            for (int f = 0; f < 3; ++f) {
                recs[j].lo[f] = fkey(3.0e38f);
                recs[j].hi[f] = fkey(-3.0e38f);
            }
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
    }
    __syncwarp();
    return carry;
}

// slot k of env e from its instance record r and prototype primitive pi
// (compile_instances' per-primitive body); the slot's box is folded into the
// record's AABB keys with atomics (shared or global memory)
__device__ __forceinline__ void rebuild_slot(const fs_obstacles& ob, int64_t e, int k, InstS& r,
                                             int pi) {
    const fs_proto_prim& pp = ob.proto_prims[pi];
    float lo[3], hi[3];
    if (r.cls < 0) {
        write_slot(ob, k, e, pp, r.p, r.q, ob.wall_seg, FS_COLL_WALL, lo, hi);
    } else {
        const fs_asset_class& cl = ob.classes[r.cls];
        write_slot(ob, k, e, pp, r.p, r.q, cl.segmentation_id, cl.collision_enabled, lo, hi);
    }
#pragma unroll
    for (int f = 0; f < 3; ++f) {
        atomicMin(&r.lo[f], fkey(lo[f]));
        atomicMax(&r.hi[f], fkey(hi[f]));
    }
}

// the instance broad-phase records of env e from its J instance records
__device__ __forceinline__ void write_inst_boxes(const fs_obstacles& ob, int64_t e,
                                                 const InstS* recs, int lane) {
    if (!ob.inst_box) return;
    for (int j = lane; j < ob.instances_per_env; j += 32) {
        float lo[3], hi[3];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            lo[f] = funkey(recs[j].lo[f]);
            hi[f] = funkey(recs[j].hi[f]);
        }
        const int32_t span = recs[j].first | (recs[j].count << 16);
        const float coll = ob.classes[recs[j].cls].collision_enabled ? 1.0f : 0.0f;
        // instance-major: a warp of consecutive envs reads record j with
        // one coalesced 512-B request per half (scene_hit_inst)
        float4* base = reinterpret_cast<float4*>(ob.inst_box);
        base[(int64_t)(2 * j) * ob.plane_stride + e] =
            make_float4(lo[0], lo[1], lo[2], __int_as_float(span));
        base[(int64_t)(2 * j + 1) * ob.plane_stride + e] = make_float4(hi[0], hi[1], hi[2], coll);
    }
}

__device__ __forceinline__ void warp_rebuild_env(const fs_obstacles& ob, int64_t e, uint64_t seed,
                                                 int64_t gid, uint32_t c, const double* bounds,
                                                 InstS* sm, int lane, uint8_t* s2i = nullptr,
                                                 uint16_t* s2p = nullptr) {
    const int nI = ob.instances_per_env + (ob.wall_proto >= 0 ? 1 : 0);
    const int used = warp_rebuild_poses(ob, e, seed, gid, c, bounds, sm, lane);
    // slot -> (instance, prototype primitive) tables for the slot writes
    bool table = s2i && s2p && used <= kSlotTable && nI <= 255;
    if (table) {
        bool big = false;       // primitive ids beyond uint16: no table
        for (int j = lane; j < nI; j += 32)
            big |= ob.proto_offset[sm[j].proto] + sm[j].count > 65536;
        table = !__any_sync(0xffffffffu, big);
    }
    if (table) {
        for (int j = lane; j < nI; j += 32) {
            const int p0 = ob.proto_offset[sm[j].proto] - sm[j].first;
            for (int k = sm[j].first; k < sm[j].first + sm[j].count; ++k) {
                s2i[k] = (uint8_t)j;
                s2p[k] = (uint16_t)(p0 + k);
            }
        }
        __syncwarp();
    }
    const int K = ob.scene.width;
    for (int k = lane; k < K; k += 32) {
        if (k >= used) {
            pad_slot(ob.scene, k, e);
            continue;
        }
        int j = 0, pi;
        if (table) {
            j = s2i[k];
            pi = s2p[k];
        } else {
            while (j + 1 < nI && sm[j + 1].first <= k) ++j;
            pi = ob.proto_offset[sm[j].proto] + (k - sm[j].first);
        }
        rebuild_slot(ob, e, k, sm[j], pi);
    }
    __syncwarp();
    write_inst_boxes(ob, e, sm, lane);
    __syncwarp();
}

// is the point farther than rr from every collision-enabled instance box of
// the rebuilt env (shared-memory boxes, lanes over instances; warp-uniform)?
// Then no primitive is within r and scene_hit is false without a global read.
__device__ __forceinline__ bool warp_far_from_instances(const fs_obstacles& ob, const InstS* sm,
                                                        const float* p, float rr, int lane) {
    const int J = ob.instances_per_env;
    bool near = false;
    for (int j = lane; j < J; j += 32) {
        if (!ob.classes[sm[j].cls].collision_enabled) continue;
        float d2 = 0.0f;
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            const float dd = fmaxf(fmaxf(funkey(sm[j].lo[f]) - p[f], p[f] - funkey(sm[j].hi[f])),
                                   0.0f);
            d2 += dd * dd;
        }
        near |= d2 < rr * rr;
    }
    return !__any_sync(0xffffffffu, near);
}

// scene_hit over the lanes of a warp (warp-uniform result)
__device__ __forceinline__ bool warp_scene_hit(const fs_scene& s, int64_t e, double px, double py,
                                               double pz, double r, int lane) {
    bool hit = false;
    for (int k = lane; k < s.width && !hit; k += 32) hit = slot_hit(s, k, e, px, py, pz, r);
    return __any_sync(0xffffffffu, hit);
}

}  // namespace fs
