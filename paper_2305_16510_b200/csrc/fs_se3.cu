// fs_se3.cu -- the rotation-group primitives of flocksim.se3 (se3.py:32-266)
// as batched float64 device kernels: one thread per row, rows contiguous
// (AoS, the reference's (..., k) trailing layout).  The same operations as
// the reference's NumPy expressions; results agree to an ulp or two of
// float64 (fused multiply-adds, libdevice transcendentals).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "flocksim_b200.h"
#include "fs_scene.cuh"   // qmul_d, qrot_d, qmat_d, rot_zyx_d

namespace fs {
int check_launch(const char* what);
}
int fs_fail_einval(const char* msg);

namespace fs {

__device__ __forceinline__ void qnorm_d(const double* q, double* o) {
    const double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
    o[0] = q[0] / n;
    o[1] = q[1] / n;
    o[2] = q[2] / n;
    o[3] = q[3] / n;
}

// quat_from_matrix (se3.py:156-197): Shepperd's method, largest pivot,
// scalar part made non-negative, renormalized
__device__ __forceinline__ void qfrom_mat_d(const double* r, double* o) {
    const double m00 = r[0], m01 = r[1], m02 = r[2], m10 = r[3], m11 = r[4], m12 = r[5];
    const double m20 = r[6], m21 = r[7], m22 = r[8];
    const double tr = m00 + m11 + m22;
    const double c[4] = {sqrt(fmax(0.0, 1.0 + tr)) / 2.0, sqrt(fmax(0.0, 1.0 + m00 - m11 - m22)) / 2.0,
                         sqrt(fmax(0.0, 1.0 - m00 + m11 - m22)) / 2.0,
                         sqrt(fmax(0.0, 1.0 - m00 - m11 + m22)) / 2.0};
    int k = 0;                              // np.argmax: first maximum
    for (int j = 1; j < 4; ++j)
        if (c[j] > c[k]) k = j;
    const double den = 4.0 * c[k] == 0.0 ? 1.0 : 4.0 * c[k];
    double q[4];
    if (k == 0) {
        q[0] = c[0]; q[1] = (m21 - m12) / den; q[2] = (m02 - m20) / den; q[3] = (m10 - m01) / den;
    } else if (k == 1) {
        q[0] = (m21 - m12) / den; q[1] = c[1]; q[2] = (m01 + m10) / den; q[3] = (m02 + m20) / den;
    } else if (k == 2) {
        q[0] = (m02 - m20) / den; q[1] = (m01 + m10) / den; q[2] = c[2]; q[3] = (m12 + m21) / den;
    } else {
        q[0] = (m10 - m01) / den; q[1] = (m02 + m20) / den; q[2] = (m12 + m21) / den; q[3] = c[3];
    }
    const double sgn = q[0] < 0.0 ? -1.0 : 1.0;
    for (int j = 0; j < 4; ++j) q[j] *= sgn;
    qnorm_d(q, o);
}

// exp_so3 (se3.py:246-266): series of sin(theta/2)/theta below 1e-8
__device__ __forceinline__ void exp_so3_d(const double* w, double* o) {
    const double th = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    const bool small = th < 1e-8;
    const double safe = small ? 1.0 : th;
    const double k = small ? 0.5 - th * th / 48.0 : sin(safe / 2.0) / safe;
    const double q[4] = {cos(th / 2.0), k * w[0], k * w[1], k * w[2]};
    qnorm_d(q, o);
}

__global__ void __launch_bounds__(256) se3_kernel(int op, int64_t n, const double* __restrict__ a,
                                                  const double* __restrict__ b,
                                                  const double* __restrict__ c, double* out,
                                                  double* out2, double gimbal_cos) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    switch (op) {
        case FS_SE3_QUAT_NORMALIZE:
            qnorm_d(a + 4 * i, out + 4 * i);
            break;
        case FS_SE3_QUAT_MULTIPLY:
            qmul_d(a + 4 * i, b + 4 * i, out + 4 * i);
            break;
        case FS_SE3_QUAT_CONJUGATE: {
            const double* q = a + 4 * i;
            double* o = out + 4 * i;
            o[0] = q[0];
            o[1] = -q[1];
            o[2] = -q[2];
            o[3] = -q[3];
            break;
        }
        case FS_SE3_QUAT_ROTATE:
        case FS_SE3_QUAT_ROTATE_INVERSE: {
            const double* q = a + 4 * i;
            const double qq[4] = {q[0], op == FS_SE3_QUAT_ROTATE ? q[1] : -q[1],
                                  op == FS_SE3_QUAT_ROTATE ? q[2] : -q[2],
                                  op == FS_SE3_QUAT_ROTATE ? q[3] : -q[3]};
            qrot_d(qq, b + 3 * i, out + 3 * i);
            break;
        }
        case FS_SE3_QUAT_TO_MATRIX:
            qmat_d(a + 4 * i, out + 9 * i);
            break;
        case FS_SE3_QUAT_FROM_MATRIX:
            qfrom_mat_d(a + 9 * i, out + 4 * i);
            break;
        case FS_SE3_ROT_ZYX:
            rot_zyx_d(a[i], b[i], c[i], out + 4 * i);
            break;
        case FS_SE3_ROT_Z: {
            double s, co;
            sincos(a[i] / 2.0, &s, &co);
            double* o = out + 4 * i;
            o[0] = co;
            o[1] = 0.0;
            o[2] = 0.0;
            o[3] = s;
            break;
        }
        case FS_SE3_YAW_OF: {
            // se3.py:226-243: psi = atan2(R10, R00); gimbal flag |R20| >= cos(1e-6)
            const double* q = a + 4 * i;
            const double w = q[0], x = q[1], y = q[2], z = q[3];
            const double r10 = 2.0 * (x * y + w * z), r00 = 1.0 - 2.0 * (y * y + z * z);
            const double r20 = 2.0 * (x * z - w * y);
            out[i] = atan2(r10, r00);
            out2[i] = fabs(r20) >= gimbal_cos ? 1.0 : 0.0;
            break;
        }
        case FS_SE3_EXP_SO3:
            exp_so3_d(a + 3 * i, out + 4 * i);
            break;
        case FS_SE3_HAT: {
            const double* w = a + 3 * i;
            double* o = out + 9 * i;
            o[0] = 0.0; o[1] = -w[2]; o[2] = w[1];
            o[3] = w[2]; o[4] = 0.0; o[5] = -w[0];
            o[6] = -w[1]; o[7] = w[0]; o[8] = 0.0;
            break;
        }
        case FS_SE3_VEE: {
            // se3.py:51-67: (S21, S02, S10) and the row's max |S + S^T|
            const double* s = a + 9 * i;
            double res = 0.0;
            for (int r = 0; r < 3; ++r)
                for (int col = 0; col < 3; ++col)
                    res = fmax(res, fabs(s[3 * r + col] + s[3 * col + r]));
            out[3 * i] = s[7];
            out[3 * i + 1] = s[2];
            out[3 * i + 2] = s[3];
            out2[i] = res;
            break;
        }
        default:
            break;
    }
}

}  // namespace fs

extern "C" int fs_se3(int32_t op, int64_t n, const double* a, const double* b, const double* c,
                      double* out, double* out2, void* stream) {
    if (op < FS_SE3_QUAT_NORMALIZE || op > FS_SE3_VEE) return fs_fail_einval("unknown se3 op");
    if (n < 0) return fs_fail_einval("length must be >= 0");
    if (n == 0) return FS_OK;
    const bool two = op == FS_SE3_QUAT_MULTIPLY || op == FS_SE3_QUAT_ROTATE ||
                     op == FS_SE3_QUAT_ROTATE_INVERSE || op == FS_SE3_ROT_ZYX;
    if (!a || !out || (two && !b) || (op == FS_SE3_ROT_ZYX && !c) ||
        ((op == FS_SE3_YAW_OF || op == FS_SE3_VEE) && !out2))
        return fs_fail_einval("null se3 buffer");
    const unsigned blocks = (unsigned)((n + 255) / 256);
    fs::se3_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(op, n, a, b, c, out, out2,
                                                             cos(1e-6));
    return fs::check_launch("se3_kernel");
}
