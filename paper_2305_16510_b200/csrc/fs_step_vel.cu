// fs_step_vel.cu -- instantiates the fused velocity-mode kernels (see fs_step.cuh).
#include "fs_step.cuh"

namespace fs {
int launch_velocity(const KParams& P, cudaStream_t s, bool rollout) {
    return launch_mode_prec<FS_MODE_VELOCITY>(P, s, rollout);
}
}  // namespace fs
