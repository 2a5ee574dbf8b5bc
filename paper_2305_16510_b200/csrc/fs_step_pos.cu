// fs_step_pos.cu -- instantiates the fused position-mode kernels (see fs_step.cuh).
#include "fs_step.cuh"

namespace fs {
int launch_position(const KParams& P, cudaStream_t s, bool rollout) {
    return launch_mode_prec<FS_MODE_POSITION>(P, s, rollout);
}
}  // namespace fs
