// fs_step_att.cu -- instantiates the fused attitude-mode kernels (see fs_step.cuh).
#include "fs_step.cuh"

namespace fs {
int launch_attitude(const KParams& P, cudaStream_t s, bool rollout) {
    return launch_mode_prec<FS_MODE_ATTITUDE>(P, s, rollout);
}
}  // namespace fs
