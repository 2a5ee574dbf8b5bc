// fs_step_mix.cu -- instantiates the fused mixed-mode kernels (see fs_step.cuh).
#include "fs_step.cuh"

namespace fs {
int launch_mixed(const KParams& P, cudaStream_t s, bool rollout) {
    return launch_mode_prec<FS_MODE_MIXED>(P, s, rollout);
}
}  // namespace fs
