// Probe: does a programmatic dependent launch (PDL) overlap the previous
// kernel, eagerly and inside a captured CUDA graph, on this driver?
// Kernel A: 148 CTAs, CTA b spins (1 + b % 8) * 2 us, triggers its
// dependents at the start, records its end time.  Kernel B (PDL secondary):
// records each CTA's start time.  Overlap <=> min(B start) < max(A end).
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a tools/pdl_probe.cu -o /tmp/pdl_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint64_t gns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void kern_a(uint64_t* end, int trigger) {
    if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const uint64_t t0 = gns();
    const uint64_t spin = 2000ull * (1 + blockIdx.x % 8);
    while (gns() - t0 < spin) {}
    __syncthreads();
    if (threadIdx.x == 0) end[blockIdx.x] = gns();
}

__global__ void kern_b(uint64_t* start) {
    if (threadIdx.x == 0) start[blockIdx.x] = gns();
}

static void report(const char* what, const uint64_t* e, const uint64_t* s, int n) {
    uint64_t emax = 0, emin = ~0ull, smin = ~0ull;
    for (int i = 0; i < n; ++i) {
        emax = e[i] > emax ? e[i] : emax;
        emin = e[i] < emin ? e[i] : emin;
        smin = s[i] < smin ? s[i] : smin;
    }
    printf("%-26s A ends %.2f..%.2f us, first B start at %+.2f us vs last A end -> %s\n", what,
           0.0, (emax - emin) / 1e3, ((double)smin - (double)emax) / 1e3,
           smin < emax ? "OVERLAP" : "serialized");
}

int main() {
    const int n = 148;
    uint64_t *e, *s;
    cudaMallocManaged(&e, n * sizeof(uint64_t));
    cudaMallocManaged(&s, n * sizeof(uint64_t));
    cudaStream_t st;
    cudaStreamCreate(&st);
    // B needs an SM's worth of smem so it cannot co-reside with A (like the step kernel)
    const int big = 200 * 1024;
    cudaFuncSetAttribute(kern_b, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    cudaFuncSetAttribute(kern_a, cudaFuncAttributeMaxDynamicSharedMemorySize, big);
    auto launch = [&](int pdl, int trigger) {
        kern_a<<<n, 128, big, st>>>(e, trigger);
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(n);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = big;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = pdl;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern_b, s);
    };
    for (int rep = 0; rep < 2; ++rep) {
        launch(0, 0);
        cudaStreamSynchronize(st);
        report("eager, plain", e, s, n);
        launch(1, 1);
        cudaStreamSynchronize(st);
        report("eager, PDL", e, s, n);
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        launch(1, 1);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        report("graph, PDL", e, s, n);
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        launch(0, 0);
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
        cudaGraphLaunch(ge, st);
        cudaStreamSynchronize(st);
        report("graph, plain", e, s, n);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
