// fs_host.h -- host-side helpers shared by the launchers.
//
// Launchers cache per-kernel setup (the opt-in dynamic shared-memory size,
// occupancy-derived grid limits, the SM count).  Those facts belong to a
// CUDA device, not to the process: the caches are keyed by the current
// device and guarded, so two host threads, or a second GPU in the same
// process, each get their own correctly initialised copy.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

namespace fs {

constexpr int kMaxDevices = 64;

inline int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    return dev;
}

// Runs init(dev) once per CUDA device (thread-safe) and returns the device.
struct PerDeviceOnce {
    std::mutex mu;
    uint64_t done = 0;
    template <class F>
    int operator()(F&& init) {
        const int dev = current_device();
        if (dev < 0 || dev >= kMaxDevices) {   // (no device / out of range: do it every time)
            init(dev < 0 ? 0 : dev);
            return dev < 0 ? 0 : dev;
        }
        std::lock_guard<std::mutex> g(mu);
        if (!((done >> dev) & 1u)) {
            init(dev);
            done |= 1ull << dev;
        }
        return dev;
    }
};

}  // namespace fs
