// Per-device launch state shared by the kernel launchers.
//
// The dynamic shared-memory opt-in (cudaFuncAttributeMaxDynamicSharedMemorySize) belongs to a
// (kernel, device context) pair, and layers may be created on several GPUs and shared across
// host threads (sfc_b200.h), so the "already raised to N bytes" cache is kept per device, read
// lock-free and raised under a mutex (the attribute is only ever raised, never lowered).
#pragma once
#include <atomic>
#include <cstddef>
#include <mutex>
#include <cuda_runtime.h>

namespace sfcb200 {

constexpr int kMaxDevices = 64;

inline int current_device() {
    int dev = 0;
    cudaGetDevice(&dev);
    return dev >= 0 && dev < kMaxDevices ? dev : 0;
}

struct SmemOptIn {
    std::atomic<size_t> bytes[kMaxDevices] = {};
    std::mutex mu;

    // Make sure `kern` may use `smem` bytes of dynamic shared memory on the current device.
    template <class Kern>
    cudaError_t ensure(Kern kern, size_t smem) {
        const int dev = current_device();
        if (bytes[dev].load(std::memory_order_acquire) >= smem) return cudaSuccess;
        std::lock_guard<std::mutex> lk(mu);
        const size_t have = bytes[dev].load(std::memory_order_relaxed);
        if (have >= smem) return cudaSuccess;
        const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        if (e == cudaSuccess) bytes[dev].store(smem, std::memory_order_release);
        return e;
    }
};

// Streaming multiprocessors of the current device (148 on B200), cached per device.
inline int device_sm_count() {
    static std::atomic<int> n[kMaxDevices] = {};
    const int dev = current_device();
    int v = n[dev].load(std::memory_order_relaxed);
    if (v <= 0) {
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        if (v <= 0) v = 148;
        n[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

}  // namespace sfcb200
