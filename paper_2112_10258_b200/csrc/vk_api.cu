// vk_api.cu -- error reporting and device queries for the C ABI.
#include <stdarg.h>

#include <atomic>
#include <stdio.h>

#include "vk_hood.cuh"

namespace vk {

static thread_local char g_last_error[512] = "";
static std::atomic<long long> g_launches{0};

void count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return VK_OK;
    set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    return VK_ERR_CUDA;
}

}  // namespace vk

extern "C" const char* vk_last_error(void) { return vk::g_last_error; }

extern "C" int vk_abi_version(void) { return VK_ABI_VERSION; }

extern "C" int vk_device_sm_count(int device) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return sms;
}

extern "C" int vk_memset_async(void* ptr, long long bytes, void* stream) {
    if (!ptr || bytes < 0) {
        vk::set_error("vk_memset_async: bad arguments");
        return VK_ERR_PARAMETER;
    }
    return vk::cuda_status(cudaMemsetAsync(ptr, 0, (size_t)bytes, vk::as_stream(stream)), "memset");
}

extern "C" long long vk_launch_count(void) { return vk::g_launches.load(); }

extern "C" long long vk_accum_work_bytes(int device) {
    const int sms = vk_device_sm_count(device);
    if (sms <= 0) {
        vk::set_error("vk_accum_work_bytes: no device %d", device);
        return -1;
    }
    return (long long)sms * vk::kAccumCtasPerSm * vk::kAccumSlot * (long long)sizeof(double);
}
