// Library-level entry points and CUDA error plumbing of libmpm_b200.so.
#include <atomic>
#include <stdio.h>
#include <string.h>

#include "mpm_common.cuh"

namespace mpm {

static thread_local char g_last_error[512] = "";

void set_last_error(const char *what, cudaError_t e)
{
    snprintf(g_last_error, sizeof g_last_error, "%s: %s (%s)", what, cudaGetErrorString(e),
             cudaGetErrorName(e));
}

// Launch-time errors only (bad configuration, no device, no kernel image): the call stays
// asynchronous.  Execution errors surface at the host's next synchronisation.
static std::atomic<unsigned long long> g_launches{0};

thread_local bool g_plain_launch = false;

unsigned long long launch_counter_add(unsigned long long n)
{
    return g_launches.fetch_add(n, std::memory_order_relaxed) + n;
}

int check_launch(const char *what, int n_kernels)
{
    g_launches.fetch_add((unsigned long long)n_kernels, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) return MPM_OK;
    set_last_error(what, e);
    return MPM_ERR_RESOURCE;
}

}  // namespace mpm

extern "C" {

const char *mpm_version(void) { return "mpm_b200 0.1 (sm_100a)"; }

const char *mpm_last_error(void) { return mpm::g_last_error; }

unsigned long long mpm_launch_count(void) { return mpm::g_launches.load(std::memory_order_relaxed); }

int mpm_device_arch(void)
{
    int dev = 0, major = 0, minor = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return 0; }
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
    return major * 10 + minor;
}

void *mpm_host_alias(void *pinned_host)
{
    void *dev = nullptr;
    if (!pinned_host || cudaHostGetDevicePointer(&dev, pinned_host, 0) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    return dev;
}

// Peer memory: a buffer exported by another process (cudaIpcGetMemHandle through torch's
// storage sharing) is opened in THIS process's current-device context.  With
// cudaIpcMemLazyEnablePeerAccess the driver enables peer access between the current device and
// the exporting device, so the mapping is valid for kernels of the current device -- over NVLink
// when the exporter is another GPU of the node.
int mpm_ipc_open(const void *handle64, void **base_out)
{
    if (!handle64 || !base_out) return MPM_ERR_REJECTED_INPUT;
    cudaIpcMemHandle_t h;
    static_assert(sizeof(h) == 64, "CUDA IPC memory handles are 64 bytes");
    memcpy(&h, handle64, sizeof h);
    cudaError_t e = cudaIpcOpenMemHandle(base_out, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        cudaGetLastError();
        mpm::set_last_error("mpm_ipc_open", e);
        return MPM_ERR_RESOURCE;
    }
    return MPM_OK;
}

// One word read back from a device pointer (blocking): the probe a rank uses to check that a
// peer mapping really is reachable from its device before it relies on it.
int mpm_peek_i32(const int32_t *dev_ptr, int32_t *out_host)
{
    if (!dev_ptr || !out_host) return MPM_ERR_REJECTED_INPUT;
    cudaError_t e = cudaMemcpy(out_host, dev_ptr, sizeof(int32_t), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        cudaGetLastError();
        mpm::set_last_error("mpm_peek_i32", e);
        return MPM_ERR_RESOURCE;
    }
    return MPM_OK;
}

int mpm_ipc_close(void *base)
{
    if (!base) return MPM_OK;
    cudaError_t e = cudaIpcCloseMemHandle(base);
    if (e != cudaSuccess) {
        cudaGetLastError();
        mpm::set_last_error("mpm_ipc_close", e);
        return MPM_ERR_RESOURCE;
    }
    return MPM_OK;
}

}  // extern "C"
