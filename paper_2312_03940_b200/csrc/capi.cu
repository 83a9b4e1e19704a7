// C-ABI plumbing: error strings, device properties.
#include <cstdio>
#include <string>

#include "../../include/peakann_b200.h"
#include "api.cuh"

namespace pk {

static thread_local std::string g_err;

void set_error(const std::string& msg) { g_err = msg; }

int fail(const char* where, cudaError_t e) {
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return 1;
}

static int g_sms = -1, g_smem = -1;

static void query_device() {
    if (g_sms > 0) return;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&g_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (g_sms <= 0) g_sms = 148;
    if (g_smem <= 0) g_smem = 227 * 1024;
}

int sm_count() {
    query_device();
    return g_sms;
}

int max_smem_optin() {
    query_device();
    return g_smem;
}

}  // namespace pk

extern "C" int pk_version(void) { return 1; }

extern "C" const char* pk_last_error(void) { return pk::g_err.c_str(); }

extern "C" int pk_device_info(int* sm_count, int* smem_optin) {
    if (sm_count) *sm_count = pk::sm_count();
    if (smem_optin) *smem_optin = pk::max_smem_optin();
    return 0;
}
