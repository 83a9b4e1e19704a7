// C-ABI plumbing: error strings, device properties.
#include <cstdio>
#include <cstring>
#include <map>
#include <set>
#include <mutex>
#include <string>
#include <vector>

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
    // keep freed scratch in the stream-ordered pool instead of returning it to
    // the driver at every synchronisation (the kernels allocate per call)
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        unsigned long long keep = ~0ull;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
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

// ---- launch accounting ---------------------------------------------------------
struct ProfRecord {
    std::string name;
    cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::map<std::string, long long> g_counts;
static std::vector<ProfRecord> g_records;
static std::vector<cudaEvent_t> g_event_pool;

static cudaEvent_t take_event() {
    if (!g_event_pool.empty()) {
        cudaEvent_t e = g_event_pool.back();
        g_event_pool.pop_back();
        return e;
    }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}

static std::set<std::string> g_prof_only;  // empty: time every launch

ProfScope::ProfScope(const char* n, cudaStream_t s) : name(n), st(s), slot(-1) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_counts[name] += 1;
    if (g_prof_on && (g_prof_only.empty() || g_prof_only.count(name))) {
        ProfRecord r{name, take_event(), take_event()};
        cudaEventRecord(r.a, st);
        g_records.push_back(r);
        slot = (int)g_records.size() - 1;
    }
}

ProfScope::~ProfScope() {
    if (slot < 0) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    cudaEventRecord(g_records[slot].b, st);
}

}  // namespace pk

extern "C" void pk_prof_enable(int on) {
    std::lock_guard<std::mutex> lk(pk::g_prof_mu);
    pk::g_prof_on = on != 0;
    // events are created up front: cudaEventCreate inside a timed region stalls
    while (on && pk::g_event_pool.size() < 4096) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) break;
        pk::g_event_pool.push_back(e);
    }
}

// comma-separated kernel names whose launches get event timing ("" = all)
extern "C" void pk_prof_only(const char* names) {
    std::lock_guard<std::mutex> lk(pk::g_prof_mu);
    pk::g_prof_only.clear();
    std::string cur;
    for (const char* c = names ? names : ""; ; ++c) {
        if (*c == ',' || *c == 0) {
            if (!cur.empty()) pk::g_prof_only.insert(cur);
            cur.clear();
            if (*c == 0) break;
        } else {
            cur += *c;
        }
    }
}

// "name count total_ms\n" per kernel; counts since the last reset, times of the
// event-bracketed launches since the last collect.  reset != 0 clears both.
extern "C" int pk_prof_collect(char* buf, int len, int reset) {
    std::lock_guard<std::mutex> lk(pk::g_prof_mu);
    std::map<std::string, double> ms;
    for (auto& r : pk::g_records) {
        cudaEventSynchronize(r.b);
        float t = 0.f;
        cudaEventElapsedTime(&t, r.a, r.b);
        ms[r.name] += t;
        pk::g_event_pool.push_back(r.a);
        pk::g_event_pool.push_back(r.b);
    }
    pk::g_records.clear();
    std::string out;
    for (auto& kv : pk::g_counts) {
        char line[256];
        snprintf(line, sizeof line, "%s %lld %.6f\n", kv.first.c_str(), kv.second, ms[kv.first]);
        out += line;
    }
    if (reset) pk::g_counts.clear();
    int n = (int)out.size() < len - 1 ? (int)out.size() : len - 1;
    memcpy(buf, out.data(), n);
    buf[n] = 0;
    return (int)out.size();
}

extern "C" int pk_version(void) { return 1; }

extern "C" const char* pk_last_error(void) { return pk::g_err.c_str(); }

extern "C" int pk_device_info(int* sm_count, int* smem_optin) {
    if (sm_count) *sm_count = pk::sm_count();
    if (smem_optin) *smem_optin = pk::max_smem_optin();
    return 0;
}
