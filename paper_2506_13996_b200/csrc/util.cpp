// Process-wide plumbing: last-error slot, SM count, launch counter, version.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "common.h"
#include "launch.h"

namespace spt {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

void set_last_error(const std::string& msg) { g_last_error = msg; }

// SPT_TRACE=1: synchronise after every launch and log it (debugging hangs / async faults).
void count_launch(const char* tag) {
    const int64_t n = g_launches.fetch_add(1, std::memory_order_relaxed);
    static const bool trace = [] {
        const char* e = getenv("SPT_TRACE");
        return e && e[0] == '1';
    }();
    if (trace) {
        fprintf(stderr, "[spt] launch %lld %s ...", (long long)n, tag ? tag : "");
        fflush(stderr);
        cudaError_t e = cudaDeviceSynchronize();
        fprintf(stderr, " %s\n", cudaGetErrorString(e));
        fflush(stderr);
    }
}
int64_t launch_count() { return g_launches.load(std::memory_order_relaxed); }
void add_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

struct Prof;
Prof*& current_prof() {
    static thread_local Prof* p = nullptr;
    return p;
}

int num_sms() {
    static thread_local int dev_cached = -1, sms = 0;
    int dev = 0;
    SPT_CUDA(cudaGetDevice(&dev));
    if (dev != dev_cached) {
        SPT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        int major = 0, minor = 0;
        SPT_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
        SPT_CUDA(cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev));
        SPT_CHECK(major == 10 && minor == 0, SPT_ERR_CUDA,
                  "sptrain_b200 is built for sm_100a (B200); device reports sm_" + std::to_string(major) +
                      std::to_string(minor));
        dev_cached = dev;
    }
    return sms;
}

}  // namespace spt

extern "C" const char* spt_last_error(void) { return spt::g_last_error.c_str(); }
extern "C" const char* spt_version(void) { return "sptrain_b200 0.1 (sm_100a, tcgen05/TMA, NCCL)"; }
extern "C" int64_t spt_kernel_launch_count(void) { return spt::launch_count(); }
