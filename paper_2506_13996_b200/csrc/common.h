// Host-side plumbing shared by the C-ABI layer: status codes, thread-local last error, CUDA checks.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/sptrain_b200.h"

namespace spt {

// Exceptions mirror proj/include/sptrain/errors.hpp:12-72; the C-ABI maps them onto spt_status.
struct SptError : std::runtime_error {
    spt_status code;
    SptError(spt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_last_error(const std::string& msg);

#define SPT_THROW(code, msg) throw ::spt::SptError((code), (msg))

#define SPT_CUDA(call)                                                                                  \
    do {                                                                                                \
        cudaError_t e_ = (call);                                                                        \
        if (e_ != cudaSuccess)                                                                          \
            SPT_THROW(SPT_ERR_CUDA, std::string(#call " failed: ") + cudaGetErrorString(e_) + " at " + \
                                        __FILE__ + ":" + std::to_string(__LINE__));                     \
    } while (0)

#define SPT_CHECK(cond, code, msg)     \
    do {                               \
        if (!(cond)) SPT_THROW(code, msg); \
    } while (0)

// Wrap a C-ABI body: exceptions -> status + spt_last_error().
template <class F>
spt_status capi_guard(F&& f) {
    try {
        f();
        return SPT_OK;
    } catch (const SptError& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc& e) {
        set_last_error(std::string("host allocation failed: ") + e.what());
        return SPT_ERR_OOM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return SPT_ERR_INTERNAL;
    }
}

int num_sms();

}  // namespace spt
