// Host-side helpers shared by the C-ABI translation units (hm_index.cpp,
// hm_bridge.cpp): the thread-local error message behind hm_last_error(),
// status mapping of C++ exceptions, device selection.
#pragma once
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "hm_b200.h"

namespace hm_host {

struct no_device_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

std::string& error_slot();  // this thread's hm_last_error() message

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}

// invalid_argument -> HM_ERR_INVALID, out_of_range -> HM_ERR_RANGE, other
// exceptions -> HM_ERR_RUNTIME (the reference's exception types)
template <typename F>
int guard(F&& f) {
    try {
        f();
        return HM_OK;
    } catch (const no_device_error& e) {
        error_slot() = e.what();
        return HM_ERR_NO_DEVICE;
    } catch (const std::invalid_argument& e) {
        error_slot() = e.what();
        return HM_ERR_INVALID;
    } catch (const std::out_of_range& e) {
        error_slot() = e.what();
        return HM_ERR_RANGE;
    } catch (const std::exception& e) {
        error_slot() = e.what();
        return HM_ERR_RUNTIME;
    } catch (...) {
        error_slot() = "unknown error";
        return HM_ERR_RUNTIME;
    }
}

inline void use_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        throw no_device_error("no CUDA device available (the B200 path has no CPU fallback)");
    if (device < 0 || device >= n) throw std::invalid_argument("device ordinal out of range");
    ck(cudaSetDevice(device), "cudaSetDevice");
}

}  // namespace hm_host
