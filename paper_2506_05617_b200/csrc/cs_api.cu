// cs_api.cu -- error plumbing and version of the C-ABI (include/convspectra_b200.h).
#include <string>

#include "cs_common.cuh"

namespace cs {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int fail(int status, const std::string &msg) {
    g_last_error = msg;
    return status;
}

int cuda_status(cudaError_t e, const char *what) {
    g_last_error = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
    return (e == cudaErrorMemoryAllocation) ? CS_ENOMEM : CS_ECUDA;
}

}  // namespace cs

extern "C" int cs_abi_version(void) { return CS_ABI_VERSION; }

extern "C" const char *cs_last_error_string(void) { return cs::g_last_error.c_str(); }
