// Library-level ABI: version, thread-local error string, launch accounting.
#include <atomic>
#include <string>

#include "pf_common.cuh"

namespace pf {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int status, const std::string& msg) {
    g_last_error = msg;
    return status;
}

int check_cuda(cudaError_t err, const char* what) {
    if (err == cudaSuccess) return PF_OK;
    g_last_error = std::string(what) + ": " + cudaGetErrorString(err);
    return PF_ERR_CUDA;
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

}  // namespace pf

extern "C" int pf_abi_version(void) { return PF_ABI_VERSION; }

extern "C" const char* pf_last_error(void) { return pf::g_last_error.c_str(); }

extern "C" uint64_t pf_launch_count(void) { return pf::g_launches.load(); }
