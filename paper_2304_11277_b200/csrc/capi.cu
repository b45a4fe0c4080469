// C-ABI plumbing: error strings, launch accounting, version.
#include <atomic>
#include <mutex>

#include "common.cuh"

namespace fsdp {

static thread_local std::string g_last_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

int check_cuda(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return (int)e;
}

void count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

}  // namespace fsdp

extern "C" const char* fsdp_last_error(void) { return fsdp::g_last_error.c_str(); }
extern "C" int fsdp_abi_version(void) { return 1; }
extern "C" uint64_t fsdp_launch_count(void) { return fsdp::g_launches.load(); }
extern "C" int fsdp_num_sms(int device) {
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
  return v;
}
