// C ABI bookkeeping: error strings, version, device probe.
#include <cstdio>
#include <string>

#include "common.cuh"

namespace sbo {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(SBO_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return SBO_OK;
}

}  // namespace sbo

extern "C" int sbo_abi_version(void) { return 1; }

extern "C" const char* sbo_last_error(void) { return sbo::g_last_error.c_str(); }

extern "C" int sbo_device_ok(int device) {
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return 0;
  return prop.major == 10 ? 1 : 0;
}
