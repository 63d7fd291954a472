// C-ABI plumbing: error text, version, device check.
#include "common.cuh"

namespace ublr {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
}  // namespace ublr

extern "C" const char* ublr_last_error(void) { return ublr::g_last_error.c_str(); }

extern "C" int ublr_version(void) { return 1; }

// Verifies a CUDA device is present and is sm_100 (the kernels are built for
// sm_100a only; there is no fallback path).
extern "C" int ublr_device_check(void) {
  int dev = 0;
  UBLR_CUDA(cudaGetDevice(&dev));
  cudaDeviceProp p;
  UBLR_CUDA(cudaGetDeviceProperties(&p, dev));
  UBLR_REQUIRE(p.major == 10 && p.minor == 0, UBLR_ERR_VALUE,
               std::string("ublr_b200 is built for sm_100a; found ") + p.name);
  return UBLR_OK;
}
