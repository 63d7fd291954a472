// Test-only host build of the RNG decode (philox_zig.cuh) so the CPU test
// suite can check Philox words and the serial ziggurat decode against numpy.
#include <cstdint>
#include "philox_zig.cuh"
#include "ziggurat_tables.h"

struct HostWords {
  uint64_t k0, k1;
  uint64_t operator()(int64_t w) const { return ublr::rng::philox_word(k0, k1, (uint64_t)w); }
};

extern "C" void host_philox_words(uint64_t k0, uint64_t k1, int64_t n, uint64_t* out) {
  for (int64_t w = 0; w < n; ++w) out[w] = ublr::rng::philox_word(k0, k1, (uint64_t)w);
}

extern "C" int64_t host_normals(uint64_t k0, uint64_t k1, int64_t n, double* out) {
  double wi[256], fi[256];
  for (int i = 0; i < 256; ++i) {
    uint64_t a = ublr::zig::H_WI_BITS[i], b = ublr::zig::H_FI_BITS[i];
    __builtin_memcpy(&wi[i], &a, 8);
    __builtin_memcpy(&fi[i], &b, 8);
  }
  HostWords ws{k0, k1};
  int64_t p = 0;
  for (int64_t i = 0; i < n;) {
    double v; bool ok;
    p += ublr::rng::zig_token(ws, p, ublr::zig::H_KI, wi, fi, v, ok);
    if (ok) out[i++] = v;
  }
  return p;  // words consumed
}

extern "C" void host_log1p(const double* x, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = ublr::rng::log1p_host_exact(x[i]);
}

// the host C library's log1p (what numpy's ziggurat calls through npy_log1p)
extern "C" void host_libm_log1p(const double* x, int64_t n, double* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = log1p(x[i]);
}
