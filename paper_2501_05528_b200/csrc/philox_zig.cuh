// numpy-compatible Philox4x64-10 + ziggurat standard normals (host + device).
//
// Restates the published algorithms behind the reference's RandomStream
// (ref/linalg.py:14-52): numpy 2.3's `Philox` bit generator (Random123
// Philox4x64 with 10 rounds; the 256-bit counter is incremented BEFORE each
// block of 4 words, so word w comes from counter w/4 + 1) and numpy's
// `random_standard_normal` ziggurat (Marsaglia-Tsang, 256 strips, one uint64
// per attempt: 8 bits strip index, 1 sign bit, 52 bits magnitude; wedge and
// tail draws consume further words as doubles (u >> 11) * 2^-53).
// The ziggurat tables are numpy's own (generated header, see
// tools/gen_ziggurat_tables.py). Non-contracted arithmetic (__dmul_rn /
// __dadd_rn) keeps accept/reject decisions identical to numpy's C code.
#pragma once
#include <cstdint>
#include <cmath>

#ifdef __CUDACC__
#define UBLR_HD __host__ __device__ __forceinline__
#else
#define UBLR_HD inline
#endif

namespace ublr {
namespace rng {

constexpr uint64_t PHILOX_M0 = 0xD2E7470EE14C6C93ULL;
constexpr uint64_t PHILOX_M1 = 0xCA5A826395121157ULL;
constexpr uint64_t PHILOX_W0 = 0x9E3779B97F4A7C15ULL;
constexpr uint64_t PHILOX_W1 = 0xBB67AE8584CAA73BULL;
constexpr double ZIG_R = 3.6541528853610087963519472518;
constexpr double ZIG_INV_R = 0.27366123732975827203338247596;

UBLR_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#ifdef __CUDA_ARCH__
  lo = a * b;
  hi = __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  lo = (uint64_t)p;
  hi = (uint64_t)(p >> 64);
#endif
}

// Philox4x64-10 of counter (c0, 0, 0, 0) under key (k0, k1).
UBLR_HD void philox4x64_10(uint64_t c0, uint64_t k0, uint64_t k1, uint64_t out[4]) {
  uint64_t x0 = c0, x1 = 0, x2 = 0, x3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += PHILOX_W0;
      k1 += PHILOX_W1;
    }
    uint64_t hi0, lo0, hi1, lo1;
    mulhilo64(PHILOX_M0, x0, hi0, lo0);
    mulhilo64(PHILOX_M1, x2, hi1, lo1);
    uint64_t y0 = hi1 ^ x1 ^ k0;
    uint64_t y1 = lo1;
    uint64_t y2 = hi0 ^ x3 ^ k1;
    uint64_t y3 = lo0;
    x0 = y0; x1 = y1; x2 = y2; x3 = y3;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

// Word w (0-based) of the numpy Philox stream keyed (k0, k1).
UBLR_HD uint64_t philox_word(uint64_t k0, uint64_t k1, uint64_t w) {
  uint64_t o[4];
  philox4x64_10((w >> 2) + 1, k0, k1, o);
  return o[w & 3];
}

UBLR_HD double u64_to_unit(uint64_t v) { return (double)(v >> 11) * (1.0 / 9007199254740992.0); }

#ifdef __CUDA_ARCH__
#define UBLR_MUL(a, b) __dmul_rn((a), (b))
#define UBLR_ADD(a, b) __dadd_rn((a), (b))
#else
#define UBLR_MUL(a, b) ((a) * (b))
#define UBLR_ADD(a, b) ((a) + (b))
#endif

// One ziggurat attempt starting at word position p of a word source `ws`
// (ws(q) returns word q). Returns the number of words consumed and sets
// `ok` when the attempt yields a normal (written to `val`).
template <class WordSource>
UBLR_HD int zig_token(WordSource& ws, int64_t p, const uint64_t* ki, const double* wi, const double* fi,
                      double& val, bool& ok) {
  uint64_t r = ws(p);
  int idx = (int)(r & 0xff);
  r >>= 8;
  int sign = (int)(r & 0x1);
  uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
  double x = UBLR_MUL((double)rabs, wi[idx]);
  if (sign) x = -x;
  if (rabs < ki[idx]) {
    val = x;
    ok = true;
    return 1;
  }
  if (idx == 0) {
    int64_t q = p + 1;
    for (;;) {
      double u1 = u64_to_unit(ws(q));
      double u2 = u64_to_unit(ws(q + 1));
      q += 2;
      double xx = UBLR_MUL(-ZIG_INV_R, log1p(-u1));
      double yy = -log1p(-u2);
      if (UBLR_ADD(yy, yy) > UBLR_MUL(xx, xx)) {
        val = ((rabs >> 8) & 0x1) ? -UBLR_ADD(ZIG_R, xx) : UBLR_ADD(ZIG_R, xx);
        ok = true;
        return (int)(q - p);
      }
    }
  }
  double u = u64_to_unit(ws(p + 1));
  double lhs = UBLR_ADD(UBLR_MUL(fi[idx - 1] - fi[idx], u), fi[idx]);
  double rhs = exp(UBLR_MUL(UBLR_MUL(-0.5, x), x));
  ok = lhs < rhs;
  val = x;
  return 2;
}

}  // namespace rng
}  // namespace ublr
