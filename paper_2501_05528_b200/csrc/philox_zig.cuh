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
#define UBLR_SUB(a, b) __dsub_rn((a), (b))
#define UBLR_DIV(a, b) __ddiv_rn((a), (b))
#else
#define UBLR_MUL(a, b) ((a) * (b))
#define UBLR_ADD(a, b) ((a) + (b))
#define UBLR_SUB(a, b) ((a) - (b))
#define UBLR_DIV(a, b) ((a) / (b))
#endif

UBLR_HD int32_t hi_word(double x) {
#ifdef __CUDA_ARCH__
  return __double2hiint(x);
#else
  uint64_t b;
  __builtin_memcpy(&b, &x, 8);
  return (int32_t)(b >> 32);
#endif
}

UBLR_HD double with_hi_word(double x, int32_t h) {
#ifdef __CUDA_ARCH__
  return __hiloint2double(h, __double2loint(x));
#else
  uint64_t b;
  __builtin_memcpy(&b, &x, 8);
  b = (b & 0xffffffffULL) | ((uint64_t)(uint32_t)h << 32);
  __builtin_memcpy(&x, &b, 8);
  return x;
#endif
}

// log(1 + x), bit for bit as the host C library computes it for numpy's
// ziggurat tail (npy_log1p -> glibc 2.39 log1p, whose x86-64 build with FMA
// is selected on the hosts of this image). The algorithm is the published
// fdlibm one: 1 + x = 2^k (1 + f) with a rounding correction c,
// log(1 + f) = f - (hfsq - s (hfsq + R(s^2))), s = f / (2 + f), R a degree-7
// minimax polynomial in s^2 evaluated in Estrin form; the fused
// multiply-adds are placed where that build fuses them (checked against the
// host log1p over 6e7 arguments, tests/test_host.py). Used for -1 < x <= 0
// (x = -u, u a 53-bit uniform) but valid for every finite x > -1.
UBLR_HD double log1p_host_exact(double x) {
  constexpr double LN2_HI = 6.93147180369123816490e-01, LN2_LO = 1.90821492927058770002e-10;
  constexpr double P1 = 6.666666666666735130e-01, P2 = 3.999999999940941908e-01, P3 = 2.857142874366239149e-01,
                   P4 = 2.222219843214978396e-01, P5 = 1.818357216161805012e-01, P6 = 1.531383769920937332e-01,
                   P7 = 1.479819860511658591e-01;
  const int32_t hx = hi_word(x), ax = hx & 0x7fffffff;
  int k = 1, hu = 0;
  double f = 0.0, c = 0.0;
  if (hx < 0x3FDA827A) {                         // x < 0.41422 (every negative x)
    if (ax >= 0x3ff00000) return x == -1.0 ? -INFINITY : NAN;
    if (ax < 0x3e200000) {                       // |x| < 2^-29
      if (ax < 0x3c900000) return x;             // |x| < 2^-54
      return fma(-UBLR_MUL(x, x), 0.5, x);
    }
    if (hx > 0 || hx <= (int32_t)0xbfd2bec3) {   // -0.2929 < x < 0.41422: no reduction
      k = 0;
      f = x;
      hu = 1;
    }
  }
  if (hx >= 0x7ff00000) return UBLR_ADD(x, x);
  if (k != 0) {
    double u;
    if (hx < 0x43400000) {
      u = UBLR_ADD(1.0, x);
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = k > 0 ? UBLR_SUB(1.0, UBLR_SUB(u, x)) : UBLR_SUB(x, UBLR_SUB(u, 1.0));
      c = UBLR_DIV(c, u);
    } else {
      u = x;
      hu = hi_word(u);
      k = (hu >> 20) - 1023;
      c = 0.0;
    }
    hu &= 0x000fffff;
    if (hu < 0x6a09e) {                           // 1 + f in [1, sqrt 2)
      u = with_hi_word(u, hu | 0x3ff00000);
    } else {                                      // halve: 1 + f in [sqrt 2 / 2, 1)
      k += 1;
      u = with_hi_word(u, hu | 0x3fe00000);
      hu = (0x00100000 - hu) >> 2;
    }
    f = UBLR_SUB(u, 1.0);
  }
  const double hfsq = UBLR_MUL(UBLR_MUL(f, 0.5), f);
  const double kd = (double)k;
  if (hu == 0) {                                  // |f| < 2^-20
    if (f == 0.0) {
      if (k == 0) return 0.0;
      c = fma(kd, LN2_LO, c);
      return fma(kd, LN2_HI, c);
    }
    const double R = UBLR_MUL(fma(-f, 0.66666666666666666, 1.0), hfsq);
    if (k == 0) return UBLR_SUB(f, R);
    return fma(kd, LN2_HI, -UBLR_SUB(UBLR_SUB(R, fma(kd, LN2_LO, c)), f));
  }
  const double s = UBLR_DIV(f, UBLR_ADD(f, 2.0));
  const double z = UBLR_MUL(s, s), z2 = UBLR_MUL(z, z), z4 = UBLR_MUL(z2, z2), z6 = UBLR_MUL(z2, z4);
  const double R2 = fma(z, P3, P2), R3 = fma(z, P5, P4), R4 = fma(z, P7, P6);
  const double R = fma(z6, R4, fma(z4, R3, fma(z, P1, UBLR_MUL(z2, R2))));
  const double t = UBLR_MUL(s, UBLR_ADD(hfsq, R));
  if (k == 0) return UBLR_SUB(f, UBLR_SUB(hfsq, t));
  return fma(kd, LN2_HI, -UBLR_SUB(UBLR_SUB(hfsq, UBLR_ADD(fma(kd, LN2_LO, c), t)), f));
}

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
      double xx = UBLR_MUL(-ZIG_INV_R, log1p_host_exact(-u1));
      double yy = -log1p_host_exact(-u2);
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
