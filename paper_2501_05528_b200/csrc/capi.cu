// C-ABI plumbing: error text, version, device check.
#include "common.cuh"
#include "nullvec.cuh"
#include <cmath>
#include <vector>

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

// numpy SeedSequence(seed, spawn_key = prefix + suffix_s).generate_state(2,
// uint64) for n spawn keys at once (host code; numpy's published algorithm:
// O'Neill's seed_seq hash mixing over a 4-word uint32 pool,
// numpy/random/bit_generator.pyx). Restated from paper_2501_05528_b200/seedseq.py
// (checked bit-for-bit against numpy in tests/test_host.py).
namespace {
constexpr uint32_t SS_INIT_A = 0x43b0d7e5u, SS_MULT_A = 0x931e8875u, SS_INIT_B = 0x8b51f9ddu,
                   SS_MULT_B = 0x58f38dedu, SS_MIX_L = 0xca01f9ddu, SS_MIX_R = 0x4973f715u;
}  // namespace

extern "C" int ublr_seedseq_keys(const uint32_t* run, int nrun, const uint32_t* prefix, int nprefix,
                                 const uint32_t* suffix, int nsuffix, int64_t n, uint64_t* keys_out) {
  UBLR_REQUIRE(run && nrun >= 1 && nprefix >= 0 && nsuffix >= 0 && n >= 0 && keys_out &&
                   (nprefix == 0 || prefix) && (nsuffix == 0 || suffix),
               UBLR_ERR_VALUE, "ublr_seedseq_keys: bad arguments");
  const int nspawn = nprefix + nsuffix;
  const int nr = (nspawn > 0 && nrun < 4) ? 4 : nrun;  // run entropy padded to the pool size
  const int L = nr + nspawn;
  std::vector<uint32_t> ent((size_t)L);
  for (int64_t s = 0; s < n; ++s) {
    for (int i = 0; i < nr; ++i) ent[i] = i < nrun ? run[i] : 0u;
    for (int i = 0; i < nprefix; ++i) ent[nr + i] = prefix[i];
    for (int i = 0; i < nsuffix; ++i) ent[nr + nprefix + i] = suffix[s * nsuffix + i];
    uint32_t hc = SS_INIT_A;
    auto hashmix = [&hc](uint32_t v) {
      v ^= hc;
      hc *= SS_MULT_A;
      v *= hc;
      return v ^ (v >> 16);
    };
    auto mix = [](uint32_t x, uint32_t y) {
      uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
      return r ^ (r >> 16);
    };
    uint32_t pool[4];
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < L ? ent[i] : 0u);
    for (int a = 0; a < 4; ++a)
      for (int d = 0; d < 4; ++d)
        if (a != d) pool[d] = mix(pool[d], hashmix(pool[a]));
    for (int a = 4; a < L; ++a)
      for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[a]));
    uint32_t hb = SS_INIT_B, st[4];
    for (int i = 0; i < 4; ++i) {
      uint32_t v = pool[i] ^ hb;
      hb *= SS_MULT_B;
      v *= hb;
      st[i] = v ^ (v >> 16);
    }
    keys_out[2 * s] = (uint64_t)st[0] | ((uint64_t)st[1] << 32);
    keys_out[2 * s + 1] = (uint64_t)st[2] | ((uint64_t)st[3] << 32);
  }
  return UBLR_OK;
}

// Null vectors of tagging-row subsets (host code; ref/tagging.py:126-139 via
// ref/linalg.py:72-94: the last column of the complete Householder Q of
// T[rows]^T). Per set: Householder QR of the ell x sz matrix A = T[rows]^T in
// LAPACK's dgeqr2 convention (v_0 = 1, beta = -sign(alpha) ||x||,
// tau = (beta - alpha) / beta), then q = H_0 H_1 ... H_{k-1} e_{ell-1}.
// Equal to numpy's qr(mode="complete")[0][:, -1] up to rounding.
extern "C" int ublr_null_vectors(const double* T, int ell, const int32_t* ptr, const int32_t* idx, int nsets,
                                 double* Z, double* res) {
  UBLR_REQUIRE(T && ell >= 1 && ptr && idx && nsets >= 0 && Z && res, UBLR_ERR_VALUE,
               "ublr_null_vectors: bad arguments");
  double Afix[ublr::nullvec::MAX_ELL * ublr::nullvec::MAX_ELL], taufix[ublr::nullvec::MAX_ELL];
  std::vector<double> Aheap, tauheap;   // ell > 32 (extra tagging columns in 3-D)
  if (ell > ublr::nullvec::MAX_ELL) {
    Aheap.resize((size_t)ell * ell);
    tauheap.resize(ell);
  }
  double* A = ell > ublr::nullvec::MAX_ELL ? Aheap.data() : Afix;
  double* tau = ell > ublr::nullvec::MAX_ELL ? tauheap.data() : taufix;
  for (int s = 0; s < nsets; ++s) {
    const int r0 = ptr[s], sz = ptr[s + 1] - ptr[s];
    UBLR_REQUIRE(sz >= 0 && sz < ell, UBLR_ERR_VALUE, "ublr_null_vectors: a set has >= ell rows (no null vector)");
    res[s] = ublr::nullvec::null_vector(T, ell, idx + r0, sz, A, tau, Z + (size_t)s * ell);
  }
  return UBLR_OK;
}

// One redraw-policy evaluation on the host (ref/tagging.py:355-379 with
// :110-139): null vectors and residuals (ublr_null_vectors), the residual
// scale max(1, ||T[rows]||_F) per set, and the aspect ratios rho_i over the
// far field of block i (1 if the max is 0, inf if the min is 0, NaN for an
// empty far field). The Python planner is a thin wrapper around it; for
// b >= 1024 the aspect ratios run on the GPU (ublr_tag_aspect) instead.
extern "C" int ublr_tag_plan_host(const double* T, int ell, const int32_t* ptr, const int32_t* idx, int b,
                                  double* Z, double* res, double* scale, double* rho) {
  int rc = ublr_null_vectors(T, ell, ptr, idx, b, Z, res);
  if (rc) return rc;
  std::vector<double> rn2(b);
  for (int j = 0; j < b; ++j) {
    double s2 = 0.0;
    for (int c = 0; c < ell; ++c) s2 += T[(size_t)j * ell + c] * T[(size_t)j * ell + c];
    rn2[j] = s2;
  }
  std::vector<char> nearm(b, 0);
  for (int i = 0; i < b; ++i) {
    double seg = 0.0;
    for (int p = ptr[i]; p < ptr[i + 1]; ++p) seg += rn2[idx[p]];
    scale[i] = fmax(1.0, sqrt(seg));
    if (!rho) continue;
    for (int p = ptr[i]; p < ptr[i + 1]; ++p) nearm[idx[p]] = 1;
    const double* z = Z + (size_t)i * ell;
    double lo = INFINITY, hi = -INFINITY;
    int j = 0;
    for (; j + 4 <= b; j += 4) {   // four independent dot products (ILP; same per-dot order)
      const double* t0 = T + (size_t)j * ell;
      double d0 = 0.0, d1 = 0.0, d2 = 0.0, d3 = 0.0;
      for (int c = 0; c < ell; ++c) {   // host: no libm fma call
        const double zc = z[c];
        d0 += t0[c] * zc;
        d1 += t0[ell + c] * zc;
        d2 += t0[2 * ell + c] * zc;
        d3 += t0[3 * ell + c] * zc;
      }
      const double dv[4] = {fabs(d0), fabs(d1), fabs(d2), fabs(d3)};
      for (int u = 0; u < 4; ++u) {
        if (nearm[j + u]) continue;
        lo = fmin(lo, dv[u]);
        hi = fmax(hi, dv[u]);
      }
    }
    for (; j < b; ++j) {
      if (nearm[j]) continue;
      double d = 0.0;
      for (int c = 0; c < ell; ++c) d += T[(size_t)j * ell + c] * z[c];
      d = fabs(d);
      lo = fmin(lo, d);
      hi = fmax(hi, d);
    }
    for (int p = ptr[i]; p < ptr[i + 1]; ++p) nearm[idx[p]] = 0;
    if (ptr[i + 1] - ptr[i] >= b) rho[i] = NAN;
    else if (hi == 0.0) rho[i] = 1.0;
    else if (lo == 0.0) rho[i] = INFINITY;
    else rho[i] = hi / lo;
  }
  return UBLR_OK;
}
