// K1 — numpy-bit-compatible Gaussian streams on the GPU.
//
// Replaces RandomStream.normal / gaussian (ref/linalg.py:38-52) for every
// test matrix of the pipeline (ref/bases.py:97-98, :163-168, :229-230;
// ref/reconstruction.py:405). Each stream is numpy's Philox4x64-10 under a
// host-derived SeedSequence key; normals come from numpy's ziggurat.
//
// The ziggurat consumes a data-dependent number of words per normal (1 on
// ~99% of attempts), so a stream is decoded in parallel:
//   A. every chunk of C words is parsed from each possible entry offset
//      e < D; parses from different entries merge after a few tokens, so a
//      chunk is summarised by (exit offset, count[e]);
//   B. chunk entries are resolved from the previous chunk's exit, giving a
//      per-chunk normal count (entries >= D are re-parsed exactly);
//   C. an exclusive scan of counts gives each chunk's first normal index;
//   D. every chunk re-parses from its entry and writes its normals.
// Any inconsistency (no merge, too few words) sets a device flag, and a
// serial fallback kernel re-decodes the affected launch exactly — there is
// no host round trip.
#include "common.cuh"
#include "philox_zig.cuh"
#include "ziggurat_tables.h"

namespace ublr {
namespace {

constexpr int C = 32;         // words per chunk
constexpr int D = 6;          // entry offsets summarised per chunk
constexpr int WIN = C + 16;   // words cached per thread
constexpr int RNG_THREADS = 128;

struct Tables {
  uint64_t ki[256];
  double wi[256];
  double fi[256];
};

__device__ __forceinline__ void load_tables(Tables* t) {
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    t->ki[i] = zig::KI[i];
    t->wi[i] = __longlong_as_double((long long)zig::WI_BITS[i]);
    t->fi[i] = __longlong_as_double((long long)zig::FI_BITS[i]);
  }
}

// Out-of-line Philox word for the rare reads past a window and the serial
// fallback: inlined, every ziggurat token site carried its own copy of the
// ten unrolled rounds and the per-CTA decode kernel outgrew the instruction
// cache (ncu: "no instructions" was the top stall of k_rng_cta).
__device__ __noinline__ uint64_t philox_word_ool(uint64_t k0, uint64_t k1, uint64_t w) {
  return rng::philox_word(k0, k1, w);
}

template <int CC>
struct WindowWords {
  static constexpr int WIN = CC + 16;
  uint64_t k0, k1;
  int64_t base;  // absolute word index of rel 0
  uint64_t buf[WIN];
  __device__ void fill() {
#pragma unroll 1
    for (int q = 0; q < WIN / 4; ++q) {
      uint64_t o[4];
      rng::philox4x64_10(((uint64_t)base >> 2) + q + 1, k0, k1, o);
      buf[4 * q + 0] = o[0];
      buf[4 * q + 1] = o[1];
      buf[4 * q + 2] = o[2];
      buf[4 * q + 3] = o[3];
    }
  }
  __device__ uint64_t operator()(int64_t rel) {
    if (rel < WIN) return buf[rel];
    return philox_word_ool(k0, k1, (uint64_t)(base + rel));
  }
};

struct DirectWords {
  uint64_t k0, k1;
  int64_t base;
  __device__ uint64_t operator()(int64_t rel) { return philox_word_ool(k0, k1, (uint64_t)(base + rel)); }
};

// Per-launch descriptor arrays live in the workspace.
struct RngPlan {
  const ublr_rng_stream_t* streams;
  const int64_t* chunk_start;  // [n_streams + 1] global chunk index of each stream's chunk 0
  int n_streams;
  int64_t n_chunks;
  uint64_t* summary;           // [n_chunks]: exit (16b) | cnt[e] (8b each, 0xff = unknown)
  int32_t* counts;             // [n_chunks]
  int64_t* prefix;             // [n_chunks + 1]
  int* flag;                   // [1]
};

__device__ __forceinline__ int find_stream(const int64_t* chunk_start, int n, int64_t g) {
  int lo = 0, hi = n;  // chunk_start[lo] <= g < chunk_start[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (chunk_start[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}

// A. chunk summaries: chunk `local` of stream st parsed from entries 0..D-1
template <int CC>
__device__ uint64_t chunk_summary(const Tables& tb, const ublr_rng_stream_t& st, int64_t local) {
  WindowWords<CC> ws;
  ws.k0 = st.key0; ws.k1 = st.key1; ws.base = local * CC;
  ws.fill();
  // parse from entry 0: token starts and accepted-suffix counts
  uint32_t starts = 0;        // bit p set if parse-0 token starts at rel p < CC
  uint8_t acc_at[CC];          // accepted flag of the token starting at p
  int64_t p = 0;
  double v; bool ok;
  while (p < CC) {
    int len = rng::zig_token(ws, p, tb.ki, tb.wi, tb.fi, v, ok);
    starts |= 1u << p;
    acc_at[p] = ok ? 1 : 0;
    p += len;
  }
  int exit0 = (int)(p - CC);
  uint8_t suffix[CC + 1];      // accepted parse-0 tokens starting at >= q (q a start)
  suffix[CC] = 0;
  int run = 0;
  for (int q = CC - 1; q >= 0; --q) {
    if (starts & (1u << q)) run += acc_at[q];
    suffix[q] = (uint8_t)run;
  }
  uint64_t rec = (uint64_t)(exit0 > 0xffff ? 0xffff : exit0);
  for (int e = 0; e < D; ++e) {
    int cnt = 0xff;
    if (e == 0) {
      cnt = suffix[0];
    } else {
      int64_t q = e;
      int before = 0;
      while (q < CC && !(starts & (1u << q))) {
        int len = rng::zig_token(ws, q, tb.ki, tb.wi, tb.fi, v, ok);
        before += ok ? 1 : 0;
        q += len;
      }
      if (q < CC) cnt = before + suffix[q];          // merged with parse 0
      else if (q - CC == exit0) cnt = before;         // same exit, no merge inside
      else cnt = 0xff;                               // diverged
    }
    rec |= (uint64_t)(cnt & 0xff) << (16 + 8 * e);
  }
  return rec;
}

__global__ void __launch_bounds__(RNG_THREADS) k_rng_summary(RngPlan P) {
  __shared__ Tables tb;
  load_tables(&tb);
  __syncthreads();
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P.n_chunks) return;
  int s = find_stream(P.chunk_start, P.n_streams, g);
  P.summary[g] = chunk_summary<C>(tb, P.streams[s], g - P.chunk_start[s]);
}

// Exact parse of chunk g from entry `entry` (slow path).
template <int CC>
__device__ int parse_count(const Tables& tb, const ublr_rng_stream_t& st, int64_t local, int64_t entry,
                           int64_t* exit_rel) {
  DirectWords ws{st.key0, st.key1, local * CC};
  int64_t p = entry;
  int cnt = 0;
  double v; bool ok;
  while (p < CC) {
    p += rng::zig_token(ws, p, tb.ki, tb.wi, tb.fi, v, ok);
    cnt += ok ? 1 : 0;
  }
  *exit_rel = p - CC;
  return cnt;
}

__device__ __forceinline__ int64_t chunk_entry(const RngPlan& P, int64_t g, int s) {
  if (g == P.chunk_start[s]) return 0;
  return (int64_t)(P.summary[g - 1] & 0xffff);
}

// B. resolve: normals produced by chunk `local` entered at `entry` (rec =
// its summary); sets *bad when the summaries are inconsistent (serial fallback)
template <int CC>
__device__ int chunk_count(const Tables& tb, const ublr_rng_stream_t& st, int64_t local, int64_t entry,
                           uint64_t rec, bool* bad) {
  int cnt = 0xff;
  if (entry == 0xffff) {
    *bad = true;
    return 0;
  }
  if (entry < D) cnt = (int)((rec >> (16 + 8 * entry)) & 0xff);
  if (cnt == 0xff) {
    if (entry >= CC) {
      *bad = true;  // a token spanning a whole chunk: serial fallback
      return 0;
    }
    int64_t ex;
    cnt = parse_count<CC>(tb, st, local, entry, &ex);
    if (ex != (int64_t)(rec & 0xffff)) *bad = true;
  }
  return cnt;
}

__global__ void __launch_bounds__(RNG_THREADS) k_rng_resolve(RngPlan P) {
  __shared__ Tables tb;
  load_tables(&tb);
  __syncthreads();
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P.n_chunks) return;
  int s = find_stream(P.chunk_start, P.n_streams, g);
  bool bad = false;
  P.counts[g] = chunk_count<C>(tb, P.streams[s], g - P.chunk_start[s], chunk_entry(P, g, s), P.summary[g], &bad);
  if (bad) atomicExch(P.flag, 1);
}

// C. scan (exclusive, int32 -> int64), two levels.
constexpr int SCAN_T = 512;
constexpr int SCAN_PER = 4;
__global__ void __launch_bounds__(SCAN_T) k_scan_blocks(const int32_t* in, int64_t n, int64_t* out,
                                                        int64_t* block_sums) {
  __shared__ int64_t sh[SCAN_T];
  int64_t base = (int64_t)blockIdx.x * SCAN_T * SCAN_PER + threadIdx.x * SCAN_PER;
  int64_t v[SCAN_PER];
  int64_t tot = 0;
  for (int q = 0; q < SCAN_PER; ++q) {
    v[q] = (base + q < n) ? in[base + q] : 0;
    tot += v[q];
  }
  sh[threadIdx.x] = tot;
  __syncthreads();
  for (int off = 1; off < SCAN_T; off <<= 1) {
    int64_t t = threadIdx.x >= off ? sh[threadIdx.x - off] : 0;
    __syncthreads();
    sh[threadIdx.x] += t;
    __syncthreads();
  }
  int64_t run = sh[threadIdx.x] - tot;
  for (int q = 0; q < SCAN_PER; ++q) {
    if (base + q < n) out[base + q] = run;
    run += v[q];
  }
  if (threadIdx.x == SCAN_T - 1) block_sums[blockIdx.x] = sh[SCAN_T - 1];
}

__global__ void __launch_bounds__(1024) k_scan_sums(int64_t* sums, int64_t nb, int64_t* total) {
  __shared__ int64_t sh[1024];
  int64_t carry = 0;
  for (int64_t base = 0; base < nb; base += 1024) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < nb ? sums[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      int64_t t = threadIdx.x >= off ? sh[threadIdx.x - off] : 0;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    if (i < nb) sums[i] = carry + sh[threadIdx.x] - v;
    int64_t blk = sh[1023];
    __syncthreads();
    carry += blk;
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void k_scan_add(int64_t* out, int64_t n, const int64_t* block_sums) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] += block_sums[i / (SCAN_T * SCAN_PER)];
}

__device__ __forceinline__ void store_normal(const ublr_rng_stream_t& st, int64_t n, double v, double* out) {
  int64_t r = n / st.cols, c = n - r * st.cols;
  int64_t row = st.rowmap ? (int64_t)st.rowmap[r] : r;
  out[st.out_offset + row * st.ld + c] = v;
}

// D. emit: chunk `local` entered at `entry` writes its normals from index n;
// returns the index after its last normal
template <int CC>
__device__ int64_t chunk_emit(const Tables& tb, const ublr_rng_stream_t& st, int64_t local, int64_t entry, int64_t n,
                              double* out) {
  WindowWords<CC> ws;
  ws.k0 = st.key0; ws.k1 = st.key1; ws.base = local * CC;
  ws.fill();
  int64_t p = entry;
  double v; bool ok;
  while (p < CC) {
    p += rng::zig_token(ws, p, tb.ki, tb.wi, tb.fi, v, ok);
    if (ok) {
      if (n < st.count) store_normal(st, n, v, out);
      ++n;
    }
  }
  return n;
}

__global__ void __launch_bounds__(RNG_THREADS) k_rng_emit(RngPlan P, double* out) {
  __shared__ Tables tb;
  load_tables(&tb);
  __syncthreads();
  int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P.n_chunks) return;
  if (*P.flag) return;
  int s = find_stream(P.chunk_start, P.n_streams, g);
  const ublr_rng_stream_t st = P.streams[s];
  int64_t first = P.chunk_start[s];
  int64_t entry = chunk_entry(P, g, s);
  if (entry >= C) return;
  int64_t n = chunk_emit<C>(tb, st, g - first, entry, P.prefix[g] - P.prefix[first], out);
  if (g + 1 == P.chunk_start[s + 1] && n < st.count) atomicExch(P.flag, 1);  // ran out of words
}

// Serial fallback: one thread per stream decodes the whole stream exactly.
__global__ void k_rng_serial(RngPlan P, double* out) {
  __shared__ Tables tb;
  load_tables(&tb);
  __syncthreads();
  if (*P.flag == 0) return;
  for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < P.n_streams; s += gridDim.x * blockDim.x) {
    const ublr_rng_stream_t st = P.streams[s];
    DirectWords ws{st.key0, st.key1, 0};
    int64_t p = 0;
    double v; bool ok;
    for (int64_t n = 0; n < st.count;) {
      p += rng::zig_token(ws, p, tb.ki, tb.wi, tb.fi, v, ok);
      if (ok) store_normal(st, n++, v, out);
    }
  }
}


// One CTA per stream for many short streams (the test blocks G_i, H_i: one
// stream per block of m_i x gc normals): the four phases above run inside
// the CTA on its stream's chunks (summaries and counts in shared memory, a
// block scan), so a whole launch set is one kernel. A chunk's entry is the
// previous chunk's parse-0 exit, so every phase is chunk-parallel; an
// inconsistency makes thread 0 re-decode the stream serially.
constexpr int CTA_MAX_CHUNKS = 4096;   // longest stream decoded by one CTA (~125k normals)
constexpr int CTA_THREADS = 256;

__host__ __device__ inline int64_t chunks_for(int64_t count, int cc) { return (count + count / 24 + 256 + cc - 1) / cc; }

template <int CC>
__global__ void __launch_bounds__(CTA_THREADS) k_rng_cta(const ublr_rng_stream_t* __restrict__ streams,
                                                         int n_streams, double* __restrict__ out) {
  __shared__ Tables tb;
  __shared__ uint64_t rec[CTA_MAX_CHUNKS];
  __shared__ int32_t part[CTA_THREADS];
  __shared__ int bad_any;
  load_tables(&tb);
  const int T = blockDim.x, tid = threadIdx.x;
  for (int s = blockIdx.x; s < n_streams; s += gridDim.x) {
    const ublr_rng_stream_t st = streams[s];
    const int nch = (int)chunks_for(st.count, CC);
    if (tid == 0) bad_any = 0;
    __syncthreads();
    for (int g = tid; g < nch; g += T) rec[g] = chunk_summary<CC>(tb, st, g);
    __syncthreads();
    bool bad = false;
    // counts, then a block scan over contiguous per-thread runs of chunks
    const int per = (nch + T - 1) / T, g0 = tid * per, g1 = min(nch, g0 + per);
    int run = 0;
    for (int g = g0; g < g1; ++g) {
      const int64_t entry = g == 0 ? 0 : (int64_t)(rec[g - 1] & 0xffff);
      run += chunk_count<CC>(tb, st, g, entry, rec[g], &bad);
    }
    part[tid] = run;
    __syncthreads();
    for (int o = 1; o < T; o <<= 1) {
      const int v = tid >= o ? part[tid - o] : 0;
      __syncthreads();
      part[tid] += v;
      __syncthreads();
    }
    int64_t n = part[tid] - run;
    for (int g = g0; g < g1 && !bad; ++g) {
      const int64_t entry = g == 0 ? 0 : (int64_t)(rec[g - 1] & 0xffff);
      if (entry >= CC) { bad = true; break; }
      n = chunk_emit<CC>(tb, st, g, entry, n, out);
    }
    if (tid == T - 1 && part[T - 1] < st.count) bad = true;   // ran out of words
    if (bad) atomicExch(&bad_any, 1);
    __syncthreads();
    if (bad_any && tid == 0) {
      DirectWords ws{st.key0, st.key1, 0};
      int64_t p = 0;
      double v; bool ok;
      for (int64_t q = 0; q < st.count;) {
        p += rng::zig_token(ws, p, tb.ki, tb.wi, tb.fi, v, ok);
        if (ok) store_normal(st, q++, v, out);
      }
    }
    __syncthreads();
  }
}

inline int64_t words_for(int64_t count) { return count + count / 24 + 256; }
inline int64_t align_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// chunk_start[s] = sum_{t < s} ceil(words(count_t) / C), from the device
// stream records (one block; replaces a pageable host->device copy, which
// would block the host behind queued work)
__global__ void k_chunk_starts(const ublr_rng_stream_t* __restrict__ streams, int n, int64_t* __restrict__ out,
                               int* __restrict__ flag) {
  __shared__ int64_t part[1024];
  const int T = blockDim.x;
  const int per = (n + T - 1) / T;
  const int s0 = threadIdx.x * per, s1 = min(n, s0 + per);
  int64_t sum = 0;
  for (int s = s0; s < s1; ++s) sum += (streams[s].count + streams[s].count / 24 + 256 + C - 1) / C;
  part[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int t = 0; t < T; ++t) {
      const int64_t v = part[t];
      part[t] = run;
      run += v;
    }
    out[n] = run;
    *flag = 0;
  }
  __syncthreads();
  int64_t run = part[threadIdx.x];
  for (int s = s0; s < s1; ++s) {
    out[s] = run;
    run += (streams[s].count + streams[s].count / 24 + 256 + C - 1) / C;
  }
}

struct Layout {
  int64_t n_chunks, chunk_start_off, summary_off, counts_off, prefix_off, bsum_off, total_off, flag_off, bytes;
};

Layout layout(const int64_t* counts, int n_streams) {
  Layout L{};
  int64_t nc = 0;
  for (int s = 0; s < n_streams; ++s) nc += (words_for(counts[s]) + C - 1) / C;
  L.n_chunks = nc;
  int64_t o = 0;
  L.chunk_start_off = o; o = align_up(o + 8 * (n_streams + 1), 256);
  L.summary_off = o; o = align_up(o + 8 * nc, 256);
  L.counts_off = o; o = align_up(o + 4 * nc, 256);
  L.prefix_off = o; o = align_up(o + 8 * (nc + 1), 256);
  int64_t nb = (nc + SCAN_T * SCAN_PER - 1) / (SCAN_T * SCAN_PER);
  L.bsum_off = o; o = align_up(o + 8 * (nb + 1), 256);
  L.total_off = o; o = align_up(o + 8, 256);
  L.flag_off = o; o = align_up(o + 8, 256);
  L.bytes = o;
  return L;
}

}  // namespace
}  // namespace ublr

using namespace ublr;

extern "C" int64_t ublr_rng_workspace_bytes(const int64_t* counts, int n_streams) {
  if (n_streams <= 0 || !counts) return 0;
  return layout(counts, n_streams).bytes;
}

extern "C" int ublr_rng_normals(const ublr_rng_stream_t* streams_dev, const int64_t* counts_host, int n_streams,
                                double* out, void* workspace, int64_t workspace_bytes, void* stream) {
  UBLR_REQUIRE(n_streams >= 0, UBLR_ERR_VALUE, "n_streams must be >= 0");
  if (n_streams == 0) return UBLR_OK;
  UBLR_REQUIRE(streams_dev && counts_host && out && workspace, UBLR_ERR_VALUE, "null pointer argument");
  for (int s = 0; s < n_streams; ++s) UBLR_REQUIRE(counts_host[s] >= 0, UBLR_ERR_VALUE, "negative stream count");
  cudaStream_t st = (cudaStream_t)stream;
  int64_t max_count = 0;
  for (int s = 0; s < n_streams; ++s) max_count = counts_host[s] > max_count ? counts_host[s] : max_count;
  static const int path = [] {
    const char* e = getenv("UBLR_RNG_PATH");  // 0 auto, 1 chunked multi-kernel, 2 one CTA per stream
    return e ? atoi(e) : 0;
  }();
  // chunk size: enough chunks per stream to give every stream a CTA of threads
  const int cc = chunks_for(max_count, 8) <= CTA_THREADS ? 8 : chunks_for(max_count, 16) <= 2 * CTA_THREADS ? 16 : C;
  const int64_t max_chunks = chunks_for(max_count, cc);
  // the per-CTA decode wins for short streams (c2: 0.081 -> 0.033 ms); for
  // long ones (c5: 8192 streams of 16k normals) the chunk-parallel kernels do
  // (2.8 vs 3.8 ms)
  if (path == 2 || (path == 0 && cc < C)) {
    UBLR_REQUIRE(max_chunks <= CTA_MAX_CHUNKS, UBLR_ERR_VALUE, "rng: stream too long for the per-CTA decode");
    int threads = (int)((max_chunks + 31) / 32 * 32);
    threads = threads > CTA_THREADS ? CTA_THREADS : threads;
    if (cc == 8) k_rng_cta<8><<<n_streams, threads, 0, st>>>(streams_dev, n_streams, out);
    else if (cc == 16) k_rng_cta<16><<<n_streams, threads, 0, st>>>(streams_dev, n_streams, out);
    else k_rng_cta<C><<<n_streams, threads, 0, st>>>(streams_dev, n_streams, out);
    UBLR_LAUNCH_CHECK();
    return UBLR_OK;
  }
  Layout L = layout(counts_host, n_streams);
  UBLR_REQUIRE(workspace_bytes >= L.bytes, UBLR_ERR_VALUE, "rng workspace too small");
  char* ws = (char*)workspace;
  // chunk starts and the fallback flag, computed on the device
  k_chunk_starts<<<1, 1024, 0, st>>>(streams_dev, n_streams, (int64_t*)(ws + L.chunk_start_off), (int*)(ws + L.flag_off));
  UBLR_LAUNCH_CHECK();
  RngPlan P;
  P.streams = streams_dev;
  P.chunk_start = (const int64_t*)(ws + L.chunk_start_off);
  P.n_streams = n_streams;
  P.n_chunks = L.n_chunks;
  P.summary = (uint64_t*)(ws + L.summary_off);
  P.counts = (int32_t*)(ws + L.counts_off);
  P.prefix = (int64_t*)(ws + L.prefix_off);
  P.flag = (int*)(ws + L.flag_off);
  int64_t grid = (L.n_chunks + RNG_THREADS - 1) / RNG_THREADS;
  k_rng_summary<<<(unsigned)grid, RNG_THREADS, 0, st>>>(P);
  UBLR_LAUNCH_CHECK();
  k_rng_resolve<<<(unsigned)grid, RNG_THREADS, 0, st>>>(P);
  UBLR_LAUNCH_CHECK();
  int64_t nb = (L.n_chunks + SCAN_T * SCAN_PER - 1) / (SCAN_T * SCAN_PER);
  int64_t* bsum = (int64_t*)(ws + L.bsum_off);
  k_scan_blocks<<<(unsigned)nb, SCAN_T, 0, st>>>(P.counts, L.n_chunks, P.prefix, bsum);
  UBLR_LAUNCH_CHECK();
  k_scan_sums<<<1, 1024, 0, st>>>(bsum, nb, P.prefix + L.n_chunks);
  UBLR_LAUNCH_CHECK();
  k_scan_add<<<(unsigned)((L.n_chunks + 255) / 256), 256, 0, st>>>(P.prefix, L.n_chunks, bsum);
  UBLR_LAUNCH_CHECK();
  k_rng_emit<<<(unsigned)grid, RNG_THREADS, 0, st>>>(P, out);
  UBLR_LAUNCH_CHECK();
  k_rng_serial<<<(unsigned)((n_streams + 63) / 64), 64, 0, st>>>(P, out);
  UBLR_LAUNCH_CHECK();
  return UBLR_OK;
}
