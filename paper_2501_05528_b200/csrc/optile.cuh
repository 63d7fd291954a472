// On-the-fly operator tiles: entries A(p, q) in permuted (block-contiguous)
// indices for the operator kinds of ublr_op_t.
//
// The reference treats A as a black box (ref/operators.py:24-35); the
// BASELINE configs use a dense synthetic matrix (config 1) or kernel
// matrices evaluated on the fly inside the sketch GEMM (configs 2-5), so
// tiles are generated in registers and written to shared memory — A is
// never materialised in HBM.
#pragma once
#include "common.cuh"

namespace ublr {

// Per-thread cached data for one fixed row p of the tile.
struct RowPoint {
  int p;
  int orig;          // perm[p] (dense / diagonal test)
  double x0, x1, x2;
};

__device__ __forceinline__ RowPoint load_row_point(const ublr_op_t& op, int p, bool valid) {
  RowPoint r;
  r.p = valid ? p : -1;
  r.orig = 0;
  r.x0 = r.x1 = r.x2 = 0.0;
  if (!valid) return r;
  if (op.kind == UBLR_OP_DENSE) {
    r.orig = op.perm ? op.perm[p] : p;
  } else {
    r.x0 = op.coords[p];
    if (op.dim > 1) r.x1 = op.coords[op.n + p];
    if (op.dim > 2) r.x2 = op.coords[2 * op.n + p];
  }
  return r;
}

// Entry A(row.p, q); q must be a valid permuted index (0 <= q < n).
template <int KIND>
__device__ __forceinline__ double op_entry(const ublr_op_t& op, const RowPoint& row, int q, const LogTables* lt) {
  if (KIND == UBLR_OP_DENSE) {
    int oq = op.perm ? op.perm[q] : q;
    return op.transpose ? op.A[(int64_t)oq * op.lda + row.orig] : op.A[(int64_t)row.orig * op.lda + oq];
  } else {
    if (q == row.p) return op.diag;
    double d = row.x0 - op.coords[q];
    double r2 = d * d;
    if (op.dim > 1) {
      d = row.x1 - op.coords[op.n + q];
      r2 = fma(d, d, r2);
    }
    if (op.dim > 2) {
      d = row.x2 - op.coords[2 * op.n + q];
      r2 = fma(d, d, r2);
    }
    if (KIND == UBLR_OP_LOG) return -0.5 * fast_log(r2, lt);
    return rsqrt(r2);
  }
}

// Entry from explicit column coordinates (kernel operators): the column
// point's coordinates come from a shared-memory ring filled ahead of time
// (ColRing), so tile generation does not wait on global loads.
template <int KIND>
__device__ __forceinline__ double kernel_entry(const ublr_op_t& op, const RowPoint& row, int q, double c0, double c1,
                                               double c2, const LogTables* lt) {
  if (q == row.p) return op.diag;
  double d = row.x0 - c0;
  double r2 = d * d;
  if (op.dim > 1) {
    d = row.x1 - c1;
    r2 = fma(d, d, r2);
  }
  if (op.dim > 2) {
    d = row.x2 - c2;
    r2 = fma(d, d, r2);
  }
  if (KIND == UBLR_OP_LOG) return -0.5 * fast_log(r2, lt);
  return rsqrt(r2);
}

// Branch-free form for a compile-time dimension: out-of-range rows/columns
// are left to the caller (their X rows are zero / their outputs are not
// stored), the diagonal is a select. Same operation order as kernel_entry,
// so the two give identical bits.
template <int KIND, int DIM>
__device__ __forceinline__ double kernel_entry_dim(const RowPoint& row, int q, double c0, double c1, double c2,
                                                   double diag, const LogTables* lt) {
  double d = row.x0 - c0;
  double r2 = d * d;
  if (DIM > 1) {
    d = row.x1 - c1;
    r2 = fma(d, d, r2);
  }
  if (DIM > 2) {
    d = row.x2 - c2;
    r2 = fma(d, d, r2);
  }
  const double v = (KIND == UBLR_OP_LOG) ? -0.5 * fast_log(r2, lt) : rsqrt(r2);
  return q == row.p ? diag : v;
}

// Three-slot shared-memory ring of column coordinates (3 dims x BK per slot)
// for the k-steps of an operator-tile producer; slot = stage % 3.
template <int BK>
struct ColRing {
  double* buf;  // 9 * BK doubles
  __device__ __forceinline__ void prefetch(const ublr_op_t& op, int stage, int q0, int qend, int nthreads) {
    const int slot = stage % 3;
    for (int e = threadIdx.x; e < op.dim * BK; e += nthreads) {
      int a = e / BK, kk = e - a * BK;
      int q = q0 + kk;
      bool ok = q < qend;
      cp_async8(&buf[(slot * 3 + a) * BK + kk], ok ? (const void*)(op.coords + (int64_t)a * op.n + q) : (const void*)op.coords,
                ok);
    }
  }
  __device__ __forceinline__ double at(int stage, int a, int kk) const { return buf[((stage % 3) * 3 + a) * BK + kk]; }
};

// Runtime -> compile-time dispatch on the operator kind.
#define UBLR_DISPATCH_KIND(kind, KIND_NAME, ...)                       \
  switch (kind) {                                                      \
    case UBLR_OP_DENSE: { constexpr int KIND_NAME = UBLR_OP_DENSE; __VA_ARGS__; } break; \
    case UBLR_OP_LOG:   { constexpr int KIND_NAME = UBLR_OP_LOG;   __VA_ARGS__; } break; \
    case UBLR_OP_INV:   { constexpr int KIND_NAME = UBLR_OP_INV;   __VA_ARGS__; } break; \
    default: ::ublr::set_error("unknown operator kind"); return UBLR_ERR_VALUE;          \
  }

inline int check_op(const ublr_op_t* op) {
  if (!op) { set_error("null operator"); return UBLR_ERR_VALUE; }
  if (op->n <= 0) { set_error("operator has no rows"); return UBLR_ERR_VALUE; }
  if (op->kind == UBLR_OP_DENSE) {
    if (!op->A || op->lda < op->n) { set_error("dense operator needs A and lda >= n (perm NULL = identity)"); return UBLR_ERR_VALUE; }
  } else if (op->kind == UBLR_OP_LOG || op->kind == UBLR_OP_INV) {
    if (!op->coords || op->dim < 1 || op->dim > 3) { set_error("kernel operator needs coords with 1 <= dim <= 3"); return UBLR_ERR_VALUE; }
  } else {
    set_error("unknown operator kind");
    return UBLR_ERR_VALUE;
  }
  return UBLR_OK;
}

}  // namespace ublr
