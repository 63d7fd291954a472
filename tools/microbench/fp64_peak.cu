// FP64 pipe microbenchmark for B200 (sm_100a): DFMA vs DMMA shapes, log/rsqrt cost.
// Used once to pick the MMA shape and to measure the FP64 roofline denominator
// (MEASURED_PEAKS.json carries only HBM and bf16 peaks).
#include <cstdio>
#include <cuda_runtime.h>
#include <cmath>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void k_dfma(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0+4, a5=a0+5, a6=a0+6, a7=a0+7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void k_m8n8k4(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 - a;
  double c[8][2];
  for (int t = 0; t < 8; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0; for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_m16n8k4(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 0.5, b = 1.0 - a0;
  double c[8][4];
  for (int t = 0; t < 8; ++t) for (int q = 0; q < 4; ++q) c[t][q] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3]) : "d"(a0), "d"(a1), "d"(b));
  }
  double s = 0; for (int t = 0; t < 8; ++t) for (int q = 0; q < 4; ++q) s += c[t][q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_m16n8k8(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 0.5, a2 = a0 + .25, a3 = a0 + .125, b0 = 1.0 - a0, b1 = b0 * .5;
  double c[8][4];
  for (int t = 0; t < 8; ++t) for (int q = 0; q < 4; ++q) c[t][q] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a0), "d"(a1), "d"(a2), "d"(a3), "d"(b0), "d"(b1));
  }
  double s = 0; for (int t = 0; t < 8; ++t) for (int q = 0; q < 4; ++q) s += c[t][q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_m16n8k16(double* out, int iters) {
  double a[8], b[4];
  for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-3 + q;
  for (int q = 0; q < 4; ++q) b[q] = 1.0 - q * 1e-3;
  double c[8][4];
  for (int t = 0; t < 8; ++t) for (int q = 0; q < 4; ++q) c[t][q] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(c[t][0]), "+d"(c[t][1]), "+d"(c[t][2]), "+d"(c[t][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
  }
  double s = 0; for (int t = 0; t < 8; ++t) for (int q = 0; q < 4; ++q) s += c[t][q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_log(double* out, int iters) {
  double x = 1.0 + threadIdx.x * 1e-5, s = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) { s += log(x); x += 1e-9; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_rsqrt(double* out, int iters) {
  double x = 1.0 + threadIdx.x * 1e-5, s = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) { s += rsqrt(x); x += 1e-9; }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Launch errors (e.g. too many registers for 1024-thread blocks) are checked
// after every launch: a failed launch returns a negative time and the row is
// reported as FAILED instead of timing an empty kernel.
template <class K>
float run(K kern, double* out, int blocks, int threads, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, 10);
  if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) return -1.f;
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(out, iters);
  if (cudaGetLastError() != cudaSuccess) return -1.f;
  cudaEventRecord(e1);
  if (cudaEventSynchronize(e1) != cudaSuccess) return -1.f;
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

static void report(const char* name, int tpb, float ms, double work, const char* unit) {
  if (ms <= 0.f) printf("%-8s tpb=%4d : FAILED (launch error: %s)\n", name, tpb, cudaGetErrorString(cudaGetLastError()));
  else printf("%-8s tpb=%4d : %.2f %s\n", name, tpb, work / (ms * 1e-3) / (unit[0] == 'T' ? 1e12 : 1e9), unit);
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 8 * 1024));
  int iters = 20000;
  for (int tpb : {256, 512, 1024}) {
    int blocks = sms * (1024 / tpb) * 1;
    double thr = (double)blocks * tpb;
    report("DFMA", tpb, run(k_dfma, out, blocks, tpb, iters), thr * iters * 64 * 2, "TFLOP/s");
    report("m8n8k4", tpb, run(k_m8n8k4, out, blocks, tpb, iters), thr / 32 * iters * 8 * (8 * 8 * 4) * 2, "TFLOP/s");
    report("m16n8k4", tpb, run(k_m16n8k4, out, blocks, tpb, iters), thr / 32 * iters * 8 * (16 * 8 * 4) * 2,
           "TFLOP/s");
    report("m16n8k8", tpb, run(k_m16n8k8, out, blocks, tpb, iters), thr / 32 * iters * 8 * (16 * 8 * 8) * 2,
           "TFLOP/s");
    report("m16n8k16", tpb, run(k_m16n8k16, out, blocks, tpb, iters / 2),
           thr / 32 * (iters / 2) * 8 * (16 * 8 * 16) * 2, "TFLOP/s");
    report("log", tpb, run(k_log, out, blocks, tpb, iters / 10), thr * (iters / 10) * 8, "Gevals/s");
    report("rsqrt", tpb, run(k_rsqrt, out, blocks, tpb, iters / 10), thr * (iters / 10) * 8, "Gevals/s");
  }
  return 0;
}
