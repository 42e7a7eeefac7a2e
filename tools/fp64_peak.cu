// FP64 roofline denominator for this repo: MEASURED_PEAKS.json has no fp64
// entry, so the interaction kernels are rated against the DFMA throughput this
// program measures on the box.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu
//   ./fp64_peak            -> one JSON line
//
// Three probes:
//   dfma   : 8 independent DFMA chains per thread, 148*k CTAs, long loop
//   mixed  : the per-pair instruction mix of the PP kernel (DMUL/DADD/DFMA +
//            rcp.approx.f64) to see how MUFU.RCP64H co-issues with the FP64 pipe
//   rcp    : max relative error of rcp.approx.ftz.f64 and of one Newton step
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
      exit(1);                                                                 \
    }                                                                          \
  } while (0)

constexpr int kChains = 8;

__global__ void dfma_chain(double* out, int iters, double a, double b) {
  double c[kChains];
#pragma unroll
  for (int k = 0; k < kChains; ++k) c[k] = threadIdx.x * 1e-9 + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
#pragma unroll
      for (int k = 0; k < kChains; ++k) c[k] = fma(c[k], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < kChains; ++k) s += c[k];
  if (s == 12345.678) out[0] = s;  // never true; keeps the chains live
}

__device__ __forceinline__ double rcp_approx(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

// One "pair" of the fast PP path: 3 DFMA den, MUFU + 3 DP reciprocal, 3 DFMA accumulate.
__global__ void pair_mix(double* out, int iters, double x0, double x1, double x2) {
  double s0 = 0, s1 = 0, s2 = 0;
  double y0 = 0.3 + threadIdx.x * 1e-7, y1 = 0.4, y2 = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int u = 0; u < 32; ++u) {
      double den = fma(-x2, y2, fma(-x1, y1, fma(-x0, y0, 1.0)));
      double r0 = rcp_approx(den);
      double q = y0 * r0;
      double e = fma(-den, r0, 1.0);
      double r = fma(q, e, q);
      s0 = fma(r, y0, s0);
      s1 = fma(r, y1, s1);
      s2 = fma(r, y2, s2);
      y0 += 1e-9;
    }
  }
  if (s0 + s1 + s2 == 12345.678) out[0] = s0;
}

__global__ void rcp_err(const double* x, int n, double* err0, double* err1) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d = x[i];
  double r0 = rcp_approx(d);
  double e = fma(-d, r0, 1.0);
  double r1 = fma(r0, e, r0);
  double exact = 1.0 / d;
  err0[i] = fabs(r0 - exact) / exact;
  err1[i] = fabs(r1 - exact) / exact;
}

int main() {
  int dev = 0;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  const int sms = prop.multiProcessorCount;
  double* dout;
  CK(cudaMalloc(&dout, 1 << 20));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));

  // --- DFMA peak
  const int threads = 256, blocks = sms * 8, iters = 4096;
  double best_tf = 0;
  for (int rep = 0; rep < 6; ++rep) {
    CK(cudaEventRecord(e0));
    dfma_chain<<<blocks, threads>>>(dout, iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double flop = 2.0 * blocks * threads * (double)iters * 16 * kChains;
    const double tf = flop / (ms * 1e-3) / 1e12;
    if (rep > 0 && tf > best_tf) best_tf = tf;
  }
  // sustained: back-to-back for ~3 s
  double sus_tf = 0;
  {
    const int launches = 200;
    CK(cudaEventRecord(e0));
    for (int l = 0; l < launches; ++l) dfma_chain<<<blocks, threads>>>(dout, iters, 0.999999, 1e-7);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double flop = 2.0 * blocks * threads * (double)iters * 16 * kChains * launches;
    sus_tf = flop / (ms * 1e-3) / 1e12;
  }

  // --- pair mix
  double pairs_per_s = 0;
  for (int rep = 0; rep < 4; ++rep) {
    CK(cudaEventRecord(e0));
    pair_mix<<<blocks, threads>>>(dout, 1024, 0.1, 0.2, 0.3);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    const double pairs = (double)blocks * threads * 1024 * 32;
    if (rep > 0) pairs_per_s = std::max(pairs_per_s, pairs / (ms * 1e-3));
  }

  // --- rcp accuracy over [1e-14, 2]
  const int n = 1 << 20;
  std::vector<double> hx(n);
  srand(7);
  for (int i = 0; i < n; ++i) {
    const double u = (rand() + 0.5) / (RAND_MAX + 1.0);
    hx[i] = std::pow(10.0, -14.0 + 14.3 * u);
  }
  double *dx, *de0, *de1;
  CK(cudaMalloc(&dx, n * 8));
  CK(cudaMalloc(&de0, n * 8));
  CK(cudaMalloc(&de1, n * 8));
  CK(cudaMemcpy(dx, hx.data(), n * 8, cudaMemcpyHostToDevice));
  rcp_err<<<(n + 255) / 256, 256>>>(dx, n, de0, de1);
  CK(cudaGetLastError());
  std::vector<double> h0(n), h1(n);
  CK(cudaMemcpy(h0.data(), de0, n * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(h1.data(), de1, n * 8, cudaMemcpyDeviceToHost));
  double m0 = 0, m1 = 0;
  for (int i = 0; i < n; ++i) {
    m0 = std::max(m0, h0[i]);
    m1 = std::max(m1, h1[i]);
  }
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
  printf(
      "{\"fp64_dfma_tflops_burst\": %.3f, \"fp64_dfma_tflops_sustained\": %.3f, "
      "\"pair_mix_pairs_per_s\": %.4e, \"rcp_approx_max_rel_err\": %.3e, "
      "\"rcp_newton1_max_rel_err\": %.3e, \"sms\": %d, \"clock_khz_attr\": %d, \"name\": \"%s\"}\n",
      best_tf, sus_tf, pairs_per_s, m0, m1, sms, clk_khz, prop.name);
  return 0;
}
