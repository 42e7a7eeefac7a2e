// FP64 tensor-core (DMMA m8n8k4) vs FP64 vector (DFMA) throughput on this
// GPU, alone and interleaved in the same warps: do they share a pipe?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_probe.bin tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// NM independent DMMA accumulators and NF independent DFMA chains per iteration
template <int NM, int NF>
__global__ void k_mix(int iters, double* out) {
  double acc[NM > 0 ? NM : 1][2];
  double f[NF > 0 ? NF : 1];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.999999 - threadIdx.x * 1e-10;
#pragma unroll
  for (int m = 0; m < (NM > 0 ? NM : 1); ++m) acc[m][0] = acc[m][1] = m * 1e-3;
#pragma unroll
  for (int k = 0; k < (NF > 0 ? NF : 1); ++k) f[k] = k * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int m = 0; m < NM; ++m) dmma(acc[m], a, b);
#pragma unroll
    for (int k = 0; k < NF; ++k) f[k] = fma(f[k], b, a);
  }
  double s = 0.0;
#pragma unroll
  for (int m = 0; m < (NM > 0 ? NM : 1); ++m) s += acc[m][0] + acc[m][1];
#pragma unroll
  for (int k = 0; k < (NF > 0 ? NF : 1); ++k) s += f[k];
  if (s == 12345.678) out[0] = s;
}

template <int NM, int NF>
void run(const char* name, int warps_per_sm, int sms, double clk_ghz) {
  const int threads = 256, blocks = sms * warps_per_sm / 8, iters = 20000;
  double* d;
  cudaMalloc(&d, 8);
  k_mix<NM, NF><<<blocks, threads>>>(100, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_mix<NM, NF><<<blocks, threads>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double cycles = ms * 1e-3 * clk_ghz * 1e9;
  const double warps = double(blocks) * threads / 32;
  const double mma_rate = warps * iters * NM / sms / cycles, fma_rate = warps * iters * NF / sms / cycles;
  const double tf = (warps * iters * (NM * 512.0 + NF * 64.0)) / (ms * 1e-3) / 1e12;
  std::printf("%-28s warps/SM=%2d %8.3f ms  DMMA %.3f/SM/clk  DFMA %.3f warp-instr/SM/clk  %.2f TFLOP/s%s\n", name,
              warps_per_sm, ms, mma_rate, fma_rate, tf, cudaGetLastError() == cudaSuccess ? "" : "  ERROR");
  cudaFree(d);
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double ghz = clk * 1e-6;
  std::printf("SMs %d clock %.3f GHz (attribute)\n", sms, ghz);
  for (int w : {8, 16, 32}) {
    run<4, 0>("DMMA x4", w, sms, ghz);
    run<8, 0>("DMMA x8", w, sms, ghz);
    run<0, 8>("DFMA x8", w, sms, ghz);
    run<1, 6>("1 DMMA + 6 DFMA", w, sms, ghz);
    run<1, 12>("1 DMMA + 12 DFMA", w, sms, ghz);
    run<2, 12>("2 DMMA + 12 DFMA", w, sms, ghz);
    run<1, 24>("1 DMMA + 24 DFMA", w, sms, ghz);
  }
  return 0;
}
