// Ceiling probe for the leaf/fit inner loop: how much of the FP64 pipe can
// the staged pair block reach with no shared memory, fetch or loop overhead?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pair_ceiling tools/pair_ceiling.cu
// Prints, per variant, warp-instructions per SM per cycle and the implied
// FP64-pipe fraction (peak: 64 DFMA lanes / SM / cycle = 2 warp-instr / SM / cycle).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp_approx(double x) {
  double r;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

// (a) MUFU.RCP64H only: 8 independent chains
__global__ void k_mufu(double* out, int iters, double seed) {
  double v[8];
  for (int c = 0; c < 8; ++c) v[c] = seed + threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = rcp_approx(v[c]);
  double s = 0;
  for (int c = 0; c < 8; ++c) s += v[c];
  if (s == 1234.5) out[0] = s;
}

// (b) the production block: 2 sources x 2 targets, staged, 10 DP + 1 MUFU per pair
template <bool MUFU>
__global__ void k_pairs(double* out, int iters, double seed) {
  double x[2][3], a[2][3];
  for (int q = 0; q < 2; ++q)
    for (int d = 0; d < 3; ++d) {
      x[q][d] = 0.5 + 1e-3 * (threadIdx.x + q + d);
      a[q][d] = 0;
    }
  double y[2][4];
  for (int s = 0; s < 2; ++s)
    for (int d = 0; d < 4; ++d) y[s][d] = 0.1 * (s + d) + seed;
  for (int i = 0; i < iters; ++i) {
    double den[4], r[4], e[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) den[c] = fma(-x[c % 2][0], y[c / 2][0], 1.0);
#pragma unroll
    for (int c = 0; c < 4; ++c) den[c] = fma(-x[c % 2][1], y[c / 2][1], den[c]);
#pragma unroll
    for (int c = 0; c < 4; ++c) den[c] = fma(-x[c % 2][2], y[c / 2][2], den[c]);
#pragma unroll
    for (int c = 0; c < 4; ++c) r[c] = MUFU ? rcp_approx(den[c]) : den[c];
#pragma unroll
    for (int c = 0; c < 4; ++c) e[c] = fma(-den[c], r[c], 1.0);
#pragma unroll
    for (int c = 0; c < 4; ++c) e[c] = fma(e[c], e[c], e[c]);
#pragma unroll
    for (int c = 0; c < 4; ++c) r[c] = y[c / 2][3] * r[c];
#pragma unroll
    for (int c = 0; c < 4; ++c) r[c] = fma(r[c], e[c], r[c]);
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int d = 0; d < 3; ++d) a[c % 2][d] = fma(r[c], y[c / 2][d], a[c % 2][d]);
    // perturb the sources so nothing is loop-invariant
#pragma unroll
    for (int s = 0; s < 2; ++s) y[s][0] = y[s][0] + 1e-300;
  }
  double s = 0;
  for (int q = 0; q < 2; ++q)
    for (int d = 0; d < 3; ++d) s += a[q][d];
  if (s == 1234.5) out[0] = s;
}

template <class F>
void run(const char* name, F launch, double warp_instr_per_thread_iter, int iters, int blocks, int threads, int sms,
         double clk_ghz) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = double(blocks) * threads / 32.0;
  const double winstr = warps * iters * warp_instr_per_thread_iter;
  const double cycles = ms * 1e-3 * clk_ghz * 1e9;
  printf("%-34s %8.3f ms  %.3f warp-instr/SM/cycle\n", name, ms, winstr / sms / cycles);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double ghz = clk_khz / 1e6;
  const int sms = p.multiProcessorCount;
  double* d;
  cudaMalloc(&d, 64);
  const int iters = 20000;
  printf("SMs %d, clock %.3f GHz (attribute; actual may differ)\n", sms, ghz);
  for (int wps : {8, 16, 32, 48}) {
    const int threads = 256, blocks = sms * wps * 32 / threads;
    printf("-- %d warps/SM\n", wps);
    run("MUFU.RCP64H only (per MUFU)", [&] { k_mufu<<<blocks, threads>>>(d, iters, 1.5); }, 8.0, iters, blocks,
        threads, sms, ghz);
    run("pair block, 40 DP + 4 MUFU (per DP)", [&] { k_pairs<true><<<blocks, threads>>>(d, iters, 0.3); }, 40.0,
        iters, blocks, threads, sms, ghz);
    run("pair block, 40 DP, no MUFU (per DP)", [&] { k_pairs<false><<<blocks, threads>>>(d, iters, 0.3); }, 40.0,
        iters, blocks, threads, sms, ghz);
  }
  printf("FP64 pipe peak = 2.0 warp-instr/SM/cycle\n");
  return 0;
}
