// Dependent-chain latencies on this GPU (cycles, one warp): DFMA, DMUL,
// MUFU.RCP64H (+DFMA), LDS.128 -> DFMA, and the throughput of the PP inner
// loop shape at several warp counts (how many warps hide its latency).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o latency_probe tools/latency_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

__device__ __forceinline__ double rcp_approx(double x) {
  double r;
  asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

__global__ void lat_dfma(double* out, long long* cyc, double a, double b) {
  double x = threadIdx.x * 1e-9 + 1.0;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    x = fma(x, a, b);
    x = fma(x, a, b);
    x = fma(x, a, b);
    x = fma(x, a, b);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}

__global__ void lat_rcp(double* out, long long* cyc, double a) {
  double x = threadIdx.x * 1e-9 + 1.5;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    x = rcp_approx(x) + a;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}

__global__ void lat_lds(double* out, long long* cyc) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (i + 1) % 1024;
  __syncthreads();
  int idx = 0;
  double acc = 0;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1024; ++i) {
    const double v = s[idx];
    idx = static_cast<int>(v);
    acc += v;
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[0] = (t1 - t0);
}

// PP fast-path loop on smem-broadcast sources; blocks x threads set occupancy.
__global__ void pp_loop(double* out, int iters) {
  __shared__ double4 src[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    src[i] = make_double4(0.3 + i * 1e-4, 0.4 - i * 1e-4, 0.5, 1e-3 * i);
  __syncthreads();
  const double x0 = 0.577 + threadIdx.x * 1e-7, x1 = 0.577, x2 = -0.577;
  double s0 = 0, s1 = 0, s2 = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int k = 0; k < 256; ++k) {
      const double4 y = src[k];
      const double den = fma(-x2, y.z, fma(-x1, y.y, fma(-x0, y.x, 1.0)));
      const double r0 = rcp_approx(den);
      double e = fma(-den, r0, 1.0);
      e = fma(e, e, e);
      const double y0 = y.w * r0;
      const double r = fma(y0, e, y0);
      s0 = fma(r, y.x, s0);
      s1 = fma(r, y.y, s1);
      s2 = fma(r, y.z, s2);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s0 + s1 + s2;
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1 << 24);
  cudaMalloc(&c, 64);
  long long h;
  lat_dfma<<<1, 32>>>(d, c, 0.9999, 1e-9);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", h / 4096.0);
  lat_rcp<<<1, 32>>>(d, c, 0.5);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("MUFU.RCP64H + DADD dependent latency: %.2f cycles\n", h / 1024.0);
  lat_lds<<<1, 32>>>(d, c);
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("LDS.64 -> F2I dependent latency: %.2f cycles\n", h / 1024.0);
  int sms = 148;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 64;
  for (int warps_per_sm : {8, 16, 24, 32, 48, 64}) {
    const int threads = 256, blocks = sms * warps_per_sm / 8;
    pp_loop<<<blocks, threads>>>(d, 1);
    cudaEventRecord(e0);
    pp_loop<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double pairs = double(blocks) * threads * iters * 256;
    printf("pp_loop warps/SM=%2d: %.3e pairs/s (%.1f%% of 10-DP/pair at 34.2 TF)\n", warps_per_sm,
           pairs / (ms * 1e-3), 100.0 * pairs * 10 * 2 / (ms * 1e-3) / 34.2e12);
  }
  return 0;
}
