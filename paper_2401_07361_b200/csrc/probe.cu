// FP64 roofline denominator, measured on the box the bench runs on.
// MEASURED_PEAKS.json carries no fp64 entry, so bench.py
// rates the interaction kernels against this DFMA-chain throughput: 8
// independent FMA chains per thread, 8 CTAs of 256 threads per SM, best of
// `reps` launches timed with CUDA events on the context's stream.
#include <algorithm>

#include "kernels.cuh"

namespace ssum {
namespace {

constexpr int kChains = 8;

__global__ void k_dfma_chain(double* out, int iters, double a, double b) {
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

__global__ void k_log_far(const double* __restrict__ x, int64_t n, const double2* __restrict__ tab_g,
                          double* __restrict__ out) {
  __shared__ double2 tab[kLogTabN * kLogTabCopies];  // as the log tiles stage it
  log_tab_stage(tab, tab_g, threadIdx.x, blockDim.x);
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) out[i] = log_tab(x[i], tab + (threadIdx.x & (kLogTabCopies - 1)));
}

}  // namespace
}  // namespace ssum

using namespace ssum;

// Accuracy probe of the far-pair log (kernels.cuh log_tab), host arrays.
extern "C" int ssum_probe_log_far(ssum_ctx* h, const double* x, int64_t n, double* out) {
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c || (n > 0 && (!x || !out)) || n < 0) return SSUM_INVALID;
  try {
    cudaSetDevice(c->device);
    if (n == 0) return SSUM_OK;
    DBuf<double> buf;
    buf.ensure(size_t(2 * n));
    SSUM_CUDA_CHECK(cudaMemcpyAsync(buf.p, x, size_t(n) * 8, cudaMemcpyHostToDevice, c->stream));
    k_log_far<<<static_cast<unsigned>((n + 255) / 256), 256, 0, c->stream>>>(buf.p, n, c->logtab.p, buf.p + n);
    SSUM_LAUNCH_CHECK();
    SSUM_CUDA_CHECK(cudaMemcpyAsync(out, buf.p + n, size_t(n) * 8, cudaMemcpyDeviceToHost, c->stream));
    SSUM_CUDA_CHECK(cudaStreamSynchronize(c->stream));
    return SSUM_OK;
  } catch (const Error& e) {
    c->last_error = e.what();
    return e.code;
  }
}

extern "C" int ssum_fp64_peak(ssum_ctx* h, int reps, double* tflops) {
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c || !tflops) return SSUM_INVALID;
  try {
    cudaSetDevice(c->device);
    int sms = 0;
    SSUM_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device));
    const int threads = 256, blocks = sms * 8, iters = 2048;
    double best = 0.0;
    for (int r = 0; r < reps + 1; ++r) {
      SSUM_CUDA_CHECK(cudaEventRecord(c->ev[6], c->stream));
      k_dfma_chain<<<blocks, threads, 0, c->stream>>>(reinterpret_cast<double*>(c->d_flags.p + 32), iters, 0.999999, 1e-7);
      SSUM_LAUNCH_CHECK();
      SSUM_CUDA_CHECK(cudaEventRecord(c->ev[7], c->stream));
      SSUM_CUDA_CHECK(cudaEventSynchronize(c->ev[7]));
      float ms = 0.f;
      SSUM_CUDA_CHECK(cudaEventElapsedTime(&ms, c->ev[6], c->ev[7]));
      const double flop = 2.0 * blocks * threads * double(iters) * 16 * kChains;
      if (r > 0) best = std::max(best, flop / (ms * 1e-3) / 1e12);  // first launch is warm-up
    }
    *tflops = best;
    return SSUM_OK;
  } catch (const Error& e) {
    c->last_error = e.what();
    return e.code;
  }
}
