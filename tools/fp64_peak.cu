// fp64_peak.cu — measured FP64 (DFMA) throughput of the device, the
// roofline denominator for FP64-bound configurations (C4 convolution).
// 8 independent DFMA chains per thread, full occupancy, CUDA-event timed.
#include <cstdio>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256, iters = 1 << 16;
  double* out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_loop<<<blocks, threads>>>(out, 1024, 0.999999, 1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fmas = 8.0 * iters * (double)blocks * threads;
  const double tflops = 2.0 * fmas / (best * 1e-3) / 1e12;
  std::printf("{\"fp64_tflops\": %.3f, \"dfma_per_s\": %.4e, \"sms\": %d, \"max_clock_mhz\": %.0f, "
              "\"dfma_per_clk_per_sm_at_max_clock\": %.2f, \"ms\": %.3f}\n",
              tflops, fmas / (best * 1e-3), sms, clk / 1e3, fmas / (best * 1e-3) / sms / (clk * 1e3), best);
  return 0;
}
