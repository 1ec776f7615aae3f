// fp64_probe.cu — FP64 latency and per-SM throughput on this GPU (clock64
// inside one CTA): a dependent DFMA chain, independent DFMA streams with 1-16
// warps, and the I2F.F64.U64 conversion the grid-point index takes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int N = 4096;

template <int ILP>
__global__ void k_fma(double* out, long long* cyc, double a, double b) {
  double x[ILP];
#pragma unroll
  for (int i = 0; i < ILP; ++i) x[i] = threadIdx.x + i;
  __syncthreads();
  const long long t0 = clock64();
  for (int n = 0; n < N; ++n)
#pragma unroll
    for (int i = 0; i < ILP; ++i) x[i] = fma(x[i], a, b);
  __syncthreads();
  const long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int i = 0; i < ILP; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void k_i2f(double* out, long long* cyc, unsigned long long a) {
  unsigned long long v = threadIdx.x;
  double s = 0;
  __syncthreads();
  const long long t0 = clock64();
  for (int n = 0; n < N; ++n) {
    const double d = (double)v;  // dependent: the next index comes from the converted value
    s += d;
    v = (unsigned long long)__double2loint(d) + a;
  }
  __syncthreads();
  const long long t1 = clock64();
  out[threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 20);
  cudaMalloc(&cyc, 1024);
  long long h;
  auto run = [&](const char* name, auto kern, int threads, double ops_per_thread) {
    for (int rep = 0; rep < 2; ++rep) kern<<<1, threads>>>(out, cyc, 1.0000001, 1e-9);
    cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    const double per_clk = ops_per_thread * threads / (double)h;
    printf("{\"probe\": \"%s\", \"threads\": %d, \"cycles\": %lld, \"lane_ops_per_clk_per_sm\": %.2f, "
           "\"cycles_per_op_per_thread\": %.2f}\n",
           name, threads, h, per_clk, (double)h / ops_per_thread);
  };
  run("dfma chain (latency)", k_fma<1>, 32, N);
  for (int w : {1, 2, 4, 8, 16, 32})
    run("dfma ilp4", k_fma<4>, 32 * w, 4.0 * N);
  for (int w : {4, 16, 32})
    run("dfma ilp8", k_fma<8>, 32 * w, 8.0 * N);
  k_i2f<<<1, 32>>>(out, cyc, 3);
  k_i2f<<<1, 32>>>(out, cyc, 3);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"probe\": \"i2f.f64.u64 + dadd + int chain\", \"cycles_per_iter\": %.2f}\n", (double)h / N);
  return 0;
}
