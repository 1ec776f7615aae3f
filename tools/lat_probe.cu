// lat_probe.cu — dependent-chain latencies on this GPU (cycles per op, one
// warp), used to size ILP/occupancy of the FP64-heavy kernels.
#include <cstdio>

template <int OP>
__global__ void chain(double* out, long long* cyc, double a, double b, int n) {
  double x = a + threadIdx.x;
  unsigned u = threadIdx.x;
  __syncwarp();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (OP == 0) x = x + b;                                  // DADD
    if (OP == 1) x = fma(x, a, b);                           // DFMA
    if (OP == 2) x = x * a;                                  // DMUL
    if (OP == 3) x = __shfl_xor_sync(0xffffffffu, x, 1);     // SHFL (64-bit: 2 x SHFL)
    if (OP == 4) x = (x > b ? x : b) + 1.0;                  // DSETP + FSEL + DADD
    if (OP == 5) u = u * 3u + 1u;                            // IMAD
    if (OP == 6) x = __longlong_as_double(__double_as_longlong(x) + 1) ;  // int64 add on a double
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = x + u;
}

template <int OP>
void run(const char* name, double* out, long long* cyc) {
  const int n = 4096;
  chain<OP><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n);
  chain<OP><<<1, 32>>>(out, cyc, 1.0000001, 1e-9, n);
  long long h;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("{\"op\": \"%s\", \"cycles_per_iter\": %.2f}\n", name, (double)h / n);
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1024 * 8);
  cudaMalloc(&cyc, 8);
  run<0>("DADD", out, cyc);
  run<1>("DFMA", out, cyc);
  run<2>("DMUL", out, cyc);
  run<3>("SHFL f64", out, cyc);
  run<4>("DSETP+FSEL+DADD", out, cyc);
  run<5>("IMAD", out, cyc);
  run<6>("IADD64", out, cyc);
  return 0;
}
