// conv_probe.cu — the C4 per-bin convolution recurrence (codegen.cpp,
// Gaussian-resolution fast sum: fw = fw E + M[jf] T[jf - jc], bw likewise
// with 1/E) alone on shared-memory tables, 2-warp blocks x 8 per SM as the
// event pass runs it: cycles per (bin, tau) against the variant:
//   0  as generated: M and T loaded per step (4 LDS + 2 DMUL + 2 DFMA per step pair)
//   1  M and T as 16-byte pairs (LDS.128)
//   2  products A[k] = M[jc + k] T[k] precomputed per warp (1 LDS + 1 DFMA per step)
//   3  variant 2 with two sub-chains per direction (step E^2)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/conv_probe.bin tools/conv_probe.cu
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <cuda_runtime.h>

constexpr int Q = 1024;
constexpr int WARPS = 2;
constexpr int BINS_PER_LANE = 4;
constexpr int KB = 128;

template <int VAR, int BPS = 8>
__global__ void __launch_bounds__(64, BPS) k_conv(const double* Mg, const double* Tg, double* out, long long* cyc, int jc0) {
  __shared__ __align__(16) double M[Q + 2];
  __shared__ __align__(16) double T[Q + 2];
  __shared__ __align__(16) double A[WARPS][2][KB];  // 16-byte aligned rows (KB even)
  for (int i = threadIdx.x; i < Q + 2; i += blockDim.x) {
    M[i] = Mg[i];
    T[i] = Tg[i];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double res = 0.0;
  long long t0 = clock64();
  for (int b = 0; b < BINS_PER_LANE; ++b) {
    const int jc = jc0 + (b & 1);  // warp-uniform centre
    const int j0 = 4, j1 = Q - 4;
    const double E = 1.0 - 1e-4 * (lane + 1 + b), Ei = 1.0 / E;
    double fw = 0.0, bw = 0.0;
    int jf = j1 - 1, jb = j0;
    for (; jf - jc + 1 > jc - jb; --jf) fw = fma(fw, E, M[jf] * T[jf - jc]);
    for (; jc - jb > jf - jc + 1; ++jb) bw = fma(bw, Ei, M[jb] * T[jc - jb]);
    if (VAR == 0 || (VAR == 1 && (jc & 1))) {  // (pairs of M and T align only for even jc)
#pragma unroll 16
      for (; jf >= jc; --jf, ++jb) {
        fw = fma(fw, E, M[jf] * T[jf - jc]);
        bw = fma(bw, Ei, M[jb] * T[jc - jb]);
      }
    } else if (VAR == 1) {
      // pairs: M[jf-1..jf] needs jf-1 even, T[jf-jc-1..jf-jc] needs jf-jc-1 even
      if (((jf - 1) & 1) || ((jf - jc - 1) & 1)) {
        fw = fma(fw, E, M[jf] * T[jf - jc]);
        bw = fma(bw, Ei, M[jb] * T[jc - jb]);
        --jf, ++jb;
      }
#pragma unroll 8
      for (; jf - 1 >= jc; jf -= 2, jb += 2) {
        const double2 m = *reinterpret_cast<const double2*>(&M[jf - 1]);
        const double2 t = *reinterpret_cast<const double2*>(&T[jf - jc - 1]);
        fw = fma(fw, E, m.y * t.y);
        fw = fma(fw, E, m.x * t.x);
        bw = fma(bw, Ei, M[jb] * T[jc - jb]);
        bw = fma(bw, Ei, M[jb + 1] * T[jc - jb - 1]);
      }
      for (; jf >= jc; --jf, ++jb) {
        fw = fma(fw, E, M[jf] * T[jf - jc]);
        bw = fma(bw, Ei, M[jb] * T[jc - jb]);
      }
    } else {
      // the remaining L steps in blocks of KB: the warp's products for a block
      // lane-parallel into its scratch, then KB recurrence steps reading them
      const int L = jf - jc + 1;
      double* af = A[warp][0];
      double* ab = A[warp][1];
      const double E2 = E * E, Ei2 = Ei * Ei;
      double fw2 = 0.0, bw2 = 0.0;
      for (int s0 = 0; s0 < L; s0 += KB) {
        const int n = min(KB, L - s0);
        __syncwarp();
        for (int i = lane; i < n; i += 32) {
          const int k = L - 1 - (s0 + i), kb = L - (s0 + i);
          af[i] = M[jc + k] * T[k];
          ab[i] = M[jc - kb] * T[kb];
        }
        __syncwarp();
        if (VAR == 4 && !(n & 1)) {  // pairs of products by 16-byte loads: half the LDS
          const double2* af2 = reinterpret_cast<const double2*>(af);
          const double2* ab2 = reinterpret_cast<const double2*>(ab);
#pragma unroll 8
          for (int i = 0; i < n / 2; ++i) {
            const double2 f = af2[i], g = ab2[i];
            fw = fma(fw, E, f.x);
            bw = fma(bw, Ei, g.x);
            fw = fma(fw, E, f.y);
            bw = fma(bw, Ei, g.y);
          }
        } else if (VAR == 2 || VAR == 4) {
#pragma unroll 16
          for (int i = 0; i < n; ++i) {
            fw = fma(fw, E, af[i]);
            bw = fma(bw, Ei, ab[i]);
          }
        } else {
#pragma unroll 8
          for (int i = 0; i < n; i += 2) {  // n even here (KB even, L even in the probe)
            fw = fma(fw, E2, af[i]);
            fw2 = fma(fw2, E2, af[i + 1]);
            bw = fma(bw, Ei2, ab[i]);
            bw2 = fma(bw2, Ei2, ab[i + 1]);
          }
        }
      }
      if (VAR == 3) {
        fw = fma(fw, E, fw2);
        bw = fma(bw, Ei, bw2);
      }
      jf = jc - 1;
    }
    res += fma(bw, Ei, fw);
    __syncwarp();
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = res;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  double *Mg, *Tg, *out;
  long long* cyc;
  cudaMalloc(&Mg, (Q + 2) * 8);
  cudaMalloc(&Tg, (Q + 2) * 8);
  cudaMalloc(&out, 148 * 32 * 64 * 8);
  cudaMalloc(&cyc, 148 * 32 * 8);
  double hM[Q + 2], hT[Q + 2];
  for (int i = 0; i < Q + 2; ++i) {
    hM[i] = 1.0 / (1.0 + (i - 512) * (i - 512) * 1e-4);
    hT[i] = exp(-1e-5 * i * i);
  }
  cudaMemcpy(Mg, hM, sizeof(hM), cudaMemcpyHostToDevice);
  cudaMemcpy(Tg, hT, sizeof(hT), cudaMemcpyHostToDevice);
  static long long hc[148 * 32];
  auto run = [&](int var, auto kern, int bps) {
    const int G = 148 * bps;
    for (int rep = 0; rep < 3; ++rep) kern<<<G, 64>>>(Mg, Tg, out, cyc, 500);
    if (cudaDeviceSynchronize() != cudaSuccess || cudaGetLastError() != cudaSuccess) {
      printf("{\"variant\": %d, \"error\": true}\n", var);
      return;
    }
    cudaMemcpy(hc, cyc, G * 8, cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < G; ++i) mx = hc[i] > mx ? hc[i] : mx;
    // per SM: bps blocks x 64 lanes x BINS_PER_LANE bins x ~(Q - 8) taus, all co-resident
    const double taus = (double)bps * 64 * BINS_PER_LANE * (Q - 8);
    double h0;
    cudaMemcpy(&h0, out, 8, cudaMemcpyDeviceToHost);
    printf("{\"variant\": %d, \"blocks_per_sm\": %d, \"cycles_max\": %lld, \"taus_per_clk_per_sm\": %.2f, "
           "\"us_per_1e6_bins_x_1016_taus\": %.1f, \"out0\": %.17g}\n",
           var, bps, mx, taus / mx, 1e6 * (Q - 8) / 148.0 / (taus / mx) / 1965.0, h0);
  };
  run(0, k_conv<0>, 8);
  run(1, k_conv<1>, 8);
  run(2, k_conv<2>, 8);
  run(3, k_conv<3>, 8);
  run(4, k_conv<4>, 8);
  run(0, k_conv<0, 16>, 16);
  run(2, k_conv<2, 16>, 16);
  run(4, k_conv<4, 16>, 16);
  return 0;
}
