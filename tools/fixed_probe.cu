// fixed_probe.cu — fixed costs of one event-pass launch on this GPU (device
// time per launch, CUDA events, no L2 flush): empty persistent grids, the
// last-block completion pattern, publishing into mapped host memory with and
// without a system-scope release, and the first TMA bulk fill of a stage.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ unsigned g_done;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int MODE>
__global__ void k_probe(double* dev_out, double* host_out, const double* data, uint64_t stride) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int last;
  if (MODE == 5 || MODE == 6) {  // one 4 KB bulk copy per warp-0, wait for it
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(4096));
      const double* src = data + (uint64_t)blockIdx.x * 512;
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(dyn)),
          "l"(src), "r"(4096), "r"(smem_u32(&bar))
          : "memory");
    }
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(ok)
          : "r"(smem_u32(&bar)), "r"(0)
          : "memory");
    if (MODE == 5) return;
  }
  if (MODE == 0) return;
  // last block pattern
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&g_done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  if (threadIdx.x == 0) g_done = 0;
  if (threadIdx.x < 32) {
    if (MODE == 1 || MODE == 6) {
      dev_out[threadIdx.x] = threadIdx.x;
    } else if (MODE == 2) {
      host_out[threadIdx.x] = threadIdx.x;
    } else if (MODE == 3) {
      host_out[threadIdx.x] = threadIdx.x;
      __syncwarp();
      if (threadIdx.x == 0)
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(host_out + 32), "l"(1ull) : "memory");
    } else if (MODE == 4) {
      host_out[threadIdx.x] = threadIdx.x;
      __syncwarp();
      if (threadIdx.x == 0) {
        __threadfence_system();
        *(volatile double*)(host_out + 32) = 1.0;
      }
    } else if (MODE == 7) {  // 16 B store only (value + sequence in one store)
      if (threadIdx.x == 0) {
        asm volatile("st.volatile.global.v2.f64 [%0], {%1, %2};" ::"l"(host_out), "d"(1.0), "d"(2.0) : "memory");
      }
    }
  }
}

template <int MODE>
float run(int grid, int block, double* d, double* h, const double* data, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k_probe<MODE><<<grid, block, 8192>>>(d, h, data, 0);
  cudaDeviceSynchronize();
  float tot = 0;
  for (int i = 0; i < reps; ++i) {
    cudaEventRecord(a);
    k_probe<MODE><<<grid, block, 8192>>>(d, h, data, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    tot += ms;
  }
  return tot / reps * 1000.0f;
}

int main() {
  double *d, *h, *hd, *data;
  cudaMalloc(&d, 4096);
  cudaHostAlloc(&h, 4096, cudaHostAllocMapped);
  cudaHostGetDevicePointer((void**)&hd, h, 0);
  cudaMalloc(&data, 64ull << 20);
  cudaMemset(data, 0, 64ull << 20);
  const int R = 200;
  struct { int g, b; } shapes[] = {{1, 64}, {148, 64}, {1184, 64}, {148, 256}, {148, 512}, {296, 256}};
  const char* names[] = {"empty", "last-block dev store", "last-block host store", "host store + st.release.sys",
                         "host store + threadfence_system", "tma first fill", "tma fill + last-block dev", "host 16B store"};
  for (auto s : shapes) {
    float t[8];
    t[0] = run<0>(s.g, s.b, d, hd, data, R);
    t[1] = run<1>(s.g, s.b, d, hd, data, R);
    t[2] = run<2>(s.g, s.b, d, hd, data, R);
    t[3] = run<3>(s.g, s.b, d, hd, data, R);
    t[4] = run<4>(s.g, s.b, d, hd, data, R);
    t[5] = run<5>(s.g, s.b, d, hd, data, R);
    t[6] = run<6>(s.g, s.b, d, hd, data, R);
    t[7] = run<7>(s.g, s.b, d, hd, data, R);
    for (int i = 0; i < 8; ++i)
      printf("{\"grid\": %d, \"block\": %d, \"probe\": \"%s\", \"us\": %.2f}\n", s.g, s.b, names[i], t[i]);
  }
  // a CUDA graph of one kernel vs two back-to-back kernels
  return 0;
}
