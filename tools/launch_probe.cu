// launch_probe.cu — device time of one launch after a 256 MiB memset (the
// bench's L2 flush), by grid shape and dynamic shared memory: how much of a
// short kernel's step is launch, shared-memory carveout and drain.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_empty(int* p) { if (p && threadIdx.x == 1023) p[0] = 1; }
__global__ void k_smem(int* p) {
  extern __shared__ int sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (p && sm[(threadIdx.x + 1) % blockDim.x] == -1) p[0] = 1;
}
int main() {
  void* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct { const char* name; int grid, block, smem; bool graph; } cfg[] = {
      {"empty 148x512", 148, 512, 0, false},
      {"smem0 148x512", 148, 512, 0, false},
      {"smem48K 148x512", 148, 512, 48 * 1024, false},
      {"smem200K 148x512", 148, 512, 200 * 1024, false},
      {"smem200K 148x512 graph", 148, 512, 200 * 1024, true},
      {"smem40K 1184x64", 1184, 64, 40 * 1024, false},
  };
  for (auto& c : cfg) {
    cudaGraphExec_t ge = nullptr;
    if (c.graph) {
      cudaGraph_t g;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      k_smem<<<c.grid, c.block, c.smem, s>>>(nullptr);
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
    }
    float tot = 0;
    const int R = 50;
    for (int i = 0; i < R + 3; ++i) {
      cudaMemsetAsync(flush, i, 256 << 20, s);
      cudaEventRecord(a, s);
      if (ge) cudaGraphLaunch(ge, s);
      else if (c.smem == 0) k_empty<<<c.grid, c.block, 0, s>>>(nullptr);
      else k_smem<<<c.grid, c.block, c.smem, s>>>(nullptr);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (i >= 3) tot += ms;
    }
    printf("{\"probe\": \"%s\", \"us\": %.2f}\n", c.name, tot / R * 1000);
  }
  return 0;
}
