// pf_counters.cuh — per-thread counters (PolynomialPdf clamps, pdf.hpp:313-316).
// Included after the generated PF_NPOLY definition.
#pragma once

#if PF_NPOLY > 0
#define PF_CLAMP_ARRAY pf_u32 clamp[PF_NPOLY];
#else
#define PF_CLAMP_ARRAY pf_u32 clamp[1];
#endif

struct pf_cnt {
  PF_CLAMP_ARRAY
};

__device__ __forceinline__ void pf_cnt_init(pf_cnt& c) {
#pragma unroll
  for (int i = 0; i < (PF_NPOLY > 0 ? PF_NPOLY : 1); ++i) c.clamp[i] = 0;
}

__device__ __forceinline__ void pf_cnt_flush(const pf_cnt& c, pf_u64* clamp) {
#if PF_NPOLY > 0
#pragma unroll
  for (int i = 0; i < PF_NPOLY; ++i)
    if (c.clamp[i]) atomicAdd(clamp + i, (pf_u64)c.clamp[i]);
#endif
}

