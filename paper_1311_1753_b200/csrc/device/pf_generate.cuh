// pf_generate.cuh — toy generation on the GPU: generate_events
// (generate.hpp:33-86) with the reference's ToyRng bit recipe.
//
// Included after pf_kernels.cuh when the module is built for a generator
// (PF_GEN).  The reference draws candidates one at a time from ONE
// std::mt19937_64 stream: per candidate, one uniform per box dimension (box
// order) and one for the accept test.  Here:
//   pf_gen_max_kernel      the envelope scan: max of raw/norm over the
//                          midpoint grid (generate.hpp:47-63), order-free
//   pf_mt_kernel           the mt19937_64 stream, one CTA: each 312-word
//                          twist is two dependency-free halves of 156 words
//                          (x[k+312] = x[k+156] ^ twist(x[k], x[k+1])), two
//                          barriers per twist; it overlaps the previous
//                          batch's evaluation (second stream)
//   pf_gen_eval_kernel     every candidate of a batch in parallel: density,
//                          accept flag, first envelope failure / raw error
//   pf_gen_scan_kernel     exclusive scan of the per-block accept counts
//   pf_gen_scatter_kernel  accepted candidates, in stream order, into the
//                          SoA output columns (stops at the n-th acceptance)
// Candidate arithmetic is the reference's, rounded explicitly (no FMA
// contraction): x = lo + (hi - lo) * u and accept iff u * envelope < density.
#pragma once

#define PF_GEN_THREADS 256
#define PF_GEN_PER_THREAD 8
#define PF_GEN_SEGMENT (PF_GEN_THREADS * PF_GEN_PER_THREAD)  // candidates per block
#define PF_MT_N 312
#define PF_MT_M 156

struct pf_gen_args {
  const double* P;
  const double* S;
  const double* C;
  int dims;             // root box dimensions
  int pad0;
  int cols[8];          // event column per box dimension (box order)
  double lo[8];         // observable lower bound
  double span[8];       // upper - lower (candidates)
  double h[8];          // grid spacing (envelope scan)
  pf_u64 points;        // grid points per dimension
  pf_u64 total;         // grid points
  double envelope;
  const double* u;      // batch stream words (raw mt19937_64 state words, as bits): dims + 1 per candidate
  pf_u64 n_cand;        // candidates in the batch
  unsigned char* flags; // per candidate: 1 accepted
  pf_u32* block_count;  // accepted per block
  pf_u32* block_base;   // exclusive scan of block_count
  pf_u64* rec;          // [0] max density bits, [1] first error key, [2] first failure,
                        // [3] candidate of the last needed acceptance, [4] accepted in batch
  double* fail_density; // density of a failing candidate (sparse)
  double* out;          // SoA: dims columns, stride out_stride
  pf_u64 out_stride;
  pf_u64 out_base;      // events already generated
  pf_u64 remaining;     // events still needed
  pf_u64* mt;           // 312-word generator state
  pf_u64 rounds;        // twists this launch
  // jump-ahead draw (pf_mt_jump_kernel)
  const pf_u64* jpoly;  // [segment][312]: x^(k J) mod phi, little-endian bit words
  pf_u64* mt_next;      // the window after the batch (the next batch's base)
  pf_u64 jump_words;    // J: words per segment
  pf_u64 u_off;         // first word of this batch's segments in u
};

__device__ __forceinline__ double pf_gen_density(const pf_gen_args& g, double* ev, pf_ctx& cx) {
  pf_cnt cnt;  // scratch: generation does not count clamps
  pf_cnt_init(cnt);
  return pf_eval_event(ev, g.P, g.S, g.C, cx, cnt);
}

// generate.hpp:47-63: max over the midpoint grid of raw / norm (last
// dimension fastest; the max is order-free so any traversal gives the same).
extern "C" __global__ void __launch_bounds__(PF_GEN_THREADS) pf_gen_max_kernel(const __grid_constant__ pf_gen_args g) {
  pf_math_init();  // the exp table in shared memory
  double best = 0.0;
  pf_u64 err_key = ~0ull;
  for (pf_u64 flat = (pf_u64)blockIdx.x * blockDim.x + threadIdx.x; flat < g.total;
       flat += (pf_u64)gridDim.x * blockDim.x) {
    double ev[PF_NCOLS];
#pragma unroll
    for (int q = 0; q < PF_NCOLS; ++q) ev[q] = 0.0;
    pf_u64 rem = flat;
    for (int d = g.dims - 1; d >= 0; --d) {
      const pf_u64 k = rem % g.points;
      rem /= g.points;
      ev[g.cols[d]] = __dadd_rn(g.lo[d], __dmul_rn((double)k + 0.5, g.h[d]));
    }
    pf_ctx cx;
    cx.err = 0;
    const double v = pf_gen_density(g, ev, cx);
    if (cx.err) {
      const pf_u64 key = (flat << 24) | cx.err;
      err_key = key < err_key ? key : err_key;
    } else if (v > best) {
      best = v;  // NaN never compares greater (generate.hpp:61)
    }
  }
  pf_u64 bits = (pf_u64)__double_as_longlong(best);  // non-negative: integer order = value order
  for (int o = 16; o > 0; o >>= 1) {
    const pf_u64 ob = __shfl_xor_sync(0xffffffffu, bits, o);
    const pf_u64 oe = __shfl_xor_sync(0xffffffffu, err_key, o);
    bits = ob > bits ? ob : bits;
    err_key = oe < err_key ? oe : err_key;
  }
  if ((threadIdx.x & 31) == 0) {
    if (bits) atomicMax(&g.rec[0], bits);
    if (err_key != ~0ull) atomicMin(&g.rec[1], err_key);
  }
}

__device__ __forceinline__ pf_u64 pf_mt_twist(pf_u64 a, pf_u64 b, pf_u64 c) {
  const pf_u64 y = (a & 0xFFFFFFFF80000000ull) | (b & 0x7FFFFFFFull);
  return c ^ (y >> 1) ^ ((y & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
}

// tempering + ToyRng::uniform (generate.hpp:22), applied by the consumers
__device__ __forceinline__ double pf_mt_uniform(pf_u64 y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return (double)(y >> 11) * 0x1.0p-53;
}

// `rounds` twists of the stream; the raw (untempered) words of round r go to
// u[312 r ..].  Thread t < 156 owns the state pair (x[t], x[t + 156]):
//   x'[t]       = x[t + 156] ^ twist(x[t], x[t + 1])
//   x'[t + 156] = x'[t] ^ twist(x[t + 156], x[t + 157])   (x[312] = x'[0])
// so a round needs only the successor's old pair, exchanged through
// double-buffered shared memory: two barriers per 312 words.  (A one-barrier
// variant, where thread 155 recomputes x'[156] itself, and a one-warp
// shuffle variant both measured slower: the twist's 64-bit integer chain,
// not the barrier, sets the round time.)
extern "C" __global__ void __launch_bounds__(160) pf_mt_kernel(const __grid_constant__ pf_gen_args g) {
  __shared__ pf_u64 sa[2][PF_MT_M + 1], sb[2][PF_MT_M + 1];
  const int t = threadIdx.x;
  const bool own = t < PF_MT_M;
  pf_u64 a = own ? g.mt[t] : 0ull, b = own ? g.mt[t + PF_MT_M] : 0ull;
  if (own) {
    sa[0][t] = a;
    sb[0][t] = b;
  }
  if (t == 0) sa[0][PF_MT_M] = b;  // x[156] is thread 0's second word
  __syncthreads();
  pf_u64* out = (pf_u64*)g.u;
  int cur = 0;
  for (pf_u64 r = 0; r < g.rounds; ++r) {
    pf_u64* o = out + r * PF_MT_N;
    pf_u64 n1 = 0ull;
    if (own) {
      n1 = pf_mt_twist(a, sa[cur][t + 1], b);
      sa[cur ^ 1][t] = n1;
      o[t] = n1;
    }
    __syncthreads();
    if (own) {
      const pf_u64 bn = t + 1 < PF_MT_M ? sb[cur][t + 1] : sa[cur ^ 1][0];
      const pf_u64 n2 = pf_mt_twist(b, bn, n1);
      sb[cur ^ 1][t] = n2;
      if (t == 0) sa[cur ^ 1][PF_MT_M] = n2;
      o[t + PF_MT_M] = n2;
      a = n1;
      b = n2;
    }
    cur ^= 1;
    __syncthreads();
  }
  if (own) {
    g.mt[t] = a;
    g.mt[t + PF_MT_M] = b;
  }
}

// Jump-ahead draw: block k writes words [u_off + k J, u_off + (k + 1) J) of
// the batch, starting from the window T^(k J)(base) (T: the generator's
// one-word window map; base = g.mt, a window in the image of T).  The start
// window is g_k(T) base with g_k = x^(k J) mod phi (tools/gen_mt_jump.py),
// evaluated by Horner over 156 coefficients at a time:
//   acc <- T^156(acc) ^ sum_m g_(i-m) T^(155-m)(base),
// where T^156 is one dependency-free half-twist and T^j(base) is the window
// of base's own stream at offset j (<= 155, so 467 words of it suffice).
// Then the block twists its window J / 312 times like pf_mt_kernel.  The last
// block leaves the window after the batch in g.mt_next.
extern "C" __global__ void __launch_bounds__(320) pf_mt_jump_kernel(const __grid_constant__ pf_gen_args g) {
  __shared__ pf_u64 bs[PF_MT_N + PF_MT_M];    // base stream, words 0 .. 467
  __shared__ pf_u64 acc[2][PF_MT_N];
  __shared__ pf_u64 sa[2][PF_MT_M + 1], sb[2][PF_MT_M + 1];
  const int t = threadIdx.x;
  const int k = blockIdx.x;
  for (int i = t; i < PF_MT_N; i += blockDim.x) {
    bs[i] = g.mt[i];
    acc[0][i] = 0ull;
  }
  __syncthreads();
  if (t < PF_MT_M) bs[PF_MT_N + t] = pf_mt_twist(bs[t], bs[t + 1], bs[t + PF_MT_M]);
  __syncthreads();
  const pf_u64* gk = g.jpoly + (pf_u64)k * PF_MT_N;
  int cur = 0;
  for (int i0 = 128 * PF_MT_M - 1; i0 >= 0; i0 -= PF_MT_M) {  // 19968 >= deg phi + 1
    // coefficients i0 - 155 .. i0: bits of gk[] (uniform across the block)
    const int lo = i0 - (PF_MT_M - 1);
    pf_u64 w0 = gk[lo >> 6], w1 = (lo >> 6) + 1 < PF_MT_N ? gk[(lo >> 6) + 1] : 0ull,
           w2 = (lo >> 6) + 2 < PF_MT_N ? gk[(lo >> 6) + 2] : 0ull,
           w3 = (lo >> 6) + 3 < PF_MT_N ? gk[(lo >> 6) + 3] : 0ull;
    const int sh = lo & 63;
    if (sh) {  // bits lo .. lo + 155 into (w0, w1, w2) from bit 0
      w0 = (w0 >> sh) | (w1 << (64 - sh));
      w1 = (w1 >> sh) | (w2 << (64 - sh));
      w2 = (w2 >> sh) | (w3 << (64 - sh));
    }
    if (t < PF_MT_N) {
      const pf_u64* A = acc[cur];
      pf_u64 v = t < PF_MT_M ? A[t + PF_MT_M] : pf_mt_twist(A[t - PF_MT_M], A[t - PF_MT_M + 1], A[t]);
      // bit b of (w0, w1, w2) is coefficient lo + b = i0 - m with m = 155 - b:
      // window offset 155 - m = b.  Branch-free and unrolled: the loads do
      // not depend on the bits, so they pipeline (a set-bit loop serialises
      // on each load's latency and measured 6x slower)
      pf_u64 x0 = 0ull, x1 = 0ull;
#pragma unroll 16
      for (int b = 0; b < 64; ++b) {
        x0 ^= ((w0 >> b) & 1ull) ? bs[b + t] : 0ull;
        x1 ^= ((w1 >> b) & 1ull) ? bs[b + 64 + t] : 0ull;
      }
#pragma unroll 14
      for (int b = 0; b < PF_MT_M - 128; ++b) x0 ^= ((w2 >> b) & 1ull) ? bs[b + 128 + t] : 0ull;
      v ^= x0 ^ x1;
      acc[cur ^ 1][t] = v;
    }
    cur ^= 1;
    __syncthreads();
  }
  // segment k: J words from the window acc[cur] (two-phase twists, as pf_mt_kernel)
  const bool own = t < PF_MT_M;
  pf_u64 a = own ? acc[cur][t] : 0ull, b = own ? acc[cur][t + PF_MT_M] : 0ull;
  int c2 = 0;
  if (own) {
    sa[0][t] = a;
    sb[0][t] = b;
  }
  if (t == 0) sa[0][PF_MT_M] = b;
  __syncthreads();
  pf_u64* out = (pf_u64*)g.u + g.u_off + (pf_u64)k * g.jump_words;
  const pf_u64 rounds = g.jump_words / PF_MT_N;
  for (pf_u64 r = 0; r < rounds; ++r) {
    pf_u64* o = out + r * PF_MT_N;
    pf_u64 n1 = 0ull;
    if (own) {
      n1 = pf_mt_twist(a, sa[c2][t + 1], b);
      sa[c2 ^ 1][t] = n1;
      o[t] = n1;
    }
    __syncthreads();
    if (own) {
      const pf_u64 bn = t + 1 < PF_MT_M ? sb[c2][t + 1] : sa[c2 ^ 1][0];
      const pf_u64 n2 = pf_mt_twist(b, bn, n1);
      sb[c2 ^ 1][t] = n2;
      if (t == 0) sa[c2 ^ 1][PF_MT_M] = n2;
      o[t + PF_MT_M] = n2;
      a = n1;
      b = n2;
    }
    c2 ^= 1;
    __syncthreads();
  }
  if (k == (int)gridDim.x - 1 && own) {
    g.mt_next[t] = a;
    g.mt_next[t + PF_MT_M] = b;
  }
}

// Candidate c of the batch: box coordinates from its first `dims` uniforms
// (generate.hpp:70-71), then its density and accept test (:72-78).
__device__ __forceinline__ void pf_gen_candidate(const pf_gen_args& g, pf_u64 c, double* ev) {
#pragma unroll
  for (int q = 0; q < PF_NCOLS; ++q) ev[q] = 0.0;
  const pf_u64* uc = (const pf_u64*)g.u + c * (pf_u64)(g.dims + 1);
  for (int d = 0; d < g.dims; ++d)
    ev[g.cols[d]] = __dadd_rn(g.lo[d], __dmul_rn(g.span[d], pf_mt_uniform(uc[d])));
}

__device__ __forceinline__ pf_u32 pf_gen_block_sum(pf_u32 v, pf_u32* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
  __syncthreads();
  pf_u32 s = 0;
  for (int w = 0; w < PF_GEN_THREADS / 32; ++w) s += sh[w];
  return s;
}

extern "C" __global__ void __launch_bounds__(PF_GEN_THREADS) pf_gen_eval_kernel(const __grid_constant__ pf_gen_args g) {
  __shared__ pf_u32 sh[PF_GEN_THREADS / 32];
  pf_math_init();  // the exp table in shared memory
  const pf_u64 base = (pf_u64)blockIdx.x * PF_GEN_SEGMENT;
  pf_u32 accepted = 0;
  pf_u64 err_key = ~0ull, fail = ~0ull;
  for (int j = 0; j < PF_GEN_PER_THREAD; ++j) {
    const pf_u64 c = base + (pf_u64)j * PF_GEN_THREADS + threadIdx.x;
    if (c >= g.n_cand) break;
    double ev[PF_NCOLS];
    pf_gen_candidate(g, c, ev);
    pf_ctx cx;
    cx.err = 0;
    const double density = pf_gen_density(g, ev, cx);
    const double ua = pf_mt_uniform(((const pf_u64*)g.u)[c * (pf_u64)(g.dims + 1) + g.dims]);
    unsigned char f = 0;
    if (cx.err) {
      const pf_u64 key = (c << 24) | cx.err;
      err_key = key < err_key ? key : err_key;
    } else if (density > g.envelope) {
      g.fail_density[c] = density;
      fail = c < fail ? c : fail;
    } else if (__dmul_rn(ua, g.envelope) < density) {
      f = 1;
      ++accepted;
    }
    g.flags[c] = f;
  }
  if (err_key != ~0ull) atomicMin(&g.rec[1], err_key);
  if (fail != ~0ull) atomicMin(&g.rec[2], fail);
  const pf_u32 s = pf_gen_block_sum(accepted, sh);
  if (threadIdx.x == 0) g.block_count[blockIdx.x] = s;
}

// one block: exclusive scan of the per-block counts, batch total into rec[4]
extern "C" __global__ void __launch_bounds__(1024) pf_gen_scan_kernel(const __grid_constant__ pf_gen_args g) {
  __shared__ pf_u64 warp_tot[32];
  __shared__ pf_u64 carry;
  const int n = (int)((g.n_cand + PF_GEN_SEGMENT - 1) / PF_GEN_SEGMENT);
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (t == 0) carry = 0;
  __syncthreads();
  for (int b0 = 0; b0 < n; b0 += 1024) {
    const int b = b0 + t;
    const pf_u64 v = b < n ? g.block_count[b] : 0u;
    pf_u64 x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const pf_u64 y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[w] = x;
    __syncthreads();
    if (w == 0) {
      pf_u64 s = warp_tot[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const pf_u64 y = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += y;
      }
      warp_tot[lane] = s;  // inclusive over warps
    }
    __syncthreads();
    const pf_u64 excl = carry + (w ? warp_tot[w - 1] : 0ull) + x - v;
    if (b < n) g.block_base[b] = (pf_u32)excl;
    __syncthreads();
    if (t == 0) carry += warp_tot[31];
    __syncthreads();
  }
  if (t == 0) g.rec[4] = carry;
}

// accepted candidates in stream order -> out[col][out_base + rank], rank <
// remaining; the candidate holding rank remaining - 1 is recorded (rec[3])
extern "C" __global__ void __launch_bounds__(PF_GEN_THREADS) pf_gen_scatter_kernel(const __grid_constant__ pf_gen_args g) {
  __shared__ pf_u32 wsum[PF_GEN_THREADS / 32];
  const pf_u64 base = (pf_u64)blockIdx.x * PF_GEN_SEGMENT;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  pf_u64 rank0 = g.block_base[blockIdx.x];
  if (rank0 >= g.remaining) return;
  for (int j = 0; j < PF_GEN_PER_THREAD; ++j) {
    const pf_u64 c = base + (pf_u64)j * PF_GEN_THREADS + threadIdx.x;
    const bool acc = c < g.n_cand && g.flags[c];
    const pf_u32 m = __ballot_sync(0xffffffffu, acc);
    if (lane == 0) wsum[w] = __popc(m);
    __syncthreads();
    pf_u32 before = 0, all = 0;
    for (int q = 0; q < PF_GEN_THREADS / 32; ++q) {
      before += q < w ? wsum[q] : 0u;
      all += wsum[q];
    }
    const pf_u64 rank = rank0 + before + __popc(m & ((1u << lane) - 1u));
    if (acc && rank < g.remaining) {
      const pf_u64* uc = (const pf_u64*)g.u + c * (pf_u64)(g.dims + 1);
      for (int d = 0; d < g.dims; ++d)
        g.out[(pf_u64)d * g.out_stride + g.out_base + rank] =
            __dadd_rn(g.lo[d], __dmul_rn(g.span[d], pf_mt_uniform(uc[d])));
      if (rank == g.remaining - 1) g.rec[3] = c;
    }
    rank0 += all;
    __syncthreads();
  }
}
