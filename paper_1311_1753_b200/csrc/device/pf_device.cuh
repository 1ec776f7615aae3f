// pf_device.cuh — device library shared by every generated evaluator.
//
// Compiled at model-creation time by NVRTC for sm_100a together with the
// per-model generated code (codegen.cpp).  Contents:
//   * double-double (DD) arithmetic: replaces the x87 `long double`
//     accumulators of the reference (engine.hpp:57-68, pdf.hpp:163-175);
//   * fixed-shape warp/block reductions: summation order is a pure function
//     of the input length, never of scheduling (engine.hpp:72-78);
//   * error/status records standing in for parfit::Error (errors.hpp);
//   * scalar math entry points used by the node kernels.
#pragma once

typedef unsigned long long pf_u64;
typedef long long pf_i64;
typedef unsigned int pf_u32;

// PF_CHECKS (PFB200_DEFINES=PF_CHECKS): device-side bounds checks on every
// TMA copy, shared-memory stage, task and record index -- the substitute for
// compute-sanitizer, which this GPU pool does not allow; a failed check traps
// (the call then fails with a CUDA error instead of reading out of bounds)
#ifdef PF_CHECKS
#define PF_CHECK(cond)                                                                       \
  do {                                                                                      \
    if (!(cond)) {                                                                          \
      printf("PF_CHECK failed: %s (block %d thread %d)\n", #cond, blockIdx.x, threadIdx.x); \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define PF_CHECK(cond) \
  do {                 \
  } while (0)
#endif

#define PF_THREADS 256
#define PF_FINAL_THREADS 1024
#define PF_LOG_FLOOR 1e-300   // engine.hpp:50 kLogFloor
#define PF_CHISQ_EPS 1e-9     // engine.hpp:51 kChiSqEps
#define PF_MAX_BOX 8
#define PF_MAX_LEVELS 14
#define PF_MAX_INLINE 64  // parameters passed inline in the kernel arguments

// error codes, mirrored by engine.cpp's message table
#define PF_E_NONPOS_SIGMA 1   // pdf.hpp:256-257
#define PF_E_NONPOS_WIDTH 2   // pdf.hpp:285
#define PF_E_OUT_OF_DOMAIN 3  // pdf.hpp:443-444
#define PF_E_ZERO_INTEGRAL 4  // pdf.hpp:186-187
#define PF_E_NONPOS_ENDPOINT 5 // ArgusPdf m0 <= 0
#define PF_E_GROUP_TIMEOUT 6   // a peer's record never arrived (exchange group)
#define PF_E_NONPOS_LIFETIME 7 // TddpPdf tau <= 0
#define PF_COMP_ALL4 8         // pf_task.comp: a TddpPdf Dalitz task returning its four components
#define PF_GROUP_MAX 16        // ranks of a peer-memory exchange group (engine.hpp kMaxGroup)
#define PF_MAX_BATCH 16        // parameter sets per launch (engine.hpp kMaxBatch)

struct pf_dd {
  double hi, lo;
};

// Per-parameter-set call record (one per k of a batch).  Initialised by the
// pre kernel of every call; copied back to the host after the call.
struct pf_krec {
  pf_u64 floor_count;        // events floored at 1e-300 (engine.hpp:190-193)
  pf_u64 first_nonfinite;    // min global index of a non-finite term (engine.hpp:210-216)
  pf_u64 first_event_error;  // min (index << 24 | node << 8 | code) raised in the event pass
  pf_u32 norm_error;         // min (node << 8 | code) raised while normalising
  pf_u32 arrive[PF_MAX_LEVELS + 1];  // last-block arrival counters
  long long fx[6];           // exact superaccumulator of the metric (pf_fx_add)
};

struct pf_task {  // one midpoint sum: node, n points per box dimension
  int node, n, dims, first_block;
  int n_blocks, comp, fine, level;  // comp: component of a TddpPdf grid (-1: a plain midpoint sum)
  pf_u64 points, per_block;
  double lo[PF_MAX_BOX];
  double h[PF_MAX_BOX];
  double vol;
  double pad;  // 192 B: a whole number of 16-byte units (TMA bulk copies)
};

// Per-call result record, written by the device straight into mapped
// (zero-copy) host memory: no memcpy nodes in the per-call graph.
struct pf_out {
  double result;  // correctly rounded metric of this shard
  pf_u64 floor_count, first_nonfinite, first_event_error;
  pf_u32 norm_error, pad;  // pad: completion sequence number (pf_publish)
  long long fx[6];  // exact digits (combined across shards on the host)
  pf_u64 check;     // pf_out_check of every field above: the record is complete
};

// The record is published with uncached system-scope stores and no
// system-scope fence (which costs ~1.5 us at the end of every call,
// pf_finalize_warp0): the host accepts it once `pad` carries the call's
// sequence number AND `check` matches every field, so a record read while
// its stores are still landing is retried (host twin: engine.cpp out_check).
__device__ __forceinline__ pf_u64 pf_mix64(pf_u64 h, pf_u64 v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h ^= h >> 31;
  h *= 0xbf58476d1ce4e5b9ull;
  return h ^ (h >> 29);
}
__device__ __forceinline__ pf_u64 pf_out_check(const pf_out& o) {
  pf_u64 h = 0x243f6a8885a308d3ull;
  h = pf_mix64(h, (pf_u64)__double_as_longlong(o.result));
  h = pf_mix64(h, o.floor_count);
  h = pf_mix64(h, o.first_nonfinite);
  h = pf_mix64(h, o.first_event_error);
  h = pf_mix64(h, ((pf_u64)o.norm_error << 32) | o.pad);
  for (int i = 0; i < 6; ++i) h = pf_mix64(h, (pf_u64)o.fx[i]);
  return h;
}

struct pf_args {
  const double* hP;     // host-mapped parameters (K x PF_NP)
  pf_out* hout;         // host-mapped results (K)
  double* hnorms;       // DEVICE: norms of the last call without a norm error (3 n_nodes)
  pf_u64* hclamp;       // (unused: the host reads the device counters on demand)
  int n_nodes;
  int fuse_final;       // K == 1: the last event block runs the final tree
  int n_levels;
  int tddp_tab;         // norm kernel: a TddpPdf column table in dynamic shared memory (pf_tddp_cols)
  const double* data;   // column-major shard: data[col * col_stride + e]
  pf_u64 col_stride;
  pf_u64 n_local;       // events (bins) in this shard
  pf_u64 event_offset;  // global index of local event 0
  int n_chunks;         // chunks in this shard
  int K;                // parameter sets in this call
  int level;            // normalisation level of this launch
  int n_tasks;
  const double* P;      // K x PF_NP parameters
  double* S;            // K x PF_SS per-call state (norms, derived constants)
  const double* C;      // model constants (ranges, boundaries, ...)
  const pf_task* tasks; // norm tasks of this level
  pf_dd* partials;      // K x n_chunks (event pass) / K x n_partials (norms)
  pf_krec* rec;         // K records
  pf_u64* clamp;        // cumulative PolynomialPdf clamp counters per node
  double total_content; // binned: N_tot (engine.hpp:153)
  pf_u32* done;         // [finished-block counter (self-resetting), per-k completion sequence]
  long long* fxbins;    // K x PF_FX_BINS x 16: binned block digits (self-resetting)
  long long* dpart;     // K x 8 (device): exact digits, norm error, event-error flag of this call
  long long** peers;    // peer-memory exchange group: every rank's receive buffer (null: none)
  int gworld;           // ranks in the group
  int grank;            // this rank
  int npin;             // K = 1: parameters passed inline (pin[0..npin))
  int s_smem;            // S staged in the event pass's shared memory (models with conv tables)
  long long* big;       // K x PF_BIG_STRIDE: wide accumulator of chunk sums >= 2^62 (pf_big_add)
  pf_u32* ticket;       // (unused: reserved)
  int fused;            // 1: this launch is the single fused kernel (setup in every CTA)
  int nwa;              // fused pass: active warps (static balanced schedule)
  int kpw;              // fused pass: chunks per active warp (at most)
  pf_u32 gmask;         // K = 1 inline: bit 0 = count this call's grid clamps
  const pf_u32* hmask;  // host-mapped: bit k = parameter set k recomputes its norms
                        // (the reference's fingerprint cache, pdf.hpp:111-123)
  double pin[PF_MAX_INLINE];
};

// ----------------------------------------------------------------------------
// error/counter context carried through one evaluation
#ifdef PF_CONV_TRACE_FULL
__device__ unsigned pf_conv_full_count[2];  // experiment: full-Q fallbacks, windows not summed
#endif

struct pf_ctx {
  pf_u32 err;  // (node << 8) | code of the first error, 0 when none
  // the event pass's warp scratch (PF_CONV_SHARED) and the mask of the lanes
  // evaluating an event together; null elsewhere: per-lane sums
  double* scr = nullptr;
  pf_u32 mask = 0u;
};

// An index as a double, exactly, without the I2F conversion pipe: below 2^32
// the integer is spliced into the mantissa of 2^52 and 2^52 subtracted
// (exact); the grid walks convert one index per point (the setup's points
// phase was bound on I2F.F64.U64).
__device__ __forceinline__ double pf_idx2d(pf_u64 i) {
  if (i < 0x100000000ull) return __hiloint2double(0x43300000, (int)(pf_u32)i) - 4503599627370496.0;
  return (double)i;
}

__device__ __forceinline__ void pf_fail(pf_ctx& cx, int node, int code) {
  if (!cx.err) cx.err = ((pf_u32)node << 8) | (pf_u32)code;
}

// Richardson combination of a node's (coarse, fine) midpoint sums
// (pdf.hpp:178-188) into S: norm, error estimate, 1 / norm; the sums are kept
// (PF_SUMS_BASE) for AddPdf nodes normalised from their children's sums.
// Returns true when the integral is zero or non-finite (pdf.hpp:186-187).
__device__ __forceinline__ bool pf_finish_norm_s(double* S, int node, double coarse, double fine) {
  const double norm = fine + (fine - coarse) / 3.0;
  const double err = fabs(fine - coarse) / 3.0;
  S[3 * node + 0] = norm;
  S[3 * node + 1] = err;
  S[3 * node + 2] = 1.0 / norm;
#ifdef PF_SUMS_BASE
  S[PF_SUMS_BASE + 2 * node] = coarse;
  S[PF_SUMS_BASE + 2 * node + 1] = fine;
#endif
  return !(norm > 0.0) || !isfinite(norm);
}

// Does parameter set k count the clamps met on the normalisation grids?  The
// reference recomputes norms only when the parameters' hash changed since the
// last refresh (pdf.hpp:111-123, hash_params :40-51); this engine recomputes
// every call, so it counts the grid clamps only when the reference would.
__device__ __forceinline__ bool pf_grid_counts(const pf_args& a, int k) {
  const pf_u32 m = a.npin ? a.gmask : __ldcv(a.hmask);
  return (m >> k) & 1u;
}

__device__ __forceinline__ void pf_finish_norm_cx(double* S, pf_ctx& cx, int node, double coarse,
                                                  double fine) {
  if (pf_finish_norm_s(S, node, coarse, fine)) pf_fail(cx, node, PF_E_ZERO_INTEGRAL);
}

// ----------------------------------------------------------------------------
// double-double arithmetic (Knuth TwoSum / Dekker FastTwoSum).  Only adds are
// involved, so FMA contraction cannot perturb them.
__device__ __forceinline__ pf_dd pf_two_sum(double a, double b) {
  double s = a + b;
  double bb = s - a;
  double e = (a - (s - bb)) + (b - bb);
  pf_dd r;
  r.hi = s;
  r.lo = e;
  return r;
}

__device__ __forceinline__ pf_dd pf_fast_two_sum(double a, double b) {
  double s = a + b;
  pf_dd r;
  r.hi = s;
  r.lo = b - (s - a);
  return r;
}

__device__ __forceinline__ pf_dd pf_dd_add(pf_dd a, pf_dd b) {
  pf_dd s = pf_two_sum(a.hi, b.hi);
  pf_dd t = pf_two_sum(a.lo, b.lo);
  double lo = s.lo + t.hi;
  pf_dd u = pf_fast_two_sum(s.hi, lo);
  lo = u.lo + t.lo;
  return pf_fast_two_sum(u.hi, lo);
}

__device__ __forceinline__ pf_dd pf_dd_add_d(pf_dd a, double b) {
  pf_dd s = pf_two_sum(a.hi, b);
  double lo = s.lo + a.lo;
  return pf_fast_two_sum(s.hi, lo);
}

__device__ __forceinline__ pf_dd pf_dd_zero() {
  pf_dd z;
  z.hi = 0.0;
  z.lo = 0.0;
  return z;
}

__device__ __forceinline__ double pf_dd_to_double(pf_dd a) { return a.hi + a.lo; }

__device__ __forceinline__ pf_dd pf_shfl_down_dd(pf_dd v, int d) {
  pf_dd r;
  r.hi = __shfl_down_sync(0xffffffffu, v.hi, d);
  r.lo = __shfl_down_sync(0xffffffffu, v.lo, d);
  return r;
}

// Fixed-shape reduction of n DD values by ONE warp (all 32 lanes must call):
// lane l sums the contiguous run [l*per, min((l+1)*per, n)) sequentially,
// then a shuffle tree (16, 8, 4, 2, 1).  Result valid in lane 0.
__device__ __forceinline__ pf_dd pf_warp_reduce_runs(const pf_dd* v, int n) {
  const int lane = threadIdx.x & 31;
  const int per = (n + 31) >> 5;
  pf_dd acc = pf_dd_zero();
  const int lo = lane * per;
  const int hi = min(lo + per, n);
  for (int i = lo; i < hi; ++i) acc = pf_dd_add(acc, v[i]);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    pf_dd o = pf_shfl_down_dd(acc, d);
    acc = pf_dd_add(acc, o);
  }
  return acc;
}

// Fixed-shape block reduction (any blockDim multiple of 32, <= 1024): a
// shuffle tree inside every warp, then one over the warp results.  All
// threads must call; the result is valid in thread 0.  sm: >= 32 slots.
__device__ __forceinline__ pf_dd pf_block_reduce(pf_dd v, pf_dd* sm) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) v = pf_dd_add(v, pf_shfl_down_dd(v, d));
  __syncthreads();  // sm may still be read by a previous call
  if (lane == 0) sm[warp] = v;
  __syncthreads();
  if (warp == 0) {
    v = lane < nw ? sm[lane] : pf_dd_zero();
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v = pf_dd_add(v, pf_shfl_down_dd(v, d));
  }
  return v;
}

// ----------------------------------------------------------------------------
// Exact fixed-point superaccumulator: value = sum_i d_i 2^(32 i - 128), six
// signed 64-bit digit accumulators, every contribution < 2^32 in magnitude
// per digit.  Adding a double is exact for |x| in [2^-128, 2^64) (bits below
// 2^-128 are truncated toward zero); additions commute, so the total does not
// depend on order, chunking or the number of devices, and the final rounding
// to double is correct (pf_fx_round).  The reference sums in x87 long double
// (engine.hpp:57-87); this is at least as accurate.
#define PF_FX_DIGITS 6

__device__ __forceinline__ void pf_fx_add(long long* acc, double x) {
  if (x == 0.0) return;
  const pf_u64 bits = (pf_u64)__double_as_longlong(x);
  const int be = (int)((bits >> 52) & 0x7ff);
  if (be == 0x7ff || be >= 1023 + 63) {  // non-finite or |x| >= 2^63: poison the sum
    atomicAdd((unsigned long long*)(acc + PF_FX_DIGITS - 1), 0x4000000000000000ull);
    return;
  }
  pf_u64 m = bits & 0xfffffffffffffull;
  int e;
  if (be == 0) {
    e = -1074;
  } else {
    m |= 0x10000000000000ull;
    e = be - 1075;
  }
  int p = e + 128;  // bit position of m's LSB above 2^-128
  if (p < 0) {
    if (p <= -53) return;
    m >>= -p;
    p = 0;
  }
  const int q = p >> 5, s = p & 31;
  // m << s spans up to 85 bits: three 32-bit digits starting at q
  const pf_u64 d0 = (m << s) & 0xffffffffull;
  const pf_u64 d1 = (s ? (m >> (32 - s)) : (m >> 32)) & 0xffffffffull;
  const pf_u64 d2 = s ? (m >> (64 - s)) : 0ull;
  const bool neg = (bits >> 63) != 0;
  const long long v[3] = {(long long)d0, (long long)d1, (long long)d2};
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (v[i] && q + i < PF_FX_DIGITS)
      atomicAdd((unsigned long long*)(acc + q + i), (unsigned long long)(neg ? -v[i] : v[i]));
}

// Register-resident superaccumulator of one lane (same digit layout): exact
// integer adds with branch-free digit placement; no atomics, no shuffles.
struct pf_fxl {
  long long d[PF_FX_DIGITS];
};

__device__ __forceinline__ void pf_fxl_add(pf_fxl& A, double x) {
  const pf_u64 bits = (pf_u64)__double_as_longlong(x);
  const int be = (int)((bits >> 52) & 0x7ff);
  const bool poison = be >= 1023 + 63;  // non-finite or |x| >= 2^63
  pf_u64 m = (bits & 0xfffffffffffffull) | (be ? 0x10000000000000ull : 0ull);
  int p = (be ? be : 1) - 1075 + 128;  // LSB position above 2^-128
  if (p < 0) {
    m = p <= -53 ? 0ull : (m >> -p);
    p = 0;
  }
  const int q = p >> 5, s = p & 31;
  const long long d0 = (long long)((m << s) & 0xffffffffull);
  const long long d1 = (long long)((s ? (m >> (32 - s)) : (m >> 32)) & 0xffffffffull);
  const long long d2 = (long long)(s ? (m >> (64 - s)) : 0ull);
  const long long sg = (bits >> 63) ? -1ll : 1ll;
#pragma unroll
  for (int i = 0; i < PF_FX_DIGITS; ++i) {
    const long long v = (i == q ? d0 : 0ll) + (i == q + 1 ? d1 : 0ll) + (i == q + 2 ? d2 : 0ll);
    A.d[i] += sg * v;
  }
  if (poison) A.d[PF_FX_DIGITS - 1] += 0x4000000000000000ll;
}

// Wide accumulator for the rare chunk sums |x| >= 2^62 (chi-squared far from
// the data: the reference's long-double sum has no such range limit,
// engine.hpp:57-87): value = sum_i b_i 2^(32 i), exact for every finite
// |x| >= 2^52.  Global atomics, out of line: never on the common path.
// Per parameter set PF_BIG_STRIDE words: [0, PF_BIG_DIGITS) accumulating
// digits and PF_BIG_COUNT their add count (both reset by the finalizing warp),
// [PF_BIG_SNAP, +PF_BIG_DIGITS) the last call's digits and PF_BIG_SNAP_COUNT
// its count, which the host reads when the published result is NaN.
#define PF_BIG_DIGITS 34
#define PF_BIG_COUNT 40
#define PF_BIG_SNAP 64
#define PF_BIG_SNAP_COUNT 104
#define PF_BIG_STRIDE 128

__device__ __noinline__ void pf_big_add(long long* big, double x) {
  const pf_u64 bits = (pf_u64)__double_as_longlong(x);
  const pf_u64 m = (bits & 0xfffffffffffffull) | 0x10000000000000ull;
  const int p = (int)((bits >> 52) & 0x7ff) - 1075;  // LSB position, >= 10 here
  const int q = p >> 5, s = p & 31;
  const pf_u64 d0 = (m << s) & 0xffffffffull;
  const pf_u64 d1 = (s ? (m >> (32 - s)) : (m >> 32)) & 0xffffffffull;
  const pf_u64 d2 = s ? (m >> (64 - s)) : 0ull;
  const bool neg = (bits >> 63) != 0;
  const long long v[3] = {(long long)d0, (long long)d1, (long long)d2};
#pragma unroll
  for (int i = 0; i < 3; ++i)
    if (v[i]) atomicAdd((unsigned long long*)(big + q + i), (unsigned long long)(neg ? -v[i] : v[i]));
  atomicAdd((unsigned long long*)(big + PF_BIG_COUNT), 1ull);
}

// a chunk sum into the lane's accumulator, or (|x| >= 2^62, finite) the wide one
__device__ __forceinline__ void pf_fxl_add_w(pf_fxl& A, double x, long long* big) {
  const double ax = fabs(x);
  if (ax >= 0x1p62 && ax <= 1.7976931348623157e308)
    pf_big_add(big, x);
  else
    pf_fxl_add(A, x);
}

// The same exact add into a lane's six digits kept in SHARED memory
// (d[i * stride]): the digit position is an address, not a chain of selects
// over six registers (the fused pass adds one chunk value per lane per chunk;
// this is about a third of pf_fxl_add's instructions)
__device__ __forceinline__ void pf_fxs_add(long long* d, int stride, double x) {
  const pf_u64 bits = (pf_u64)__double_as_longlong(x);
  const int be = (int)((bits >> 52) & 0x7ff);
  if (be >= 1023 + 63) {  // non-finite or |x| >= 2^63: poison the sum
    d[(PF_FX_DIGITS - 1) * stride] += 0x4000000000000000ll;
    return;
  }
  pf_u64 m = (bits & 0xfffffffffffffull) | (be ? 0x10000000000000ull : 0ull);
  int p = (be ? be : 1) - 1075 + 128;  // LSB position above 2^-128
  if (p < 0) {
    m = p <= -53 ? 0ull : (m >> -p);
    p = 0;
  }
  const int q = p >> 5, s = p & 31;
  const long long sg = (bits >> 63) ? -1ll : 1ll;
  const long long d0 = (long long)((m << s) & 0xffffffffull);
  const long long d1 = (long long)((s ? (m >> (32 - s)) : (m >> 32)) & 0xffffffffull);
  const long long d2 = (long long)(s ? (m >> (64 - s)) : 0ull);
  d[q * stride] += sg * d0;  // q <= 5 here (|x| < 2^63, LSB >= 2^-128)
  if (q + 1 < PF_FX_DIGITS) d[(q + 1) * stride] += sg * d1;
  if (q + 2 < PF_FX_DIGITS) d[(q + 2) * stride] += sg * d2;
}

// Warp-wide integer sum of the lanes' accumulators into the global one.
// warp total of the lanes' digits (integer shuffles; exact), valid in lane 0
__device__ __forceinline__ void pf_fxl_warp_sum(pf_fxl& A) {
#pragma unroll
  for (int i = 0; i < PF_FX_DIGITS; ++i) {
    long long v = A.d[i];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_down_sync(0xffffffffu, v, d);
    A.d[i] = v;
  }
}

// Same-address atomics serialise in one L2 slice (~1 op/clk): the event pass
// spreads its blocks' digits over PF_FX_BINS 128-byte slots
#define PF_FX_BINS 32
#define PF_FX_BIN_STRIDE 16

// Correctly rounded double of the accumulator (host twin: pfb::fx_round).
__device__ __forceinline__ double pf_fx_round(const long long* acc) {
  unsigned dig[PF_FX_DIGITS];
  long long carry = 0;
  for (int i = 0; i < PF_FX_DIGITS; ++i) {  // carry-normalise to 32-bit digits
    const long long v = acc[i] + carry;
    dig[i] = (unsigned)(v & 0xffffffffll);
    carry = v >> 32;
  }
  if (carry > 0 || carry < -1) return __longlong_as_double(0x7ff8000000000000ll);  // poisoned
  const bool neg = carry < 0;
  if (neg) {  // magnitude of the 192-bit two's complement value
    unsigned c = 1;
    for (int i = 0; i < PF_FX_DIGITS; ++i) {
      const unsigned long long t = (unsigned long long)(~dig[i]) + c;
      dig[i] = (unsigned)t;
      c = (unsigned)(t >> 32);
    }
  }
  int top = PF_FX_DIGITS - 1;
  while (top >= 0 && dig[top] == 0) --top;
  if (top < 0) return 0.0;
  const int lz = __clz(dig[top]);
  const pf_u64 hi = dig[top];
  const pf_u64 mid = top >= 1 ? dig[top - 1] : 0u;
  const pf_u64 lo = top >= 2 ? dig[top - 2] : 0u;
  bool sticky = false;
  for (int i = top - 3; i >= 0; --i) sticky |= dig[i] != 0;
  // 64-bit window with the leading one at bit 63, the rest into `sticky`
  pf_u64 win = (hi << (32 + lz)) | (mid << lz);
  if (lz) {
    win |= lo >> (32 - lz);
    sticky |= (lo & ((1ull << (32 - lz)) - 1)) != 0;
  } else {
    sticky |= lo != 0;
  }
  pf_u64 mant = win >> 11;  // 53 significant bits
  const pf_u64 rem = win & 0x7ffull;
  if ((rem & 0x400ull) && ((rem & 0x3ffull) || sticky || (mant & 1ull))) ++mant;  // nearest even
  int msb = 32 * top + 31 - lz;
  if (mant >> 53) {
    mant >>= 1;
    ++msb;
  }
  const double r = ldexp((double)mant, msb - 52 - 128);
  return neg ? -r : r;
}

// ----------------------------------------------------------------------------
// scalar math used by the node kernels
//
// pf_exp: table-driven exp.  x = (128 e + j) ln2/128 + r, |r| <= ln2/256;
// exp(x) = 2^e * 2^(j/128) * (1 + expm1(r)) with 2^(j/128) = hi + lo from a
// 128-entry shared-memory table and expm1(r) a degree-5 Taylor polynomial
// (truncation r^6/720 < 6e-19).  One rounding dominates: error ~0.51 ulp,
// 12 FP64 instructions instead of libdevice's ~17.  Branch-free range
// handling: x is clamped to +-1100 (NaN kept) and 2^e applied in two exact
// steps, so underflow to 0 and overflow to inf come out of the last multiply.
#include "pf_exp_table.cuh"

__shared__ double2 pf_exp_tab[128];
#ifdef PF_QFAST
__shared__ __align__(16) double pf_exp2_1024[1024];  // 2^(j/1024) (pf_qfast_terms)
#endif

// every kernel calls this before the first pf_exp (includes __syncthreads)
__device__ __forceinline__ void pf_math_init() {
  for (int i = threadIdx.x; i < 128; i += blockDim.x)
    pf_exp_tab[i] = make_double2(pf_exp_tab_g[2 * i], pf_exp_tab_g[2 * i + 1]);
#ifdef PF_QFAST
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) pf_exp2_1024[i] = pf_exp2_1024_g[i];
#endif
  __syncthreads();
}

__device__ __forceinline__ double pf_exp_core(double x);

__device__ __forceinline__ double pf_exp(double x) {
#ifdef PF_EXP_LIBDEVICE
  return exp(x);
#endif
  // branch-free range handling: the two-step 2^e scaling below is exact for
  // |x| <= 1100 (0 / inf beyond exp's range come out of the final multiply);
  // larger |x| and +-inf are clamped by compare-selects that keep NaN.
  x = x < -1100.0 ? -1100.0 : x;
  x = x > 1100.0 ? 1100.0 : x;
  return pf_exp_core(x);
}

// exp for arguments known to be <= 0 (Gaussian exponents): one clamp fewer
__device__ __forceinline__ double pf_exp_neg(double x) {
#ifdef PF_EXP_LIBDEVICE
  return exp(x);
#endif
  x = x < -1100.0 ? -1100.0 : x;
  return pf_exp_core(x);
}

__device__ __forceinline__ double pf_exp_core(double x) {
  const double kd = fma(x, PF_EXP_INVLN2N, 0x1.8p52);
  const int ki = __double2loint(kd);
  const double k = kd - 0x1.8p52;
  double r = fma(k, -PF_EXP_LN2N_HI, x);
  r = fma(k, -PF_EXP_LN2N_LO, r);
  const double2 t = pf_exp_tab[ki & 127];
  const double r2 = r * r;
  const double q = fma(fma(fma(r, 1.0 / 120.0, 1.0 / 24.0), r, 1.0 / 6.0), r, 0.5);
  const double p = fma(r2, q, r);
  const double s = fma(t.x, p, t.y) + t.x;
  // 2^e in two factors (e in [-1477, 1477]): 2^e1 folded exactly into the
  // exponent field of s (integer add), 2^(e - e1) by the one rounding multiply
  const int e = ki >> 7;
  const int e1 = e >> 1;
  const double sc = __hiloint2double(__double2hiint(s) + (e1 << 20), __double2loint(s));
  return sc * __hiloint2double((e - e1 + 1023) << 20, 0);
}

// F = 1 + e^x for x <= 0: the mixture factor of the log-sum-exp NLL form
// (codegen.cpp emit_event_log), multiplied per lane and logged once per chunk.
// Only F matters, not e^x: below x = -40, e^x < 2^-57 vanishes in 1 + e^x, so
// the exponent is clamped at -60 on the integer pipe instead of clamping x
// (x is finite and |x| < 2^40 whenever the caller keeps F).  Degree-4
// polynomial on the 2^(j/128) table: |r| <= 0.00272, truncation r^5/120 <=
// 1.3e-15 relative in e^x, i.e. < 1.3e-15 absolute in log F per event
// (per-term budget, far inside the 1e-12 relative NLL bar).
// Constants whose low 32 bits are zero become SASS immediates (no registers).
#define PF_F_INVLN2N 0x1.71547p+7            // ~128/ln2: only picks k
#define PF_F_LN2N_HI 0x1.62e42p-8            // 21 significant bits: k * hi exact
#define PF_F_LN2N_LO 0x1.fdf473de6af28p-29   // ln2/128 - hi
__device__ __forceinline__ double pf_one_plus_exp_neg(double x) {
  const double kd = fma(x, PF_F_INVLN2N, 0x1.8p52);
  const int ki = __double2loint(kd);
  const double k = kd - 0x1.8p52;
  double r = fma(k, -PF_F_LN2N_HI, x);
  r = fma(k, -PF_F_LN2N_LO, r);
  const double2 t = pf_exp_tab[ki & 127];
  double q = fma(r, 0x1.55555p-5, 1.0 / 6.0);
  q = fma(q, r, 0.5);
  q = fma(q, r, 1.0);
  const double p = r * q;                    // e^r - 1
  const double s = fma(t.x, p, t.y) + t.x;   // 2^(j/128) e^r, in [0.99, 2.01)
  const int e = max(ki >> 7, -60);
  return 1.0 + __hiloint2double(__double2hiint(s) + (e << 20), __double2loint(s));
}

// A power factor of the log form (codegen.cpp log_factored) is a positive
// normal in [2^-20, 2^21): its log is within 14.6 in magnitude, which bounds
// sum_j pow_j log fac_j per call (pf_stage_post) without a per-event log.
__device__ __forceinline__ bool pf_fac_in_range(double v) {
  return ((unsigned)__double2hiint(v) >> 20) - 1003u < 41u;
}

// running product of power factors: mantissas in [1, 2) multiplied, binary
// exponents summed (so products of any length neither over- nor underflow)
__device__ __forceinline__ void pf_fac_accum(double& m, int& e, double v) {
  const int hi = __double2hiint(v);
  e += (hi >> 20) - 1023;
  m *= __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(v));
}

// ----------------------------------------------------------------------------
// DalitzPlotPdf pieces.  The kinematic boundary and the per-call constants
// are the C oracle's sequence (pf_oracle.c, -ffp-contract=off), explicitly
// rounded, so no event changes side of the boundary; the per-event amplitude
// uses pf_dalitz_res_fast (reciprocals by Newton-refined MUFU seeds), within
// a few ulp of pf_dalitz_res.
struct pf_cplx {
  double re, im;
};

// q^2 of a two-body split of invariant mass^2 s into masses ma, mb, given
// quarter = 1 / (4 s) (shared by every resonance of the channel)
__device__ __forceinline__ double pf_q2(double s, double quarter, double ma, double mb) {
  const double sp = __dadd_rn(ma, mb), sm = __dsub_rn(ma, mb);
  const double v = __dmul_rn(__dmul_rn(__dsub_rn(s, __dmul_rn(sp, sp)), __dsub_rn(s, __dmul_rn(sm, sm))), quarter);
  return v > 0.0 ? v : 0.0;
}

// one resonance: Z B(q)/B(q0) / (m^2 - s - i m Gamma(s)),
// Gamma(s) = G (q/q0)^(2J+1) (m / sqrt s) (B(q)/B(q0))^2, B_1(q)^2 = 1/(1 + R^2 q^2).
// Channel terms: quarter = 1/(4 s), rs = 1/sqrt(s) = sqrt(4 quarter)/2 (one
// division and one root per channel).  Per call (pf_stage_pre): m2 = m^2,
// iq0 = 1/q0, br0 = 1 + R^2 q0^2.
__device__ __forceinline__ pf_cplx pf_dalitz_res(double s, double quarter, double rs, double Z, double m,
                                                 double m2, double G, double iq0, double br0, double mi,
                                                 double mj, double R2, int spin) {
  const double q2 = pf_q2(s, quarter, mi, mj);
  const double x = __dmul_rn(__dsqrt_rn(q2), iq0);
  double bf2 = 1.0, ratio = x, sbf = 1.0;  // (B(q)/B(q0))^2, (q/q0)^(2J+1), B(q)/B(q0)
  if (spin == 1) {
    bf2 = __ddiv_rn(br0, __dadd_rn(1.0, __dmul_rn(R2, q2)));
    ratio = __dmul_rn(__dmul_rn(x, x), x);
    sbf = __dsqrt_rn(bf2);
  }
  const double gs = __dmul_rn(__dmul_rn(__dmul_rn(G, ratio), __dmul_rn(m, rs)), bf2);
  const double a = __dsub_rn(m2, s), b = __dmul_rn(m, gs);
  const double den = __dadd_rn(__dmul_rn(a, a), __dmul_rn(b, b));
  const double f = __ddiv_rn(__dmul_rn(Z, sbf), den);
  pf_cplx r;
  r.re = __dmul_rn(f, a);
  r.im = __dmul_rn(f, b);
  return r;
}

// Fast reciprocal / reciprocal square root: the MUFU 64-bit seeds (about 22
// bits) refined by two Newton steps each (quadratic convergence, ~1 ulp).
// Used in the amplitude arithmetic, where the 1e-12 bar leaves room and the
// IEEE sequences (__ddiv_rn / __dsqrt_rn, with their slow-path branches)
// dominated the event cost; the kinematic boundary stays exact.
// One third-order step each: the seed's relative error e (~2^-22) becomes
// O(e^3), below the double rounding.
__device__ __forceinline__ double pf_rcp_fast(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);  // 1/x = y / (1 - e) = y (1 + e + e^2 + ...)
  return fma(y, fma(e, e, e), y);
}

__device__ __forceinline__ double pf_rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x * y, y, 1.0);  // 1 - x y^2; 1/sqrt(x) = y (1 - e)^(-1/2)
  return fma(y * e, fma(e, 0.375, 0.5), y);
}

// pf_dalitz_res with the fast primitives: rsq = 1/sqrt(s) of the channel,
// qt = 1/(4 s), sbr0 = sqrt(1 + R^2 q0^2) per call.  (B/B0)^2 and B/B0 share
// one reciprocal square root of 1 + R^2 q^2.
__device__ __forceinline__ pf_cplx pf_dalitz_res_fast(double s, double quarter, double rs, double Z, double m,
                                                      double m2, double G, double iq0, double br0, double sbr0,
                                                      double mi, double mj, double R2, int spin) {
  const double sp = mi + mj, sm = mi - mj;
  const double q2 = fmax(fma(-sp, sp, s) * fma(-sm, sm, s) * quarter, 0.0);
  const double x = q2 > 0.0 ? q2 * pf_rsqrt_fast(q2) * iq0 : 0.0;
  double bf2 = 1.0, ratio = x, sbf = 1.0;
  if (spin == 1) {
    const double ru = pf_rsqrt_fast(fma(R2, q2, 1.0));
    bf2 = br0 * (ru * ru);
    ratio = x * x * x;
    sbf = sbr0 * ru;
  }
  const double gs = G * ratio * (m * rs) * bf2;
  const double a = m2 - s, b = m * gs;
  const double f = Z * sbf * pf_rcp_fast(fma(a, a, b * b));
  pf_cplx r;
  r.re = f * a;
  r.im = f * b;
  return r;
}

// sin/cos and sinh/cosh of |u| <= 1/8 by Taylor polynomials in u^2 (terms
// to u^11 and u^12: the first omitted term is below 1e-19 relative), the
// TddpPdf mixing factors when x t / tau and y t / tau are small
__device__ __forceinline__ void pf_trig_small(double u, double& s, double& c) {
  const double u2 = u * u;
  double ps = fma(u2, -1.0 / 39916800.0, 1.0 / 362880.0);
  ps = fma(ps, u2, -1.0 / 5040.0);
  ps = fma(ps, u2, 1.0 / 120.0);
  ps = fma(ps, u2, -1.0 / 6.0);
  s = fma(u * u2, ps, u);
  double pc = fma(u2, 1.0 / 479001600.0, -1.0 / 3628800.0);
  pc = fma(pc, u2, 1.0 / 40320.0);
  pc = fma(pc, u2, -1.0 / 720.0);
  pc = fma(pc, u2, 1.0 / 24.0);
  pc = fma(pc, u2, -0.5);
  c = fma(u2, pc, 1.0);
}

__device__ __forceinline__ void pf_hyp_small(double u, double& s, double& c) {
  const double u2 = u * u;
  double ps = fma(u2, 1.0 / 39916800.0, 1.0 / 362880.0);
  ps = fma(ps, u2, 1.0 / 5040.0);
  ps = fma(ps, u2, 1.0 / 120.0);
  ps = fma(ps, u2, 1.0 / 6.0);
  s = fma(u * u2, ps, u);
  double pc = fma(u2, 1.0 / 479001600.0, 1.0 / 3628800.0);
  pc = fma(pc, u2, 1.0 / 40320.0);
  pc = fma(pc, u2, 1.0 / 720.0);
  pc = fma(pc, u2, 1.0 / 24.0);
  pc = fma(pc, u2, 0.5);
  c = fma(u2, pc, 1.0);
}

// inside the kinematic boundary of the (m12^2, m13^2) plane
__device__ __forceinline__ bool pf_dalitz_inside(double s12, double s13, double M, double m1, double m2,
                                                 double m3) {
  const double a12 = __dadd_rn(m1, m2), b12 = __dsub_rn(M, m3);
  if (!(s12 >= __dmul_rn(a12, a12) && s12 <= __dmul_rn(b12, b12))) return false;
  const double r12 = __dsqrt_rn(s12);
  const double e1 = __ddiv_rn(__dadd_rn(__dsub_rn(s12, __dmul_rn(m2, m2)), __dmul_rn(m1, m1)), __dmul_rn(2.0, r12));
  const double e3 = __ddiv_rn(__dsub_rn(__dsub_rn(__dmul_rn(M, M), s12), __dmul_rn(m3, m3)), __dmul_rn(2.0, r12));
  double t1 = __dsub_rn(__dmul_rn(e1, e1), __dmul_rn(m1, m1));
  double t3 = __dsub_rn(__dmul_rn(e3, e3), __dmul_rn(m3, m3));
  const double p1 = __dsqrt_rn(t1 > 0.0 ? t1 : 0.0), p3 = __dsqrt_rn(t3 > 0.0 ? t3 : 0.0);
  const double e = __dadd_rn(e1, e3), pp = __dadd_rn(p1, p3), pm = __dsub_rn(p1, p3);
  const double lo = __dsub_rn(__dmul_rn(e, e), __dmul_rn(pp, pp));
  const double hi = __dsub_rn(__dmul_rn(e, e), __dmul_rn(pm, pm));
  return s13 >= lo && s13 <= hi;
}

// Per-channel quantities shared by every resonance of the channel (same s,
// same daughters): q = |p*| of the split, and for spin 1 the Blatt-Weisskopf
// reciprocal root 1/sqrt(1 + R^2 q^2) and its square.
struct pf_dalitz_ch {
  double s, rs, q, ru, ru2;
};

__device__ __forceinline__ pf_dalitz_ch pf_dalitz_channel(double s, double rs, double mi, double mj, double R2) {
  pf_dalitz_ch c;
  c.s = s;
  c.rs = rs;
  const double sp = mi + mj, sm = mi - mj;
  const double q2 = fmax(fma(-sp, sp, s) * fma(-sm, sm, s) * (0.25 * (rs * rs)), 0.0);
  c.q = q2 > 0.0 ? q2 * pf_rsqrt_fast(q2) : 0.0;
  c.ru = pf_rsqrt_fast(fma(R2, q2, 1.0));
  c.ru2 = c.ru * c.ru;
  return c;
}

// one resonance of a channel: pf_dalitz_res_fast with the channel's shared terms
__device__ __forceinline__ pf_cplx pf_dalitz_res_ch(const pf_dalitz_ch& c, double Z, double m, double m2, double G,
                                                    double iq0, double br0, double sbr0, int spin) {
  const double x = c.q * iq0;
  double bf2 = 1.0, ratio = x, sbf = 1.0;
  if (spin == 1) {
    bf2 = br0 * c.ru2;
    ratio = x * x * x;
    sbf = sbr0 * c.ru;
  }
  const double gs = G * ratio * (m * c.rs) * bf2;
  const double a = m2 - c.s, b = m * gs;
  const double f = Z * sbf * pf_rcp_fast(fma(a, a, b * b));
  pf_cplx r;
  r.re = f * a;
  r.im = f * b;
  return r;
}

// The same decision as pf_dalitz_inside, cheaply: the limits lo/hi of s13
// come from the fast reciprocals.  With p >= 1e-3 E the fast and exact
// sequences differ by < 5e-13 (e^2 + p^2), so a point farther than
// 1e-11 (e^2 + p^2) from both limits is decided alike; closer points, and
// p < 1e-3 E (ill-conditioned square root), take the exact sequence.
__device__ __forceinline__ bool pf_dalitz_inside_fast(double s12, double s13, double M, double m1, double m2,
                                                      double m3) {
  const double a12 = __dadd_rn(m1, m2), b12 = __dsub_rn(M, m3);
  if (!(s12 >= __dmul_rn(a12, a12) && s12 <= __dmul_rn(b12, b12))) return false;
  const double ir = 0.5 * pf_rsqrt_fast(s12);  // 1 / (2 sqrt s12)
  const double e1 = (s12 - m2 * m2 + m1 * m1) * ir;
  const double e3 = (M * M - s12 - m3 * m3) * ir;
  const double t1 = e1 * e1 - m1 * m1, t3 = e3 * e3 - m3 * m3;
  // p = sqrt(t) is ill-conditioned where p << E (the edges of the s12 range):
  // there the exact sequence decides
  if (!(t1 >= 1e-6 * (e1 * e1)) || !(t3 >= 1e-6 * (e3 * e3))) return pf_dalitz_inside(s12, s13, M, m1, m2, m3);
  const double p1 = t1 * pf_rsqrt_fast(t1), p3 = t3 * pf_rsqrt_fast(t3);
  const double e = e1 + e3, pp = p1 + p3, pm = p1 - p3;
  const double ee = e * e;
  const double lo = ee - pp * pp, hi = ee - pm * pm;
  const double tol = 1e-11 * (ee + pp * pp);
  if (s13 < lo - tol || s13 > hi + tol) return false;
  if (s13 > lo + tol && s13 < hi - tol) return true;
  return pf_dalitz_inside(s12, s13, M, m1, m2, m3);
}

// pf_dalitz_inside_fast split for a grid row (s12 fixed): the s12 side once
// per row, then per point the same decision as pf_dalitz_inside_fast.
struct pf_dalitz_row {
  bool in12, exact;
  double lo, hi, tol;
};

__device__ __forceinline__ pf_dalitz_row pf_dalitz_row_limits(double s12, double M, double m1, double m2, double m3) {
  pf_dalitz_row R;
  R.exact = false;
  R.lo = R.hi = R.tol = 0.0;
  const double a12 = __dadd_rn(m1, m2), b12 = __dsub_rn(M, m3);
  R.in12 = s12 >= __dmul_rn(a12, a12) && s12 <= __dmul_rn(b12, b12);
  if (!R.in12) return R;
  const double ir = 0.5 * pf_rsqrt_fast(s12);
  const double e1 = (s12 - m2 * m2 + m1 * m1) * ir;
  const double e3 = (M * M - s12 - m3 * m3) * ir;
  const double t1 = e1 * e1 - m1 * m1, t3 = e3 * e3 - m3 * m3;
  if (!(t1 >= 1e-6 * (e1 * e1)) || !(t3 >= 1e-6 * (e3 * e3))) {
    R.exact = true;
    return R;
  }
  const double p1 = t1 * pf_rsqrt_fast(t1), p3 = t3 * pf_rsqrt_fast(t3);
  const double e = e1 + e3, pp = p1 + p3, pm = p1 - p3;
  const double ee = e * e;
  R.lo = ee - pp * pp;
  R.hi = ee - pm * pm;
  R.tol = 1e-11 * (ee + pp * pp);
  return R;
}

__device__ __forceinline__ bool pf_dalitz_row_inside(const pf_dalitz_row& R, double s12, double s13, double M,
                                                     double m1, double m2, double m3) {
  if (!R.in12) return false;
  if (!R.exact) {
    if (s13 < R.lo - R.tol || s13 > R.hi + R.tol) return false;
    if (s13 > R.lo + R.tol && s13 < R.hi - R.tol) return true;
  }
  return pf_dalitz_inside(s12, s13, M, m1, m2, m3);
}

// ----------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, global -> shared) completed on mbarriers.
__device__ __forceinline__ unsigned pf_smem_addr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void pf_mbar_init(pf_u64* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(pf_smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void pf_fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void pf_mbar_expect_tx(pf_u64* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(pf_smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void pf_tma_load(void* dst, const void* src, unsigned bytes, pf_u64* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          pf_smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(pf_smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void pf_mbar_wait(pf_u64* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "PF_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra PF_WAIT;\n"
      "}\n" ::"r"(pf_smem_addr(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ double pf_log(double x) { return log(x); }
__device__ __forceinline__ double pf_pow(double x, double y) { return pow(x, y); }

// 1e-300 as an integer: for x >= +0 the IEEE bit pattern orders like x
#define PF_FLOOR_BITS 0x01a56e1fc2f8f359LL

// ln 2 split so that E * PF_LN2_HI is exact for |E| < 2^21 (fdlibm constants)
#define PF_LN2_HI 6.93147180369123816490e-01
#define PF_LN2_LO 1.90821492927058770002e-10

// Running product with an exponent register: prod(v) = m * 2^E, m in [1, 2).
// Replaces one log per event by one log per thread and chunk; the per-event
// rounding added is one ulp of m (below the reference's own per-term log
// rounding), and nothing can over- or underflow.
struct pf_prod {
  double m;
  int e;
};

__device__ __forceinline__ void pf_prod_init(pf_prod& p) {
  p.m = 1.0;
  p.e = 0;
}

// v is in 2^[-500, 600] here (the caller rescales rarer magnitudes) and m
// stays within 2^[-400, 400) between renormalisations, so m * v can neither
// over- nor underflow; renormalising only when m leaves that band keeps the
// serial chain to one DMUL and one integer compare.
__device__ __forceinline__ void pf_prod_mul(pf_prod& p, double v) {
  double m = p.m * v;
  const unsigned hi = (unsigned)__double2hiint(m);
  if (hi - 0x26F00000u >= 0x32000000u) {  // biased exponent outside [623, 1423)
    const int ex = (int)((hi >> 20) & 0x7ff) - 1023;
    p.e += ex;
    m = __hiloint2double((int)hi - (ex << 20), __double2loint(m));
  }
  p.m = m;
}

// -log(prod) as a DD value
__device__ __forceinline__ pf_dd pf_prod_neglog(const pf_prod& p) {
  double lm = pf_log(p.m);
  double e = (double)p.e;
  pf_dd s = pf_two_sum(-(e * PF_LN2_HI), -lm);
  s.lo += -(e * PF_LN2_LO);
  return pf_fast_two_sum(s.hi, s.lo);
}
