// pf_kernels.cuh — kernel bodies of the per-call CUDA graph.
//
// Included by the generated evaluator AFTER it has defined:
//   PF_NP, PF_SS, PF_NCOLS, PF_NLOAD, PF_EPT, PF_BINNED, PF_NPOLY,
//   pf_load_col(q)                                 data columns read per event
//   pf_stage_pre(k, P, S, C, cx, cnt, tid, nt)      parameter-derived constants
//   pf_stage_post(level, k, P, S, C, cx, cnt, tid, nt)  constants needing norms
//   pf_norm_point(node, flat, task, P, S, C, cx, cnt)   raw at a grid midpoint
//   pf_eval_event(ev, P, S, C, cx, cnt)            normalised density (NLL) or
//                                                  N_tot * density (chi2)
//
// Per-call graph (engine.cpp):
//   small normalisation grids:  setup ──PDL──> event(+final tree)
//   large grids:                pre -> norm level 0..L ──PDL──> event(+final)
//   batched (K > 1):            ... -> event -> final (one block per k)
// Parameters are read from, and results written to, mapped host memory.
// Every reduction has a fixed shape: a call is bitwise reproducible and
// independent of the number of devices.

// griddepcontrol (programmatic dependent launch); no-ops without PDL
#ifdef PF_EVENT_TRACE
__device__ __forceinline__ unsigned long long pf_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// per block: [in, prologue done, PDL wait done, main loop done, block done,
// published]; setup: slot 0 of block 4095 (in), slot 1 (out)
__device__ unsigned long long pf_trace_buf[4096 * 6];
__device__ unsigned long long pf_trace_w[4096 * 2];
#define PF_ETRACE(slot, v) (pf_trace_buf[(pf_u64)blockIdx.x * 6 + (slot)] = (v))
#endif
__device__ __forceinline__ void pf_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }
__device__ __forceinline__ void pf_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void pf_rec_init(pf_krec* r) {
  r->floor_count = 0ull;
  r->first_nonfinite = ~0ull;
  r->first_event_error = ~0ull;
  r->norm_error = ~0u;
  for (int i = 0; i <= PF_MAX_LEVELS; ++i) r->arrive[i] = 0u;
  for (int i = 0; i < PF_FX_DIGITS; ++i) r->fx[i] = 0ll;
}

__device__ __forceinline__ void pf_load_params(const pf_args& a, int k) {
  for (int i = threadIdx.x; i < PF_NP; i += blockDim.x)
    ((double*)a.P)[(pf_u64)k * PF_NP + i] = a.npin ? a.pin[i] : a.hP[(pf_u64)k * PF_NP + i];
}

// Richardson combination of a node's (coarse, fine) sums (pdf.hpp:178-188)
__device__ __forceinline__ void pf_finish_norm(double* S, pf_krec* r, int node, double coarse,
                                               double fine) {
  if (pf_finish_norm_s(S, node, coarse, fine))
    atomicMin(&r->norm_error, ((pf_u32)node << 8) | PF_E_ZERO_INTEGRAL);
}

// a finished (coarse, fine) task pair: a node's norm, or one component sum of
// a TddpPdf's separable grid (combined by pf_stage_post)
__device__ __forceinline__ void pf_finish_task(double* S, pf_krec* r, const pf_task& T, double coarse,
                                               double fine) {
  if (T.comp >= 0)
    pf_store_comp(S, T.node, T.comp, coarse, fine);
  else
    pf_finish_norm(S, r, T.node, coarse, fine);
}

// ---------------------------------------------------------------------------
#define PF_SETUP_THREADS 512  // 128 registers: the level's 8 reductions interleave unspilled
#ifndef PF_SETUP_CLUSTER
#define PF_SETUP_CLUSTER 1    // CTAs (one thread-block cluster) per parameter set
#endif
#ifndef PF_SETUP_MAXQ
#define PF_SETUP_MAXQ 8       // most midpoint sums in one level (2 per node)
#endif

// thread-block cluster helpers (distributed shared memory, sm_90+)
__device__ __forceinline__ unsigned pf_cluster_rank() {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void pf_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ double pf_dsmem_load(const double* p, unsigned rank) {
  unsigned ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(pf_smem_addr(p)), "r"(rank));
  double v;
  asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
  return v;
}
// ---------------------------------------------------------------------------
// The setup work of one parameter set, shared by the setup kernel (a cluster
// of CL CTAs splitting the grid points) and the fused kernel (every CTA
// computes all of it, CL = 1): P and S in shared memory on return, identical
// in every CTA.  Grid-point clamps go to `cnt`, stage clamps to `cnt_stage`.
struct pf_no_hook {
  __device__ void operator()() const {}
};

// the setup's task table (shared memory; filled by the setup core, or by a
// TMA bulk copy at kernel entry, pf_setup_prefetch)
__shared__ __align__(16) pf_task pf_tk[16];

// The setup's inputs, global -> shared by TMA bulk copies issued by one
// thread at kernel entry and completing on `bar`: the task table and the exp
// tables.  Their latency (cold after the L2 flush) then overlaps the
// parameter copy and the TMA issue of the event stages instead of stalling
// the setup (fused pass; measured 1.5 of its 7 us before).
__device__ __forceinline__ void pf_setup_prefetch(const pf_args& a, pf_u64* bar) {
  const unsigned tb = (unsigned)(min(a.n_tasks, 16) * (int)sizeof(pf_task));
  unsigned total = tb + 2048u;
#ifdef PF_QFAST
  total += 8192u;
#endif
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  pf_mbar_expect_tx(bar, total);
  if (tb) pf_tma_load(pf_tk, a.tasks, tb, bar);
  pf_tma_load(pf_exp_tab, pf_exp_tab_g, 2048u, bar);
#ifdef PF_QFAST
  pf_tma_load(pf_exp2_1024, pf_exp2_1024_g, 8192u, bar);
#endif
}

// after_init runs once the setup's own global loads (parameters, tasks,
// tables) have landed: the fused pass starts its L2 prefetch there
// preloaded: the task and exp tables arrive by pf_setup_prefetch on this
// mbarrier (phase 0) instead of being copied here
template <int CL, class Hook = pf_no_hook>
__device__ __forceinline__ void pf_setup_core(const pf_args& a, int k, unsigned rank, double* P, double* S,
                                              pf_krec* r, bool init_rec, pf_ctx& cx, pf_cnt& cnt,
                                              pf_cnt& cnt_stage, const Hook& after_init = Hook(),
                                              pf_u64* preloaded = nullptr) {
  // this CTA's run partials per task (double-double), double-buffered by level parity
  __shared__ pf_dd wpart[2][PF_SETUP_MAXQ][4];
  __shared__ double red[PF_SETUP_MAXQ][PF_SETUP_THREADS];  // the threads' partials
  pf_task* tk = pf_tk;
#ifdef PF_SETUP_TRACE
  __shared__ long long trs[32];
  __shared__ const char* trn[32];
  int ntr = 0;
  long long tr0 = clock64();
#define PF_TRACE(tag) if (threadIdx.x == 0 && ntr < 32) { trs[ntr] = clock64() - tr0; trn[ntr++] = tag; }
#else
#define PF_TRACE(tag)
#endif
  // K = 1: parameters arrive inline in the kernel arguments (constant bank,
  // updated per call on the instantiated graph); batches read mapped memory
  for (int i = threadIdx.x; i < PF_NP; i += blockDim.x)
    P[i] = a.npin ? a.pin[i] : a.hP[(pf_u64)k * PF_NP + i];
  for (int i = threadIdx.x; i < PF_SS; i += blockDim.x) S[i] = 0.0;
  const int nt = min(a.n_tasks, 16);
  if (!preloaded)
    for (int i = threadIdx.x; i < nt * (int)(sizeof(pf_task) / 8); i += blockDim.x)
      reinterpret_cast<pf_u64*>(tk)[i] = reinterpret_cast<const pf_u64*>(a.tasks)[i];
  if (init_rec && threadIdx.x == 0 && rank == 0) pf_rec_init(r);
  PF_TRACE("copy");
  if (preloaded) {
    pf_mbar_wait(preloaded, 0u);
    __syncthreads();
  } else {
    pf_math_init();  // includes __syncthreads
  }
  after_init();
  // the record is initialised before any CTA of the cluster reports into it
  if (CL > 1) pf_cluster_sync();
  PF_TRACE("init");
  pf_stage_pre(k, P, S, a.C, cx, cnt_stage, threadIdx.x, blockDim.x);
  PF_TRACE("pre");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int t0 = 0;
  for (int level = 0; level < a.n_levels; ++level) {
    int t1 = t0;
    while (t1 < nt && tk[t1].level == level) ++t1;
    const int nl = min(t1 - t0, PF_SETUP_MAXQ);  // (coarse, fine) task pairs of the level's nodes
    // every midpoint sum of the level first (this CTA's share of the points).
    // A thread adds its few points in plain double (a handful per task);
    // every tree above that is double-double, so the sum is good to ~1e-17
    // relative whatever the split into threads and CTAs -- its rounding to
    // double is the correctly rounded sum, as the reference's long double
    // sum rounded to double (pdf.hpp:163-175) nearly always is, and the same
    // for the cluster, single-CTA (fused) and multi-block paths.
    // one loop per task (constant q: no per-point task search); the loops'
    // few iterations are independent evaluations
#ifdef PF_SETUP_QLOOP
    // one copy of the task loop's code (the setup runs once per call from a
    // cold instruction cache: its code size is its cost)
#pragma unroll 1
    for (int q = 0; q < PF_SETUP_MAXQ; ++q) {
      double xq = 0.0;
      if (q < nl) {
        PF_CHECK(t0 + q < nt && t0 + q < 16);
        const pf_task& T = tk[t0 + q];
        xq = pf_norm_accum(T.node, rank * PF_SETUP_THREADS + threadIdx.x, T.points, PF_SETUP_THREADS * CL, T, P, S,
                           a.C, cx, cnt);
      }
      red[q][threadIdx.x] = xq;
    }
    PF_TRACE("points");
#else
    double x[PF_SETUP_MAXQ];
#pragma unroll
    for (int q = 0; q < PF_SETUP_MAXQ; ++q) {
      x[q] = 0.0;
      if (q < nl) {
        PF_CHECK(t0 + q < nt && t0 + q < 16);
        const pf_task& T = tk[t0 + q];
        x[q] = pf_norm_accum(T.node, rank * PF_SETUP_THREADS + threadIdx.x, T.points, PF_SETUP_THREADS * CL, T, P, S,
                             a.C, cx, cnt);
      }
    }
    PF_TRACE("points");
#endif
    // the threads' partials through shared memory; then warp w sums run
    // (w % 4) of task (w / 4) -- 128 partials -- in double-double and 4 runs
    // per task are added in double-double: every task's sum is good to
    // ~1e-17 relative for a fraction of the cost of per-warp trees of all tasks
#ifndef PF_SETUP_QLOOP
#pragma unroll
    for (int q = 0; q < PF_SETUP_MAXQ; ++q) red[q][threadIdx.x] = x[q];
#endif
    __syncthreads();
    static_assert(PF_SETUP_THREADS == 512, "16 warps: 4 runs of 128 partials for each of 4 tasks per pass");
    for (int q0 = 0; q0 < nl; q0 += 4) {
      const int q = q0 + warp / 4;
      if (q < nl) {
        const int base = (warp % 4) * 128;
        pf_dd acc = pf_dd_zero();
#pragma unroll
        for (int i = 0; i < 4; ++i) acc = pf_dd_add_d(acc, red[q][base + 32 * i + lane]);
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) acc = pf_dd_add(acc, pf_shfl_down_dd(acc, d));
        if (lane == 0) wpart[level & 1][q][warp % 4] = acc;
      }
    }
    PF_TRACE("wtree");
    // partials of every rank visible cluster-wide (double-buffered by level
    // parity: a rank cannot overwrite a buffer another rank may still read
    // without first passing the next level's barrier)
    if (CL > 1)
      pf_cluster_sync();
    else
      __syncthreads();
    PF_TRACE("csync");
    // one warp per node: lanes 0-15 its coarse sum, lanes 16-31 its fine sum;
    // lane l < 4 of each half holds run l of every rank, combined over ranks
    // by a fixed tree, then a 4-lane tree; lane 0 finishes the node
    if (2 * warp < nl) {
      const int q = 2 * warp + (lane >> 4);
      const int l = lane & 15;
      pf_dd y = pf_dd_zero();
      if (l < 4) {
        const pf_dd* src = &wpart[level & 1][q][l];
        pf_dd v[CL];
#pragma unroll
        for (int rk = 0; rk < CL; ++rk)
          v[rk] = CL > 1 ? pf_dd{pf_dsmem_load(&src->hi, (unsigned)rk), pf_dsmem_load(&src->lo, (unsigned)rk)} : *src;
#pragma unroll
        for (int w = 1; w < CL; w <<= 1)
#pragma unroll
          for (int rk = 0; rk + w < CL; rk += 2 * w) v[rk] = pf_dd_add(v[rk], v[rk + w]);
        y = v[0];
      }
#pragma unroll
      for (int d = 2; d > 0; d >>= 1) y = pf_dd_add(y, pf_shfl_down_dd(y, d));
      // midpoint_sum returns static_cast<double>(sum) * vol (pdf.hpp:173-175)
      const double sum = __dmul_rn(pf_dd_to_double(y), tk[t0 + q].vol);
      const double fine = __shfl_down_sync(0xffffffffu, sum, 16);
      if (lane == 0) pf_finish_task(S, r, tk[t0 + q], sum, fine);
    }
    __syncthreads();
    PF_TRACE("finish");
    pf_stage_post(level, k, P, S, a.C, cx, cnt_stage, threadIdx.x, blockDim.x);
    PF_TRACE("post");
    t0 = t1;
  }
#ifdef PF_SETUP_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0)
    for (int i = 0; i < ntr; ++i) printf("setup %-8s %lld\n", trn[i], trs[i]);
#endif
#undef PF_TRACE
}

// ---------------------------------------------------------------------------
// setup: call records, pre stage and EVERY normalisation level for one
// parameter set in one thread-block cluster of PF_SETUP_CLUSTER CTAs (small
// grids).  Midpoint sums at n and 2n (pdf.hpp:148-176): thread t of CTA c
// sums points c * 512 + t, + 512 * PF_SETUP_CLUSTER, ... ; a fixed-shape
// block reduction gives each CTA's partial, and every CTA adds the partials
// of all ranks (read over DSMEM) in rank order, so all CTAs hold identical
// norms and stage constants for the next level.  Rank 0 writes the per-call
// state to global memory for the event pass.
extern "C" __global__ void __launch_bounds__(PF_SETUP_THREADS) pf_setup_kernel(const __grid_constant__ pf_args a) {
  // parameters and the per-call state live in shared memory while the CTA
  // works (every S read/write is an LDS/STS, not an L2 round trip)
  extern __shared__ __align__(16) double pf_sdyn[];
  pf_pdl_trigger();  // let the event kernel start streaming its data now
  const unsigned rank = PF_SETUP_CLUSTER > 1 ? pf_cluster_rank() : 0u;
  const int k = blockIdx.x / PF_SETUP_CLUSTER;
#ifdef PF_EVENT_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0) pf_trace_buf[4095 * 6 + 0] = pf_gtime();
#endif
  double* P = pf_sdyn;
  double* S = pf_sdyn + PF_NP;
  pf_krec* r = a.rec + k;
  pf_ctx cx;
  cx.err = 0;
  pf_cnt cnt;        // clamps met on this CTA's grid points
  pf_cnt_init(cnt);
  pf_cnt cnt_stage;  // clamps met in the pre/post stages (every CTA runs them; rank 0 reports)
  pf_cnt_init(cnt_stage);
  pf_setup_core<PF_SETUP_CLUSTER>(a, k, rank, P, S, r, true, cx, cnt, cnt_stage);
  if (cx.err) atomicMin(&r->norm_error, cx.err);
  if (pf_grid_counts(a, k)) {
    pf_cnt_flush(cnt, a.clamp);
    if (rank == 0) pf_cnt_flush(cnt_stage, a.clamp);
  }
  __syncthreads();
  if (rank == 0) {
    double* gS = a.S + (pf_u64)k * PF_SS;
    double* gP = (double*)a.P + (pf_u64)k * PF_NP;
    for (int i = threadIdx.x; i < PF_SS; i += blockDim.x) gS[i] = S[i];
    for (int i = threadIdx.x; i < PF_NP; i += blockDim.x) gP[i] = P[i];
  }
#ifdef PF_EVENT_TRACE
  if (threadIdx.x == 0 && blockIdx.x == 0) pf_trace_buf[4095 * 6 + 1] = pf_gtime();
#endif
  // no CTA leaves while another may still read its shared memory
  if (PF_SETUP_CLUSTER > 1) pf_cluster_sync();
}

// ---------------------------------------------------------------------------
// pre (large grids): parameters, call records and the pre stage.
#if defined(PF_S_SMEM) && PF_SS * 8 <= 96 * 1024 && PF_SS % 2 == 0 && !defined(PF_QFAST)
#define PF_S_STAGE_TMA 1  // the norm kernel works on a shared-memory copy of S (engine.cpp norm_smem)
#endif

extern "C" __global__ void __launch_bounds__(PF_THREADS) pf_pre_kernel(const __grid_constant__ pf_args a) {
  // (a shared-memory copy of S staged by TMA and written back measured slower
  // for C4's tables: 8.3 vs 7.1 us)
  pf_math_init();
  const int k = blockIdx.x;
  pf_krec* r = a.rec + k;
  pf_load_params(a, k);
  if (threadIdx.x == 0) pf_rec_init(r);
  __syncthreads();
  pf_ctx cx;
  cx.err = 0;
  pf_cnt cnt;
  pf_cnt_init(cnt);
  pf_stage_pre(k, a.P + (pf_u64)k * PF_NP, a.S + (pf_u64)k * PF_SS, a.C, cx, cnt, threadIdx.x,
               blockDim.x);
  if (cx.err) atomicMin(&r->norm_error, cx.err);
  if (pf_grid_counts(a, k)) pf_cnt_flush(cnt, a.clamp);
}

// ---------------------------------------------------------------------------
// norm (large grids): one level, many blocks per midpoint sum; the last
// block to arrive combines the block partials, applies Richardson and runs
// the post stage.
#ifndef PF_NORM_RUN
#define PF_NORM_RUN 32  // grid points per thread and run (>= 2-D boxes; engine.cpp build_tasks, kNormRun)
#endif
#ifndef PF_NORM_MIN_BLOCKS
#define PF_NORM_MIN_BLOCKS 2  // resident norm blocks per SM: <= 128 registers (C5 TDDP grid: 164 regs, 1 block/SM, 147 us -> 2 blocks, 122 us despite spills)
#endif
extern "C" __global__ void __launch_bounds__(PF_THREADS, PF_NORM_MIN_BLOCKS) pf_norm_kernel(const __grid_constant__ pf_args a) {
  __shared__ pf_dd sm[PF_THREADS];
  __shared__ int s_last;
  __shared__ double sums[64][4];
#ifdef PF_NORM_POINT_TRACE
  const unsigned long long g_in = pf_gtime();
#endif
  if (a.level == a.n_levels - 1) pf_pdl_trigger();
  const int k = blockIdx.y;
  const double* P = a.P + (pf_u64)k * PF_NP;
  double* S = a.S + (pf_u64)k * PF_SS;
#ifdef PF_S_STAGE_TMA
#define PF_NORM_S_STAGED 1
  // convolution tables read per (point, tau): the points read a shared-memory
  // copy of the per-call state (LDS, not global loads on the recurrence's
  // critical path), brought in with the exp table by two TMA bulk copies (a
  // thread loop took 3.5 us); the last block below still finishes into global S
  extern __shared__ __align__(16) double pf_norm_S[];
  __shared__ __align__(8) pf_u64 nbar;
  if (threadIdx.x == 0) {
    pf_mbar_init(&nbar, 1);
    pf_fence_mbar_init();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    pf_mbar_expect_tx(&nbar, (unsigned)(PF_SS * 8 + 2048));
    pf_tma_load(pf_norm_S, S, (unsigned)(PF_SS * 8), &nbar);
    pf_tma_load(pf_exp_tab, pf_exp_tab_g, 2048u, &nbar);
  }
  __syncthreads();
  pf_mbar_wait(&nbar, 0u);
#else
  pf_math_init();
#endif
  // per block and value one partial: task t owns blocks [first_block,
  // first_block + n_blocks); value c (a TddpPdf's four Dalitz components,
  // comp 8) at part[c * gridDim.x + block]
  pf_dd* part = a.partials + (pf_u64)k * gridDim.x * 4;
  int t = 0;
  while (t + 1 < a.n_tasks && (int)blockIdx.x >= a.tasks[t + 1].first_block) ++t;
  const pf_task& T = a.tasks[t];
  PF_CHECK(t < a.n_tasks && (int)blockIdx.x >= T.first_block && (int)blockIdx.x < T.first_block + T.n_blocks);
  const pf_u64 b = (pf_u64)((int)blockIdx.x - T.first_block);
  const pf_u64 lo = b * T.per_block;
  const pf_u64 hi = min(lo + T.per_block, T.points);
  pf_ctx cx;
  cx.err = 0;
  pf_cnt cnt;
  pf_cnt_init(cnt);
  const bool multi = T.comp == PF_COMP_ALL4;
  pf_dd acc[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) acc[c] = pf_dd_zero();
#ifdef PF_NORM_S_STAGED
  const double* Sp = pf_norm_S;
#else
  const double* Sp = S;
#endif
  if (multi) {
    // all four components from ONE evaluation of both amplitudes per point,
    // in runs of PF_NORM_RUN consecutive points walked row by row; channel A
    // (s13) from the block's column table when the engine gave it room
    const double* tab = nullptr;
    if (a.tddp_tab) {
      extern __shared__ __align__(16) double pf_norm_tab[];
      pf_tddp_cols(T.node, T, P, Sp, a.C, pf_norm_tab, threadIdx.x, PF_THREADS);
      __syncthreads();
      tab = pf_norm_tab;
    }
    for (pf_u64 i = lo + (pf_u64)threadIdx.x * PF_NORM_RUN; i < hi; i += (pf_u64)PF_THREADS * PF_NORM_RUN) {
      double v4[4];
      pf_norm_run4(T.node, i, (int)min((pf_u64)PF_NORM_RUN, hi - i), T, P, Sp, a.C, v4, tab);
#pragma unroll
      for (int c = 0; c < 4; ++c) acc[c] = pf_dd_add_d(acc[c], v4[c]);
    }
  } else if (T.dims >= 2 && T.per_block >= (pf_u64)PF_THREADS * PF_NORM_RUN) {
    // runs of PF_NORM_RUN consecutive points per thread, walked row by row
    // (a DalitzPlotPdf's channel 13 from the block's column table)
    const double* tab = nullptr;
    if (a.tddp_tab) {
      extern __shared__ __align__(16) double pf_norm_tab[];
      pf_dalitz_cols(T.node, T, P, Sp, a.C, pf_norm_tab, threadIdx.x, PF_THREADS);
      __syncthreads();
      tab = pf_norm_tab;
    }
    for (pf_u64 i = lo + (pf_u64)threadIdx.x * PF_NORM_RUN; i < hi; i += (pf_u64)PF_THREADS * PF_NORM_RUN)
      acc[0] = pf_dd_add_d(acc[0], pf_norm_run(T.node, i, (int)min((pf_u64)PF_NORM_RUN, hi - i), T, P, Sp, a.C, cx, cnt,
                                               tab));
  } else {
#ifdef PF_NORM_POINT_TRACE
    const long long c0 = clock64();
    const unsigned long long g_pts = pf_gtime();
#endif
    for (pf_u64 i = lo + threadIdx.x; i < hi; i += PF_THREADS)
      acc[0] = pf_dd_add_d(acc[0], pf_norm_point(T.node, i, T, P, Sp, a.C, cx, cnt));
#ifdef PF_NORM_POINT_TRACE
    (void)c0;
    if (threadIdx.x == 0 && blockIdx.x < 2000) {
      pf_trace_buf[(2000 + blockIdx.x) * 6 + 0] = g_in;
      pf_trace_buf[(2000 + blockIdx.x) * 6 + 1] = g_pts;
      pf_trace_buf[(2000 + blockIdx.x) * 6 + 2] = pf_gtime();
    }
#endif
  }
  for (int c = 0; c < (multi ? 4 : 1); ++c) {
    pf_dd s = pf_block_reduce(acc[c], sm);
    if (threadIdx.x == 0) part[(pf_u64)c * gridDim.x + blockIdx.x] = s;
  }
  if (cx.err) atomicMin(&a.rec[k].norm_error, cx.err);
  if (pf_grid_counts(a, k)) pf_cnt_flush(cnt, a.clamp);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev = atomicAdd(&a.rec[k].arrive[a.level], 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
#ifdef PF_NORM_POINT_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 2000) pf_trace_buf[(2000 + blockIdx.x) * 6 + 3] = pf_gtime();
#endif
  if (!s_last) return;
  __threadfence();
#ifdef PF_CONV_TRACE_FULL
  if (threadIdx.x == 0) {
    printf("norm level %d: full-Q fallbacks %u, windows not summed %u\n", a.level, pf_conv_full_count[0],
           pf_conv_full_count[1]);
    pf_conv_full_count[0] = pf_conv_full_count[1] = 0u;
  }
#endif
  // one warp per task (the tasks' partials in parallel: each sum is the
  // same fixed-shape reduction whichever warp does it)
  for (int tt = (int)(threadIdx.x >> 5); tt < a.n_tasks; tt += PF_THREADS / 32) {
    const pf_task& U = a.tasks[tt];
    const int nv = U.comp == PF_COMP_ALL4 ? 4 : 1;
    for (int c = 0; c < nv; ++c) {
      pf_dd s = pf_warp_reduce_runs(part + (pf_u64)c * gridDim.x + U.first_block, U.n_blocks);
      if ((threadIdx.x & 31) == 0) sums[tt][c] = __dmul_rn(pf_dd_to_double(s), U.vol);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int tt = 0; tt + 1 < a.n_tasks; tt += 2) {
      if (a.tasks[tt].comp == PF_COMP_ALL4) {
        for (int c = 0; c < 4; ++c) pf_store_comp(S, a.tasks[tt].node, c, sums[tt][c], sums[tt + 1][c]);
      } else {
        pf_finish_task(S, a.rec + k, a.tasks[tt], sums[tt][0], sums[tt + 1][0]);
      }
    }
  __syncthreads();
  pf_ctx cx2;
  cx2.err = 0;
  pf_cnt cnt2;
  pf_cnt_init(cnt2);
  pf_stage_post(a.level, k, P, S, a.C, cx2, cnt2, threadIdx.x, blockDim.x);
  if (cx2.err) atomicMin(&a.rec[k].norm_error, cx2.err);
  if (pf_grid_counts(a, k)) pf_cnt_flush(cnt2, a.clamp);
#ifdef PF_NORM_POINT_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 2000) pf_trace_buf[(2000 + blockIdx.x) * 6 + 4] = pf_gtime();
#endif
}

// ---------------------------------------------------------------------------
// event pass.  A chunk (the reduction unit, 256 * PF_EPT events) belongs to
// ONE warp, which walks it in PF_NSUB sub-chunks of 32 * PF_EPT events.
// Sub-chunks are staged global -> shared by TMA bulk copies into a per-warp
// ring of PF_NST stages (mbarrier completion), PF_NST - 1 copies in flight
// while the warp computes; the compute loop reads the stage with
// conflict-free LDS (lane l takes events 32 j + l), so the code stays small
// and the memory stream never waits on the math.  Per lane: a chunk
// accumulator (pf_lacc_*: log-domain sum and mixture-factor product, or a
// running density product) is carried over the chunk's sub-chunks and turned
// into -log terms once per chunk, which are added EXACTLY into the lane's
// fixed-point accumulator.  No block-level barrier in the main loop.  The
// first stages are issued BEFORE waiting on the setup grid (PDL).

#define PF_SUB (32 * PF_EPT)
#ifndef PF_NSUB
#define PF_NSUB 8  // sub-chunks per chunk: chunk = PF_NSUB * 32 * PF_EPT events
#endif
#ifndef PF_UNROLL
#define PF_UNROLL 8  // events interleaved per lane in the event loop
#endif
constexpr int pf_unroll = PF_UNROLL;
#ifndef PF_NST
#define PF_NST 3
#endif
#ifndef PF_EV_WARPS
#define PF_EV_WARPS 2  // warps per event block: fine-grained block scheduling
#endif
#define PF_EV_THREADS (32 * PF_EV_WARPS)
#define PF_STAGE (PF_NLOAD * PF_SUB)  // doubles per stage

// One event's term for the rare-path rescans (errors / non-finite terms).
__device__ __noinline__ pf_u32 pf_event_flags(const pf_args& a, const double* P, const double* S,
                                              const double* st, int i, double* v_out) {
  pf_ctx cx;
  cx.err = 0;
  pf_cnt cnt;  // scratch: rescans do not count clamps twice
  pf_cnt_init(cnt);
  double ev[PF_NCOLS];
#pragma unroll
  for (int q = 0; q < PF_NCOLS; ++q) ev[q] = 0.0;
#pragma unroll
  for (int q = 0; q < PF_NLOAD; ++q) ev[pf_load_col(q)] = st[q * PF_SUB + i];
  *v_out = pf_eval_event(ev, P, S, a.C, cx, cnt);
  return cx.err;
}

// Rare path, out of line: the first event (in this lane's order) that raised
// an error or produced a non-finite term is found by re-evaluating.
__device__ __noinline__ void pf_rescan(const pf_args& a, int k, const double* P, const double* S,
                                       pf_u64 base, int lane, const double* st, int n_valid, bool want_err) {
  for (int j = 0; j < PF_EPT; ++j) {
    const int i = 32 * j + lane;
    if (i >= n_valid) break;
    double v;
    const pf_u32 err = pf_event_flags(a, P, S, st, i, &v);
    if (want_err) {
      if (err) {
        atomicMin(&a.rec[k].first_event_error, ((a.event_offset + base + i) << 24) | (pf_u64)err);
        return;
      }
    } else {
#if PF_BINNED
      const double mu = v * st[(PF_NLOAD - 1) * PF_SUB + i];
      const double diff = st[(PF_NLOAD - 2) * PF_SUB + i] - mu;
      const double term = diff * diff / fmax(mu, PF_CHISQ_EPS);
      const bool bad = !isfinite(term);
#else
      const bool bad = !(v < PF_LOG_FLOOR) && !(v <= 1.7976931348623157e308);
#endif
      if (bad) {
        atomicMin(&a.rec[k].first_nonfinite, a.event_offset + base + i);
        return;
      }
    }
  }
}

// Per-lane chunk accumulator, carried across the PF_NSUB sub-chunks of a
// chunk (in shared memory, fixed order) and turned into the chunk's sum of
// -log terms once per chunk (pf_lacc_terms), so the lane's logs are
// amortised over PF_NSUB * PF_EPT events:
//   log form 1: {sum of L, per power factor: mantissa product, exponent sum}
//   log form 2: {sum of L, product of mixture factors F (F <= n_children)}
//   linear:     {m, e}: running density product m * 2^e   (pf_prod)
//   binned:     double-double sum of chi-squared terms
#ifndef PF_NFAC
#define PF_NFAC 0
#endif
#ifndef PF_FSPLIT
#define PF_FSPLIT 0
#endif
#define PF_NFAC_A (PF_NFAC > 0 ? PF_NFAC : 1)
#if !PF_BINNED && PF_LOGFORM
#define PF_LACC_N (1 + (PF_FSPLIT ? 2 : 1) * PF_NFAC)
#else
#define PF_LACC_N 2
#endif
struct pf_lacc {
  double v[PF_LACC_N];
};

__device__ __forceinline__ pf_lacc pf_lacc_merge(pf_lacc x, const pf_lacc& y) {
#if PF_BINNED
  const pf_dd s = pf_dd_add(pf_dd{x.v[0], x.v[1]}, pf_dd{y.v[0], y.v[1]});
  x.v[0] = s.hi;
  x.v[1] = s.lo;
#elif PF_LOGFORM
  x.v[0] += y.v[0];
#pragma unroll
  for (int j = 0; j < PF_NFAC; ++j) {
    if (PF_FSPLIT) {
      x.v[1 + 2 * j] *= y.v[1 + 2 * j];  // mantissa products (< 2^64 per chunk lane)
      x.v[2 + 2 * j] += y.v[2 + 2 * j];  // exponent sums (exact integers)
    } else {
      x.v[1 + j] *= y.v[1 + j];
    }
  }
#else
  pf_prod p;
  p.m = x.v[0];
  p.e = (int)x.v[1];
  pf_prod_mul(p, y.v[0]);  // y's mantissa is renormalised: inside 2^[-400, 400)
  x.v[0] = p.m;
  x.v[1] = (double)(p.e + (int)y.v[1]);
#endif
  return x;
}

// the chunk lane's sum of -log terms (double-double)
__device__ __forceinline__ pf_dd pf_lacc_terms(const pf_lacc& x, const double* __restrict__ P) {
#if PF_BINNED
  return pf_dd{x.v[0], x.v[1]};
#elif PF_LOGFORM
  double f = 0.0;
#pragma unroll
  for (int j = 0; j < PF_NFAC; ++j) {
    if (PF_FSPLIT) {
      const double e = x.v[2 + 2 * j];
      f += pf_fac_pow(j, P) * (pf_log(x.v[1 + 2 * j]) + (e * PF_LN2_HI + e * PF_LN2_LO));
    } else {
      f += pf_log(x.v[1 + j]);
    }
  }
  return pf_two_sum(-x.v[0], -f);
#else
  pf_prod p;
  p.m = x.v[0];
  p.e = (int)x.v[1];
  return pf_prod_neglog(p);
#endif
}

#if !PF_BINNED && PF_LOGFORM
// log-form event accumulation shared by the fast loop and the fix-up
struct pf_lform {
  double lsum;
  double fm[PF_NFAC_A];
  int fe[PF_NFAC_A];
};

__device__ __forceinline__ void pf_lform_init(pf_lform& A) {
  A.lsum = 0.0;
#pragma unroll
  for (int j = 0; j < PF_NFAC_A; ++j) {
    A.fm[j] = 1.0;
    A.fe[j] = 0;
  }
}

__device__ __forceinline__ void pf_lform_add(pf_lform& A, double Lv, const double* fac) {
  A.lsum += Lv;
#pragma unroll
  for (int j = 0; j < PF_NFAC; ++j) {
    if (PF_FSPLIT)
      pf_fac_accum(A.fm[j], A.fe[j], fac[j]);
    else
      A.fm[j] *= fac[j];
  }
}

__device__ __forceinline__ pf_lacc pf_lform_pack(const pf_lform& A) {
  pf_lacc x;
  x.v[0] = A.lsum;
#pragma unroll
  for (int j = 0; j < PF_NFAC; ++j) {
    if (PF_FSPLIT) {
      x.v[1 + 2 * j] = A.fm[j];
      x.v[2 + 2 * j] = (double)A.fe[j];
    } else {
      x.v[1 + j] = A.fm[j];
    }
  }
  return x;
}

// Rare path of the log-domain pass, out of line: one of this lane's events
// in the sub-chunk is near the floor, overflows, is subnormal or NaN (or the
// log form is unusable, e.g. a negative mixture coefficient).  The lane's
// sub-chunk is recomputed with the reference's linear form for exactly those
// events (engine.hpp:186-195: floor 1e-300 counted, non-finite index kept).
__device__ __noinline__ pf_lacc pf_lane_fixup(const pf_args& a, int k, const double* P, const double* S,
                                              pf_u64 base, int lane, const double* st, int n_valid) {
  pf_ctx cx;
  cx.err = 0;
  pf_cnt cnt;
  pf_cnt_init(cnt);
  pf_u32 floors = 0;
  bool bad = false;
  pf_lform A;
  pf_lform_init(A);
  for (int j = 0; j < PF_EPT; ++j) {
    const int i = 32 * j + lane;
    if (i >= n_valid) continue;
    double ev[PF_NCOLS];
#pragma unroll
    for (int q = 0; q < PF_NCOLS; ++q) ev[q] = 0.0;
#pragma unroll
    for (int q = 0; q < PF_NLOAD; ++q) ev[pf_load_col(q)] = st[q * PF_SUB + i];
    double Lv, fac[PF_NFAC_A];
    if (pf_eval_event_log(ev, P, S, Lv, fac)) {
      pf_lform_add(A, Lv, fac);
    } else {
      double v = pf_eval_event(ev, P, S, a.C, cx, cnt);
      if (v < PF_LOG_FLOOR) {
        v = PF_LOG_FLOOR;
        ++floors;
      } else if (!(v <= 1.7976931348623157e308)) {
        bad = true;
        v = 1.0;
      }
      A.lsum += pf_log(v);
    }
  }
  if (cx.err) pf_rescan(a, k, P, S, base, lane, st, n_valid, true);
  if (bad) pf_rescan(a, k, P, S, base, lane, st, n_valid, false);
  if (floors) atomicAdd(&a.rec[k].floor_count, (pf_u64)floors);
  pf_cnt_flush(cnt, a.clamp);
  return pf_lform_pack(A);
}
#endif

// this lane's accumulator over one staged sub-chunk for parameter set k.
// FULL: all 32 * PF_EPT events are real (every sub-chunk but the data's last).
#ifndef PF_LOG_FAST_SLOT
struct pf_fk {};  // no fast path: nothing hoisted
__device__ __forceinline__ pf_fk pf_fk_load(const double*, const double*, const double*) { return pf_fk{}; }
#endif
__device__ __forceinline__ pf_fk pf_fk_get(const pf_args& a, int k) {
  return pf_fk_load(a.P + (pf_u64)k * PF_NP, a.S + (pf_u64)k * PF_SS, a.C);
}

#ifdef PF_QFAST
#ifndef PF_QUNROLL
#define PF_QUNROLL (PF_EPT / 2)
#endif
constexpr int pf_qunroll = PF_QUNROLL;
// Mixture fast path: AddPdf of two Exp/Gauss children of one observable, the
// per-call proof K.qfast holding (codegen.cpp: every event's terms in range,
// no floor, |d| <= 700, d's quadratic terms <= 256).  Centred at m (a
// Gaussian child's mean), t = x - m; u_i = log(coef_i raw_i) are quadratics
// in t; base child b, d = u_o - u_b:
//   -log v = -(max(u_o, u_b) + log(1 + e^-|d|)),  max = u_b + (d + |d|) / 2,
// so per event: t, d by two FMAs, u_b by one (ExpPdf base), the lane sums
// of u_b and d + |d| (exact), and e^-|d| = 2^(k/1024) e^r by a 1024-entry
// table and a quartic (|r| <= ln2/2048: truncation r^5/120 < 4e-20: smooth
// at the ulp level in the parameters, which the reference minimiser's
// finite differences need) multiplied into two products of (1 + e^-|d|).
// The result is the log-form accumulator {sum L, product F} of the other
// paths.  16 FP64 instructions per event (the general fast path: 19).
template <bool FULL>
__device__ __forceinline__ pf_lacc pf_qfast_terms(const double* st, int lane, int n_valid, const pf_fk& K) {
  const double zm = K.q[0], qA = K.q[1], qB = K.q[2], qC = K.q[3];
  const double ba = K.q[4], bb = K.q[5], bc = K.q[6];
  double s1 = 0.0, s2 = 0.0, p0 = 1.0, p1 = 1.0;
  const double2* s2v = reinterpret_cast<const double2*>(st);
#pragma unroll pf_qunroll
  for (int j = 0; j < PF_EPT / 2; ++j) {
    const int i = 32 * j + lane;  // this lane's events 2i and 2i + 1 of the stage
    const double2 xv = s2v[i];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const bool valid = FULL || 2 * i + h < n_valid;
      const double t = (h ? xv.y : xv.x) - zm;
#ifdef PF_QTRIVIAL
      s1 += t;  // experiment: the stream without the per-event math
      continue;
#endif
      const double d = fma(fma(qA, t, qB), t, qC);
#ifdef PF_QFAST_LINEAR_BASE
      const double ub = fma(bb, t, bc);
      (void)ba;
#else
      const double ub = fma(fma(ba, t, bb), t, bc);
#endif
      const double ad = fabs(d);
      s1 += valid ? ub : 0.0;
#ifdef PF_QMAX_INT
      // max(d, 0) by masking d's bits with its sign (integer pipe): the sum of
      // max(d, 0) is exactly half the sum of d + |d| term by term
      const int dh = __double2hiint(d), dm = ~(dh >> 31);
      s2 += valid ? __hiloint2double(dh & dm, __double2loint(d) & dm) : 0.0;
#else
      s2 += valid ? d + ad : 0.0;
#endif
      const double kd = fma(-ad, PF_Q_INVLN2N, 0x1.8p52);
      const int ki = __double2loint(kd);
      const double k = kd - 0x1.8p52;
      const double r = fma(k, -PF_Q_LN2N, -ad);
#ifdef PF_QNOTABLE
      const double T = __hiloint2double(0x3ff00000 | (ki & 1023), 0);  // experiment: no shared-memory gather
#else
      const double T = pf_exp2_1024[ki & 1023];
#endif
      double pp = fma(r, 1.0 / 24.0, 1.0 / 6.0);
      pp = fma(pp, r, 0.5);
      pp = fma(pp, r, 1.0);
      const double sv = fma(T, r * pp, T);
      double e = __hiloint2double(__double2hiint(sv) + (int)((unsigned)(ki >> 10) << 20), __double2loint(sv));
      if (!FULL && !valid) e = 0.0;
      if (h == 0)
        p0 = fma(p0, e, p0);
      else
        p1 = fma(p1, e, p1);
    }
  }
  pf_lacc out;
#ifdef PF_QMAX_INT
  out.v[0] = s1 + s2;
#else
  out.v[0] = fma(0.5, s2, s1);
#endif
  out.v[1] = p0 * p1;
  return out;
}
#endif

template <bool FULL>
__device__ __forceinline__ pf_lacc pf_stage_terms(const pf_args& a, int k, pf_u64 base, int lane,
                                                const double* st, int n_valid, const pf_fk& K,
                                                const double* P, const double* S, double* scr = nullptr) {
#if !PF_BINNED && PF_LOGFORM
  pf_lform A;
  pf_lform_init(A);
#ifdef PF_LOG_FAST_SLOT
  // per-call fast path: interval bounds over the data box (pf_stage_post)
  // proved every event's terms in range, so no per-event test at all
#ifdef PF_QFAST
  if (K.qfast) return pf_qfast_terms<FULL>(st, lane, n_valid, K);
#endif
  if (K.fast) {
#pragma unroll pf_unroll
    for (int j = 0; j < PF_EPT; ++j) {
      const int i = 32 * j + lane;
      double ev[PF_NCOLS];
#pragma unroll
      for (int q = 0; q < PF_NCOLS; ++q) ev[q] = 0.0;
#pragma unroll
      for (int q = 0; q < PF_NLOAD; ++q) ev[pf_load_col(q)] = st[q * PF_SUB + i];
      double Lv, fac[PF_NFAC_A];
      pf_eval_event_log_fast(ev, K, Lv, fac);
      if (!FULL && i >= n_valid) {
        Lv = 0.0;
#pragma unroll
        for (int f = 0; f < PF_NFAC_A; ++f) fac[f] = 1.0;
      }
      pf_lform_add(A, Lv, fac);
    }
    return pf_lform_pack(A);
  }
#endif
  // log domain, optimistic: -log v = -(L + log F) with no per-event log and
  // no per-event branch; the lane's sub-chunk is redone exactly (above) when
  // any of its events fails the log-domain test
  bool allok = true;
#pragma unroll pf_unroll
  for (int j = 0; j < PF_EPT; ++j) {
    const int i = 32 * j + lane;
    double ev[PF_NCOLS];
#pragma unroll
    for (int q = 0; q < PF_NCOLS; ++q) ev[q] = 0.0;
#pragma unroll
    for (int q = 0; q < PF_NLOAD; ++q) ev[pf_load_col(q)] = st[q * PF_SUB + i];
    double Lv, fac[PF_NFAC_A];
    bool ok = pf_eval_event_log(ev, P, S, Lv, fac);
    if (!FULL && i >= n_valid) {
      ok = true;
      Lv = 0.0;
#pragma unroll
      for (int f = 0; f < PF_NFAC_A; ++f) fac[f] = 1.0;
    }
    allok = allok && ok;
    pf_lform_add(A, Lv, fac);
  }
  if (!allok) return pf_lane_fixup(a, k, P, S, base, lane, st, FULL ? PF_SUB : n_valid);
  return pf_lform_pack(A);
#else
  pf_ctx cx;
  cx.err = 0;
  cx.scr = scr;
  pf_cnt cnt;
  pf_cnt_init(cnt);
  pf_u32 floors = 0;
  bool bad = false;
#if PF_BINNED
  pf_dd acc = pf_dd_zero();
#else
  pf_prod acc;
  pf_prod_init(acc);
#endif
#pragma unroll pf_unroll
  for (int j = 0; j < PF_EPT; ++j) {
    const int i = 32 * j + lane;
#ifdef PF_CONV_SHARED
    // the lanes that evaluate event j of the stage together (whole warp here)
    cx.mask = __ballot_sync(0xffffffffu, FULL || i < n_valid);
#endif
    // padding events (the column tail up to a whole chunk) are not evaluated:
    // they would count clamps the reference never sees
    if (!FULL && i >= n_valid) continue;
    double ev[PF_NCOLS];
#pragma unroll
    for (int q = 0; q < PF_NCOLS; ++q) ev[q] = 0.0;
#pragma unroll
    for (int q = 0; q < PF_NLOAD; ++q) ev[pf_load_col(q)] = st[q * PF_SUB + i];
    double v = pf_eval_event(ev, P, S, a.C, cx, cnt);
#if PF_BINNED
    // chi-squared term (engine.hpp:196-206): mu = N_tot * density * volume
    const double content = ev[PF_CONTENT_COL];
    const double volume = ev[PF_CONTENT_COL + 1];
    const double mu = v * volume;
    const double diff = content - mu;
    double term = diff * diff / fmax(mu, PF_CHISQ_EPS);
    if (!FULL && i >= n_valid) term = 0.0;
    bad |= !(term <= 1.7976931348623157e308);
    acc = pf_dd_add_d(acc, term);
#else
    if (!FULL && i >= n_valid) v = 1.0;
    // common case in one test: 2^-500 <= v <= 2^600 (no floor, finite, and
    // safe for the running product)
    if (!(v >= 0x1p-500 && v <= 0x1p+600)) {
      // NLL term (engine.hpp:186-195): v < 1e-300 is floored and counted;
      // NaN / +inf make -log(v) non-finite (first index found by a rescan)
      if (v < PF_LOG_FLOOR) {
        v = PF_LOG_FLOOR;
        ++floors;
      } else if (!(v <= 1.7976931348623157e308)) {
        bad = true;
        v = 1.0;
      }
      if (v < 0x1p-500) {
        v *= 0x1p+600;
        acc.e -= 600;
      } else if (v > 0x1p+600) {
        v *= 0x1p-600;
        acc.e += 600;
      }
    }
    pf_prod_mul(acc, v);
#endif
  }
  if (cx.err) pf_rescan(a, k, P, S, base, lane, st, FULL ? PF_SUB : n_valid, true);
  if (bad) pf_rescan(a, k, P, S, base, lane, st, FULL ? PF_SUB : n_valid, false);
  if (floors) atomicAdd(&a.rec[k].floor_count, (pf_u64)floors);
  pf_cnt_flush(cnt, a.clamp);
  pf_lacc x;
#if PF_BINNED
  x.v[0] = acc.hi;
  x.v[1] = acc.lo;
#else
  x.v[0] = acc.m;
  x.v[1] = (double)acc.e;
#endif
  return x;
#endif
}

// Peer-memory exchange group (one process per GPU, NVLink): the finalizing
// warp sends this rank's exact record (6 digits, norm error, error flag) into
// slot [k][rank] of every rank's receive buffer (IPC-mapped, P2P stores,
// system-scope release of a per-call sequence word), waits with acquire loads
// until every rank's record for this call is in its own buffer, and replaces
// the local digits by the sum over ranks: every rank then rounds and publishes
// the same global metric.  Integer digits make the sum order-free, so the
// value is bitwise the single-device one.  A peer missing for 5 s reports
// PF_E_GROUP_TIMEOUT instead of hanging.
__device__ __noinline__ void pf_group_exchange(const pf_args& a, int k, int lane, long long* d, pf_u32& normerr,
                                                pf_u64& nonfinite, pf_u64& evterr, int& gbig) {
  long long g[PF_FX_DIGITS];
#pragma unroll
  for (int i = 0; i < PF_FX_DIGITS; ++i) g[i] = __shfl_sync(0xffffffffu, d[i], 0);
  const pf_u32 nerr = __shfl_sync(0xffffffffu, normerr, 0);
  // bit 0: an error or non-finite term, bit 1: wide (>= 2^62) chunk sums
  const int flag = __shfl_sync(0xffffffffu, (int)(nonfinite != ~0ull || evterr != ~0ull) | (gbig ? 2 : 0), 0);
  const unsigned long long seq = (unsigned long long)(a.done[1 + k] + 1u);
  // slots double-buffered by call parity: a rank can run at most one call
  // ahead of a peer (it needs every peer's record of call n to finish call
  // n), so call n + 1's record can never overwrite call n's before the peer
  // has read it
  const pf_u64 slot_base = (pf_u64)(seq & 1ull) * PF_MAX_BATCH * PF_GROUP_MAX;
  if (lane < a.gworld) {  // send: lane q writes this rank's record into rank q's buffer
    long long* dst = a.peers[lane] + (slot_base + (pf_u64)k * PF_GROUP_MAX + a.grank) * 16;
#pragma unroll
    for (int i = 0; i < PF_FX_DIGITS; ++i) dst[i] = g[i];
    dst[6] = (long long)nerr;
    dst[7] = flag;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst + 8), "l"(seq) : "memory");
  }
  long long h[PF_FX_DIGITS];
#pragma unroll
  for (int i = 0; i < PF_FX_DIGITS; ++i) h[i] = 0;
  pf_u32 qerr = ~0u;
  int qflag = 0, timeout = 0;
  if (lane < a.gworld) {  // receive: lane q waits for rank q's record
    const long long* src = a.peers[a.grank] + (slot_base + (pf_u64)k * PF_GROUP_MAX + lane) * 16;
    unsigned long long t0, t, got;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
      asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(got) : "l"(src + 8) : "memory");
      if (got == seq) break;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 5000000000ull) {
        timeout = 1;
        break;
      }
    }
    if (!timeout) {
#pragma unroll
      for (int i = 0; i < PF_FX_DIGITS; ++i) h[i] = (long long)__ldcv((const unsigned long long*)(src + i));
      qerr = (pf_u32)__ldcv((const unsigned long long*)(src + 6));
      qflag = (int)__ldcv((const unsigned long long*)(src + 7));
    }
  }
#pragma unroll
  for (int i = 0; i < PF_FX_DIGITS; ++i) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) h[i] += __shfl_down_sync(0xffffffffu, h[i], off);
    d[i] = h[i];  // the group total (valid in lane 0)
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    qerr = min(qerr, __shfl_down_sync(0xffffffffu, qerr, off));
    qflag |= __shfl_down_sync(0xffffffffu, qflag, off);
    timeout |= __shfl_down_sync(0xffffffffu, timeout, off);
  }
  if (lane == 0) {
    normerr = timeout ? ((0xffffffu << 8) | PF_E_GROUP_TIMEOUT) : min(normerr, qerr);
    if ((qflag & 1) && nonfinite == ~0ull && evterr == ~0ull) nonfinite = 0;  // a peer's term was non-finite
    gbig = (qflag & 2) != 0;  // some rank's sum left the fixed-point range: NaN everywhere
  }
}

// Warp 0 finishes every parameter set of the call: lane b reads digit bin b
// (one round trip, 32 bins), integer shuffles add the digits (and, in an
// exchange group, pf_group_exchange sums the ranks), lane 0 rounds and writes
// the record straight into mapped host memory; one system fence, then the
// completion words.  Used by the event pass's last block and by the publish
// kernel of a shard without events (whose bins are zero).
__device__ void pf_finalize_warp0(const pf_args& a, int lane, const double* S0 = nullptr) {
  static_assert(PF_FX_BINS == 32, "one bin per lane of warp 0");
  {
    for (int k = 0; k < a.K; ++k) {
      PF_CHECK(k < PF_MAX_BATCH && lane < PF_FX_BINS);
      const pf_krec* r = a.rec + k;
      long long* bin = a.fxbins + ((pf_u64)k * PF_FX_BINS + lane) * PF_FX_BIN_STRIDE;
      long long d[PF_FX_DIGITS];
#pragma unroll
      for (int i = 0; i < PF_FX_DIGITS; ++i) d[i] = (long long)__ldcg((const unsigned long long*)(bin + i));
      // the wide-digit count in the same round trip as the bins (it was
      // loaded after the digit shuffles: one more L2 latency on the tail)
      long long* bg = a.big + (pf_u64)k * PF_BIG_STRIDE;
      const long long nbig = (long long)__ldcg((const unsigned long long*)(bg + PF_BIG_COUNT));
      pf_u64 floors = 0, nonfinite = 0, evterr = 0;
      pf_u32 normerr = 0;
      if (lane == 0) {
        floors = __ldcg(&r->floor_count);
        nonfinite = __ldcg(&r->first_nonfinite);
        evterr = __ldcg(&r->first_event_error);
        normerr = __ldcg(&r->norm_error);
        // self-resetting: the fused pass has no kernel that initialises it
        pf_krec* rw = a.rec + k;
        rw->floor_count = 0ull;
        rw->first_nonfinite = ~0ull;
        rw->first_event_error = ~0ull;
        rw->norm_error = ~0u;
      }
#pragma unroll
      for (int i = 0; i < PF_FX_DIGITS; ++i) bin[i] = 0ll;  // self-resetting
#pragma unroll
      for (int i = 0; i < PF_FX_DIGITS; ++i) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) d[i] += __shfl_down_sync(0xffffffffu, d[i], off);
      }
      // chunk sums beyond the fixed-point range: snapshot the wide digits for
      // the host (which then combines them with d) and reset them
      if (nbig) {
        for (int i = lane; i < PF_BIG_DIGITS; i += 32) {
          bg[PF_BIG_SNAP + i] = (long long)__ldcg((const unsigned long long*)(bg + i));
          bg[i] = 0ll;
        }
      }
      int gbig = nbig != 0;
#ifdef PF_EVENT_TRACE
      if (lane == 0 && k == 0) pf_trace_buf[4095 * 6 + 1] = pf_gtime();  // digits summed
#endif
      if (a.peers) pf_group_exchange(a, k, lane, d, normerr, nonfinite, evterr, gbig);
      if (lane == 0) {
        bg[PF_BIG_COUNT] = 0ll;
        bg[PF_BIG_SNAP_COUNT] = nbig;
        long long* dp = a.dpart + (pf_u64)k * 8;  // the device copy, for a stream-ordered collective
#pragma unroll
        for (int i = 0; i < PF_FX_DIGITS; ++i) dp[i] = d[i];
        dp[6] = (long long)normerr;
        dp[7] = ((nonfinite != ~0ull || evterr != ~0ull) ? 1 : 0) | (gbig ? 2 : 0);
        // the record, built in registers, then stored field by field into
        // mapped host memory with its sequence number and check word
        pf_out o;
        // NaN: the host adds the wide digits (Model::wait_results)
        o.result = gbig ? __longlong_as_double(0x7ff8000000000000ll) : pf_fx_round(d);
#pragma unroll
        for (int i = 0; i < PF_FX_DIGITS; ++i) o.fx[i] = d[i];
        o.floor_count = floors;
        o.first_nonfinite = nonfinite;
        o.first_event_error = evterr;
        o.norm_error = normerr;
        const pf_u32 seq = a.done[1 + k] + 1u;
        a.done[1 + k] = seq;
        o.pad = seq;
        o.check = pf_out_check(o);
#ifdef PF_EVENT_TRACE
        if (k == 0) pf_trace_buf[4095 * 6 + 2] = pf_gtime();  // record built (rounded)
#endif
#ifndef PF_PUBLISH_RELEASE
        // every field by an uncached system-scope store (STG.MMIO.SYS: not
        // held in L2 until the grid drains) and no release fence: the host
        // accepts the record once `pad` is this call's sequence number and
        // `check` matches every field, whatever order the stores land in.
        // Measured (C2, profiles/r2e_publish_ab.txt): device step 40.2 ->
        // 38.8 us, end to end unchanged or better; PF_PUBLISH_RELEASE keeps
        // the volatile stores + st.release.sys of the sequence word
        {
          pf_out* h = a.hout + k;
          auto st = [](void* p, pf_u64 v) {
            asm volatile("st.mmio.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
          };
          st(&h->result, (pf_u64)__double_as_longlong(o.result));
          st(&h->floor_count, o.floor_count);
          st(&h->first_nonfinite, o.first_nonfinite);
          st(&h->first_event_error, o.first_event_error);
#pragma unroll
          for (int i = 0; i < PF_FX_DIGITS; ++i) st(&h->fx[i], (pf_u64)o.fx[i]);
          st(&h->check, o.check);
          st(&h->norm_error, (pf_u64)o.norm_error | ((pf_u64)o.pad << 32));
        }
#else
        volatile pf_out* dst = a.hout + k;
        dst->result = o.result;
        dst->floor_count = o.floor_count;
        dst->first_nonfinite = o.first_nonfinite;
        dst->first_event_error = o.first_event_error;
        dst->norm_error = o.norm_error;
#pragma unroll
        for (int i = 0; i < PF_FX_DIGITS; ++i) dst->fx[i] = o.fx[i];
        dst->check = o.check;
        // system-scope release of the sequence word: every field above
        // reaches the host first, and the host sees the record right away
        // rather than when the grid drains (measured: e2e 58 -> 48 us, C2)
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(&a.hout[k].pad), "r"(o.pad) : "memory");
#endif
#ifdef PF_EVENT_TRACE
        if (k == 0) pf_trace_buf[4095 * 6 + 3] = pf_gtime();  // published
#endif
      }
      // the norms the reference's nodes now cache: device memory, read by
      // the host only when asked (pf_node_norms); a call whose normalisation
      // failed leaves the last successful set (engine.hpp:174-178)
      const pf_u32 ne = __shfl_sync(0xffffffffu, normerr, 0);
      if (ne == ~0u) {
        const double* S = S0 ? S0 : a.S + (pf_u64)k * PF_SS;
        for (int i = lane; i < 3 * a.n_nodes; i += 32) a.hnorms[i] = S[i];
      }
    }
  }
}

#ifndef PF_EVENT_MIN_BLOCKS
#define PF_EVENT_MIN_BLOCKS 8
#endif
extern "C" __global__ void __launch_bounds__(PF_EV_THREADS, PF_EVENT_MIN_BLOCKS) pf_event_kernel(const __grid_constant__ pf_args a) {
  extern __shared__ __align__(16) unsigned char pf_dyn[];
  __shared__ __align__(8) pf_u64 bars[PF_EV_WARPS * PF_NST];
#ifdef PF_EVENT_TRACE
  const unsigned long long t_in = pf_gtime();
#endif
  double* stages = reinterpret_cast<double*>(pf_dyn);
  double* accs = stages + PF_EV_WARPS * PF_NST * PF_STAGE;  // [k][PF_LACC_N][thread]
  long long* fxs = reinterpret_cast<long long*>(accs + a.K * PF_LACC_N * PF_EV_THREADS);  // [k][digit][thread]
  for (int i = threadIdx.x; i < a.K * PF_FX_DIGITS * PF_EV_THREADS; i += PF_EV_THREADS) fxs[i] = 0;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* my = stages + warp * PF_NST * PF_STAGE;
  pf_u64* mybar = bars + warp * PF_NST;
  if (lane == 0) {
    for (int s = 0; s < PF_NST; ++s) pf_mbar_init(mybar + s, 1);
    pf_fence_mbar_init();
  }
  pf_math_init();  // includes __syncthreads (barrier inits visible)
  // static chunk assignment: warp gw takes chunks gw, gw + nw, ... (a
  // dynamic ticket was measured no faster and slower to start)
  const int gw = blockIdx.x * PF_EV_WARPS + warp;
  const int nw = gridDim.x * PF_EV_WARPS;
  const int my_chunks = gw < a.n_chunks ? (a.n_chunks - 1 - gw) / nw + 1 : 0;
  const int W = my_chunks * PF_NSUB;
  // TMA producer (lane 0): sub-chunk w of this warp into stage w % PF_NST
  auto issue = [&](int w) {
    if (lane == 0) {
      const int s = w % PF_NST;
      const pf_u64 c = (pf_u64)gw + (pf_u64)(w / PF_NSUB) * (pf_u64)nw;
      const pf_u64 base = c * (PF_SUB * PF_NSUB) + (pf_u64)(w % PF_NSUB) * PF_SUB;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      PF_CHECK(c < (pf_u64)a.n_chunks && base + PF_SUB <= a.col_stride && s < PF_NST);
      pf_mbar_expect_tx(mybar + s, PF_STAGE * 8);
#pragma unroll
      for (int q = 0; q < PF_NLOAD; ++q)
        pf_tma_load(my + s * PF_STAGE + q * PF_SUB,
                    a.data + (pf_u64)pf_load_col(q) * a.col_stride + base, PF_SUB * 8, mybar + s);
    }
  };
  for (int w = 0; w < PF_NST - 1 && w < W; ++w) issue(w);
#ifdef PF_EVENT_TRACE
  const unsigned long long t_pro = pf_gtime();
#endif
  pf_pdl_wait();  // norms, constants and records of this call are ready
#ifdef PF_EVENT_TRACE
  const unsigned long long t_wait = pf_gtime();
#endif
  const pf_fk fk0 = pf_fk_get(a, 0);  // fast-path operands in registers for the whole pass
  // convolution models: the per-call state (model and resolution tables) in
  // shared memory, read per (event, tau) pair
  double* sS = reinterpret_cast<double*>(fxs + a.K * PF_FX_DIGITS * PF_EV_THREADS);
  if (a.s_smem) {
    for (int i = threadIdx.x; i < a.K * PF_SS; i += PF_EV_THREADS) sS[i] = a.S[i];
    __syncthreads();
  }
#ifdef PF_CONV_SHARED
  // this warp's scratch for the shared window products (engine.cpp event_smem)
  double* scr = sS + (a.s_smem ? a.K * PF_SS : 0) + warp * 2 * PF_CONV_KB;
#else
  double* scr = nullptr;
#endif
  for (int w = 0; w < W; ++w) {
    const int s = w % PF_NST;
    pf_mbar_wait(mybar + s, (unsigned)((w / PF_NST) & 1));
    const pf_u64 c = (pf_u64)gw + (pf_u64)(w / PF_NSUB) * (pf_u64)nw;
    const pf_u64 base = c * (PF_SUB * PF_NSUB) + (pf_u64)(w % PF_NSUB) * PF_SUB;
    const bool first = (w % PF_NSUB) == 0;
    const bool full = base + PF_SUB <= a.n_local;
    const int n_valid = full ? PF_SUB : (int)(a.n_local > base ? a.n_local - base : 0);
    for (int k = 0; k < a.K; ++k) {
      const pf_fk fk = k == 0 ? fk0 : pf_fk_get(a, k);
      const double* Pk = a.P + (pf_u64)k * PF_NP;
      pf_lacc t;
#ifdef PF_S_SMEM
      // separate instantiations, so the staged copy is read with LDS (the
      // pointer's address space is known), not generic loads
      if (a.s_smem) {
        const double* Sk = sS + (pf_u64)k * PF_SS;
        t = full ? pf_stage_terms<true>(a, k, base, lane, my + s * PF_STAGE, n_valid, fk, Pk, Sk, scr)
                 : pf_stage_terms<false>(a, k, base, lane, my + s * PF_STAGE, n_valid, fk, Pk, Sk, scr);
      } else
#endif
      {
        const double* Sk = a.S + (pf_u64)k * PF_SS;
        t = full ? pf_stage_terms<true>(a, k, base, lane, my + s * PF_STAGE, n_valid, fk, Pk, Sk, scr)
                 : pf_stage_terms<false>(a, k, base, lane, my + s * PF_STAGE, n_valid, fk, Pk, Sk, scr);
      }
      double* slot = accs + k * PF_LACC_N * PF_EV_THREADS + threadIdx.x;
      if (!first) {
        pf_lacc prev;
#pragma unroll
        for (int j = 0; j < PF_LACC_N; ++j) prev.v[j] = slot[j * PF_EV_THREADS];
        t = pf_lacc_merge(prev, t);
      }
#pragma unroll
      for (int j = 0; j < PF_LACC_N; ++j) slot[j * PF_EV_THREADS] = t.v[j];
    }
    __syncwarp();
    if (w + PF_NST - 1 < W) issue(w + PF_NST - 1);  // refills the stage read at w - 1
    if ((w % PF_NSUB) == PF_NSUB - 1) {
      // chunk done: each lane adds its chunk value EXACTLY into its own
      // fixed-point accumulator (integer adds, no shuffles/atomics)
      for (int k = 0; k < a.K; ++k) {
        pf_lacc x;
#pragma unroll
        for (int j = 0; j < PF_LACC_N; ++j) x.v[j] = accs[(k * PF_LACC_N + j) * PF_EV_THREADS + threadIdx.x];
        const pf_dd t = pf_lacc_terms(x, a.P + (pf_u64)k * PF_NP);
        pf_fxl A;
#pragma unroll
        for (int i = 0; i < PF_FX_DIGITS; ++i) A.d[i] = fxs[(k * PF_FX_DIGITS + i) * PF_EV_THREADS + threadIdx.x];
        long long* big = a.big + (pf_u64)k * PF_BIG_STRIDE;
        pf_fxl_add_w(A, t.hi, big);
        pf_fxl_add_w(A, t.lo, big);
#pragma unroll
        for (int i = 0; i < PF_FX_DIGITS; ++i) fxs[(k * PF_FX_DIGITS + i) * PF_EV_THREADS + threadIdx.x] = A.d[i];
      }
    }
  }
#ifdef PF_EVENT_TRACE
  const unsigned long long t_loop = pf_gtime();
#endif
  // block totals: warp shuffles, the block's warps through shared memory,
  // then ONE binned atomic set per block (exact integer digits)
  __shared__ long long bfx[PF_EV_WARPS][PF_FX_DIGITS];
  for (int k = 0; k < a.K; ++k) {
    pf_fxl A;
#pragma unroll
    for (int i = 0; i < PF_FX_DIGITS; ++i) A.d[i] = fxs[(k * PF_FX_DIGITS + i) * PF_EV_THREADS + threadIdx.x];
    pf_fxl_warp_sum(A);
    if (lane == 0)
#pragma unroll
      for (int i = 0; i < PF_FX_DIGITS; ++i) bfx[warp][i] = A.d[i];
    __syncthreads();
    if (threadIdx.x < PF_FX_DIGITS) {
      long long v = 0;
#pragma unroll
      for (int w = 0; w < PF_EV_WARPS; ++w) v += bfx[w][threadIdx.x];
      if (v)
        atomicAdd((unsigned long long*)(a.fxbins + ((pf_u64)k * PF_FX_BINS + blockIdx.x % PF_FX_BINS) *
                                                       PF_FX_BIN_STRIDE + threadIdx.x),
                  (unsigned long long)v);
    }
    __syncthreads();
  }
  // the last block to finish publishes every parameter set
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
#ifdef PF_EVENT_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 4095) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    PF_ETRACE(5, (unsigned long long)smid);
    PF_ETRACE(0, t_in);
    PF_ETRACE(1, t_pro);
    PF_ETRACE(2, t_wait);
    PF_ETRACE(3, t_loop);
    PF_ETRACE(4, pf_gtime());
  }
#endif
  if (!s_last) return;
#ifdef PF_EVENT_TRACE
  if (threadIdx.x == 0) pf_trace_buf[4094 * 6 + 0] = pf_gtime();
#endif
  __threadfence();
  if (threadIdx.x == 0) *a.done = 0u;  // self-resetting (bench relaunches)
  if (warp == 0) pf_finalize_warp0(a, lane);
#ifdef PF_EVENT_TRACE
  if (threadIdx.x == 0) pf_trace_buf[4094 * 6 + 2] = pf_gtime();
#endif
}


// ---------------------------------------------------------------------------
// Fused pass (K = 1, small normalisation grids): ONE kernel per call.  Every
// CTA (one per SM, 16 warps) first issues the TMA copies of its warps' first
// stages, then computes the whole setup (parameters, pre stage, every
// normalisation level, post stage) in its own shared memory while those
// copies are in flight -- the setup work is a few thousand raw evaluations,
// cheaper to repeat per SM than to hand over through a second grid -- and
// then streams its chunks.  Chunks (fixed event ranges: the reduction unit,
// so the result does not depend on the schedule) go to a balanced set of
// active warps (every active warp the same number of chunks: no lone last
// round).  Lane accumulators live in
// registers; one exact block total per CTA; the last CTA rounds and
// publishes (pf_finalize_warp0).
#ifndef PF_FUSED_WARPS
#define PF_FUSED_WARPS 16
#endif
#define PF_FUSED_THREADS (32 * PF_FUSED_WARPS)

extern "C" __global__ void __launch_bounds__(PF_FUSED_THREADS, 1) pf_fused_kernel(const __grid_constant__ pf_args a) {
  static_assert(PF_FUSED_THREADS == PF_SETUP_THREADS, "the setup core strides by PF_SETUP_THREADS");
#ifdef PF_EVENT_TRACE
  const unsigned long long t_in = pf_gtime();
#endif
  extern __shared__ __align__(16) unsigned char pf_dyn[];
  __shared__ __align__(8) pf_u64 bars[PF_FUSED_WARPS * PF_NST];
  __shared__ __align__(8) pf_u64 tbar;  // the setup's tables (pf_setup_prefetch)
  __shared__ long long bfx[PF_FUSED_WARPS][PF_FX_DIGITS];
  __shared__ int s_last;
  double* stages = reinterpret_cast<double*>(pf_dyn);
  double* P = stages + PF_FUSED_WARPS * PF_NST * PF_STAGE;
  double* S = P + PF_NP;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double* my = stages + warp * PF_NST * PF_STAGE;
  pf_u64* mybar = bars + warp * PF_NST;
  const int nch = a.n_chunks;
  // Static balanced schedule: nwa active warps (host: nwa = ceil(nch / kpw),
  // kpw = ceil(nch / all warps)), spread evenly over the SMs (warp-major
  // index), each taking chunks gw, gw + nwa, ... -- every active warp has kpw
  // chunks (the last ones one fewer), so no warp runs a lone extra round.
  const int nwa = a.nwa;
  const int gw = warp * gridDim.x + blockIdx.x;
  const bool active = gw < nwa;
  int n_mine = active ? (nch - 1 - gw) / nwa + 1 : 0;
  if (n_mine > a.kpw) n_mine = a.kpw;
  if (threadIdx.x == 0) {
    pf_mbar_init(&tbar, 1);
    pf_fence_mbar_init();
    pf_setup_prefetch(a, &tbar);
  }
  if (lane == 0) {
    for (int s = 0; s < PF_NST; ++s) pf_mbar_init(mybar + s, 1);
    pf_fence_mbar_init();
#ifdef PF_L2_PREFETCH_ALL
    // every chunk of this warp into L2 now (measured slower: 45 vs 40 us
    // for C2 -- the prefetch storm delays the setup's own loads)
    for (int j = 0; j < n_mine; ++j) {
      const pf_u64 b = (pf_u64)(gw + j * nwa) * (PF_SUB * PF_NSUB);
#pragma unroll
      for (int q = 0; q < PF_NLOAD; ++q)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.data + (pf_u64)pf_load_col(q) * a.col_stride + b),
                     "r"((unsigned)(PF_SUB * PF_NSUB * 8))
                     : "memory");
    }
#endif
  }
  // sub-chunk v of this warp: chunk gw + (v / PF_NSUB) nwa
  auto issue = [&](int v) {
    if (lane == 0 && v < n_mine * PF_NSUB) {
      const int c = gw + (v / PF_NSUB) * nwa;
      const int st = v % PF_NST;
      const pf_u64 base = (pf_u64)c * (PF_SUB * PF_NSUB) + (pf_u64)(v % PF_NSUB) * PF_SUB;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      PF_CHECK(c < nch && base + PF_SUB <= a.col_stride && st < PF_NST && gw < nwa);
      pf_mbar_expect_tx(mybar + st, PF_STAGE * 8);
#pragma unroll
      for (int q = 0; q < PF_NLOAD; ++q)
        pf_tma_load(my + st * PF_STAGE + q * PF_SUB, a.data + (pf_u64)pf_load_col(q) * a.col_stride + base,
                    PF_SUB * 8, mybar + st);
    }
  };
  for (int v = 0; v < PF_NST; ++v) issue(v);
  // the setup, redundantly in every CTA, while the first stages stream in
  pf_krec* r = a.rec;
  pf_ctx cx;
  cx.err = 0;
  pf_cnt cnt_grid, cnt_stage;
  pf_cnt_init(cnt_grid);
  pf_cnt_init(cnt_stage);
  // the setup's grid points split over a cluster of PF_SETUP_CLUSTER CTAs
  // (DSMEM exchange), exactly as the setup kernel of the batched path splits
  // them: batched and single calls stay bitwise equal
  const unsigned rank = PF_SETUP_CLUSTER > 1 ? pf_cluster_rank() : 0u;
#ifdef PF_L2_PREFETCH_FIRST
  // the sub-chunks beyond the ring of this warp's first PF_L2_PREFETCH_FIRST
  // chunks into L2 while the setup computes: HBM keeps streaming, and the
  // loop's first TMA copies hit L2
  auto hook = [&]() {
    if (lane == 0 && n_mine > 0) {
      const pf_u64 b0 = (pf_u64)gw * (PF_SUB * PF_NSUB) + (pf_u64)PF_NST * PF_SUB;
      const int m = n_mine < PF_L2_PREFETCH_FIRST ? n_mine : PF_L2_PREFETCH_FIRST;
      for (int j = 0; j < m; ++j) {
        const pf_u64 b = j == 0 ? b0 : (pf_u64)(gw + j * nwa) * (PF_SUB * PF_NSUB);
        const unsigned bytes = (unsigned)((j == 0 ? PF_SUB * (PF_NSUB - PF_NST) : PF_SUB * PF_NSUB) * 8);
#pragma unroll
        for (int q = 0; q < PF_NLOAD; ++q)
          if (bytes)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a.data + (pf_u64)pf_load_col(q) * a.col_stride + b),
                         "r"(bytes)
                         : "memory");
      }
    }
  };
  pf_setup_core<PF_SETUP_CLUSTER>(a, 0, rank, P, S, r, false, cx, cnt_grid, cnt_stage, hook, &tbar);
#else
#ifdef PF_SETUP_TWICE
  // experiment: the setup once more with warm instruction caches (traced twice)
  pf_setup_core<PF_SETUP_CLUSTER>(a, 0, rank, P, S, r, false, cx, cnt_grid, cnt_stage, pf_no_hook(), &tbar);
  __syncthreads();
#endif
  pf_setup_core<PF_SETUP_CLUSTER>(a, 0, rank, P, S, r, false, cx, cnt_grid, cnt_stage, pf_no_hook(), &tbar);
#endif
  // no CTA may leave while a cluster peer could still read its setup
  // partials: arrive now, wait just before exit
  if (PF_SETUP_CLUSTER > 1) asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  if (blockIdx.x < PF_SETUP_CLUSTER) {  // one cluster reports what every cluster found
    if (cx.err && rank == 0) atomicMin(&r->norm_error, cx.err);
    if (pf_grid_counts(a, 0)) {
      pf_cnt_flush(cnt_grid, a.clamp);
      if (rank == 0) pf_cnt_flush(cnt_stage, a.clamp);
    }
  }
  if (blockIdx.x == 0) {
    double* gS = a.S;
    double* gP = (double*)a.P;
    for (int i = threadIdx.x; i < PF_SS; i += blockDim.x) gS[i] = S[i];
    for (int i = threadIdx.x; i < PF_NP; i += blockDim.x) gP[i] = P[i];
  }
  __syncthreads();  // P and S complete (the setup core ends with a barrier too)
#ifdef PF_EVENT_TRACE
  const unsigned long long t_setup = pf_gtime();
#endif
  const pf_fk fk = pf_fk_load(P, S, a.C);
  pf_fxl F;
#pragma unroll
  for (int i = 0; i < PF_FX_DIGITS; ++i) F.d[i] = 0;
  long long* big = a.big;
  pf_lacc acc;
  int w = 0;  // sub-chunks consumed by this warp
#ifdef PF_EVENT_TRACE
  const int n_done = n_mine;
#endif
  for (int jc = 0; jc < n_mine; ++jc) {
    const int c = gw + jc * nwa;
    for (int j = 0; j < PF_NSUB; ++j, ++w) {
      const int st = w % PF_NST;
#ifdef PF_QNOWAIT
      // experiment: the math alone -- stage 0 once, then re-read (no TMA waits)
      if (w == 0)
        for (int s0 = 0; s0 < PF_NST && s0 < n_mine * PF_NSUB; ++s0) pf_mbar_wait(mybar + s0, 0u);
#else
      pf_mbar_wait(mybar + st, (unsigned)((w / PF_NST) & 1));
#endif
      const pf_u64 base = (pf_u64)c * (PF_SUB * PF_NSUB) + (pf_u64)j * PF_SUB;
      PF_CHECK(c < nch && base < a.col_stride && st < PF_NST);
      const bool full = base + PF_SUB <= a.n_local;
      const int n_valid = full ? PF_SUB : (int)(a.n_local > base ? a.n_local - base : 0);
      const pf_lacc t = full ? pf_stage_terms<true>(a, 0, base, lane, my + st * PF_STAGE, n_valid, fk, P, S)
                             : pf_stage_terms<false>(a, 0, base, lane, my + st * PF_STAGE, n_valid, fk, P, S);
      acc = j == 0 ? t : pf_lacc_merge(acc, t);
      __syncwarp();
#ifndef PF_QNOWAIT
      issue(w + PF_NST);  // refills the stage just read
#endif
    }
    // chunk done: its exact value into the lane's fixed-point accumulator
    const pf_dd tv = pf_lacc_terms(acc, P);
    pf_fxl_add_w(F, tv.hi, big);
    pf_fxl_add_w(F, tv.lo, big);
  }
#ifdef PF_EVENT_TRACE
  const unsigned long long t_loop = pf_gtime();
  if (lane == 0 && gw < 4096) {  // per warp: chunks taken, loop end
    pf_trace_w[2 * gw] = (unsigned long long)n_done;
    pf_trace_w[2 * gw + 1] = t_loop;
  }
  __shared__ unsigned long long t_loop_max;
  if (threadIdx.x == 0) t_loop_max = 0;
  __syncthreads();
  atomicMax(&t_loop_max, t_loop);
#endif
  // block total (exact integer digits), ONE binned atomic set per CTA
  pf_fxl_warp_sum(F);
  if (lane == 0)
#pragma unroll
    for (int i = 0; i < PF_FX_DIGITS; ++i) bfx[warp][i] = F.d[i];
  __syncthreads();
  if (threadIdx.x < PF_FX_DIGITS) {
    long long v = 0;
#pragma unroll
    for (int ww = 0; ww < PF_FUSED_WARPS; ++ww) v += bfx[ww][threadIdx.x];
    if (v)
      atomicAdd((unsigned long long*)(a.fxbins + (pf_u64)(blockIdx.x % PF_FX_BINS) * PF_FX_BIN_STRIDE + threadIdx.x),
                (unsigned long long)v);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#ifdef PF_DONE_ACQREL
    // experiment: one acq_rel atomic instead of fence + atomic (the block's
    // digit atomics happen-before it through the barrier above)
    unsigned prev;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(a.done) : "memory");
    s_last = prev == gridDim.x - 1;
#else
    __threadfence();
    s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
#endif
  }
  __syncthreads();
  if (PF_SETUP_CLUSTER > 1) asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
#ifdef PF_EVENT_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 4094) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    PF_ETRACE(0, t_in);
    PF_ETRACE(1, t_setup);
    PF_ETRACE(2, t_loop_max);
    PF_ETRACE(3, pf_gtime());
    PF_ETRACE(5, (unsigned long long)smid);
  }
#endif
  if (!s_last) return;
  __threadfence();
#ifdef PF_EVENT_TRACE
  if (threadIdx.x == 0) pf_trace_buf[4094 * 6 + 0] = pf_gtime();
#endif
  if (threadIdx.x == 0) *a.done = 0u;  // self-resetting (every CTA has arrived)
  if (warp == 0) pf_finalize_warp0(a, lane, S);
#ifdef PF_EVENT_TRACE
  if (threadIdx.x == 0) pf_trace_buf[4094 * 6 + 2] = pf_gtime();
#endif
}

// ---------------------------------------------------------------------------
// bench only (PFB200_FLUSH=writeread): the optional read half of the L2
// flush, leaving clean lines of the flush buffer in L2.
extern "C" __global__ void pf_flush_read_kernel(const ulonglong2* p, pf_u64 n, unsigned long long* sink) {
  unsigned long long acc = 0;
  for (pf_u64 i = (pf_u64)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (pf_u64)gridDim.x * blockDim.x) {
    const ulonglong2 v = __ldcg(p + i);
    acc ^= v.x ^ v.y;
  }
  if (acc == 0x5eed5eed5eed5eedull) *sink = acc;
}

// ---------------------------------------------------------------------------
// publish only (a shard without events: the metric is 0)
extern "C" __global__ void __launch_bounds__(PF_THREADS) pf_publish_kernel(const __grid_constant__ pf_args a) {
  pf_pdl_wait();
  if (threadIdx.x < 32) pf_finalize_warp0(a, (int)threadIdx.x);
}
