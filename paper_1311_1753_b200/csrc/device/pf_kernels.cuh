// pf_kernels.cuh — kernel bodies of the per-call CUDA graph.
//
// Included by the generated evaluator AFTER it has defined:
//   PF_NP, PF_SS, PF_NCOLS, PF_NLOAD, PF_EPT, PF_BINNED, PF_NPOLY,
//   pf_load_col(q) (data columns read per event),
//   pf_stage_pre(k, P, S, C, cx, tid, nt)       parameter-derived constants
//   pf_stage_post(level, k, P, S, C, cx, tid, nt) constants needing norms
//   pf_norm_point(node, flat, task, P, S, C, cx)  raw at one grid midpoint
//   pf_eval_event(ev, P, S, C, cx)               normalised density (NLL) or
//                                                 N_tot * density (chi2)
//   pf_norm_nodes_of_level(level, nodes[]), PF_NORM_COUNT(level)
//
// Launch sequence per call (engine.cpp):  pre -> norm(level 0..L) -> event
// -> final.  Every reduction has a fixed shape, so a call is bitwise
// reproducible and independent of the number of devices.

// ---------------------------------------------------------------------------
// pre: initialise the call record and the parameter-derived constants.
extern "C" __global__ void __launch_bounds__(PF_THREADS) pf_pre_kernel(pf_args a) {
  const int k = blockIdx.x;
  pf_krec* r = a.rec + k;
  if (threadIdx.x == 0) {
    r->floor_count = 0ull;
    r->first_nonfinite = ~0ull;
    r->first_event_error = ~0ull;
    r->norm_error = ~0u;
    for (int i = 0; i <= PF_MAX_LEVELS; ++i) r->arrive[i] = 0u;
    r->result_hi = 0.0;
    r->result_lo = 0.0;
  }
  __syncthreads();
  pf_ctx cx;
  cx.err = 0;
  pf_cnt cnt;
  pf_cnt_init(cnt);
  pf_stage_pre(k, a.P + (pf_u64)k * PF_NP, a.S + (pf_u64)k * PF_SS, a.C, cx, cnt,
               threadIdx.x, blockDim.x);
  if (cx.err) atomicMin(&r->norm_error, cx.err);
  pf_cnt_flush(cnt, a.clamp);
}

// ---------------------------------------------------------------------------
// norm: midpoint sums at n and 2n per box dimension for every normalised node
// of one level (pdf.hpp:148-176), Richardson combination (pdf.hpp:178-188)
// by the last block to arrive, then the post-level constants.
extern "C" __global__ void __launch_bounds__(PF_THREADS) pf_norm_kernel(pf_args a) {
  __shared__ pf_dd sm[PF_THREADS];
  __shared__ int s_last;
  const int k = blockIdx.y;
  const double* P = a.P + (pf_u64)k * PF_NP;
  double* S = a.S + (pf_u64)k * PF_SS;
  // one partial per block: task t owns [first_block, first_block + n_blocks)
  pf_dd* part = a.partials + (pf_u64)k * gridDim.x;
  // locate this block's task (n_tasks is small)
  int t = 0;
  while (t + 1 < a.n_tasks && (int)blockIdx.x >= a.tasks[t + 1].first_block) ++t;
  const pf_task& T = a.tasks[t];
  const pf_u64 b = (pf_u64)((int)blockIdx.x - T.first_block);
  const pf_u64 lo = b * T.per_block;
  const pf_u64 hi = min(lo + T.per_block, T.points);
  pf_ctx cx;
  cx.err = 0;
  pf_cnt cnt;
  pf_cnt_init(cnt);
  pf_dd acc = pf_dd_zero();
  for (pf_u64 i = lo + threadIdx.x; i < hi; i += PF_THREADS)
    acc = pf_dd_add_d(acc, pf_norm_point(T.node, i, T, P, S, a.C, cx, cnt));
  sm[threadIdx.x] = acc;
  __syncthreads();
  if (threadIdx.x < 32) {
    pf_dd s = pf_warp_reduce_runs(sm, PF_THREADS);
    if (threadIdx.x == 0) part[blockIdx.x] = s;
  }
  if (cx.err) atomicMin(&a.rec[k].norm_error, cx.err);
  pf_cnt_flush(cnt, a.clamp);
  // last block of this (level, k) finalises
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned prev = atomicAdd(&a.rec[k].arrive[a.level], 1u);
    s_last = (prev == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  __shared__ double sums[64];
  for (int tt = 0; tt < a.n_tasks; ++tt) {
    const pf_task& U = a.tasks[tt];
    const pf_dd* pv = part + U.first_block;
    if (threadIdx.x < 32) {
      pf_dd s = pf_warp_reduce_runs(pv, U.n_blocks);
      // midpoint_sum returns static_cast<double>(sum) * vol (pdf.hpp:173-175)
      if (threadIdx.x == 0) sums[tt] = __dmul_rn(pf_dd_to_double(s), U.vol);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // tasks come in (coarse, fine) pairs per node
    for (int tt = 0; tt + 1 < a.n_tasks; tt += 2) {
      const int node = a.tasks[tt].node;
      const double coarse = sums[tt], fine = sums[tt + 1];
      const double norm = fine + (fine - coarse) / 3.0;
      const double err = fabs(fine - coarse) / 3.0;
      S[3 * node + 0] = norm;
      S[3 * node + 1] = err;
      S[3 * node + 2] = 1.0 / norm;
      if (!(norm > 0.0) || !isfinite(norm))
        atomicMin(&a.rec[k].norm_error, ((pf_u32)node << 8) | PF_E_ZERO_INTEGRAL);
    }
  }
  __syncthreads();
  pf_ctx cx2;
  cx2.err = 0;
  pf_cnt cnt2;
  pf_cnt_init(cnt2);
  pf_stage_post(a.level, k, P, S, a.C, cx2, cnt2, threadIdx.x, blockDim.x);
  if (cx2.err) atomicMin(&a.rec[k].norm_error, cx2.err);
  pf_cnt_flush(cnt2, a.clamp);
}

// ---------------------------------------------------------------------------
// event pass: PF_EPT events per thread, PF_THREADS * PF_EPT per chunk.  Data
// are read once per chunk and reused for every parameter set k.
extern "C" __global__ void __launch_bounds__(PF_THREADS) pf_event_kernel(pf_args a) {
  extern __shared__ pf_dd smk[];  // K x PF_THREADS
  const int tid = threadIdx.x;
  const int warp = tid >> 5;
  for (int c = blockIdx.x; c < a.n_chunks; c += gridDim.x) {
    const pf_u64 base = (pf_u64)c * (PF_THREADS * PF_EPT);
    double val[PF_NLOAD][PF_EPT];
    bool ok[PF_EPT];
    const bool full = base + (pf_u64)(PF_THREADS * PF_EPT) <= a.n_local;
#if PF_EPT >= 2
#pragma unroll
    for (int i = 0; i < PF_EPT / 2; ++i) {
      const pf_u64 e = base + 2ull * (pf_u64)(tid + PF_THREADS * i);
      ok[2 * i] = full || e < a.n_local;
      ok[2 * i + 1] = full || e + 1 < a.n_local;
#pragma unroll
      for (int q = 0; q < PF_NLOAD; ++q) {
        const double* col = a.data + (pf_u64)pf_load_col(q) * a.col_stride;
        if (full) {
          double2 w = __ldg(reinterpret_cast<const double2*>(col + e));
          val[q][2 * i] = w.x;
          val[q][2 * i + 1] = w.y;
        } else {
          val[q][2 * i] = ok[2 * i] ? __ldg(col + e) : 0.0;
          val[q][2 * i + 1] = ok[2 * i + 1] ? __ldg(col + e + 1) : 0.0;
        }
      }
    }
#else
    {
      const pf_u64 e = base + (pf_u64)tid;
      ok[0] = e < a.n_local;
#pragma unroll
      for (int q = 0; q < PF_NLOAD; ++q) {
        const double* col = a.data + (pf_u64)pf_load_col(q) * a.col_stride;
        val[q][0] = ok[0] ? __ldg(col + e) : 0.0;
      }
    }
#endif
    for (int k = 0; k < a.K; ++k) {
      const double* P = a.P + (pf_u64)k * PF_NP;
      const double* S = a.S + (pf_u64)k * PF_SS;
      pf_ctx cx;
      cx.err = 0;
      pf_cnt cnt;
      pf_cnt_init(cnt);
      pf_u32 floors = 0;
#if PF_BINNED
      pf_dd acc = pf_dd_zero();
#else
      pf_prod acc;
      pf_prod_init(acc);
#endif
#pragma unroll
      for (int j = 0; j < PF_EPT; ++j) {
        if (!ok[j]) continue;
#if PF_EPT >= 2
        const pf_u64 e = base + 2ull * (pf_u64)(tid + PF_THREADS * (j >> 1)) + (pf_u64)(j & 1);
#else
        const pf_u64 e = base + (pf_u64)tid;
#endif
        double ev[PF_NCOLS];
#pragma unroll
        for (int q = 0; q < PF_NCOLS; ++q) ev[q] = 0.0;
#pragma unroll
        for (int q = 0; q < PF_NLOAD; ++q) ev[pf_load_col(q)] = val[q][j];
        pf_u32 err0 = cx.err;
        double v = pf_eval_event(ev, P, S, a.C, cx, cnt);
        if (cx.err != err0 && err0 == 0) {
          const pf_u64 g = a.event_offset + e;
          atomicMin(&a.rec[k].first_event_error, (g << 24) | (pf_u64)cx.err);
        }
#if PF_BINNED
        // chi-squared term (engine.hpp:196-206): mu = N_tot * density * volume
        const double content = ev[PF_CONTENT_COL];
        const double volume = ev[PF_CONTENT_COL + 1];
        const double mu = v * volume;
        const double diff = content - mu;
        const double term = diff * diff / fmax(mu, PF_CHISQ_EPS);
        if (!isfinite(term)) atomicMin(&a.rec[k].first_nonfinite, a.event_offset + e);
        acc = pf_dd_add_d(acc, term);
#else
        // NLL term (engine.hpp:186-195): floor at 1e-300, counted
        if (v < PF_LOG_FLOOR) {
          v = PF_LOG_FLOOR;
          ++floors;
        } else if (!(v <= 1.7976931348623157e308)) {
          // +inf or NaN: -log(v) is not finite
          atomicMin(&a.rec[k].first_nonfinite, a.event_offset + e);
          v = 1.0;
        }
        pf_prod_mul(acc, v);
#endif
      }
#if PF_BINNED
      smk[k * PF_THREADS + tid] = acc;
#else
      smk[k * PF_THREADS + tid] = pf_prod_neglog(acc);
#endif
      if (floors) atomicAdd(&a.rec[k].floor_count, (pf_u64)floors);
      pf_cnt_flush(cnt, a.clamp);
    }
    __syncthreads();
    for (int k = warp; k < a.K; k += PF_THREADS / 32) {
      pf_dd s = pf_warp_reduce_runs(smk + k * PF_THREADS, PF_THREADS);
      if ((tid & 31) == 0) a.partials[(pf_u64)k * a.n_chunks + c] = s;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// final: the reference's pairwise tree over chunk partials, one block per k.
extern "C" __global__ void __launch_bounds__(PF_FINAL_THREADS) pf_final_kernel(pf_args a) {
  __shared__ pf_dd sm[PF_FINAL_THREADS];
  const int k = blockIdx.x;
  pf_dd r = pf_pairwise_block(a.partials + (pf_u64)k * a.n_chunks, (pf_u64)a.n_chunks, sm);
  if (threadIdx.x == 0) {
    a.rec[k].result_hi = r.hi;
    a.rec[k].result_lo = r.lo;
  }
}
