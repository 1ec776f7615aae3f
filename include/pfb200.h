/*
 * pfb200.h — C ABI of the B200-native likelihood-evaluation engine.
 *
 * This is the drop-in boundary for the hot path of the reference `parfit`
 * (GooFit re-architecture, /root/reference/proj/include/parfit/).  Every
 * entry point replaces one reference interface; the citation is given per
 * function.  Plain C types only: pointers, sizes, fixed-width integers.
 *
 * Ownership: the caller owns every input buffer; pf_model_create copies the
 * event table into HBM (the reference copies it into its EventTable,
 * engine.hpp:143,151) and the model owns all device state afterwards.
 *
 * Errors: functions return 0 on success, nonzero on failure, and fill
 * `pf_status.message` with the reference's stable "code: detail" text
 * (errors.hpp:9-16), e.g. "non-finite-metric: first offending event index 7".
 *
 * Threading: a model may move between threads but evaluates one call at a
 * time (engine.hpp:134-136).  pf_eval_metric blocks until the scalar is on
 * the host, exactly like BoundModel::eval_metric.
 */
#ifndef PFB200_H
#define PFB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PF_ABI_VERSION 1

#if defined(__GNUC__)
#define PF_API __attribute__((visibility("default")))
#else
#define PF_API
#endif

/* Node kinds: pdf.hpp:20-30 (Exponential..Convolution) plus ArgusPdf and
 * DalitzPlotPdf, which the reference lacks (BASELINE configs 3 and 5; see
 * DESIGN.md).  DalitzPlotPdf: obs = {m^2_12, m^2_13}; params = per resonance
 * {mass, width, Re c, Im c}; reals = {M, m1, m2, m3, R, then per resonance
 * channel (12, 13 or 23) and spin (0 or 1)}.
 * TddpPdf (time-dependent Dalitz, BASELINE config 5): obs = {m^2_12, m^2_13,
 * t}; params = the DalitzPlotPdf resonance params, then {tau, x, y}; reals =
 * the DalitzPlotPdf reals (m1 == m2: daughters 1 and 2 CP conjugates).
 * Density |A g+(t) + Abar g-(t)|^2 =
 *   e^-(t/tau) [ (|A|^2 + |Abar|^2)/2 cosh(y t/tau) + (|A|^2 - |Abar|^2)/2 cos(x t/tau)
 *                - Re(A* Abar) sinh(y t/tau) - Im(A* Abar) sin(x t/tau) ],
 * Abar(s12, s13) = A(s12, s23) (the CP-mirrored point). */
enum pf_kind {
  PF_EXPONENTIAL = 0,
  PF_GAUSSIAN = 1,
  PF_BREIT_WIGNER = 2,
  PF_POLYNOMIAL = 3,
  PF_PRODUCT = 4,
  PF_SUM = 5,
  PF_COMPOSITE = 6,
  PF_MAPPED = 7,
  PF_CONVOLUTION = 8,
  PF_ARGUS = 9,
  PF_DALITZ = 10,
  PF_TDDP = 11
};

/* MetricKind, engine.hpp:48 */
enum pf_metric { PF_NLL = 0, PF_CHISQ = 1 };

/* Role, variable.hpp:13 */
enum pf_role { PF_OBSERVABLE = 0, PF_PARAMETER = 1 };

/* Variable, variable.hpp:18-27.  Identity is the index in pf_graph.variables:
 * two nodes naming the same index share one registry slot. */
typedef struct pf_variable {
  const char* name;
  double value;
  double lower;
  double upper;
  double step;
  int32_t fixed;
  int32_t role; /* pf_role */
} pf_variable;

/* One PdfNode (pdf.hpp:61-205) as declared by the user, before finalize.
 *   children: node indices (ProdPdf/AddPdf order; Composite = {outer, inner};
 *             Convolution = {model, resolution}; Mapped = targets)
 *   params:   variable indices in node-local declaration order
 *   obs:      variable indices (primitives only)
 *   reals:    MappedPdf boundaries (n_children + 1 strictly increasing values)
 *   quadrature_points: ConvolutionPdf Q (pdf.hpp:464-466), 0 otherwise. */
typedef struct pf_node {
  int32_t kind; /* pf_kind */
  const char* name;
  int32_t n_children;
  const int32_t* children;
  int32_t n_params;
  const int32_t* params;
  int32_t n_obs;
  const int32_t* obs;
  int32_t n_reals;
  const double* reals;
  int64_t quadrature_points;
} pf_node;

typedef struct pf_graph {
  int32_t n_variables;
  const pf_variable* variables;
  int32_t n_nodes;
  const pf_node* nodes;
  int32_t root;
} pf_graph;

/* The flat column-major EventTable (dataset.hpp:135-182).
 * Unbinned: n_obs columns.  Binned: n_obs bin-centre columns, then content,
 * then volume (to_event_table, dataset.hpp:161-182); total_content is
 * BinnedDataSet::total_content() (dataset.hpp:356-358). */
typedef struct pf_data {
  int32_t binned;
  int32_t n_obs;
  const int32_t* obs; /* variable indices in column order */
  uint64_t n_events;  /* events, or bins */
  const double* values;
  double total_content;
} pf_data;

/* Device placement / sharding.
 *   device:        CUDA ordinal of the first device.
 *   n_devices:     >1 shards events over devices device..device+n-1 in this
 *                  process (contiguous subtrees of the reduction tree).
 *   shard_index/shard_count: this process evaluates only the contiguous
 *                  chunk range shard_index of shard_count (power of two);
 *                  pf_eval_partial returns its exact accumulator and
 *                  pf_combine_partials reproduces the global value.
 *                  shard_count = 1: whole data set.
 *   oversubscribe: 1 lets n_devices exceed the visible devices: shard s
 *                  runs on device (device + s) mod count.  The shards still
 *                  combine on the host (no kernel waits on another), so this
 *                  exercises the multi-device path on a one-GPU box; 0 (the
 *                  default) rejects a count above the visible devices. */
typedef struct pf_options {
  int32_t device;
  int32_t n_devices;
  int32_t shard_index;
  int32_t shard_count;
  int32_t verbose;
  int32_t oversubscribe;
  int32_t reserved[2];
} pf_options;

/* number of CUDA devices visible to this process (cudaGetDeviceCount; 0
 * when the driver reports none) */
PF_API int32_t pf_device_count(void);

typedef struct pf_status {
  int32_t code; /* 0 ok */
  char message[512];
} pf_status;

/* Per-call diagnostics returned alongside the metric. */
typedef struct pf_eval_info {
  uint64_t log_floor_delta; /* events floored at 1e-300 in this call */
  int32_t penalty;          /* 1 when the 1e300 penalty was returned */
  int32_t norms_recomputed; /* always 1: norms are recomputed every call on
                               the device (the reference's fingerprint,
                               pdf.hpp:40-51, misses on any param change) */
} pf_eval_info;

typedef struct pf_model pf_model;

/* ---- model-core: finalize without a device ------------------------------ */

/* GraphFinalizer::finalize (pdf.hpp:504-613) on the host only: validates the
 * graph, assigns pre-order ids, fills the registry order and the IndexTable.
 *   reserved_columns: 2 for binned data sets (engine.hpp:149)
 *   param_order[n]:  variable index of registry slot i (capacity cap_params)
 *   table/table_len: concatenated IndexTable rows (index_table.hpp:12-16)
 *   n_columns:       data + reserved + synthetic columns.
 * Returns the number of parameters through *n_params. */
PF_API int pf_graph_finalize(const pf_graph* graph, int32_t n_data_obs, const int32_t* data_obs,
                      int32_t reserved_columns, int32_t* param_order, int32_t cap_params,
                      int32_t* n_params, uint32_t* table, int32_t cap_table,
                      int32_t* table_len, int32_t* n_columns, pf_status* status);

/* Generated per-model CUDA source (the fused evaluator) for inspection and
 * for the NVRTC compile check that runs without a GPU.  Writes at most cap
 * bytes (NUL-terminated) and the full length to *len. */
PF_API int pf_graph_codegen(const pf_graph* graph, const pf_data* data, uint32_t grid_points,
                     char* out, size_t cap, size_t* len, pf_status* status);

/* Compiles the generated source for sm_100a with NVRTC (no GPU needed) and
 * returns the cubin size; used by build() and the CPU tests. */
PF_API int pf_graph_compile_check(const pf_graph* graph, const pf_data* data,
                           uint32_t grid_points, size_t* cubin_bytes, pf_status* status);

/* ---- parallel-engine: the hot path -------------------------------------- */

/* BoundModel(pdf, data, GridSpec) — engine.hpp:139-154 (setData).
 * Finalizes the graph, uploads the EventTable to HBM in SoA layout, compiles
 * the fused evaluator for sm_100a and captures the per-call CUDA graphs. */
PF_API int pf_model_create(const pf_graph* graph, const pf_data* data, uint32_t grid_points,
                    const pf_options* options, pf_model** out, pf_status* status);

PF_API void pf_model_destroy(pf_model* model);

/* BoundModel::n_events / registry().n_parameters (engine.hpp:156-162). */
PF_API uint64_t pf_model_n_events(const pf_model* model);
PF_API int32_t pf_model_n_params(const pf_model* model);
/* variable index (into pf_graph.variables) of registry slot i */
PF_API int32_t pf_model_param_variable(const pf_model* model, int32_t slot);
PF_API int32_t pf_model_n_nodes(const pf_model* model);
PF_API int32_t pf_model_binned(const pf_model* model);

/* BoundModel::eval_metric(params, metric, backend) — engine.hpp:165-218. */
PF_API int pf_eval_metric(pf_model* model, const double* params, size_t n_params, int32_t metric,
                   double* out, pf_eval_info* info, pf_status* status);

/* K parameter vectors (row-major K x n_params) in one pass over the events:
 * out[k] equals pf_eval_metric(params + k*n_params) bit for bit.  Serves the
 * independent probes of numeric_gradient / numeric_hessian (fit.hpp:138-208). */
PF_API int pf_eval_metric_batch(pf_model* model, const double* params, size_t k, size_t n_params,
                         int32_t metric, double* out, pf_status* status);

/* The metric is accumulated EXACTLY in a fixed-point superaccumulator of
 * PF_FX_DIGITS signed 64-bit digits (value = sum_i d_i 2^(32 i - 128)) and
 * rounded once, so it does not depend on summation order or sharding.
 * Chunk sums of 2^62 or more (chi-squared far from the data) go to a wider
 * device-side accumulator that pf_eval_metric / pf_eval_metric_batch fold in
 * on the host; the partial and exchange-group paths carry only the six
 * digits and fail such a call with "metric-overflow". */
#define PF_FX_DIGITS 6

/* This process's shard accumulator (PF_FX_DIGITS digits), for multi-process
 * sharding; *penalty set when the 1e300 penalty applies. */
PF_API int pf_eval_partial(pf_model* model, const double* params, size_t n_params, int32_t metric,
                           int64_t* partial_fx, int32_t* penalty, pf_status* status);

/* Multi-process exchange without a host round trip (single-device models):
 * pf_eval_launch enqueues one evaluation on the model's stream and returns
 * at once (*penalty set, nothing enqueued, when the parameters are invalid).
 * The event pass also writes a device record of 8 int64 at
 * pf_model_partial_device(): the PF_FX_DIGITS exact digits, the norm error
 * word (~0u when none) and a flag word: bit 0 a non-finite term or event
 * error, bit 1 chunk sums beyond the six digits (see PF_FX_DIGITS).
 * A collective enqueued on pf_model_stream() (cudaStream_t as an integer)
 * after the launch sees the record. */
PF_API int pf_eval_launch(pf_model* model, const double* params, size_t n_params, int32_t metric,
                          int32_t* penalty, pf_status* status);
PF_API uint64_t pf_model_stream(const pf_model* model);
PF_API uint64_t pf_model_partial_device(const pf_model* model);

/* Exchange group over peer memory (one process per GPU on one NVLink node):
 * every rank exports its model's receive buffer (pf_group_handle: a 64-byte
 * CUDA IPC handle), the handles are all-gathered by the caller (any
 * transport), and every rank calls pf_group_join with all of them, then
 * barriers.  From then on each evaluation's event pass stores its exact
 * record into every rank's buffer over NVLink and sums the group's digits on
 * the device: pf_eval_metric returns the GLOBAL metric on every rank, bitwise
 * the single-device value, with no host collective.  All ranks must issue the
 * same sequence of evaluations (as a fit does). */
PF_API int pf_group_handle(pf_model* model, void* handle64, pf_status* status);
PF_API int pf_group_join(pf_model* model, int32_t world, int32_t rank, const void* handles, pf_status* status);

/* Exact combine of shard_count accumulators (shard_count x PF_FX_DIGITS) and
 * the correctly rounded metric: bitwise the single-device value. */
PF_API double pf_combine_partials(const int64_t* partials_fx, int32_t shard_count);

/* PdfNode::cached_norm / norm_error_estimate (pdf.hpp:88-92) for every node
 * in pre-order; valid[i] = 0 where the reference would throw
 * "stale-normalization" (nodes that are never normalised). */
PF_API int pf_node_norms(pf_model* model, double* norms, double* errs, int32_t* valid, int32_t n_nodes);

/* BoundModel::log_floor_count (engine.hpp:163) and
 * PolynomialPdf::clamp_count (pdf.hpp:320), cumulative. */
PF_API uint64_t pf_log_floor_count(const pf_model* model);
PF_API uint64_t pf_clamp_count(const pf_model* model, int32_t node);

/* ---- measurement ---------------------------------------------------------- */

/* Device-side timing of the hot path with CUDA events on the model's own
 * stream (the stream every graph and kernel of the model is launched on).
 *   step_ms_*:            one full pf_eval_metric graph (setup kernel with
 *                         validity + normalisation, event pass; params and
 *                         result through mapped host memory)
 *   event_kernel_ms_mean: the event-pass kernel alone (roofline numerator)
 * flush_l2 != 0 writes a 256 MiB scratch buffer before every timed launch,
 * outside the timed window, so no step starts with a warm L2. */
typedef struct pf_bench_result {
  double step_ms_mean;
  double step_ms_min;
  double event_kernel_ms_mean;
  double event_kernel_ms_min;
  double metric;
  uint64_t kernels_per_step;
  uint64_t h2d_bytes_per_step;
  uint64_t d2h_bytes_per_step;
} pf_bench_result;

PF_API int pf_bench(pf_model* model, const double* params, size_t n_params, int32_t metric,
                    int32_t steps, int32_t flush_l2, pf_bench_result* out, pf_status* status);

/* Event range [first, first + count) of shard `shard_index` of `shard_count`
 * for a data set of n_events under chunk size `chunk` (the subtree split of
 * the reduction tree, engine.hpp:63-68). */
PF_API void pf_shard_events(uint64_t n_events, uint64_t chunk, int32_t shard_count,
                            int32_t shard_index, uint64_t* first, uint64_t* count);

/* Events per reduction chunk of a bound model (warp sub-chunks x 32 lanes x
 * events per lane); shard boundaries fall on whole chunks. */
PF_API uint64_t pf_model_chunk(const pf_model* model);
/* 1 when this model's single-parameter-set call is the one fused kernel
 * (pf_fused_kernel: setup in every CTA + event pass), 0 for the setup/norm
 * kernels + event pass graph; known once a call has run */
PF_API int32_t pf_model_fused(const pf_model* model);

/* ---- fit-manager --------------------------------------------------------- */

/* FitConfig, fit.hpp:23-28 */
typedef struct pf_fit_config {
  int32_t minimizer; /* 0 QuasiNewton (BFGS), 1 NelderMead */
  int32_t batch_probes; /* 1: evaluate independent FD probes in one pass */
  uint64_t max_iterations;
  double gradient_tolerance;
  double simplex_tolerance;
} pf_fit_config;

/* FitResult, fit.hpp:32-43.  Arrays sized to pf_model_n_params. */
typedef struct pf_fit_result {
  int32_t status; /* 0 converged, 1 max-iterations, 2 failed */
  int32_t uncertainties_available;
  double metric_value;
  uint64_t n_metric_calls;
  double wall_time_s;
  double grad_max_norm;
  double* params;        /* external values, registry order */
  double* uncertainties; /* external; 0 for fixed parameters */
} pf_fit_result;

/* parfit::fit(BoundModel&, MetricKind, Backend, FitConfig) — fit.hpp:498-581.
 *   start:  initial external values (registry order), e.g. export_values()
 *   fixed:  per registry slot, nonzero keeps the value fixed
 *   lower/upper/step: Variable limits and steps (BoundTransform, fit.hpp:77-129) */
PF_API int pf_fit(pf_model* model, int32_t metric, const pf_fit_config* config, const double* start,
           const int32_t* fixed, const double* lower, const double* upper, const double* step,
           pf_fit_result* result, pf_status* status);

/* ---- event-store: toy generation ----------------------------------------- */

/* generate_events(pdf, observables, n_events, seed, GridSpec) —
 * generate.hpp:33-86 (ToyRng, :19-27).  The graph's parameters take their
 * current values (pf_variable.value).  obs: the data set's observables
 * (variable indices, column order).  out: column-major n_obs x n_events.
 * last (optional, n_obs): the observables' values afterwards — the last
 * accepted event for the PDF's box observables, their current value
 * otherwise (the reference sets Variable::value per accepted event, :79).
 * Runs on options->device (null: device 0).  gen_ms (optional): device time
 * of the batch loop (draw, evaluate, compact; buffer allocation excluded).
 * Errors: bad-arity (n_events < 1), the norm and raw errors of the PDF,
 * envelope-failure (generate.hpp:65-76). */
PF_API int pf_generate_events(const pf_graph* graph, const int32_t* obs, int32_t n_obs,
                              uint64_t n_events, uint64_t seed, uint32_t grid_points,
                              const pf_options* options, double* out, double* last, double* gen_ms,
                              pf_status* status);

/* Diagnostics: copies up to n of the model's %globaltimer stamps (built with
 * PFB200_DEFINES=PF_EVENT_TRACE; per event block: entry, prologue, PDL wait,
 * main loop, done, published; block 4095: setup entry/exit) into out.
 * Returns the number copied (0 when the module has no trace buffer). */
PF_API int64_t pf_debug_trace(pf_model* model, uint64_t* out, int64_t n);

/* Library version / number of CUDA kernels launched so far by this process
 * (all models), for the bench's gpu_launches accounting. */
PF_API int32_t pf_abi_version(void);
PF_API uint64_t pf_kernel_launches(void);

#ifdef __cplusplus
}
#endif

#endif /* PFB200_H */
