// engine.hpp — BoundModel on B200: HBM event store, compiled evaluator and
// per-call CUDA graphs.  Restates engine.hpp:137-236 of the reference.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "codegen.hpp"
#include "graph.hpp"

namespace pfb {

constexpr double kPenaltyValue = 1e300;  // engine.hpp:52
constexpr int kMaxBatch = 16;            // parameter sets per launch
constexpr int kEventWarps = 2;           // warps per event-pass block (PF_EV_WARPS)
constexpr uint64_t kConvNormPointsPerBlock = 32;  // windowed convolution grid points per norm block
constexpr int kEventBlocksPerSM = 8;     // resident event blocks per SM (PF_EVENT_MIN_BLOCKS)
constexpr int kCompAll4 = 8;               // Task.comp: a TddpPdf Dalitz task yielding its 4 components (PF_COMP_ALL4)
constexpr int kMaxGroup = 16;              // PF_GROUP_MAX: ranks of a peer-memory exchange group
constexpr int kFxBins = 32;               // PF_FX_BINS (x 16 int64 per bin)
constexpr double kSmallNormWork = 65536; // raw evaluations: single-CTA setup path
// wide accumulator of chunk sums >= 2^62 (pf_device.cuh PF_BIG_*)
constexpr int kBigDigits = 34, kBigSnap = 64, kBigSnapCount = 104, kBigStride = 128;

// host mirrors of the device structs (pf_device.cuh); layouts must match
struct KRec {
  uint64_t floor_count;
  uint64_t first_nonfinite;
  uint64_t first_event_error;
  uint32_t norm_error;
  uint32_t arrive[15];
  int64_t fx[6];
};
static_assert(sizeof(KRec) == 136, "pf_krec layout");

struct Task {
  int node, n, dims, first_block;
  int n_blocks, comp, fine, level;  // comp: component of a TddpPdf grid (-1: a plain midpoint sum)
  uint64_t points, per_block;
  double lo[8];
  double h[8];
  double vol;
  double pad;
};
static_assert(sizeof(Task) == 192, "pf_task layout");

struct Out {
  double result;
  uint64_t floor_count, first_nonfinite, first_event_error;
  uint32_t norm_error, pad;
  int64_t fx[6];
  uint64_t check;  // pf_out_check (pf_device.cuh): the record is complete
};
static_assert(sizeof(Out) == 96, "pf_out layout");
// host twin of pf_out_check
uint64_t out_check(const Out& o);

// Correctly rounded double of a superaccumulator (digits d_i 2^(32 i - 128));
// host twin of pf_fx_round (pf_device.cuh).  NaN when poisoned.
double fx_round(const int64_t* fx);
// the same for D digits d_i 2^(32 i - 128) (D <= 64)
double fx_round_n(const int64_t* fx, int D);

struct Args {
  const double* hP;
  Out* hout;
  double* hnorms;
  uint64_t* hclamp;
  int n_nodes;
  int fuse_final;
  int n_levels;
  int tddp_tab;  // norm kernel: TddpPdf column table in dynamic shared memory
  const double* data;
  uint64_t col_stride;
  uint64_t n_local;
  uint64_t event_offset;
  int n_chunks;
  int K;
  int level;
  int n_tasks;
  const double* P;
  double* S;
  const double* C;
  const Task* tasks;
  void* partials;
  KRec* rec;
  uint64_t* clamp;
  double total_content;
  uint32_t* done;
  int64_t* fxbins;
  int64_t* dpart;
  int64_t** peers;  // group exchange: every rank's receive buffer (null: no group)
  int gworld;
  int grank;
  int npin;
  int s_smem;  // the event pass stages S in shared memory (event_s_staged)
  int64_t* big;  // kMaxBatch x kBigStride wide accumulator (pf_big_add)
  uint32_t* ticket;  // (unused: reserved)
  int fused;
  int nwa;  // fused pass: active warps
  int kpw;  // fused pass: chunks per active warp
  uint32_t gmask;          // K = 1 inline: count this call's grid clamps (bit 0)
  const uint32_t* hmask;   // mapped: bit k = parameter set k recomputes its norms
  double pin[64];
};

struct Module {
  cudaLibrary_t lib = nullptr;
  cudaKernel_t setup = nullptr, pre = nullptr, norm = nullptr, event = nullptr, final = nullptr,
               publish = nullptr, fused = nullptr;
  size_t fused_static_smem = 0;  // static shared memory of pf_fused_kernel
  // largest dynamic shared memory any model sharing this module asked of
  // pf_norm_kernel (TddpPdf column tables depend on the grid): only raised
  mutable size_t norm_dyn_max = 0;
  cudaKernel_t flush_read = nullptr;  // bench: read half of the L2 flush
  // generator modules only (PF_GEN, pf_generate.cuh)
  cudaKernel_t gen_max = nullptr, gen_mt = nullptr, gen_mt_jump = nullptr, gen_eval = nullptr,
               gen_scan = nullptr, gen_scatter = nullptr;
};

// NVRTC compile of (library headers + generated source) for sm_100a.
std::vector<char> compile_cubin(const Layout& L, std::string* log);

struct Shard {
  int device = 0;
  cudaStream_t stream = nullptr;
  uint64_t chunk_lo = 0, chunk_hi = 0;  // global chunk range
  uint64_t n_local = 0, event_offset = 0, col_stride = 0;
  int n_chunks = 0;
  const Module* mod = nullptr;
  double* d_data = nullptr;
  double* d_P = nullptr;
  double* d_S = nullptr;
  double* d_C = nullptr;
  Task* d_tasks = nullptr;  // all levels, concatenated
  void* d_partials = nullptr;
  uint32_t* d_done = nullptr;   // [finished-block counter, kMaxBatch completion sequences]
  uint32_t seq[kMaxBatch] = {};  // completion sequence the host expects next, per k
  int64_t* d_fxbins = nullptr;  // kMaxBatch x kFxBins x 16 binned digits of the event pass
  int64_t* d_part = nullptr;    // kMaxBatch x 8: exact digits + error words of the last call (device)
  int64_t* d_big = nullptr;     // kMaxBatch x kBigStride wide accumulator + last-call snapshot
  int64_t* d_recv = nullptr;    // group exchange: kMaxBatch x kMaxGroup x 16 receive slots
  int64_t** d_peers = nullptr;  // group exchange: device array of every rank's d_recv (IPC-mapped)
  std::vector<void*> ipc_mapped;
  KRec* d_rec = nullptr;
  uint64_t* d_clamp = nullptr;  // [n_poly counted | n_poly discarded]
  Out* h_out = nullptr;         // mapped, kMaxBatch
  double* h_norms = nullptr;    // DEVICE: 3 n_nodes norms of the last call without a norm error
  uint64_t* h_clamp = nullptr;  // mapped
  std::map<int, cudaGraphExec_t> graphs;
  int kernels_per_graph = 0;
  Args event_args{};  // K = 1 event-pass arguments (timing)
  Args first_args{};  // K = 1 arguments of the first kernel (params inline)
  cudaGraph_t graph1 = nullptr;       // K = 1 template graph (kept for node updates)
  cudaGraphNode_t first_node = nullptr;
  int event_grid = 1;
  bool fused = false;          // K = 1 graph is the single fused kernel
  void* d_scratch = nullptr;  // L2 flush buffer (bench only)
};

struct BenchResult {
  double step_ms_mean = 0, step_ms_min = 0, event_ms_mean = 0, event_ms_min = 0, metric = 0;
  uint64_t kernels_per_step = 0, h2d_bytes = 0, d2h_bytes = 0;
};

void subtree_range(uint64_t n, int shard_count, int index, uint64_t* lo, uint64_t* hi);
size_t event_smem(const Layout& L, int K);
size_t fused_smem(const Layout& L);
constexpr int kFusedWarps = 16;  // PF_FUSED_WARPS
constexpr size_t kFusedSmemLimit = 227 * 1024;  // static + dynamic shared memory of one CTA
bool event_s_staged(const Layout& L, int K);
int sm_count(int device);

class Model {
 public:
  // generator: also compile the toy-generation kernels (pf_generate.cuh)
  Model(const pf_graph& g, const pf_data& d, uint32_t grid_points, const pf_options& opt,
        bool generator = false);
  ~Model();
  Model(const Model&) = delete;
  Model& operator=(const Model&) = delete;

  // BoundModel::eval_metric (engine.hpp:165-218)
  double eval(const double* params, size_t n, int metric, pf_eval_info* info);
  // K independent evaluations, bitwise equal to K eval() calls
  void eval_batch(const double* params, size_t K, size_t n, int metric, double* out);
  // this process's shard partial (shard_count > 1)
  void eval_partial(const double* params, size_t n, int metric, int64_t* fx, int* penalty);
  void eval_launch(const double* params, size_t n, int metric, int* penalty);
  void group_handle(void* out) const;
  void group_join(int world, int rank, const void* handles);
  cudaStream_t stream() const { return shards_[0].stream; }
  int64_t* partial_device() const { return shards_[0].d_part; }
  int64_t debug_trace(uint64_t* out, int64_t n);
  BenchResult bench(const double* params, size_t n, int metric, int steps, bool flush);
  // bench's L2 flush on shard 0's stream: write 256 MiB, then (unless
  // PFB200_FLUSH=write) read it back so the lines left in L2 are clean
  void flush_l2(int i);
  // generate_events (generate.hpp:33-86) at the parameters' current values:
  // n events; box dimension d is written to out[d] (host, n doubles; null:
  // not copied) (generate.cpp)
  void generate(uint64_t n, uint64_t seed, uint32_t grid_points, double* const* out, double* gen_ms);

  const Program& program() const { return pg_; }
  const Layout& layout() const { return L_; }
  uint64_t n_events() const { return n_events_; }
  uint64_t chunk() const { return chunk_; }
  bool fused_path() const { return !shards_.empty() && shards_[0].fused; }
  bool binned() const { return binned_; }
  uint64_t floor_count() const { return floor_total_; }
  uint64_t clamp_count(int node);
  void norms(double* norms, double* errs, int32_t* valid, int n);

 private:
  struct Raw {  // per-k outcome of one device pass
    bool penalty = false;
    bool wide = false;  // chunk sums beyond the fixed-point digits (value from wide_value)
    double value = 0;
    int64_t fx[6] = {0, 0, 0, 0, 0, 0};
  };
  void check_call(size_t n, int metric) const;
  bool params_valid(const double* p) const;
  void run(const double* params, int K, std::vector<Raw>& out, bool partial_only);
  void launch_graphs(const double* params, int K);
  void wait_results(int K, std::vector<Raw>& out, bool partial_only);
  double wide_value(int k);
  cudaGraphExec_t graph_for(Shard& s, int K);
  Args base_args(Shard& s, int K);
  void build_tasks(uint32_t grid_points);
  void add_tddp_tasks(int node, uint32_t grid_points, int lvl, int* blocks);
  std::string error_message(uint32_t code_node) const;
  bool conv_windowed(int node) const {
    return std::find(L_.conv_windowed.begin(), L_.conv_windowed.end(), node) != L_.conv_windowed.end();
  }
  [[noreturn]] void throw_device_error(uint32_t code_node) const;
  bool fused_ok(const Shard& sh) const;
  int fused_grid(const Shard& sh) const;
  size_t setup_smem_bytes() const {
    return sizeof(double) * (std::max(L_.np, 1) + std::max(L_.ss, 1));
  }

  Program pg_;
  Layout L_;
  bool binned_ = false;
  uint64_t n_events_ = 0;
  double total_content_ = 0;
  uint64_t chunk_ = 0, n_chunks_total_ = 0;
  int shard_count_ = 1, shard_index_ = 0;
  bool small_norms_ = true;
  int group_world_ = 1, group_rank_ = 0;  // peer-memory exchange group (group_join)
  std::vector<Shard> shards_;
  std::vector<Task> tasks_;  // host copy, all levels
  std::vector<int> level_first_task_, level_n_tasks_, level_blocks_;
  int max_norm_blocks_ = 0;
  size_t tddp_tab_bytes_ = 0;  // norm kernel: TddpPdf column table (dynamic shared memory), 0: none
  double* h_params_ = nullptr;  // mapped, kMaxBatch x np
  uint32_t* h_mask_ = nullptr;  // mapped: grid-clamp counting mask of the call (pf_grid_counts)
  uint32_t call_mask_ = 0;      // the mask of the call in flight
  std::vector<uint64_t> call_hash_;  // hash_params of each parameter set of the call in flight
  uint64_t norm_hash_ = 0;      // hash_params of the last call whose norms were computed
  bool have_norm_hash_ = false;
  uint64_t floor_total_ = 0;
  std::vector<uint64_t> clamp_total_;
  std::vector<double> norms_, errs_;
  std::vector<int32_t> norm_valid_;
  bool norms_on_device_ = false;  // a call succeeded since norms_ was last read from the device
  void fetch_norms();
};

uint64_t kernel_launch_count();

}  // namespace pfb
