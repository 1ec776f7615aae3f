// engine.cpp — the B200 BoundModel.
//
// setData (engine.hpp:139-154 of the reference): finalize the graph, upload
// the EventTable once into HBM (column-major, one shard per device), compile
// the fused evaluator with NVRTC for sm_100a and capture one CUDA graph per
// batch width:  setup (validity + normalisation; or pre + norm levels for big
// grids) -PDL-> event pass, which publishes the result itself.  Parameters
// and results travel through mapped host memory (K = 1: parameters inline in
// the kernel arguments), so there are no memcpy nodes.
// eval_metric (engine.hpp:165-218): host-side contract checks and penalty
// rules, one graph launch per shard, one synchronisation.
#include "engine.hpp"

#include <nvrtc.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <limits>
#include <mutex>
#include <sstream>
#include <unordered_map>

namespace pfb {

namespace {

std::atomic<uint64_t> g_launches{0};

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error("cuda-error", std::string(what) + ": " + cudaGetErrorString(e));
}

void ckr(nvrtcResult r, const char* what) {
  if (r != NVRTC_SUCCESS) throw Error("nvrtc-error", std::string(what) + ": " + nvrtcGetErrorString(r));
}

struct ModuleCache {
  std::mutex mu;
  std::unordered_map<std::string, std::vector<char>> cubins;          // by source
  std::map<std::pair<std::string, int>, Module*> modules;             // by (source, device)
};

ModuleCache& cache() {
  static ModuleCache* c = new ModuleCache();  // intentionally leaked (process lifetime)
  return *c;
}

}  // namespace

// TMA stage ring (PF_EV_WARPS x PF_NST stages x PF_NLOAD x 32 PF_EPT doubles)
// plus the per-lane chunk and fixed-point accumulators of K parameter sets
// Models with convolution tables read the per-call state S per (event, tau)
// pair: the event pass copies it into shared memory when it fits
// (PF_S_SMEM; the kernel's pointer then resolves to LDS, not L1).
bool event_s_staged(const Layout& L, int K) {
  if (const char* env = std::getenv("PFB200_EVENT_S_SMEM"))  // A/B hook
    if (std::atoi(env) == 0) return false;
  return !L.conv_tables.empty() && static_cast<size_t>(K) * L.ss * sizeof(double) <= 96 * 1024;
}

size_t event_smem(const Layout& L, int K) {
  const size_t stages = static_cast<size_t>(kEventWarps) * L.nst * L.load_cols.size() * 32 *
                        static_cast<size_t>(L.ept) * sizeof(double);
  // per lane and parameter set: a chunk accumulator (pf_lacc, lacc_n
  // doubles) and an exact fixed-point accumulator (6 x 8 B)
  size_t bytes = stages + static_cast<size_t>(K) * 32 * kEventWarps * (8 * L.lacc_n + 48);
  if (event_s_staged(L, K)) bytes += static_cast<size_t>(K) * L.ss * sizeof(double);
  // per warp: the scratch of the warp-shared convolution window products
  if (L.conv_shared) bytes += static_cast<size_t>(kEventWarps) * 2 * kConvKB * sizeof(double);
  return bytes;
}

// fused kernel: every warp's TMA ring, then P and S of the one parameter set
size_t fused_smem(const Layout& L) {
  return static_cast<size_t>(kFusedWarps) * L.nst * L.load_cols.size() * 32 * static_cast<size_t>(L.ept) *
             sizeof(double) +
         sizeof(double) * (std::max(L.np, 1) + std::max(L.ss, 1));
}

// grid points per thread and run of the normalisation kernel (PF_NORM_RUN;
// env PFB200_NORM_RUN with PFB200_DEFINES=PF_NORM_RUN=n: A/B hook)
uint64_t norm_run() {
  if (const char* env = std::getenv("PFB200_NORM_RUN")) return std::max<uint64_t>(1, std::strtoull(env, nullptr, 10));
  return 32;
}

// the normalisation kernel's copy of the per-call state (convolution models,
// pf_norm_kernel under PF_S_SMEM)
size_t norm_smem(const Layout& L) {
  const size_t b = static_cast<size_t>(L.ss) * sizeof(double);
  return !L.conv_tables.empty() && b <= 96 * 1024 && L.ss % 2 == 0 ? b : 0;
}

size_t event_smem_max(const Layout& L) {
  size_t m = 0;
  for (int K = 1; K <= kMaxBatch; ++K) m = std::max(m, event_smem(L, K));
  return m;
}

namespace {

const Module* load_module(const Layout& L, int device) {
  ModuleCache& c = cache();
  std::lock_guard<std::mutex> lock(c.mu);
  auto key = std::make_pair(L.structure_key, device);
  auto it = c.modules.find(key);
  if (it != c.modules.end()) return it->second;
  auto cit = c.cubins.find(L.structure_key);
  if (cit == c.cubins.end()) {
    std::string log;
    cit = c.cubins.emplace(L.structure_key, compile_cubin(L, &log)).first;
  }
  Module* m = new Module();
  ck(cudaSetDevice(device), "cudaSetDevice");
  ck(cudaLibraryLoadData(&m->lib, cit->second.data(), nullptr, nullptr, 0, nullptr, nullptr, 0),
     "cudaLibraryLoadData");
  ck(cudaLibraryGetKernel(&m->setup, m->lib, "pf_setup_kernel"), "get pf_setup_kernel");
  ck(cudaLibraryGetKernel(&m->publish, m->lib, "pf_publish_kernel"), "get pf_publish_kernel");
  ck(cudaLibraryGetKernel(&m->pre, m->lib, "pf_pre_kernel"), "get pf_pre_kernel");
  ck(cudaLibraryGetKernel(&m->norm, m->lib, "pf_norm_kernel"), "get pf_norm_kernel");
  ck(cudaLibraryGetKernel(&m->event, m->lib, "pf_event_kernel"), "get pf_event_kernel");
  ck(cudaLibraryGetKernel(&m->fused, m->lib, "pf_fused_kernel"), "get pf_fused_kernel");
  ck(cudaLibraryGetKernel(&m->flush_read, m->lib, "pf_flush_read_kernel"), "get pf_flush_read_kernel");
  if (L.source.rfind("#define PF_GEN 1\n", 0) == 0) {
    ck(cudaLibraryGetKernel(&m->gen_max, m->lib, "pf_gen_max_kernel"), "get pf_gen_max_kernel");
    ck(cudaLibraryGetKernel(&m->gen_mt, m->lib, "pf_mt_kernel"), "get pf_mt_kernel");
    ck(cudaLibraryGetKernel(&m->gen_mt_jump, m->lib, "pf_mt_jump_kernel"), "get pf_mt_jump_kernel");
    ck(cudaLibraryGetKernel(&m->gen_eval, m->lib, "pf_gen_eval_kernel"), "get pf_gen_eval_kernel");
    ck(cudaLibraryGetKernel(&m->gen_scan, m->lib, "pf_gen_scan_kernel"), "get pf_gen_scan_kernel");
    ck(cudaLibraryGetKernel(&m->gen_scatter, m->lib, "pf_gen_scatter_kernel"), "get pf_gen_scatter_kernel");
  }
  ck(cudaKernelSetAttributeForDevice(m->event, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     static_cast<int>(event_smem_max(L)), device),
     "event kernel smem attribute");
  if (norm_smem(L) > 0) {
    ck(cudaKernelSetAttributeForDevice(m->norm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(norm_smem(L)), device),
       "norm kernel smem attribute");
    m->norm_dyn_max = norm_smem(L);
  }
  {
    cudaFuncAttributes fa{};
    if (cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(m->fused)) == cudaSuccess)
      m->fused_static_smem = fa.sharedSizeBytes;
    else
      m->fused_static_smem = 64 * 1024, cudaGetLastError();
    if (fused_smem(L) + m->fused_static_smem <= kFusedSmemLimit)
      ck(cudaKernelSetAttributeForDevice(m->fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(fused_smem(L)), device),
         "fused kernel smem attribute");
  }
  c.modules.emplace(key, m);
  return m;
}

void launch(cudaKernel_t k, dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args& a,
            bool pdl = false, int cluster = 1) {
  void* args[] = {&a};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  cfg.attrs = attr;
  if (pdl) {  // programmatic dependent launch: overlaps this grid's start with its predecessor
    attr[cfg.numAttrs].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[cfg.numAttrs].val.programmaticStreamSerializationAllowed = 1;
    ++cfg.numAttrs;
  }
  if (cluster > 1) {  // thread-block cluster (distributed shared memory)
    attr[cfg.numAttrs].id = cudaLaunchAttributeClusterDimension;
    attr[cfg.numAttrs].val.clusterDim.x = static_cast<unsigned>(cluster);
    attr[cfg.numAttrs].val.clusterDim.y = 1;
    attr[cfg.numAttrs].val.clusterDim.z = 1;
    ++cfg.numAttrs;
  }
  ck(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k), args), "cudaLaunchKernelEx");
}

}  // namespace

// Split [lo, hi) the way the reference's pairwise tree does (engine.hpp:63-68)
// and descend `depth` levels following the bits of `index` (MSB first).
void subtree_range(uint64_t n, int shard_count, int index, uint64_t* lo, uint64_t* hi) {
  uint64_t a = 0, b = n;
  int depth = 0;
  while ((1 << depth) < shard_count) ++depth;
  for (int level = 0; level < depth; ++level) {
    uint64_t mid = a + (b - a) / 2;
    if ((index >> (depth - 1 - level)) & 1)
      a = mid;
    else
      b = mid;
  }
  *lo = a;
  *hi = b;
}

uint64_t kernel_launch_count() { return g_launches.load(); }

int sm_count(int device) {
  static int cached[64] = {0};
  if (device >= 0 && device < 64 && cached[device]) return cached[device];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device);
  if (device >= 0 && device < 64) cached[device] = n;
  return n;
}

std::vector<char> compile_cubin(const Layout& L, std::string* log) {
  nvrtcProgram prog;
  const char* headers[] = {device_header_source(), kernels_header_source(), counters_header_source(),
                           exp_table_header_source(), generate_header_source()};
  const char* names[] = {"pf_device.cuh", "pf_kernels.cuh", "pf_counters.cuh", "pf_exp_table.cuh",
                         "pf_generate.cuh"};
  ckr(nvrtcCreateProgram(&prog, L.source.c_str(), "pf_model.cu", 5, headers, names),
      "nvrtcCreateProgram");
  const char* opts[] = {"--gpu-architecture=sm_100a", "-lineinfo", "--std=c++17",
                        "--device-as-default-execution-space"};
  nvrtcResult r = nvrtcCompileProgram(prog, 4, opts);
  size_t log_size = 0;
  nvrtcGetProgramLogSize(prog, &log_size);
  std::string lg(log_size, '\0');
  if (log_size) nvrtcGetProgramLog(prog, &lg[0]);
  if (log) *log = lg;
  if (r != NVRTC_SUCCESS) {
    nvrtcDestroyProgram(&prog);
    throw Error("nvrtc-error", "compiling the evaluator failed:\n" + lg);
  }
  size_t n = 0;
  ckr(nvrtcGetCUBINSize(prog, &n), "nvrtcGetCUBINSize");
  std::vector<char> cubin(n);
  ckr(nvrtcGetCUBIN(prog, cubin.data()), "nvrtcGetCUBIN");
  nvrtcDestroyProgram(&prog);
  return cubin;
}

// ---------------------------------------------------------------------------

Model::Model(const pf_graph& g, const pf_data& d, uint32_t grid_points, const pf_options& opt,
             bool generator) {
  if (grid_points < 2) throw Error("bad-grid", "GridSpec needs >= 2 points");  // pdf.hpp:35-37
  if (!d.obs && d.n_obs > 0) throw Error("bad-data", "null observable list");
  binned_ = d.binned != 0;
  n_events_ = d.n_events;
  total_content_ = d.total_content;
  pg_ = finalize(g, d.n_obs, d.obs, binned_ ? 2 : 0);
  L_ = pfb::generate(pg_, binned_, d.n_events);
  if (generator) {
    L_.source = "#define PF_GEN 1\n" + L_.source;
    L_.structure_key = L_.source;
  }
  if (binned_) L_.constants[L_.nc_total_slot] = total_content_;
  if (L_.data_range_base >= 0) {
    // (min, max) of every data column over ALL events, for the per-call
    // log-form range proof (a NaN or infinite datum disables the fast path)
    for (int c = 0; c < d.n_obs; ++c) {
      double lo = std::numeric_limits<double>::infinity(), hi = -lo;
      bool finite = d.n_events > 0;
      const double* col = d.values + static_cast<size_t>(c) * d.n_events;
      for (uint64_t e = 0; e < d.n_events; ++e) {
        const double v = col[e];
        finite = finite && std::isfinite(v);
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
      }
      if (!finite) lo = hi = std::numeric_limits<double>::quiet_NaN();
      L_.constants[L_.data_range_base + 2 * c] = lo;
      L_.constants[L_.data_range_base + 2 * c + 1] = hi;
    }
  }
  clamp_total_.assign(pg_.nodes.size(), 0);
  norms_.assign(pg_.nodes.size(), 1.0);  // PdfNode::norm_ default (pdf.hpp:199)
  errs_.assign(pg_.nodes.size(), 0.0);
  norm_valid_.assign(pg_.nodes.size(), 0);

  const int n_devices = std::max(1, opt.n_devices);
  shard_count_ = std::max(1, opt.shard_count);
  shard_index_ = opt.shard_index;
  if (n_devices > 1 && shard_count_ > 1)
    throw Error("bad-backend", "n_devices and shard_count cannot both exceed 1");
  auto pow2 = [](int v) { return v > 0 && (v & (v - 1)) == 0; };
  if (!pow2(n_devices) || !pow2(shard_count_))
    throw Error("bad-backend", "device and shard counts must be powers of two");
  if (shard_index_ < 0 || shard_index_ >= shard_count_)
    throw Error("bad-backend", "shard_index out of range");

  chunk_ = 32ull * static_cast<uint64_t>(L_.ept) * static_cast<uint64_t>(L_.nsub);
  n_chunks_total_ = (n_events_ + chunk_ - 1) / chunk_;
  const int n_cols_data = d.n_obs + (binned_ ? 2 : 0);
  build_tasks(grid_points);
  double norm_work = 0;
  for (const Task& t : tasks_) {
    const Node& nd = pg_.nodes[t.node];
    const bool pairs = nd.kind == PF_CONVOLUTION && nd.box.size() == 1 && !conv_windowed(t.node);
    norm_work += static_cast<double>(t.points) *
                 (pairs ? 1.0 + subtree_cost(pg_, nd.children[1]) : subtree_cost(pg_, t.node));
  }
  int most_in_level = 0;
  for (int n : level_n_tasks_) most_in_level = std::max(most_in_level, n);
  bool multi = false;
  for (const Task& t : tasks_) multi |= t.comp == kCompAll4;  // four values per task: the norm kernel only
  small_norms_ = norm_work <= kSmallNormWork && setup_smem_bytes() <= 48 * 1024 && tasks_.size() <= 16 &&
                 most_in_level <= L_.setup_maxq && !multi;

  ck(cudaSetDevice(opt.device), "cudaSetDevice");
  // parameters and results live in mapped (zero-copy) pinned memory: the
  // per-call graph has no memcpy nodes
  ck(cudaHostAlloc(reinterpret_cast<void**>(&h_params_), sizeof(double) * kMaxBatch * std::max(L_.np, 1),
                   cudaHostAllocMapped | cudaHostAllocPortable),
     "cudaHostAlloc params");
  ck(cudaHostAlloc(reinterpret_cast<void**>(&h_mask_), sizeof(uint32_t) * 16, cudaHostAllocMapped | cudaHostAllocPortable),
     "cudaHostAlloc mask");
  std::memset(h_mask_, 0, sizeof(uint32_t) * 16);

  const int G = n_devices;
  const int groups = std::max(G, shard_count_);
  int visible = 0;
  if (cudaGetDeviceCount(&visible) != cudaSuccess || visible < 1)
    throw Error("cuda-error", "no CUDA device visible (there is no CPU fallback)");
  if (!opt.oversubscribe && opt.device + G > visible)
    throw Error("bad-backend", std::to_string(G) + " devices requested from device " + std::to_string(opt.device) +
                                   ", " + std::to_string(visible) + " visible");
  shards_.resize(G);
  for (int s = 0; s < G; ++s) {
    Shard& sh = shards_[s];
    sh.device = opt.oversubscribe ? (opt.device + s) % visible : opt.device + s;
    int part = shard_count_ > 1 ? shard_index_ : s;
    // balanced contiguous chunk ranges; the exact accumulator makes the sum
    // independent of where the shards split
    subtree_range(n_chunks_total_, groups, part, &sh.chunk_lo, &sh.chunk_hi);
    sh.n_chunks = static_cast<int>(sh.chunk_hi - sh.chunk_lo);
    sh.event_offset = std::min(sh.chunk_lo * chunk_, n_events_);
    uint64_t end = std::min(sh.chunk_hi * chunk_, n_events_);
    sh.n_local = end - sh.event_offset;
    // columns padded to whole chunks: every TMA stage copy stays in bounds
    sh.col_stride = (sh.n_local + chunk_ - 1) / chunk_ * chunk_;
    ck(cudaSetDevice(sh.device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&sh.stream, cudaStreamNonBlocking), "cudaStreamCreate");
    sh.mod = load_module(L_, sh.device);
    if (tddp_tab_bytes_ > 0) {
      // the module (and its kernel attribute) is shared by every model of the
      // same structure: raise the limit, never lower it under another model
      std::lock_guard<std::mutex> lock(cache().mu);
      const size_t need = std::max(tddp_tab_bytes_, norm_smem(L_));
      if (need > sh.mod->norm_dyn_max) {
        ck(cudaKernelSetAttributeForDevice(sh.mod->norm, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(need), sh.device),
           "norm kernel smem attribute (TddpPdf column table)");
        sh.mod->norm_dyn_max = need;
      }
    }
    const size_t np = std::max(L_.np, 1);
    ck(cudaMalloc(&sh.d_P, sizeof(double) * kMaxBatch * np), "cudaMalloc P");
    ck(cudaMalloc(&sh.d_S, sizeof(double) * kMaxBatch * std::max(L_.ss, 1)), "cudaMalloc S");
    ck(cudaMemset(sh.d_S, 0, sizeof(double) * kMaxBatch * std::max(L_.ss, 1)), "memset S");
    ck(cudaMalloc(&sh.d_C, sizeof(double) * std::max<size_t>(L_.constants.size(), 1)), "cudaMalloc C");
    if (!L_.constants.empty())
      ck(cudaMemcpy(sh.d_C, L_.constants.data(), sizeof(double) * L_.constants.size(),
                    cudaMemcpyHostToDevice),
         "upload C");
    ck(cudaMalloc(&sh.d_tasks, sizeof(Task) * std::max<size_t>(tasks_.size(), 1)), "cudaMalloc tasks");
    if (!tasks_.empty())
      ck(cudaMemcpy(sh.d_tasks, tasks_.data(), sizeof(Task) * tasks_.size(), cudaMemcpyHostToDevice),
         "upload tasks");
    size_t part_elems = static_cast<size_t>(kMaxBatch) *
                        std::max<size_t>(std::max<size_t>(sh.n_chunks, max_norm_blocks_), 1);
    ck(cudaMalloc(&sh.d_partials, 16 * 4 * part_elems), "cudaMalloc partials");  // 4 values per block (kCompAll4)
    ck(cudaMalloc(&sh.d_done, sizeof(uint32_t) * (1 + kMaxBatch)), "cudaMalloc done");
    ck(cudaMemset(sh.d_done, 0, sizeof(uint32_t) * (1 + kMaxBatch)), "memset done");
    ck(cudaMalloc(&sh.d_recv, sizeof(int64_t) * 2 * 16 * kMaxGroup * kMaxBatch), "cudaMalloc group receive");
    ck(cudaMemset(sh.d_recv, 0, sizeof(int64_t) * 2 * 16 * kMaxGroup * kMaxBatch), "memset group receive");
    ck(cudaMalloc(&sh.d_part, sizeof(int64_t) * 8 * kMaxBatch), "cudaMalloc partial");
    ck(cudaMemset(sh.d_part, 0, sizeof(int64_t) * 8 * kMaxBatch), "memset partial");
    ck(cudaMalloc(&sh.d_big, sizeof(int64_t) * kBigStride * kMaxBatch), "cudaMalloc wide digits");
    ck(cudaMemset(sh.d_big, 0, sizeof(int64_t) * kBigStride * kMaxBatch), "memset wide digits");
    const size_t bins = sizeof(int64_t) * kMaxBatch * kFxBins * 16;
    ck(cudaMalloc(&sh.d_fxbins, bins), "cudaMalloc fxbins");
    ck(cudaMemset(sh.d_fxbins, 0, bins), "memset fxbins");
    ck(cudaMalloc(&sh.d_rec, sizeof(KRec) * kMaxBatch), "cudaMalloc rec");
    {  // the records' reset state (pf_rec_init); every call's finalizer restores it
      std::vector<KRec> init(kMaxBatch);
      for (KRec& r : init) {
        std::memset(&r, 0, sizeof r);
        r.first_nonfinite = ~0ull;
        r.first_event_error = ~0ull;
        r.norm_error = ~0u;
      }
      ck(cudaMemcpy(sh.d_rec, init.data(), sizeof(KRec) * kMaxBatch, cudaMemcpyHostToDevice), "init rec");
    }
    ck(cudaMalloc(&sh.d_clamp, sizeof(uint64_t) * 2 * std::max(L_.n_poly, 1)), "cudaMalloc clamp");
    ck(cudaMemset(sh.d_clamp, 0, sizeof(uint64_t) * 2 * std::max(L_.n_poly, 1)), "memset clamp");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&sh.h_out), sizeof(Out) * kMaxBatch, cudaHostAllocMapped),
       "mapped out");
    // pinned memory may be recycled from a freed model: clear the completion
    // words (pad) so no stale value can equal the sequence the host expects
    std::memset(sh.h_out, 0, sizeof(Out) * kMaxBatch);
    ck(cudaMalloc(&sh.h_norms, sizeof(double) * 3 * pg_.nodes.size()), "cudaMalloc norms");
    ck(cudaHostAlloc(reinterpret_cast<void**>(&sh.h_clamp), sizeof(uint64_t) * std::max(L_.n_poly, 1),
                     cudaHostAllocMapped),
       "mapped clamp");
    std::memset(sh.h_clamp, 0, sizeof(uint64_t) * std::max(L_.n_poly, 1));
    // the EventTable shard, column-major with a padded stride (double2 loads)
    if (sh.n_local > 0) {
      ck(cudaMalloc(&sh.d_data, sizeof(double) * sh.col_stride * n_cols_data), "cudaMalloc events");
      ck(cudaMemcpy2D(sh.d_data, sizeof(double) * sh.col_stride, d.values + sh.event_offset,
                      sizeof(double) * n_events_, sizeof(double) * sh.n_local, n_cols_data,
                      cudaMemcpyHostToDevice),
         "upload events");
      // padding events (masked out of every sum) sit at each observable's
      // lower edge so no node raises a domain error on them
      const uint64_t pad = sh.col_stride - sh.n_local;
      if (pad > 0) {
        std::vector<double> fill(pad);
        for (int c = 0; c < n_cols_data; ++c) {
          std::fill(fill.begin(), fill.end(), c < d.n_obs ? pg_.vars[d.obs[c]].lower : 0.0);
          ck(cudaMemcpy(sh.d_data + c * sh.col_stride + sh.n_local, fill.data(), sizeof(double) * pad,
                        cudaMemcpyHostToDevice),
             "pad events");
        }
      }
    }
  }
}

Model::~Model() {
  for (Shard& sh : shards_) {
    cudaSetDevice(sh.device);
    for (auto& kv : sh.graphs) cudaGraphExecDestroy(kv.second);
    if (sh.graph1) cudaGraphDestroy(sh.graph1);
    if (sh.stream) cudaStreamDestroy(sh.stream);
    cudaFree(sh.d_data);
    cudaFree(sh.d_P);
    cudaFree(sh.d_S);
    cudaFree(sh.d_C);
    cudaFree(sh.d_tasks);
    cudaFree(sh.d_partials);
    cudaFree(sh.d_done);
    cudaFree(sh.d_fxbins);
    cudaFree(sh.d_part);
    cudaFree(sh.d_big);
    for (void* p : sh.ipc_mapped) cudaIpcCloseMemHandle(p);
    cudaFree(sh.d_peers);
    cudaFree(sh.d_recv);
    cudaFree(sh.d_rec);
    cudaFree(sh.d_clamp);
    cudaFreeHost(sh.h_out);
    cudaFree(sh.h_norms);
    cudaFreeHost(sh.h_clamp);
    cudaFree(sh.d_scratch);
  }
  cudaFreeHost(h_params_);
  cudaFreeHost(h_mask_);
}

// Norm tasks: for every normalised node, midpoint sums at n and 2n points per
// box dimension (pdf.hpp:148-188).  Box spacing and cell volume are computed
// exactly as midpoint_sum does so the grid coordinates agree bit for bit.
void Model::build_tasks(uint32_t grid_points) {
  tasks_.clear();
  level_first_task_.assign(L_.level_nodes.size(), 0);
  level_n_tasks_.assign(L_.level_nodes.size(), 0);
  level_blocks_.assign(L_.level_nodes.size(), 0);
  max_norm_blocks_ = 0;
  for (size_t lvl = 0; lvl < L_.level_nodes.size(); ++lvl) {
    level_first_task_[lvl] = static_cast<int>(tasks_.size());
    int blocks = 0;
    for (int node : L_.level_nodes[lvl]) {
      const Node& nd = pg_.nodes[node];
      const int dims = static_cast<int>(nd.box.size());
      if (nd.kind == PF_TDDP) {
        add_tddp_tasks(node, grid_points, static_cast<int>(lvl), &blocks);
        continue;
      }
      if (dims > 8) throw Error("bad-graph", nd.name + ": more than 8 box dimensions");
      // a convolution's grid runs over (point, tau_j) pairs (codegen.cpp
      // emit_norm_point): Q elements per point, each one resolution call
      const bool pairs = nd.kind == PF_CONVOLUTION && dims == 1 && !conv_windowed(node);
      const double cost = pairs ? 1.0 + subtree_cost(pg_, nd.children[1]) : subtree_cost(pg_, node);
      for (int fine = 0; fine < 2; ++fine) {
        Task t;
        std::memset(&t, 0, sizeof t);
        const uint64_t n = static_cast<uint64_t>(grid_points) * (fine ? 2 : 1);
        t.node = node;
        t.n = static_cast<int>(n);
        t.dims = dims;
        t.fine = fine;
        uint64_t total = 1;
        for (int dd = 0; dd < dims; ++dd) {
          const Var& v = pg_.vars[nd.box[dd].var];
          t.lo[dd] = v.lower;
          t.h[dd] = (v.upper - v.lower) / static_cast<double>(n);
          total *= n;
        }
        double vol = 1.0;
        for (int dd = 0; dd < dims; ++dd) vol *= t.h[dd];
        t.vol = vol;
        if (pairs) total *= static_cast<uint64_t>(nd.q);
        t.points = total;
        // about 4096 raw evaluations per block, at most 4096 blocks per task;
        // boxes of >= 2 dimensions: runs of 32 points per thread
        // (PF_NORM_RUN, walked row by row) for all 256 threads of a block
        uint64_t per = static_cast<uint64_t>(std::max(1.0, std::floor(4096.0 / cost)));
        if (dims >= 2 && !pairs) per = std::max<uint64_t>(per, 256ull * norm_run());
        // a windowed convolution point is one thread's loop (a few hundred
        // dependent steps): one warp's worth of points per block spreads the
        // grid over many SMs (C4: 12 blocks of 256 points took 25 us)
        if (conv_windowed(node)) {
          per = kConvNormPointsPerBlock;
          if (const char* env = std::getenv("PFB200_CONV_NORM_PER"))  // A/B hook
            per = std::max<uint64_t>(1, std::strtoull(env, nullptr, 10));
        }
        uint64_t nb = (total + per - 1) / per;
        if (nb > 4096) {
          nb = 4096;
          per = (total + nb - 1) / nb;
          nb = (total + per - 1) / per;
        }
        t.per_block = per;
        t.n_blocks = static_cast<int>(nb);
        t.level = static_cast<int>(lvl);
        t.first_block = blocks;
        t.comp = -1;
        blocks += t.n_blocks;
        tasks_.push_back(t);
      }
    }
    level_n_tasks_[lvl] = static_cast<int>(tasks_.size()) - level_first_task_[lvl];
    level_blocks_[lvl] = blocks;
    max_norm_blocks_ = std::max(max_norm_blocks_, blocks);
  }
  // TddpPdf Dalitz tasks: a column table per norm block when it fits beside
  // two resident blocks per SM (pf_tddp_cols; env PFB200_NOTDDPTAB: A/B hook)
  if (L_.tddp_tab_arrays > 0 && !std::getenv("PFB200_NOTDDPTAB")) {
    uint64_t n = 0;
    for (const Task& t : tasks_)
      if (t.comp == kCompAll4 || (t.dims == 2 && pg_.nodes[t.node].kind == PF_DALITZ))
        n = std::max<uint64_t>(n, static_cast<uint64_t>(t.n));
    const size_t bytes = static_cast<size_t>(L_.tddp_tab_arrays) * (n + n / 32) * sizeof(double);
    if (n > 0 && bytes <= 100 * 1024) tddp_tab_bytes_ = bytes;
  }
}

// TddpPdf: its 3-D midpoint sums (pdf.hpp:148-176 over (s12, s13, t)) are
// separable, sum_c D_c T_c: four Dalitz-grid component sums D_c and four
// time-grid sums T_c, each at n and 2n points per dimension (codegen.cpp
// emit_tddp_components; pf_stage_post combines them)
void Model::add_tddp_tasks(int node, uint32_t grid_points, int lvl, int* blocks) {
  const Node& nd = pg_.nodes[node];
  auto box_of = [&](int col) -> const BoxDim& {
    for (const BoxDim& b : nd.box)
      if (b.column == col) return b;
    throw Error("bad-graph", nd.name + ": observable outside the box");
  };
  const BoxDim* dims[3] = {&box_of(nd.obs_cols[0]), &box_of(nd.obs_cols[1]), &box_of(nd.obs_cols[2])};
  const double cost = subtree_cost(pg_, node);
  // the Dalitz grid: ONE task pair whose points yield all four components
  // (kCompAll4: both amplitudes evaluated once per point); the time grid:
  // one pair per component (cheap)
  for (int comp : {kCompAll4, 4, 5, 6, 7}) {
    const bool time = comp != kCompAll4;
    for (int fine = 0; fine < 2; ++fine) {
      Task t;
      std::memset(&t, 0, sizeof t);
      const uint64_t n = static_cast<uint64_t>(grid_points) * (fine ? 2 : 1);
      t.node = node;
      t.comp = comp;
      t.n = static_cast<int>(n);
      t.dims = time ? 1 : 2;
      t.fine = fine;
      double vol = 1.0;
      uint64_t total = 1;
      for (int d = 0; d < t.dims; ++d) {
        const Var& v = pg_.vars[dims[time ? 2 : d]->var];
        t.lo[d] = v.lower;
        t.h[d] = (v.upper - v.lower) / static_cast<double>(n);
        vol *= t.h[d];
        total *= n;
      }
      t.vol = vol;
      t.points = total;
      uint64_t per = static_cast<uint64_t>(std::max(1.0, std::floor(4096.0 / (time ? 8.0 : cost))));
      if (!time) per = std::max<uint64_t>(per, 256ull * norm_run());  // runs of PF_NORM_RUN points per thread (pf_norm_run4)
      uint64_t nb = (total + per - 1) / per;
      if (nb > 4096) {
        nb = 4096;
        per = (total + nb - 1) / nb;
        nb = (total + per - 1) / per;
      }
      t.per_block = per;
      t.n_blocks = static_cast<int>(nb);
      t.level = lvl;
      t.first_block = *blocks;
      *blocks += t.n_blocks;
      tasks_.push_back(t);
    }
  }
}

Args Model::base_args(Shard& sh, int K) {
  Args a;
  std::memset(&a, 0, sizeof a);
  ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(const_cast<double**>(&a.hP)), h_params_, 0),
     "mapped params");
  ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&a.hout), sh.h_out, 0), "mapped out");
  a.hnorms = sh.h_norms;  // device memory
  ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(&a.hclamp), sh.h_clamp, 0), "mapped clamp");
  ck(cudaHostGetDevicePointer(reinterpret_cast<void**>(const_cast<uint32_t**>(&a.hmask)), h_mask_, 0),
     "mapped mask");
  a.n_nodes = static_cast<int>(pg_.nodes.size());
  a.fuse_final = K == 1 ? 1 : 0;
  a.n_levels = static_cast<int>(L_.level_nodes.size());
  a.data = sh.d_data;
  a.col_stride = sh.col_stride;
  a.n_local = sh.n_local;
  a.event_offset = sh.event_offset;
  a.n_chunks = sh.n_chunks;
  a.K = K;
  a.P = sh.d_P;
  a.S = sh.d_S;
  a.C = sh.d_C;
  a.tasks = sh.d_tasks;
  a.n_tasks = static_cast<int>(tasks_.size());
  a.partials = sh.d_partials;
  a.done = sh.d_done;
  a.fxbins = sh.d_fxbins;
  a.dpart = sh.d_part;
  a.big = sh.d_big;
  a.peers = sh.d_peers;
  a.gworld = group_world_;
  a.grank = group_rank_;
  a.rec = sh.d_rec;
  a.s_smem = event_s_staged(L_, K) ? 1 : 0;
  a.total_content = total_content_;
  // norm-stage clamps are counted once (shard 0); the others discard them
  const bool counts_norm = (&sh == &shards_[0]) && shard_index_ == 0;
  a.clamp = counts_norm ? sh.d_clamp : sh.d_clamp + std::max(L_.n_poly, 1);
  return a;
}

// One call = one graph:  setup (or pre + norm levels) --PDL--> event pass
// (+ fused final tree for K = 1, or a final kernel with one block per k).
cudaGraphExec_t Model::graph_for(Shard& sh, int K) {
  auto it = sh.graphs.find(K);
  if (it != sh.graphs.end()) return it->second;
  ck(cudaSetDevice(sh.device), "cudaSetDevice");
  Args a = base_args(sh, K);
  int kernels = 0;
  // never more event blocks per SM than are co-resident (wide stages or a big
  // K need more shared memory): a persistent grid with a second partial wave
  // would leave SMs idle at the end
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, reinterpret_cast<const void*>(sh.mod->event),
                                                    32 * kEventWarps, event_smem(L_, K)) != cudaSuccess ||
      occ < 1)
    occ = kEventBlocksPerSM;
  cudaGraph_t graph;
  ck(cudaStreamBeginCapture(sh.stream, cudaStreamCaptureModeThreadLocal), "begin capture");
  const bool fused = K == 1 && fused_ok(sh);
  if (K == 1) sh.fused = false;
  if (fused) {
    // ONE kernel: setup in every CTA, then the event pass (pf_fused_kernel)
    Args f = a;
    f.clamp = sh.d_clamp;
    f.fused = 1;
    {  // balanced static schedule: kpw chunks for each of nwa active warps
      const int all = fused_grid(sh) * kFusedWarps;
      const int n = std::max(sh.n_chunks, 1);
      f.kpw = (n + all - 1) / all;
      f.nwa = (n + f.kpw - 1) / f.kpw;
    }
    launch(sh.mod->fused, dim3(fused_grid(sh)), dim3(32 * kFusedWarps), fused_smem(L_), sh.stream, f, false,
           L_.setup_cluster);
    ++kernels;
    sh.event_args = f;
    sh.event_grid = fused_grid(sh);
    sh.fused = true;
  } else if (small_norms_) {
    launch(sh.mod->setup, dim3(K * L_.setup_cluster), dim3(512), setup_smem_bytes(), sh.stream, a, false,
           L_.setup_cluster);
    ++kernels;
  } else {
    launch(sh.mod->pre, dim3(K), dim3(256), 0, sh.stream, a);
    ++kernels;
    for (size_t lvl = 0; lvl < L_.level_nodes.size(); ++lvl) {
      Args b = a;
      b.level = static_cast<int>(lvl);
      b.n_tasks = level_n_tasks_[lvl];
      b.tasks = sh.d_tasks + level_first_task_[lvl];
      b.tddp_tab = tddp_tab_bytes_ > 0 ? 1 : 0;
      launch(sh.mod->norm, dim3(level_blocks_[lvl], K), dim3(256), std::max(norm_smem(L_), tddp_tab_bytes_),
             sh.stream, b);
      ++kernels;
    }
  }
  Args e = a;
  e.clamp = sh.d_clamp;
  if (fused) {
  } else if (sh.n_local > 0) {
    // one warp per chunk, 2-warp blocks: the block scheduler balances SMs
    // persistent grid: one wave of 2-warp blocks; every warp strides over
    // many chunks, so its TMA ring streams without restarts
    int per_sm = kEventBlocksPerSM;
    if (const char* env = std::getenv("PFB200_EV_BLOCKS")) per_sm = std::max(1, std::atoi(env));
    const size_t smem = event_smem(L_, K);
    per_sm = std::min(per_sm, occ);
    const int grid = std::max(1, std::min((sh.n_chunks + kEventWarps - 1) / kEventWarps,
                                          sm_count(sh.device) * per_sm));
    // the event pass closes its own reduction tree and publishes the results
    launch(sh.mod->event, dim3(grid), dim3(32 * kEventWarps), smem, sh.stream, e, /*pdl=*/true);
    kernels += 1;
    if (K == 1) {
      sh.event_args = e;
      sh.event_grid = grid;
    }
  } else {
    launch(sh.mod->publish, dim3(1), dim3(256), 0, sh.stream, e);
    ++kernels;
  }
  ck(cudaStreamEndCapture(sh.stream, &graph), "end capture");
  cudaGraphExec_t exec;
  ck(cudaGraphInstantiate(&exec, graph, 0), "cudaGraphInstantiate");
  if (K == 1 && L_.np <= 64) {
    // keep the template: its root kernel node receives the parameters inline
    // (cudaGraphExecKernelNodeSetParams) on every call
    size_t n_roots = 1;
    ck(cudaGraphGetRootNodes(graph, &sh.first_node, &n_roots), "cudaGraphGetRootNodes");
    sh.graph1 = graph;
    sh.first_args = fused ? sh.event_args : a;
  } else {
    cudaGraphDestroy(graph);
  }
  sh.kernels_per_graph = kernels;
  sh.graphs.emplace(K, exec);
  return exec;
}

// The single-kernel path: small normalisation grids (the setup runs in every
// CTA), a ring that runs at most one chunk ahead, shared memory that fits,
// and events on this shard.  PFB200_FUSED=0 selects the two-kernel graph.
// one CTA per SM, rounded down to whole setup clusters
int Model::fused_grid(const Shard& sh) const {
  const int c = std::max(1, L_.setup_cluster);
  return std::max(c, sm_count(sh.device) / c * c);
}

bool Model::fused_ok(const Shard& sh) const {
  if (const char* env = std::getenv("PFB200_FUSED"))
    if (std::atoi(env) == 0) return false;
  return small_norms_ && sh.n_local > 0 && L_.nst <= L_.nsub &&
         fused_smem(L_) + sh.mod->fused_static_smem <= kFusedSmemLimit && L_.setup_maxq <= 8;
}

void Model::check_call(size_t n, int metric) const {
  if (n != pg_.param_vars.size())
    throw Error("size-mismatch", "eval_metric: parameter vector length");
  if (binned_ && metric == PF_NLL) throw Error("metric-mismatch", "NLL needs an unbinned data set");
  if (!binned_ && metric == PF_CHISQ)
    throw Error("metric-mismatch", "chi-squared needs a binned data set");
  if (metric != PF_NLL && metric != PF_CHISQ) throw Error("bad-metric", "unknown metric kind");
}

// AddPdf::params_valid (pdf.hpp:381-390) over the whole tree (pdf.hpp:96-100)
bool Model::params_valid(const double* p) const {
  for (const Node& n : pg_.nodes) {
    if (n.kind != PF_SUM) continue;
    double fsum = 0.0;
    for (int slot : n.params) {
      double f = p[slot];
      if (f < 0.0 || f > 1.0) return false;
      fsum += f;
    }
    if (fsum > 1.0) return false;
  }
  return true;
}

std::string Model::error_message(uint32_t code_node) const {
  const int code = code_node & 0xff;
  const int node = static_cast<int>(code_node >> 8);
  const std::string name = node < static_cast<int>(pg_.nodes.size()) ? pg_.nodes[node].name : "?";
  switch (code) {
    case 1: return "nonpositive-sigma: " + name;
    case 2: return "nonpositive-width: " + name;
    case 3: return "out-of-domain: " + name + ": x outside mapped range";
    case 4: return "zero-integral: degenerate PDF '" + name + "'";
    case 5: return "nonpositive-endpoint: " + name;
    case 7: return "nonpositive-lifetime: " + name;
  }
  return "device-error: code " + std::to_string(code);
}

void Model::throw_device_error(uint32_t code_node) const {
  const std::string m = error_message(code_node);
  const size_t colon = m.find(": ");
  throw Error(m.substr(0, colon), colon == std::string::npos ? "" : m.substr(colon + 2));
}

void Model::run(const double* params, int K, std::vector<Raw>& out, bool partial_only) {
  launch_graphs(params, K);
  wait_results(K, out, partial_only);
}

// hash_params (pdf.hpp:40-51): FNV-1a over the parameters' bytes
static uint64_t hash_params(const double* p, int n) {
  uint64_t h = 14695981039346656037ull;
  for (int k = 0; k < n; ++k) {
    uint64_t bits;
    std::memcpy(&bits, p + k, sizeof bits);
    for (int i = 0; i < 8; ++i) {
      h ^= (bits >> (8 * i)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
  return h;
}

void Model::launch_graphs(const double* params, int K) {
  if (L_.np > 0) std::memcpy(h_params_, params, sizeof(double) * K * L_.np);
  // the reference recomputes norms (and so meets the grid's clamps) only
  // when the parameters' hash differs from the last refresh's (pdf.hpp:111-123)
  call_mask_ = 0;
  call_hash_.assign(K, 0);
  {
    uint64_t cur = norm_hash_;
    bool have = have_norm_hash_;
    for (int k = 0; k < K; ++k) {
      call_hash_[k] = hash_params(params + static_cast<size_t>(k) * L_.np, L_.np);
      if (!have || call_hash_[k] != cur) call_mask_ |= 1u << k;
      cur = call_hash_[k];
      have = true;
    }
  }
  *reinterpret_cast<volatile uint32_t*>(h_mask_) = call_mask_;
  for (Shard& sh : shards_) {
    cudaGraphExec_t g = graph_for(sh, K);
    ck(cudaSetDevice(sh.device), "cudaSetDevice");
    if (K == 1 && sh.fused && L_.np <= 64) {
      // a one-kernel call: launched directly (one API call instead of a
      // kernel-node update plus a graph launch), parameters inline
      Args inl = sh.event_args;
      inl.npin = L_.np;
      inl.gmask = call_mask_;
      std::memcpy(inl.pin, params, sizeof(double) * L_.np);
      launch(sh.mod->fused, dim3(sh.event_grid), dim3(32 * kFusedWarps), fused_smem(L_), sh.stream, inl, false,
             L_.setup_cluster);
      g_launches += 1;
      ++sh.seq[0];
      continue;
    }
    if (K == 1 && sh.graph1) {
      cudaKernelNodeParams kp = {};
      const bool setup = small_norms_;
      kp.func = reinterpret_cast<void*>(sh.fused ? sh.mod->fused : setup ? sh.mod->setup : sh.mod->pre);
      kp.gridDim = dim3(sh.fused ? fused_grid(sh) : setup ? L_.setup_cluster : 1);
      kp.blockDim = dim3(sh.fused ? 32 * kFusedWarps : setup ? 512 : 256);
      kp.sharedMemBytes = sh.fused ? static_cast<unsigned>(fused_smem(L_))
                                   : setup ? static_cast<unsigned>(setup_smem_bytes()) : 0u;
      Args inl = sh.first_args;
      inl.npin = L_.np;
      inl.gmask = call_mask_;
      std::memcpy(inl.pin, params, sizeof(double) * L_.np);
      void* ptrs[] = {&inl};
      kp.kernelParams = ptrs;
      kp.extra = nullptr;
      ck(cudaGraphExecKernelNodeSetParams(g, sh.first_node, &kp), "cudaGraphExecKernelNodeSetParams");
    }
    ck(cudaGraphLaunch(g, sh.stream), "cudaGraphLaunch");
    g_launches += sh.kernels_per_graph;
    for (int k = 0; k < K; ++k) ++sh.seq[k];
  }
}

void Model::wait_results(int K, std::vector<Raw>& out, bool partial_only) {
  const size_t np = std::max(L_.np, 1);
  // the result is in mapped memory as soon as the publishing block has
  // written its completion word: spin on it (a stream synchronisation costs
  // a wake-up); the stream is queried now and then so errors still surface
  // the record is stored without a system fence: it is complete once its
  // sequence number and check word agree with its fields (pf_out_check)
  for (Shard& sh : shards_) {
    for (int k = 0; k < K; ++k) {
      const volatile uint32_t* word = &sh.h_out[k].pad;
      for (uint64_t spin = 1;; ++spin) {
        if (*word == sh.seq[k]) {
          std::atomic_thread_fence(std::memory_order_acquire);
          const volatile Out& v = sh.h_out[k];
          Out o;
          o.result = v.result;
          o.floor_count = v.floor_count;
          o.first_nonfinite = v.first_nonfinite;
          o.first_event_error = v.first_event_error;
          o.norm_error = v.norm_error;
          o.pad = v.pad;
          for (int i = 0; i < 6; ++i) o.fx[i] = v.fx[i];
          o.check = v.check;
          if (o.pad == sh.seq[k] && o.check == out_check(o)) break;
        }
        if ((spin & 1023) == 0) {
          const cudaError_t e = cudaStreamQuery(sh.stream);
          if (e == cudaSuccess && spin > (1u << 22))  // the kernel ended long ago: its stores have landed
            throw Error("device-error", "evaluation finished without publishing its result");
          if (e != cudaSuccess && e != cudaErrorNotReady) ck(e, "evaluation");
        }
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
  (void)np;
  out.assign(K, Raw());
  const size_t nn = pg_.nodes.size();
  // errors first, in parameter-set order (the sequential reference stops at
  // the first throwing call)
  for (int k = 0; k < K; ++k) {
    uint32_t norm_err = ~0u;
    uint64_t ev_err = ~0ull, nonfinite = ~0ull;
    for (Shard& sh : shards_) {
      norm_err = std::min(norm_err, sh.h_out[k].norm_error);
      ev_err = std::min(ev_err, sh.h_out[k].first_event_error);
      nonfinite = std::min(nonfinite, sh.h_out[k].first_nonfinite);
    }
    if (norm_err != ~0u && (norm_err & 0xff) == 6)
      throw Error("group-timeout", "a rank of the exchange group did not deliver its record within 5 s");
    if (norm_err != ~0u) {  // refresh_normalizations threw (engine.hpp:174-178)
      out[k].penalty = true;
      continue;
    }
    if (k < static_cast<int>(call_hash_.size())) {  // the fingerprint the reference now holds
      norm_hash_ = call_hash_[k];
      have_norm_hash_ = true;
    }
    // norms are replicated on every shard; the device keeps the last
    // successful set, read when asked (fetch_norms)
    norms_on_device_ = true;
    (void)nn;
    if (ev_err != ~0ull) throw Error("event-error", error_message(static_cast<uint32_t>(ev_err & 0xffffff)));
    for (Shard& sh : shards_) floor_total_ += sh.h_out[k].floor_count;
    // shard accumulators are exact: summing their digits and rounding once
    // gives the single-device value bit for bit
    for (int i = 0; i < 6; ++i) {
      int64_t s = 0;
      for (Shard& sh : shards_) s += sh.h_out[k].fx[i];
      out[k].fx[i] = s;
    }
    out[k].value = shards_.size() == 1 ? shards_[0].h_out[k].result : fx_round(out[k].fx);
    for (Shard& sh : shards_) out[k].wide |= std::isnan(sh.h_out[k].result) && nonfinite == ~0ull;
    if (out[k].wide && !partial_only) out[k].value = wide_value(k);
    if (!partial_only) {
      // any non-finite term makes the reference's sum non-finite
      // (engine.hpp:210-216); the device neutralised it and kept its index
      if (nonfinite != ~0ull)
        throw Error("non-finite-metric", "first offending event index " + std::to_string(nonfinite));
      if (!std::isfinite(out[k].value)) throw Error("non-finite-metric", "non-finite reduction");
    }
  }
}

uint64_t out_check(const Out& o) {
  auto mix = [](uint64_t h, uint64_t v) {
    h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
    h ^= h >> 31;
    h *= 0xbf58476d1ce4e5b9ull;
    return h ^ (h >> 29);
  };
  uint64_t h = 0x243f6a8885a308d3ull, bits;
  std::memcpy(&bits, &o.result, 8);
  h = mix(h, bits);
  h = mix(h, o.floor_count);
  h = mix(h, o.first_nonfinite);
  h = mix(h, o.first_event_error);
  h = mix(h, (static_cast<uint64_t>(o.norm_error) << 32) | o.pad);
  for (int i = 0; i < 6; ++i) h = mix(h, static_cast<uint64_t>(o.fx[i]));
  return h;
}

void Model::fetch_norms() {
  if (!norms_on_device_) return;
  Shard& sh = shards_[0];
  const size_t nn = pg_.nodes.size();
  std::vector<double> hn(3 * nn);
  ck(cudaSetDevice(sh.device), "cudaSetDevice");
  ck(cudaStreamSynchronize(sh.stream), "cudaStreamSynchronize");
  ck(cudaMemcpy(hn.data(), sh.h_norms, sizeof(double) * 3 * nn, cudaMemcpyDeviceToHost), "norms D2H");
  for (size_t i = 0; i < nn; ++i) {
    if (!pg_.nodes[i].normalised) continue;
    norms_[i] = hn[3 * i];
    errs_[i] = hn[3 * i + 1];
    norm_valid_[i] = 1;
  }
  norms_on_device_ = false;
}

// Rare path: some chunk sums were >= 2^62 (pf_big_add), beyond the six
// fixed-point digits.  The shards' wide digits (2^(32 j)) and fixed-point
// digits (2^(32 i - 128)) are added exactly on one 2^-128 grid and rounded
// once, so the value is still the correctly rounded exact sum of the chunk
// sums.  A poisoned fixed-point top digit (a non-finite chunk sum) gives NaN.
double Model::wide_value(int k) {
  if (group_world_ > 1)  // the exchanged digits are the group's, the wide ones only this rank's
    throw Error("metric-overflow", "chunk sums exceed the 2^63 range of the exact cross-rank digits");
  constexpr int D = 4 + kBigDigits + 2;
  int64_t acc[D] = {};
  std::vector<int64_t> snap(kBigStride);
  for (Shard& sh : shards_) {
    const int64_t* fx = sh.h_out[k].fx;
    if (fx[5] >= (1ll << 61) || fx[5] <= -(1ll << 61)) return std::numeric_limits<double>::quiet_NaN();
    for (int i = 0; i < 6; ++i) acc[i] += fx[i];
    if (!std::isnan(sh.h_out[k].result)) continue;
    ck(cudaSetDevice(sh.device), "cudaSetDevice");
    ck(cudaStreamSynchronize(sh.stream), "evaluation");
    ck(cudaMemcpy(snap.data(), sh.d_big + static_cast<size_t>(k) * kBigStride, sizeof(int64_t) * kBigStride,
                  cudaMemcpyDeviceToHost),
       "wide digits");
    if (snap[kBigSnapCount] == 0) continue;
    for (int j = 0; j < kBigDigits; ++j) acc[4 + j] += snap[kBigSnap + j];
  }
  return fx_round_n(acc, D);
}

// BoundModel::eval_metric (engine.hpp:165-218)
double Model::eval(const double* params, size_t n, int metric, pf_eval_info* info) {
  check_call(n, metric);
  if (info) std::memset(info, 0, sizeof *info);
  if (!params_valid(params)) {
    if (info) info->penalty = 1;
    return kPenaltyValue;
  }
  const uint64_t floors0 = floor_total_;
  std::vector<Raw> out;
  run(params, 1, out, false);
  if (info) {
    info->norms_recomputed = 1;
    info->log_floor_delta = floor_total_ - floors0;
  }
  if (out[0].penalty) {
    if (info) info->penalty = 1;
    return kPenaltyValue;
  }
  return out[0].value;
}

void Model::eval_batch(const double* params, size_t K, size_t n, int metric, double* result) {
  check_call(n, metric);
  // invalid parameter sets are answered on the host; the rest go to the GPU
  std::vector<size_t> live;
  for (size_t k = 0; k < K; ++k) {
    if (params_valid(params + k * n))
      live.push_back(k);
    else
      result[k] = kPenaltyValue;
  }
  std::vector<double> packed;
  std::vector<Raw> out;
  for (size_t first = 0; first < live.size(); first += kMaxBatch) {
    const size_t cnt = std::min<size_t>(kMaxBatch, live.size() - first);
    packed.resize(cnt * std::max<size_t>(n, 1));
    for (size_t j = 0; j < cnt; ++j)
      std::memcpy(packed.data() + j * n, params + live[first + j] * n, sizeof(double) * n);
    run(packed.data(), static_cast<int>(cnt), out, false);
    for (size_t j = 0; j < cnt; ++j)
      result[live[first + j]] = out[j].penalty ? kPenaltyValue : out[j].value;
  }
}

void Model::eval_partial(const double* params, size_t n, int metric, int64_t* fx, int* penalty) {
  check_call(n, metric);
  *penalty = 0;
  for (int i = 0; i < 6; ++i) fx[i] = 0;
  if (!params_valid(params)) {
    *penalty = 1;
    return;
  }
  std::vector<Raw> out;
  run(params, 1, out, true);
  if (out[0].penalty) {
    *penalty = 1;
    return;
  }
  if (out[0].wide)
    throw Error("metric-overflow", "a shard's chunk sums exceed the 2^63 range of the exact cross-shard digits");
  for (int i = 0; i < 6; ++i) fx[i] = out[0].fx[i];
}

// Enqueue one evaluation without waiting (multi-process exchange): the event
// pass also writes its exact digits to the device partial buffer, so a
// collective can follow on the same stream.  The host records the call as
// published; mapped results stay valid once the stream has drained.
void Model::eval_launch(const double* params, size_t n, int metric, int* penalty) {
  check_call(n, metric);
  if (shards_.size() != 1) throw Error("bad-backend", "eval_launch needs a single-device model");
  *penalty = 0;
  if (!params_valid(params)) {
    *penalty = 1;
    return;
  }
  launch_graphs(params, 1);
}

// Peer-memory exchange group (pf_group_handle / pf_group_join): the
// receive buffer of this model is exported as a CUDA IPC handle; joining maps
// every other rank's buffer into this process, so the event pass of every
// rank can store its exact record into all of them (pf_group_exchange).
void Model::group_handle(void* out) const {
  if (shards_.size() != 1) throw Error("bad-backend", "exchange groups need single-device models");
  const Shard& sh = shards_[0];
  ck(cudaSetDevice(sh.device), "cudaSetDevice");
  cudaIpcMemHandle_t h;
  ck(cudaIpcGetMemHandle(&h, sh.d_recv), "cudaIpcGetMemHandle");
  std::memcpy(out, &h, sizeof h);
}

void Model::group_join(int world, int rank, const void* handles) {
  if (shards_.size() != 1) throw Error("bad-backend", "exchange groups need single-device models");
  if (world < 1 || world > kMaxGroup || rank < 0 || rank >= world)
    throw Error("bad-backend", "exchange group: rank/world out of range");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  Shard& sh = shards_[0];
  ck(cudaSetDevice(sh.device), "cudaSetDevice");
  ck(cudaStreamSynchronize(sh.stream), "cudaStreamSynchronize");
  for (void* p : sh.ipc_mapped) cudaIpcCloseMemHandle(p);
  sh.ipc_mapped.clear();
  std::vector<int64_t*> ptrs(world);
  for (int q = 0; q < world; ++q) {
    if (q == rank) {
      ptrs[q] = sh.d_recv;
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, static_cast<const char*>(handles) + 64 * q, 64);
    void* p = nullptr;
    ck(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    sh.ipc_mapped.push_back(p);
    ptrs[q] = static_cast<int64_t*>(p);
  }
  if (!sh.d_peers) ck(cudaMalloc(&sh.d_peers, sizeof(int64_t*) * kMaxGroup), "cudaMalloc peers");
  ck(cudaMemcpy(sh.d_peers, ptrs.data(), sizeof(int64_t*) * world, cudaMemcpyHostToDevice), "peers H2D");
  // every rank restarts its per-call sequence at 0 (callers barrier after
  // joining, before the first evaluation)
  ck(cudaMemset(sh.d_recv, 0, sizeof(int64_t) * 2 * 16 * kMaxGroup * kMaxBatch), "memset group receive");
  ck(cudaMemset(sh.d_done, 0, sizeof(uint32_t) * (1 + kMaxBatch)), "memset done");
  for (int k = 0; k < kMaxBatch; ++k) sh.seq[k] = 0;
  std::memset(sh.h_out, 0, sizeof(Out) * kMaxBatch);
  group_world_ = world;
  group_rank_ = rank;
  // the captured graphs carry the old arguments: rebuild on next use
  for (auto& kv : sh.graphs) cudaGraphExecDestroy(kv.second);
  sh.graphs.clear();
  if (sh.graph1) cudaGraphDestroy(sh.graph1);
  sh.graph1 = nullptr;
  ck(cudaDeviceSynchronize(), "group join");
}

// PolynomialPdf clamp counter (pdf.hpp:320): the device's cumulative
// counters of every shard, read when asked
uint64_t Model::clamp_count(int node) {
  if (node < 0 || node >= static_cast<int>(clamp_total_.size())) return 0;
  if (L_.poly_index[node] < 0) return 0;
  uint64_t total = 0;
  for (Shard& sh : shards_) {
    uint64_t v = 0;
    ck(cudaSetDevice(sh.device), "cudaSetDevice");
    ck(cudaStreamSynchronize(sh.stream), "cudaStreamSynchronize");
    ck(cudaMemcpy(&v, sh.d_clamp + L_.poly_index[node], sizeof v, cudaMemcpyDeviceToHost), "clamp D2H");
    total += v;
  }
  return total;
}

void Model::norms(double* norms, double* errs, int32_t* valid, int n) {
  fetch_norms();
  for (int i = 0; i < n && i < static_cast<int>(norms_.size()); ++i) {
    if (norms) norms[i] = norms_[i];
    if (errs) errs[i] = errs_[i];
    if (valid) valid[i] = norm_valid_[i];
  }
}

}  // namespace pfb

namespace pfb {

// Device timing with CUDA events on the shard-0 stream (pfb200.h pf_bench).
int64_t Model::debug_trace(uint64_t* out, int64_t n) {
  Shard& sh = shards_[0];
  void* ptr = nullptr;
  size_t bytes = 0;
  // n < 0: the per-warp buffer (pf_trace_w) instead of the per-block one
  const char* name = n < 0 ? "pf_trace_w" : "pf_trace_buf";
  if (n < 0) n = -n;
  if (cudaLibraryGetGlobal(&ptr, &bytes, sh.mod->lib, name) != cudaSuccess || !ptr) {
    cudaGetLastError();
    return 0;
  }
  const int64_t m = std::min<int64_t>(n, static_cast<int64_t>(bytes / sizeof(uint64_t)));
  ck(cudaSetDevice(sh.device), "cudaSetDevice");
  ck(cudaStreamSynchronize(sh.stream), "cudaStreamSynchronize");
  ck(cudaMemcpy(out, ptr, sizeof(uint64_t) * m, cudaMemcpyDeviceToHost), "trace D2H");
  return m;
}

void Model::flush_l2(int i) {
  Shard& sh = shards_[0];
  const size_t bytes = 256ull << 20;
  if (!sh.d_scratch) ck(cudaMalloc(&sh.d_scratch, bytes + 64), "cudaMalloc scratch");
  ck(cudaMemsetAsync(sh.d_scratch, i & 0xff, bytes, sh.stream), "flush");
  // write only (the protocol's flush); PFB200_FLUSH=writeread also reads the
  // buffer back (clean lines in L2): measured the same C2 step (45.0 vs 45.4 us)
  const char* mode = std::getenv("PFB200_FLUSH");
  if (!mode || std::string(mode) != "writeread") return;
  const void* p = sh.d_scratch;
  uint64_t n16 = bytes / 16;
  void* sink = static_cast<char*>(sh.d_scratch) + bytes;
  void* args[] = {&p, &n16, &sink};
  ck(cudaLaunchKernel(reinterpret_cast<const void*>(sh.mod->flush_read), dim3(sm_count(sh.device) * 4), dim3(512),
                      args, 0, sh.stream),
     "flush read");
}

BenchResult Model::bench(const double* params, size_t n, int metric, int steps, bool flush) {
  BenchResult r;
  r.metric = eval(params, n, metric, nullptr);  // builds the K = 1 graph
  Shard& sh = shards_[0];
  ck(cudaSetDevice(sh.device), "cudaSetDevice");

  cudaEvent_t e0, e1;
  ck(cudaEventCreate(&e0), "cudaEventCreate");
  ck(cudaEventCreate(&e1), "cudaEventCreate");
  cudaGraphExec_t g = graph_for(sh, 1);
  double sum = 0, mn = 1e300;
  const uint64_t launches0 = g_launches.load();
  Args inl = sh.event_args;  // the fused call exactly as launch_graphs issues it
  inl.npin = L_.np;
  inl.gmask = 0;
  if (L_.np > 0 && L_.np <= 64) std::memcpy(inl.pin, params, sizeof(double) * L_.np);
  const bool direct = sh.fused && L_.np <= 64;
  for (int i = 0; i < steps; ++i) {
    if (flush) flush_l2(i);
    ck(cudaEventRecord(e0, sh.stream), "record");
    if (direct)
      launch(sh.mod->fused, dim3(sh.event_grid), dim3(32 * kFusedWarps), fused_smem(L_), sh.stream, inl, false,
             L_.setup_cluster);
    else
      ck(cudaGraphLaunch(g, sh.stream), "cudaGraphLaunch");
    ck(cudaEventRecord(e1, sh.stream), "record");
    ck(cudaEventSynchronize(e1), "sync");
    g_launches += sh.kernels_per_graph;
    float ms = 0;
    ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    sum += ms;
    mn = std::min(mn, static_cast<double>(ms));
  }
  r.kernels_per_step = steps ? (g_launches.load() - launches0) / steps : 0;
  r.step_ms_mean = steps ? sum / steps : 0;
  r.step_ms_min = steps ? mn : 0;
  sum = 0;
  mn = 1e300;
  if (sh.n_local > 0) {
    for (int i = 0; i < steps; ++i) {
      if (flush) flush_l2(i);
      Args a = sh.event_args;
      if (sh.fused) {  // the whole call is this one kernel: parameters inline, as in the graph
        a.npin = L_.np;
        std::memcpy(a.pin, params, sizeof(double) * L_.np);
      }
      ck(cudaEventRecord(e0, sh.stream), "record");
      if (sh.fused)
        launch(sh.mod->fused, dim3(sh.event_grid), dim3(32 * kFusedWarps), fused_smem(L_), sh.stream, a, false,
               L_.setup_cluster);
      else
        launch(sh.mod->event, dim3(sh.event_grid), dim3(32 * kEventWarps), event_smem(L_, 1), sh.stream,
               a, false);
      ck(cudaEventRecord(e1, sh.stream), "record");
      ck(cudaEventSynchronize(e1), "sync");
      ++g_launches;
      float ms = 0;
      ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
      sum += ms;
      mn = std::min(mn, static_cast<double>(ms));
    }
  }
  r.event_ms_mean = steps ? sum / steps : 0;
  r.event_ms_min = steps ? mn : 0;
  ck(cudaStreamSynchronize(sh.stream), "cudaStreamSynchronize");
  for (int k = 0; k < kMaxBatch; ++k) sh.seq[k] = sh.h_out[k].pad;  // bench launches published too
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  r.h2d_bytes = sizeof(double) * std::max(L_.np, 1);
  r.d2h_bytes = sizeof(Out);
  return r;
}

}  // namespace pfb

namespace pfb {

double fx_round(const int64_t* acc) { return fx_round_n(acc, 6); }

double fx_round_n(const int64_t* acc, int D) {
  uint32_t dig[64];
  int64_t carry = 0;
  for (int i = 0; i < D; ++i) {
    const int64_t v = acc[i] + carry;
    dig[i] = static_cast<uint32_t>(v & 0xffffffffll);
    carry = v >> 32;
  }
  if (carry > 0 || carry < -1) return std::numeric_limits<double>::quiet_NaN();
  const bool neg = carry < 0;
  if (neg) {
    uint32_t c = 1;
    for (int i = 0; i < D; ++i) {
      const uint64_t t = static_cast<uint64_t>(static_cast<uint32_t>(~dig[i])) + c;
      dig[i] = static_cast<uint32_t>(t);
      c = static_cast<uint32_t>(t >> 32);
    }
  }
  int top = D - 1;
  while (top >= 0 && dig[top] == 0) --top;
  if (top < 0) return 0.0;
  const int lz = __builtin_clz(dig[top]);
  const uint64_t hi = dig[top];
  const uint64_t mid = top >= 1 ? dig[top - 1] : 0u;
  const uint64_t lo = top >= 2 ? dig[top - 2] : 0u;
  bool sticky = false;
  for (int i = top - 3; i >= 0; --i) sticky |= dig[i] != 0;
  uint64_t win = (hi << (32 + lz)) | (mid << lz);
  if (lz) {
    win |= lo >> (32 - lz);
    sticky |= (lo & ((1ull << (32 - lz)) - 1)) != 0;
  } else {
    sticky |= lo != 0;
  }
  uint64_t mant = win >> 11;
  const uint64_t rem = win & 0x7ffull;
  if ((rem & 0x400ull) && ((rem & 0x3ffull) || sticky || (mant & 1ull))) ++mant;
  int msb = 32 * top + 31 - lz;
  if (mant >> 53) {
    mant >>= 1;
    ++msb;
  }
  const double r = std::ldexp(static_cast<double>(mant), msb - 52 - 128);
  return neg ? -r : r;
}

}  // namespace pfb
