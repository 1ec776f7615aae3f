// generate.cpp — generate_events (generate.hpp:33-86) on the GPU.
//
// The reference: refresh the norms at the registry's current values (:39-43),
// scan the midpoint grid for the density maximum (:47-63), envelope = 1.1 x
// max (:64-66), then accept-reject candidates drawn from ONE mt19937_64
// stream (ToyRng, :19-27): per candidate one uniform per box dimension (box
// order) and one for the test `u * envelope < density`; a candidate density
// above the envelope throws envelope-failure (:72-76).
//
// Here the stream is produced on the device by a one-CTA kernel in batches
// of whole twists, every candidate of a batch is evaluated in parallel by
// the model's fused evaluator, and the accepted ones are compacted in stream
// order.  Identical seeds give the reference's events: candidates, the test
// and the stream are bit-exact; only the density itself can differ from the
// reference's by rounding (~1e-16 relative), which changes a decision with
// probability ~1e-16 per candidate (tests/test_gpu_generate.py checks whole
// samples against the reference).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>

#include "engine.hpp"

namespace pfb {

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error("cuda-error", std::string(what) + ": " + cudaGetErrorString(e));
}

struct GenArgs {  // pf_gen_args (pf_generate.cuh); layouts must match
  const double* P;
  const double* S;
  const double* C;
  int dims;
  int pad0;
  int cols[8];
  double lo[8];
  double span[8];
  double h[8];
  uint64_t points;
  uint64_t total;
  double envelope;
  const double* u;
  uint64_t n_cand;
  unsigned char* flags;
  uint32_t* block_count;
  uint32_t* block_base;
  uint64_t* rec;
  double* fail_density;
  double* out;
  uint64_t out_stride;
  uint64_t out_base;
  uint64_t remaining;
  uint64_t* mt;
  uint64_t rounds;
  const uint64_t* jpoly;
  uint64_t* mt_next;
  uint64_t jump_words;
  uint64_t u_off;
};

#include "mt_jump_table.inc"  // tools/gen_mt_jump.py

constexpr uint64_t kSegment = 256 * 8;  // PF_GEN_SEGMENT
constexpr uint64_t kMtN = 312;

void launch_gen(cudaKernel_t k, unsigned grid, unsigned block, cudaStream_t s, GenArgs& a) {
  void* args[] = {&a};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = s;
  ck(cudaLaunchKernelExC(&cfg, reinterpret_cast<const void*>(k), args), "generator launch");
}

// std::mt19937_64(seed): x_i = f (x_{i-1} ^ (x_{i-1} >> 62)) + i
void mt_seed(uint64_t seed, uint64_t* mt) {
  mt[0] = seed;
  for (uint64_t i = 1; i < kMtN; ++i) mt[i] = 6364136223846793005ull * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i;
}

struct Events {
  cudaEvent_t a = nullptr, b = nullptr;
  Events() {
    ck(cudaEventCreate(&a), "event");
    ck(cudaEventCreate(&b), "event");
  }
  ~Events() {
    cudaEventDestroy(a);
    cudaEventDestroy(b);
  }
};

// the generator's second stream: the mt19937_64 draw of the next batch
struct Side {
  cudaStream_t s = nullptr;
  cudaEvent_t ready = nullptr, drawn[2] = {nullptr, nullptr}, used[2] = {nullptr, nullptr};
  explicit Side(int device) {
    ck(cudaSetDevice(device), "cudaSetDevice");
    ck(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "event");
    for (int i = 0; i < 2; ++i) {
      ck(cudaEventCreateWithFlags(&drawn[i], cudaEventDisableTiming), "event");
      ck(cudaEventCreateWithFlags(&used[i], cudaEventDisableTiming), "event");
    }
  }
  ~Side() {  // a draw past the last batch may still be running
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    cudaEventDestroy(ready);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(drawn[i]);
      cudaEventDestroy(used[i]);
    }
  }
};

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { cudaFree(p); }
  template <class T>
  T* alloc(size_t bytes) {
    ck(cudaMalloc(&p, std::max<size_t>(bytes, 8)), "generator buffer");
    return static_cast<T*>(p);
  }
};

}  // namespace

void Model::generate(uint64_t n, uint64_t seed, uint32_t grid_points, double* const* out, double* gen_ms) {
  Shard& sh = shards_[0];
  if (!sh.mod->gen_max) throw Error("bad-model", "model was not built for generation");
  const Node& root = pg_.nodes[0];
  const int dims = static_cast<int>(root.box.size());
  if (dims < 1 || dims > 8) throw Error("bad-graph", "generate_events: 1-8 box dimensions");

  // refresh_normalizations at the registry's current values (:39-43); a
  // failing norm throws here (no penalty outside eval_metric)
  std::vector<double> p(pg_.param_vars.size());
  for (size_t i = 0; i < p.size(); ++i) p[i] = pg_.vars[pg_.param_vars[i]].value;
  std::vector<Raw> raw;
  run(p.data(), 1, raw, true);
  if (sh.h_out[0].norm_error != ~0u) throw_device_error(sh.h_out[0].norm_error);

  ck(cudaSetDevice(sh.device), "cudaSetDevice");
  cudaStream_t s = sh.stream;
  Events ev;  // gen_ms: the batch loop (draw, evaluate, compact), after the buffers exist

  GenArgs g;
  std::memset(&g, 0, sizeof g);
  g.P = sh.d_P;
  g.S = sh.d_S;
  g.C = sh.d_C;
  g.dims = dims;
  uint64_t total = 1;
  for (int d = 0; d < dims; ++d) {
    const Var& v = pg_.vars[root.box[d].var];
    g.cols[d] = root.box[d].column;
    g.lo[d] = v.lower;
    g.span[d] = v.upper - v.lower;
    g.h[d] = (v.upper - v.lower) / static_cast<double>(grid_points);  // generate.hpp:57
    if (total > (1ull << 40) / grid_points) throw Error("bad-grid", "generate_events: envelope grid too large");
    total *= grid_points;
  }
  g.points = grid_points;
  g.total = total;

  DevBuf b_rec;
  g.rec = b_rec.alloc<uint64_t>(8 * sizeof(uint64_t));
  uint64_t rec[8] = {0, ~0ull, ~0ull, ~0ull, 0, 0, 0, 0};
  ck(cudaMemcpyAsync(g.rec, rec, sizeof rec, cudaMemcpyHostToDevice, s), "rec init");

  // envelope scan (:47-66)
  const unsigned scan_grid =
      static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 8ull * sm_count(sh.device)));
  launch_gen(sh.mod->gen_max, scan_grid, 256, s, g);
  ck(cudaMemcpyAsync(rec, g.rec, sizeof rec, cudaMemcpyDeviceToHost, s), "rec read");
  ck(cudaStreamSynchronize(s), "envelope scan");
  if (rec[1] != ~0ull) throw_device_error(static_cast<uint32_t>(rec[1] & 0xffffff));
  double dmax;
  std::memcpy(&dmax, &rec[0], sizeof dmax);
  const double envelope = dmax * 1.1;
  if (!(envelope > 0)) throw Error("envelope-failure", "density maximum is not positive");
  g.envelope = envelope;

  // batches of whole candidates that are also whole twists and whole blocks
  const uint64_t w = static_cast<uint64_t>(dims) + 1;
  const uint64_t per_twist = kMtN / std::gcd(kMtN, w);  // candidates per whole number of twists
  const uint64_t unit = std::lcm(kSegment, per_twist);
  const uint64_t full = unit * std::max<uint64_t>(1, (1ull << 22) / unit);
  auto round_up = [&](double c) {
    const double u = std::ceil(std::max(c, 1.0) / static_cast<double>(unit));
    return std::min(full, unit * static_cast<uint64_t>(std::min(u, 1e12)));
  };

  // the stream is drawn by jumps (every batch: 128 segments of J words, each
  // from its own jumped window, pf_mt_jump_kernel) when a candidate's words
  // divide a twist; otherwise by the one-CTA sequential kernel
  const bool jump = kMtN % w == 0 && !std::getenv("PFB200_MT_SEQUENTIAL");
  const uint64_t seg_words = static_cast<uint64_t>(kMtJumpSegments) * kMtJumpWords;
  const uint64_t cap = jump ? (kMtN + seg_words) / w : full;  // candidates per batch, at most

  DevBuf b_u[2], b_flags, b_cnt, b_base, b_fail, b_out, b_mt, b_mt2, b_poly;
  double* u[2] = {b_u[0].alloc<double>(sizeof(double) * cap * w), b_u[1].alloc<double>(sizeof(double) * cap * w)};
  const uint64_t cap_blocks = (cap + kSegment - 1) / kSegment;
  g.flags = b_flags.alloc<unsigned char>(cap);
  g.block_count = b_cnt.alloc<uint32_t>(sizeof(uint32_t) * cap_blocks);
  g.block_base = b_base.alloc<uint32_t>(sizeof(uint32_t) * cap_blocks);
  g.fail_density = b_fail.alloc<double>(sizeof(double) * cap);
  g.out = b_out.alloc<double>(sizeof(double) * n * dims);
  g.out_stride = n;
  uint64_t* mt_cur = b_mt.alloc<uint64_t>(sizeof(uint64_t) * kMtN);
  uint64_t* mt_other = jump ? b_mt2.alloc<uint64_t>(sizeof(uint64_t) * kMtN) : nullptr;
  g.mt = mt_cur;
  std::vector<uint64_t> mt(kMtN);
  mt_seed(seed, mt.data());
  ck(cudaMemcpyAsync(mt_cur, mt.data(), sizeof(uint64_t) * kMtN, cudaMemcpyHostToDevice, s), "mt seed");
  if (jump) {
    g.jpoly = b_poly.alloc<uint64_t>(sizeof(uint64_t) * kMtN * kMtJumpSegments);
    ck(cudaMemcpyAsync(const_cast<uint64_t*>(g.jpoly), kMtJumpPoly, sizeof(uint64_t) * kMtN * kMtJumpSegments,
                       cudaMemcpyHostToDevice, s),
       "jump table");
    g.jump_words = kMtJumpWords;
  }

  // the stream of batch b + 1 is drawn (second stream) while batch b is
  // evaluated; sequential draws size their batches by the measured
  // acceptance so the stream drawn past the last needed candidate stays small
  Side side(sh.device);
  uint64_t size[2] = {round_up(4.0 * static_cast<double>(n)), 0};
  ck(cudaEventRecord(side.ready, s), "event record");  // the seeded state
  ck(cudaStreamWaitEvent(side.s, side.ready, 0), "stream wait");
  int draws = 0;
  auto draw = [&](int slot, uint64_t B) {
    GenArgs m = g;
    m.u = u[slot];
    if (jump) {
      uint64_t words = 0;
      if (draws == 0) {  // the seeded window is not in the image of T: one plain twist first
        m.mt = mt_cur;
        m.rounds = 1;
        launch_gen(sh.mod->gen_mt, 1, 160, side.s, m);
        words = kMtN;
      }
      m.mt = mt_cur;
      m.mt_next = mt_other;
      m.u_off = words;
      launch_gen(sh.mod->gen_mt_jump, static_cast<unsigned>(kMtJumpSegments), 320, side.s, m);
      std::swap(mt_cur, mt_other);
      size[slot] = (words + seg_words) / w;
    } else {
      m.rounds = B * w / kMtN;
      size[slot] = B;
      launch_gen(sh.mod->gen_mt, 1, 160, side.s, m);
    }
    ++draws;
    ck(cudaEventRecord(side.drawn[slot], side.s), "event record");
  };
  ck(cudaEventRecord(ev.a, s), "event record");
  draw(0, size[0]);
  uint64_t done = 0, cand_total = 0, acc_total = 0;
  for (int b = 0;; ++b) {
    const int slot = b & 1;
    const uint64_t B = size[slot];
    g.u = u[slot];
    g.n_cand = B;
    g.out_base = done;
    g.remaining = n - done;
    uint64_t r[8] = {0, ~0ull, ~0ull, ~0ull, 0, 0, 0, 0};
    ck(cudaMemcpyAsync(g.rec, r, sizeof r, cudaMemcpyHostToDevice, s), "rec reset");
    ck(cudaStreamWaitEvent(s, side.drawn[slot], 0), "stream wait");
    const unsigned blocks = static_cast<unsigned>((B + kSegment - 1) / kSegment);
    launch_gen(sh.mod->gen_eval, blocks, 256, s, g);
    launch_gen(sh.mod->gen_scan, 1, 1024, s, g);
    launch_gen(sh.mod->gen_scatter, blocks, 256, s, g);
    ck(cudaEventRecord(side.used[slot], s), "event record");
    ck(cudaMemcpyAsync(r, g.rec, sizeof r, cudaMemcpyDeviceToHost, s), "rec read");
    bool prefetched = false;
    if (acc_total > 0) {
      const double rate = static_cast<double>(acc_total) / static_cast<double>(cand_total);
      const double expect = static_cast<double>(done) + rate * static_cast<double>(B);
      if (expect < static_cast<double>(n)) {
        ck(cudaStreamWaitEvent(side.s, side.used[slot ^ 1], 0), "stream wait");
        draw(slot ^ 1, round_up(1.2 * (static_cast<double>(n) - expect) / rate));
        prefetched = true;
      }
    }
    ck(cudaStreamSynchronize(s), "generator batch");
    const uint64_t accepted = r[4];
    const uint64_t need = n - done;
    // only candidates up to the one that completes the sample are drawn by
    // the reference; an error or failure after it never happens there
    const uint64_t limit = accepted >= need ? r[3] : B - 1;
    const uint64_t ce = r[1] == ~0ull ? ~0ull : r[1] >> 24;
    const uint64_t cf = r[2];
    if (std::min(ce, cf) <= limit) {
      if (ce <= cf) throw_device_error(static_cast<uint32_t>(r[1] & 0xffffff));
      double density = 0;
      ck(cudaMemcpy(&density, g.fail_density + cf, sizeof density, cudaMemcpyDeviceToHost), "failure");
      throw Error("envelope-failure",
                  "density " + std::to_string(density) + " exceeds envelope " + std::to_string(envelope));
    }
    done += std::min(accepted, need);
    cand_total += B;
    acc_total += accepted;
    if (done >= n) break;
    if (!prefetched) {
      const double rate = acc_total ? static_cast<double>(acc_total) / static_cast<double>(cand_total) : 0.0;
      draw(slot ^ 1, rate > 0 ? round_up(1.2 * static_cast<double>(n - done) / rate) : full);
    }
  }
  ck(cudaEventRecord(ev.b, s), "event record");
  for (int d = 0; d < dims; ++d)  // straight into the caller's column of that observable
    if (out[d])
      ck(cudaMemcpyAsync(out[d], g.out + static_cast<size_t>(d) * n, sizeof(double) * n, cudaMemcpyDeviceToHost, s),
         "events D2H");
  ck(cudaStreamSynchronize(s), "generator");
  float ms = 0;
  cudaEventElapsedTime(&ms, ev.a, ev.b);
  if (gen_ms) *gen_ms = ms;
}

}  // namespace pfb
