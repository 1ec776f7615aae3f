// abi.cpp — extern "C" entry points of include/pfb200.h.  Every C++
// exception becomes a nonzero return plus the reference's "code: detail"
// message (errors.hpp:9-16).
#include <cuda_runtime.h>
#include <algorithm>
#include <cstring>
#include <memory>
#include <new>
#include <vector>

#include "codegen.hpp"
#include "engine.hpp"
#include "fit.hpp"
#include "graph.hpp"
#include "pfb200.h"

struct pf_model {
  std::unique_ptr<pfb::Model> impl;
};

namespace {

void set_status(pf_status* st, int code, const char* msg) {
  if (!st) return;
  st->code = code;
  std::strncpy(st->message, msg, sizeof(st->message) - 1);
  st->message[sizeof(st->message) - 1] = '\0';
}

template <class F>
int guarded(pf_status* st, F&& f) {
  try {
    f();
    set_status(st, 0, "");
    return 0;
  } catch (const pfb::Error& e) {
    set_status(st, 1, e.what());
  } catch (const std::bad_alloc&) {
    set_status(st, 2, "out-of-memory: host allocation failed");
  } catch (const std::exception& e) {
    set_status(st, 3, e.what());
  } catch (...) {
    set_status(st, 4, "unknown-error: non-standard exception");
  }
  return st ? st->code : 1;
}

pfb::Config to_config(const pf_fit_config* c) {
  pfb::Config cfg;
  if (c) {
    cfg.minimizer = c->minimizer;
    cfg.batch_probes = c->batch_probes != 0;
    cfg.max_iterations = c->max_iterations;
    cfg.gradient_tolerance = c->gradient_tolerance;
    cfg.simplex_tolerance = c->simplex_tolerance;
  }
  return cfg;
}

}  // namespace

extern "C" {

int32_t pf_abi_version(void) { return PF_ABI_VERSION; }
int32_t pf_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}
uint64_t pf_kernel_launches(void) { return pfb::kernel_launch_count(); }

int pf_graph_finalize(const pf_graph* graph, int32_t n_data_obs, const int32_t* data_obs,
                      int32_t reserved_columns, int32_t* param_order, int32_t cap_params,
                      int32_t* n_params, uint32_t* table, int32_t cap_table, int32_t* table_len,
                      int32_t* n_columns, pf_status* status) {
  return guarded(status, [&] {
    if (!graph) throw pfb::Error("bad-graph", "null graph");
    pfb::Program pg = pfb::finalize(*graph, n_data_obs, data_obs, reserved_columns);
    const int np = static_cast<int>(pg.param_vars.size());
    if (n_params) *n_params = np;
    if (param_order)
      for (int i = 0; i < std::min(np, cap_params); ++i) param_order[i] = pg.param_vars[i];
    int len = 0;
    for (const auto& row : pg.table)
      for (uint32_t v : row) {
        if (table && len < cap_table) table[len] = v;
        ++len;
      }
    if (table_len) *table_len = len;
    if (n_columns) *n_columns = pg.n_columns;
  });
}

int pf_graph_codegen(const pf_graph* graph, const pf_data* data, uint32_t grid_points, char* out,
                     size_t cap, size_t* len, pf_status* status) {
  return guarded(status, [&] {
    if (!graph || !data) throw pfb::Error("bad-graph", "null argument");
    (void)grid_points;
    pfb::Program pg = pfb::finalize(*graph, data->n_obs, data->obs, data->binned ? 2 : 0);
    pfb::Layout L = pfb::generate(pg, data->binned != 0);
    if (len) *len = L.source.size();
    if (out && cap) {
      size_t n = std::min(cap - 1, L.source.size());
      std::memcpy(out, L.source.data(), n);
      out[n] = '\0';
    }
  });
}

int pf_graph_compile_check(const pf_graph* graph, const pf_data* data, uint32_t grid_points,
                           size_t* cubin_bytes, pf_status* status) {
  return guarded(status, [&] {
    if (!graph || !data) throw pfb::Error("bad-graph", "null argument");
    (void)grid_points;
    pfb::Program pg = pfb::finalize(*graph, data->n_obs, data->obs, data->binned ? 2 : 0);
    pfb::Layout L = pfb::generate(pg, data->binned != 0);
    std::string log;
    std::vector<char> cubin = pfb::compile_cubin(L, &log);
    if (cubin_bytes) *cubin_bytes = cubin.size();
  });
}

int pf_model_create(const pf_graph* graph, const pf_data* data, uint32_t grid_points,
                    const pf_options* options, pf_model** out, pf_status* status) {
  return guarded(status, [&] {
    if (!graph || !data || !out) throw pfb::Error("bad-graph", "null argument");
    pf_options opt;
    std::memset(&opt, 0, sizeof opt);
    opt.n_devices = 1;
    opt.shard_count = 1;
    if (options) opt = *options;
    auto m = std::make_unique<pf_model>();
    m->impl = std::make_unique<pfb::Model>(*graph, *data, grid_points, opt);
    *out = m.release();
  });
}

void pf_model_destroy(pf_model* model) { delete model; }

int pf_generate_events(const pf_graph* graph, const int32_t* obs, int32_t n_obs, uint64_t n_events,
                       uint64_t seed, uint32_t grid_points, const pf_options* options, double* out,
                       double* last, double* gen_ms, pf_status* status) {
  return guarded(status, [&] {
    if (n_events < 1) throw pfb::Error("bad-arity", "generate_events: n_events >= 1");  // generate.hpp:37
    if (!graph || !out || (n_obs > 0 && !obs)) throw pfb::Error("bad-graph", "null argument");
    if (n_obs < 1) throw pfb::Error("empty-observables", "UnbinnedDataSet needs >= 1 observable");
    pf_options opt;
    std::memset(&opt, 0, sizeof opt);
    if (options) opt.device = options->device;
    opt.n_devices = 1;
    opt.shard_count = 1;
    // the evaluator is bound to one placeholder event at the observables'
    // lower edges; generation uses its parameters, norms and constants
    std::vector<double> row(n_obs);
    for (int32_t c = 0; c < n_obs; ++c) {
      if (obs[c] < 0 || obs[c] >= graph->n_variables) throw pfb::Error("bad-graph", "observable index");
      row[c] = graph->variables[obs[c]].lower;
    }
    pf_data d;
    std::memset(&d, 0, sizeof d);
    d.n_obs = n_obs;
    d.obs = obs;
    d.n_events = 1;
    d.values = row.data();
    pfb::Model m(*graph, d, grid_points, opt, /*generator=*/true);
    const auto& box = m.program().nodes[0].box;
    std::vector<double*> dst(box.size(), nullptr);  // box dimension -> the caller's column
    for (int32_t c = 0; c < n_obs; ++c)
      for (size_t b = 0; b < box.size(); ++b)
        if (box[b].var == obs[c]) dst[b] = out + static_cast<size_t>(c) * n_events;
    m.generate(n_events, seed, grid_points, dst.data(), gen_ms);
    for (int32_t c = 0; c < n_obs; ++c) {
      double* col = out + static_cast<size_t>(c) * n_events;
      bool in_box = false;
      for (size_t b = 0; b < box.size(); ++b) in_box |= box[b].var == obs[c];
      // an observable outside the PDF's box keeps its current value (add_event snapshot)
      if (!in_box) std::fill(col, col + n_events, graph->variables[obs[c]].value);
      if (last) last[c] = col[n_events - 1];
    }
  });
}

uint64_t pf_model_n_events(const pf_model* m) { return m ? m->impl->n_events() : 0; }
int32_t pf_model_n_params(const pf_model* m) {
  return m ? static_cast<int32_t>(m->impl->program().param_vars.size()) : 0;
}
int32_t pf_model_param_variable(const pf_model* m, int32_t slot) {
  if (!m || slot < 0 || slot >= static_cast<int32_t>(m->impl->program().param_vars.size())) return -1;
  return m->impl->program().param_vars[slot];
}
int32_t pf_model_n_nodes(const pf_model* m) {
  return m ? static_cast<int32_t>(m->impl->program().nodes.size()) : 0;
}
int32_t pf_model_binned(const pf_model* m) { return m && m->impl->binned() ? 1 : 0; }

int pf_eval_metric(pf_model* model, const double* params, size_t n_params, int32_t metric,
                   double* out, pf_eval_info* info, pf_status* status) {
  return guarded(status, [&] {
    if (!model || !out) throw pfb::Error("bad-model", "null argument");
    *out = model->impl->eval(params, n_params, metric, info);
  });
}

int pf_eval_metric_batch(pf_model* model, const double* params, size_t k, size_t n_params,
                         int32_t metric, double* out, pf_status* status) {
  return guarded(status, [&] {
    if (!model || !out) throw pfb::Error("bad-model", "null argument");
    model->impl->eval_batch(params, k, n_params, metric, out);
  });
}

int pf_eval_partial(pf_model* model, const double* params, size_t n_params, int32_t metric,
                    int64_t* partial_fx, int32_t* penalty, pf_status* status) {
  return guarded(status, [&] {
    if (!model || !partial_fx || !penalty) throw pfb::Error("bad-model", "null argument");
    int pen = 0;
    model->impl->eval_partial(params, n_params, metric, partial_fx, &pen);
    *penalty = pen;
  });
}

int pf_eval_launch(pf_model* model, const double* params, size_t n_params, int32_t metric, int32_t* penalty,
                   pf_status* status) {
  return guarded(status, [&] {
    if (!model || !penalty) throw pfb::Error("bad-model", "null argument");
    int pen = 0;
    model->impl->eval_launch(params, n_params, metric, &pen);
    *penalty = pen;
  });
}

uint64_t pf_model_stream(const pf_model* model) {
  return model ? reinterpret_cast<uint64_t>(model->impl->stream()) : 0;
}

uint64_t pf_model_partial_device(const pf_model* model) {
  return model ? reinterpret_cast<uint64_t>(model->impl->partial_device()) : 0;
}

double pf_combine_partials(const int64_t* partials_fx, int32_t shard_count) {
  int64_t fx[PF_FX_DIGITS] = {0, 0, 0, 0, 0, 0};
  for (int32_t s = 0; s < shard_count; ++s)
    for (int i = 0; i < PF_FX_DIGITS; ++i) fx[i] += partials_fx[s * PF_FX_DIGITS + i];
  return pfb::fx_round(fx);
}

int pf_node_norms(pf_model* model, double* norms, double* errs, int32_t* valid, int32_t n_nodes) {
  if (!model) return 1;
  model->impl->norms(norms, errs, valid, n_nodes);
  return 0;
}

int pf_bench(pf_model* model, const double* params, size_t n_params, int32_t metric, int32_t steps,
             int32_t flush_l2, pf_bench_result* out, pf_status* status) {
  return guarded(status, [&] {
    if (!model || !out) throw pfb::Error("bad-model", "null argument");
    pfb::BenchResult r = model->impl->bench(params, n_params, metric, steps, flush_l2 != 0);
    out->step_ms_mean = r.step_ms_mean;
    out->step_ms_min = r.step_ms_min;
    out->event_kernel_ms_mean = r.event_ms_mean;
    out->event_kernel_ms_min = r.event_ms_min;
    out->metric = r.metric;
    out->kernels_per_step = r.kernels_per_step;
    out->h2d_bytes_per_step = r.h2d_bytes;
    out->d2h_bytes_per_step = r.d2h_bytes;
  });
}

void pf_shard_events(uint64_t n_events, uint64_t chunk, int32_t shard_count, int32_t shard_index,
                     uint64_t* first, uint64_t* count) {
  // balanced contiguous chunk ranges (the exact accumulator makes any split
  // give the same metric)
  uint64_t chunks = chunk ? (n_events + chunk - 1) / chunk : 0, lo = 0, hi = 0;
  pfb::subtree_range(chunks, shard_count, shard_index, &lo, &hi);
  uint64_t a = std::min(lo * chunk, n_events), b = std::min(hi * chunk, n_events);
  if (first) *first = a;
  if (count) *count = b - a;
}

uint64_t pf_model_chunk(const pf_model* m) { return m ? m->impl->chunk() : 0; }
int32_t pf_model_fused(const pf_model* m) { return m && m->impl->fused_path() ? 1 : 0; }

uint64_t pf_log_floor_count(const pf_model* m) { return m ? m->impl->floor_count() : 0; }
uint64_t pf_clamp_count(const pf_model* m, int32_t node) { return m ? m->impl->clamp_count(node) : 0; }

int pf_fit(pf_model* model, int32_t metric, const pf_fit_config* config, const double* start,
           const int32_t* fixed, const double* lower, const double* upper, const double* step,
           pf_fit_result* result, pf_status* status) {
  return guarded(status, [&] {
    if (!model || !start || !fixed || !lower || !upper || !step || !result)
      throw pfb::Error("bad-model", "null argument");
    const size_t np = model->impl->program().param_vars.size();
    std::vector<double> s(start, start + np), lo(lower, lower + np), hi(upper, upper + np),
        st(step, step + np);
    std::vector<int> fx(fixed, fixed + np);
    pfb::Model* m = model->impl.get();
    auto one = [&](const std::vector<double>& p) { return m->eval(p.data(), p.size(), metric, nullptr); };
    auto many = [&](const std::vector<std::vector<double>>& ps, std::vector<double>& out) {
      std::vector<double> flat;
      flat.reserve(ps.size() * np);
      for (const auto& p : ps) flat.insert(flat.end(), p.begin(), p.end());
      out.resize(ps.size());
      m->eval_batch(flat.data(), ps.size(), np, metric, out.data());
    };
    pfb::FitOutput r = pfb::fit(one, many, metric == PF_CHISQ, s, fx, lo, hi, st, to_config(config));
    result->status = static_cast<int32_t>(r.status);
    result->uncertainties_available = r.uncertainties_available ? 1 : 0;
    result->metric_value = r.metric_value;
    result->n_metric_calls = r.n_calls;
    result->wall_time_s = r.wall_time_s;
    result->grad_max_norm = r.grad_max_norm;
    for (size_t i = 0; i < np; ++i) {
      if (result->params) result->params[i] = r.params[i];
      if (result->uncertainties)
        result->uncertainties[i] = r.uncertainties_available ? r.uncertainties[i] : 0.0;
    }
  });
}

}  // extern "C"

extern "C" PF_API int64_t pf_debug_trace(pf_model* model, uint64_t* out, int64_t n) {
  if (!model || !out || n == 0) return 0;  // n < 0: the per-warp trace buffer
  try {
    return model->impl->debug_trace(out, n);
  } catch (...) {
    return 0;
  }
}

int pf_group_handle(pf_model* model, void* handle64, pf_status* status) {
  return guarded(status, [&] {
    if (!model || !handle64) throw pfb::Error("bad-model", "null argument");
    model->impl->group_handle(handle64);
  });
}

int pf_group_join(pf_model* model, int32_t world, int32_t rank, const void* handles, pf_status* status) {
  return guarded(status, [&] {
    if (!model || !handles) throw pfb::Error("bad-model", "null argument");
    model->impl->group_join(world, rank, handles);
  });
}
