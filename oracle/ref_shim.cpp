// ref_shim.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// A C entry layer over the UNMODIFIED reference headers
// (/root/reference/proj/include/parfit/*.hpp, compiled from where they lie,
// see oracle/Makefile).  It builds reference objects from the same pf_graph /
// pf_data description the product consumes (include/pfb200.h), so tests and
// bench.py's reference arm can run the reference's own BoundModel::eval_metric
// and parfit::fit on identical inputs.  Output: oracle/_ref/libparfit_ref.so.
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "parfit/engine.hpp"
#include "parfit/fit.hpp"
#include "parfit/generate.hpp"
#include "pfb200.h"

using namespace parfit;

namespace {

struct RefModel {
  std::vector<VariablePtr> vars;
  std::vector<PdfPtr> nodes;  // by desc index
  PdfPtr root;
  std::unique_ptr<BoundModel> bm;
  std::vector<PdfNode*> preorder;
};

void put(char* err, const std::string& s) {
  if (!err) return;
  std::strncpy(err, s.c_str(), 511);
  err[511] = '\0';
}

std::vector<VariablePtr> make_vars(const pf_graph* g) {
  std::vector<VariablePtr> vars;
  for (int i = 0; i < g->n_variables; ++i) {
    const pf_variable& v = g->variables[i];
    auto p = std::make_shared<Variable>();
    p->name = v.name ? v.name : "";
    p->value = v.value;
    p->lower = v.lower;
    p->upper = v.upper;
    p->step = v.step;
    p->fixed = v.fixed != 0;
    p->role = v.role == PF_PARAMETER ? Role::Parameter : Role::Observable;
    vars.push_back(p);
  }
  return vars;
}

PdfPtr build(const pf_graph* g, int idx, std::vector<VariablePtr>& vars, std::vector<PdfPtr>& memo) {
  if (memo[idx]) return memo[idx];
  const pf_node& n = g->nodes[idx];
  std::string name = n.name ? n.name : "";
  std::vector<PdfPtr> ch;
  for (int i = 0; i < n.n_children; ++i) ch.push_back(build(g, n.children[i], vars, memo));
  std::vector<VariablePtr> ps;
  for (int i = 0; i < n.n_params; ++i) ps.push_back(vars[n.params[i]]);
  VariablePtr x = n.n_obs > 0 ? vars[n.obs[0]] : nullptr;
  PdfPtr p;
  switch (n.kind) {
    case PF_EXPONENTIAL: p = exp_pdf(name, x, ps.at(0)); break;
    case PF_GAUSSIAN: p = gaussian_pdf(name, x, ps.at(0), ps.at(1)); break;
    case PF_BREIT_WIGNER: p = breit_wigner_pdf(name, x, ps.at(0), ps.at(1)); break;
    case PF_POLYNOMIAL: p = polynomial_pdf(name, x, ps); break;
    case PF_PRODUCT: p = prod_pdf(name, ch); break;
    case PF_SUM: p = add_pdf(name, ch, ps); break;
    case PF_COMPOSITE: p = composite_pdf(name, ch.at(0), ch.at(1)); break;
    case PF_MAPPED:
      p = mapped_pdf(name, std::vector<double>(n.reals, n.reals + n.n_reals), ch);
      break;
    case PF_CONVOLUTION:
      p = convolution_pdf(name, ch.at(0), ch.at(1), static_cast<std::size_t>(n.quadrature_points));
      break;
    default: throw Error("unsupported", "reference has no node kind " + std::to_string(n.kind));
  }
  memo[idx] = p;
  return p;
}

void collect(PdfNode* n, std::vector<PdfNode*>& out) {
  out.push_back(n);
  if (n->kind() == PdfKind::Composite) {
    auto* c = static_cast<CompositePdf*>(n);
    collect(c->outer().get(), out);
    collect(c->inner().get(), out);
  } else {
    for (const auto& c : n->children()) collect(c.get(), out);
  }
}

Backend backend_of(int threads) { return threads <= 0 ? Backend::serial() : Backend::with_threads(threads); }

}  // namespace

extern "C" {

// bins: per observable bin counts (binned data only)
void* ref_model_create(const pf_graph* g, const pf_data* d, const uint64_t* bins, uint32_t grid,
                       char* err) {
  try {
    auto m = std::make_unique<RefModel>();
    m->vars = make_vars(g);
    m->nodes.assign(g->n_nodes, nullptr);
    m->root = build(g, g->root, m->vars, m->nodes);
    std::vector<VariablePtr> obs;
    for (int i = 0; i < d->n_obs; ++i) obs.push_back(m->vars[d->obs[i]]);
    if (!d->binned) {
      UnbinnedDataSet ds(obs);
      for (uint64_t e = 0; e < d->n_events; ++e) {
        for (int c = 0; c < d->n_obs; ++c) obs[c]->value = d->values[c * d->n_events + e];
        ds.add_event();
      }
      m->bm = std::make_unique<BoundModel>(m->root, ds, GridSpec(grid));
    } else {
      std::vector<std::size_t> b(bins, bins + d->n_obs);
      BinnedDataSet ds(obs, b);
      std::vector<double> pt(d->n_obs);
      for (uint64_t e = 0; e < d->n_events; ++e) {
        for (int c = 0; c < d->n_obs; ++c) pt[c] = d->values[c * d->n_events + e];
        double w = d->values[d->n_obs * d->n_events + e];
        if (w != 0.0) ds.fill(pt, w);
      }
      m->bm = std::make_unique<BoundModel>(m->root, ds, GridSpec(grid));
    }
    collect(m->root.get(), m->preorder);
    return m.release();
  } catch (const std::exception& e) {
    put(err, e.what());
    return nullptr;
  }
}

void ref_model_destroy(void* h) { delete static_cast<RefModel*>(h); }

int32_t ref_n_params(void* h) {
  return static_cast<int32_t>(static_cast<RefModel*>(h)->bm->registry().n_parameters());
}

// registry slot -> variable index of the description
int32_t ref_param_variable(void* h, int32_t slot) {
  auto* m = static_cast<RefModel*>(h);
  const auto& p = m->bm->registry().parameters().at(slot);
  for (size_t i = 0; i < m->vars.size(); ++i)
    if (m->vars[i] == p) return static_cast<int32_t>(i);
  return -1;
}

int ref_eval(void* h, const double* p, size_t n, int metric, int threads, double* out, char* err) {
  try {
    auto* m = static_cast<RefModel*>(h);
    *out = m->bm->eval_metric(std::span<const double>(p, n),
                              metric == PF_CHISQ ? MetricKind::ChiSquared : MetricKind::NegLogLikelihood,
                              backend_of(threads));
    return 0;
  } catch (const std::exception& e) {
    put(err, e.what());
    return 1;
  }
}

uint64_t ref_floor_count(void* h) { return static_cast<RefModel*>(h)->bm->log_floor_count(); }

int32_t ref_n_nodes(void* h) { return static_cast<int32_t>(static_cast<RefModel*>(h)->preorder.size()); }

// cached_norm per pre-order node; valid[i] = 0 when the reference throws stale-normalization
void ref_norms(void* h, double* norms, double* errs, int32_t* valid, int32_t n) {
  auto* m = static_cast<RefModel*>(h);
  for (int32_t i = 0; i < n && i < static_cast<int32_t>(m->preorder.size()); ++i) {
    PdfNode* node = m->preorder[i];
    try {
      norms[i] = node->cached_norm();
      errs[i] = node->norm_error_estimate();
      valid[i] = 1;
    } catch (const Error&) {
      norms[i] = 0;
      errs[i] = 0;
      valid[i] = 0;
    }
  }
}

uint64_t ref_clamp_count(void* h, int32_t node) {
  auto* m = static_cast<RefModel*>(h);
  if (node < 0 || node >= static_cast<int32_t>(m->preorder.size())) return 0;
  auto* p = dynamic_cast<PolynomialPdf*>(m->preorder[node]);
  return p ? p->clamp_count() : 0;
}

// parfit::fit; params/uncert sized n_params (registry order)
int ref_fit(void* h, int metric, int threads, int minimizer, double* params, double* uncert,
            double* metric_value, uint64_t* calls, int32_t* status, int32_t* unc_avail,
            double* grad_max, double* wall, char* err) {
  try {
    auto* m = static_cast<RefModel*>(h);
    FitConfig cfg;
    cfg.minimizer = minimizer ? MinimizerKind::NelderMead : MinimizerKind::QuasiNewton;
    FitResult r = fit(*m->bm, metric == PF_CHISQ ? MetricKind::ChiSquared : MetricKind::NegLogLikelihood,
                      backend_of(threads), cfg);
    for (size_t i = 0; i < r.params.size(); ++i) {
      params[i] = r.params[i];
      uncert[i] = r.uncertainties_available ? r.uncertainties[i] : 0.0;
    }
    *metric_value = r.metric_value;
    *calls = r.n_metric_calls;
    *status = static_cast<int32_t>(r.status);
    *unc_avail = r.uncertainties_available ? 1 : 0;
    *grad_max = r.grad_max_norm;
    *wall = r.wall_time_s;
    return 0;
  } catch (const std::exception& e) {
    put(err, e.what());
    return 1;
  }
}

double ref_reduce(const double* terms, size_t n) { return reduce(std::span<const double>(terms, n)); }

// generate_events (generate.hpp:33-86) into column-major out[n_obs * n]
int ref_generate(const pf_graph* g, const int32_t* obs_idx, int32_t n_obs, uint64_t n, uint64_t seed,
                 uint32_t grid, double* out, char* err) {
  try {
    auto vars = make_vars(g);
    std::vector<PdfPtr> memo(g->n_nodes);
    PdfPtr root = build(g, g->root, vars, memo);
    std::vector<VariablePtr> obs;
    for (int i = 0; i < n_obs; ++i) obs.push_back(vars[obs_idx[i]]);
    UnbinnedDataSet ds = generate_events(root, obs, n, seed, GridSpec(grid));
    for (uint64_t e = 0; e < n; ++e)
      for (int c = 0; c < n_obs; ++c) out[c * n + e] = ds.rows()[e][c];
    return 0;
  } catch (const std::exception& e) {
    put(err, e.what());
    return 1;
  }
}

}  // extern "C"
