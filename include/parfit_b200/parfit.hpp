// parfit_b200/parfit.hpp — C++ drop-in for the reference's public API.
//
// Same namespace, class names, factory functions and signatures as
// /root/reference/proj/include/parfit/{variable,dataset,pdf,engine,fit}.hpp,
// so code written against the reference recompiles unchanged after switching
//     #include "parfit/parfit.hpp"   ->   #include "parfit_b200/parfit.hpp"
// and linking libpfb200.so.  Every metric evaluation runs on the GPU through
// the C ABI (pfb200.h); this header only describes graphs and data sets.
//
// generate_events runs on the GPU too (pf_generate_events; same ToyRng stream,
// so a seed gives the reference's sample).  Not part of the drop-in (host-side
// utilities off the hot path, SURVEY §2 "OUT OF SCOPE"): PdfNode::raw/density
// for plotting, the JSON config front-end and the CLI.
#ifndef PARFIT_B200_PARFIT_HPP
#define PARFIT_B200_PARFIT_HPP

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <istream>
#include <memory>
#include <ostream>
#include <random>
#include <sstream>
#include <numeric>
#include <span>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "pfb200.h"

namespace parfit {

// ---- errors.hpp -----------------------------------------------------------
class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& msg) : std::runtime_error(msg) {}
  Error(const std::string& code, const std::string& detail) : std::runtime_error(code + ": " + detail) {}
};

inline void check(int rc, const pf_status& st) {
  if (rc) throw Error(st.message);
}

// ---- variable.hpp ---------------------------------------------------------
enum class Role { Observable, Parameter };

struct Variable {
  std::string name;
  double value = 0, lower = 0, upper = 0, step = 0;
  bool fixed = false;
  Role role = Role::Observable;
  int global_index = -1;
};
using VariablePtr = std::shared_ptr<Variable>;

inline VariablePtr new_observable(const std::string& name, double lower, double upper) {
  if (!(lower < upper)) throw Error("invalid-range", "observable '" + name + "': lower must be < upper");
  auto v = std::make_shared<Variable>();
  v->name = name;
  v->value = v->lower = lower;
  v->upper = upper;
  v->role = Role::Observable;
  return v;
}

inline VariablePtr new_parameter(const std::string& name, double init, double step, double lower,
                                 double upper) {
  if (!(lower < upper)) throw Error("invalid-range", "parameter '" + name + "': lower must be < upper");
  if (!(lower <= init && init <= upper))
    throw Error("invalid-range", "parameter '" + name + "': init outside [lower, upper]");
  if (!(step > 0)) throw Error("invalid-step", "parameter '" + name + "': step must be > 0");
  auto v = std::make_shared<Variable>();
  v->name = name;
  v->value = init;
  v->lower = lower;
  v->upper = upper;
  v->step = step;
  v->role = Role::Parameter;
  return v;
}

class ParameterRegistry {
 public:
  std::size_t register_parameter(const VariablePtr& v) {
    if (!v) throw Error("null-variable", "register_parameter");
    if (v->role != Role::Parameter) throw Error("wrong-role", "'" + v->name + "' is not a parameter");
    return add(params_, pby_, v);
  }
  std::size_t register_observable(const VariablePtr& v) {
    if (!v) throw Error("null-variable", "register_observable");
    if (v->role != Role::Observable) throw Error("wrong-role", "'" + v->name + "' is not an observable");
    return add(obs_, oby_, v);
  }
  const std::vector<VariablePtr>& parameters() const { return params_; }
  const std::vector<VariablePtr>& observables() const { return obs_; }
  std::size_t n_parameters() const { return params_.size(); }
  std::vector<double> export_values() const {
    std::vector<double> out;
    for (const auto& p : params_) out.push_back(p->value);
    return out;
  }
  void import_values(const std::vector<double>& vals) {
    if (vals.size() != params_.size()) throw Error("size-mismatch", "import_values: wrong parameter count");
    for (std::size_t i = 0; i < vals.size(); ++i) params_[i]->value = vals[i];
  }

 private:
  static std::size_t add(std::vector<VariablePtr>& list, std::unordered_map<std::string, Variable*>& by,
                         const VariablePtr& v) {
    auto it = by.find(v->name);
    if (it != by.end()) {
      if (it->second != v.get()) throw Error("name-collision", "distinct Variables both named '" + v->name + "'");
      return static_cast<std::size_t>(it->second->global_index);
    }
    v->global_index = static_cast<int>(list.size());
    list.push_back(v);
    by.emplace(v->name, v.get());
    return static_cast<std::size_t>(v->global_index);
  }
  std::vector<VariablePtr> params_, obs_;
  std::unordered_map<std::string, Variable*> pby_, oby_;
};

// ---- dataset.hpp ----------------------------------------------------------
class UnbinnedDataSet {
 public:
  explicit UnbinnedDataSet(std::vector<VariablePtr> observables) : obs_(std::move(observables)) {
    if (obs_.empty()) throw Error("empty-observables", "UnbinnedDataSet needs >= 1 observable");
    for (std::size_t i = 0; i < obs_.size(); ++i)
      for (std::size_t j = i + 1; j < obs_.size(); ++j)
        if (obs_[i] == obs_[j] || obs_[i]->name == obs_[j]->name) throw Error("duplicate-observable", obs_[i]->name);
    cols_.resize(obs_.size());
  }
  explicit UnbinnedDataSet(const VariablePtr& obs) : UnbinnedDataSet(std::vector<VariablePtr>{obs}) {}
  void add_event() {  // snapshot (dataset.hpp:28-33); stored column-major
    for (std::size_t c = 0; c < obs_.size(); ++c) cols_[c].push_back(obs_[c]->value);
  }
  const std::vector<VariablePtr>& observables() const { return obs_; }
  std::size_t n_events() const { return cols_.empty() ? 0 : cols_[0].size(); }
  std::size_t n_columns() const { return obs_.size(); }
  const std::vector<std::vector<double>>& columns() const { return cols_; }

 private:
  friend class detail_generate;
  std::vector<VariablePtr> obs_;
  std::vector<std::vector<double>> cols_;
};

// Text event store (dataset.hpp:184-245): '#' header naming the observables,
// one event per line, %.17g.  Same header checks and error codes.
inline void write_text(const UnbinnedDataSet& ds, std::ostream& out) {
  out << '#';
  for (const auto& o : ds.observables()) out << ' ' << o->name;
  out << '\n';
  char buf[40];
  const auto& cols = ds.columns();
  for (std::size_t e = 0; e < ds.n_events(); ++e) {
    for (std::size_t c = 0; c < cols.size(); ++c) {
      std::snprintf(buf, sizeof buf, "%.17g", cols[c][e]);
      if (c) out << ' ';
      out << buf;
    }
    out << '\n';
  }
}

inline void write_text_file(const UnbinnedDataSet& ds, const std::string& path) {
  std::ofstream f(path);
  if (!f) throw Error("io-error", "cannot open '" + path + "' for writing");
  write_text(ds, f);
}

inline UnbinnedDataSet read_text(std::istream& in, const std::vector<VariablePtr>& observables) {
  std::string line;
  if (!std::getline(in, line) || line.empty() || line[0] != '#') throw Error("bad-format", "missing '#' header line");
  {
    std::istringstream hs(line.substr(1));
    std::string name;
    std::size_t i = 0;
    while (hs >> name) {
      if (i >= observables.size() || observables[i]->name != name)
        throw Error("bad-format", "header observable '" + name + "' does not match expected order");
      ++i;
    }
    if (i != observables.size()) throw Error("bad-format", "header names fewer observables than expected");
  }
  UnbinnedDataSet ds(observables);
  while (std::getline(in, line)) {
    if (line.empty()) continue;
    std::istringstream ls(line);
    for (const auto& o : observables) {
      double v;
      if (!(ls >> v)) throw Error("bad-format", "short row in data file");
      o->value = v;
    }
    ds.add_event();
  }
  return ds;
}

inline UnbinnedDataSet read_text_file(const std::string& path, const std::vector<VariablePtr>& observables) {
  std::ifstream f(path);
  if (!f) throw Error("io-error", "cannot open '" + path + "'");
  return read_text(f, observables);
}

class BinnedDataSet {
 public:
  BinnedDataSet(std::vector<VariablePtr> observables, std::vector<std::size_t> bins)
      : obs_(std::move(observables)), bins_(std::move(bins)) {
    if (obs_.empty()) throw Error("empty-observables", "BinnedDataSet needs >= 1 observable");
    if (obs_.size() != bins_.size()) throw Error("dimension-mismatch", "observable/bin count mismatch");
    std::size_t total = 1;
    for (std::size_t b : bins_) {
      if (b < 1) throw Error("dimension-mismatch", "bins must be >= 1");
      total *= b;
    }
    contents_.assign(total, 0.0);
  }
  void fill(const std::vector<double>& point, double weight = 1.0) {
    if (point.size() != obs_.size()) throw Error("dimension-mismatch", "fill point arity");
    contents_[flat_bin(point)] += weight;
  }
  std::size_t flat_bin(const std::vector<double>& point) const {  // dataset.hpp:78-101
    std::size_t idx = 0;
    for (std::size_t i = 0; i < obs_.size(); ++i) {
      const auto& o = *obs_[i];
      const double w = (o.upper - o.lower) / static_cast<double>(bins_[i]);
      const double x = point[i];
      if (x < o.lower || x > o.upper) throw Error("out-of-range", "fill: '" + o.name + "' outside range");
      std::size_t b = static_cast<std::size_t>((x - o.lower) / w);
      if (b >= bins_[i]) {
        if (x == o.upper) b = bins_[i] - 1;
        else throw Error("out-of-range", "fill: '" + o.name + "' outside range");
      }
      if (x == o.upper && b != bins_[i] - 1) throw Error("out-of-range", "fill: '" + o.name + "' at excluded edge");
      idx = idx * bins_[i] + b;
    }
    return idx;
  }
  double bin_center(std::size_t obs, std::size_t b) const {
    const auto& o = *obs_[obs];
    return o.lower + (static_cast<double>(b) + 0.5) * ((o.upper - o.lower) / static_cast<double>(bins_[obs]));
  }
  double bin_volume() const {
    double v = 1.0;
    for (std::size_t i = 0; i < obs_.size(); ++i)
      v *= (obs_[i]->upper - obs_[i]->lower) / static_cast<double>(bins_[i]);
    return v;
  }
  double total_content() const { return std::accumulate(contents_.begin(), contents_.end(), 0.0); }
  const std::vector<VariablePtr>& observables() const { return obs_; }
  const std::vector<std::size_t>& bins() const { return bins_; }
  const std::vector<double>& contents() const { return contents_; }
  std::size_t n_bins() const { return contents_.size(); }

 private:
  std::vector<VariablePtr> obs_;
  std::vector<std::size_t> bins_;
  std::vector<double> contents_;
};

// Flat column-major event store (dataset.hpp:135-182)
struct EventTable {
  std::size_t n_events = 0, n_columns = 0;
  std::vector<double> values;
  double at(std::size_t e, std::size_t c) const { return values[c * n_events + e]; }
};

inline EventTable to_event_table(const UnbinnedDataSet& ds) {
  EventTable t;
  t.n_events = ds.n_events();
  t.n_columns = ds.n_columns();
  for (const auto& col : ds.columns()) t.values.insert(t.values.end(), col.begin(), col.end());
  return t;
}

inline EventTable to_event_table(const BinnedDataSet& ds) {
  const std::size_t nobs = ds.observables().size();
  EventTable t;
  t.n_events = ds.n_bins();
  t.n_columns = nobs + 2;
  t.values.resize(t.n_events * t.n_columns);
  const double vol = ds.bin_volume();
  std::vector<std::size_t> idx(nobs);
  for (std::size_t flat = 0; flat < ds.n_bins(); ++flat) {
    std::size_t rem = flat;
    for (std::size_t i = nobs; i-- > 0;) {
      idx[i] = rem % ds.bins()[i];
      rem /= ds.bins()[i];
    }
    for (std::size_t i = 0; i < nobs; ++i) t.values[i * t.n_events + flat] = ds.bin_center(i, idx[i]);
    t.values[nobs * t.n_events + flat] = ds.contents()[flat];
    t.values[(nobs + 1) * t.n_events + flat] = vol;
  }
  return t;
}

// ---- pdf.hpp ----------------------------------------------------------------
enum class PdfKind { Exponential, Gaussian, BreitWigner, Polynomial, Product, Sum, Composite, Mapped,
                     Convolution, Argus, Dalitz, Tddp };

struct GridSpec {
  std::size_t points = 1024;
  GridSpec() = default;
  explicit GridSpec(std::size_t p) : points(p) {
    if (p < 2) throw Error("bad-grid", "GridSpec needs >= 2 points");
  }
};

class PdfNode;
using PdfPtr = std::shared_ptr<PdfNode>;
class BoundModel;
class IndexTable;
IndexTable finalize(ParameterRegistry& registry, const PdfPtr& root,
                    const std::vector<VariablePtr>& data_observables, int reserved);

// A node of the PDF graph.  Kernels run on the GPU; after an evaluation the
// node exposes the normalisation the device computed (pdf.hpp:88-92).
class PdfNode {
 public:
  PdfNode(std::string name, PdfKind kind) : name_(std::move(name)), kind_(kind) {}
  virtual ~PdfNode() = default;
  const std::string& name() const { return name_; }
  PdfKind kind() const { return kind_; }
  std::size_t id() const { return id_; }
  const std::vector<PdfPtr>& children() const { return children_; }
  const std::vector<VariablePtr>& declared_parameters() const { return params_; }
  const std::vector<VariablePtr>& declared_observables() const { return obs_; }
  double cached_norm() const {
    refresh();
    if (!norm_valid_) throw Error("stale-normalization", name_);
    return norm_;
  }
  double norm_error_estimate() const {
    refresh();
    return norm_err_;
  }
  const std::vector<double>& reals() const { return reals_; }
  std::size_t quadrature() const { return q_; }

 protected:
  std::string name_;
  PdfKind kind_;
  std::vector<PdfPtr> children_;
  std::vector<VariablePtr> params_, obs_;
  std::vector<double> reals_;
  std::size_t q_ = 0;
  mutable std::size_t id_ = 0;
  mutable double norm_ = 1.0, norm_err_ = 0.0;
  mutable bool norm_valid_ = false;
  mutable BoundModel* owner_ = nullptr;  // the model that evaluated this node last
  void refresh() const;                  // its norms, fetched on first use
  friend class BoundModel;
  friend IndexTable finalize(ParameterRegistry&, const PdfPtr&, const std::vector<VariablePtr>&, int);
  static void need_obs(const std::string& n, const VariablePtr& v, const char* what = "x") {
    if (!v || v->role != Role::Observable) throw Error("wrong-role", n + ": " + what + " must be an observable");
  }
  static void need_par(const std::string& n, const VariablePtr& v, const char* what) {
    if (!v || v->role != Role::Parameter) throw Error("wrong-role", n + ": " + what + " must be a parameter");
  }
};

class ExpPdf final : public PdfNode {
 public:
  ExpPdf(std::string name, VariablePtr x, VariablePtr alpha) : PdfNode(std::move(name), PdfKind::Exponential) {
    need_obs(name_, x);
    need_par(name_, alpha, "alpha");
    obs_ = {std::move(x)};
    params_ = {std::move(alpha)};
  }
};

class GaussianPdf final : public PdfNode {
 public:
  GaussianPdf(std::string name, VariablePtr x, VariablePtr mean, VariablePtr sigma)
      : PdfNode(std::move(name), PdfKind::Gaussian) {
    need_obs(name_, x);
    need_par(name_, mean, "mean");
    need_par(name_, sigma, "sigma");
    if (!(sigma->lower > 0)) throw Error("nonpositive-sigma", name_ + ": sigma limits must exclude 0");
    obs_ = {std::move(x)};
    params_ = {std::move(mean), std::move(sigma)};
  }
};

class BreitWignerPdf final : public PdfNode {
 public:
  BreitWignerPdf(std::string name, VariablePtr x, VariablePtr mass, VariablePtr width)
      : PdfNode(std::move(name), PdfKind::BreitWigner) {
    need_obs(name_, x);
    need_par(name_, mass, "mass");
    need_par(name_, width, "width");
    if (!(width->lower > 0)) throw Error("nonpositive-width", name_ + ": width limits must exclude 0");
    obs_ = {std::move(x)};
    params_ = {std::move(mass), std::move(width)};
  }
};

class PolynomialPdf final : public PdfNode {
 public:
  PolynomialPdf(std::string name, VariablePtr x, std::vector<VariablePtr> coeffs)
      : PdfNode(std::move(name), PdfKind::Polynomial) {
    need_obs(name_, x);
    if (coeffs.empty()) throw Error("bad-arity", name_ + ": need >= 1 coefficient");
    for (const auto& c : coeffs) need_par(name_, c, "coefficients");
    obs_ = {std::move(x)};
    params_ = std::move(coeffs);
  }
  std::uint64_t clamp_count() const { return model_ ? pf_clamp_count(model_, static_cast<int32_t>(id_)) : 0; }

 private:
  friend class BoundModel;
  mutable const pf_model* model_ = nullptr;
};

// ArgusPdf(x; m0, c, p) (GooFit upper-threshold form; not in the reference)
class ArgusPdf final : public PdfNode {
 public:
  ArgusPdf(std::string name, VariablePtr x, VariablePtr m0, VariablePtr c, VariablePtr p)
      : PdfNode(std::move(name), PdfKind::Argus) {
    need_obs(name_, x);
    need_par(name_, m0, "m0");
    need_par(name_, c, "c");
    need_par(name_, p, "p");
    if (!(m0->lower > 0)) throw Error("nonpositive-endpoint", name_ + ": m0 limits must exclude 0");
    obs_ = {std::move(x)};
    params_ = {std::move(m0), std::move(c), std::move(p)};
  }
};

// Time-integrated isobar model over the Dalitz plot of M -> 1 2 3 (not in the
// reference; BASELINE config 5): |sum_r c_r BW_r|^2 inside the kinematic
// boundary.  Observables m12^2, m13^2; per resonance (mass, width, Re c, Im c)
// parameters, channel 12 / 13 / 23 and spin 0 / 1 (pfb200.h PF_DALITZ).
struct DalitzResonance {
  VariablePtr mass, width, re, im;
  int channel = 12;
  int spin = 1;
};

class DalitzPlotPdf final : public PdfNode {
 public:
  DalitzPlotPdf(std::string name, VariablePtr m12sq, VariablePtr m13sq, const std::vector<DalitzResonance>& res,
                double M, double m1, double m2, double m3, double radius = 1.5)
      : PdfNode(std::move(name), PdfKind::Dalitz) {
    need_obs(name_, m12sq, "m12sq");
    need_obs(name_, m13sq, "m13sq");
    if (!(M > m1 + m2 + m3 && m1 >= 0 && m2 >= 0 && m3 >= 0 && radius >= 0))
      throw Error("bad-kinematics", name_ + ": need M > m1 + m2 + m3, masses and R >= 0");
    if (res.empty()) throw Error("bad-arity", name_ + ": need >= 1 resonance");
    reals_ = {M, m1, m2, m3, radius};
    for (const auto& r : res) {
      need_par(name_, r.mass, "mass");
      need_par(name_, r.width, "width");
      need_par(name_, r.re, "Re c");
      need_par(name_, r.im, "Im c");
      if (r.channel != 12 && r.channel != 13 && r.channel != 23)
        throw Error("bad-channel", name_ + ": channel must be 12, 13 or 23");
      if (r.spin != 0 && r.spin != 1) throw Error("bad-spin", name_ + ": spin must be 0 or 1");
      if (!(r.width->lower > 0)) throw Error("nonpositive-width", name_ + ": width limits must exclude 0");
      params_.insert(params_.end(), {r.mass, r.width, r.re, r.im});
      reals_.push_back(r.channel);
      reals_.push_back(r.spin);
    }
    obs_ = {std::move(m12sq), std::move(m13sq)};
  }
};

// Time-dependent Dalitz-plot PDF with mixing (not in the reference; BASELINE
// config 5, GooFit's TDDP): |A g+(t) + Abar g-(t)|^2 with Abar(s12, s13) =
// A(s12, s23), observables m12^2, m13^2, t; the DalitzPlotPdf resonances, then
// tau, x, y (pfb200.h PF_TDDP).  Daughters 1 and 2 are CP conjugates (m1 == m2).
class TddpPdf final : public PdfNode {
 public:
  TddpPdf(std::string name, VariablePtr m12sq, VariablePtr m13sq, VariablePtr t,
          const std::vector<DalitzResonance>& res, double M, double m1, double m2, double m3, VariablePtr tau,
          VariablePtr x, VariablePtr y, double radius = 1.5)
      : PdfNode(std::move(name), PdfKind::Tddp) {
    DalitzPlotPdf amp(name_, m12sq, m13sq, res, M, m1, m2, m3, radius);  // the same checks
    need_obs(name_, t, "t");
    need_par(name_, tau, "tau");
    need_par(name_, x, "x");
    need_par(name_, y, "y");
    if (!(tau->lower > 0)) throw Error("nonpositive-lifetime", name_ + ": tau limits must exclude 0");
    if (m1 != m2) throw Error("bad-kinematics", name_ + ": daughters 1 and 2 must be CP conjugates (m1 == m2)");
    reals_ = amp.reals();
    params_ = amp.declared_parameters();
    params_.insert(params_.end(), {std::move(tau), std::move(x), std::move(y)});
    obs_ = {std::move(m12sq), std::move(m13sq), std::move(t)};
  }
};

class ProdPdf final : public PdfNode {
 public:
  ProdPdf(std::string name, std::vector<PdfPtr> children) : PdfNode(std::move(name), PdfKind::Product) {
    if (children.size() < 2) throw Error("bad-arity", name_ + ": product needs >= 2 children");
    children_ = std::move(children);
  }
};

class AddPdf final : public PdfNode {
 public:
  AddPdf(std::string name, std::vector<PdfPtr> children, std::vector<VariablePtr> fractions)
      : PdfNode(std::move(name), PdfKind::Sum) {
    if (children.size() < 2) throw Error("bad-arity", name_ + ": sum needs >= 2 children");
    if (fractions.size() != children.size() - 1)
      throw Error("fraction-count-mismatch", name_ + ": need n_children - 1 fractions");
    for (const auto& f : fractions) need_par(name_, f, "fractions");
    children_ = std::move(children);
    params_ = std::move(fractions);
  }
};

class CompositePdf final : public PdfNode {
 public:
  CompositePdf(std::string name, PdfPtr outer, PdfPtr inner) : PdfNode(std::move(name), PdfKind::Composite) {
    if (!outer || !inner) throw Error("bad-arity", name_ + ": null child");
    children_ = {std::move(outer), std::move(inner)};
  }
  const PdfPtr& outer() const { return children_[0]; }
  const PdfPtr& inner() const { return children_[1]; }
};

class MappedPdf final : public PdfNode {
 public:
  MappedPdf(std::string name, std::vector<double> boundaries, std::vector<PdfPtr> targets)
      : PdfNode(std::move(name), PdfKind::Mapped) {
    if (targets.empty()) throw Error("bad-arity", name_ + ": need >= 1 target");
    if (boundaries.size() != targets.size() + 1) throw Error("bad-arity", name_ + ": need n_targets + 1 boundaries");
    for (std::size_t i = 1; i < boundaries.size(); ++i)
      if (!(boundaries[i - 1] < boundaries[i])) throw Error("non-monotone-boundaries", name_);
    children_ = std::move(targets);
    reals_ = std::move(boundaries);
  }
  const std::vector<double>& boundaries() const { return reals_; }
};

class ConvolutionPdf final : public PdfNode {
 public:
  ConvolutionPdf(std::string name, PdfPtr model, PdfPtr resolution, std::size_t quadrature_points = 1024)
      : PdfNode(std::move(name), PdfKind::Convolution) {
    if (!model || !resolution) throw Error("bad-arity", name_ + ": null child");
    if (quadrature_points < 2) throw Error("bad-grid", name_ + ": need >= 2 quadrature points");
    children_ = {std::move(model), std::move(resolution)};
    q_ = quadrature_points;
  }
  const PdfPtr& model() const { return children_[0]; }
  const PdfPtr& resolution() const { return children_[1]; }
  std::size_t quadrature_points() const { return q_; }
};

inline PdfPtr exp_pdf(std::string n, VariablePtr x, VariablePtr a) {
  return std::make_shared<ExpPdf>(std::move(n), std::move(x), std::move(a));
}
inline PdfPtr gaussian_pdf(std::string n, VariablePtr x, VariablePtr m, VariablePtr s) {
  return std::make_shared<GaussianPdf>(std::move(n), std::move(x), std::move(m), std::move(s));
}
inline PdfPtr breit_wigner_pdf(std::string n, VariablePtr x, VariablePtr m, VariablePtr w) {
  return std::make_shared<BreitWignerPdf>(std::move(n), std::move(x), std::move(m), std::move(w));
}
inline PdfPtr polynomial_pdf(std::string n, VariablePtr x, std::vector<VariablePtr> c) {
  return std::make_shared<PolynomialPdf>(std::move(n), std::move(x), std::move(c));
}
inline PdfPtr argus_pdf(std::string n, VariablePtr x, VariablePtr m0, VariablePtr c, VariablePtr p) {
  return std::make_shared<ArgusPdf>(std::move(n), std::move(x), std::move(m0), std::move(c), std::move(p));
}
inline PdfPtr dalitz_pdf(std::string n, VariablePtr m12sq, VariablePtr m13sq, const std::vector<DalitzResonance>& res,
                         double M, double m1, double m2, double m3, double radius = 1.5) {
  return std::make_shared<DalitzPlotPdf>(std::move(n), std::move(m12sq), std::move(m13sq), res, M, m1, m2, m3,
                                         radius);
}
inline PdfPtr tddp_pdf(std::string n, VariablePtr m12sq, VariablePtr m13sq, VariablePtr t,
                       const std::vector<DalitzResonance>& res, double M, double m1, double m2, double m3,
                       VariablePtr tau, VariablePtr x, VariablePtr y, double radius = 1.5) {
  return std::make_shared<TddpPdf>(std::move(n), std::move(m12sq), std::move(m13sq), std::move(t), res, M, m1, m2,
                                   m3, std::move(tau), std::move(x), std::move(y), radius);
}
inline PdfPtr prod_pdf(std::string n, std::vector<PdfPtr> ch) {
  return std::make_shared<ProdPdf>(std::move(n), std::move(ch));
}
inline PdfPtr add_pdf(std::string n, std::vector<PdfPtr> ch, std::vector<VariablePtr> f) {
  return std::make_shared<AddPdf>(std::move(n), std::move(ch), std::move(f));
}
inline PdfPtr composite_pdf(std::string n, PdfPtr outer, PdfPtr inner) {
  return std::make_shared<CompositePdf>(std::move(n), std::move(outer), std::move(inner));
}
inline PdfPtr mapped_pdf(std::string n, std::vector<double> b, std::vector<PdfPtr> t) {
  return std::make_shared<MappedPdf>(std::move(n), std::move(b), std::move(t));
}
inline PdfPtr convolution_pdf(std::string n, PdfPtr model, PdfPtr res, std::size_t q = 1024) {
  return std::make_shared<ConvolutionPdf>(std::move(n), std::move(model), std::move(res), q);
}

// GooFit spellings (Listing 1)
using GooPdf = PdfNode;

// ---- graph description for the C ABI -----------------------------------------
namespace detail {

struct GraphDesc {
  std::vector<VariablePtr> vars;
  std::unordered_map<const Variable*, int> vidx;
  std::vector<const PdfNode*> nodes;
  std::unordered_map<const PdfNode*, int> nidx;
  std::vector<pf_variable> cvars;
  std::vector<pf_node> cnodes;
  std::vector<std::vector<int32_t>> ints;
  pf_graph graph{};
  int32_t root = -1;

  int var(const VariablePtr& v) {
    auto it = vidx.find(v.get());
    if (it != vidx.end()) return it->second;
    const int i = static_cast<int>(vars.size());
    vidx.emplace(v.get(), i);
    vars.push_back(v);
    return i;
  }
  int add(const PdfNode* n) {
    auto it = nidx.find(n);
    if (it != nidx.end()) return it->second;
    const int i = static_cast<int>(nodes.size());
    nidx.emplace(n, i);
    nodes.push_back(n);
    for (const auto& c : n->children()) add(c.get());
    for (const auto& p : n->declared_parameters()) var(p);
    for (const auto& o : n->declared_observables()) var(o);
    return i;
  }
  void build(const PdfPtr& pdf, const std::vector<VariablePtr>& data_obs) {
    for (const auto& o : data_obs) var(o);
    root = pdf ? add(pdf.get()) : -1;
    cvars.resize(vars.size());
    for (std::size_t i = 0; i < vars.size(); ++i) {
      const Variable& v = *vars[i];
      cvars[i] = pf_variable{v.name.c_str(), v.value, v.lower, v.upper, v.step, v.fixed ? 1 : 0,
                             v.role == Role::Parameter ? PF_PARAMETER : PF_OBSERVABLE};
    }
    cnodes.resize(nodes.size());
    ints.assign(nodes.size() * 3, {});
    for (std::size_t i = 0; i < nodes.size(); ++i) {
      const PdfNode* n = nodes[i];
      auto& ch = ints[3 * i];
      auto& pa = ints[3 * i + 1];
      auto& ob = ints[3 * i + 2];
      for (const auto& c : n->children()) ch.push_back(nidx.at(c.get()));
      for (const auto& p : n->declared_parameters()) pa.push_back(vidx.at(p.get()));
      for (const auto& o : n->declared_observables()) ob.push_back(vidx.at(o.get()));
      cnodes[i] = pf_node{static_cast<int32_t>(n->kind()), n->name().c_str(), static_cast<int32_t>(ch.size()),
                          ch.data(), static_cast<int32_t>(pa.size()), pa.data(),
                          static_cast<int32_t>(ob.size()), ob.data(), static_cast<int32_t>(n->reals().size()),
                          n->reals().data(), static_cast<int64_t>(n->quadrature())};
    }
    graph = pf_graph{static_cast<int32_t>(cvars.size()), cvars.data(), static_cast<int32_t>(cnodes.size()),
                     cnodes.data(), root};
  }
};

inline void preorder(const PdfNode* n, std::vector<const PdfNode*>& out) {
  out.push_back(n);
  for (const auto& c : n->children()) preorder(c.get(), out);
}

}  // namespace detail

// IndexTable (index_table.hpp): the finalized slot rows, read side
class IndexTable {
 public:
  IndexTable() = default;
  IndexTable(std::vector<std::vector<std::uint32_t>> rows, std::size_t ncols, std::size_t np)
      : rows_(std::move(rows)), ncols_(ncols), np_(np) {}
  std::size_t n_nodes() const { return rows_.size(); }
  std::size_t n_columns() const { return ncols_; }
  std::size_t n_parameters() const { return np_; }
  std::span<const std::uint32_t> node(std::size_t id) const {
    if (id >= rows_.size()) throw Error("bad-node-id", "IndexTable::node");
    return rows_[id];
  }
  std::uint32_t param_index(std::size_t id, std::size_t slot) const {
    auto s = node(id);
    if (slot >= s[0]) throw Error("out-of-bounds", "param slot");
    return s[1 + slot];
  }
  std::uint32_t obs_column(std::size_t id, std::size_t slot) const {
    auto s = node(id);
    if (slot >= s[1 + s[0]]) throw Error("out-of-bounds", "observable slot");
    return s[2 + s[0] + slot];
  }
  bool operator==(const IndexTable& o) const { return rows_ == o.rows_ && ncols_ == o.ncols_ && np_ == o.np_; }

 private:
  std::vector<std::vector<std::uint32_t>> rows_;
  std::size_t ncols_ = 0, np_ = 0;
};

// parfit::finalize (pdf.hpp:615-619)
inline IndexTable finalize(ParameterRegistry& registry, const PdfPtr& root,
                           const std::vector<VariablePtr>& data_observables, int reserved) {
  detail::GraphDesc g;
  g.build(root, data_observables);
  std::vector<int32_t> data(data_observables.size());
  for (std::size_t i = 0; i < data.size(); ++i) data[i] = g.vidx.at(data_observables[i].get());
  std::vector<int32_t> order(4096);
  std::vector<uint32_t> table(1 << 16);
  int32_t np = 0, tlen = 0, ncols = 0;
  pf_status st{};
  check(pf_graph_finalize(&g.graph, static_cast<int32_t>(data.size()), data.data(), reserved, order.data(),
                          static_cast<int32_t>(order.size()), &np, table.data(), static_cast<int32_t>(table.size()),
                          &tlen, &ncols, &st),
        st);
  for (int32_t i = 0; i < np; ++i) registry.register_parameter(g.vars[order[i]]);
  std::vector<std::vector<std::uint32_t>> rows;
  for (int32_t k = 0; k < tlen;) {
    const uint32_t p = table[k], o = table[k + 1 + p];
    rows.emplace_back(table.begin() + k, table.begin() + k + 2 + p + o);
    k += static_cast<int32_t>(2 + p + o);
  }
  if (root) {
    std::vector<const PdfNode*> pre;
    detail::preorder(root.get(), pre);
    for (std::size_t i = 0; i < pre.size(); ++i) pre[i]->id_ = i;
  }
  return IndexTable(std::move(rows), static_cast<std::size_t>(ncols), static_cast<std::size_t>(np));
}

inline IndexTable finalize(ParameterRegistry& registry, const PdfPtr& root,
                           const std::vector<VariablePtr>& data_observables) {
  return finalize(registry, root, data_observables, 0);
}

inline double lookup_param(const IndexTable& t, std::size_t node, std::size_t slot, std::span<const double> p) {
  const std::uint32_t gi = t.param_index(node, slot);
  if (gi >= p.size()) throw Error("out-of-bounds", "parameter vector shorter than index");
  return p[gi];
}

// ---- engine.hpp -----------------------------------------------------------------
struct Backend {
  enum class Kind { Serial, Threads, Gpu };
  Kind kind = Kind::Gpu;
  unsigned threads = 1;
  std::size_t chunk_size = 4096;
  int devices = 1;  // >1: events sharded over devices 0..devices-1 of this process
  static Backend serial() { return Backend{Kind::Serial, 1, 4096, 1}; }
  static Backend with_threads(unsigned n, std::size_t chunk = 4096) {
    if (n < 1) throw Error("bad-backend", "threads must be >= 1");
    return Backend{Kind::Threads, n, chunk, 1};
  }
  static Backend gpus(int n = 1) { return Backend{Kind::Gpu, 1, 4096, n}; }
};

enum class MetricKind { NegLogLikelihood, ChiSquared };
inline constexpr double kLogFloor = 1e-300;
inline constexpr double kChiSqEps = 1e-9;
inline constexpr double kPenaltyValue = 1e300;

// BoundModel = setData (engine.hpp:137-236): the event table lives in HBM.
// Backend::Serial / Threads are accepted and select nothing (the GPU always
// evaluates); Backend::gpus(n) shards over n devices at construction.
class BoundModel {
 public:
  BoundModel(PdfPtr pdf, const UnbinnedDataSet& ds, GridSpec grid = GridSpec{}, Backend backend = Backend::gpus())
      : pdf_(std::move(pdf)), grid_(grid), binned_(false) {
    events_ = to_event_table(ds);
    create(ds.observables(), 0.0, backend);
  }
  BoundModel(PdfPtr pdf, const BinnedDataSet& ds, GridSpec grid = GridSpec{}, Backend backend = Backend::gpus())
      : pdf_(std::move(pdf)), grid_(grid), binned_(true) {
    events_ = to_event_table(ds);
    create(ds.observables(), ds.total_content(), backend);
  }
  ~BoundModel() {
    for (const PdfNode* node : pre_)
      if (node->owner_ == this) node->owner_ = nullptr;
    pf_model_destroy(model_);
  }
  BoundModel(const BoundModel&) = delete;
  BoundModel& operator=(const BoundModel&) = delete;

  ParameterRegistry& registry() { return registry_; }
  const ParameterRegistry& registry() const { return registry_; }
  const IndexTable& table() const { return table_; }
  const PdfPtr& pdf() const { return pdf_; }
  const GridSpec& grid() const { return grid_; }
  std::size_t n_events() const { return events_.n_events; }
  bool binned() const { return binned_; }
  std::uint64_t log_floor_count() const { return pf_log_floor_count(model_); }
  pf_model* handle() const { return model_; }

  double eval_metric(std::span<const double> params, MetricKind metric, const Backend& = Backend::gpus()) {
    double out = 0;
    pf_status st{};
    const int rc = pf_eval_metric(model_, params.data(), params.size(),
                                  metric == MetricKind::ChiSquared ? PF_CHISQ : PF_NLL, &out, nullptr, &st);
    evaluated();
    check(rc, st);
    return out;
  }

  // the node norms of the last evaluation (pdf.hpp:88-92), fetched on demand
  void refresh_norms() {
    if (stale_) sync_norms();
  }
  void mark_evaluated() { evaluated(); }

  // K probes in one pass over the events (bitwise equal to K eval_metric calls)
  std::vector<double> eval_metric_batch(const std::vector<std::vector<double>>& ps, MetricKind metric) {
    const std::size_t n = registry_.n_parameters();
    std::vector<double> flat;
    for (const auto& p : ps) flat.insert(flat.end(), p.begin(), p.end());
    std::vector<double> out(ps.size());
    pf_status st{};
    const int rc = pf_eval_metric_batch(model_, flat.data(), ps.size(), n,
                                        metric == MetricKind::ChiSquared ? PF_CHISQ : PF_NLL, out.data(), &st);
    evaluated();
    check(rc, st);
    return out;
  }

 private:
  void create(const std::vector<VariablePtr>& obs, double total, const Backend& backend) {
    desc_.build(pdf_, obs);
    std::vector<int32_t> oi(obs.size());
    for (std::size_t i = 0; i < obs.size(); ++i) oi[i] = desc_.vidx.at(obs[i].get());
    pf_data data{binned_ ? 1 : 0, static_cast<int32_t>(obs.size()), oi.data(), events_.n_events,
                 events_.values.data(), total};
    pf_options opt{};
    opt.n_devices = std::max(1, backend.devices);
    opt.shard_count = 1;
    pf_status st{};
    check(pf_model_create(&desc_.graph, &data, static_cast<uint32_t>(grid_.points), &opt, &model_, &st), st);
    for (int32_t i = 0; i < pf_model_n_params(model_); ++i)
      registry_.register_parameter(desc_.vars[pf_model_param_variable(model_, i)]);
    ParameterRegistry scratch;
    table_ = finalize(scratch, pdf_, obs, binned_ ? 2 : 0);
    detail::preorder(pdf_.get(), pre_);
    for (std::size_t i = 0; i < pre_.size(); ++i)
      if (auto* poly = dynamic_cast<const PolynomialPdf*>(pre_[i])) poly->model_ = model_;
  }
  void evaluated() {
    stale_ = true;
    if (!pre_.empty() && pre_[0]->owner_ != this)
      for (const PdfNode* node : pre_) node->owner_ = this;
  }
  void sync_norms() {
    stale_ = false;
    const int n = static_cast<int>(pre_.size());
    std::vector<double> norms(n), errs(n);
    std::vector<int32_t> valid(n);
    pf_node_norms(model_, norms.data(), errs.data(), valid.data(), n);
    for (int i = 0; i < n; ++i)
      if (valid[i]) {
        auto* node = const_cast<PdfNode*>(pre_[i]);
        node->norm_ = norms[i];
        node->norm_err_ = errs[i];
        node->norm_valid_ = true;
      }
  }

  bool stale_ = false;
  PdfPtr pdf_;
  GridSpec grid_;
  bool binned_;
  EventTable events_;
  detail::GraphDesc desc_;
  ParameterRegistry registry_;
  IndexTable table_;
  std::vector<const PdfNode*> pre_;
  pf_model* model_ = nullptr;
};

// ---- generate.hpp --------------------------------------------------------
// ToyRng (generate.hpp:19-27): the fixed uniform bit recipe
// (mt19937_64() >> 11) * 2^-53, host side.
class ToyRng {
 public:
  explicit ToyRng(std::uint64_t seed) : engine_(seed) {}
  double uniform() { return 0x1.0p-53 * static_cast<double>(engine_() >> 11); }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }

 private:
  std::mt19937_64 engine_;
};

class detail_generate {
 public:
  static void fill(UnbinnedDataSet& ds, const std::vector<double>& cols, std::size_t n) {
    for (std::size_t c = 0; c < ds.obs_.size(); ++c)
      ds.cols_[c].assign(cols.begin() + static_cast<std::ptrdiff_t>(c * n),
                         cols.begin() + static_cast<std::ptrdiff_t>((c + 1) * n));
  }
};

// generate_events (generate.hpp:33-86), accept-reject on the GPU with the
// reference's envelope and ToyRng stream: the same seed gives the same
// sample; box observables are left at the last accepted event.
inline UnbinnedDataSet generate_events(const PdfPtr& pdf, const std::vector<VariablePtr>& observables,
                                       std::size_t n_events, std::uint64_t seed, GridSpec grid = GridSpec{}) {
  if (n_events < 1) throw Error("bad-arity", "generate_events: n_events >= 1");
  UnbinnedDataSet ds(observables);
  detail::GraphDesc g;
  g.build(pdf, observables);
  std::vector<int32_t> oi(observables.size());
  for (std::size_t i = 0; i < observables.size(); ++i) oi[i] = g.vidx.at(observables[i].get());
  std::vector<double> cols(observables.size() * n_events), last(observables.size());
  pf_options opt{};
  opt.n_devices = 1;
  opt.shard_count = 1;
  pf_status st{};
  check(pf_generate_events(&g.graph, oi.data(), static_cast<int32_t>(oi.size()), n_events, seed,
                           static_cast<uint32_t>(grid.points), &opt, cols.data(), last.data(), nullptr, &st),
        st);
  detail_generate::fill(ds, cols, n_events);
  for (std::size_t i = 0; i < observables.size(); ++i) observables[i]->value = last[i];
  return ds;
}

inline void PdfNode::refresh() const {
  if (owner_) owner_->refresh_norms();
}

// ---- fit.hpp ------------------------------------------------------------------
enum class MinimizerKind { QuasiNewton, NelderMead };
struct FitConfig {
  MinimizerKind minimizer = MinimizerKind::QuasiNewton;
  std::size_t max_iterations = 10000;
  double gradient_tolerance = 1e-6;
  double simplex_tolerance = 1e-8;
  bool batch_probes = true;  // FD stencil evaluated in one GPU pass (same values)
};
enum class FitStatus { Converged, MaxIterations, Failed };

struct FitResult {
  FitStatus status = FitStatus::Failed;
  std::vector<std::string> names;
  std::vector<double> params, uncertainties;
  bool uncertainties_available = false;
  double metric_value = 0.0;
  std::size_t n_metric_calls = 0;
  double wall_time_s = 0.0;
  double grad_max_norm = std::nan("");
  bool converged() const { return status == FitStatus::Converged; }
  std::string to_report() const {  // fit.hpp:46-71
    std::string out;
    char buf[96];
    const char* st = status == FitStatus::Converged ? "converged"
                     : status == FitStatus::MaxIterations ? "max-iterations" : "failed";
    out += std::string("status ") + st + "\n";
    std::snprintf(buf, sizeof buf, "metric_value %.17g\n", metric_value);
    out += buf;
    out += "metric_calls " + std::to_string(n_metric_calls) + "\n";
    std::snprintf(buf, sizeof buf, "wall_time_s %.6g\ngrad_max_norm %.6g\n", wall_time_s, grad_max_norm);
    out += buf;
    out += std::string("uncertainties ") + (uncertainties_available ? "available" : "unavailable") + "\n";
    for (std::size_t i = 0; i < names.size(); ++i) {
      std::snprintf(buf, sizeof buf, " %.17g %.17g\n", params[i], uncertainties_available ? uncertainties[i] : 0.0);
      out += "param " + names[i] + buf;
    }
    return out;
  }
};

// parfit::fit (fit.hpp:498-581), run by the native driver in libpfb200.so
inline FitResult fit(BoundModel& bm, MetricKind metric, const Backend& = Backend::gpus(),
                     const FitConfig& cfg = FitConfig{}) {
  auto& reg = bm.registry();
  const std::size_t n = reg.n_parameters();
  std::vector<double> start(n), lo(n), hi(n), step(n), outp(n), outu(n);
  std::vector<int32_t> fixed(n);
  for (std::size_t i = 0; i < n; ++i) {
    const auto& p = *reg.parameters()[i];
    start[i] = p.value;
    lo[i] = p.lower;
    hi[i] = p.upper;
    step[i] = p.step;
    fixed[i] = p.fixed ? 1 : 0;
  }
  pf_fit_config c{cfg.minimizer == MinimizerKind::NelderMead ? 1 : 0, cfg.batch_probes ? 1 : 0,
                  cfg.max_iterations, cfg.gradient_tolerance, cfg.simplex_tolerance};
  pf_fit_result r{};
  r.params = outp.data();
  r.uncertainties = outu.data();
  pf_status st{};
  const int rc = pf_fit(bm.handle(), metric == MetricKind::ChiSquared ? PF_CHISQ : PF_NLL, &c, start.data(),
                        fixed.data(), lo.data(), hi.data(), step.data(), &r, &st);
  bm.mark_evaluated();  // node norms: those of the fit's last evaluation
  check(rc, st);
  FitResult out;
  out.status = static_cast<FitStatus>(r.status);
  for (const auto& p : reg.parameters()) out.names.push_back(p->name);
  out.params = outp;
  out.uncertainties_available = r.uncertainties_available != 0;
  if (out.uncertainties_available) out.uncertainties = outu;
  out.metric_value = r.metric_value;
  out.n_metric_calls = r.n_metric_calls;
  out.wall_time_s = r.wall_time_s;
  out.grad_max_norm = r.grad_max_norm;
  if (out.status != FitStatus::Failed) reg.import_values(out.params);
  return out;
}

// GooFit's FitManager spelling: FitManager fitter(bm); fitter.fit();
class FitManager {
 public:
  explicit FitManager(BoundModel& bm, MetricKind metric = MetricKind::NegLogLikelihood)
      : bm_(bm), metric_(metric) {}
  FitResult fit(const FitConfig& cfg = FitConfig{}) { return parfit::fit(bm_, metric_, Backend::gpus(), cfg); }

 private:
  BoundModel& bm_;
  MetricKind metric_;
};

}  // namespace parfit

#endif  // PARFIT_B200_PARFIT_HPP
