// fit.hpp — FitManager contract of the reference (fit.hpp:19-581): MINUIT-
// style sine bound transform, five-point finite-difference gradient, BFGS
// with Armijo backtracking and a gradient-norm endgame, Nelder-Mead, and
// uncertainties from the inverse finite-difference Hessian.
//
// The arithmetic of every step is the reference's, so given bitwise-equal
// objective values the iterates, the call count and the result are bitwise
// equal too.  Independent probes (the 4n gradient stencil points and the
// Hessian stencil) may be evaluated as ONE batched device pass
// (Objective::batch); this changes neither the values nor their use.
#pragma once

#include <cstdint>
#include <functional>
#include <vector>

namespace pfb {

struct Objective {
  virtual ~Objective() = default;
  virtual double f(const std::vector<double>& u) = 0;
  // default: sequential calls
  virtual void batch(const std::vector<std::vector<double>>& us, std::vector<double>& out) {
    out.resize(us.size());
    for (size_t i = 0; i < us.size(); ++i) out[i] = f(us[i]);
  }
};

class Transform {  // BoundTransform, fit.hpp:77-129
 public:
  Transform(std::vector<double> lower, std::vector<double> upper, std::vector<double> step)
      : lo_(std::move(lower)), hi_(std::move(upper)), step_(std::move(step)) {}
  double to_external(size_t i, double u) const;
  double to_internal(size_t i, double p) const;
  double jacobian(size_t i, double u) const;
  double fd_step(size_t i, double u) const;

 private:
  std::vector<double> lo_, hi_, step_;
};

enum class Status { Converged = 0, MaxIterations = 1, Failed = 2 };

struct Config {
  int minimizer = 0;  // 0 BFGS, 1 Nelder-Mead
  bool batch_probes = true;
  uint64_t max_iterations = 10000;
  double gradient_tolerance = 1e-6;
  double simplex_tolerance = 1e-8;
};

struct Outcome {
  std::vector<double> u;
  double f = 0.0;
  Status status = Status::Failed;
  std::vector<double> grad;
};

double max_abs(const std::vector<double>& v);

// numeric_gradient (fit.hpp:138-171); `one_sided` as the reference's flag
std::vector<double> gradient(Objective& obj, const std::vector<double>& u,
                             const std::vector<double>& h, bool batch, bool* one_sided);
// numeric_hessian (fit.hpp:180-208)
std::vector<std::vector<double>> hessian(Objective& obj, const std::vector<double>& u,
                                         const std::vector<double>& h, bool batch);
// invert_spd (fit.hpp:212-244)
bool invert_spd(const std::vector<std::vector<double>>& a, std::vector<std::vector<double>>& inv);

Outcome bfgs(Objective& obj, std::vector<double> u, const Config& cfg,
             const std::function<std::vector<double>(const std::vector<double>&)>& grad);
Outcome nelder_mead(Objective& obj, std::vector<double> u0, const Config& cfg,
                    const std::vector<double>& scale);

struct FitOutput {
  Status status = Status::Failed;
  std::vector<double> params, uncertainties;
  bool uncertainties_available = false;
  double metric_value = 0.0;
  uint64_t n_calls = 0;
  double wall_time_s = 0.0;
  double grad_max_norm = 0.0;
};

// parfit::fit (fit.hpp:498-581) over an external-space metric.
//   metric(p)            one evaluation (external parameters, full vector)
//   metric_batch(ps,out) K evaluations in one pass (may be empty)
FitOutput fit(const std::function<double(const std::vector<double>&)>& metric,
              const std::function<void(const std::vector<std::vector<double>>&,
                                       std::vector<double>&)>& metric_batch,
              bool chi_squared, const std::vector<double>& start, const std::vector<int>& fixed,
              const std::vector<double>& lower, const std::vector<double>& upper,
              const std::vector<double>& step, const Config& cfg);

}  // namespace pfb
