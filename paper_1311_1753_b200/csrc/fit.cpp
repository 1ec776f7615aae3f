// fit.cpp — FitManager restated from the reference's fit.hpp (cited per
// function).  Host code: the minimiser is sequential by nature; the hot
// objective behind it runs on the GPU.
#include "fit.hpp"

#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>

#include "graph.hpp"

namespace pfb {

// p = a + (b - a) (sin u + 1) / 2  (fit.hpp:89-91)
double Transform::to_external(size_t i, double u) const {
  return lo_[i] + (hi_[i] - lo_[i]) * (std::sin(u) + 1.0) / 2.0;
}

double Transform::to_internal(size_t i, double p) const {  // fit.hpp:93-97
  double z = 2.0 * (p - lo_[i]) / (hi_[i] - lo_[i]) - 1.0;
  z = std::min(std::max(z, -1.0), 1.0);
  return std::asin(z);
}

double Transform::jacobian(size_t i, double u) const {  // fit.hpp:100-102
  return (hi_[i] - lo_[i]) * std::cos(u) / 2.0;
}

double Transform::fd_step(size_t i, double u) const {  // fit.hpp:121-125
  const double j = std::abs(jacobian(i, u));
  const double scaled = j > 1e-12 ? step_[i] / j : step_[i];
  return std::max(1e-5, 2e-3 * scaled);
}

double max_abs(const std::vector<double>& v) {  // fit.hpp:173-177
  double m = 0.0;
  for (double x : v) m = std::max(m, std::abs(x));
  return m;
}

// Richardson five-point stencil with the one-sided fallback (fit.hpp:138-171).
// Batched: the 4n stencil points go to the device in one pass; the values
// are then consumed in the reference's order, so g is bitwise identical.
namespace {
double stencil(Objective& obj, const std::vector<double>& u, double h, const double* v,
               bool* one_sided) {
  const double fp = v[0], fm = v[1], fp2 = v[2], fm2 = v[3];
  if (std::isfinite(fp) && std::isfinite(fm) && std::isfinite(fp2) && std::isfinite(fm2))
    return (8.0 * (fp - fm) - (fp2 - fm2)) / (12.0 * h);
  if (std::isfinite(fp) && std::isfinite(fm)) return (fp - fm) / (2.0 * h);
  const double f0 = obj.f(u);
  if (one_sided) *one_sided = true;
  if (std::isfinite(fp)) return (fp - f0) / h;
  if (std::isfinite(fm)) return (f0 - fm) / h;
  throw Error("non-finite-objective", "gradient probe failed both sides");
}
}  // namespace

std::vector<double> gradient(Objective& obj, const std::vector<double>& u,
                             const std::vector<double>& h, bool batch, bool* one_sided) {
  const size_t n = u.size();
  std::vector<double> g(n);
  if (batch) {
    std::vector<std::vector<double>> probes;
    probes.reserve(4 * n);
    for (size_t i = 0; i < n; ++i) {
      std::vector<double> p = u;
      p[i] = u[i] + h[i];
      probes.push_back(p);
      p[i] = u[i] - h[i];
      probes.push_back(p);
      p[i] = u[i] + 2.0 * h[i];
      probes.push_back(p);
      p[i] = u[i] - 2.0 * h[i];
      probes.push_back(p);
    }
    std::vector<double> vals;
    obj.batch(probes, vals);
    for (size_t i = 0; i < n; ++i) g[i] = stencil(obj, u, h[i], vals.data() + 4 * i, one_sided);
    return g;
  }
  std::vector<double> probe = u;
  for (size_t i = 0; i < n; ++i) {
    double v[4];
    probe[i] = u[i] + h[i];
    v[0] = obj.f(probe);
    probe[i] = u[i] - h[i];
    v[1] = obj.f(probe);
    probe[i] = u[i] + 2.0 * h[i];
    v[2] = obj.f(probe);
    probe[i] = u[i] - 2.0 * h[i];
    v[3] = obj.f(probe);
    probe[i] = u[i];
    g[i] = stencil(obj, u, h[i], v, one_sided);
  }
  return g;
}

// numeric_hessian (fit.hpp:180-208): probe list in the reference's call order
std::vector<std::vector<double>> hessian(Objective& obj, const std::vector<double>& u,
                                         const std::vector<double>& h, bool batch) {
  const size_t n = u.size();
  std::vector<std::vector<double>> probes;
  probes.push_back(u);
  std::vector<double> x = u;
  for (size_t i = 0; i < n; ++i) {
    x[i] = u[i] + h[i];
    probes.push_back(x);
    x[i] = u[i] - h[i];
    probes.push_back(x);
    x[i] = u[i];
    for (size_t j = i + 1; j < n; ++j) {
      x[i] = u[i] + h[i];
      x[j] = u[j] + h[j];
      probes.push_back(x);
      x[j] = u[j] - h[j];
      probes.push_back(x);
      x[i] = u[i] - h[i];
      x[j] = u[j] + h[j];
      probes.push_back(x);
      x[j] = u[j] - h[j];
      probes.push_back(x);
      x[i] = u[i];
      x[j] = u[j];
    }
  }
  std::vector<double> v;
  if (batch) {
    obj.batch(probes, v);
  } else {
    v.resize(probes.size());
    for (size_t k = 0; k < probes.size(); ++k) v[k] = obj.f(probes[k]);
  }
  std::vector<std::vector<double>> H(n, std::vector<double>(n, 0.0));
  const double f0 = v[0];
  size_t k = 1;
  for (size_t i = 0; i < n; ++i) {
    const double fp = v[k++], fm = v[k++];
    H[i][i] = (fp - 2.0 * f0 + fm) / (h[i] * h[i]);
    for (size_t j = i + 1; j < n; ++j) {
      const double fpp = v[k++], fpm = v[k++], fmp = v[k++], fmm = v[k++];
      H[i][j] = H[j][i] = (fpp - fpm - fmp + fmm) / (4.0 * h[i] * h[j]);
    }
  }
  return H;
}

// Cholesky inverse (fit.hpp:212-244)
bool invert_spd(const std::vector<std::vector<double>>& A, std::vector<std::vector<double>>& inv) {
  const size_t n = A.size();
  std::vector<std::vector<double>> Lm(n, std::vector<double>(n, 0.0));
  for (size_t i = 0; i < n; ++i) {
    for (size_t j = 0; j <= i; ++j) {
      double s = A[i][j];
      for (size_t k = 0; k < j; ++k) s -= Lm[i][k] * Lm[j][k];
      if (i == j) {
        if (!(s > 0.0) || !std::isfinite(s)) return false;
        Lm[i][i] = std::sqrt(s);
      } else {
        Lm[i][j] = s / Lm[j][j];
      }
    }
  }
  inv.assign(n, std::vector<double>(n, 0.0));
  std::vector<double> y(n);
  for (size_t c = 0; c < n; ++c) {
    for (size_t i = 0; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
      for (size_t k = 0; k < i; ++k) s -= Lm[i][k] * y[k];
      y[i] = s / Lm[i][i];
    }
    for (size_t i = n; i-- > 0;) {
      double s = y[i];
      for (size_t k = i + 1; k < n; ++k) s -= Lm[k][i] * inv[k][c];
      inv[i][c] = s / Lm[i][i];
    }
  }
  return true;
}

namespace {
void reset_identity(std::vector<std::vector<double>>& H) {
  for (size_t i = 0; i < H.size(); ++i) {
    std::fill(H[i].begin(), H[i].end(), 0.0);
    H[i][i] = 1.0;
  }
}
}  // namespace

// BFGS + Armijo backtracking (c1 = 1e-4, halving) + endgame (fit.hpp:270-400)
Outcome bfgs(Objective& obj, std::vector<double> u, const Config& cfg,
             const std::function<std::vector<double>(const std::vector<double>&)>& grad) {
  const size_t n = u.size();
  Outcome out;
  double fu = obj.f(u);
  if (!std::isfinite(fu)) {
    out.u = std::move(u);
    out.status = Status::Failed;
    return out;
  }
  std::vector<std::vector<double>> H(n, std::vector<double>(n, 0.0));
  reset_identity(H);
  std::vector<double> g = grad(u);
  const double c1 = 1e-4;
  bool reset_used = false;
  Status status = Status::MaxIterations;
  for (uint64_t iter = 0; iter < cfg.max_iterations; ++iter) {
    if (max_abs(g) <= cfg.gradient_tolerance) {
      status = Status::Converged;
      break;
    }
    std::vector<double> d(n, 0.0);
    for (size_t i = 0; i < n; ++i)
      for (size_t j = 0; j < n; ++j) d[i] -= H[i][j] * g[j];
    double gd = 0.0;
    for (size_t i = 0; i < n; ++i) gd += g[i] * d[i];
    if (!(gd < 0.0)) {  // restart from steepest descent
      reset_identity(H);
      for (size_t i = 0; i < n; ++i) d[i] = -g[i];
      gd = 0.0;
      for (size_t i = 0; i < n; ++i) gd += g[i] * d[i];
      if (!(gd < 0.0)) {
        status = Status::Converged;
        break;
      }
    }
    double t = 1.0;
    std::vector<double> u_new(n);
    double f_new = fu;
    bool accepted = false;
    while (t > 1e-16) {
      for (size_t i = 0; i < n; ++i) u_new[i] = u[i] + t * d[i];
      f_new = obj.f(u_new);
      if (std::isfinite(f_new) && f_new <= fu + c1 * t * gd) {
        accepted = true;
        break;
      }
      t *= 0.5;
    }
    bool stagnant = accepted;
    if (accepted)
      for (size_t i = 0; i < n; ++i)
        if (u_new[i] != u[i]) {
          stagnant = false;
          break;
        }
    if (!accepted || stagnant) {
      if (!accepted && !reset_used) {
        reset_used = true;
        reset_identity(H);
        continue;
      }
      // endgame: damped quasi-Newton steps accepted on gradient-norm decrease
      bool moved = false;
      const double gnorm = max_abs(g);
      double td = 1.0;
      for (int attempt = 0; attempt < 8 && !moved; ++attempt, td *= 0.5) {
        bool distinct = false;
        for (size_t i = 0; i < n; ++i) {
          u_new[i] = u[i] + td * d[i];
          if (u_new[i] != u[i]) distinct = true;
        }
        if (!distinct) break;
        std::vector<double> g_try = grad(u_new);
        if (max_abs(g_try) < gnorm) {
          const double f_try = obj.f(u_new);
          if (std::isfinite(f_try)) {
            u = u_new;
            fu = f_try;
            g = std::move(g_try);
            moved = true;
          }
        }
      }
      if (!moved) break;
      reset_used = false;
      continue;
    }
    reset_used = false;
    std::vector<double> g_new = grad(u_new);
    std::vector<double> s(n), y(n);
    double sy = 0.0;
    for (size_t i = 0; i < n; ++i) {
      s[i] = u_new[i] - u[i];
      y[i] = g_new[i] - g[i];
      sy += s[i] * y[i];
    }
    if (sy > 0.0 && std::isfinite(sy)) {
      std::vector<double> Hy(n, 0.0);
      for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < n; ++j) Hy[i] += H[i][j] * y[j];
      double yHy = 0.0;
      for (size_t i = 0; i < n; ++i) yHy += y[i] * Hy[i];
      for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j < n; ++j)
          H[i][j] += (sy + yHy) * s[i] * s[j] / (sy * sy) - (Hy[i] * s[j] + s[i] * Hy[j]) / sy;
    }
    u = std::move(u_new);
    fu = f_new;
    g = std::move(g_new);
  }
  if (status != Status::Converged && max_abs(g) <= cfg.gradient_tolerance) status = Status::Converged;
  out.u = std::move(u);
  out.f = fu;
  out.grad = std::move(g);
  out.status = status;
  return out;
}

// Nelder-Mead (reflection 1, expansion 2, contraction 0.5, shrink 0.5),
// fit.hpp:404-490
Outcome nelder_mead(Objective& obj, std::vector<double> u0, const Config& cfg,
                    const std::vector<double>& scale) {
  const size_t n = u0.size();
  Outcome out;
  std::vector<std::vector<double>> simplex;
  std::vector<double> fv;
  simplex.push_back(u0);
  fv.push_back(obj.f(u0));
  if (!std::isfinite(fv[0])) {
    out.u = std::move(u0);
    out.status = Status::Failed;
    return out;
  }
  for (size_t i = 0; i < n; ++i) {
    std::vector<double> v = u0;
    v[i] += scale[i];
    simplex.push_back(v);
    fv.push_back(obj.f(v));
  }
  auto order = [&] {
    std::vector<size_t> idx(simplex.size());
    for (size_t i = 0; i < idx.size(); ++i) idx[i] = i;
    std::sort(idx.begin(), idx.end(), [&](size_t a, size_t b) { return fv[a] < fv[b]; });
    std::vector<std::vector<double>> s2;
    std::vector<double> f2;
    for (size_t i : idx) {
      s2.push_back(simplex[i]);
      f2.push_back(fv[i]);
    }
    simplex = std::move(s2);
    fv = std::move(f2);
  };
  order();
  Status status = Status::MaxIterations;
  for (uint64_t iter = 0; iter < cfg.max_iterations; ++iter) {
    const double spread = std::abs(fv.back() - fv.front()) / std::max(1.0, std::abs(fv.front()));
    if (spread <= cfg.simplex_tolerance) {
      status = Status::Converged;
      break;
    }
    std::vector<double> centroid(n, 0.0);
    for (size_t i = 0; i < n; ++i) {
      for (size_t v = 0; v < n; ++v) centroid[i] += simplex[v][i];
      centroid[i] /= static_cast<double>(n);
    }
    auto point = [&](double coeff) {
      std::vector<double> p(n);
      for (size_t i = 0; i < n; ++i) p[i] = centroid[i] + coeff * (centroid[i] - simplex.back()[i]);
      return p;
    };
    std::vector<double> refl = point(1.0);
    const double f_refl = obj.f(refl);
    if (f_refl < fv.front()) {
      std::vector<double> expd = point(2.0);
      const double f_exp = obj.f(expd);
      if (f_exp < f_refl) {
        simplex.back() = expd;
        fv.back() = f_exp;
      } else {
        simplex.back() = refl;
        fv.back() = f_refl;
      }
    } else if (f_refl < fv[fv.size() - 2]) {
      simplex.back() = refl;
      fv.back() = f_refl;
    } else {
      std::vector<double> con = point(-0.5);
      const double f_con = obj.f(con);
      if (f_con < fv.back()) {
        simplex.back() = con;
        fv.back() = f_con;
      } else {
        for (size_t v = 1; v < simplex.size(); ++v) {
          for (size_t i = 0; i < n; ++i)
            simplex[v][i] = simplex[0][i] + 0.5 * (simplex[v][i] - simplex[0][i]);
          fv[v] = obj.f(simplex[v]);
        }
      }
    }
    order();
  }
  out.u = simplex.front();
  out.f = fv.front();
  out.status = status;
  return out;
}

namespace {

// internal-space objective over the free parameters (fit.hpp:508-522)
struct Internal : Objective {
  const std::function<double(const std::vector<double>&)>& metric;
  const std::function<void(const std::vector<std::vector<double>>&, std::vector<double>&)>& mbatch;
  const Transform& tr;
  const std::vector<size_t>& free_idx;
  const std::vector<double>& p_template;
  uint64_t calls = 0;

  Internal(const std::function<double(const std::vector<double>&)>& m,
           const std::function<void(const std::vector<std::vector<double>>&, std::vector<double>&)>& b,
           const Transform& t, const std::vector<size_t>& fi, const std::vector<double>& pt)
      : metric(m), mbatch(b), tr(t), free_idx(fi), p_template(pt) {}

  std::vector<double> expand(const std::vector<double>& u) const {
    std::vector<double> p = p_template;
    for (size_t k = 0; k < u.size(); ++k) p[free_idx[k]] = tr.to_external(free_idx[k], u[k]);
    return p;
  }
  // diagnostics: PFB200_FIT_TRACE=<file> appends every evaluated point
  // (external parameters) and its metric, %.17g, one line per call
  static void trace(const std::vector<double>& p, double v) {
    static const char* path = std::getenv("PFB200_FIT_TRACE");
    if (!path) return;
    if (FILE* fh = std::fopen(path, "a")) {
      std::fprintf(fh, "%.17g", v);
      for (double x : p) std::fprintf(fh, " %.17g", x);
      std::fprintf(fh, "\n");
      std::fclose(fh);
    }
  }
  double f(const std::vector<double>& u) override {
    ++calls;
    const std::vector<double> p = expand(u);
    const double v = metric(p);
    trace(p, v);
    return v;
  }
  void batch(const std::vector<std::vector<double>>& us, std::vector<double>& out) override {
    if (!mbatch) {
      Objective::batch(us, out);
      return;
    }
    std::vector<std::vector<double>> ps;
    ps.reserve(us.size());
    for (const auto& u : us) ps.push_back(expand(u));
    calls += us.size();
    mbatch(ps, out);
    for (size_t i = 0; i < ps.size() && i < out.size(); ++i) trace(ps[i], out[i]);
  }
};

}  // namespace

// parfit::fit orchestration (fit.hpp:498-581)
FitOutput fit(const std::function<double(const std::vector<double>&)>& metric,
              const std::function<void(const std::vector<std::vector<double>>&,
                                       std::vector<double>&)>& metric_batch,
              bool chi_squared, const std::vector<double>& start, const std::vector<int>& fixed,
              const std::vector<double>& lower, const std::vector<double>& upper,
              const std::vector<double>& step, const Config& cfg) {
  std::vector<size_t> free_idx;
  for (size_t i = 0; i < start.size(); ++i)
    if (!fixed[i]) free_idx.push_back(i);
  if (free_idx.empty()) throw Error("no-parameters", "fit needs >= 1 free parameter");
  const auto t0 = std::chrono::steady_clock::now();
  Transform tr(lower, upper, step);
  Internal obj(metric, metric_batch, tr, free_idx, start);
  const bool batch = cfg.batch_probes && static_cast<bool>(metric_batch);
  auto grad = [&](const std::vector<double>& u) {
    std::vector<double> h(u.size());
    for (size_t k = 0; k < u.size(); ++k) h[k] = tr.fd_step(free_idx[k], u[k]);
    return gradient(obj, u, h, batch, nullptr);
  };
  std::vector<double> u0(free_idx.size());
  for (size_t k = 0; k < free_idx.size(); ++k) u0[k] = tr.to_internal(free_idx[k], start[free_idx[k]]);

  Outcome mo;
  if (cfg.minimizer == 0) {
    mo = bfgs(obj, u0, cfg, grad);
  } else {
    std::vector<double> scale(u0.size());
    for (size_t k = 0; k < u0.size(); ++k) scale[k] = tr.fd_step(free_idx[k], u0[k]) * 100.0;
    mo = nelder_mead(obj, u0, cfg, scale);
  }

  FitOutput r;
  r.status = mo.status;
  r.params = obj.expand(mo.u);
  r.metric_value = mo.f;
  if (mo.grad.empty() && mo.status != Status::Failed) mo.grad = grad(mo.u);
  r.grad_max_norm = mo.grad.empty() ? std::numeric_limits<double>::quiet_NaN() : max_abs(mo.grad);
  if (mo.status != Status::Failed) {
    std::vector<double> hh(mo.u.size());
    for (size_t k = 0; k < mo.u.size(); ++k) hh[k] = 10.0 * tr.fd_step(free_idx[k], mo.u[k]);
    std::vector<std::vector<double>> cov;
    auto H = hessian(obj, mo.u, hh, batch);
    if (invert_spd(H, cov)) {
      r.uncertainties_available = true;
      r.uncertainties.assign(start.size(), 0.0);
      const double scale = chi_squared ? 2.0 : 1.0;  // fit.hpp:566-567
      for (size_t k = 0; k < mo.u.size(); ++k) {
        const double var_int = scale * cov[k][k];
        const double j = tr.jacobian(free_idx[k], mo.u[k]);
        r.uncertainties[free_idx[k]] = var_int > 0 ? std::sqrt(var_int) * std::abs(j) : 0.0;
      }
    }
  }
  r.n_calls = obj.calls;
  r.wall_time_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  return r;
}

}  // namespace pfb
