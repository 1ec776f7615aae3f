// graph.cpp — GraphFinalizer restatement (pdf.hpp:504-613) plus the
// constructor-time validation of every node kind (pdf.hpp:210-497).
#include "graph.hpp"

#include <algorithm>
#include <functional>
#include <set>
#include <unordered_map>

namespace pfb {

const char* kind_name(int kind) {
  switch (kind) {
    case PF_EXPONENTIAL: return "ExpPdf";
    case PF_GAUSSIAN: return "GaussianPdf";
    case PF_BREIT_WIGNER: return "BreitWignerPdf";
    case PF_POLYNOMIAL: return "PolynomialPdf";
    case PF_PRODUCT: return "ProdPdf";
    case PF_SUM: return "AddPdf";
    case PF_COMPOSITE: return "CompositePdf";
    case PF_MAPPED: return "MappedPdf";
    case PF_CONVOLUTION: return "ConvolutionPdf";
    case PF_ARGUS: return "ArgusPdf";
    case PF_DALITZ: return "DalitzPlotPdf";
    case PF_TDDP: return "TddpPdf";
  }
  return "unknown";
}

namespace {

// ParameterRegistry::register_into (variable.hpp:121-135): idempotent per
// variable identity, rejects a second identity under the same name.
struct Registry {
  std::vector<int> params, observables;
  std::unordered_map<std::string, int> param_by_name, obs_by_name;
  std::unordered_map<int, int> param_slot;

  int register_parameter(const std::vector<Var>& vars, int v) {
    if (vars[v].role != PF_PARAMETER)
      throw Error("wrong-role", "'" + vars[v].name + "' is not a parameter");
    auto it = param_by_name.find(vars[v].name);
    if (it != param_by_name.end()) {
      if (it->second != v)
        throw Error("name-collision", "distinct Variables both named '" + vars[v].name + "'");
      return param_slot.at(v);
    }
    int slot = static_cast<int>(params.size());
    params.push_back(v);
    param_by_name.emplace(vars[v].name, v);
    param_slot.emplace(v, slot);
    return slot;
  }

  void register_observable(const std::vector<Var>& vars, int v) {
    if (vars[v].role != PF_OBSERVABLE)
      throw Error("wrong-role", "'" + vars[v].name + "' is not an observable");
    auto it = obs_by_name.find(vars[v].name);
    if (it != obs_by_name.end()) {
      if (it->second != v)
        throw Error("name-collision", "distinct Variables both named '" + vars[v].name + "'");
      return;
    }
    observables.push_back(v);
    obs_by_name.emplace(vars[v].name, v);
  }
};

void require(bool ok, const std::string& code, const std::string& detail) {
  if (!ok) throw Error(code, detail);
}

// Constructor contracts of each node class.
void validate_node(const pf_graph& g, int idx) {
  const pf_node& n = g.nodes[idx];
  const std::string name = n.name ? n.name : "";
  auto var_ok = [&](int v) { return v >= 0 && v < g.n_variables; };
  auto node_ok = [&](int c) { return c >= 0 && c < g.n_nodes; };
  auto is_obs = [&](int v) { return var_ok(v) && g.variables[v].role == PF_OBSERVABLE; };
  auto is_par = [&](int v) { return var_ok(v) && g.variables[v].role == PF_PARAMETER; };
  for (int i = 0; i < n.n_children; ++i)
    require(node_ok(n.children[i]), "bad-arity", name + ": null child");
  switch (n.kind) {
    case PF_EXPONENTIAL:  // pdf.hpp:212-232
      require(n.n_obs == 1 && is_obs(n.obs[0]), "wrong-role", name + ": x must be an observable");
      require(n.n_params == 1 && is_par(n.params[0]), "wrong-role",
              name + ": alpha must be a parameter");
      break;
    case PF_GAUSSIAN:  // pdf.hpp:237-249
      require(n.n_obs == 1 && is_obs(n.obs[0]), "wrong-role", name + ": x must be an observable");
      require(n.n_params == 2 && is_par(n.params[0]), "wrong-role",
              name + ": mean must be a parameter");
      require(is_par(n.params[1]), "wrong-role", name + ": sigma must be a parameter");
      require(g.variables[n.params[1]].lower > 0, "nonpositive-sigma",
              name + ": sigma limits must exclude 0");
      break;
    case PF_BREIT_WIGNER:  // pdf.hpp:266-278
      require(n.n_obs == 1 && is_obs(n.obs[0]), "wrong-role", name + ": x must be an observable");
      require(n.n_params == 2 && is_par(n.params[0]), "wrong-role",
              name + ": mass must be a parameter");
      require(is_par(n.params[1]), "wrong-role", name + ": width must be a parameter");
      require(g.variables[n.params[1]].lower > 0, "nonpositive-width",
              name + ": width limits must exclude 0");
      break;
    case PF_POLYNOMIAL:  // pdf.hpp:294-305
      require(n.n_obs == 1 && is_obs(n.obs[0]), "wrong-role", name + ": x must be an observable");
      require(n.n_params >= 1, "bad-arity", name + ": need >= 1 coefficient");
      for (int i = 0; i < n.n_params; ++i)
        require(is_par(n.params[i]), "wrong-role", name + ": coefficients must be parameters");
      break;
    case PF_ARGUS:  // ArgusPdf(x; m0, c, p), new
      require(n.n_obs == 1 && is_obs(n.obs[0]), "wrong-role", name + ": x must be an observable");
      require(n.n_params == 3, "bad-arity", name + ": need m0, c, p");
      for (int i = 0; i < 3; ++i)
        require(is_par(n.params[i]), "wrong-role", name + ": m0, c, p must be parameters");
      require(g.variables[n.params[0]].lower > 0, "nonpositive-endpoint",
              name + ": m0 limits must exclude 0");
      break;
    case PF_DALITZ:    // DalitzPlotPdf(m12^2, m13^2; resonances), new
    case PF_TDDP: {    // TddpPdf(m12^2, m13^2, t; resonances, tau, x, y), new
      const bool td = n.kind == PF_TDDP;
      require(n.n_obs == (td ? 3 : 2) && is_obs(n.obs[0]) && is_obs(n.obs[1]) && (!td || is_obs(n.obs[2])),
              "wrong-role", name + (td ? ": m12^2, m13^2 and t must be observables" : ": m12^2 and m13^2 must be observables"));
      const int nres = (n.n_params - (td ? 3 : 0)) / 4;
      require(nres >= 1 && n.n_params == 4 * nres + (td ? 3 : 0), "bad-arity",
              name + (td ? ": need (mass, width, Re c, Im c) per resonance, then tau, x, y"
                         : ": need (mass, width, Re c, Im c) per resonance"));
      if (td) {
        require(is_par(n.params[4 * nres]) && is_par(n.params[4 * nres + 1]) && is_par(n.params[4 * nres + 2]),
                "wrong-role", name + ": tau, x, y must be parameters");
        require(g.variables[n.params[4 * nres]].lower > 0, "nonpositive-lifetime", name + ": tau limits must exclude 0");
        require(n.n_reals >= 5 && n.reals[1] == n.reals[2], "bad-kinematics",
                name + ": daughters 1 and 2 must be CP conjugates (m1 == m2)");
      }
      require(n.n_reals == 5 + 2 * nres, "bad-arity", name + ": need M, m1, m2, m3, R and (channel, spin) per resonance");
      for (int i = 0; i < 4 * nres; ++i)
        require(is_par(n.params[i]), "wrong-role", name + ": resonance constants must be parameters");
      for (int r = 0; r < nres; ++r) {
        const double ch = n.reals[5 + 2 * r], sp = n.reals[6 + 2 * r];
        require(ch == 12 || ch == 13 || ch == 23, "bad-channel", name + ": channel must be 12, 13 or 23");
        require(sp == 0 || sp == 1, "bad-spin", name + ": spin must be 0 or 1");
        require(g.variables[n.params[4 * r + 1]].lower > 0, "nonpositive-width",
                name + ": width limits must exclude 0");
      }
      require(n.reals[0] > n.reals[1] + n.reals[2] + n.reals[3] && n.reals[1] >= 0 && n.reals[2] >= 0 &&
                  n.reals[3] >= 0 && n.reals[4] >= 0,
              "bad-kinematics", name + ": need M > m1 + m2 + m3, masses and R >= 0");
      break;
    }
    case PF_PRODUCT:  // pdf.hpp:332-337
      require(n.n_children >= 2, "bad-arity", name + ": product needs >= 2 children");
      require(n.n_params == 0 && n.n_obs == 0, "bad-arity", name + ": product has no own variables");
      break;
    case PF_SUM:  // pdf.hpp:354-366
      require(n.n_children >= 2, "bad-arity", name + ": sum needs >= 2 children");
      require(n.n_params == n.n_children - 1, "fraction-count-mismatch",
              name + ": need n_children - 1 fractions");
      for (int i = 0; i < n.n_params; ++i)
        require(is_par(n.params[i]), "wrong-role", name + ": fractions must be parameters");
      break;
    case PF_COMPOSITE:  // pdf.hpp:397-401
      require(n.n_children == 2, "bad-arity", name + ": null child");
      break;
    case PF_MAPPED:  // pdf.hpp:422-432
      require(n.n_children >= 1, "bad-arity", name + ": need >= 1 target");
      require(n.n_reals == n.n_children + 1, "bad-arity", name + ": need n_targets + 1 boundaries");
      for (int i = 1; i < n.n_reals; ++i)
        require(n.reals[i - 1] < n.reals[i], "non-monotone-boundaries", name);
      break;
    case PF_CONVOLUTION:  // pdf.hpp:464-470
      require(n.n_children == 2, "bad-arity", name + ": null child");
      require(n.quadrature_points >= 2, "bad-grid", name + ": need >= 2 quadrature points");
      break;
    default:
      throw Error("bad-kind", name + ": unknown node kind " + std::to_string(n.kind));
  }
}

}  // namespace

Program finalize(const pf_graph& g, int n_data_obs, const int32_t* data_obs, int reserved) {
  Program pg;
  if (g.n_variables < 0 || g.n_nodes < 0) throw Error("bad-graph", "negative sizes");
  pg.vars.resize(g.n_variables);
  for (int i = 0; i < g.n_variables; ++i) {
    const pf_variable& v = g.variables[i];
    Var& w = pg.vars[i];
    w.name = v.name ? v.name : "";
    w.value = v.value;
    w.lower = v.lower;
    w.upper = v.upper;
    w.step = v.step;
    w.fixed = v.fixed != 0;
    w.role = v.role;
  }
  for (int i = 0; i < g.n_nodes; ++i) validate_node(g, i);
  if (g.n_nodes == 0 || g.root < 0) return pg;  // empty graph (test_model_core.cpp:96-100)
  if (g.root >= g.n_nodes) throw Error("bad-graph", "root index out of range");

  // data columns (GraphFinalizer ctor, pdf.hpp:508-515)
  std::unordered_map<int, int> columns;
  pg.n_data_obs = n_data_obs;
  pg.reserved = reserved;
  for (int c = 0; c < n_data_obs; ++c) {
    int v = data_obs[c];
    if (v < 0 || v >= g.n_variables) throw Error("bad-graph", "data observable index");
    columns[v] = c;
    pg.data_obs.push_back(v);
  }
  int next_column = n_data_obs + reserved;

  // pre-order collection; Composite: outer synthetic, then inner (pdf.hpp:540-549)
  std::vector<std::pair<int, bool>> order;
  std::function<void(int, bool, int)> collect = [&](int idx, bool synthetic, int depth) {
    if (depth > 256) throw Error("bad-graph", "graph is cyclic or too deep");
    order.emplace_back(idx, synthetic);
    const pf_node& n = g.nodes[idx];
    if (n.kind == PF_COMPOSITE) {
      collect(n.children[0], true, depth + 1);
      collect(n.children[1], synthetic, depth + 1);
    } else {
      for (int i = 0; i < n.n_children; ++i) collect(n.children[i], synthetic, depth + 1);
    }
  };
  collect(g.root, false, 0);

  Registry reg;
  auto column_of = [&](int v, bool synthetic) -> int {
    auto it = columns.find(v);
    if (it != columns.end()) return it->second;
    if (!synthetic)
      throw Error("unbound-observable", "'" + pg.vars[v].name + "' is not in the bound data set");
    int col = next_column++;
    columns.emplace(v, col);
    return col;
  };

  // rows (pdf.hpp:521-533); children ids follow from pre-order positions
  pg.nodes.resize(order.size());
  for (size_t id = 0; id < order.size(); ++id) {
    const pf_node& n = g.nodes[order[id].first];
    Node& node = pg.nodes[id];
    node.kind = n.kind;
    node.name = n.name ? n.name : "";
    node.desc_index = order[id].first;
    node.synthetic = order[id].second;
    node.q = n.quadrature_points;
    node.reals.assign(n.reals, n.reals + n.n_reals);
    std::vector<uint32_t> row;
    row.push_back(static_cast<uint32_t>(n.n_params));
    for (int i = 0; i < n.n_params; ++i) {
      int slot = reg.register_parameter(pg.vars, n.params[i]);
      node.params.push_back(slot);
      row.push_back(static_cast<uint32_t>(slot));
    }
    row.push_back(static_cast<uint32_t>(n.n_obs));
    for (int i = 0; i < n.n_obs; ++i) {
      reg.register_observable(pg.vars, n.obs[i]);
      int col = column_of(n.obs[i], node.synthetic);
      node.obs_vars.push_back(n.obs[i]);
      node.obs_cols.push_back(col);
      row.push_back(static_cast<uint32_t>(col));
    }
    pg.table.push_back(std::move(row));
  }
  // children ids: walk the same pre-order with a cursor
  {
    size_t cursor = 0;
    std::function<int(int)> link = [&](int parent) -> int {
      int id = static_cast<int>(cursor++);
      pg.nodes[id].parent = parent;
      const pf_node& n = g.nodes[pg.nodes[id].desc_index];
      for (int i = 0; i < n.n_children; ++i) pg.nodes[id].children.push_back(link(id));
      return id;
    };
    link(-1);
  }
  pg.n_columns = next_column;
  pg.param_vars = reg.params;
  // IndexTableBuilder::finish validation (index_table.hpp:69-84) holds by construction

  // column ranges (synthetic columns take their observable's range)
  pg.col_lower.assign(pg.n_columns, 0.0);
  pg.col_upper.assign(pg.n_columns, 0.0);
  for (auto& [v, c] : columns) {
    pg.col_lower[c] = pg.vars[v].lower;
    pg.col_upper[c] = pg.vars[v].upper;
  }

  // resolve_box (pdf.hpp:562-607)
  std::function<void(int)> resolve = [&](int id) {
    Node& node = pg.nodes[id];
    node.box.clear();
    switch (node.kind) {
      case PF_COMPOSITE: {
        resolve(node.children[0]);
        if (pg.nodes[node.children[0]].box.size() != 1)
          throw Error("arity-mismatch", node.name + ": composite outer must be one-dimensional");
        resolve(node.children[1]);
        node.box = pg.nodes[node.children[1]].box;
        break;
      }
      case PF_CONVOLUTION: {
        resolve(node.children[0]);
        resolve(node.children[1]);
        const auto& mb = pg.nodes[node.children[0]].box;
        const auto& rb = pg.nodes[node.children[1]].box;
        if (mb.size() != 1 || rb.size() != 1 || mb[0].var != rb[0].var)
          throw Error("dimensionality-mismatch",
                      node.name + ": convolution children must share one observable");
        node.box = mb;
        break;
      }
      default: {
        if (node.children.empty()) {
          for (size_t i = 0; i < node.obs_vars.size(); ++i)
            node.box.push_back({node.obs_vars[i], columns.at(node.obs_vars[i])});
        } else {
          for (int c : node.children) {
            resolve(c);
            for (const auto& e : pg.nodes[c].box) {
              bool seen = false;
              for (const auto& have : node.box)
                if (have.var == e.var) {
                  seen = true;
                  break;
                }
              if (!seen) node.box.push_back(e);
            }
          }
          if (node.kind == PF_MAPPED && node.box.size() != 1)
            throw Error("dimensionality-mismatch",
                        node.name + ": mapped targets must share one observable");
        }
        break;
      }
    }
  };
  // the reference resolves every collected node; resolving the root covers all
  resolve(0);
  for (size_t id = 0; id < pg.nodes.size(); ++id)
    if (pg.nodes[id].box.empty() && !pg.nodes[id].children.empty()) resolve(static_cast<int>(id));

  // normalised set: the root and every child of an AddPdf (pdf.hpp:107-132)
  pg.nodes[0].normalised = true;
  for (auto& node : pg.nodes)
    if (node.kind == PF_SUM)
      for (int c : node.children) pg.nodes[c].normalised = true;
  // An AddPdf whose children are all normalised over its own box needs no
  // grid of its own: midpoint_sum (pdf.hpp:148-176) is linear and AddPdf::raw
  // (pdf.hpp:368-379) is sum_i c_i raw_i / norm_i, so its coarse and fine sums
  // are the children's sums weighted by c_i / norm_i (equal up to rounding,
  // ~1e-16 relative).  It completes in its children's level (no extra level).
  for (auto& node : pg.nodes) {
    if (node.kind != PF_SUM || !node.normalised) continue;
    bool same = true;
    for (int c : node.children) {
      const Node& ch = pg.nodes[c];
      same = same && ch.normalised && ch.box.size() == node.box.size();
      for (size_t d = 0; same && d < node.box.size(); ++d) same = ch.box[d].var == node.box[d].var;
    }
    node.folded = same;
  }
  // A ProdPdf whose children live on disjoint observables that make up its
  // box has a separable grid: its n- and 2n-point midpoint sums (pdf.hpp:
  // 148-176 over the product box, ProdPdf::raw pdf.hpp:339-344) are the
  // products of the children's own midpoint sums (equal up to rounding).
  // The children's 1-D sums become its tasks: 2 x 3n evaluations instead of
  // 5 n^2 for a 2-D product.
  for (auto& node : pg.nodes) {
    if (node.kind != PF_PRODUCT || !node.normalised || node.children.size() < 2) continue;
    std::set<int> seen;
    size_t dims = 0;
    bool ok = true;
    for (int c : node.children) {
      for (const auto& b : pg.nodes[c].box) ok = ok && seen.insert(b.var).second;
      dims += pg.nodes[c].box.size();
    }
    std::set<int> own;
    for (const auto& b : node.box) own.insert(b.var);
    node.folded = ok && dims == node.box.size() && seen == own;
  }
  // levels: 1 + max level of normalised strict descendants (folded: their max)
  std::function<int(int)> max_desc_level = [&](int id) -> int {
    int best = -1;
    for (int c : pg.nodes[id].children) {
      int sub = max_desc_level(c);
      if (pg.nodes[c].normalised) sub = std::max(sub, pg.nodes[c].level);
      best = std::max(best, sub);
    }
    const Node& nd = pg.nodes[id];
    if (nd.normalised) pg.nodes[id].level = nd.folded && nd.kind == PF_SUM ? std::max(best, 0) : best + 1;
    return best;
  };
  max_desc_level(0);
  pg.max_level = pg.nodes[0].level;
  return pg;
}

double subtree_cost(const Program& pg, int node) {
  const Node& n = pg.nodes[node];
  double c = 1.0;
  if (n.kind == PF_DALITZ) return 8.0 * static_cast<double>(n.params.size() / 4);  // per resonance
  if (n.kind == PF_TDDP) return 16.0 * static_cast<double>(n.params.size() / 4) + 8.0;  // two amplitudes + time
  if (n.kind == PF_CONVOLUTION) {
    // model values are hoisted per call; the resolution runs Q times
    return 1.0 + static_cast<double>(n.q) * subtree_cost(pg, n.children[1]);
  }
  if (n.kind == PF_MAPPED) {
    double m = 0;
    for (int ch : n.children) m = std::max(m, subtree_cost(pg, ch));
    return 1.0 + m;
  }
  for (int ch : n.children) c += subtree_cost(pg, ch);
  return c;
}

}  // namespace pfb
