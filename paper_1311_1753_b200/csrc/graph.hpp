// graph.hpp — finalized PDF graph ("program") built from a pf_graph.
//
// Restates the reference's GraphFinalizer (pdf.hpp:504-613), the parameter
// registry (variable.hpp:65-121) and the IndexTable (index_table.hpp:12-99):
// pre-order node ids, registry order = parameter-vector layout, observable
// columns (data, then reserved binned columns, then synthetic Composite
// columns) and each node's integration box.  The result is the single
// description from which codegen.cpp emits the fused device evaluator.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pfb200.h"

namespace pfb {

// parfit::Error equivalent: message "code: detail" (errors.hpp:11-16)
class Error : public std::runtime_error {
 public:
  Error(const std::string& code, const std::string& detail)
      : std::runtime_error(code + ": " + detail), code_(code) {}
  const std::string& code() const { return code_; }

 private:
  std::string code_;
};

struct Var {
  std::string name;
  double value = 0, lower = 0, upper = 0, step = 0;
  bool fixed = false;
  int role = PF_OBSERVABLE;
};

struct BoxDim {
  int var;     // variable index
  int column;  // resolved event column
};

struct Node {
  int kind = 0;
  std::string name;
  int desc_index = -1;          // index in pf_graph.nodes
  bool synthetic = false;       // below a Composite outer (pdf.hpp:540-549)
  std::vector<int> children;    // node ids (pre-order)
  std::vector<int> params;      // registry slots, node-local order
  std::vector<int> obs_vars;    // variable indices
  std::vector<int> obs_cols;    // event columns
  std::vector<double> reals;    // MappedPdf boundaries
  int64_t q = 0;                // ConvolutionPdf quadrature points
  std::vector<BoxDim> box;      // resolve_box (pdf.hpp:562-607)
  bool normalised = false;      // root or child of an AddPdf (pdf.hpp:107-132)
  int level = -1;               // normalisation level (0 = no normalised descendants)
  bool folded = false;          // AddPdf normalised from its children's grid sums (no grid)
  int parent = -1;
};

struct Program {
  std::vector<Var> vars;
  std::vector<Node> nodes;                       // pre-order
  std::vector<int> param_vars;                   // registry slot -> var index
  std::vector<std::vector<uint32_t>> table;      // IndexTable rows
  int n_data_obs = 0;
  int reserved = 0;
  int n_columns = 0;
  std::vector<int> data_obs;                     // var index per data column
  std::vector<double> col_lower, col_upper;      // per column (reserved: 0)
  int max_level = 0;
};

// Validates constructor contracts (pdf.hpp:210-497) and finalizes.
Program finalize(const pf_graph& g, int n_data_obs, const int32_t* data_obs, int reserved);

// Subtree cost per event in "raw evaluations" (ConvolutionPdf multiplies by Q).
double subtree_cost(const Program& pg, int node);

// True when `node`'s subtree evaluation depends on the norms of `other`.
const char* kind_name(int kind);

}  // namespace pfb
