// codegen.hpp — emits the fused per-model CUDA evaluator (NVRTC source).
//
// The reference evaluates a virtual PdfNode::raw tree per event through the
// IndexTable's double indirection (pdf.hpp:79-80, 140-145).  Here the tree
// is flattened at model creation into straight-line device code: parameter
// slots and event columns become compile-time constants, so the only
// per-event work is the arithmetic itself.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "graph.hpp"

namespace pfb {

struct ConvTable {
  int node;       // ConvolutionPdf node id
  int slot;       // S offset of the Q model values
  int q;
  int after;      // stage after which it can be filled (-1 = pre)
};

constexpr int kConvKB = 128;  // products per chain per block of the warp-shared window sum

struct Layout {
  int n_nodes = 0;
  int np = 0;                 // parameters
  int ss = 0;                 // per-call state doubles per parameter set
  int nc = 0;                 // model constant doubles
  int nc_total_slot = -1;     // C index of N_tot (binned)
  bool binned = false;
  int ept = 8;                // events per lane per sub-chunk (32 * ept events)
  int nsub = 2;               // sub-chunks per chunk (chunk = nsub * 32 * ept events)
  int setup_cluster = 1;      // CTAs of a setup cluster: the setup kernel's and the fused pass's (same split: batched == sequential bitwise; 4 measured 41 -> 64 us for C2: 4-CTA clusters of 1-CTA/SM kernels do not all fit at once)
  int nst = 3;                // TMA stages per event warp (PF_NST)
  int setup_maxq = 8;         // most midpoint sums in one level (PF_SETUP_MAXQ)
  int lacc_n = 2;             // doubles of the per-lane chunk accumulator (PF_LACC_N)
  int unroll = 8;             // events interleaved per lane in the event loop (PF_UNROLL)
  int data_range_base = -1;   // C slots: (min, max) per data column, filled at bind time
  std::vector<int> load_cols; // data columns read per event
  std::vector<int> poly_index; // node -> clamp counter index (-1 otherwise)
  int n_poly = 0;
  std::vector<double> constants;  // C buffer contents (boundaries, conv L/h)
  std::vector<ConvTable> conv_tables;
  // convolutions with a Gaussian resolution: their normalisation grid is
  // evaluated per grid point (window + term recurrence), not per (point, tau) pair
  std::vector<int> conv_windowed;
  // the root is such a convolution: the event pass gives each warp a
  // shared-memory scratch of 2 x kConvKB products (PF_CONV_SHARED)
  bool conv_shared = false;
  // TddpPdf grids: doubles per column of the norm kernel's column table
  // (qt and the channel-A lineshapes, PF_TDDP_TAB_ARRAYS); 0: none
  int tddp_tab_arrays = 0;
  std::vector<std::vector<int>> level_nodes;  // normalised nodes per level
  std::string source;         // generated CUDA source (without library headers)
  std::string structure_key;  // cache key of the compiled module
};

// binned: chi-squared evaluator (content/volume columns after the obs).
// n_events (0: unknown) lets small data sets use short chunks, so that the
// event pass spreads over every SM.
Layout generate(const Program& pg, bool binned, uint64_t n_events = 0);

// Embedded library headers (pf_device.cuh, pf_kernels.cuh).
const char* device_header_source();
const char* kernels_header_source();
const char* counters_header_source();
const char* exp_table_header_source();
const char* generate_header_source();

}  // namespace pfb
