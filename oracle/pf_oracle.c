/*
 * pf_oracle.c — TEST INFRASTRUCTURE ONLY: a plain-C restatement of the
 * reference's likelihood path, used as the checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg.  Never linked into
 * the product (paper_1311_1753_b200/libpfb200.so).
 *
 * Follows /root/reference/proj/include/parfit/ (cited per function):
 *   finalize         pdf.hpp:504-613, variable.hpp:65-135
 *   raw kernels      pdf.hpp:210-497 (+ ArgusPdf, which the reference lacks:
 *                    GooFit's upper-threshold form, parity unpinned)
 *   normalisation    pdf.hpp:111-188 (long double midpoint sums, Richardson)
 *   eval_metric      engine.hpp:165-218 (floor, chi2, penalty, non-finite)
 *   reduce           engine.hpp:57-87 (4096-term long double chunks + pairwise)
 * Pinned against the reference itself (oracle/_ref, tests/test_oracle.py) and
 * against the golden vectors in tests/golden/.
 * Compiled with -ffp-contract=off and no -march, like the reference build.
 */
#include <math.h>
#include <stdint.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pfb200.h"

#define PO_MAX 64
#define KLOGFLOOR 1e-300
#define KCHISQEPS 1e-9
#define KPENALTY 1e300
#define KREDUCECHUNK 4096

typedef struct {
  int kind;
  const char* name;
  int nch, ch[PO_MAX];
  int np, p[PO_MAX];       /* registry slots */
  int no, ovar[PO_MAX], ocol[PO_MAX];
  int nreal;
  double reals[PO_MAX];
  long q;
  int synthetic;
  int nbox, bvar[8], bcol[8];
  int needs_child_norms;   /* AddPdf */
  double norm, err;
  int norm_valid;
  uint64_t fingerprint;
  uint64_t clamp;
} onode;

typedef struct {
  pf_variable* vars;
  int nvars;
  onode* nodes;
  int nn;
  int param_var[PO_MAX * 8];
  int np;
  int ncols, ndata;
  int binned;
  uint64_t n;
  double* values; /* column-major, ndata (+2) columns */
  double total;
  unsigned grid;
  double* terms;
  uint64_t floor_count;
  /* error state of the current evaluation */
  int err_code;
  char err_msg[512];
} omodel;

static void fail(omodel* m, const char* code, const char* detail) {
  if (m->err_code) return;
  m->err_code = 1;
  snprintf(m->err_msg, sizeof m->err_msg, "%s: %s", code, detail);
}

/* ---- finalize (pdf.hpp:517-537) ------------------------------------------ */
typedef struct {
  int idx, synthetic;
} visit;

static int collect(const pf_graph* g, int idx, int synthetic, visit* out, int n) {
  out[n].idx = idx;
  out[n].synthetic = synthetic;
  ++n;
  const pf_node* nd = &g->nodes[idx];
  if (nd->kind == PF_COMPOSITE) {
    n = collect(g, nd->children[0], 1, out, n);
    n = collect(g, nd->children[1], synthetic, out, n);
  } else {
    for (int i = 0; i < nd->n_children; ++i) n = collect(g, nd->children[i], synthetic, out, n);
  }
  return n;
}

static int count_nodes(const pf_graph* g, int idx) {
  int c = 1;
  for (int i = 0; i < g->nodes[idx].n_children; ++i) c += count_nodes(g, g->nodes[idx].children[i]);
  return c;
}

static void resolve_box(omodel* m, int id, int* colmap);

/* pre-order ids: a node's children start right after it, each followed by
 * its own subtree; *cursor ends one past the subtree of `id` */
static int find_child_ids(omodel* m, const pf_graph* g, visit* order, int id, int* cursor) {
  const pf_node* nd = &g->nodes[order[id].idx];
  onode* o = &m->nodes[id];
  o->nch = nd->n_children;
  *cursor = id + 1;
  for (int i = 0; i < nd->n_children; ++i) {
    int cid = *cursor;
    o->ch[i] = cid;
    find_child_ids(m, g, order, cid, cursor);
  }
  return id;
}

static void box_add(onode* o, int var, int col) {
  for (int i = 0; i < o->nbox; ++i)
    if (o->bvar[i] == var) return;
  o->bvar[o->nbox] = var;
  o->bcol[o->nbox] = col;
  o->nbox++;
}

static void resolve_box(omodel* m, int id, int* colmap) { /* pdf.hpp:562-607 */
  onode* o = &m->nodes[id];
  o->nbox = 0;
  if (o->kind == PF_COMPOSITE) {
    resolve_box(m, o->ch[0], colmap);
    resolve_box(m, o->ch[1], colmap);
    onode* in = &m->nodes[o->ch[1]];
    for (int i = 0; i < in->nbox; ++i) box_add(o, in->bvar[i], in->bcol[i]);
  } else if (o->kind == PF_CONVOLUTION) {
    resolve_box(m, o->ch[0], colmap);
    resolve_box(m, o->ch[1], colmap);
    onode* md = &m->nodes[o->ch[0]];
    box_add(o, md->bvar[0], md->bcol[0]);
  } else if (o->nch == 0) {
    for (int i = 0; i < o->no; ++i) box_add(o, o->ovar[i], colmap[o->ovar[i]]);
  } else {
    for (int c = 0; c < o->nch; ++c) {
      resolve_box(m, o->ch[c], colmap);
      onode* cn = &m->nodes[o->ch[c]];
      for (int i = 0; i < cn->nbox; ++i) box_add(o, cn->bvar[i], cn->bcol[i]);
    }
  }
}

/* ---- raw kernels (pdf.hpp:210-497) --------------------------------------- */
static double raw(omodel* m, int id, double* evt, const double* p);
/* DalitzPlotPdf (no reference kernel; parity unpinned): the GPU's
 * pf_device.cuh pf_q2 / pf_dalitz_res / pf_dalitz_inside, same operation order
 * (this file is compiled with -ffp-contract=off; the GPU uses explicitly
 * rounded operations). */
static double po_q2(double s, double quarter, double ma, double mb) {
  const double sp = ma + mb, sm = ma - mb;
  const double v = ((s - sp * sp) * (s - sm * sm)) * quarter;
  return v > 0.0 ? v : 0.0;
}

static void po_dalitz_res(double s, double quarter, double rs, double Z, double m, double m2, double G, double iq0,
                          double br0, double mi, double mj, double R2, int spin, double* re, double* im) {
  const double q2 = po_q2(s, quarter, mi, mj);
  const double x = sqrt(q2) * iq0;
  double bf2 = 1.0, ratio = x, sbf = 1.0;
  if (spin == 1) {
    bf2 = br0 / (1.0 + R2 * q2);
    ratio = (x * x) * x;
    sbf = sqrt(bf2);
  }
  const double gs = ((G * ratio) * (m * rs)) * bf2;
  const double a = m2 - s, b = m * gs;
  const double den = a * a + b * b;
  const double f = (Z * sbf) / den;
  *re = f * a;
  *im = f * b;
}

static int po_dalitz_inside(double s12, double s13, double M, double m1, double m2, double m3) {
  const double a12 = m1 + m2, b12 = M - m3;
  if (!(s12 >= a12 * a12 && s12 <= b12 * b12)) return 0;
  const double r12 = sqrt(s12);
  const double e1 = ((s12 - m2 * m2) + m1 * m1) / (2.0 * r12);
  const double e3 = ((M * M - s12) - m3 * m3) / (2.0 * r12);
  const double t1 = e1 * e1 - m1 * m1, t3 = e3 * e3 - m3 * m3;
  const double p1 = sqrt(t1 > 0.0 ? t1 : 0.0), p3 = sqrt(t3 > 0.0 ? t3 : 0.0);
  const double e = e1 + e3, pp = p1 + p3, pm = p1 - p3;
  const double lo = e * e - pp * pp, hi = e * e - pm * pm;
  return s13 >= lo && s13 <= hi;
}

/* the isobar amplitude sum at (s12, s13, s23), the kinematic boundary aside */
static void po_dalitz_amp(const onode* o, int nres, double s12, double s13, double s23, const double* p,
                          double* are_out, double* aim_out) {
  const double M = o->reals[0], m1 = o->reals[1], m2 = o->reals[2], m3 = o->reals[3], R = o->reals[4];
  const double R2 = R * R;
  const double ms[4] = {M, m1, m2, m3};
  double are = 0.0, aim = 0.0;
  for (int r = 0; r < nres; ++r) {
    const int ch = (int)o->reals[5 + 2 * r], spin = (int)o->reals[6 + 2 * r];
    const int i = ch / 10, j = ch % 10, k = 6 - i - j;
    const double sij = ch == 12 ? s12 : ch == 13 ? s13 : s23;
    const double sik = ch == 12 ? s13 : s12;
    const double sjk = ch == 12 ? s23 : ch == 13 ? s23 : s13;
    const double qt = 0.25 / sij, rs = sqrt(4.0 * qt);  /* 1/(4 s), 1/sqrt(s) */
    double Z = 1.0;
    if (spin == 1) {
      const double a = M * M - ms[k] * ms[k];
      const double b = ms[i] * ms[i] - ms[j] * ms[j];
      Z = (sjk - sik) + (4.0 * (a * b)) * qt;
    }
    const double m = p[o->p[4 * r]], mm2 = m * m, G = p[o->p[4 * r + 1]];
    const double q20 = po_q2(mm2, 0.25 / mm2, ms[i], ms[j]);
    double bre, bim;
    po_dalitz_res(sij, qt, rs, Z, m, mm2, G, 1.0 / sqrt(q20), 1.0 + R2 * q20, ms[i], ms[j], R2, spin, &bre, &bim);
    const double cre = p[o->p[4 * r + 2]], cim = p[o->p[4 * r + 3]];
    are = are + (cre * bre - cim * bim);
    aim = aim + (cre * bim + cim * bre);
  }
  *are_out = are;
  *aim_out = aim;
}

static double po_dalitz_s23(const onode* o, double s12, double s13) {
  const double M = o->reals[0], m1 = o->reals[1], m2 = o->reals[2], m3 = o->reals[3];
  double msum = M * M;
  msum = msum + m1 * m1;
  msum = msum + m2 * m2;
  msum = msum + m3 * m3;
  return (msum - s12) - s13;
}

static double po_dalitz(const onode* o, const double* evt, const double* p) {
  const double s12 = evt[o->ocol[0]], s13 = evt[o->ocol[1]];
  if (!po_dalitz_inside(s12, s13, o->reals[0], o->reals[1], o->reals[2], o->reals[3])) return 0.0;
  double are, aim;
  po_dalitz_amp(o, o->np / 4, s12, s13, po_dalitz_s23(o, s12, s13), p, &are, &aim);
  return are * are + aim * aim;
}

/* TddpPdf (no reference kernel; GooFit's TDDP of PAPER.md:299-309 restated):
   |A g+(t) + Abar g-(t)|^2 with Abar(s12, s13) = A(s12, s23), T = t / tau:
   e^-T [(|A|^2+|Abar|^2)/2 cosh(yT) + (|A|^2-|Abar|^2)/2 cos(xT)
         - Re(A* Abar) sinh(yT) - Im(A* Abar) sin(xT)] */
static double po_tddp(const onode* o, const double* evt, const double* p) {
  const int nres = (o->np - 3) / 4;
  const double s12 = evt[o->ocol[0]], s13 = evt[o->ocol[1]], t = evt[o->ocol[2]];
  if (!po_dalitz_inside(s12, s13, o->reals[0], o->reals[1], o->reals[2], o->reals[3])) return 0.0;
  const double s23 = po_dalitz_s23(o, s12, s13);
  double are, aim, bre, bim;
  po_dalitz_amp(o, nres, s12, s13, s23, p, &are, &aim);
  po_dalitz_amp(o, nres, s12, s23, s13, p, &bre, &bim);
  const double tau = p[o->p[4 * nres]], x = p[o->p[4 * nres + 1]], y = p[o->p[4 * nres + 2]];
  const double T = t / tau;
  const double a2 = are * are + aim * aim, b2 = bre * bre + bim * bim;
  const double cre = are * bre + aim * bim, cim = are * bim - aim * bre;
  const double v = ((0.5 * (a2 + b2)) * cosh(y * T) + (0.5 * (a2 - b2)) * cos(x * T)) - cre * sinh(y * T) -
                   cim * sin(x * T);
  return exp(-T) * v;
}

static double density(omodel* m, int id, double* evt, const double* p) { /* pdf.hpp:83-91 */
  onode* o = &m->nodes[id];
  if (!o->norm_valid) {
    fail(m, "stale-normalization", o->name);
    return 0.0;
  }
  return raw(m, id, evt, p) / o->norm;
}

static double raw(omodel* m, int id, double* evt, const double* p) {
  onode* o = &m->nodes[id];
  switch (o->kind) {
    case PF_EXPONENTIAL: /* pdf.hpp:219-224 */
      return exp(p[o->p[0]] * evt[o->ocol[0]]);
    case PF_GAUSSIAN: { /* pdf.hpp:251-260 */
      double x = evt[o->ocol[0]], mean = p[o->p[0]], sigma = p[o->p[1]];
      if (!(sigma > 0)) {
        fail(m, "nonpositive-sigma", o->name);
        return 0.0;
      }
      return exp(-0.5 * (x - mean) * (x - mean) / (sigma * sigma));
    }
    case PF_BREIT_WIGNER: { /* pdf.hpp:280-288 */
      double x = evt[o->ocol[0]], mm = p[o->p[0]], g = p[o->p[1]];
      if (!(g > 0)) {
        fail(m, "nonpositive-width", o->name);
        return 0.0;
      }
      double d = x * x - mm * mm;
      return 1.0 / (d * d + mm * mm * g * g);
    }
    case PF_POLYNOMIAL: { /* pdf.hpp:307-318 */
      double x = evt[o->ocol[0]], acc = 0.0;
      for (int i = o->np; i-- > 0;) acc = acc * x + p[o->p[i]];
      if (acc < 0.0) {
        o->clamp++;
        return 0.0;
      }
      return acc;
    }
    case PF_DALITZ: {
      for (int r = 0; r < o->np / 4; ++r)
        if (!(p[o->p[4 * r + 1]] > 0.0)) {
          char buf[300];
          snprintf(buf, sizeof buf, "%s: width must be > 0", o->name);
          fail(m, "nonpositive-width", buf);
          return 0.0;
        }
      return po_dalitz(o, evt, p);
    }
    case PF_TDDP: {
      const int nres = (o->np - 3) / 4;
      for (int r = 0; r < nres; ++r)
        if (!(p[o->p[4 * r + 1]] > 0.0)) {
          char buf[300];
          snprintf(buf, sizeof buf, "%s: width must be > 0", o->name);
          fail(m, "nonpositive-width", buf);
          return 0.0;
        }
      if (!(p[o->p[4 * nres]] > 0.0)) {
        fail(m, "nonpositive-lifetime", o->name);
        return 0.0;
      }
      return po_tddp(o, evt, p);
    }
    case PF_ARGUS: { /* GooFit ArgusPdf, upper threshold; no reference kernel */
      double x = evt[o->ocol[0]];
      double t = x / p[o->p[0]];
      if (t >= 1.0) return 0.0;
      t = 1.0 - t * t;
      return x * pow(t, p[o->p[2]]) * exp(p[o->p[1]] * t);
    }
    case PF_PRODUCT: { /* pdf.hpp:339-344 */
      double acc = 1.0;
      for (int i = 0; i < o->nch; ++i) acc *= raw(m, o->ch[i], evt, p);
      return acc;
    }
    case PF_SUM: { /* pdf.hpp:368-379 */
      double fsum = 0.0, acc = 0.0;
      for (int i = 0; i < o->np; ++i) {
        double f = p[o->p[i]];
        fsum += f;
        acc += f * density(m, o->ch[i], evt, p);
      }
      acc += (1.0 - fsum) * density(m, o->ch[o->nch - 1], evt, p);
      return acc;
    }
    case PF_COMPOSITE: { /* pdf.hpp:406-415 */
      double g = raw(m, o->ch[1], evt, p);
      int col = m->nodes[o->ch[0]].bcol[0];
      double saved = evt[col];
      evt[col] = g;
      double v = raw(m, o->ch[0], evt, p);
      evt[col] = saved;
      return v;
    }
    case PF_MAPPED: { /* pdf.hpp:436-452 */
      double x = evt[o->bcol[0]];
      int nb = o->nreal;
      if (x < o->reals[0] || x > o->reals[nb - 1]) {
        char buf[300];
        snprintf(buf, sizeof buf, "%s: x outside mapped range", o->name);
        fail(m, "out-of-domain", buf);
        return 0.0;
      }
      int r;
      if (x == o->reals[nb - 1]) {
        r = o->nch - 1;
      } else {
        int lo = 0, hi = nb - 1;
        while (hi - lo > 1) {
          int mid = (lo + hi) / 2;
          if (x < o->reals[mid]) hi = mid;
          else lo = mid;
        }
        r = lo;
      }
      return raw(m, o->ch[r], evt, p);
    }
    case PF_CONVOLUTION: { /* pdf.hpp:476-493 */
      const pf_variable* dim = &m->vars[o->bvar[0]];
      int col = o->bcol[0];
      double x = evt[col];
      double h = (dim->upper - dim->lower) / (double)o->q;
      double sum = 0.0;
      for (long j = 0; j < o->q; ++j) {
        double tau = dim->lower + ((double)j + 0.5) * h;
        evt[col] = tau;
        double mv = raw(m, o->ch[0], evt, p);
        evt[col] = x - tau;
        double r = raw(m, o->ch[1], evt, p);
        sum += mv * r;
      }
      evt[col] = x;
      return sum * h;
    }
  }
  return 0.0;
}

/* ---- normalisation (pdf.hpp:111-188) ------------------------------------- */
static uint64_t hash_params(const double* p, int n) { /* pdf.hpp:40-51 */
  uint64_t h = 14695981039346656037ull;
  for (int k = 0; k < n; ++k) {
    uint64_t bits;
    memcpy(&bits, &p[k], sizeof bits);
    for (int i = 0; i < 8; ++i) {
      h ^= (bits >> (8 * i)) & 0xffu;
      h *= 1099511628211ull;
    }
  }
  return h;
}

/* TddpPdf: the 3-D midpoint sum over (s12, s13, t) evaluated by its
   separability, sum_ij sum_l D(s12_i, s13_j) . T(t_l) = sum_c D_c T_c (the
   four Dalitz bilinears times the four time functions, po_tddp), in long
   double like midpoint_sum.  Mathematically the same sum as the brute-force
   walk over n^3 points (checked against it at small n, tests/test_oracle.py),
   which at n = 1024 would take 10^10 evaluations. */
static double tddp_midpoint_sum(omodel* m, int id, const double* p, uint64_t n) {
  onode* o = &m->nodes[id];
  const int nres = (o->np - 3) / 4;
  int b12 = -1, b13 = -1, bt = -1;
  for (int d = 0; d < o->nbox; ++d) {
    if (o->bcol[d] == o->ocol[0]) b12 = d;
    if (o->bcol[d] == o->ocol[1]) b13 = d;
    if (o->bcol[d] == o->ocol[2]) bt = d;
  }
  const pf_variable *v12 = &m->vars[o->bvar[b12]], *v13 = &m->vars[o->bvar[b13]], *vt = &m->vars[o->bvar[bt]];
  const double h12 = (v12->upper - v12->lower) / (double)n, h13 = (v13->upper - v13->lower) / (double)n;
  const double ht = (vt->upper - vt->lower) / (double)n;
  for (int r = 0; r < nres; ++r)
    if (!(p[o->p[4 * r + 1]] > 0.0)) {
      fail(m, "nonpositive-width", o->name);
      return 0.0;
    }
  const double tau = p[o->p[4 * nres]], x = p[o->p[4 * nres + 1]], y = p[o->p[4 * nres + 2]];
  if (!(tau > 0.0)) {
    fail(m, "nonpositive-lifetime", o->name);
    return 0.0;
  }
  long double D[4] = {0.0L, 0.0L, 0.0L, 0.0L}, T[4] = {0.0L, 0.0L, 0.0L, 0.0L};
  for (uint64_t i = 0; i < n; ++i) {
    const double s12 = v12->lower + ((double)i + 0.5) * h12;
    for (uint64_t j = 0; j < n; ++j) {
      const double s13 = v13->lower + ((double)j + 0.5) * h13;
      if (!po_dalitz_inside(s12, s13, o->reals[0], o->reals[1], o->reals[2], o->reals[3])) continue;
      const double s23 = po_dalitz_s23(o, s12, s13);
      double are, aim, bre, bim;
      po_dalitz_amp(o, nres, s12, s13, s23, p, &are, &aim);
      po_dalitz_amp(o, nres, s12, s23, s13, p, &bre, &bim);
      const double a2 = are * are + aim * aim, b2 = bre * bre + bim * bim;
      D[0] += 0.5 * (a2 + b2);
      D[1] += 0.5 * (a2 - b2);
      D[2] += are * bre + aim * bim;
      D[3] += are * bim - aim * bre;
    }
  }
  for (uint64_t l = 0; l < n; ++l) {
    const double t = vt->lower + ((double)l + 0.5) * ht;
    const double Tt = t / tau, e = exp(-Tt);
    T[0] += e * cosh(y * Tt);
    T[1] += e * cos(x * Tt);
    T[2] -= e * sinh(y * Tt);
    T[3] -= e * sin(x * Tt);
  }
  long double sum = 0.0L;
  for (int c = 0; c < 4; ++c) sum += D[c] * T[c];
  return (double)sum * ((h12 * h13) * ht);
}

static double midpoint_sum(omodel* m, int id, const double* p, uint64_t n) {
  onode* o = &m->nodes[id];
  if (o->kind == PF_TDDP && !getenv("PO_TDDP_BRUTE")) return tddp_midpoint_sum(m, id, p, n);
  int dims = o->nbox;
  double lo[8], h[8];
  uint64_t total = 1;
  if (dims == 0) {
    fail(m, "no-observables", o->name);
    return 0.0;
  }
  for (int d = 0; d < dims; ++d) {
    const pf_variable* v = &m->vars[o->bvar[d]];
    lo[d] = v->lower;
    h[d] = (v->upper - v->lower) / (double)n;
    total *= n;
  }
  double* evt = calloc((size_t)m->ncols + 1, sizeof(double));
  long double sum = 0.0L;
  for (uint64_t flat = 0; flat < total && !m->err_code; ++flat) {
    uint64_t rem = flat;
    for (int d = dims; d-- > 0;) {
      uint64_t k = rem % n;
      rem /= n;
      evt[o->bcol[d]] = lo[d] + ((double)k + 0.5) * h[d];
    }
    sum += raw(m, id, evt, p);
  }
  free(evt);
  double vol = 1.0;
  for (int d = 0; d < dims; ++d) vol *= h[d];
  return (double)sum * vol;
}

static void compute_normalization(omodel* m, int id, const double* p) {
  onode* o = &m->nodes[id];
  double coarse = midpoint_sum(m, id, p, m->grid);
  if (m->err_code) return;
  double fine = midpoint_sum(m, id, p, 2ull * m->grid);
  if (m->err_code) return;
  o->norm = fine + (fine - coarse) / 3.0;
  o->err = fabs(fine - coarse) / 3.0;
  if (!(o->norm > 0.0) || !isfinite(o->norm)) {
    char buf[300];
    snprintf(buf, sizeof buf, "degenerate PDF '%s'", o->name);
    fail(m, "zero-integral", buf);
  }
}

static void refresh(omodel* m, int id, const double* p);

static void propagate(omodel* m, int id, const double* p) {
  onode* o = &m->nodes[id];
  for (int i = 0; i < o->nch && !m->err_code; ++i) {
    if (o->needs_child_norms) refresh(m, o->ch[i], p);
    else propagate(m, o->ch[i], p);
  }
}

static void refresh(omodel* m, int id, const double* p) {
  onode* o = &m->nodes[id];
  propagate(m, id, p);
  if (m->err_code) return;
  uint64_t fp = hash_params(p, m->np);
  if (o->norm_valid && o->fingerprint == fp) return;
  compute_normalization(m, id, p);
  if (m->err_code) return;
  o->fingerprint = fp;
  o->norm_valid = 1;
}

static int params_valid(omodel* m, const double* p) { /* pdf.hpp:96-100, 381-390 */
  for (int id = 0; id < m->nn; ++id) {
    onode* o = &m->nodes[id];
    if (o->kind != PF_SUM) continue;
    double fsum = 0.0;
    for (int i = 0; i < o->np; ++i) {
      double f = p[o->p[i]];
      if (f < 0.0 || f > 1.0) return 0;
      fsum += f;
    }
    if (fsum > 1.0) return 0;
  }
  return 1;
}

/* ---- reduce (engine.hpp:57-87) ------------------------------------------- */
static long double pairwise(const long double* v, size_t n) {
  if (n == 0) return 0.0L;
  if (n == 1) return v[0];
  size_t half = n / 2;
  return pairwise(v, half) + pairwise(v + half, n - half);
}

double po_reduce(const double* t, size_t n) {
  if (n == 0) return 0.0;
  size_t nc = (n + KREDUCECHUNK - 1) / KREDUCECHUNK;
  long double* parts = malloc(nc * sizeof(long double));
  for (size_t c = 0; c < nc; ++c) {
    size_t lo = c * KREDUCECHUNK, hi = lo + KREDUCECHUNK < n ? lo + KREDUCECHUNK : n;
    long double s = 0.0L;
    for (size_t i = lo; i < hi; ++i) s += t[i];
    parts[c] = s;
  }
  double r = (double)pairwise(parts, nc);
  free(parts);
  return r;
}

/* ---- public entry points ------------------------------------------------- */
void* po_create(const pf_graph* g, const pf_data* d, uint32_t grid, char* err) {
  omodel* m = calloc(1, sizeof(omodel));
  m->grid = grid;
  m->nvars = g->n_variables;
  m->vars = malloc(sizeof(pf_variable) * (g->n_variables + 1));
  memcpy(m->vars, g->variables, sizeof(pf_variable) * g->n_variables);
  int total = count_nodes(g, g->root);
  visit* order = malloc(sizeof(visit) * total);
  collect(g, g->root, 0, order, 0);
  m->nn = total;
  m->nodes = calloc(total, sizeof(onode));
  int* colmap = malloc(sizeof(int) * (g->n_variables + 1));
  for (int i = 0; i < g->n_variables; ++i) colmap[i] = -1;
  for (int c = 0; c < d->n_obs; ++c) colmap[d->obs[c]] = c;
  m->ndata = d->n_obs;
  m->binned = d->binned;
  int next_col = d->n_obs + (d->binned ? 2 : 0);
  /* registry (variable.hpp:121-135): first appearance wins the next slot */
  int* slot_of = malloc(sizeof(int) * (g->n_variables + 1));
  for (int i = 0; i < g->n_variables; ++i) slot_of[i] = -1;
  for (int id = 0; id < total; ++id) {
    const pf_node* nd = &g->nodes[order[id].idx];
    onode* o = &m->nodes[id];
    o->kind = nd->kind;
    o->name = nd->name;
    o->synthetic = order[id].synthetic;
    o->q = (long)nd->quadrature_points;
    o->nreal = nd->n_reals;
    for (int i = 0; i < nd->n_reals; ++i) o->reals[i] = nd->reals[i];
    o->needs_child_norms = nd->kind == PF_SUM;
    o->np = nd->n_params;
    for (int i = 0; i < nd->n_params; ++i) {
      int v = nd->params[i];
      if (slot_of[v] < 0) {
        slot_of[v] = m->np;
        m->param_var[m->np++] = v;
      }
      o->p[i] = slot_of[v];
    }
    o->no = nd->n_obs;
    for (int i = 0; i < nd->n_obs; ++i) {
      int v = nd->obs[i];
      if (colmap[v] < 0) {
        if (!o->synthetic) {
          char buf[300];
          snprintf(buf, sizeof buf, "unbound-observable: '%s' is not in the bound data set",
                   g->variables[v].name);
          if (err) snprintf(err, 512, "%s", buf);
          free(order);
          free(colmap);
          free(slot_of);
          free(m->nodes);
          free(m->vars);
          free(m);
          return NULL;
        }
        colmap[v] = next_col++;
      }
      o->ovar[i] = v;
      o->ocol[i] = colmap[v];
    }
  }
  int cursor = 0;
  find_child_ids(m, g, order, 0, &cursor);
  m->ncols = next_col;
  resolve_box(m, 0, colmap);
  free(order);
  free(colmap);
  free(slot_of);
  m->n = d->n_events;
  int ncol_data = d->n_obs + (d->binned ? 2 : 0);
  m->values = malloc(sizeof(double) * (m->n * ncol_data + 1));
  memcpy(m->values, d->values, sizeof(double) * m->n * ncol_data);
  m->total = d->total_content;
  m->terms = malloc(sizeof(double) * (m->n + 1));
  return m;
}

void po_destroy(void* h) {
  omodel* m = h;
  if (!m) return;
  free(m->values);
  free(m->terms);
  free(m->nodes);
  free(m->vars);
  free(m);
}

int po_n_params(void* h) { return ((omodel*)h)->np; }
int po_param_variable(void* h, int slot) { return ((omodel*)h)->param_var[slot]; }
int po_n_nodes(void* h) { return ((omodel*)h)->nn; }
uint64_t po_floor_count(void* h) { return ((omodel*)h)->floor_count; }
uint64_t po_clamp_count(void* h, int node) { return ((omodel*)h)->nodes[node].clamp; }

void po_norms(void* h, double* norms, double* errs, int* valid, int n) {
  omodel* m = h;
  for (int i = 0; i < n && i < m->nn; ++i) {
    norms[i] = m->nodes[i].norm;
    errs[i] = m->nodes[i].err;
    valid[i] = m->nodes[i].norm_valid;
  }
}

/* The event loop of eval_metric (engine.hpp:184-209) over events [lo, hi) on
   a private copy of the model state: raw() bumps clamp counters and records
   errors in the model, so every worker thread owns a copy of the node array
   and error slot; terms go to disjoint slots of the shared terms array.  The
   reduce stays serial and in the reference's fixed order, so the result does
   not depend on the thread count. */
typedef struct {
  omodel mc;             /* private copy (nodes copied too) */
  const double* p;
  int metric;
  double norm;
  uint64_t lo, hi;
  uint64_t floors;
  uint64_t err_event;    /* first erroring event, or UINT64_MAX */
} po_work;

static void* po_event_range(void* arg) {
  po_work* w = arg;
  omodel* m = &w->mc;
  double* evt = calloc((size_t)m->ncols + 1, sizeof(double));
  const int nc = m->ndata + (m->binned ? 2 : 0);
  w->floors = 0;
  w->err_event = UINT64_MAX;
  for (uint64_t e = w->lo; e < w->hi; ++e) {
    for (int c = 0; c < nc; ++c) evt[c] = m->values[(uint64_t)c * m->n + e];
    if (w->metric == PF_NLL) {
      double v = raw(m, 0, evt, w->p) / w->norm;
      if (v < KLOGFLOOR) {
        v = KLOGFLOOR;
        w->floors++;
      }
      m->terms[e] = -log(v);
    } else {
      double content = evt[m->ndata], volume = evt[m->ndata + 1];
      double mu = m->total * (raw(m, 0, evt, w->p) / w->norm) * volume;
      double diff = content - mu;
      m->terms[e] = diff * diff / (mu > KCHISQEPS ? mu : KCHISQEPS);
    }
    if (m->err_code) {
      w->err_event = e;
      break;
    }
  }
  free(evt);
  return NULL;
}

/* BoundModel::eval_metric (engine.hpp:165-218); threads > 1 splits the event
   loop over that many POSIX threads (the reference's Backend::with_threads,
   engine.hpp:98-130), bit-identical to threads = 1 */
int po_eval_mt(void* h, const double* p, size_t n, int metric, int threads, double* out, char* err) {
  omodel* m = h;
  m->err_code = 0;
  m->err_msg[0] = 0;
  if (n != (size_t)m->np) {
    snprintf(err, 512, "size-mismatch: eval_metric: parameter vector length");
    return 1;
  }
  if (m->binned && metric == PF_NLL) {
    snprintf(err, 512, "metric-mismatch: NLL needs an unbinned data set");
    return 1;
  }
  if (!m->binned && metric == PF_CHISQ) {
    snprintf(err, 512, "metric-mismatch: chi-squared needs a binned data set");
    return 1;
  }
  if (!params_valid(m, p)) {
    *out = KPENALTY;
    return 0;
  }
  refresh(m, 0, p);
  if (m->err_code) { /* degenerate normalisation: penalty (engine.hpp:174-178) */
    m->err_code = 0;
    *out = KPENALTY;
    return 0;
  }
  if (threads < 1) threads = 1;
  if ((uint64_t)threads > m->n / 4096 + 1) threads = (int)(m->n / 4096 + 1);
  po_work* w = calloc((size_t)threads, sizeof(po_work));
  pthread_t* tid = calloc((size_t)threads, sizeof(pthread_t));
  for (int t = 0; t < threads; ++t) {
    w[t].mc = *m;
    w[t].mc.nodes = malloc(sizeof(onode) * (size_t)m->nn);
    memcpy(w[t].mc.nodes, m->nodes, sizeof(onode) * (size_t)m->nn);
    w[t].p = p;
    w[t].metric = metric;
    w[t].norm = m->nodes[0].norm;
    w[t].lo = m->n * (uint64_t)t / (uint64_t)threads;
    w[t].hi = m->n * (uint64_t)(t + 1) / (uint64_t)threads;
    if (threads > 1) pthread_create(&tid[t], NULL, po_event_range, &w[t]);
  }
  if (threads == 1) po_event_range(&w[0]);
  else
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
  int rc = 0;
  for (int t = 0; t < threads; ++t) {
    m->floor_count += w[t].floors;
  }
  /* clamp counters: every copy started from the model's value */
  for (int i = 0; i < m->nn; ++i) {
    uint64_t tot = 0;
    for (int t = 0; t < threads; ++t) tot += w[t].mc.nodes[i].clamp;
    m->nodes[i].clamp = tot - (uint64_t)(threads - 1) * m->nodes[i].clamp;
  }
  for (int t = 0; t < threads && !rc; ++t)
    if (w[t].err_event != UINT64_MAX) { /* the first error in event order */
      snprintf(err, 512, "%s", w[t].mc.err_msg);
      rc = 1;
    }
  for (int t = 0; t < threads; ++t) free(w[t].mc.nodes);
  free(w);
  free(tid);
  if (rc) return 1;
  double r = po_reduce(m->terms, m->n);
  if (!isfinite(r)) {
    for (uint64_t e = 0; e < m->n; ++e)
      if (!isfinite(m->terms[e])) {
        snprintf(err, 512, "non-finite-metric: first offending event index %llu", (unsigned long long)e);
        return 1;
      }
    snprintf(err, 512, "non-finite-metric: non-finite reduction");
    return 1;
  }
  *out = r;
  return 0;
}

int po_eval(void* h, const double* p, size_t n, int metric, double* out, char* err) {
  return po_eval_mt(h, p, n, metric, 1, out, err);
}

/* raw/density of the root at explicit points (column-major, ncols_data) */
int po_density(void* h, const double* p, const double* pts, uint64_t npts, double* out, char* err) {
  omodel* m = h;
  m->err_code = 0;
  refresh(m, 0, p);
  if (m->err_code) {
    snprintf(err, 512, "%s", m->err_msg);
    return 1;
  }
  double* evt = calloc((size_t)m->ncols + 1, sizeof(double));
  for (uint64_t e = 0; e < npts; ++e) {
    for (int c = 0; c < m->ndata; ++c) evt[c] = pts[(uint64_t)c * npts + e];
    out[e] = raw(m, 0, evt, p) / m->nodes[0].norm;
  }
  free(evt);
  return 0;
}

/* ---- std::mt19937_64 (Matsumoto & Nishimura 2004 parameters) -------------
 * ToyRng's bit recipe (generate.hpp:19-27): u = (g() >> 11) * 2^-53.  Used
 * only to regenerate the reference tests' seeded inputs (e.g. the
 * acceptance.cpp:313-318 golden data set). */
typedef struct {
  uint64_t mt[312];
  int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ull) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFull);
      uint64_t xa = x >> 1;
      if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

/* n uniforms in [0, 1) from mt19937_64(seed) */
void po_mt64_uniform(uint64_t seed, uint64_t n, double* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (uint64_t i = 0; i < n; ++i) out[i] = (double)(mt64_next(&g) >> 11) * 0x1.0p-53;
}

/* Test support for the GPU's ArgusPdf log form (codegen.cpp emit_logterm):
 * y / m0 there is Markstein's FMA sequence on the correctly rounded
 * reciprocal, q = y * inv, r = fma(-q, m0, y), q' = fma(r, inv, q).  Counts
 * the operand pairs (y in [lo, hi), m0 in [mlo, mhi), uniform from a
 * splitmix64 stream) where q' differs from the IEEE quotient y / m0. */
static uint64_t po_splitmix(uint64_t* s) {
  uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

int64_t po_markstein_mismatches(uint64_t n, uint64_t seed, double lo, double hi, double mlo, double mhi) {
  int64_t bad = 0;
  uint64_t s = seed;
  for (uint64_t i = 0; i < n; ++i) {
    const double u = (double)(po_splitmix(&s) >> 11) * 0x1.0p-53;
    const double v = (double)(po_splitmix(&s) >> 11) * 0x1.0p-53;
    const double y = lo + (hi - lo) * u, m0 = mlo + (mhi - mlo) * v;
    const double inv = 1.0 / m0;
    const double q = y * inv;
    const double r = fma(fma(-q, m0, y), inv, q);
    if (r != y / m0) ++bad;
  }
  return bad;
}
