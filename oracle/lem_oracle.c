/*
 * lem_oracle.c -- CPU restatement of the reference D8 timestep.
 *
 * TEST INFRASTRUCTURE ONLY: this is the parity checker for the B200 path.
 * It is never linked into, loaded by, or called from the product library.
 * Compile with -O2 -ffp-contract=off (the reference's own flags,
 * CMakeLists.txt:14) so that every expression rounds exactly as the
 * reference's does.
 *
 * Each function restates one reference function; citations are to the
 * reference tree's proj/ directory.
 */
#include "lem_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* include/lem/erosion.hpp:16-24 -- default SimParams. */
void lo_default_params(lo_params* p) {
  p->K = 2e-6;
  p->m_exp = 0.5;
  p->n_exp = 1.0;
  p->uplift_rate = 2e-3;
  p->dt = 1000.0;
  p->epsilon = 1e-6;
  p->dx = 1.0;
  p->dy = 1.0;
  p->max_newton_iters = 100;
}

/* include/lem/neighborhood.hpp:17-23 -- offset_length. */
double lo_offset_length(int dx, int dy, double sx, double sy) {
  const double ox = dx * sx;
  const double oy = dy * sy;
  if (dy == 0) return fabs(ox);
  if (dx == 0) return fabs(oy);
  return sqrt(ox * ox + oy * oy);
}

/* src/neighborhood.cpp:9-45 -- frozen D8 / D4 stencils. */
int lo_make_nbh(int connectivity, double dx, double dy, lo_nbh* n) {
  static const int d8x[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
  static const int d8y[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
  static const int d4x[4] = {0, -1, 1, 0};
  static const int d4y[4] = {-1, 0, 0, 1};
  memset(n, 0, sizeof(*n));
  if (connectivity != 4 && connectivity != 8) return LO_ECONFIG;
  n->connectivity = connectivity;
  n->dx = dx;
  n->dy = dy;
  for (int i = 0; i < connectivity; ++i) {
    n->ox[i] = connectivity == 8 ? d8x[i] : d4x[i];
    n->oy[i] = connectivity == 8 ? d8y[i] : d4y[i];
    n->dist[i] = lo_offset_length(n->ox[i], n->oy[i], dx, dy);
  }
  return LO_OK;
}

/* src/terrain.cpp:12-17 -- splitmix64. */
uint64_t lo_splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* src/terrain.cpp:19-31 -- generate_terrain. */
void lo_generate_terrain(uint32_t w, uint32_t h, uint64_t seed, double* out) {
  const size_t n = (size_t)w * h;
  for (size_t i = 0; i < n; ++i) {
    const uint64_t z = lo_splitmix64(seed + (uint64_t)i * 0x9E3779B97F4A7C15ull);
    out[i] = (double)(z >> 11) * 0x1.0p-53;
  }
}

uint64_t lo_fnv1a64(const void* data, size_t nbytes) {
  const unsigned char* p = (const unsigned char*)data;
  uint64_t h = 1469598103934665603ull;
  for (size_t i = 0; i < nbytes; ++i) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

static int is_perimeter(size_t c, int w, int h) {
  const int x = (int)(c % (size_t)w), y = (int)(c / (size_t)w);
  return x == 0 || x == w - 1 || y == 0 || y == h - 1;
}

/* include/lem/flow_graph.hpp:44-59 steepest_receiver, :74-80 compute_receivers,
 * with include/lem/grid_graph.hpp:37-47 for_each_neighbor (off-grid skipped). */
void lo_receivers(const double* elev, int w, int h, const lo_nbh* nbh, uint32_t* rec) {
  const size_t n = (size_t)w * h;
  for (size_t c = 0; c < n; ++c) {
    if (is_perimeter(c, w, h)) {
      rec[c] = LO_NOFLOW;
      continue;
    }
    const int x = (int)(c % (size_t)w), y = (int)(c / (size_t)w);
    double s_max = 0.0;
    uint32_t n_max = LO_NOFLOW;
    const double ec = elev[c];
    for (int i = 0; i < nbh->connectivity; ++i) {
      const int nx = x + nbh->ox[i], ny = y + nbh->oy[i];
      if (nx < 0 || nx >= w || ny < 0 || ny >= h) continue;
      const uint32_t nb = (uint32_t)ny * (uint32_t)w + (uint32_t)nx;
      const double s = (ec - elev[nb]) / nbh->dist[i];
      if (s > s_max) {
        s_max = s;
        n_max = nb;
      }
    }
    rec[c] = n_max;
  }
}

/* include/lem/flow_graph.hpp:64-72 donors_of, :82-90 compute_donors. */
void lo_donors(const uint32_t* rec, int w, int h, const lo_nbh* nbh, uint32_t* donor,
               uint8_t* dnum) {
  const size_t n = (size_t)w * h;
  const int dmax = nbh->connectivity;
  for (size_t c = 0; c < n; ++c) {
    const int x = (int)(c % (size_t)w), y = (int)(c / (size_t)w);
    uint8_t k = 0;
    for (int i = 0; i < nbh->connectivity; ++i) {
      const int nx = x + nbh->ox[i], ny = y + nbh->oy[i];
      if (nx < 0 || nx >= w || ny < 0 || ny >= h) continue;
      const uint32_t nb = (uint32_t)ny * (uint32_t)w + (uint32_t)nx;
      if (rec[nb] == (uint32_t)c) donor[(size_t)dmax * c + k++] = nb;
    }
    for (int i = k; i < dmax; ++i) donor[(size_t)dmax * c + i] = LO_NOFLOW;
    dnum[c] = k;
  }
}

/* Same kernels over tests/fixtures.hpp ExplicitGraph (CSR adjacency). */
void lo_receivers_explicit(size_t n, const uint32_t* adj_off, const uint32_t* adj_nbr,
                           const double* adj_dist, const uint8_t* boundary,
                           const double* elev, uint32_t* rec) {
  for (size_t c = 0; c < n; ++c) {
    if (boundary[c]) {
      rec[c] = LO_NOFLOW;
      continue;
    }
    double s_max = 0.0;
    uint32_t n_max = LO_NOFLOW;
    for (uint32_t j = adj_off[c]; j < adj_off[c + 1]; ++j) {
      const double s = (elev[c] - elev[adj_nbr[j]]) / adj_dist[j];
      if (s > s_max) {
        s_max = s;
        n_max = adj_nbr[j];
      }
    }
    rec[c] = n_max;
  }
}

void lo_donors_explicit(size_t n, int dmax, const uint32_t* adj_off, const uint32_t* adj_nbr,
                        const uint32_t* rec, uint32_t* donor, uint8_t* dnum) {
  for (size_t c = 0; c < n; ++c) {
    uint8_t k = 0;
    for (uint32_t j = adj_off[c]; j < adj_off[c + 1]; ++j)
      if (rec[adj_nbr[j]] == (uint32_t)c) donor[(size_t)dmax * c + k++] = adj_nbr[j];
    for (int i = k; i < dmax; ++i) donor[(size_t)dmax * c + i] = LO_NOFLOW;
    dnum[c] = k;
  }
}

/* src/traversal.cpp:19-48 -- generate_queue (BFS level sets). */
int lo_generate_queue(size_t n, const uint32_t* rec, const uint32_t* donor,
                      const uint8_t* dnum, int dmax, uint32_t* order, uint32_t* levels,
                      uint32_t* nlevels) {
  size_t sz = 0;
  uint32_t nl = 0;
  levels[0] = 0;
  for (size_t c = 0; c < n; ++c)
    if (rec[c] == LO_NOFLOW) order[sz++] = (uint32_t)c;
  levels[++nl] = (uint32_t)sz;
  size_t lo = 0, hi = sz;
  while (lo < hi) {
    for (size_t i = lo; i < hi; ++i) {
      const uint32_t c = order[i];
      const size_t base = (size_t)dmax * c;
      for (int k = 0; k < dnum[c]; ++k) {
        if (sz >= n) return LO_ESTRUCTURE; /* cannot happen for a consistent table */
        order[sz++] = donor[base + k];
      }
    }
    lo = hi;
    hi = sz;
    if (hi > lo) levels[++nl] = (uint32_t)hi;
  }
  *nlevels = nl;
  if (sz != n) return LO_ESTRUCTURE;
  return LO_OK;
}

/* include/lem/accumulation.hpp:21-28 add_donor_flow; src/accumulation.cpp:7-26
 * accumulate_into / accumulate (uniform weight w0), order swept back to front. */
void lo_accumulate(size_t n, const uint32_t* order, const uint32_t* donor,
                   const uint8_t* dnum, int dmax, double w0, double* A) {
  for (size_t c = 0; c < n; ++c) A[c] = w0;
  for (size_t i = n; i-- > 0;) {
    const uint32_t c = order[i];
    const size_t base = (size_t)dmax * c;
    double a = A[c];
    for (int k = 0; k < dnum[c]; ++k) a += A[donor[base + k]];
    A[c] = a;
  }
}

/* src/erosion.cpp:52-57 -- uplift (interior only). */
void lo_uplift(double* elev, int w, int h, double du) {
  const size_t n = (size_t)w * h;
  for (size_t c = 0; c < n; ++c)
    if (!is_perimeter(c, w, h)) elev[c] += du;
}

/* src/erosion.cpp:19-34 -- newton_erode_cell. */
double lo_newton(double h0, double hn, double F, double n_exp, double eps, int max_iters,
                 int* iters, int* converged) {
  double hh = h0;
  double h_prev = h0;
  for (int it = 1; it <= max_iters; ++it) {
    const double diff = hh - hn;
    const double residual = hh - h0 + F * pow(diff, n_exp);
    const double slope = 1.0 + F * n_exp * pow(diff, n_exp - 1.0);
    hh -= residual / slope;
    if (hh < hn) hh = hn;
    const double delta = hh - h_prev;
    h_prev = hh;
    if (fabs(delta) <= eps) {
      *iters = it;
      *converged = 1;
      return hh;
    }
  }
  *iters = max_iters;
  *converged = 0;
  return hh;
}

/* include/lem/grid_graph.hpp:53-57 -- distance_between. */
static double distance_between(uint32_t a, uint32_t b, int w, const lo_nbh* nbh) {
  const int dx = (int)(b % (uint32_t)w) - (int)(a % (uint32_t)w);
  const int dy = (int)(b / (uint32_t)w) - (int)(a / (uint32_t)w);
  return lo_offset_length(dx, dy, nbh->dx, nbh->dy);
}

/* src/erosion.cpp:36-50 erode_one_cell and :66-81 erode (levels 1..L-1). */
int lo_erode(double* elev, int w, int h, const lo_nbh* nbh, const uint32_t* order,
             const uint32_t* levels, uint32_t nlevels, const uint32_t* rec, const double* A,
             const lo_params* p, uint64_t* iters, uint32_t* err_cell) {
  (void)h;
  uint64_t total = 0;
  for (uint32_t l = 1; l < nlevels; ++l) {
    for (uint32_t i = levels[l]; i < levels[l + 1]; ++i) {
      const uint32_t c = order[i];
      const uint32_t r = rec[c];
      const double dist = distance_between(c, r, w, nbh);
      const double F = p->K * p->dt * pow(A[c], p->m_exp) / pow(dist, p->n_exp);
      int it = 0, conv = 0;
      const double hnew =
          lo_newton(elev[c], elev[r], F, p->n_exp, p->epsilon, p->max_newton_iters, &it, &conv);
      if (!conv) {
        *iters = total;
        *err_cell = c;
        return LO_ECONVERGENCE;
      }
      elev[c] = hnew;
      total += (uint64_t)it;
    }
  }
  *iters = total;
  return LO_OK;
}

/* src/simulation.cpp:31-89 -- simulate_front + simulate_step (queue order, D8
 * or D4 routing, uniform cell-area weights). */
int lo_step(double* elev, int w, int h, int connectivity, const lo_params* p,
            lo_step_out* out) {
  lo_nbh nbh;
  if (lo_make_nbh(connectivity, p->dx, p->dy, &nbh) != LO_OK) return LO_ECONFIG;
  const size_t n = (size_t)w * h;
  const int dmax = connectivity;
  uint32_t* rec = out->rec ? out->rec : (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* donor = out->donor ? out->donor : (uint32_t*)malloc(n * dmax * sizeof(uint32_t));
  uint8_t* dnum = out->dnum ? out->dnum : (uint8_t*)malloc(n);
  uint32_t* order = out->order ? out->order : (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* levels = out->levels ? out->levels : (uint32_t*)malloc((n + 2) * sizeof(uint32_t));
  double* A = out->A ? out->A : (double*)malloc(n * sizeof(double));
  int rc = LO_OK;

  lo_receivers(elev, w, h, &nbh, rec);
  uint32_t pits = 0;
  for (size_t c = 0; c < n; ++c)
    if (rec[c] == LO_NOFLOW && !is_perimeter(c, w, h)) ++pits;
  out->interior_noflow = pits;
  lo_donors(rec, w, h, &nbh, donor, dnum);
  rc = lo_generate_queue(n, rec, donor, dnum, dmax, order, levels, &out->nlevels);
  if (rc == LO_OK) {
    lo_accumulate(n, order, donor, dnum, dmax, p->dx * p->dy, A);
    lo_uplift(elev, w, h, p->uplift_rate * p->dt);
    out->err_cell = LO_NOFLOW;
    rc = lo_erode(elev, w, h, &nbh, order, levels, out->nlevels, rec, A, p, &out->newton_iters,
                  &out->err_cell);
  }
  if (!out->rec) free(rec);
  if (!out->donor) free(donor);
  if (!out->dnum) free(dnum);
  if (!out->order) free(order);
  if (!out->levels) free(levels);
  if (!out->A) free(A);
  return rc;
}

/* src/mfd.cpp:33-64 compute_mfd: every strictly lower in-bounds neighbour of
 * an interior cell (stencil order) gets weight pow((e[c] - e[nb]) / dist,
 * exponent), normalised by their sum (accumulated in stencil order). */
void lo_compute_mfd(const double* elev, int w, int h, const lo_nbh* nbh, double exponent,
                    uint32_t* recs, double* alpha, uint8_t* rnum) {
  const size_t n = (size_t)w * h;
  const int dmax = nbh->connectivity;
  for (size_t c = 0; c < n; ++c) {
    const size_t base = (size_t)dmax * c;
    for (int i = 0; i < dmax; ++i) {
      recs[base + i] = LO_NOFLOW;
      alpha[base + i] = 0.0;
    }
    rnum[c] = 0;
    if (is_perimeter(c, w, h)) continue;
    const int x = (int)(c % (size_t)w), y = (int)(c / (size_t)w);
    double wsum = 0.0;
    int k = 0;
    for (int i = 0; i < nbh->connectivity; ++i) {
      const int nx = x + nbh->ox[i], ny = y + nbh->oy[i];
      if (nx < 0 || nx >= w || ny < 0 || ny >= h) continue;
      const uint32_t nb = (uint32_t)ny * (uint32_t)w + (uint32_t)nx;
      if (elev[nb] >= elev[c]) continue;  /* receivers must be strictly lower */
      const double slope = (elev[c] - elev[nb]) / nbh->dist[i];
      const double wt = pow(slope, exponent);
      recs[base + k] = nb;
      alpha[base + k] = wt;
      wsum += wt;
      ++k;
    }
    rnum[c] = (uint8_t)k;
    for (int i = 0; i < k; ++i) alpha[base + i] /= wsum;
  }
}

/* src/mfd.cpp:8-31 build_mfd_donor_table: donors of each cell in ascending
 * donor order (cells visited in ascending order). */
static void lo_mfd_donors(size_t n, int dmax, const uint32_t* recs, const double* alpha,
                          const uint8_t* rnum, uint32_t* donors, double* dalpha, uint8_t* dnum) {
  memset(dnum, 0, n);
  for (size_t c = 0; c < n; ++c) {
    const size_t base = (size_t)dmax * c;
    for (int k = 0; k < rnum[c]; ++k) {
      const uint32_t r = recs[base + k];
      const size_t slot = (size_t)dmax * r + dnum[r];
      donors[slot] = (uint32_t)c;
      dalpha[slot] = alpha[base + k];
      ++dnum[r];
    }
  }
}

static int lo_u32_less(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

/* src/mfd.cpp:66-104 generate_mfd_order: level 0 = cells without receivers
 * (ascending); a cell joins the wave after its last receiver is placed; each
 * level sorted ascending. */
int lo_mfd_order(size_t n, int dmax, const uint32_t* recs, const uint8_t* rnum, uint32_t* order,
                 uint32_t* levels, uint32_t* nlevels) {
  uint32_t* donors = (uint32_t*)malloc(n * dmax * sizeof(uint32_t));
  double* dalpha = (double*)malloc(n * dmax * sizeof(double));
  uint8_t* dnum = (uint8_t*)malloc(n);
  uint8_t* remaining = (uint8_t*)malloc(n);
  double* zero = (double*)calloc(n * dmax, sizeof(double));
  lo_mfd_donors(n, dmax, recs, zero, rnum, donors, dalpha, dnum);
  memcpy(remaining, rnum, n);
  size_t len = 0;
  uint32_t nl = 0;
  levels[nl++] = 0;
  for (size_t c = 0; c < n; ++c)
    if (remaining[c] == 0) order[len++] = (uint32_t)c;
  levels[nl++] = (uint32_t)len;
  size_t lo = 0, hi = len;
  while (lo < hi) {
    for (size_t i = lo; i < hi; ++i) {
      const uint32_t c = order[i];
      for (int k = 0; k < dnum[c]; ++k) {
        const uint32_t d = donors[(size_t)dmax * c + k];
        if (--remaining[d] == 0) order[len++] = d;
      }
    }
    qsort(order + hi, len - hi, sizeof(uint32_t), lo_u32_less);
    lo = hi;
    hi = len;
    if (hi > lo) levels[nl++] = (uint32_t)hi;
  }
  *nlevels = nl - 1;
  free(donors);
  free(dalpha);
  free(dnum);
  free(remaining);
  free(zero);
  return len == n ? LO_OK : LO_ESTRUCTURE;
}

/* src/mfd.cpp:106-132 accumulate_mfd_into / accumulate_mfd and
 * include/lem/mfd.hpp:62-69 add_mfd_donor_flow. */
void lo_accumulate_mfd(size_t n, int dmax, const uint32_t* recs, const double* alpha,
                       const uint8_t* rnum, const uint32_t* order, const uint32_t* levels,
                       uint32_t nlevels, double w0, double* A) {
  uint32_t* donors = (uint32_t*)malloc(n * dmax * sizeof(uint32_t));
  double* dalpha = (double*)malloc(n * dmax * sizeof(double));
  uint8_t* dnum = (uint8_t*)malloc(n);
  lo_mfd_donors(n, dmax, recs, alpha, rnum, donors, dalpha, dnum);
  for (size_t c = 0; c < n; ++c) A[c] = w0;
  for (uint32_t l = nlevels; l-- > 0;) {
    for (uint32_t i = levels[l]; i < levels[l + 1]; ++i) {
      const uint32_t c = order[i];
      const size_t base = (size_t)dmax * c;
      double a = A[c];
      for (int k = 0; k < dnum[c]; ++k) a += dalpha[base + k] * A[donors[base + k]];
      A[c] = a;
    }
  }
  free(donors);
  free(dalpha);
  free(dnum);
}

/* src/simulation.cpp:31-89 with Routing::kMfd: D8 receivers, donors and
 * queue (erosion follows the D8 receiver), MFD graph on the pre-uplift
 * elevation, MFD plan and accumulation, uplift, erosion. */
int lo_step_mfd(double* elev, int w, int h, int connectivity, const lo_params* p, double exponent,
                lo_step_out* out, uint32_t* mfd_order, uint32_t* mfd_levels, uint32_t* mfd_nlevels) {
  lo_nbh nbh;
  if (lo_make_nbh(connectivity, p->dx, p->dy, &nbh) != LO_OK) return LO_ECONFIG;
  const size_t n = (size_t)w * h;
  const int dmax = connectivity;
  uint32_t* rec = out->rec ? out->rec : (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* donor = out->donor ? out->donor : (uint32_t*)malloc(n * dmax * sizeof(uint32_t));
  uint8_t* dnum = out->dnum ? out->dnum : (uint8_t*)malloc(n);
  uint32_t* order = out->order ? out->order : (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* levels = out->levels ? out->levels : (uint32_t*)malloc((n + 2) * sizeof(uint32_t));
  double* A = out->A ? out->A : (double*)malloc(n * sizeof(double));
  uint32_t* recs = (uint32_t*)malloc(n * dmax * sizeof(uint32_t));
  double* alpha = (double*)malloc(n * dmax * sizeof(double));
  uint8_t* rnum = (uint8_t*)malloc(n);
  uint32_t* morder = mfd_order ? mfd_order : (uint32_t*)malloc(n * sizeof(uint32_t));
  uint32_t* mlevels = mfd_levels ? mfd_levels : (uint32_t*)malloc((n + 2) * sizeof(uint32_t));
  uint32_t mnl = 0;
  int rc = LO_OK;

  lo_receivers(elev, w, h, &nbh, rec);
  uint32_t pits = 0;
  for (size_t c = 0; c < n; ++c)
    if (rec[c] == LO_NOFLOW && !is_perimeter(c, w, h)) ++pits;
  out->interior_noflow = pits;
  lo_donors(rec, w, h, &nbh, donor, dnum);
  rc = lo_generate_queue(n, rec, donor, dnum, dmax, order, levels, &out->nlevels);
  if (rc == LO_OK) {
    lo_compute_mfd(elev, w, h, &nbh, exponent, recs, alpha, rnum);
    rc = lo_mfd_order(n, dmax, recs, rnum, morder, mlevels, &mnl);
  }
  if (rc == LO_OK) {
    lo_accumulate_mfd(n, dmax, recs, alpha, rnum, morder, mlevels, mnl, p->dx * p->dy, A);
    lo_uplift(elev, w, h, p->uplift_rate * p->dt);
    out->err_cell = LO_NOFLOW;
    rc = lo_erode(elev, w, h, &nbh, order, levels, out->nlevels, rec, A, p, &out->newton_iters,
                  &out->err_cell);
  }
  if (mfd_nlevels) *mfd_nlevels = mnl;
  if (!out->rec) free(rec);
  if (!out->donor) free(donor);
  if (!out->dnum) free(dnum);
  if (!out->order) free(order);
  if (!out->levels) free(levels);
  if (!out->A) free(A);
  if (!mfd_order) free(morder);
  if (!mfd_levels) free(mlevels);
  free(recs);
  free(alpha);
  free(rnum);
  return rc;
}

/* src/scheduler.cpp:466-500 -- run_simulation loop (rb_serial strategy). */
int lo_run(double* elev, int w, int h, int connectivity, const lo_params* p, uint32_t steps,
           uint64_t* newton_total, uint32_t* err_cell) {
  const size_t n = (size_t)w * h;
  lo_step_out o;
  memset(&o, 0, sizeof(o));
  o.rec = (uint32_t*)malloc(n * sizeof(uint32_t));
  o.donor = (uint32_t*)malloc(n * connectivity * sizeof(uint32_t));
  o.dnum = (uint8_t*)malloc(n);
  o.order = (uint32_t*)malloc(n * sizeof(uint32_t));
  o.levels = (uint32_t*)malloc((n + 2) * sizeof(uint32_t));
  o.A = (double*)malloc(n * sizeof(double));
  uint64_t total = 0;
  int rc = LO_OK;
  for (uint32_t s = 0; s < steps && rc == LO_OK; ++s) {
    rc = lo_step(elev, w, h, connectivity, p, &o);
    total += o.newton_iters;
  }
  *newton_total = total;
  *err_cell = o.err_cell;
  free(o.rec);
  free(o.donor);
  free(o.dnum);
  free(o.order);
  free(o.levels);
  free(o.A);
  return rc;
}

/* ---- Priority-Flood fill (src/depressions.cpp:26-68) ----------------------
 * Min-heap entries (spill elevation, cell); the lower elevation first, ties
 * by the lower cell index (HeapGreater, depressions.cpp:17-22).  The
 * perimeter seeds the flood at its own elevation (:38-44); every neighbour
 * (D8, stencil order, :50-56) not yet visited is raised to the spill
 * elevation (exact, :58-59) or to spill + eps when at or below it (epsilon
 * ascending, :60-62) and pushed with its new elevation. */
typedef struct { double v; uint32_t c; } lo_he;

static int lo_he_less(lo_he a, lo_he b) { return a.v < b.v || (a.v == b.v && a.c < b.c); }

static void lo_heap_push(lo_he* hp, size_t* n, lo_he e) {
  size_t i = (*n)++;
  while (i > 0) {
    const size_t p = (i - 1) / 2;
    if (!lo_he_less(e, hp[p])) break;
    hp[i] = hp[p];
    i = p;
  }
  hp[i] = e;
}

static lo_he lo_heap_pop(lo_he* hp, size_t* n) {
  const lo_he top = hp[0];
  const lo_he last = hp[--(*n)];
  size_t i = 0;
  for (;;) {
    size_t c = 2 * i + 1;
    if (c >= *n) break;
    if (c + 1 < *n && lo_he_less(hp[c + 1], hp[c])) ++c;
    if (!lo_he_less(hp[c], last)) break;
    hp[i] = hp[c];
    i = c;
  }
  if (*n > 0) hp[i] = last;
  return top;
}

void lo_fill(const double* elev, int w, int h, int mode, double eps, double* out) {
  const size_t n = (size_t)w * h;
  memcpy(out, elev, n * sizeof(double));
  if (mode == LO_FILL_OFF) return;
  static const int ox[8] = {-1, 0, 1, -1, 1, -1, 0, 1}, oy[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
  lo_he* hp = (lo_he*)malloc(n * sizeof(lo_he));
  char* vis = (char*)calloc(n, 1);
  size_t hn = 0;
  for (size_t c = 0; c < n; ++c) {
    const int x = (int)(c % (size_t)w), y = (int)(c / (size_t)w);
    if (!(x == 0 || y == 0 || x == w - 1 || y == h - 1)) continue;
    lo_he e = {out[c], (uint32_t)c};
    lo_heap_push(hp, &hn, e);
    vis[c] = 1;
  }
  while (hn > 0) {
    const lo_he top = lo_heap_pop(hp, &hn);
    const int cx = (int)(top.c % (uint32_t)w), cy = (int)(top.c / (uint32_t)w);
    for (int k = 0; k < 8; ++k) {
      const int nx = cx + ox[k], ny = cy + oy[k];
      if (nx < 0 || ny < 0 || nx >= w || ny >= h) continue;
      const size_t nc = (size_t)ny * w + nx;
      if (vis[nc]) continue;
      vis[nc] = 1;
      if (mode == LO_FILL_EXACT) {
        if (out[nc] < top.v) out[nc] = top.v;
      } else if (out[nc] <= top.v) {
        out[nc] = top.v + eps;
      }
      lo_he e = {out[nc], (uint32_t)nc};
      lo_heap_push(hp, &hn, e);
    }
  }
  free(hp);
  free(vis);
}
