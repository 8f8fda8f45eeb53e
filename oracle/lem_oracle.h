/*
 * lem_oracle.h -- CPU restatement of the reference D8 timestep (TEST INFRASTRUCTURE).
 *
 * This is the parity CHECKER for the B200 path, not part of the product.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  Every function restates one reference function and cites it
 * (paths relative to the reference tree's proj/ directory).
 *
 * Conventions mirror the reference exactly:
 *   - row-major cells, index = y*width + x          (include/lem/raster.hpp:56-59)
 *   - no-receiver sentinel UINT32_MAX               (include/lem/raster.hpp:16)
 *   - frozen D8 stencil order                       (src/neighborhood.cpp:12)
 *   - no FMA contraction (-ffp-contract=off)        (CMakeLists.txt:14)
 */
#ifndef LEM_ORACLE_H
#define LEM_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LO_NOFLOW 0xFFFFFFFFu

enum { LO_OK = 0, LO_ECONFIG = 1, LO_ESTRUCTURE = 2, LO_ECONVERGENCE = 3 };

/* Neighbourhood (include/lem/neighborhood.hpp:31-45). */
typedef struct lo_nbh {
  int connectivity;   /* 4 or 8 */
  int ox[8], oy[8];   /* offsets in stencil order */
  double dist[8];     /* offset_length of each offset */
  double dx, dy;
} lo_nbh;

/* SimParams (include/lem/erosion.hpp:15-25). */
typedef struct lo_params {
  double K, m_exp, n_exp, uplift_rate, dt, epsilon, dx, dy;
  int max_newton_iters;
} lo_params;

void lo_default_params(lo_params* p);
int lo_make_nbh(int connectivity, double dx, double dy, lo_nbh* out);
double lo_offset_length(int dx, int dy, double sx, double sy);

uint64_t lo_splitmix64(uint64_t x);
void lo_generate_terrain(uint32_t w, uint32_t h, uint64_t seed, double* out);
uint64_t lo_fnv1a64(const void* data, size_t nbytes);

void lo_receivers(const double* elev, int w, int h, const lo_nbh* nbh, uint32_t* rec);
void lo_donors(const uint32_t* rec, int w, int h, const lo_nbh* nbh, uint32_t* donor,
               uint8_t* dnum);

/* Explicit-graph variants (tests/fixtures.hpp:22-41 ExplicitGraph): CSR adjacency. */
void lo_receivers_explicit(size_t n, const uint32_t* adj_off, const uint32_t* adj_nbr,
                           const double* adj_dist, const uint8_t* boundary,
                           const double* elev, uint32_t* rec);
void lo_donors_explicit(size_t n, int dmax, const uint32_t* adj_off, const uint32_t* adj_nbr,
                        const uint32_t* rec, uint32_t* donor, uint8_t* dnum);

/* Returns LO_OK or LO_ESTRUCTURE; levels needs room for n+2 entries. */
int lo_generate_queue(size_t n, const uint32_t* rec, const uint32_t* donor,
                      const uint8_t* dnum, int dmax, uint32_t* order, uint32_t* levels,
                      uint32_t* nlevels);
void lo_accumulate(size_t n, const uint32_t* order, const uint32_t* donor,
                   const uint8_t* dnum, int dmax, double w0, double* A);
void lo_uplift(double* elev, int w, int h, double du);
double lo_newton(double h0, double hn, double F, double n_exp, double eps, int max_iters,
                 int* iters, int* converged);
int lo_erode(double* elev, int w, int h, const lo_nbh* nbh, const uint32_t* order,
             const uint32_t* levels, uint32_t nlevels, const uint32_t* rec, const double* A,
             const lo_params* p, uint64_t* iters, uint32_t* err_cell);

/* One whole reference step (src/simulation.cpp:68-89).  All output arrays
 * are caller-owned; any may be NULL except the ones the step itself needs
 * (a scratch workspace is allocated internally for NULL ones). */
typedef struct lo_step_out {
  uint32_t* rec;      /* N      */
  uint32_t* donor;    /* N*dmax */
  uint8_t* dnum;      /* N      */
  uint32_t* order;    /* N      */
  uint32_t* levels;   /* N+2    */
  uint32_t nlevels;
  double* A;          /* N      */
  uint64_t newton_iters;
  uint32_t interior_noflow;
  uint32_t err_cell;
} lo_step_out;

int lo_step(double* elev, int w, int h, int connectivity, const lo_params* p,
            lo_step_out* out);
int lo_run(double* elev, int w, int h, int connectivity, const lo_params* p, uint32_t steps,
           uint64_t* newton_total, uint32_t* err_cell);

/* Multiple-flow-direction routing (src/mfd.cpp, include/lem/mfd.hpp).
 * recs / alpha: N*dmax receiver slots (stencil order) and their normalised
 * weights; rnum: receivers per cell.  dmax = connectivity. */
void lo_compute_mfd(const double* elev, int w, int h, const lo_nbh* nbh, double exponent,
                    uint32_t* recs, double* alpha, uint8_t* rnum);
/* Dependency-counting level order; levels needs n+2 entries. LO_ESTRUCTURE on a cycle. */
int lo_mfd_order(size_t n, int dmax, const uint32_t* recs, const uint8_t* rnum, uint32_t* order,
                 uint32_t* levels, uint32_t* nlevels);
/* A = w0 + alpha-weighted donor pulls in ascending donor order, last level first. */
void lo_accumulate_mfd(size_t n, int dmax, const uint32_t* recs, const double* alpha,
                       const uint8_t* rnum, const uint32_t* order, const uint32_t* levels,
                       uint32_t nlevels, double w0, double* A);
/* simulate_step with StepSetup::routing = kMfd (src/simulation.cpp:31-89):
 * the D8 plan erodes, the MFD accumulation feeds it.  out as lo_step (A = the
 * MFD drainage area); mfd_order / mfd_levels (N, N+2; may be NULL) receive
 * the MFD plan. */
int lo_step_mfd(double* elev, int w, int h, int connectivity, const lo_params* p, double exponent,
                lo_step_out* out, uint32_t* mfd_order, uint32_t* mfd_levels, uint32_t* mfd_nlevels);

/* Priority-Flood depression filling (src/depressions.cpp:26-68,
 * include/lem/depressions.hpp:8-27): mode 0 off, 1 exact (raise to the spill
 * elevation), 2 epsilon ascending (spill + eps).  A binary min-heap over
 * (elevation, cell index) -- the reference's std::priority_queue order. */
enum { LO_FILL_OFF = 0, LO_FILL_EXACT = 1, LO_FILL_EPSILON = 2 };
void lo_fill(const double* elev, int w, int h, int mode, double eps, double* out);

#ifdef __cplusplus
}
#endif
#endif
