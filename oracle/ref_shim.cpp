// ref_shim.cpp -- extern "C" wrapper over the UNMODIFIED reference library
// (TEST INFRASTRUCTURE ONLY).
//
// oracle/Makefile compiles this file together with the reference's own
// sources, where they lie under /root/reference/proj/src, into
// oracle/_ref/liblemref.so.  It lets the Python tests and bench.py's CPU
// baseline call the reference's real entry points:
//   lem::simulate_step   (src/simulation.cpp:68-89)      -- per-step goldens
//   lem::run_simulation  (src/scheduler.cpp:466-500)     -- timed CPU baseline
//   lem::generate_terrain(src/terrain.cpp:19-31)
// Nothing here is part of the product path.
#include <cstdint>
#include <cstring>
#include <chrono>
#include <exception>
#include <string>

#include <lem/depressions.hpp>
#include <lem/error.hpp>
#include <lem/scheduler.hpp>
#include <lem/simulation.hpp>
#include <lem/strategy.hpp>
#include <lem/terrain.hpp>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

thread_local std::string g_err;

struct LrParams {
  double K, m_exp, n_exp, uplift_rate, dt, epsilon, dx, dy;
  int max_newton_iters;
};

lem::SimParams to_params(const LrParams* p) {
  lem::SimParams s;
  s.K = p->K;
  s.m_exp = p->m_exp;
  s.n_exp = p->n_exp;
  s.uplift_rate = p->uplift_rate;
  s.dt = p->dt;
  s.epsilon = p->epsilon;
  s.dx = p->dx;
  s.dy = p->dy;
  s.max_newton_iters = p->max_newton_iters;
  return s;
}

// Status codes mirror include/lemgpu.h: 0 ok, 1 config, 2 structure,
// 3 convergence, 5 other.
template <typename F>
int guarded(F&& f, std::uint32_t* err_cell) {
  try {
    f();
    return 0;
  } catch (const lem::ConvergenceError& e) {
    g_err = e.what();
    if (err_cell) *err_cell = e.cell();
    return 3;
  } catch (const lem::StructureError& e) {
    g_err = e.what();
    return 2;
  } catch (const lem::ConfigError& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

}  // namespace

extern "C" {

const char* lr_last_error() { return g_err.c_str(); }

int lr_max_threads() {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void lr_generate_terrain(std::uint32_t w, std::uint32_t h, std::uint64_t seed, double* out) {
  lem::Raster<double> r = lem::generate_terrain(w, h, seed);
  std::memcpy(out, r.storage().data(), r.size() * sizeof(double));
}

// One lem::simulate_step on elev (in/out) exposing the workspace arrays.
int lr_simulate_step(int w, int h, int connectivity, const LrParams* p, double* elev,
                     std::uint32_t* rec, std::uint32_t* donor, std::uint8_t* dnum,
                     std::uint32_t* order, std::uint32_t* levels, std::uint32_t* nlevels,
                     double* A, std::uint64_t* newton, std::uint32_t* pits,
                     std::uint32_t* err_cell) {
  return guarded(
      [&] {
        const std::size_t n = static_cast<std::size_t>(w) * h;
        lem::Raster<double> r(w, h, std::vector<double>(elev, elev + n));
        const lem::Neighborhood nbh = lem::Neighborhood::make(connectivity, p->dx, p->dy);
        const lem::GridGraph g(w, h, nbh);
        lem::SimParams sp = to_params(p);
        sp.validate();
        lem::SimWorkspace ws;
        lem::StepSetup setup;
        lem::StepDiagnostics d;
        try {
          d = lem::simulate_step(r, g, sp, setup, ws);
        } catch (...) {
          std::memcpy(elev, r.storage().data(), n * sizeof(double));
          throw;
        }
        std::memcpy(elev, r.storage().data(), n * sizeof(double));
        if (rec) std::memcpy(rec, ws.fg.rec.data(), n * 4);
        if (donor) std::memcpy(donor, ws.fg.donor.data(), ws.fg.donor.size() * 4);
        if (dnum) std::memcpy(dnum, ws.fg.dnum.data(), n);
        if (order) std::memcpy(order, ws.plan.order.data(), n * 4);
        if (levels) std::memcpy(levels, ws.plan.levels.data(), ws.plan.levels.size() * 4);
        if (nlevels) *nlevels = static_cast<std::uint32_t>(ws.plan.nlevels());
        if (A) std::memcpy(A, ws.accum.values.storage().data(), n * sizeof(double));
        if (newton) *newton = d.newton_iters;
        if (pits) *pits = d.interior_noflow;
      },
      err_cell);
}

// One lem::simulate_step with StepSetup::routing = kMfd (src/simulation.cpp:
// 31-89): h, the MFD drainage area (ws.accum) and the MFD plan (ws.mfd_plan).
int lr_simulate_step_mfd(int w, int h, int connectivity, const LrParams* p, double exponent, double* elev,
                         double* A, std::uint32_t* mfd_order, std::uint32_t* mfd_levels,
                         std::uint32_t* mfd_nlevels, std::uint64_t* newton, std::uint32_t* err_cell) {
  return guarded(
      [&] {
        const std::size_t n = static_cast<std::size_t>(w) * h;
        lem::Raster<double> r(w, h, std::vector<double>(elev, elev + n));
        const lem::Neighborhood nbh = lem::Neighborhood::make(connectivity, p->dx, p->dy);
        const lem::GridGraph g(w, h, nbh);
        lem::SimParams sp = to_params(p);
        sp.validate();
        lem::SimWorkspace ws;
        lem::StepSetup setup;
        setup.routing = lem::Routing::kMfd;
        setup.mfd_exponent = exponent;
        lem::StepDiagnostics d;
        try {
          d = lem::simulate_step(r, g, sp, setup, ws);
        } catch (...) {
          std::memcpy(elev, r.storage().data(), n * sizeof(double));
          throw;
        }
        std::memcpy(elev, r.storage().data(), n * sizeof(double));
        if (A) std::memcpy(A, ws.accum.values.storage().data(), n * sizeof(double));
        if (mfd_order) std::memcpy(mfd_order, ws.mfd_plan.order.data(), n * 4);
        if (mfd_levels) std::memcpy(mfd_levels, ws.mfd_plan.levels.data(), ws.mfd_plan.levels.size() * 4);
        if (mfd_nlevels) *mfd_nlevels = static_cast<std::uint32_t>(ws.mfd_plan.nlevels());
        if (newton) *newton = d.newton_iters;
      },
      err_cell);
}

// run_simulation with a routing choice (0 d8, 1 mfd) and MFD exponent.
int lr_run_routing(int w, int h, int connectivity, const LrParams* p, const char* strategy,
                   std::uint32_t workers, std::uint32_t steps, int routing, double exponent, double* elev,
                   std::uint64_t* newton, std::uint32_t* err_cell) {
  return guarded(
      [&] {
        const std::size_t n = static_cast<std::size_t>(w) * h;
        auto kind = lem::strategy_from_string(strategy);
        if (!kind) throw lem::ConfigError(std::string("unknown strategy ") + strategy);
        lem::RunConfig cfg;
        cfg.width = static_cast<std::uint32_t>(w);
        cfg.height = static_cast<std::uint32_t>(h);
        cfg.timesteps = steps;
        cfg.strategy = {*kind, workers};
        cfg.params = to_params(p);
        cfg.connectivity = connectivity;
        cfg.routing = routing ? lem::Routing::kMfd : lem::Routing::kD8;
        cfg.mfd_exponent = exponent;
        lem::Raster<double> r(w, h, std::vector<double>(elev, elev + n));
        lem::RunResult res = lem::run_simulation(std::move(r), cfg);
        std::memcpy(elev, res.elevation.storage().data(), n * sizeof(double));
        if (newton) *newton = res.newton_iters;
      },
      err_cell);
}

// lem::run_simulation(Raster initial, cfg) under a named strategy.
// seconds_out receives the wall time of the stepping loop.
int lr_run(int w, int h, int connectivity, const LrParams* p, const char* strategy,
           std::uint32_t workers, std::uint32_t steps, double* elev, std::uint64_t* newton,
           std::uint32_t* err_cell) {
  return guarded(
      [&] {
        const std::size_t n = static_cast<std::size_t>(w) * h;
        auto kind = lem::strategy_from_string(strategy);
        if (!kind) throw lem::ConfigError(std::string("unknown strategy ") + strategy);
        lem::RunConfig cfg;
        cfg.width = static_cast<std::uint32_t>(w);
        cfg.height = static_cast<std::uint32_t>(h);
        cfg.timesteps = steps;
        cfg.strategy = {*kind, workers};
        cfg.params = to_params(p);
        cfg.connectivity = connectivity;
        lem::Raster<double> r(w, h, std::vector<double>(elev, elev + n));
        lem::RunResult res = lem::run_simulation(std::move(r), cfg);
        std::memcpy(elev, res.elevation.storage().data(), n * sizeof(double));
        if (newton) *newton = res.newton_iters;
      },
      err_cell);
}

// Timed CPU baseline: `warmup` untimed then `steps` timed lem::strategy_step
// calls of one strategy on a persistent workspace (the run_simulation loop
// body, scheduler.cpp:490-498).  seconds[i] = wall time of timed step i,
// including the per-step FlowGraph::resize the phase timers miss.
// fill_mode: 0 off, 1 exact, 2 epsilon ascending (run_simulation's
// generate_terrain + priority_flood_fill, scheduler.cpp:503-506)
int lr_bench_routing(int w, int h, int connectivity, const LrParams* p, const char* strategy,
                     std::uint32_t workers, std::uint64_t seed, std::uint32_t warmup, std::uint32_t steps,
                     double* seconds, std::uint64_t* newton, int fill_mode, double fill_eps, int routing,
                     double exponent);
int lr_bench(int w, int h, int connectivity, const LrParams* p, const char* strategy,
             std::uint32_t workers, std::uint64_t seed, std::uint32_t warmup, std::uint32_t steps,
             double* seconds, std::uint64_t* newton, int fill_mode, double fill_eps) {
  return lr_bench_routing(w, h, connectivity, p, strategy, workers, seed, warmup, steps, seconds, newton, fill_mode,
                          fill_eps, 0, 1.0);
}
// ... with StepSetup::routing (0 d8, 1 mfd) and the MFD exponent
int lr_bench_routing(int w, int h, int connectivity, const LrParams* p, const char* strategy,
                     std::uint32_t workers, std::uint64_t seed, std::uint32_t warmup, std::uint32_t steps,
                     double* seconds, std::uint64_t* newton, int fill_mode, double fill_eps, int routing,
                     double exponent) {
  return guarded(
      [&] {
        auto kind = lem::strategy_from_string(strategy);
        if (!kind) throw lem::ConfigError(std::string("unknown strategy ") + strategy);
        lem::Raster<double> r = lem::generate_terrain(w, h, seed);
        if (fill_mode) {
          lem::FillOptions o;
          o.mode = fill_mode == 1 ? lem::FillMode::kExact : lem::FillMode::kEpsilonAscending;
          o.epsilon_increment = fill_eps;
          r = lem::priority_flood_fill(r, o);
        }
        const lem::Neighborhood nbh = lem::Neighborhood::make(connectivity, p->dx, p->dy);
        const lem::GridGraph g(w, h, nbh);
        const lem::SimParams sp = to_params(p);
        lem::StepSetup setup;
        setup.order = lem::uses_stack_order(*kind) ? lem::OrderKind::kStack : lem::OrderKind::kQueue;
        setup.routing = routing ? lem::Routing::kMfd : lem::Routing::kD8;
        setup.mfd_exponent = exponent;
        const lem::Strategy st{*kind, workers};
        lem::SimWorkspace ws;
        std::uint64_t it = 0;
        for (std::uint32_t s = 0; s < warmup + steps; ++s) {
          const auto t0 = std::chrono::steady_clock::now();
          lem::StepDiagnostics d = lem::strategy_step(r, g, sp, setup, st, ws);
          const auto t1 = std::chrono::steady_clock::now();
          if (s >= warmup) {
            seconds[s - warmup] = std::chrono::duration<double>(t1 - t0).count();
            it += d.newton_iters;
          }
        }
        if (newton) *newton = it;
      },
      nullptr);
}

// lem::priority_flood_fill (src/depressions.cpp:26-68): mode 0 off, 1 exact, 2 epsilon ascending
int lr_fill(int w, int h, const double* elev, int mode, double eps, double* out) {
  return guarded(
      [&] {
        lem::Raster<double> r(w, h, std::vector<double>(elev, elev + (std::size_t)w * h));
        lem::FillOptions o;
        o.mode = mode == 1 ? lem::FillMode::kExact : mode == 2 ? lem::FillMode::kEpsilonAscending : lem::FillMode::kOff;
        o.epsilon_increment = eps;
        const lem::Raster<double> f = lem::priority_flood_fill(r, o);
        std::memcpy(out, f.storage().data(), sizeof(double) * (std::size_t)w * h);
      },
      nullptr);
}

}  // extern "C"
