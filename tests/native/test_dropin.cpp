// Drop-in check of the rb_gpu strategy THROUGH THE REFERENCE'S OWN C++ API.
//
// Links the unmodified reference library (oracle/_ref/liblemref.so, built from
// /root/reference/proj/src) and the C++ shim paper_1803_02977_b200/host/
// lem_rb_gpu.cpp over the C-ABI.  Every check compares bytes with the
// reference's own strategies, the way proj/tests/acceptance.cpp:85-110
// compares strategies with each other.  Needs a GPU; built by oracle/Makefile.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <lem/error.hpp>
#include <lem/raster_io.hpp>
#include <lem/scheduler.hpp>
#include <lem/terrain.hpp>

#include "lem_rb_gpu.hpp"

using namespace lem;

static int g_fail = 0;
#define CHECK(cond, ...)                       \
  do {                                         \
    if (!(cond)) {                             \
      std::printf("FAIL %s:%d ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);                \
      std::printf("\n");                       \
      ++g_fail;                                \
    }                                          \
  } while (0)

static RunConfig cfg_of(int w, int h, std::uint64_t seed, std::uint32_t steps) {
  RunConfig c;
  c.width = w;
  c.height = h;
  c.seed = seed;
  c.timesteps = steps;
  c.strategy = {StrategyKind::kRbPrivateQueues, 8};
  return c;
}

// run_simulation: reference strategy vs rb_gpu, byte-identical elevations
static void check_run(RunConfig c, const char* name) {
  Raster<double> init = generate_terrain(c.width, c.height, c.seed);
  RunResult want = run_simulation(init, c);
  RunResult got = gpu::run_simulation_rb_gpu(init, c);
  auto diff = first_difference(want.elevation, got.elevation);
  CHECK(!diff, "%s: elevation differs at cell %u", name, diff ? *diff : 0u);
  CHECK(want.newton_iters == got.newton_iters, "%s: newton %llu vs %llu", name,
        (unsigned long long)want.newton_iters, (unsigned long long)got.newton_iters);
  CHECK(want.interior_noflow_last == got.interior_noflow_last, "%s: pits", name);
  std::printf("%s %s (%ux%u, %u steps)\n", diff ? "FAIL" : "ok  ", name, c.width, c.height, c.timesteps);
}

int main() {
  // 1. whole runs, several shapes / params (acceptance.cpp:85-110 style)
  check_run(cfg_of(100, 80, 1, 40), "d8 100x80");
  check_run(cfg_of(1000, 1000, 42, 30), "d8 1000^2");
  {
    RunConfig c = cfg_of(64, 50, 5, 20);
    c.connectivity = 4;
    check_run(c, "d4 64x50");
  }
  {
    RunConfig c = cfg_of(90, 61, 7, 20);
    c.params.dx = 0.5;
    c.params.dy = 2.0;
    check_run(c, "anisotropic spacing");
  }
  {
    RunConfig c = cfg_of(120, 80, 8, 20);
    c.params.m_exp = 0.35;
    c.params.K = 5e-6;
    check_run(c, "m=0.35 K=5e-6");
  }

  // 2. strategy_step is interchangeable step by step with a CPU strategy
  {
    const int w = 77, h = 65;
    Raster<double> a = generate_terrain(w, h, 9), b = a;
    const GridGraph g(w, h, Neighborhood::d8());
    SimParams p;
    StepSetup s;
    SimWorkspace wa, wb;
    std::uint64_t na = 0, nb = 0;
    for (int step = 0; step < 12; ++step) {
      na += strategy_step(a, g, p, s, {StrategyKind::kRbSerial, 1}, wa).newton_iters;
      if (step % 2 == 0)
        nb += gpu::strategy_step_rb_gpu(b, g, p, s, wb).newton_iters;
      else
        nb += strategy_step(b, g, p, s, {StrategyKind::kRbParAll, 4}, wb).newton_iters;
    }
    CHECK(a == b && na == nb, "alternating gpu/cpu steps diverge");
    std::printf("%s interleaved rb_gpu / rb_par_all steps == rb_serial\n", a == b ? "ok  " : "FAIL");
    gpu::release_workspace(wb);
  }

  // 3. the workspace of one step: FlowGraph, TraversalPlan, AccumField
  {
    const int w = 60, h = 45;
    Raster<double> a = generate_terrain(w, h, 3), b = a;
    const GridGraph g(w, h, Neighborhood::d8());
    SimParams p;
    StepSetup s;
    SimWorkspace wa, wb;
    simulate_step(a, g, p, s, wa);
    gpu::strategy_step_rb_gpu(b, g, p, s, wb);
    gpu::fill_workspace(wb);
    const bool ok = wa.fg.rec == wb.fg.rec && wa.fg.dnum == wb.fg.dnum && wa.fg.donor == wb.fg.donor &&
                    wa.plan.order == wb.plan.order && wa.plan.levels == wb.plan.levels &&
                    wa.accum.values == wb.accum.values && a == b;
    CHECK(ok, "workspace arrays differ");
    std::printf("%s FlowGraph / TraversalPlan / AccumField identical to simulate_step\n", ok ? "ok  " : "FAIL");
    gpu::release_workspace(wb);
  }

  // 4. error behaviour (error.hpp:10-43)
  {
    RunConfig c = cfg_of(40, 40, 5, 2);
    c.params.max_newton_iters = 1;
    Raster<double> init = generate_terrain(40, 40, 5);
    bool got = false;
    try {
      gpu::run_simulation_rb_gpu(init, c);
    } catch (const ConvergenceError& e) {
      got = e.cell() < 1600;
    }
    CHECK(got, "ConvergenceError not raised");
    init[123] = std::nan("");
    bool cfg = false;
    try {
      c.params.max_newton_iters = 100;
      gpu::run_simulation_rb_gpu(init, c);
    } catch (const ConfigError& e) {
      cfg = std::string(e.what()).find("cell 123") != std::string::npos;
    }
    CHECK(cfg, "non-finite input not rejected");
    StepSetup mfd;
    mfd.routing = Routing::kMfd;
    mfd.mfd_exponent = 0.0;  // config.cpp:166
    bool mf = false;
    try {
      SimWorkspace ws;
      Raster<double> r = generate_terrain(10, 10, 1);
      gpu::strategy_step_rb_gpu(r, GridGraph(10, 10, Neighborhood::d8()), SimParams{}, mfd, ws);
    } catch (const ConfigError&) {
      mf = true;
    }
    CHECK(mf, "mfd_exponent 0 accepted");
    std::printf("%s ConvergenceError(cell) / ConfigError behaviour\n", (got && cfg && mf) ? "ok  " : "FAIL");
  }

  // 4b. MFD routing (simulation.cpp:53-60): rb_gpu steps == rb_par_all steps,
  // alternating with D8 steps on the same workspace (routing switched per step)
  {
    Raster<double> a = generate_terrain(150, 110, 21), b = a;
    const GridGraph g(150, 110, Neighborhood::d8());
    SimWorkspace wa, wb;
    const Strategy par{StrategyKind::kRbParAll, 4};
    bool ok = true;
    for (int s = 0; s < 6; ++s) {
      StepSetup st;
      st.routing = (s % 3 == 2) ? Routing::kD8 : Routing::kMfd;
      st.mfd_exponent = s < 3 ? 1.0 : 1.4;
      strategy_step(a, g, SimParams{}, st, par, wa);
      gpu::strategy_step_rb_gpu(b, g, SimParams{}, st, wb);
      if (first_difference(a, b)) ok = false;
    }
    CHECK(ok, "MFD routing differs from rb_par_all");
    std::printf("%s MFD routing (exponents 1, 1.4) interleaved with D8 == rb_par_all\n", ok ? "ok  " : "FAIL");
  }

  // 5. on_step callback sees every step's raster (scheduler.cpp:496)
  {
    RunConfig c = cfg_of(50, 40, 11, 6);
    Raster<double> init = generate_terrain(50, 40, 11);
    std::vector<double> want, got;
    run_simulation(init, c, [&](std::uint32_t, const Raster<double>& r, const StepDiagnostics&) {
      want.push_back(r[1234]);
    });
    gpu::run_simulation_rb_gpu(init, c, [&](std::uint32_t, const Raster<double>& r, const StepDiagnostics&) {
      got.push_back(r[1234]);
    });
    CHECK(want == got, "callback rasters differ");
    std::printf("%s on_step callbacks\n", want == got ? "ok  " : "FAIL");
  }
  // 5. Priority-Flood fill and the filled-DEM run (scheduler.cpp:503-506)
  for (FillMode m : {FillMode::kExact, FillMode::kEpsilonAscending}) {
    const Raster<double> t = generate_terrain(300, 200, 5);
    FillOptions o;
    o.mode = m;
    auto diff = first_difference(priority_flood_fill(t, o), gpu::priority_flood_fill_rb_gpu(t, o));
    CHECK(!diff, "fill mode %d differs at cell %u", (int)m, diff ? *diff : 0u);
    std::printf("%s priority_flood_fill mode %d (300x200)\n", diff ? "FAIL" : "ok  ", (int)m);
  }
  {
    RunConfig c = cfg_of(200, 150, 3, 10);
    c.fill.mode = FillMode::kEpsilonAscending;
    RunResult want = run_simulation(c);
    RunResult got = gpu::run_simulation_rb_gpu(c);
    auto diff = first_difference(want.elevation, got.elevation);
    CHECK(!diff, "filled run differs at cell %u", diff ? *diff : 0u);
    CHECK(want.newton_iters == got.newton_iters, "filled run newton");
    std::printf("%s run_simulation(cfg) with epsilon fill (200x150, 10 steps)\n", diff ? "FAIL" : "ok  ");
  }
  std::printf("%d failure(s)\n", g_fail);
  return g_fail ? 1 : 0;
}
