// lem_rb_gpu.cpp -- see lem_rb_gpu.hpp.  Host-only C++ over the C-ABI.
#include "lem_rb_gpu.hpp"

#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <unordered_map>

#include <lem/error.hpp>
#include <lem/neighborhood.hpp>

#include "lemgpu.h"

namespace lem::gpu {
namespace {

struct Ctx {
  lemgpu_ctx* h = nullptr;
  int w = 0, hgt = 0, conn = 0, device = 0;
  int routing = 0;            // lemgpu_set_routing state (0 d8, 1 mfd)
  double mfd_exponent = 1.0;
  SimParams params{};
  ~Ctx() {
    if (h) lemgpu_destroy(h);
  }
};

std::mutex g_mu;
std::unordered_map<const SimWorkspace*, std::unique_ptr<Ctx>>& table() {
  static std::unordered_map<const SimWorkspace*, std::unique_ptr<Ctx>> t;
  return t;
}

// ErrorCollector::rethrow mapping (scheduler.cpp:45-49).
[[noreturn]] void raise(int status, const std::string& msg, std::uint32_t cell) {
  switch (status) {
    case LEMGPU_ECONFIG:
      throw ConfigError(msg);
    case LEMGPU_ESTRUCTURE:
      throw StructureError(msg);
    case LEMGPU_ECONVERGENCE:
      throw ConvergenceError(cell, msg);
    default:
      throw Error(msg);
  }
}

void check(lemgpu_ctx* h, int rc) {
  if (rc != LEMGPU_OK) raise(rc, lemgpu_error_message(h), lemgpu_error_cell(h));
}

lemgpu_params to_abi(const SimParams& p, int connectivity) {
  lemgpu_params q{};
  q.K = p.K;
  q.m_exp = p.m_exp;
  q.n_exp = p.n_exp;
  q.uplift_rate = p.uplift_rate;
  q.dt = p.dt;
  q.epsilon = p.epsilon;
  q.dx = p.dx;
  q.dy = p.dy;
  q.max_newton_iters = p.max_newton_iters;
  q.connectivity = connectivity;
  return q;
}

bool same(const SimParams& a, const SimParams& b) {
  return a.K == b.K && a.m_exp == b.m_exp && a.n_exp == b.n_exp && a.uplift_rate == b.uplift_rate &&
         a.dt == b.dt && a.epsilon == b.epsilon && a.dx == b.dx && a.dy == b.dy &&
         a.max_newton_iters == b.max_newton_iters;
}

std::unique_ptr<Ctx> make_ctx(int w, int h, int conn, const SimParams& p, int device) {
  auto c = std::make_unique<Ctx>();
  const lemgpu_params q = to_abi(p, conn);
  lemgpu_options o{};
  o.phase_clocks = 1;  // StepDiagnostics::timings / RunResult::phase_totals
  const int rc = lemgpu_create_ex(device, static_cast<std::uint32_t>(w), static_cast<std::uint32_t>(h), 1, &q, nullptr,
                                  &o, &c->h);
  if (rc != LEMGPU_OK) raise(rc, lemgpu_error_message(nullptr), kNoFlow);
  c->w = w;
  c->hgt = h;
  c->conn = conn;
  c->device = device;
  c->params = p;
  return c;
}

Ctx& ctx_for(SimWorkspace& ws, const GridGraph& g, const SimParams& p, int device) {
  std::lock_guard<std::mutex> lock(g_mu);
  auto& slot = table()[&ws];
  const int conn = g.neighborhood().connectivity;
  if (!slot || slot->w != g.width() || slot->hgt != g.height() || slot->conn != conn ||
      slot->device != device || !same(slot->params, p))
    slot = make_ctx(g.width(), g.height(), conn, p, device);
  return *slot;
}

StepDiagnostics to_diag(const lemgpu_diag& d) {
  StepDiagnostics out;
  for (int i = 0; i < kNumPhases; ++i) out.timings.seconds[i] = d.seconds[i];
  out.newton_iters = d.newton_iters;
  out.interior_noflow = d.interior_noflow;
  return out;
}

void check_setup(const StepSetup& setup) {
  // the device path is the breadth-first queue plan; Routing::kMfd feeds it the
  // multiple-flow drainage area (simulation.cpp:53-60), like rb_par_all
  if (setup.routing == Routing::kMfd && !(setup.mfd_exponent > 0.0))
    throw ConfigError("mfd_exponent must be > 0");  // config.cpp:166
  if (setup.order == OrderKind::kStack) throw ConfigError("rb_gpu uses the breadth-first queue order");
}

// StepSetup::routing / mfd_exponent onto the context (graphs rebuilt only on a change)
void apply_routing(Ctx& c, const StepSetup& setup) {
  const int r = setup.routing == Routing::kMfd ? 1 : 0;
  const double e = r ? setup.mfd_exponent : 1.0;
  if (r == c.routing && e == c.mfd_exponent) return;
  check(c.h, lemgpu_set_routing(c.h, r, e));
  c.routing = r;
  c.mfd_exponent = e;
}

}  // namespace

StepDiagnostics strategy_step_rb_gpu(Raster<double>& elev, const GridGraph& grid, const SimParams& params,
                                     const StepSetup& setup, SimWorkspace& ws, int device) {
  check_setup(setup);
  params.validate();
  Ctx& c = ctx_for(ws, grid, params, device);
  apply_routing(c, setup);
  lemgpu_diag d{};
  check(c.h, lemgpu_step_host(c.h, elev.storage().data(), &d));
  return to_diag(d);
}

RunResult run_simulation_rb_gpu(Raster<double> initial, const RunConfig& cfg, const StepCallback& on_step,
                                int device) {
  cfg.validate();
  if (initial.width() != static_cast<int>(cfg.width) || initial.height() != static_cast<int>(cfg.height))
    throw ConfigError("initial raster is " + std::to_string(initial.width()) + "x" +
                      std::to_string(initial.height()) + " but config says " + std::to_string(cfg.width) + "x" +
                      std::to_string(cfg.height));
  StepSetup setup;
  setup.routing = cfg.routing;
  setup.mfd_exponent = cfg.mfd_exponent;
  check_setup(setup);
  auto c = make_ctx(initial.width(), initial.height(), cfg.connectivity, cfg.params, device);
  apply_routing(*c, setup);
  check(c->h, lemgpu_upload_elev(c->h, initial.storage().data()));  // rejects non-finite input
  RunResult res;
  res.elevation = std::move(initial);
  res.per_step.reserve(cfg.timesteps);
  if (!on_step) {
    std::vector<lemgpu_diag> d(cfg.timesteps);
    if (cfg.timesteps) check(c->h, lemgpu_step(c->h, cfg.timesteps, d.data()));
    for (const auto& x : d) res.per_step.push_back(to_diag(x));
  } else {
    // The callback needs each step's raster (lem run's snapshots,
    // proj/tools/lem.cpp:143-147).  Pipelined: step s+1 runs on the device
    // while step s's raster comes down on a side stream (lemgpu_snapshot_async)
    // into one of two pinned staging rasters and the callback sees it.
    Raster<double> stage[2] = {Raster<double>(res.elevation.width(), res.elevation.height()),
                               Raster<double>(res.elevation.width(), res.elevation.height())};
    const std::size_t bytes = stage[0].size() * sizeof(double);
    bool pinned[2];
    for (int i = 0; i < 2; ++i) pinned[i] = lemgpu_host_register(stage[i].storage().data(), bytes) == LEMGPU_OK;
    lemgpu_diag dg[2]{};
    auto deliver = [&](std::uint32_t s) {
      check(c->h, lemgpu_snapshot_wait(c->h));
      const lemgpu_diag& d = dg[s & 1u];
      if (d.status != 0) check(c->h, lemgpu_sync(c->h, nullptr, 0, nullptr));  // throws the step's error
      StepDiagnostics sd = to_diag(d);
      on_step(s, stage[s & 1u], sd);
      res.per_step.push_back(std::move(sd));
    };
    try {
      for (std::uint32_t s = 1; s <= cfg.timesteps; ++s) {
        check(c->h, lemgpu_step_async(c->h, 1));  // runs beside the previous snapshot's copy and callback
        if (s > 1) deliver(s - 1);
        check(c->h, lemgpu_snapshot_async(c->h, stage[s & 1u].storage().data(), &dg[s & 1u]));
      }
      if (cfg.timesteps) deliver(cfg.timesteps);
      check(c->h, lemgpu_sync(c->h, nullptr, 0, nullptr));
    } catch (...) {
      lemgpu_snapshot_wait(c->h);
      for (int i = 0; i < 2; ++i)
        if (pinned[i]) lemgpu_host_unregister(stage[i].storage().data());
      throw;
    }
    for (int i = 0; i < 2; ++i)
      if (pinned[i]) lemgpu_host_unregister(stage[i].storage().data());
  }
  check(c->h, lemgpu_download_elev(c->h, res.elevation.storage().data()));
  for (const auto& d : res.per_step) {
    res.phase_totals += d.timings;
    res.newton_iters += d.newton_iters;
    res.interior_noflow_last = d.interior_noflow;
  }
  return res;
}

namespace {
int fill_mode(const FillOptions& o) {
  return o.mode == FillMode::kExact ? LEMGPU_FILL_EXACT
         : o.mode == FillMode::kEpsilonAscending ? LEMGPU_FILL_EPSILON
                                                 : LEMGPU_FILL_OFF;
}
}  // namespace

Raster<double> priority_flood_fill_rb_gpu(const Raster<double>& elev, const FillOptions& opts, int device) {
  Raster<double> out = elev;
  if (opts.mode == FillMode::kOff) return out;
  auto c = make_ctx(elev.width(), elev.height(), 8, SimParams{}, device);
  check(c->h, lemgpu_upload_elev(c->h, elev.storage().data()));
  check(c->h, lemgpu_fill(c->h, fill_mode(opts), opts.epsilon_increment));
  check(c->h, lemgpu_download_elev(c->h, out.storage().data()));
  return out;
}

RunResult run_simulation_rb_gpu(const RunConfig& cfg, const StepCallback& on_step, int device) {
  cfg.validate();
  Raster<double> terrain(static_cast<int>(cfg.width), static_cast<int>(cfg.height));
  {
    auto c = make_ctx(terrain.width(), terrain.height(), cfg.connectivity, cfg.params, device);
    const std::uint64_t seed = cfg.seed;
    check(c->h, lemgpu_generate_terrain(c->h, &seed));
    check(c->h, lemgpu_fill(c->h, fill_mode(cfg.fill), cfg.fill.epsilon_increment));
    check(c->h, lemgpu_download_elev(c->h, terrain.storage().data()));
  }
  return run_simulation_rb_gpu(std::move(terrain), cfg, on_step, device);
}

void fill_workspace(SimWorkspace& ws) {
  Ctx* c = nullptr;
  {
    std::lock_guard<std::mutex> lock(g_mu);
    auto it = table().find(&ws);
    if (it == table().end() || !it->second) throw ConfigError("no rb_gpu step has run in this workspace");
    c = it->second.get();
  }
  const std::size_t n = static_cast<std::size_t>(c->w) * c->hgt;
  ws.fg.resize(c->w, c->hgt, c->conn);
  std::vector<std::uint32_t> levels(n + 2);
  std::uint32_t nl = 0;
  ws.accum.values = Raster<double>(c->w, c->hgt);
  ws.accum.cell_area = c->params.cell_area();
  ws.plan.order.resize(n);
  check(c->h, lemgpu_download_graph(c->h, ws.fg.rec.data(), ws.fg.dnum.data(), ws.fg.donor.data(),
                                    ws.plan.order.data(), levels.data(), &nl,
                                    ws.accum.values.storage().data()));
  ws.plan.levels.assign(levels.begin(), levels.begin() + nl + 1);
}

void release_workspace(SimWorkspace& ws) {
  std::lock_guard<std::mutex> lock(g_mu);
  table().erase(&ws);
}

}  // namespace lem::gpu
