// lem_rb_gpu.hpp -- C++ drop-in of the B200 step behind the reference's own
// step entry points (the "rb_gpu" execution strategy).
//
// Compiled INSIDE the reference tree (it includes <lem/...> headers): a
// maintainer adds StrategyKind::kRbGpu to proj/include/lem/strategy.hpp:12-56
// and one case to the strategy_step switch (proj/src/scheduler.cpp:425-462)
// that forwards here; see INTEGRATION.md.  Everything below talks to the GPU
// only through the C-ABI of include/lemgpu.h.
#pragma once

#include <lem/config.hpp>
#include <lem/depressions.hpp>
#include <lem/raster.hpp>
#include <lem/scheduler.hpp>
#include <lem/simulation.hpp>

namespace lem::gpu {

// lem::strategy_step for StrategyKind::kRbGpu (scheduler.hpp:38-41): one
// timestep of `elev` (host raster, updated in place) on CUDA device `device`.
// The device context (all device buffers) is cached per SimWorkspace and
// reused across steps, like the workspace's own scratch (simulation.hpp:43-52).
// Throws ConfigError / StructureError / ConvergenceError(cell) / Error exactly
// where the reference strategies do.
StepDiagnostics strategy_step_rb_gpu(Raster<double>& elev, const GridGraph& grid,
                                     const SimParams& params, const StepSetup& setup,
                                     SimWorkspace& ws, int device = 0);

// lem::run_simulation (scheduler.hpp:61-65) with strategy rb_gpu: the elevation
// stays on the device for the whole run; it is copied back per step only when
// on_step is set (the callback needs the raster), and once at the end.
RunResult run_simulation_rb_gpu(Raster<double> initial, const RunConfig& cfg,
                                const StepCallback& on_step = {}, int device = 0);

// lem::run_simulation(const RunConfig&, ...) (scheduler.hpp:64-65,
// scheduler.cpp:503-506) with strategy rb_gpu: generate_terrain(cfg.seed) and
// the optional depression fill (cfg.fill) on the device, then the run.
RunResult run_simulation_rb_gpu(const RunConfig& cfg, const StepCallback& on_step = {}, int device = 0);

// lem::priority_flood_fill (depressions.hpp:21-27) on the device (lemgpu_fill),
// bit-identical in both modes.
Raster<double> priority_flood_fill_rb_gpu(const Raster<double>& elev, const FillOptions& opts, int device = 0);

// Copy the last step's flow graph, plan and accumulation into ws.fg / ws.plan /
// ws.accum in the reference layouts (for parity checks and inspection).
void fill_workspace(SimWorkspace& ws);

// Drop the device context cached for ws (also done automatically at exit).
void release_workspace(SimWorkspace& ws);

}  // namespace lem::gpu
