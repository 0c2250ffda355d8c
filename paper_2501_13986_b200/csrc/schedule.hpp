// The reference's per-row schedule model and its dumps, computed by the
// product (not borrowed from the reference): the scratch-budget phase plan of
// scheduler::build_schedule (scheduler.cpp:139-389), its traffic model
// (traffic_report, scheduler.cpp:391-404), the per-row counters the
// reference's TpPlan reports as ExecStats (engine.cpp:92-195,
// engine_impl.hpp:96-186), schedule_to_json (scheduler.cpp:406-445) and the
// emit_text listing of a subkernel's op stream (kernelgen.cpp:305-360).
//
// The GPU kernels do not execute this plan — they stage per unit (problem.hpp)
// and move each input word once — but the counters are part of the drop-in
// contract (test_engine.cpp:350-363 asserts forward ExecStats == traffic x
// rows), and the JSON / listing dumps let the reference's compile / verify
// workflow inspect a plan built here.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "problem.hpp"

namespace cgf {

enum class Space : std::uint8_t { X, Y, W, Z };
enum class Strategy : std::uint8_t { SinglePhase, StreamZ, Greedy };

// A stageable word range (rows == 1) or strided weight tile.
struct SchedResource {
  Space space = Space::X;
  std::uint32_t offset = 0, rows = 1, cols = 0, row_stride = 0;
  std::uint32_t words() const { return rows * cols; }
};

struct SchedPhase {
  std::vector<std::uint32_t> resident, loaded, retained, z_flush, instructions;
};

struct ScheduleModel {
  Strategy strategy = Strategy::SinglePhase;
  std::uint32_t budget = 4096;
  std::vector<SchedResource> resources;  // ids in first-use order
  std::vector<SchedPhase> phases;
  std::vector<std::uint32_t> order;      // position -> split index (Sub::split_index)
  // per-row counters (words / flops)
  std::uint64_t fwd_loads = 0, fwd_stores = 0, fwd_flops = 0;  // = traffic_report
  std::uint64_t bwd_loads = 0, bwd_flops = 0;                  // backward ExecStats (no stores)
};

struct BudgetError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Throws BudgetError when a subkernel's working set exceeds the budget or the
// greedy planner cannot place an instruction (the reference's messages).
ScheduleModel build_schedule_model(const Problem& p, std::uint32_t budget);

// schedule_to_json's document (same keys and values; 2-space indent).
std::string schedule_json(const Problem& p, const ScheduleModel& s);

// emit_text of gen_forward / gen_backward for one split subkernel.
std::string listing_text(const Sub& s, bool backward);

}  // namespace cgf
