// Shared by the drop-in shims (engine_b200.cpp, conv_b200.cpp): the private
// state behind cgforge::engine::TpPlan (engine.hpp forward-declares
// detail::PlanImpl) — the reference's problem and schedule, kept for
// problem() / schedule() and the traffic model, plus the GPU plan handle.
#pragma once

#include <type_traits>

#include "cgf.h"
#include "cgforge/engine.hpp"

namespace cgforge::engine {

namespace detail {
struct PlanImpl {
  tpspec::ValidatedProblem problem;
  scheduler::Schedule schedule;
  cgf_plan* gpu = nullptr;
  PlanImpl() = default;
  PlanImpl(const PlanImpl&) = delete;
  PlanImpl& operator=(const PlanImpl&) = delete;
  ~PlanImpl() {
    if (gpu) cgf_plan_destroy(gpu);
  }
};
}  // namespace detail

namespace b200 {
// C ABI status -> the reference's exception types.
[[noreturn]] void rethrow(int rc);
inline void check(int rc) {
  if (rc != CGF_OK) rethrow(rc);
}
template <typename T>
constexpr int dtype() {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "float or double");
  return std::is_same_v<T, float> ? CGF_F32 : CGF_F64;
}
}  // namespace b200

}  // namespace cgforge::engine
