// Drop-in replacement for cgforge's src/engine.cpp: `cgforge::engine::TpPlan`
// (include/cgforge/engine.hpp, unchanged) computed by the B200 kernels
// through the C ABI in include/cgf.h. A maintainer links this file (and
// conv_b200.cpp) instead of src/engine.cpp / src/conv.cpp plus libcgf.so; the
// rest of cgforge (irreps, cg, tpspec, scheduler, oracle) is untouched.
// INTEGRATION.md has the recipe.
//
// Semantics kept from the reference:
//  * shape checks before any compute, same ShapeError messages (engine.cpp:206-220);
//  * outputs resized only when the size differs and fully overwritten
//    (ensure_zeroed, engine.cpp:270-274);
//  * ExecStats come from libcgf's own restatement of the reference's per-row
//    schedule model (cgf_tp_stats: forward = traffic_report x rows, the
//    counters test_engine.cpp:350-363 asserts; backward / double-backward the
//    reference's phase counters) -- nothing is read from the reference's
//    scheduler objects;
//  * results are bitwise independent of Options::workers and ExecMode (the GPU
//    kernels ignore both) and of DispatchStyle (one fused pass);
//  * C ABI codes are rethrown as the reference's exception types.
#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "cgforge/rng.hpp"
#include "plan_impl_b200.hpp"

namespace cgforge::engine {

namespace b200 {

void rethrow(int rc) {
  const std::string m = cgf_last_error();
  switch (rc) {
    case CGF_E_SHAPE: throw ShapeError(m);
    case CGF_E_PARSE: throw irreps::ParseError(m);
    case CGF_E_BUDGET: throw scheduler::BudgetError(m);
    case CGF_E_TRIANGLE: throw cg::TriangleError(m);
    case CGF_E_INVALID: throw std::invalid_argument(m);
    case CGF_E_INTERNAL: throw std::logic_error(m);
    default: throw std::runtime_error("cgf: " + m);
  }
}

}  // namespace b200

namespace {

template <typename T>
void require_size(const char* what, const std::vector<T>& v, std::int64_t rows, int cols) {
  const std::int64_t want = rows * cols;
  if (static_cast<std::int64_t>(v.size()) == want) return;
  throw ShapeError(std::string("shape mismatch for ") + what + ": expected " + std::to_string(rows) + "x" +
                   std::to_string(cols) + " = " + std::to_string(want) + " elements, got " +
                   std::to_string(v.size()));
}

template <typename T>
void require_batch(const tpspec::ValidatedProblem& p, const Batch<T>& in) {
  require_size("x", in.x, in.rows, p.dim_x);
  require_size("y", in.y, in.rows, p.dim_y);
  require_size("w", in.w, in.rows, static_cast<int>(p.total_weights));
}

template <typename T>
void sized(std::vector<T>& v, std::size_t n) {
  if (v.size() != n) v.assign(n, T(0));
}

ExecStats model_stats(const cgf_plan* g, int op, std::int64_t rows) {
  std::uint64_t s[3] = {0, 0, 0};
  b200::check(cgf_tp_stats(g, op, rows, 0, s));
  ExecStats st;
  st.loads_words = s[0];
  st.stores_words = s[1];
  st.flops = s[2];
  return st;
}

}  // namespace

TpPlan::TpPlan(const tpspec::ValidatedProblem& p, const scheduler::Schedule& s)
    : impl_(std::make_unique<detail::PlanImpl>()) {
  impl_->problem = p;
  impl_->schedule = s;
  // The GPU planner re-splits the ORIGINAL instructions (problem_to_json
  // writes those) at the lane width the caller split with: the largest chunk
  // of `p` (split_multiplicities(p, L) leaves chunks of min(L, mult)), so the
  // split -- and the schedule model under the same budget -- is the caller's.
  int lanes = 1;
  for (const auto& r : p.resolved) lanes = std::max({lanes, r.b, r.b_prime});
  const std::string js = tpspec::problem_to_json(p);
  b200::check(cgf_plan_create(js.c_str(), std::min(lanes, 32), s.budget_words, &impl_->gpu));
}

TpPlan::~TpPlan() = default;
TpPlan::TpPlan(TpPlan&&) noexcept = default;
TpPlan& TpPlan::operator=(TpPlan&&) noexcept = default;

const tpspec::ValidatedProblem& TpPlan::problem() const { return impl_->problem; }
const scheduler::Schedule& TpPlan::schedule() const { return impl_->schedule; }

template <typename T>
ExecStats TpPlan::forward(const Batch<T>& in, std::vector<T>& z, const Options&) const {
  const auto& p = impl_->problem;
  require_batch(p, in);
  sized(z, static_cast<std::size_t>(in.rows) * p.dim_z);
  if (in.rows > 0)
    b200::check(cgf_tp_forward_host(impl_->gpu, b200::dtype<T>(), in.x.data(), in.y.data(), in.w.data(), z.data(),
                                    in.rows, 0));
  return model_stats(impl_->gpu, CGF_OP_FORWARD, in.rows);
}

template <typename T>
ExecStats TpPlan::backward(const Batch<T>& in, const std::vector<T>& gz, Grads<T>& out, const Options&) const {
  const auto& p = impl_->problem;
  require_batch(p, in);
  require_size("g_z", gz, in.rows, p.dim_z);
  sized(out.x, in.x.size());
  sized(out.y, in.y.size());
  sized(out.w, in.w.size());
  if (in.rows > 0)
    b200::check(cgf_tp_backward_host(impl_->gpu, b200::dtype<T>(), in.x.data(), in.y.data(), in.w.data(), gz.data(),
                                     out.x.data(), out.y.data(), out.w.data(), in.rows, 0));
  return model_stats(impl_->gpu, CGF_OP_BACKWARD, in.rows);
}

template <typename T>
ExecStats TpPlan::double_backward(const Batch<T>& in, const std::vector<T>& gz, const Grads<T>& up,
                                  DoubleGrads<T>& out, DispatchStyle, const Options&) const {
  const auto& p = impl_->problem;
  require_batch(p, in);
  require_size("g_z", gz, in.rows, p.dim_z);
  require_size("dL/da", up.x, in.rows, p.dim_x);
  require_size("dL/db", up.y, in.rows, p.dim_y);
  require_size("dL/dC", up.w, in.rows, static_cast<int>(p.total_weights));
  sized(out.x, in.x.size());
  sized(out.y, in.y.size());
  sized(out.w, in.w.size());
  sized(out.gz, gz.size());
  if (in.rows > 0)
    b200::check(cgf_tp_double_backward_host(impl_->gpu, b200::dtype<T>(), in.x.data(), in.y.data(), in.w.data(),
                                            gz.data(), up.x.data(), up.y.data(), up.w.data(), out.x.data(),
                                            out.y.data(), out.w.data(), out.gz.data(), in.rows, 0));
  return model_stats(impl_->gpu, CGF_OP_DOUBLE_BACKWARD, in.rows);
}

// N(0, 1) rows drawn from one stream in the order x, y, w (engine.cpp:394-403).
template <typename T>
Batch<T> random_batch(const tpspec::ValidatedProblem& p, std::int64_t rows, std::uint64_t seed) {
  rng::NormalGen gen(seed);
  Batch<T> b;
  b.rows = rows;
  b.x = gen.normal_vec<T>(static_cast<std::size_t>(rows) * p.dim_x);
  b.y = gen.normal_vec<T>(static_cast<std::size_t>(rows) * p.dim_y);
  b.w = gen.normal_vec<T>(static_cast<std::size_t>(rows) * p.total_weights);
  return b;
}

template ExecStats TpPlan::forward<float>(const Batch<float>&, std::vector<float>&, const Options&) const;
template ExecStats TpPlan::forward<double>(const Batch<double>&, std::vector<double>&, const Options&) const;
template ExecStats TpPlan::backward<float>(const Batch<float>&, const std::vector<float>&, Grads<float>&,
                                           const Options&) const;
template ExecStats TpPlan::backward<double>(const Batch<double>&, const std::vector<double>&, Grads<double>&,
                                            const Options&) const;
template ExecStats TpPlan::double_backward<float>(const Batch<float>&, const std::vector<float>&,
                                                  const Grads<float>&, DoubleGrads<float>&, DispatchStyle,
                                                  const Options&) const;
template ExecStats TpPlan::double_backward<double>(const Batch<double>&, const std::vector<double>&,
                                                   const Grads<double>&, DoubleGrads<double>&, DispatchStyle,
                                                   const Options&) const;
template Batch<float> random_batch<float>(const tpspec::ValidatedProblem&, std::int64_t, std::uint64_t);
template Batch<double> random_batch<double>(const tpspec::ValidatedProblem&, std::int64_t, std::uint64_t);

}  // namespace cgforge::engine
