// Problem descriptors: irreps, real-basis CG blocks, instruction validation,
// multiplicity splitting and the GPU work-unit plan.
//
// Mirrors the reference's descriptor API (include/cgforge/{irreps,cg,tpspec}.hpp):
// the same parsing rules, validation rules, weight layout and CG convention, so
// a problem JSON means the same thing to both. The unit plan at the bottom is
// the B200-side static scheduler (replaces scheduler::build_schedule's
// scratch-budget phases, scheduler.cpp:139-389).
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace cgf {

// ----------------------------------------------------------------- errors --
// One exception type per reference exception; the C ABI maps each to a code.
struct ParseError : std::runtime_error {       // irreps::ParseError, json errors
  using std::runtime_error::runtime_error;
};
struct ValidationError : std::runtime_error {  // tpspec::validate violations
  using std::runtime_error::runtime_error;
};
struct ShapeError : std::invalid_argument {    // engine::ShapeError
  using std::invalid_argument::invalid_argument;
};
struct TriangleError : std::invalid_argument {  // cg::TriangleError
  using std::invalid_argument::invalid_argument;
};
struct UnsupportedError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Sets cgf_last_error()'s message on this thread (capi.cpp).
void set_last_error(const std::string& msg);

// ----------------------------------------------------------------- irreps --
struct MulIrrep {
  int mult = 1;
  int l = 0;
  bool odd = false;
  int dim() const { return mult * (2 * l + 1); }
};

struct Irreps {
  std::vector<MulIrrep> blocks;
  int dim() const;
  int offset(int seg) const;  // seg == size() gives dim()
  std::string str() const;
};

// `<mult>x<l><e|o>` joined by '+', textual order, no merging (irreps.cpp:60-122).
Irreps parse_irreps(const std::string& text);

// --------------------------------------------------------------------- CG --
struct CGEntry {
  int i, j, k;
  double v;
};
struct CGBlock {
  int l1, l2, l3;
  std::vector<CGEntry> entries;  // sorted (k, i, j)
};
// Same convention as cg::cg_block (cg.cpp:58-134): Racah sum, real basis on
// all three modes, global phase fix, drop |v| <= 1e-12, unit norm per k.
std::shared_ptr<const CGBlock> cg_block(int l1, int l2, int l3);

// ----------------------------------------------------------------- tpspec --
enum class Kind : std::uint8_t { B, C };  // B = uvu (diagonal W), C = uvw (dense W)

struct Instruction {
  int x_seg = 1, y_seg = 1, z_seg = 1;  // 1-based
  Kind kind = Kind::B;
};

// One (possibly split) subkernel with resolved offsets (tpspec.hpp:39-60).
struct Sub {
  Kind kind = Kind::B;
  int l1 = 0, l2 = 0, l3 = 0;
  int b = 0, bp = 0;  // z-side rows, x-side lanes
  std::uint32_t x_off = 0, y_off = 0, z_off = 0, w_off = 0, w_stride = 1;
  int origin = 0;       // user instruction index
  int split_index = 0;  // position in the split (pre-schedule) order
  std::shared_ptr<const CGBlock> cg;
  int dx() const { return 2 * l1 + 1; }
  int dy() const { return 2 * l2 + 1; }
  int dz() const { return 2 * l3 + 1; }
  std::uint64_t fwd_flops() const;  // kernelgen::flop_count(gen_forward) rule
  std::uint64_t bwd_flops() const;  // kernelgen::flop_count(gen_backward) rule
};

struct Problem {
  Irreps x_ir, y_ir, z_ir;
  std::vector<Instruction> instructions;
  std::vector<Sub> resolved;  // one per instruction (unsplit)
  std::vector<Sub> subs;      // split to <= lane_width, schedule order
  int dim_x = 0, dim_y = 0, dim_z = 0;
  std::uint32_t n_w = 0;
  int lane_width = 32;

  std::uint64_t fwd_flops_per_row() const;
  std::uint64_t bwd_flops_per_row() const;
};

// validate (tpspec.cpp:8-99) + split_multiplicities (scheduler.cpp:32-81) +
// normalised order (stable sort by z offset, scheduler.cpp:146-151).
// Throws ValidationError listing every violation.
Problem make_problem(const Irreps& x, const Irreps& y, const Irreps& z,
                     const std::vector<Instruction>& ins, int lane_width = 32);
// Problem JSON schema of tpspec::parse_problem_json (tpspec.cpp:105-130).
Problem parse_problem_json(const std::string& text, int lane_width = 32);

// --------------------------------------------------------- unit planning --
// A unit is the smallest set of subkernels that owns its outputs: every
// subkernel sharing an x chunk (owner of gx / dx) or a z piece (owner of z /
// dgz) lands in the same unit. One warp runs a row's units back to back; each
// unit's inputs are staged into one shared-memory slot.
struct Piece {
  std::uint32_t off;    // word offset within the row
  std::uint32_t words;  // contiguous words
};
struct Unit {
  std::vector<int> subs;        // indices into Problem::subs, schedule order
  std::vector<Piece> x_chunks;  // distinct x chunks read (and gx / dx written)
  std::vector<Piece> z_pieces;  // distinct z pieces written (gz / dgz read)
  int merged = 1;               // same-shape chunks folded in (subs = merged groups of equal length)
  int x_chunk_of(const Sub& s) const;
  int z_piece_of(const Sub& s) const;
};
std::vector<Unit> plan_units(const Problem& p);

}  // namespace cgf
