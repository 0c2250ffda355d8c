// Tensor-core (tcgen05, kind::tf32, 3xTF32) path for uvw (kind C) problems
// with one weight set shared by every row — the e3nn FullyConnectedTP shape
// of config C3. The sparse CG contraction stays on the SIMT pipes; the dense
// W contraction, which dominates the flops, runs on the 5th-gen tensor cores.
//
// Forward, per 128-row tile and output z segment s (all instructions p that
// write s accumulate into one TMEM accumulator):
//   A_{p,k}[row, c]  = sum_{(i,j,k) in CG_p} v * x[row][p.x][c][i] * y[row][p.y][j]   (SIMT, smem)
//   D_{s,k}[row, r] += sum_c A_{p,k}[row, c] * W_p[r][c]                             (tcgen05.mma)
//   z[row][s][r][k]  = D_{s,k}[row, r]                                               (TMEM -> HBM)
// which is the reference's C-kind forward (kernelgen.cpp:611-623: out[r][s] =
// sum_c W[r,c] z'[c][s]) with the multiplicity split undone: the reference
// splits b, b' into 32-lane chunks only because its interpreter is lane-bound.
#pragma once

#include <string>

#include "codegen.hpp"
#include "problem.hpp"

namespace cgf {

// True when every instruction is kind C with b % 16 == 0, b <= 256,
// b' % 16 == 0, 16-aligned x segments and each z segment's accumulator (dz * b columns) fits TMEM.
bool uvw_eligible(const Problem& p, std::string* why = nullptr);

struct UvwSource {
  KernelSource main;      // cgf_uvw_fwd_f32
  KernelSource prep;      // cgf_uvw_prep_f32: W -> swizzled hi / lo tf32 images
  std::size_t wimg_bytes = 0;
  int tile_rows = 128;
  int dims_x = 0;
  int prep_rows = 32;  // batch rows per block of the prep kernel (the gz planes pre-pass)
};

UvwSource generate_uvw_forward(const Problem& p);
// gx of the backward as the forward of the transposed problem (x <-> gz).
UvwSource generate_uvw_backward_x(const Problem& p);
// dL/dy of the backward (shared W).
UvwSource generate_uvw_backward_y(const Problem& p);
// Shared dL/dW for instructions [first, first + count), count <= 6: per-CTA
// partials; `prep` is the fixed-order reduction over CTAs.
UvwSource generate_uvw_backward_w(const Problem& p, int first, int count);

}  // namespace cgf
