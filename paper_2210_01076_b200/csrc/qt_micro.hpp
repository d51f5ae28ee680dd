// qt_micro.hpp -- lowering of a planned pass into the lean kernel's
// micro-op stream (host).
//
// The round compiler (qt_plan.cpp compile_round) emits fused LAYER ops; the
// lean tile kernel does not decode them: each layer becomes a short run of
// layer words (qt_ir.hpp): one 8-byte word per layer whose flag bits select
// compiled bodies -- [table][signs][one rotation / 2x2 per slot].
//
// Diagonal tables of unit phases are re-expressed as plane rotations of each
// amplitude's (re, im): e^{i phi} as three shears (3 FP64 ops per amplitude
// instead of a complex multiply's 4). Shears stay well-conditioned while
// |phi| stays away from pi, so every table is first multiplied by a common
// phase e^{-i gamma} that centres its 2^R angles (largest circular gap
// opposite): |phi| <= pi - pi/2^R. The removed scalars commute with
// everything; their product is carried through the plan and folded into the
// plan's last table (kept as complex multiplies), so every launch sequence
// leaves the exact state.
#pragma once

#include <cstdint>
#include <vector>

#include "qt_ir.hpp"

namespace qtb {

struct MicroPass {
  std::vector<uint32_t> words;        // layer words as (x, y) pairs
  std::vector<double> pool;           // 16-B aligned entries (even offsets)
  std::vector<uint16_t> round_first;  // per round: first micro-op
  std::vector<uint16_t> round_count;  // per round: micro-op count
  bool ok = false;                    // lowered (lean passes only)
  size_t size() const { return words.size() / 2; }
};

// True when every device op of the pass is a plain fused layer or an X / CX
// register permutation without diagonal flags (the lean kernel's op set).
bool pass_is_lean(const PlanPass& ps);

// Lowers every lean tile pass of the plan (others: ok = false). The table
// phases removed for conditioning are folded into the plan's last table.
// Passes whose lowering exceeds the limits (one launch's micro-op / pool /
// round capacity) are left to the generic kernel.
struct MicroLimits {
  size_t ops, pool, rounds;
};
std::vector<MicroPass> lower_plan_micro(const Plan& plan, int reg_bits, const MicroLimits& lim);

// FP64-pipe instructions per amplitude of a lowered pass (roofline
// accounting): shear table 3 per non-identity entry / 2^R, complex table 4,
// rotation 2 (scaled form), complex 2x2 8 (per amplitude of the slot pairs).
double micro_fp64_per_amp(const MicroPass& mp, int reg_bits);

}  // namespace qtb
