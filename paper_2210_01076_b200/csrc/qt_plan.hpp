// qt_plan.hpp -- fusion and pass planning (host).
#pragma once

#include <string>
#include <vector>

#include "qt_ir.hpp"

namespace qtb {

struct PlanOptions {
  int tile_bits = kDefaultTileBits;  // qubits per shared-memory tile
  int low_bits = 4;    // lowest physical bits always in the tile (coalescing)
  int reg_bits = kDefaultRegBits;    // qubits per register round (2^R amps/thread)
  int lookahead = 4096;// ops scanned per pass
  bool fuse_layers = true;  // round compiler: MULTI / diagonal-table layers
  int max_round_ops = 48;   // logical ops per register round (param space)
  // register-set search per round (qt_plan.cpp make_rounds) from this many
  // local qubits up: it costs host time per round and pays off only where a
  // pass streams enough amplitudes (small states are launch/host-bound)
  int round_search_min_bits = 22;
  // estimated FP64 ops per amplitude a tile pass may carry (0 = no cap): a
  // non-diagonal op counts ~3 (scaled rotation + its share of a table).
  // Balances FP64-heavy passes against HBM-bound ones (QTB_PASS_FP64).
  double max_pass_fp64 = 0.0;
  // per pass, also try tiles seeded with every window of consecutive
  // physical bits and keep the fill with the most FP64 work (QTB_WINDOW_SEARCH)
  bool window_search = false;
  // > 1: beam search over the window choice of every pass (QTB_WINDOW_BEAM)
  int window_beam = 0;
  // tile shrinking (0 = off): a pass's tile drops the reserved low bits in
  // [shrink_run_bits, low_bits) that none of its ops needs as an X-role bit,
  // down to shrink_min_bits tile bits (QTB_SHRINK_MIN / QTB_SHRINK_RUN)
  int shrink_min_bits = 0;
  int shrink_run_bits = 2;
  // exchanges pick their local victim bits among the top victim_span local
  // bits (QTB_VICTIM_SPAN)
  int victim_span = 10;
};

// Cost model of the compiled-mode plan search (qt_state.cpp State::plan):
// FP64 pipe rate (DFMA/s, B200 probe at load clocks) and the ring kernel's
// measured streaming rate (B/s, tools/tilebits_bench.py: ~5.9 TB/s).
constexpr double kPlanFp64PerS = 1.67e13;
constexpr double kPlanHbmBytesPerS = 5.87e12;
constexpr double kPlanExposedHbm = 0.56;  // share of a pass's HBM time not hidden under its FP64 time
constexpr int kPlanSearchMinBits = 24;
constexpr size_t kPlanBeamMaxOps = 20000;  // fused ops; larger circuits keep the phase-1 plan
constexpr int kPlanBeamWidth = 16;  // window beam of the plan search's second phase

// Merges runs of uncontrolled single-qubit ops on the same qubit into one
// 2x2 (matrix product) and drops exact identities. Order-preserving:
// an op merges into the latest op touching its qubit only. Then pushes
// single-qubit diagonal factors forward into the next single-qubit op on
// their qubit (qt_plan.cpp push_phases).
void fuse_ops(std::vector<LOp>& ops, int nqubits);
// U = diag(p0, p1) . [[c, -s], [s, c]] . diag(1, q1) (qt_plan.cpp); false when
// c or s is ~0 (U diagonal or anti-diagonal).
bool zyz_split(const cplx* u, cplx& p0, cplx& p1, double& c, double& s, cplx& q1);

// Plans `ops` (logical qubits) for a state of nqubits bits of which the top
// nqubits - nlocal are sharded (global). perm maps logical -> physical and
// is updated by the exchanges the plan inserts.
Plan make_plan(const std::vector<LOp>& ops, int nqubits, int nlocal,
               const std::vector<int>& perm, const PlanOptions& opt);

// Device op for `op` (physical qubits) inside a pass whose tile holds the
// physical bits tile_phys and whose round uses register tile-bits reg.
void encode_single(const LOp& op, const std::vector<int>& tile_phys,
                   const std::vector<int>& reg, EncRound& out);

// Device encoding of one round (fuse: build MULTI / table / sign layers;
// otherwise one device op per logical op).
EncRound compile_round(const PlanPass& pass, const PlanRound& round, bool fuse);

// Kernel-side op type of an LOp.
uint32_t dtype_of(const LOp& op);

// detail=true adds every round's register bits and encoded device ops.
// fp64_lowered (optional, per pass, < 0 = none): FP64 ops per amplitude of
// the pass as lowered for the lean / compiled kernels (qt_micro.cpp), which
// then replaces the device-op accounting in "fp64_per_amp".
std::string plan_to_json(const Plan& p, bool detail = false,
                         const std::vector<double>* fp64_lowered = nullptr);

// FP64 pipe operations per amplitude of an op (roofline accounting).
double op_fp64_per_amp(const LOp& op);

}  // namespace qtb
