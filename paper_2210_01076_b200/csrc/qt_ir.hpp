// qt_ir.hpp -- intermediate representation shared by the host planner and
// the sm_100a kernels.
//
//   qt_gate (C ABI, reference GateKind)  --lower-->  LOp (logical ops)
//   LOp list  --fuse + plan-->  Plan = passes of rounds of DOp (device ops)
//
// Reference counterparts: the gate database (gate.cpp:42-106) and the
// element-op forms (element_ops.cpp:24-133) become LOp kinds; the stage
// planner (plan.cpp:100-163, chunk/form partitions plan.cpp:26-89) becomes
// the pass/round planner in qt_plan.cpp.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace qtb {

// ---------------------------------------------------------------------------
// Logical ops (host)
// ---------------------------------------------------------------------------

struct cplx {
  double re = 0.0, im = 0.0;
};

inline cplx cmul(cplx a, cplx b) {
  return cplx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
inline cplx cadd(cplx a, cplx b) { return cplx{a.re + b.re, a.im + b.im}; }

enum class LKind : uint8_t {
  Dense,  // general 2x2 on target
  Diag,   // diag(m00, m11) on target (target has a Z role)
  Anti,   // [[0, m01], [m10, 0]] on target (scaled bit flip)
  Swap,   // exchange qubits target and target2
};

// One logical op: an (optionally singly-controlled) 2x2 or a SWAP.
// Control semantics: the op acts where bit `control` == 1.
struct LOp {
  LKind kind = LKind::Dense;
  int target = 0;
  int target2 = -1;  // Swap only
  int control = -1;
  cplx m[4];         // row-major 2x2
  uint32_t gate = 0; // index of the originating gate (for plan audit)
};

// ---------------------------------------------------------------------------
// Device ops (host-built, consumed by the kernels)
// ---------------------------------------------------------------------------

enum DType : uint32_t {
  D_DENSE = 0,   // 2x2 complex on reg slot a                  (8 DFMA/amp)
  D_REAL = 1,    // 2x2 real on reg slot a                     (4 DFMA/amp)
  D_DIAG = 2,    // diag(d0, d1) on a bit anywhere             (4 DFMA/amp)
  D_SIGN = 3,    // multiply by -1 where bit set (Z, CZ)       (integer ops)
  D_XPERM = 4,   // plain swap of the pair on reg slot a (X, CX)
  D_ANTI = 5,    // scaled swap [[0,m01],[m10,0]] on slot a    (4 DFMA/amp)
  D_SWAP2 = 6,   // swap qubits on reg slots a and b
  D_PHASE1 = 7,  // multiply by d1 where bit set (S, T, phase) (4 DFMA/amp)
};

// Variant id of a device op: the kernel dispatches on it to a fully
// specialised code path (register slots known at compile time, no per-slot
// predication). cs / ds are -1 when the control / diagonal target is not a
// register bit of the round; SWAP2 stores its second slot in ds.
constexpr uint32_t vid(uint32_t type, int a, int cs, int ds) {
  return (type << 9) | (uint32_t(a) << 6) | (uint32_t(cs + 1) << 3) | uint32_t(ds + 1);
}

// 96 bytes; lives in the kernel-parameter constant bank (read uniformly).
struct alignas(16) DOp {
  uint32_t variant;  // vid(type, a, cs, ds)
  uint32_t lmask;    // control bits among the round's NON-register tile bits
  uint32_t dl;       // diag target among non-register tile bits (mask) or 0
  uint32_t pad;
  uint64_t gmask;    // control bits outside the tile (global index bits)
  uint64_t dg;       // diag target outside the tile (mask) or 0
  double m[8];       // interleaved row-major 2x2 (diag: m[0..1]=d0, m[6..7]=d1)
};
static_assert(sizeof(DOp) == 96, "DOp layout");

constexpr int kMaxTileBits = 13;  // 2^13 x 16 B = 128 KiB of smem
constexpr int kMaxRegBits = 4;

struct DRound {
  uint16_t op_first;  // into the pass's op array
  uint16_t op_count;
  uint8_t reg[kMaxRegBits];  // tile-bit indices of the register bits
};
static_assert(sizeof(DRound) == 8, "DRound layout");

// Per-launch capacity of the kernel-parameter block (<= 32764 bytes): a
// pass with more ops / rounds is split by the planner.
constexpr int kSmallOps = 32, kSmallRounds = 16;
constexpr int kLargeOps = 288, kLargeRounds = 96;

// ---------------------------------------------------------------------------
// Host plan
// ---------------------------------------------------------------------------

struct PlanRound {
  std::vector<int> reg;          // tile-bit indices
  std::vector<int> ops;          // indices into the pass op list (LOp order)
};

struct PlanPass {
  enum Kind { Tile, Exchange } kind = Tile;
  std::vector<int> tile_phys;    // physical bits of tile bits (low first)
  std::vector<LOp> ops;          // physical-qubit ops, in application order
  std::vector<PlanRound> rounds;
  // Exchange: swap physical global bits with local bits
  std::vector<std::pair<int, int>> exchange;  // (global phys bit, local phys bit)
};

struct Plan {
  int nqubits = 0;
  int nlocal = 0;                // physical bits held per shard
  std::vector<PlanPass> passes;
  std::vector<int> perm_before;  // logical -> physical at plan start
  std::vector<int> perm_after;   // logical -> physical at plan end
  size_t gates = 0;
};

}  // namespace qtb
