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
  // single ops (data: one 2x2 matrix, 8 doubles, in the pass pool)
  D_DENSE = 0,   // 2x2 complex on reg slot a                  (8 DFMA/amp)
  D_REAL = 1,    // 2x2 real on reg slot a                     (4 DFMA/amp)
  D_DIAG = 2,    // diag(d0, d1) on a bit anywhere             (4 DFMA/amp)
  D_SIGN = 3,    // multiply by -1 where bit set (Z, CZ)       (integer ops)
  D_XPERM = 4,   // plain swap of the pair on reg slot a (X, CX)
  D_ANTI = 5,    // scaled swap [[0,m01],[m10,0]] on slot a    (4 DFMA/amp)
  D_SWAP2 = 6,   // swap qubits on reg slots a and b
  D_PHASE1 = 7,  // multiply by d1 where bit set (S, T, phase) (4 DFMA/amp)
  // the fused LAYER op built by the round compiler (qt_plan.cpp): [diag table
  // if kOpTable][sign terms: base mask dl, arg >> 16 conditional terms][a
  // real rotation (2 doubles: three-shear form) on every reg slot in mask a]
  // [a complex 2x2 (8 doubles) on every reg slot in lmask], ascending slots.
  // A lone diagonal table or sign op is a layer with empty masks.
  D_LAYER = 9,
  // (8, 10, 11: retired op types, kept unused so ids stay stable)
};

// ---------------------------------------------------------------------------
// Lean layer words: the lean kernel's instruction stream (qt_micro.cpp
// lowers the D_LAYER / D_XPERM ops of a pass into them). One uint2 per layer:
//   x = pool offset (doubles, even) | rotation slots << 16 | 2x2 slots << 20
//       | flags | tile-uniform sign terms << 28 | M_LAST
//   y = unconditional sign-slot mask | conditional sign terms << 16 (M_SIGN),
//       or the D_XPERM header (M_PERM)
// Pool data of a layer, in order: [nv tile-uniform sign terms (global-bit
// condition, slot mask: 2 words each)][diagonal table of 2^R entries]
// [sign terms (2 words each)]
// [scaled rotation (t, 0) or (u, 1) per rotation slot: qt_micro.cpp
// push_rotation][8 doubles per 2x2 slot].
// Tile-uniform sign terms (condition on global bits only) negate the
// table's output slots with one uniform test per term instead of flipping signs
// per amplitude.
// ---------------------------------------------------------------------------
constexpr uint32_t M_ROT_SHIFT = 16;     // rotation slot mask (4 bits)
constexpr uint32_t M_DENSE_SHIFT = 20;   // complex 2x2 slot mask (4 bits)
constexpr uint32_t M_STAB = 1u << 24;    // table of unit phases as shears (a, b)
constexpr uint32_t M_CTAB = 1u << 25;    // table as complex multiplies (re, im)
constexpr uint32_t M_SIGN = 1u << 26;    // sign flips (mask / terms in y)
constexpr uint32_t M_PERM = 1u << 27;    // X / CX register permutation
constexpr uint32_t M_NV_SHIFT = 28;      // tile-uniform sign terms of the table (2 bits)
constexpr uint32_t M_LAST = 1u << 30;    // the round's last word (every round has one)
// A lone diagonal gate the round compiler could not merge into a table (its
// target or a control is a non-register tile bit or a global bit): per slot s
// in the slot mask, multiply by d1 where the target bit is set, else d0.
//   y = slot mask (16 bits) | (target slot + 1) << 16 (0: thread / tile bit)
//       | M_TD_PHASE1 (d0 == 1: only set bits change)
//   pool: [lmask (tile-local control bits), dl (tile-local target bit),
//          gmask (global control bits), dg (global target bit), d0, d1]
constexpr uint32_t M_TDIAG = 1u << 31;
constexpr uint32_t M_TD_PHASE1 = 1u << 24;
constexpr int kMaxTableVariantTerms = 3;

// Variant id of a device op: the kernel dispatches on it to a fully
// specialised code path (register slots known at compile time, no per-slot
// predication). cs / ds are -1 when the control / diagonal target is not a
// register bit of the round; SWAP2 stores its second slot in ds; D_LAYER
// stores its rotation-slot mask in a.
constexpr uint32_t vid(uint32_t type, int a, int cs, int ds) {
  return (type << 10) | (uint32_t(a) << 6) | (uint32_t(cs + 1) << 3) | uint32_t(ds + 1);
}

// Header word of a device op: variant id in the low 14 bits, flags above.
constexpr uint32_t kOpVariantMask = 0x3fff;
constexpr uint32_t kOpLctl = 1u << 16;  // lmask != 0
constexpr uint32_t kOpGctl = 1u << 17;  // gmask != 0
constexpr uint32_t kOpDl = 1u << 18;    // dl != 0
constexpr uint32_t kOpDg = 1u << 19;    // dg != 0
constexpr uint32_t kOpFlagMask = kOpLctl | kOpGctl | kOpDl | kOpDg;
// dense dispatch index of the variant (tools/gen_variants.py) in bits 20..27
constexpr uint32_t kOpIndexShift = 20;
constexpr uint32_t kOpTable = 1u << 28;  // D_LAYER: a 2^R-entry table leads the pool data

// 32 bytes; lives in the kernel-parameter constant bank (read uniformly).
// Matrices / tables / sign terms are in the pass's double pool at `arg`.
struct alignas(8) DOp {
  uint32_t hdr;      // vid(type, a, cs, ds) | flags
  uint32_t arg;      // pool offset (doubles); D_LAYER: offset | nterms << 16
  uint32_t lmask;    // control bits among the round's NON-register tile bits
  uint32_t dl;       // diag target among non-register tile bits (mask) or 0
  uint64_t gmask;    // control bits outside the tile (global index bits)
  uint64_t dg;       // diag target outside the tile (mask) or 0
};
static_assert(sizeof(DOp) == 32, "DOp layout");

// One sign term of a D_LAYER op (two pool words): negate the register slots
// in `slots` when (j & lcond) == lcond and (g & gcond) == gcond.
struct SignTerm {
  uint32_t slots;    // bit s set: slot s is negated
  uint32_t lcond;    // non-register tile bits that must be 1
  uint64_t gcond;    // global bits that must be 1
};

constexpr int kMaxTileBits = 13;  // 2^13 x 16 B = 128 KiB of smem
constexpr int kMaxRegBits = 4;
// Defaults (overridable per state; QTB_TILE_BITS / QTB_REG_BITS for sweeps):
// 2^10-amplitude tiles (16 KiB smem), 3 register bits -> 128 threads of 8
// amplitudes, <= 64 registers, 8 CTAs (32 warps) per SM -- measured best on
// C3 on B200 (the pass is latency-bound, so resident warps win over R = 4).
constexpr int kDefaultTileBits = 10;
constexpr int kDefaultRegBits = 3;
// compiled passes (qt_jit.cpp): R = 4, 2^12-amplitude tiles whose lowest 4
// physical bits are always in the tile (256-B runs) -- measured best on C3
// (221 ms vs 226 ms with 128-B runs); hybrid mode (the incremental engine)
// keeps 128-B runs (tuned on C5)
constexpr int kJitTileBits = 12;
constexpr int kJitRegBits = 4;
constexpr int kJitLowBits = 4;
constexpr int kHybridLowBits = 3;
// hybrid passes: R = 3 -- compiled the R = 4 ring kernel is faster (C5 at
// 28 q: 2.16 vs 2.36 ms per pass), but the misses run the interpreter, whose
// R = 4 variant is slower (5.5 vs 4.7 ms): measured on C5's modifiers, R = 3
// keeps the last-10% class faster and the uniform class unchanged
constexpr int kHybridRegBits = 3;
constexpr int kJitDirectBits = 3;
// hybrid compiled passes (incremental engine) from this many local qubits up
constexpr int kHybridMinQubits = 20;

struct DRound {
  uint16_t op_first;  // into the pass's op array
  uint16_t op_count;
  uint8_t reg[kMaxRegBits];   // tile-bit indices of the register bits (slot order)
  uint8_t sreg[kMaxRegBits];  // the same bits ascending (thread-index deposit)
  uint32_t sbit[kMaxRegBits]; // swz(1 << reg[i]) * 16: smem byte-offset term of slot bit i
};
static_assert(sizeof(DRound) == 28, "DRound layout");

// Host copy of the device smem swizzle (qt_device.cuh swz): GF(2)-linear.
constexpr uint32_t swz_host(uint32_t j) {
  return j ^ ((j >> 3) & 7u) ^ ((j >> 6) & 7u) ^ ((j >> 9) & 7u) ^ ((j >> 12) & 7u);
}

// Per-launch capacity of the kernel-parameter block (<= 32764 bytes): a
// pass with more ops / rounds / pool is split by the planner.
constexpr int kSmallOps = 32, kSmallRounds = 16, kSmallPool = 320;
constexpr int kLargeOps = 256, kLargeRounds = 96, kLargePool = 2560;

// A device-encoded round (host side): its ops and their pool data.
struct EncRound {
  std::vector<DOp> ops;
  std::vector<double> pool;  // offsets in ops are relative to this vector
};

// ---------------------------------------------------------------------------
// Host plan
// ---------------------------------------------------------------------------

struct PlanRound {
  std::vector<int> reg;          // tile-bit indices
  std::vector<int> ops;          // indices into the pass op list (LOp order)
  EncRound enc;                  // device encoding (compile_round)
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
