// qt_plan.cpp -- gate fusion and the fused-pass planner (host).
//
// Replaces the reference's per-net stage planner (plan.cpp:100-163), task
// chunking / partition forming (plan.cpp:26-89) and the per-update job DAG
// (engine.cpp:392-491). Where the reference materialises one stage per gate
// (one full read+write of the touched blocks per gate), the planner packs
// gates into PASSES: each pass streams the state through shared-memory
// tiles of 2^k amplitudes exactly once and applies every gate whose
// non-diagonal targets lie in the tile's qubit set. Inside a tile, gates are
// grouped into ROUNDS of R register qubits (each thread holds 2^R amplitudes
// in registers while the round's gates are applied).
//
// Legality: an op may be hoisted over earlier, not-yet-scheduled ops only if
// it commutes with them qubit by qubit: two ops commute on a shared qubit
// when both act diagonally there (diagonal targets, controls); see roles().
#include "qt_plan.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <unordered_map>

namespace qtb {

namespace {

enum Role : uint8_t { ZRole = 1, XRole = 2 };

struct QR {
  int q;
  Role r;
};

// Qubits an op touches with their roles (<= 3).
inline int roles(const LOp& op, QR* out) {
  int n = 0;
  switch (op.kind) {
    case LKind::Dense:
    case LKind::Anti:
      out[n++] = {op.target, XRole};
      break;
    case LKind::Diag:
      out[n++] = {op.target, ZRole};
      break;
    case LKind::Swap:
      out[n++] = {op.target, XRole};
      out[n++] = {op.target2, XRole};
      break;
  }
  if (op.control >= 0) out[n++] = {op.control, ZRole};
  return n;
}

inline bool is_one(cplx c) { return c.re == 1.0 && c.im == 0.0; }
inline bool is_zero(cplx c) { return c.re == 0.0 && c.im == 0.0; }

void reclassify(LOp& op) {
  const bool off0 = is_zero(op.m[1]) && is_zero(op.m[2]);
  const bool diag0 = is_zero(op.m[0]) && is_zero(op.m[3]);
  op.kind = off0 ? LKind::Diag : (diag0 ? LKind::Anti : LKind::Dense);
}

LOp to_phys(const LOp& op, const std::vector<int>& cur) {
  LOp p = op;
  p.target = cur[op.target];
  if (op.target2 >= 0) p.target2 = cur[op.target2];
  if (op.control >= 0) p.control = cur[op.control];
  return p;
}

}  // namespace

uint32_t dtype_of(const LOp& op) {
  switch (op.kind) {
    case LKind::Swap:
      return D_SWAP2;
    case LKind::Anti:
      if (is_one(op.m[1]) && is_one(op.m[2])) return D_XPERM;
      return D_ANTI;
    case LKind::Diag:
      if (is_one(op.m[0])) {
        if (op.m[3].re == -1.0 && op.m[3].im == 0.0) return D_SIGN;
        return D_PHASE1;
      }
      return D_DIAG;
    case LKind::Dense: {
      bool real = true;
      for (int k = 0; k < 4; ++k) real = real && op.m[k].im == 0.0;
      return real ? D_REAL : D_DENSE;
    }
  }
  return D_DENSE;
}

double op_fp64_per_amp(const LOp& op) {
  switch (dtype_of(op)) {
    case D_DENSE: return 8.0;
    case D_REAL: return 4.0;
    case D_DIAG: return 4.0;
    case D_PHASE1: return 4.0;
    case D_ANTI: return 4.0;
    default: return 0.0;
  }
}

namespace {

// min(|u00|, |u10|) for the diag . rotation . diag factorisation (QTB_ZYZ
// overrides, for sweeps; > 1 disables it). zyz_split is accurate for any
// c, s > 0, the threshold only keeps clear of zero / subnormal divisions.
double zyz_min() {
  static const double v = [] {
    const char* e = std::getenv("QTB_ZYZ");
    return e ? std::atof(e) : 1e-100;
  }();
  return v;
}

inline cplx conjc(cplx a) { return cplx{a.re, -a.im}; }

}  // namespace

// U = diag(p0, p1) . [[c, -s], [s, c]] . diag(1, q1) with c = |u00|,
// s = |u10| (u00 = p0 c, u01 = -p0 s q1, u10 = p1 s, u11 = p1 c q1).
// p0, p1 are the normalised first column; q1 is taken from the LARGER of
// u11 (c >= s: q1 = u11 conj(p1) / c) and u01 (c < s: q1 = -u01 conj(p0) / s),
// so every reconstructed entry is within O(eps) of U for a unitary U (the
// phase of a small column entry is ill-determined, but it only ever
// multiplies that small magnitude). False when c or s is below zyz_min().
bool zyz_split(const cplx* u, cplx& p0, cplx& p1, double& c, double& s, cplx& q1) {
  c = std::hypot(u[0].re, u[0].im);
  s = std::hypot(u[2].re, u[2].im);
  if (!(c > zyz_min() && s > zyz_min())) return false;
  p0 = cplx{u[0].re / c, u[0].im / c};
  p1 = cplx{u[2].re / s, u[2].im / s};
  if (c >= s) {
    const cplx t = cmul(u[3], conjc(p1));
    q1 = cplx{t.re / c, t.im / c};
  } else {
    const cplx t = cmul(u[1], conjc(p0));
    q1 = cplx{-t.re / s, -t.im / s};
  }
  return true;
}

namespace {

// Phase pushing (after fusion): single-qubit diagonal factors are carried
// forward on their qubit -- they commute with everything that acts on it
// diagonally (controls, CZ, other diagonals) -- and merged into the next
// single-qubit X-role op there:
//  * a dense U absorbs them (U' = U . D) and is split U' = diag(p0, p1) . V
//    with V = [[c, u01'/p0], [s, u11'/p1]], c = |u00'|, s = |u10'| real >= 0
//    (so the round compiler's ZYZ of V leaves no output phases); diag(p0, p1)
//    is carried on;
//  * an anti-diagonal op becomes a pure swap: [[0, a], [b, 0]] . D =
//    diag(a d1, b d0) . X;
//  * any other X-role use (a CX / controlled-U target, SWAP) and the end of
//    the list flush the carried factor as one diagonal op.
// So a layered circuit pays one diagonal table per rotation layer (the
// rotations' input phases) instead of an extra one at every round end.
void push_phases(std::vector<LOp>& ops, int nqubits) {
  std::vector<LOp> out;
  out.reserve(ops.size() + static_cast<size_t>(nqubits));
  std::vector<cplx> d0(nqubits, cplx{1.0, 0.0}), d1(nqubits, cplx{1.0, 0.0});
  std::vector<char> has(nqubits, 0);
  auto flush = [&](int q, uint32_t gate) {
    if (!has[q]) return;
    has[q] = 0;
    if (is_one(d0[q]) && is_one(d1[q])) return;
    LOp f;
    f.kind = LKind::Diag;
    f.target = q;
    f.m[0] = d0[q];
    f.m[1] = cplx{0.0, 0.0};
    f.m[2] = cplx{0.0, 0.0};
    f.m[3] = d1[q];
    f.gate = gate;
    out.push_back(f);
    d0[q] = d1[q] = cplx{1.0, 0.0};
  };
  for (const LOp& op : ops) {
    const int t = op.target;
    if (op.control < 0 && op.kind == LKind::Diag) {
      d0[t] = cmul(op.m[0], d0[t]);
      d1[t] = cmul(op.m[3], d1[t]);
      has[t] = 1;
      continue;
    }
    if (op.control < 0 && op.kind == LKind::Anti) {
      LOp x = op;
      const cplx a = cmul(op.m[1], d1[t]), b = cmul(op.m[2], d0[t]);
      x.m[1] = x.m[2] = cplx{1.0, 0.0};
      out.push_back(x);
      d0[t] = a;
      d1[t] = b;
      has[t] = 1;
      continue;
    }
    if (op.control < 0 && op.kind == LKind::Dense) {
      LOp u = op;
      u.m[0] = cmul(op.m[0], d0[t]);
      u.m[1] = cmul(op.m[1], d1[t]);
      u.m[2] = cmul(op.m[2], d0[t]);
      u.m[3] = cmul(op.m[3], d1[t]);
      cplx p0, p1, q1;
      double c, sn;
      if (zyz_split(u.m, p0, p1, c, sn, q1)) {
        // V = diag(p0, p1)^-1 U' = [[c, -s q1], [s, c q1]]
        u.m[0] = cplx{c, 0.0};
        u.m[1] = cplx{-sn * q1.re, -sn * q1.im};
        u.m[2] = cplx{sn, 0.0};
        u.m[3] = cplx{c * q1.re, c * q1.im};
        d0[t] = p0;
        d1[t] = p1;
        has[t] = 1;
      } else {
        d0[t] = d1[t] = cplx{1.0, 0.0};
        has[t] = 0;
      }
      reclassify(u);
      out.push_back(u);
      continue;
    }
    QR rl[3];
    const int nr = roles(op, rl);
    for (int k = 0; k < nr; ++k)
      if (rl[k].r == XRole) flush(rl[k].q, op.gate);
    out.push_back(op);
  }
  const uint32_t last = ops.empty() ? 0u : ops.back().gate;
  for (int q = 0; q < nqubits; ++q) flush(q, last);
  ops.swap(out);
}

}  // namespace

void fuse_ops(std::vector<LOp>& ops, int nqubits) {
  std::vector<LOp> out;
  out.reserve(ops.size());
  std::vector<int> last(nqubits, -1);  // index in out of the latest op on q
  std::vector<char> dead;
  dead.reserve(ops.size());
  for (const LOp& op : ops) {
    const bool single = op.kind != LKind::Swap && op.control < 0;
    if (single) {
      const int p = last[op.target];
      if (p >= 0 && !dead[p]) {
        LOp& prev = out[p];
        if (prev.kind != LKind::Swap && prev.control < 0 &&
            prev.target == op.target) {
          // apply prev first, then op: M = op.m * prev.m
          cplx r[4];
          r[0] = cadd(cmul(op.m[0], prev.m[0]), cmul(op.m[1], prev.m[2]));
          r[1] = cadd(cmul(op.m[0], prev.m[1]), cmul(op.m[1], prev.m[3]));
          r[2] = cadd(cmul(op.m[2], prev.m[0]), cmul(op.m[3], prev.m[2]));
          r[3] = cadd(cmul(op.m[2], prev.m[1]), cmul(op.m[3], prev.m[3]));
          for (int k = 0; k < 4; ++k) prev.m[k] = r[k];
          reclassify(prev);
          continue;
        }
      }
    }
    out.push_back(op);
    dead.push_back(0);
    const int idx = static_cast<int>(out.size()) - 1;
    last[op.target] = idx;
    if (op.target2 >= 0) last[op.target2] = idx;
    if (op.control >= 0) last[op.control] = idx;
  }
  // drop exact identities (e.g. RZ(0), merged X.X)
  std::vector<LOp> kept;
  kept.reserve(out.size());
  for (const LOp& op : out) {
    if (op.kind == LKind::Diag && is_one(op.m[0]) && is_one(op.m[3])) continue;
    kept.push_back(op);
  }
  ops.swap(kept);
  push_phases(ops, nqubits);
}

namespace {

// Placement of a physical qubit in a round: register slot, else tile bit,
// else outside the tile.
struct Place {
  const std::vector<int>& tile_phys;
  const std::vector<int>& reg;
  int tile(int phys) const {
    for (size_t i = 0; i < tile_phys.size(); ++i)
      if (tile_phys[i] == phys) return static_cast<int>(i);
    return -1;
  }
  int slot(int phys) const {
    const int ti = tile(phys);
    if (ti < 0) return -1;
    for (size_t i = 0; i < reg.size(); ++i)
      if (reg[i] == ti) return static_cast<int>(i);
    return -1;
  }
};

void push_matrix(std::vector<double>& pool, const cplx* m) {
  for (int k = 0; k < 4; ++k) {
    pool.push_back(m[k].re);
    pool.push_back(m[k].im);
  }
}

}  // namespace

void encode_single(const LOp& op, const std::vector<int>& tile_phys,
                   const std::vector<int>& reg, EncRound& out) {
  const Place pl{tile_phys, reg};
  DOp d{};
  const uint32_t type = dtype_of(op);
  int a = 0, cs = -1, ds = -1;
  if (op.kind == LKind::Diag) {
    ds = pl.slot(op.target);
    if (ds < 0) {
      const int ti = pl.tile(op.target);
      if (ti >= 0) d.dl = 1u << ti;  // thread-uniform bit
      else d.dg = 1ull << op.target; // tile-uniform bit
    }
  } else {
    a = pl.slot(op.target);
    if (a < 0) throw std::logic_error("op target is not a register bit of its round");
    if (op.kind == LKind::Swap) {
      int b = pl.slot(op.target2);
      if (b < 0) throw std::logic_error("swap target is not a register bit");
      if (a > b) std::swap(a, b);
      ds = b;  // SWAP2 carries its second slot in ds
    }
  }
  if (op.control >= 0) {
    cs = pl.slot(op.control);
    if (cs < 0) {
      const int ti = pl.tile(op.control);
      if (ti >= 0) d.lmask = 1u << ti;
      else d.gmask = 1ull << op.control;
    }
  }
  d.hdr = vid(type, a, cs, ds) | (d.lmask ? kOpLctl : 0u) | (d.gmask ? kOpGctl : 0u) |
          (d.dl ? kOpDl : 0u) | (d.dg ? kOpDg : 0u);
  d.arg = static_cast<uint32_t>(out.pool.size());
  push_matrix(out.pool, op.m);
  out.ops.push_back(d);
}

// ---------------------------------------------------------------------------
// Round compiler: turns a round's op sequence into fused LAYERS
//   [pre diagonal table][pre sign terms][one 2x2 per register slot]
// Dense single-qubit gates on distinct register slots commute, so each
// layer's MULTI op applies up to R of them in one dispatch. A well-conditioned
// complex 2x2 U is factored U = diag(p0,p1) . [[c,-s],[s,c]] . diag(1,q1)
// (ZYZ with the global phase folded in): the real rotation goes to the layer
// (4 FP64 ops per amplitude instead of 8) and the diagonals join the
// neighbouring tables, where every diagonal factor of the round (RZ, S, T,
// CZ, controlled phases on register slots) is merged into one per-slot
// multiply or one integer sign flip.
// ---------------------------------------------------------------------------
namespace {

struct LayerState {
  int R, NS;
  std::vector<cplx> pre, post;
  bool pre_used = false, post_used = false;
  std::vector<SignTerm> pre_signs, post_signs;
  uint32_t post_slots = 0;  // register slots the post factors depend on
  cplx M[kMaxRegBits][4];
  uint32_t mmask = 0;
  uint32_t cmask = 0;  // slots of mmask holding complex 2x2s (the rest: real)

  explicit LayerState(int r) : R(r), NS(1 << r), pre(1 << r), post(1 << r) {
    for (auto& c : pre) c = cplx{1.0, 0.0};
    for (auto& c : post) c = cplx{1.0, 0.0};
  }
};

bool table_trivial(const std::vector<cplx>& t) {
  for (const cplx& c : t)
    if (c.re != 1.0 || c.im != 0.0) return false;
  return true;
}

void emit_table(const std::vector<cplx>& t, EncRound& out) {
  if (table_trivial(t)) return;
  DOp d{};
  d.hdr = vid(D_LAYER, 0, -1, -1) | kOpTable;  // a layer with no 2x2s
  d.arg = static_cast<uint32_t>(out.pool.size());
  for (const cplx& c : t) {
    out.pool.push_back(c.re);
    out.pool.push_back(c.im);
  }
  out.ops.push_back(d);
}

// Sign terms: unconditional ones (slot patterns only) collapse into one base
// mask carried in the op itself (dl field); only thread/tile-conditional
// terms go to the pool.
void emit_signs(const std::vector<SignTerm>& terms, EncRound& out) {
  if (terms.empty()) return;
  uint32_t base = 0;
  std::vector<SignTerm> cond;
  for (const SignTerm& t : terms) {
    if (t.lcond == 0 && t.gcond == 0) base ^= t.slots;
    else cond.push_back(t);
  }
  if (base == 0 && cond.empty()) return;
  DOp d{};
  d.hdr = vid(D_LAYER, 0, -1, -1);  // a layer with no table and no 2x2s
  d.dl = base;
  const uint32_t off = static_cast<uint32_t>(out.pool.size());
  d.arg = off | (static_cast<uint32_t>(cond.size()) << 16);
  for (const SignTerm& t : cond) {
    const uint64_t w0 = static_cast<uint64_t>(t.slots) | (static_cast<uint64_t>(t.lcond) << 32);
    double dw0, dw1;
    std::memcpy(&dw0, &w0, 8);
    std::memcpy(&dw1, &t.gcond, 8);
    out.pool.push_back(dw0);
    out.pool.push_back(dw1);
  }
  out.ops.push_back(d);
}

// A table that is emitted anyway absorbs the unconditional sign terms
// (multiplying entries by -1 is free); conditional terms stay sign ops.
void fold_signs(std::vector<cplx>& table, std::vector<SignTerm>& terms) {
  if (table_trivial(table)) return;
  std::vector<SignTerm> rest;
  for (const SignTerm& t : terms) {
    if (t.lcond == 0 && t.gcond == 0) {
      for (size_t s = 0; s < table.size(); ++s)
        if ((t.slots >> s) & 1u) table[s] = cplx{-table[s].re, -table[s].im};
    } else {
      rest.push_back(t);
    }
  }
  terms.swap(rest);
}

// Emits a layer as ONE device op (kernel k_layer): the layer's pre table,
// its pre sign terms (unconditional ones as the base mask in dl, conditional
// ones in the pool) and one 2x2 per register slot in L.mmask: rotations on
// the real slots (mask in the variant's a field), then complex 2x2s on the
// others (mask in lmask).
void emit_layer(LayerState& L, EncRound& out) {
  DOp d{};
  const bool tab = !table_trivial(L.pre);
  uint32_t base = 0;
  std::vector<SignTerm> cond;
  for (const SignTerm& t : L.pre_signs) {
    if (t.lcond == 0 && t.gcond == 0) base ^= t.slots;
    else cond.push_back(t);
  }
  const uint32_t rmask = L.mmask & ~L.cmask;
  d.hdr = vid(D_LAYER, static_cast<int>(rmask), -1, -1) |
          (tab ? kOpTable : 0u);
  d.dl = base;
  d.arg = static_cast<uint32_t>(out.pool.size()) | (static_cast<uint32_t>(cond.size()) << 16);
  if (tab) {
    for (const cplx& c : L.pre) {
      out.pool.push_back(c.re);
      out.pool.push_back(c.im);
    }
  }
  for (const SignTerm& t : cond) {
    const uint64_t w0 = static_cast<uint64_t>(t.slots) | (static_cast<uint64_t>(t.lcond) << 32);
    double dw0, dw1;
    std::memcpy(&dw0, &w0, 8);
    std::memcpy(&dw1, &t.gcond, 8);
    out.pool.push_back(dw0);
    out.pool.push_back(dw1);
  }
  for (int i = 0; i < L.R; ++i) {
    if (!(L.mmask & (1u << i))) continue;
    // rotation [[c, -s], [s, c]] (c >= 0, to_rotations) as (c, s): the
    // generic kernel applies it as three in-place shears (pair_shear), the
    // lean layer words as a scaled two-FMA rotation (qt_micro.cpp)
    if (rmask & (1u << i)) {
      out.pool.push_back(L.M[i][0].re);
      out.pool.push_back(L.M[i][2].re);
    }
  }
  for (int i = 0; i < L.R; ++i)
    if (L.cmask & (1u << i)) push_matrix(out.pool, L.M[i]);
  d.lmask = L.cmask;  // layers: the complex-slot mask (no control bits)
  out.ops.push_back(d);
  L.mmask = 0;
  L.cmask = 0;
}

// Real slots are stored as rotations (2 doubles per slot, half the constant
// loads): a real orthogonal 2x2 is a rotation [[c,-s],[s,c]] or a reflection
// [[c,s],[s,-c]] = rotation . Z, whose Z joins the layer's (earlier-applied)
// sign terms. Anything else makes that slot complex.
void to_rotations(LayerState& L) {
  if (!L.mmask) return;
  for (int i = 0; i < L.R; ++i) {
    if (!(L.mmask & (1u << i)) || (L.cmask & (1u << i))) continue;
    const double m0 = L.M[i][0].re, m1 = L.M[i][1].re, m2 = L.M[i][2].re, m3 = L.M[i][3].re;
    bool rot = m0 == m3 && m1 == -m2;
    if (!rot && m0 == -m3 && m1 == m2) {
      SignTerm z{};
      for (int s = 0; s < L.NS; ++s)
        if ((s >> i) & 1) z.slots |= 1u << s;
      L.pre_signs.push_back(z);
      L.M[i][1] = cplx{-m2, 0.0};
      L.M[i][3] = cplx{m0, 0.0};
      rot = true;
    }
    if (!rot) {
      L.cmask |= 1u << i;
      continue;
    }
    if (L.M[i][0].re < 0.0) {
      // R(theta) = -R(theta - pi): keep |theta| <= pi/2 (shear factors <= 1);
      // the scalar -1 commutes with everything and joins the layer's signs
      for (int k = 0; k < 4; ++k) L.M[i][k] = cplx{-L.M[i][k].re, 0.0};
      SignTerm all{};
      all.slots = (L.NS >= 32) ? 0xffffffffu : ((1u << L.NS) - 1u);
      L.pre_signs.push_back(all);
    }
  }
}

// Emits the layer (pre part + 2x2s) as one op; the post part becomes the
// next layer's pre part.
void close_layer(LayerState& L, EncRound& out) {
  to_rotations(L);
  fold_signs(L.pre, L.pre_signs);
  if (L.mmask) {
    emit_layer(L, out);
  } else {
    emit_table(L.pre, out);
    emit_signs(L.pre_signs, out);
  }
  L.pre.swap(L.post);
  L.pre_signs.swap(L.post_signs);
  for (auto& c : L.post) c = cplx{1.0, 0.0};
  L.post_signs.clear();
  L.post_slots = 0;
}

void flush_all(LayerState& L, EncRound& out) {
  close_layer(L, out);
  fold_signs(L.pre, L.pre_signs);
  emit_table(L.pre, out);
  emit_signs(L.pre_signs, out);
  for (auto& c : L.pre) c = cplx{1.0, 0.0};
  L.pre_signs.clear();
}

inline bool bit_of(int s, int slot) { return slot >= 0 && ((s >> slot) & 1); }

#include "qt_variant_ids.inc"

// Stores each op's dense dispatch index (the kernel's switch key).
void set_dispatch_index(EncRound& out, int R) {
  for (DOp& d : out.ops) {
    const uint32_t type = (d.hdr & kOpVariantMask) >> 10;
    if (type == D_LAYER || type == D_XPERM) continue;  // k_layer / k_perm
    const uint16_t idx = variant_index(R, d.hdr & kOpVariantMask);
    if (idx == 0xffff) throw std::logic_error("device op without a kernel variant");
    d.hdr = (d.hdr & ~(0xffu << kOpIndexShift)) | (static_cast<uint32_t>(idx) << kOpIndexShift);
  }
}

}  // namespace

EncRound compile_round(const PlanPass& pass, const PlanRound& round, bool fuse) {
  EncRound out;
  const int R = static_cast<int>(round.reg.size());
  const Place pl{pass.tile_phys, round.reg};
  if (!fuse) {
    for (int idx : round.ops) encode_single(pass.ops[idx], pass.tile_phys, round.reg, out);
    set_dispatch_index(out, R);
    return out;
  }
  LayerState L(R);
  for (int idx : round.ops) {
    const LOp& op = pass.ops[idx];
    const uint32_t type = dtype_of(op);
    const int cslot = op.control >= 0 ? pl.slot(op.control) : -1;
    // ---- sign flips (Z, CZ) anywhere: an integer sign term --------------------
    if (type == D_SIGN) {
      SignTerm t{};
      const int tslot = pl.slot(op.target);
      uint32_t deps = 0;
      for (int s = 0; s < L.NS; ++s) {
        const bool tgt = tslot >= 0 ? bit_of(s, tslot) : true;
        const bool ctl = op.control < 0 || cslot < 0 ? true : bit_of(s, cslot);
        if (tgt && ctl) t.slots |= 1u << s;
      }
      if (tslot >= 0) deps |= 1u << tslot;
      else if (pl.tile(op.target) >= 0) t.lcond |= 1u << pl.tile(op.target);
      else t.gcond |= 1ull << op.target;
      if (op.control >= 0) {
        if (cslot >= 0) deps |= 1u << cslot;
        else if (pl.tile(op.control) >= 0) t.lcond |= 1u << pl.tile(op.control);
        else t.gcond |= 1ull << op.control;
      }
      // a term on slots without a 2x2 in the open layer commutes with that
      // layer's 2x2s: it joins the layer's pre part, so the layer stays open
      // for later 2x2s on those slots
      if (deps & L.mmask) {
        L.post_signs.push_back(t);
        L.post_slots |= deps;
      } else {
        L.pre_signs.push_back(t);
      }
      continue;
    }
    // ---- diagonal ops living on register slots: one table ----------------------
    if (type == D_DIAG || type == D_PHASE1) {
      const int tslot = pl.slot(op.target);
      if (tslot >= 0 && (op.control < 0 || cslot >= 0)) {
        const uint32_t deps = (1u << tslot) | (cslot >= 0 ? 1u << cslot : 0u);
        std::vector<cplx>& tab = (deps & L.mmask) ? L.post : L.pre;  // as for signs
        for (int s = 0; s < L.NS; ++s) {
          if (op.control >= 0 && !bit_of(s, cslot)) continue;
          tab[s] = cmul(tab[s], bit_of(s, tslot) ? op.m[3] : op.m[0]);
        }
        if (deps & L.mmask) L.post_slots |= deps;
        continue;
      }
    }
    // ---- uncontrolled dense on a register slot: into the layer -----------------
    if ((type == D_DENSE || type == D_REAL) && op.control < 0) {
      const int a = pl.slot(op.target);
      cplx R2[4] = {op.m[0], op.m[1], op.m[2], op.m[3]};
      cplx d1 = {1.0, 0.0}, p0 = {1.0, 0.0}, p1 = {1.0, 0.0};
      bool factored = false;
      bool real = type == D_REAL;
      if (!real) {
        double c, sn;
        if (zyz_split(op.m, p0, p1, c, sn, d1)) {
          // U = diag(p0, p1) . [[c, -s], [s, c]] . diag(1, q1)
          R2[0] = {c, 0.0};
          R2[1] = {-sn, 0.0};
          R2[2] = {sn, 0.0};
          R2[3] = {c, 0.0};
          factored = true;
          real = true;
        }
      }
      if ((L.mmask & (1u << a)) || (L.post_slots & (1u << a))) close_layer(L, out);
      if (factored) {
        for (int s = 0; s < L.NS; ++s)
          if (bit_of(s, a)) L.pre[s] = cmul(L.pre[s], d1);
        for (int s = 0; s < L.NS; ++s) L.post[s] = cmul(L.post[s], bit_of(s, a) ? p1 : p0);
        L.post_slots |= 1u << a;
      }
      for (int k = 0; k < 4; ++k) L.M[a][k] = R2[k];
      L.mmask |= 1u << a;
      if (real) L.cmask &= ~(1u << a);
      else L.cmask |= 1u << a;
      continue;
    }
    // ---- anything else: flush, then a single op --------------------------------
    flush_all(L, out);
    encode_single(op, pass.tile_phys, round.reg, out);
  }
  flush_all(L, out);
  set_dispatch_index(out, R);
  return out;
}

namespace {

// One greedy register round over `remaining` (application order, with
// hoisting): an op joins when it commutes with every skipped op on its
// qubits and its X-role qubits are (or, without `preset`, can still become)
// register bits. Returns the number of X-role ops scheduled.
int greedy_round(const PlanPass& pass, const std::vector<int>& remaining, int R,
                 const std::vector<int>& tix, const std::vector<int>* preset,
                 const PlanOptions& opt, PlanRound& round, std::vector<int>& rest) {
  const int k = static_cast<int>(pass.tile_phys.size());
  const int nphys = static_cast<int>(tix.size());
  std::vector<char> blockAll(nphys, 0), blockX(nphys, 0), inReg(k, 0);
  round = PlanRound{};
  rest.clear();
  if (preset) {
    round.reg = *preset;
    for (int ti : *preset) inReg[ti] = 1;
  }
  int xops = 0;
  QR rl[3];
  for (int idx : remaining) {
    const LOp& op = pass.ops[idx];
    const int nr = roles(op, rl);
    bool can = static_cast<int>(round.ops.size()) < opt.max_round_ops;
    for (int t = 0; t < nr && can; ++t) {
      if (blockAll[rl[t].q] || (rl[t].r == XRole && blockX[rl[t].q])) can = false;
    }
    bool isx = false;
    if (can) {
      int need[2], nn = 0;
      for (int t = 0; t < nr; ++t) {
        if (rl[t].r != XRole) continue;
        isx = true;
        const int ti = tix[rl[t].q];
        if (!inReg[ti]) {
          bool dup = false;
          for (int u = 0; u < nn; ++u) dup = dup || need[u] == ti;
          if (!dup) need[nn++] = ti;
        }
      }
      if (nn == 0 || (!preset && static_cast<int>(round.reg.size()) + nn <= R)) {
        for (int u = 0; u < nn; ++u) {
          inReg[need[u]] = 1;
          round.reg.push_back(need[u]);
        }
        round.ops.push_back(idx);
        xops += isx ? 1 : 0;
      } else {
        can = false;
      }
    }
    if (!can) {
      rest.push_back(idx);
      for (int t = 0; t < nr; ++t) {
        if (rl[t].r == XRole) blockAll[rl[t].q] = 1;
        else blockX[rl[t].q] = 1;
      }
    }
  }
  // pad the register set with the highest unused tile bits
  for (int ti = k - 1; static_cast<int>(round.reg.size()) < R && ti >= 0; --ti) {
    if (!inReg[ti]) {
      inReg[ti] = 1;
      round.reg.push_back(ti);
    }
  }
  return xops;
}

// Splits the ops of one pass (physical qubits, application order) into
// register rounds of R tile bits, then device-encodes every round. Each
// round's register set is chosen among the first few tile bits that still
// have X-role ops: every R-subset is tried and the one that schedules the
// most X-role ops wins (ties: the plain first-need greedy), so rounds hold
// full layers instead of whatever the op order reaches first.
void make_rounds(PlanPass& pass, int R, int nphys, const PlanOptions& opt, bool search) {
  const int k = static_cast<int>(pass.tile_phys.size());
  std::vector<int> tix(nphys, -1);
  for (int i = 0; i < k; ++i) tix[pass.tile_phys[i]] = i;
  std::vector<int> remaining(pass.ops.size());
  for (size_t i = 0; i < remaining.size(); ++i) remaining[i] = static_cast<int>(i);
  constexpr int kCand = 8;  // candidate register bits (at most 70 R-subsets for R = 4)
  PlanRound best, trial;
  std::vector<int> best_rest, trial_rest;
  QR rl[3];
  while (!remaining.empty()) {
    int best_x = greedy_round(pass, remaining, R, tix, nullptr, opt, best, best_rest);
    // candidate register bits: tile bits with X-role ops, in first-need order
    std::vector<int> cand;
    for (int idx : remaining) {
      if (!search) break;
      const int nr = roles(pass.ops[idx], rl);
      for (int t = 0; t < nr; ++t) {
        if (rl[t].r != XRole) continue;
        const int ti = tix[rl[t].q];
        if (std::find(cand.begin(), cand.end(), ti) == cand.end()) cand.push_back(ti);
      }
      if (static_cast<int>(cand.size()) >= kCand) break;
    }
    const int m = static_cast<int>(cand.size());
    if (search && m > R && R <= 4) {
      std::vector<int> pick(R);
      // all R-subsets of cand (m <= 8: at most 70)
      for (uint32_t bits = 0; bits < (1u << m); ++bits) {
        if (__builtin_popcount(bits) != R) continue;
        int j = 0;
        for (int i = 0; i < m; ++i)
          if ((bits >> i) & 1u) pick[j++] = cand[i];
        const int x = greedy_round(pass, remaining, R, tix, &pick, opt, trial, trial_rest);
        if (x > best_x) {
          best_x = x;
          std::swap(best, trial);
          std::swap(best_rest, trial_rest);
        }
      }
    }
    best.enc = compile_round(pass, best, opt.fuse_layers);
    pass.rounds.push_back(std::move(best));
    remaining.swap(best_rest);
  }
}

// A launch carries at most kLargeOps device ops, kLargeRounds rounds and
// kLargePool pool doubles (kernel parameter space); deeper passes become
// consecutive launches on the same tile (only FP64-bound passes are that
// deep, so the extra HBM sweep hides).
void split_pass(PlanPass& pass, std::vector<PlanPass>& out) {
  size_t r = 0;
  while (r < pass.rounds.size()) {
    PlanPass part;
    part.kind = PlanPass::Tile;
    part.tile_phys = pass.tile_phys;
    size_t nops = 0, npool = 0;
    while (r < pass.rounds.size() &&
           static_cast<int>(part.rounds.size()) < kLargeRounds &&
           nops + pass.rounds[r].enc.ops.size() <= static_cast<size_t>(kLargeOps) &&
           npool + pass.rounds[r].enc.pool.size() <= static_cast<size_t>(kLargePool)) {
      PlanRound pr;
      pr.reg = pass.rounds[r].reg;
      for (int idx : pass.rounds[r].ops) {
        pr.ops.push_back(static_cast<int>(part.ops.size()));
        part.ops.push_back(pass.ops[idx]);
      }
      pr.enc = std::move(pass.rounds[r].enc);
      nops += pr.enc.ops.size();
      npool += pr.enc.pool.size();
      part.rounds.push_back(std::move(pr));
      ++r;
    }
    if (part.rounds.empty())
      throw std::logic_error("a register round exceeds the kernel parameter space");
    out.push_back(std::move(part));
  }
}

}  // namespace

Plan make_plan(const std::vector<LOp>& ops, int nqubits, int nlocal,
               const std::vector<int>& perm, const PlanOptions& opt) {
  Plan plan;
  plan.nqubits = nqubits;
  plan.nlocal = nlocal;
  plan.perm_before = perm;
  std::vector<int> cur = perm;  // logical -> physical
  std::vector<int> inv(nqubits);
  for (int q = 0; q < nqubits; ++q) inv[cur[q]] = q;

  const int K = std::min(opt.tile_bits, nlocal);
  // keep at least two free tile slots so any op (SWAP: two targets) fits
  const int m = std::max(0, std::min(opt.low_bits, K - 2));
  const int R = std::min(opt.reg_bits, K);
  const size_t nops = ops.size();
  std::vector<char> done(nops, 0);
  size_t first = 0;
  QR rl[3];

  std::vector<char> blockAll(nqubits), blockX(nqubits), inQ(nlocal);
  std::vector<std::vector<int>> beam_seeds;  // window choice of every pass (beam search)
  size_t beam_pos = 0;
  bool beam_tried = false;
  while (true) {
    while (first < nops && done[first]) ++first;
    if (first >= nops) break;

    // ---- exchange when the head op needs a global (sharded) qubit --------
    bool head_global = false;
    {
      const int nr = roles(ops[first], rl);
      for (int t = 0; t < nr; ++t)
        if (rl[t].r == XRole && cur[rl[t].q] >= nlocal) head_global = true;
    }
    if (head_global) {
      // global physical bits with upcoming X-role use, in order of need
      std::vector<int> need_g;
      std::vector<size_t> next_x(nqubits, std::numeric_limits<size_t>::max());
      size_t scanned = 0;
      for (size_t i = first; i < nops && scanned < static_cast<size_t>(opt.lookahead); ++i) {
        if (done[i]) continue;
        ++scanned;
        const int nr = roles(ops[i], rl);
        for (int t = 0; t < nr; ++t) {
          if (rl[t].r != XRole) continue;
          const int q = rl[t].q;
          if (next_x[q] == std::numeric_limits<size_t>::max()) next_x[q] = i;
          const int p = cur[q];
          if (p >= nlocal && std::find(need_g.begin(), need_g.end(), p) == need_g.end())
            need_g.push_back(p);
        }
      }
      const int g = nqubits - nlocal;
      // at most g globals per exchange, and no more than there are local
      // victim bits (shards of fewer bits than the rank bits)
      if (static_cast<int>(need_g.size()) > std::min(g, nlocal)) need_g.resize(std::min(g, nlocal));
      // victims: among the top local bits, the furthest next X use first.
      // The candidates reach down to kVictimSpan bits below the top (runs of
      // >= 2^(nlocal - kVictimSpan) amplitudes per exchange step): with only
      // the top few bits as candidates, the qubits swapped out are needed
      // again soon and swapped straight back (C4 at 8 shards: 20 exchanges
      // instead of 12).
      const int ncand = std::min(nlocal, std::max({4, static_cast<int>(need_g.size()),
                                                   std::min(nlocal, opt.victim_span)}));
      std::vector<int> cand;
      for (int p = nlocal - 1; p >= nlocal - ncand; --p) cand.push_back(p);
      std::stable_sort(cand.begin(), cand.end(), [&](int a, int b) {
        return next_x[inv[a]] > next_x[inv[b]];
      });
      PlanPass ex;
      ex.kind = PlanPass::Exchange;
      for (size_t i = 0; i < need_g.size(); ++i) {
        const int G = need_g[i], V = cand[i];
        ex.exchange.emplace_back(G, V);
        const int qg = inv[G], qv = inv[V];
        cur[qg] = V;
        cur[qv] = G;
        inv[V] = qg;
        inv[G] = qv;
      }
      plan.passes.push_back(std::move(ex));
      continue;
    }

    // ---- tile pass --------------------------------------------------------
    // One greedy fill: scan the undone ops in order; an op joins when nothing
    // it must follow was skipped and its X-role bits are (or can still
    // become) tile bits. `seed` bits are in the tile from the start.
    struct Fill {
      std::vector<size_t> taken;
      std::vector<char> inQ;
      int qcount = 0;
      double fp64 = 0.0;
    };
    auto fill_pass = [&](const std::vector<char>& done, size_t first, const std::vector<int>& seed, Fill& f) {
      std::fill(blockAll.begin(), blockAll.end(), 0);
      std::fill(blockX.begin(), blockX.end(), 0);
      f.taken.clear();
      f.inQ.assign(nlocal, 0);
      for (int b = 0; b < m; ++b) f.inQ[b] = 1;
      f.qcount = m;
      for (int p : seed)
        if (p >= 0 && p < nlocal && !f.inQ[p] && f.qcount < K) {
          f.inQ[p] = 1;
          ++f.qcount;
        }
      f.fp64 = 0.0;
      int nblocked = 0;
      size_t scanned = 0;
      for (size_t i = first; i < nops && scanned < static_cast<size_t>(opt.lookahead); ++i) {
        if (done[i]) continue;
        ++scanned;
        const LOp& op = ops[i];
        const int nr = roles(op, rl);
        bool can = true;
        const double cost = (op.kind == LKind::Dense) ? 3.0 : 0.0;
        if (opt.max_pass_fp64 > 0.0 && !f.taken.empty() && f.fp64 + cost > opt.max_pass_fp64) can = false;
        for (int t = 0; t < nr; ++t) {
          if (blockAll[rl[t].q] || (rl[t].r == XRole && blockX[rl[t].q])) can = false;
        }
        if (can) {
          int need[2], nn = 0;
          for (int t = 0; t < nr; ++t) {
            if (rl[t].r != XRole) continue;
            const int p = cur[rl[t].q];
            if (p >= nlocal) {
              can = false;
              break;
            }
            if (!f.inQ[p]) {
              bool dup = false;
              for (int u = 0; u < nn; ++u) dup = dup || need[u] == p;
              if (!dup) need[nn++] = p;
            }
          }
          if (can && f.qcount + nn <= K) {
            for (int u = 0; u < nn; ++u) f.inQ[need[u]] = 1;
            f.qcount += nn;
          } else {
            can = false;
          }
        }
        if (can) {
          f.fp64 += cost;
          f.taken.push_back(i);
        } else {
          for (int t = 0; t < nr; ++t) {
            if (rl[t].r == XRole) {
              if (!blockAll[rl[t].q]) {
                blockAll[rl[t].q] = 1;
                ++nblocked;
              }
            } else {
              blockX[rl[t].q] = 1;
            }
          }
          if (nblocked == nqubits) break;
        }
      }
    };
    // candidate seeds of a pass: none (first-need greedy) and every window of
    // K - m consecutive physical bits
    auto candidate_seeds = [&]() {
      std::vector<std::vector<int>> c(1);
      const int w = K - m;
      for (int s0 = m; s0 + w <= nlocal; ++s0) {
        c.emplace_back();
        for (int b = 0; b < w; ++b) c.back().push_back(s0 + b);
      }
      return c;
    };
    // Beam search over the window choices (single-GPU plans only: no exchange
    // changes the qubit map underneath): every level is one more pass, a node
    // is the set of ops done so far, the `window_beam` nodes with the most
    // FP64 work done survive a level, and the first level on which a node has
    // every op done gives the seed sequence the passes below follow.
    if (opt.window_search && opt.window_beam > 1 && nlocal == nqubits && beam_seeds.empty() && !beam_tried) {
      beam_tried = true;
      struct Node {
        std::vector<char> done;
        size_t first = 0, left = 0;
        double fp = 0.0;
        std::vector<std::vector<int>> seeds;
      };
      std::vector<Node> beam(1);
      beam[0].done = done;
      beam[0].first = first;
      for (size_t i = 0; i < nops; ++i) beam[0].left += done[i] ? 0 : 1;
      const std::vector<std::vector<int>> cands = candidate_seeds();
      Fill f;
      bool found = false;
      for (int level = 0; level < 4096 && !found && !beam.empty(); ++level) {
        std::vector<Node> next;
        std::unordered_map<std::string, size_t> seen;
        for (const Node& nd : beam) {
          for (const std::vector<int>& sd : cands) {
            fill_pass(nd.done, nd.first, sd, f);
            if (f.taken.empty()) continue;
            Node ch;
            ch.done = nd.done;
            for (size_t i : f.taken) ch.done[i] = 1;
            std::string key(ch.done.begin(), ch.done.end());
            auto it = seen.find(key);
            if (it != seen.end()) continue;
            seen.emplace(std::move(key), next.size());
            ch.first = nd.first;
            while (ch.first < nops && ch.done[ch.first]) ++ch.first;
            ch.left = nd.left - f.taken.size();
            ch.fp = nd.fp + f.fp64;
            ch.seeds = nd.seeds;
            ch.seeds.push_back(sd);
            if (ch.left == 0) {
              beam_seeds = ch.seeds;
              found = true;
              break;
            }
            next.push_back(std::move(ch));
          }
          if (found) break;
        }
        if (found) break;
        std::sort(next.begin(), next.end(), [](const Node& a, const Node& b) {
          if (a.fp != b.fp) return a.fp > b.fp;
          return a.left < b.left;
        });
        if (next.size() > static_cast<size_t>(opt.window_beam)) next.resize(static_cast<size_t>(opt.window_beam));
        beam.swap(next);
      }
      beam_pos = 0;
    }
    Fill best;
    if (beam_pos < beam_seeds.size()) {
      fill_pass(done, first, beam_seeds[beam_pos++], best);
    } else {
      fill_pass(done, first, {}, best);
    }
    if (opt.window_search && beam_seeds.empty()) {
      // Candidate tiles: windows of K - m consecutive physical bits at every
      // start; the fill that carries the most FP64 work (ties: most ops) wins.
      // The first-need greedy above follows the op order, which on layered
      // circuits spends tile bits on qubits whose neighbours block them after
      // one layer; a window over qubits that can advance together carries
      // several layers.
      Fill trial;
      std::vector<int> seed;
      const int w = K - m;
      for (int s0 = m; s0 + w <= nlocal; ++s0) {
        seed.clear();
        for (int b = 0; b < w; ++b) seed.push_back(s0 + b);
        fill_pass(done, first, seed, trial);
        if (trial.taken.empty()) continue;
        if (trial.fp64 > best.fp64 + 1e-9 ||
            (trial.fp64 > best.fp64 - 1e-9 && trial.taken.size() > best.taken.size()))
          std::swap(best, trial);
      }
    }
    PlanPass pass;
    for (size_t i : best.taken) {
      done[i] = 1;
      pass.ops.push_back(to_phys(ops[i], cur));
    }
    inQ = best.inQ;
    int qcount = best.qcount;
    // seeded bits no op of the pass uses as an X-role bit leave the tile again
    if (opt.window_search) {
      std::vector<char> xb(nlocal, 0);
      for (const LOp& pop : pass.ops) {
        const int nr = roles(pop, rl);
        for (int t = 0; t < nr; ++t)
          if (rl[t].r == XRole && rl[t].q < nlocal) xb[rl[t].q] = 1;
      }
      for (int p = m; p < nlocal; ++p)
        if (inQ[p] && !xb[p]) {
          inQ[p] = 0;
          --qcount;
        }
    }
    // Tile shrinking (opt.shrink_min_bits): the low bits were reserved for
    // coalescing only; those above the run bits that no op of the pass uses
    // as an X-role bit leave the tile (highest first) while it keeps at least
    // shrink_min_bits bits. The pass holds the same ops; the smaller tile
    // needs less shared memory, so more CTAs of the compiled kernel (each with
    // its own ring of tile buffers) are resident per SM and their load /
    // compute / store phases overlap.
    if (opt.shrink_min_bits > 0 && qcount > opt.shrink_min_bits) {
      std::vector<char> xbit(nlocal, 0);
      for (const LOp& pop : pass.ops) {
        const int nr = roles(pop, rl);
        for (int t = 0; t < nr; ++t)
          if (rl[t].r == XRole && rl[t].q < nlocal) xbit[rl[t].q] = 1;
      }
      for (int b = m - 1; b >= std::max(0, opt.shrink_run_bits) && qcount > opt.shrink_min_bits; --b) {
        if (inQ[b] && !xbit[b]) {
          inQ[b] = 0;
          --qcount;
        }
      }
    }
    // complete the tile to K bits with the lowest unused local bits
    for (int p = 0; p < nlocal && qcount < (opt.shrink_min_bits > 0 ? std::min(K, opt.shrink_min_bits) : K); ++p) {
      if (!inQ[p]) {
        inQ[p] = 1;
        ++qcount;
      }
    }
    for (int p = 0; p < nlocal; ++p)
      if (inQ[p]) pass.tile_phys.push_back(p);
    if (pass.ops.empty()) throw std::logic_error("planner made no progress");
    make_rounds(pass, R, nqubits, opt, nlocal >= opt.round_search_min_bits);
    split_pass(pass, plan.passes);
  }
  plan.perm_after = cur;
  plan.gates = nops;
  return plan;
}

std::string plan_to_json(const Plan& p, bool detail, const std::vector<double>* fp64_lowered) {
  std::ostringstream os;
  const unsigned long long amps = 1ull << p.nlocal;
  os << "{\"nqubits\":" << p.nqubits << ",\"nlocal\":" << p.nlocal
     << ",\"ops\":" << p.gates << ",\"passes\":[";
  for (size_t i = 0; i < p.passes.size(); ++i) {
    const PlanPass& ps = p.passes[i];
    if (i) os << ",";
    if (ps.kind == PlanPass::Exchange) {
      os << "{\"kind\":\"exchange\",\"swap\":[";
      for (size_t e = 0; e < ps.exchange.size(); ++e) {
        if (e) os << ",";
        os << "[" << ps.exchange[e].first << "," << ps.exchange[e].second << "]";
      }
      os << "]}";
      continue;
    }
    // FP64-pipe instructions per amplitude of the encoded (fused) ops
    double fp = 0.0;
    size_t ndev = 0;
    for (const PlanRound& pr : ps.rounds) {
      ndev += pr.enc.ops.size();
      for (const DOp& d : pr.enc.ops) {
        const uint32_t v = d.hdr & kOpVariantMask, type = v >> 10, a = (v >> 6) & 15;
        const bool ctl = ((v >> 3) & 7) != 0;
        switch (type) {
          case D_DENSE: fp += ctl ? 4.0 : 8.0; break;
          case D_REAL: case D_ANTI: fp += ctl ? 2.0 : 4.0; break;
          case D_DIAG: case D_PHASE1: fp += 4.0; break;
          case D_LAYER:  // a layer: rotations (a), complex 2x2s (lmask), table
            fp += 3.0 * __builtin_popcount(a) + 8.0 * __builtin_popcount(d.lmask) +
                  ((d.hdr & kOpTable) ? 4.0 : 0.0);
            break;
          default: break;
        }
      }
    }
    os << "{\"kind\":\"tile\",\"device_ops\":" << ndev << ",\"tile\":[";
    for (size_t t = 0; t < ps.tile_phys.size(); ++t) {
      if (t) os << ",";
      os << ps.tile_phys[t];
    }
    os << "],\"rounds\":" << ps.rounds.size() << ",\"ops\":" << ps.ops.size()
       << ",\"gates\":[";
    std::vector<uint32_t> gs;
    for (const LOp& op : ps.ops) gs.push_back(op.gate);
    std::sort(gs.begin(), gs.end());
    gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
    for (size_t t = 0; t < gs.size(); ++t) {
      if (t) os << ",";
      os << gs[t];
    }
    if (fp64_lowered && i < fp64_lowered->size() && (*fp64_lowered)[i] >= 0.0) fp = (*fp64_lowered)[i];
    os << "],\"read_amps\":" << amps << ",\"write_amps\":" << amps
       << ",\"fp64_per_amp\":" << fp;
    if (detail) {
      os << ",\"round_detail\":[";
      char num[64];
      for (size_t r = 0; r < ps.rounds.size(); ++r) {
        const PlanRound& pr = ps.rounds[r];
        if (r) os << ",";
        os << "{\"reg\":[";
        for (size_t i = 0; i < pr.reg.size(); ++i) os << (i ? "," : "") << pr.reg[i];
        os << "],\"ops\":[";
        const int NS = 1 << pr.reg.size();
        for (size_t o = 0; o < pr.enc.ops.size(); ++o) {
          const DOp& d = pr.enc.ops[o];
          if (o) os << ",";
          const uint32_t v = d.hdr & kOpVariantMask;
          const uint32_t type = v >> 10, a = (v >> 6) & 15;
          os << "[" << type << "," << a << "," << static_cast<int>((v >> 3) & 7) - 1
             << "," << static_cast<int>(v & 7) - 1 << "," << d.lmask << "," << d.gmask
             << "," << d.dl << "," << d.dg << ",[";
          size_t off = d.arg & 0xffff, len = 8;
          const bool tab = (d.hdr & kOpTable) != 0;
          auto put = [&](size_t from, size_t n) {
            for (size_t k = 0; k < n; ++k) {
              std::snprintf(num, sizeof(num), "%s%.17g", k ? "," : "", pr.enc.pool[from + k]);
              os << num;
            }
          };
          if (type == D_LAYER) {
            // layer: [..., [2x2 data], tabflag, [table], [[base,0,0], terms...]]
            const uint32_t nt = d.arg >> 16;
            const size_t toff = off, soff = off + (tab ? 2 * NS : 0), moff = soff + 2 * nt;
            put(moff, 2 * __builtin_popcount(a) + 8 * __builtin_popcount(d.lmask));
            os << "]," << (tab ? 1 : 0) << ",[";
            if (tab) put(toff, 2 * NS);
            os << "],[[" << d.dl << ",0,0]";
            for (uint32_t t = 0; t < nt; ++t) {
              uint64_t w0, w1;
              std::memcpy(&w0, &pr.enc.pool[soff + 2 * t], 8);
              std::memcpy(&w1, &pr.enc.pool[soff + 2 * t + 1], 8);
              os << ",[" << (w0 & 0xffffffffull) << "," << (w0 >> 32) << "," << w1 << "]";
            }
            os << "]]";
            continue;
          }
          put(off, len);
          os << "]," << (tab ? 1 : 0) << "]";
        }
        os << "]}";
      }
      os << "]";
    }
    os << "}";
  }
  os << "],\"perm_after\":[";
  for (size_t q = 0; q < p.perm_after.size(); ++q) {
    if (q) os << ",";
    os << p.perm_after[q];
  }
  os << "]}";
  return os.str();
}

}  // namespace qtb
