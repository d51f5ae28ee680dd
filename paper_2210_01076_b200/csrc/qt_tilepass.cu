// qt_tilepass.cu -- the fused tile-pass kernel (the hot path).
//
// The reference applies one gate per stage with two CPU loops:
// run_permute_tasks (engine.cpp:315-350: swap/scale element ops, one
// ElementOpSeq::op(k) per pair, element_ops.cpp:82-133) and
// run_mxv_partition (engine.cpp:352-383: Kronecker-row mat-vec over every
// superposition gate of a net, kron_row_visit plan.hpp:98-127), both on host
// copy-on-write blocks.
//
// Here a whole run of gates is applied by ONE launch that streams the
// 2^n complex128 state through shared memory exactly once:
//   HBM --(16-B coalesced loads)--> smem tile of 2^k amplitudes
//       --> R-qubit register rounds: each thread holds 2^R amplitudes (indices
//           differing in the round's R tile bits) in registers and applies
//           the round's device ops
//       --> smem --> HBM
// so a pass costs 32 B of HBM traffic per amplitude however many gates it
// carries. Device ops live in the kernel-parameter constant bank (headers +
// a pool of tables / rotations / matrices / sign terms). The host round
// compiler (qt_plan.cpp) turns each round into LAYER ops: a diagonal table
// over the round's register slots (every merged diagonal factor), integer
// sign flips (CZ, Z), then one 2x2 per register slot -- real rotations as
// three in-place shears after the ZYZ split, complex 2x2s otherwise -- all
// in one dispatch (k_layer: runtime slot masks over compiled slot bodies).
// X / CX are register permutations (k_perm). The generic instantiation adds
// specialised single-op variants (controlled 2x2s, diagonals on
// non-register bits, SWAP) for what a layer cannot hold. Controls /
// diagonal bits outside the register slots are thread- or tile-uniform
// predicates. Tensor cores do not apply (2x2 complex FP64 operands): a pass
// is bounded by HBM when shallow and by the FP64 pipe / issue when deep
// (DESIGN.md).
#include <cuda_runtime.h>

#include <cstdint>

#include "qt_device.cuh"
#include "qt_kernels.hpp"

namespace qtb {

namespace {

// ---- op variants (R register bits, 2^R slots per thread) -------------------
//
// Register discipline: every output of a pair is written by ONE final FMA
// that reads its own input register last (partial sums of the other terms
// are formed first), so ptxas can allocate each result into the input's
// register and the dispatch switch needs no phi moves for the 2^R
// loop-carried amplitudes.

template <int R, int A, int CS>
__device__ __forceinline__ void pair_dense(double2 (&v)[1 << R], double m0r, double m0i,
                                           double m1r, double m1i, double m2r, double m2i,
                                           double m3r, double m3i) {
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (s & (1 << A)) continue;
    if (CS >= 0 && !(s & (1 << CS))) continue;
    const int s1 = s | (1 << A);
    // na = m00 a + m01 b, nb = m10 a + m11 b (complex)
    const double p0 = fma(m1r, v[s1].x, fma(-m1i, v[s1].y, -m0i * v[s].y));
    const double p1 = fma(m1r, v[s1].y, fma(m1i, v[s1].x, m0i * v[s].x));
    const double p2 = fma(m2r, v[s].x, fma(-m2i, v[s].y, -m3i * v[s1].y));
    const double p3 = fma(m2r, v[s].y, fma(m2i, v[s].x, m3i * v[s1].x));
    v[s].x = fma(m0r, v[s].x, p0);
    v[s].y = fma(m0r, v[s].y, p1);
    v[s1].x = fma(m3r, v[s1].x, p2);
    v[s1].y = fma(m3r, v[s1].y, p3);
  }
}

template <int R, int A, int CS>
__device__ __forceinline__ void pair_real(double2 (&v)[1 << R], double m0, double m1,
                                          double m2, double m3) {
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (s & (1 << A)) continue;
    if (CS >= 0 && !(s & (1 << CS))) continue;
    const int s1 = s | (1 << A);
    const double p0 = m1 * v[s1].x, p1 = m1 * v[s1].y;
    const double p2 = m2 * v[s].x, p3 = m2 * v[s].y;
    v[s].x = fma(m0, v[s].x, p0);
    v[s].y = fma(m0, v[s].y, p1);
    v[s1].x = fma(m3, v[s1].x, p2);
    v[s1].y = fma(m3, v[s1].y, p3);
  }
}

// Real rotation [[c, -s], [s, c]] (|theta| <= pi/2) as three shears, each an
// in-place FMA: x += a y; y += b x; x += a y with a = -tan(theta/2), b =
// sin(theta) -- 3 FP64 ops per amplitude instead of 4, no temporaries.
template <int R, int A>
__device__ __forceinline__ void pair_shear(double2 (&v)[1 << R], double a, double b) {
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (s & (1 << A)) continue;
    const int s1 = s | (1 << A);
    v[s].x = fma(a, v[s1].x, v[s].x);
    v[s].y = fma(a, v[s1].y, v[s].y);
    v[s1].x = fma(b, v[s].x, v[s1].x);
    v[s1].y = fma(b, v[s].y, v[s1].y);
    v[s].x = fma(a, v[s1].x, v[s].x);
    v[s].y = fma(a, v[s1].y, v[s].y);
  }
}

template <int R, int A, int CS, typename P>
__device__ __forceinline__ void k_dense(double2 (&v)[1 << R], const P& p, int o) {
  pair_dense<R, A, CS>(v, p.pool[o], p.pool[o + 1], p.pool[o + 2], p.pool[o + 3],
                       p.pool[o + 4], p.pool[o + 5], p.pool[o + 6], p.pool[o + 7]);
}

template <int R, int A, int CS, typename P>
__device__ __forceinline__ void k_real(double2 (&v)[1 << R], const P& p, int o) {
  pair_real<R, A, CS>(v, p.pool[o], p.pool[o + 2], p.pool[o + 4], p.pool[o + 6]);
}

// Register-identity-preserving swap: XOR swap on the bit patterns, so no
// amplitude changes register (a plain swap makes ptxas insert a copy of all
// 2^R loop-carried amplitudes at the op-loop head for every op).
__device__ __forceinline__ void xswap(double& a, double& b) {
  // opaque to NVVM / ptxas: a source-level XOR swap is folded back into a
  // renaming, which is exactly what must not happen
  long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  asm volatile(
      "{\n\t"
      "xor.b64 %0, %0, %1;\n\t"
      "xor.b64 %1, %1, %0;\n\t"
      "xor.b64 %0, %0, %1;\n\t"
      "}"
      : "+l"(x), "+l"(y));
  a = __longlong_as_double(x);
  b = __longlong_as_double(y);
}

__device__ __forceinline__ void xswap2(double2& a, double2& b) {
  xswap(a.x, b.x);
  xswap(a.y, b.y);
}

template <int R, int A, int CS>
__device__ __forceinline__ void k_xperm(double2 (&v)[1 << R]) {
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (s & (1 << A)) continue;
    if (CS >= 0 && !(s & (1 << CS))) continue;
    xswap2(v[s], v[s | (1 << A)]);
  }
}

// in-place complex scale: the final FMA of each part reads its own input
__device__ __forceinline__ void cscale(double2& x, double br, double bi) {
  const double p0 = -bi * x.y, p1 = bi * x.x;
  x.x = fma(br, x.x, p0);
  x.y = fma(br, x.y, p1);
}

template <int R, int A, int CS, typename P>
__device__ __forceinline__ void k_anti(double2 (&v)[1 << R], const P& p, int o) {
  const double m1r = p.pool[o + 2], m1i = p.pool[o + 3];
  const double m2r = p.pool[o + 4], m2i = p.pool[o + 5];
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (s & (1 << A)) continue;
    if (CS >= 0 && !(s & (1 << CS))) continue;
    const int s1 = s | (1 << A);
    xswap2(v[s], v[s1]);  // then scale in place: (m01 b, m10 a)
    cscale(v[s], m1r, m1i);
    cscale(v[s1], m2r, m2i);
  }
}

// diag(d0, d1) on a bit: DS >= 0 -> register slot bit DS (compile-time
// choice per slot); DS < 0 -> the thread-uniform bit `bit`.
template <int R, int CS, int DS, typename P>
__device__ __forceinline__ void k_diag(double2 (&v)[1 << R], const P& p, int o,
                                       bool bit) {
  const double d0r = p.pool[o], d0i = p.pool[o + 1];
  const double d1r = p.pool[o + 6], d1i = p.pool[o + 7];
  const double ur = bit ? d1r : d0r, ui = bit ? d1i : d0i;
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (CS >= 0 && !(s & (1 << CS))) continue;
    if (DS >= 0) {
      if (s & (1 << DS)) cscale(v[s], d1r, d1i);
      else cscale(v[s], d0r, d0i);
    } else {
      cscale(v[s], ur, ui);
    }
  }
}

// diag(1, d1): only amplitudes whose bit is set are touched
template <int R, int CS, int DS, typename P>
__device__ __forceinline__ void k_phase1(double2 (&v)[1 << R], const P& p, int o,
                                         bool bit) {
  const double d1r = p.pool[o + 6], d1i = p.pool[o + 7];
  if (DS < 0 && !bit) return;
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (CS >= 0 && !(s & (1 << CS))) continue;
    if (DS >= 0 && !(s & (1 << DS))) continue;
    cscale(v[s], d1r, d1i);
  }
}

// diag(1, -1): integer sign flips (Z, CZ)
template <int R, int CS, int DS>
__device__ __forceinline__ void k_sign(double2 (&v)[1 << R], bool bit) {
  if (DS < 0 && !bit) return;
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (CS >= 0 && !(s & (1 << CS))) continue;
    if (DS >= 0 && !(s & (1 << DS))) continue;
    v[s] = neg2(v[s]);
  }
}

template <int R, int A, int B>
__device__ __forceinline__ void k_swap2(double2 (&v)[1 << R]) {
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if ((s & (1 << A)) && !(s & (1 << B))) xswap2(v[s], v[s ^ (1 << A) ^ (1 << B)]);
  }
}

// per-slot complex factor table (all merged diagonal gates of a layer)
template <int R, typename P>
__device__ __forceinline__ void k_dtab(double2 (&v)[1 << R], const P& p, int o) {
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) cscale(v[s], p.pool[o + 2 * s], p.pool[o + 2 * s + 1]);
}

// Sign terms: `base` = the unconditional terms (folded on the host) and nt
// thread/tile-conditional terms at pool[o]; then one integer XOR per
// component (branch-free: the mask differs between threads).
// hi ^ (ms & 0x80000000) in one LOP3 (LUT 0x78 = a ^ (b & c))
__device__ __forceinline__ int xor_sign(int hi, uint32_t ms) {
  int r;
  asm("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(r) : "r"(hi), "r"(ms), "n"(0x80000000));
  return r;
}

template <int R, typename P>
__device__ __forceinline__ void apply_signs(double2 (&v)[1 << R], const P& p, int o,
                                            uint32_t nt, uint32_t base, uint32_t jb,
                                            const uint64_t* sg) {
  uint32_t mask = base;
  for (int t = 0; t < static_cast<int>(nt); ++t) {
    const uint64_t w0 = static_cast<uint64_t>(__double_as_longlong(p.pool[o + 2 * t]));
    const uint64_t gc = static_cast<uint64_t>(__double_as_longlong(p.pool[o + 2 * t + 1]));
    const uint32_t lc = static_cast<uint32_t>(w0 >> 32);
    bool on = (jb & lc) == lc;
    if (gc) on = on && (*sg & gc) == gc;
    mask ^= on ? static_cast<uint32_t>(w0) : 0u;
  }
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    // bit s of the mask to the sign bit: one shift, then one and-xor LOP3
    // (hi ^ (ms & 0x80000000)) per high word
    const uint32_t ms = mask << (31 - s);
    v[s] = make_double2(__hiloint2double(xor_sign(__double2hiint(v[s].x), ms), __double2loint(v[s].x)),
                        __hiloint2double(xor_sign(__double2hiint(v[s].y), ms), __double2loint(v[s].y)));
  }
}

// slot bodies of a layer, slots A..R-1 (compile-time slot index, runtime mask)
template <int R, int A, typename P>
__device__ __forceinline__ void layer_rot(double2 (&v)[1 << R], const P& p, uint32_t mask,
                                          int& o) {
  if constexpr (A < R) {
    if (mask & (1u << A)) {
      // rotation (c, s) as three in-place shears a = -s / (1 + c), b = s
      // (pair_shear; the division is correctly rounded, as on the host)
      const double c = p.pool[o], sn = p.pool[o + 1];
      pair_shear<R, A>(v, -sn / (1.0 + c), sn);
      o += 2;
    }
    layer_rot<R, A + 1>(v, p, mask, o);
  }
}

template <int R, int A, typename P>
__device__ __forceinline__ void layer_dense(double2 (&v)[1 << R], const P& p, uint32_t mask,
                                            int& o) {
  if constexpr (A < R) {
    if (mask & (1u << A)) {
      k_dense<R, A, -1>(v, p, o);
      o += 8;
    }
    layer_dense<R, A + 1>(v, p, mask, o);
  }
}

// A fused LAYER in one dispatch (the round compiler's unit, types MULTI /
// MULTIR): the layer's diagonal table (kOpTable), its sign terms (base mask
// in dl, conditional terms counted in arg >> 16), then one 2x2 per register
// slot in the slot mask, ascending slots (they commute exactly, so one fixed
// order): real rotations (three-shear form, after the ZYZ split) or complex
// 2x2s. Pool
// data in that order. A lone table / sign op is a layer with an empty mask.
// The slot loop is a runtime (CTA-uniform) mask over R compiled slot bodies:
// one copy of each body keeps the hot loop inside the instruction cache.
template <int R, typename P>
__device__ __forceinline__ void k_layer(double2 (&v)[1 << R], const P& p, uint32_t hdr,
                                        uint32_t arg, uint32_t base, uint32_t cmask,
                                        uint32_t jb, const uint64_t* sg) {
  int o = static_cast<int>(arg & 0xffffu);
  const uint32_t nt = arg >> 16;
  if (hdr & kOpTable) {
    k_dtab<R>(v, p, o);
    o += 2 << R;
  }
  if (nt | base) {
    apply_signs<R>(v, p, o, nt, base, jb, sg);
    o += 2 * static_cast<int>(nt);
  }
  const uint32_t rmask = (hdr >> 6) & 15u;
  // (offsets advance slot by slot: no popcount, which would leave the
  // uniform datapath and turn every constant load into a per-thread LDC)
  if (rmask) layer_rot<R, 0>(v, p, rmask, o);
  if (cmask) layer_dense<R, 0>(v, p, cmask, o);
}

// X / CX as a register permutation: swap the pairs of slot A (runtime target
// slot, one compiled body per slot) where the control holds -- a register
// slot (runtime, CTA-uniform per pair), a thread bit (lmask: per-thread,
// branch-free masked XOR swaps) and / or a bit outside the tile (gmask:
// tile-uniform, checked once).
__device__ __forceinline__ void mswap(double& a, double& b, uint64_t m) {
  long long x = __double_as_longlong(a), y = __double_as_longlong(b);
  const long long t = (x ^ y) & static_cast<long long>(m);
  asm volatile("" : "+l"(x), "+l"(y));
  a = __longlong_as_double(x ^ t);
  b = __longlong_as_double(y ^ t);
}

template <int R, int A>
__device__ __forceinline__ void perm_slot(double2 (&v)[1 << R], int cs, bool masked,
                                          uint64_t m) {
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (s & (1 << A)) continue;
    if (cs >= 0 && !((s >> cs) & 1)) continue;  // CTA-uniform
    const int s1 = s | (1 << A);
    if (masked) {
      mswap(v[s].x, v[s1].x, m);
      mswap(v[s].y, v[s1].y, m);
    } else {
      xswap2(v[s], v[s1]);
    }
  }
}

template <int R, int A>
__device__ __forceinline__ void perm_dispatch(double2 (&v)[1 << R], int a, int cs, bool masked,
                                              uint64_t m) {
  if constexpr (A < R) {
    if (a == A) perm_slot<R, A>(v, cs, masked, m);
    else perm_dispatch<R, A + 1>(v, a, cs, masked, m);
  }
}

template <int R>
__device__ __forceinline__ void k_perm(double2 (&v)[1 << R], uint32_t hdr, const DOp& d,
                                       uint32_t jb, const uint64_t* sg) {
  if ((hdr & kOpGctl) && (*sg & d.gmask) != d.gmask) return;  // tile-uniform
  const int a = static_cast<int>((hdr >> 6) & 15u);
  const int cs = static_cast<int>((hdr >> 3) & 7u) - 1;
  const bool masked = (hdr & kOpLctl) != 0;
  const uint64_t m = masked && (jb & d.lmask) == d.lmask ? ~0ull : 0ull;
  perm_dispatch<R, 0>(v, a, cs, masked, m);
}

// Applies one device op. `jb` = the thread's tile-local index with the
// register bits cleared; `sg` = the tile's global base index (smem).
// Controls / diagonal bits outside the register slots are only evaluated for
// ops whose header flags say they have them.
template <int R, bool GENERIC, typename P>
__device__ __forceinline__ void apply_op(double2 (&v)[1 << R], const P& p, const DOp& d,
                                         uint32_t hdr, uint32_t jb, const uint64_t* sg) {
  const uint32_t type = (hdr & kOpVariantMask) >> 10;
  if (type == D_XPERM) {  // X / CX on a register slot: the lean kernel has it too
    k_perm<R>(v, hdr, d, jb, sg);
    return;
  }
  if (!GENERIC || type == D_LAYER) {
    // the fused layer ops carry no flags
    k_layer<R>(v, p, hdr, d.arg, d.dl, d.lmask, jb, sg);
    return;
  }
  bool bit = false;
  if (hdr & kOpFlagMask) {
    if ((hdr & kOpLctl) && (jb & d.lmask) != d.lmask) return;
    if (hdr & kOpDl) bit = (jb & d.dl) != 0;
    if (hdr & (kOpGctl | kOpDg)) {
      const uint64_t g = *sg;
      if ((g & d.gmask) != d.gmask) return;
      bit = bit || (g & d.dg) != 0;
    }
  }
  const uint32_t arg = d.arg;
  const uint32_t idx = (hdr >> kOpIndexShift) & 0xffu;
#include "qt_variants.inc"
}

// ---- lean kernel: layer-word interpreter (qt_micro.cpp lowers the layers) ----

// diagonal table of unit phases: each e^{i phi_s} rotates (re, im) by three
// in-place shears (a, b) = (-tan(phi/2), sin(phi)), |phi| well inside pi
template <int R>
__device__ __forceinline__ void m_stab(double2 (&v)[1 << R], const double2* t) {
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    const double2 ab = t[s];
    v[s].x = fma(ab.x, v[s].y, v[s].x);
    v[s].y = fma(ab.y, v[s].x, v[s].y);
    v[s].x = fma(ab.x, v[s].y, v[s].x);
  }
}

template <int R>
__device__ __forceinline__ void m_ctab(double2 (&v)[1 << R], const double2* t) {
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    const double2 c = t[s];
    cscale(v[s], c.x, c.y);
  }
}

// Scaled rotation of the lean layer words (qt_micro.cpp push_rotation): two
// FMAs per real pair, the scale carried by the plan.
//   (t, 0):  x' = x - t y,  y' = y + t x        (c [[1, -t], [t, 1]])
//   (u, 1):  x' = u x - y,  y' = x + u y        (s [[u, -1], [1, u]])
template <int R, int A>
__device__ __forceinline__ void pair_srot(double2 (&v)[1 << R], double k, bool uform) {
  if (uform) {
#pragma unroll
    for (int s = 0; s < (1 << R); ++s) {
      if (s & (1 << A)) continue;
      const int s1 = s | (1 << A);
      const double2 x = v[s], y = v[s1];
      v[s].x = fma(k, x.x, -y.x);
      v[s].y = fma(k, x.y, -y.y);
      v[s1].x = fma(k, y.x, x.x);
      v[s1].y = fma(k, y.y, x.y);
    }
  } else {
#pragma unroll
    for (int s = 0; s < (1 << R); ++s) {
      if (s & (1 << A)) continue;
      const int s1 = s | (1 << A);
      const double2 x = v[s], y = v[s1];
      v[s].x = fma(-k, y.x, x.x);
      v[s].y = fma(-k, y.y, x.y);
      v[s1].x = fma(k, x.x, y.x);
      v[s1].y = fma(k, x.y, y.y);
    }
  }
}

template <int R, int A>
__device__ __forceinline__ void m_rots(double2 (&v)[1 << R], const double2*& q, uint32_t x) {
  if constexpr (A < R) {
    if (x & (1u << (M_ROT_SHIFT + A))) {
      const double2 ab = *q++;
      pair_srot<R, A>(v, ab.x, ab.y != 0.0);
    }
    m_rots<R, A + 1>(v, q, x);
  }
}

template <int R, int A>
__device__ __forceinline__ void m_denses(double2 (&v)[1 << R], const double2*& q, uint32_t x) {
  if constexpr (A < R) {
    if (x & (1u << (M_DENSE_SHIFT + A))) {
      const double2 m0 = q[0], m1 = q[1], m2 = q[2], m3 = q[3];
      q += 4;
      pair_dense<R, A, -1>(v, m0.x, m0.y, m1.x, m1.y, m2.x, m2.y, m3.x, m3.y);
    }
    m_denses<R, A + 1>(v, q, x);
  }
}

// Runs the layer words [o, o1) of a round. Each word's flag bits select the
// compiled bodies: [table (variant chosen by tile-uniform conditions)]
// [sign flips][rotation per slot][complex 2x2 per slot] (qt_ir.hpp).
template <int R, bool TD, typename P>
__device__ __forceinline__ void run_layers(double2 (&v)[1 << R], const P& p, uint32_t o,
                                           uint32_t jb, const uint64_t* sg) {
  constexpr int NS = 1 << R;
  const unsigned long long* mw = reinterpret_cast<const unsigned long long*>(p.ops);
  const double2* pl = reinterpret_cast<const double2*>(p.pool);
  // the round's words end with the one flagged M_LAST (no loop bound to keep)
  for (uint32_t x = 0; !(x & M_LAST); ++o) {
    const unsigned long long wv = mw[o];  // one 64-bit uniform load
    const uint2 w = make_uint2(static_cast<uint32_t>(wv), static_cast<uint32_t>(wv >> 32));
    x = w.x;
    uint32_t off = x & 0xffffu;  // doubles, even
    if (x & M_PERM) {
      DOp d{};
      d.lmask = static_cast<uint32_t>(__double_as_longlong(p.pool[off]));
      d.gmask = static_cast<uint64_t>(__double_as_longlong(p.pool[off + 1]));
      k_perm<R>(v, w.y, d, jb, sg);
      continue;
    }
    if (TD && (x & M_TDIAG)) {
      // a lone diagonal on a thread / tile bit (or a register slot under a
      // thread / tile control): per-thread predicates, uniform slot loop
      // (its own instantiation: the handler costs the lean loop registers)
      const uint32_t lm = static_cast<uint32_t>(__double_as_longlong(p.pool[off]));
      const uint32_t dl = static_cast<uint32_t>(__double_as_longlong(p.pool[off + 1]));
      const uint64_t gm = static_cast<uint64_t>(__double_as_longlong(p.pool[off + 2]));
      const uint64_t dg = static_cast<uint64_t>(__double_as_longlong(p.pool[off + 3]));
      const uint64_t g = *sg;
      if ((jb & lm) != lm || (g & gm) != gm) continue;
      const bool tb = (jb & dl) != 0 || (g & dg) != 0;
      const int ds = static_cast<int>((w.y >> 16) & 15u) - 1;
      const bool ph1 = (w.y & M_TD_PHASE1) != 0;
      // the factor is loaded per slot (short live range: the lean R = 3
      // instantiation stays within its 64 registers)
      const double2* dp = pl + (off >> 1) + 2;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        if (!((w.y >> s) & 1u)) continue;
        const bool b = ds >= 0 ? ((s >> ds) & 1) != 0 : tb;
        if (ph1 && !b) continue;
        const double2 d = dp[b ? 1 : 0];
        cscale(v[s], d.x, d.y);
      }
      continue;
    }
    if (x & (M_STAB | M_CTAB)) {
      const uint32_t nv = (x >> M_NV_SHIFT) & 3u;
      const double2* t = pl + (off >> 1) + nv;  // after nv (condition, slots) pairs
      if (x & M_STAB) m_stab<R>(v, t);
      else m_ctab<R>(v, t);
      if (nv) {
        // tile-uniform sign terms: negate the slots of every term whose
        // condition the tile's global bits meet (exact, so after the table)
        const uint64_t g = *sg;
        uint32_t fl = 0;
#pragma unroll
        for (uint32_t j = 0; j < kMaxTableVariantTerms; ++j) {
          if (j < nv) {
            const uint64_t gc = static_cast<uint64_t>(__double_as_longlong(p.pool[off + 2 * j]));
            if ((g & gc) == gc)
              fl ^= static_cast<uint32_t>(__double_as_longlong(p.pool[off + 2 * j + 1]));
          }
        }
        if (fl) {
#pragma unroll
          for (int s = 0; s < NS; ++s)
            if (fl & (1u << s)) v[s] = neg2(v[s]);
        }
      }
      off += 2 * nv + 2 * NS;
    }
    if (x & M_SIGN) {
      const uint32_t nt = w.y >> 16;
      apply_signs<R>(v, p, static_cast<int>(off), nt, w.y & 0xffffu, jb, sg);
      off += 2 * nt;
    }
    const double2* q = pl + (off >> 1);
    m_rots<R, 0>(v, q, x);
    if (x & (15u << M_DENSE_SHIFT)) m_denses<R, 0>(v, q, x);
  }
}

// R = 3: 8 amplitudes per thread in registers, up to 512 threads (2^12
// tiles) at <= 64 registers (32 warps per SM); R = 4: 16 amplitudes per
// thread, up to 256 threads (2^12 tiles) at <= 128 registers. The kernel is
// latency-bound at low occupancy, so the R = 3 bound trades registers for
// resident warps. R <= 2 runs only on tiny states (launch-bound): the same
// 64-register bound keeps its generic instantiations from spilling.
// kTileMaxThreads (qt_kernels.hpp) must match.
template <int R>
constexpr int kMinBlocks = 2;  // R <= 2 (tiny states) too: 64 registers, no spills
template <int R>
constexpr int kMaxThreads = R >= 4 ? 256 : 512;

// async 16-B global -> shared copy (LDGSTS, L1 bypass)
__device__ __forceinline__ void cp_async16(uint32_t sdst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sdst), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
// bulk L2 prefetch of `bytes` (multiple of 16) at a 16-B aligned address
__device__ __forceinline__ void prefetch_l2(const void* g, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint64_t next_tile_base(uint64_t base, uint64_t outer) {
  return ((base | ~outer) + 1) & outer;
}

// GENERIC = false: the lean instantiation: it runs the pass's layer words
// (qt_micro.cpp: table / sign / per-slot rotation and 2x2 bodies, X / CX
// permutations); every extra variant body costs registers and
// instruction cache in the hot loop, so passes made only of layer ops (e.g.
// every pass of config 3) run this one.
// PIPE = true: two smem tile buffers; tile i+1 streams in with cp.async
// (no register staging) while tile i runs its register rounds, so every CTA
// keeps a tile of loads in flight through its compute phase.
template <int R, int KM, bool PIPE, typename P>
__global__ void __launch_bounds__(kMaxThreads<R>, kMinBlocks<R>)
    tile_pass_kernel(double2* psi, const __grid_constant__ P p) {
  constexpr bool GENERIC = KM == kKernelGeneric;
  extern __shared__ double2 sm[];
  constexpr int NS = 1 << R;
  const KPassHead& h = p.h;
  const uint32_t t = threadIdx.x;

  // global offset of this thread's load slots: tile bits [0, k-R) from the
  // thread index (coalesced: low tile bits are the low physical bits), tile
  // bits [k-R, k) from the slot index (host-precomputed byte offsets
  // h.slot_gb, CTA-uniform)
  const uint64_t off_t = pdep64(t, h.lo_mask);
  // smem byte offset of the thread's slots: swz is GF(2)-linear, so
  // swz(t | s << (k-R)) * 16 = st4 ^ h.slot_sb[s]
  const uint32_t st4 = swz(t) << 4;
  // L2 prefetch of the next tile: the threads whose low pf_bits are zero
  // each cover one contiguous run per slot
  const bool pf_lead = h.pf_bits != 0 && (t & ((1u << h.pf_bits) - 1u)) == 0;
  const uint32_t pf_bytes = 16u << h.pf_bits;

  // per-tile uniform values live in smem while the register rounds run
  __shared__ uint64_t s_tile[2];  // [0] tile base, [1] global base (+ rank bits)

  // contiguous tile range per CTA; the tile base advances by a masked
  // increment over the outer (non-tile) bits
  const uint64_t per = (h.ntiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = uint64_t(blockIdx.x) * per;
  const uint64_t t1 = t0 + per < h.ntiles ? t0 + per : h.ntiles;
  uint64_t base = pdep64(t0, h.outer_mask);
  const uint32_t sm0 = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  const uint32_t tbytes = 16u << h.k;
  if (PIPE && t0 < t1) {
    const char* src = reinterpret_cast<const char*>(h.src + base + off_t);
#pragma unroll
    for (int s = 0; s < NS; ++s) cp_async16(sm0 + (st4 ^ h.slot_sb[s]), src + h.slot_gb[s]);
    cp_async_commit();
  }
  uint32_t cur = 0;  // PIPE: byte offset of the current buffer
  bool bad = false;
  for (uint64_t tile = t0; tile < t1; ++tile) {
    char* const smb = reinterpret_cast<char*>(sm) + cur;
    if (t == 0) {
      s_tile[0] = base;
      s_tile[1] = h.gbase_hi | base;
    }
    if (PIPE) {
      if (tile + 1 < t1) {
        const char* src = reinterpret_cast<const char*>(
            h.src + next_tile_base(base, h.outer_mask) + off_t);
        const uint32_t nb = sm0 + (cur ^ tbytes);
#pragma unroll
        for (int s = 0; s < NS; ++s) cp_async16(nb + (st4 ^ h.slot_sb[s]), src + h.slot_gb[s]);
        cp_async_commit();
        cp_async_wait<1>();
      } else {
        cp_async_wait<0>();
      }
    } else {
      const char* src = reinterpret_cast<const char*>(h.src + base + off_t);
      double2 ld[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s)
        ld[s] = __ldcs(reinterpret_cast<const double2*>(src + h.slot_gb[s]));
      if (pf_lead && tile + 1 < t1) {
        const char* nsrc = reinterpret_cast<const char*>(
            h.src + next_tile_base(base, h.outer_mask) + off_t);
#pragma unroll
        for (int s = 0; s < NS; ++s) prefetch_l2(nsrc + h.slot_gb[s], pf_bytes);
      }
#pragma unroll
      for (int s = 0; s < NS; ++s)
        *reinterpret_cast<double2*>(smb + (st4 ^ h.slot_sb[s])) = ld[s];
    }
    __syncthreads();

    for (uint32_t r = 0; r < h.nrounds; ++r) {
      const DRound& rd = p.rounds[r];
      // deposit t into the non-register tile bits (insert zeros ascending)
      uint32_t jb = t;
#pragma unroll
      for (int i = 0; i < R; ++i) jb = insert_zero(jb, rd.sreg[i]);
      // swz is GF(2)-linear: swz(jb | bits) * 16 = sj4 ^ (XOR of rd.sbit)
      const uint32_t sj4 = swz(jb) << 4;
      double2 v[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        uint32_t a = sj4;
#pragma unroll
        for (int i = 0; i < R; ++i)
          if (s & (1 << i)) a ^= rd.sbit[i];
        v[s] = *reinterpret_cast<const double2*>(smb + a);
      }
      const uint32_t o1 = uint32_t(rd.op_first) + rd.op_count;
      if constexpr (!GENERIC) {
        run_layers<R, KM == kKernelLeanTdiag>(v, p, rd.op_first, jb, &s_tile[1]);
      } else {
        // the next op's header is loaded while the current op runs (the
        // dispatch chain of an op starts from it; the op array always has a
        // readable slot after the last op: pool data follows it)
        uint32_t hdr = p.ops[rd.op_first].hdr;
        for (uint32_t o = rd.op_first; o < o1; ++o) {
          const uint32_t hdr_next = p.ops[o + 1].hdr;
          apply_op<R, GENERIC>(v, p, p.ops[o], hdr, jb, &s_tile[1]);
          hdr = hdr_next;
        }
      }
      // opaque copy: forces the 2^R store addresses to be regenerated here
      // instead of being kept live (2^R registers) across the op loop
      // (and the slot terms re-read from the constant bank)
      uint32_t sj4b = sj4, rr = r;
      asm volatile("" : "+r"(sj4b), "+r"(rr));
      const DRound& rd2 = p.rounds[rr];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        uint32_t a = sj4b;
#pragma unroll
        for (int i = 0; i < R; ++i)
          if (s & (1 << i)) a ^= rd2.sbit[i];
        *reinterpret_cast<double2*>(smb + a) = v[s];
      }
      __syncthreads();
    }

    base = s_tile[0];
    {
      char* dst = reinterpret_cast<char*>(psi + base + off_t);
      if (h.check) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const double2 x = *reinterpret_cast<const double2*>(smb + (st4 ^ h.slot_sb[s]));
          bad = bad || !finite2(x);
          __stcs(reinterpret_cast<double2*>(dst + h.slot_gb[s]), x);
        }
      } else {
#pragma unroll
        for (int s = 0; s < NS; ++s)
          __stcs(reinterpret_cast<double2*>(dst + h.slot_gb[s]),
                 *reinterpret_cast<const double2*>(smb + (st4 ^ h.slot_sb[s])));
      }
    }
    base = next_tile_base(base, h.outer_mask);
    if (PIPE) cur ^= tbytes;
    __syncthreads();  // smem reuse by the next tile
  }
  if (__syncthreads_or(bad) && t == 0) atomicOr(h.flag, 1);
}

template <typename P, int KM, bool PIPE>
void* kernel_ptr(int R) {
  switch (R) {
    case 1: return reinterpret_cast<void*>(&tile_pass_kernel<1, KM, PIPE, P>);
    case 2: return reinterpret_cast<void*>(&tile_pass_kernel<2, KM, PIPE, P>);
    case 3: return reinterpret_cast<void*>(&tile_pass_kernel<3, KM, PIPE, P>);
    default: return reinterpret_cast<void*>(&tile_pass_kernel<4, KM, PIPE, P>);
  }
}

template <typename P, int KM>
void* kernel_ptr(int R, bool pipe) {
  return pipe ? kernel_ptr<P, KM, true>(R) : kernel_ptr<P, KM, false>(R);
}

template <typename P>
void* kernel_ptr(int R, int kmode, bool pipe) {
  if (kmode == kKernelGeneric) return kernel_ptr<P, kKernelGeneric>(R, pipe);
  if (kmode == kKernelLeanTdiag) return kernel_ptr<P, kKernelLeanTdiag>(R, pipe);
  return kernel_ptr<P, kKernelLean>(R, pipe);
}

template <typename P, int KM, bool PIPE>
cudaError_t launch(double2* psi, const P& p, int grid, cudaStream_t s) {
  const size_t smem = (PIPE ? 2 : 1) * (sizeof(double2) << p.h.k);
  const int threads = 1 << (p.h.k - p.h.reg_bits);
  switch (p.h.reg_bits) {
    case 1:
      tile_pass_kernel<1, KM, PIPE, P><<<grid, threads, smem, s>>>(psi, p);
      break;
    case 2:
      tile_pass_kernel<2, KM, PIPE, P><<<grid, threads, smem, s>>>(psi, p);
      break;
    case 3:
      tile_pass_kernel<3, KM, PIPE, P><<<grid, threads, smem, s>>>(psi, p);
      break;
    default:
      tile_pass_kernel<4, KM, PIPE, P><<<grid, threads, smem, s>>>(psi, p);
      break;
  }
  return cudaGetLastError();
}

template <typename P, int KM>
cudaError_t launch_pipe(double2* psi, const P& p, int grid, bool pipe, cudaStream_t s) {
  return pipe ? launch<P, KM, true>(psi, p, grid, s) : launch<P, KM, false>(psi, p, grid, s);
}

template <typename P>
cudaError_t launch_any(double2* psi, const P& p, int grid, int kmode, bool pipe,
                       cudaStream_t s) {
  if (kmode == kKernelGeneric) return launch_pipe<P, kKernelGeneric>(psi, p, grid, pipe, s);
  if (kmode == kKernelLeanTdiag) return launch_pipe<P, kKernelLeanTdiag>(psi, p, grid, pipe, s);
  return launch_pipe<P, kKernelLean>(psi, p, grid, pipe, s);
}

}  // namespace

int tile_pass_occupancy(int k, int R, bool large, int kmode, bool pipe) {
  // per-device cache: (pipe, kmode, large, k, R) -> resident CTAs per SM
  static thread_local int cache_dev = -1;
  static thread_local int cache[12][kMaxTileBits + 1][kMaxRegBits + 1];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cache_dev) {
    for (auto& a : cache)
      for (auto& row : a)
        for (int& v : row) v = -1;
    cache_dev = dev;
  }
  int& slot = cache[(large ? 1 : 0) + 2 * kmode + (pipe ? 6 : 0)][k][R];
  if (slot >= 0) return slot;
  const size_t smem = (pipe ? 2 : 1) * (sizeof(double2) << k);
  const int threads = 1 << (k - R);
  void* fn = large ? kernel_ptr<KPassLarge>(R, kmode, pipe)
                   : kernel_ptr<KPassSmall>(R, kmode, pipe);
  int occ = 0;
  // the attribute is per function: always allow the largest tile (2^13
  // single-buffered, 2^12 double-buffered)
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(double2) << kMaxTileBits)) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) !=
          cudaSuccess) {
    cudaGetLastError();
    occ = 0;
  }
  slot = occ;
  return occ;
}

cudaError_t launch_tile_pass(double2* psi, const KPassSmall& p, int grid, int kmode,
                             bool pipe, cudaStream_t s) {
  return launch_any(psi, p, grid, kmode, pipe, s);
}

cudaError_t launch_tile_pass(double2* psi, const KPassLarge& p, int grid, int kmode,
                             bool pipe, cudaStream_t s) {
  return launch_any(psi, p, grid, kmode, pipe, s);
}

}  // namespace qtb
