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
//           every op of the round
//       --> smem --> HBM
// so a pass costs 32 B of HBM traffic per amplitude however many gates it
// carries. Ops live in the kernel-parameter constant bank and each op is
// dispatched (one switch per op) to a fully specialised variant: target,
// control and diagonal-target register slots are template parameters, so no
// per-amplitude predication is executed; controls / diagonal bits outside the
// register slots are thread- or tile-uniform predicates. Tensor cores do not
// apply (2x2 complex FP64 operands): a pass is bounded by HBM when shallow
// and by the FP64 pipe when deep ("Rooflines").
#include <cuda_runtime.h>

#include <cstdint>

#include "qt_device.cuh"
#include "qt_kernels.hpp"

namespace qtb {

namespace {

// ---- op variants (R register bits, NS = 2^R slots per thread) -------------

#define QT_LD_M                                            \
  const double m0r = op.m[0], m0i = op.m[1], m1r = op.m[2], \
               m1i = op.m[3], m2r = op.m[4], m2i = op.m[5], \
               m3r = op.m[6], m3i = op.m[7]

template <int R, int A, int CS>
__device__ __forceinline__ void k_dense(double2 (&v)[1 << R], const DOp& op) {
  QT_LD_M;
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (s & (1 << A)) continue;
    if (CS >= 0 && !(s & (1 << CS))) continue;
    const int s1 = s | (1 << A);
    const double2 a = v[s], b = v[s1];
    v[s].x = m0r * a.x - m0i * a.y + m1r * b.x - m1i * b.y;
    v[s].y = m0r * a.y + m0i * a.x + m1r * b.y + m1i * b.x;
    v[s1].x = m2r * a.x - m2i * a.y + m3r * b.x - m3i * b.y;
    v[s1].y = m2r * a.y + m2i * a.x + m3r * b.y + m3i * b.x;
  }
}

template <int R, int A, int CS>
__device__ __forceinline__ void k_real(double2 (&v)[1 << R], const DOp& op) {
  const double m0 = op.m[0], m1 = op.m[2], m2 = op.m[4], m3 = op.m[6];
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (s & (1 << A)) continue;
    if (CS >= 0 && !(s & (1 << CS))) continue;
    const int s1 = s | (1 << A);
    const double2 a = v[s], b = v[s1];
    v[s].x = m0 * a.x + m1 * b.x;
    v[s].y = m0 * a.y + m1 * b.y;
    v[s1].x = m2 * a.x + m3 * b.x;
    v[s1].y = m2 * a.y + m3 * b.y;
  }
}

template <int R, int A, int CS>
__device__ __forceinline__ void k_xperm(double2 (&v)[1 << R]) {
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (s & (1 << A)) continue;
    if (CS >= 0 && !(s & (1 << CS))) continue;
    const int s1 = s | (1 << A);
    const double2 t = v[s];
    v[s] = v[s1];
    v[s1] = t;
  }
}

template <int R, int A, int CS>
__device__ __forceinline__ void k_anti(double2 (&v)[1 << R], const DOp& op) {
  const double m1r = op.m[2], m1i = op.m[3], m2r = op.m[4], m2i = op.m[5];
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (s & (1 << A)) continue;
    if (CS >= 0 && !(s & (1 << CS))) continue;
    const int s1 = s | (1 << A);
    const double2 a = v[s], b = v[s1];
    v[s] = cmulz(b, m1r, m1i);
    v[s1] = cmulz(a, m2r, m2i);
  }
}

// diag(d0, d1) on a bit: DS >= 0 -> register slot bit DS (compile-time
// choice per slot); DS < 0 -> the thread-uniform bit `bit`.
template <int R, int CS, int DS>
__device__ __forceinline__ void k_diag(double2 (&v)[1 << R], const DOp& op,
                                       bool bit) {
  const double d0r = op.m[0], d0i = op.m[1], d1r = op.m[6], d1i = op.m[7];
  const double ur = bit ? d1r : d0r, ui = bit ? d1i : d0i;
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (CS >= 0 && !(s & (1 << CS))) continue;
    if (DS >= 0) {
      if (s & (1 << DS)) v[s] = cmulz(v[s], d1r, d1i);
      else v[s] = cmulz(v[s], d0r, d0i);
    } else {
      v[s] = cmulz(v[s], ur, ui);
    }
  }
}

// diag(1, d1): only amplitudes whose bit is set are touched
template <int R, int CS, int DS>
__device__ __forceinline__ void k_phase1(double2 (&v)[1 << R], const DOp& op,
                                         bool bit) {
  const double d1r = op.m[6], d1i = op.m[7];
  if (DS < 0 && !bit) return;
#pragma unroll
  for (int s = 0; s < (1 << R); ++s) {
    if (CS >= 0 && !(s & (1 << CS))) continue;
    if (DS >= 0 && !(s & (1 << DS))) continue;
    v[s] = cmulz(v[s], d1r, d1i);
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
    if ((s & (1 << A)) && !(s & (1 << B))) {
      const int s2 = s ^ (1 << A) ^ (1 << B);
      const double2 t = v[s];
      v[s] = v[s2];
      v[s2] = t;
    }
  }
}

// Applies one op. `jb` = the thread's tile-local index with the register
// bits cleared, `g` = the tile's global base index.
template <int R>
__device__ __forceinline__ void apply_op(double2 (&v)[1 << R], const DOp& op,
                                         uint32_t jb, const uint64_t* sg) {
  // thread-uniform control predicate (controls outside the register slots);
  // the tile's global base is read from smem only by ops that need it
  if ((jb & op.lmask) != op.lmask) return;
  bool bit = (jb & op.dl) != 0;
  if ((op.gmask | op.dg) != 0) {
    const uint64_t g = *sg;
    if ((g & op.gmask) != op.gmask) return;
    bit = bit || (g & op.dg) != 0;
  }
  (void)bit;
  switch (op.variant) {
#include "qt_variants.inc"
    default:
      break;
  }
}

// R = 4 (the default): 16 amplitudes per thread in registers, 256 threads
// per 2^12-amplitude tile, <= 128 registers so two CTAs (64 KiB smem each)
// stay resident per SM -- one streams its tile while the other computes.
template <int R>
constexpr int kMinBlocks = R >= 4 ? 2 : (R == 3 ? 2 : 4);
template <int R>
constexpr int kMaxThreads = R >= 4 ? 256 : 512;

template <int R, typename P>
__global__ void __launch_bounds__(kMaxThreads<R>, kMinBlocks<R>)
    tile_pass_kernel(double2* psi, const __grid_constant__ P p) {
  extern __shared__ double2 sm[];
  constexpr int NS = 1 << R;
  const KPassHead& h = p.h;
  const uint32_t lo_bits = h.k - R;
  const uint32_t t = threadIdx.x;

  // global offsets of this thread's load slots: tile bits [0, k-R) from the
  // thread index (coalesced: low tile bits are the low physical bits), tile
  // bits [k-R, k) from the slot index
  const uint64_t off_t = pdep64(t, h.lo_mask);
  // the R physical bits of the slot index (CTA-uniform)
  uint32_t hpos[R];
  {
    uint64_t mk = h.hi_mask;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      hpos[i] = static_cast<uint32_t>(__ffsll(static_cast<long long>(mk)) - 1);
      mk &= mk - 1;
    }
  }
#define QT_SLOT_OFF(s)                                   \
  ([&] {                                                 \
    uint64_t o_ = 0;                                     \
    _Pragma("unroll") for (int i_ = 0; i_ < R; ++i_) if ((s) & (1 << i_)) o_ |= 1ull << hpos[i_]; \
    return o_;                                           \
  }())

  // per-tile uniform values live in smem while the register rounds run
  __shared__ uint64_t s_tile[2];  // [0] tile base, [1] global base (+ rank bits)

  // contiguous tile range per CTA; the tile base advances by a masked
  // increment over the outer (non-tile) bits
  const uint64_t per = (h.ntiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = uint64_t(blockIdx.x) * per;
  const uint64_t t1 = t0 + per < h.ntiles ? t0 + per : h.ntiles;
  uint64_t base = pdep64(t0, h.outer_mask);
  bool bad = false;
  for (uint64_t tile = t0; tile < t1; ++tile) {
    if (t == 0) {
      s_tile[0] = base;
      s_tile[1] = h.gbase_hi | base;
    }
    {
      const double2* src = h.src + base + off_t;
      double2 ld[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) ld[s] = __ldcs(src + QT_SLOT_OFF(s));
#pragma unroll
      for (int s = 0; s < NS; ++s) sm[swz(t | (uint32_t(s) << lo_bits))] = ld[s];
    }
    __syncthreads();

    for (uint32_t r = 0; r < h.nrounds; ++r) {
      const DRound rd = p.rounds[r];
      uint32_t rb[R];
#pragma unroll
      for (int i = 0; i < R; ++i) rb[i] = rd.reg[i];
      // deposit t into the non-register tile bits (insert zeros ascending)
      uint32_t sr[R];
#pragma unroll
      for (int i = 0; i < R; ++i) sr[i] = rb[i];
#pragma unroll
      for (int i = 0; i < R; ++i)
#pragma unroll
        for (int j2 = i + 1; j2 < R; ++j2)
          if (sr[j2] < sr[i]) {
            const uint32_t tmp = sr[i];
            sr[i] = sr[j2];
            sr[j2] = tmp;
          }
      uint32_t jb = t;
#pragma unroll
      for (int i = 0; i < R; ++i) jb = insert_zero(jb, sr[i]);
      // swz is GF(2)-linear: swz(jb | bits) = swz(jb) ^ swz(bits)
      const uint32_t sjb = swz(jb);
      uint32_t srb[R];
#pragma unroll
      for (int i = 0; i < R; ++i) srb[i] = swz(1u << rb[i]);
      double2 v[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        uint32_t a = sjb;
#pragma unroll
        for (int i = 0; i < R; ++i)
          if (s & (1 << i)) a ^= srb[i];
        v[s] = sm[a];
      }
      const uint32_t o1 = uint32_t(rd.op_first) + rd.op_count;
      for (uint32_t o = rd.op_first; o < o1; ++o) apply_op<R>(v, p.ops[o], jb, &s_tile[1]);
      // opaque copy: forces the 2^R store addresses to be regenerated here
      // instead of being kept live (2^R registers) across the op loop
      uint32_t sjb2 = sjb;
      asm volatile("" : "+r"(sjb2));
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        uint32_t a = sjb2;
#pragma unroll
        for (int i = 0; i < R; ++i)
          if (s & (1 << i)) a ^= srb[i];
        sm[a] = v[s];
      }
      __syncthreads();
    }

    base = s_tile[0];
    {
      double2* dst = psi + base + off_t;
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const double2 x = sm[swz(t | (uint32_t(s) << lo_bits))];
        bad = bad || !finite2(x);
        __stcs(dst + QT_SLOT_OFF(s), x);
      }
    }
    base = ((base | ~h.outer_mask) + 1) & h.outer_mask;
    __syncthreads();  // smem reuse by the next tile
  }
#undef QT_SLOT_OFF
  if (__syncthreads_or(bad) && t == 0) atomicOr(h.flag, 1);
}

template <typename P>
void* kernel_ptr(int R) {
  switch (R) {
    case 1: return reinterpret_cast<void*>(&tile_pass_kernel<1, P>);
    case 2: return reinterpret_cast<void*>(&tile_pass_kernel<2, P>);
    case 3: return reinterpret_cast<void*>(&tile_pass_kernel<3, P>);
    default: return reinterpret_cast<void*>(&tile_pass_kernel<4, P>);
  }
}

template <typename P>
cudaError_t launch(double2* psi, const P& p, int grid, cudaStream_t s) {
  const size_t smem = sizeof(double2) << p.h.k;
  const int threads = 1 << (p.h.k - p.h.reg_bits);
  switch (p.h.reg_bits) {
    case 1:
      tile_pass_kernel<1, P><<<grid, threads, smem, s>>>(psi, p);
      break;
    case 2:
      tile_pass_kernel<2, P><<<grid, threads, smem, s>>>(psi, p);
      break;
    case 3:
      tile_pass_kernel<3, P><<<grid, threads, smem, s>>>(psi, p);
      break;
    default:
      tile_pass_kernel<4, P><<<grid, threads, smem, s>>>(psi, p);
      break;
  }
  return cudaGetLastError();
}

}  // namespace

int tile_pass_occupancy(int k, int R, bool large) {
  // per-device cache: (large, k, R) -> resident CTAs per SM
  static thread_local int cache_dev = -1;
  static thread_local int cache[2][kMaxTileBits + 1][kMaxRegBits + 1];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cache_dev) {
    for (auto& a : cache)
      for (auto& row : a)
        for (int& v : row) v = -1;
    cache_dev = dev;
  }
  int& slot = cache[large ? 1 : 0][k][R];
  if (slot >= 0) return slot;
  const size_t smem = sizeof(double2) << k;
  const int threads = 1 << (k - R);
  void* fn = large ? kernel_ptr<KPassLarge>(R) : kernel_ptr<KPassSmall>(R);
  int occ = 0;
  // the attribute is per function: always allow the largest tile (2^13)
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(double2) << kMaxTileBits)) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) !=
          cudaSuccess) {
    cudaGetLastError();
    occ = 1;
  }
  slot = occ;
  return occ;
}

cudaError_t launch_tile_pass(double2* psi, const KPassSmall& p, int grid,
                             cudaStream_t s) {
  return launch(psi, p, grid, s);
}

cudaError_t launch_tile_pass(double2* psi, const KPassLarge& p, int grid,
                             cudaStream_t s) {
  return launch(psi, p, grid, s);
}

}  // namespace qtb
