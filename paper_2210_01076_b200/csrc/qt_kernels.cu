// qt_kernels.cu -- sm_100a kernels of the qTask hot path.
//
// The reference applies one gate per stage with two CPU loops:
// run_permute_tasks (engine.cpp:315-350: swap/scale element ops, one
// ElementOpSeq::op(k) per pair, element_ops.cpp:82-133) and
// run_mxv_partition (engine.cpp:352-383: Kronecker-row mat-vec over every
// superposition gate of a net, kron_row_visit plan.hpp:98-127). Both read
// and write host copy-on-write blocks.
//
// Here the whole gate sequence is applied by FUSED TILE PASSES. One pass
// streams the 2^n complex128 state through shared memory exactly once:
//   HBM --(16-B coalesced loads)--> smem tile of 2^k amplitudes
//       --> R-qubit register rounds: each thread holds 2^R amplitudes
//           (indices differing in the round's R tile bits) in registers
//           and applies every op of the round (2x2 dense/real, diagonal,
//           sign, bit-flip, swap; controls and diagonal targets anywhere)
//       --> smem --> HBM
// so a pass costs 32 B of HBM traffic per amplitude however many gates it
// carries. Tensor cores do not apply (2x2 complex FP64 operands); the
// kernel is bounded by HBM for shallow passes and by the FP64 pipe for deep
// ones ("Rooflines").
#include <cuda_runtime.h>

#include <cstdint>

#include "qt_kernels.hpp"

namespace qtb {

namespace {

// XOR swizzle of 16-B smem slots: folds every higher 3-bit group of the
// index onto the low 3 bits so lanes that differ in (almost any) three tile
// bits land in distinct 16-B bank groups. Linear over GF(2):
// swz(a | b) == swz(a) ^ swz(b) for disjoint a, b.
__device__ __forceinline__ uint32_t swz(uint32_t j) {
  return j ^ ((j >> 3) & 7u) ^ ((j >> 6) & 7u) ^ ((j >> 9) & 7u) ^
         ((j >> 12) & 7u);
}

// software parallel-bit-deposit: bit i of x goes to the i-th set bit of mask
__device__ __forceinline__ uint64_t pdep64(uint64_t x, uint64_t mask) {
  uint64_t r = 0;
  for (uint64_t b = 1; mask; b <<= 1) {
    const uint64_t low = mask & (~mask + 1);
    if (x & b) r |= low;
    mask ^= low;
  }
  return r;
}

__device__ __forceinline__ uint32_t insert_zero(uint32_t x, uint32_t p) {
  return ((x >> p) << (p + 1)) | (x & ((1u << p) - 1u));
}

__device__ __forceinline__ bool finite2(double2 v) {
  // exponent all-ones <=> inf/nan; integer test keeps the FP64 pipe free
  const uint32_t hx = __double2hiint(v.x), hy = __double2hiint(v.y);
  return ((hx & 0x7ff00000u) != 0x7ff00000u) &&
         ((hy & 0x7ff00000u) != 0x7ff00000u);
}

__device__ __forceinline__ double2 neg2(double2 v) {
  // sign flip with integer ops (no FP64 instruction)
  return make_double2(
      __hiloint2double(__double2hiint(v.x) ^ 0x80000000, __double2loint(v.x)),
      __hiloint2double(__double2hiint(v.y) ^ 0x80000000, __double2loint(v.y)));
}

__device__ __forceinline__ double2 cmulz(double2 a, double br, double bi) {
  return make_double2(a.x * br - a.y * bi, a.x * bi + a.y * br);
}

// Tile-local index of register slot s: the thread's base index with the
// round's register bits set from s (s is a compile-time constant after
// unrolling, so this is 0-3 ORs).
struct SlotIdx {
  uint32_t jb, r0, r1, r2;
  __device__ __forceinline__ uint32_t operator()(int s) const {
    return jb | ((s & 1) ? r0 : 0u) | ((s & 2) ? r1 : 0u) | ((s & 4) ? r2 : 0u);
  }
};

template <int NS, int A>
__device__ __forceinline__ void op_dense(double2 (&v)[NS],
                                         const SlotIdx& js,
                                         uint32_t lmask, bool gok,
                                         const double* __restrict__ m) {
  const double m0r = m[0], m0i = m[1], m1r = m[2], m1i = m[3];
  const double m2r = m[4], m2i = m[5], m3r = m[6], m3i = m[7];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (s & (1 << A)) continue;
    const int s1 = s | (1 << A);
    const bool ok = gok && ((js(s) & lmask) == lmask);
    const double2 a = v[s], b = v[s1];
    double2 na, nb;
    na.x = m0r * a.x - m0i * a.y + m1r * b.x - m1i * b.y;
    na.y = m0r * a.y + m0i * a.x + m1r * b.y + m1i * b.x;
    nb.x = m2r * a.x - m2i * a.y + m3r * b.x - m3i * b.y;
    nb.y = m2r * a.y + m2i * a.x + m3r * b.y + m3i * b.x;
    v[s] = ok ? na : a;
    v[s1] = ok ? nb : b;
  }
}

template <int NS, int A>
__device__ __forceinline__ void op_real(double2 (&v)[NS],
                                        const SlotIdx& js,
                                        uint32_t lmask, bool gok,
                                        const double* __restrict__ m) {
  const double m0 = m[0], m1 = m[2], m2 = m[4], m3 = m[6];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (s & (1 << A)) continue;
    const int s1 = s | (1 << A);
    const bool ok = gok && ((js(s) & lmask) == lmask);
    const double2 a = v[s], b = v[s1];
    double2 na, nb;
    na.x = m0 * a.x + m1 * b.x;
    na.y = m0 * a.y + m1 * b.y;
    nb.x = m2 * a.x + m3 * b.x;
    nb.y = m2 * a.y + m3 * b.y;
    v[s] = ok ? na : a;
    v[s1] = ok ? nb : b;
  }
}

template <int NS, int A>
__device__ __forceinline__ void op_xperm(double2 (&v)[NS],
                                         const SlotIdx& js,
                                         uint32_t lmask, bool gok) {
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (s & (1 << A)) continue;
    const int s1 = s | (1 << A);
    const bool ok = gok && ((js(s) & lmask) == lmask);
    const double2 a = v[s], b = v[s1];
    v[s] = ok ? b : a;
    v[s1] = ok ? a : b;
  }
}

template <int NS, int A>
__device__ __forceinline__ void op_anti(double2 (&v)[NS],
                                        const SlotIdx& js,
                                        uint32_t lmask, bool gok,
                                        const double* __restrict__ m) {
  const double m1r = m[2], m1i = m[3], m2r = m[4], m2i = m[5];
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (s & (1 << A)) continue;
    const int s1 = s | (1 << A);
    const bool ok = gok && ((js(s) & lmask) == lmask);
    const double2 a = v[s], b = v[s1];
    const double2 na = cmulz(b, m1r, m1i);
    const double2 nb = cmulz(a, m2r, m2i);
    v[s] = ok ? na : a;
    v[s1] = ok ? nb : b;
  }
}

template <int NS, int A, int B>
__device__ __forceinline__ void op_swap2(double2 (&v)[NS]) {
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if ((s & (1 << A)) && !(s & (1 << B))) {
      const int s2 = s ^ (1 << A) ^ (1 << B);
      const double2 t = v[s];
      v[s] = v[s2];
      v[s2] = t;
    }
  }
}

template <int NS>
__device__ __forceinline__ void apply_op(double2 (&v)[NS],
                                         const SlotIdx& js, uint64_t g,
                                         const DOp* __restrict__ opp) {
  const uint32_t type = opp->type;
  const uint32_t lmask = opp->lmask;
  const uint64_t gmask = opp->gmask;
  const bool gok = (g & gmask) == gmask;
  const double* m = opp->m;
  switch (type) {
    case D_DENSE:
    case D_REAL:
    case D_XPERM:
    case D_ANTI: {
      const uint32_t a = opp->a;
      constexpr int A1 = NS > 2 ? 1 : 0;
      constexpr int A2 = NS > 4 ? 2 : 0;
      if (type == D_DENSE) {
        if (a == 0) op_dense<NS, 0>(v, js, lmask, gok, m);
        else if (a == 1) op_dense<NS, A1>(v, js, lmask, gok, m);
        else op_dense<NS, A2>(v, js, lmask, gok, m);
      } else if (type == D_REAL) {
        if (a == 0) op_real<NS, 0>(v, js, lmask, gok, m);
        else if (a == 1) op_real<NS, A1>(v, js, lmask, gok, m);
        else op_real<NS, A2>(v, js, lmask, gok, m);
      } else if (type == D_XPERM) {
        if (a == 0) op_xperm<NS, 0>(v, js, lmask, gok);
        else if (a == 1) op_xperm<NS, A1>(v, js, lmask, gok);
        else op_xperm<NS, A2>(v, js, lmask, gok);
      } else {
        if (a == 0) op_anti<NS, 0>(v, js, lmask, gok, m);
        else if (a == 1) op_anti<NS, A1>(v, js, lmask, gok, m);
        else op_anti<NS, A2>(v, js, lmask, gok, m);
      }
      break;
    }
    case D_DIAG:
    case D_PHASE1:
    case D_SIGN: {
      const uint32_t dl = opp->dl;
      const bool gbit = (g & opp->dg) != 0;
      if (type == D_SIGN) {
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const bool ok = gok && ((js(s) & lmask) == lmask);
          const bool bit = gbit || (js(s) & dl) != 0;
          v[s] = (ok && bit) ? neg2(v[s]) : v[s];
        }
      } else if (type == D_PHASE1) {
        const double d1r = m[6], d1i = m[7];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const bool ok = gok && ((js(s) & lmask) == lmask);
          const bool bit = gbit || (js(s) & dl) != 0;
          const double2 w = cmulz(v[s], d1r, d1i);
          v[s] = (ok && bit) ? w : v[s];
        }
      } else {
        const double d0r = m[0], d0i = m[1], d1r = m[6], d1i = m[7];
#pragma unroll
        for (int s = 0; s < NS; ++s) {
          const bool ok = gok && ((js(s) & lmask) == lmask);
          const bool bit = gbit || (js(s) & dl) != 0;
          const double2 w = cmulz(v[s], bit ? d1r : d0r, bit ? d1i : d0i);
          v[s] = ok ? w : v[s];
        }
      }
      break;
    }
    case D_SWAP2: {
      if constexpr (NS >= 4) {
        uint32_t a = opp->a, b = opp->b;
        if (a > b) {
          const uint32_t t = a;
          a = b;
          b = t;
        }
        if (a == 0 && b == 1) op_swap2<NS, 0, 1>(v);
        if constexpr (NS >= 8) {
          if (a == 0 && b == 2) op_swap2<NS, 0, (NS >= 8 ? 2 : 1)>(v);
          if (a == 1 && b == 2) op_swap2<NS, 1, (NS >= 8 ? 2 : 1)>(v);
        }
      }
      break;
    }
    default:
      break;
  }
}

template <int R>
__global__ void __launch_bounds__(512, 2)
    tile_pass_kernel(double2* psi, const KPass p) {
  extern __shared__ double2 sm[];
  constexpr int NS = 1 << R;
  const uint32_t k = p.k;
  const uint32_t lo_bits = k - R;
  const uint32_t t = threadIdx.x;
  (void)k;

  // global offsets of this thread's load slots: tile bits [0, k-R) from the
  // thread index (coalesced: low tile bits are the low physical bits),
  // tile bits [k-R, k) from the slot index
  const uint64_t off_t = pdep64(t, p.lo_mask);
  // slot s adds the physical bits of tile bits k-R+i for the set bits i of s
  uint64_t hb[R];
  {
    uint64_t mk = p.hi_mask;
#pragma unroll
    for (int i = 0; i < R; ++i) {
      hb[i] = mk & (~mk + 1);
      mk ^= hb[i];
    }
  }
#define QT_OFF_S(s) (((s) & 1 ? hb[0] : 0) | (R > 1 && ((s) & 2) ? hb[R > 1 ? 1 : 0] : 0) | \
                     (R > 2 && ((s) & 4) ? hb[R > 2 ? 2 : 0] : 0))

  // contiguous tile range per CTA; the tile base advances by a masked
  // increment over the outer (non-tile) bits
  const uint64_t per = (p.ntiles + gridDim.x - 1) / gridDim.x;
  const uint64_t t0 = uint64_t(blockIdx.x) * per;
  const uint64_t t1 = t0 + per < p.ntiles ? t0 + per : p.ntiles;
  uint64_t base = pdep64(t0, p.outer_mask);
  bool bad = false;
  for (uint64_t tile = t0; tile < t1; ++tile,
                base = ((base | ~p.outer_mask) + 1) & p.outer_mask) {
    const uint64_t g = p.gbase_hi | base;
    const double2* src = p.src + base + off_t;
    double2* dst = psi + base + off_t;

    double2 ld[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) ld[s] = __ldcs(src + QT_OFF_S(s));
#pragma unroll
    for (int s = 0; s < NS; ++s) sm[swz(t | (uint32_t(s) << lo_bits))] = ld[s];
    __syncthreads();

    for (uint32_t r = 0; r < p.nrounds; ++r) {
      const DRound rd = p.rounds[r];
      uint32_t rb[R];
#pragma unroll
      for (int i = 0; i < R; ++i) rb[i] = rd.reg[i];
      // sorted copy for the zero-insertion deposit of t
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
      SlotIdx js;
      js.jb = jb;
      js.r0 = 1u << rb[0];
      js.r1 = R > 1 ? 1u << rb[R > 1 ? 1 : 0] : 0u;
      js.r2 = R > 2 ? 1u << rb[R > 2 ? 2 : 0] : 0u;
      // swizzled smem slot of register slot s: swz is GF(2)-linear, so
      // swz(jb | bits) = swz(jb) ^ swz(bits): 4 registers regenerate all 8
      const uint32_t sjb = swz(jb), sr0 = swz(js.r0), sr1 = swz(js.r1),
                     sr2 = swz(js.r2);
#define QT_SADDR(s) (sjb ^ (((s) & 1) ? sr0 : 0u) ^ (((s) & 2) ? sr1 : 0u) ^ \
                     (((s) & 4) ? sr2 : 0u))
      double2 v[NS];
#pragma unroll
      for (int s = 0; s < NS; ++s) v[s] = sm[QT_SADDR(s)];
      const DOp* __restrict__ op = p.ops + rd.op_first;
      for (uint32_t o = 0; o < rd.op_count; ++o) apply_op<NS>(v, js, g, op + o);
#pragma unroll
      for (int s = 0; s < NS; ++s) sm[QT_SADDR(s)] = v[s];
#undef QT_SADDR
      __syncthreads();
    }

#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const double2 x = sm[swz(t | (uint32_t(s) << lo_bits))];
      bad = bad || !finite2(x);
      __stcs(dst + QT_OFF_S(s), x);
    }
    __syncthreads();  // smem reuse by the next tile
  }
  if (__syncthreads_or(bad) && t == 0) atomicOr(p.flag, 1);
#undef QT_OFF_S
}

__global__ void set_basis_kernel(double2* __restrict__ psi, uint64_t n,
                                 uint64_t index) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride)
    psi[i] = make_double2(i == index ? 1.0 : 0.0, 0.0);
}

// level 1: block b sums the contiguous range [b*chunk, (b+1)*chunk) with a
// fixed per-thread stride order and a fixed tree; level 2 sums the block
// partials in a fixed tree. Same n -> same bits, run to run.
__global__ void norm_level1(const double2* __restrict__ psi, uint64_t n,
                            double* __restrict__ partial) {
  __shared__ double red[256];
  const uint64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const uint64_t lo = uint64_t(blockIdx.x) * chunk;
  const uint64_t hi = lo + chunk < n ? lo + chunk : n;
  double acc = 0.0;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double2 v = psi[i];
    acc += v.x * v.x + v.y * v.y;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void norm_level2(const double* __restrict__ partial, int np,
                            double* __restrict__ out) {
  __shared__ double red[1024];
  double acc = 0.0;
  for (int i = threadIdx.x; i < np; i += blockDim.x) acc += partial[i];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = red[0];
}

__global__ void bitswap_kernel(double2* __restrict__ psi, uint64_t pairs,
                               int b1, int b2) {
  // enumerate x with bit b1 = 1, bit b2 = 0 (b1 < b2); partner x ^ both
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
       k < pairs; k += stride) {
    uint64_t x = ((k >> b1) << (b1 + 1)) | (k & ((1ull << b1) - 1));
    x = ((x >> b2) << (b2 + 1)) | (x & ((1ull << b2) - 1));
    x |= 1ull << b1;
    const uint64_t y = x ^ (1ull << b1) ^ (1ull << b2);
    const double2 a = psi[x], b = psi[y];
    psi[x] = b;
    psi[y] = a;
  }
}

struct PermArg {
  uint8_t p[64];
};

__global__ void gather_kernel(const double2* __restrict__ psi,
                              double2* __restrict__ out, uint64_t first,
                              uint64_t count, PermArg perm, int nq) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
       i < count; i += stride) {
    const uint64_t l = first + i;
    uint64_t ph = 0;
    for (int q = 0; q < nq; ++q)
      if ((l >> q) & 1ull) ph |= 1ull << perm.p[q];
    out[i] = psi[ph];
  }
}

__global__ void gather_shard_kernel(const double2* __restrict__ psi,
                                    double2* __restrict__ out, uint64_t first,
                                    uint64_t count, PermArg perm, int nq,
                                    int nlocal, uint64_t rank) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  const uint64_t lmask = (1ull << nlocal) - 1;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
       i < count; i += stride) {
    const uint64_t l = first + i;
    uint64_t ph = 0;
    for (int q = 0; q < nq; ++q)
      if ((l >> q) & 1ull) ph |= 1ull << perm.p[q];
    out[i] = (ph >> nlocal) == rank ? psi[ph & lmask] : make_double2(0.0, 0.0);
  }
}

__global__ void fp64_probe_kernel(double* out, int iters) {
  double a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  const double b = 0.999999999, c = 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.678) out[0] = s;  // keep the chains alive
}

__global__ void check_finite_kernel(const double2* __restrict__ psi,
                                    uint64_t n, int* flag) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  bool bad = false;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride)
    bad = bad || !finite2(psi[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

int grid_for(uint64_t work, int block) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t want = (work + block - 1) / block;
  const uint64_t cap = uint64_t(sms) * 8;
  return static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap);
}

}  // namespace

static void* tile_kernel_ptr(int R) {
  switch (R) {
    case 1: return reinterpret_cast<void*>(&tile_pass_kernel<1>);
    case 2: return reinterpret_cast<void*>(&tile_pass_kernel<2>);
    default: return reinterpret_cast<void*>(&tile_pass_kernel<3>);
  }
}

int tile_pass_occupancy(int k, int R) {
  // per-device cache: (k, R) -> resident CTAs per SM
  static thread_local int cache_dev = -1;
  static thread_local int cache[kMaxTileBits + 1][kMaxRegBits + 1];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cache_dev) {
    for (auto& row : cache)
      for (int& v : row) v = -1;
    cache_dev = dev;
  }
  if (cache[k][R] >= 0) return cache[k][R];
  const size_t smem = sizeof(double2) << k;
  const int threads = 1 << (k - R);
  void* fn = tile_kernel_ptr(R);
  int occ = 0;
  // the attribute is per function: always allow the largest tile (2^13)
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(double2) << 13)) != cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem) !=
          cudaSuccess) {
    cudaGetLastError();
    occ = 1;
  }
  cache[k][R] = occ;
  return occ;
}

cudaError_t launch_tile_pass(double2* psi, const KPass& p, int grid,
                             cudaStream_t s) {
  const size_t smem = sizeof(double2) << p.k;
  const int threads = 1 << (p.k - p.reg_bits);
  switch (p.reg_bits) {
    case 1:
      tile_pass_kernel<1><<<grid, threads, smem, s>>>(psi, p);
      break;
    case 2:
      tile_pass_kernel<2><<<grid, threads, smem, s>>>(psi, p);
      break;
    default:
      tile_pass_kernel<3><<<grid, threads, smem, s>>>(psi, p);
      break;
  }
  return cudaGetLastError();
}

cudaError_t launch_set_basis(double2* psi, uint64_t n, uint64_t index,
                             cudaStream_t s) {
  set_basis_kernel<<<grid_for(n, 256), 256, 0, s>>>(psi, n, index);
  return cudaGetLastError();
}

cudaError_t launch_norm(const double2* psi, uint64_t n, double* scratch,
                        double* out, cudaStream_t s) {
  norm_level1<<<kNormBlocks, 256, 0, s>>>(psi, n, scratch);
  norm_level2<<<1, 1024, 0, s>>>(scratch, kNormBlocks, out);
  return cudaGetLastError();
}

cudaError_t launch_bitswap(double2* psi, int nbits, int b1, int b2,
                           cudaStream_t s) {
  if (b1 > b2) {
    const int t = b1;
    b1 = b2;
    b2 = t;
  }
  const uint64_t pairs = 1ull << (nbits - 2);
  bitswap_kernel<<<grid_for(pairs, 256), 256, 0, s>>>(psi, pairs, b1, b2);
  return cudaGetLastError();
}

cudaError_t launch_gather(const double2* psi, double2* out, uint64_t first,
                          uint64_t count, const uint8_t* perm_host, int nq,
                          cudaStream_t s) {
  PermArg pa{};
  for (int q = 0; q < nq && q < 64; ++q) pa.p[q] = perm_host[q];
  gather_kernel<<<grid_for(count, 256), 256, 0, s>>>(psi, out, first, count,
                                                     pa, nq);
  return cudaGetLastError();
}

cudaError_t launch_gather_shard(const double2* psi, double2* out,
                                uint64_t first, uint64_t count,
                                const uint8_t* perm_host, int nq, int nlocal,
                                uint64_t rank, cudaStream_t s) {
  PermArg pa{};
  for (int q = 0; q < nq && q < 64; ++q) pa.p[q] = perm_host[q];
  gather_shard_kernel<<<grid_for(count, 256), 256, 0, s>>>(
      psi, out, first, count, pa, nq, nlocal, rank);
  return cudaGetLastError();
}

cudaError_t launch_fp64_probe(double* out, int grid, int block, int iters,
                              cudaStream_t s) {
  fp64_probe_kernel<<<grid, block, 0, s>>>(out, iters);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(const double2* psi, uint64_t n, int* flag,
                                cudaStream_t s) {
  check_finite_kernel<<<grid_for(n, 256), 256, 0, s>>>(psi, n, flag);
  return cudaGetLastError();
}

}  // namespace qtb
