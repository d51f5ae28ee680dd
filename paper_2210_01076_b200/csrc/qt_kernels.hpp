// qt_kernels.hpp -- host-callable launchers of the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "qt_ir.hpp"

namespace qtb {

// Header of one tile-pass launch.
struct KPassHead {
  uint32_t k;          // tile bits
  uint32_t nrounds;
  uint32_t nops;
  uint32_t reg_bits;   // R
  uint64_t ntiles;
  uint64_t gbase_hi;   // shard offset in the global index (rank << nlocal)
  uint64_t lo_mask;    // physical bits of tile bits [0, k-R)  (thread bits)
  uint64_t hi_mask;    // physical bits of tile bits [k-R, k)  (load slots)
  uint64_t outer_mask; // buffer bits outside the tile
  const double2* src;  // tiles are read from src and written to psi (may alias)
  int* flag;           // set to 1 if any written amplitude is non-finite
  // 1: check the written amplitudes for inf/nan. Only the last tile pass of a
  // launch sequence checks: a non-finite amplitude never becomes finite again
  // under the (finite, linear) gate ops, so the final state shows it.
  uint32_t check;
  // > 0: while a tile is processed, the CTA prefetches its NEXT tile into L2
  // (cp.async.bulk.prefetch) as runs of 2^pf_bits contiguous amplitudes
  // (the tile's lowest physical bits are 0 .. pf_bits-1); 0 = off
  uint32_t pf_bits;
  uint64_t slot_gb[1 << kMaxRegBits];  // byte offset of load slot s (s deposited into hi_mask)
  uint32_t slot_sb[1 << kMaxRegBits];  // swz(s << (k - R)) * 16: smem byte term of slot s
};

// Kernel parameters (passed by value as a __grid_constant__: the rounds and
// ops are read from the constant bank, uniformly across the CTA).
template <int OPS, int ROUNDS, int POOL>
struct KPass {
  KPassHead h;
  DRound rounds[ROUNDS];
  // generic kernel: device ops; lean kernel: the same bytes hold the pass's
  // micro-ops (uint2, 4 per DOp slot; DRound op_first / op_count index them)
  DOp ops[OPS];
  alignas(16) double pool[POOL];  // matrices, diagonal tables, sign terms
};
using KPassSmall = KPass<kSmallOps, kSmallRounds, kSmallPool>;
using KPassLarge = KPass<kLargeOps, kLargeRounds, kLargePool>;
static_assert(sizeof(KPassLarge) <= 32764, "kernel parameter limit");
// micro-op capacity of a launch (lean kernel)
template <typename P>
constexpr int micro_capacity() { return static_cast<int>(sizeof(P::ops) / 8); }

// Fused tile pass over a state of 2^nlocal amplitudes. generic = false
// selects the lean instantiation that only handles the fused layer ops
// (MULTI, MULTIR, DTAB, STAB).
// kmode: kKernelLean (layer words), kKernelLeanTdiag (layer words incl.
// M_TDIAG: its handler costs the lean loop registers, so it has its own
// instantiation) or kKernelGeneric (device ops). pipe = true: the
// double-buffered instantiation (the next tile is copied into a second smem
// buffer with cp.async while the current one is worked on; 2x the dynamic
// shared memory).
constexpr int kKernelLean = 0, kKernelGeneric = 1, kKernelLeanTdiag = 2;
cudaError_t launch_tile_pass(double2* psi, const KPassSmall& p, int grid, int kmode,
                             bool pipe, cudaStream_t s);
cudaError_t launch_tile_pass(double2* psi, const KPassLarge& p, int grid, int kmode,
                             bool pipe, cudaStream_t s);
// Max threads per CTA of the tile-pass kernel for R register bits (its
// launch bounds): a pass's tile has at most R + log2(this) bits.
constexpr int tile_max_threads(int R) { return R >= 4 ? 256 : 512; }
// Max resident CTAs per SM of the tile-pass kernel for (k, R).
int tile_pass_occupancy(int k, int R, bool large, int kmode, bool pipe);

// Sets every amplitude to 0 and amplitude `index` to 1.
cudaError_t launch_set_basis(double2* psi, uint64_t n, uint64_t index,
                             cudaStream_t s);
// Deterministic sum of |a|^2 in two fixed-shape levels; result to *out
// (device). scratch must hold kNormBlocks doubles.
constexpr int kNormBlocks = 1184;  // 8 x 148 SMs
cudaError_t launch_norm(const double2* psi, uint64_t n, double* scratch,
                        double* out, cudaStream_t s);
// Swaps physical index bits b1 < b2 of a 2^nbits vector in place.
// Copies the runs of an exchange's own region (State::exchange, two-buffer
// scheme): offsets pdep(r, above) | vpat, 2^run_bits amplitudes each.
cudaError_t launch_copy_runs(double2* dst, const double2* src, uint64_t above, uint64_t vpat,
                             int run_bits, uint64_t total, cudaStream_t s);
cudaError_t launch_bitswap(double2* psi, int nbits, int b1, int b2,
                           cudaStream_t s);
// out[i] = psi[phys(first + i)] where phys permutes logical index bits by
// perm (logical bit q -> physical bit perm[q]); nq <= 64.
cudaError_t launch_gather(const double2* psi, double2* out, uint64_t first,
                          uint64_t count, const uint8_t* perm_host, int nq,
                          cudaStream_t s);
// Sharded variant: physical index ph = perm(l); out = psi[ph & local mask]
// if ph >> nlocal == rank, else 0.
cudaError_t launch_gather_shard(const double2* psi, double2* out,
                                uint64_t first, uint64_t count,
                                const uint8_t* perm_host, int nq, int nlocal,
                                uint64_t rank, cudaStream_t s);
// FP64 throughput probe: iters x 16 independent FMA chains per thread.
cudaError_t launch_fp64_probe(double* out, int grid, int block, int iters,
                              cudaStream_t s);
// ---- top-K by |a|^2 (qt_state.cpp State::top_k drives these) ----
constexpr int kTopkBits = 11;
constexpr int kTopkBins = 1 << kTopkBits;
struct TopkItem {
  uint64_t index;  // logical index (chunk base + position)
  uint64_t key;    // bits of |a|^2 (std::norm, no FMA)
  double2 amp;
};
// hist[(key >> shift) & (bins-1)] += 1 for keys with (key & pmask) == prefix
cudaError_t launch_topk_hist(const double2* psi, uint64_t count, uint64_t prefix,
                             uint64_t pmask, int shift, unsigned long long* hist,
                             cudaStream_t s);
// appends every amplitude with key >= lo (at most cap written)
cudaError_t launch_topk_collect(const double2* psi, uint64_t count, uint64_t base, uint64_t lo,
                                TopkItem* out, unsigned long long* n, uint64_t cap,
                                cudaStream_t s);
// per-block (fixed partition of `per` amplitudes) counts of key == t
cudaError_t launch_topk_ties(const double2* psi, uint64_t count, uint64_t per, int blocks,
                             uint64_t t, unsigned long long* ties, cudaStream_t s);
// keys > t appended into out[0, n_gt); the first r keys == t in index order
// into out[n_gt + rank] (tie_off = exclusive prefix of the tie counts)
cudaError_t launch_topk_final(const double2* psi, uint64_t count, uint64_t per, int blocks,
                              uint64_t base, uint64_t t, uint64_t r, uint64_t n_gt,
                              const unsigned long long* tie_off, TopkItem* out,
                              unsigned long long* n, cudaStream_t s);

// Checks a range for non-finite values (flag |= 1).
cudaError_t launch_check_finite(const double2* psi, uint64_t n, int* flag,
                                cudaStream_t s);

}  // namespace qtb
