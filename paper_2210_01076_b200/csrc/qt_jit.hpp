// qt_jit.hpp -- compiled tile passes (host).
//
// The lean tile kernel interprets layer words (qt_micro.cpp): every op pays
// a dispatch, and every matrix / table constant a uniform constant load. A
// circuit that is simulated more than once can instead be compiled: each
// lowered pass becomes one straight-line sm_100a kernel (NVRTC, loaded with
// cudaLibraryLoadData) whose register rounds, slot addresses and FP64
// constants are literals (hex-float immediates) and no dispatch instruction
// is left in the hot loop. Compiled passes are cached process-wide by an
// exact binary key of the pass (jit_key: layer words, pool, tile geometry),
// so re-running a circuit (or the same pass in another circuit) skips
// compilation; hybrid mode compiles misses on background threads.
//
// NVRTC is loaded at run time (dlopen libnvrtc.so.12); without it compiled
// mode (1) fails at state creation and hybrid mode (2) is the interpreter.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "qt_ir.hpp"
#include "qt_kernels.hpp"
#include "qt_micro.hpp"

namespace qtb {

// Everything a compiled pass bakes in (besides the lowered layer words).
struct JitPassSpec {
  int k = 0, R = 0;
  uint64_t ntiles = 0;
  uint64_t lo_mask = 0, outer_mask = 0;
  uint64_t slot_gb[1 << kMaxRegBits] = {};
  uint32_t slot_sb[1 << kMaxRegBits] = {};
  bool check = false;
  bool pipe = false;    // double-buffered tiles: the next tile streams in (cp.async) during the rounds
  int pf_bits = 0;      // > 0: L2 prefetch of the next tile in runs of 2^pf_bits amplitudes
  // smem bank swizzle of the ring kernel, GF(2)-linear on the tile index j:
  // bank group = (j & 7) ^ XOR of swzv[b] over the set bits b >= 3 of j,
  // chosen per pass so every round's quarter-warp hits 8 distinct 16-B bank
  // groups (make_jit_spec); default swzv[b] = 1 << (b % 3) (= qt_device.cuh swz)
  uint8_t swzv[kMaxTileBits + 3] = {};
  int debug = 0;        // QTB_JIT_DEBUG test builds: 1 bounds checks, 2 group skew (ring kernel)
  int device = 0;       // CUDA ordinal the kernel is loaded for (part of the cache key:
                        // launch attributes / occupancy are per device)
  bool kparam = false;  // FP64 constants in a kernel-parameter block (ring kernel), not literals
  bool ring = false;    // persistent CTA, two consumer groups, 3-buffer cp.async + mbarrier ring (jit_source_ring)
  // ring kernel: results leave through shared memory and the TMA engine
  // (cp.async.bulk shared -> global, one bulk copy per contiguous run) instead
  // of 2^R st.global per thread, which sit in the LSU queue at HBM write speed
  // and block the other group's shared-memory traffic
  // 1: the whole tile is staged in place and its buffer refilled one tile
  //    later; 2: every warp drains its own results through a 2 KiB staging
  //    area (two halves of 1 KiB), waiting on its own bulk reads only
  int tma_store = 0;
  // Fused exchange (ring kernel, sharded states with peer memory): the pass
  // before an exchange of k global bits stores every amplitude straight to
  // its place after the exchange -- rank and local index decided by the
  // amplitude's k victim bits (local physical bits fuse_v[i]) -- through a
  // table of the peers' buffers passed as a kernel parameter.
  int fuse_k = 0;
  int fuse_v[3] = {0, 0, 0};
  int min_blocks = 0;   // launch bounds (0 = by R: <= 64 registers for R <= 3, <= 128 for R = 4)
  std::vector<DRound> rounds;  // reg / sreg / sbit per round
  std::vector<int> tile_phys;  // physical bit of each tile bit (ascending)
  // first / last round read / write HBM directly when their register bits
  // leave physical bits [0, coalesce_bits) to the threads (0 = never)
  int coalesce_bits = 0;
};

// Kernel parameter of a fused-exchange pass: peer[v] = the buffer of the rank
// that owns the amplitudes whose victim bits spell v; rfix = this rank's global
// bits deposited at the victim positions (the local index after the exchange).
struct JitFuseParams {
  double2* peer[8];
  unsigned long long rfix;
};

struct JitKernel {
  int fuse_k = 0;  // > 0: a fused-exchange pass (takes a JitFuseParams)
  cudaKernel_t fn = nullptr;
  int threads = 0;
  size_t smem = 0;
  int occupancy = 0;  // resident CTAs per SM
  std::shared_ptr<const std::vector<double>> kp;  // the kernel-parameter constants (kparam passes)
};

// Tile geometry of a planned pass (buf_bits = log2 of the local buffer).
JitPassSpec make_jit_spec(const PlanPass& ps, int reg_bits, int buf_bits, bool check);

// CUDA C++ source of one compiled pass.
// With spec.kparam the pass's distinct FP64 constants are returned in
// *kparams (the launch passes them as the kernel-parameter block).
std::string jit_source(const JitPassSpec& spec, const MicroPass& mp,
                       std::vector<double>* kparams = nullptr);

// Exact cache key of a compiled pass: the bytes of every input of
// jit_source (looking a pass up costs no source generation).
std::string jit_key(const JitPassSpec& spec, const MicroPass& mp);

// Compiles (or finds in the cache) the kernels of `keys` (sources generated
// on a miss only), in parallel. Throws on compile / load failure.
std::vector<JitKernel> jit_kernels(const std::vector<std::string>& keys,
                                   const std::vector<std::function<std::string(std::vector<double>*)>>& sources,
                                   const std::vector<JitPassSpec*>& specs);

// Hybrid mode: a cached kernel, or false (the caller runs the interpreter
// kernel and may queue the pass with jit_compile_async).
bool jit_lookup(const std::string& key, JitKernel* out);
// Compiles a pass on a background thread into the cache (no-op when it is
// queued or compiling already).
void jit_compile_async(const std::string& key, const JitPassSpec& spec, const MicroPass& mp,
                       int device);
// Passes queued or compiling in the background.
size_t jit_pending();
constexpr int kJitBackgroundThreads = 4;
constexpr size_t kJitMaxBacklog = 96;  // queued background compiles (newest kept)
constexpr size_t kJitStackBytes = size_t(256) << 20;  // per compile thread (reserved, not touched)

// Launches a compiled pass (grid = occupancy x SMs, capped by the tiles).
cudaError_t jit_launch(const JitKernel& k, uint64_t ntiles, int sms, double2* psi,
                       const double2* src, int* flag, uint64_t gbase_hi, cudaStream_t s, const JitFuseParams* fuse = nullptr);

// NVRTC compile only (no device needed): CUBIN bytes of a source.
std::vector<char> jit_compile_cubin(const std::string& src);

// True if NVRTC could be loaded (compiled mode available).
bool jit_available(std::string* why = nullptr);

// Process-wide compile statistics (for benchmarks).
struct JitStats {
  uint64_t compiled = 0, cache_hits = 0, misses = 0, background = 0, failed = 0;
  uint64_t disk_hits = 0, disk_writes = 0;  // persistent cubin cache (qt_jit.cpp)
  double compile_ms = 0.0;
};
JitStats jit_stats();

}  // namespace qtb
