// qt_state.cpp -- device state, plan upload, stream-ordered pass launches,
// qubit exchanges, readout and checkpoints.
//
// Replaces the reference's storage and scheduling layer: per-stage COW
// block stores (engine.hpp:18-29, resolve_block engine.cpp:291-301,
// input_block_copy engine.cpp:303-313), the one-shot thread pool spawned per
// update (executor.cpp:64-89) and the readout (engine.cpp:510-564). The state
// is one flat HBM buffer of double2 (bit-compatible with
// std::complex<double>); gate application is a sequence of fused tile passes
// launched in order on one CUDA stream.
#include "qt_state.hpp"
#include "qt_micro.hpp"
#include "qt_jit.hpp"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <atomic>
#include <cmath>
#include <mutex>
#include <limits>
#include <thread>

#include "qt_gates.hpp"
#include "qt_kernels.hpp"

#include <nvtx3/nvToolsExt.h>

namespace qtb {

void fail(int code, const std::string& msg) { throw QtError{code, msg}; }

void cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return;
  if (e == cudaErrorMemoryAllocation)
    fail(QT_ERR_OOM, std::string(what) + ": " + cudaGetErrorString(e));
  if (e == cudaErrorNoDevice || e == cudaErrorInsufficientDriver)
    fail(QT_ERR_NO_DEVICE, std::string(what) + ": " + cudaGetErrorString(e));
  fail(QT_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

namespace {
int ilog2(uint64_t x) {
  int r = 0;
  while ((1ull << r) < x) ++r;
  return r;
}
}  // namespace

State::State(int nqubits, Mode mode, int shards, int rank, const void* nccl_id,
             const qt_config* cfg, std::shared_ptr<LocalGroup> group)
    : n_(nqubits), mode_(mode), rank_(rank), world_(shards) {
  if (nqubits < 1 || nqubits > 40) fail(QT_ERR_BAD_QUBIT, "qubit count must be in [1, 40]");
  if (shards < 1 || (shards & (shards - 1)) != 0)
    fail(QT_ERR_ARG, "shard count must be a power of two");
  const int g = ilog2(static_cast<uint64_t>(shards));
  nlocal_ = n_ - g;
  if (mode != Mode::Single && nlocal_ < 4)
    fail(QT_ERR_ARG, "too many shards for this qubit count");
  buf_bits_ = mode == Mode::Loopback ? n_ : nlocal_;

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    fail(QT_ERR_NO_DEVICE, "no CUDA device visible");
  device_ = (cfg && cfg->device >= 0) ? cfg->device : 0;
  if (!(cfg && cfg->device >= 0)) cudaGetDevice(&device_);
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cudaDeviceGetAttribute(&sms_, cudaDevAttrMultiProcessorCount, device_);

  // compiled passes (qt_jit.cpp): straight-line kernels per pass; they
  // default to wider rounds and tiles (R = 4, 2^12 tiles, 128-B runs):
  // without per-op dispatch the 128-register rounds win
  jit_mode_ = cfg ? std::max(0, std::min(2, static_cast<int>(cfg->compiled))) : 0;
  if (const char* e = std::getenv("QTB_JIT")) jit_mode_ = std::max(0, std::min(2, std::atoi(e)));
  if (jit_mode_) {
    std::string why;
    if (!jit_available(&why)) {
      // hybrid mode is an optimisation of the interpreter path: without
      // NVRTC it is just the interpreter; explicit compiled mode fails
      if (jit_mode_ == 2) jit_mode_ = 0;
      else fail(QT_ERR_ARG, "compiled passes unavailable: " + why);
    }
  }
  // hybrid pays off where passes stream enough amplitudes to amortise the
  // cache lookups (small states are launch-bound)
  if (jit_mode_ == 2 && nlocal_ < kHybridMinQubits) jit_mode_ = 0;
  // geometry: compiled R = 4 / 2^12 tiles / 128-B runs; hybrid R = 3 (its
  // misses run on the interpreter, whose R = 4 variant is slow) with 2^12
  // tiles / 128-B runs; interpreter R = 3 / 2^10 tiles / 256-B runs
  opt_.reg_bits = jit_mode_ == 1 ? kJitRegBits : jit_mode_ == 2 ? kHybridRegBits : kDefaultRegBits;
  opt_.tile_bits = jit_mode_ ? kJitTileBits : kDefaultTileBits;
  if (jit_mode_) opt_.low_bits = jit_mode_ == 1 ? kJitLowBits : kHybridLowBits;
  if (cfg && cfg->tile_qubits > 0)
    opt_.tile_bits = std::min(cfg->tile_qubits, kMaxTileBits);
  // tuning overrides (benchmark sweeps only)
  if (const char* e = std::getenv("QTB_REG_BITS")) opt_.reg_bits = std::max(1, std::min(kMaxRegBits, std::atoi(e)));
  if (const char* e = std::getenv("QTB_TILE_BITS")) opt_.tile_bits = std::max(2, std::min(kMaxTileBits, std::atoi(e)));
  // a tile's non-register bits index the CTA's threads (launch bounds)
  {
    int tb = 0;
    while ((2 << tb) <= tile_max_threads(opt_.reg_bits)) ++tb;
    opt_.tile_bits = std::min(opt_.tile_bits, opt_.reg_bits + tb);
  }
  if (const char* e = std::getenv("QTB_LOW_BITS")) opt_.low_bits = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("QTB_PASS_FP64")) opt_.max_pass_fp64 = std::atof(e);
  if (const char* e = std::getenv("QTB_VICTIM_SPAN")) opt_.victim_span = std::atoi(e);
  // window search: unset = a candidate of the compiled-mode plan search, 0 = never, 1 = always
  if (const char* e = std::getenv("QTB_WINDOW_SEARCH")) {
    window_mode_ = std::atoi(e) != 0 ? 1 : 0;
    opt_.window_search = window_mode_ == 1;
  }
  if (const char* e = std::getenv("QTB_WINDOW_BEAM")) opt_.window_beam = std::atoi(e);
  if (const char* e = std::getenv("QTB_SHRINK_MIN")) opt_.shrink_min_bits = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("QTB_SHRINK_RUN")) opt_.shrink_run_bits = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("QTB_PLAN_SEARCH")) plan_search_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("QTB_EXCHANGE_TMP")) no_alt_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("QTB_JIT_MINB")) jit_min_blocks_ = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("QTB_DIRECT_BITS")) direct_bits_ = std::max(0, std::atoi(e));
  if (const char* e = std::getenv("QTB_PIPE")) pipe_ = std::atoi(e) != 0;
  if (const char* e = std::getenv("QTB_PIPE_MAXFP")) pipe_max_fp64_ = std::atof(e);
  if (const char* e = std::getenv("QTB_PF")) {
    pf_bits_ = std::atoi(e);
    pf_ = pf_bits_ != 0;
  }

  cuda_check(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking), "stream");
  cuda_check(cudaMalloc(&psi_, sizeof(double2) << buf_bits_), "state allocation");
  pool_.push_back(psi_);
  cuda_check(cudaMalloc(&d_scratch_, sizeof(double) * (kNormBlocks + 64)), "scratch");
  cuda_check(cudaMalloc(&d_flag_, sizeof(int)), "flag");
  cuda_check(cudaMemsetAsync(d_flag_, 0, sizeof(int), stream_), "flag init");
  cuda_check(cudaMallocHost(&h_flag_, sizeof(int)), "pinned flag");
  cuda_check(cudaEventCreate(&ev0_), "event");
  cuda_check(cudaEventCreate(&ev1_), "event");
  perm_.resize(n_);
  for (int q = 0; q < n_; ++q) perm_[q] = q;

  if (mode == Mode::Sharded) {
    if (rank < 0 || rank >= shards) fail(QT_ERR_ARG, "rank out of range");
    if (group) {
      if (group->world() != shards) fail(QT_ERR_ARG, "group size differs from the shard count");
      comm_.reset(new LocalComm(group, rank, device_));
    } else {
      std::string err;
      comm_.reset(NcclComm::create(nccl_id, rank, shards, device_, &err));
      if (!comm_) fail(QT_ERR_NCCL, err);
    }
  }
  set_basis(0);
}

State::~State() {
  cudaSetDevice(device_);
  if (stream_) cudaStreamSynchronize(stream_);
  for (auto& kv : ckpt_) cudaFree(kv.second.first);
  if (alt_) cudaFree(alt_);
  for (auto& t : timings_) {
    cudaEventDestroy(t.start);
    cudaEventDestroy(t.stop);
  }
  comm_.reset();
  for (double2* b : pool_) cudaFree(b);
  cudaFree(d_scratch_);
  cudaFree(d_flag_);
  cudaFree(d_tmp_);
  if (h_flag_) cudaFreeHost(h_flag_);
  if (ev0_) cudaEventDestroy(ev0_);
  if (ev1_) cudaEventDestroy(ev1_);
  if (stream_) cudaStreamDestroy(stream_);
}

void State::set_basis(uint64_t index) {
  if (n_ < 64 && index >= (1ull << n_)) fail(QT_ERR_ARG, "basis index out of range");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  for (int q = 0; q < n_; ++q) perm_[q] = q;
  uint64_t local = index;
  uint64_t target = ~0ull;  // index within this buffer, or none
  if (mode_ == Mode::Sharded) {
    const uint64_t owner = index >> nlocal_;
    local = index & ((1ull << nlocal_) - 1);
    if (owner == static_cast<uint64_t>(rank_)) target = local;
  } else {
    target = local;
  }
  cuda_check(launch_set_basis(psi_, buffer_amps(), target, stream_), "set_basis");
}

void State::write(uint64_t first, uint64_t count, const double* src) {
  if (n_ < 64 && (first > (1ull << n_) || count > (1ull << n_) - first))
    fail(QT_ERR_ARG, "amplitude range out of bounds");
  for (int q = 0; q < n_; ++q)
    if (perm_[q] != q) fail(QT_ERR_ARG, "write needs the canonical qubit order (call set_basis)");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  uint64_t lo = first, hi = first + count;
  if (mode_ == Mode::Sharded) {
    const uint64_t s0 = static_cast<uint64_t>(rank_) << nlocal_;
    const uint64_t s1 = s0 + (1ull << nlocal_);
    lo = std::max(lo, s0);
    hi = std::min(hi, s1);
    if (lo >= hi) return;
    cuda_check(cudaMemcpyAsync(psi_ + (lo - s0), src + 2 * (lo - first),
                               (hi - lo) * sizeof(double2),
                               cudaMemcpyHostToDevice, stream_),
               "write");
  } else {
    cuda_check(cudaMemcpyAsync(psi_ + lo, src, count * sizeof(double2),
                               cudaMemcpyHostToDevice, stream_),
               "write");
  }
  cuda_check(cudaStreamSynchronize(stream_), "write sync");
}

void State::read(uint64_t first, uint64_t count, double* dst) {
  if (n_ < 64 && (first > (1ull << n_) || count > (1ull << n_) - first))
    fail(QT_ERR_ARG, "amplitude range out of bounds");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  bool identity = true;
  for (int q = 0; q < n_; ++q) identity = identity && perm_[q] == q;
  if (identity && mode_ != Mode::Sharded) {
    cuda_check(cudaMemcpyAsync(dst, psi_ + first, count * sizeof(double2),
                               cudaMemcpyDeviceToHost, stream_),
               "read");
    sync();
    return;
  }
  // gather through the logical->physical map, in device-sized chunks
  const uint64_t chunk = 1ull << 22;
  if (d_tmp_amps_ < std::min(count, chunk)) {
    cudaFree(d_tmp_);
    d_tmp_ = nullptr;
    d_tmp_amps_ = std::min(count, chunk);
    cuda_check(cudaMalloc(&d_tmp_, d_tmp_amps_ * sizeof(double2)), "gather buffer");
  }
  std::vector<uint8_t> pm(n_);
  for (int q = 0; q < n_; ++q) pm[q] = static_cast<uint8_t>(perm_[q]);
  for (uint64_t off = 0; off < count; off += chunk) {
    const uint64_t c = std::min(chunk, count - off);
    if (mode_ == Mode::Sharded) {
      cuda_check(launch_gather_shard(psi_, d_tmp_, first + off, c, pm.data(), n_,
                                     nlocal_, static_cast<uint64_t>(rank_), stream_),
                 "gather");
    } else {
      cuda_check(launch_gather(psi_, d_tmp_, first + off, c, pm.data(), n_, stream_),
                 "gather");
    }
    cuda_check(cudaMemcpyAsync(dst + 2 * off, d_tmp_, c * sizeof(double2),
                               cudaMemcpyDeviceToHost, stream_),
               "read");
  }
  sync();
}

namespace {

// Estimated device time of a plan (ms): per tile pass the larger of its FP64
// time (lowered ops per amplitude at the FP64 rate) and its HBM time (32 B
// per local amplitude at the ring kernel's streaming rate); exchanges at a
// fixed cost of one pass.
double plan_cost_ms(const Plan& p, int reg_bits, int nlocal) {
  const std::vector<MicroPass> mp = lower_plan_micro(
      p, reg_bits, MicroLimits{size_t(1) << 20, size_t(1) << 20, size_t(1) << 20});
  const double amps = std::ldexp(1.0, nlocal);
  const double hbm = 32.0 * amps / kPlanHbmBytesPerS * 1e3;
  double t = 0.0;
  for (size_t i = 0; i < p.passes.size(); ++i) {
    double fp = 0.0;
    if (p.passes[i].kind == PlanPass::Tile && mp[i].ok)
      fp = micro_fp64_per_amp(mp[i], std::min<int>(reg_bits, static_cast<int>(p.passes[i].tile_phys.size()))) *
           amps / kPlanFp64PerS * 1e3;
    // measured on B200 (profiles/r02_ablation.md): a pass costs its FP64 time
    // plus the share of its HBM time the ring kernel does not hide under the
    // arithmetic, and never less than the streaming time
    t += std::max(hbm, fp + kPlanExposedHbm * hbm);
  }
  return t;
}

}  // namespace

// Compiled mode on large states searches the planner's per-pass FP64 cap
// (PlanOptions::max_pass_fp64): the greedy planner fills every pass as far
// as the tile allows, which makes a few FP64-bound passes next to HBM-bound
// ones; capping the FP64 a pass may carry moves work into passes with FP64
// to spare and changes where pass boundaries fall. The candidate plans are
// built in parallel and the one with the least estimated time (plan_cost_ms)
// wins (C3: 22 -> 18 passes, 196 -> 180 ms).
Plan State::plan(const std::vector<LOp>& ops) const {
  // the beam search visits (beam x windows x passes) fills: bounded to circuits
  // it finishes on in well under a second
  const bool beam_ok = ops.size() <= kPlanBeamMaxOps;
  if (jit_mode_ == 0 && nlocal_ >= kPlanSearchMinBits && opt_.max_pass_fp64 <= 0.0 && plan_search_ &&
      window_mode_ < 0) {
    // interpreter (one-shot applies): the first-need greedy plan against the
    // beam-searched window plan, by the same cost model (C3: 37 -> 18 passes,
    // 346 -> 305 ms; random circuits keep the greedy plan)
    Plan greedy, window;
    PlanOptions ow = opt_;
    ow.window_search = true;
    ow.window_beam = beam_ok ? kPlanBeamWidth : 0;
    std::thread tw([&] { window = make_plan(ops, n_, nlocal_, perm_, ow); });
    greedy = make_plan(ops, n_, nlocal_, perm_, opt_);
    tw.join();
    if (window.passes.size() >= greedy.passes.size()) return greedy;
    return plan_cost_ms(window, opt_.reg_bits, nlocal_) < plan_cost_ms(greedy, opt_.reg_bits, nlocal_) - 1e-9
               ? window
               : greedy;
  }
  if (jit_mode_ != 1 || nlocal_ < kPlanSearchMinBits || opt_.max_pass_fp64 > 0.0 || !plan_search_)
    return make_plan(ops, n_, nlocal_, perm_, opt_);
  // Phase 1 candidates: every cap with the first-need greedy tiles and with
  // the window search (PlanOptions::window_search: fewer, deeper passes on
  // layered circuits -- C3 18 -> 13 passes; no gain on random circuits).
  // Phase 2, only when a window plan won: the beam search over the window
  // choices (window_beam) with the configured and one fewer reserved low bit
  // (a window one qubit wider; C3: 10-11 passes, 150-154 ms).
  struct Cand {
    double cap;
    bool window;
    int beam, low;
  };
  std::vector<double> caps{0.0};
  for (double c = 150.0; c <= 264.0; c += 6.0) caps.push_back(c);
  auto run = [&](const std::vector<Cand>& cands, Plan* best_plan, double* best_cost, Cand* best_cand) {
    std::vector<Plan> plans(cands.size());
    std::vector<double> cost(cands.size(), 0.0);
    std::vector<std::thread> th;
    std::atomic<size_t> next{0};
    const unsigned nt = std::max(1u, std::min<unsigned>(static_cast<unsigned>(cands.size()),
                                                        std::thread::hardware_concurrency()));
    for (unsigned w = 0; w < nt; ++w)
      th.emplace_back([&] {
        for (size_t i; (i = next.fetch_add(1)) < cands.size();) {
          PlanOptions o = opt_;
          o.max_pass_fp64 = cands[i].cap;
          o.window_search = cands[i].window;
          o.window_beam = cands[i].beam;
          o.low_bits = cands[i].low;
          plans[i] = make_plan(ops, n_, nlocal_, perm_, o);
          cost[i] = plan_cost_ms(plans[i], o.reg_bits, nlocal_);
        }
      });
    for (std::thread& t : th) t.join();
    for (size_t i = 0; i < cands.size(); ++i)
      if (cost[i] < *best_cost - 1e-9) {
        *best_cost = cost[i];
        *best_plan = std::move(plans[i]);
        *best_cand = cands[i];
      }
  };
  std::vector<Cand> c1;
  for (double c : caps) {
    if (window_mode_ != 1) c1.push_back(Cand{c, false, 0, opt_.low_bits});
    if (window_mode_ != 0) c1.push_back(Cand{c, true, opt_.window_beam, opt_.low_bits});
  }
  Plan best;
  double best_cost = std::numeric_limits<double>::infinity();
  Cand best_cand{0.0, false, 0, opt_.low_bits};
  run(c1, &best, &best_cost, &best_cand);
  if (best_cand.window && window_mode_ < 0 && opt_.window_beam <= 1 && beam_ok) {
    std::vector<Cand> c2;
    for (double c : caps) {
      c2.push_back(Cand{c, true, kPlanBeamWidth, opt_.low_bits});
      if (opt_.low_bits > 3) c2.push_back(Cand{c, true, kPlanBeamWidth, opt_.low_bits - 1});
    }
    run(c2, &best, &best_cost, &best_cand);
  }
  return best;
}

void State::apply(const qt_gate* gates, size_t count) {
  // re-applying the gate list of the previous call from the same qubit map
  // reuses its plan, lowering and compiled passes (no host planning)
  std::string key(reinterpret_cast<const char*>(gates), count * sizeof(qt_gate));
  key.append(reinterpret_cast<const char*>(perm_.data()), perm_.size() * sizeof(int));
  if (last_.valid && last_.key == key) {
    cuda_check(cudaSetDevice(device_), "cudaSetDevice");
    stats = qt_run_stats{};
    stats.gates = count;
    if (jit_mode_ == 2) {
      // hybrid: passes compiled since the last call are picked up
      Prepared pr = prepare(last_.plan);
      launch_prepared(last_.plan, pr, nullptr);
    } else {
      launch_prepared(last_.plan, last_.prep, nullptr);
    }
    perm_ = last_.plan.perm_after;
    return;
  }
  std::vector<LOp> ops;
  ops.reserve(count);
  std::string err;
  for (size_t i = 0; i < count; ++i) {
    const int rc = lower_gate(gates[i], n_, static_cast<uint32_t>(i), ops, &err);
    if (rc != QT_OK) fail(rc, err);
  }
  fuse_ops(ops, n_);
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  decide_fusion();
  const auto t0 = std::chrono::steady_clock::now();
  last_.valid = false;
  last_.plan = plan(ops);
  const auto t1 = std::chrono::steady_clock::now();
  stats = qt_run_stats{};
  stats.gates = count;
  stats.plan_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  last_.prep = prepare(last_.plan);
  last_.key = std::move(key);
  last_.valid = true;
  launch_prepared(last_.plan, last_.prep, nullptr);
  perm_ = last_.plan.perm_after;
}

int State::grow_pool(int count, double max_fraction_of_free) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  const size_t bytes = sizeof(double2) * buffer_amps();
  // one budget from the free memory at the start: the pool may take
  // max_fraction_of_free of it in total (not of what each allocation leaves)
  size_t fre0 = 0, tot = 0;
  cudaMemGetInfo(&fre0, &tot);
  const double budget = max_fraction_of_free * static_cast<double>(fre0);
  // keep a reserve for plan / exchange buffers and the caller
  const size_t reserve = std::max<size_t>(tot / 50, size_t(2) << 30);
  size_t taken = 0;
  while (static_cast<int>(pool_.size()) < count) {
    size_t fre = 0;
    cudaMemGetInfo(&fre, &tot);
    if (fre < reserve + bytes) break;
    if (static_cast<double>(taken + bytes) > budget) break;
    double2* b = nullptr;
    if (cudaMalloc(&b, bytes) != cudaSuccess) {
      cudaGetLastError();
      break;
    }
    pool_.push_back(b);
    taken += bytes;
  }
  return static_cast<int>(pool_.size());
}

void State::bind(int i, const std::vector<int>& perm) {
  if (i < 0 || i >= static_cast<int>(pool_.size())) fail(QT_ERR_ARG, "bad buffer");
  bound_ = i;
  psi_ = pool_[i];
  perm_ = perm;
}

std::shared_ptr<State::PreparedPlan> State::prepare_ops(const std::vector<LOp>& ops,
                                                        const std::vector<int>* perm) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  auto pp = std::make_shared<PreparedPlan>();
  const auto t0 = std::chrono::steady_clock::now();
  pp->plan = make_plan(ops, n_, nlocal_, perm ? *perm : perm_, opt_);
  pp->prep = prepare(pp->plan);
  pp->plan_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return pp;
}

void State::apply_prepared(const PreparedPlan& pp, uint64_t ngates, const double2* src,
                           const std::vector<int>* src_perm) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  if (src == psi_) src = nullptr;
  if (src && src_perm) perm_ = *src_perm;
  stats = qt_run_stats{};
  stats.gates = ngates;
  stats.plan_ms = pp.plan_ms;
  if (jit_mode_ == 2) {
    // hybrid: passes compiled since the plan was prepared are picked up
    const Prepared fresh = prepare(pp.plan);
    launch_prepared(pp.plan, fresh, src);
  } else {
    launch_prepared(pp.plan, pp.prep, src);
  }
  perm_ = pp.plan.perm_after;
}

void State::apply_ops(const std::vector<LOp>& ops, uint64_t ngates,
                      const double2* src, const std::vector<int>* src_perm) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  if (src == psi_) src = nullptr;
  if (src && src_perm) perm_ = *src_perm;
  const auto t0 = std::chrono::steady_clock::now();
  const Plan p = plan(ops);
  const auto t1 = std::chrono::steady_clock::now();
  stats = qt_run_stats{};
  stats.gates = ngates;
  stats.plan_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  upload_and_launch(p, src);
  perm_ = p.perm_after;
}

namespace {

// Fills a kernel-parameter block for one tile pass: rounds, then the ops of
// each round in order (encoded against the round's register bits).
template <typename P>
void fill_pass(P& kp, const PlanPass& ps) {
  kp.h.nrounds = static_cast<uint32_t>(ps.rounds.size());
  uint32_t nops = 0, npool = 0;
  for (size_t r = 0; r < ps.rounds.size(); ++r) {
    const PlanRound& pr = ps.rounds[r];
    DRound& dr = kp.rounds[r];
    dr = DRound{};
    dr.op_first = static_cast<uint16_t>(nops);
    dr.op_count = static_cast<uint16_t>(pr.enc.ops.size());
    const size_t nreg = std::min(pr.reg.size(), static_cast<size_t>(kMaxRegBits));
    std::vector<int> sorted(pr.reg.begin(), pr.reg.begin() + nreg);
    std::sort(sorted.begin(), sorted.end());
    for (size_t i = 0; i < nreg; ++i) {
      dr.reg[i] = static_cast<uint8_t>(pr.reg[i]);
      dr.sreg[i] = static_cast<uint8_t>(sorted[i]);
      dr.sbit[i] = swz_host(1u << pr.reg[i]) << 4;
    }
    for (DOp d : pr.enc.ops) {
      // pool offsets are round-relative: rebase onto the launch's pool
      const uint32_t type = (d.hdr & kOpVariantMask) >> 10;
      if (type == D_LAYER)
        d.arg = ((d.arg & 0xffff) + npool) | (d.arg & 0xffff0000u);  // offset | nterms << 16
      else d.arg += npool;
      kp.ops[nops++] = d;
    }
    for (double x : pr.enc.pool) kp.pool[npool++] = x;
  }
  kp.h.nops = nops;
}

// The lean kernel's parameters: rounds index the pass's micro-ops, which
// occupy the op array's bytes; the pool is the lowered one.
template <typename P>
void fill_pass_micro(P& kp, const PlanPass& ps, const MicroPass& mp) {
  kp.h.nrounds = static_cast<uint32_t>(ps.rounds.size());
  for (size_t r = 0; r < ps.rounds.size(); ++r) {
    const PlanRound& pr = ps.rounds[r];
    DRound& dr = kp.rounds[r];
    dr = DRound{};
    dr.op_first = mp.round_first[r];
    dr.op_count = mp.round_count[r];
    const size_t nreg = std::min(pr.reg.size(), static_cast<size_t>(kMaxRegBits));
    std::vector<int> sorted(pr.reg.begin(), pr.reg.begin() + nreg);
    std::sort(sorted.begin(), sorted.end());
    for (size_t i = 0; i < nreg; ++i) {
      dr.reg[i] = static_cast<uint8_t>(pr.reg[i]);
      dr.sreg[i] = static_cast<uint8_t>(sorted[i]);
      dr.sbit[i] = swz_host(1u << pr.reg[i]) << 4;
    }
  }
  std::memcpy(reinterpret_cast<char*>(kp.ops), mp.words.data(), mp.words.size() * 4);
  std::memcpy(kp.pool, mp.pool.data(), mp.pool.size() * sizeof(double));
  kp.h.nops = static_cast<uint32_t>(mp.size());
}

template <typename P>
bool micro_fits(const PlanPass& ps, const MicroPass& mp) {
  return mp.ok && mp.size() <= static_cast<size_t>(micro_capacity<P>()) &&
         mp.pool.size() <= sizeof(P::pool) / sizeof(double) &&
         ps.rounds.size() <= sizeof(P::rounds) / sizeof(DRound);
}

}  // namespace

State::Prepared State::prepare(const Plan& plan) {
  Prepared pr;
  pr.micro = lower_plan_micro(
      plan, opt_.reg_bits,
      MicroLimits{static_cast<size_t>(micro_capacity<KPassLarge>()),
                  sizeof(KPassLarge::pool) / sizeof(double),
                  sizeof(KPassLarge::rounds) / sizeof(DRound)});
  size_t last_tile = plan.passes.size();
  for (size_t pi = 0; pi < plan.passes.size(); ++pi)
    if (plan.passes[pi].kind == PlanPass::Tile) last_tile = pi;
  pr.jk.assign(plan.passes.size(), JitKernel{});
  const std::vector<MicroPass>& micro = pr.micro;
  std::vector<JitKernel>& jk = pr.jk;
  if (jit_mode_) {
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<JitPassSpec> specs(plan.passes.size());
    std::vector<std::string> keys;
    std::vector<std::function<std::string(std::vector<double>*)>> srcs;
    std::vector<JitPassSpec*> sp_ptr;
    std::vector<size_t> idx;
    for (size_t pi = 0; pi < plan.passes.size(); ++pi) {
      const PlanPass& ps = plan.passes[pi];
      if (ps.kind != PlanPass::Tile || !micro[pi].ok) continue;
      JitPassSpec& sp = specs[pi];
      sp = make_jit_spec(ps, opt_.reg_bits, buf_bits_, pi == last_tile);
      sp.pipe = pipe_ && (2 * (sizeof(double2) << sp.k)) <= 200 * 1024 &&
                (pipe_max_fp64_ <= 0.0 || micro_fp64_per_amp(micro[pi], sp.R) <= pipe_max_fp64_);
      if (sp.pipe) sp.ring = false;
      sp.min_blocks = jit_min_blocks_;
      sp.device = device_;
      sp.coalesce_bits = direct_bits_;
      if (fuse_ok_ && sp.ring && pi + 1 < plan.passes.size() &&
          plan.passes[pi + 1].kind == PlanPass::Exchange && plan.passes[pi + 1].exchange.size() <= 3) {
        const PlanPass& ex = plan.passes[pi + 1];
        sp.fuse_k = static_cast<int>(ex.exchange.size());
        for (int i = 0; i < sp.fuse_k; ++i) sp.fuse_v[i] = ex.exchange[i].second;
        sp.tma_store = 0;
        sp.kparam = false;
      }
      if (pf_ && !sp.pipe) {
        int run = 0;
        while (run < sp.k - sp.R && ps.tile_phys[run] == run) ++run;
        sp.pf_bits = std::max(run, pf_bits_);
      }
      std::string key = jit_key(sp, micro[pi]);
      if (jit_mode_ == 2) {
        // hybrid: cached passes run compiled, the others on the interpreter
        // while they compile in the background for the next update
        if (!jit_lookup(key, &jk[pi])) jit_compile_async(key, sp, micro[pi], device_);
        continue;
      }
      keys.push_back(std::move(key));
      const MicroPass* m = &micro[pi];
      const JitPassSpec* spc = &sp;
      srcs.push_back([m, spc](std::vector<double>* kp) { return jit_source(*spc, *m, kp); });
      sp_ptr.push_back(&sp);
      idx.push_back(pi);
    }
    if (!keys.empty()) {
      std::vector<JitKernel> ks = jit_kernels(keys, srcs, sp_ptr);
      for (size_t i = 0; i < idx.size(); ++i) jk[idx[i]] = ks[i];
    }
    stats.plan_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  }
  return pr;
}

void State::upload_and_launch(const Plan& plan, const double2* src) { launch_prepared(plan, prepare(plan), src); }

void State::launch_prepared(const Plan& plan, const Prepared& pr, const double2* src) {
  cuda_check(cudaEventRecord(ev0_, stream_), "event");
  size_t timing_idx = timings_used_;  // events accumulate until collected
  // NVTX ranges per pass / exchange (nvtx3 is header-only: the calls are
  // no-ops unless a profiler injects itself, e.g. nsys / ncu --nvtx)
  auto tstart = [&](int kind) {
    nvtxRangePushA(kind == 1 ? "qtask exchange" : "qtask tile pass");
    if (!timing_) return;
    if (timing_idx >= timings_.size()) {
      PassTiming t;
      cudaEventCreate(&t.start);
      cudaEventCreate(&t.stop);
      timings_.push_back(t);
    }
    timings_[timing_idx].kind = kind;
    cudaEventRecord(timings_[timing_idx].start, stream_);
  };
  auto tstop = [&]() {
    nvtxRangePop();
    if (!timing_) return;
    cudaEventRecord(timings_[timing_idx].stop, stream_);
    ++timing_idx;
  };
  const uint64_t buf_mask = buffer_amps() - 1;
  // out-of-place start: the first tile pass reads src; otherwise copy
  if (src && (plan.passes.empty() || plan.passes[0].kind != PlanPass::Tile)) {
    cuda_check(cudaMemcpyAsync(psi_, src, sizeof(double2) * buffer_amps(),
                               cudaMemcpyDeviceToDevice, stream_),
               "state copy");
    stats.kernel_launches += 1;
    stats.hbm_bytes += 2ull * sizeof(double2) * buffer_amps();
    src = nullptr;
  }
  if (!kp_small_) kp_small_.reset(new KPassSmall);
  if (!kp_large_) kp_large_.reset(new KPassLarge);
  const std::vector<MicroPass>& micro = pr.micro;
  const std::vector<JitKernel>& jk = pr.jk;
  size_t last_tile = plan.passes.size();
  for (size_t pi = 0; pi < plan.passes.size(); ++pi)
    if (plan.passes[pi].kind == PlanPass::Tile) last_tile = pi;
  for (size_t pi = 0; pi < plan.passes.size(); ++pi) {
    const PlanPass& ps = plan.passes[pi];
    if (ps.kind == PlanPass::Exchange && pi > 0 && jk[pi - 1].fuse_k > 0) continue;  // done by the pass before it
    if (ps.kind == PlanPass::Exchange) {
      tstart(1);
      exchange(ps);
      tstop();
      stats.swaps += 1;
      stats.kernel_launches += ps.exchange.size();
      continue;
    }
    if (jk[pi].fn && jk[pi].fuse_k > 0) {
      // pass + exchange in one kernel: stores go to the peers' second buffers
      const PlanPass& ex = plan.passes[pi + 1];
      const int k = static_cast<int>(ex.exchange.size());
      std::vector<int> group;  // the 2^k ranks that differ from this one in the exchanged rank bits
      uint64_t rfix = 0;
      fused_exchange_map(rank_, nlocal_, ex.exchange, &group, &rfix);
      const double2* rd = src ? src : psi_;
      src = nullptr;
      tstart(0);
      std::string err;
      std::vector<int> sorted_group(group);
      std::sort(sorted_group.begin(), sorted_group.end());
      const bool ok = comm_->with_peer_buffers(alt_, sorted_group, stream_, [&](void* const* table) {
        JitFuseParams fx{};
        for (uint32_t v = 0; v < (1u << k); ++v) {
          if (!table[group[v]]) return false;
          fx.peer[v] = static_cast<double2*>(table[group[v]]);
        }
        fx.rfix = rfix;
        return jit_launch(jk[pi], 1ull << (buf_bits_ - static_cast<int>(ps.tile_phys.size())), sms_, psi_, rd,
                          d_flag_, static_cast<uint64_t>(rank_) << nlocal_, stream_, &fx) == cudaSuccess;
      }, &err);
      if (!ok) fail(QT_ERR_NCCL, err.empty() ? "fused exchange failed" : err);
      tstop();
      std::swap(psi_, alt_);
      pool_[0] = psi_;
      const uint64_t region = 1ull << (nlocal_ - k);
      stats.passes += 1;
      stats.swaps += 1;
      stats.fused_exchanges += 1;
      stats.kernel_launches += 1;
      stats.hbm_bytes += 2ull * sizeof(double2) * buffer_amps();
      stats.exchanged_bytes += static_cast<uint64_t>((1 << k) - 1) * region * sizeof(double2);
      continue;
    }
    if (jk[pi].fn) {
      tstart(0);
      cuda_check(jit_launch(jk[pi], 1ull << (buf_bits_ - static_cast<int>(ps.tile_phys.size())), sms_,
                            psi_, src ? src : psi_, d_flag_,
                            mode_ == Mode::Sharded ? (static_cast<uint64_t>(rank_) << nlocal_) : 0,
                            stream_),
                 "compiled pass launch");
      src = nullptr;
      tstop();
      stats.passes += 1;
      stats.kernel_launches += 1;
      stats.hbm_bytes += 2ull * sizeof(double2) * buffer_amps();
      continue;
    }
    const int k = static_cast<int>(ps.tile_phys.size());
    const int R = std::min(opt_.reg_bits, k);
    KPassHead h{};
    h.k = static_cast<uint32_t>(k);
    h.reg_bits = static_cast<uint32_t>(R);
    h.flag = d_flag_;
    h.src = src ? src : psi_;
    src = nullptr;
    uint64_t tile_mask = 0;
    for (int i = 0; i < k; ++i) {
      const uint64_t b = 1ull << ps.tile_phys[i];
      tile_mask |= b;
      if (i < k - R) h.lo_mask |= b;
      else h.hi_mask |= b;
    }
    h.outer_mask = buf_mask & ~tile_mask;
    h.check = pi == last_tile ? 1u : 0u;
    if (pf_) {
      // contiguous low run of the tile (physical bits 0, 1, ...), within the
      // thread bits so a run starts at a thread's slot
      int run = 0;
      while (run < k - R && ps.tile_phys[run] == run) ++run;
      h.pf_bits = static_cast<uint32_t>(run);
    }
    for (uint32_t s = 0; s < (1u << R); ++s) {
      uint64_t off = 0;
      for (int i = 0; i < R; ++i)
        if ((s >> i) & 1u) off |= 1ull << ps.tile_phys[k - R + i];
      h.slot_gb[s] = off * sizeof(double2);
      h.slot_sb[s] = swz_host(s << (k - R)) << 4;
    }
    h.ntiles = 1ull << (buf_bits_ - k);
    h.gbase_hi = mode_ == Mode::Sharded ? (static_cast<uint64_t>(rank_) << nlocal_) : 0;
    // lean kernel (micro-ops) when the pass lowered and fits a launch;
    // otherwise the generic kernel decodes the device ops
    const MicroPass& mp = micro[pi];
    bool generic = !(micro_fits<KPassSmall>(ps, mp) || micro_fits<KPassLarge>(ps, mp));
    bool large;
    if (!generic) {
      large = !micro_fits<KPassSmall>(ps, mp);
    } else {
      size_t nops = 0, npool = 0;
      for (const PlanRound& pr : ps.rounds) {
        nops += pr.enc.ops.size();
        npool += pr.enc.pool.size();
      }
      large = nops > static_cast<size_t>(kSmallOps) ||
              npool > static_cast<size_t>(kSmallPool) ||
              ps.rounds.size() > static_cast<size_t>(kSmallRounds);
    }
    int kmode = generic ? kKernelGeneric : kKernelLean;
    if (!generic)
      for (size_t w = 0; w < mp.size(); ++w)
        if (mp.words[2 * w] & M_TDIAG) kmode = kKernelLeanTdiag;
    int occ_pipe = pipe_ ? tile_pass_occupancy(k, R, large, kmode, true) : 0;
    const bool pipe = occ_pipe > 0;
    const int occ = std::max(1, pipe ? occ_pipe : tile_pass_occupancy(k, R, large, kmode, false));
    const uint64_t cap = static_cast<uint64_t>(occ) * sms_;
    const int grid = static_cast<int>(std::min<uint64_t>(h.ntiles, cap));
    tstart(0);
    if (large) {
      kp_large_->h = h;
      if (generic) fill_pass(*kp_large_, ps);
      else fill_pass_micro(*kp_large_, ps, mp);
      cuda_check(launch_tile_pass(psi_, *kp_large_, grid, kmode, pipe, stream_), "tile pass launch");
    } else {
      kp_small_->h = h;
      if (generic) fill_pass(*kp_small_, ps);
      else fill_pass_micro(*kp_small_, ps, mp);
      cuda_check(launch_tile_pass(psi_, *kp_small_, grid, kmode, pipe, stream_), "tile pass launch");
    }
    tstop();
    stats.passes += 1;
    stats.kernel_launches += 1;
    stats.hbm_bytes += 2ull * sizeof(double2) * buffer_amps();
  }
  cuda_check(cudaEventRecord(ev1_, stream_), "event");
  timings_used_ = timing_idx;
  stats.rewritten_amplitudes = plan.passes.empty() ? 0 : (1ull << n_);
}

// The all-to-all of one exchange pass, as grouped send/recv steps. The pass
// swaps k global (rank) bits G_j with k local victim bits V_j: this rank
// keeps the part of its shard whose victim bits equal its own global bits
// (rho) and trades, with each of the 2^k - 1 partners p (rank bits G_j set to
// c_j), the region whose victim bits equal c -- receiving p's region whose
// victim bits equal rho, into the same place. Regions are cut into runs of
// 2^min(V) contiguous amplitudes and the runs into pieces that fit `tmp_amps`
// (all peers' pieces side by side).
std::vector<ExchangeStep> exchange_schedule(int rank, int nlocal,
                                            const std::vector<std::pair<int, int>>& ex,
                                            uint64_t tmp_amps) {
  const int k = static_cast<int>(ex.size());
  std::vector<int> gbit(k), vbit(k);
  uint64_t vmask = 0;
  int minv = nlocal;
  for (int j = 0; j < k; ++j) {
    gbit[j] = ex[j].first - nlocal;
    vbit[j] = ex[j].second;
    vmask |= 1ull << vbit[j];
    minv = std::min(minv, vbit[j]);
  }
  int rho = 0;
  for (int j = 0; j < k; ++j) rho |= ((rank >> gbit[j]) & 1) << j;
  const uint64_t run_len = 1ull << minv;
  const uint64_t region = 1ull << (nlocal - k);
  const uint64_t runs = region / run_len;
  const int npeer = (1 << k) - 1;
  uint64_t piece = run_len;
  while (piece * static_cast<uint64_t>(npeer) > tmp_amps && piece > 1) piece >>= 1;
  const uint64_t per_run = run_len / piece;
  // bits >= minv that are not V bits enumerate the runs of a region
  uint64_t above = 0;
  for (int b = minv; b < nlocal; ++b)
    if (!((vmask >> b) & 1)) above |= 1ull << b;
  auto pdep = [](uint64_t x, uint64_t mask) {
    uint64_t r = 0;
    for (uint64_t b = 1; mask; b <<= 1) {
      const uint64_t low = mask & (~mask + 1);
      if (x & b) r |= low;
      mask ^= low;
    }
    return r;
  };
  std::vector<int> peers;
  std::vector<uint64_t> vbase;  // the victim-bit pattern of each partner's region
  for (int c = 0; c < (1 << k); ++c) {
    if (c == rho) continue;
    int pr = rank;
    uint64_t vb = 0;
    for (int j = 0; j < k; ++j) {
      pr = (pr & ~(1 << gbit[j])) | (((c >> j) & 1) << gbit[j]);
      vb |= static_cast<uint64_t>((c >> j) & 1) << vbit[j];
    }
    peers.push_back(pr);
    vbase.push_back(vb);
  }
  // m consecutive pieces per peer per step (one NCCL group of npeer * m
  // send / receive pairs, matched in issue order), so low victim bits
  // (short runs) do not multiply the number of groups
  const uint64_t total = runs * per_run;
  const uint64_t m = std::max<uint64_t>(1, std::min<uint64_t>(total, tmp_amps / (piece * npeer)));
  std::vector<ExchangeStep> steps;
  steps.reserve((total + m - 1) / m);
  for (uint64_t p0 = 0; p0 < total; p0 += m) {
    ExchangeStep st;
    st.piece = piece;
    const uint64_t p1 = std::min(total, p0 + m);
    for (int i = 0; i < npeer; ++i) {
      for (uint64_t p = p0; p < p1; ++p) {
        const uint64_t run_base = pdep(p / per_run, above);
        st.peer.push_back(peers[i]);
        st.send_off.push_back((run_base | vbase[i]) + (p % per_run) * piece);
        st.recv_off.push_back((static_cast<uint64_t>(i) * m + (p - p0)) * piece);
      }
    }
    steps.push_back(std::move(st));
  }
  return steps;
}

namespace {

// The exchange's victim bits: this rank keeps the region whose victim-bit
// pattern equals its own global bits; it is made of runs of 2^minv
// amplitudes (minv = the lowest victim bit).
int min_victim(int nlocal, const std::vector<std::pair<int, int>>& ex) {
  int m = nlocal;
  for (const auto& gv : ex) m = std::min(m, gv.second);
  return m;
}

// this rank's own region of an exchange: the amplitudes whose victim bits
// equal its global bits -- runs of 2^min_victim amplitudes at offsets
// pdep(r, above) | vpat
void own_region(int rank, int nlocal, const std::vector<std::pair<int, int>>& ex,
                uint64_t* above, uint64_t* vpat) {
  const int minv = min_victim(nlocal, ex);
  uint64_t vmask = 0;
  *vpat = 0;
  for (const auto& gv : ex) {
    vmask |= 1ull << gv.second;
    if ((rank >> (gv.first - nlocal)) & 1) *vpat |= 1ull << gv.second;
  }
  *above = 0;
  for (int b = minv; b < nlocal; ++b)
    if (!((vmask >> b) & 1)) *above |= 1ull << b;
}

}  // namespace

// Destination map of a fused exchange on `rank`: group[v] = the rank that owns,
// after the exchange, the amplitudes whose k victim bits spell v (bit i of v =
// bit exchange[i].second of the local index); rfix = this rank's exchanged
// rank bits deposited at the victim positions -- the amplitude at local index x
// moves to rank group[v(x)], local index (x with the victim bits cleared) | rfix.
void fused_exchange_map(int rank, int nlocal, const std::vector<std::pair<int, int>>& exchange,
                        std::vector<int>* group, uint64_t* rfix) {
  const int k = static_cast<int>(exchange.size());
  group->clear();
  *rfix = 0;
  for (uint32_t v = 0; v < (1u << k); ++v) {
    int r = rank;
    for (int i = 0; i < k; ++i) {
      const int gb = exchange[i].first - nlocal;
      r = (r & ~(1 << gb)) | (static_cast<int>((v >> i) & 1u) << gb);
    }
    group->push_back(r);
  }
  for (int i = 0; i < k; ++i)
    if ((rank >> (exchange[i].first - nlocal)) & 1) *rfix |= 1ull << exchange[i].second;
}

// The second shard buffer of the two-buffer exchange, allocated once when it fits.
void State::ensure_alt() {
  if (alt_ || alt_tried_ || bound_ != 0) return;
  // one decision at a time per process (emulated ranks share a device)
  static std::mutex alloc_mu;
  std::lock_guard<std::mutex> lk(alloc_mu);
  alt_tried_ = true;
  size_t fr = 0, tot = 0;
  const size_t bytes = sizeof(double2) << nlocal_;
  if (!no_alt_ && cudaMemGetInfo(&fr, &tot) == cudaSuccess && fr > bytes + (size_t(4) << 30)) {
    if (cudaMalloc(&alt_, bytes) != cudaSuccess) {
      cudaGetLastError();
      alt_ = nullptr;
    }
  }
}

// Fused exchanges (compiled mode, transports with peer memory): the pass
// before an exchange stores every amplitude straight to the rank and index it
// has after the exchange, so the exchange costs no HBM traffic of its own and
// its transfer overlaps the pass's arithmetic. Every rank must take the same
// path: decided once, collectively (all ranks hold a second shard buffer).
void State::decide_fusion() {
  if (fuse_decided_) return;
  fuse_decided_ = true;
  fuse_ok_ = false;
  if (mode_ != Mode::Sharded || !comm_ || !comm_->peer_access() || jit_mode_ != 1 || world_ > 8) return;
  if (const char* e = std::getenv("QTB_FUSE_EXCHANGE"))
    if (std::atoi(e) == 0) return;
  ensure_alt();
  double* mine = d_scratch_ + kNormBlocks;
  double* all = d_scratch_ + kNormBlocks + 1;
  const double have = (alt_ && bound_ == 0) ? 1.0 : 0.0;
  cuda_check(cudaMemcpyAsync(mine, &have, sizeof(double), cudaMemcpyHostToDevice, stream_), "fusion vote");
  std::string err;
  if (!comm_->allgather_double(mine, all, 1, stream_, &err)) fail(QT_ERR_NCCL, err);
  std::vector<double> votes(world_, 0.0);
  cuda_check(cudaMemcpyAsync(votes.data(), all, sizeof(double) * world_, cudaMemcpyDeviceToHost, stream_),
             "fusion vote readback");
  cuda_check(cudaStreamSynchronize(stream_), "fusion vote sync");
  fuse_ok_ = true;
  for (double v : votes) fuse_ok_ = fuse_ok_ && v == 1.0;
}

void State::exchange(const PlanPass& pass) {
  if (mode_ == Mode::Loopback) {
    for (const auto& gv : pass.exchange)
      cuda_check(launch_bitswap(psi_, buf_bits_, gv.first, gv.second, stream_),
                 "bitswap");
    stats.exchanged_bytes += pass.exchange.size() * (buffer_amps() / 2) * sizeof(double2);
    return;
  }
  if (mode_ != Mode::Sharded) fail(QT_ERR_ARG, "exchange on an unsharded state");
  const int k = static_cast<int>(pass.exchange.size());
  const int npeer = (1 << k) - 1;
  const uint64_t region = 1ull << (nlocal_ - k);
  // The step structure (piece size, offsets) depends only on the shard
  // geometry, never on this rank's buffer scheme: every rank of the group
  // must make the same sequence of grouped send/recv calls. At most 1/8 of
  // the shard (<= 2 GiB) is in flight per step, at least one amplitude per
  // peer.
  uint64_t cap = std::max<uint64_t>(1, (1ull << nlocal_) / 8);
  cap = std::min<uint64_t>(cap, 1ull << 27);
  cap = std::max<uint64_t>(cap, static_cast<uint64_t>(npeer));
  const std::vector<ExchangeStep> steps = exchange_schedule(rank_, nlocal_, pass.exchange, cap);
  // Two-buffer exchange (when a second shard fits in HBM): every peer's
  // piece is received straight into its final place in the second buffer,
  // this rank's own region is copied over with one device copy, and the
  // buffers swap roles -- the only HBM traffic beyond the transfer itself is
  // that 1/2^k of the shard (the receive-buffer scheme below copies the other
  // (2^k-1)/2^k back out of the receive buffer).
  ensure_alt();
  const bool two = alt_ && bound_ == 0;
  if (!two && d_tmp_amps_ < cap) {
    static std::mutex alloc_mu2;
    std::lock_guard<std::mutex> lk(alloc_mu2);
    cuda_check(cudaStreamSynchronize(stream_), "sync");
    cudaFree(d_tmp_);
    d_tmp_ = nullptr;
    d_tmp_amps_ = cap;
    cuda_check(cudaMalloc(&d_tmp_, d_tmp_amps_ * sizeof(double2)), "exchange buffer");
  }
  std::string err;
  std::vector<const void*> sends;
  std::vector<void*> recvs;
  std::vector<int> peers;
  for (const ExchangeStep& st : steps) {
    const size_t ne = st.peer.size();
    sends.resize(ne);
    recvs.resize(ne);
    peers.resize(ne);
    for (size_t i = 0; i < ne; ++i) {
      peers[i] = st.peer[i];
      sends[i] = psi_ + st.send_off[i];
      recvs[i] = two ? alt_ + st.send_off[i] : d_tmp_ + st.recv_off[i];
    }
    if (!comm_->sendrecv(static_cast<int>(ne), peers.data(), sends.data(), recvs.data(),
                         st.piece * sizeof(double2), stream_, &err))
      fail(QT_ERR_NCCL, err);
    if (!two)
      for (size_t i = 0; i < ne; ++i)
        cuda_check(cudaMemcpyAsync(const_cast<void*>(sends[i]), recvs[i],
                                   st.piece * sizeof(double2), cudaMemcpyDeviceToDevice, stream_),
                   "exchange copy");
  }
  stats.exchanged_bytes += static_cast<uint64_t>(npeer) * region * sizeof(double2);
  if (two) {
    // this rank's own region: the victim bits equal its global bits
    uint64_t above = 0, vpat = 0;
    own_region(rank_, nlocal_, pass.exchange, &above, &vpat);
    cuda_check(launch_copy_runs(alt_, psi_, above, vpat, min_victim(nlocal_, pass.exchange), region,
                                stream_),
               "exchange own region");
    std::swap(psi_, alt_);
    pool_[0] = psi_;
    stats.exchange_local_bytes += 2ull * region * sizeof(double2);
  } else {
    stats.exchange_local_bytes += 2ull * npeer * region * sizeof(double2);
  }
}

// Top-K readout (the reference's amplitude report, qtask_cli.cpp:53-86:
// partial_sort by std::norm descending, index ascending) without copying the
// state to the host: an exact radix select over the 64-bit |a|^2 key, 11 bits
// per pass (a pass = one HBM sweep + a 16 KiB histogram readback); as soon as
// the selected bin holds <= 2^16 keys, one collecting pass gathers every key
// >= the bin's floor and the host sorts those few. Fully tied states (e.g. a
// uniform superposition) go to the exact threshold and rank its ties in
// logical index order (two more sweeps). Permuted (loopback) states are
// streamed in logical-order chunks through the gather kernel.
// Sharded states (one rank per GPU): every rank selects the k largest of its
// shard -- read in the order of the full logical index, so ties break exactly
// as on one GPU -- the ranks all-gather their k (key, index) pairs and each
// merges them into the same global list. Collective: every rank calls it.
std::vector<TopkItem> State::top_k(uint64_t k) {
  if (mode_ != Mode::Sharded) {
    std::vector<int> pm(perm_.begin(), perm_.end());
    return top_k_local(k, n_, pm);
  }
  // local logical qubits (ascending) and the fixed bits of this rank's global ones
  std::vector<int> local_q, pm;
  uint64_t fixed = 0;
  for (int q = 0; q < n_; ++q) {
    if (perm_[q] < nlocal_) {
      local_q.push_back(q);
      pm.push_back(perm_[q]);
    } else if ((static_cast<uint64_t>(rank_) >> (perm_[q] - nlocal_)) & 1ull) {
      fixed |= 1ull << q;
    }
  }
  const uint64_t kl = std::min<uint64_t>(k, 1ull << nlocal_);
  if (kl == 0) return {};
  std::vector<TopkItem> mine = top_k_local(kl, nlocal_, pm);
  for (TopkItem& it : mine) {
    uint64_t full = fixed;
    for (int i = 0; i < nlocal_; ++i)
      if ((it.index >> i) & 1ull) full |= 1ull << local_q[i];
    it.index = full;
  }
  TopkItem pad{};
  pad.index = ~0ull;
  mine.resize(kl, pad);
  static_assert(sizeof(TopkItem) == 4 * sizeof(double), "TopkItem travels as four doubles");
  double *d_in = nullptr, *d_out = nullptr;
  cuda_check(cudaMalloc(&d_in, sizeof(TopkItem) * kl), "topk gather");
  cuda_check(cudaMalloc(&d_out, sizeof(TopkItem) * kl * world_), "topk gather");
  struct Free2 {
    void *a, *b;
    ~Free2() {
      cudaFree(a);
      cudaFree(b);
    }
  } guard_{d_in, d_out};
  cuda_check(cudaMemcpyAsync(d_in, mine.data(), sizeof(TopkItem) * kl, cudaMemcpyHostToDevice, stream_),
             "topk gather upload");
  std::string err;
  if (!comm_->allgather_double(d_in, d_out, 4 * kl, stream_, &err)) fail(QT_ERR_NCCL, err);
  std::vector<TopkItem> all(kl * world_);
  cuda_check(cudaMemcpyAsync(all.data(), d_out, sizeof(TopkItem) * all.size(), cudaMemcpyDeviceToHost, stream_),
             "topk gather readback");
  sync();
  all.erase(std::remove_if(all.begin(), all.end(), [](const TopkItem& a) { return a.index == ~0ull; }), all.end());
  std::sort(all.begin(), all.end(), [](const TopkItem& a, const TopkItem& b) {
    return a.key != b.key ? a.key > b.key : a.index < b.index;
  });
  if (all.size() > k) all.resize(k);
  return all;
}

// The k largest |a|^2 of the 2^bits amplitudes of psi_, read through the bit
// permutation pm (position i of the returned index <-> physical bit pm[i]).
std::vector<TopkItem> State::top_k_local(uint64_t k, int bits, const std::vector<int>& perm) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  const uint64_t total = 1ull << bits;
  k = std::min(k, total);
  if (k == 0) return {};
  bool identity = true;
  for (int q = 0; q < bits; ++q) identity = identity && perm[q] == q;
  const uint64_t chunk = 1ull << 22;
  std::vector<uint8_t> pm(bits);
  for (int q = 0; q < bits; ++q) pm[q] = static_cast<uint8_t>(perm[q]);
  if (!identity && d_tmp_amps_ < std::min(total, chunk)) {
    cudaFree(d_tmp_);
    d_tmp_ = nullptr;
    d_tmp_amps_ = std::min(total, chunk);
    cuda_check(cudaMalloc(&d_tmp_, d_tmp_amps_ * sizeof(double2)), "gather buffer");
  }
  auto for_chunks = [&](const auto& fn) {
    if (identity) {
      fn(static_cast<const double2*>(psi_), total, uint64_t{0});
      return;
    }
    for (uint64_t off = 0; off < total; off += chunk) {
      const uint64_t c = std::min(chunk, total - off);
      cuda_check(launch_gather(psi_, d_tmp_, off, c, pm.data(), bits, stream_), "gather");
      fn(static_cast<const double2*>(d_tmp_), c, off);
    }
  };
  const uint64_t cap = 1ull << 16;
  unsigned long long *d_hist = nullptr, *d_n = nullptr;
  TopkItem* d_items = nullptr;
  cuda_check(cudaMalloc(&d_hist, sizeof(unsigned long long) * kTopkBins), "topk hist");
  cuda_check(cudaMalloc(&d_n, sizeof(unsigned long long)), "topk counter");
  cuda_check(cudaMalloc(&d_items, sizeof(TopkItem) * (k + cap)), "topk items");
  struct Free {
    void* a[3];
    ~Free() {
      for (void* p : a) cudaFree(p);
    }
  } guard_{{d_hist, d_n, d_items}};
  std::vector<unsigned long long> h(kTopkBins);
  std::vector<TopkItem> items;
  auto finish = [&](uint64_t count) {
    items.resize(count);
    cuda_check(cudaMemcpyAsync(items.data(), d_items, sizeof(TopkItem) * count,
                               cudaMemcpyDeviceToHost, stream_),
               "topk readback");
    sync();
    std::sort(items.begin(), items.end(), [](const TopkItem& a, const TopkItem& b) {
      return a.key != b.key ? a.key > b.key : a.index < b.index;
    });
    if (items.size() > k) items.resize(k);
  };
  uint64_t prefix = 0, pmask = 0, c_gt = 0;
  int shift = 64;
  while (shift > 0) {
    const int bits = std::min(kTopkBits, shift);
    shift -= bits;
    cuda_check(cudaMemsetAsync(d_hist, 0, sizeof(unsigned long long) * kTopkBins, stream_),
               "topk hist reset");
    for_chunks([&](const double2* src, uint64_t c, uint64_t) {
      cuda_check(launch_topk_hist(src, c, prefix, pmask, shift, d_hist, stream_), "topk hist");
    });
    cuda_check(cudaMemcpyAsync(h.data(), d_hist, sizeof(unsigned long long) * kTopkBins,
                               cudaMemcpyDeviceToHost, stream_),
               "topk hist readback");
    sync();
    uint64_t above = 0;
    int b = (1 << bits) - 1;
    for (; b > 0; --b) {
      if (c_gt + above + h[b] >= k) break;
      above += h[b];
    }
    c_gt += above;
    prefix |= static_cast<uint64_t>(b) << shift;
    pmask |= ((1ull << bits) - 1) << shift;
    if (h[b] <= cap) {
      // every key >= the bin's floor: c_gt + h[b] <= k + cap of them
      const uint64_t want = c_gt + h[b];
      cuda_check(cudaMemsetAsync(d_n, 0, sizeof(unsigned long long), stream_), "topk counter");
      for_chunks([&](const double2* src, uint64_t c, uint64_t base) {
        cuda_check(launch_topk_collect(src, c, base, prefix, d_items, d_n, k + cap, stream_),
                   "topk collect");
      });
      finish(want);
      return items;
    }
  }
  // exact threshold key t = prefix with c_gt keys above it: rank its ties
  const uint64_t t = prefix, r = k - c_gt;
  const int blocks_max = 8 * sms_;
  std::vector<std::vector<unsigned long long>> tie_off;
  unsigned long long* d_ties = nullptr;
  cuda_check(cudaMalloc(&d_ties, sizeof(unsigned long long) * blocks_max), "topk ties");
  struct FreeOne {
    void* p;
    ~FreeOne() { cudaFree(p); }
  } guard2_{d_ties};
  uint64_t running = 0;
  for_chunks([&](const double2* src, uint64_t c, uint64_t) {
    const int blocks = static_cast<int>(std::min<uint64_t>(blocks_max, (c + 255) / 256));
    const uint64_t per = (c + blocks - 1) / blocks;
    cuda_check(launch_topk_ties(src, c, per, blocks, t, d_ties, stream_), "topk ties");
    std::vector<unsigned long long> cnt(blocks);
    cuda_check(cudaMemcpyAsync(cnt.data(), d_ties, sizeof(unsigned long long) * blocks,
                               cudaMemcpyDeviceToHost, stream_),
               "topk ties readback");
    sync();
    std::vector<unsigned long long> off(blocks);
    for (int i = 0; i < blocks; ++i) {
      off[i] = running;
      running += cnt[i];
    }
    tie_off.push_back(std::move(off));
  });
  cuda_check(cudaMemsetAsync(d_n, 0, sizeof(unsigned long long), stream_), "topk counter");
  size_t ci = 0;
  for_chunks([&](const double2* src, uint64_t c, uint64_t base) {
    const std::vector<unsigned long long>& off = tie_off[ci++];
    const int blocks = static_cast<int>(off.size());
    const uint64_t per = (c + blocks - 1) / blocks;
    cuda_check(cudaMemcpyAsync(d_ties, off.data(), sizeof(unsigned long long) * blocks,
                               cudaMemcpyHostToDevice, stream_),
               "topk tie offsets");
    cuda_check(launch_topk_final(src, c, per, blocks, base, t, r, c_gt, d_ties, d_items, d_n,
                                 stream_),
               "topk final");
    sync();  // d_ties is rewritten for the next chunk
  });
  finish(k);
  return items;
}

double State::norm_squared() {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  double* out = d_scratch_ + kNormBlocks;
  cuda_check(launch_norm(psi_, buffer_amps(), d_scratch_, out, stream_), "norm");
  std::vector<double> parts(world_, 0.0);
  if (mode_ == Mode::Sharded) {
    std::string err;
    double* gathered = d_scratch_ + kNormBlocks + 1;
    if (!comm_->allgather_double(out, gathered, 1, stream_, &err)) fail(QT_ERR_NCCL, err);
    cuda_check(cudaMemcpyAsync(parts.data(), gathered, sizeof(double) * world_,
                               cudaMemcpyDeviceToHost, stream_),
               "norm readback");
  } else {
    cuda_check(cudaMemcpyAsync(parts.data(), out, sizeof(double),
                               cudaMemcpyDeviceToHost, stream_),
               "norm readback");
  }
  sync();
  double acc = 0.0;
  for (int r = 0; r < (mode_ == Mode::Sharded ? world_ : 1); ++r) acc += parts[r];
  return acc;
}

void State::sync() {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cuda_check(cudaMemcpyAsync(h_flag_, d_flag_, sizeof(int), cudaMemcpyDeviceToHost, stream_),
             "flag readback");
  cuda_check(cudaStreamSynchronize(stream_), "stream sync");
  if (comm_) {
    std::string err;
    if (!comm_->check_async(&err)) fail(QT_ERR_NCCL, err);
  }
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, ev0_, ev1_) == cudaSuccess) stats.device_ms = ms;
  cudaGetLastError();  // an unrecorded event pair is not an error here
  if (*h_flag_) {
    const int f = *h_flag_;
    *h_flag_ = 0;
    cuda_check(cudaMemsetAsync(d_flag_, 0, sizeof(int), stream_), "flag reset");
    cuda_check(cudaStreamSynchronize(stream_), "stream sync");
    // bit 2: a QTB_JIT_DEBUG bounds check of a compiled pass failed
    if (f & 4) fail(QT_ERR_CUDA, "compiled pass: index out of bounds (QTB_JIT_DEBUG)");
    fail(QT_ERR_NUMERIC, "non-finite amplitude");
  }
}

std::vector<std::pair<int, float>> State::last_timings(bool consume) {
  sync();
  std::vector<std::pair<int, float>> out;
  for (size_t i = 0; i < timings_used_; ++i) {
    float ms = -1.f;
    if (cudaEventElapsedTime(&ms, timings_[i].start, timings_[i].stop) != cudaSuccess) {
      cudaGetLastError();
      ms = -1.f;
    }
    out.emplace_back(timings_[i].kind, ms);
  }
  if (consume) timings_used_ = 0;
  return out;
}

void State::checkpoint_save(int slot) {
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  auto it = ckpt_.find(slot);
  if (it == ckpt_.end()) {
    double2* buf = nullptr;
    cuda_check(cudaMalloc(&buf, sizeof(double2) * buffer_amps()), "checkpoint allocation");
    it = ckpt_.emplace(slot, std::make_pair(buf, perm_)).first;
  }
  cuda_check(cudaMemcpyAsync(it->second.first, psi_, sizeof(double2) * buffer_amps(),
                             cudaMemcpyDeviceToDevice, stream_),
             "checkpoint save");
  it->second.second = perm_;
}

void State::checkpoint_restore(int slot) {
  auto it = ckpt_.find(slot);
  if (it == ckpt_.end()) fail(QT_ERR_ARG, "unknown checkpoint slot");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cuda_check(cudaMemcpyAsync(psi_, it->second.first, sizeof(double2) * buffer_amps(),
                             cudaMemcpyDeviceToDevice, stream_),
             "checkpoint restore");
  perm_ = it->second.second;
}

void State::checkpoint_drop_all() {
  cudaStreamSynchronize(stream_);
  for (auto& kv : ckpt_) cudaFree(kv.second.first);
  ckpt_.clear();
}

void State::checkpoint_drop(int slot) {
  auto it = ckpt_.find(slot);
  if (it == ckpt_.end()) return;
  cudaStreamSynchronize(stream_);
  cudaFree(it->second.first);
  ckpt_.erase(it);
}

void State::copy_from(const State& other) {
  if (other.buf_bits_ != buf_bits_) fail(QT_ERR_ARG, "geometry mismatch");
  cuda_check(cudaSetDevice(device_), "cudaSetDevice");
  cuda_check(cudaMemcpyAsync(psi_, other.psi_, sizeof(double2) * buffer_amps(),
                             cudaMemcpyDeviceToDevice, stream_),
             "state copy");
  perm_ = other.perm_;
}

}  // namespace qtb
