// qt_sim.cpp -- the incremental engine behind qtask::Simulator.
//
// Reference semantics kept (engine.hpp:46-151, engine.cpp:58-124, 392-504,
// circuit.cpp:8-135):
//   * modifiers validate exactly like Circuit (UnknownNet, InvalidPosition,
//     BadQubit, NetConflict, UnknownGate, non-finite angle -> Error);
//   * update_state simulates everything on the first call and afterwards only
//     what the modifiers since the last call affect;
//   * amplitude queries throw StaleStateError while modifiers are pending;
//   * NumericError keeps the pending edits so a later update retries;
//   * results are deterministic (fixed plan, fixed reduction order).
// What changes: the reference tracks affected work as a partition DAG with
// per-stage copy-on-write block stores (graph.cpp:116-251, engine.hpp:18-29).
// On BASELINE-style circuits every update rewrote 100% of the amplitudes
// (SURVEY.md 0.6), so the savings come from skipping gates upstream of the
// edit. Here the state after gate position P is kept as a device-resident
// checkpoint for a chain of segment boundaries P_1 < P_2 < ...; an edit at
// position p invalidates the checkpoints after p, and update_state restarts
// from the last surviving one, writing the re-simulated segments out of
// place into free chain buffers (the first pass of a segment reads the
// previous checkpoint, so saving a checkpoint costs no extra HBM traffic).
#include "qt_sim.hpp"
#include "qt_jit.hpp"

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>

#include "qt_gates.hpp"

#include <nvtx3/nvToolsExt.h>

namespace qtb {

constexpr uint64_t kMinSegmentGates = 256;
// the partition model runs (auto) for states of at most this many partition
// blocks: its graph holds one node per block for every MxV stage
constexpr uint64_t kModelMaxBlocks = 1024;
constexpr size_t kSegmentPlanCache = 512;  // cached segment plans (cleared when full)

Sim::Sim(int nqubits, const qt_config* cfg) : n_(nqubits) {
  if (nqubits < 1 || nqubits > 40)
    fail(QT_ERR_BAD_QUBIT, "qubit count must be in [1, 40]");
  if (cfg) cfg_ = *cfg;
  if (cfg_.block_size == 0) cfg_.block_size = 256;
  // plan.cpp:7-13
  const bool pow2 = cfg_.block_size >= 2 && (cfg_.block_size & (cfg_.block_size - 1)) == 0;
  if (!pow2) fail(QT_ERR_ARG, "block size must be a power of two >= 2");
  const uint64_t dim = 1ull << n_;
  bs_ = cfg_.block_size < dim ? cfg_.block_size : dim;  // plan.hpp:26-35
  nblocks_ = dim / bs_;
  qt_config scfg = cfg_;
  // the incremental engine runs hybrid compiled passes by default: segments
  // re-simulated unchanged after an edit hit the compile cache (-1: the
  // interpreter only)
  if (scfg.compiled == 0) scfg.compiled = 2;
  if (scfg.compiled < 0) scfg.compiled = 0;
  st_.reset(new State(n_, Mode::Single, 1, 0, nullptr, &scfg));
  const int want = cfg_.max_checkpoints > 0 ? cfg_.max_checkpoints + 1 : 48;
  const double frac = cfg_.checkpoint_fraction > 0 ? cfg_.checkpoint_fraction : 0.85;
  nbuf_ = st_->grow_pool(want, frac);
  if (const char* e = std::getenv("QTB_SIM_TRACE")) trace_ = std::atoi(e) != 0;
  const int pm = cfg_.partition_model;
  if (pm > 0 || (pm == 0 && nblocks_ <= kModelMaxBlocks)) {
    model_.reset(new PartitionModel(n_, cfg_.block_size));
    model_thread_ = std::thread([this] { model_worker(); });
  }
}

Sim::~Sim() {
  if (model_thread_.joinable()) {
    {
      std::lock_guard<std::mutex> lk(q_mu_);
      stop_ = true;
    }
    q_cv_.notify_all();
    model_thread_.join();
  }
}

void Sim::post(std::function<void(PartitionModel&)> ev) {
  if (!model_) return;
  {
    std::lock_guard<std::mutex> lk(q_mu_);
    events_.push_back(std::move(ev));
  }
  q_cv_.notify_one();
}

void Sim::model_worker() {
  for (;;) {
    std::function<void(PartitionModel&)> ev;
    {
      std::unique_lock<std::mutex> lk(q_mu_);
      q_cv_.wait(lk, [&] { return stop_ || !events_.empty(); });
      if (stop_) return;  // destruction: the model goes away, pending events with it
      ev = std::move(events_.front());
      events_.pop_front();
      busy_ = true;
    }
    {
      std::lock_guard<std::mutex> mk(model_mu_);
      try {
        ev(*model_);
      } catch (const std::exception& e) {
        if (model_error_.empty()) model_error_ = e.what();
      }
    }
    {
      std::lock_guard<std::mutex> lk(q_mu_);
      busy_ = false;
    }
    drained_cv_.notify_all();
  }
}

const PartitionModel* Sim::model(std::unique_lock<std::mutex>* lk) {
  if (!model_) return nullptr;
  {
    std::unique_lock<std::mutex> q(q_mu_);
    drained_cv_.wait(q, [&] { return events_.empty() && !busy_; });
  }
  *lk = std::unique_lock<std::mutex>(model_mu_);
  if (!model_error_.empty()) fail(QT_ERR_ARG, "partition model: " + model_error_);
  return model_.get();
}

// ---- circuit model (circuit.cpp) -------------------------------------------

uint32_t Sim::new_net(size_t at) {
  const uint32_t id = next_net_++;
  nets_.emplace(id, std::vector<uint32_t>{});
  index_.insert(id, at);
  order_valid_ = false;
  pending_ = true;
  return id;
}

uint32_t Sim::insert_net_front() {
  const uint32_t id = new_net(0);
  post([id](PartitionModel& m) { m.insert_net(id, 0); });
  return id;
}
uint32_t Sim::insert_net_back() {
  const uint32_t id = new_net(index_.nets());
  post([id](PartitionModel& m) { m.insert_net_back(id); });
  return id;
}

uint32_t Sim::insert_net_after(uint32_t after) {
  if (!index_.has(after)) fail(QT_ERR_INVALID_POSITION, "insert_net: unknown anchor net");
  const uint32_t id = new_net(index_.rank(after) + 1);
  post([id, after](PartitionModel& m) { m.insert_net(id, after); });
  return id;
}

void Sim::remove_net(uint32_t net) {
  auto it = nets_.find(net);
  if (it == nets_.end()) fail(QT_ERR_UNKNOWN_NET, "remove_net: unknown net");
  const std::vector<uint32_t> gs = it->second;
  for (uint32_t g : gs) remove_gate(g);
  nets_.erase(net);
  index_.erase(net);
  order_valid_ = false;
  post([net](PartitionModel& m) { m.remove_net(net); });
  pending_ = true;
}

const std::vector<uint32_t>& Sim::net_gates(uint32_t net) const {
  auto it = nets_.find(net);
  if (it == nets_.end()) fail(QT_ERR_UNKNOWN_NET, "unknown net");
  return it->second;
}

void Sim::gate_info(uint32_t gate, qt_gate* out, uint32_t* net) const {
  auto it = gates_.find(gate);
  if (it == gates_.end()) fail(QT_ERR_UNKNOWN_GATE, "unknown gate");
  if (out) *out = it->second.g;
  if (net) *net = it->second.net;
}

const std::vector<uint32_t>& Sim::net_order() const {
  if (!order_valid_) {
    index_.order(&order_);
    order_valid_ = true;
  }
  return order_;
}

uint64_t Sim::position_of_net_end(uint32_t net) const {
  if (!index_.has(net)) fail(QT_ERR_UNKNOWN_NET, "unknown net");
  return index_.gates_before(net) + index_.gates_of(net);
}

uint64_t Sim::position_of_gate(uint32_t gate) const {
  auto it = gates_.find(gate);
  if (it == gates_.end()) fail(QT_ERR_UNKNOWN_GATE, "unknown gate");
  // a net holds at most one gate per qubit (circuit.cpp:122-135): a short scan
  const auto& gs = nets_.at(it->second.net);
  return index_.gates_before(it->second.net) +
         static_cast<uint64_t>(std::find(gs.begin(), gs.end(), gate) - gs.begin());
}

void Sim::edited_at(uint64_t pos) {
  // checkpoints strictly after the edit no longer describe the circuit
  while (!chain_.empty() && chain_.back().pos > pos) chain_.pop_back();
  pending_ = true;
}

uint32_t Sim::insert_gate(int kind, const double* params, uint32_t net,
                          int target, int control) {
  auto it = nets_.find(net);
  if (it == nets_.end()) fail(QT_ERR_UNKNOWN_NET, "insert_gate: unknown net");
  qt_gate g{};
  g.kind = kind;
  g.target = target;
  g.control = is_two_qubit_kind(kind) ? control : (control < 0 ? -1 : control);
  if (params) {
    g.theta = params[0];
    g.phi = params[1];
    g.lambda = params[2];
  }
  if (!valid_kind(kind)) fail(QT_ERR_ARG, "unknown gate kind");
  // circuit.cpp:51-65
  if (target < 0 || target >= n_) fail(QT_ERR_BAD_QUBIT, "target qubit out of range");
  if (is_two_qubit_kind(kind)) {
    if (control < 0 || control >= n_) fail(QT_ERR_BAD_QUBIT, "second qubit out of range");
    if (control == target) fail(QT_ERR_BAD_QUBIT, "two-qubit gate needs distinct qubits");
  } else if (control != -1) {
    fail(QT_ERR_BAD_QUBIT, "single-qubit gate takes no control");
  }
  if (!std::isfinite(g.theta) || !std::isfinite(g.phi) || !std::isfinite(g.lambda))
    fail(QT_ERR_ARG, "rotation angle must be finite");
  // circuit.cpp:122-135
  const bool two = is_two_qubit_kind(kind);
  for (uint32_t other : it->second) {
    const qt_gate& o = gates_.at(other).g;
    const bool hits = o.target == target || (two && o.target == control) ||
                      o.control == target ||
                      (two && o.control >= 0 && o.control == control);
    if (hits) fail(QT_ERR_NET_CONFLICT, "gate would depend on another gate in the net");
  }
  const uint64_t pos = position_of_net_end(net);
  const uint32_t id = next_gate_++;
  gates_.emplace(id, GateRec{g, net});
  it->second.push_back(id);
  index_.add_gates(net, 1);
  edited_at(pos);
  post([id, g, net](PartitionModel& m) { m.insert_gate(id, g, net); });
  return id;
}

void Sim::remove_gate(uint32_t gate) {
  auto it = gates_.find(gate);
  if (it == gates_.end()) fail(QT_ERR_UNKNOWN_GATE, "remove_gate: unknown gate");
  const uint64_t pos = position_of_gate(gate);
  auto& gs = nets_.at(it->second.net);
  gs.erase(std::find(gs.begin(), gs.end(), gate));
  index_.add_gates(it->second.net, -1);
  gates_.erase(it);
  edited_at(pos);
  post([gate](PartitionModel& m) { m.remove_gate(gate); });
}

std::vector<qt_gate> Sim::flatten(std::vector<uint32_t>* ids, uint64_t from) const {
  std::vector<qt_gate> out;
  const uint64_t total = index_.gates();
  if (ids) ids->clear();
  if (from >= total) return out;
  out.reserve(total - from);
  if (ids) ids->reserve(total - from);
  // the net holding position `from`, then the nets after it
  uint64_t first = 0;
  const uint32_t start = index_.net_at_gate(from, &first);
  std::vector<uint32_t> tail;
  index_.order(&tail, index_.rank(start));
  uint64_t skip = from - first;
  for (uint32_t net : tail) {
    const auto& gs = nets_.at(net);
    for (size_t i = static_cast<size_t>(std::min<uint64_t>(skip, gs.size())); i < gs.size(); ++i) {
      out.push_back(gates_.at(gs[i]).g);
      if (ids) ids->push_back(gs[i]);
    }
    skip = 0;
  }
  return out;
}

// ---- update (engine.cpp:392-504) -------------------------------------------

void Sim::update_state() {
  const auto t0 = std::chrono::steady_clock::now();
  struct Range {  // NVTX range of the whole update (no-op without a profiler)
    Range() { nvtxRangePushA("qtask update_state"); }
    ~Range() { nvtxRangePop(); }
  } nvtx_range;
  qt_run_stats stats{};
  stats.full = ran_full_ ? 0 : 1;
  if (ran_full_ && !pending_) {
    last_ = stats;  // nothing pending: nothing executes
    post([](PartitionModel& m) { m.update(); });
    return;
  }
  const uint64_t N = index_.gates();
  if (!ran_full_) chain_.clear();
  const uint64_t restart = chain_.empty() ? 0 : chain_.back().pos;
  const size_t chain_keep = chain_.size();
  stats.restart_gate = restart;
  // only the gates from the restart position on are touched: ids[i - restart]
  // is the gate at circuit position i
  std::vector<uint32_t> ids;
  const std::vector<qt_gate> gates = flatten(&ids, restart);
  // segment boundaries of the last run, by gate identity: re-simulated
  // segments after an edit keep the same gates, hence the same plans (and
  // compiled passes in hybrid mode)
  std::vector<uint64_t> old_bounds;
  for (uint32_t g : bound_ids_) {
    if (!gates_.count(g)) continue;
    const uint64_t p = position_of_gate(g);
    if (p > restart) old_bounds.push_back(p);
  }
  std::sort(old_bounds.begin(), old_bounds.end());

  // segment length: the chain has nbuf_ buffers for N gates
  uint64_t seg = cfg_.segment_gates > 0 ? static_cast<uint64_t>(cfg_.segment_gates) : 0;
  if (seg == 0) {
    // >= 256 gates per segment from 20 qubits up: shorter segments break pass
    // fusion more than they save in restart distance (C5: 139 -> 300 gates
    // per segment cut the uniform-position update from 191 to 140 ms)
    seg = (N + static_cast<uint64_t>(nbuf_) - 1) / static_cast<uint64_t>(nbuf_);
    // small states are launch-bound: fine checkpoints (short restarts) win there
    seg = std::max<uint64_t>(seg, n_ >= kHybridMinQubits ? kMinSegmentGates : 64);
  }

  std::vector<char> used(nbuf_, 0);
  for (const Ckpt& c : chain_) used[c.buf] = 1;
  auto take_free = [&]() -> int {
    for (int b = 0; b < nbuf_; ++b)
      if (!used[b]) {
        used[b] = 1;
        return b;
      }
    return -1;
  };

  std::string err;
  bool clobbered = false;  // an existing checkpoint was advanced in place
  try {
    if (chain_.empty()) {
      // the initial |0...0> (engine.cpp:303-313)
      int b = take_free();
      std::vector<int> id(n_);
      for (int q = 0; q < n_; ++q) id[q] = q;
      st_->bind(b, id);
      st_->set_basis(0);
      chain_.push_back(Ckpt{0, b, id, 0});
    }
    uint64_t a = restart;
    // the last 10 % of the circuit gets half-length segments: edits there
    // (the reference's level-by-level building, the tail class of C5)
    // restart closer to the edit and re-plan (and run uncompiled) fewer gates
    const uint64_t tail_start = N - N / 10;
    while (a < N) {
      const uint64_t len = (a >= tail_start && seg >= 128) ? seg / 2 : seg;
      uint64_t b = std::min(N, a + len);
      auto ob = std::upper_bound(old_bounds.begin(), old_bounds.end(), a);
      if (ob != old_bounds.end() && *ob - a >= len / 2 && *ob - a <= 2 * len) b = *ob;
      int dst = take_free();
      bool in_place = false;
      if (dst < 0) {
        // no free buffer: run the rest in place on the newest checkpoint
        b = N;
        dst = chain_.back().buf;
        in_place = true;
        if (chain_.size() <= chain_keep) clobbered = true;
      }
      const Ckpt src = chain_.back();
      // a segment's gates (by identity) from the same qubit map plan the
      // same way: the plan and its lowering are cached across updates
      std::string key(reinterpret_cast<const char*>(ids.data() + (a - restart)), (b - a) * sizeof(uint32_t));
      key.append(reinterpret_cast<const char*>(src.perm.data()), src.perm.size() * sizeof(int));
      std::shared_ptr<State::PreparedPlan> pp;
      auto hit = seg_plans_.find(key);
      if (hit != seg_plans_.end()) {
        pp = hit->second;
      } else {
        std::vector<LOp> ops;
        ops.reserve(static_cast<size_t>(b - a));
        for (uint64_t i = a; i < b; ++i) {
          const int rc = lower_gate(gates[i - restart], n_, static_cast<uint32_t>(i), ops, &err);
          if (rc != QT_OK) fail(rc, err);
        }
        fuse_ops(ops, n_);
        pp = st_->prepare_ops(ops, &src.perm);
        if (seg_plans_.size() >= kSegmentPlanCache) seg_plans_.clear();
        seg_plans_.emplace(std::move(key), pp);
      }
      if (in_place) {
        st_->bind(dst, src.perm);
        st_->apply_prepared(*pp, b - a);
        chain_.back().pos = b;
        chain_.back().perm = st_->perm();
      } else {
        st_->bind(dst, src.perm);
        st_->apply_prepared(*pp, b - a, st_->buffer(src.buf), &src.perm);
        chain_.push_back(Ckpt{b, dst, st_->perm(), 0});
      }
      if (trace_) {
        const JitStats js = jit_stats();
        std::fprintf(stderr, "qtask-b200 sim: segment [%llu, %llu) passes %llu hits %llu misses %llu host %.2f ms\n",
                     static_cast<unsigned long long>(a), static_cast<unsigned long long>(b),
                     static_cast<unsigned long long>(st_->stats.passes),
                     static_cast<unsigned long long>(js.cache_hits - trace_hits_),
                     static_cast<unsigned long long>(js.misses - trace_misses_),
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
        trace_hits_ = js.cache_hits;
        trace_misses_ = js.misses;
      }
      stats.passes += st_->stats.passes;
      stats.kernel_launches += st_->stats.kernel_launches;
      stats.hbm_bytes += st_->stats.hbm_bytes;
      stats.gates += b - a;
      stats.plan_ms += st_->stats.plan_ms;
      stats.segments += 1;
      a = b;
    }
    st_->bind(chain_.back().buf, chain_.back().perm);
    const auto ts = std::chrono::steady_clock::now();
    st_->sync();  // raises QT_ERR_NUMERIC on a non-finite amplitude
    if (trace_)
      std::fprintf(stderr, "qtask-b200 sim: launched at %.2f ms, synced after %.2f ms more\n",
                   std::chrono::duration<double, std::milli>(ts - t0).count(),
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ts).count());
    bound_ids_.clear();
    for (Ckpt& c : chain_) {
      // checkpoints before the restart keep the gate that followed them
      // (gates before an edit are untouched); the others take it from this run
      if (c.pos >= restart) c.next_id = c.pos < N ? ids[c.pos - restart] : 0;
      if (c.pos > 0 && c.pos < N && c.next_id) bound_ids_.push_back(c.next_id);
    }
  } catch (const QtError&) {
    // keep the pending edits; checkpoints written by this run are dropped
    if (chain_.size() > chain_keep) chain_.resize(chain_keep);
    if (clobbered && !chain_.empty()) chain_.pop_back();
    if (!chain_.empty()) st_->bind(chain_.back().buf, chain_.back().perm);
    throw;
  }
  // UpdateStats (engine.hpp:32-39) in GPU terms: every re-simulated segment
  // rewrites the whole state, i.e. all partition blocks.
  stats.executed_partitions = stats.passes;
  stats.rewritten_amplitudes = stats.segments > 0 ? (1ull << n_) : 0;
  stats.device_ms = 0.0;
  const auto t1 = std::chrono::steady_clock::now();
  stats.device_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
  last_ = stats;
  pending_ = false;
  ran_full_ = true;
  post([](PartitionModel& m) { m.update(); });
}

void Sim::amplitudes(uint64_t first, uint64_t last, double* out) {
  if (pending_) fail(QT_ERR_STALE_STATE, "modifiers pending; call update_state first");
  if (first > last || (n_ < 64 && last >= (1ull << n_)))
    fail(QT_ERR_ARG, "amplitude range out of bounds");
  st_->read(first, last - first + 1, out);
}

std::vector<TopkItem> Sim::top_k(uint64_t k) {
  if (pending_) fail(QT_ERR_STALE_STATE, "modifiers pending; call update_state first");
  return st_->top_k(k);
}

double Sim::norm_squared() {
  // engine.cpp:551-564 reads the last committed state without a pending check
  return st_->norm_squared();
}

}  // namespace qtb
