// qtask/engine.hpp -- drop-in qtask::Simulator (reference
// proj/include/qtask/engine.hpp:46-100) over the B200 engine's C ABI
// (qtask_c.h, libqtask_b200.so). Same member names, signatures, semantics
// and exception types: circuits built from nets and gates, insert / remove
// modifiers, update_state() (first call simulates everything, later calls
// re-simulate from the last device checkpoint at or before the earliest
// edit), amplitude(s) / norm_squared readout, StaleStateError while
// modifiers are pending. The CPU partition-DAG introspection members
// (stage_views, graph, node_name, frontier_nodes, dump_graph) are not part
// of the GPU engine.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "qtask/gate.hpp"
#include "qtask/types.hpp"

namespace qtask {

// Reference Config (plan.hpp:17-20) + GPU knobs (0 = auto). Aggregate-init
// compatible with the reference's Config{block_size, threads}.
struct Config {
  std::uint64_t block_size = 256;
  unsigned threads = 0;
  int device = -1;
  int tile_qubits = 0;
  int max_checkpoints = 0;
  double checkpoint_fraction = 0.0;
  int segment_gates = 0;
  int compiled = 0;  // 0: hybrid compiled passes (NVRTC, cached segments), -1: interpreter only
};

// Reference UpdateStats (engine.hpp:32-39) in GPU terms.
struct UpdateStats {
  bool full = false;
  std::size_t executed_partitions = 0;  // fused tile passes executed
  std::uint64_t rewritten_amplitudes = 0;
  std::uint64_t restart_gate = 0;       // first re-simulated gate position
  std::uint64_t gates = 0;              // gates re-applied
  std::uint64_t segments = 0;           // checkpoint segments re-run
  double wall_ms = 0.0;
};

struct Gate {  // reference Gate (circuit.hpp:14-21)
  GateId id = kNoGate;
  GateKind kind = GateKind::X;
  double theta = 0.0;
  NetId net = kNoNet;
  int target = 0;
  int control = -1;
};

class Simulator;

// Read-only circuit view (reference Circuit, circuit.hpp:32-66).
class CircuitView {
 public:
  explicit CircuitView(const qt_sim* s) : s_(s) {}
  int num_qubits() const { return qt_sim_num_qubits(s_); }
  std::size_t num_gates() const { return qt_sim_num_gates(s_); }
  std::vector<NetId> net_order() const {
    std::vector<NetId> out(qt_sim_num_nets(s_));
    detail::check(qt_sim_net_order(s_, out.data(), out.size()));
    return out;
  }
  std::vector<GateId> net(NetId id) const {
    std::size_t n = 0;
    detail::check(qt_sim_net_gates(s_, id, nullptr, 0, &n));
    std::vector<GateId> out(n);
    detail::check(qt_sim_net_gates(s_, id, out.data(), n, &n));
    return out;
  }
  Gate gate(GateId id) const {
    qt_gate g{};
    std::uint32_t net = 0;
    detail::check(qt_sim_gate_info(s_, id, &g, &net));
    return Gate{id, static_cast<GateKind>(g.kind), g.theta, net, g.target, g.control};
  }
  // Flattened gate list in simulation order (what a dense oracle consumes).
  std::vector<qt_gate> gates() const {
    std::size_t n = 0;
    detail::check(qt_sim_export_gates(s_, nullptr, 0, &n));
    std::vector<qt_gate> out(n);
    detail::check(qt_sim_export_gates(s_, out.data(), n, &n));
    return out;
  }

 private:
  const qt_sim* s_;
};

class Simulator {
 public:
  explicit Simulator(int num_qubits, Config cfg = Config{}) : cfg_(cfg) {
    // validate_config (plan.cpp:7-13): the C ABI reads 0 as "default", the
    // reference rejects it like any non power of two
    if (cfg.block_size < 2 || (cfg.block_size & (cfg.block_size - 1)) != 0)
      throw Error("block size must be a power of two >= 2");
    qt_config c{};
    c.block_size = cfg.block_size;
    c.threads = cfg.threads;
    c.device = cfg.device;
    c.tile_qubits = cfg.tile_qubits;
    c.max_checkpoints = cfg.max_checkpoints;
    c.checkpoint_fraction = cfg.checkpoint_fraction;
    c.segment_gates = cfg.segment_gates;
    c.compiled = cfg.compiled;
    detail::check(qt_sim_create(num_qubits, &c, &s_));
  }
  ~Simulator() { qt_sim_destroy(s_); }
  Simulator(const Simulator&) = delete;
  Simulator& operator=(const Simulator&) = delete;
  Simulator(Simulator&& o) noexcept : s_(std::exchange(o.s_, nullptr)), cfg_(o.cfg_) {}

  int num_qubits() const { return qt_sim_num_qubits(s_); }
  const Config& config() const { return cfg_; }
  std::uint64_t block_size() const { return qt_sim_block_size(s_); }
  std::uint64_t total_blocks() const { return qt_sim_total_blocks(s_); }
  CircuitView circuit() const { return CircuitView(s_); }

  // -- circuit modifiers (engine.hpp:57-64)
  NetId insert_net_front() { return net(qt_sim_insert_net_front(s_, &tmp_)); }
  NetId insert_net_back() { return net(qt_sim_insert_net_back(s_, &tmp_)); }
  NetId insert_net_after(NetId after) { return net(qt_sim_insert_net_after(s_, after, &tmp_)); }
  void remove_net(NetId n) { detail::check(qt_sim_remove_net(s_, n)); }
  GateId insert_gate(GateKind kind, NetId net, int target) {
    return insert(kind, nullptr, net, target, -1);
  }
  GateId insert_gate(GateKind kind, double theta, NetId net, int target) {
    const double p[3] = {theta, 0.0, 0.0};
    return insert(kind, p, net, target, -1);
  }
  GateId insert_gate(GateKind kind, NetId net, int target, int control) {
    return insert(kind, nullptr, net, target, control);
  }
  // additive: U3(theta, phi, lambda)
  GateId insert_u3(double theta, double phi, double lambda, NetId net, int target) {
    const double p[3] = {theta, phi, lambda};
    return insert(GateKind::U3, p, net, target, -1);
  }
  void remove_gate(GateId g) { detail::check(qt_sim_remove_gate(s_, g)); }

  // -- state update (engine.hpp:71)
  void update_state() { detail::check(qt_sim_update_state(s_)); }

  // -- queries (engine.hpp:77-83)
  Complex amplitude(std::uint64_t index) const {
    double v[2];
    detail::check(qt_sim_amplitude(s_, index, v));
    return Complex{v[0], v[1]};
  }
  std::vector<Complex> amplitudes(std::uint64_t first, std::uint64_t last) const {
    if (first > last) detail::check(QT_ERR_ARG);
    std::vector<Complex> out(last - first + 1);
    detail::check(qt_sim_amplitudes(s_, first, last, reinterpret_cast<double*>(out.data())));
    return out;
  }
  double norm_squared() const {
    double v = 0.0;
    detail::check(qt_sim_norm_squared(s_, &v));
    return v;
  }
  // Amplitude report (reference tools/qtask_cli.cpp:53-86, additive here):
  // the k amplitudes of largest std::norm, ties by smaller index, selected
  // on the device; (index, amplitude) pairs, largest first.
  std::vector<std::pair<std::uint64_t, Complex>> top_k(std::uint64_t k) const {
    const std::uint64_t dim = std::uint64_t{1} << num_qubits();
    if (k > dim) k = dim;
    std::vector<std::uint64_t> idx(k ? k : 1);
    std::vector<Complex> amp(k ? k : 1);
    std::uint64_t n = 0;
    detail::check(qt_sim_top_k(s_, k, idx.data(), reinterpret_cast<double*>(amp.data()), &n));
    std::vector<std::pair<std::uint64_t, Complex>> out(n);
    for (std::uint64_t i = 0; i < n; ++i) out[i] = {idx[i], amp[i]};
    return out;
  }
  UpdateStats last_update() const {
    qt_run_stats s{};
    qt_sim_last_update(s_, &s);
    UpdateStats u;
    u.full = s.full != 0;
    u.executed_partitions = s.executed_partitions;
    u.rewritten_amplitudes = s.rewritten_amplitudes;
    u.restart_gate = s.restart_gate;
    u.gates = s.gates;
    u.segments = s.segments;
    u.wall_ms = s.device_ms;
    return u;
  }
  bool pending_modifiers() const { return qt_sim_pending(s_) != 0; }

 private:
  NetId net(int rc) {
    detail::check(rc);
    return tmp_;
  }
  GateId insert(GateKind kind, const double* p, NetId net, int target, int control) {
    std::uint32_t g = 0;
    detail::check(qt_sim_insert_gate(s_, static_cast<int>(kind), p, net, target, control, &g));
    return g;
  }

  qt_sim* s_ = nullptr;
  Config cfg_;
  std::uint32_t tmp_ = 0;
};

}  // namespace qtask
