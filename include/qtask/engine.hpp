// qtask/engine.hpp -- drop-in qtask::Simulator (reference
// proj/include/qtask/engine.hpp:18-151) over the B200 engine's C ABI
// (qtask_c.h, libqtask_b200.so). Same member names, signatures, semantics
// and exception types: circuits built from nets and gates, insert / remove
// modifiers, update_state() (first call simulates everything, later calls
// re-simulate from the last device checkpoint at or before the earliest
// edit), amplitude(s) / norm_squared readout, StaleStateError while
// modifiers are pending, circuit() as a Circuit. UpdateStats and the
// introspection members (stage_views, graph, node_name, frontier_nodes,
// dump_graph) report the reference's partition DAG in its own units, from
// the engine's host partition model (csrc/qt_partition.hpp; on for states of
// at most 1024 partition blocks unless Config::partition_model says
// otherwise). The device does not execute partitions: it runs fused tile
// passes over whole checkpoint segments (UpdateStats::passes / gates /
// segments / restart_gate report that work).
#pragma once

#include <cstdint>
#include <deque>
#include <memory>
#include <ostream>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "qtask/circuit.hpp"
#include "qtask/gate.hpp"
#include "qtask/graph.hpp"
#include "qtask/plan.hpp"
#include "qtask/types.hpp"

namespace qtask {

/// Per-stage block store (engine.hpp:18-29). On the B200 engine the
/// amplitudes live in HBM checkpoints; the store records which blocks the
/// stage's executed partitions have materialised (copy-on-write semantics of
/// the reference: untouched blocks resolve to an earlier stage).
struct BlockStore {
  std::uint64_t block_size = 0;
  std::vector<std::uint8_t> flags;
  bool materialized(std::uint64_t b) const { return b < flags.size() && flags[b] != 0; }
};

/// Result of the most recent update_state (engine.hpp:32-39), plus the
/// device work behind it.
struct UpdateStats {
  bool full = false;
  std::size_t executed_partitions = 0;
  std::size_t materialized_blocks = 0;
  std::vector<std::uint64_t> rewritten_blocks;  // sorted
  std::uint64_t rewritten_amplitudes = 0;
  // false: the partition model is off for this state; the fields above then
  // count the device work (passes as partitions, the whole state rewritten)
  bool reference_units = false;
  // device work of the update
  std::uint64_t passes = 0;          // fused tile passes executed
  std::uint64_t restart_gate = 0;    // first re-simulated gate position
  std::uint64_t gates = 0;           // gates re-applied
  std::uint64_t segments = 0;        // checkpoint segments re-run
  double wall_ms = 0.0;
};

class Simulator {
 public:
  explicit Simulator(int num_qubits, Config cfg = Config{}) : cfg_(cfg), circuit_(num_qubits) {
    validate_config(cfg);  // the C ABI would read 0 as "default"
    qt_config c{};
    c.block_size = cfg.block_size;
    c.threads = cfg.threads;
    c.device = cfg.device;
    c.tile_qubits = cfg.tile_qubits;
    c.max_checkpoints = cfg.max_checkpoints;
    c.checkpoint_fraction = cfg.checkpoint_fraction;
    c.segment_gates = cfg.segment_gates;
    c.compiled = cfg.compiled;
    c.partition_model = cfg.partition_model;
    detail::check(qt_sim_create(num_qubits, &c, &s_));
  }
  ~Simulator() { qt_sim_destroy(s_); }
  Simulator(const Simulator&) = delete;
  Simulator& operator=(const Simulator&) = delete;

  int num_qubits() const { return circuit_.num_qubits(); }
  const Config& config() const { return cfg_; }
  std::uint64_t block_size() const { return qt_sim_block_size(s_); }
  std::uint64_t total_blocks() const { return qt_sim_total_blocks(s_); }
  const Circuit& circuit() const { return circuit_; }

  // -- circuit modifiers (engine.hpp:57-64)
  NetId insert_net_front() {
    std::uint32_t id = 0;
    detail::check(qt_sim_insert_net_front(s_, &id));
    ++version_;
    return circuit_.add_net(0, id);
  }
  NetId insert_net_back() {
    std::uint32_t id = 0;
    detail::check(qt_sim_insert_net_back(s_, &id));
    ++version_;
    return circuit_.add_net(circuit_.net_order().size(), id);
  }
  NetId insert_net_after(NetId after) {
    std::uint32_t id = 0;
    detail::check(qt_sim_insert_net_after(s_, after, &id));
    ++version_;
    return circuit_.add_net(circuit_.net_position(after) + 1, id);
  }
  void remove_net(NetId n) {
    detail::check(qt_sim_remove_net(s_, n));
    ++version_;
    circuit_.remove_net(n);
  }
  GateId insert_gate(GateKind kind, NetId net, int target) {
    return insert(kind, 0.0, 0.0, 0.0, net, target, -1);
  }
  GateId insert_gate(GateKind kind, double theta, NetId net, int target) {
    return insert(kind, theta, 0.0, 0.0, net, target, -1);
  }
  GateId insert_gate(GateKind kind, NetId net, int target, int control) {
    return insert(kind, 0.0, 0.0, 0.0, net, target, control);
  }
  // additive: U3(theta, phi, lambda) = RZ(phi) RY(theta) RZ(lambda)
  GateId insert_u3(double theta, double phi, double lambda, NetId net, int target) {
    return insert(GateKind::U3, theta, phi, lambda, net, target, -1);
  }
  void remove_gate(GateId g) {
    detail::check(qt_sim_remove_gate(s_, g));
    ++version_;
    circuit_.remove_gate(g);
  }

  // -- state update (engine.hpp:71)
  void update_state() {
    detail::check(qt_sim_update_state(s_));
    ++version_;
  }

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
  void dump_graph(std::ostream& os) const {
    std::size_t need = 0;
    detail::check(qt_sim_dump_graph(s_, nullptr, 0, &need));
    std::string buf(need, '\0');
    detail::check(qt_sim_dump_graph(s_, &buf[0], need, &need));
    os << buf.c_str();
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

  const UpdateStats& last_update() const {
    qt_run_stats s{};
    qt_sim_last_update(s_, &s);
    UpdateStats u;
    u.full = s.full != 0;
    u.passes = s.passes;
    u.restart_gate = s.restart_gate;
    u.gates = s.gates;
    u.segments = s.segments;
    u.wall_ms = s.device_ms;
    qt_update_account a{};
    detail::check(qt_sim_update_account(s_, &a, nullptr, 0));
    if (a.valid) {
      u.reference_units = true;
      u.full = a.full != 0;
      u.executed_partitions = a.executed_partitions;
      u.materialized_blocks = a.materialized_blocks;
      u.rewritten_amplitudes = a.rewritten_amplitudes;
      u.rewritten_blocks.resize(a.rewritten_block_count);
      detail::check(qt_sim_update_account(s_, &a, u.rewritten_blocks.data(), u.rewritten_blocks.size()));
    } else {
      u.executed_partitions = s.executed_partitions;
      u.rewritten_amplitudes = s.rewritten_amplitudes;
    }
    last_ = std::move(u);
    return last_;
  }
  bool pending_modifiers() const { return qt_sim_pending(s_) != 0; }

  // -- introspection (engine.hpp:87-100), from the host partition model.
  // Pointers stay valid while the circuit and state are not modified.
  struct StageView {
    StageId id = 0;
    NetId net = kNoNet;
    GateId gate = kNoGate;
    StageKind kind = StageKind::PermuteScale;
    const std::vector<PartitionSpec>* partitions = nullptr;
    const std::vector<NodeId>* nodes = nullptr;
    const BlockStore* store = nullptr;  // null for Sync stages
  };
  /// Stages in execution order (empty when the partition model is off).
  std::vector<StageView> stage_views() const {
    const Snapshot& sn = snapshot();
    std::vector<StageView> out;
    for (std::size_t i = 0; i < sn.stages.size(); ++i) {
      StageView v;
      v.id = sn.stages[i].id;
      v.net = sn.stages[i].net;
      v.gate = sn.stages[i].gate;
      v.kind = sn.stages[i].kind;
      v.partitions = &sn.parts[i];
      v.nodes = &sn.nodes[i];
      v.store = v.kind == StageKind::Sync ? nullptr : &sn.stores[i];
      out.push_back(v);
    }
    return out;
  }
  const PartitionGraph& graph() const { return snapshot().graph; }
  std::string node_name(NodeId id) const {
    std::size_t need = 0;
    detail::check(qt_sim_node_name(s_, id, nullptr, 0, &need));
    std::string buf(need, '\0');
    detail::check(qt_sim_node_name(s_, id, &buf[0], need, &need));
    return std::string(buf.c_str());
  }
  const std::set<NodeId>& frontier_nodes() const { return snapshot().frontiers; }

 private:
  struct StageRec {
    StageId id;
    NetId net;
    GateId gate;
    StageKind kind;
  };
  struct Snapshot {
    std::uint64_t version = ~std::uint64_t{0};
    std::vector<StageRec> stages;
    std::vector<std::vector<PartitionSpec>> parts;
    std::vector<std::vector<NodeId>> nodes;
    std::vector<BlockStore> stores;
    PartitionGraph graph;
    std::set<NodeId> frontiers;
  };

  const Snapshot& snapshot() const {
    if (!snaps_.empty() && snaps_.back()->version == version_) return *snaps_.back();
    auto sn = std::make_shared<Snapshot>();
    sn->version = version_;
    qt_model_sizes z{};
    detail::check(qt_sim_model_snapshot(s_, &z, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr));
    std::vector<qt_model_stage> st(z.stages);
    std::vector<qt_model_part> pa(z.parts);
    std::vector<qt_model_task> ta(z.tasks);
    std::vector<std::uint64_t> ed(2 * z.edges), fr(z.frontiers);
    std::vector<std::uint8_t> mat(z.stages * z.blocks);
    if (z.valid)
      detail::check(qt_sim_model_snapshot(s_, &z, st.data(), pa.data(), ta.data(), ed.data(), mat.data(),
                                          fr.data()));
    const std::uint64_t nb = z.blocks;
    const std::uint64_t bs = nb ? (std::uint64_t{1} << num_qubits()) / nb : 0;
    PartitionGraph& g = sn->graph;
    PartitionGraph::Node out;
    out.id = kOutputNode;
    out.is_output = true;
    out.read = BlockRange{0, nb ? nb - 1 : 0};
    if (z.valid) g.nodes_.emplace(kOutputNode, out);
    for (std::size_t i = 0; i < st.size(); ++i) {
      const StageKind kind = static_cast<StageKind>(st[i].kind);
      sn->stages.push_back(StageRec{st[i].id, st[i].net, st[i].gate, kind});
      std::vector<PartitionSpec> ps;
      std::vector<NodeId> ns;
      for (std::uint64_t k = 0; k < st[i].num_parts; ++k) {
        const qt_model_part& p = pa[st[i].first_part + k];
        PartitionSpec spec;
        spec.first_block = p.first_block;
        spec.last_block = p.last_block;
        for (std::uint64_t t = 0; t < p.num_tasks; ++t) {
          const qt_model_task& tk = ta[p.first_task + t];
          spec.tasks.push_back(TaskSpec{tk.first_op, tk.last_op, tk.region_lo, tk.region_hi});
        }
        ps.push_back(std::move(spec));
        ns.push_back(p.node);
        // graph node: read / write ranges by stage kind (engine.cpp:159-171)
        PartitionGraph::Node nd;
        nd.id = p.node;
        nd.stage = st[i].id;
        nd.index = static_cast<std::uint32_t>(k);
        nd.kind = kind;
        const BlockRange own{p.first_block, p.last_block}, full{0, nb - 1};
        nd.read = kind == StageKind::PermuteScale ? own : full;
        nd.write = kind == StageKind::Sync ? full : own;
        nd.has_write = true;
        g.nodes_.emplace(nd.id, std::move(nd));
      }
      g.stages_.emplace_back(st[i].id, ns);
      sn->parts.push_back(std::move(ps));
      sn->nodes.push_back(std::move(ns));
      BlockStore bsr;
      bsr.block_size = bs;
      if (kind != StageKind::Sync) bsr.flags.assign(mat.begin() + i * nb, mat.begin() + (i + 1) * nb);
      sn->stores.push_back(std::move(bsr));
    }
    for (std::size_t e = 0; e < z.edges; ++e) {
      const NodeId a = ed[2 * e], b = ed[2 * e + 1];
      g.edges_.emplace_back(a, b);
      g.nodes_[a].succs.insert(b);
      g.nodes_[b].preds.insert(a);
    }
    sn->frontiers.insert(fr.begin(), fr.end());
    snaps_.push_back(std::move(sn));
    while (snaps_.size() > 16) snaps_.pop_front();  // views into older snapshots may still be held
    return *snaps_.back();
  }

  GateId insert(GateKind kind, double theta, double phi, double lambda, NetId net, int target,
                int control) {
    const double p[3] = {theta, phi, lambda};
    std::uint32_t g = 0;
    detail::check(qt_sim_insert_gate(s_, static_cast<int>(kind), p, net, target, control, &g));
    ++version_;
    return circuit_.add_gate(g, kind, theta, phi, lambda, net, target, control);
  }

  qt_sim* s_ = nullptr;
  Config cfg_;
  Circuit circuit_;
  std::uint64_t version_ = 0;
  mutable UpdateStats last_;
  mutable std::deque<std::shared_ptr<Snapshot>> snaps_;
};

}  // namespace qtask
