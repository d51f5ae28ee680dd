// qt_partition.hpp -- host model of the reference's partition DAG, for the
// drop-in's reference-unit accounting and introspection.
//
// The B200 engine does not execute partitions: it re-simulates gate ranges
// from device checkpoints (qt_sim.cpp). The reference exposes its CPU data
// structure through the API, though -- UpdateStats in partition / block
// units (engine.hpp:32-39), stage_views / graph / node_name /
// frontier_nodes / dump_graph (engine.hpp:77-100) -- and its acceptance
// suite checks them (acceptance.cpp:180-395). This model restates the
// structure's semantics on the host, from the same modifier stream:
//   * element-op forms and their index hulls (element_ops.cpp:24-133),
//     task chunking, partition forming, one-partition-per-block MxV stages
//     (plan.cpp:26-89) and the per-net stage order (engine.cpp:204-285);
//   * the partition graph: nearest-writer / nearest-reader edge discovery
//     with interval masking, transitive pruning, reconnection on removal,
//     affected closure (graph.cpp:93-251);
//   * frontiers, the affected set of an update, and its accounting
//     (engine.cpp:186-202, 392-504): executed partitions, materialised
//     blocks, rewritten blocks; per-stage block materialisation (COW stores).
// Nothing here touches amplitudes. Its cost is the reference's (O(stages x
// partitions) per edit), so qt_sim.cpp runs it on a background thread and
// only for states with few partition blocks.
#pragma once

#include <cstdint>
#include <map>
#include <ostream>
#include <set>
#include <string>
#include <unordered_map>
#include <vector>

#include "qtask_c.h"

namespace qtb {

enum class PmKind : int32_t { Sync = 0, MatrixVector = 1, PermuteScale = 2 };

struct PmTask {
  uint64_t first_op = 0, last_op = 0, lo = 0, hi = 0;  // ops and their index hull (inclusive)
};
struct PmPart {
  uint64_t first_block = 0, last_block = 0;  // inclusive
  std::vector<PmTask> tasks;
};
struct PmRange {
  uint64_t first = 0, last = 0;  // inclusive
};

struct PmAccount {
  bool valid = false;
  bool full = false;
  uint64_t executed_partitions = 0;
  uint64_t materialized_blocks = 0;
  uint64_t rewritten_amplitudes = 0;
  std::vector<uint64_t> rewritten_blocks;  // sorted
};

class PartitionModel {
 public:
  // block_size: the configured block size (task chunk length); the block
  // granularity is min(block_size, 2^n) (plan.hpp:26-35)
  PartitionModel(int nqubits, uint64_t block_size);

  // -- the modifier stream (already validated by the engine) ------------
  void insert_net(uint32_t net, uint32_t after);  // after = 0: at the front
  void insert_net_back(uint32_t net);
  void remove_net(uint32_t net);                  // removes its gates first
  void insert_gate(uint32_t gate, const qt_gate& g, uint32_t net);
  void remove_gate(uint32_t gate);
  // a successful update_state: the affected set is executed
  void update();

  // -- reference-unit results ------------------------------------------
  const PmAccount& account() const { return last_; }
  struct StageInfo {
    uint32_t id = 0, net = 0, gate = 0;
    PmKind kind = PmKind::PermuteScale;
    const std::vector<PmPart>* parts = nullptr;
    const std::vector<uint64_t>* nodes = nullptr;
    const std::vector<uint8_t>* materialized = nullptr;  // per block (empty: Sync)
  };
  std::vector<StageInfo> stages() const;  // execution order
  std::vector<std::pair<uint64_t, uint64_t>> edges() const;  // sorted
  std::string node_name(uint64_t node) const;
  void dump_dot(std::ostream& os) const;
  const std::set<uint64_t>& frontiers() const { return frontiers_; }
  uint64_t num_blocks() const { return nblocks_; }
  uint64_t block() const { return bs_; }

 private:
  struct Node {
    uint32_t stage = 0, index = 0;
    PmKind kind = PmKind::PermuteScale;
    PmRange read, write;
    bool has_write = false, is_output = false;
    std::set<uint64_t> preds, succs;
  };
  struct Stage {
    uint32_t id = 0, net = 0, gate = 0;
    PmKind kind = PmKind::PermuteScale;
    std::vector<PmPart> parts;
    std::vector<uint64_t> nodes;
    uint64_t block_count = 0;
    std::vector<uint8_t> materialized;
  };
  struct GateRec {
    qt_gate g;
    uint32_t net;
    bool superposition;
  };

  // stage bookkeeping (engine.cpp:126-285)
  size_t exec_index(uint32_t net, size_t local) const;
  uint32_t make_stage(Stage&& st, uint32_t net, size_t local);
  void drop_stage(uint32_t sid, bool frontier_succs);
  void add_permute_stage(uint32_t net, uint32_t gate);
  void rebuild_mxv(uint32_t net);
  std::vector<PmPart> permute_parts(const qt_gate& g) const;

  // the graph (graph.cpp)
  std::vector<uint64_t> connect(uint32_t stage, PmKind kind, const std::vector<PmRange>& reads,
                                const std::vector<PmRange>& writes, const std::vector<bool>& has_write,
                                size_t at);
  struct Removal {
    std::vector<uint64_t> removed;
    std::vector<std::vector<uint64_t>> successors;
  };
  Removal disconnect(uint32_t stage);
  bool justified(uint64_t from, uint64_t to) const;
  std::set<uint64_t> affected(const std::set<uint64_t>& from) const;
  void link(uint64_t a, uint64_t b);
  void unlink(uint64_t a, uint64_t b);
  size_t position(uint32_t stage) const;
  void reposition();

  int n_;
  uint64_t cfg_bs_, bs_, nblocks_;
  // circuit mirror
  std::vector<uint32_t> order_;
  std::unordered_map<uint32_t, std::vector<uint32_t>> net_gates_;
  std::unordered_map<uint32_t, GateRec> gates_;
  // stages
  std::map<uint32_t, Stage> stages_;
  std::vector<uint32_t> exec_;  // stage ids in execution order (== graph order)
  std::unordered_map<uint32_t, std::vector<uint32_t>> net_stages_;
  std::unordered_map<uint32_t, uint32_t> gate_stage_;
  std::unordered_map<uint32_t, size_t> pos_;  // stage -> index in exec_
  uint32_t next_stage_ = 1;
  // graph
  std::map<uint64_t, Node> nodes_;
  uint64_t next_node_ = 1;
  std::set<uint64_t> frontiers_;
  bool ran_full_ = false;
  PmAccount last_;
};

}  // namespace qtb
