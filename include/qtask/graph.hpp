// qtask/graph.hpp -- drop-in for the reference's partition-graph view
// (reference proj/include/qtask/graph.hpp:17-125). Simulator::graph()
// returns a snapshot of the engine's host partition model
// (csrc/qt_partition.hpp, which restates graph.cpp's edge discovery,
// pruning and reconnection): nodes with their stage, partition index,
// read / write block ranges and edges, plus the reference's read-only
// queries (edges, topological order, acyclicity, affected closure).
#pragma once

#include <algorithm>
#include <cstdint>
#include <map>
#include <set>
#include <utility>
#include <vector>

#include "qtask/plan.hpp"
#include "qtask/types.hpp"

namespace qtask {

/// Inclusive range of block indices (graph.hpp:17-26).
struct BlockRange {
  std::uint64_t first = 0;
  std::uint64_t last = 0;
  friend bool operator==(const BlockRange& a, const BlockRange& b) {
    return a.first == b.first && a.last == b.last;
  }
};

inline bool intersects(const BlockRange& a, const BlockRange& b) {
  return std::max(a.first, b.first) <= std::min(a.last, b.last);
}

using NodeId = std::uint64_t;
inline constexpr NodeId kOutputNode = 0;

class Simulator;

class PartitionGraph {
 public:
  struct Node {
    NodeId id = 0;
    StageId stage = 0;
    std::uint32_t index = 0;
    StageKind kind = StageKind::PermuteScale;
    BlockRange read;
    BlockRange write;
    bool has_write = false;
    bool is_output = false;
    std::set<NodeId> preds;
    std::set<NodeId> succs;
  };

  bool contains(NodeId id) const { return nodes_.count(id) != 0; }
  const Node& node(NodeId id) const {
    auto it = nodes_.find(id);
    if (it == nodes_.end()) throw Error("unknown partition-graph node");
    return it->second;
  }
  std::size_t num_nodes() const { return nodes_.size(); }
  std::size_t num_stages() const { return stages_.size(); }
  const std::vector<NodeId>& stage_nodes(StageId stage) const {
    for (const auto& s : stages_)
      if (s.first == stage) return s.second;
    throw Error("stage not present in partition graph");
  }
  std::size_t stage_position(StageId stage) const {
    for (std::size_t i = 0; i < stages_.size(); ++i)
      if (stages_[i].first == stage) return i;
    throw Error("stage not present in partition graph");
  }

  /// Frontier partitions plus every node reachable from them.
  std::set<NodeId> affected_from(const std::set<NodeId>& frontiers) const {
    std::set<NodeId> seen;
    std::vector<NodeId> stack(frontiers.begin(), frontiers.end());
    while (!stack.empty()) {
      const NodeId id = stack.back();
      stack.pop_back();
      if (!seen.insert(id).second) continue;
      for (NodeId s : node(id).succs)
        if (!seen.count(s)) stack.push_back(s);
    }
    return seen;
  }

  /// All nodes including output, in a valid topological order (Kahn).
  std::vector<NodeId> topo_order() const {
    std::map<NodeId, std::size_t> indeg;
    std::vector<NodeId> ready, out;
    for (const auto& kv : nodes_) {
      indeg[kv.first] = kv.second.preds.size();
      if (kv.second.preds.empty()) ready.push_back(kv.first);
    }
    while (!ready.empty()) {
      const NodeId id = ready.back();
      ready.pop_back();
      out.push_back(id);
      for (NodeId s : nodes_.at(id).succs)
        if (--indeg[s] == 0) ready.push_back(s);
    }
    return out;
  }
  bool is_acyclic() const { return topo_order().size() == nodes_.size(); }

  /// Directed edges as (source, destination) pairs, sorted.
  std::vector<std::pair<NodeId, NodeId>> edges() const { return edges_; }

 private:
  friend class Simulator;
  std::map<NodeId, Node> nodes_;
  std::vector<std::pair<StageId, std::vector<NodeId>>> stages_;  // execution order
  std::vector<std::pair<NodeId, NodeId>> edges_;
};

}  // namespace qtask
