// qtask/circuit.hpp -- drop-in for the reference circuit model (reference
// proj/include/qtask/circuit.hpp:14-73, circuit.cpp:8-135): gates, nets and
// an ordered net list with the same validation and exception types.
// Header-only host code; the drop-in Simulator keeps one as the mirror that
// circuit() returns. Differences: up to 40 qubits (the device engine's
// limit, circuit.cpp:9-11 caps at 30), the additive U3 parameters, and
// net positions answered from an index rebuilt after edits instead of a
// linear search per call.
#pragma once

#include <algorithm>
#include <cmath>
#include <optional>
#include <unordered_map>
#include <vector>

#include "qtask/gate.hpp"
#include "qtask/types.hpp"

namespace qtask {

/// One gate. `control` is -1 unless two-qubit: the control of a Cnot / Cz,
/// the second qubit of a Swap. phi / lambda: U3 only (additive).
struct Gate {
  GateId id = kNoGate;
  GateKind kind = GateKind::X;
  double theta = 0.0;
  NetId net = kNoNet;
  int target = 0;
  int control = -1;
  double phi = 0.0;
  double lambda = 0.0;
};

/// Structurally parallel gates (no shared qubit), in insertion order.
struct Net {
  NetId id = kNoNet;
  std::vector<GateId> gates;
};

class Simulator;
class Circuit;
bool check_net_conflict(const Circuit& circuit, NetId net, int target,
                        std::optional<int> control = std::nullopt);

class Circuit {
 public:
  explicit Circuit(int num_qubits) : num_qubits_(num_qubits) {
    if (num_qubits < 1 || num_qubits > 40) throw BadQubitError("qubit count must be in [1, 40]");
  }

  int num_qubits() const { return num_qubits_; }

  NetId insert_net_front() { return add_net(0); }
  NetId insert_net_back() { return add_net(order_.size()); }
  NetId insert_net_after(NetId after) {
    if (!nets_.count(after)) throw InvalidPositionError("insert_net: unknown anchor net");
    return add_net(net_position(after) + 1);
  }
  /// Removes a net and its gates. Throws UnknownNetError.
  void remove_net(NetId net) {
    auto it = nets_.find(net);
    if (it == nets_.end()) throw UnknownNetError("remove_net: unknown net");
    for (GateId g : it->second.gates) gates_.erase(g);
    const std::size_t at = net_position(net);
    nets_.erase(it);
    order_.erase(order_.begin() + static_cast<std::ptrdiff_t>(at));
    dirty_ = true;
  }

  GateId insert_gate(GateKind kind, double theta, NetId net, int target, int control = -1) {
    return add_gate(next_gate_, kind, theta, 0.0, 0.0, net, target, control);
  }
  void remove_gate(GateId gate) {
    auto it = gates_.find(gate);
    if (it == gates_.end()) throw UnknownGateError("remove_gate: unknown gate");
    std::vector<GateId>& gs = nets_.at(it->second.net).gates;
    gs.erase(std::find(gs.begin(), gs.end(), gate));
    gates_.erase(it);
  }

  bool has_net(NetId net) const { return nets_.count(net) != 0; }
  bool has_gate(GateId gate) const { return gates_.count(gate) != 0; }
  const Net& net(NetId id) const {
    auto it = nets_.find(id);
    if (it == nets_.end()) throw UnknownNetError("unknown net");
    return it->second;
  }
  const Gate& gate(GateId id) const {
    auto it = gates_.find(id);
    if (it == gates_.end()) throw UnknownGateError("unknown gate");
    return it->second;
  }
  const std::vector<NetId>& net_order() const { return order_; }
  /// Position of a net in simulation order. Throws UnknownNetError.
  std::size_t net_position(NetId id) const {
    if (dirty_) {
      pos_.clear();
      for (std::size_t i = 0; i < order_.size(); ++i) pos_[order_[i]] = i;
      dirty_ = false;
    }
    auto it = pos_.find(id);
    if (it == pos_.end()) throw UnknownNetError("unknown net");
    return it->second;
  }
  std::size_t num_gates() const { return gates_.size(); }

 private:
  friend class Simulator;

  NetId add_net(std::size_t at, NetId given = kNoNet) {
    const NetId id = given != kNoNet ? given : next_net_;
    next_net_ = std::max(next_net_, id + 1);
    nets_.emplace(id, Net{id, {}});
    order_.insert(order_.begin() + static_cast<std::ptrdiff_t>(at), id);
    dirty_ = true;
    return id;
  }
  // circuit.cpp:51-86 validation; `id` lets the Simulator mirror the
  // engine's handles
  GateId add_gate(GateId id, GateKind kind, double theta, double phi, double lambda, NetId net,
                  int target, int control) {
    auto it = nets_.find(net);
    if (it == nets_.end()) throw UnknownNetError("insert_gate: unknown net");
    if (target < 0 || target >= num_qubits_) throw BadQubitError("target qubit out of range");
    if (is_two_qubit(kind)) {
      if (control < 0 || control >= num_qubits_) throw BadQubitError("second qubit out of range");
      if (control == target) throw BadQubitError("two-qubit gate needs distinct qubits");
    } else if (control != -1) {
      throw BadQubitError("single-qubit gate takes no control");
    }
    if (!std::isfinite(theta) || !std::isfinite(phi) || !std::isfinite(lambda))
      throw Error("rotation angle must be finite");
    if (check_net_conflict(*this, net, target, control >= 0 ? std::optional<int>(control) : std::nullopt))
      throw NetConflictError("gate would depend on another gate in the net");
    gates_.emplace(id, Gate{id, kind, theta, net, target, control, phi, lambda});
    it->second.gates.push_back(id);
    next_gate_ = std::max(next_gate_, id + 1);
    return id;
  }

  int num_qubits_;
  std::vector<NetId> order_;
  std::unordered_map<NetId, Net> nets_;
  std::unordered_map<GateId, Gate> gates_;
  mutable std::unordered_map<NetId, std::size_t> pos_;
  mutable bool dirty_ = true;
  NetId next_net_ = 1;
  GateId next_gate_ = 1;
};

/// True iff a gate on (target[, control]) would share a qubit with a gate
/// already in the net (circuit.cpp:122-135).
inline bool check_net_conflict(const Circuit& circuit, NetId net, int target,
                               std::optional<int> control) {
  for (GateId g : circuit.net(net).gates) {
    const Gate& o = circuit.gate(g);
    if (o.target == target || (control && o.target == *control) || o.control == target ||
        (control && o.control >= 0 && o.control == *control))
      return true;
  }
  return false;
}

}  // namespace qtask
