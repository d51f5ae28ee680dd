// qtask/oracle.hpp -- TEST INFRASTRUCTURE. The reference's dense oracle API
// (reference proj/include/qtask/oracle.hpp:9-21) for C++ test programs that
// check the drop-in (tests/cpp): it forwards to oracle/liboracle.so, the C
// restatement of oracle.cpp:15-60 that tests/test_oracle.py memcmp-pins to
// the reference compiled from its sources. Not part of the product headers
// (include/): the B200 engine never includes or links it.
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "qtask/circuit.hpp"
#include "qtask/types.hpp"

extern "C" int qo_apply(int n, double* state, const void* gates, size_t count, int threads);

namespace qtask::oracle {

using DenseState = std::vector<Complex>;

inline DenseState initial_state(int num_qubits) {
  DenseState s(std::size_t{1} << num_qubits, Complex{0.0, 0.0});
  s[0] = Complex{1.0, 0.0};
  return s;
}

namespace detail {
inline qt_gate to_pod(const Gate& g) {
  qt_gate p{};
  p.kind = static_cast<int32_t>(g.kind);
  p.target = g.target;
  p.control = g.control;
  p.theta = g.theta;
  p.phi = g.phi;
  p.lambda = g.lambda;
  return p;
}
}  // namespace detail

/// Applies one gate in place (single-threaded, as the reference's).
inline void apply_gate_dense(DenseState& state, const Gate& gate, int num_qubits) {
  const qt_gate p = detail::to_pod(gate);
  if (qo_apply(num_qubits, reinterpret_cast<double*>(state.data()), &p, 1, 1) != 0)
    throw Error("oracle: unsupported gate");
}

/// Applies the nets in order (oracle.cpp:52-60).
inline DenseState simulate_dense(const Circuit& circuit) {
  std::vector<qt_gate> gs;
  for (NetId n : circuit.net_order())
    for (GateId g : circuit.net(n).gates) gs.push_back(detail::to_pod(circuit.gate(g)));
  DenseState s = initial_state(circuit.num_qubits());
  if (qo_apply(circuit.num_qubits(), reinterpret_cast<double*>(s.data()), gs.data(), gs.size(), 1) != 0)
    throw Error("oracle: unsupported gate");
  return s;
}

}  // namespace qtask::oracle
