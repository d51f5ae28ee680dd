// qtask/gate.hpp -- drop-in for the reference's gate kinds (reference
// proj/include/qtask/gate.hpp:13-37). Same enumerators in the same order
// (they are the qt_gate_kind values), plus the additive U3 and Cz.
#pragma once

#include <array>
#include <cmath>

#include "qtask/types.hpp"

namespace qtask {

enum class GateKind {
  Cnot = QT_CNOT,
  X = QT_X,
  Y = QT_Y,
  Z = QT_Z,
  H = QT_H,
  S = QT_S,
  Sdg = QT_SDG,
  T = QT_T,
  Tdg = QT_TDG,
  Rx = QT_RX,
  Ry = QT_RY,
  Rz = QT_RZ,
  Swap = QT_SWAP,
  U3 = QT_U3,  // additive: RZ(phi) RY(theta) RZ(lambda)
  Cz = QT_CZ,  // additive: H CX H
};

inline const char* kind_name(GateKind k) {
  switch (k) {
    case GateKind::Cnot: return "CNOT";
    case GateKind::X: return "X";
    case GateKind::Y: return "Y";
    case GateKind::Z: return "Z";
    case GateKind::H: return "H";
    case GateKind::S: return "S";
    case GateKind::Sdg: return "SDG";
    case GateKind::T: return "T";
    case GateKind::Tdg: return "TDG";
    case GateKind::Rx: return "RX";
    case GateKind::Ry: return "RY";
    case GateKind::Rz: return "RZ";
    case GateKind::Swap: return "SWAP";
    case GateKind::U3: return "U3";
    case GateKind::Cz: return "CZ";
  }
  return "?";
}

inline bool is_rotation(GateKind k) {
  return k == GateKind::Rx || k == GateKind::Ry || k == GateKind::Rz;
}

inline bool is_two_qubit(GateKind k) {
  return k == GateKind::Cnot || k == GateKind::Swap || k == GateKind::Cz;
}

/// Dense unitary of a gate (reference gate.hpp:38-48): dim 2, or 4 for the
/// two-qubit kinds with the sub-index (first << 1) | second. The entries
/// come from the engine's gate database, which restates gate.cpp:42-90
/// bit for bit.
struct GateMatrix {
  int dim = 2;
  std::array<Complex, 16> m{};

  Complex at(int r, int c) const { return m[r * dim + c]; }
  Complex& at(int r, int c) { return m[r * dim + c]; }
};

/// Structural-zero threshold of the classification (gate.hpp:50-53).
inline constexpr double kZeroThreshold = 1e-12;

enum class GateClass { NonSuperposition, Superposition };

/// gate_matrix(kind, theta) (gate.cpp:42-90); U3 takes phi / lambda too.
inline GateMatrix gate_matrix(GateKind kind, double theta = 0.0, double phi = 0.0,
                              double lambda = 0.0) {
  double raw[32];
  int dim = 2;
  detail::check(qt_gate_matrix(static_cast<int>(kind), theta, phi, lambda, raw, &dim));
  GateMatrix g;
  g.dim = dim;
  for (int i = 0; i < dim * dim; ++i) g.m[i] = Complex{raw[2 * i], raw[2 * i + 1]};
  return g;
}

/// NonSuperposition iff at most one entry per row exceeds kZeroThreshold
/// (gate.cpp:92-106).
inline GateClass classify_gate(GateKind kind, double theta = 0.0) {
  const GateMatrix g = gate_matrix(kind, theta);
  for (int r = 0; r < g.dim; ++r) {
    int nz = 0;
    for (int c = 0; c < g.dim; ++c) nz += std::abs(g.at(r, c)) > kZeroThreshold ? 1 : 0;
    if (nz > 1) return GateClass::Superposition;
  }
  return GateClass::NonSuperposition;
}

/// U U^dagger == I within tol (gate.cpp:108-122).
inline bool is_unitary(const GateMatrix& g, double tol = 1e-12) {
  for (int r = 0; r < g.dim; ++r)
    for (int c = 0; c < g.dim; ++c) {
      Complex acc = 0;
      for (int k = 0; k < g.dim; ++k) acc += g.at(r, k) * std::conj(g.at(c, k));
      if (std::abs(acc - (r == c ? Complex{1, 0} : Complex{0, 0})) > tol) return false;
    }
  return true;
}

}  // namespace qtask
