// qtask/gate.hpp -- drop-in for the reference's gate kinds (reference
// proj/include/qtask/gate.hpp:13-37). Same enumerators in the same order
// (they are the qt_gate_kind values), plus the additive U3 and Cz.
#pragma once

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

}  // namespace qtask
