// qt_gates.cpp -- host gate database and lowering of qt_gate to logical ops.
//
// Matrices restate the reference gate database (gate.cpp:42-90) with the
// same libm calls and the same std::complex evaluation order, so the inputs
// the GPU consumes are bit-identical to the oracle's. classify (gate.cpp:92-
// 106, kZeroThreshold gate.hpp:53) decides only the reference's bookkeeping
// semantics (SuperpositionGateError, UpdateStats); the kernels pick their op
// form from the matrix structure.
#include <cmath>
#include <cstring>

#include "qt_gates.hpp"
#include "qtask_c.h"

namespace qtb {

namespace {
constexpr double kInvSqrt2 = 0.70710678118654752440084436210484903928;


inline cplx mk(double re, double im) { return cplx{re, im}; }
}  // namespace

bool is_two_qubit_kind(int kind) {
  return kind == QT_CNOT || kind == QT_SWAP || kind == QT_CZ;
}
bool is_rotation_kind(int kind) {
  return kind == QT_RX || kind == QT_RY || kind == QT_RZ || kind == QT_U3;
}
bool valid_kind(int kind) { return kind >= QT_CNOT && kind <= QT_CZ; }

Mat2 gate_matrix_1q(int kind, double theta) {
  const double half = theta / 2.0;
  const cplx zero = mk(0.0, 0.0), one = mk(1.0, 0.0);
  const cplx i = mk(0.0, 1.0), mi = mk(-0.0, -1.0);
  Mat2 g;
  switch (kind) {
    case QT_X: g = {zero, one, one, zero}; break;
    case QT_Y: g = {zero, mi, i, zero}; break;
    case QT_Z: g = {one, zero, zero, mk(-1.0, 0.0)}; break;
    case QT_H:
      g = {mk(kInvSqrt2, 0.0), mk(kInvSqrt2, 0.0), mk(kInvSqrt2, 0.0),
           mk(-kInvSqrt2, 0.0)};
      break;
    case QT_S: g = {one, zero, zero, i}; break;
    case QT_SDG: g = {one, zero, zero, mi}; break;
    case QT_T:
      g = {one, zero, zero,
           mk(1.0 * std::cos(M_PI / 4.0), 1.0 * std::sin(M_PI / 4.0))};
      break;
    case QT_TDG:
      g = {one, zero, zero,
           mk(1.0 * std::cos(-M_PI / 4.0), 1.0 * std::sin(-M_PI / 4.0))};
      break;
    case QT_RX: {
      const double c = std::cos(half), s = std::sin(half);
      const cplx off = mk(-0.0 * s, -1.0 * s);  // (-i) * sin(half)
      g = {mk(c, 0.0), off, off, mk(c, 0.0)};
      break;
    }
    case QT_RY: {
      const double c = std::cos(half), s = std::sin(half);
      g = {mk(c, 0.0), mk(-s, 0.0), mk(s, 0.0), mk(c, 0.0)};
      break;
    }
    case QT_RZ:
      g = {mk(1.0 * std::cos(-half), 1.0 * std::sin(-half)), zero, zero,
           mk(1.0 * std::cos(half), 1.0 * std::sin(half))};
      break;
    default:
      g = {one, zero, zero, one};
      break;
  }
  return g;
}

Mat2 matmul(const Mat2& a, const Mat2& b) {
  Mat2 r;
  r[0] = cadd(cmul(a[0], b[0]), cmul(a[1], b[2]));
  r[1] = cadd(cmul(a[0], b[1]), cmul(a[1], b[3]));
  r[2] = cadd(cmul(a[2], b[0]), cmul(a[3], b[2]));
  r[3] = cadd(cmul(a[2], b[1]), cmul(a[3], b[3]));
  return r;
}

Mat2 u3_matrix(double theta, double phi, double lambda) {
  // time order RZ(lambda), RY(theta), RZ(phi) -> M = RZ(phi) RY(theta) RZ(lambda)
  return matmul(gate_matrix_1q(QT_RZ, phi),
                matmul(gate_matrix_1q(QT_RY, theta),
                       gate_matrix_1q(QT_RZ, lambda)));
}

static double cabs(cplx c) { return std::hypot(c.re, c.im); }

bool is_superposition(int kind, double theta) {
  // gate.cpp:92-106: NonSuperposition iff at most one |entry| > 1e-12 per row.
  if (kind == QT_CNOT || kind == QT_SWAP || kind == QT_CZ) return false;
  Mat2 g = kind == QT_U3 ? u3_matrix(theta, 0.0, 0.0)
                         : gate_matrix_1q(kind, theta);
  for (int r = 0; r < 2; ++r) {
    int nz = 0;
    for (int c = 0; c < 2; ++c) nz += cabs(g[r * 2 + c]) > kZeroThreshold;
    if (nz > 1) return true;
  }
  return false;
}

bool is_superposition_gate(const qt_gate& g) {
  if (g.kind == QT_U3) {
    const Mat2 m = u3_matrix(g.theta, g.phi, g.lambda);
    for (int r = 0; r < 2; ++r) {
      int nz = 0;
      for (int c = 0; c < 2; ++c) nz += cabs(m[r * 2 + c]) > kZeroThreshold;
      if (nz > 1) return true;
    }
    return false;
  }
  return is_superposition(g.kind, g.theta);
}

static LOp from_mat(const Mat2& m, int target, int control, uint32_t gate) {
  LOp op;
  op.target = target;
  op.control = control;
  op.gate = gate;
  for (int k = 0; k < 4; ++k) op.m[k] = m[k];
  const bool off0 = m[1].re == 0.0 && m[1].im == 0.0 && m[2].re == 0.0 &&
                    m[2].im == 0.0;
  const bool diag0 = m[0].re == 0.0 && m[0].im == 0.0 && m[3].re == 0.0 &&
                     m[3].im == 0.0;
  op.kind = off0 ? LKind::Diag : (diag0 ? LKind::Anti : LKind::Dense);
  return op;
}

int lower_gate(const qt_gate& g, int n, uint32_t index, std::vector<LOp>& out,
               std::string* err) {
  if (!valid_kind(g.kind)) {
    if (err) *err = "unknown gate kind";
    return QT_ERR_ARG;
  }
  if (g.target < 0 || g.target >= n) {
    if (err) *err = "target qubit out of range";
    return QT_ERR_BAD_QUBIT;
  }
  if (is_two_qubit_kind(g.kind)) {
    if (g.control < 0 || g.control >= n) {
      if (err) *err = "second qubit out of range";
      return QT_ERR_BAD_QUBIT;
    }
    if (g.control == g.target) {
      if (err) *err = "two-qubit gate needs distinct qubits";
      return QT_ERR_BAD_QUBIT;
    }
  } else if (g.control != -1) {
    if (err) *err = "single-qubit gate takes no control";
    return QT_ERR_BAD_QUBIT;
  }
  if (!std::isfinite(g.theta) || !std::isfinite(g.phi) ||
      !std::isfinite(g.lambda)) {
    if (err) *err = "rotation angle must be finite";
    return QT_ERR_ARG;
  }
  const cplx zero{0.0, 0.0}, one{1.0, 0.0};
  switch (g.kind) {
    case QT_CNOT: {  // gate.cpp:70-77: controlled bit flip, scale 1
      out.push_back(from_mat({zero, one, one, zero}, g.target, g.control,
                             index));
      return QT_OK;
    }
    case QT_CZ: {
      out.push_back(from_mat({one, zero, zero, cplx{-1.0, 0.0}}, g.target,
                             g.control, index));
      return QT_OK;
    }
    case QT_SWAP: {
      LOp op;
      op.kind = LKind::Swap;
      op.target = g.target;
      op.target2 = g.control;
      op.gate = index;
      out.push_back(op);
      return QT_OK;
    }
    case QT_U3:
      out.push_back(from_mat(u3_matrix(g.theta, g.phi, g.lambda), g.target, -1,
                             index));
      return QT_OK;
    default:
      out.push_back(from_mat(gate_matrix_1q(g.kind, g.theta), g.target, -1,
                             index));
      return QT_OK;
  }
}

}  // namespace qtb
