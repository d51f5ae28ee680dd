// qt_gates.hpp -- host gate database (restates gate.cpp:42-106) + lowering.
#pragma once

#include <array>
#include <string>
#include <vector>

#include "qt_ir.hpp"
#include "qtask_c.h"

namespace qtb {

using Mat2 = std::array<cplx, 4>;

// structural-zero threshold of the gate classification (gate.hpp:50-53)
constexpr double kZeroThreshold = 1e-12;

bool valid_kind(int kind);
bool is_two_qubit_kind(int kind);
bool is_rotation_kind(int kind);
Mat2 gate_matrix_1q(int kind, double theta);
Mat2 u3_matrix(double theta, double phi, double lambda);
Mat2 matmul(const Mat2& a, const Mat2& b);
bool is_superposition(int kind, double theta);
bool is_superposition_gate(const qt_gate& g);

// Validates (circuit.cpp:51-76 semantics) and appends the logical op(s) of
// one gate. Returns QT_OK or a QT_ERR_* code with *err set.
int lower_gate(const qt_gate& g, int n, uint32_t index, std::vector<LOp>& out,
               std::string* err);

}  // namespace qtb
