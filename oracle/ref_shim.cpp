// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" shim over the UNMODIFIED qTask reference library, compiled from
// its own sources under /root/reference/proj/src by oracle/Makefile into
// oracle/_ref/libqtask_ref.so (git-ignored; travels to the GPU box with the
// snapshot).  It exposes:
//   * ref_oracle_run      -> qtask::oracle::apply_gate_dense (oracle.cpp:15-50)
//                            over a gate list, timed around the gate loop only
//   * ref_sim_*           -> qtask::Simulator (engine.hpp:46-100): the
//                            reference's incremental engine, driven through
//                            its public modifier / update / readout API
//   * ref_qasm_parse      -> qtask::qasm::parse + levelize (qasm.cpp:34-405)
//   * ref_qasm_build      -> qtask::qasm::build_circuit (qasm.cpp:407-426)
//                            into a ref_sim handle
// so tests can pin oracle/qt_oracle.c against the reference and bench.py's
// reference arm can time the reference's own CPU implementation.
//
// Gates use the qt_gate layout of include/qtask_c.h. Additive kinds U3 (13)
// and CZ (14) are lowered to reference gates.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <sstream>
#include <exception>
#include <vector>

#include "qtask/engine.hpp"
#include "qtask/oracle.hpp"
#include "qtask/qasm.hpp"

namespace {

struct RefGate {
  int32_t kind;
  int32_t target;
  int32_t control;
  int32_t reserved;
  double theta, phi, lambda;
};

struct Prim {
  qtask::GateKind kind;
  double theta;
  int target;
  int control;
};

int lower(const RefGate& g, std::vector<Prim>& out) {
  using K = qtask::GateKind;
  if (g.kind >= 0 && g.kind <= 12) {
    out.push_back(Prim{static_cast<K>(g.kind), g.theta, g.target,
                       qtask::is_two_qubit(static_cast<K>(g.kind)) ? g.control
                                                                   : -1});
    return 0;
  }
  if (g.kind == 13) {  // U3 -> RZ(lambda) RY(theta) RZ(phi)
    out.push_back(Prim{K::Rz, g.lambda, g.target, -1});
    out.push_back(Prim{K::Ry, g.theta, g.target, -1});
    out.push_back(Prim{K::Rz, g.phi, g.target, -1});
    return 0;
  }
  if (g.kind == 14) {  // CZ -> H CX H
    out.push_back(Prim{K::H, 0.0, g.target, -1});
    out.push_back(Prim{K::Cnot, 0.0, g.target, g.control});
    out.push_back(Prim{K::H, 0.0, g.target, -1});
    return 0;
  }
  return -1;
}

int error_code(const std::exception& e) {
  if (dynamic_cast<const qtask::NetConflictError*>(&e)) return -2;
  if (dynamic_cast<const qtask::UnknownNetError*>(&e)) return -3;
  if (dynamic_cast<const qtask::UnknownGateError*>(&e)) return -4;
  if (dynamic_cast<const qtask::BadQubitError*>(&e)) return -5;
  if (dynamic_cast<const qtask::InvalidPositionError*>(&e)) return -6;
  if (dynamic_cast<const qtask::StaleStateError*>(&e)) return -7;
  if (dynamic_cast<const qtask::NumericError*>(&e)) return -8;
  if (dynamic_cast<const qtask::SuperpositionGateError*>(&e)) return -9;
  return -1;
}

}  // namespace

extern "C" {

// Applies gates[0..count) with the reference dense oracle to |basis>, writes
// the final 2^n state (interleaved) to out (if non-null) and the wall time of
// the gate loop to *seconds. Returns 0 or a negative error.
int ref_oracle_run(int n, uint64_t basis, const RefGate* gates, size_t count,
                   double* out, double* seconds) {
  try {
    std::vector<Prim> prims;
    for (size_t i = 0; i < count; ++i) {
      if (lower(gates[i], prims) != 0) return -1;
    }
    qtask::oracle::DenseState st(std::uint64_t{1} << n,
                                 qtask::Complex{0.0, 0.0});
    st[basis] = qtask::Complex{1.0, 0.0};
    std::vector<qtask::Gate> gs;
    gs.reserve(prims.size());
    for (const Prim& p : prims) {
      qtask::Gate g;
      g.kind = p.kind;
      g.theta = p.theta;
      g.target = p.target;
      g.control = p.control;
      gs.push_back(g);
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (const qtask::Gate& g : gs) {
      qtask::oracle::apply_gate_dense(st, g, n);
    }
    const auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    if (out) std::memcpy(out, st.data(), st.size() * sizeof(qtask::Complex));
    return 0;
  } catch (const std::exception& e) {
    return error_code(e);
  }
}

// Reference gate matrix (gate.cpp:42-90) of a 1q kind, interleaved row major.
int ref_gate_matrix(int kind, double theta, double* m) {
  try {
    const qtask::GateMatrix g =
        qtask::gate_matrix(static_cast<qtask::GateKind>(kind), theta);
    for (int k = 0; k < g.dim * g.dim; ++k) {
      m[2 * k] = g.m[k].real();
      m[2 * k + 1] = g.m[k].imag();
    }
    return g.dim;
  } catch (const std::exception& e) {
    return error_code(e);
  }
}

int ref_classify(int kind, double theta) {
  return qtask::classify_gate(static_cast<qtask::GateKind>(kind), theta) ==
                 qtask::GateClass::Superposition
             ? 1
             : 0;
}

// ---- the reference incremental engine ------------------------------------

void* ref_sim_create(int n, uint64_t block_size, unsigned threads) {
  try {
    return new qtask::Simulator(n, qtask::Config{block_size, threads});
  } catch (...) {
    return nullptr;
  }
}

void ref_sim_destroy(void* s) { delete static_cast<qtask::Simulator*>(s); }

// where: 0 = front, 1 = back, 2 = after `after`. Returns the net id (> 0) or
// a negative error.
int64_t ref_sim_insert_net(void* s, int where, uint32_t after) {
  auto* sim = static_cast<qtask::Simulator*>(s);
  try {
    if (where == 0) return sim->insert_net_front();
    if (where == 1) return sim->insert_net_back();
    return sim->insert_net_after(after);
  } catch (const std::exception& e) {
    return error_code(e);
  }
}

int ref_sim_remove_net(void* s, uint32_t net) {
  try {
    static_cast<qtask::Simulator*>(s)->remove_net(net);
    return 0;
  } catch (const std::exception& e) {
    return error_code(e);
  }
}

// Reference kinds only (0..12). Returns the gate id (> 0) or an error.
int64_t ref_sim_insert_gate(void* s, int kind, double theta, uint32_t net,
                            int target, int control) {
  auto* sim = static_cast<qtask::Simulator*>(s);
  try {
    const auto k = static_cast<qtask::GateKind>(kind);
    if (qtask::is_two_qubit(k)) return sim->insert_gate(k, net, target, control);
    return sim->insert_gate(k, theta, net, target);
  } catch (const std::exception& e) {
    return error_code(e);
  }
}

int ref_sim_remove_gate(void* s, uint32_t gate) {
  try {
    static_cast<qtask::Simulator*>(s)->remove_gate(gate);
    return 0;
  } catch (const std::exception& e) {
    return error_code(e);
  }
}

int ref_sim_update(void* s) {
  try {
    static_cast<qtask::Simulator*>(s)->update_state();
    return 0;
  } catch (const std::exception& e) {
    return error_code(e);
  }
}

int ref_sim_amplitudes(void* s, uint64_t first, uint64_t last, double* out) {
  try {
    const auto v = static_cast<qtask::Simulator*>(s)->amplitudes(first, last);
    std::memcpy(out, v.data(), v.size() * sizeof(qtask::Complex));
    return 0;
  } catch (const std::exception& e) {
    return error_code(e);
  }
}

double ref_sim_norm(void* s) {
  return static_cast<qtask::Simulator*>(s)->norm_squared();
}

// stats: [full, executed_partitions, materialized_blocks, rewritten_amps]
void ref_sim_stats(void* s, uint64_t* out4) {
  const auto& st = static_cast<qtask::Simulator*>(s)->last_update();
  out4[0] = st.full ? 1 : 0;
  out4[1] = st.executed_partitions;
  out4[2] = st.materialized_blocks;
  out4[3] = st.rewritten_amplitudes;
}

// The reference's partition graph as DOT text (engine.cpp dump_graph) and
// the last update's rewritten blocks: the checker for the drop-in's host
// partition model (tests/test_partition_model.py). Returns the text length
// (+1); copies at most cap bytes.
size_t ref_sim_dump(void* s, char* buf, size_t cap) {
  std::ostringstream os;
  static_cast<qtask::Simulator*>(s)->dump_graph(os);
  const std::string t = os.str();
  if (buf && cap) {
    const size_t n = t.size() < cap - 1 ? t.size() : cap - 1;
    std::memcpy(buf, t.data(), n);
    buf[n] = 0;
  }
  return t.size() + 1;
}

size_t ref_sim_rewritten_blocks(void* s, uint64_t* out, size_t cap) {
  const auto& b = static_cast<qtask::Simulator*>(s)->last_update().rewritten_blocks;
  for (size_t i = 0; i < b.size() && i < cap; ++i) out[i] = b[i];
  return b.size();
}

// ---- the reference OpenQASM front end -------------------------------------

// Flattened statements, 8 doubles each: [kind (0 gate, 1 barrier), gate,
// theta, has_theta, q0, q1 (-1 if absent), line, column] plus, in `levels`,
// each statement's ASAP level (-1 for barriers). Returns the statement count,
// or -1 (ParseError) / -2 (UnsupportedGateError) with *line / *col set, or
// -3 for any other failure. *nq = qreg size.
int64_t ref_qasm_parse(const char* text, size_t len, double* out, int32_t* levels,
                       size_t cap, uint32_t* nq, int* line, int* col) {
  try {
    const auto p = qtask::qasm::parse(std::string_view(text, len));
    const auto lv = qtask::qasm::levelize(p);
    std::vector<int32_t> level(p.statements.size(), -1);
    for (size_t l = 0; l < lv.size(); ++l)
      for (size_t i : lv[l]) level[i] = static_cast<int32_t>(l);
    *nq = static_cast<uint32_t>(p.num_qubits);
    for (size_t i = 0; i < p.statements.size() && i < cap; ++i) {
      const auto& st = p.statements[i];
      double* r = out + 8 * i;
      r[0] = st.kind == qtask::qasm::Statement::Kind::Barrier ? 1 : 0;
      r[1] = static_cast<double>(static_cast<int>(st.gate));
      r[2] = st.theta;
      r[3] = st.has_theta ? 1 : 0;
      r[4] = st.qubits.size() > 0 ? st.qubits[0] : -1;
      r[5] = st.qubits.size() > 1 ? st.qubits[1] : -1;
      r[6] = st.line;
      r[7] = st.column;
      levels[i] = level[i];
    }
    return static_cast<int64_t>(p.statements.size());
  } catch (const qtask::qasm::ParseError& e) {
    *line = e.line();
    *col = e.column();
    return -1;
  } catch (const qtask::qasm::UnsupportedGateError& e) {
    *line = e.line();
    *col = e.column();
    return -2;
  } catch (...) {
    return -3;
  }
}

int ref_qasm_build(void* s, const char* text, size_t len) {
  try {
    qtask::qasm::build_circuit(*static_cast<qtask::Simulator*>(s),
                               qtask::qasm::parse(std::string_view(text, len)));
    return 0;
  } catch (const std::exception& e) {
    return error_code(e);
  }
}

}  // extern "C"
