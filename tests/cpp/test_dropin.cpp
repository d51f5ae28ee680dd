// test_dropin.cpp -- C++ callers of the reference API compile unchanged
// against the drop-in (include/qtask/engine.hpp) and get the reference's
// behaviour from the B200 engine. Restates the reference's own engine tests
// (proj/tests/test_engine.cpp) and acceptance criteria 1, 2, 6, 7
// (proj/tests/acceptance.cpp) as plain checks; the dense oracle is
// oracle/liboracle.so (test infrastructure). Prints one [PASS]/[FAIL] per
// check; exit status = number of failures.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "qtask/engine.hpp"
#include "qtask/oracle.hpp"
#include "qtask/qasm.hpp"

using namespace qtask;

namespace {

int g_fail = 0;

void report(const char* name, bool ok, const std::string& detail = "") {
  std::printf("[%s] %s%s%s\n", ok ? "PASS" : "FAIL", name, detail.empty() ? "" : " -- ",
              detail.c_str());
  if (!ok) ++g_fail;
}

std::vector<Complex> dense_oracle(const Simulator& sim) {
  // the reference's oracle API over the test-only C restatement
  return oracle::simulate_dense(sim.circuit());
}

double max_dev(const Simulator& sim) {
  const std::vector<Complex> ref = dense_oracle(sim);
  const std::vector<Complex> got = sim.amplitudes(0, ref.size() - 1);
  double d = 0.0;
  for (std::size_t i = 0; i < ref.size(); ++i) d = std::max(d, std::abs(got[i] - ref[i]));
  return d;
}

struct Entangle5 {  // acceptance.cpp:43-63 (Listing-1 circuit)
  Simulator sim;
  NetId n1, n2, n3, n4, n5;
  GateId g6 = 0, g7 = 0, g8 = 0, g9 = 0;
  explicit Entangle5(Config cfg = Config{4, 1})
      : sim(5, cfg), n1(sim.insert_net_back()), n2(sim.insert_net_back()),
        n3(sim.insert_net_back()), n4(sim.insert_net_back()), n5(sim.insert_net_back()) {
    for (int q = 4; q >= 0; --q) sim.insert_gate(GateKind::H, n1, q);
    g6 = sim.insert_gate(GateKind::Cnot, n2, 3, 4);
    g7 = sim.insert_gate(GateKind::Cnot, n3, 1, 4);
    g8 = sim.insert_gate(GateKind::Cnot, n4, 2, 3);
    g9 = sim.insert_gate(GateKind::Cnot, n5, 0, 2);
  }
};

template <typename E, typename F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

struct GateDesc {
  GateKind kind;
  double theta;
  int target, control;
};

GateDesc random_gate(std::mt19937_64& rng, int n) {  // test_support.hpp:137-167
  static const GateKind kinds[] = {GateKind::Cnot, GateKind::X, GateKind::Y, GateKind::Z,
                                   GateKind::H, GateKind::S, GateKind::Sdg, GateKind::T,
                                   GateKind::Tdg, GateKind::Rx, GateKind::Ry, GateKind::Rz,
                                   GateKind::Swap};
  GateDesc g{kinds[rng() % (n >= 2 ? 13 : 12)], 0.0, 0, -1};
  if (n < 2 && is_two_qubit(g.kind)) g.kind = GateKind::H;
  g.target = static_cast<int>(rng() % n);
  if (is_two_qubit(g.kind)) {
    do {
      g.control = static_cast<int>(rng() % n);
    } while (g.control == g.target);
  }
  if (is_rotation(g.kind)) {
    switch (rng() % 4) {
      case 0: g.theta = M_PI; break;
      case 1: g.theta = M_PI / 2; break;
      case 2: g.theta = 0.0; break;
      default: g.theta = std::uniform_real_distribution<double>(-2 * M_PI, 2 * M_PI)(rng);
    }
  }
  return g;
}

GateId insert(Simulator& sim, NetId net, const GateDesc& g) {
  if (g.control >= 0) return sim.insert_gate(g.kind, net, g.target, g.control);
  if (is_rotation(g.kind)) return sim.insert_gate(g.kind, g.theta, net, g.target);
  return sim.insert_gate(g.kind, net, g.target);
}

}  // namespace

int main() {
  {
    Simulator sim(3);
    report("fresh simulator reads the initial state",
           sim.amplitude(0) == Complex{1, 0} && sim.amplitude(5) == Complex{0, 0} &&
               std::abs(sim.norm_squared() - 1.0) < 1e-12);
  }
  {
    Simulator sim(3);
    bool ok = throws<InvalidPositionError>([&] { sim.insert_net_after(99); }) &&
              throws<UnknownNetError>([&] { sim.remove_net(7); }) &&
              throws<UnknownGateError>([&] { sim.remove_gate(7); });
    const NetId net = sim.insert_net_back();
    ok = ok && throws<UnknownNetError>([&] { sim.insert_gate(GateKind::H, 42, 0); }) &&
         throws<BadQubitError>([&] { sim.insert_gate(GateKind::H, net, 3); }) &&
         throws<BadQubitError>([&] { sim.insert_gate(GateKind::Cnot, net, 1, 1); });
    sim.insert_gate(GateKind::Cnot, net, 1, 2);
    ok = ok && throws<NetConflictError>([&] { sim.insert_gate(GateKind::X, net, 2); }) &&
         throws<NetConflictError>([&] { sim.insert_gate(GateKind::Cnot, net, 0, 1); });
    report("modifier errors map to the reference exception types", ok);
  }
  {
    Simulator sim(2);
    const NetId net = sim.insert_net_back();
    bool ok = throws<StaleStateError>([&] { sim.amplitude(0); });
    sim.update_state();
    ok = ok && sim.amplitude(0) == Complex{1, 0};
    sim.insert_gate(GateKind::X, net, 0);
    ok = ok && throws<StaleStateError>([&] { sim.amplitudes(0, 3); });
    sim.update_state();
    ok = ok && sim.amplitude(1) == Complex{1, 0};
    report("amplitude queries require a clean state", ok);
  }
  {
    Entangle5 lc;
    lc.sim.update_state();
    bool ok = lc.sim.last_update().full;
    for (std::uint64_t i = 0; i < 32; ++i)
      ok = ok && std::abs(lc.sim.amplitude(i) - Complex{1 / std::sqrt(32.0), 0}) < 1e-12;
    report("Listing-1 circuit: uniform superposition", ok);
    lc.sim.remove_gate(lc.g8);
    lc.sim.insert_gate(GateKind::Cnot, lc.n4, 1, 2);
    lc.sim.update_state();
    const double d = max_dev(lc.sim);
    report("incremental update equals a fresh simulation of the edited circuit",
           !lc.sim.last_update().full && d <= 1e-10, "max dev " + std::to_string(d));
    lc.sim.update_state();
    report("update with no pending work executes nothing",
           lc.sim.last_update().executed_partitions == 0);
  }
  {
    // acceptance criterion 1: 200 random full circuits vs the oracle
    std::mt19937_64 rng(20240501);
    double worst = 0.0, worst_norm = 0.0;
    for (int trial = 0; trial < 200; ++trial) {
      const int n = 1 + static_cast<int>(rng() % 10);
      Simulator sim(n, Config{std::uint64_t{1} << (1 + rng() % 10), 1});
      std::vector<NetId> nets{sim.insert_net_back()};
      const int count = 1 + static_cast<int>(rng() % 60);
      for (int i = 0; i < count; ++i) {
        const GateDesc g = random_gate(rng, n);
        if (rng() % 3 == 0) nets.push_back(sim.insert_net_back());
        try {
          insert(sim, nets.back(), g);
        } catch (const NetConflictError&) {
          nets.push_back(sim.insert_net_back());
          insert(sim, nets.back(), g);
        }
      }
      sim.update_state();
      worst = std::max(worst, max_dev(sim));
      worst_norm = std::max(worst_norm, std::abs(sim.norm_squared() - 1.0));
    }
    report("criterion 1: 200 random circuits <= 1e-10", worst <= 1e-10,
           "max dev " + std::to_string(worst));
    report("criterion 6: normalisation", worst_norm <= 1e-9,
           "worst " + std::to_string(worst_norm));
  }
  {
    // acceptance criterion 2: random modifier sequences, incremental updates
    std::mt19937_64 rng(87123);
    double worst = 0.0;
    for (int trial = 0; trial < 100; ++trial) {
      const int n = 1 + static_cast<int>(rng() % 10);
      Config cfg{std::uint64_t{1} << (1 + rng() % 9), 1};
      cfg.max_checkpoints = 3;
      cfg.segment_gates = 1 + static_cast<int>(rng() % 6);
      Simulator sim(n, cfg);
      std::vector<NetId> nets;
      std::vector<GateId> gates;
      const int steps = 10 + static_cast<int>(rng() % 50);
      for (int s = 0; s < steps; ++s) {
        const int roll = static_cast<int>(rng() % 12);
        if (roll < 3 || nets.empty()) {
          if (nets.empty() || rng() % 2 == 0) nets.push_back(sim.insert_net_back());
          else nets.push_back(sim.insert_net_after(nets[rng() % nets.size()]));
        } else if (roll < 9) {
          try {
            gates.push_back(insert(sim, nets[rng() % nets.size()], random_gate(rng, n)));
          } catch (const NetConflictError&) {
          }
        } else if (roll < 10 && !gates.empty()) {
          const std::size_t at = rng() % gates.size();
          sim.remove_gate(gates[at]);
          gates.erase(gates.begin() + static_cast<std::ptrdiff_t>(at));
        } else {
          sim.update_state();
          worst = std::max(worst, max_dev(sim));
        }
      }
      sim.update_state();
      worst = std::max(worst, max_dev(sim));
    }
    report("criterion 2: 100 random modifier sequences <= 1e-10", worst <= 1e-10,
           "max dev " + std::to_string(worst));
  }
  {
    // acceptance criterion 7 restated for the GPU: bit-identical reruns
    std::mt19937_64 rng(3333);
    bool ok = true;
    for (int trial = 0; trial < 10; ++trial) {
      std::vector<GateDesc> desc;
      const int n = 1 + static_cast<int>(rng() % 8);
      for (int i = 0; i < 40; ++i) desc.push_back(random_gate(rng, n));
      std::vector<std::vector<Complex>> res;
      for (unsigned threads : {1u, 2u, 8u}) {
        Simulator sim(n, Config{8, threads});
        for (const GateDesc& g : desc) insert(sim, sim.insert_net_back(), g);
        sim.update_state();
        res.push_back(sim.amplitudes(0, (std::uint64_t{1} << n) - 1));
      }
      const std::size_t bytes = res[0].size() * sizeof(Complex);
      ok = ok && std::memcmp(res[0].data(), res[1].data(), bytes) == 0 &&
           std::memcmp(res[0].data(), res[2].data(), bytes) == 0;
    }
    report("criterion 7: amplitudes bit-identical across runs / thread settings", ok);
  }
  {
    // OpenQASM front end (qtask/qasm.hpp): the reference's test_qasm.cpp checks
    const std::string src =
        "// GHZ-like\nOPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg q[3];\ncreg c[3];\n"
        "h q[0];\ncx q[0],q[1];\nbarrier q;\ncx q[1],q[2];\nrz(-pi/2) q[2];\n";
    const qasm::QasmProgram p = qasm::parse(src);
    bool ok = p.num_qubits == 3 && p.statements.size() == 5 &&
              p.statements[1].qubits == std::vector<int>{0, 1} &&
              std::abs(p.statements[4].theta + M_PI / 2) < 1e-15;
    const auto lv = qasm::levelize(p);
    ok = ok && lv.size() == 4 && lv[0].size() == 1 && lv[3].size() == 1;
    const qasm::QasmProgram q = qasm::parse(qasm::to_qasm(p));
    ok = ok && q.statements.size() == p.statements.size() && q.statements[4].theta == p.statements[4].theta;
    report("qasm: parse / levelize / round trip", ok);
    int line = 0;
    try {
      qasm::parse("OPENQASM 2.0;\nqreg q[2];\nh q[5];\n");
    } catch (const qasm::ParseError& e) {
      line = e.line();
    }
    report("qasm: errors carry the line",
           line == 3 && throws<qasm::UnsupportedGateError>([&] {
             qasm::parse("OPENQASM 2.0;\nqreg q[3];\nccx q[0],q[1],q[2];\n");
           }) && throws<qasm::ParseError>([&] { qasm::parse("OPENQASM 3.0;\nqreg q[1];\n"); }));
    Simulator sim(3);
    qasm::build_circuit(sim, p);
    sim.update_state();
    // (|000> + |111>)/sqrt(2) with RZ(-pi/2) on q2: e^{+i pi/4} on |000>, e^{-i pi/4} on |111>
    const double r = 1 / std::sqrt(2.0);
    const Complex a0 = std::polar(r, M_PI / 4), a7 = std::polar(r, -M_PI / 4);
    const auto top = sim.top_k(3);
    const bool ghz = (top.size() == 3) &&
                     ((top[0].first == 0 && top[1].first == 7) ||
                      (top[0].first == 7 && top[1].first == 0)) &&
                     std::norm(top[0].second) >= std::norm(top[1].second) &&
                     std::abs(std::abs(top[0].second) - r) < 1e-12;
    report("top_k: the two GHZ amplitudes first (largest norm first)", ghz);
    report("qasm: build_circuit + update_state",
           sim.circuit().net_order().size() == 4 && std::abs(sim.amplitude(0) - a0) < 1e-12 &&
               std::abs(sim.amplitude(7) - a7) < 1e-12 && max_dev(sim) <= 1e-12);
  }
  std::printf("%s: %d failure(s)\n", g_fail ? "FAILURES" : "all passed", g_fail);
  return g_fail;
}
