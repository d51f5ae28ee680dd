// qtask/qasm.hpp -- drop-in for the reference's OpenQASM 2.0 front end
// (reference proj/include/qtask/qasm.hpp:11-66, proj/src/qasm.cpp:34-426):
// the on-disk input format feeding the gate path. Header-only, host code.
//
// Accepted subset (same as the reference): `OPENQASM 2.0;`, `include
// "qelib1.inc";`, ONE `qreg`, any `creg` (ignored), `barrier ...;` (a global
// level separator, operands ignored), and the gates h x y z s sdg t tdg
// rx(θ) ry(θ) rz(θ) cx swap on indexed qubits. θ := ['-'] term {('*'|'/') term},
// term := number | pi. `//` comments. Any other statement name (measure, ccx,
// u1, id, ...) -> UnsupportedGateError; malformed input -> ParseError, both
// carrying the 1-based line / column of the offending token.
//
// levelize() is the reference's ASAP levelling (qasm.cpp:376-405) and
// build_circuit() appends one net per level (qasm.cpp:407-426); OpenQASM
// `cx a,b` is control a, target b; `swap a,b` is target a, control b.
#pragma once

#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdlib>
#include <sstream>
#include <string>
#include <string_view>
#include <vector>

#include "qtask/engine.hpp"
#include "qtask/gate.hpp"
#include "qtask/types.hpp"

namespace qtask::qasm {

class ParseError : public Error {
 public:
  ParseError(const std::string& message, int line, int column)
      : Error("qasm:" + std::to_string(line) + ":" + std::to_string(column) + ": " + message),
        line_(line), column_(column) {}
  int line() const { return line_; }
  int column() const { return column_; }

 private:
  int line_, column_;
};

class UnsupportedGateError : public Error {
 public:
  UnsupportedGateError(const std::string& name, int line, int column)
      : Error("qasm:" + std::to_string(line) + ":" + std::to_string(column) +
              ": unsupported statement '" + name + "'"),
        line_(line), column_(column) {}
  int line() const { return line_; }
  int column() const { return column_; }

 private:
  int line_, column_;
};

struct Statement {
  enum class Kind { Gate, Barrier };
  Kind kind = Kind::Gate;
  GateKind gate = GateKind::X;
  double theta = 0.0;
  bool has_theta = false;
  std::vector<int> qubits;  // cx: control first, target second
  int line = 0;
  int column = 0;
};

struct QasmProgram {
  std::size_t num_qubits = 0;
  std::string qreg_name = "q";
  std::vector<Statement> statements;
};

namespace detail {

inline bool rotation(GateKind k) {
  return k == GateKind::Rx || k == GateKind::Ry || k == GateKind::Rz;
}
inline bool two_qubit(GateKind k) { return k == GateKind::Cnot || k == GateKind::Swap; }

inline const char* gate_word(GateKind k) {
  switch (k) {
    case GateKind::Cnot: return "cx";
    case GateKind::X: return "x";
    case GateKind::Y: return "y";
    case GateKind::Z: return "z";
    case GateKind::H: return "h";
    case GateKind::S: return "s";
    case GateKind::Sdg: return "sdg";
    case GateKind::T: return "t";
    case GateKind::Tdg: return "tdg";
    case GateKind::Rx: return "rx";
    case GateKind::Ry: return "ry";
    case GateKind::Rz: return "rz";
    case GateKind::Swap: return "swap";
    default: return nullptr;  // U3 / Cz have no QASM 2.0 qelib spelling here
  }
}

inline bool gate_of(const std::string& w, GateKind* out) {
  static const GateKind all[] = {GateKind::Cnot, GateKind::X,   GateKind::Y,  GateKind::Z,
                                 GateKind::H,    GateKind::S,   GateKind::Sdg, GateKind::T,
                                 GateKind::Tdg,  GateKind::Rx,  GateKind::Ry, GateKind::Rz,
                                 GateKind::Swap};
  for (GateKind k : all) {
    if (w == gate_word(k)) {
      *out = k;
      return true;
    }
  }
  return false;
}

// Token cursor over the source text: identifiers, numbers, "strings" and
// one-character symbols; whitespace and // comments are skipped.
class Cursor {
 public:
  enum Type { Ident, Number, String, Symbol, End };
  struct Tok {
    Type type = End;
    std::string text;
    int line = 1, column = 1;
  };

  explicit Cursor(std::string_view src) : s_(src) { advance(); }
  const Tok& tok() const { return t_; }

  void advance() {
    skip_blank();
    t_ = Tok{};
    t_.line = line_;
    t_.column = col_;
    if (i_ >= s_.size()) return;
    const char c = s_[i_];
    if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
      t_.type = Ident;
      while (i_ < s_.size() && (std::isalnum(static_cast<unsigned char>(s_[i_])) || s_[i_] == '_'))
        t_.text += take();
    } else if (std::isdigit(static_cast<unsigned char>(c)) || c == '.') {
      t_.type = Number;
      while (i_ < s_.size()) {
        const char d = s_[i_];
        const bool exp_sign = (d == '+' || d == '-') && !t_.text.empty() &&
                              (t_.text.back() == 'e' || t_.text.back() == 'E');
        if (std::isdigit(static_cast<unsigned char>(d)) || d == '.' || d == 'e' || d == 'E' ||
            exp_sign)
          t_.text += take();
        else
          break;
      }
    } else if (c == '"') {
      t_.type = String;
      take();
      while (i_ < s_.size() && s_[i_] != '"') t_.text += take();
      if (i_ >= s_.size()) throw ParseError("unterminated string", t_.line, t_.column);
      take();
    } else {
      t_.type = Symbol;
      t_.text = std::string(1, take());
    }
  }

 private:
  char take() {
    const char c = s_[i_++];
    if (c == '\n') {
      ++line_;
      col_ = 1;
    } else {
      ++col_;
    }
    return c;
  }
  void skip_blank() {
    while (i_ < s_.size()) {
      if (std::isspace(static_cast<unsigned char>(s_[i_]))) {
        take();
      } else if (s_[i_] == '/' && i_ + 1 < s_.size() && s_[i_ + 1] == '/') {
        while (i_ < s_.size() && s_[i_] != '\n') take();
      } else {
        break;
      }
    }
  }

  std::string_view s_;
  std::size_t i_ = 0;
  int line_ = 1, col_ = 1;
  Tok t_;
};

class Reader {
 public:
  explicit Reader(std::string_view src) : c_(src) {}

  QasmProgram read() {
    word("OPENQASM");
    const Cursor::Tok v = want(Cursor::Number, "version");
    if (v.text != "2.0") throw ParseError("unsupported OPENQASM version " + v.text, v.line, v.column);
    sym(";");
    bool have_qreg = false;
    while (c_.tok().type != Cursor::End) {
      const Cursor::Tok head = want(Cursor::Ident, "statement");
      if (head.text == "include") {
        const Cursor::Tok f = want(Cursor::String, "include file");
        if (f.text != "qelib1.inc")
          throw ParseError("unsupported include \"" + f.text + "\"", f.line, f.column);
        sym(";");
      } else if (head.text == "qreg") {
        if (have_qreg)
          throw ParseError("a second qreg is not supported", head.line, head.column);
        have_qreg = true;
        std::size_t size = 0;
        prog_.qreg_name = reg_decl(&size);
        prog_.num_qubits = size;
      } else if (head.text == "creg") {
        std::size_t ignored = 0;
        reg_decl(&ignored);
      } else if (head.text == "barrier") {
        barrier(head);
      } else {
        gate(head, have_qreg);
      }
    }
    if (!have_qreg) throw ParseError("no qreg declaration", 1, 1);
    return std::move(prog_);
  }

 private:
  bool at(const char* s) const {
    return c_.tok().type == Cursor::Symbol && c_.tok().text == s;
  }
  Cursor::Tok want(Cursor::Type type, const std::string& what) {
    if (c_.tok().type != type) throw ParseError("expected " + what, c_.tok().line, c_.tok().column);
    Cursor::Tok t = c_.tok();
    c_.advance();
    return t;
  }
  void sym(const char* s) {
    if (!at(s))
      throw ParseError(std::string("expected '") + s + "'", c_.tok().line, c_.tok().column);
    c_.advance();
  }
  void word(const char* w) {
    if (c_.tok().type != Cursor::Ident || c_.tok().text != w)
      throw ParseError(std::string("expected '") + w + "'", c_.tok().line, c_.tok().column);
    c_.advance();
  }

  std::string reg_decl(std::size_t* size) {
    const Cursor::Tok name = want(Cursor::Ident, "register name");
    sym("[");
    const Cursor::Tok n = want(Cursor::Number, "register size");
    sym("]");
    sym(";");
    const long v = std::strtol(n.text.c_str(), nullptr, 10);
    if (v < 1) throw ParseError("register size must be >= 1", n.line, n.column);
    *size = static_cast<std::size_t>(v);
    return name.text;
  }

  int qubit() {
    const Cursor::Tok reg = want(Cursor::Ident, "qubit operand");
    if (reg.text != prog_.qreg_name)
      throw ParseError("unknown register '" + reg.text + "'", reg.line, reg.column);
    if (!at("["))
      throw ParseError("whole-register operands are not supported (use q[i])", c_.tok().line,
                       c_.tok().column);
    c_.advance();
    const Cursor::Tok i = want(Cursor::Number, "qubit index");
    sym("]");
    const long q = std::strtol(i.text.c_str(), nullptr, 10);
    if (q < 0 || static_cast<std::size_t>(q) >= prog_.num_qubits)
      throw ParseError("qubit index outside the register", i.line, i.column);
    return static_cast<int>(q);
  }

  double term() {
    if (c_.tok().type == Cursor::Ident && c_.tok().text == "pi") {
      c_.advance();
      return M_PI;
    }
    return std::strtod(want(Cursor::Number, "angle").text.c_str(), nullptr);
  }

  double angle() {
    double sign = 1.0;
    if (at("-")) {
      c_.advance();
      sign = -1.0;
    }
    double v = term();
    while (at("*") || at("/")) {
      const bool mul = at("*");
      c_.advance();
      const double r = term();
      v = mul ? v * r : v / r;
    }
    return sign * v;
  }

  void barrier(const Cursor::Tok& head) {
    Statement st;
    st.kind = Statement::Kind::Barrier;
    st.line = head.line;
    st.column = head.column;
    while (!at(";")) {  // operands do not matter: a barrier separates all levels
      if (c_.tok().type == Cursor::End) throw ParseError("expected ';'", c_.tok().line, c_.tok().column);
      c_.advance();
    }
    c_.advance();
    prog_.statements.push_back(st);
  }

  void gate(const Cursor::Tok& head, bool have_qreg) {
    Statement st;
    if (!gate_of(head.text, &st.gate)) throw UnsupportedGateError(head.text, head.line, head.column);
    if (!have_qreg) throw ParseError("gate used before the qreg declaration", head.line, head.column);
    st.line = head.line;
    st.column = head.column;
    if (rotation(st.gate)) {
      sym("(");
      st.theta = angle();
      st.has_theta = true;
      sym(")");
    } else if (at("(")) {
      throw ParseError("unexpected parameter list", c_.tok().line, c_.tok().column);
    }
    st.qubits.push_back(qubit());
    while (at(",")) {
      c_.advance();
      st.qubits.push_back(qubit());
    }
    sym(";");
    const std::size_t arity = two_qubit(st.gate) ? 2 : 1;
    if (st.qubits.size() != arity)
      throw ParseError("wrong operand count for '" + head.text + "'", head.line, head.column);
    if (arity == 2 && st.qubits[0] == st.qubits[1])
      throw ParseError("two-qubit gate on one qubit", head.line, head.column);
    prog_.statements.push_back(std::move(st));
  }

  Cursor c_;
  QasmProgram prog_;
};

}  // namespace detail

/// Parses OpenQASM 2.0 text (the subset above).
inline QasmProgram parse(std::string_view text) { return detail::Reader(text).read(); }

/// Regenerates QASM text (statement order preserved, angles with 17 digits).
inline std::string to_qasm(const QasmProgram& p) {
  std::ostringstream os;
  os.precision(17);
  os << "OPENQASM 2.0;\ninclude \"qelib1.inc\";\nqreg " << p.qreg_name << "[" << p.num_qubits
     << "];\n";
  for (const Statement& st : p.statements) {
    if (st.kind == Statement::Kind::Barrier) {
      os << "barrier " << p.qreg_name << ";\n";
      continue;
    }
    const char* w = detail::gate_word(st.gate);
    os << (w ? w : "?");
    if (st.has_theta) os << "(" << st.theta << ")";
    for (std::size_t i = 0; i < st.qubits.size(); ++i)
      os << (i ? "," : " ") << p.qreg_name << "[" << st.qubits[i] << "]";
    os << ";\n";
  }
  return os.str();
}

/// ASAP levels: a gate lands one past the deepest earlier gate on any of its
/// qubits; a barrier moves every later gate past all levels seen so far.
/// Returns statement indices grouped by ascending level.
inline std::vector<std::vector<std::size_t>> levelize(const QasmProgram& p) {
  std::vector<int> depth(p.num_qubits, -1);
  std::vector<std::vector<std::size_t>> levels;
  int floor_level = 0, deepest = -1;
  for (std::size_t i = 0; i < p.statements.size(); ++i) {
    const Statement& st = p.statements[i];
    if (st.kind == Statement::Kind::Barrier) {
      floor_level = deepest + 1;
      continue;
    }
    int lv = floor_level;
    for (int q : st.qubits) lv = std::max(lv, depth[q] + 1);
    for (int q : st.qubits) depth[q] = lv;
    deepest = std::max(deepest, lv);
    if (levels.size() <= static_cast<std::size_t>(lv)) levels.resize(lv + 1);
    levels[lv].push_back(i);
  }
  return levels;
}

/// Appends one net per level and inserts its gates.
inline void build_circuit(Simulator& sim, const QasmProgram& p) {
  for (const auto& level : levelize(p)) {
    const NetId net = sim.insert_net_back();
    for (std::size_t i : level) {
      const Statement& st = p.statements[i];
      if (st.gate == GateKind::Cnot)
        sim.insert_gate(GateKind::Cnot, net, st.qubits[1], st.qubits[0]);
      else if (st.gate == GateKind::Swap)
        sim.insert_gate(GateKind::Swap, net, st.qubits[0], st.qubits[1]);
      else if (st.has_theta)
        sim.insert_gate(st.gate, st.theta, net, st.qubits[0]);
      else
        sim.insert_gate(st.gate, net, st.qubits[0]);
    }
  }
}

}  // namespace qtask::qasm
