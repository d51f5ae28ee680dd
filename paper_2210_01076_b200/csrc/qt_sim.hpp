// qt_sim.hpp -- incremental simulator with the reference's programming model
// (qtask::Simulator, engine.hpp:46-151) on the device state of qt_state.
#pragma once

#include <cstdint>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "qt_state.hpp"

namespace qtb {

class Sim {
 public:
  Sim(int nqubits, const qt_config* cfg);

  int nqubits() const { return n_; }
  uint64_t block_size() const { return bs_; }
  uint64_t total_blocks() const { return nblocks_; }

  uint32_t insert_net_front();
  uint32_t insert_net_back();
  uint32_t insert_net_after(uint32_t after);
  void remove_net(uint32_t net);
  uint32_t insert_gate(int kind, const double* params, uint32_t net, int target,
                       int control);
  void remove_gate(uint32_t gate);

  void update_state();
  bool pending() const { return pending_; }

  void amplitudes(uint64_t first, uint64_t last, double* out);
  double norm_squared();
  std::vector<TopkItem> top_k(uint64_t k);
  const qt_run_stats& last_update() const { return last_; }

  size_t num_gates() const { return gates_.size(); }
  const std::vector<uint32_t>& net_order() const { return order_; }
  const std::vector<uint32_t>& net_gates(uint32_t net) const;
  void gate_info(uint32_t gate, qt_gate* out, uint32_t* net) const;
  std::vector<qt_gate> flatten(std::vector<uint32_t>* ids = nullptr) const;
  State& state() { return *st_; }

 private:
  struct GateRec {
    qt_gate g;
    uint32_t net;
  };
  uint64_t position_of_net_end(uint32_t net) const;
  uint64_t position_of_gate(uint32_t gate) const;
  void edited_at(uint64_t pos);
  uint32_t new_net(size_t at);

  int n_;
  uint64_t bs_, nblocks_;
  qt_config cfg_{};
  std::vector<uint32_t> order_;
  std::unordered_map<uint32_t, std::vector<uint32_t>> nets_;
  std::unordered_map<uint32_t, GateRec> gates_;
  uint32_t next_net_ = 1, next_gate_ = 1;
  bool pending_ = false, ran_full_ = false;

  struct Ckpt {
    uint64_t pos;           // state after the first `pos` gates
    int buf;                // pool buffer holding it
    std::vector<int> perm;  // its logical -> physical qubit map
  };
  std::unique_ptr<State> st_;
  std::vector<Ckpt> chain_;  // valid checkpoints, increasing pos
  std::vector<uint32_t> bound_ids_;  // first gate of each segment of the last run (pos > 0)
  // plans of segments by (gate ids, input qubit map): segments re-simulated
  // unchanged after an edit skip planning
  std::unordered_map<std::string, std::shared_ptr<State::PreparedPlan>> seg_plans_;
  int nbuf_ = 1;
  qt_run_stats last_{};
  bool trace_ = false;  // QTB_SIM_TRACE=1: per-segment timing / cache lines on stderr
  uint64_t trace_hits_ = 0, trace_misses_ = 0;
};

}  // namespace qtb
