// qt_sim.hpp -- incremental simulator with the reference's programming model
// (qtask::Simulator, engine.hpp:46-151) on the device state of qt_state.
#pragma once

#include <condition_variable>
#include <cstdint>
#include <deque>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <string>
#include <unordered_map>
#include <vector>

#include "qt_netindex.hpp"
#include "qt_partition.hpp"
#include "qt_state.hpp"

namespace qtb {

class Sim {
 public:
  Sim(int nqubits, const qt_config* cfg);
  ~Sim();

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
  const std::vector<uint32_t>& net_order() const;
  const std::vector<uint32_t>& net_gates(uint32_t net) const;
  void gate_info(uint32_t gate, qt_gate* out, uint32_t* net) const;
  // gates (and their ids) in circuit order from gate position `from` on
  std::vector<qt_gate> flatten(std::vector<uint32_t>* ids = nullptr, uint64_t from = 0) const;
  State& state() { return *st_; }

  // The reference-unit partition model (qt_partition.hpp), caught up with
  // every modifier / update so far; nullptr when it is off for this state
  // (auto: at most kModelMaxBlocks partition blocks). Callers hold the
  // returned lock while reading the model.
  const PartitionModel* model(std::unique_lock<std::mutex>* lk);

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
  // net order with subtree gate counts (qt_netindex.hpp): positions of nets
  // and gates in O(log nets); order_ is the flat copy net_order() hands out
  NetIndex index_;
  mutable std::vector<uint32_t> order_;
  mutable bool order_valid_ = true;
  std::unordered_map<uint32_t, std::vector<uint32_t>> nets_;
  std::unordered_map<uint32_t, GateRec> gates_;
  uint32_t next_net_ = 1, next_gate_ = 1;
  bool pending_ = false, ran_full_ = false;

  struct Ckpt {
    uint64_t pos;           // state after the first `pos` gates
    int buf;                // pool buffer holding it
    std::vector<int> perm;  // its logical -> physical qubit map
    uint32_t next_id = 0;   // the gate that followed it when it was written (0: none)
  };
  std::unique_ptr<State> st_;
  std::vector<Ckpt> chain_;  // valid checkpoints, increasing pos
  std::vector<uint32_t> bound_ids_;  // first gate of each segment of the last run (pos > 0)
  // plans of segments by (gate ids, input qubit map): segments re-simulated
  // unchanged after an edit skip planning
  std::unordered_map<std::string, std::shared_ptr<State::PreparedPlan>> seg_plans_;
  int nbuf_ = 1;
  qt_run_stats last_{};
  // partition model on its own thread: modifiers post events, queries wait
  // for the queue to drain (the reference's graph upkeep costs O(stages x
  // partitions) per edit; it never delays the device work)
  void post(std::function<void(PartitionModel&)> ev);
  void model_worker();
  std::unique_ptr<PartitionModel> model_;
  std::mutex q_mu_, model_mu_;
  std::condition_variable q_cv_, drained_cv_;
  std::deque<std::function<void(PartitionModel&)>> events_;
  bool busy_ = false, stop_ = false;
  std::string model_error_;
  std::thread model_thread_;
  bool trace_ = false;  // QTB_SIM_TRACE=1: per-segment timing / cache lines on stderr
  uint64_t trace_hits_ = 0, trace_misses_ = 0;
};

}  // namespace qtb
