// qt_state.hpp -- device-resident state vector + stateless gate application.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "qt_comm.hpp"
#include "qt_ir.hpp"
#include "qt_kernels.hpp"
#include "qt_plan.hpp"
#include "qt_jit.hpp"
#include "qt_micro.hpp"
#include "qtask_c.h"

namespace qtb {

// Destination map of a fused exchange (qt_state.cpp; audited by qt_fused_exchange_map).
void fused_exchange_map(int rank, int nlocal, const std::vector<std::pair<int, int>>& exchange,
                        std::vector<int>* group, uint64_t* rfix);

// Thrown inside the library; the C API converts it to a status code.
struct QtError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string& msg);
void cuda_check(cudaError_t e, const char* what);

enum class Mode { Single, Loopback, Sharded };

// Per-pass timing record (when timing is enabled).
struct PassTiming {
  cudaEvent_t start = nullptr, stop = nullptr;
  int kind = 0;  // 0 tile, 1 exchange
};

// One grouped send/recv step of a sharded exchange (State::exchange): for
// each entry i, send `piece` amplitudes at shard offset send_off[i] to
// peer[i] and receive as many from peer[i] into the exchange buffer at
// recv_off[i], then copy them back over send_off[i] (or, two-buffer scheme,
// receive straight into the second buffer at send_off[i]). A peer can appear
// in several entries of a step; its sends and receives match in order.
struct ExchangeStep {
  uint64_t piece = 0;
  std::vector<int> peer;
  std::vector<uint64_t> send_off, recv_off;
};
// The steps of one exchange pass on `rank` (pairs: global physical bit,
// local victim bit), for an exchange buffer of tmp_amps amplitudes.
std::vector<ExchangeStep> exchange_schedule(int rank, int nlocal,
                                            const std::vector<std::pair<int, int>>& ex,
                                            uint64_t tmp_amps);

class State {
 public:
  // Sharded states exchange through NCCL (nccl_id) or, when `group` is
  // given, through the in-process transport of that group (qt_comm.hpp).
  State(int nqubits, Mode mode, int shards, int rank, const void* nccl_id,
        const qt_config* cfg, std::shared_ptr<LocalGroup> group = nullptr);
  ~State();

  int nqubits() const { return n_; }
  int nlocal() const { return nlocal_; }
  Mode mode() const { return mode_; }
  cudaStream_t stream() const { return stream_; }
  double2* data() { return psi_; }
  uint64_t buffer_amps() const { return 1ull << buf_bits_; }
  const std::vector<int>& perm() const { return perm_; }

  void set_basis(uint64_t index);
  void write(uint64_t first, uint64_t count, const double* src);
  void read(uint64_t first, uint64_t count, double* dst);
  // Applies pre-lowered logical ops (already fused). If src is given (a
  // buffer of the same geometry, perm src_perm), the state is computed from
  // src out of place: the first pass reads src and writes the bound buffer.
  void apply_ops(const std::vector<LOp>& ops, uint64_t ngates,
                 const double2* src = nullptr,
                 const std::vector<int>* src_perm = nullptr);

  // Extra full-state buffers (the incremental engine's checkpoint chain).
  // Buffer 0 is the one allocated at construction. Returns how many exist.
  int grow_pool(int count, double max_fraction_of_free);
  int pool_size() const { return static_cast<int>(pool_.size()); }
  double2* buffer(int i) const { return pool_[i]; }
  int bound() const { return bound_; }
  void bind(int i, const std::vector<int>& perm);
  void apply(const qt_gate* gates, size_t count);
  double norm_squared();
  // The k amplitudes of largest |a|^2 (ties: smaller logical index first),
  // sorted; logical indices. Single / loopback states (State::top_k).
  std::vector<TopkItem> top_k(uint64_t k);
  std::vector<TopkItem> top_k_local(uint64_t k, int bits, const std::vector<int>& perm);
  void sync();  // also raises QT_ERR_NUMERIC if a pass saw a non-finite value
  // a call on this rank failed: release the group's other ranks
  void abort_comm(const std::string& why) {
    if (comm_) comm_->abort(why);
  }

  void checkpoint_save(int slot);
  void checkpoint_restore(int slot);
  void checkpoint_drop(int slot);
  void checkpoint_drop_all();
  bool has_checkpoint(int slot) const { return ckpt_.count(slot) != 0; }
  // D2D copy of the whole local buffer + perm between two states of the same
  // geometry (used by the incremental engine's checkpoint chain).
  void copy_from(const State& other);

  Plan plan(const std::vector<LOp>& ops) const;
  const PlanOptions& options() const { return opt_; }

  // A plan with its host-side preparation (lowering, compiled passes), for
  // callers that re-run the same ops (the incremental engine's segments).
  struct PreparedPlan;
  // Plans `ops` from qubit map `perm` (nullptr: the current one).
  std::shared_ptr<PreparedPlan> prepare_ops(const std::vector<LOp>& ops,
                                            const std::vector<int>* perm);
  // apply_ops with the planning already done.
  void apply_prepared(const PreparedPlan& pp, uint64_t ngates, const double2* src = nullptr,
                      const std::vector<int>* src_perm = nullptr);
  void set_timing(bool on) { timing_ = on; }
  // Device ms of every launch of the last apply (timing enabled).
  std::vector<std::pair<int, float>> last_timings(bool consume = true);

  qt_run_stats stats{};

 private:
  // the per-plan host work before launching: lowering + compiled passes
  struct Prepared {
    std::vector<MicroPass> micro;
    std::vector<JitKernel> jk;
  };
  Prepared prepare(const Plan& plan);

 public:
  struct PreparedPlan {
    Plan plan;
    Prepared prep;
    double plan_ms = 0.0;
  };

 private:
  void launch_prepared(const Plan& plan, const Prepared& pr, const double2* src);
  void upload_and_launch(const Plan& plan, const double2* src);
  // apply(): the previous call's plan, reused when the same gate list is
  // applied again from the same qubit map
  struct LastApply {
    bool valid = false;
    std::string key;
    Plan plan;
    Prepared prep;
  };
  LastApply last_;
  void exchange(const PlanPass& pass);

  int n_ = 0, nlocal_ = 0, buf_bits_ = 0;
  Mode mode_ = Mode::Single;
  int rank_ = 0, world_ = 1, device_ = 0;
  cudaStream_t stream_ = nullptr;
  double2* psi_ = nullptr;
  double* d_scratch_ = nullptr;   // norm partials + result + gather
  int* d_flag_ = nullptr;
  int* h_flag_ = nullptr;         // pinned
  // kernel-parameter blocks (ops travel in the launch's constant bank)
  std::unique_ptr<KPassSmall> kp_small_;
  std::unique_ptr<KPassLarge> kp_large_;
  double2* alt_ = nullptr;        // second shard buffer of the two-buffer exchange
  bool alt_tried_ = false;
  bool no_alt_ = false;           // QTB_EXCHANGE_TMP=1: always the receive-buffer scheme
  double2* d_tmp_ = nullptr;      // exchange receive buffer
  size_t d_tmp_amps_ = 0;
  std::vector<int> perm_;         // logical -> physical
  std::vector<double2*> pool_;
  int bound_ = 0;
  std::map<int, std::pair<double2*, std::vector<int>>> ckpt_;
  std::unique_ptr<Comm> comm_;
  PlanOptions opt_;
  // tile-pass streaming mode: double-buffered cp.async (pipe_) and / or L2
  // prefetch of the next tile (pf_); QTB_PIPE / QTB_PF override
  bool pipe_ = false;
  bool pf_ = false;
  int pf_bits_ = 0;  // QTB_PF=b: prefetch runs of up to 2^b amplitudes (compiled direct rounds)
  // compiled passes: double-buffer only passes with at most this many FP64
  // ops per amplitude (<= 0: every pass when pipe_)
  double pipe_max_fp64_ = 0.0;
  // compiled passes (qt_jit.cpp; cfg->compiled or QTB_JIT): 1 = every
  // lowered tile pass runs its own straight-line kernel (compiled on first
  // use); 2 = hybrid: passes found in the compile cache run compiled, the
  // others on the interpreter while they compile in the background
  int jit_mode_ = 0;
  bool plan_search_ = true;  // compiled mode: search the per-pass FP64 cap (QTB_PLAN_SEARCH=0: off)
  int jit_min_blocks_ = 0;  // compiled passes' launch-bound override (QTB_JIT_MINB)
  // compiled passes: first / last round straight from / to HBM when physical
  // bits [0, direct_bits_) stay thread bits (128-B runs); 0 = always stage
  int direct_bits_ = kJitDirectBits;
  void ensure_alt();
  void decide_fusion();
  bool fuse_decided_ = false, fuse_ok_ = false;  // fused exchanges (collective decision, first apply)
  int window_mode_ = -1;  // QTB_WINDOW_SEARCH: -1 auto (plan-search candidate), 0 never, 1 always
  int occupancy_ = 1, sms_ = 148;
  bool timing_ = false;
  std::vector<PassTiming> timings_;
  size_t timings_used_ = 0;
  cudaEvent_t ev0_ = nullptr, ev1_ = nullptr;
};

}  // namespace qtb
