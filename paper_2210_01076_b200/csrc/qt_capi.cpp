// qt_capi.cpp -- extern "C" entry points of include/qtask_c.h.
//
// Every entry point converts internal failures (QtError, std::bad_alloc,
// anything else) into a QT_ERR_* status and a thread-local message, so no
// C++ exception crosses the C ABI. include/qtask/engine.hpp maps the codes
// back onto the reference exception types (types.hpp:21-64).
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <sstream>
#include <string>

#include "qt_gates.hpp"
#include "qt_jit.hpp"
#include "qt_kernels.hpp"
#include "qt_micro.hpp"
#include "qt_plan.hpp"
#include "qt_netindex.hpp"
#include "qt_sim.hpp"
#include "qt_state.hpp"
#include "qtask_c.h"
#include "qtask/qasm.hpp"

struct qt_state {
  qtb::State* s;
};
struct qt_sim {
  qtb::Sim* s;
};

namespace {
thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return QT_OK;
  } catch (const qtb::QtError& e) {
    g_err = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return QT_ERR_OOM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return QT_ERR_ARG;
  } catch (...) {
    g_err = "unknown failure";
    return QT_ERR_ARG;
  }
}

// Collective calls of a sharded state: a failure on this rank releases the
// rest of an in-process group (their rendezvous report it) instead of
// leaving them waiting for this rank.
template <typename F>
int guard_collective(qt_state* st, F&& f) {
  const int rc = guard(std::forward<F>(f));
  if (rc != QT_OK) st->s->abort_comm(g_err);
  return rc;
}


int null_arg() {
  g_err = "null argument";
  return QT_ERR_ARG;
}

int copy_out(const std::string& s, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = s.size() + 1;
  if (buf && cap > 0) {
    const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
    std::memcpy(buf, s.data(), n);
    buf[n] = 0;
  }
  return QT_OK;
}
}  // namespace

extern "C" {

int qt_plan_probe_ex(int num_qubits, int global_qubits, int tile_qubits, int detail,
                     const qt_gate* gates, size_t count, char* buf, size_t cap,
                     size_t* needed);

const char* qt_last_error(void) { return g_err.c_str(); }

const char* qt_version(void) { return "qtask-b200 0.1 sm_100a"; }

int qt_device_count(int* out) {
  if (!out) return null_arg();
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *out = n;
  return QT_OK;
}

// ---- state ------------------------------------------------------------------

int qt_state_create(int num_qubits, const qt_config* cfg, qt_state** out) {
  if (!out) return null_arg();
  return guard([&] {
    *out = new qt_state{new qtb::State(num_qubits, qtb::Mode::Single, 1, 0, nullptr, cfg)};
  });
}

int qt_state_create_sharded(int num_qubits, int rank, int world,
                            const void* nccl_id, const qt_config* cfg,
                            qt_state** out) {
  if (!out || !nccl_id) return null_arg();
  return guard([&] {
    *out = new qt_state{new qtb::State(num_qubits, qtb::Mode::Sharded, world, rank, nccl_id, cfg)};
  });
}

struct qt_group {
  std::shared_ptr<qtb::LocalGroup> g;
};

int qt_group_create(int world, qt_group** out) {
  if (!out) return null_arg();
  return guard([&] {
    if (world < 1 || (world & (world - 1)) != 0) qtb::fail(QT_ERR_ARG, "group size must be a power of two");
    *out = new qt_group{std::make_shared<qtb::LocalGroup>(world)};
  });
}

int qt_group_destroy(qt_group* g) {
  if (!g) return QT_OK;
  return guard([&] { delete g; });
}

int qt_state_create_group(int num_qubits, qt_group* group, int rank, const qt_config* cfg,
                          qt_state** out) {
  if (!out || !group) return null_arg();
  return guard([&] {
    *out = new qt_state{new qtb::State(num_qubits, qtb::Mode::Sharded, group->g->world(), rank,
                                       nullptr, cfg, group->g)};
  });
}

int qt_state_create_loopback(int num_qubits, int shards, const qt_config* cfg,
                             qt_state** out) {
  if (!out) return null_arg();
  return guard([&] {
    *out = new qt_state{new qtb::State(num_qubits, qtb::Mode::Loopback, shards, 0, nullptr, cfg)};
  });
}

int qt_nccl_unique_id(void* out128) {
  if (!out128) return null_arg();
  return guard([&] {
    std::string err;
    if (!qtb::NcclComm::unique_id(out128, &err)) qtb::fail(QT_ERR_NCCL, err);
  });
}

int qt_state_destroy(qt_state* st) {
  if (!st) return QT_OK;
  return guard([&] {
    delete st->s;
    delete st;
  });
}

int qt_state_num_qubits(const qt_state* st) { return st ? st->s->nqubits() : -1; }

int qt_set_basis(qt_state* st, uint64_t index) {
  if (!st) return null_arg();
  return guard([&] { st->s->set_basis(index); });
}

int qt_write(qt_state* st, uint64_t first, uint64_t count, const double* in) {
  if (!st || (!in && count)) return null_arg();
  return guard([&] { st->s->write(first, count, in); });
}

int qt_read(qt_state* st, uint64_t first, uint64_t count, double* outp) {
  if (!st || (!outp && count)) return null_arg();
  return guard([&] { st->s->read(first, count, outp); });
}

int qt_apply(qt_state* st, const qt_gate* gates, size_t count) {
  if (!st || (!gates && count)) return null_arg();
  return guard_collective(st, [&] { st->s->apply(gates, count); });
}

int qt_norm_squared(qt_state* st, double* outp) {
  if (!st || !outp) return null_arg();
  return guard_collective(st, [&] { *outp = st->s->norm_squared(); });
}

int qt_sync(qt_state* st) {
  if (!st) return null_arg();
  return guard([&] { st->s->sync(); });
}

int qt_last_stats(const qt_state* st, qt_run_stats* outp) {
  if (!st || !outp) return null_arg();
  *outp = st->s->stats;
  return QT_OK;
}

int qt_checkpoint_save(qt_state* st, int slot) {
  if (!st) return null_arg();
  return guard([&] { st->s->checkpoint_save(slot); });
}

int qt_checkpoint_restore(qt_state* st, int slot) {
  if (!st) return null_arg();
  return guard([&] { st->s->checkpoint_restore(slot); });
}

int qt_plan_json(const qt_state* st, const qt_gate* gates, size_t count,
                 char* buf, size_t cap, size_t* needed) {
  if (!st || (!gates && count)) return null_arg();
  return guard([&] {
    std::vector<qtb::LOp> ops;
    std::string err;
    const int n = st->s->nqubits();
    for (size_t i = 0; i < count; ++i) {
      const int rc = qtb::lower_gate(gates[i], n, static_cast<uint32_t>(i), ops, &err);
      if (rc != QT_OK) qtb::fail(rc, err);
    }
    qtb::fuse_ops(ops, n);
    const qtb::Plan p = st->s->plan(ops);
    const int R = st->s->options().reg_bits;
    const std::vector<qtb::MicroPass> mp = qtb::lower_plan_micro(
        p, R,
        qtb::MicroLimits{static_cast<size_t>(qtb::micro_capacity<qtb::KPassLarge>()),
                         sizeof(qtb::KPassLarge::pool) / sizeof(double),
                         sizeof(qtb::KPassLarge::rounds) / sizeof(qtb::DRound)});
    std::vector<double> fp(p.passes.size(), -1.0);
    for (size_t i = 0; i < p.passes.size(); ++i)
      if (mp[i].ok)
        fp[i] = qtb::micro_fp64_per_amp(mp[i], std::min<int>(R, static_cast<int>(p.passes[i].tile_phys.size())));
    copy_out(qtb::plan_to_json(p, false, &fp), buf, cap, needed);
  });
}

int qt_plan_probe(int num_qubits, int global_qubits, int tile_qubits,
                  const qt_gate* gates, size_t count, char* buf, size_t cap,
                  size_t* needed) {
  return qt_plan_probe_ex(num_qubits, global_qubits, tile_qubits, 0, gates, count,
                          buf, cap, needed);
}

// detail != 0: the JSON carries every round's register bits and encoded ops
// (tests/test_planner.py replays them with an independent numpy emulator).
int qt_plan_probe_ex(int num_qubits, int global_qubits, int tile_qubits, int detail,
                     const qt_gate* gates, size_t count, char* buf, size_t cap,
                     size_t* needed) {
  if (!gates && count) return null_arg();
  return guard([&] {
    if (num_qubits < 1 || num_qubits > 40 || global_qubits < 0 ||
        global_qubits >= num_qubits)
      qtb::fail(QT_ERR_BAD_QUBIT, "bad qubit counts");
    std::vector<qtb::LOp> ops;
    std::string err;
    for (size_t i = 0; i < count; ++i) {
      const int rc = qtb::lower_gate(gates[i], num_qubits, static_cast<uint32_t>(i), ops, &err);
      if (rc != QT_OK) qtb::fail(rc, err);
    }
    qtb::fuse_ops(ops, num_qubits);
    qtb::PlanOptions opt;
    if (tile_qubits > 0) opt.tile_bits = tile_qubits < qtb::kMaxTileBits ? tile_qubits : qtb::kMaxTileBits;
    if (const char* e = std::getenv("QTB_VICTIM_SPAN")) opt.victim_span = std::atoi(e);
    std::vector<int> perm(num_qubits);
    for (int q = 0; q < num_qubits; ++q) perm[q] = q;
    const qtb::Plan p = qtb::make_plan(ops, num_qubits, num_qubits - global_qubits, perm, opt);
    copy_out(qtb::plan_to_json(p, detail != 0), buf, cap, needed);
  });
}

// ---- extensions used by the Python host layer / bench ------------------------

// cudaStream_t of the state (events recorded on it time the passes).
void* qt_state_stream(qt_state* st) { return st ? static_cast<void*>(st->s->stream()) : nullptr; }

int qt_set_timing(qt_state* st, int on) {
  if (!st) return null_arg();
  st->s->set_timing(on != 0);
  return QT_OK;
}

// Per-launch device ms of the last apply: kinds[i] 0 = tile pass, 1 = exchange.
int qt_last_timings(qt_state* st, int* kinds, float* ms, size_t cap, size_t* count) {
  if (!st) return null_arg();
  return guard([&] {
    const auto t = st->s->last_timings(kinds != nullptr || ms != nullptr);
    if (count) *count = t.size();
    for (size_t i = 0; i < t.size() && i < cap; ++i) {
      if (kinds) kinds[i] = t[i].first;
      if (ms) ms[i] = t[i].second;
    }
  });
}

// FP64 pipe probe: returns DFMA/s measured with CUDA events.
int qt_probe_fp64(int device, double* dfma_per_s) {
  if (!dfma_per_s) return null_arg();
  return guard([&] {
    qtb::cuda_check(cudaSetDevice(device), "cudaSetDevice");
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    double* d = nullptr;
    qtb::cuda_check(cudaMalloc(&d, sizeof(double)), "probe alloc");
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = sms * 4, block = 256, iters = 4096;
    qtb::cuda_check(qtb::launch_fp64_probe(d, grid, block, iters, 0), "probe");
    cudaEventRecord(a, 0);
    qtb::cuda_check(qtb::launch_fp64_probe(d, grid, block, iters, 0), "probe");
    cudaEventRecord(b, 0);
    qtb::cuda_check(cudaEventSynchronize(b), "probe sync");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(d);
    *dfma_per_s = double(grid) * block * iters * 16.0 / (ms * 1e-3);
  });
}

// ---- incremental simulator ----------------------------------------------------

int qt_sim_create(int num_qubits, const qt_config* cfg, qt_sim** out) {
  if (!out) return null_arg();
  return guard([&] { *out = new qt_sim{new qtb::Sim(num_qubits, cfg)}; });
}

int qt_sim_destroy(qt_sim* sim) {
  if (!sim) return QT_OK;
  return guard([&] {
    delete sim->s;
    delete sim;
  });
}

int qt_sim_num_qubits(const qt_sim* sim) { return sim ? sim->s->nqubits() : -1; }
uint64_t qt_sim_block_size(const qt_sim* sim) { return sim ? sim->s->block_size() : 0; }
uint64_t qt_sim_total_blocks(const qt_sim* sim) { return sim ? sim->s->total_blocks() : 0; }

int qt_sim_insert_net_front(qt_sim* sim, uint32_t* net) {
  if (!sim || !net) return null_arg();
  return guard([&] { *net = sim->s->insert_net_front(); });
}
int qt_sim_insert_net_back(qt_sim* sim, uint32_t* net) {
  if (!sim || !net) return null_arg();
  return guard([&] { *net = sim->s->insert_net_back(); });
}
int qt_sim_insert_net_after(qt_sim* sim, uint32_t after, uint32_t* net) {
  if (!sim || !net) return null_arg();
  return guard([&] { *net = sim->s->insert_net_after(after); });
}
int qt_sim_remove_net(qt_sim* sim, uint32_t net) {
  if (!sim) return null_arg();
  return guard([&] { sim->s->remove_net(net); });
}
int qt_sim_insert_gate(qt_sim* sim, int kind, const double* params, uint32_t net,
                       int target, int control, uint32_t* gate) {
  if (!sim || !gate) return null_arg();
  return guard([&] { *gate = sim->s->insert_gate(kind, params, net, target, control); });
}
int qt_sim_remove_gate(qt_sim* sim, uint32_t gate) {
  if (!sim) return null_arg();
  return guard([&] { sim->s->remove_gate(gate); });
}
int qt_sim_update_state(qt_sim* sim) {
  if (!sim) return null_arg();
  return guard([&] { sim->s->update_state(); });
}
int qt_sim_pending(const qt_sim* sim) { return sim && sim->s->pending() ? 1 : 0; }

int qt_sim_amplitude(qt_sim* sim, uint64_t index, double* out2) {
  if (!sim || !out2) return null_arg();
  return guard([&] { sim->s->amplitudes(index, index, out2); });
}
int qt_sim_amplitudes(qt_sim* sim, uint64_t first, uint64_t last, double* outp) {
  if (!sim || !outp) return null_arg();
  return guard([&] { sim->s->amplitudes(first, last, outp); });
}
namespace {
void put_topk(const std::vector<qtb::TopkItem>& items, uint64_t* idx, double* amps,
              uint64_t* count) {
  for (size_t i = 0; i < items.size(); ++i) {
    if (idx) idx[i] = items[i].index;
    if (amps) {
      amps[2 * i] = items[i].amp.x;
      amps[2 * i + 1] = items[i].amp.y;
    }
  }
  if (count) *count = items.size();
}
}  // namespace

int qt_sim_top_k(qt_sim* sim, uint64_t k, uint64_t* idx, double* amps, uint64_t* count) {
  if (!sim) return null_arg();
  return guard([&] { put_topk(sim->s->top_k(k), idx, amps, count); });
}

int qt_top_k(qt_state* st, uint64_t k, uint64_t* idx, double* amps, uint64_t* count) {
  if (!st) return null_arg();
  return guard_collective(st, [&] { put_topk(st->s->top_k(k), idx, amps, count); });
}

int qt_sim_norm_squared(qt_sim* sim, double* outp) {
  if (!sim || !outp) return null_arg();
  return guard([&] { *outp = sim->s->norm_squared(); });
}
int qt_sim_last_update(const qt_sim* sim, qt_run_stats* outp) {
  if (!sim || !outp) return null_arg();
  *outp = sim->s->last_update();
  return QT_OK;
}

int qt_sim_update_account(qt_sim* sim, qt_update_account* out, uint64_t* blocks, size_t cap) {
  if (!sim || !out) return null_arg();
  return guard([&] {
    *out = qt_update_account{};
    std::unique_lock<std::mutex> lk;
    const qtb::PartitionModel* m = sim->s->model(&lk);
    if (!m) return;
    const qtb::PmAccount& a = m->account();
    out->valid = 1;
    out->full = a.full ? 1 : 0;
    out->executed_partitions = a.executed_partitions;
    out->materialized_blocks = a.materialized_blocks;
    out->rewritten_amplitudes = a.rewritten_amplitudes;
    out->rewritten_block_count = a.rewritten_blocks.size();
    if (blocks)
      for (size_t i = 0; i < a.rewritten_blocks.size() && i < cap; ++i) blocks[i] = a.rewritten_blocks[i];
  });
}

int qt_sim_model_snapshot(qt_sim* sim, qt_model_sizes* sizes, qt_model_stage* stages,
                          qt_model_part* parts, qt_model_task* tasks, uint64_t* edges,
                          uint8_t* materialized, uint64_t* frontiers) {
  if (!sim || !sizes) return null_arg();
  return guard([&] {
    *sizes = qt_model_sizes{};
    std::unique_lock<std::mutex> lk;
    const qtb::PartitionModel* m = sim->s->model(&lk);
    if (!m) return;
    const auto views = m->stages();
    const auto es = m->edges();
    sizes->valid = 1;
    sizes->stages = views.size();
    sizes->blocks = m->num_blocks();
    sizes->edges = es.size();
    sizes->frontiers = m->frontiers().size();
    uint64_t np = 0, nt = 0;
    for (size_t si = 0; si < views.size(); ++si) {
      const auto& v = views[si];
      if (stages)
        stages[si] = qt_model_stage{v.id, v.net, v.gate, static_cast<int32_t>(v.kind), np,
                                    static_cast<uint64_t>(v.parts->size())};
      for (size_t k = 0; k < v.parts->size(); ++k) {
        const qtb::PmPart& p = (*v.parts)[k];
        if (parts)
          parts[np] = qt_model_part{p.first_block, p.last_block, (*v.nodes)[k], nt,
                                    static_cast<uint64_t>(p.tasks.size())};
        for (const qtb::PmTask& t : p.tasks) {
          if (tasks) tasks[nt] = qt_model_task{t.first_op, t.last_op, t.lo, t.hi};
          ++nt;
        }
        ++np;
      }
      if (materialized) {
        uint8_t* row = materialized + si * m->num_blocks();
        for (uint64_t b = 0; b < m->num_blocks(); ++b)
          row[b] = v.materialized->empty() ? 0 : (*v.materialized)[b];
      }
    }
    sizes->parts = np;
    sizes->tasks = nt;
    if (edges)
      for (size_t i = 0; i < es.size(); ++i) {
        edges[2 * i] = es[i].first;
        edges[2 * i + 1] = es[i].second;
      }
    if (frontiers) {
      size_t i = 0;
      for (uint64_t f : m->frontiers()) frontiers[i++] = f;
    }
  });
}

int qt_sim_node_name(qt_sim* sim, uint64_t node, char* buf, size_t cap, size_t* needed) {
  if (!sim) return null_arg();
  return guard([&] {
    std::unique_lock<std::mutex> lk;
    const qtb::PartitionModel* m = sim->s->model(&lk);
    if (!m) qtb::fail(QT_ERR_ARG, "the partition model is off for this simulator");
    copy_out(m->node_name(node), buf, cap, needed);
  });
}

int qt_sim_dump_graph(qt_sim* sim, char* buf, size_t cap, size_t* needed) {
  if (!sim) return null_arg();
  return guard([&] {
    std::unique_lock<std::mutex> lk;
    const qtb::PartitionModel* m = sim->s->model(&lk);
    if (!m) qtb::fail(QT_ERR_ARG, "the partition model is off for this simulator");
    std::ostringstream os;
    m->dump_dot(os);
    copy_out(os.str(), buf, cap, needed);
  });
}

struct qt_pm {
  qtb::PartitionModel m;
};

int qt_pm_create(int num_qubits, uint64_t block_size, qt_pm** out) {
  if (!out) return null_arg();
  return guard([&] {
    if (num_qubits < 1 || num_qubits > 30) qtb::fail(QT_ERR_BAD_QUBIT, "qubit count must be in [1, 30]");
    if (block_size < 2 || (block_size & (block_size - 1)) != 0)
      qtb::fail(QT_ERR_ARG, "block size must be a power of two >= 2");
    *out = new qt_pm{qtb::PartitionModel(num_qubits, block_size)};
  });
}
int qt_pm_destroy(qt_pm* pm) {
  delete pm;
  return QT_OK;
}
int qt_pm_insert_net(qt_pm* pm, uint32_t net, int where, uint32_t after) {
  if (!pm) return null_arg();
  return guard([&] {
    if (where == 1) pm->m.insert_net_back(net);
    else pm->m.insert_net(net, where == 0 ? 0 : after);
  });
}
int qt_pm_remove_net(qt_pm* pm, uint32_t net) {
  if (!pm) return null_arg();
  return guard([&] { pm->m.remove_net(net); });
}
int qt_pm_insert_gate(qt_pm* pm, uint32_t gate, const qt_gate* g, uint32_t net) {
  if (!pm || !g) return null_arg();
  return guard([&] { pm->m.insert_gate(gate, *g, net); });
}
int qt_pm_remove_gate(qt_pm* pm, uint32_t gate) {
  if (!pm) return null_arg();
  return guard([&] { pm->m.remove_gate(gate); });
}
int qt_pm_update(qt_pm* pm) {
  if (!pm) return null_arg();
  return guard([&] { pm->m.update(); });
}
int qt_pm_account(qt_pm* pm, qt_update_account* out, uint64_t* blocks, size_t cap) {
  if (!pm || !out) return null_arg();
  return guard([&] {
    const qtb::PmAccount& a = pm->m.account();
    *out = qt_update_account{};
    out->valid = a.valid ? 1 : 0;
    out->full = a.full ? 1 : 0;
    out->executed_partitions = a.executed_partitions;
    out->materialized_blocks = a.materialized_blocks;
    out->rewritten_amplitudes = a.rewritten_amplitudes;
    out->rewritten_block_count = a.rewritten_blocks.size();
    if (blocks)
      for (size_t i = 0; i < a.rewritten_blocks.size() && i < cap; ++i) blocks[i] = a.rewritten_blocks[i];
  });
}
int qt_pm_dump_graph(qt_pm* pm, char* buf, size_t cap, size_t* needed) {
  if (!pm) return null_arg();
  return guard([&] {
    std::ostringstream os;
    pm->m.dump_dot(os);
    copy_out(os.str(), buf, cap, needed);
  });
}

int qt_gate_matrix(int kind, double theta, double phi, double lambda, double* m, int* dim) {
  if (!m || !dim) return null_arg();
  return guard([&] {
    if (!qtb::valid_kind(kind)) qtb::fail(QT_ERR_ARG, "unknown gate kind");
    if (qtb::is_two_qubit_kind(kind)) {
      // 4x4 with the sub-index (first << 1) | second (gate.hpp:39-41)
      for (int i = 0; i < 32; ++i) m[i] = 0.0;
      auto set = [&](int r, int c) { m[2 * (r * 4 + c)] = 1.0; };
      if (kind == QT_CNOT) { set(0, 0); set(1, 1); set(2, 3); set(3, 2); }
      else if (kind == QT_SWAP) { set(0, 0); set(1, 2); set(2, 1); set(3, 3); }
      else { set(0, 0); set(1, 1); set(2, 2); m[2 * 15] = -1.0; }
      *dim = 4;
      return;
    }
    const qtb::Mat2 g = kind == QT_U3 ? qtb::u3_matrix(theta, phi, lambda) : qtb::gate_matrix_1q(kind, theta);
    for (int i = 0; i < 4; ++i) {
      m[2 * i] = g[i].re;
      m[2 * i + 1] = g[i].im;
    }
    *dim = 2;
  });
}

int qt_classify_gate(int kind, double theta, double phi, double lambda) {
  qt_gate g{};
  g.kind = kind;
  g.theta = theta;
  g.phi = phi;
  g.lambda = lambda;
  if (!qtb::valid_kind(kind)) return QT_ERR_ARG;
  return qtb::is_superposition_gate(g) ? 1 : 0;
}

size_t qt_sim_num_gates(const qt_sim* sim) { return sim ? sim->s->num_gates() : 0; }
size_t qt_sim_num_nets(const qt_sim* sim) { return sim ? sim->s->net_order().size() : 0; }

int qt_sim_net_order(const qt_sim* sim, uint32_t* outp, size_t cap) {
  if (!sim || (!outp && cap)) return null_arg();
  const auto& o = sim->s->net_order();
  for (size_t i = 0; i < o.size() && i < cap; ++i) outp[i] = o[i];
  return QT_OK;
}

int qt_sim_net_gates(const qt_sim* sim, uint32_t net, uint32_t* outp, size_t cap,
                     size_t* count) {
  if (!sim) return null_arg();
  return guard([&] {
    const auto& gs = sim->s->net_gates(net);
    if (count) *count = gs.size();
    for (size_t i = 0; i < gs.size() && i < cap && outp; ++i) outp[i] = gs[i];
  });
}

int qt_sim_gate_info(const qt_sim* sim, uint32_t gate, qt_gate* outp, uint32_t* net) {
  if (!sim) return null_arg();
  return guard([&] { sim->s->gate_info(gate, outp, net); });
}

int qt_sim_export_gates(const qt_sim* sim, qt_gate* outp, size_t cap, size_t* count) {
  if (!sim) return null_arg();
  return guard([&] {
    const auto gs = sim->s->flatten();
    if (count) *count = gs.size();
    for (size_t i = 0; i < gs.size() && i < cap && outp; ++i) outp[i] = gs[i];
  });
}

int qt_exchange_schedule(int rank, int nlocal, int k, const int* gbit, const int* vbit,
                         uint64_t tmp_amps, uint64_t* rows, size_t cap, size_t* count,
                         uint64_t* piece) {
  if ((k > 0 && (!gbit || !vbit)) || k < 1 || nlocal < k || nlocal > 62) return null_arg();
  return guard([&] {
    std::vector<std::pair<int, int>> ex;
    for (int j = 0; j < k; ++j) ex.emplace_back(nlocal + gbit[j], vbit[j]);
    const auto steps = qtb::exchange_schedule(rank, nlocal, ex, tmp_amps);
    size_t n = 0;
    for (size_t si = 0; si < steps.size(); ++si) {
      for (size_t i = 0; i < steps[si].peer.size(); ++i, ++n) {
        if (rows && n < cap) {
          rows[4 * n] = si;
          rows[4 * n + 1] = static_cast<uint64_t>(steps[si].peer[i]);
          rows[4 * n + 2] = steps[si].send_off[i];
          rows[4 * n + 3] = steps[si].recv_off[i];
        }
      }
      if (piece) *piece = steps[si].piece;
    }
    if (count) *count = n;
  });
}

}  // extern "C"

// ---- OpenQASM 2.0 front end ---------------------------------------------------

namespace {
template <typename F>
int qasm_guard(int* err_line, int* err_col, F&& f) {
  try {
    f();
    return QT_OK;
  } catch (const qtask::qasm::ParseError& e) {
    if (err_line) *err_line = e.line();
    if (err_col) *err_col = e.column();
    g_err = e.what();
    return QT_ERR_QASM_PARSE;
  } catch (const qtask::qasm::UnsupportedGateError& e) {
    if (err_line) *err_line = e.line();
    if (err_col) *err_col = e.column();
    g_err = e.what();
    return QT_ERR_QASM_UNSUPPORTED;
  } catch (const qtask::Error& e) {  // the drop-in wrapper's mapped error
    g_err = e.what();
    return QT_ERR_ARG;
  }
}
}  // namespace

extern "C" {

int qt_qasm_parse(const char* text, size_t len, qt_qasm_stmt* outp, size_t cap,
                  size_t* count, uint32_t* num_qubits, int* err_line, int* err_col) {
  if (!text && len) return null_arg();
  int rc = QT_OK;
  const int g = guard([&] {
    rc = qasm_guard(err_line, err_col, [&] {
      const qtask::qasm::QasmProgram prog =
          qtask::qasm::parse(std::string_view(text ? text : "", len));
      std::vector<int> level(prog.statements.size(), -1);
      const auto levels = qtask::qasm::levelize(prog);
      for (size_t l = 0; l < levels.size(); ++l)
        for (size_t i : levels[l]) level[i] = static_cast<int>(l);
      if (count) *count = prog.statements.size();
      if (num_qubits) *num_qubits = static_cast<uint32_t>(prog.num_qubits);
      for (size_t i = 0; i < prog.statements.size() && i < cap && outp; ++i) {
        const auto& st = prog.statements[i];
        qt_qasm_stmt r{};
        r.kind = st.kind == qtask::qasm::Statement::Kind::Barrier ? 1 : 0;
        r.gate = static_cast<int32_t>(st.gate);
        r.theta = st.theta;
        r.has_theta = st.has_theta ? 1 : 0;
        r.nqubits = static_cast<int32_t>(st.qubits.size());
        for (size_t k = 0; k < st.qubits.size() && k < 2; ++k) r.qubits[k] = st.qubits[k];
        r.line = st.line;
        r.column = st.column;
        r.level = level[i];
        outp[i] = r;
      }
    });
  });
  return g != QT_OK ? g : rc;
}

int qt_qasm_build(qt_sim* sim, const char* text, size_t len, int* err_line, int* err_col) {
  if (!sim || (!text && len)) return null_arg();
  int rc = QT_OK;
  const int g = guard([&] {
    rc = qasm_guard(err_line, err_col, [&] {
      const qtask::qasm::QasmProgram prog =
          qtask::qasm::parse(std::string_view(text ? text : "", len));
      // build_circuit (qasm.cpp:407-426) through this handle's modifier calls
      for (const auto& lv : qtask::qasm::levelize(prog)) {
        uint32_t net = 0;
        qtask::detail::check(qt_sim_insert_net_back(sim, &net));
        for (size_t i : lv) {
          const auto& st = prog.statements[i];
          uint32_t gid = 0;
          const double th[3] = {st.theta, 0.0, 0.0};
          int t = st.qubits[0], c = -1;
          if (st.gate == qtask::GateKind::Cnot) {
            t = st.qubits[1];
            c = st.qubits[0];
          } else if (st.gate == qtask::GateKind::Swap) {
            c = st.qubits[1];
          }
          qtask::detail::check(qt_sim_insert_gate(sim, static_cast<int>(st.gate),
                                                  st.has_theta ? th : nullptr, net, t, c, &gid));
        }
      }
    });
  });
  return g != QT_OK ? g : rc;
}

}  // extern "C"

int qt_jit_probe(int num_qubits, int tile_qubits, int reg_bits, int low_bits, int compile,
                 int source_pass, const qt_gate* gates, size_t count, char* buf, size_t cap,
                 size_t* needed) {
  if (!gates && count) return null_arg();
  return guard([&] {
    if (num_qubits < 1 || num_qubits > 40) qtb::fail(QT_ERR_BAD_QUBIT, "bad qubit count");
    std::vector<qtb::LOp> ops;
    std::string err;
    for (size_t i = 0; i < count; ++i) {
      const int rc = qtb::lower_gate(gates[i], num_qubits, static_cast<uint32_t>(i), ops, &err);
      if (rc != QT_OK) qtb::fail(rc, err);
    }
    qtb::fuse_ops(ops, num_qubits);
    qtb::PlanOptions opt;
    if (reg_bits > 0) opt.reg_bits = std::min(reg_bits, qtb::kMaxRegBits);
    if (tile_qubits > 0) opt.tile_bits = std::min(tile_qubits, qtb::kMaxTileBits);
    if (low_bits > 0) opt.low_bits = low_bits;
    if (const char* e = std::getenv("QTB_PASS_FP64")) opt.max_pass_fp64 = std::atof(e);
    if (const char* e = std::getenv("QTB_VICTIM_SPAN")) opt.victim_span = std::atoi(e);
    if (const char* e = std::getenv("QTB_WINDOW_SEARCH")) opt.window_search = std::atoi(e) != 0;
    if (const char* e = std::getenv("QTB_WINDOW_BEAM")) opt.window_beam = std::atoi(e);
    if (const char* e = std::getenv("QTB_SHRINK_MIN")) opt.shrink_min_bits = std::max(0, std::atoi(e));
    if (const char* e = std::getenv("QTB_SHRINK_RUN")) opt.shrink_run_bits = std::max(0, std::atoi(e));
    std::vector<int> perm(num_qubits);
    for (int q = 0; q < num_qubits; ++q) perm[q] = q;
    const qtb::Plan p = qtb::make_plan(ops, num_qubits, num_qubits, perm, opt);
    const std::vector<qtb::MicroPass> mp = qtb::lower_plan_micro(
        p, opt.reg_bits,
        qtb::MicroLimits{static_cast<size_t>(qtb::micro_capacity<qtb::KPassLarge>()),
                         sizeof(qtb::KPassLarge::pool) / sizeof(double),
                         sizeof(qtb::KPassLarge::rounds) / sizeof(qtb::DRound)});
    size_t last_tile = p.passes.size();
    for (size_t i = 0; i < p.passes.size(); ++i)
      if (p.passes[i].kind == qtb::PlanPass::Tile) last_tile = i;
    if (source_pass == -2) {
      // the lowered layer words of every pass (tests/emulator.py replays them)
      std::string js = "{\"nqubits\":" + std::to_string(num_qubits) + ",\"passes\":[";
      char hx[32];
      for (size_t i = 0; i < p.passes.size(); ++i) {
        const qtb::PlanPass& ps = p.passes[i];
        if (i) js += ",";
        if (!mp[i].ok) {
          js += "{\"kind\":\"generic\"}";
          continue;
        }
        const int R = std::min<int>(opt.reg_bits, static_cast<int>(ps.tile_phys.size()));
        js += "{\"kind\":\"lowered\",\"R\":" + std::to_string(R) + ",\"tile_phys\":[";
        for (size_t t = 0; t < ps.tile_phys.size(); ++t)
          js += (t ? "," : "") + std::to_string(ps.tile_phys[t]);
        js += "],\"rounds\":[";
        for (size_t r = 0; r < ps.rounds.size(); ++r) {
          js += std::string(r ? "," : "") + "{\"reg\":[";
          for (size_t q = 0; q < ps.rounds[r].reg.size(); ++q)
            js += (q ? "," : "") + std::to_string(ps.rounds[r].reg[q]);
          js += "],\"first\":" + std::to_string(mp[i].round_first[r]) +
                ",\"count\":" + std::to_string(mp[i].round_count[r]) + "}";
        }
        js += "],\"words\":[";
        for (size_t w = 0; w < mp[i].size(); ++w)
          js += std::string(w ? "," : "") + "[" + std::to_string(mp[i].words[2 * w]) + "," +
                std::to_string(mp[i].words[2 * w + 1]) + "]";
        js += "],\"pool\":[";
        for (size_t k = 0; k < mp[i].pool.size(); ++k) {
          uint64_t b;
          std::memcpy(&b, &mp[i].pool[k], 8);
          std::snprintf(hx, sizeof(hx), "\"%016llx\"", static_cast<unsigned long long>(b));
          js += std::string(k ? "," : "") + hx;
        }
        js += "]}";
      }
      copy_out(js + "]}", buf, cap, needed);
      return;
    }
    size_t lowered = 0, bytes = 0, compiled = 0, cubin = 0;
    double ms = 0.0, fp = 0.0;
    std::string per = "[", rounds = "[";
    for (size_t i = 0; i < p.passes.size(); ++i) {
      if (!mp[i].ok) continue;
      ++lowered;
      const double f = qtb::micro_fp64_per_amp(mp[i], std::min<int>(opt.reg_bits, static_cast<int>(p.passes[i].tile_phys.size())));
      fp += f;
      per += (per.size() > 1 ? "," : "") + std::to_string(f);
      rounds += (rounds.size() > 1 ? "," : "") + std::to_string(p.passes[i].rounds.size());
      qtb::JitPassSpec sp = qtb::make_jit_spec(p.passes[i], opt.reg_bits, num_qubits, i == last_tile);
      // the state's tuning overrides (QTB_PIPE / QTB_JIT_MINB), as qt_state.cpp applies them
      if (const char* e = std::getenv("QTB_PIPE")) sp.pipe = std::atoi(e) != 0 && 2 * (16u << sp.k) <= 200u * 1024u;
      if (sp.pipe) sp.ring = false;
      if (const char* e = std::getenv("QTB_JIT_MINB")) sp.min_blocks = std::atoi(e);
      sp.coalesce_bits = qtb::kJitDirectBits;
      if (const char* e = std::getenv("QTB_DIRECT_BITS")) sp.coalesce_bits = std::atoi(e);
      // compile checks of the fused-exchange variant: QTB_PROBE_FUSE="v0[,v1[,v2]]"
      // (the victim bits of a pretended exchange after every pass)
      if (const char* e = std::getenv("QTB_PROBE_FUSE")) {
        sp.fuse_k = 0;
        for (const char* c = e; *c && sp.fuse_k < 3;) {
          sp.fuse_v[sp.fuse_k++] = std::atoi(c);
          while (*c && *c != ',') ++c;
          if (*c == ',') ++c;
        }
        if (sp.ring && sp.fuse_k > 0) {
          sp.tma_store = 0;
          sp.kparam = false;
        } else {
          sp.fuse_k = 0;
        }
      }
      const std::string src = qtb::jit_source(sp, mp[i]);
      if (source_pass >= 0) {
        if (static_cast<size_t>(source_pass) == i) {
          copy_out(src, buf, cap, needed);
          return;
        }
        continue;
      }
      bytes += src.size();
      if (compile) {
        const auto t0 = std::chrono::steady_clock::now();
        cubin += qtb::jit_compile_cubin(src).size();
        ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        ++compiled;
      }
    }
    if (source_pass >= 0) qtb::fail(QT_ERR_ARG, "source_pass is not a lowered tile pass");
    char js[256];
    std::snprintf(js, sizeof(js),
                  "{\"passes\":%zu,\"lowered\":%zu,\"source_bytes\":%zu,\"compiled\":%zu,"
                  "\"compile_ms\":%.1f,\"cubin_bytes\":%zu,\"fp64_per_amp\":%.1f,",
                  p.passes.size(), lowered, bytes, compiled, ms, cubin, fp);
    copy_out(std::string(js) + "\"pass_fp64\":" + per + "],\"pass_rounds\":" + rounds + "]}", buf, cap,
             needed);
  });
}

int qt_jit_stats(uint64_t* compiled, uint64_t* cache_hits, double* compile_ms) {
  if (!compiled || !cache_hits || !compile_ms) return null_arg();
  const qtb::JitStats st = qtb::jit_stats();
  *compiled = st.compiled;
  *cache_hits = st.cache_hits;
  *compile_ms = st.compile_ms;
  return QT_OK;
}

int qt_jit_disk_stats(uint64_t* disk_hits, uint64_t* disk_writes) {
  if (!disk_hits || !disk_writes) return null_arg();
  const qtb::JitStats st = qtb::jit_stats();
  *disk_hits = st.disk_hits;
  *disk_writes = st.disk_writes;
  return QT_OK;
}

int qt_fused_exchange_map(int rank, int nlocal, int k, const int* gbit, const int* vbit,
                          int* peer_rank, uint64_t* rfix) {
  if (!gbit || !vbit || !peer_rank || !rfix) return null_arg();
  return guard([&] {
    if (k < 1 || k > 3 || nlocal < 1) qtb::fail(QT_ERR_ARG, "fused exchange of 1..3 bits");
    std::vector<std::pair<int, int>> ex;
    for (int i = 0; i < k; ++i) ex.emplace_back(nlocal + gbit[i], vbit[i]);
    std::vector<int> group;
    uint64_t fix = 0;
    qtb::fused_exchange_map(rank, nlocal, ex, &group, &fix);
    for (size_t v = 0; v < group.size(); ++v) peer_rank[v] = group[v];
    *rfix = fix;
  });
}

int qt_netindex_audit(uint64_t seed, uint32_t ops, uint64_t* mismatches) {
  if (!mismatches) return null_arg();
  return guard([&] {
    qtb::NetIndex ix;
    std::vector<std::pair<uint32_t, uint64_t>> flat;  // (net, gates) in order
    uint64_t bad = 0, rng = seed * 0x9e3779b97f4a7c15ull + 1;
    auto next = [&] {
      rng ^= rng << 13;
      rng ^= rng >> 7;
      rng ^= rng << 17;
      return rng;
    };
    uint32_t next_id = 1;
    std::vector<uint32_t> order;
    for (uint32_t step = 0; step < ops; ++step) {
      const uint64_t r = next() % 10;
      if (flat.empty() || r < 3) {
        const size_t at = static_cast<size_t>(next() % (flat.size() + 1));
        ix.insert(next_id, at);
        flat.insert(flat.begin() + static_cast<std::ptrdiff_t>(at), {next_id, 0});
        ++next_id;
      } else if (r < 4) {
        const size_t at = static_cast<size_t>(next() % flat.size());
        ix.erase(flat[at].first);
        flat.erase(flat.begin() + static_cast<std::ptrdiff_t>(at));
      } else {
        const size_t at = static_cast<size_t>(next() % flat.size());
        int64_t d = static_cast<int64_t>(next() % 5) - 1;
        if (static_cast<int64_t>(flat[at].second) + d < 0) d = 1;
        ix.add_gates(flat[at].first, d);
        flat[at].second = static_cast<uint64_t>(static_cast<int64_t>(flat[at].second) + d);
      }
      // compare
      uint64_t total = 0;
      for (const auto& e : flat) total += e.second;
      bad += ix.nets() != flat.size();
      bad += ix.gates() != total;
      if (!flat.empty()) {
        const size_t at = static_cast<size_t>(next() % flat.size());
        uint64_t before = 0;
        for (size_t i = 0; i < at; ++i) before += flat[i].second;
        bad += ix.rank(flat[at].first) != at;
        bad += ix.gates_before(flat[at].first) != before;
        bad += ix.gates_of(flat[at].first) != flat[at].second;
        if (total) {
          const uint64_t pos = next() % total;
          uint64_t acc = 0, first = 0;
          uint32_t want = 0;
          for (const auto& e : flat) {
            if (pos < acc + e.second) {
              want = e.first;
              first = acc;
              break;
            }
            acc += e.second;
          }
          uint64_t got_first = 0;
          bad += ix.net_at_gate(pos, &got_first) != want;
          bad += got_first != first;
        }
        const size_t from = static_cast<size_t>(next() % (flat.size() + 1));
        ix.order(&order, from);
        bad += order.size() != flat.size() - from;
        for (size_t i = 0; i < order.size() && from + i < flat.size(); ++i) bad += order[i] != flat[from + i].first;
      }
    }
    *mismatches = bad;
  });
}

int qt_jit_pending(uint64_t* pending) {
  if (!pending) return null_arg();
  *pending = qtb::jit_pending();
  return QT_OK;
}
