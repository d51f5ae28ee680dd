/*
 * qtask_c.h -- C ABI of the B200-native qTask hot path (libqtask_b200.so).
 *
 * Drop-in boundary for the reference's data-parallel core:
 * the reference has no FFI; its hot path sits behind the C++ class
 * qtask::Simulator (/root/reference/proj/include/qtask/engine.hpp:46-151),
 * whose private kernels run_permute_tasks / run_mxv_partition
 * (engine.hpp:129-135, engine.cpp:315-383) and scheduler TaskPool
 * (executor.hpp:18-48) this library replaces.  Two layers are exported:
 *
 *  1. qt_state_*  -- a device-resident 2^n complex128 state vector and
 *     stateless gate application (the replacement for the two CPU kernels
 *     plus the COW block stores, engine.hpp:18-29).
 *  2. qt_sim_*    -- the incremental simulator with the reference's
 *     programming model (modifiers, update_state, readout), one entry point
 *     per public member of qtask::Simulator. include/qtask/engine.hpp wraps
 *     these in the reference's C++ API and exception types.
 *
 * Conventions: index bit t <-> qubit t; amplitudes are
 * interleaved (re, im) doubles, bit-compatible with std::complex<double>.
 * Every function returns QT_OK (0) or a negative QT_ERR_* code; the message
 * of the last failure on the calling thread is qt_last_error().
 * Handles are single-writer (engine.hpp:41-45): one host thread at a time.
 */
#ifndef QTASK_C_H_
#define QTASK_C_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: one per reference exception type (types.hpp:21-64) -- */
#define QT_OK 0
#define QT_ERR_ARG (-1)              /* qtask::Error                      */
#define QT_ERR_NET_CONFLICT (-2)     /* qtask::NetConflictError           */
#define QT_ERR_UNKNOWN_NET (-3)      /* qtask::UnknownNetError            */
#define QT_ERR_UNKNOWN_GATE (-4)     /* qtask::UnknownGateError           */
#define QT_ERR_BAD_QUBIT (-5)        /* qtask::BadQubitError              */
#define QT_ERR_INVALID_POSITION (-6) /* qtask::InvalidPositionError       */
#define QT_ERR_STALE_STATE (-7)      /* qtask::StaleStateError            */
#define QT_ERR_NUMERIC (-8)          /* qtask::NumericError               */
#define QT_ERR_SUPERPOSITION (-9)    /* qtask::SuperpositionGateError     */
#define QT_ERR_QASM_PARSE (-10)      /* qtask::qasm::ParseError           */
#define QT_ERR_QASM_UNSUPPORTED (-11) /* qtask::qasm::UnsupportedGateError */
#define QT_ERR_CUDA (-20)            /* CUDA runtime failure              */
#define QT_ERR_OOM (-21)             /* device allocation failed          */
#define QT_ERR_NCCL (-22)            /* NCCL failure                      */
#define QT_ERR_NO_DEVICE (-23)       /* no CUDA device visible            */

/* ---- gate kinds: reference GateKind order (gate.hpp:13-27) + additive -- */
enum qt_gate_kind {
  QT_CNOT = 0, QT_X = 1, QT_Y = 2, QT_Z = 3, QT_H = 4, QT_S = 5, QT_SDG = 6,
  QT_T = 7, QT_TDG = 8, QT_RX = 9, QT_RY = 10, QT_RZ = 11, QT_SWAP = 12,
  /* additive; same phase convention as their lowering: */
  QT_U3 = 13, /* == RZ(phi) * RY(theta) * RZ(lambda)  (time order RZ(l),RY,RZ(p)) */
  QT_CZ = 14  /* == H(t) CX(c->t) H(t) = diag(1,1,1,-1)                         */
};

/* One gate. Reference Gate record (circuit.hpp:14-21) as POD:
 * control is -1 for 1-qubit kinds; for CNOT/CZ it is the control qubit, for
 * SWAP the second swapped qubit. theta is the rotation angle of RX/RY/RZ;
 * U3 uses (theta, phi, lambda). 40 bytes. */
typedef struct qt_gate {
  int32_t kind;
  int32_t target;
  int32_t control;
  int32_t reserved; /* must be 0 */
  double theta;
  double phi;
  double lambda;
} qt_gate;

/* Engine configuration. The first two fields are the reference Config
 * (plan.hpp:17-20: power-of-two block_size >= 2, threads 0 = auto); on the
 * GPU block_size is the partition-block granularity of UpdateStats and
 * threads is accepted and ignored. The rest are GPU knobs (0 = auto). */
typedef struct qt_config {
  uint64_t block_size;
  uint32_t threads;
  int32_t device;            /* CUDA ordinal; -1 = current device          */
  int32_t tile_qubits;       /* qubits per shared-memory tile (0 = auto)   */
  int32_t max_checkpoints;   /* incremental checkpoint slots (0 = auto)    */
  double checkpoint_fraction;/* share of free HBM for checkpoints (0=auto) */
  int32_t segment_gates;     /* gates per checkpoint segment (0 = auto)    */
  int32_t compiled;          /* 1: compile each tile pass into its own
                                straight-line kernel (NVRTC, cached by
                                pass), for circuits run more than once;
                                2: hybrid -- cached passes run compiled,
                                the others on the interpreter kernel while
                                they compile in the background. qt_state:
                                0 = interpreter. qt_sim: 0 = hybrid (its
                                re-simulated segments repeat), -1 =
                                interpreter only                            */
  int32_t partition_model;   /* qt_sim: the reference-unit partition model
                                (UpdateStats in partitions / blocks, stage
                                views, graph): 0 = auto (states of <= 1024
                                partition blocks), 1 = on, -1 = off         */
  int32_t reserved;
} qt_config;

/* Result of the last qt_apply / update (UpdateStats, engine.hpp:32-39, in
 * GPU terms plus the bytes the roofline is computed from). */
typedef struct qt_run_stats {
  int32_t full;                 /* reference UpdateStats::full             */
  int32_t reserved0;
  uint64_t executed_partitions; /* partition blocks rewritten (ref. sem.)  */
  uint64_t rewritten_amplitudes;/* amplitudes rewritten                    */
  uint64_t gates;               /* gates applied (after lowering)          */
  uint64_t passes;              /* fused tile passes launched              */
  uint64_t kernel_launches;     /* all kernels launched by the call        */
  uint64_t hbm_bytes;           /* algorithmic bytes: 16 B*(R+W) per pass  */
  uint64_t exchanged_bytes;     /* bytes sent over the interconnect        */
  uint64_t swaps;               /* global<->local qubit exchanges          */
  uint64_t restart_gate;        /* first gate re-simulated (incremental)   */
  uint64_t segments;            /* checkpoint segments executed            */
  double device_ms;             /* device time of the call (CUDA events)   */
  double plan_ms;               /* host planning time                      */
  uint64_t exchange_local_bytes;/* local HBM bytes the exchanges copied    */
  uint64_t fused_exchanges;     /* exchanges done by the pass before them
                                   (stores straight into peer memory)     */
} qt_run_stats;

const char* qt_last_error(void);
int qt_device_count(int* out);
/* Library version string, e.g. "qtask-b200 0.1 sm_100a". */
const char* qt_version(void);

/* ======================================================================= */
/* 1. State vector: stateless gate application                             */
/* ======================================================================= */
typedef struct qt_state qt_state;

/* |0...0> on one GPU. cfg may be NULL. n in [1, 40] (no n <= 30 cap,
 * circuit.cpp:9-11 is lifted; limited by HBM). */
int qt_state_create(int num_qubits, const qt_config* cfg, qt_state** out);
/* One shard of a state sharded on its top log2(world) qubits across
 * `world` ranks (one process per GPU). nccl_id is the 128-byte
 * ncclUniqueId made by qt_nccl_unique_id on rank 0 and broadcast by the
 * caller. */
int qt_state_create_sharded(int num_qubits, int rank, int world,
                            const void* nccl_id, const qt_config* cfg,
                            qt_state** out);
/* An in-process group of `world` emulated ranks (power of two): each rank
 * is a qt_state made by qt_state_create_group and driven by its own host
 * thread; the ranks' exchanges are rendezvous of those threads with the data
 * moved by device-to-device copies ordered by CUDA events (qt_comm.hpp
 * LocalComm). Same kernels, rank offsets, exchange schedule and norm combine
 * as qt_state_create_sharded, on one GPU (or several GPUs of one process).
 * The group must outlive its states. */
typedef struct qt_group qt_group;
int qt_group_create(int world, qt_group** out);
int qt_group_destroy(qt_group* g);
int qt_state_create_group(int num_qubits, qt_group* group, int rank,
                          const qt_config* cfg, qt_state** out);
/* `shards` emulated ranks held as slices of one GPU's memory, exchanged
 * with device copies -- exercises the sharded scheduler bit-exactly on
 * one GPU ("loopback comm backend"). */
int qt_state_create_loopback(int num_qubits, int shards,
                             const qt_config* cfg, qt_state** out);
int qt_nccl_unique_id(void* out128);
int qt_state_destroy(qt_state* st);

int qt_state_num_qubits(const qt_state* st);
/* Sets |index> (logical basis index). */
int qt_set_basis(qt_state* st, uint64_t index);
/* Writes / reads amplitudes [first, first+count) in logical index order,
 * interleaved doubles, host memory. Reads synchronise. Sharded states read
 * and write only the amplitudes this rank owns when `count` spans other
 * ranks' ranges, unless the loopback backend holds them all. */
int qt_write(qt_state* st, uint64_t first, uint64_t count,
             const double* interleaved);
int qt_read(qt_state* st, uint64_t first, uint64_t count, double* interleaved);
/* Applies gates in order. The array is copied; stream-ordered (returns
 * before the device finishes). Fails with QT_ERR_NUMERIC at the next
 * synchronising call if an amplitude became non-finite. */
int qt_apply(qt_state* st, const qt_gate* gates, size_t count);
/* Sum |a|^2 by a deterministic tree reduction (fixed order, bit-stable
 * across runs); sharded: fixed-order combine over ranks. */
int qt_norm_squared(qt_state* st, double* out);
/* Top-K readout (the reference's amplitude report, qtask_cli.cpp:53-86):
 * the min(k, 2^n) amplitudes of largest |a|^2 (std::norm; ties: smaller
 * index first), sorted, with their logical indices -- selected on the
 * device, only k records cross PCIe. *count = records written.
 * Sharded states: collective -- every rank selects the k largest of its
 * shard (read in logical-index order, so ties break as on one GPU), the
 * ranks all-gather their records and each merges the same global list. */
int qt_top_k(qt_state* st, uint64_t k, uint64_t* indices, double* amps_interleaved,
             uint64_t* count);
int qt_sync(qt_state* st);
int qt_last_stats(const qt_state* st, qt_run_stats* out);
/* Device-resident checkpoint slots (HBM copies of the state). */
int qt_checkpoint_save(qt_state* st, int slot);
int qt_checkpoint_restore(qt_state* st, int slot);
/* Pass plan of a gate list for this state as JSON (per pass: tile qubits,
 * rounds, ops, R/W amplitudes) for roofline auditing. Writes at most cap
 * bytes (NUL-terminated); *needed gets the full size. Host-only. */
int qt_plan_json(const qt_state* st, const qt_gate* gates, size_t count,
                 char* buf, size_t cap, size_t* needed);

/* Host-only planner probe (no device needed): plans `gates` for an n-qubit
 * state with `global_qubits` sharded bits and writes the JSON plan. */
int qt_plan_probe(int num_qubits, int global_qubits, int tile_qubits,
                  const qt_gate* gates, size_t count, char* buf, size_t cap,
                  size_t* needed);

/* Compiled-pass probe (no device needed): plans `gates` for a one-GPU state
 * of num_qubits (tile / register / low-bit settings, 0 = defaults), lowers
 * every tile pass and generates its compiled kernel; compile != 0 also runs
 * NVRTC on each. JSON {"passes","lowered","source_bytes","compiled",
 * "compile_ms","cubin_bytes"}; source_pass >= 0 returns that pass's CUDA
 * source instead, source_pass == -2 the lowered layer words of every pass
 * (JSON; tests/emulator.py replays them). */
int qt_jit_probe(int num_qubits, int tile_qubits, int reg_bits, int low_bits,
                 int compile, int source_pass, const qt_gate* gates,
                 size_t count, char* buf, size_t cap, size_t* needed);
/* Process-wide compiled-pass statistics (qt_config.compiled states): passes
 * compiled, compile-cache hits, total NVRTC + load milliseconds. */
int qt_jit_stats(uint64_t* compiled, uint64_t* cache_hits, double* compile_ms);
/* Persistent cubin cache ($QTB_JIT_CACHE_DIR, default ~/.cache/qtask_b200;
 * "off" disables): compiled passes found on disk (no NVRTC run) and entries
 * written by this process. */
int qt_jit_disk_stats(uint64_t* disk_hits, uint64_t* disk_writes);
/* Passes queued or compiling in the background (hybrid mode). */
int qt_jit_pending(uint64_t* pending);

/* ======================================================================= */
/* 2. Incremental simulator: qtask::Simulator (engine.hpp:46-100)          */
/* ======================================================================= */
typedef struct qt_sim qt_sim;

int qt_sim_create(int num_qubits, const qt_config* cfg, qt_sim** out);
int qt_sim_destroy(qt_sim* sim);
int qt_sim_num_qubits(const qt_sim* sim);
/* Effective block size (plan.hpp:26-35) and block count. */
uint64_t qt_sim_block_size(const qt_sim* sim);
uint64_t qt_sim_total_blocks(const qt_sim* sim);

/* Modifiers (engine.hpp:57-64). Net and gate ids are never reused; 0 is
 * "none" (types.hpp:13-18). */
int qt_sim_insert_net_front(qt_sim* sim, uint32_t* net);
int qt_sim_insert_net_back(qt_sim* sim, uint32_t* net);
int qt_sim_insert_net_after(qt_sim* sim, uint32_t after, uint32_t* net);
int qt_sim_remove_net(qt_sim* sim, uint32_t net);
/* control = -1 for 1-qubit kinds. params = (theta, phi, lambda) or NULL. */
int qt_sim_insert_gate(qt_sim* sim, int kind, const double* params,
                       uint32_t net, int target, int control, uint32_t* gate);
int qt_sim_remove_gate(qt_sim* sim, uint32_t gate);

/* engine.hpp:71. First call simulates everything; later calls re-simulate
 * from the last valid device checkpoint at or before the earliest edit. */
int qt_sim_update_state(qt_sim* sim);
int qt_sim_pending(const qt_sim* sim); /* 1 if modifiers are pending */

/* Queries (engine.hpp:77-80): QT_ERR_STALE_STATE while modifiers pend. */
int qt_sim_amplitude(qt_sim* sim, uint64_t index, double* out2);
int qt_sim_amplitudes(qt_sim* sim, uint64_t first, uint64_t last,
                      double* interleaved);
int qt_sim_norm_squared(qt_sim* sim, double* out);
/* qt_top_k on the simulator's committed state (QT_ERR_STALE_STATE while
 * modifiers pend, like amplitude queries). */
int qt_sim_top_k(qt_sim* sim, uint64_t k, uint64_t* indices, double* amps_interleaved,
                 uint64_t* count);
int qt_sim_last_update(const qt_sim* sim, qt_run_stats* out);

/* Circuit introspection (Circuit, circuit.hpp:32-66): counts and the
 * flattened gate list in simulation order (nets in order, gates in
 * insertion order within a net). */
size_t qt_sim_num_gates(const qt_sim* sim);
size_t qt_sim_num_nets(const qt_sim* sim);
int qt_sim_net_order(const qt_sim* sim, uint32_t* out, size_t cap);
int qt_sim_net_gates(const qt_sim* sim, uint32_t net, uint32_t* out,
                     size_t cap, size_t* count);
int qt_sim_gate_info(const qt_sim* sim, uint32_t gate, qt_gate* out,
                     uint32_t* net);
int qt_sim_export_gates(const qt_sim* sim, qt_gate* out, size_t cap,
                        size_t* count);

/* ---- reference-unit partition model (qt_config.partition_model) ----------
 * The reference's partition DAG restated on the host from the modifier
 * stream (csrc/qt_partition.hpp): UpdateStats in partition / block units
 * (engine.hpp:32-39) and the introspection members (engine.hpp:77-100).
 * valid = 0 when the model is off for this simulator. */
typedef struct qt_update_account {
  int32_t valid;
  int32_t full;
  uint64_t executed_partitions;
  uint64_t materialized_blocks;
  uint64_t rewritten_amplitudes;
  uint64_t rewritten_block_count;
} qt_update_account;
/* The last update's accounting; up to `cap` rewritten block indices (sorted)
 * into `blocks` (may be NULL). */
int qt_sim_update_account(qt_sim* sim, qt_update_account* out, uint64_t* blocks, size_t cap);

typedef struct qt_model_stage {
  uint32_t id, net, gate;
  int32_t kind;          /* 0 Sync, 1 MatrixVector, 2 PermuteScale */
  uint64_t first_part;   /* into the partition array */
  uint64_t num_parts;
} qt_model_stage;
typedef struct qt_model_part {
  uint64_t first_block, last_block;  /* inclusive */
  uint64_t node;                     /* graph node id */
  uint64_t first_task, num_tasks;    /* into the task array */
} qt_model_part;
typedef struct qt_model_task {
  uint64_t first_op, last_op, region_lo, region_hi;  /* inclusive */
} qt_model_task;
typedef struct qt_model_sizes {
  int32_t valid;
  int32_t reserved;
  uint64_t stages, parts, tasks, edges, blocks, frontiers;
} qt_model_sizes;
/* Snapshot of the model: stages in execution order, their partitions and
 * tasks, the graph's edges as (from, to) node pairs sorted, each stage's
 * materialised blocks (stages x blocks bytes, row-major) and the frontier
 * nodes. Call with NULL arrays for the sizes, then with arrays that large. */
int qt_sim_model_snapshot(qt_sim* sim, qt_model_sizes* sizes, qt_model_stage* stages,
                          qt_model_part* parts, qt_model_task* tasks, uint64_t* edges,
                          uint8_t* materialized, uint64_t* frontiers);
/* Reference node names (engine.cpp:570-586) and the DOT dump (graph.cpp:
 * 302-327); two-call pattern on `needed`. */
int qt_sim_node_name(qt_sim* sim, uint64_t node, char* buf, size_t cap, size_t* needed);
int qt_sim_dump_graph(qt_sim* sim, char* buf, size_t cap, size_t* needed);
/* The reference gate database (gate.cpp:42-106): the dense matrix (dim 2 or
 * 4, row-major, interleaved re/im into m[2*dim*dim]) and the classification
 * (1 = superposition). */
int qt_gate_matrix(int kind, double theta, double phi, double lambda, double* m, int* dim);
int qt_classify_gate(int kind, double theta, double phi, double lambda);

/* Host-only handle on the partition model alone (no device): the same
 * restatement qt_sim runs, driven directly with modifier events whose ids
 * and validity the caller guarantees -- for differential tests against the
 * reference engine. where: 0 = front, 1 = back, 2 = after `after`. */
typedef struct qt_pm qt_pm;
int qt_pm_create(int num_qubits, uint64_t block_size, qt_pm** out);
int qt_pm_destroy(qt_pm* pm);
int qt_pm_insert_net(qt_pm* pm, uint32_t net, int where, uint32_t after);
int qt_pm_remove_net(qt_pm* pm, uint32_t net);
int qt_pm_insert_gate(qt_pm* pm, uint32_t gate, const qt_gate* g, uint32_t net);
int qt_pm_remove_gate(qt_pm* pm, uint32_t gate);
int qt_pm_update(qt_pm* pm);
int qt_pm_account(qt_pm* pm, qt_update_account* out, uint64_t* blocks, size_t cap);
int qt_pm_dump_graph(qt_pm* pm, char* buf, size_t cap, size_t* needed);

/* Host-only audit of a sharded exchange (State::exchange): the grouped
 * send/recv steps `rank` performs to swap the k global rank bits gbit[j]
 * (0-based above the local bits) with local victim bits vbit[j], for an
 * exchange buffer of tmp_amps amplitudes. Rows of 4 uint64: step, peer,
 * send offset (amplitudes into the shard), receive offset (into the buffer);
 * *piece = amplitudes per row. Call with cap 0 to size. */
int qt_exchange_schedule(int rank, int nlocal, int k, const int* gbit, const int* vbit,
                         uint64_t tmp_amps, uint64_t* rows, size_t cap, size_t* count,
                         uint64_t* piece);

/* Host-only audit of a fused exchange (the compiled pass in front of an
 * exchange stores straight into the peers' buffers): for `rank` and the k
 * pairs (global bit gbit[j] above the local bits, local victim bit vbit[j]),
 * peer_rank[v] (2^k entries) = the rank that receives the amplitudes whose
 * victim bits spell v, *rfix = the bits set at the victim positions of the
 * index they land at: local index x -> (x with the victim bits cleared) | rfix. */
int qt_fused_exchange_map(int rank, int nlocal, int k, const int* gbit, const int* vbit,
                          int* peer_rank, uint64_t* rfix);

/* Host-only audit of the circuit's net order index (csrc/qt_netindex.hpp, the
 * O(log nets) replacement of the list walks of circuit.cpp:67-120): drives
 * `ops` seeded random net inserts / removals and gate-count changes into the
 * index and into a plain array, comparing rank, gates-before, net-at-position
 * and the order after every step. *mismatches = failed comparisons. */
int qt_netindex_audit(uint64_t seed, uint32_t ops, uint64_t* mismatches);

/* ---- OpenQASM 2.0 front end (reference qasm.hpp:11-66, qasm.cpp:34-426) --
 * Same accepted subset, errors (line / column of the offending token) and
 * ASAP levelling as the reference; implementation: include/qtask/qasm.hpp. */
typedef struct qt_qasm_stmt {
  int32_t kind;      /* 0 gate, 1 barrier */
  int32_t gate;      /* qt_gate_kind (gates only) */
  double theta;      /* rx / ry / rz angle */
  int32_t has_theta;
  int32_t nqubits;   /* operands: cx = control, target; swap = target, control */
  int32_t qubits[2];
  int32_t line, column;
  int32_t level;     /* ASAP level (levelize), -1 for barriers */
  int32_t reserved;
} qt_qasm_stmt;

/* Parses `len` bytes of QASM text. On success *count statements (up to cap
 * are written; call with cap 0 to size), *num_qubits the qreg size. On
 * QT_ERR_QASM_PARSE / QT_ERR_QASM_UNSUPPORTED, *err_line / *err_col locate
 * the offending token. */
int qt_qasm_parse(const char* text, size_t len, qt_qasm_stmt* out, size_t cap,
                  size_t* count, uint32_t* num_qubits, int* err_line,
                  int* err_col);
/* build_circuit (qasm.cpp:407-426): parses `text` and appends one net per ASAP
 * level to `sim` (qt_sim_create'd with at least the qreg size). */
int qt_qasm_build(qt_sim* sim, const char* text, size_t len, int* err_line,
                  int* err_col);

#ifdef __cplusplus
}
#endif

#endif /* QTASK_C_H_ */
