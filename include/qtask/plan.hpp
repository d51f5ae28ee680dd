// qtask/plan.hpp -- drop-in for the reference's planning types (reference
// proj/include/qtask/plan.hpp:17-71): Config, the block arithmetic, and the
// task / partition / stage-kind records the partition introspection reports.
// On the B200 engine the partitions are accounting units of the host
// partition model (csrc/qt_partition.hpp); the device runs fused tile passes.
#pragma once

#include <cstdint>
#include <vector>

#include "qtask/types.hpp"

namespace qtask {

/// Reference Config (plan.hpp:17-20) + GPU knobs (0 = auto). Aggregate-init
/// compatible with the reference's Config{block_size, threads}.
struct Config {
  std::uint64_t block_size = 256;
  unsigned threads = 0;
  int device = -1;
  int tile_qubits = 0;
  int max_checkpoints = 0;
  double checkpoint_fraction = 0.0;
  int segment_gates = 0;
  int compiled = 0;         // 0: hybrid compiled passes (NVRTC, cached segments), -1: interpreter only
  int partition_model = 0;  // reference-unit accounting / introspection: 0 auto (<= 1024 blocks), 1 on, -1 off
};

/// block_size must be a power of two >= 2 (plan.cpp:7-13).
inline void validate_config(const Config& cfg) {
  if (cfg.block_size < 2 || (cfg.block_size & (cfg.block_size - 1)) != 0)
    throw Error("block size must be a power of two >= 2");
}

/// Blocks never exceed the state vector (plan.hpp:26-35).
inline std::uint64_t effective_block_size(int num_qubits, std::uint64_t block_size) {
  const std::uint64_t dim = std::uint64_t{1} << num_qubits;
  return block_size < dim ? block_size : dim;
}

inline std::uint64_t num_blocks(int num_qubits, std::uint64_t block_size) {
  return (std::uint64_t{1} << num_qubits) / effective_block_size(num_qubits, block_size);
}

/// A run of consecutive element ops (or matrix rows) and the inclusive hull
/// of the state indices it touches (plan.hpp:39-44).
struct TaskSpec {
  std::uint64_t first_op = 0;
  std::uint64_t last_op = 0;
  std::uint64_t region_lo = 0;
  std::uint64_t region_hi = 0;
};

/// A node of the partition graph: chain-overlapping tasks of one stage and
/// their inclusive block range (plan.hpp:48-52).
struct PartitionSpec {
  std::uint64_t first_block = 0;
  std::uint64_t last_block = 0;
  std::vector<TaskSpec> tasks;
};

enum class StageKind { Sync, MatrixVector, PermuteScale };

}  // namespace qtask
