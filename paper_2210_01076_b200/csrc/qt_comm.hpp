// qt_comm.hpp -- NCCL, loaded at run time (dlopen "libnccl.so.2"): the
// process that created the ncclUniqueId (normally torch.distributed's) and
// this library share one NCCL; no link-time dependency, so single-GPU use
// never touches it.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <string>

namespace qtb {

struct NcclApi;

class Comm {
 public:
  // Returns nullptr and sets *err on failure.
  static Comm* create(const void* unique_id, int rank, int world, int device,
                      std::string* err);
  static bool unique_id(void* out128, std::string* err);
  ~Comm();

  int rank() const { return rank_; }
  int world() const { return world_; }

  // Grouped point-to-point: sends[i] (bytes) to peers[i] and receives the
  // same byte count from peers[i] into recvs[i], all in one NCCL group.
  bool sendrecv(int npeers, const int* peers, const void* const* sends,
                void* const* recvs, size_t bytes, cudaStream_t s,
                std::string* err);
  // out[r] = in from rank r (one double each), device buffers.
  bool allgather_double(const double* in, double* out, cudaStream_t s,
                        std::string* err);
  bool check_async(std::string* err);

 private:
  Comm() = default;
  NcclApi* api_ = nullptr;
  void* comm_ = nullptr;
  int rank_ = 0, world_ = 1;
};

}  // namespace qtb
