// qt_comm.hpp -- the transport under a sharded state's exchanges.
//
// Two implementations of one interface (Comm):
//  * NcclComm: NCCL over NVLink / NVSwitch, loaded at run time (dlopen
//    "libnccl.so.2"): the process that created the ncclUniqueId (normally
//    torch.distributed's) and this library share one NCCL; no link-time
//    dependency, so single-GPU use never touches it.
//  * LocalComm: an in-process group of emulated ranks on one device (one
//    State and one host thread per rank): every grouped send / receive is a
//    rendezvous of the participating ranks' host threads, and the data moves
//    as device-to-device copies ordered by CUDA events between the ranks'
//    streams (no kernel ever waits on another). It runs State::exchange's
//    real step loop with the sharded kernels' rank offsets, on one GPU.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <mutex>
#include <functional>
#include <string>
#include <vector>

namespace qtb {

class Comm {
 public:
  virtual ~Comm() = default;
  int rank() const { return rank_; }
  int world() const { return world_; }
  // Grouped point-to-point: sends[i] (bytes) to peers[i] and receives the
  // same byte count from peers[i] into recvs[i], as one group (a peer may
  // appear several times: its sends and receives match in order): on return
  // (stream order) every receive has landed and every send buffer may be
  // overwritten.
  virtual bool sendrecv(int npeers, const int* peers, const void* const* sends,
                        void* const* recvs, size_t bytes, cudaStream_t s,
                        std::string* err) = 0;
  // out[r * count ...] = the count doubles of rank r's in, device buffers
  // (bit patterns travel unchanged: also used for packed integer records).
  virtual bool allgather_double(const double* in, double* out, size_t count, cudaStream_t s,
                                std::string* err) = 0;
  // Peer memory (fused exchanges, qt_state.cpp): true when this rank's kernels
  // can store straight into the other ranks' buffers (in-process group: same
  // device; NCCL ranks live in separate processes and would need an IPC or
  // multicast mapping: not available here, so they keep the send/recv path).
  virtual bool peer_access() const { return false; }
  // Collective over `peers` (this rank included): publishes `mine`, waits
  // (stream order) until every peer's earlier work is done, calls
  // launch(table) with table[r] = rank r's published pointer (nullptr for
  // ranks outside `peers`), then makes the stream wait for every peer's launch.
  virtual bool with_peer_buffers(void* mine, const std::vector<int>& peers, cudaStream_t s,
                                 const std::function<bool(void* const* table)>& launch,
                                 std::string* err) {
    if (err) *err = "transport has no peer access";
    return false;
  }
  virtual bool check_async(std::string* err) = 0;
  virtual const char* kind() const = 0;
  // This rank failed mid-call: release peers waiting on it (in-process
  // group) instead of letting them time out.
  virtual void abort(const std::string& why) {}

 protected:
  int rank_ = 0, world_ = 1;
};

struct NcclApi;

class NcclComm : public Comm {
 public:
  // Returns nullptr and sets *err on failure.
  static NcclComm* create(const void* unique_id, int rank, int world, int device,
                          std::string* err);
  static bool unique_id(void* out128, std::string* err);
  ~NcclComm() override;
  bool sendrecv(int npeers, const int* peers, const void* const* sends, void* const* recvs,
                size_t bytes, cudaStream_t s, std::string* err) override;
  bool allgather_double(const double* in, double* out, size_t count, cudaStream_t s,
                        std::string* err) override;
  bool check_async(std::string* err) override;
  const char* kind() const override { return "nccl"; }

 private:
  NcclComm() = default;
  NcclApi* api_ = nullptr;
  void* comm_ = nullptr;
};

// The shared rendezvous of an in-process group (one per emulated world).
class LocalGroup {
 public:
  explicit LocalGroup(int world);
  ~LocalGroup();
  int world() const { return world_; }

 private:
  friend class LocalComm;
  struct Slot {
    uint64_t seq = 0;        // calls posted by this rank (sendrecv or allgather)
    uint64_t read_seq = 0;   // calls whose reads this rank has issued
    std::vector<std::vector<const void*>> send_to;  // per destination rank, in order (this call)
    const double* gather_src = nullptr;
    void* peer_buf = nullptr;  // with_peer_buffers: this rank's published buffer
    cudaEvent_t ready = nullptr;  // the rank's stream reached the call
    cudaEvent_t read = nullptr;   // the rank's reads of its peers are issued
    int device = -1;
  };
  int world_;
  bool broken_ = false;
  std::string why_;
  std::mutex mu_;
  std::condition_variable cv_;
  std::vector<Slot> slots_;
};

class LocalComm : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalGroup> g, int rank, int device);
  ~LocalComm() override;
  bool sendrecv(int npeers, const int* peers, const void* const* sends, void* const* recvs,
                size_t bytes, cudaStream_t s, std::string* err) override;
  bool allgather_double(const double* in, double* out, size_t count, cudaStream_t s,
                        std::string* err) override;
  bool peer_access() const override { return true; }
  bool with_peer_buffers(void* mine, const std::vector<int>& peers, cudaStream_t s,
                         const std::function<bool(void* const* table)>& launch,
                         std::string* err) override;
  bool check_async(std::string*) override { return true; }
  const char* kind() const override { return "local"; }
  void abort(const std::string& why) override;

 private:
  // posts this rank's call, waits until `peers` posted the same call, makes
  // the stream wait for their ready events; then, after `copy` issued the
  // reads, the same for the read events (so no peer overwrites what is read)
  template <typename Copy>
  bool rendezvous(const std::vector<int>& peers, cudaStream_t s, Copy copy, std::string* err);
  std::shared_ptr<LocalGroup> g_;
};

}  // namespace qtb
