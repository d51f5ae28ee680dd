// qt_comm.cpp -- transports for global<->local qubit exchanges: NCCL over
// NVLink, and an in-process group of emulated ranks (qt_comm.hpp).
//
// The reference is single-process (executor.hpp:40-47); sharding the state
// on its top qubits across GPUs is new in this build.
// NCCL is resolved with dlopen so the library has no link-time NCCL
// dependency and picks up the libnccl.so.2 torch already loaded.
#include "qt_comm.hpp"

#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstring>

namespace qtb {

namespace {
// ABI subset of nccl.h (stable across NCCL 2.x)
using ncclResult_t = int;
using ncclComm_t = void*;
struct ncclUniqueId {
  char internal[128];
};
constexpr int ncclUint8 = 1;
constexpr int ncclFloat64 = 8;
}  // namespace

struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi* load_api(std::string* err) {
  static NcclApi api;
  static bool tried = false, ok = false;
  if (tried) {
    if (!ok && err) *err = "libnccl.so.2 unavailable";
    return ok ? &api : nullptr;
  }
  tried = true;
  api.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!api.h) api.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!api.h) {
    if (err) *err = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
    return nullptr;
  }
#define QT_SYM(field, name)                                              \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(api.h, name)); \
  if (!api.field) {                                                      \
    if (err) *err = std::string("missing NCCL symbol ") + name;          \
    return nullptr;                                                      \
  }
  QT_SYM(GetUniqueId, "ncclGetUniqueId");
  QT_SYM(CommInitRank, "ncclCommInitRank");
  QT_SYM(CommDestroy, "ncclCommDestroy");
  QT_SYM(Send, "ncclSend");
  QT_SYM(Recv, "ncclRecv");
  QT_SYM(GroupStart, "ncclGroupStart");
  QT_SYM(GroupEnd, "ncclGroupEnd");
  QT_SYM(AllGather, "ncclAllGather");
  QT_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
  QT_SYM(GetErrorString, "ncclGetErrorString");
#undef QT_SYM
  ok = true;
  return &api;
}

static bool nccl_ok(NcclApi* api, ncclResult_t r, const char* what,
                    std::string* err) {
  if (r == 0) return true;
  if (err) *err = std::string(what) + ": " + api->GetErrorString(r);
  return false;
}

bool NcclComm::unique_id(void* out128, std::string* err) {
  NcclApi* api = load_api(err);
  if (!api) return false;
  ncclUniqueId id;
  if (!nccl_ok(api, api->GetUniqueId(&id), "ncclGetUniqueId", err)) return false;
  std::memcpy(out128, id.internal, 128);
  return true;
}

NcclComm* NcclComm::create(const void* unique_id, int rank, int world, int device,
                           std::string* err) {
  NcclApi* api = load_api(err);
  if (!api) return nullptr;
  if (cudaSetDevice(device) != cudaSuccess) {
    if (err) *err = "cudaSetDevice failed";
    return nullptr;
  }
  ncclUniqueId id;
  std::memcpy(id.internal, unique_id, 128);
  ncclComm_t c = nullptr;
  if (!nccl_ok(api, api->CommInitRank(&c, world, id, rank), "ncclCommInitRank",
               err))
    return nullptr;
  NcclComm* cm = new NcclComm();
  cm->api_ = api;
  cm->comm_ = c;
  cm->rank_ = rank;
  cm->world_ = world;
  return cm;
}

NcclComm::~NcclComm() {
  if (api_ && comm_) api_->CommDestroy(comm_);
}

bool NcclComm::sendrecv(int npeers, const int* peers, const void* const* sends,
                        void* const* recvs, size_t bytes, cudaStream_t s,
                        std::string* err) {
  if (!nccl_ok(api_, api_->GroupStart(), "ncclGroupStart", err)) return false;
  for (int i = 0; i < npeers; ++i) {
    if (!nccl_ok(api_, api_->Send(sends[i], bytes, ncclUint8, peers[i], comm_, s),
                 "ncclSend", err) ||
        !nccl_ok(api_, api_->Recv(recvs[i], bytes, ncclUint8, peers[i], comm_, s),
                 "ncclRecv", err)) {
      api_->GroupEnd();
      return false;
    }
  }
  return nccl_ok(api_, api_->GroupEnd(), "ncclGroupEnd", err);
}

bool NcclComm::allgather_double(const double* in, double* out, size_t count, cudaStream_t s,
                                std::string* err) {
  return nccl_ok(api_, api_->AllGather(in, out, count, ncclFloat64, comm_, s),
                 "ncclAllGather", err);
}

bool NcclComm::check_async(std::string* err) {
  ncclResult_t r = 0;
  api_->CommGetAsyncError(comm_, &r);
  return nccl_ok(api_, r, "NCCL async error", err);
}

// ---- in-process group ------------------------------------------------------

namespace {
constexpr auto kRendezvousTimeout = std::chrono::seconds(600);
}

LocalGroup::LocalGroup(int world) : world_(world), slots_(world) {}

LocalGroup::~LocalGroup() {
  for (Slot& sl : slots_) {
    if (sl.device >= 0) cudaSetDevice(sl.device);
    if (sl.ready) cudaEventDestroy(sl.ready);
    if (sl.read) cudaEventDestroy(sl.read);
  }
}

LocalComm::LocalComm(std::shared_ptr<LocalGroup> g, int rank, int device) : g_(std::move(g)) {
  rank_ = rank;
  world_ = g_->world();
  LocalGroup::Slot& me = g_->slots_[rank];
  me.device = device;
  me.send_to.assign(world_, {});
  cudaEventCreateWithFlags(&me.ready, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&me.read, cudaEventDisableTiming);
}

LocalComm::~LocalComm() = default;

template <typename Copy>
bool LocalComm::rendezvous(const std::vector<int>& peers, cudaStream_t s, Copy copy,
                           std::string* err) {
  LocalGroup& g = *g_;
  LocalGroup::Slot& me = g.slots_[rank_];
  uint64_t seq = 0;
  {
    std::unique_lock<std::mutex> lk(g.mu_);
    if (cudaEventRecord(me.ready, s) != cudaSuccess) {
      if (err) *err = "local transport: event record failed";
      return false;
    }
    seq = ++me.seq;
    g.cv_.notify_all();
    const bool ok = g.cv_.wait_for(lk, kRendezvousTimeout, [&] {
      if (g.broken_) return true;
      for (int p : peers)
        if (g.slots_[p].seq < seq) return false;
      return true;
    });
    if (g.broken_) {
      if (err) *err = "local transport: a peer rank failed: " + g.why_;
      return false;
    }
    if (!ok) {
      if (err) *err = "local transport: a peer rank never reached the exchange";
      return false;
    }
  }
  // the peers' sends are ready (stream order) and stay untouched until they
  // pass the read barrier below, which waits for this rank's reads
  for (int p : peers)
    if (p != rank_) cudaStreamWaitEvent(s, g.slots_[p].ready, 0);
  if (!copy()) {
    if (err) *err = "local transport: device copy failed";
    return false;
  }
  {
    std::unique_lock<std::mutex> lk(g.mu_);
    cudaEventRecord(me.read, s);
    me.read_seq = seq;
    g.cv_.notify_all();
    const bool ok = g.cv_.wait_for(lk, kRendezvousTimeout, [&] {
      if (g.broken_) return true;
      for (int p : peers)
        if (g.slots_[p].read_seq < seq) return false;
      return true;
    });
    if (g.broken_) {
      if (err) *err = "local transport: a peer rank failed: " + g.why_;
      return false;
    }
    if (!ok) {
      if (err) *err = "local transport: a peer rank never finished the exchange";
      return false;
    }
  }
  for (int p : peers)
    if (p != rank_) cudaStreamWaitEvent(s, g.slots_[p].read, 0);
  return true;
}

void LocalComm::abort(const std::string& why) {
  std::lock_guard<std::mutex> lk(g_->mu_);
  if (!g_->broken_) {
    g_->broken_ = true;
    g_->why_ = "rank " + std::to_string(rank_) + ": " + why;
  }
  g_->cv_.notify_all();
}

bool LocalComm::sendrecv(int npeers, const int* peers, const void* const* sends,
                         void* const* recvs, size_t bytes, cudaStream_t s, std::string* err) {
  LocalGroup::Slot& me = g_->slots_[rank_];
  std::vector<int> pv;
  {
    std::lock_guard<std::mutex> lk(g_->mu_);
    for (auto& v : me.send_to) v.clear();
    for (int i = 0; i < npeers; ++i) {
      me.send_to[peers[i]].push_back(sends[i]);
      if (std::find(pv.begin(), pv.end(), peers[i]) == pv.end()) pv.push_back(peers[i]);
    }
  }
  return rendezvous(pv, s, [&] {
    std::vector<size_t> next(world_, 0);
    for (int i = 0; i < npeers; ++i) {
      const std::vector<const void*>& from = g_->slots_[peers[i]].send_to[rank_];
      const size_t j = next[peers[i]]++;
      if (j >= from.size()) return false;  // the peer sends fewer pieces
      if (cudaMemcpyAsync(recvs[i], from[j], bytes, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return false;
    }
    return true;
  }, err);
}

bool LocalComm::with_peer_buffers(void* mine, const std::vector<int>& peers, cudaStream_t s,
                                  const std::function<bool(void* const* table)>& launch,
                                  std::string* err) {
  {
    std::lock_guard<std::mutex> lk(g_->mu_);
    g_->slots_[rank_].peer_buf = mine;
  }
  return rendezvous(peers, s, [&] {
    std::vector<void*> table(world_, nullptr);
    {
      std::lock_guard<std::mutex> lk(g_->mu_);
      for (int p : peers) table[p] = g_->slots_[p].peer_buf;
    }
    return launch(table.data());
  }, err);
}

bool LocalComm::allgather_double(const double* in, double* out, size_t count, cudaStream_t s,
                                 std::string* err) {
  LocalGroup::Slot& me = g_->slots_[rank_];
  std::vector<int> all(world_);
  for (int r = 0; r < world_; ++r) all[r] = r;
  {
    std::lock_guard<std::mutex> lk(g_->mu_);
    me.gather_src = in;
  }
  return rendezvous(all, s, [&] {
    for (int r = 0; r < world_; ++r)
      if (cudaMemcpyAsync(out + r * count, g_->slots_[r].gather_src, sizeof(double) * count,
                          cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return false;
    return true;
  }, err);
}

}  // namespace qtb
