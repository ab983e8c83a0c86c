#include "comm.hpp"

#include <dlfcn.h>

#include <string>

namespace moa {

namespace {

// Minimal NCCL ABI (stable since 2.x): opaque communicator, 128-byte id.
using ncclResult = int;
struct NcclId {
  char internal[kNcclIdBytes];
};
constexpr int kNcclInt32 = 2, kNcclFloat32 = 7;

struct NcclApi {
  ncclResult (*get_unique_id)(NcclId*) = nullptr;
  ncclResult (*comm_init_rank)(void**, int, NcclId, int) = nullptr;
  ncclResult (*comm_destroy)(void*) = nullptr;
  ncclResult (*send)(const void*, std::size_t, int, int, void*, cudaStream_t) = nullptr;
  ncclResult (*recv)(void*, std::size_t, int, int, void*, cudaStream_t) = nullptr;
  ncclResult (*group_start)() = nullptr;
  ncclResult (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static bool loaded = false;
  if (loaded) return api;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) throw DeviceError(std::string("nccl: cannot load libnccl.so.2: ") + dlerror());
  auto sym = [&](const char* name) {
    void* p = dlsym(h, name);
    if (!p) throw DeviceError(std::string("nccl: missing symbol ") + name);
    return p;
  };
  api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
  api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
  api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
  api.send = reinterpret_cast<decltype(api.send)>(sym("ncclSend"));
  api.recv = reinterpret_cast<decltype(api.recv)>(sym("ncclRecv"));
  api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
  api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
  api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
  loaded = true;
  return api;
}

void check(ncclResult r, const char* what) {
  if (r != 0) throw DeviceError(std::string("nccl: ") + what + ": " + nccl().error_string(r));
}

}  // namespace

PeerComm::PeerComm(int rank, int world) : rank_(rank), world_(world) {
  if (world < 1 || rank < 0 || rank >= world) throw ValidationError("comm: rank must be in [0, world)");
}

// ---- NCCL ----

void NcclComm::unique_id(std::uint8_t* out) {
  NcclId id;
  check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  for (int i = 0; i < kNcclIdBytes; ++i) out[i] = static_cast<std::uint8_t>(id.internal[i]);
}

NcclComm::NcclComm(const std::uint8_t* id, int rank, int world) : PeerComm(rank, world) {
  NcclId nid;
  for (int i = 0; i < kNcclIdBytes; ++i) nid.internal[i] = static_cast<char>(id[i]);
  check(nccl().comm_init_rank(&comm_, world, nid, rank), "ncclCommInitRank");
}

NcclComm::~NcclComm() {
  if (comm_) nccl().comm_destroy(comm_);
}

void NcclComm::begin() { check(nccl().group_start(), "ncclGroupStart"); }
void NcclComm::end() { check(nccl().group_end(), "ncclGroupEnd"); }

namespace {
int nccl_type(int elem) { return elem == PeerComm::kI32 ? kNcclInt32 : kNcclFloat32; }
}  // namespace

void NcclComm::send(const void* buf, long long bytes, int elem, int peer, cudaStream_t st) {
  check(nccl().send(buf, static_cast<std::size_t>(bytes / 4), nccl_type(elem), peer, comm_, st), "ncclSend");
}
void NcclComm::recv(void* buf, long long bytes, int elem, int peer, cudaStream_t st) {
  check(nccl().recv(buf, static_cast<std::size_t>(bytes / 4), nccl_type(elem), peer, comm_, st), "ncclRecv");
}

// ---- in-process loopback ----

LoopbackHub::LoopbackHub(int world)
    : world_(world), q_(static_cast<std::size_t>(world) * world), head_(static_cast<std::size_t>(world) * world, 0) {
  if (world < 1) throw ValidationError("loopback: world must be >= 1");
}

void LoopbackHub::barrier() {
  std::unique_lock<std::mutex> lk(mu_);
  const long long gen = generation_;
  if (++arrived_ == world_) {
    arrived_ = 0;
    ++generation_;
    cv_.notify_all();
  } else {
    cv_.wait(lk, [&] { return generation_ != gen; });
  }
}

void LoopbackHub::post(int from, int to, const Msg& m) {
  std::lock_guard<std::mutex> lk(mu_);
  q_[static_cast<std::size_t>(from) * world_ + to].push_back(m);
}

LoopbackHub::Msg LoopbackHub::take(int from, int to) {
  std::lock_guard<std::mutex> lk(mu_);
  const std::size_t k = static_cast<std::size_t>(from) * world_ + to;
  if (head_[k] >= q_[k].size()) throw RunError("loopback: receive without a matching send");
  Msg m = q_[k][head_[k]++];
  if (head_[k] == q_[k].size()) {
    q_[k].clear();
    head_[k] = 0;
  }
  return m;
}

LoopbackComm::LoopbackComm(std::shared_ptr<LoopbackHub> hub, int rank)
    : PeerComm(rank, hub->world()), hub_(std::move(hub)) {}

void LoopbackComm::begin() {
  if (open_) throw RunError("loopback: nested group");
  open_ = true;
  recvs_.clear();
  streams_.clear();
}

void LoopbackComm::send(const void* buf, long long bytes, int elem, int peer, cudaStream_t st) {
  streams_.push_back(st);
  hub_->post(rank(), peer, {buf, bytes, elem});
}

void LoopbackComm::recv(void* buf, long long bytes, int elem, int peer, cudaStream_t st) {
  streams_.push_back(st);
  recvs_.push_back({buf, bytes, elem, peer});
}

// Every rank of the group calls end() (as with NCCL, where a rank with
// nothing to exchange this tick simply issues no group -- here too: ranks
// exchange only in ticks where some chunk completes, which the replicated
// schedule makes identical on every rank).
void LoopbackComm::end() {
  if (!open_) throw RunError("loopback: end without begin");
  open_ = false;
  for (cudaStream_t st : streams_) MOA_CUDA(cudaStreamSynchronize(st));  // send buffers final
  hub_->barrier();                                                      // all sends posted
  for (const Recv& r : recvs_) {
    const LoopbackHub::Msg m = hub_->take(r.peer, rank());
    if (m.bytes != r.bytes || m.elem != r.elem) throw RunError("loopback: send / receive size or type mismatch");
    MOA_CUDA(cudaMemcpy(r.dst, m.src, static_cast<std::size_t>(r.bytes), cudaMemcpyDefault));
  }
  hub_->barrier();  // senders may reuse their buffers
}

}  // namespace moa
