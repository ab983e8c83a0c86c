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

void PeerComm::unique_id(std::uint8_t* out) {
  NcclId id;
  check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  for (int i = 0; i < kNcclIdBytes; ++i) out[i] = static_cast<std::uint8_t>(id.internal[i]);
}

PeerComm::PeerComm(const std::uint8_t* id, int rank, int world) : rank_(rank), world_(world) {
  if (world < 1 || rank < 0 || rank >= world) throw ValidationError("comm: rank must be in [0, world)");
  NcclId nid;
  for (int i = 0; i < kNcclIdBytes; ++i) nid.internal[i] = static_cast<char>(id[i]);
  check(nccl().comm_init_rank(&comm_, world, nid, rank), "ncclCommInitRank");
}

PeerComm::~PeerComm() {
  if (comm_) nccl().comm_destroy(comm_);
}

void PeerComm::begin() { check(nccl().group_start(), "ncclGroupStart"); }
void PeerComm::end() { check(nccl().group_end(), "ncclGroupEnd"); }

void PeerComm::send_i32(const int* buf, long long n, int peer, cudaStream_t st) {
  check(nccl().send(buf, static_cast<std::size_t>(n), kNcclInt32, peer, comm_, st), "ncclSend");
}
void PeerComm::recv_i32(int* buf, long long n, int peer, cudaStream_t st) {
  check(nccl().recv(buf, static_cast<std::size_t>(n), kNcclInt32, peer, comm_, st), "ncclRecv");
}
void PeerComm::send_f32(const float* buf, long long n, int peer, cudaStream_t st) {
  check(nccl().send(buf, static_cast<std::size_t>(n), kNcclFloat32, peer, comm_, st), "ncclSend");
}
void PeerComm::recv_f32(float* buf, long long n, int peer, cudaStream_t st) {
  check(nccl().recv(buf, static_cast<std::size_t>(n), kNcclFloat32, peer, comm_, st), "ncclRecv");
}

}  // namespace moa
