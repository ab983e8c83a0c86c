// Inter-GPU hand-off for tree-partitioned requests.  The engine talks to a
// PeerComm: grouped point-to-point sends / receives of chunk payloads.
//  * NcclComm -- ncclSend / ncclRecv in groups over NVLink / NVSwitch; NCCL
//    is loaded with dlopen on first use, so single-GPU use of the library has
//    no NCCL dependency (inside a torch process the already-loaded
//    libnccl.so.2 is reused).
//  * LoopbackComm -- several engines in ONE process (one thread each, any
//    devices, possibly the same one) exchanging through a shared hub with
//    device-to-device copies.  NCCL refuses two ranks on one GPU, so this is
//    how the partitioned engine is exercised on a single-GPU box; the engine
//    issues the identical message sequence to both.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <memory>
#include <mutex>
#include <vector>

#include "common.hpp"

namespace moa {

void cuda_check(cudaError_t e, const char* what);  // model.cpp
#ifndef MOA_CUDA
#define MOA_CUDA(x) ::moa::cuda_check((x), #x)
#endif

constexpr int kNcclIdBytes = 128;

class PeerComm {
 public:
  PeerComm(int rank, int world);
  virtual ~PeerComm() = default;
  PeerComm(const PeerComm&) = delete;
  PeerComm& operator=(const PeerComm&) = delete;

  int rank() const { return rank_; }
  int world() const { return world_; }

  // Grouped P2P: call begin(), any number of send/recv, end().  Received data
  // is visible to work enqueued on `st` after end().
  virtual void begin() = 0;
  virtual void send(const void* buf, long long bytes, int elem, int peer, cudaStream_t st) = 0;
  virtual void recv(void* buf, long long bytes, int elem, int peer, cudaStream_t st) = 0;
  virtual void end() = 0;

  void send_i32(const int* b, long long n, int peer, cudaStream_t st) { send(b, 4 * n, kI32, peer, st); }
  void recv_i32(int* b, long long n, int peer, cudaStream_t st) { recv(b, 4 * n, kI32, peer, st); }
  void send_f32(const float* b, long long n, int peer, cudaStream_t st) { send(b, 4 * n, kF32, peer, st); }
  void recv_f32(float* b, long long n, int peer, cudaStream_t st) { recv(b, 4 * n, kF32, peer, st); }

  static constexpr int kI32 = 0, kF32 = 1;

 private:
  int rank_ = 0, world_ = 1;
};

class NcclComm final : public PeerComm {
 public:
  // Collective over `world` processes (one GPU each) sharing `id`.
  NcclComm(const std::uint8_t* id, int rank, int world);
  ~NcclComm() override;
  static void unique_id(std::uint8_t* out);  // ncclGetUniqueId

  void begin() override;
  void send(const void* buf, long long bytes, int elem, int peer, cudaStream_t st) override;
  void recv(void* buf, long long bytes, int elem, int peer, cudaStream_t st) override;
  void end() override;

 private:
  void* comm_ = nullptr;
};

// Rendezvous point for LoopbackComm ranks living in one process.
class LoopbackHub {
 public:
  explicit LoopbackHub(int world);
  int world() const { return world_; }

  struct Msg {
    const void* src;
    long long bytes;
    int elem;
  };
  void barrier();
  void post(int from, int to, const Msg& m);
  Msg take(int from, int to);

 private:
  int world_;
  std::mutex mu_;
  std::condition_variable cv_;
  int arrived_ = 0;
  long long generation_ = 0;
  std::vector<std::vector<Msg>> q_;  // [from * world + to], FIFO
  std::vector<std::size_t> head_;
};

class LoopbackComm final : public PeerComm {
 public:
  LoopbackComm(std::shared_ptr<LoopbackHub> hub, int rank);

  void begin() override;
  void send(const void* buf, long long bytes, int elem, int peer, cudaStream_t st) override;
  void recv(void* buf, long long bytes, int elem, int peer, cudaStream_t st) override;
  void end() override;

 private:
  struct Recv {
    void* dst;
    long long bytes;
    int elem, peer;
  };
  std::shared_ptr<LoopbackHub> hub_;
  std::vector<Recv> recvs_;
  std::vector<cudaStream_t> streams_;
  bool open_ = false;
};

}  // namespace moa
