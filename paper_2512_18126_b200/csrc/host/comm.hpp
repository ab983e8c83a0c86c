// Inter-GPU hand-off for tree-partitioned requests: NCCL point-to-point
// (ncclSend / ncclRecv in groups) over NVLink / NVSwitch.  NCCL is loaded with
// dlopen on first use, so single-GPU use of the library has no NCCL
// dependency; inside a torch process the already-loaded libnccl.so.2 is reused.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "common.hpp"

namespace moa {

constexpr int kNcclIdBytes = 128;

class PeerComm {
 public:
  // Collective over `world` processes (one GPU each) sharing `id`.
  PeerComm(const std::uint8_t* id, int rank, int world);
  ~PeerComm();
  PeerComm(const PeerComm&) = delete;
  PeerComm& operator=(const PeerComm&) = delete;

  static void unique_id(std::uint8_t* out);  // ncclGetUniqueId

  int rank() const { return rank_; }
  int world() const { return world_; }

  // Grouped P2P: call begin(), any number of send/recv, end().
  void begin();
  void send_i32(const int* buf, long long n, int peer, cudaStream_t st);
  void recv_i32(int* buf, long long n, int peer, cudaStream_t st);
  void send_f32(const float* buf, long long n, int peer, cudaStream_t st);
  void recv_f32(float* buf, long long n, int peer, cudaStream_t st);
  void end();

 private:
  void* comm_ = nullptr;
  int rank_ = 0, world_ = 1;
};

}  // namespace moa
