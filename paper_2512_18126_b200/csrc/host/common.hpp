// Host foundations: agent ids, token sequences, errors and the deterministic
// RNG.  Same semantics as the reference's agent.hpp:16-37, errors.hpp:10-33
// and rng.hpp:14-103 (splitmix64 / fnv1a / RngStream), re-declared here so the
// B200 library has no dependency on the reference tree.
#pragma once

#include <compare>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <string_view>
#include <vector>

namespace moa {

using Token = std::int32_t;
using TokenSeq = std::vector<Token>;

// Invalid input / violated precondition (reference exit code 2).
struct ValidationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// Protocol or runtime failure (reference exit code 3).
struct RunError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
// Device / CUDA failure: a RunError with its own status code at the C-ABI.
// a valid request this build/device cannot serve (C-ABI MOA_ERR_UNSUPPORTED)
struct UnsupportedError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DeviceError : RunError {
  using RunError::RunError;
};
// Embedding provider failure (errors.hpp:24-33): Transport, MissingCredentials, BadResponse.
struct ProviderError : std::runtime_error {
  enum Kind { Transport, MissingCredentials, BadResponse };
  ProviderError(Kind k, const std::string& what) : std::runtime_error(what), kind(k) {}
  Kind kind;
};

struct AgentId {
  int layer = 1;
  int position = 0;
  int req = 0;  // request of a concurrent batch (engine-internal; 0 for a single request)
  auto operator<=>(const AgentId&) const = default;
  // the reference's "layer:position" (agent.hpp:16-38); labels of synthetic
  // prompts and RNG streams always use this form, whatever the request
  std::string str() const { return std::to_string(layer) + ":" + std::to_string(position); }
  AgentId in_request(int r) const { return AgentId{layer, position, r}; }
  AgentId topo() const { return AgentId{layer, position, 0}; }
};

namespace rng {

inline std::uint64_t mix64(std::uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

inline std::uint64_t fnv1a(std::string_view s) {
  std::uint64_t h = 0xcbf29ce484222325ULL;
  for (unsigned char c : s) {
    h ^= c;
    h *= 0x100000001b3ULL;
  }
  return h;
}

inline double unit_from_bits(std::uint64_t x) { return static_cast<double>(x >> 11) * 0x1.0p-53; }

inline std::uint64_t hash_combine(std::uint64_t a, std::uint64_t b) {
  return mix64(a ^ (b + 0x9e3779b97f4a7c15ULL + (a << 6) + (a >> 2)));
}

inline std::uint64_t hash_u64(std::uint64_t seed, std::string_view label, std::uint64_t i) {
  return mix64(hash_combine(hash_combine(seed, fnv1a(label)), i));
}

class Stream {
 public:
  explicit Stream(std::uint64_t s) : state_(s) {}
  static Stream derive(std::uint64_t master, std::string_view label) {
    return Stream(hash_combine(master, fnv1a(label)));
  }
  std::uint64_t next_u64() { return mix64(state_++); }
  double next_uniform() { return unit_from_bits(next_u64()); }
  std::int64_t next_int(std::int64_t lo, std::int64_t hi) {
    if (hi < lo) return lo;
    std::uint64_t span = static_cast<std::uint64_t>(hi - lo) + 1;
    return lo + static_cast<std::int64_t>(next_u64() % span);
  }
  std::uint64_t state() const { return state_; }

 private:
  std::uint64_t state_;
};

// scenario.cpp:257-264
inline TokenSeq synth_tokens(std::uint64_t seed, std::string_view label, int count) {
  TokenSeq out;
  out.reserve(count > 0 ? count : 0);
  for (int i = 0; i < count; ++i)
    out.push_back(static_cast<Token>(hash_u64(seed, label, static_cast<std::uint64_t>(i)) % 50000));
  return out;
}

}  // namespace rng
}  // namespace moa
