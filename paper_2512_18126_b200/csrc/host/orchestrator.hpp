// run_query over the GPU engine: prompt synthesis, source/plan registration,
// slot-filling driver, exit groups and the completion gate, exactly as the
// reference wires them (orchestrator.cpp:130-295, scenario.cpp:10-116), with
// agent outputs produced by greedy decode on the device.
#pragma once

#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "engine.hpp"
#include "graph.hpp"
#include "metricq.hpp"

namespace moa {

enum class ScheduleMode { SequentialPd, DpOnly, DpChunkedPrefill, IncrementalOverlap };  // pdsim.hpp:38
enum class ExitScope { Cluster, Layer };                                                   // orchestrator.hpp:17

struct OutLen {             // OutputLenDist (agent.hpp:40-103)
  int lo = 64, hi = 64;      // Fixed when lo == hi, else Uniform [lo, hi]
  std::vector<int> values;   // Empirical when non-empty: uniform over this support
  int min() const;
  int sample(std::uint64_t ss, const AgentId& a) const;  // RngStream::derive(ss, "outlen:" + a)
};

struct RunConfig {  // orchestrator.hpp:23-53 (+ model per agent, which replaces rates)
  Topology topology = Topology::tree({1}, {});
  std::map<AgentId, int> model_of;
  std::map<AgentId, OutLen> out_len;
  ScheduleMode mode = ScheduleMode::IncrementalOverlap;
  bool early_exit = false;
  ExitScope exit_scope = ExitScope::Cluster;
  double tau = kDefaultTau;
  bool include_diagonal = true;
  std::optional<double> force_q;
  int chunk_size = 32;
  std::uint64_t seed = 0;
  int query_tokens = 256, leaf_prefix_tokens = 64, agg_prefix_tokens = 96, separator_tokens = 0,
      suffix_tokens = 32;
  int hidden = 64;
  std::uint64_t provider_seed = 0;
  // embedding provider: -1 = the reference's MockProvider (hidden, provider_seed);
  // >= 0 = hidden states of engine model `embed_model` (width = its d_model)
  int embed_model = -1;
  // caller EmbeddingProvider (embedding.hpp:38-44): tokens -> out[n][hidden], width = hidden
  std::function<void(const TokenSeq&, int hidden, double* out)> embed_fn;

  void validate() const;
};

struct MetricQRecord {  // trace.hpp:69-78
  int tick = 0;
  int group = 0;
  int eval_index = 0;
  AgentId completed;
  bool evaluated = false;
  QualityScore score;
  ExitDecision decision;
  std::vector<AgentId> pruned;
};

struct QueryResult {
  std::vector<AgentId> agents;  // registration order
  std::map<AgentId, AgentRecord> records;
  std::map<AgentId, TokenSeq> prompts;  // literal tokens
  std::map<AgentId, TokenSeq> outputs;  // literal tokens (emitted prefix for pruned agents)
  std::map<AgentId, std::vector<float>> logprobs, entropy;
  std::vector<MetricQRecord> metricq;
  int ticks = 0;
  long long tokens = 0;          // output tokens of invoked, unpruned agents
  long long decoded_tokens = 0;  // every token the GPU produced (incl. pruned)
  double e2e_ms = 0.0;           // first tick -> last completion (device events)
  double wall_ms = 0.0;          // host wall clock around the whole call
  double weight_bytes = 0.0;     // sum of per-forward weight reads
  long long rows = 0;
  int forwards = 0;
  double host_ms = 0.0;       // host time inside engine ticks
  double host_wait_ms = 0.0;  // of which: blocked on the GPU (the host is ahead)
  double ee_ms = 0.0;         // host time the early-exit evaluations held the engine between ticks
  // trace context (RunTrace JSONL, trace.hpp)
  std::vector<double> tick_ms;  // device ms at the end of each tick (engine tracing on)
  std::vector<std::string> model_tags;
  std::uint64_t seed = 0;
  int sample = 0;
  TopologyKind topology_kind = TopologyKind::Tree;
  int mode = 3;
  bool early_exit = false;
  int hidden = 64;
  std::uint64_t provider_seed = 0;
  double tau = kDefaultTau;
  bool include_diagonal = true;
};

// GPU placement along the tree: leaves are spread in
// contiguous blocks over the ranks (so a cluster's leaves share a rank when
// there are fewer ranks than leaves, and each gets its own when there are
// enough); every dependent agent runs on the rank of its first precursor (the
// cluster aggregator sits with its cluster's first leaf, the root on rank 0).
std::map<AgentId, int> tree_placement(const Topology& topo, int world);

// One orchestrated request on `eng` (which must hold every model the config
// names).  `resolve` = copy literal prompts/outputs back to the host.
QueryResult run_query(GpuEngine& eng, const RunConfig& cfg, int sample, bool resolve = true);

// Several independent requests served concurrently by one engine (continuous
// batching): every request keeps its own prompts, slot plans, exit groups
// and RNG streams (sample s_i, exactly as run_query(s_i)); their agents share
// the engine's ticks, so decode rows of all requests ride one weight pass per
// model.  Results are per request, keyed by the topology's agent ids; e2e_ms
// is each request's own first-tick -> last-completion latency.  The engine
// needs capacity for every request's agents.
std::vector<QueryResult> run_queries(GpuEngine& eng, const RunConfig& cfg, const std::vector<int>& samples,
                                     bool resolve = true);

}  // namespace moa
