// RunSummary over a set of request traces: run_repetitions / summarize /
// critical_path_prefill_share / percentile (orchestrator.hpp:59-86,
// orchestrator.cpp:297-382).  The summary works on a plain trace view so the
// same code scores the GPU engine's requests (device seconds) and, in the
// CPU tests, the reference's own virtual-time traces (oracle/_ref).
#pragma once

#include <map>
#include <vector>

#include "graph.hpp"
#include "orchestrator.hpp"

namespace moa {

struct TracePrefill {  // PrefillInterval (trace.hpp:31-37)
  double start = 0.0, end = 0.0;
  bool wasted = false;
};

struct TraceAgent {  // the AgentRecord fields summarize reads (trace.hpp:40-66)
  int model = 0;     // model index (the reference keys activation by model_tag)
  bool invoked = false, pruned = false;
  int prefill_only_calls = 0, recomputed_tokens = 0;
  double complete_t = 0.0;
  std::vector<TracePrefill> prefill;
};

struct TraceView {  // RunTrace (trace.hpp:90-124) after roll_up
  double e2e_latency = 0.0;
  double ee_latency_total = 0.0;
  std::map<AgentId, TraceAgent> agents;
};

struct ModelActivation {  // trace.hpp:84-88
  int instances = 0, invoked = 0, pruned = 0;
};

struct RunSummary {  // orchestrator.hpp:61-76
  int samples = 0;
  double mean_e2e = 0.0, p50_e2e = 0.0, p95_e2e = 0.0;
  double mean_ee_share = 0.0, mean_prefill_only_calls = 0.0, mean_recomputed_tokens = 0.0;
  double prefill_share = 0.0;
  std::map<int, ModelActivation> activation_counts;
  std::map<int, double> activation;  // invoked / instances
};

// Linear interpolation between closest ranks (orchestrator.cpp:306-314).
double percentile(std::vector<double> v, double p);

// Committed prefill seconds on the chain of latest-completing surviving
// precursors ending at the root, over e2e (orchestrator.cpp:325-350).
double critical_path_prefill_share(const Topology& topo, const TraceView& trace);

RunSummary summarize(const Topology& topo, const std::vector<TraceView>& traces);  // orchestrator.cpp:352-382

// A GPU request as a trace view, in device seconds: prefill intervals are the
// ticks that ran an agent's prefill rows, complete_t the end of its completion
// tick (engine tracing must have been on: QueryResult::tick_ms), ee latency
// the host time the early-exit evaluations held the engine between ticks.
TraceView trace_view(const QueryResult& r);

// run_repetitions (orchestrator.cpp:297-302): samples 0..n-1 one request at a
// time, engine tracing on for the duration (restored afterwards).
std::vector<QueryResult> run_repetitions(GpuEngine& eng, const RunConfig& cfg, int repetitions, bool resolve = false);

}  // namespace moa
