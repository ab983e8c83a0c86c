#include "summary.hpp"

#include <algorithm>
#include <cmath>

namespace moa {

double percentile(std::vector<double> v, double p) {
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const double rank = p * static_cast<double>(v.size() - 1);
  const auto lo = static_cast<std::size_t>(std::floor(rank));
  const auto hi = static_cast<std::size_t>(std::ceil(rank));
  const double frac = rank - std::floor(rank);
  return v[lo] * (1.0 - frac) + v[hi] * frac;
}

namespace {

double mean(const std::vector<double>& v) {
  if (v.empty()) return 0.0;
  double s = 0.0;
  for (double x : v) s += x;
  return s / static_cast<double>(v.size());
}

}  // namespace

double critical_path_prefill_share(const Topology& topo, const TraceView& trace) {
  double prefill = 0.0;
  AgentId at = topo.root();
  for (;;) {
    const auto self = trace.agents.find(at);
    if (self == trace.agents.end()) throw RunError("summarize: trace has no record for " + at.str());
    for (const TracePrefill& p : self->second.prefill)
      if (!p.wasted) prefill += p.end - p.start;
    // step to the latest-completing surviving precursor (first one on ties)
    const AgentId* next = nullptr;
    double best = -1.0;
    for (const AgentId& p : topo.precursors(at)) {
      const auto it = trace.agents.find(p);
      if (it == trace.agents.end() || it->second.pruned) continue;
      if (it->second.complete_t > best) {
        best = it->second.complete_t;
        next = &p;
      }
    }
    if (!next) break;
    at = *next;
  }
  return trace.e2e_latency > 0 ? prefill / trace.e2e_latency : 0.0;
}

RunSummary summarize(const Topology& topo, const std::vector<TraceView>& traces) {
  RunSummary s;
  s.samples = static_cast<int>(traces.size());
  std::vector<double> e2e, ee_share, calls, recomputed, share;
  for (const TraceView& t : traces) {
    int poc = 0, rec = 0;
    for (const auto& [id, a] : t.agents) {
      poc += a.prefill_only_calls;
      rec += a.recomputed_tokens;
      ModelActivation& act = s.activation_counts[a.model];  // RunTrace::roll_up (trace.cpp:190-207)
      act.instances += 1;
      act.invoked += a.invoked && !a.pruned;
      act.pruned += a.pruned;
    }
    e2e.push_back(t.e2e_latency);
    ee_share.push_back(t.e2e_latency > 0.0 ? t.ee_latency_total / t.e2e_latency : 0.0);
    calls.push_back(static_cast<double>(poc));
    recomputed.push_back(static_cast<double>(rec));
    share.push_back(critical_path_prefill_share(topo, t));
  }
  s.mean_e2e = mean(e2e);
  s.p50_e2e = percentile(e2e, 0.50);
  s.p95_e2e = percentile(e2e, 0.95);
  s.mean_ee_share = mean(ee_share);
  s.mean_prefill_only_calls = mean(calls);
  s.mean_recomputed_tokens = mean(recomputed);
  s.prefill_share = mean(share);
  for (const auto& [m, a] : s.activation_counts)
    s.activation[m] = a.instances > 0 ? static_cast<double>(a.invoked) / static_cast<double>(a.instances) : 0.0;
  return s;
}

TraceView trace_view(const QueryResult& r) {
  if (r.tick_ms.size() < static_cast<std::size_t>(std::max(r.ticks, 0)))
    throw RunError("summarize: request ran without engine tracing (no per-tick device times)");
  auto at = [&](int tick) -> double {
    if (tick < 0) return 0.0;
    return r.tick_ms[static_cast<std::size_t>(tick)] / 1e3;
  };
  TraceView v;
  v.e2e_latency = r.e2e_ms / 1e3;
  v.ee_latency_total = r.ee_ms / 1e3;
  for (const auto& [id, ar] : r.records) {
    TraceAgent a;
    a.model = ar.model;
    a.invoked = ar.invoked;
    a.pruned = ar.pruned;
    a.prefill_only_calls = ar.prefill_only_calls;
    a.recomputed_tokens = ar.recomputed_tokens;
    a.complete_t = ar.complete >= 0 ? at(ar.complete) : -1.0;
    // one interval per tick that ran this agent's prefill rows (a tick's
    // rows of one agent are one contiguous append)
    for (const PrefillInterval& p : ar.prefill)
      a.prefill.push_back(TracePrefill{p.tick > 0 ? at(p.tick - 1) : 0.0, at(p.tick), false});
    v.agents[id] = std::move(a);
  }
  return v;
}

std::vector<QueryResult> run_repetitions(GpuEngine& eng, const RunConfig& cfg, int repetitions, bool resolve) {
  if (repetitions <= 0) throw ValidationError("run_repetitions: repetitions must be > 0");
  const bool was = eng.tracing();
  eng.set_tracing(true);
  std::vector<QueryResult> out;
  try {
    for (int i = 0; i < repetitions; ++i) out.push_back(run_query(eng, cfg, i, resolve));
  } catch (...) {
    eng.set_tracing(was);
    throw;
  }
  eng.set_tracing(was);
  return out;
}

}  // namespace moa
