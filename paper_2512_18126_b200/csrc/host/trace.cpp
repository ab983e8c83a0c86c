#include "trace.hpp"

#include <array>
#include <cmath>
#include <cstdlib>
#include <map>
#include <cstdio>
#include <sstream>

namespace moa {

namespace {

// JSON numbers as the reference prints them (nlohmann: shortest round-trip)
std::string num(double v) {
  if (!std::isfinite(v)) return "null";
  char buf[32];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  // prefer the shortest representation that round-trips
  for (int p = 1; p <= 17; ++p) {
    char t[32];
    std::snprintf(t, sizeof t, "%.*g", p, v);
    if (std::strtod(t, nullptr) == v) {
      std::string s(t);
      if (s.find_first_of(".eE") == std::string::npos && s.find("inf") == std::string::npos) s += ".0";
      return s;
    }
  }
  return buf;
}

std::string str(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    o += c;
  }
  return o + "\"";
}

const char* mode_name(int m) {
  switch (m) {
    case 0: return "sequential-pd";
    case 1: return "dp-only";
    case 2: return "dp-chunked-prefill";
    default: return "incremental-overlap";
  }
}

}  // namespace

std::string trace_jsonl(const QueryResult& r) {
  auto at = [&](int tick) -> double {
    if (tick < 0) return -1.0;
    if (tick < static_cast<int>(r.tick_ms.size())) return r.tick_ms[static_cast<std::size_t>(tick)] / 1e3;
    return -1.0;
  };
  std::ostringstream out;
  const std::string label = std::string(r.topology_kind == TopologyKind::AllToAll ? "all_to_all" : "tree") + "|" +
                            mode_name(r.mode) + (r.early_exit ? "|ee" : "");
  // activation per model tag
  std::map<std::string, std::array<int, 3>> act;
  int poc = 0, rec = 0, recl = 0, wasted = 0, evals = 0;
  for (const AgentId& a : r.agents) {
    const AgentRecord& ar = r.records.at(a);
    auto& v = act[r.model_tags.at(static_cast<std::size_t>(ar.model))];
    v[0] += 1;
    v[1] += ar.invoked && !ar.pruned;
    v[2] += ar.pruned;
    poc += ar.prefill_only_calls;
    rec += ar.recomputed_tokens;
    recl += ar.reclaimed_tokens;
    wasted += ar.wasted_prefill_tokens;
  }
  for (const auto& m : r.metricq) evals += m.evaluated;
  out << "{\"record\":\"meta\",\"mode\":" << str(label) << ",\"seed\":" << r.seed << ",\"sample_index\":" << r.sample
      << ",\"e2e_latency\":" << num(r.e2e_ms / 1e3) << ",\"horizon\":" << num(at(r.ticks - 1))
      << ",\"ee_evals\":" << evals << ",\"ee_latency_total\":0.0,\"ee_latency_share\":0.0"
      << ",\"prefill_only_calls_total\":" << poc << ",\"recomputed_tokens_total\":" << rec
      << ",\"reclaimed_tokens_total\":" << recl << ",\"wasted_prefill_tokens_total\":" << wasted << ",\"activation\":{";
  bool first = true;
  for (const auto& [tag, v] : act) {
    out << (first ? "" : ",") << str(tag) << ":{\"instances\":" << v[0] << ",\"invoked\":" << v[1]
        << ",\"pruned\":" << v[2] << "}";
    first = false;
  }
  out << "},\"device\":\"B200\",\"ticks\":" << r.ticks << ",\"provider\":{\"kind\":\"mock\",\"hidden\":" << r.hidden
      << ",\"seed\":" << r.provider_seed << "},\"tau\":" << num(r.tau)
      << ",\"include_diagonal\":" << (r.include_diagonal ? "true" : "false") << "}\n";

  for (const auto& [id, ar] : r.records) {
    double exposed = 0.0;  // prefill time after the last precursor finished (not hidden behind waiting)
    const double ready = at(ar.precursor_ready_tick);
    out << "{\"record\":\"agent\",\"agent\":" << str(id.str()) << ",\"model_tag\":"
        << str(r.model_tags.at(static_cast<std::size_t>(ar.model))) << ",\"monolithic\":true"
        << ",\"invoked\":" << (ar.invoked ? "true" : "false") << ",\"pruned\":" << (ar.pruned ? "true" : "false")
        << ",\"empty_input\":" << (ar.empty_input ? "true" : "false") << ",\"submit_t\":" << num(at(ar.submit_tick) < 0 ? 0.0 : at(ar.submit_tick))
        << ",\"precursor_ready_t\":" << num(ready < 0 ? 0.0 : ready) << ",\"prompt_tokens\":" << ar.prompt_tokens
        << ",\"output_tokens\":" << ar.output_tokens << ",\"prefill\":[";
    for (std::size_t i = 0; i < ar.prefill.size(); ++i) {
      const auto& p = ar.prefill[i];
      const double s = p.tick > 0 ? at(p.tick - 1) : 0.0, e = at(p.tick);
      if (e > ready && ready >= 0) exposed += e - std::max(s, ready);
      out << (i ? "," : "") << "{\"start\":" << num(s) << ",\"end\":" << num(e) << ",\"begin_token\":" << p.begin
          << ",\"end_token\":" << p.end << ",\"wasted\":false}";
    }
    out << "],\"prefill_only_calls\":" << ar.prefill_only_calls << ",\"recomputed_tokens\":" << ar.recomputed_tokens
        << ",\"reclaimed_tokens\":" << ar.reclaimed_tokens << ",\"wasted_prefill_tokens\":" << ar.wasted_prefill_tokens
        << ",\"transfer_seconds\":0.0,\"transfer_end\":-1.0,\"decode_start\":" << num(at(ar.decode_start))
        << ",\"decode_end\":" << num(at(ar.decode_end)) << ",\"complete_t\":" << num(at(ar.complete))
        << ",\"exposed_prefill\":" << num(exposed) << ",\"pe_busy\":0.0,\"de_busy\":0.0";
    auto ot = r.outputs.find(id);
    if (ot != r.outputs.end()) {
      out << ",\"output_token_ids\":[";
      for (std::size_t i = 0; i < ot->second.size(); ++i) out << (i ? "," : "") << ot->second[i];
      out << "],\"logprobs\":[";
      const auto& lp = r.logprobs.at(id);
      for (std::size_t i = 0; i < lp.size(); ++i) out << (i ? "," : "") << num(lp[i]);
      out << "]";
    }
    out << "}\n";
  }

  for (const MetricQRecord& m : r.metricq) {
    out << "{\"record\":\"metricq\",\"t\":" << num(at(m.tick)) << ",\"group\":" << str("ee:" + std::to_string(m.group))
        << ",\"eval_index\":" << m.eval_index << ",\"completed\":" << str(m.completed.str())
        << ",\"evaluated\":" << (m.evaluated ? "true" : "false");
    if (m.evaluated) {
      const QualityScore& q = m.score;
      out << ",\"score\":{\"outputs\":" << q.outputs << ",\"confidences\":[";
      for (std::size_t i = 0; i < q.confidences.size(); ++i) out << (i ? "," : "") << num(q.confidences[i]);
      out << "],\"c_bar\":" << num(q.c_bar) << ",\"sim\":[";
      const int n = q.outputs;
      for (int i = 0; i < n; ++i) {
        out << (i ? "," : "") << "[";
        for (int j = 0; j < n; ++j) out << (j ? "," : "") << num(q.sim[static_cast<std::size_t>(i * n + j)]);
        out << "]";
      }
      out << "],\"weight_sum\":" << num(q.weight_sum) << ",\"weighted\":" << num(q.weighted)
          << ",\"calibrated\":" << num(q.calibrated) << ",\"q\":" << num(q.q) << ",\"tau\":" << num(q.tau) << "}";
    }
    out << ",\"decision\":{\"q\":" << num(m.decision.q) << ",\"draw\":" << num(m.decision.draw)
        << ",\"exited\":" << (m.decision.exited ? "true" : "false") << "},\"pruned\":[";
    for (std::size_t i = 0; i < m.pruned.size(); ++i) out << (i ? "," : "") << str(m.pruned[i].str());
    out << "]}\n";
  }
  return out.str();
}

}  // namespace moa
