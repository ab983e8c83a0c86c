// RunTrace JSONL for a GPU request, in the reference's format (trace.hpp:
// 18-124, trace.cpp:209-337): one "meta" record, one "agent" record per agent
// (id order), one "metricq" record per early-exit evaluation, one "event"
// record per prefill / decode / chunk / prune.  Times are seconds of device
// time since the request's first tick (the reference's are virtual seconds).
// Extension fields (ignored by the reference parser): per agent the literal
// output token ids and logprobs, so the reference MetricQEvaluator can
// re-score the GPU's completions (tools/replay_verify.py).
#pragma once

#include <string>
#include <vector>

#include "orchestrator.hpp"

namespace moa {

std::string trace_jsonl(const QueryResult& r);

}  // namespace moa
