// Reference-side adapters over the C-ABI, compiled
// against the reference's own headers (/root/reference/proj/core/include) and
// linked with libmoa_b200.so by oracle/ref/Makefile (target `integration`).
// TEST INFRASTRUCTURE: this is the code a maintainer adds on the reference
// side; tests/test_integration.py builds and runs it.
//
//   GpuEngineBackend  replaces  EngineBackend     engine_service.hpp:73-82
//   GpuWorld          replaces  SimWorld          pdsim.hpp:61-156
#pragma once

#include <functional>
#include <map>
#include <string>
#include <vector>

#include <nlohmann/json.hpp>

#include "moa_b200.h"
#include "moaserve/agent.hpp"
#include "moaserve/engine_service.hpp"
#include "moaserve/errors.hpp"

namespace moaserve {

// MOA status -> the reference's error classes (errors.hpp:10-33)
inline void moa_throw(int rc) {
  if (rc == MOA_OK) return;
  if (rc == MOA_ERR_VALIDATION) throw ValidationError(moa_last_error());
  throw RunError(moa_last_error());
}

// The split-entrypoint plugin (engine_service.hpp:73-82) served by the GPU
// engine: prefill_only / reclaim map 1:1; generate decodes max_new greedy
// tokens and returns the EngineService /generate body shape
// (engine_service.cpp:115-171: agent, prompt_tokens, remainder, chunks),
// with the decoded tokens in each chunk.
class GpuEngineBackend : public EngineBackend {
 public:
  GpuEngineBackend(moa_engine* eng, int max_new, int apc_chunk) : eng_(eng), max_new_(max_new), apc_(apc_chunk) {}

  bool prefill_only(const AgentId& a, int start, const TokenSeq& t) override {
    moa_throw(moa_prefill_only(eng_, a.layer, a.position, start, t.data(), static_cast<int>(t.size())));
    return true;  // the split entrypoint always exists (no sticky degrade)
  }

  nlohmann::ordered_json generate(const AgentId& a, const TokenSeq& prompt) override {
    int scheduled = 0, decoded = 0, fin = 0, canc = 0;
    moa_throw(moa_agent_state(eng_, a.layer, a.position, &scheduled, &decoded, &fin, &canc));
    moa_throw(moa_generate(eng_, a.layer, a.position, prompt.data(), static_cast<int>(prompt.size()), max_new_, apc_,
                           0));
    nlohmann::ordered_json out{{"agent", a.str()},
                               {"prompt_tokens", prompt.size()},
                               {"remainder", static_cast<int>(prompt.size()) - scheduled}};
    nlohmann::ordered_json chunks = nlohmann::ordered_json::array();
    std::vector<moa_event> ev(256);
    int busy = 1, n = 0;
    bool done = max_new_ == 0;
    while (busy && !done) {  // drive ticks until this agent finishes
      moa_throw(moa_step(eng_, ev.data(), static_cast<int>(ev.size()), &n, &busy));
      for (int i = 0; i < n; ++i) {
        if (ev[i].layer != a.layer || ev[i].position != a.position) continue;
        if (ev[i].kind == MOA_EV_CHUNK) {
          TokenSeq toks(static_cast<std::size_t>(ev[i].b));
          moa_throw(moa_read_output(eng_, a.layer, a.position, ev[i].b, toks.data(), nullptr, nullptr));
          chunks.push_back({{"t", ev[i].tick},
                            {"begin", ev[i].a},
                            {"end", ev[i].b},
                            {"tokens", TokenSeq(toks.begin() + ev[i].a, toks.end())}});
        }
        if (ev[i].kind == MOA_EV_DECODE_END) done = true;
      }
    }
    out["chunks"] = chunks;
    return out;
  }

  void reclaim(const AgentId& a, int keep) override { moa_throw(moa_reclaim(eng_, a.layer, a.position, keep)); }

 private:
  moa_engine* eng_;
  int max_new_, apc_;
};

// SimWorld's protocol (pdsim.hpp:61-156) over the GPU engine.  SimDriver
// (scenario.hpp:19-62) holds a `SimWorld&`, so a maintainer either makes the
// driver a template over its world type or calls moa_run_query, which runs
// the same driver natively.  The one semantic inversion: submit_generate
// takes the output length (planned.size()); the engine decodes the tokens.
class GpuWorld {
 public:
  using ChunkFn = std::function<void(double, int, int, const TokenSeq&)>;  // (t, begin, end, tokens)
  using EndFn = std::function<void(double)>;

  GpuWorld(moa_engine* e, std::map<std::string, int> model_index) : e_(e), models_(std::move(model_index)) {}

  void add_agent(const AgentId& id, const std::string& model_tag) {
    auto it = models_.find(model_tag);
    if (it == models_.end()) throw ValidationError("GpuWorld: unknown model tag " + model_tag);
    moa_throw(moa_add_agent(e_, id.layer, id.position, it->second));
  }
  void submit_prefill_only(const AgentId& id, int start, const TokenSeq& t) {
    moa_throw(moa_prefill_only(e_, id.layer, id.position, start, t.data(), static_cast<int>(t.size())));
  }
  void submit_generate(const AgentId& id, const TokenSeq& prompt, const TokenSeq& planned, int apc, int pc) {
    moa_throw(moa_generate(e_, id.layer, id.position, prompt.data(), static_cast<int>(prompt.size()),
                           static_cast<int>(planned.size()), apc, pc));
  }
  void cancel(const AgentId& id) { moa_throw(moa_cancel(e_, id.layer, id.position)); }
  void reclaim(const AgentId& id, int keep) { moa_throw(moa_reclaim(e_, id.layer, id.position, keep)); }
  void on_chunk(const AgentId& id, ChunkFn fn) { chunk_fns_[id].push_back(std::move(fn)); }
  void on_decode_end(const AgentId& id, EndFn fn) { end_fns_[id].push_back(std::move(fn)); }

  // Runs ticks until the engine is idle, dispatching chunk / decode-end
  // events (time = the tick index: the engine's virtual clock).
  void run() {
    std::vector<moa_event> ev(1024);
    int busy = 1, n = 0;
    while (busy) {
      moa_throw(moa_step(e_, ev.data(), static_cast<int>(ev.size()), &n, &busy));
      for (int i = 0; i < n; ++i) dispatch(ev[static_cast<std::size_t>(i)]);
    }
  }

 private:
  void dispatch(const moa_event& e) {
    const AgentId id{e.layer, e.position};
    if (e.kind == MOA_EV_CHUNK) {
      auto it = chunk_fns_.find(id);
      if (it == chunk_fns_.end()) return;
      TokenSeq toks(static_cast<std::size_t>(e.b));
      moa_throw(moa_read_output(e_, e.layer, e.position, e.b, toks.data(), nullptr, nullptr));
      const TokenSeq chunk(toks.begin() + e.a, toks.end());
      for (auto& fn : it->second) fn(static_cast<double>(e.tick), e.a, e.b, chunk);
    } else if (e.kind == MOA_EV_DECODE_END) {
      auto it = end_fns_.find(id);
      if (it == end_fns_.end()) return;
      for (auto& fn : it->second) fn(static_cast<double>(e.tick));
    }
  }

  moa_engine* e_;
  std::map<std::string, int> models_;
  std::map<AgentId, std::vector<ChunkFn>> chunk_fns_;
  std::map<AgentId, std::vector<EndFn>> end_fns_;
};

}  // namespace moaserve
