// The reference's HttpShellRouter cases (test_engine_service.cpp:436-558),
// run against the GPU engine through the reference-side adapter
// (gpu_backend.hpp) instead of the reference's FakeBackend.  TEST
// INFRASTRUCTURE: built by oracle/ref/Makefile `integration`, driven by
// tests/test_integration.py.
//
//   backend_cases link   -- no GPU: the adapter compiled and linked against the
//                           reference headers + libmoa_b200.so; calls only
//                           host entry points (routing) through the C-ABI
//   backend_cases gpu    -- the router cases on cuda:0 (tiny agent model);
//                           one JSON line per case with the engine's prompt,
//                           decoded tokens and logprobs (the Python side
//                           teacher-forces them against the oracle)
#include <cstdio>
#include <cstring>
#include <iostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "gpu_backend.hpp"
#include "moaserve/router.hpp"

using namespace moaserve;
using json = nlohmann::ordered_json;

namespace {

const AgentId kSelf{2, 0};
const AgentId kA{1, 0};
const AgentId kB{1, 1};

TokenSeq seq(std::initializer_list<Token> t) { return TokenSeq(t); }

PromptTemplate two_slot_template() {
  return PromptTemplate(seq({10, 11}), {SlotSpec{kA, seq({20})}, SlotSpec{kB, seq({21})}}, seq({30}));
}

void expect(bool c, const std::string& what) {
  if (!c) throw std::runtime_error("check failed: " + what);
}

// Records every call (FakeBackend's log, test_engine_service.cpp:71-107)
// and forwards it to the GPU backend; `delivered` is read back from the
// engine (scheduled prompt length) after every call.
struct Recording final : EngineBackend {
  struct Call {
    char kind;  // 'p' prefill, 'g' generate, 'r' reclaim
    int arg;
    TokenSeq tokens;
  };
  GpuEngineBackend& inner;
  moa_engine* eng;
  std::vector<Call> calls;
  json last;
  Recording(GpuEngineBackend& b, moa_engine* e) : inner(b), eng(e) {}

  int scheduled() const {
    int s = 0, d = 0, f = 0, c = 0;
    moa_throw(moa_agent_state(eng, kSelf.layer, kSelf.position, &s, &d, &f, &c));
    return s;
  }
  bool prefill_only(const AgentId& a, int start, const TokenSeq& t) override {
    calls.push_back({'p', start, t});
    expect(start == scheduled(), "prefill contiguity");
    const bool ok = inner.prefill_only(a, start, t);
    expect(scheduled() == start + static_cast<int>(t.size()), "prefill appended");
    return ok;
  }
  json generate(const AgentId& a, const TokenSeq& p) override {
    calls.push_back({'g', 0, p});
    last = inner.generate(a, p);
    return last;
  }
  void reclaim(const AgentId& a, int keep) override {
    calls.push_back({'r', keep, {}});
    inner.reclaim(a, keep);
    expect(scheduled() == keep, "reclaim truncates the scheduled prompt");
  }
};

json tokens_json(moa_engine* eng, int n) {
  std::vector<int32_t> tok(static_cast<std::size_t>(n));
  std::vector<float> lp(static_cast<std::size_t>(n));
  moa_throw(moa_read_output(eng, kSelf.layer, kSelf.position, n, tok.data(), lp.data(), nullptr));
  return json{{"tokens", tok}, {"logprobs", lp}};
}

int run_gpu(int max_new, int apc) {
  moa_model_spec m{};
  std::snprintf(m.tag, sizeof m.tag, "%s", "agg");
  // the `tiny` shape of oracle/model.py (d256 L4 4x64 heads FFN1024, vocab 50000), seed 2
  m.d = 256;
  m.n_layers = 4;
  m.n_heads = 4;
  m.n_kv_heads = 4;
  m.head_dim = 64;
  m.ffn = 1024;
  m.vocab = 50000;
  m.rope_theta = 10000.0;
  m.norm_eps = 1e-5;
  m.lm_gain = 4.0;
  m.seed = 2;
  m.max_agents = 1;
  moa_engine_opts o{};
  o.max_ctx = 256;
  o.max_out = max_new + 8;
  o.max_rows = 256;
  o.device = 0;
  moa_engine* eng = nullptr;
  moa_throw(moa_engine_create(&m, 1, &o, &eng));
  GpuEngineBackend gpu(eng, max_new, apc);
  auto fresh = [&]() {
    moa_throw(moa_engine_reset(eng));
    moa_throw(moa_add_agent(eng, kSelf.layer, kSelf.position, 0));
  };
  auto emit = [&](const char* name, const Recording& rec, const HttpShellRouter& router) {
    json line{{"case", name}, {"prompt", router.plan().final_prompt()}, {"calls", json::array()}};
    for (const auto& c : rec.calls) line["calls"].push_back(json{{"kind", std::string(1, c.kind)}, {"arg", c.arg}, {"tokens", c.tokens}});
    line["generate"] = rec.last;
    const json out = tokens_json(eng, max_new);
    line["tokens"] = out["tokens"];
    line["logprobs"] = out["logprobs"];
    std::cout << line.dump() << std::endl;
  };

  {  // "shell router streams an incremental fill through the backend"
    fresh();
    Recording rec(gpu, eng);
    HttpShellRouter router(rec, kSelf, two_slot_template(), true);
    router.start();
    router.on_chunk(kA, seq({100, 101}));
    router.on_precursor_done(kA);
    router.on_chunk(kB, seq({200}));
    expect(!router.done(), "not done before the last precursor");
    router.on_precursor_done(kB);
    expect(router.done() && !router.degraded(), "done, not degraded");
    expect(rec.calls.size() == 6, "six calls");
    expect(rec.calls[0].tokens == seq({10, 11, 20}) && rec.calls[1].tokens == seq({100, 101}) &&
               rec.calls[2].tokens == seq({21}) && rec.calls[3].tokens == seq({200}) && rec.calls[4].tokens == seq({30}),
           "streamed increments");
    expect(rec.calls[5].kind == 'g' && rec.calls[5].tokens == seq({10, 11, 20, 100, 101, 21, 200, 30}), "generate");
    expect(router.generate_response().at("prompt_tokens") == 8 && router.generate_response().at("remainder") == 0,
           "generate body");
    emit("incremental", rec, router);
  }
  {  // "non-incremental shell router accumulates and generates once"
    fresh();
    Recording rec(gpu, eng);
    HttpShellRouter router(rec, kSelf, two_slot_template(), false);
    router.start();
    router.on_chunk(kA, seq({100, 101}));
    router.on_precursor_done(kA);
    router.on_chunk(kB, seq({200}));
    router.on_precursor_done(kB);
    expect(router.done() && rec.calls.size() == 1 && rec.calls[0].kind == 'g', "one generate");
    expect(router.generate_response().at("remainder") == 8, "whole prompt is the remainder");
    emit("non_incremental", rec, router);
  }
  {  // "shell router coalesces increments below the token threshold"
    fresh();
    Recording rec(gpu, eng);
    HttpShellRouter router(rec, kSelf, two_slot_template(), true, 5);
    router.start();
    router.on_chunk(kA, seq({100}));
    expect(rec.calls.empty(), "below threshold");
    router.on_chunk(kA, seq({101, 102}));
    expect(rec.calls.size() == 1 && rec.calls[0].arg == 0 && rec.calls[0].tokens == seq({10, 11, 20, 100, 101, 102}),
           "first flush");
    router.on_chunk(kA, seq({103}));
    router.on_precursor_done(kA);
    expect(rec.calls.size() == 1, "still buffered");
    router.on_chunk(kB, seq({200, 201, 202}));
    expect(rec.calls.size() == 2 && rec.calls[1].arg == 6 && rec.calls[1].tokens == seq({103, 21, 200, 201, 202}),
           "second flush");
    router.on_precursor_done(kB);
    expect(rec.calls.size() == 3 && rec.calls[2].kind == 'g', "generate carries the suffix");
    expect(router.generate_response().at("remainder") == 1, "suffix is the remainder");
    emit("coalescing", rec, router);
  }
  {  // "shell router flushes the buffer before rolling a slot back"
    fresh();
    Recording rec(gpu, eng);
    HttpShellRouter router(rec, kSelf, two_slot_template(), true, 100);
    router.start();
    router.on_chunk(kA, seq({100, 101}));
    expect(rec.calls.empty(), "buffered");
    router.on_precursor_cancelled(kA);
    expect(rec.calls.size() == 2 && rec.calls[0].kind == 'p' && rec.calls[1].kind == 'r' && rec.calls[1].arg == 2,
           "flush then reclaim to the prefix");
    router.on_chunk(kB, seq({200}));
    router.on_precursor_done(kB);
    expect(router.done() && rec.calls.size() == 3 && rec.calls[2].tokens == seq({10, 11, 21, 200, 30}),
           "generate after rollback");
    emit("rollback", rec, router);
  }
  {  // engine errors surface as the reference's error classes
    fresh();
    bool threw = false;
    try {
      gpu.prefill_only(kSelf, 99, seq({4}));
    } catch (const RunError&) {
      threw = true;
    }
    expect(threw, "non-contiguous prefill -> RunError");
    gpu.prefill_only(kSelf, 0, seq({1, 2, 3}));
    threw = false;
    try {
      gpu.generate(kSelf, seq({9}));
    } catch (const RunError&) {
      threw = true;
    }
    expect(threw, "generate not extending the prefix -> RunError");
    threw = false;
    try {
      gpu.prefill_only(kSelf, 3, seq({60000}));
    } catch (const ValidationError&) {
      threw = true;
    }
    expect(threw, "token outside the vocabulary -> ValidationError");
  }
  {  // GpuWorld: SimWorld's protocol with callbacks (the SimDriver call pattern)
    fresh();
    GpuWorld world(eng, {{"agg", 0}});
    std::vector<std::pair<int, int>> chunks;
    double end_t = -1;
    world.on_chunk(kSelf, [&](double, int b, int e, const TokenSeq& t) {
      expect(static_cast<int>(t.size()) == e - b, "chunk size");
      chunks.emplace_back(b, e);
    });
    world.on_decode_end(kSelf, [&](double t) { end_t = t; });
    world.submit_prefill_only(kSelf, 0, seq({10, 11, 20, 100, 101}));
    world.submit_generate(kSelf, seq({10, 11, 20, 100, 101, 21, 200, 30}), TokenSeq(static_cast<std::size_t>(max_new)),
                          apc, 0);
    world.run();
    expect(end_t >= 0 && !chunks.empty() && chunks.back().second == max_new, "chunks and decode end");
    json line{{"case", "gpu_world"}, {"prompt", seq({10, 11, 20, 100, 101, 21, 200, 30})}, {"chunks", chunks}};
    const json out = tokens_json(eng, max_new);
    line["tokens"] = out["tokens"];
    line["logprobs"] = out["logprobs"];
    std::cout << line.dump() << std::endl;
  }
  moa_throw(moa_engine_destroy(eng));
  return 0;
}

int run_link() {
  // host-only entry points through the adapter's error mapping: a tree
  // topology and a slot plan (no device needed)
  const int widths[3] = {4, 2, 1}, clusters[3] = {2, 2, 2};
  int pre_off[8] = {0}, pre[16] = {0};
  moa_throw(moa_topology(0, 3, widths, clusters, pre_off, pre, 16));
  expect(pre_off[7] - pre_off[4] == 6, "tree precursors");
  bool threw = false;
  try {
    const int bad[2] = {2, 0};
    moa_throw(moa_topology(0, 2, bad, clusters, pre_off, pre, 16));
  } catch (const ValidationError&) {
    threw = true;
  }
  expect(threw, "invalid topology -> ValidationError");
  std::cout << json{{"link", "ok"}, {"version", moa_version()}}.dump() << std::endl;
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "link";
  try {
    if (mode == "gpu") return run_gpu(argc > 2 ? std::atoi(argv[2]) : 12, argc > 3 ? std::atoi(argv[3]) : 4);
    return run_link();
  } catch (const std::exception& e) {
    std::cerr << "backend_cases: " << e.what() << std::endl;
    return 1;
  }
}
