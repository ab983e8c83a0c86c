// oracle/ref/refwrap.cpp -- TEST INFRASTRUCTURE, NOT PRODUCT CODE.
//
// A JSON-in / JSON-out C entry point over the reference's own proj/core
// sources (compiled read-only from /root/reference by oracle/ref/Makefile
// into oracle/_ref/libmoaref.so).  tests/ and tests/golden/make_golden.py use
// it to pin the Python oracle against the reference implementation itself;
// bench.py's `--impl reference` arm may time `time_run_query` (the reference
// simulator's own run_repetitions, orchestrator.cpp:297-302).  Nothing in the
// product path links or loads this library.
#include <chrono>
#include <cstring>
#include <string>

#include <nlohmann/json.hpp>

#include "moaserve/embedding.hpp"
#include "moaserve/errors.hpp"
#include "moaserve/metricq.hpp"
#include "moaserve/orchestrator.hpp"
#include "moaserve/prompt.hpp"
#include "moaserve/rng.hpp"
#include "moaserve/router.hpp"
#include "moaserve/scenario.hpp"
#include "moaserve/topology.hpp"

using namespace moaserve;
using json = nlohmann::ordered_json;

namespace {

json ids(const std::vector<AgentId>& v) {
  json a = json::array();
  for (const auto& x : v) a.push_back(x.str());
  return a;
}

Topology topo_from(const json& j) {
  std::string kind = j.value("kind", "tree");
  std::vector<int> widths = j.at("widths").get<std::vector<int>>();
  if (kind == "all_to_all") return Topology::all_to_all(widths);
  if (j.contains("cluster_sizes"))
    return Topology::tree_custom(widths, j.at("cluster_sizes").get<std::vector<std::vector<int>>>());
  return Topology::tree(widths, j.at("branching").get<std::vector<int>>());
}

json cmd_topology(const json& req) {
  Topology t = topo_from(req);
  json out;
  json layers = json::array();
  for (const auto& l : t.layers()) layers.push_back(ids(l));
  out["layers"] = layers;
  json pre = json::object();
  for (const auto& l : t.layers())
    for (const auto& a : l) pre[a.str()] = ids(t.precursors(a));
  out["precursors"] = pre;
  json succ = json::object();
  for (const auto& l : t.layers())
    for (const auto& a : l) succ[a.str()] = ids(t.successors(a));
  out["successors"] = succ;
  json clusters = json::object();
  for (int l = 2; l <= t.depth(); ++l) {
    json cl = json::array();
    for (const auto& c : t.clusters_of_layer(l)) cl.push_back(ids(c));
    clusters[std::to_string(l)] = cl;
  }
  out["clusters"] = clusters;
  try {
    out["root"] = t.root().str();
  } catch (const ValidationError&) {
    out["root"] = nullptr;
  }
  return out;
}

json action_json(const RouteAction& a) {
  json j;
  switch (a.kind) {
    case RouteAction::Kind::PrefillOnly: j["kind"] = "prefill_only"; break;
    case RouteAction::Kind::Generate: j["kind"] = "generate"; break;
    case RouteAction::Kind::Reclaim: j["kind"] = "reclaim"; break;
  }
  j["start"] = a.start;
  j["tokens"] = a.tokens;
  return j;
}

json cmd_slotplan(const json& req) {
  std::vector<SlotSpec> slots;
  for (const auto& s : req.at("slots")) {
    SlotSpec spec;
    spec.precursor = AgentId::parse(s.at("precursor").get<std::string>());
    spec.separator = s.value("separator", TokenSeq{});
    slots.push_back(spec);
  }
  PromptTemplate tmpl(req.value("prefix", TokenSeq{}), slots, req.value("suffix", TokenSeq{}));
  SlotPlan plan(AgentId::parse(req.value("self", std::string("2:0"))), tmpl,
                req.value("incremental", true));
  json steps = json::array();
  for (const auto& ev : req.at("events")) {
    std::string op = ev.at("op").get<std::string>();
    std::vector<RouteAction> acts;
    json step;
    try {
      if (op == "start") acts = plan.start();
      else if (op == "chunk")
        acts = plan.on_chunk(AgentId::parse(ev.at("producer").get<std::string>()),
                             ev.at("tokens").get<TokenSeq>());
      else if (op == "done")
        acts = plan.on_precursor_done(AgentId::parse(ev.at("producer").get<std::string>()));
      else if (op == "cancelled")
        acts = plan.on_precursor_cancelled(AgentId::parse(ev.at("producer").get<std::string>()));
      json a = json::array();
      for (const auto& x : acts) a.push_back(action_json(x));
      step["actions"] = a;
    } catch (const ValidationError& e) {
      step["error"] = "ValidationError";
      step["what"] = e.what();
    } catch (const RunError& e) {
      step["error"] = "RunError";
      step["what"] = e.what();
    }
    steps.push_back(step);
    if (step.contains("error")) break;
  }
  json out;
  out["steps"] = steps;
  out["calls"] = plan.prefill_only_calls();
  out["reclaims"] = plan.reclaims();
  out["scheduled"] = plan.scheduled();
  out["generate_issued"] = plan.generate_issued();
  if (plan.generate_issued()) out["final_prompt"] = plan.final_prompt();
  return out;
}

json cmd_mock_embed(const json& req) {
  ProviderSpec spec;
  spec.kind = ProviderSpec::Kind::DeterministicMock;
  spec.hidden = req.value("hidden", 64);
  spec.seed = req.value("seed", std::uint64_t{0});
  auto p = make_provider(spec);
  Eigen::MatrixXd m = p->embed(req.at("tokens").get<TokenSeq>());
  json rows = json::array();
  for (Eigen::Index r = 0; r < m.rows(); ++r) {
    json row = json::array();
    for (Eigen::Index c = 0; c < m.cols(); ++c) row.push_back(m(r, c));
    rows.push_back(row);
  }
  return json{{"embedding", rows}};
}

json score_json(const QualityScore& qs) {
  json j;
  j["outputs"] = qs.outputs;
  j["confidences"] = qs.confidences;
  j["c_bar"] = qs.c_bar;
  json sim = json::array();
  for (Eigen::Index i = 0; i < qs.sim.rows(); ++i) {
    json row = json::array();
    for (Eigen::Index k = 0; k < qs.sim.cols(); ++k) row.push_back(qs.sim(i, k));
    sim.push_back(row);
  }
  j["sim"] = sim;
  j["weight_sum"] = qs.weight_sum;
  j["weighted"] = qs.weighted;
  j["calibrated"] = qs.calibrated;
  j["q"] = qs.q;
  return j;
}

// Incremental MetricQ over a completion sequence with the mock provider (or
// explicit embeddings), plus Bernoulli draws from RngStream::derive(ss, label)
// exactly as the EE gate does (orchestrator.cpp:214-217, :253-255).
json cmd_metricq(const json& req) {
  std::unique_ptr<EmbeddingProvider> provider;
  int hidden = req.value("hidden", 64);
  if (req.contains("embeddings")) {
    std::map<std::string, Eigen::MatrixXd> recs;
    const auto& outs = req.at("outputs");
    const auto& embs = req.at("embeddings");
    for (std::size_t i = 0; i < outs.size(); ++i) {
      const auto& e = embs[i];
      Eigen::MatrixXd m(static_cast<Eigen::Index>(e.size()), hidden);
      for (std::size_t r = 0; r < e.size(); ++r)
        for (int c = 0; c < hidden; ++c) m(static_cast<Eigen::Index>(r), c) = e[r][c].get<double>();
      recs[embedding_key(outs[i].get<TokenSeq>())] = m;
    }
    provider = make_map_provider(std::move(recs), hidden);
  } else {
    ProviderSpec spec;
    spec.hidden = hidden;
    spec.seed = req.value("seed", std::uint64_t{0});
    spec.memoize = true;
    provider = make_provider(spec);
  }
  MetricQOptions opts;
  opts.tau = req.value("tau", kDefaultTau);
  opts.include_diagonal = req.value("include_diagonal", true);
  MetricQEvaluator ev(*provider, opts);
  RngStream rng = RngStream::derive(req.value("rng_master", std::uint64_t{0}),
                                    req.value("rng_label", std::string("ee:0")));
  json evals = json::array();
  const auto& outs = req.at("outputs");
  const auto& lps = req.at("logprobs");
  for (std::size_t i = 0; i < outs.size(); ++i) {
    TokenLogProbs lp;
    lp.values = lps[i].get<std::vector<double>>();
    QualityScore qs = ev.add_completion(outs[i].get<TokenSeq>(), lp);
    ExitDecision d = decide_exit(qs.q, rng);
    json j = score_json(qs);
    j["draw"] = d.draw;
    j["exited"] = d.exited;
    evals.push_back(j);
  }
  return json{{"evals", evals}};
}

RunConfig config_from(const json& req) {
  RunConfig cfg;
  cfg.topology = topo_from(req.at("topology"));
  const json& profs = req.at("profiles");  // {"leaf": {...}, "agg": {...}} by layer index list
  const json& assign = req.at("assign");   // [[tag per position cycle], ...] per layer
  for (const auto& layer : cfg.topology.layers()) {
    for (const auto& a : layer) {
      const auto& cyc = assign[std::min<std::size_t>(a.layer - 1, assign.size() - 1)];
      std::string tag = cyc[static_cast<std::size_t>(a.position) % cyc.size()].get<std::string>();
      const json& pj = profs.at(tag);
      AgentProfile p;
      p.model_tag = tag;
      p.prefill_rate = pj.value("prefill_rate", p.prefill_rate);
      p.decode_rate = pj.value("decode_rate", p.decode_rate);
      p.output_len = OutputLenDist::fixed_len(pj.value("output_len", 64));
      if (pj.contains("output_min"))
        p.output_len = OutputLenDist::uniform(pj.at("output_min").get<int>(),
                                              pj.at("output_max").get<int>());
      p.conf_logprob_mu = pj.value("conf_logprob_mu", p.conf_logprob_mu);
      p.conf_logprob_sigma = pj.value("conf_logprob_sigma", p.conf_logprob_sigma);
      p.semantic_overlap = pj.value("semantic_overlap", p.semantic_overlap);
      cfg.topology.assign_profile(a, p);
    }
  }
  cfg.mode = schedule_mode_from_string(req.value("mode", std::string("incremental-overlap")));
  cfg.early_exit = req.value("early_exit", false);
  cfg.exit_scope = exit_scope_from_string(req.value("exit_scope", std::string("cluster")));
  cfg.tau = req.value("tau", kDefaultTau);
  cfg.include_diagonal = req.value("include_diagonal", true);
  cfg.ee_eval_latency = req.value("ee_eval_latency", 0.0);
  if (req.contains("force_q")) cfg.force_q = req.at("force_q").get<double>();
  cfg.chunk_size = req.value("chunk_size", 32);
  cfg.seed = req.value("seed", std::uint64_t{0});
  cfg.repetitions = req.value("repetitions", 1);
  cfg.query_tokens = req.value("query_tokens", 256);
  cfg.leaf_prefix_tokens = req.value("leaf_prefix_tokens", 64);
  cfg.agg_prefix_tokens = req.value("agg_prefix_tokens", 96);
  cfg.separator_tokens = req.value("separator_tokens", 0);
  cfg.suffix_tokens = req.value("suffix_tokens", 32);
  cfg.kv_transfer_per_block = req.value("kv_transfer_per_block", 0.0);
  cfg.provider.hidden = req.value("hidden", 64);
  cfg.provider.seed = req.value("provider_seed", std::uint64_t{0});
  cfg.provider.memoize = true;
  return cfg;
}

json cmd_run_query(const json& req) {
  RunConfig cfg = config_from(req);
  RunTrace tr = run_query(cfg, req.value("sample", 0));
  json out;
  out["e2e"] = tr.e2e_latency;
  out["ee_evals"] = tr.ee_evals;
  json mq = json::array();
  for (const auto& r : tr.metricq) {
    json j;
    j["group"] = r.group;
    j["eval_index"] = r.eval_index;
    j["completed"] = r.completed.str();
    j["evaluated"] = r.evaluated;
    j["q"] = r.decision.q;
    j["draw"] = r.decision.draw;
    j["exited"] = r.decision.exited;
    j["pruned"] = ids(r.pruned);
    mq.push_back(j);
  }
  out["metricq"] = mq;
  json agents = json::object();
  for (const auto& [id, a] : tr.agents) {
    agents[id.str()] = {{"invoked", a.invoked},
                        {"pruned", a.pruned},
                        {"prompt_tokens", a.prompt_tokens},
                        {"output_tokens", a.output_tokens},
                        {"prefill_only_calls", a.prefill_only_calls},
                        {"reclaimed_tokens", a.reclaimed_tokens},
                        {"complete_t", a.complete_t}};
  }
  out["agents"] = agents;
  return out;
}

// Wall-clock of the reference CPU path (run_repetitions over `reps` samples),
// single-threaded, as shipped (orchestrator.cpp:297-302).
json cmd_time_run_query(const json& req) {
  RunConfig cfg = config_from(req);
  int reps = req.value("reps", 24);
  auto t0 = std::chrono::steady_clock::now();
  double sink = 0.0;
  for (int i = 0; i < reps; ++i) sink += run_query(cfg, i).e2e_latency;
  auto t1 = std::chrono::steady_clock::now();
  return json{{"seconds", std::chrono::duration<double>(t1 - t0).count()},
              {"reps", reps},
              {"sink", sink}};
}

// run_repetitions + summarize as shipped (orchestrator.cpp:297-382), plus the
// per-trace fields summarize reads, so the C-ABI's moa_summarize can be fed
// the same traces (tests/test_summary.py).
json cmd_summarize(const json& req) {
  RunConfig cfg = config_from(req);
  cfg.repetitions = req.value("reps", 24);
  if (req.contains("ee_eval_latency")) cfg.ee_eval_latency = req.at("ee_eval_latency").get<double>();
  std::vector<RunTrace> traces = run_repetitions(cfg);
  json tj = json::array();
  for (const auto& t : traces) {
    json agents = json::array();
    for (const auto& [id, a] : t.agents) {
      json pf = json::array();
      for (const auto& p : a.prefill) pf.push_back({p.start, p.end, p.wasted});
      agents.push_back({{"layer", id.layer},
                        {"position", id.position},
                        {"model_tag", a.model_tag},
                        {"invoked", a.invoked},
                        {"pruned", a.pruned},
                        {"prefill_only_calls", a.prefill_only_calls},
                        {"recomputed_tokens", a.recomputed_tokens},
                        {"complete_t", a.complete_t},
                        {"prefill", pf}});
    }
    tj.push_back({{"e2e_latency", t.e2e_latency},
                  {"ee_latency_total", t.ee_latency_total},
                  {"prefill_share", critical_path_prefill_share(cfg.topology, t)},
                  {"agents", agents}});
  }
  json out;
  out["summary"] = summarize(cfg, traces).to_json();
  out["traces"] = tj;
  return out;
}

json cmd_rng(const json& req) {
  std::uint64_t seed = req.value("seed", std::uint64_t{0});
  std::string label = req.value("label", std::string(""));
  int n = req.value("n", 8);
  json out;
  std::vector<std::uint64_t> h;
  std::vector<double> u;
  for (int i = 0; i < n; ++i) {
    h.push_back(hash_u64(seed, label, static_cast<std::uint64_t>(i)));
    u.push_back(hash_unit(seed, label, static_cast<std::uint64_t>(i)));
  }
  out["hash_u64"] = h;
  out["hash_unit"] = u;
  RngStream s = RngStream::derive(seed, label);
  std::vector<double> draws;
  for (int i = 0; i < n; ++i) draws.push_back(s.next_uniform());
  out["stream_uniform"] = draws;
  out["hash_combine"] = hash_combine(seed, static_cast<std::uint64_t>(n));
  out["synth"] = synth_tokens(seed, label, n);
  return out;
}

// OutputLenDist::sample (agent.hpp:88-99) on RngStream::derive(seed, "outlen:" + agent)
json cmd_outlen(const json& req) {
  const std::uint64_t seed = req.value("seed", std::uint64_t{0});
  const std::string agent = req.value("agent", std::string("1:0"));
  const json& d = req.at("dist");
  OutputLenDist dist;
  const std::string kind = d.at("kind").get<std::string>();
  if (kind == "fixed") dist = OutputLenDist::fixed_len(d.at("n").get<int>());
  else if (kind == "uniform") dist = OutputLenDist::uniform(d.at("lo").get<int>(), d.at("hi").get<int>());
  else dist = OutputLenDist::empirical(d.at("values").get<std::vector<int>>());
  dist.validate("outlen");
  RngStream rng = RngStream::derive(seed, "outlen:" + agent);
  return json{{"n", dist.sample(rng)}};
}

thread_local std::string g_out;

}  // namespace

extern "C" const char* moaref_call(const char* request) {
  json out;
  try {
    json req = json::parse(request);
    std::string cmd = req.at("cmd").get<std::string>();
    if (cmd == "topology") out = cmd_topology(req);
    else if (cmd == "slotplan") out = cmd_slotplan(req);
    else if (cmd == "mock_embed") out = cmd_mock_embed(req);
    else if (cmd == "metricq") out = cmd_metricq(req);
    else if (cmd == "run_query") out = cmd_run_query(req);
    else if (cmd == "time_run_query") out = cmd_time_run_query(req);
    else if (cmd == "rng") out = cmd_rng(req);
    else if (cmd == "summarize") out = cmd_summarize(req);
    else if (cmd == "outlen") out = cmd_outlen(req);
    else out = json{{"error", "unknown"}, {"what", cmd}};
  } catch (const ValidationError& e) {
    out = json{{"error", "ValidationError"}, {"what", e.what()}};
  } catch (const RunError& e) {
    out = json{{"error", "RunError"}, {"what", e.what()}};
  } catch (const std::exception& e) {
    out = json{{"error", "exception"}, {"what", e.what()}};
  }
  g_out = out.dump(-1, ' ', false, nlohmann::ordered_json::error_handler_t::replace);
  return g_out.c_str();
}
