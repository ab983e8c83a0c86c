#include "orchestrator.hpp"

#include <algorithm>

#include <chrono>

namespace moa {

void RunConfig::validate() const {  // orchestrator.cpp:21-62
  if (topology.layers().back().size() != 1)
    throw ValidationError("run: last layer must hold a single aggregator");
  if (!(tau > 0.0 && tau <= 1.0)) throw ValidationError("run.tau: must be in (0, 1]");
  if (chunk_size <= 0) throw ValidationError("run.chunk_size: must be > 0");
  if (force_q && !(*force_q >= 0.0 && *force_q <= 1.0)) throw ValidationError("run.force_q: must be in [0, 1]");
  if (query_tokens < 0 || leaf_prefix_tokens < 0 || agg_prefix_tokens < 0 || separator_tokens < 0 ||
      suffix_tokens < 0)
    throw ValidationError("run: token counts must be >= 0");
  if (hidden <= 0) throw ValidationError("provider.hidden: must be > 0");
  for (const auto& layer : topology.layers())
    for (const auto& a : layer) {
      if (!model_of.count(a)) throw ValidationError("run: no model assigned to agent " + a.str());
      auto it = out_len.find(a);
      if (it == out_len.end()) throw ValidationError("run: no output length for agent " + a.str());
      const OutLen& ol = it->second;
      if (ol.values.empty() && (ol.lo < 0 || ol.hi < ol.lo))
        throw ValidationError("run: output length needs 0 <= min <= max for agent " + a.str());
      for (int v : ol.values)
        if (v < 0) throw ValidationError("run: empirical output lengths must be >= 0 for agent " + a.str());
      // quality scores need at least one token of logprobs per output (orchestrator.cpp:42-60)
      if (early_exit && ol.min() < 1)
        throw ValidationError("run: early exit needs output_len >= 1 for agent " + a.str());
    }
}

int OutLen::min() const { return values.empty() ? lo : *std::min_element(values.begin(), values.end()); }

int OutLen::sample(std::uint64_t ss, const AgentId& a) const {
  if (!values.empty()) {
    rng::Stream s = rng::Stream::derive(ss, "outlen:" + a.str());
    return values[static_cast<std::size_t>(s.next_int(0, static_cast<std::int64_t>(values.size()) - 1))];
  }
  if (hi == lo) return lo;  // Fixed (a Uniform of one value draws the same)
  rng::Stream s = rng::Stream::derive(ss, "outlen:" + a.str());
  return static_cast<int>(s.next_int(lo, hi));
}

std::map<AgentId, int> tree_placement(const Topology& topo, int world) {
  std::map<AgentId, int> at;
  const auto& leaves = topo.layers().front();
  const int n = static_cast<int>(leaves.size());
  for (int i = 0; i < n; ++i) at[leaves[static_cast<std::size_t>(i)]] = static_cast<int>((1LL * i * world) / n);
  for (std::size_t l = 1; l < topo.layers().size(); ++l)
    for (const AgentId& a : topo.layers()[l]) at[a] = at.at(topo.precursors(a).front());
  return at;
}

namespace {

bool incremental(ScheduleMode m) { return m == ScheduleMode::IncrementalOverlap; }

// SimDriver (scenario.cpp:10-116) over the GPU engine.
class Driver {
 public:
  Driver(GpuEngine& eng, ScheduleMode mode, int chunk) : eng_(eng), mode_(mode), chunk_(chunk) {}

  void add_source(const AgentId& a, int model, int owner, TokenSeq prompt, int n) {
    eng_.add_agent(a, model, owner);
    order_.push_back(a);
    dependent_[a] = false;
    out_len_[a] = n;
    plans_.emplace(a, SlotPlan(a, PromptTemplate(std::move(prompt), {}, {}), false));
  }

  void add_plan(const AgentId& a, int model, int owner, PromptTemplate tmpl, int n) {
    eng_.add_agent(a, model, owner);
    order_.push_back(a);
    dependent_[a] = !tmpl.slots().empty();
    out_len_[a] = n;
    for (const auto& s : tmpl.slots()) consumers_[s.precursor].push_back(a);
    plans_.emplace(a, SlotPlan(a, std::move(tmpl), incremental(mode_)));
  }

  void start() {
    for (const auto& [dep, cs] : consumers_)
      for (const AgentId& c : cs) {
        const AgentId d = dep, cc = c;
        eng_.on_chunk(d, [this, d, cc](int, int, const TokenSeq& toks) { apply(cc, plans_.at(cc).on_chunk(d, toks)); });
      }
    for (const AgentId& a : order_) eng_.on_decode_end(a, [this, a](int) { completed(a); });
    for (const AgentId& a : order_) apply(a, plans_.at(a).start());
  }

  void apply(const AgentId& a, const std::vector<RouteAction>& acts) {
    for (const RouteAction& x : acts) {
      switch (x.kind) {
        case RouteAction::Kind::PrefillOnly:
          eng_.submit_prefill_only(a, x.start, x.tokens);
          break;
        case RouteAction::Kind::Generate: {
          const int pc = (mode_ == ScheduleMode::DpChunkedPrefill && dependent_.at(a)) ? chunk_ : 0;
          eng_.submit_generate(a, x.tokens, out_len_.at(a), chunk_, pc);
          break;
        }
        case RouteAction::Kind::Reclaim:
          eng_.reclaim(a, x.start);
          break;
      }
    }
  }

  void release(const AgentId& p) {
    auto it = consumers_.find(p);
    if (it == consumers_.end()) return;
    for (const AgentId& c : it->second) {
      eng_.note_precursor_ready(c);
      apply(c, plans_.at(c).on_precursor_done(p));
    }
  }

  void prune(const AgentId& p) {
    eng_.cancel(p);
    auto it = consumers_.find(p);
    if (it == consumers_.end()) return;
    for (const AgentId& c : it->second) {
      SlotPlan& plan = plans_.at(c);
      apply(c, plan.on_precursor_cancelled(p));
      if (plan.all_inputs_pruned()) eng_.mark_empty_input(c);
    }
  }

  std::function<void(const AgentId&)> gate;
  const std::vector<AgentId>& order() const { return order_; }

 private:
  void completed(const AgentId& a) {
    if (gate)
      gate(a);
    else
      release(a);
  }

  GpuEngine& eng_;
  ScheduleMode mode_;
  int chunk_;
  std::vector<AgentId> order_;
  std::map<AgentId, SlotPlan> plans_;
  std::map<AgentId, int> out_len_;
  std::map<AgentId, std::vector<AgentId>> consumers_;
  std::map<AgentId, bool> dependent_;
};

struct ExitGroup {
  int index = 0;
  std::vector<AgentId> members;
  GpuMetricQ* eval = nullptr;
  rng::Stream stream{0};
  bool exited = false;
  int evals = 0;
};

}  // namespace

namespace {

// One request of a (possibly concurrent) batch: its driver, exit groups and
// result.  Engine agent ids carry the request index; prompt / RNG labels use
// the topology ids (AgentId::str ignores the request).
struct Request {
  Request(GpuEngine& eng, const RunConfig& cfg, int req, int sample, int group_base)
      : eng(eng), cfg(cfg), req(req), sample(sample), group_base(group_base), drv(eng, cfg.mode, cfg.chunk_size) {}

  GpuEngine& eng;
  const RunConfig& cfg;
  int req, sample, group_base;
  Driver drv;
  QueryResult res;
  std::vector<std::unique_ptr<ExitGroup>> groups;
  std::map<AgentId, ExitGroup*> group_of;

  AgentId id(const AgentId& topo_id) const { return topo_id.in_request(req); }

  void build(const std::map<AgentId, int>& owner) {
    const Topology& topo = cfg.topology;
    const std::uint64_t ss = rng::hash_combine(cfg.seed, static_cast<std::uint64_t>(sample));
    // prompt synthesis + registration (orchestrator.cpp:151-191)
    const TokenSeq query = rng::synth_tokens(ss, "query", cfg.query_tokens);
    int max_out = 0;
    for (const auto& layer : topo.layers())
      for (const AgentId& a : layer) {
        const int n = cfg.out_len.at(a).sample(ss, a);
        max_out = std::max(max_out, n);
        if (topo.precursors(a).empty()) {
          TokenSeq prompt = rng::synth_tokens(ss, "leaf_prefix:" + a.str(), cfg.leaf_prefix_tokens);
          prompt.insert(prompt.end(), query.begin(), query.end());
          drv.add_source(id(a), cfg.model_of.at(a), owner.at(a), std::move(prompt), n);
        } else {
          std::vector<Slot> slots;
          const auto& pre = topo.precursors(a);
          for (std::size_t k = 0; k < pre.size(); ++k)
            slots.push_back(Slot{id(pre[k]), rng::synth_tokens(ss, "sep:" + a.str() + ":" + std::to_string(k),
                                                               cfg.separator_tokens)});
          PromptTemplate tmpl(rng::synth_tokens(ss, "agg_prefix:" + a.str(), cfg.agg_prefix_tokens), std::move(slots),
                              rng::synth_tokens(ss, "suffix:" + a.str(), cfg.suffix_tokens));
          drv.add_plan(id(a), cfg.model_of.at(a), owner.at(a), std::move(tmpl), n);
        }
      }

    // Tree-partitioned serving without an early-exit gate: an agent's chunks
    // go only to the ranks of its consumers (their slot plans prefill them)
    // and to rank 0 (which resolves the request's outputs).  With the gate
    // every rank evaluates it on every completion, so chunks go everywhere.
    if (eng.world() > 1 && !(cfg.early_exit && topo.depth() > 1)) {
      std::map<AgentId, std::uint64_t> dests;
      for (const auto& layer : topo.layers())
        for (const AgentId& a : layer) dests[a] |= 1ULL;
      for (const auto& layer : topo.layers())
        for (const AgentId& c : layer)
          for (const AgentId& p : topo.precursors(c)) dests[p] |= 1ULL << owner.at(c);
      for (const auto& [a, m] : dests) eng.set_chunk_dests(id(a), m);
    }
    // exit groups (orchestrator.cpp:193-220)
    if (!(cfg.early_exit && topo.depth() > 1)) return;
    std::vector<std::vector<AgentId>> sets;
    if (cfg.exit_scope == ExitScope::Layer || topo.kind() == TopologyKind::AllToAll) {
      for (int l = 1; l < topo.depth(); ++l) sets.push_back(topo.layer(l));
    } else {
      for (int l = 2; l <= topo.depth(); ++l)
        for (auto& c : topo.clusters_of_layer(l)) sets.push_back(c);
    }
    for (std::size_t g = 0; g < sets.size(); ++g) {
      auto grp = std::make_unique<ExitGroup>();
      grp->index = static_cast<int>(g);
      for (const AgentId& m : sets[g]) grp->members.push_back(id(m));
      const int width = cfg.embed_model >= 0 ? eng.model(cfg.embed_model).spec().d : cfg.hidden;
      grp->eval = &eng.ee_evaluator(group_base + static_cast<int>(g), width, cfg.provider_seed, cfg.tau,
                                    cfg.include_diagonal, static_cast<int>(sets[g].size()), std::max(1, max_out));
      grp->stream = rng::Stream::derive(ss, "ee:" + std::to_string(g));
      for (const AgentId& m : grp->members) group_of[m] = grp.get();
      groups.push_back(std::move(grp));
    }
    // completion gate (orchestrator.cpp:222-276); evaluations run between ticks
    drv.gate = [this](const AgentId& producer) {
      auto it = group_of.find(producer);
      if (it == group_of.end() || it->second->exited) {
        drv.release(producer);
        return;
      }
      ExitGroup* grp = it->second;
      eng.defer([this, producer, grp]() {
        const auto t0 = std::chrono::steady_clock::now();
        struct Clock {  // ee_latency_total analogue (orchestrator.cpp:236-240)
          std::chrono::steady_clock::time_point t0;
          double& acc;
          ~Clock() { acc += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
        } clock{t0, res.ee_ms};
        MetricQRecord rec;
        rec.tick = eng.tick();
        rec.group = grp->index;
        rec.eval_index = grp->evals;
        rec.completed = producer.topo();
        if (grp->exited) {
          res.metricq.push_back(rec);
          drv.release(producer);
          return;
        }
        grp->evals += 1;
        rec.evaluated = true;
        const int n = eng.record(producer).output_tokens;
        if (cfg.embed_fn) {
          TokenSeq toks(static_cast<std::size_t>(n));
          eng.read_outputs(producer, n, toks.data(), nullptr, nullptr);
          std::vector<double> emb(static_cast<std::size_t>(n) * static_cast<std::size_t>(cfg.hidden));
          cfg.embed_fn(toks, cfg.hidden, emb.data());
          rec.score = grp->eval->add_completion_host(emb.data(), eng.d_out_lp(), eng.out_offset(producer), n);
        } else if (cfg.embed_model >= 0) {
          eng.hidden_embed(cfg.embed_model, producer, n, *grp->eval);
          rec.score = grp->eval->add_completion_embedded(eng.d_out_lp(), eng.out_offset(producer), n);
        } else {
          rec.score = grp->eval->add_completion(eng.d_out_tok(), eng.d_out_lp(), eng.out_offset(producer), n);
        }
        const double q = cfg.force_q ? *cfg.force_q : rec.score.q;
        rec.decision = decide_exit(q, grp->stream);
        std::vector<AgentId> pruned;
        if (rec.decision.exited) {
          grp->exited = true;
          for (const AgentId& m : grp->members) {
            if (m == producer || eng.finished(m) || eng.cancelled(m)) continue;
            pruned.push_back(m);
          }
        }
        for (const AgentId& m : pruned) {
          drv.prune(m);
          rec.pruned.push_back(m.topo());
        }
        res.metricq.push_back(rec);
        drv.release(producer);
      });
    };
  }

  void roll_up(bool resolve) {
    int last = -1;
    for (const AgentId& ea : drv.order()) {
      const AgentId a = ea.topo();
      res.agents.push_back(a);
      AgentRecord r = eng.record(ea);
      r.id = a;
      res.records[a] = r;
      last = std::max(last, r.complete);
      if (r.invoked && !r.pruned) res.tokens += r.output_tokens;
      res.decoded_tokens += eng.decoded(ea);
    }
    res.ticks = last + 1;
    res.e2e_ms = eng.ms_since_start(last);
    if (eng.tracing())
      for (int t = 0; t <= last; ++t) res.tick_ms.push_back(eng.ms_since_start(t));
    for (int m = 0; m < eng.n_models(); ++m) res.model_tags.push_back(eng.model(m).spec().tag);
    res.seed = cfg.seed;
    res.sample = sample;
    res.topology_kind = cfg.topology.kind();
    res.mode = static_cast<int>(cfg.mode);
    res.early_exit = cfg.early_exit;
    res.hidden = cfg.hidden;
    res.provider_seed = cfg.provider_seed;
    res.tau = cfg.tau;
    res.include_diagonal = cfg.include_diagonal;
    res.weight_bytes = eng.bytes_moved();
    res.rows = eng.rows_processed();
    res.forwards = eng.kernel_forwards();
    res.host_ms = eng.host_ms();
    res.host_wait_ms = eng.host_wait_ms();
    if (!resolve) return;
    for (const AgentId& ea : drv.order()) {
      const AgentId a = ea.topo();
      res.prompts[a] = eng.resolve(eng.prompt(ea));
      const int n = eng.record(ea).output_tokens;
      TokenSeq out(static_cast<std::size_t>(n));
      std::vector<float> lp(static_cast<std::size_t>(n)), ent(static_cast<std::size_t>(n));
      if (n > 0) eng.read_outputs(ea, n, out.data(), lp.data(), ent.data());
      res.outputs[a] = std::move(out);
      res.logprobs[a] = std::move(lp);
      res.entropy[a] = std::move(ent);
    }
  }
};

}  // namespace

std::vector<QueryResult> run_queries(GpuEngine& eng, const RunConfig& cfg, const std::vector<int>& samples,
                                     bool resolve) {
  const auto t0 = std::chrono::steady_clock::now();
  cfg.validate();
  if (samples.empty()) throw ValidationError("run: at least one request is required");
  eng.reset();
  const std::map<AgentId, int> owner = tree_placement(cfg.topology, eng.world());
  const int groups_per_request = cfg.topology.agent_count();  // upper bound on exit groups per request
  std::vector<std::unique_ptr<Request>> reqs;
  for (std::size_t i = 0; i < samples.size(); ++i) {
    reqs.push_back(std::make_unique<Request>(eng, cfg, static_cast<int>(i), samples[i],
                                             static_cast<int>(i) * groups_per_request));
    reqs.back()->build(owner);
  }
  eng.mark_start();
  for (auto& r : reqs) r->drv.start();
  eng.run();
  std::vector<QueryResult> out;
  const double wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  for (auto& r : reqs) {
    r->roll_up(resolve);
    r->res.wall_ms = wall;
    out.push_back(std::move(r->res));
  }
  return out;
}

QueryResult run_query(GpuEngine& eng, const RunConfig& cfg, int sample, bool resolve) {
  return std::move(run_queries(eng, cfg, {sample}, resolve).front());
}

}  // namespace moa
