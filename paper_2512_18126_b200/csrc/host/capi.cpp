// extern "C" boundary (include/moa_b200.h).  Exceptions never cross it: they
// become status codes plus a thread-local message.
#include "../../../include/moa_b200.h"
#include "trace.hpp"

#include <cstring>
#include <memory>
#include <string>

#include "../kernels/kernels.cuh"
#include "engine.hpp"
#include "graph.hpp"
#include "metricq.hpp"
#include "orchestrator.hpp"
#include "summary.hpp"

struct moa_engine {
  std::unique_ptr<moa::GpuEngine> eng;
};

struct moa_query {
  moa::QueryResult r;
};

struct moa_slotplan {
  moa::SlotPlan plan;
};

namespace {

thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return MOA_OK;
  } catch (const moa::ValidationError& e) {
    g_err = e.what();
    return MOA_ERR_VALIDATION;
  } catch (const moa::UnsupportedError& e) {
    g_err = e.what();
    return MOA_ERR_UNSUPPORTED;
  } catch (const moa::DeviceError& e) {
    g_err = e.what();
    return MOA_ERR_DEVICE;
  } catch (const moa::RunError& e) {
    g_err = e.what();
    return MOA_ERR_RUNTIME;
  } catch (const moa::ProviderError& e) {
    g_err = e.what();
    return e.kind == moa::ProviderError::Transport            ? MOA_ERR_PROVIDER_TRANSPORT
           : e.kind == moa::ProviderError::MissingCredentials ? MOA_ERR_PROVIDER_CREDENTIALS
                                                              : MOA_ERR_PROVIDER_BAD_RESPONSE;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MOA_ERR_RUNTIME;
  }
}

void need(const void* p, const char* what) {
  if (!p) throw moa::ValidationError(std::string(what) + ": null pointer");
}

moa::GpuEngine& E(moa_engine* e) {
  need(e, "engine");
  return *e->eng;
}

moa::TokenSeq seq(const int32_t* t, int n) {
  if (n < 0) throw moa::ValidationError("token count must be >= 0");
  if (n > 0) need(t, "tokens");
  moa::TokenSeq s(t, t + n);
  for (auto v : s)
    if (v < 0) throw moa::ValidationError("tokens must be >= 0");
  return s;
}

moa::Topology topology_of(int kind, int n_layers, const int* widths, const int* cluster_sizes) {
  need(widths, "widths");
  if (n_layers <= 0) throw moa::ValidationError("topology: widths must be non-empty");
  std::vector<int> w(widths, widths + n_layers);
  if (kind == MOA_TOPO_ALL_TO_ALL) return moa::Topology::all_to_all(w);
  need(cluster_sizes, "cluster_sizes");
  std::vector<std::vector<int>> cs;
  int off = 0;
  for (int l = 1; l < n_layers; ++l) {
    if (w[static_cast<std::size_t>(l)] <= 0)
      throw moa::ValidationError("topology: layer " + std::to_string(l + 1) + " has non-positive width");
    cs.emplace_back(cluster_sizes + off, cluster_sizes + off + w[static_cast<std::size_t>(l)]);
    off += w[static_cast<std::size_t>(l)];
  }
  return moa::Topology::tree_custom(w, cs);
}

moa::RunConfig run_config_of(const moa_run_config* c) {
  need(c, "config");
  moa::RunConfig cfg;
  cfg.topology = topology_of(c->topo_kind, c->n_layers, c->widths, c->cluster_sizes);
  need(c->model_cycle, "model_cycle");
  need(c->cycle_len, "cycle_len");
  need(c->out_lo, "out_lo");
  need(c->out_hi, "out_hi");
  std::vector<int> off(static_cast<std::size_t>(c->n_layers) + 1, 0), voff(off);
  for (int l = 0; l < c->n_layers; ++l) {
    if (c->cycle_len[l] <= 0) throw moa::ValidationError("config: assignment cycle must not be empty");
    off[static_cast<std::size_t>(l) + 1] = off[static_cast<std::size_t>(l)] + c->cycle_len[l];
    const int nv = c->out_values_len ? c->out_values_len[l] : 0;
    if (nv < 0) throw moa::ValidationError("config: out_values_len must be >= 0");
    if (nv > 0) need(c->out_values, "out_values");
    voff[static_cast<std::size_t>(l) + 1] = voff[static_cast<std::size_t>(l)] + nv;
  }
  for (const auto& layer : cfg.topology.layers())
    for (const auto& a : layer) {
      const int l = a.layer - 1;
      cfg.model_of[a] = c->model_cycle[off[static_cast<std::size_t>(l)] + a.position % c->cycle_len[l]];
      moa::OutLen ol{c->out_lo[l], c->out_hi[l], {}};
      const int nv = c->out_values_len ? c->out_values_len[l] : 0;
      if (nv > 0)
        ol.values.assign(c->out_values + voff[static_cast<std::size_t>(l)],
                         c->out_values + voff[static_cast<std::size_t>(l)] + nv);
      cfg.out_len[a] = std::move(ol);
    }
  switch (c->mode) {
    case MOA_MODE_SEQUENTIAL_PD: cfg.mode = moa::ScheduleMode::SequentialPd; break;
    case MOA_MODE_DP_ONLY: cfg.mode = moa::ScheduleMode::DpOnly; break;
    case MOA_MODE_DP_CHUNKED_PREFILL: cfg.mode = moa::ScheduleMode::DpChunkedPrefill; break;
    case MOA_MODE_INCREMENTAL_OVERLAP: cfg.mode = moa::ScheduleMode::IncrementalOverlap; break;
    default: throw moa::ValidationError("mode: unknown schedule mode");
  }
  cfg.early_exit = c->early_exit != 0;
  cfg.exit_scope = c->exit_scope == MOA_SCOPE_LAYER ? moa::ExitScope::Layer : moa::ExitScope::Cluster;
  cfg.tau = c->tau;
  cfg.include_diagonal = c->include_diagonal != 0;
  if (c->use_force_q) cfg.force_q = c->force_q;
  cfg.chunk_size = c->chunk_size;
  cfg.seed = c->seed;
  cfg.query_tokens = c->query_tokens;
  cfg.leaf_prefix_tokens = c->leaf_prefix_tokens;
  cfg.agg_prefix_tokens = c->agg_prefix_tokens;
  cfg.separator_tokens = c->separator_tokens;
  cfg.suffix_tokens = c->suffix_tokens;
  cfg.hidden = c->hidden;
  cfg.provider_seed = c->provider_seed;
  cfg.embed_model = c->embed_model;
  if (c->embed_fn) {
    if (c->embed_model >= 0) throw moa::ValidationError("config: embed_fn and embed_model are exclusive");
    auto fn = c->embed_fn;
    void* user = c->embed_user;
    cfg.embed_fn = [fn, user](const moa::TokenSeq& t, int hidden, double* out) {
      const int rc = fn(user, t.data(), static_cast<int>(t.size()), hidden, out);
      if (rc == MOA_OK) return;
      const std::string what = "embedding provider failed (status " + std::to_string(rc) + ")";
      if (rc == MOA_ERR_PROVIDER_TRANSPORT) throw moa::ProviderError(moa::ProviderError::Transport, what);
      if (rc == MOA_ERR_PROVIDER_CREDENTIALS) throw moa::ProviderError(moa::ProviderError::MissingCredentials, what);
      throw moa::ProviderError(moa::ProviderError::BadResponse, what);
    };
  }
  return cfg;
}

}  // namespace

extern "C" {

const char* moa_last_error(void) { return g_err.c_str(); }
const char* moa_version(void) { return "moa_b200 0.1 (sm_100a)"; }

int moa_device_count(int* n) {
  return guard([&] {
    need(n, "n");
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) c = 0;
    *n = c;
  });
}

int moa_engine_create(const moa_model_spec* models, int n_models, const moa_engine_opts* opts, moa_engine** out) {
  return guard([&] {
    need(models, "models");
    need(out, "out");
    if (n_models <= 0) throw moa::ValidationError("engine: at least one model is required");
    std::vector<moa::ModelSpec> specs;
    std::vector<int> caps;
    for (int i = 0; i < n_models; ++i) {
      const moa_model_spec& m = models[i];
      moa::ModelSpec s;
      s.tag = std::string(m.tag, strnlen(m.tag, sizeof(m.tag)));
      s.d = m.d;
      s.n_layers = m.n_layers;
      s.n_heads = m.n_heads;
      s.n_kv_heads = m.n_kv_heads;
      s.head_dim = m.head_dim;
      s.ffn = m.ffn;
      s.vocab = m.vocab;
      s.rope_theta = m.rope_theta;
      s.norm_eps = m.norm_eps;
      s.lm_gain = m.lm_gain;
      s.seed = m.seed;
      specs.push_back(s);
      caps.push_back(m.max_agents);
    }
    moa::EngineOptions o;
    if (opts) {
      o.max_ctx = opts->max_ctx;
      o.max_out = opts->max_out;
      o.max_rows = opts->max_rows;
      o.device = opts->device;
      o.keep_logits = opts->keep_logits != 0;
      o.tensor_cores = opts->gemv_only == 0;
    }
    auto e = std::make_unique<moa_engine>();
    e->eng = std::make_unique<moa::GpuEngine>(specs, caps, o);
    *out = e.release();
  });
}

int moa_engine_destroy(moa_engine* eng) {
  return guard([&] { delete eng; });
}

int moa_engine_reset(moa_engine* eng) {
  return guard([&] { E(eng).reset(); });
}

int moa_nccl_unique_id(uint8_t* out) {
  return guard([&] {
    need(out, "out");
    moa::NcclComm::unique_id(out);
  });
}

int moa_engine_attach_comm(moa_engine* eng, const uint8_t* id, int rank, int world) {
  return guard([&] {
    need(id, "id");
    moa::GpuEngine& g = E(eng);
    MOA_CUDA(cudaSetDevice(g.device()));
    g.attach_comm(std::make_unique<moa::NcclComm>(id, rank, world));
  });
}

struct moa_loopback {
  std::shared_ptr<moa::LoopbackHub> hub;
};

int moa_loopback_create(int world, moa_loopback** out) {
  return guard([&] {
    need(out, "out");
    *out = new moa_loopback{std::make_shared<moa::LoopbackHub>(world)};
  });
}

int moa_loopback_destroy(moa_loopback* hub) {
  delete hub;
  return 0;
}

int moa_engine_attach_loopback(moa_engine* eng, moa_loopback* hub, int rank) {
  return guard([&] {
    need(hub, "hub");
    moa::GpuEngine& g = E(eng);
    MOA_CUDA(cudaSetDevice(g.device()));
    g.attach_comm(std::make_unique<moa::LoopbackComm>(hub->hub, rank));
  });
}

int moa_placement(int kind, int n_layers, const int* widths, const int* cluster_sizes, int world, int* ranks) {
  return guard([&] {
    need(ranks, "ranks");
    if (world < 1) throw moa::ValidationError("placement: world must be >= 1");
    moa::Topology t = topology_of(kind, n_layers, widths, cluster_sizes);
    const auto at = moa::tree_placement(t, world);
    int k = 0;
    for (const auto& layer : t.layers())
      for (const auto& a : layer) ranks[k++] = at.at(a);
  });
}

int moa_engine_probe(moa_engine* eng, int enable) {
  return guard([&] { E(eng).set_probing(enable != 0); });
}

int moa_engine_probe_stats(moa_engine* eng, int kind, int* launches, double* ms, double* bytes, double* flops) {
  return guard([&] {
    need(launches, "launches");
    need(ms, "ms");
    need(bytes, "bytes");
    if (kind < 0 || kind >= moa::KernelProbes::kKinds) throw moa::ValidationError("probe kind out of range");
    double f = 0.0;
    E(eng).probe_stats(kind, launches, ms, bytes, &f);
    if (flops) *flops = f;
  });
}

int moa_add_agent(moa_engine* eng, int layer, int position, int model) {
  return guard([&] { E(eng).add_agent(moa::AgentId{layer, position}, model); });
}

int moa_prefill_only(moa_engine* eng, int layer, int position, int start, const int32_t* tokens, int n) {
  return guard([&] { E(eng).submit_prefill_only(moa::AgentId{layer, position}, start, seq(tokens, n)); });
}

int moa_generate(moa_engine* eng, int layer, int position, const int32_t* prompt, int n, int max_new, int apc_chunk,
                 int prefill_chunk) {
  return guard([&] {
    E(eng).submit_generate(moa::AgentId{layer, position}, seq(prompt, n), max_new, apc_chunk, prefill_chunk);
  });
}

int moa_cancel(moa_engine* eng, int layer, int position) {
  return guard([&] { E(eng).cancel(moa::AgentId{layer, position}); });
}

int moa_reclaim(moa_engine* eng, int layer, int position, int keep) {
  return guard([&] { E(eng).reclaim(moa::AgentId{layer, position}, keep); });
}

int moa_step(moa_engine* eng, moa_event* events, int cap, int* n_events, int* busy) {
  return guard([&] {
    moa::GpuEngine& g = E(eng);
    g.clear_events();
    g.step();
    const auto& ev = g.events();
    int n = 0;
    for (const auto& e : ev) {
      if (events && n < cap) events[n] = moa_event{e.kind, e.tick, e.agent.layer, e.agent.position, e.a, e.b};
      ++n;
    }
    if (n_events) *n_events = n;
    if (busy) *busy = g.busy() ? 1 : 0;
  });
}

int moa_busy(moa_engine* eng, int* busy) {
  return guard([&] {
    need(busy, "busy");
    *busy = E(eng).busy() ? 1 : 0;
  });
}

int moa_read_output(moa_engine* eng, int layer, int position, int n, int32_t* tokens, float* logprobs,
                    float* entropy) {
  return guard([&] {
    moa::GpuEngine& g = E(eng);
    const moa::AgentId id{layer, position};
    if (n > g.decoded(id)) throw moa::ValidationError("read_output: only " + std::to_string(g.decoded(id)) +
                                                      " tokens decoded");
    g.read_outputs(id, n, tokens, logprobs, entropy);
  });
}

int moa_read_logits(moa_engine* eng, int layer, int position, int k, float* logits, int cap) {
  return guard([&] {
    need(logits, "logits");
    moa::GpuEngine& g = E(eng);
    const moa::AgentId id{layer, position};
    if (k < 0 || k >= g.decoded(id)) throw moa::ValidationError("read_logits: token index out of range");
    const int vocab = g.model(g.record(id).model).spec().vocab;
    if (cap < vocab)
      throw moa::ValidationError("read_logits: buffer of " + std::to_string(cap) + " floats < vocab " +
                                 std::to_string(vocab));
    g.read_logits(id, k, logits);
  });
}

int moa_agent_state(moa_engine* eng, int layer, int position, int* scheduled, int* decoded, int* finished,
                    int* cancelled) {
  return guard([&] {
    moa::GpuEngine& g = E(eng);
    const moa::AgentId id{layer, position};
    if (scheduled) *scheduled = static_cast<int>(g.prompt(id).size());
    if (decoded) *decoded = g.decoded(id);
    if (finished) *finished = g.finished(id) ? 1 : 0;
    if (cancelled) *cancelled = g.cancelled(id) ? 1 : 0;
  });
}

int moa_run_query(moa_engine* eng, const moa_run_config* cfg, int sample, int resolve, moa_run_summary* summary,
                  moa_query** out) {
  return guard([&] {
    moa::GpuEngine& g = E(eng);
    auto q = std::make_unique<moa_query>();
    q->r = moa::run_query(g, run_config_of(cfg), sample, resolve != 0);
    if (summary) {
      const auto& r = q->r;
      summary->ticks = r.ticks;
      summary->n_agents = static_cast<int>(r.agents.size());
      summary->n_evals = static_cast<int>(r.metricq.size());
      summary->forwards = r.forwards;
      summary->tokens = r.tokens;
      summary->decoded_tokens = r.decoded_tokens;
      summary->rows = r.rows;
      summary->e2e_ms = r.e2e_ms;
      summary->wall_ms = r.wall_ms;
      summary->weight_bytes = r.weight_bytes;
      summary->host_ms = r.host_ms;
      summary->host_wait_ms = r.host_wait_ms;
    }
    if (out) *out = q.release();
  });
}

int moa_run_batch(moa_engine* eng, const moa_run_config* cfg, const int* samples, int n, int resolve,
                  moa_run_summary* summaries, moa_query** out) {
  return guard([&] {
    need(samples, "samples");
    if (n <= 0) throw moa::ValidationError("run_batch: n must be > 0");
    std::vector<int> smp(samples, samples + n);
    auto rs = moa::run_queries(E(eng), run_config_of(cfg), smp, resolve != 0);
    for (int i = 0; i < n; ++i) {
      const auto& r = rs[static_cast<std::size_t>(i)];
      if (summaries) {
        moa_run_summary& s = summaries[i];
        s.ticks = r.ticks;
        s.n_agents = static_cast<int>(r.agents.size());
        s.n_evals = static_cast<int>(r.metricq.size());
        s.forwards = r.forwards;
        s.tokens = r.tokens;
        s.decoded_tokens = r.decoded_tokens;
        s.rows = r.rows;
        s.e2e_ms = r.e2e_ms;
        s.wall_ms = r.wall_ms;
        s.weight_bytes = r.weight_bytes;
        s.host_ms = r.host_ms;
        s.host_wait_ms = r.host_wait_ms;
      }
      if (out) {
        auto q = std::make_unique<moa_query>();
        q->r = std::move(rs[static_cast<std::size_t>(i)]);
        out[i] = q.release();
      }
    }
  });
}

int moa_read_residual(moa_engine* eng, int model, int rows, float* out, long long cap) {
  return guard([&] {
    need(out, "out");
    if (model < 0 || model >= E(eng).n_models()) throw moa::ValidationError("engine: model index out of range");
    moa::DeviceModel& dm = E(eng).model(model);
    const long long n = static_cast<long long>(rows) * dm.spec().d;
    if (rows < 0 || rows > dm.max_rows() || n > cap) throw moa::ValidationError("read_residual: rows out of range");
    MOA_CUDA(cudaStreamSynchronize(E(eng).stream()));
    MOA_CUDA(cudaMemcpy(out, dm.residual(), sizeof(float) * n, cudaMemcpyDeviceToHost));
  });
}

int moa_engine_trace(moa_engine* eng, int enable) {
  return guard([&] { E(eng).set_tracing(enable != 0); });
}

int moa_engine_mark_start(moa_engine* eng) {
  return guard([&] { E(eng).mark_start(); });
}

int moa_engine_tick(moa_engine* eng, int* tick) {
  return guard([&] {
    need(tick, "tick");
    *tick = E(eng).tick();
  });
}

int moa_tick_seconds(moa_engine* eng, int tick, double* seconds) {
  return guard([&] {
    need(seconds, "seconds");
    *seconds = E(eng).ms_since_start(tick) / 1e3;
  });
}

int moa_agent_record_get(moa_engine* eng, int layer, int position, moa_agent_record* rec) {
  return guard([&] {
    need(rec, "rec");
    const moa::AgentId id{layer, position};
    const moa::AgentRecord& r = E(eng).record(id);
    *rec = moa_agent_record{layer,
                            position,
                            r.model,
                            r.invoked,
                            r.pruned,
                            r.empty_input,
                            r.prompt_tokens,
                            r.output_tokens,
                            r.prefill_only_calls,
                            r.recomputed_tokens,
                            r.reclaimed_tokens,
                            r.decode_start,
                            r.decode_end,
                            r.complete,
                            r.precursor_ready_tick};
  });
}

int moa_query_trace(const moa_query* q, char* buf, long long cap, long long* len) {
  return guard([&] {
    need(q, "query");
    need(len, "len");
    const std::string s = moa::trace_jsonl(q->r);
    *len = static_cast<long long>(s.size());
    if (buf && cap > *len) std::memcpy(buf, s.c_str(), s.size() + 1);
  });
}

int moa_query_ticks(const moa_query* q, double* ms, int cap, int* n) {
  return guard([&] {
    need(q, "query");
    need(n, "n");
    *n = static_cast<int>(q->r.tick_ms.size());
    if (ms)
      for (int i = 0; i < std::min(cap, *n); ++i) ms[i] = q->r.tick_ms[static_cast<std::size_t>(i)];
  });
}

int moa_query_agent(const moa_query* q, int i, moa_agent_record* rec) {
  return guard([&] {
    need(q, "query");
    need(rec, "rec");
    if (i < 0 || i >= static_cast<int>(q->r.agents.size())) throw moa::ValidationError("agent index out of range");
    const auto& a = q->r.agents[static_cast<std::size_t>(i)];
    const auto& r = q->r.records.at(a);
    *rec = moa_agent_record{a.layer,
                            a.position,
                            r.model,
                            r.invoked,
                            r.pruned,
                            r.empty_input,
                            r.prompt_tokens,
                            r.output_tokens,
                            r.prefill_only_calls,
                            r.recomputed_tokens,
                            r.reclaimed_tokens,
                            r.decode_start,
                            r.decode_end,
                            r.complete,
                            r.precursor_ready_tick};
  });
}

int moa_query_tokens(const moa_query* q, int i, int which, int32_t* dst, int cap, int* n) {
  return guard([&] {
    need(q, "query");
    if (i < 0 || i >= static_cast<int>(q->r.agents.size())) throw moa::ValidationError("agent index out of range");
    const auto& a = q->r.agents[static_cast<std::size_t>(i)];
    const auto& m = which == 0 ? q->r.prompts : q->r.outputs;
    auto it = m.find(a);
    if (it == m.end()) throw moa::ValidationError("query: tokens were not resolved (resolve = 0)");
    const int len = static_cast<int>(it->second.size());
    if (n) *n = len;
    if (dst) std::memcpy(dst, it->second.data(), sizeof(int32_t) * std::min(cap, len));
  });
}

int moa_query_logprobs(const moa_query* q, int i, float* logprobs, float* entropy, int cap, int* n) {
  return guard([&] {
    need(q, "query");
    if (i < 0 || i >= static_cast<int>(q->r.agents.size())) throw moa::ValidationError("agent index out of range");
    const auto& a = q->r.agents[static_cast<std::size_t>(i)];
    auto it = q->r.logprobs.find(a);
    if (it == q->r.logprobs.end()) throw moa::ValidationError("query: outputs were not resolved");
    const int len = static_cast<int>(it->second.size());
    if (n) *n = len;
    if (logprobs) std::memcpy(logprobs, it->second.data(), sizeof(float) * std::min(cap, len));
    if (entropy) std::memcpy(entropy, q->r.entropy.at(a).data(), sizeof(float) * std::min(cap, len));
  });
}

int moa_query_eval(const moa_query* q, int i, moa_eval_record* rec, double* sim_row, int cap) {
  return guard([&] {
    need(q, "query");
    need(rec, "rec");
    if (i < 0 || i >= static_cast<int>(q->r.metricq.size())) throw moa::ValidationError("eval index out of range");
    const auto& m = q->r.metricq[static_cast<std::size_t>(i)];
    moa_eval_record r{};
    r.tick = m.tick;
    r.group = m.group;
    r.eval_index = m.eval_index;
    r.layer = m.completed.layer;
    r.position = m.completed.position;
    r.evaluated = m.evaluated;
    r.exited = m.decision.exited;
    r.n_pruned = static_cast<int>(m.pruned.size());
    r.outputs = m.score.outputs;
    r.q = m.decision.q;
    r.draw = m.decision.draw;
    r.c = m.score.confidences.empty() ? 0.0 : m.score.confidences.back();
    r.c_bar = m.score.c_bar;
    r.weight_sum = m.score.weight_sum;
    r.weighted = m.score.weighted;
    r.calibrated = m.score.calibrated;
    for (int k = 0; k < r.n_pruned && k < 16; ++k) {
      r.pruned_layer[k] = m.pruned[static_cast<std::size_t>(k)].layer;
      r.pruned_position[k] = m.pruned[static_cast<std::size_t>(k)].position;
    }
    *rec = r;
    if (sim_row && m.score.outputs > 0) {
      const int n = m.score.outputs;
      for (int j = 0; j < n && j < cap; ++j) sim_row[j] = m.score.sim[static_cast<std::size_t>(n - 1) * n + j];
    }
  });
}

int moa_query_free(moa_query* q) {
  return guard([&] { delete q; });
}

namespace {

void fill_summary(const moa::RunSummary& s, moa_summary* out) {
  *out = moa_summary{};
  out->samples = s.samples;
  out->mean_e2e = s.mean_e2e;
  out->p50_e2e = s.p50_e2e;
  out->p95_e2e = s.p95_e2e;
  out->mean_ee_share = s.mean_ee_share;
  out->mean_prefill_only_calls = s.mean_prefill_only_calls;
  out->mean_recomputed_tokens = s.mean_recomputed_tokens;
  out->prefill_share = s.prefill_share;
  for (const auto& [m, a] : s.activation_counts) {
    if (m < 0 || m >= MOA_SUMMARY_MAX_MODELS) throw moa::ValidationError("summarize: model index out of range");
    out->n_models = std::max(out->n_models, m + 1);
    out->instances[m] = a.instances;
    out->invoked[m] = a.invoked;
    out->pruned[m] = a.pruned;
    out->activation[m] = s.activation.at(m);
  }
}

void fill_run_summary(const moa::QueryResult& r, moa_run_summary& s) {
  s.ticks = r.ticks;
  s.n_agents = static_cast<int>(r.agents.size());
  s.n_evals = static_cast<int>(r.metricq.size());
  s.forwards = r.forwards;
  s.tokens = r.tokens;
  s.decoded_tokens = r.decoded_tokens;
  s.rows = r.rows;
  s.e2e_ms = r.e2e_ms;
  s.wall_ms = r.wall_ms;
  s.weight_bytes = r.weight_bytes;
  s.host_ms = r.host_ms;
  s.host_wait_ms = r.host_wait_ms;
}

}  // namespace

int moa_summarize(int kind, int n_layers, const int* widths, const int* cluster_sizes, const moa_trace_view* traces,
                  int n, moa_summary* out) {
  return guard([&] {
    need(out, "out");
    if (n < 0) throw moa::ValidationError("summarize: n must be >= 0");
    if (n > 0) need(traces, "traces");
    const moa::Topology topo = topology_of(kind, n_layers, widths, cluster_sizes);
    std::vector<moa::TraceView> views;
    for (int i = 0; i < n; ++i) {
      const moa_trace_view& t = traces[i];
      if (t.n_agents < 0 || (t.n_agents > 0 && !t.agents)) throw moa::ValidationError("summarize: bad trace agents");
      moa::TraceView v;
      v.e2e_latency = t.e2e_latency;
      v.ee_latency_total = t.ee_latency_total;
      for (int k = 0; k < t.n_agents; ++k) {
        const moa_trace_agent& a = t.agents[k];
        if (a.n_prefill < 0 || (a.n_prefill > 0 && !a.prefill))
          throw moa::ValidationError("summarize: bad prefill spans");
        moa::TraceAgent ta;
        ta.model = a.model;
        ta.invoked = a.invoked != 0;
        ta.pruned = a.pruned != 0;
        ta.prefill_only_calls = a.prefill_only_calls;
        ta.recomputed_tokens = a.recomputed_tokens;
        ta.complete_t = a.complete_t;
        for (int j = 0; j < a.n_prefill; ++j)
          ta.prefill.push_back(moa::TracePrefill{a.prefill[j].start, a.prefill[j].end, a.prefill[j].wasted != 0});
        v.agents[moa::AgentId{a.layer, a.position}] = std::move(ta);
      }
      views.push_back(std::move(v));
    }
    fill_summary(moa::summarize(topo, views), out);
  });
}

int moa_percentile(const double* v, int n, double p, double* out) {
  return guard([&] {
    need(out, "out");
    if (n < 0) throw moa::ValidationError("percentile: n must be >= 0");
    if (n > 0) need(v, "v");
    *out = moa::percentile(std::vector<double>(v, v + n), p);
  });
}

int moa_run_repetitions(moa_engine* eng, const moa_run_config* cfg, int repetitions, moa_summary* out,
                        moa_run_summary* per_sample) {
  return guard([&] {
    need(out, "out");
    const moa::RunConfig rc = run_config_of(cfg);
    const auto rs = moa::run_repetitions(E(eng), rc, repetitions, false);
    std::vector<moa::TraceView> views;
    for (std::size_t i = 0; i < rs.size(); ++i) {
      views.push_back(moa::trace_view(rs[i]));
      if (per_sample) fill_run_summary(rs[i], per_sample[i]);
    }
    fill_summary(moa::summarize(rc.topology, views), out);
  });
}

int moa_query_trace_view(const moa_query* q, moa_trace_view* view, moa_trace_agent* agents, int cap,
                         moa_prefill_span* spans, int span_cap, int* n_agents, int* n_spans) {
  return guard([&] {
    need(q, "query");
    const moa::TraceView v = moa::trace_view(q->r);
    int na = 0, ns = 0;
    for (const auto& [id, a] : v.agents) {
      const int first = ns;
      for (const auto& p : a.prefill) {
        if (spans && ns < span_cap) spans[ns] = moa_prefill_span{p.start, p.end, p.wasted ? 1 : 0};
        ++ns;
      }
      if (agents && na < cap) {
        agents[na] = moa_trace_agent{id.layer, id.position, a.model, a.invoked ? 1 : 0, a.pruned ? 1 : 0,
                                     a.prefill_only_calls, a.recomputed_tokens, a.complete_t,
                                     static_cast<int>(a.prefill.size()),
                                     spans && ns <= span_cap ? spans + first : nullptr};
      }
      ++na;
    }
    if (view) *view = moa_trace_view{v.e2e_latency, v.ee_latency_total, std::min(na, cap), agents};
    if (n_agents) *n_agents = na;
    if (n_spans) *n_spans = ns;
  });
}

int moa_mock_embed(const int32_t* tokens, int n, int hidden, uint64_t seed, double* out, int device) {
  return guard([&] {
    if (n <= 0) return;
    need(tokens, "tokens");
    need(out, "out");
    if (hidden <= 0) throw moa::ValidationError("provider.hidden: must be > 0");
    MOA_CUDA(cudaSetDevice(device));
    int* d_tok = nullptr;
    double* d_emb = nullptr;
    MOA_CUDA(cudaMalloc(&d_tok, sizeof(int) * n));
    MOA_CUDA(cudaMalloc(&d_emb, sizeof(double) * n * hidden));
    MOA_CUDA(cudaMemcpy(d_tok, tokens, sizeof(int) * n, cudaMemcpyHostToDevice));
    moa::k::ee_mock_embed(d_tok, 0, n, hidden, seed, d_emb, nullptr);
    MOA_CUDA(cudaGetLastError());
    MOA_CUDA(cudaMemcpy(out, d_emb, sizeof(double) * n * hidden, cudaMemcpyDeviceToHost));
    cudaFree(d_tok);
    cudaFree(d_emb);
  });
}

}  // extern "C"

struct moa_mq_group {
  int device = 0;
  cudaStream_t st = nullptr;
  int hidden = 0, max_tokens = 0;
  std::uint64_t seed = 0;
  int* d_tok = nullptr;
  std::unique_ptr<moa::GpuMetricQ> ev;
  ~moa_mq_group() {
    ev.reset();
    if (d_tok) cudaFree(d_tok);
    if (st) cudaStreamDestroy(st);
  }
};

namespace {
void fill_quality(const moa::QualityScore& qs, moa_quality* out, double* sim, int sim_cap) {
  if (out) {
    out->outputs = qs.outputs;
    out->c = qs.confidences.back();
    out->c_bar = qs.c_bar;
    out->weight_sum = qs.weight_sum;
    out->weighted = qs.weighted;
    out->calibrated = qs.calibrated;
    out->q = qs.q;
    out->tau = qs.tau;
  }
  if (sim && sim_cap >= static_cast<int>(qs.sim.size()))
    std::memcpy(sim, qs.sim.data(), sizeof(double) * qs.sim.size());
}

void check_group_input(const moa_mq_group* g, const double* logprobs, int n) {
  if (!g) throw moa::ValidationError("metricq: null group");
  need(logprobs, "logprobs");
  if (n <= 0) throw moa::ValidationError("logprobs: need at least one token");
  if (n > g->max_tokens) throw moa::ValidationError("metricq: completion longer than the evaluator capacity");
}
}  // namespace

extern "C" {

int moa_mq_group_create(int hidden, uint64_t provider_seed, double tau, int include_diagonal, int max_members,
                        int max_tokens, int device, moa_mq_group** out) {
  return guard([&] {
    need(out, "out");
    if (max_members <= 0 || max_tokens <= 0)
      throw moa::ValidationError("metricq: max_members and max_tokens must be > 0");
    MOA_CUDA(cudaSetDevice(device));
    auto g = std::make_unique<moa_mq_group>();
    g->device = device;
    g->hidden = hidden;
    g->max_tokens = max_tokens;
    g->seed = provider_seed;
    MOA_CUDA(cudaStreamCreateWithFlags(&g->st, cudaStreamNonBlocking));
    MOA_CUDA(cudaMalloc(&g->d_tok, sizeof(int) * max_tokens));
    g->ev = std::make_unique<moa::GpuMetricQ>(hidden, provider_seed, tau, include_diagonal != 0, max_members,
                                              max_tokens, g->st);
    *out = g.release();
  });
}

int moa_mq_group_add_completion(moa_mq_group* g, const int32_t* tokens, const double* logprobs, int n,
                                moa_quality* out, double* sim, int sim_cap) {
  return guard([&] {
    check_group_input(g, logprobs, n);
    need(tokens, "tokens");
    const double c = moa::geometric_mean_confidence(std::vector<double>(logprobs, logprobs + n));
    MOA_CUDA(cudaSetDevice(g->device));
    MOA_CUDA(cudaMemcpyAsync(g->d_tok, tokens, sizeof(int) * n, cudaMemcpyHostToDevice, g->st));
    moa::k::ee_mock_embed(g->d_tok, 0, n, g->hidden, g->seed, g->ev->emb_buffer(), g->st);
    fill_quality(g->ev->add_completion_conf(c, n), out, sim, sim_cap);
  });
}

int moa_mq_group_add_embedded(moa_mq_group* g, const double* emb, const double* logprobs, int n, moa_quality* out,
                              double* sim, int sim_cap) {
  return guard([&] {
    check_group_input(g, logprobs, n);
    need(emb, "emb");
    const double c = moa::geometric_mean_confidence(std::vector<double>(logprobs, logprobs + n));
    MOA_CUDA(cudaSetDevice(g->device));
    MOA_CUDA(cudaMemcpyAsync(g->ev->emb_buffer(), emb, sizeof(double) * n * g->hidden, cudaMemcpyHostToDevice,
                             g->st));
    fill_quality(g->ev->add_completion_conf(c, n), out, sim, sim_cap);
  });
}

int moa_mq_group_completions(const moa_mq_group* g, int* n) {
  return guard([&] {
    need(n, "n");
    if (!g) throw moa::ValidationError("metricq: null group");
    *n = g->ev->completions();
  });
}

int moa_mq_group_free(moa_mq_group* g) {
  return guard([&] { delete g; });
}

int moa_rng_derive(uint64_t master, const char* label, uint64_t* state) {
  return guard([&] {
    need(label, "label");
    need(state, "state");
    *state = moa::rng::Stream::derive(master, label).state();
  });
}

int moa_decide_exit(double q, uint64_t* state, double* draw, int* exited) {
  return guard([&] {
    need(state, "state");
    moa::rng::Stream s(*state);
    const moa::ExitDecision d = moa::decide_exit(q, s);
    *state = s.state();
    if (draw) *draw = d.draw;
    if (exited) *exited = d.exited ? 1 : 0;
  });
}

int moa_metricq_run(const int32_t* tokens, const float* logprobs, const int* lens, int m, int hidden, uint64_t seed,
                    double tau, int include_diagonal, uint64_t master, const char* label, double* out6,
                    double* draw, int* exited, double* sim_out, int device) {
  return guard([&] {
    need(lens, "lens");
    need(label, "label");
    if (m <= 0) throw moa::ValidationError("metricq: need at least one completion");
    long long total = 0;
    int maxn = 0;
    for (int i = 0; i < m; ++i) {
      if (lens[i] <= 0) throw moa::ValidationError("logprobs: need at least one token");
      total += lens[i];
      maxn = std::max(maxn, lens[i]);
    }
    need(tokens, "tokens");
    need(logprobs, "logprobs");
    MOA_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    MOA_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    int* d_tok = nullptr;
    float* d_lp = nullptr;
    MOA_CUDA(cudaMalloc(&d_tok, sizeof(int) * total));
    MOA_CUDA(cudaMalloc(&d_lp, sizeof(float) * total));
    MOA_CUDA(cudaMemcpy(d_tok, tokens, sizeof(int) * total, cudaMemcpyHostToDevice));
    MOA_CUDA(cudaMemcpy(d_lp, logprobs, sizeof(float) * total, cudaMemcpyHostToDevice));
    {
      moa::GpuMetricQ ev(hidden, seed, tau, include_diagonal != 0, m, maxn, st);
      moa::rng::Stream s = moa::rng::Stream::derive(master, label);
      long long base = 0;
      moa::QualityScore qs;
      for (int i = 0; i < m; ++i) {
        qs = ev.add_completion(d_tok, d_lp, base, lens[i]);
        base += lens[i];
        const moa::ExitDecision d = moa::decide_exit(qs.q, s);
        if (out6) {
          double* o = out6 + 6 * i;
          o[0] = qs.confidences.back();
          o[1] = qs.c_bar;
          o[2] = qs.weight_sum;
          o[3] = qs.weighted;
          o[4] = qs.calibrated;
          o[5] = qs.q;
        }
        if (draw) draw[i] = d.draw;
        if (exited) exited[i] = d.exited ? 1 : 0;
      }
      if (sim_out) std::memcpy(sim_out, qs.sim.data(), sizeof(double) * qs.sim.size());
    }
    cudaFree(d_tok);
    cudaFree(d_lp);
    cudaStreamDestroy(st);
  });
}

int moa_topology(int kind, int n_layers, const int* widths, const int* cluster_sizes, int* pre_off, int* pre,
                 int cap) {
  return guard([&] {
    moa::Topology t = topology_of(kind, n_layers, widths, cluster_sizes);
    std::map<moa::AgentId, int> index;
    int k = 0;
    for (const auto& layer : t.layers())
      for (const auto& a : layer) index[a] = k++;
    int n = 0, i = 0;
    for (const auto& layer : t.layers())
      for (const auto& a : layer) {
        if (pre_off) pre_off[i] = n;
        for (const auto& p : t.precursors(a)) {
          if (pre && n < cap) pre[n] = index.at(p);
          ++n;
        }
        ++i;
      }
    if (pre_off) pre_off[i] = n;
  });
}

int moa_slotplan_create(int self_layer, int self_position, const int32_t* prefix, int n_prefix, const int* slot_layer,
                        const int* slot_position, const int32_t* sep_tokens, const int* sep_lens, int n_slots,
                        const int32_t* suffix, int n_suffix, int incremental, moa_slotplan** out) {
  return guard([&] {
    need(out, "out");
    std::vector<moa::Slot> slots;
    int off = 0;
    for (int i = 0; i < n_slots; ++i) {
      const int len = sep_lens ? sep_lens[i] : 0;
      slots.push_back(moa::Slot{moa::AgentId{slot_layer[i], slot_position[i]},
                                moa::TokenSeq(sep_tokens + off, sep_tokens + off + len)});
      off += len;
    }
    moa::PromptTemplate t(moa::TokenSeq(prefix, prefix + n_prefix), slots, moa::TokenSeq(suffix, suffix + n_suffix));
    *out = new moa_slotplan{moa::SlotPlan(moa::AgentId{self_layer, self_position}, t, incremental != 0)};
  });
}

int moa_slotplan_event(moa_slotplan* p, int op, int layer, int position, const int32_t* tokens, int n, int32_t* buf,
                       int cap, int* n_words) {
  return guard([&] {
    need(p, "plan");
    std::vector<moa::RouteAction> acts;
    const moa::AgentId who{layer, position};
    switch (op) {
      case 0: acts = p->plan.start(); break;
      case 1: acts = p->plan.on_chunk(who, moa::TokenSeq(tokens, tokens + n)); break;
      case 2: acts = p->plan.on_precursor_done(who); break;
      case 3: acts = p->plan.on_precursor_cancelled(who); break;
      default: throw moa::ValidationError("slotplan: unknown op");
    }
    int w = 0;
    auto put = [&](int32_t v) {
      if (buf && w < cap) buf[w] = v;
      ++w;
    };
    for (const auto& a : acts) {
      put(a.kind == moa::RouteAction::Kind::PrefillOnly ? 0 : a.kind == moa::RouteAction::Kind::Generate ? 1 : 2);
      put(a.start);
      put(static_cast<int32_t>(a.tokens.size()));
      for (auto t : a.tokens) put(t);
    }
    if (n_words) *n_words = w;
  });
}

int moa_slotplan_free(moa_slotplan* p) {
  return guard([&] { delete p; });
}

int moa_k_attention(uintptr_t q, uintptr_t rows, int R, uintptr_t meta, int nh, int nkv, int hd, uintptr_t kpool,
                    uintptr_t vpool, long long kv_stride, int max_ctx, uintptr_t out, int prefill, uintptr_t stream,
                    int slots) {
  return guard([&] {
    if ((hd != 64 && hd != 128) || nh % nkv || R <= 0) throw moa::ValidationError("attention: unsupported shape");
    const auto st = reinterpret_cast<cudaStream_t>(stream);
    const auto* qp = reinterpret_cast<const moa::k::bf16*>(q);
    const auto* rp = reinterpret_cast<const moa::k::RowDesc*>(rows);
    const auto* mp = reinterpret_cast<const int*>(meta);
    const auto* kp = reinterpret_cast<const moa::k::bf16*>(kpool);
    const auto* vp = reinterpret_cast<const moa::k::bf16*>(vpool);
    auto* op = reinterpret_cast<moa::k::bf16*>(out);
    const bool tma = (prefill & 2) != 0;  // bit 1: the TMA-staged per-row kernel
    const bool cluster = (prefill & 4) != 0;  // bit 2: the cluster-split kernel, splits = bits 8-15 (0: heuristic)
    const bool pf_tc = (prefill & 8) != 0;    // bit 3 (with bit 0): the runs by the tcgen05 prefill kernel
    const bool runs_only = (prefill & 16) != 0;  // bit 4 (with bit 0): no per-row kernel (timing the runs)
    const int ns_req = (prefill >> 8) & 0xff;
    const int ks_req = std::max(1, (prefill >> 16) & 0xff);  // bits 16-23: key splits of the tcgen05 prefill kernel
    prefill &= 1;
    if (prefill && pf_tc) {
      if (!moa::k::attention_prefill_tc_supported(nh, nkv, hd)) throw moa::ValidationError("attention: tcgen05 prefill shape");
      const long long pool_rows = static_cast<long long>(slots) * kv_stride / hd;
      moa::k::TmaMap qm, km, vm;
      if (!moa::k::make_tmap_q3d(&qm, qp, R, nh, hd, nh / nkv) || !moa::k::make_tmap_bf16(&km, kp, pool_rows, hd, 64) ||
          !moa::k::make_tmap_bf16(&vm, vp, pool_rows, hd, 64))
        throw moa::DeviceError("attention: TMA map creation failed");
      static float* pws = nullptr;
      if (ks_req > 1 && !pws) MOA_CUDA(cudaMalloc(&pws, sizeof(float) * moa::k::attention_prefill_tc_ws_floats(128)));
      const int P = 128 / (nh / nkv);
      if (ks_req > 8 || (R + P - 1) / P * nkv * ks_req > moa::k::kPfTcMaxCtas)
        throw moa::ValidationError("attention: key splits exceed the workspace");
      moa::k::attention_prefill_tc(qm, km, vm, rp, R, mp, nh, nkv, hd, kv_stride, 0, max_ctx, op, st, ks_req, pws);
    } else if (prefill) {
      moa::k::attention_prefill(qp, rp, R, mp, nh, nkv, hd, kp, vp, kv_stride, 0, max_ctx, op, st);
    }
    if (prefill && runs_only) {
      MOA_CUDA(cudaStreamSynchronize(st));
    } else if (cluster) {
      const long long pool_rows = static_cast<long long>(slots) * kv_stride / hd;
      moa::k::TmaMap km, vm;
      if (!moa::k::make_tmap_bf16(&km, kp, pool_rows, hd, 64) || !moa::k::make_tmap_bf16(&vm, vp, pool_rows, hd, 64))
        throw moa::DeviceError("attention: TMA map creation failed");
      if (ns_req > 16 || (ns_req & (ns_req - 1))) throw moa::ValidationError("attention: splits must be 1, 2, 4, 8 or 16");
      const int ns = ns_req ? ns_req : moa::k::attention_decode_cluster_splits(R, nkv, (max_ctx + 63) / 64);
      moa::k::attention_decode_cluster(km, vm, qp, rp, R, ns, mp, nh, nkv, hd, kv_stride, 0, max_ctx, op, st,
                                       prefill != 0);
      MOA_CUDA(cudaStreamSynchronize(st));
    } else {  // prefill: the per-row kernel takes the rows alone in their run
      float* ws = nullptr;
      int* cnt = nullptr;
      MOA_CUDA(cudaMalloc(&ws, sizeof(float) * moa::k::attention_ws_floats(R, nh, hd, max_ctx)));
      MOA_CUDA(cudaMalloc(&cnt, sizeof(int) * R * nh));
      MOA_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * R * nh, st));
      const int ks = tma ? moa::k::attention_decode_tma_keys(hd) : moa::k::kv_split(hd);
      int ns = 1;
      while (ns * ks < max_ctx) ns <<= 1;
      if (tma) {
        // the pools hold `slots` agents of one layer
        const long long pool_rows = static_cast<long long>(slots) * kv_stride / hd;
        moa::k::TmaMap km, vm;
        if (!moa::k::make_tmap_bf16(&km, kp, pool_rows, hd, 64) || !moa::k::make_tmap_bf16(&vm, vp, pool_rows, hd, 64))
          throw moa::DeviceError("attention: TMA map creation failed");
        moa::k::attention_decode_tma(km, vm, qp, rp, R, ns, mp, nh, nkv, hd, kv_stride, 0, max_ctx, op, ws, cnt, st,
                                     prefill != 0);
      } else {
        moa::k::attention(qp, rp, R, ns, mp, nh, nkv, hd, kp, vp, kv_stride, 0, max_ctx, op, ws, cnt, st,
                          prefill != 0);
      }
      MOA_CUDA(cudaStreamSynchronize(st));
      cudaFree(ws);
      cudaFree(cnt);
    }
    MOA_CUDA(cudaGetLastError());
  });
}

int moa_k_gemv(uintptr_t A, uintptr_t X, int R, uintptr_t W, int N, int K, uintptr_t out, uintptr_t stream) {
  return guard([&] {
    if (K % 256) throw moa::ValidationError("gemv: K must be a multiple of 256");
    if ((A == 0) == (X == 0)) throw moa::ValidationError("gemv: exactly one of A (bf16) / X (fp32, normed) is required");
    moa::k::GemvArgs a;
    a.A = reinterpret_cast<const moa::k::bf16*>(A);
    a.X = reinterpret_cast<const float*>(X);
    a.R = R;
    a.N = N;
    a.K = K;
    a.W = reinterpret_cast<const moa::k::bf16*>(W);
    a.epi = moa::k::kEpiF32;
    a.out = reinterpret_cast<float*>(out);
    moa::k::gemv(a, reinterpret_cast<cudaStream_t>(stream));
    MOA_CUDA(cudaGetLastError());
  });
}

int moa_k_gemm_tc(uintptr_t A, int M, uintptr_t W, int N, int K, uintptr_t out, uintptr_t stream) {
  return guard([&] {
    if (!moa::k::gemm_tc_supported(N, K)) throw moa::ValidationError("gemm_tc: needs N % 128 == 0 and K % 64 == 0");
    if (M <= 0) return;
    moa::k::TmaMap ma, mw;
    if (!moa::k::make_tmap_bf16(&ma, reinterpret_cast<const moa::k::bf16*>(A), M, K, 128) ||
        !moa::k::make_tmap_bf16(&mw, reinterpret_cast<const moa::k::bf16*>(W), N, K, 128))
      throw moa::DeviceError("gemm_tc: cuTensorMapEncodeTiled failed");
    moa::k::GemvArgs a;
    a.R = M;
    a.N = N;
    a.K = K;
    a.epi = moa::k::kEpiF32;
    a.out = reinterpret_cast<float*>(out);
    moa::k::gemm_tc(ma, mw, a, reinterpret_cast<cudaStream_t>(stream));
    MOA_CUDA(cudaGetLastError());
  });
}

int moa_k_noop(uintptr_t p, int ctas, uintptr_t stream) {
  return guard([&] { moa::k::noop_chain_link(reinterpret_cast<int*>(p), ctas, reinterpret_cast<cudaStream_t>(stream)); });
}

int moa_k_chain_stamp(uintptr_t buf) {
  return guard([&] {
    moa::k::forward_chain_stamp(reinterpret_cast<unsigned long long*>(buf));
    moa::k::gemv_tc_chain_stamp(reinterpret_cast<unsigned long long*>(buf));
    moa::k::gemm_tc_chain_stamp(reinterpret_cast<unsigned long long*>(buf));
    moa::k::attn_decode_chain_stamp(reinterpret_cast<unsigned long long*>(buf));
    moa::k::attn_prefill_tc_chain_stamp(reinterpret_cast<unsigned long long*>(buf));
  });
}

int moa_k_gemv_tc(uintptr_t A, int R, uintptr_t W, int N, int K, uintptr_t out, uintptr_t stream) {
  return guard([&] {
    moa::k::GemvArgs a;
    a.R = R;
    a.N = N;
    a.K = K;
    a.epi = moa::k::kEpiF32;
    a.out = reinterpret_cast<float*>(out);
    if (R <= 0 || R > moa::k::kGemvTcWideRows || K % 64 || N % 2)
      throw moa::ValidationError("gemv_tc: needs 1 <= R <= 64, K % 64 == 0, even N");
    // A holds 16, 32 or 64 rows (R <= 16 / 32 / 64), the activation tile's box
    const int arows = moa::k::gemv_tc_box_rows(R);
    moa::k::TmaMap mw, mx;
    if (!moa::k::make_tmap_bf16(&mw, reinterpret_cast<const moa::k::bf16*>(W), N, K, 128) ||
        !moa::k::make_tmap_bf16(&mx, reinterpret_cast<const moa::k::bf16*>(A), arows, K, arows))
      throw moa::DeviceError("gemv_tc: cuTensorMapEncodeTiled failed");
    static float* ws = nullptr;
    static int* cnt = nullptr;
    static long long ws_cap = 0, cnt_cap = 0;
    const long long need = moa::k::gemv_tc_ws_floats(N, K), tiles = (N + 127) / 128;
    if (need > ws_cap) {
      if (ws) cudaFree(ws);
      MOA_CUDA(cudaMalloc(&ws, sizeof(float) * need));
      ws_cap = need;
    }
    if (tiles > cnt_cap) {
      if (cnt) cudaFree(cnt);
      MOA_CUDA(cudaMalloc(&cnt, sizeof(int) * tiles));
      MOA_CUDA(cudaMemset(cnt, 0, sizeof(int) * tiles));
      cnt_cap = tiles;
    }
    moa::k::gemv_tc(mw, mx, a, ws, cnt, reinterpret_cast<cudaStream_t>(stream));
    MOA_CUDA(cudaGetLastError());
  });
}

int moa_k_init_uniform(uintptr_t dst, long long rows, long long cols, uint64_t base, float scale, int row_map, int hd,
                       uintptr_t stream) {
  return guard([&] {
    moa::k::init_uniform_rows(reinterpret_cast<moa::k::bf16*>(dst), rows, cols, base, scale, row_map, hd,
                              reinterpret_cast<cudaStream_t>(stream));
    MOA_CUDA(cudaGetLastError());
  });
}

}  // extern "C"
