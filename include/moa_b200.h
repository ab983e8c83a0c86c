/*
 * moa_b200.h -- C-ABI of the B200 Faster-MoA agent-execution hot path.
 *
 * Drop-in boundary for the reference's proj/core path (arXiv 2512.18126,
 * "moaserve").  Plain C types only: caller-owned host buffers in, results
 * copied into caller buffers out; the engine owns weights, KV caches and
 * generated tokens on the GPU.  Every function returns a status code
 * (MOA_OK on success); moa_last_error() returns the thread-local message of
 * the last failure.  Status codes map onto the reference's error types
 * (errors.hpp:10-33): MOA_ERR_VALIDATION = ValidationError (CLI exit 2),
 * MOA_ERR_RUNTIME = RunError (CLI exit 3).
 *
 * Reference interfaces replaced (file:line under /root/reference/proj):
 *   engine protocol   SimWorld            core/include/moaserve/pdsim.hpp:61-156
 *   request entry     run_query           core/include/moaserve/orchestrator.hpp:57
 *   early-exit        MetricQEvaluator    core/include/moaserve/metricq.hpp:25-122
 *   embedding plugin  EmbeddingProvider   core/include/moaserve/embedding.hpp:38-44
 *   routing           Topology / SlotPlan core/include/moaserve/topology.hpp:28-80,
 *                                         core/include/moaserve/router.hpp:36-90
 * INTEGRATION.md shows the C++ adapter a maintainer adds on the reference side.
 */
#ifndef MOA_B200_H
#define MOA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MOA_OK 0
#define MOA_ERR_VALIDATION 2 /* ValidationError (errors.hpp:10-13)            */
#define MOA_ERR_RUNTIME 3    /* RunError        (errors.hpp:17-20)            */
#define MOA_ERR_DEVICE 4     /* CUDA failure (a RunError on the reference side) */
#define MOA_ERR_UNSUPPORTED 5
/* ProviderError kinds (errors.hpp:24-33), raised by an EmbeddingProvider */
#define MOA_ERR_PROVIDER_TRANSPORT 6
#define MOA_ERR_PROVIDER_CREDENTIALS 7
#define MOA_ERR_PROVIDER_BAD_RESPONSE 8

typedef struct moa_engine moa_engine;
typedef struct moa_query moa_query;
typedef struct moa_slotplan moa_slotplan;

const char* moa_last_error(void);
const char* moa_version(void);
int moa_device_count(int* n);

/* ---- engine lifecycle ------------------------------------------------- */

/* One agent model (builder-chosen Llama-style shape; random uniform-hash
 * init from (seed, tag) -- bit-identical with oracle/model.py). */
typedef struct {
  char tag[32];
  int d, n_layers, n_heads, n_kv_heads, head_dim, ffn, vocab;
  double rope_theta, norm_eps, lm_gain;
  uint64_t seed;
  int max_agents; /* agents that may bind this model at once */
} moa_model_spec;

typedef struct {
  int max_ctx;     /* KV positions per agent                 */
  int max_out;     /* output tokens per agent                */
  int max_rows;    /* rows per tick (prefill budget)         */
  int device;      /* CUDA device ordinal                    */
  int keep_logits; /* debug: retain fp32 logits per token    */
  int gemv_only;   /* 1: never use the tcgen05 prefill GEMM  */
} moa_engine_opts;

int moa_engine_create(const moa_model_spec* models, int n_models, const moa_engine_opts* opts,
                      moa_engine** out);
int moa_engine_destroy(moa_engine* eng);
/* Drops every request; weights and buffers stay resident. */
int moa_engine_reset(moa_engine* eng);
/* Kernel probes: CUDA events around every forward kernel (graphs bypassed)
 * with each launch's algorithmic (unique) bytes and dense flops.  kind:
 * decode regime (rows <= 16): 0 embed, 1 qkv GEMV, 2 per-row attention,
 * 3 o-proj GEMV, 4 gate/up GEMV, 5 down GEMV, 6 LM head, 7 fused small-agent
 * QKV + attention (+ o-proj); prefill regime: 8 tiled prompt attention,
 * 9 qkv GEMM, 10 o-proj GEMM, 11 gate/up GEMM, 12 down GEMM.  flops may be NULL. */
int moa_engine_probe(moa_engine* eng, int enable);
int moa_engine_probe_stats(moa_engine* eng, int kind, int* launches, double* ms, double* bytes, double* flops);

/* ---- tree-partitioned serving over several GPUs (one process per GPU) ----
 * Rank 0 creates the id, the caller broadcasts it (e.g. torch.distributed),
 * every rank attaches before its first request.  run_query then places the
 * agents along the tree (moa_placement), every rank runs the same tick
 * schedule, computes only its own agents, and moves each output chunk from its
 * owner to the other ranks with NCCL P2P. */
int moa_nccl_unique_id(uint8_t* out /* 128 bytes */);
int moa_engine_attach_comm(moa_engine* eng, const uint8_t* id /* 128 bytes */, int rank, int world);
/* Same protocol for several engines inside ONE process (one thread per
 * engine, any devices -- the same GPU included, which NCCL refuses): a hub
 * joins `world` engines, chunk payloads move by device-to-device copy.  Used
 * to run the partitioned engine on a single-GPU box. */
typedef struct moa_loopback moa_loopback;
int moa_loopback_create(int world, moa_loopback** out);
int moa_loopback_destroy(moa_loopback* hub);
int moa_engine_attach_loopback(moa_engine* eng, moa_loopback* hub, int rank);
/* ranks[k] = owning rank of agent k (layer-major order) for `world` GPUs. */
int moa_placement(int kind, int n_layers, const int* widths, const int* cluster_sizes, int world, int* ranks);

/* ---- SimWorld engine protocol (pdsim.hpp:61-156) ------------------------
 * Agents are (layer, position) = AgentId (agent.hpp:16-37).  Tokens passed
 * in are literal ids in [0, vocab).  Time advances by moa_step ticks.      */
int moa_add_agent(moa_engine* eng, int layer, int position, int model);
/* submit_prefill_only (pdsim.cpp:155-174): start must equal the scheduled
 * prompt length (contiguity) or MOA_ERR_RUNTIME. */
int moa_prefill_only(moa_engine* eng, int layer, int position, int start, const int32_t* tokens,
                     int n);
/* submit_generate (pdsim.cpp:176-214): prompt must extend the scheduled
 * prefix; the engine decodes max_new greedy tokens and announces them every
 * apc_chunk tokens.  prefill_chunk > 0 splits the remainder (DpChunkedPrefill). */
int moa_generate(moa_engine* eng, int layer, int position, const int32_t* prompt, int n, int max_new,
                 int apc_chunk, int prefill_chunk);
int moa_cancel(moa_engine* eng, int layer, int position);            /* pdsim.cpp:374-398 */
int moa_reclaim(moa_engine* eng, int layer, int position, int keep); /* pdsim.cpp:400-418 */

#define MOA_EV_CHUNK 1      /* a = begin, b = end (output offsets)   */
#define MOA_EV_DECODE_END 2 /* a = output tokens                     */
#define MOA_EV_CANCEL 3     /* a = tokens emitted before the cancel  */
#define MOA_EV_RECLAIM 4    /* a = keep point                        */
typedef struct {
  int kind, tick, layer, position, a, b;
} moa_event;

/* Runs one engine tick; returns the tick's events (chunk/decode_end/...) and
 * whether work remains.  Chunk tokens are read with moa_read_output. */
int moa_step(moa_engine* eng, moa_event* events, int cap, int* n_events, int* busy);
int moa_busy(moa_engine* eng, int* busy);
/* First n outputs of an agent (tokens, fp32 logprob of the greedy token,
 * fp32 softmax entropy).  Any pointer may be NULL. */
int moa_read_output(moa_engine* eng, int layer, int position, int n, int32_t* tokens, float* logprobs,
                    float* entropy);
/* fp32 logits of output token k (keep_logits engines); cap = floats in
 * `logits`, at least the agent model's vocab (else VALIDATION). */
int moa_read_logits(moa_engine* eng, int layer, int position, int k, float* logits, int cap);
int moa_agent_state(moa_engine* eng, int layer, int position, int* scheduled, int* decoded,
                    int* finished, int* cancelled);

/* ---- run_query (orchestrator.cpp:130-295) ------------------------------ */
#define MOA_TOPO_TREE 0
#define MOA_TOPO_ALL_TO_ALL 1
#define MOA_MODE_SEQUENTIAL_PD 0
#define MOA_MODE_DP_ONLY 1
#define MOA_MODE_DP_CHUNKED_PREFILL 2
#define MOA_MODE_INCREMENTAL_OVERLAP 3
#define MOA_SCOPE_CLUSTER 0
#define MOA_SCOPE_LAYER 1

typedef struct {
  int topo_kind;
  int n_layers;
  const int* widths;        /* [n_layers]                                        */
  const int* cluster_sizes; /* tree: sum(widths[1:]) sizes, layer by layer; NULL = all-to-all */
  const int* model_cycle;   /* concatenated per-layer model-index cycles (config.cpp:252-265) */
  const int* cycle_len;     /* [n_layers]                                        */
  const int* out_lo;        /* [n_layers] output length: fixed (lo == hi) or U(lo, hi) */
  const int* out_hi;
  int mode, early_exit, exit_scope;
  double tau;
  int include_diagonal;
  int use_force_q;
  double force_q;
  int chunk_size;
  uint64_t seed;
  int query_tokens, leaf_prefix_tokens, agg_prefix_tokens, separator_tokens, suffix_tokens;
  int hidden; /* mock embedding width (ProviderSpec::hidden) */
  uint64_t provider_seed;
  int embed_model; /* -1: MockProvider; >= 0: hidden states of this engine model (EmbeddingProvider,
                      embedding.hpp:38-44; width = its d_model) */
  /* Caller-supplied EmbeddingProvider (embedding.hpp:38-44), used when
   * non-NULL (embed_model must be -1): embed_fn(user, tokens, n, hidden, out)
   * fills out[n][hidden] (row-major fp64) with the completion's embedding and
   * returns MOA_OK, or MOA_ERR_PROVIDER_* (the request then fails with that
   * code; moa_last_error reports the provider).  Called on the thread running
   * the request, between engine ticks, once per early-exit evaluation. */
  int (*embed_fn)(void* user, const int32_t* tokens, int n, int hidden, double* out);
  void* embed_user;
  /* OutputLenDist::Empirical (agent.hpp:40-103): out_values_len[l] > 0 makes
   * layer l's output length a uniform draw from the next out_values_len[l]
   * entries of out_values (layers concatenated); NULL / 0 = out_lo..out_hi. */
  const int* out_values;
  const int* out_values_len;
} moa_run_config;

typedef struct {
  int ticks;
  int n_agents;
  int n_evals;
  int forwards;
  long long tokens;         /* output tokens of invoked, unpruned agents */
  long long decoded_tokens; /* every token decoded (incl. pruned partials) */
  long long rows;
  double e2e_ms;       /* device events: first tick -> last completion */
  double wall_ms;      /* host wall clock of the whole call            */
  double weight_bytes; /* weight bytes the forwards had to read        */
  double host_ms;      /* host time spent inside engine ticks          */
  double host_wait_ms; /* of which: blocked on the GPU (staging ring)  */
} moa_run_summary;

typedef struct {
  int layer, position, model;
  int invoked, pruned, empty_input;
  int prompt_tokens, output_tokens;
  int prefill_only_calls, recomputed_tokens, reclaimed_tokens;
  int decode_start, decode_end, complete, precursor_ready;
} moa_agent_record;

typedef struct {
  int tick, group, eval_index, layer, position, evaluated, exited, n_pruned, outputs;
  double q, draw, c, c_bar, weight_sum, weighted, calibrated;
  int pruned_layer[16], pruned_position[16];
} moa_eval_record;

/* resolve != 0 copies literal prompts/outputs back (needed by moa_query_*). */
int moa_run_query(moa_engine* eng, const moa_run_config* cfg, int sample, int resolve,
                  moa_run_summary* summary, moa_query** out /* may be NULL */);
/* Continuous batching: n independent requests (samples[i]) served
 * concurrently by one engine -- each keeps its own prompts, slot plans, exit
 * groups and RNG streams exactly as moa_run_query(samples[i]); their agents
 * share the engine's ticks (one weight pass per model per tick for all of
 * them).  summaries[i] / out[i] (out may be NULL) describe request i; e2e_ms
 * is its own first-tick -> last-completion latency.  The engine needs agent
 * capacity for n requests. */
int moa_run_batch(moa_engine* eng, const moa_run_config* cfg, const int* samples, int n, int resolve,
                  moa_run_summary* summaries, moa_query** out);
/* RunTrace JSONL of a request (reference format, trace.cpp:209-337; times in
 * device seconds since the first tick).  Timestamps need engine tracing on
 * before the request (moa_engine_trace); *len = bytes, written to buf when
 * cap > *len. */
int moa_engine_trace(moa_engine* eng, int enable);
/* Test hook: the fp32 residual rows [rows][d] of model `model`'s last forward
 * (tick row order, before the final RMSNorm) -- per-layer parity checks. */
int moa_read_residual(moa_engine* eng, int model, int rows, float* out, long long cap);
/* Engine clock for protocol-level callers (the HTTP engine service,
 * engine_service.cpp:49-171): mark time zero on the engine stream, then read
 * the device time at the end of a tick (seconds; needs moa_engine_trace on
 * while that tick ran).  moa_agent_record: the engine's record of one agent
 * (ticks of decode start / end, prompt / output sizes). */
int moa_engine_mark_start(moa_engine* eng);
int moa_engine_tick(moa_engine* eng, int* tick); /* ticks run so far (the next tick's index) */
int moa_tick_seconds(moa_engine* eng, int tick, double* seconds);
int moa_agent_record_get(moa_engine* eng, int layer, int position, moa_agent_record* rec);
int moa_query_trace(const moa_query* q, char* buf, long long cap, long long* len);
/* Device time (ms since the request's first tick) at the end of every tick;
 * needs engine tracing (moa_engine_trace).  *n = ticks, min(cap, *n) written. */
int moa_query_ticks(const moa_query* q, double* ms, int cap, int* n);
int moa_query_agent(const moa_query* q, int i, moa_agent_record* rec);
/* which: 0 = prompt, 1 = output. */
int moa_query_tokens(const moa_query* q, int i, int which, int32_t* dst, int cap, int* n);
int moa_query_logprobs(const moa_query* q, int i, float* logprobs, float* entropy, int cap, int* n);
int moa_query_eval(const moa_query* q, int i, moa_eval_record* rec, double* sim_row, int cap);
int moa_query_free(moa_query* q);

/* ---- RunSummary (orchestrator.hpp:59-86, orchestrator.cpp:297-382) ------ */
/* A request trace as summarize reads it (RunTrace after roll_up,
 * trace.hpp:31-124): times in any one unit (the GPU engine reports device
 * seconds).  Activation is keyed by model index (the reference keys it by
 * model_tag; a caller maps tags to indices). */
typedef struct {
  double start, end;
  int wasted;
} moa_prefill_span;
typedef struct {
  int layer, position, model;
  int invoked, pruned;
  int prefill_only_calls, recomputed_tokens;
  double complete_t;
  int n_prefill;
  const moa_prefill_span* prefill;
} moa_trace_agent;
typedef struct {
  double e2e_latency;
  double ee_latency_total;
  int n_agents;
  const moa_trace_agent* agents;
} moa_trace_view;
#define MOA_SUMMARY_MAX_MODELS 16
typedef struct {
  int samples;
  double mean_e2e, p50_e2e, p95_e2e; /* percentile: linear interpolation, orchestrator.cpp:306-314 */
  double mean_ee_share, mean_prefill_only_calls, mean_recomputed_tokens;
  double prefill_share; /* critical_path_prefill_share averaged (orchestrator.cpp:325-350) */
  int n_models;         /* activation rows 0..n_models-1 */
  int instances[MOA_SUMMARY_MAX_MODELS], invoked[MOA_SUMMARY_MAX_MODELS], pruned[MOA_SUMMARY_MAX_MODELS];
  double activation[MOA_SUMMARY_MAX_MODELS]; /* invoked (and not pruned) / instances */
} moa_summary;
/* summarize(cfg, traces) over caller-supplied traces; the topology is given
 * as for moa_topology (kind 0 tree / 1 all-to-all). */
int moa_summarize(int kind, int n_layers, const int* widths, const int* cluster_sizes, const moa_trace_view* traces,
                  int n, moa_summary* out);
/* percentile (orchestrator.cpp:306-314) of v[0..n) at p in [0, 1]. */
int moa_percentile(const double* v, int n, double p, double* out);
/* run_repetitions + summarize on the GPU engine: samples 0..repetitions-1,
 * one request at a time, engine tracing on (per-tick device times), times in
 * device seconds; e2e_latency = first tick -> last completion, ee latency =
 * the time early-exit evaluations held the engine between ticks.
 * per_sample (may be NULL) receives each request's moa_run_summary. */
int moa_run_repetitions(moa_engine* eng, const moa_run_config* cfg, int repetitions, moa_summary* out,
                        moa_run_summary* per_sample);
/* The trace view of a finished request (needs engine tracing while it ran):
 * *n_agents agents written to agents (cap), their prefill spans to spans
 * (span_cap; agents[i].prefill points into spans). */
int moa_query_trace_view(const moa_query* q, moa_trace_view* view, moa_trace_agent* agents, int cap,
                         moa_prefill_span* spans, int span_cap, int* n_agents, int* n_spans);

/* ---- early-exit signals (metricq.hpp:25-122, embedding.cpp:86-120) ------ */
/* MockProvider::embed on the GPU: out[n][hidden] fp64, bit-exact. */
int moa_mock_embed(const int32_t* tokens, int n, int hidden, uint64_t seed, double* out, int device);
/* Incremental MetricQ over m completions (lengths lens[i], concatenated
 * tokens / logprobs), exit draws from RngStream::derive(master, label).
 * Per completion i: out6[i] = {c, c_bar, W, P, B, q}, draw[i], exited[i];
 * sim_out = final m x m similarity matrix (row-major). */
int moa_metricq_run(const int32_t* tokens, const float* logprobs, const int* lens, int m, int hidden,
                    uint64_t seed, double tau, int include_diagonal, uint64_t master, const char* label,
                    double* out6, double* draw, int* exited, double* sim_out, int device);

/* Incremental evaluator handle, one per exit group: MetricQEvaluator
 * (metricq.hpp:102-122, metricq.cpp:148-194) with its state on the GPU.
 * add_completion = MockProvider embeddings (embedding.cpp:86-120) computed on
 * the device from the tokens; add_embedded = rows supplied by any
 * EmbeddingProvider (embedding.hpp:38-44; emb row-major [n][hidden] fp64).
 * logprobs are the reference's TokenLogProbs values (validated: non-empty,
 * finite, <= 0 -> VALIDATION); the confidence is their sequential fp64 mean,
 * exp'd on the host (bit-exact).  After the call `out` holds the group score
 * (QualityScore) and, when sim != NULL and sim_cap >= outputs^2, the grown
 * similarity matrix (row-major).  Groups wider than max_tokens use the n x n
 * cross-Gram route. */
typedef struct moa_mq_group moa_mq_group;
typedef struct {
  int outputs;
  double c; /* this completion's confidence */
  double c_bar, weight_sum, weighted, calibrated, q, tau;
} moa_quality;
int moa_mq_group_create(int hidden, uint64_t provider_seed, double tau, int include_diagonal, int max_members,
                        int max_tokens, int device, moa_mq_group** out);
int moa_mq_group_add_completion(moa_mq_group* g, const int32_t* tokens, const double* logprobs, int n,
                                moa_quality* out, double* sim, int sim_cap);
int moa_mq_group_add_embedded(moa_mq_group* g, const double* emb, const double* logprobs, int n, moa_quality* out,
                              double* sim, int sim_cap);
int moa_mq_group_completions(const moa_mq_group* g, int* n);
int moa_mq_group_free(moa_mq_group* g);
/* RngStream (rng.hpp:46-83): state of derive(master, label); decide_exit
 * (metricq.cpp:125-131) draws next_uniform from *state (advanced) and exits
 * iff draw < q -- add_and_decide = add + decide on the group's stream. */
int moa_rng_derive(uint64_t master, const char* label, uint64_t* state);
int moa_decide_exit(double q, uint64_t* state, double* draw, int* exited);

/* ---- routing (topology.cpp:43-196, router.cpp:9-184) ------------------- */
/* precursor lists: for agent k (layer-major order) pre_off[k]..pre_off[k+1]
 * index into pre (as layer-major agent indices). */
int moa_topology(int kind, int n_layers, const int* widths, const int* cluster_sizes, int* pre_off,
                 int* pre, int cap);
int moa_slotplan_create(int self_layer, int self_position, const int32_t* prefix, int n_prefix,
                        const int* slot_layer, const int* slot_position, const int32_t* sep_tokens,
                        const int* sep_lens, int n_slots, const int32_t* suffix, int n_suffix,
                        int incremental, moa_slotplan** out);
/* op: 0 start, 1 chunk, 2 done, 3 cancelled.  Actions are serialised into
 * buf as [kind, start, n, tokens...]* (kind 0 prefill_only, 1 generate,
 * 2 reclaim); *n_words receives the length. */
int moa_slotplan_event(moa_slotplan* p, int op, int layer, int position, const int32_t* tokens, int n,
                       int32_t* buf, int cap, int* n_words);
int moa_slotplan_free(moa_slotplan* p);

/* ---- kernel entry points (device pointers; tests and profiling) -------- */
/* out[R][N] fp32 = A . W^T with A = bf16 A [R][K], or A = bf16(rmsnorm(X)) for
 * fp32 X (pass 0 for the unused one).  W bf16 [N][K]. */
int moa_k_gemv(uintptr_t A, uintptr_t X, int R, uintptr_t W, int N, int K, uintptr_t out, uintptr_t stream);
/* out[M][N] fp32 = A[M][K] . W[N][K]^T on the tcgen05 tensor cores (TMA, TMEM);
 * N % 128 == 0, K % 64 == 0. */
int moa_k_gemm_tc(uintptr_t A, int M, uintptr_t W, int N, int K, uintptr_t out, uintptr_t stream);
/* Decode GEMV on the tensor cores (swap-AB, split-K): out[R][N] fp32 =
 * A[R][K] . W[N][K]^T for R <= 16; A must have >= 16 allocated rows. */
/* Causal attention over a KV pool (layer 0 of `slots` kv_stride-sized slots): out[R][nh][hd] bf16 from
 * q[R][nh][hd] bf16, rows = moa row descriptors {kv, pos, tok, out}, meta[0] = live rows.  prefill bit 0:
 * the tiled prefill kernel (rows in same-agent runs) + the per-row kernel for rows alone in their run; bit 1:
 * the per-row kernel is the TMA-staged one (attn_decode.cu) instead of the register-staged one; bit 2: the
 * cluster-split kernel (attn_decode.cu) with (prefill >> 8) & 0xff splits (1..16; 0: the engine's choice); bit 3
 * (with bit 0): the runs by the tcgen05 prefill kernel (attn_prefill_tc.cu) instead of the mma.sync one; bit 4
 * (with bit 0): no per-row kernel (rows alone in their run left untouched: timing the prefill kernels);
 * (prefill >> 16) & 0xff (with bits 0 and 3): key splits of the tcgen05 prefill kernel, 1..8 (0: 1), at most
 * 296 CTAs in all (row blocks x kv heads x splits). */
int moa_k_attention(uintptr_t q, uintptr_t rows, int R, uintptr_t meta, int nh, int nkv, int hd, uintptr_t kpool,
                    uintptr_t vpool, long long kv_stride, int max_ctx, uintptr_t out, int prefill, uintptr_t stream,
                    int slots);
int moa_k_noop(uintptr_t p, int ctas, uintptr_t stream); /* trivial PDL kernel: launch-chain cost probe */
int moa_k_chain_stamp(uintptr_t buf); /* debug: decode-chain per-CTA globaltimer stamps (stamp.cuh), 0 = off */
/* Swap-AB tensor-core GEMV out[R][N] = A[:R] . W^T, fp32 out; A holds 16 rows (R <= 16), 32 (17 <= R <= 32)
 * or 64 (33 <= R <= 64: the wide variants the engine runs for incremental-prefill chunks). */
int moa_k_gemv_tc(uintptr_t A, int R, uintptr_t W, int N, int K, uintptr_t out, uintptr_t stream);
/* Hash-uniform weight init of a logical [rows][cols] tensor into a device row
 * layout (0 identity, 1 RoPE-pair interleave per hd rows, 2 even rows, 3 odd rows). */
int moa_k_init_uniform(uintptr_t dst, long long rows, long long cols, uint64_t base, float scale, int row_map, int hd,
                       uintptr_t stream);

#ifdef __cplusplus
}
#endif
#endif /* MOA_B200_H */
