// GpuEngine: the reference's SimWorld engine protocol (pdsim.hpp:61-156) with
// real agents on the GPU.  Requests grow by contiguous prefill_only appends
// and are sealed by generate; decode is greedy; decoded tokens land in the
// agent's output cache and are announced every apc_chunk tokens.
//
// Time is the engine *tick* (one batched forward per model over every runnable
// row); DESIGN.md §5 / oracle/engine.py state the tick contract this class
// must reproduce exactly.  Generated tokens stay on the device: the host
// handles them as symbolic ids (ref(slot, k) < 0) that the kernels resolve,
// so scheduling never waits for the GPU except at early-exit evaluations.
#pragma once

#include <cuda_runtime.h>

#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <vector>

#include "common.hpp"
#include "comm.hpp"
#include "metricq.hpp"
#include "model.hpp"

namespace moa {

struct EngineOptions {
  int max_ctx = 4096;     // KV positions per agent
  int max_out = 4096;     // output tokens per agent
  int max_rows = 16384;   // rows per model per tick
  int device = 0;
  bool keep_logits = false;  // debug: keep fp32 logits of every produced token
  bool time_ticks = true;    // record a CUDA event after every tick
  bool tensor_cores = true;  // tcgen05 GEMMs for ticks with >= 128 rows of a model (else GEMV only)
};

struct PrefillInterval {
  int tick, begin, end;
};

struct AgentRecord {
  AgentId id;
  int model = 0;
  bool invoked = false, pruned = false, empty_input = false;
  int submit_tick = 0, precursor_ready_tick = 0;
  int prompt_tokens = 0, output_tokens = 0;
  int prefill_only_calls = 0, recomputed_tokens = 0, reclaimed_tokens = 0, wasted_prefill_tokens = 0;
  int decode_start = -1, decode_end = -1, complete = -1;
  std::vector<PrefillInterval> prefill;
};

struct EngineEvent {
  enum Kind { Chunk = 1, DecodeEnd = 2, Cancel = 3, Reclaim = 4 };
  int kind;
  int tick;
  AgentId agent;
  int a, b;  // chunk [a, b); decode_end (n, 0); cancel (emitted, 0); reclaim (keep, 0)
};

class GpuEngine {
 public:
  using ChunkFn = std::function<void(int begin, int end, const TokenSeq& tokens)>;
  using EndFn = std::function<void(int tick)>;

  GpuEngine(std::vector<ModelSpec> models, std::vector<int> agents_per_model, EngineOptions opt);
  ~GpuEngine();
  GpuEngine(const GpuEngine&) = delete;
  GpuEngine& operator=(const GpuEngine&) = delete;

  // ---- SimWorld protocol ----
  // owner = rank that computes the agent (-1: this rank).  Every rank
  // registers every agent in the same order (replicated control plane);
  // only owned agents bind KV and contribute rows to the forwards.
  void add_agent(const AgentId& id, int model, int owner = -1);
  // Tree-partitioned serving: chunks of an agent's output are sent by its
  // owner to every other rank (NCCL P2P) into the same output-cache slots.
  void attach_comm(std::unique_ptr<PeerComm> comm);
  // Ranks (bit mask) that receive the agent's chunks; default every rank.  The
  // caller narrows it to the ranks that consume them (identically on every
  // rank: sender and receivers must agree).
  void set_chunk_dests(const AgentId& id, std::uint64_t ranks);
  int rank() const { return comm_ ? comm_->rank() : 0; }
  int world() const { return comm_ ? comm_->world() : 1; }
  bool is_local(const AgentId& id) const { return req(id).local; }
  void submit_prefill_only(const AgentId& id, int expected_start, const TokenSeq& tokens);
  void submit_generate(const AgentId& id, const TokenSeq& full_prompt, int max_new, int apc_chunk,
                       int prefill_chunk = 0);
  void cancel(const AgentId& id);
  void reclaim(const AgentId& id, int keep);
  void on_chunk(const AgentId& id, ChunkFn fn);
  void on_decode_end(const AgentId& id, EndFn fn);
  void defer(std::function<void()> fn) { deferred_.push_back(std::move(fn)); }
  void note_precursor_ready(const AgentId& id);
  void mark_empty_input(const AgentId& id);

  bool busy() const;
  void step();
  void run(int max_ticks = 1 << 22);
  // Drop every request (device buffers and weights stay resident).
  void reset();
  int tick() const { return tick_; }

  // ---- introspection / readback ----
  bool has(const AgentId& id) const { return reqs_.count(id) > 0; }
  bool finished(const AgentId& id) const { return req(id).finished; }
  bool cancelled(const AgentId& id) const { return req(id).cancelled; }
  int decoded(const AgentId& id) const { return req(id).n_out; }
  int slot_of(const AgentId& id) const { return req(id).slot; }
  const TokenSeq& prompt(const AgentId& id) const { return req(id).prompt; }
  const AgentRecord& record(const AgentId& id) const { return req(id).rec; }
  const std::vector<AgentId>& order() const { return order_; }
  const std::vector<EngineEvent>& events() const { return events_; }
  void clear_events() { events_.clear(); }

  Token ref(int slot, int k) const { return static_cast<Token>(-1 - (slot * opt_.max_out + k)); }
  // Literal token values for a (possibly symbolic) sequence; synchronises.
  TokenSeq resolve(const TokenSeq& seq);
  // Copies the first n outputs of an agent to host (synchronises).
  void read_outputs(const AgentId& id, int n, int* tok, float* lp, float* ent);
  void read_logits(const AgentId& id, int k, float* dst);  // keep_logits only

  cudaStream_t stream() const { return stream_; }
  int device() const { return opt_.device; }
  const int* d_out_tok() const { return out_tok_; }
  const float* d_out_lp() const { return out_lp_; }
  long long out_offset(const AgentId& id) const { return static_cast<long long>(req(id).slot) * opt_.max_out; }
  const EngineOptions& options() const { return opt_; }
  DeviceModel& model(int m) { return *models_[static_cast<std::size_t>(m)]; }
  int n_models() const { return static_cast<int>(models_.size()); }
  // Kernel probes (bench roofline): attach to every model; stats after a run.
  void set_probing(bool on);
  void probe_stats(int kind, int* count, double* ms, double* bytes, double* flops);
  // Pooled early-exit evaluator #i (device buffers reused across requests).
  GpuMetricQ& ee_evaluator(int i, int hidden, std::uint64_t seed, double tau, bool diag, int members,
                           int max_tokens);
  // Hidden-state embedding provider: the first n output tokens of `src` run
  // through model `m` (positions 0..n-1 in a KV slot reserved for this duty),
  // and the final residual rows, RMS-normalised in fp64, land in the
  // evaluator's embedding buffer.  Runs on the engine stream between ticks.
  void hidden_embed(int m, const AgentId& src, int n, GpuMetricQ& ev);

  // Timing: event recorded at run start / after a tick (time_ticks).
  void mark_start();
  double ms_since_start(int tick);  // synchronises on that tick's event (completion ticks / tracing)
  double bytes_moved() const { return weight_bytes_; }
  long long rows_processed() const { return rows_total_; }
  int kernel_forwards() const { return forwards_; }
  int overlapped_ticks() const { return overlapped_ticks_; }
  // RunTrace timestamps: run_query reads every tick's device time (synchronises)
  void set_tracing(bool on) { tracing_ = on; }
  bool tracing() const { return tracing_; }  // ticks whose model forwards ran on parallel streams
  double host_ms() const { return host_ms_; }  // host time spent inside step() (incl. EE syncs)
  double host_api_ms() const { return host_api_ms_; }    // of which: uploads + graph launches
  double host_wait_ms() const { return host_wait_ms_; }  // of which: blocked on the staging ring (GPU behind)

 private:
  struct Job {
    int b, e;
  };
  struct Req {
    AgentId id;
    int model = 0, slot = 0, kv = 0, owner = 0;
    bool local = true;
    std::uint64_t dests = ~0ULL;  // ranks receiving this agent's chunks
    TokenSeq prompt;
    int prefilled = 0, max_computed = 0;
    std::uint64_t gen = 0;
    std::deque<Job> queue;
    bool gen_pending = false, dec_started = false, finished = false, cancelled = false;
    int max_new = 0, apc = 0, n_out = 0, chunk_begin = 0;
    std::vector<ChunkFn> chunk_fns;
    std::vector<EndFn> end_fns;
    AgentRecord rec;
  };
  Req& req(const AgentId& id);
  const Req& req(const AgentId& id) const;
  void start_decode(Req& r, int n_out);
  void check_tokens(const Req& r, const TokenSeq& tokens, std::size_t from) const;
  void upload_and_forward(int m, const std::vector<k::RowDesc>& rows, const std::vector<int>& lsel,
                          const std::vector<int>& lout, cudaStream_t st);
  void upload_and_forward_run(int m, int K, const std::vector<k::RowDesc>& rows, const std::vector<int>& lout,
                              cudaStream_t st);

  EngineOptions opt_;
  std::unique_ptr<PeerComm> comm_;
  cudaStream_t stream_ = nullptr;
  // per-model streams: forwards of different models in one tick run side by side
  std::vector<cudaStream_t> mstreams_;
  std::vector<cudaEvent_t> mdone_;
  cudaEvent_t tick_fork_ = nullptr;
  // tick metadata uploads run on a copy stream per model into the blob the
  // previous tick is not reading, so the copy overlaps that tick's forward
  std::vector<cudaStream_t> cstreams_;
  std::vector<cudaEvent_t> blob_free_, blob_ready_;  // [model][2]
  bool async_upload_ = true;
  std::vector<cudaEvent_t> run_free_, run_ready_;  // [model][2] decode-run blobs
  std::vector<int> run_par_;
  int max_run_ = DeviceModel::kMaxRun;  // MOA_DECODE_RUN=K (1: off)
  bool in_run_ = false;                 // inside run(): decode runs allowed
  bool overlap_models_ = true;
  bool tracing_ = false;
  std::map<int, int> embed_kv_;  // model -> reserved KV slot of the hidden-state provider
  int overlapped_ticks_ = 0;
  std::vector<std::unique_ptr<DeviceModel>> models_;
  std::map<AgentId, Req> reqs_;
  std::vector<AgentId> order_;
  std::deque<std::function<void()>> deferred_;
  std::vector<EngineEvent> events_;
  int tick_ = 0;
  int slots_ = 0, max_slots_ = 0;
  // device output cache [slot][max_out]
  int* out_tok_ = nullptr;
  float* out_lp_ = nullptr;
  float* out_ent_ = nullptr;
  float* logits_ = nullptr;  // keep_logits: [slot][max_out][V_max]
  float* logits_scratch_ = nullptr;
  int logits_v_ = 0;
  // pinned staging ring for row descriptors
  struct Staging {
    char* host = nullptr;
    cudaEvent_t done = nullptr;
  };
  std::vector<Staging> ring_;
  std::vector<std::unique_ptr<GpuMetricQ>> ee_pool_;
  KernelProbes probes_;
  bool probing_ = false;
  std::size_t ring_next_ = 0, ring_bytes_ = 0;
  // timing
  cudaEvent_t start_ev_ = nullptr;
  std::vector<cudaEvent_t> tick_ev_;
  std::vector<char> tick_timed_;  // tick_ev_[t] recorded (completion ticks, or every tick while tracing)
  double weight_bytes_ = 0.0;
  long long rows_total_ = 0;
  int forwards_ = 0;
  double host_ms_ = 0.0, host_api_ms_ = 0.0, host_wait_ms_ = 0.0;
};

}  // namespace moa
