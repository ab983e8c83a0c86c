// Tick engine over the device models.  Protocol checks follow pdsim.cpp
// (cited per method); the tick schedule is the contract in oracle/engine.py.
#include "engine.hpp"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace moa {

namespace {
constexpr int kRing = 64;
}

GpuEngine::GpuEngine(std::vector<ModelSpec> models, std::vector<int> agents_per_model, EngineOptions opt)
    : opt_(opt) {
  if (models.empty()) throw ValidationError("engine: at least one model is required");
  if (agents_per_model.size() != models.size())
    throw ValidationError("engine: one agent capacity per model is required");
  if (opt_.max_ctx <= 0 || opt_.max_out <= 0 || opt_.max_rows <= 0)
    throw ValidationError("engine: max_ctx, max_out and max_rows must be > 0");
  MOA_CUDA(cudaSetDevice(opt_.device));
  MOA_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  for (int c : agents_per_model) max_slots_ += c;
  if (static_cast<long long>(max_slots_) * opt_.max_out >= (1LL << 31))
    throw ValidationError("engine: agents x max_out exceeds the symbolic token range");
  for (std::size_t m = 0; m < models.size(); ++m) {
    const int cap = std::max(1, agents_per_model[m]);
    static const bool graphs = [] {
      const char* e = std::getenv("MOA_GRAPHS");
      return !(e && e[0] == '0');
    }();
    models_.push_back(std::make_unique<DeviceModel>(models[m], cap, opt_.max_ctx, opt_.max_rows + max_slots_,
                                                    max_slots_, stream_, graphs));
    logits_v_ = std::max(logits_v_, models[m].vocab);
    models_.back()->set_tensor_cores(opt_.tensor_cores);
  }
  const long long nout = static_cast<long long>(max_slots_) * opt_.max_out;
  MOA_CUDA(cudaMalloc(&out_tok_, sizeof(int) * nout));
  MOA_CUDA(cudaMalloc(&out_lp_, sizeof(float) * nout));
  MOA_CUDA(cudaMalloc(&out_ent_, sizeof(float) * nout));
  MOA_CUDA(cudaMemsetAsync(out_tok_, 0, sizeof(int) * nout, stream_));
  if (opt_.keep_logits) {
    MOA_CUDA(cudaMalloc(&logits_, sizeof(float) * nout * logits_v_));
    // one scratch region per model: forwards of different models run side by side on their own streams
    MOA_CUDA(cudaMalloc(&logits_scratch_,
                        sizeof(float) * static_cast<long long>(models.size()) * max_slots_ * logits_v_));
  }
  ring_bytes_ = sizeof(k::RowDesc) * (opt_.max_rows + max_slots_) + sizeof(int) * (2 * max_slots_ + 3) + 16;
  for (const auto& dm : models_) ring_bytes_ = std::max(ring_bytes_, DeviceModel::kMaxRun * dm->run_stride());
  for (int i = 0; i < kRing; ++i) {
    Staging s;
    MOA_CUDA(cudaMallocHost(&s.host, ring_bytes_));
    MOA_CUDA(cudaEventCreateWithFlags(&s.done, cudaEventDisableTiming));
    ring_.push_back(s);
  }
  MOA_CUDA(cudaEventCreate(&start_ev_));
  MOA_CUDA(cudaEventCreateWithFlags(&tick_fork_, cudaEventDisableTiming));
  // Per-model forward streams, equal priorities by default.  MOA_STREAM_PRIO
  // (A/B): 1 = the model with the largest weight stream gets the highest
  // priority (its chain is the longest of a fanned-out tick), 2 = every other
  // model does.  Measured on C3's leaf ticks (8B + 1B): 1 is 6% slower (p50
  // 3.59 vs 3.39 ms).
  int prio_lo = 0, prio_hi = 0;
  MOA_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  double big = 0.0;
  for (const auto& dm : models_) big = std::max(big, dm->spec().weight_bytes());
  int prio_mode = 0;
  if (const char* e = std::getenv("MOA_STREAM_PRIO")) prio_mode = std::atoi(e);
  for (std::size_t m = 0; m < models_.size(); ++m) {
    cudaStream_t s2;
    cudaEvent_t e2;
    const bool is_big = models_[m]->spec().weight_bytes() >= big;
    const bool first = models_.size() > 1 && ((prio_mode == 1 && is_big) || (prio_mode == 2 && !is_big));
    MOA_CUDA(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, first ? prio_hi : prio_lo));
    MOA_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
    mstreams_.push_back(s2);
    mdone_.push_back(e2);
    MOA_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
    cstreams_.push_back(s2);
    for (int b = 0; b < 2; ++b) {
      MOA_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
      blob_free_.push_back(e2);
      MOA_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
      blob_ready_.push_back(e2);
    }
  }
  if (const char* e = std::getenv("MOA_ASYNC_UPLOAD")) async_upload_ = std::string(e) != "0";
  for (std::size_t m = 0; m < models_.size(); ++m)
    for (int b = 0; b < 2; ++b) {
      cudaEvent_t e2;
      MOA_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
      run_free_.push_back(e2);
      MOA_CUDA(cudaEventCreateWithFlags(&e2, cudaEventDisableTiming));
      run_ready_.push_back(e2);
    }
  run_par_.assign(models_.size(), 0);
  if (const char* e = std::getenv("MOA_DECODE_RUN")) max_run_ = std::max(1, std::min(DeviceModel::kMaxRun, std::atoi(e)));
  if (const char* e = std::getenv("MOA_OVERLAP")) overlap_models_ = overlap_models_ && std::string(e) != "0";
  MOA_CUDA(cudaStreamSynchronize(stream_));
}

GpuEngine::~GpuEngine() {
  cudaSetDevice(opt_.device);
  if (stream_) cudaStreamSynchronize(stream_);
  ee_pool_.clear();
  models_.clear();
  for (auto& s : ring_) {
    cudaFreeHost(s.host);
    cudaEventDestroy(s.done);
  }
  for (auto e : tick_ev_) cudaEventDestroy(e);
  for (auto s2 : mstreams_) {
    cudaStreamSynchronize(s2);
    cudaStreamDestroy(s2);
  }
  for (auto e2 : mdone_) cudaEventDestroy(e2);
  for (auto s2 : cstreams_) {
    cudaStreamSynchronize(s2);
    cudaStreamDestroy(s2);
  }
  for (auto e2 : blob_free_) cudaEventDestroy(e2);
  for (auto e2 : blob_ready_) cudaEventDestroy(e2);
  for (auto e2 : run_free_) cudaEventDestroy(e2);
  for (auto e2 : run_ready_) cudaEventDestroy(e2);
  if (tick_fork_) cudaEventDestroy(tick_fork_);
  if (start_ev_) cudaEventDestroy(start_ev_);
  for (void* p : {static_cast<void*>(out_tok_), static_cast<void*>(out_lp_), static_cast<void*>(out_ent_),
                  static_cast<void*>(logits_), static_cast<void*>(logits_scratch_)})
    if (p) cudaFree(p);
  if (stream_) cudaStreamDestroy(stream_);
}

GpuEngine::Req& GpuEngine::req(const AgentId& id) {
  auto it = reqs_.find(id);
  if (it == reqs_.end()) throw RunError("sim: unknown agent " + id.str());
  return it->second;
}

const GpuEngine::Req& GpuEngine::req(const AgentId& id) const {
  auto it = reqs_.find(id);
  if (it == reqs_.end()) throw RunError("sim: unknown agent " + id.str());
  return it->second;
}

void GpuEngine::add_agent(const AgentId& id, int model, int owner) {
  if (reqs_.count(id)) throw ValidationError("sim: agent " + id.str() + " added twice");
  if (model < 0 || model >= n_models()) throw ValidationError("engine: unknown model index for " + id.str());
  if (slots_ >= max_slots_) throw ValidationError("engine: agent capacity exhausted");
  if (owner >= world()) throw ValidationError("engine: owner rank out of range for " + id.str());
  Req r;
  r.id = id;
  r.model = model;
  r.owner = owner < 0 ? rank() : owner;
  r.local = r.owner == rank();
  r.kv = r.local ? models_[static_cast<std::size_t>(model)]->bind_agent() : -1;
  r.slot = slots_++;
  r.rec.id = id;
  r.rec.model = model;
  r.rec.submit_tick = tick_;
  reqs_.emplace(id, std::move(r));
  order_.push_back(id);
}

void GpuEngine::set_chunk_dests(const AgentId& id, std::uint64_t ranks) { req(id).dests = ranks; }

// Literal token ids index the model's embedding table on the device: reject
// anything outside [0, vocab) (negative ids are the engine's own symbolic
// references to decoded tokens, created only by the host orchestrator).
void GpuEngine::check_tokens(const Req& r, const TokenSeq& tokens, std::size_t from) const {
  const int vocab = models_[static_cast<std::size_t>(r.model)]->spec().vocab;
  for (std::size_t i = from; i < tokens.size(); ++i)
    if (tokens[i] >= vocab)
      throw ValidationError("engine: token " + std::to_string(tokens[i]) + " of agent " + r.id.str() +
                            " outside the model's vocabulary [0, " + std::to_string(vocab) + ")");
}

// pdsim.cpp:155-174
void GpuEngine::submit_prefill_only(const AgentId& id, int expected_start, const TokenSeq& tokens) {
  Req& r = req(id);
  if (r.cancelled) return;
  if (r.gen_pending || r.dec_started) throw RunError("sim: prefill_only after generate for agent " + id.str());
  const int sched = static_cast<int>(r.prompt.size());
  if (expected_start != sched)
    throw RunError("sim: contiguity violation for agent " + id.str() + ": prefill starts at " +
                   std::to_string(expected_start) + " but " + std::to_string(sched) +
                   " tokens are scheduled");
  if (tokens.empty()) return;
  if (sched + static_cast<int>(tokens.size()) > opt_.max_ctx)
    throw ValidationError("engine: prompt of " + id.str() + " exceeds max_ctx");
  check_tokens(r, tokens, 0);
  r.prompt.insert(r.prompt.end(), tokens.begin(), tokens.end());
  r.rec.prefill_only_calls += 1;
  r.queue.push_back(Job{sched, sched + static_cast<int>(tokens.size())});
}

// pdsim.cpp:176-214 (max_new replaces the planned output)
void GpuEngine::submit_generate(const AgentId& id, const TokenSeq& full, int max_new, int apc_chunk,
                                int prefill_chunk) {
  Req& r = req(id);
  if (r.cancelled) return;
  if (r.gen_pending || r.dec_started) throw RunError("sim: generate submitted twice for agent " + id.str());
  const int sched = static_cast<int>(r.prompt.size());
  if (static_cast<int>(full.size()) < sched || !std::equal(r.prompt.begin(), r.prompt.end(), full.begin()))
    throw RunError("sim: generate prompt for agent " + id.str() + " does not extend the prefilled prefix");
  if (apc_chunk <= 0) throw ValidationError("sim: apc_chunk must be > 0");
  if (max_new < 0) throw ValidationError("sim: max_new must be >= 0");
  if (max_new > opt_.max_out) throw ValidationError("engine: max_new exceeds max_out");
  if (static_cast<int>(full.size()) + max_new > opt_.max_ctx)
    throw ValidationError("engine: prompt + output of " + id.str() + " exceeds max_ctx");
  check_tokens(r, full, static_cast<std::size_t>(sched));
  r.prompt = full;
  r.max_new = max_new;
  r.apc = apc_chunk;
  r.gen_pending = true;
  r.rec.prompt_tokens = static_cast<int>(full.size());
  r.rec.invoked = true;
  const int n = static_cast<int>(full.size());
  const int step = prefill_chunk > 0 ? prefill_chunk : n - sched;
  for (int b = sched; b < n; b += step) r.queue.push_back(Job{b, std::min(b + step, n)});
}

// pdsim.cpp:374-398: output truncated to the tokens already decoded
void GpuEngine::cancel(const AgentId& id) {
  Req& r = req(id);
  if (r.finished) throw RunError("sim: cancel after completion for agent " + id.str());
  if (r.cancelled) return;
  r.cancelled = true;
  r.rec.pruned = true;
  r.gen += 1;
  r.queue.clear();
  r.gen_pending = false;
  r.rec.output_tokens = r.dec_started ? r.n_out : 0;
  events_.push_back(EngineEvent{EngineEvent::Cancel, tick_, id, r.rec.output_tokens, 0});
}

// pdsim.cpp:400-418, except that jobs below `keep` survive (truncated at
// keep): between ticks nothing is in flight, so the rewind is exact.
void GpuEngine::reclaim(const AgentId& id, int keep) {
  Req& r = req(id);
  if (r.gen_pending || r.dec_started) throw RunError("sim: reclaim after generate for agent " + id.str());
  const int sched = static_cast<int>(r.prompt.size());
  if (keep < 0 || keep > sched)
    throw RunError("sim: reclaim point " + std::to_string(keep) + " outside scheduled prompt of " +
                   std::to_string(sched) + " tokens");
  r.gen += 1;
  std::deque<Job> kept;
  for (const Job& j : r.queue)
    if (j.b < keep) kept.push_back(Job{j.b, std::min(j.e, keep)});
  r.queue.swap(kept);
  r.prompt.resize(static_cast<std::size_t>(keep));
  if (r.prefilled > keep) {
    r.rec.reclaimed_tokens += r.prefilled - keep;
    r.prefilled = keep;
  }
  events_.push_back(EngineEvent{EngineEvent::Reclaim, tick_, id, keep, 0});
}

void GpuEngine::on_chunk(const AgentId& id, ChunkFn fn) { req(id).chunk_fns.push_back(std::move(fn)); }
void GpuEngine::on_decode_end(const AgentId& id, EndFn fn) { req(id).end_fns.push_back(std::move(fn)); }

void GpuEngine::note_precursor_ready(const AgentId& id) {
  Req& r = req(id);
  r.rec.precursor_ready_tick = std::max(r.rec.precursor_ready_tick, tick_);
}

void GpuEngine::mark_empty_input(const AgentId& id) { req(id).rec.empty_input = true; }

bool GpuEngine::busy() const {
  for (const auto& [id, r] : reqs_) {
    if (r.cancelled || r.finished) continue;
    if (!r.queue.empty() || r.gen_pending || r.dec_started) return true;
  }
  return false;
}

void GpuEngine::start_decode(Req& r, int n_out) {
  r.gen_pending = false;
  r.dec_started = true;
  r.rec.decode_start = tick_;
  r.n_out = n_out;
}

void GpuEngine::upload_and_forward(int m, const std::vector<k::RowDesc>& rows, const std::vector<int>& lsel,
                                   const std::vector<int>& lout, cudaStream_t st) {
  DeviceModel& dm = *models_[static_cast<std::size_t>(m)];
  Staging& s = ring_[ring_next_];
  ring_next_ = (ring_next_ + 1) % ring_.size();
  {
    const auto t_wait = std::chrono::steady_clock::now();
    MOA_CUDA(cudaEventSynchronize(s.done));  // the copy that last used this slot has consumed it
    host_wait_ms_ += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_wait).count();
  }
  // staging layout = the device blob: [sel | meta] (padded) then the rows
  const std::size_t rb = sizeof(k::RowDesc) * rows.size();
  const int sb = dm.buffers().sel_bytes;
  std::memcpy(s.host + sb, rows.data(), rb);
  const int L = dm.max_logit_rows();
  int max_pos = 0;
  TickStats ts;
  bool distinct = rows.size() <= 64;  // every row a different agent (pure decode)?
  int runs = 0, singles = 0;           // maximal same-agent runs of consecutive positions; runs of one row
  auto joined = [&](std::size_t i) {    // rows i - 1 and i are one run
    return i > 0 && i < rows.size() && rows[i - 1].kv == rows[i].kv && rows[i - 1].pos + 1 == rows[i].pos;
  };
  for (std::size_t i = 0; i < rows.size(); ++i) {
    const auto& rd = rows[i];
    max_pos = std::max(max_pos, rd.pos);
    ts.keys += rd.pos + 1;
    for (std::size_t j = 0; j < i && distinct; ++j) distinct = rows[j].kv != rd.kv;
    runs += !joined(i);
    const bool single = !joined(i) && !joined(i + 1);
    singles += single;
    if (single) {
      ts.single_keys += rd.pos + 1;
    } else {
      ts.run_pairs += rd.pos + 1;
      if (!joined(i + 1)) ts.run_keys += rd.pos + 1;  // last row of its run: the run's key prefix
    }
  }
  ts.singles = singles;
  // prefill tick: same-agent runs (prompts and the aggregators' 32-row chunks)
  // -> the tcgen05 prefill attention, each run's keys streamed once per GQA
  // group instead of once per row (from 64 rows: C1 -5%, C2 -1%, C3 -0.5%
  // against the 512 the mma.sync kernel needed; from 32 rows, so a single
  // 32-row chunk qualifies: C3 -0.4% more, C1 / C2 unchanged)
  static const std::size_t min_rows = [] {
    const char* e = std::getenv("MOA_PREFILL_MIN_ROWS");
    return static_cast<std::size_t>(e ? std::atoi(e) : 32);
  }();
  const bool prefill = rows.size() >= min_rows && static_cast<std::size_t>(runs) * 16 <= rows.size();
  // [lsel (L)][lout (L)][meta: R, Rl, max_pos] -- the graph's kernels read meta
  int* sel = reinterpret_cast<int*>(s.host);
  std::memcpy(sel, lsel.data(), sizeof(int) * lsel.size());
  std::memcpy(sel + L, lout.data(), sizeof(int) * lout.size());
  sel[2 * L] = static_cast<int>(rows.size());
  sel[2 * L + 1] = static_cast<int>(lsel.size());
  sel[2 * L + 2] = max_pos;
  int b = 0;
  if (async_upload_) {
    // into the blob the previous forward of this model is not reading, on the
    // model's copy stream: the copy runs while that forward executes
    b = dm.blob() ^ 1;
    dm.use_blob(b);
    const std::size_t ev = 2 * static_cast<std::size_t>(m) + static_cast<std::size_t>(b);
    cudaStream_t cs = cstreams_[static_cast<std::size_t>(m)];
    MOA_CUDA(cudaStreamWaitEvent(cs, blob_free_[ev], 0));  // the forward that last read blob b is done
    MOA_CUDA(cudaMemcpyAsync(dm.buffers().sel, s.host, sb + rb, cudaMemcpyHostToDevice, cs));
    MOA_CUDA(cudaEventRecord(s.done, cs));
    MOA_CUDA(cudaEventRecord(blob_ready_[ev], cs));
    MOA_CUDA(cudaStreamWaitEvent(st, blob_ready_[ev], 0));
  } else {
    MOA_CUDA(cudaMemcpyAsync(dm.buffers().sel, s.host, sb + rb, cudaMemcpyHostToDevice, st));
    MOA_CUDA(cudaEventRecord(s.done, st));
  }
  float* logits = (opt_.keep_logits && !lsel.empty())
                      ? logits_scratch_ + static_cast<long long>(m) * max_slots_ * logits_v_
                      : nullptr;
  dm.forward(static_cast<int>(rows.size()), static_cast<int>(lsel.size()), max_pos, ts, out_tok_, out_tok_,
             out_lp_, out_ent_, logits, st, distinct, prefill, singles > 0);
  if (logits) {  // debug path: scatter each logits row to its (slot, k) home
    const long long V = dm.spec().vocab;
    for (std::size_t i = 0; i < lsel.size(); ++i)
      MOA_CUDA(cudaMemcpyAsync(logits_ + static_cast<long long>(lout[i]) * logits_v_,
                               logits + static_cast<long long>(i) * V, sizeof(float) * V,
                               cudaMemcpyDeviceToDevice, st));
  }
  if (async_upload_) MOA_CUDA(cudaEventRecord(blob_free_[2 * static_cast<std::size_t>(m) + static_cast<std::size_t>(b)], st));
  rows_total_ += static_cast<long long>(rows.size());
  weight_bytes_ += dm.weight_bytes();
  forwards_ += 1;
}

void GpuEngine::upload_and_forward_run(int m, int K, const std::vector<k::RowDesc>& rows, const std::vector<int>& lout,
                                       cudaStream_t st) {
  DeviceModel& dm = *models_[static_cast<std::size_t>(m)];
  Staging& s = ring_[ring_next_];
  ring_next_ = (ring_next_ + 1) % ring_.size();
  {
    const auto t_wait = std::chrono::steady_clock::now();
    MOA_CUDA(cudaEventSynchronize(s.done));
    host_wait_ms_ += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_wait).count();
  }
  // K compact tick blobs [lsel | lout | meta] (padded) + rows: tick j's rows
  // advance one position and read the token decoded by tick j - 1
  const std::size_t stride = dm.run_stride();
  const int L = dm.max_logit_rows(), sb = dm.buffers().sel_bytes, R = static_cast<int>(rows.size());
  int max_pos = 0;
  for (int j = 0; j < K; ++j) {
    char* base = s.host + j * stride;
    int* sel = reinterpret_cast<int*>(base);
    auto* rd = reinterpret_cast<k::RowDesc*>(base + sb);
    for (int i = 0; i < R; ++i) {
      k::RowDesc d = rows[static_cast<std::size_t>(i)];
      d.pos += j;
      d.tok = j == 0 ? d.tok : d.tok - j;  // ref(slot, k) = -1 - (slot * max_out + k): k advances with the tick
      d.out = d.out + j;
      rd[i] = d;
      sel[i] = i;
      sel[L + i] = lout[static_cast<std::size_t>(i)] + j;
      max_pos = std::max(max_pos, d.pos);
    }
    sel[2 * L] = R;
    sel[2 * L + 1] = R;
    sel[2 * L + 2] = max_pos;
  }
  const int p = run_par_[static_cast<std::size_t>(m)] ^= 1;
  const std::size_t ev = 2 * static_cast<std::size_t>(m) + static_cast<std::size_t>(p);
  cudaStream_t cs = cstreams_[static_cast<std::size_t>(m)];
  MOA_CUDA(cudaStreamWaitEvent(cs, run_free_[ev], 0));
  MOA_CUDA(cudaMemcpyAsync(dm.run_blob(p), s.host, K * stride, cudaMemcpyHostToDevice, cs));
  MOA_CUDA(cudaEventRecord(s.done, cs));
  MOA_CUDA(cudaEventRecord(run_ready_[ev], cs));
  MOA_CUDA(cudaStreamWaitEvent(st, run_ready_[ev], 0));
  dm.forward_run(K, R, max_pos, out_tok_, out_tok_, out_lp_, out_ent_, st, p);
  MOA_CUDA(cudaEventRecord(run_free_[ev], st));
  rows_total_ += static_cast<long long>(K) * R;
  weight_bytes_ += K * dm.weight_bytes();
  forwards_ += K;
}

void GpuEngine::step() {
  const auto host_t0 = std::chrono::steady_clock::now();
  struct HostTimer {
    std::chrono::steady_clock::time_point t0;
    double* acc;
    ~HostTimer() { *acc += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(); }
  } host_timer{host_t0, &host_ms_};
  enum Kind { Decode, Prefill, Bootstrap, Empty };
  struct Plan {
    Req* r;
    Kind kind;
    Job job;
    bool yields;
  };
  std::vector<Plan> plan;
  const std::size_t nm = models_.size();
  std::vector<std::vector<k::RowDesc>> rows(nm);
  std::vector<std::vector<int>> lsel(nm), lout(nm);
  int budget = opt_.max_rows;
  auto add_row = [&](Req& r, int pos, Token tok, int out_k) {
    if (!r.local) return;  // another rank computes it; the schedule advances identically here
    auto& rv = rows[static_cast<std::size_t>(r.model)];
    int oi = -1;
    if (out_k >= 0) {
      oi = r.slot * opt_.max_out + out_k;
      lsel[static_cast<std::size_t>(r.model)].push_back(static_cast<int>(rv.size()));
      lout[static_cast<std::size_t>(r.model)].push_back(oi);
    }
    rv.push_back(k::RowDesc{r.kv, pos, tok, oi});
  };
  for (const AgentId& id : order_) {
    Req& r = reqs_.at(id);
    if (r.cancelled || r.finished) continue;
    if (r.dec_started) {
      if (r.n_out < r.max_new) {
        add_row(r, static_cast<int>(r.prompt.size()) + r.n_out - 1, ref(r.slot, r.n_out - 1), r.n_out);
        plan.push_back(Plan{&r, Decode, {}, false});
        budget -= 1;
      }
      continue;
    }
    if (!r.queue.empty()) {
      // every queued job, in order, while it fits the tick's row budget
      while (!r.queue.empty() && r.queue.front().e - r.queue.front().b <= budget) {
        const Job j = r.queue.front();
        r.queue.pop_front();
        budget -= j.e - j.b;
        const bool yields = r.gen_pending && j.e == static_cast<int>(r.prompt.size()) && r.max_new > 0;
        for (int p = j.b; p < j.e; ++p)
          add_row(r, p, r.prompt[static_cast<std::size_t>(p)], (yields && p == j.e - 1) ? 0 : -1);
        plan.push_back(Plan{&r, Prefill, j, yields});
      }
      continue;
    }
    if (r.gen_pending && r.prefilled == static_cast<int>(r.prompt.size())) {
      if (r.max_new == 0) {
        plan.push_back(Plan{&r, Empty, {}, false});
      } else {
        const int P = static_cast<int>(r.prompt.size());
        add_row(r, std::max(P - 1, 0), P > 0 ? r.prompt[static_cast<std::size_t>(P - 1)] : 0, 0);
        plan.push_back(Plan{&r, Bootstrap, {}, false});
        budget -= 1;
      }
    }
  }
  // Forwards of different models in one tick are independent (disjoint
  // weights, KV pools, workspaces and output slots): each runs on its model's
  // stream after the previous tick, and the engine stream joins them -- a
  // successor's incremental prefill overlaps its predecessors' decode.
  int active = 0;
  for (std::size_t m = 0; m < nm; ++m) active += !rows[m].empty();
  // Decode run: when every row of this tick is a decode row and no request
  // reaches a chunk boundary or its end before tick t + K - 1, the K ticks
  // differ only by one position and one token each -- they run as one graph
  // launch (no host decision can change them: callbacks fire only on chunk /
  // completion events, which the run ends on).
  int K = 1;
  // With several ranks every rank computes the same K from the replicated
  // plan (remote agents' rows included: they bound the run by their chunk
  // events too), so runs end on the ticks whose hand-offs all ranks issue;
  // a rank whose own rows cannot run (workspace) falls back to single ticks,
  // which changes no tick number or event.
  if (in_run_ && max_run_ > 1 && !tracing_ && !probing_ && !opt_.keep_logits && !plan.empty()) {
    K = max_run_;
    for (const Plan& p : plan) {
      const Req& r = *p.r;
      if (p.kind != Decode) {
        K = 1;
        break;
      }
      for (int j = 0; j < K; ++j) {  // first tick of the run that emits an event
        const int n = r.n_out + j + 1;
        if (n - r.chunk_begin >= r.apc || n == r.max_new) {
          K = j + 1;
          break;
        }
      }
    }
    for (std::size_t m = 0; m < nm && K > 1; ++m)
      if (!rows[m].empty() && (!models_[m]->runs_supported() || static_cast<int>(rows[m].size()) >
                                                                     models_[m]->max_logit_rows()))
        K = 1;
  }
  const bool fan_out = active > 1 && overlap_models_;
  if (fan_out) MOA_CUDA(cudaEventRecord(tick_fork_, stream_));
  for (std::size_t m = 0; m < nm; ++m)
    if (!rows[m].empty()) {
      const auto t_api = std::chrono::steady_clock::now();
      cudaStream_t st = stream_;
      if (fan_out) {
        st = mstreams_[m];
        MOA_CUDA(cudaStreamWaitEvent(st, tick_fork_, 0));
      }
      if (K > 1)
        upload_and_forward_run(static_cast<int>(m), K, rows[m], lout[m], st);
      else
        upload_and_forward(static_cast<int>(m), rows[m], lsel[m], lout[m], st);
      if (fan_out) {
        MOA_CUDA(cudaEventRecord(mdone_[m], st));
        MOA_CUDA(cudaStreamWaitEvent(stream_, mdone_[m], 0));
      }
      host_api_ms_ += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_api).count();
    }
  overlapped_ticks_ += fan_out;
  // the first K - 1 ticks of a decode run: no event, no timing
  for (int j = 0; j + 1 < K; ++j) {
    for (Plan& p : plan) p.r->n_out += 1;
    if (opt_.time_ticks) {
      if (static_cast<int>(tick_ev_.size()) <= tick_) {
        cudaEvent_t e;
        MOA_CUDA(cudaEventCreate(&e));
        tick_ev_.push_back(e);
        tick_timed_.push_back(0);
      }
      tick_timed_[static_cast<std::size_t>(tick_)] = 0;
    }
    tick_ += 1;
  }
  // state update
  for (Plan& p : plan) {
    Req& r = *p.r;
    switch (p.kind) {
      case Decode:
        r.n_out += 1;
        break;
      case Prefill: {
        const int recomputed = std::max(0, std::min(p.job.e, r.max_computed) - p.job.b);
        r.max_computed = std::max(r.max_computed, p.job.e);
        r.rec.prefill.push_back(PrefillInterval{tick_, p.job.b, p.job.e});
        r.rec.recomputed_tokens += recomputed;
        if (p.job.b != r.prefilled) throw RunError("sim: internal contiguity breach for agent " + r.id.str());
        r.prefilled = p.job.e;
        if (p.yields)
          start_decode(r, 1);
        else if (r.gen_pending && r.prefilled == static_cast<int>(r.prompt.size()) && r.max_new == 0)
          start_decode(r, 0);
        break;
      }
      case Bootstrap:
        start_decode(r, 1);
        break;
      case Empty:
        start_decode(r, 0);
        break;
    }
  }
  // Tick-end timing event: a timed event record costs ~4 us of device time
  // between two ticks' graphs, so it is recorded only where a time is read --
  // ticks on which a decode completes (request e2e, orchestrator.cpp:290-292)
  // and every tick while tracing.
  if (opt_.time_ticks) {
    bool completes = tracing_;
    for (const Plan& p : plan)
      completes = completes || (p.r->dec_started && !p.r->finished && !p.r->cancelled && p.r->n_out == p.r->max_new);
    if (static_cast<int>(tick_ev_.size()) <= tick_) {
      cudaEvent_t e;
      MOA_CUDA(cudaEventCreate(&e));
      tick_ev_.push_back(e);
      tick_timed_.push_back(0);
    }
    tick_timed_[static_cast<std::size_t>(tick_)] = completes;
    if (completes) MOA_CUDA(cudaEventRecord(tick_ev_[static_cast<std::size_t>(tick_)], stream_));
  }
  const int t = tick_;
  tick_ += 1;
  // phase A: chunk emission (pdsim.cpp:339-362).  With several ranks the
  // chunk's tokens / logprobs / entropies first move from the owner to every
  // other rank (grouped NCCL P2P on the engine stream, so they land before
  // the next tick's forward and before this tick's early-exit evaluations).
  if (world() > 1) {
    bool any = false;
    for (const AgentId& id : order_) {
      Req& r = reqs_.at(id);
      if (r.cancelled || r.finished || !r.dec_started) continue;
      const int n = r.n_out;
      if (!(n > r.chunk_begin && (n - r.chunk_begin >= r.apc || n == r.max_new))) continue;
      if (!any) comm_->begin();
      any = true;
      const long long off = static_cast<long long>(r.slot) * opt_.max_out + r.chunk_begin;
      const long long cnt = n - r.chunk_begin;
      for (int p = 0; p < world(); ++p) {
        if (p == rank()) continue;
        if (r.local) {
          if (!((r.dests >> p) & 1)) continue;  // this rank needs no copy of the chunk
          comm_->send_i32(out_tok_ + off, cnt, p, stream_);
          comm_->send_f32(out_lp_ + off, cnt, p, stream_);
          comm_->send_f32(out_ent_ + off, cnt, p, stream_);
        } else if (p == r.owner && ((r.dests >> rank()) & 1)) {
          comm_->recv_i32(out_tok_ + off, cnt, p, stream_);
          comm_->recv_f32(out_lp_ + off, cnt, p, stream_);
          comm_->recv_f32(out_ent_ + off, cnt, p, stream_);
        }
      }
    }
    if (any) comm_->end();
  }
  std::vector<Req*> done;
  for (const AgentId& id : order_) {
    Req& r = reqs_.at(id);
    if (r.cancelled || r.finished || !r.dec_started) continue;
    const int n = r.n_out;
    if (n > r.chunk_begin && (n - r.chunk_begin >= r.apc || n == r.max_new)) {
      const int b = r.chunk_begin;
      r.chunk_begin = n;
      const std::uint64_t gen = r.gen;
      TokenSeq toks;
      toks.reserve(static_cast<std::size_t>(n - b));
      for (int q = b; q < n; ++q) toks.push_back(ref(r.slot, q));
      events_.push_back(EngineEvent{EngineEvent::Chunk, t, id, b, n});
      const auto fns = r.chunk_fns;
      for (const auto& fn : fns) {
        fn(b, n, toks);
        if (r.gen != gen) break;  // a callback cancelled this request
      }
    }
    if (r.n_out == r.max_new && !r.cancelled) done.push_back(&r);
  }
  // phase B: completions
  for (Req* r : done) {
    if (r->cancelled || r->finished) continue;
    r->finished = true;
    r->rec.decode_end = t;
    r->rec.complete = t;
    r->rec.output_tokens = r->max_new;
    events_.push_back(EngineEvent{EngineEvent::DecodeEnd, t, r->id, r->max_new, 0});
    const auto fns = r->end_fns;
    for (const auto& fn : fns) fn(t);
  }
  // phase C: deferred work (early-exit evaluations), FIFO
  while (!deferred_.empty()) {
    auto fn = std::move(deferred_.front());
    deferred_.pop_front();
    fn();
  }
}

void GpuEngine::run(int max_ticks) {
  // decode runs only here: the caller regains control only through event
  // callbacks, which end a run.  step() alone keeps one tick per call (the
  // protocol lets a caller cancel / reclaim between any two ticks).
  struct RunsOn {
    bool& f;
    explicit RunsOn(bool& x) : f(x) { f = true; }
    ~RunsOn() { f = false; }
  } runs_on(in_run_);
  while (busy()) {
    step();
    if (tick_ > max_ticks) throw RunError("engine: tick limit exceeded");
  }
  if (std::getenv("MOA_HOST_PROFILE"))
    std::fprintf(stderr, "[moa] ticks %d host %.3f ms (api %.3f ms, ring wait %.3f ms, forwards %d)\n", tick_,
                 host_ms_, host_api_ms_, host_wait_ms_, forwards_);
}

TokenSeq GpuEngine::resolve(const TokenSeq& seq) {
  bool any = false;
  for (Token t : seq) any |= t < 0;
  if (!any) return seq;
  std::vector<int> host(static_cast<std::size_t>(slots_) * opt_.max_out);
  MOA_CUDA(cudaMemcpyAsync(host.data(), out_tok_, sizeof(int) * host.size(), cudaMemcpyDeviceToHost, stream_));
  MOA_CUDA(cudaStreamSynchronize(stream_));
  TokenSeq out(seq);
  for (Token& t : out)
    if (t < 0) t = host[static_cast<std::size_t>(-1 - t)];
  return out;
}

void GpuEngine::read_outputs(const AgentId& id, int n, int* tok, float* lp, float* ent) {
  const Req& r = req(id);
  if (n < 0 || n > opt_.max_out) throw ValidationError("engine: read_outputs count out of range");
  const long long off = static_cast<long long>(r.slot) * opt_.max_out;
  if (tok) MOA_CUDA(cudaMemcpyAsync(tok, out_tok_ + off, sizeof(int) * n, cudaMemcpyDeviceToHost, stream_));
  if (lp) MOA_CUDA(cudaMemcpyAsync(lp, out_lp_ + off, sizeof(float) * n, cudaMemcpyDeviceToHost, stream_));
  if (ent) MOA_CUDA(cudaMemcpyAsync(ent, out_ent_ + off, sizeof(float) * n, cudaMemcpyDeviceToHost, stream_));
  MOA_CUDA(cudaStreamSynchronize(stream_));
}

void GpuEngine::read_logits(const AgentId& id, int kk, float* dst) {
  if (!logits_) throw ValidationError("engine: keep_logits is off");
  const Req& r = req(id);
  const int V = models_[static_cast<std::size_t>(r.model)]->spec().vocab;
  const long long home = (static_cast<long long>(r.slot) * opt_.max_out + kk) * logits_v_;
  MOA_CUDA(cudaMemcpyAsync(dst, logits_ + home, sizeof(float) * V, cudaMemcpyDeviceToHost, stream_));
  MOA_CUDA(cudaStreamSynchronize(stream_));
}

void GpuEngine::reset() {
  MOA_CUDA(cudaStreamSynchronize(stream_));
  reqs_.clear();
  order_.clear();
  deferred_.clear();
  events_.clear();
  tick_ = 0;
  slots_ = 0;
  rows_total_ = 0;
  weight_bytes_ = 0.0;
  forwards_ = 0;
  overlapped_ticks_ = 0;
  host_ms_ = host_api_ms_ = host_wait_ms_ = 0.0;
  for (auto& m : models_) m->reset_bindings();
  embed_kv_.clear();
}

void GpuEngine::hidden_embed(int m, const AgentId& src, int n, GpuMetricQ& ev) {
  if (m < 0 || m >= n_models()) throw ValidationError("provider: embedding model index out of range");
  DeviceModel& dm = *models_[static_cast<std::size_t>(m)];
  if (ev.hidden() != dm.spec().d) throw ValidationError("provider: evaluator width differs from the embedding model");
  if (n > opt_.max_ctx) throw ValidationError("provider: completion longer than the embedding model's context");
  auto it = embed_kv_.find(m);
  if (it == embed_kv_.end()) it = embed_kv_.emplace(m, dm.bind_agent()).first;
  const Req& r = req(src);
  std::vector<k::RowDesc> rows;
  rows.reserve(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) rows.push_back(k::RowDesc{it->second, i, ref(r.slot, i), -1});
  upload_and_forward(m, rows, {}, {}, stream_);
  k::ee_hidden_embed(dm.residual(), n, dm.spec().d, dm.spec().norm_eps, ev.emb_buffer(), stream_);
  MOA_CUDA(cudaGetLastError());
}

GpuMetricQ& GpuEngine::ee_evaluator(int i, int hidden, std::uint64_t seed, double tau, bool diag, int members,
                                     int max_tokens) {
  if (static_cast<int>(ee_pool_.size()) <= i) ee_pool_.resize(static_cast<std::size_t>(i) + 1);
  auto& e = ee_pool_[static_cast<std::size_t>(i)];
  if (!e || !e->fits(hidden, members, max_tokens))
    e = std::make_unique<GpuMetricQ>(hidden, seed, tau, diag, std::max(members, 8), std::max(max_tokens, 512), stream_);
  e->reset(seed, tau, diag);
  return *e;
}

void GpuEngine::attach_comm(std::unique_ptr<PeerComm> comm) {
  if (!reqs_.empty()) throw RunError("engine: attach the communicator before adding agents");
  comm_ = std::move(comm);
}

void GpuEngine::set_probing(bool on) {
  MOA_CUDA(cudaStreamSynchronize(stream_));
  probing_ = on;
  probes_.reset();
  for (auto& m : models_) m->attach_probes(on ? &probes_ : nullptr);
}

void GpuEngine::probe_stats(int kind, int* count, double* ms, double* bytes, double* flops) {
  MOA_CUDA(cudaStreamSynchronize(stream_));
  int n = 0;
  double t = 0.0, b = 0.0, f = 0.0;
  for (const auto& r : probes_.recs) {
    if (r.kind != kind) continue;
    float e = 0.f;
    MOA_CUDA(cudaEventElapsedTime(&e, r.a, r.b));
    ++n;
    t += e;
    b += r.bytes;
    f += r.flops;
  }
  *count = n;
  *ms = t;
  *bytes = b;
  *flops = f;
}

void GpuEngine::mark_start() { MOA_CUDA(cudaEventRecord(start_ev_, stream_)); }

double GpuEngine::ms_since_start(int t) {
  if (t < 0 || t >= static_cast<int>(tick_ev_.size())) return 0.0;
  if (!tick_timed_[static_cast<std::size_t>(t)])
    throw RunError("engine: tick " + std::to_string(t) + " has no timing event (enable tracing)");
  MOA_CUDA(cudaEventSynchronize(tick_ev_[static_cast<std::size_t>(t)]));
  float ms = 0.f;
  MOA_CUDA(cudaEventElapsedTime(&ms, start_ev_, tick_ev_[static_cast<std::size_t>(t)]));
  return ms;
}

}  // namespace moa
