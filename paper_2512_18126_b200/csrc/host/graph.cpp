// See graph.hpp for the reference citations of each type.
#include "graph.hpp"

#include <algorithm>
#include <set>

namespace moa {

namespace {

std::vector<std::vector<AgentId>> grid(const std::vector<int>& widths) {
  if (widths.empty()) throw ValidationError("topology: widths must be non-empty");
  std::vector<std::vector<AgentId>> g;
  for (std::size_t l = 0; l < widths.size(); ++l) {
    if (widths[l] <= 0)
      throw ValidationError("topology: layer " + std::to_string(l + 1) + " has non-positive width " +
                            std::to_string(widths[l]));
    std::vector<AgentId> row;
    for (int p = 0; p < widths[l]; ++p) row.push_back(AgentId{static_cast<int>(l) + 1, p});
    g.push_back(std::move(row));
  }
  return g;
}

}  // namespace

Topology Topology::tree(const std::vector<int>& widths, const std::vector<int>& branching) {
  grid(widths);
  if (branching.size() + 1 != widths.size())
    throw ValidationError("topology: expected " + std::to_string(widths.size() - 1) +
                          " branching factors, got " + std::to_string(branching.size()));
  std::vector<std::vector<int>> sizes;
  for (std::size_t l = 0; l < branching.size(); ++l) {
    if (branching[l] <= 0)
      throw ValidationError("topology: branching factor for layer " + std::to_string(l + 2) +
                            " must be positive");
    if (widths[l + 1] * branching[l] != widths[l])
      throw ValidationError("topology: layer " + std::to_string(l + 2) + " width " +
                            std::to_string(widths[l + 1]) + " times branching " +
                            std::to_string(branching[l]) + " does not cover layer " +
                            std::to_string(l + 1) + " width " + std::to_string(widths[l]));
    sizes.emplace_back(static_cast<std::size_t>(widths[l + 1]), branching[l]);
  }
  return tree_custom(widths, sizes);
}

Topology Topology::tree_custom(const std::vector<int>& widths,
                               const std::vector<std::vector<int>>& cluster_sizes) {
  Topology t;
  t.layers_ = grid(widths);
  if (cluster_sizes.size() + 1 != widths.size())
    throw ValidationError("topology: expected cluster sizes for " +
                          std::to_string(widths.size() - 1) + " layer transitions");
  for (std::size_t l = 0; l < cluster_sizes.size(); ++l) {
    const auto& s = cluster_sizes[l];
    if (s.size() != static_cast<std::size_t>(widths[l + 1]))
      throw ValidationError("topology: layer " + std::to_string(l + 2) + " has " +
                            std::to_string(widths[l + 1]) + " agents but " +
                            std::to_string(s.size()) + " cluster sizes");
    int sum = 0;
    for (int v : s) {
      if (v <= 0)
        throw ValidationError("topology: layer " + std::to_string(l + 2) +
                              " has a non-positive cluster size");
      sum += v;
    }
    if (sum != widths[l])
      throw ValidationError("topology: layer " + std::to_string(l + 2) + " cluster sizes sum to " +
                            std::to_string(sum) + " but layer " + std::to_string(l + 1) +
                            " has width " + std::to_string(widths[l]));
  }
  t.kind_ = TopologyKind::Tree;
  t.sizes_ = cluster_sizes;
  t.build_edges();
  return t;
}

Topology Topology::all_to_all(const std::vector<int>& widths) {
  Topology t;
  t.layers_ = grid(widths);
  t.kind_ = TopologyKind::AllToAll;
  t.build_edges();
  return t;
}

void Topology::build_edges() {
  pre_.clear();
  for (const auto& a : layers_.front()) pre_[a] = {};
  for (std::size_t l = 1; l < layers_.size(); ++l) {
    const auto& prev = layers_[l - 1];
    if (kind_ == TopologyKind::AllToAll) {
      for (const auto& a : layers_[l]) pre_[a] = prev;
      continue;
    }
    // contiguous partition of layer l by position (topology.cpp:125-134)
    auto it = prev.begin();
    for (std::size_t j = 0; j < layers_[l].size(); ++j) {
      auto end = it + sizes_[l - 1][j];
      pre_[layers_[l][j]] = std::vector<AgentId>(it, end);
      it = end;
    }
  }
}

int Topology::agent_count() const {
  int n = 0;
  for (const auto& l : layers_) n += static_cast<int>(l.size());
  return n;
}

const std::vector<AgentId>& Topology::layer(int l) const {
  if (l < 1 || l > depth())
    throw ValidationError("topology: layer " + std::to_string(l) + " out of range [1, " +
                          std::to_string(depth()) + "]");
  return layers_[static_cast<std::size_t>(l - 1)];
}

const std::vector<AgentId>& Topology::precursors(const AgentId& a) const {
  auto it = pre_.find(a);
  if (it == pre_.end()) throw ValidationError("topology: unknown agent " + a.str());
  return it->second;
}

std::vector<AgentId> Topology::successors(const AgentId& a) const {
  std::vector<AgentId> out;
  if (a.layer >= depth()) return out;
  for (const auto& b : layers_[static_cast<std::size_t>(a.layer)]) {
    const auto& p = pre_.at(b);
    if (std::find(p.begin(), p.end(), a) != p.end()) out.push_back(b);
  }
  return out;
}

std::vector<std::vector<AgentId>> Topology::clusters_of_layer(int l) const {
  if (l < 2 || l > depth())
    throw ValidationError("topology: clusters_of_layer expects a layer in [2, " +
                          std::to_string(depth()) + "], got " + std::to_string(l));
  std::vector<std::vector<AgentId>> out;
  for (const auto& a : layers_[static_cast<std::size_t>(l - 1)]) out.push_back(pre_.at(a));
  return out;
}

const AgentId& Topology::root() const {
  if (layers_.back().size() != 1)
    throw ValidationError("topology: last layer has width " +
                          std::to_string(layers_.back().size()) +
                          "; a single aggregator is required");
  return layers_.back().front();
}

// ---------------------------------------------------------------------------

PromptTemplate::PromptTemplate(TokenSeq prefix, std::vector<Slot> slots, TokenSeq suffix)
    : prefix_(std::move(prefix)), slots_(std::move(slots)), suffix_(std::move(suffix)) {
  std::set<AgentId> seen;
  for (const auto& s : slots_)
    if (!seen.insert(s.precursor).second)
      throw ValidationError("prompt template: precursor " + s.precursor.str() +
                            " appears in more than one slot");
}

PromptTemplate PromptTemplate::without(const AgentId& pruned) const {
  std::vector<Slot> kept;
  for (const auto& s : slots_)
    if (!(s.precursor == pruned)) kept.push_back(s);
  if (kept.size() == slots_.size())
    throw ValidationError("prompt template: cannot drop " + pruned.str() + "; it has no slot");
  return PromptTemplate(prefix_, std::move(kept), suffix_);
}

TokenSeq assemble(const PromptTemplate& t, const std::map<AgentId, TokenSeq>& outputs) {
  TokenSeq out = t.prefix();
  for (const auto& s : t.slots()) {
    auto it = outputs.find(s.precursor);
    if (it == outputs.end())
      throw ValidationError("assemble: missing output for precursor " + s.precursor.str());
    out.insert(out.end(), s.separator.begin(), s.separator.end());
    out.insert(out.end(), it->second.begin(), it->second.end());
  }
  out.insert(out.end(), t.suffix().begin(), t.suffix().end());
  return out;
}

// ---------------------------------------------------------------------------

SlotPlan::SlotPlan(AgentId self, PromptTemplate tmpl, bool incremental)
    : self_(self), tmpl_(std::move(tmpl)), incremental_(incremental) {
  for (const auto& s : tmpl_.slots()) slots_.push_back(State{s, {}, 0, false, false, 0});
  had_slots_ = !slots_.empty();
}

int SlotPlan::find(const AgentId& p) const {
  for (std::size_t i = 0; i < slots_.size(); ++i)
    if (slots_[i].spec.precursor == p) return static_cast<int>(i);
  return -1;
}

std::map<AgentId, TokenSeq> SlotPlan::received() const {
  std::map<AgentId, TokenSeq> m;
  for (const auto& s : slots_) m[s.spec.precursor] = s.received;
  return m;
}

const TokenSeq& SlotPlan::final_prompt() const {
  if (!generated_) throw RunError("router: final prompt requested before generate");
  return final_;
}

std::vector<RouteAction> SlotPlan::start() {
  if (started_) throw RunError("router: started twice for agent " + self_.str());
  started_ = true;
  return step();
}

std::vector<RouteAction> SlotPlan::on_chunk(const AgentId& producer, const TokenSeq& tokens) {
  int i = find(producer);
  if (i < 0) return {};  // pruned slot: late chunk dropped (router.cpp:46)
  if (generated_)
    throw RunError("router: chunk from " + producer.str() + " after generate for " + self_.str());
  State& s = slots_[static_cast<std::size_t>(i)];
  if (s.closed) throw RunError("router: chunk after stream close from " + producer.str());
  s.received.insert(s.received.end(), tokens.begin(), tokens.end());
  return started_ ? step() : std::vector<RouteAction>{};
}

std::vector<RouteAction> SlotPlan::on_precursor_done(const AgentId& producer) {
  int i = find(producer);
  if (i < 0) return {};
  slots_[static_cast<std::size_t>(i)].closed = true;
  return started_ ? step() : std::vector<RouteAction>{};
}

std::vector<RouteAction> SlotPlan::on_precursor_cancelled(const AgentId& producer) {
  int i = find(producer);
  if (i < 0) return {};
  if (generated_)
    throw RunError("router: precursor " + producer.str() + " pruned after generate for " +
                   self_.str());
  if (i < active_)
    throw RunError("router: completed precursor " + producer.str() + " cannot be pruned");
  std::vector<RouteAction> acts;
  const State& s = slots_[static_cast<std::size_t>(i)];
  if (i == active_ && s.sep_issued && scheduled_ > s.mark) {
    // roll the engine back to where this slot began (router.cpp:80-88)
    acts.push_back(RouteAction{RouteAction::Kind::Reclaim, s.mark, {}});
    ++reclaims_;
    scheduled_ = s.mark;
    stream_.resize(static_cast<std::size_t>(s.mark));
  }
  tmpl_ = tmpl_.without(producer);
  slots_.erase(slots_.begin() + i);
  if (!started_) return acts;
  auto more = step();
  acts.insert(acts.end(), more.begin(), more.end());
  return acts;
}

void SlotPlan::emit_pending(std::vector<RouteAction>& out) {
  if (pending_.empty()) return;
  RouteAction a{RouteAction::Kind::PrefillOnly, scheduled_, std::move(pending_)};
  pending_.clear();
  scheduled_ += static_cast<int>(a.tokens.size());
  stream_.insert(stream_.end(), a.tokens.begin(), a.tokens.end());
  ++calls_;
  out.push_back(std::move(a));
}

std::vector<RouteAction> SlotPlan::step() {
  std::vector<RouteAction> out;
  if (generated_) return out;
  auto seal = [&](TokenSeq prompt) {
    final_ = std::move(prompt);
    out.push_back(RouteAction{RouteAction::Kind::Generate, 0, final_});
    generated_ = true;
  };
  if (!incremental_) {  // accumulate-then-generate (router.cpp:118-132)
    for (const auto& s : slots_)
      if (!s.closed) return out;
    seal(assemble(tmpl_, received()));
    return out;
  }
  if (scheduled_ == 0 && pending_.empty() && active_ == 0)
    pending_.insert(pending_.end(), tmpl_.prefix().begin(), tmpl_.prefix().end());
  // Feed the active slot; a closed, fully forwarded slot hands over to the next.
  while (active_ < static_cast<int>(slots_.size())) {
    State& s = slots_[static_cast<std::size_t>(active_)];
    if (!s.sep_issued) {
      s.mark = scheduled_ + static_cast<int>(pending_.size());
      pending_.insert(pending_.end(), s.spec.separator.begin(), s.spec.separator.end());
      s.sep_issued = true;
    }
    if (s.issued < static_cast<int>(s.received.size())) {
      pending_.insert(pending_.end(), s.received.begin() + s.issued, s.received.end());
      s.issued = static_cast<int>(s.received.size());
    }
    if (!s.closed) break;
    ++active_;
  }
  if (active_ < static_cast<int>(slots_.size())) {
    emit_pending(out);
    return out;
  }
  if (!suffix_done_) {
    pending_.insert(pending_.end(), tmpl_.suffix().begin(), tmpl_.suffix().end());
    suffix_done_ = true;
  }
  emit_pending(out);
  TokenSeq full = assemble(tmpl_, received());
  if (full != stream_)
    throw RunError("router: issued prompt diverged from template assembly for " + self_.str());
  seal(std::move(full));
  return out;
}

}  // namespace moa
