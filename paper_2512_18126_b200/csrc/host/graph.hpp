// Tree / all-to-all agent graph, prompt templates and the slot-filling shell
// router.  Semantics follow the reference's proj/core:
//   Topology        topology.hpp:28-80, topology.cpp:43-196
//   PromptTemplate  prompt.hpp:27-85,   prompt.cpp:8-78
//   SlotPlan        router.hpp:36-90,   router.cpp:9-184
// Token sequences may carry *symbolic* ids (< 0) that name a token the GPU
// has produced but the host has not read back; every
// operation here only concatenates, slices and compares them.
#pragma once

#include <map>
#include <optional>
#include <vector>

#include "common.hpp"

namespace moa {

enum class TopologyKind { Tree, AllToAll };

class Topology {
 public:
  static Topology tree(const std::vector<int>& widths, const std::vector<int>& branching);
  static Topology tree_custom(const std::vector<int>& widths,
                              const std::vector<std::vector<int>>& cluster_sizes);
  static Topology all_to_all(const std::vector<int>& widths);

  TopologyKind kind() const { return kind_; }
  int depth() const { return static_cast<int>(layers_.size()); }
  int agent_count() const;
  const std::vector<std::vector<AgentId>>& layers() const { return layers_; }
  const std::vector<AgentId>& layer(int l) const;
  const std::vector<AgentId>& precursors(const AgentId& a) const;
  std::vector<AgentId> successors(const AgentId& a) const;
  std::vector<std::vector<AgentId>> clusters_of_layer(int l) const;
  const AgentId& root() const;

 private:
  Topology() = default;
  void build_edges();
  TopologyKind kind_ = TopologyKind::Tree;
  std::vector<std::vector<AgentId>> layers_;
  std::vector<std::vector<int>> sizes_;
  std::map<AgentId, std::vector<AgentId>> pre_;
};

struct Slot {
  AgentId precursor;
  TokenSeq separator;
};

class PromptTemplate {
 public:
  PromptTemplate() = default;
  PromptTemplate(TokenSeq prefix, std::vector<Slot> slots, TokenSeq suffix);
  const TokenSeq& prefix() const { return prefix_; }
  const std::vector<Slot>& slots() const { return slots_; }
  const TokenSeq& suffix() const { return suffix_; }
  PromptTemplate without(const AgentId& pruned) const;

 private:
  TokenSeq prefix_;
  std::vector<Slot> slots_;
  TokenSeq suffix_;
};

TokenSeq assemble(const PromptTemplate& t, const std::map<AgentId, TokenSeq>& outputs);

struct RouteAction {
  enum class Kind { PrefillOnly, Generate, Reclaim };
  Kind kind = Kind::PrefillOnly;
  int start = 0;
  TokenSeq tokens;
};

// Incremental slot filling for one dependent agent (router.hpp:20-35).
class SlotPlan {
 public:
  SlotPlan(AgentId self, PromptTemplate tmpl, bool incremental);

  std::vector<RouteAction> start();
  std::vector<RouteAction> on_chunk(const AgentId& producer, const TokenSeq& tokens);
  std::vector<RouteAction> on_precursor_done(const AgentId& producer);
  std::vector<RouteAction> on_precursor_cancelled(const AgentId& producer);

  bool started() const { return started_; }
  bool generate_issued() const { return generated_; }
  int scheduled() const { return scheduled_; }
  int prefill_only_calls() const { return calls_; }
  int reclaims() const { return reclaims_; }
  bool all_inputs_pruned() const { return had_slots_ && slots_.empty(); }
  const TokenSeq& final_prompt() const;
  const PromptTemplate& current_template() const { return tmpl_; }

 private:
  struct State {
    Slot spec;
    TokenSeq received;
    int issued = 0;
    bool sep_issued = false;
    bool closed = false;
    int mark = 0;
  };
  int find(const AgentId& p) const;
  std::map<AgentId, TokenSeq> received() const;
  std::vector<RouteAction> step();
  void emit_pending(std::vector<RouteAction>& out);

  AgentId self_;
  PromptTemplate tmpl_;
  bool incremental_;
  bool started_ = false;
  bool had_slots_ = false;
  bool suffix_done_ = false;
  bool generated_ = false;
  int active_ = 0;
  int scheduled_ = 0;
  int calls_ = 0;
  int reclaims_ = 0;
  std::vector<State> slots_;
  TokenSeq pending_;
  TokenSeq stream_;
  TokenSeq final_;
};

}  // namespace moa
