// pe_graph.h — host graph model, loader and compiler (the boundary's
// `parse_program`, REF parser.h:28).
//
// A program enters as `.pir` text (SPEC tensor_ir "External Interfaces";
// reader in pe_pir.cc) or as structured arrays (pe_graph_create_from_arrays),
// is shape-checked (the base-dialect rules REF validate.cc:161-225 enforces)
// and compiled into the SoA tables of pe::GraphView.  Host-only C++; no
// exceptions cross the C-ABI.
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "pe.h"
#include "pe_graph_view.h"

namespace pe {

struct HostOp {
  std::string id;
  Kind kind = kAdd;
  std::vector<int32_t> operands;  // value indices
  std::vector<int64_t> shape;     // result type
  std::string scope;
  std::vector<int> lhs_batch, rhs_batch, lhs_contract, rhs_contract;
  std::vector<int> dims;  // reduce dims / transpose perm / broadcast map
  std::vector<int64_t> start, limit;
  int dim = -1;
  double value = 0.;
};

struct HostArg {
  std::string id;
  std::vector<int64_t> shape;
  std::string scope;
};

struct HostClass {
  Role role;
  int rdim;
  std::vector<std::pair<int, int>> members;  // (operand, dim)
};

struct HostGraph {
  std::string name;
  std::vector<std::string> axis_names;
  std::vector<int64_t> axis_sizes;
  std::vector<HostArg> args;
  std::vector<HostOp> ops;
  int32_t result = -1;

  // compiled tables (see GraphView)
  std::vector<int32_t> vshape;
  std::vector<uint8_t> vrank;
  std::vector<uint8_t> okind, omask, orule_err;
  std::vector<int32_t> oopnd_off, oopnd, slot_op;
  std::vector<int32_t> ocls_off;
  std::vector<uint8_t> cls_role;
  std::vector<int8_t> cls_rdim;
  std::vector<int32_t> cls_moff;
  std::vector<uint16_t> mem;
  std::vector<int16_t> slot_cls, op_rcls;
  std::vector<int32_t> user_off, users, init_uses;
  std::vector<std::vector<int32_t>> groups;  // scope groups

  int32_t num_values() const { return (int32_t)(args.size() + ops.size()); }
  int32_t value_index(const std::string& name) const;
  int32_t axis_index(const std::string& name) const;
  const std::vector<int64_t>& value_shape(int32_t v) const {
    return v < (int32_t)args.size() ? args[v].shape : ops[v - args.size()].shape;
  }
  // GraphView over the host vectors (worklist fields left empty)
  GraphView host_view() const;
};

// SPEC build_worklist (search module): worklist entries are scope groups or
// single arguments; TileValue ordinals enumerate entry x dim x auto axis
// (ordinal = (entry*4 + dim)*n_auto + auto-axis rank).  ord_mem lists, per
// ordinal, the members for which the action is statically legal (rank and
// divisibility, REF rewrite.cc:63-74); the dynamic part (carries_tiling) is
// checked per candidate.
struct Worklist {
  std::vector<int32_t> auto_axes, ent_off, ent_mem, grp_off, grp_mem, ord_off, ord_mem;
  std::vector<int32_t> ent_val;  // action value per entry: group index or argument
  bool groups = true;
  bool resurface = false;  // stuck resurfacing (pe.h resurface_stuck)
  bool infer_rest = false;  // InferRest is an action (pe.h infer_rest_action)
  int32_t n_ops = 0;
  int32_t n_entries() const { return (int32_t)ent_off.size() - 1; }
  // ordinals of the static entries (arguments / groups)
  int32_t n_static_ordinals() const {
    return n_entries() * kMaxRank * (int32_t)auto_axes.size();
  }
  // TileValue ordinals: static entries, then one block per op when stuck
  // nodes can resurface
  int32_t n_ordinals() const {
    return (n_entries() + (resurface ? n_ops : 0)) * kMaxRank * (int32_t)auto_axes.size();
  }
  // every action ordinal but Stop: the TileValue ones, then InferRest
  int32_t n_action_ordinals() const { return n_ordinals() + (infer_rest ? 1 : 0); }
};
// keep = per-argument filter (empty = all arguments; ranker top-k)
Worklist build_worklist(const HostGraph& g, uint32_t auto_axes_mask, bool group_scopes,
                        bool scoped_only = false, bool resurface = false,
                        const std::vector<char>& keep = std::vector<char>());
// the argument filter a search config asks for (empty = all)
std::vector<char> worklist_filter(const HostGraph& g, const pe_search_config& cfg);
// points the worklist fields of `v` at the (host) vectors of `w`
void attach_worklist(GraphView& v, const Worklist& w);

struct LoadError {
  int code = 0;  // pe_status
  int line = 0, column = 0;
  std::string message;
};

// `.pir` text -> HostGraph (pe_pir.cc): syntax only (names resolved,
// nothing shape-checked yet).
bool read_pir(const char* text, size_t len, HostGraph& g, LoadError& err);
// Shape-check + compile a HostGraph however it was built (pe_graph.cc).
bool finish_graph(HostGraph& g, LoadError& err);
// read_pir + finish_graph.  Returns false and fills `err` on failure.
bool load_graph(const char* text, size_t len, HostGraph& g, LoadError& err);

// SPEC:568 scope normalisation used for grouping.
std::string normalize_scope(const std::string& s);

}  // namespace pe
