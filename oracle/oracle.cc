// oracle.cc — CPU parity oracle for the candidate-evaluation hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library; the
// product engine (paper_2112_02958_b200/) never links or calls it.
//
// Layers:
//   * propagate / lower_to_spmd / collective_stats: the REFERENCE ITSELF,
//     compiled from /root/reference/proj with patches A-C (oracle/patch_ref.py,
//     SURVEY.md Appendix A) into oracle/_ref/.
//   * cost model (SPEC cost module, absent from the reference: CMakeLists.txt:24)
//     and the rollout policy / scope grouping (SPEC search module, absent:
//     CMakeLists.txt:26): our restatement, conventions frozen in SURVEY.md
//     Appendix B.5 and DESIGN.md §4.
// Parity pins: tests/test_oracle_golden.py checks this oracle against every
// worked example of SPEC.md (Fig. 2/3 types, 2048 B all_reduce, Megatron
// 4 x all_reduce / 1024 B, 10,752 B peak liveness, 16,896 flops, legal-action
// counts).
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "partir/error.h"
#include "partir/ir.h"
#include "partir/parser.h"
#include "partir/printer.h"
#include "partir/propagate.h"
#include "partir/rewrite.h"
#include "partir/spmd.h"
#include "partir/interp.h"
#include "pe.h"

using namespace partir;

extern "C" void oracle_default_cost_params(pe_cost_params* out);
extern "C" void oracle_default_search_config(pe_search_config* out);

namespace {

// ---- scope grouping (normalisation rule SPEC:568) ----------
// Strip digit-only path segments and a trailing `_<digits>` suffix of every
// segment: "layer_3/attention/q_proj" -> "layer/attention/q_proj".
std::string normalize_scope(const std::string& s) {
  std::string out;
  size_t i = 0;
  while (i <= s.size()) {
    size_t j = s.find('/', i);
    if (j == std::string::npos) j = s.size();
    std::string seg = s.substr(i, j - i);
    bool all_digits = !seg.empty() &&
        std::all_of(seg.begin(), seg.end(), [](char c) { return c >= '0' && c <= '9'; });
    if (!all_digits) {
      size_t k = seg.size();
      while (k > 0 && seg[k - 1] >= '0' && seg[k - 1] <= '9') --k;
      if (k < seg.size() && k > 0 && seg[k - 1] == '_') seg = seg.substr(0, k - 1);
      if (!out.empty()) out += '/';
      out += seg;
    }
    i = j + 1;
  }
  return out;
}

struct Setup {
  Program root;
  std::vector<std::string> names;          // value index -> id (args, then ops)
  std::map<std::string, int> op_index;     // original op id -> op index
  std::vector<std::vector<int>> groups;    // group -> member arg indices
  std::vector<std::vector<int>> entries;   // worklist entries (groups or singletons)
  std::vector<int> entry_val;              // action value per entry
  std::vector<int> auto_axes;
  pe_search_config cfg;
  pe_cost_params cp;
  int64_t baseline_bytes = 1;
};

void build_groups(Setup& s) {
  std::map<std::string, int> key_to_group;
  for (size_t a = 0; a < s.root.args.size(); ++a) {
    const std::string& sc = s.root.args[a].scope;
    if (sc.empty()) {
      s.groups.push_back({(int)a});
      continue;
    }
    std::string key = normalize_scope(sc);
    auto it = key_to_group.find(key);
    if (it == key_to_group.end()) {
      key_to_group[key] = (int)s.groups.size();
      s.groups.push_back({(int)a});
    } else {
      s.groups[it->second].push_back((int)a);
    }
  }
  // ranker top-k filter (pe.h worklist_args; SPEC build_worklist "optionally
  // filtered to ranker top-k"): an argument entry is kept when listed, a
  // group when any member is listed
  std::vector<char> keep(s.root.args.size(), s.cfg.worklist_args ? 0 : 1);
  for (uint32_t i = 0; s.cfg.worklist_args && i < s.cfg.n_worklist_args; ++i)
    if (s.cfg.worklist_args[i] < keep.size()) keep[s.cfg.worklist_args[i]] = 1;
  s.cfg.worklist_args = nullptr;  // read once
  // worklist entries and the action value each one decodes to (the group
  // index for TILE_GROUP, the argument for TILE)
  if (s.cfg.group_scopes) {
    for (size_t gi = 0; gi < s.groups.size(); ++gi) {
      if (s.cfg.scoped_only && s.root.args[s.groups[gi][0]].scope.empty()) continue;
      bool any = false;
      for (int m : s.groups[gi]) any = any || keep[m];
      if (!any) continue;
      s.entries.push_back(s.groups[gi]);
      s.entry_val.push_back((int)gi);
    }
  } else {
    for (size_t a = 0; a < s.root.args.size(); ++a) {
      if (s.cfg.scoped_only && s.root.args[a].scope.empty()) continue;
      if (!keep[a]) continue;
      s.entries.push_back({(int)a});
      s.entry_val.push_back((int)a);
    }
  }
}

// ---- cost model (SPEC cost module; conventions SURVEY.md B.5) -----------
int64_t local_bytes(const DistType& t, const Mesh& m) {
  int64_t b = 4;
  for (int64_t d : t.local(m)) b *= d;
  return b;
}

struct Cost {
  int64_t peak = 0, flops = 0;
};

// peak_liveness: arguments live for the whole program; an op result is live
// over [def, last use]; the returned value to the end (B.5.1).  flops on
// LOCAL shapes (B.5.3).
Cost cost_of(const SpmdProgram& sp) {
  Cost c;
  const Mesh& m = sp.mesh;
  int64_t base = 0;
  for (const SpmdArg& a : sp.args) base += local_bytes(a.type, m);
  size_t n = sp.ops.size();
  std::map<std::string, size_t> def;
  for (size_t j = 0; j < n; ++j) def[sp.ops[j].id] = j;
  std::vector<size_t> last(n);
  for (size_t j = 0; j < n; ++j) last[j] = j;
  for (size_t k = 0; k < n; ++k)
    for (const std::string& o : sp.ops[k].operands) {
      auto it = def.find(o);
      if (it != def.end()) last[it->second] = std::max(last[it->second], k);
    }
  {
    auto it = def.find(sp.result_id);
    if (it != def.end() && n > 0) last[it->second] = n - 1;
  }
  std::vector<int64_t> delta(n + 1, 0);
  for (size_t j = 0; j < n; ++j) {
    int64_t b = sp.ops[j].result_type.byte_size();
    delta[j] += b;
    delta[last[j] + 1] -= b;
  }
  int64_t run = 0, best = 0;
  for (size_t i = 0; i < n; ++i) {
    run += delta[i];
    best = std::max(best, run);
  }
  c.peak = base + best;
  for (const Operation& op : sp.ops) {
    switch (op.kind) {
      case OpKind::kDot: {
        std::vector<int64_t> l = sp.type_of(op.operands[0]).local(m);
        std::vector<int64_t> r = sp.type_of(op.operands[1]).local(m);
        int64_t f = 2;
        for (int64_t d : l) f *= d;  // batch x lhs free x contract
        std::set<int> rused(op.dot.rhs_batch.begin(), op.dot.rhs_batch.end());
        rused.insert(op.dot.rhs_contract.begin(), op.dot.rhs_contract.end());
        for (int i = 0; i < (int)r.size(); ++i)
          if (!rused.count(i)) f *= r[i];  // rhs free
        c.flops += f;
        break;
      }
      case OpKind::kAdd: case OpKind::kSub: case OpKind::kMul: case OpKind::kDiv:
      case OpKind::kMaximum: case OpKind::kNeg: case OpKind::kExp:
      case OpKind::kTanh: case OpKind::kRsqrt:
        c.flops += op.result_type.num_elements();
        break;
      case OpKind::kReduceSum: case OpKind::kReduceMax: {
        int64_t e = 1;
        for (int64_t d : sp.type_of(op.operands[0]).local(m)) e *= d;
        c.flops += e;
        break;
      }
      default:
        break;  // constant/transpose/reshape/broadcast/slice/concat/collectives: 0
    }
  }
  return c;
}

// runtime_estimate and reward with a fixed IEEE operation order (B.5.4-5).
void finish_costs(pe_result& r, const pe_cost_params& cp, int64_t baseline) {
  int64_t ar = 0, ag = 0, arc = 0, agc = 0;
  for (int a = 0; a < PE_MAX_AXES; ++a) {
    ar += r.ar_bytes[a];
    ag += r.ag_bytes[a];
    arc += r.ar_cnt[a];
    agc += r.ag_cnt[a];
  }
  r.reduction_bytes = ar;
  r.baseline_bytes = baseline;
  volatile double rt = (double)r.flops / cp.flops_per_second;
  volatile double comm = (double)(ar + ag) / cp.bytes_per_second;
  rt = rt + comm;
  volatile double lat = cp.collective_latency_s * (double)(arc + agc);
  rt = rt + lat;
  r.runtime_s = rt;
  r.feasible = r.peak_bytes <= cp.memory_budget_bytes ? 1 : 0;
  if (!r.feasible) {
    r.reward = 0.0;
  } else {
    volatile double t1 = (double)ar / (double)baseline;
    volatile double t2 = (double)r.peak_bytes / (double)cp.memory_budget_bytes;
    volatile double t3 = (double)r.n_steps;
    volatile double d = 1.0;
    volatile double x = cp.w_comm * t1;
    d = d + x;
    x = cp.w_mem * t2;
    d = d + x;
    x = cp.w_steps * t3;
    d = d + x;
    r.reward = 1.0 / d;
  }
}

uint32_t spec_word(const DistType& t, const Mesh& m) {
  uint32_t w = 0;
  for (size_t d = 0; d < t.spec.dim_axes.size() && d < 4; ++d)
    if (!t.spec.dim_axes[d].empty())
      w |= (uint32_t)(m.axis_index(t.spec.dim_axes[d]) + 1) << (4 * d);
  for (const std::string& a : t.spec.pending_sum) w |= 1u << (16 + m.axis_index(a));
  w |= (uint32_t)t.global.rank() << 24;
  return w;
}

struct TraceWriter {
  int32_t* buf;
  uint32_t cap;
  uint32_t n = 1;
  bool overflow = false;
  void put(int64_t v) {
    if (buf == nullptr) return;
    if (n < cap) buf[n] = (int32_t)v;
    else overflow = true;
    ++n;
  }
  void finish() {
    if (buf == nullptr || cap == 0) return;
    buf[0] = overflow ? -(int32_t)n : (int32_t)n;
  }
};

void score(const Setup& s, const Program& p, const std::vector<StuckNode>& stuck,
           pe_result& r, int32_t* trace, uint32_t trace_words) {
  SpmdProgram sp = lower_to_spmd(p);
  CollectiveStats st = collective_stats(sp);
  const Mesh& m = sp.mesh;
  for (auto& [axis, e] : st.all_reduce) {
    r.ar_cnt[m.axis_index(axis)] = (int32_t)e.count;
    r.ar_bytes[m.axis_index(axis)] = e.bytes;
  }
  for (auto& [axis, e] : st.all_gather) {
    r.ag_cnt[m.axis_index(axis)] = (int32_t)e.count;
    r.ag_bytes[m.axis_index(axis)] = e.bytes;
  }
  for (auto& [axis, e] : st.slice_by_coord) r.sbc_cnt[m.axis_index(axis)] = (int32_t)e.count;
  Cost c = cost_of(sp);
  r.peak_bytes = c.peak;
  r.flops = c.flops;
  r.n_spmd_ops = (int32_t)sp.ops.size();
  r.n_stuck = (int32_t)stuck.size();
  finish_costs(r, s.cp, s.baseline_bytes);
  if (trace == nullptr) return;
  TraceWriter tw{trace, trace_words};
  tw.put((int64_t)sp.args.size());
  std::map<std::string, int64_t> buf_index;
  for (size_t i = 0; i < sp.args.size(); ++i) {
    tw.put(spec_word(sp.args[i].type, m));
    buf_index[sp.args[i].id] = (int64_t)i;
  }
  tw.put(spec_word(sp.type_of(sp.result_id), m));
  tw.put((int64_t)stuck.size());
  for (const StuckNode& sn : stuck) {
    auto it = s.op_index.find(sn.op_id);
    tw.put(it == s.op_index.end() ? -1 : it->second);
    tw.put((int64_t)sn.reason);
  }
  tw.put((int64_t)sp.ops.size());
  for (size_t j = 0; j < sp.ops.size(); ++j) {
    const Operation& op = sp.ops[j];
    int axis = op.axis.empty() ? -1 : m.axis_index(op.axis);
    int dim = (op.kind == OpKind::kAllGather || op.kind == OpKind::kSliceByCoord) ? op.dim : -1;
    tw.put((int64_t)op.kind | ((int64_t)(axis + 1) << 8) | ((int64_t)(dim + 1) << 12) |
           ((int64_t)op.operands.size() << 16));
    int64_t b = op.result_type.byte_size();
    tw.put(b & 0xffffffff);
    tw.put(b >> 32);
    tw.put(spec_word(sp.type_of(op.id), m));
    for (const std::string& o : op.operands) {
      auto it = buf_index.find(o);
      tw.put(it == buf_index.end() ? -1 : it->second);
    }
    buf_index[op.id] = (int64_t)(sp.args.size() + j);
  }
  tw.finish();
}

bool member_legal(const Setup& s, const Program& p, int arg, int dim, int axis) {
  const Argument& a = s.root.args[arg];
  if (dim >= a.type.rank()) return false;
  if (a.type.shape[dim] % s.root.mesh.axes[axis].size != 0) return false;
  return !carries_tiling(p, a.id);
}

// Applies one action; returns false when illegal.  Throws partir::Error from
// propagate (internal / validation failures).
bool apply_action(const Setup& s, Program& p, std::vector<StuckNode>& stuck,
                  const pe_action& act) {
  if (act.kind == PE_ACT_INFER_REST) {
    // the reference's own infer_rest (REF propagate.cc:484-544) over the
    // auto axes; the stuck list is that of the resulting fixpoint
    std::vector<std::string> axes;
    for (int ax : s.auto_axes) axes.push_back(s.root.mesh.axes[ax].name);
    p = infer_rest(p, axes);
    PropagateResult pr = propagate(p);
    p = std::move(pr.program);
    stuck = std::move(pr.stuck);
    return true;
  }
  const std::string& axis = s.root.mesh.axes.at(act.axis).name;
  if (act.kind == PE_ACT_TILE) {
    if (act.value >= s.names.size()) return false;
    try {
      p = apply_tile_action(p, s.names[act.value], act.dim, axis);
    } catch (const IllegalActionError&) {
      return false;
    }
  } else if (act.kind == PE_ACT_TILE_GROUP) {
    if (act.value >= s.groups.size()) return false;
    int applied = 0;
    for (int m : s.groups[act.value]) {
      try {
        p = apply_tile_action(p, s.root.args[m].id, act.dim, axis);
        ++applied;
      } catch (const IllegalActionError&) {
      }
    }
    if (applied == 0) return false;
  } else {
    return false;
  }
  PropagateResult pr = propagate(p);
  p = std::move(pr.program);
  stuck = std::move(pr.stuck);
  return true;
}

void eval_one(const Setup& s, const pe_action* acts, uint32_t n, pe_result& r,
              int32_t* trace, uint32_t trace_words) {
  std::memset(&r, 0, sizeof(r));
  r.fail_step = -1;
  Program p = s.root;
  std::vector<StuckNode> stuck;
  try {
    for (uint32_t k = 0; k < n; ++k) {
      if (acts[k].kind == PE_ACT_STOP) break;
      // tiles the engine inferred while expanding an INFER_REST decision are
      // re-derived here by the reference's infer_rest itself
      if (acts[k].pad & PE_ACT_FLAG_INFERRED) continue;
      if (!apply_action(s, p, stuck, acts[k])) {
        r.status = PE_CAND_ILLEGAL;
        r.fail_step = (int32_t)k;
        break;
      }
      r.n_steps++;
    }
    score(s, p, stuck, r, trace, trace_words);
  } catch (const Error&) {
    int32_t steps = r.n_steps, fs = r.n_steps;
    std::memset(&r, 0, sizeof(r));
    r.status = PE_CAND_INTERNAL;
    r.n_steps = steps;
    r.fail_step = fs;
    if (trace != nullptr && trace_words > 0) trace[0] = 0;
  }
}

// splitmix64 (declared rollout RNG)
uint64_t splitmix_next(uint64_t& st) {
  st += 0x9E3779B97F4A7C15ull;
  uint64_t z = st;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Stuck resurfacing (pe.h resurface_stuck; SPEC Worklist "plus stuck nodes
// resurfaced by propagation", "deterministic order (argument order, then
// stuck discovery order)"): after every decision the ops of the fixpoint's
// stuck list (REF propagate.cc:412-454, in its order) join the worklist
// once each.
struct Resurfaced {
  std::vector<int> ops;     // op indices in discovery order
  std::vector<char> seen;   // per op
};

void resurface(const Setup& s, const std::vector<StuckNode>& stuck, Resurfaced& R) {
  if (!s.cfg.resurface_stuck) return;
  if (R.seen.empty()) R.seen.assign(s.root.ops.size(), 0);
  for (const StuckNode& sn : stuck) {
    auto it = s.op_index.find(sn.op_id);
    if (it == s.op_index.end() || R.seen[it->second]) continue;
    R.seen[it->second] = 1;
    R.ops.push_back(it->second);
  }
}

// TileValue ordinals (worklist entries x dims x auto axes)
uint32_t tile_ordinals(const Setup& s) {
  size_t entries = s.entries.size() + (s.cfg.resurface_stuck ? s.root.ops.size() : 0);
  return (uint32_t)(entries * PE_MAX_RANK * s.auto_axes.size());
}
// every action ordinal but Stop: TileValue, then InferRest when it is an
// action (pe.h infer_rest_action; SPEC legal_actions order)
uint32_t num_ordinals(const Setup& s) {
  return tile_ordinals(s) + (s.cfg.infer_rest_action ? 1 : 0);
}
// SPEC legal_actions: InferRest "if any argument untiled"
bool infer_rest_legal(const Setup& s, const Program& p) {
  if (!s.cfg.infer_rest_action) return false;
  for (const Argument& a : s.root.args)
    if (!carries_tiling(p, a.id)) return true;
  return false;
}

// TileValue(op result, d, axis) is legal when apply_tile_action would
// accept it (REF rewrite.cc:53-75): the value exists at top level, the dim
// divides, and it carries no tiling yet.
bool op_value_legal(const Setup& s, const Program& p, int o, int d, int axis) {
  const Operation& op0 = s.root.ops[o];
  if (d >= op0.result_type.rank()) return false;
  if (op0.result_type.shape[d] % s.root.mesh.axes[axis].size != 0) return false;
  bool exists = false;
  for (const Operation& op : p.ops)
    if (op.id == op0.id) exists = true;
  return exists && !carries_tiling(p, op0.id);
}

std::vector<uint32_t> legal_ordinals(const Setup& s, const Program& p,
                                     const Resurfaced& R = Resurfaced()) {
  std::vector<uint32_t> out;
  std::vector<char> carries(s.root.args.size());
  for (size_t a = 0; a < s.root.args.size(); ++a) carries[a] = carries_tiling(p, s.root.args[a].id);
  uint32_t na = (uint32_t)s.auto_axes.size();
  for (size_t e = 0; e < s.entries.size(); ++e)
    for (int d = 0; d < PE_MAX_RANK; ++d)
      for (uint32_t ai = 0; ai < na; ++ai) {
        int axis = s.auto_axes[ai];
        bool ok = false;
        for (int m : s.entries[e]) {
          const Argument& a = s.root.args[m];
          if (d < a.type.rank() && a.type.shape[d] % s.root.mesh.axes[axis].size == 0 &&
              !carries[m]) {
            ok = true;
            break;
          }
        }
        if (ok) out.push_back((uint32_t)((e * PE_MAX_RANK + d) * na + ai));
      }
  // resurfaced stuck nodes, in discovery order
  size_t E = s.entries.size();
  for (int o : R.ops)
    for (int d = 0; d < PE_MAX_RANK; ++d)
      for (uint32_t ai = 0; ai < na; ++ai)
        if (op_value_legal(s, p, o, d, s.auto_axes[ai]))
          out.push_back((uint32_t)(((E + o) * PE_MAX_RANK + d) * na + ai));
  return out;
}

pe_action ordinal_action(const Setup& s, uint32_t ord) {
  uint32_t na = (uint32_t)s.auto_axes.size();
  pe_action a{};
  if (s.cfg.infer_rest_action && ord == tile_ordinals(s)) {
    a.kind = PE_ACT_INFER_REST;
    return a;
  }
  uint32_t ai = ord % na;
  uint32_t d = (ord / na) % PE_MAX_RANK;
  uint32_t e = ord / na / PE_MAX_RANK;
  a.axis = (uint8_t)s.auto_axes[ai];
  a.dim = (uint8_t)d;
  if (e >= s.entries.size()) {  // resurfaced stuck node: TileValue(op result)
    a.kind = PE_ACT_TILE;
    a.value = (uint32_t)(s.root.args.size() + (e - s.entries.size()));
    return a;
  }
  a.kind = s.cfg.group_scopes ? PE_ACT_TILE_GROUP : PE_ACT_TILE;
  a.value = (uint32_t)s.entry_val[e];
  return a;
}

void rollout_one(const Setup& s, const pe_action* prefix, uint32_t n_prefix, uint64_t seed,
                 pe_action* acts_out, uint32_t* n_out, pe_result& r, uint64_t* legal_out) {
  std::memset(&r, 0, sizeof(r));
  r.fail_step = -1;
  Program p = s.root;
  std::vector<StuckNode> stuck;
  Resurfaced R;
  uint32_t nacts = 0;
  uint32_t maxd = s.cfg.max_decisions;
  uint32_t nwords = (num_ordinals(s) + 63) / 64;
  if (legal_out) std::fill(legal_out, legal_out + nwords, 0ull);
  try {
    bool terminal = false;
    const pe_action ir_marker{0, 0, 0, PE_ACT_INFER_REST, 0};
    for (uint32_t k = 0; k < n_prefix; ++k) {
      if (prefix[k].kind == PE_ACT_STOP) {
        terminal = true;
        break;
      }
      // tiles an engine inferred for an InferRest decision are re-derived
      // here by the reference's infer_rest on the decision itself
      if (prefix[k].pad & PE_ACT_FLAG_INFERRED) continue;
      if (!apply_action(s, p, stuck, prefix[k])) {
        r.status = PE_CAND_ILLEGAL;
        r.fail_step = (int32_t)k;
        terminal = true;
        break;
      }
      resurface(s, stuck, R);
      // decisions are recorded; InferRest as its (unexpanded) decision
      if (nacts < maxd) acts_out[nacts] = prefix[k].kind == PE_ACT_INFER_REST ? ir_marker : prefix[k];
      ++nacts;
      r.n_steps++;
    }
    if (r.status == PE_CAND_OK) {
      std::vector<uint32_t> legal = legal_ordinals(s, p, R);
      bool ir = infer_rest_legal(s, p);
      if (legal_out) {
        for (uint32_t o : legal) legal_out[o / 64] |= 1ull << (o % 64);
        if (ir) legal_out[tile_ordinals(s) / 64] |= 1ull << (tile_ordinals(s) % 64);
      }
      uint64_t st = seed;
      while (!terminal) {
        // uniform over TileValue + InferRest, then Stop (weight 1 before the
        // first decision, 2 after)
        if ((uint32_t)r.n_steps >= maxd || legal.size() + (ir ? 1 : 0) == 0) break;
        uint64_t ws = r.n_steps >= 1 ? 2 : 1;
        uint64_t total = legal.size() + (ir ? 1 : 0) + ws;
        uint64_t pick = splitmix_next(st) % total;
        if (pick >= legal.size() + (ir ? 1 : 0)) break;
        pe_action a = pick == legal.size() ? ir_marker : ordinal_action(s, legal[pick]);
        if (!apply_action(s, p, stuck, a)) {
          r.status = PE_CAND_ILLEGAL;  // cannot happen: legal by construction
          r.fail_step = (int32_t)nacts;
          break;
        }
        resurface(s, stuck, R);
        if (nacts < maxd) acts_out[nacts] = a;
        ++nacts;
        r.n_steps++;
        legal = legal_ordinals(s, p, R);
        ir = infer_rest_legal(s, p);
      }
    }
    *n_out = std::min(nacts, maxd);
    score(s, p, stuck, r, nullptr, 0);
  } catch (const Error&) {
    int32_t steps = r.n_steps;
    std::memset(&r, 0, sizeof(r));
    r.status = PE_CAND_INTERNAL;
    r.n_steps = steps;
    r.fail_step = steps;
    *n_out = std::min(nacts, maxd);
  }
}

template <typename F>
void parallel_for(uint32_t n, int threads, F&& f) {
  if (threads <= 1 || n <= 1) {
    for (uint32_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<uint32_t> next{0};
  std::vector<std::thread> pool;
  int t = std::min<int>(threads, (int)n);
  for (int k = 0; k < t; ++k)
    pool.emplace_back([&] {
      for (;;) {
        uint32_t i = next.fetch_add(1);
        if (i >= n) break;
        f(i);
      }
    });
  for (auto& th : pool) th.join();
}

int make_setup(Setup& s, const char* pir, size_t len, const pe_search_config* cfg,
               const pe_cost_params* cp, char* err, size_t errcap) {
  try {
    s.root = parse_program(std::string_view(pir, len));
  } catch (const Error& e) {
    if (err) std::snprintf(err, errcap, "%s", e.what());
    return 1;
  }
  if (s.root.mesh.axes.size() > PE_MAX_AXES) {
    if (err) std::snprintf(err, errcap, "more than %d mesh axes", PE_MAX_AXES);
    return 4;
  }
  oracle_default_search_config(&s.cfg);
  oracle_default_cost_params(&s.cp);
  if (cfg) s.cfg = *cfg;
  if (cp) s.cp = *cp;
  for (const Argument& a : s.root.args) s.names.push_back(a.id);
  for (size_t i = 0; i < s.root.ops.size(); ++i) {
    s.names.push_back(s.root.ops[i].id);
    s.op_index[s.root.ops[i].id] = (int)i;
  }
  for (size_t a = 0; a < s.root.mesh.axes.size(); ++a)
    if (s.cfg.auto_axes_mask & (1u << a)) s.auto_axes.push_back((int)a);
  build_groups(s);
  try {
    SpmdProgram sp = lower_to_spmd(s.root);
    s.baseline_bytes = std::max<int64_t>(1, cost_of(sp).peak);
  } catch (const Error& e) {
    if (err) std::snprintf(err, errcap, "%s", e.what());
    return 70;
  }
  return 0;
}

}  // namespace

extern "C" {

void oracle_default_cost_params(pe_cost_params* out) {
  out->memory_budget_bytes = 16ll << 30;
  out->flops_per_second = 1e14;
  out->bytes_per_second = 1e11;
  out->collective_latency_s = 1e-6;
  out->w_mem = 0.1;
  out->w_comm = 1.0;
  out->w_steps = 0.01;
}

void oracle_default_search_config(pe_search_config* out) {
  std::memset(out, 0, sizeof(*out));
  out->auto_axes_mask = 0xffffffffu;
  out->max_decisions = 32;
  out->group_scopes = 1;
  out->episodes = 500;
  out->seed = 0;
  out->uct_c = 1.414;
  out->leaf_batch = 8192;
}

// Evaluate explicit action sequences.  Returns 0 on success, else an error
// code with a message in err.
int oracle_eval_batch(const char* pir, size_t len, const pe_search_config* cfg,
                      const pe_cost_params* cp, const pe_action* acts, const uint32_t* off,
                      uint32_t n, pe_result* out, int32_t* trace, uint32_t trace_words,
                      int threads, char* err, size_t errcap) {
  Setup s;
  int rc = make_setup(s, pir, len, cfg, cp, err, errcap);
  if (rc) return rc;
  parallel_for(n, threads, [&](uint32_t c) {
    eval_one(s, acts + off[c], off[c + 1] - off[c], out[c],
             trace ? trace + (size_t)c * trace_words : nullptr, trace_words);
  });
  return 0;
}

int oracle_rollout_batch(const char* pir, size_t len, const pe_search_config* cfg,
                         const pe_cost_params* cp, const pe_action* prefix,
                         const uint32_t* prefix_off, const uint64_t* seeds, uint32_t n,
                         pe_action* acts_out, uint32_t* n_acts_out, pe_result* out,
                         uint64_t* legal_out, int threads, char* err, size_t errcap) {
  Setup s;
  int rc = make_setup(s, pir, len, cfg, cp, err, errcap);
  if (rc) return rc;
  uint32_t maxd = s.cfg.max_decisions;
  uint32_t nwords = (num_ordinals(s) + 63) / 64;
  parallel_for(n, threads, [&](uint32_t c) {
    rollout_one(s, prefix + prefix_off[c], prefix_off[c + 1] - prefix_off[c], seeds[c],
                acts_out + (size_t)c * maxd, n_acts_out + c, out[c],
                legal_out ? legal_out + (size_t)c * nwords : nullptr);
  });
  return 0;
}

// Introspection used by tests.
int oracle_info(const char* pir, size_t len, const pe_search_config* cfg, int64_t* out4,
                char* err, size_t errcap) {
  Setup s;
  int rc = make_setup(s, pir, len, cfg, nullptr, err, errcap);
  if (rc) return rc;
  out4[0] = s.baseline_bytes;
  out4[1] = (int64_t)s.groups.size();
  out4[2] = (int64_t)num_ordinals(s);
  out4[3] = (int64_t)s.entries.size();
  return 0;
}

// legal ordinals of the state reached by `acts` (SPEC legal_actions).
int oracle_legal(const char* pir, size_t len, const pe_search_config* cfg, const pe_action* acts,
                 uint32_t n, uint32_t* ords_out, uint32_t cap, uint32_t* n_out, char* err,
                 size_t errcap) {
  Setup s;
  int rc = make_setup(s, pir, len, cfg, nullptr, err, errcap);
  if (rc) return rc;
  Program p = s.root;
  std::vector<StuckNode> stuck;
  Resurfaced R;
  try {
    for (uint32_t k = 0; k < n; ++k) {
      if (!apply_action(s, p, stuck, acts[k])) return 3;
      resurface(s, stuck, R);
    }
  } catch (const Error& e) {
    if (err) std::snprintf(err, errcap, "%s", e.what());
    return 70;
  }
  std::vector<uint32_t> l = legal_ordinals(s, p, R);
  if (infer_rest_legal(s, p)) l.push_back(tile_ordinals(s));
  *n_out = (uint32_t)l.size();
  for (uint32_t i = 0; i < l.size() && i < cap; ++i) ords_out[i] = l[i];
  return 0;
}

// Semantics check of a plan with the reference interpreter (REF
// interp.cc:640-678 check_equivalence: eval_spmd of the lowered program vs
// eval_base of the original on seeded random inputs).  Used to verify plans
// found by the GPU search.
int oracle_check_equivalence(const char* pir, size_t len, const pe_search_config* cfg,
                             const pe_action* acts, uint32_t n, int trials, uint64_t seed,
                             double* max_abs_diff, int* pass, int* order_preserving, char* err,
                             size_t errcap) {
  Setup s;
  int rc = make_setup(s, pir, len, cfg, nullptr, err, errcap);
  if (rc) return rc;
  Program p = s.root;
  std::vector<StuckNode> stuck;
  try {
    for (uint32_t k = 0; k < n; ++k) {
      if (acts[k].kind == PE_ACT_STOP) break;
      if (acts[k].pad & PE_ACT_FLAG_INFERRED) continue;
      if (!apply_action(s, p, stuck, acts[k])) return 3;
    }
    SpmdProgram sp = lower_to_spmd(p);
    EquivalenceReport rep = check_equivalence(s.root, sp, trials, seed);
    *max_abs_diff = rep.max_abs_diff;
    *pass = rep.pass ? 1 : 0;
    *order_preserving = rep.order_preserving ? 1 : 0;
  } catch (const Error& e) {
    if (err) std::snprintf(err, errcap, "%s", e.what());
    return 70;
  }
  return 0;
}

// Text of the program after `acts` (tiled IR) and its SPMD form, for
// debugging parity failures.
int oracle_debug_text(const char* pir, size_t len, const pe_search_config* cfg,
                      const pe_action* acts, uint32_t n, char* out, size_t cap) {
  Setup s;
  char err[256];
  int rc = make_setup(s, pir, len, cfg, nullptr, err, sizeof(err));
  if (rc) {
    std::snprintf(out, cap, "%s", err);
    return rc;
  }
  Program p = s.root;
  std::vector<StuckNode> stuck;
  std::string text;
  try {
    for (uint32_t k = 0; k < n; ++k)
      if (!apply_action(s, p, stuck, acts[k])) {
        text += "illegal at " + std::to_string(k) + "\n";
        break;
      }
    text += print_program(p);
    SpmdProgram sp = lower_to_spmd(p);
    text += print_spmd(sp);
  } catch (const Error& e) {
    text += std::string("error: ") + e.what() + "\n";
  }
  std::snprintf(out, cap, "%s", text.c_str());
  return 0;
}

}  // extern "C"
