// pe_graph.cc — graph checking and compilation (host C++).
//
// A HostGraph arrives from the `.pir` reader (pe_pir.cc) or from structured
// arrays (pe_graph_create_from_arrays).  This file checks its shapes (the
// rules REF validate enforces for the base dialect, validate.cc:161-225) and
// precompiles the per-op propagation rules of REF registry.cc:123-206 into
// the flat tables of pe::GraphView.
#include "pe_graph.h"

#include <algorithm>
#include <cctype>
#include <cstdlib>
#include <cstring>
#include <map>
#include <set>

#include "pe.h"
#include "pe_rules.h"

namespace pe {
namespace {

// ---------------------------------------------------------------- checking
// Shape checking of the base dialect: every op's declared result type must
// equal the type its kind infers from its operands (the shape rules of
// SPEC tensor_ir; the reference enforces them in validate, REF
// validate.cc:161-225).  On top of those, the engine's own limits: rank <= 4,
// <= 4 mesh axes, dims and axis sizes that fit int32 (its value records).
struct Bad {
  LoadError e;
};
[[noreturn]] void reject(const std::string& msg, int code = PE_ERR_VALIDATION) {
  Bad b;
  b.e.code = code;
  b.e.message = msg;
  throw b;
}

std::string type_text(const std::vector<int64_t>& dims) {
  std::string t = "f32[";
  for (size_t i = 0; i < dims.size(); ++i) {
    if (i) t += ',';
    t += std::to_string(dims[i]);
  }
  return t + "]";
}

using Shape = std::vector<int64_t>;
// Inference per kind: fills `out` or returns why the op is malformed.
using Infer = std::string (*)(const HostOp& op, const std::vector<Shape>& in, Shape& out);

std::string want_arity(const std::vector<Shape>& in, size_t n) {
  if (in.size() == n) return "";
  return "takes " + std::to_string(n) + " operand" + (n == 1 ? "" : "s") + ", has " +
         std::to_string(in.size());
}
bool dim_ok(int d, size_t rank) { return d >= 0 && (size_t)d < rank; }

std::string infer_nullary(const HostOp& op, const std::vector<Shape>& in, Shape& out) {
  out = op.shape;
  return want_arity(in, 0);
}
std::string infer_unary(const HostOp&, const std::vector<Shape>& in, Shape& out) {
  std::string w = want_arity(in, 1);
  if (w.empty()) out = in[0];
  return w;
}
std::string infer_binary(const HostOp&, const std::vector<Shape>& in, Shape& out) {
  std::string w = want_arity(in, 2);
  if (!w.empty()) return w;
  if (in[0] != in[1]) return "pointwise operands " + type_text(in[0]) + " and " + type_text(in[1]) + " disagree";
  out = in[0];
  return "";
}
std::string infer_dot(const HostOp& op, const std::vector<Shape>& in, Shape& out) {
  std::string w = want_arity(in, 2);
  if (!w.empty()) return w;
  const Shape &l = in[0], &r = in[1];
  if (op.lhs_batch.size() != op.rhs_batch.size() || op.lhs_contract.size() != op.rhs_contract.size())
    return "lhs and rhs dimension lists have different lengths";
  std::vector<char> lused(l.size(), 0), rused(r.size(), 0);
  auto pair_up = [&](const std::vector<int>& a, const std::vector<int>& b, const char* what) {
    for (size_t i = 0; i < a.size(); ++i) {
      if (!dim_ok(a[i], l.size()) || !dim_ok(b[i], r.size()))
        return std::string(what) + " dim pair " + std::to_string(i) + " is out of range";
      if (l[a[i]] != r[b[i]]) return std::string(what) + " dims of different sizes";
      if (lused[a[i]]++ || rused[b[i]]++) return std::string(what) + " dim listed twice";
    }
    return std::string();
  };
  std::string e = pair_up(op.lhs_batch, op.rhs_batch, "batch");
  if (e.empty()) e = pair_up(op.lhs_contract, op.rhs_contract, "contracting");
  if (!e.empty()) return e;
  out.clear();  // batch dims, then lhs free dims, then rhs free dims
  for (int b : op.lhs_batch) out.push_back(l[b]);
  for (size_t i = 0; i < l.size(); ++i)
    if (!lused[i]) out.push_back(l[i]);
  for (size_t i = 0; i < r.size(); ++i)
    if (!rused[i]) out.push_back(r[i]);
  return "";
}
std::string infer_reduce(const HostOp& op, const std::vector<Shape>& in, Shape& out) {
  std::string w = want_arity(in, 1);
  if (!w.empty()) return w;
  std::vector<char> gone(in[0].size(), 0);
  for (int d : op.dims) {
    if (!dim_ok(d, in[0].size())) return "reduced dim " + std::to_string(d) + " is out of range";
    if (gone[d]++) return "reduced dim " + std::to_string(d) + " listed twice";
  }
  out.clear();
  for (size_t i = 0; i < in[0].size(); ++i)
    if (!gone[i]) out.push_back(in[0][i]);
  return "";
}
std::string infer_transpose(const HostOp& op, const std::vector<Shape>& in, Shape& out) {
  std::string w = want_arity(in, 1);
  if (!w.empty()) return w;
  std::vector<char> hit(in[0].size(), 0);
  if (op.dims.size() != in[0].size()) return "permutation length differs from the operand rank";
  out.clear();
  for (int d : op.dims) {
    if (!dim_ok(d, in[0].size()) || hit[d]++) return "perm is not a permutation of the operand dims";
    out.push_back(in[0][d]);
  }
  return "";
}
std::string infer_reshape(const HostOp& op, const std::vector<Shape>& in, Shape& out) {
  std::string w = want_arity(in, 1);
  if (!w.empty()) return w;
  int64_t from = 1, to = 1;
  for (int64_t d : in[0]) from *= d;
  for (int64_t d : op.shape) to *= d;
  if (from != to) return "reshape from " + type_text(in[0]) + " must keep the element count";
  out = op.shape;
  return "";
}
std::string infer_broadcast(const HostOp& op, const std::vector<Shape>& in, Shape& out) {
  std::string w = want_arity(in, 1);
  if (!w.empty()) return w;
  if (op.dims.size() != in[0].size()) return "map needs one entry per operand dim";
  for (size_t i = 0; i < op.dims.size(); ++i) {
    int m = op.dims[i];
    if (!dim_ok(m, op.shape.size())) return "map entry " + std::to_string(m) + " is out of range";
    if (i > 0 && m <= op.dims[i - 1]) return "map entries must increase";
    if (op.shape[m] != in[0][i]) return "operand dim " + std::to_string(i) + " does not fit result dim " + std::to_string(m);
  }
  out = op.shape;
  return "";
}
std::string infer_slice(const HostOp& op, const std::vector<Shape>& in, Shape& out) {
  std::string w = want_arity(in, 1);
  if (!w.empty()) return w;
  size_t r = in[0].size();
  if (op.start.size() != r || op.limit.size() != r) return "start and limit need one entry per dim";
  out.clear();
  for (size_t i = 0; i < r; ++i) {
    if (!(0 <= op.start[i] && op.start[i] < op.limit[i] && op.limit[i] <= in[0][i]))
      return "bounds of dim " + std::to_string(i) + " are not 0 <= start < limit <= size";
    out.push_back(op.limit[i] - op.start[i]);
  }
  return "";
}
std::string infer_concat(const HostOp& op, const std::vector<Shape>& in, Shape& out) {
  if (in.size() < 2) return "concatenates at least two operands";
  if (!dim_ok(op.dim, in[0].size())) return "concatenation dim is out of range";
  out = in[0];
  for (size_t k = 1; k < in.size(); ++k) {
    if (in[k].size() != in[0].size()) return "operands of different ranks";
    for (size_t d = 0; d < in[0].size(); ++d)
      if ((int)d != op.dim && in[k][d] != in[0][d])
        return "operand " + std::to_string(k) + " differs outside the concatenation dim";
    out[op.dim] += in[k][op.dim];
  }
  return "";
}

Infer infer_for(Kind k) {
  switch (k) {
    case kConstant: return infer_nullary;
    case kNeg: case kExp: case kTanh: case kRsqrt: return infer_unary;
    case kAdd: case kSub: case kMul: case kDiv: case kMaximum: return infer_binary;
    case kDot: return infer_dot;
    case kReduceSum: case kReduceMax: return infer_reduce;
    case kTranspose: return infer_transpose;
    case kReshape: return infer_reshape;
    case kBroadcastInDim: return infer_broadcast;
    case kSlice: return infer_slice;
    case kConcatenate: return infer_concat;
    default: return nullptr;
  }
}

void check_dims(const std::string& who, const Shape& s) {
  if ((int)s.size() > kMaxRank) reject(who + ": rank " + std::to_string(s.size()) + " > 4");
  for (int64_t d : s) {
    if (d < 1) reject(who + ": every dimension must be >= 1");
    if (d > kMaxDim) reject(who + ": dimension " + std::to_string(d) + " exceeds 2^31-1", PE_ERR_INVALID_ARGUMENT);
  }
}

void check_graph(const HostGraph& g) {
  if ((int)g.axis_names.size() > kMaxAxes) reject("the engine supports at most 4 mesh axes", PE_ERR_INVALID_ARGUMENT);
  for (size_t a = 0; a < g.axis_names.size(); ++a) {
    const std::string who = "mesh axis \"" + g.axis_names[a] + "\"";
    if (g.axis_names[a].empty()) reject("mesh axes need non-empty names");
    if (g.axis_sizes[a] < 1) reject(who + ": size must be >= 1");
    if (g.axis_sizes[a] > kMaxDim) reject(who + ": size exceeds 2^31-1", PE_ERR_INVALID_ARGUMENT);
    for (size_t b = 0; b < a; ++b)
      if (g.axis_names[b] == g.axis_names[a]) reject(who + " is declared twice");
  }
  if (g.name.empty()) reject("the function has no name");
  for (const HostArg& a : g.args) check_dims("parameter %" + a.id, a.shape);
  std::vector<Shape> in;
  Shape got;
  for (const HostOp& op : g.ops) {
    const std::string who = "%" + op.id;
    check_dims(who, op.shape);
    if (op.operands.size() > 8191) reject(who + ": more than 8191 operands", PE_ERR_INVALID_ARGUMENT);
    Infer f = infer_for(op.kind);
    if (!f) reject(who + ": kind is outside the base dialect");
    in.clear();
    for (int32_t v : op.operands) in.push_back(g.value_shape(v));
    std::string why = f(op, in, got);
    if (!why.empty()) reject(who + ": " + why);
    if ((int)got.size() > kMaxRank) reject(who + ": inferred rank exceeds 4");
    if (got != op.shape)
      reject(who + ": declared " + type_text(op.shape) + " but the operands give " + type_text(got));
  }
  if (g.result < 0) reject("the function returns nothing");
}
// ---------------------------------------------------------------- rules
// Per-op propagation rule with GLOBAL operand shapes (REF registry.cc).
// Class order and member order follow the reference exactly: they fix the
// order in which slices are created during a pull.
bool rule_for(const HostGraph& g, const HostOp& op, std::vector<HostClass>& cls) {
  auto pass = [&](int rd, std::vector<std::pair<int, int>> m) {
    cls.push_back({kPass, rd, std::move(m)});
  };
  auto blocked = [&](std::vector<std::pair<int, int>> m) { cls.push_back({kBlocked, -1, std::move(m)}); };
  auto contract = [&](std::vector<std::pair<int, int>> m) {
    cls.push_back({kContract, -1, std::move(m)});
  };
  auto rank_of = [&](int k) { return (int)g.value_shape(op.operands[k]).size(); };
  switch (op.kind) {
    case kConstant:
      return true;
    case kAdd: case kSub: case kMul: case kDiv: case kMaximum:
      for (int d = 0; d < rank_of(0); ++d) pass(d, {{0, d}, {1, d}});
      return true;
    case kNeg: case kExp: case kTanh: case kRsqrt:
      for (int d = 0; d < rank_of(0); ++d) pass(d, {{0, d}});
      return true;
    case kDot: {
      std::set<int> lu(op.lhs_batch.begin(), op.lhs_batch.end());
      lu.insert(op.lhs_contract.begin(), op.lhs_contract.end());
      std::set<int> ru(op.rhs_batch.begin(), op.rhs_batch.end());
      ru.insert(op.rhs_contract.begin(), op.rhs_contract.end());
      int out = 0;
      for (size_t i = 0; i < op.lhs_batch.size(); ++i)
        pass(out++, {{0, op.lhs_batch[i]}, {1, op.rhs_batch[i]}});
      for (int i = 0; i < rank_of(0); ++i)
        if (!lu.count(i)) pass(out++, {{0, i}});
      for (int i = 0; i < rank_of(1); ++i)
        if (!ru.count(i)) pass(out++, {{1, i}});
      for (size_t i = 0; i < op.lhs_contract.size(); ++i)
        contract({{0, op.lhs_contract[i]}, {1, op.rhs_contract[i]}});
      return true;
    }
    case kReduceSum: case kReduceMax: {
      std::set<int> red(op.dims.begin(), op.dims.end());
      int out = 0;
      for (int d = 0; d < rank_of(0); ++d) {
        if (red.count(d)) {
          if (op.kind == kReduceSum) contract({{0, d}});
          else blocked({{0, d}});
        } else {
          pass(out++, {{0, d}});
        }
      }
      return true;
    }
    case kTranspose:
      for (int i = 0; i < (int)op.dims.size(); ++i) pass(i, {{0, op.dims[i]}});
      return true;
    case kReshape: {
      const auto& a = g.value_shape(op.operands[0]);
      ReshapeRule r = reshape_rule(a.data(), (int)a.size(), op.shape.data(), (int)op.shape.size());
      if (r.error) return false;
      for (int c = 0; c < r.n_cls; ++c) {
        std::vector<std::pair<int, int>> m;
        for (int d = 0; d < (int)a.size(); ++d)
          if (r.cls_of_dim[d] == c) m.push_back({0, d});
        cls.push_back({(Role)r.role[c], r.rdim[c], m});
      }
      return true;
    }
    case kBroadcastInDim:
      for (int d = 0; d < (int)op.dims.size(); ++d) pass(op.dims[d], {{0, d}});
      return true;
    case kSlice: {
      const auto& a = g.value_shape(op.operands[0]);
      for (int d = 0; d < (int)a.size(); ++d) {
        bool full = op.start[d] == 0 && op.limit[d] == a[d];
        if (full) pass(d, {{0, d}});
        else blocked({{0, d}});
      }
      return true;
    }
    case kConcatenate: {
      int rank = rank_of(0);
      int n = (int)op.operands.size();
      for (int d = 0; d < rank; ++d) {
        std::vector<std::pair<int, int>> m;
        for (int i = 0; i < n; ++i) m.push_back({i, d});
        if (d == op.dim) blocked(std::move(m));
        else pass(d, std::move(m));
      }
      return true;
    }
    default:
      return false;
  }
}

void compile(HostGraph& g) {
  int32_t A = (int32_t)g.args.size(), N = (int32_t)g.ops.size(), V = A + N;
  g.vshape.assign((size_t)V * 4, 0);
  g.vrank.assign(V, 0);
  for (int32_t v = 0; v < V; ++v) {
    const auto& s = g.value_shape(v);
    g.vrank[v] = (uint8_t)s.size();
    for (size_t d = 0; d < s.size(); ++d) g.vshape[(size_t)v * 4 + d] = (int32_t)s[d];
  }
  g.okind.resize(N);
  g.omask.assign(N, 0);
  g.orule_err.assign(N, 0);
  g.oopnd_off.assign(N + 1, 0);
  g.ocls_off.assign(N + 1, 0);
  g.op_rcls.assign((size_t)N * 4, -1);
  g.cls_moff.assign(1, 0);
  for (int32_t o = 0; o < N; ++o) {
    const HostOp& op = g.ops[o];
    g.okind[o] = op.kind;
    g.oopnd_off[o + 1] = g.oopnd_off[o] + (int32_t)op.operands.size();
    for (int32_t v : op.operands) {
      g.oopnd.push_back(v);
      g.slot_op.push_back(o);
    }
    if (op.kind == kDot) {
      std::set<int> ru(op.rhs_batch.begin(), op.rhs_batch.end());
      ru.insert(op.rhs_contract.begin(), op.rhs_contract.end());
      int rr = (int)g.value_shape(op.operands[1]).size();
      for (int i = 0; i < rr; ++i)
        if (!ru.count(i)) g.omask[o] |= (uint8_t)(1u << i);
    } else if (op.kind == kBroadcastInDim) {
      for (int m : op.dims) g.omask[o] |= (uint8_t)(1u << m);
    }
  }
  int32_t E = g.oopnd_off[N];
  g.slot_cls.assign((size_t)E * 4, -1);
  for (int32_t o = 0; o < N; ++o) {
    const HostOp& op = g.ops[o];
    std::vector<HostClass> cls;
    if (!rule_for(g, op, cls)) {
      g.orule_err[o] = 1;
      cls.clear();
    }
    int32_t base_cls = (int32_t)g.cls_role.size();
    for (size_t c = 0; c < cls.size(); ++c) {
      g.cls_role.push_back(cls[c].role);
      g.cls_rdim.push_back((int8_t)cls[c].rdim);
      for (auto [k, d] : cls[c].members) {
        g.mem.push_back((uint16_t)((k << 2) | d));
        int16_t& slot = g.slot_cls[(size_t)(g.oopnd_off[o] + k) * 4 + d];
        if (slot < 0) slot = (int16_t)c;  // class_of: first class containing it
      }
      g.cls_moff.push_back((int32_t)g.mem.size());
      // class_for_result: first pass-through class with this result dim
      if (cls[c].role == kPass && cls[c].rdim >= 0 && cls[c].rdim < 4 &&
          g.op_rcls[(size_t)o * 4 + cls[c].rdim] < 0)
        g.op_rcls[(size_t)o * 4 + cls[c].rdim] = (int16_t)c;
    }
    g.ocls_off[o + 1] = base_cls + (int32_t)cls.size();
  }
  // users CSR and count_uses on the root
  g.user_off.assign(V + 1, 0);
  for (int32_t v : g.oopnd) g.user_off[v + 1]++;
  for (int32_t v = 0; v < V; ++v) g.user_off[v + 1] += g.user_off[v];
  g.users.assign(E, 0);
  std::vector<int32_t> fill(g.user_off.begin(), g.user_off.end() - 1);
  for (int32_t s = 0; s < E; ++s) g.users[fill[g.oopnd[s]]++] = s;
  g.init_uses.assign(V, 0);
  for (int32_t v : g.oopnd) g.init_uses[v]++;
  g.init_uses[g.result]++;
  // scope groups
  std::map<std::string, int> key;
  for (int32_t a = 0; a < A; ++a) {
    const std::string& sc = g.args[a].scope;
    if (sc.empty()) {
      g.groups.push_back({a});
      continue;
    }
    std::string k = normalize_scope(sc);
    auto it = key.find(k);
    if (it == key.end()) {
      key[k] = (int)g.groups.size();
      g.groups.push_back({a});
    } else {
      g.groups[it->second].push_back(a);
    }
  }
}

}  // namespace

std::string normalize_scope(const std::string& s) {
  std::string out;
  size_t i = 0;
  while (i <= s.size()) {
    size_t j = s.find('/', i);
    if (j == std::string::npos) j = s.size();
    std::string seg = s.substr(i, j - i);
    bool digits = !seg.empty() && std::all_of(seg.begin(), seg.end(), [](char c) {
      return c >= '0' && c <= '9';
    });
    if (!digits) {
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

int32_t HostGraph::value_index(const std::string& name) const {
  for (size_t a = 0; a < args.size(); ++a)
    if (args[a].id == name) return (int32_t)a;
  for (size_t o = 0; o < ops.size(); ++o)
    if (ops[o].id == name) return (int32_t)(args.size() + o);
  return -1;
}

int32_t HostGraph::axis_index(const std::string& name) const {
  for (size_t a = 0; a < axis_names.size(); ++a)
    if (axis_names[a] == name) return (int32_t)a;
  return -1;
}

GraphView HostGraph::host_view() const {
  GraphView v{};
  v.A = (int32_t)args.size();
  v.N = (int32_t)ops.size();
  v.E = (int32_t)oopnd.size();
  v.n_axes = (int32_t)axis_names.size();
  v.axis_sz32[0] = 1;  // "no axis": divide by 1
  v.axis_magic[0] = 1u << 31;
  v.axis_mshift[0] = 31;
  for (int a = 0; a < v.n_axes; ++a) {
    v.axis_size[a] = axis_sizes[a];
    {
      uint64_t d = (uint64_t)axis_sizes[a];
      int l = 0;
      while ((uint64_t(1) << l) < d) ++l;  // ceil(log2 d)
      int s = 31 + l;
      v.axis_sz32[a + 1] = (uint32_t)d;
      v.axis_mshift[a + 1] = s;
      v.axis_magic[a + 1] = (uint32_t)(((uint64_t(1) << s) + d - 1) / d);
    }
    int rank = 0;
    for (int b = 0; b < v.n_axes; ++b)
      if (axis_names[b] < axis_names[a]) ++rank;
    v.axis_name_rank[a] = rank;
  }
  for (int pm = 0; pm < 16; ++pm) {
    int best = -1;
    for (int ax = 0; ax < v.n_axes; ++ax)
      if ((pm >> ax) & 1)
        if (best < 0 || v.axis_name_rank[ax] < v.axis_name_rank[best]) best = ax;
    v.pend_front[pm] = (int8_t)best;
  }
  v.result = result;
  v.vshape = vshape.data();
  v.vrank = vrank.data();
  v.okind = okind.data();
  v.omask = omask.data();
  v.oopnd_off = oopnd_off.data();
  v.oopnd = oopnd.data();
  v.slot_op = slot_op.data();
  v.orule_err = orule_err.data();
  v.ocls_off = ocls_off.data();
  v.cls_role = cls_role.data();
  v.cls_rdim = cls_rdim.data();
  v.cls_moff = cls_moff.data();
  v.mem = mem.data();
  v.slot_cls = slot_cls.data();
  v.op_rcls = op_rcls.data();
  v.user_off = user_off.data();
  v.users = users.data();
  v.init_uses = init_uses.data();
  return v;
}

std::vector<char> worklist_filter(const HostGraph& g, const pe_search_config& cfg) {
  std::vector<char> keep;
  if (!cfg.worklist_args) return keep;
  keep.assign(g.args.size(), 0);
  for (uint32_t i = 0; i < cfg.n_worklist_args; ++i)
    if (cfg.worklist_args[i] < g.args.size()) keep[cfg.worklist_args[i]] = 1;
  return keep;
}

Worklist build_worklist(const HostGraph& g, uint32_t auto_axes_mask, bool group_scopes,
                        bool scoped_only, bool resurface, const std::vector<char>& keep) {
  auto kept = [&](int32_t a) { return keep.empty() || keep[a]; };
  Worklist w;
  w.groups = group_scopes;
  w.resurface = resurface;
  w.n_ops = (int32_t)g.ops.size();
  for (int32_t a = 0; a < (int32_t)g.axis_names.size(); ++a)
    if (auto_axes_mask & (1u << a)) w.auto_axes.push_back(a);
  w.grp_off.push_back(0);
  for (const auto& grp : g.groups) {
    for (int32_t m : grp) w.grp_mem.push_back(m);
    w.grp_off.push_back((int32_t)w.grp_mem.size());
  }
  w.ent_off.push_back(0);
  if (group_scopes) {
    for (int32_t gi = 0; gi < (int32_t)g.groups.size(); ++gi) {
      const auto& grp = g.groups[gi];
      if (scoped_only && g.args[grp[0]].scope.empty()) continue;
      bool any = false;
      for (int32_t m : grp) any = any || kept(m);
      if (!any) continue;
      for (int32_t m : grp) w.ent_mem.push_back(m);
      w.ent_off.push_back((int32_t)w.ent_mem.size());
      w.ent_val.push_back(gi);
    }
  } else {
    for (int32_t a = 0; a < (int32_t)g.args.size(); ++a) {
      if (scoped_only && g.args[a].scope.empty()) continue;
      if (!kept(a)) continue;
      w.ent_mem.push_back(a);
      w.ent_off.push_back((int32_t)w.ent_mem.size());
      w.ent_val.push_back(a);
    }
  }
  w.ord_off.push_back(0);
  for (int32_t e = 0; e < w.n_entries(); ++e)
    for (int32_t d = 0; d < kMaxRank; ++d)
      for (int32_t ax : w.auto_axes) {
        for (int32_t i = w.ent_off[e]; i < w.ent_off[e + 1]; ++i) {
          int32_t m = w.ent_mem[i];
          const auto& s = g.args[m].shape;
          if (d < (int32_t)s.size() && s[d] % g.axis_sizes[ax] == 0) w.ord_mem.push_back(m);
        }
        w.ord_off.push_back((int32_t)w.ord_mem.size());
      }
  return w;
}

void attach_worklist(GraphView& v, const Worklist& w) {
  v.n_entries = w.n_entries();
  v.n_auto = (int32_t)w.auto_axes.size();
  for (int i = 0; i < kMaxAxes; ++i) v.auto_axes[i] = i < v.n_auto ? w.auto_axes[i] : 0;
  v.entries_are_groups = w.groups ? 1 : 0;
  v.ent_off = w.ent_off.data();
  v.ent_mem = w.ent_mem.data();
  v.ent_val = w.ent_val.data();
  v.n_groups = (int32_t)w.grp_off.size() - 1;
  v.grp_off = w.grp_off.data();
  v.grp_mem = w.grp_mem.data();
  v.n_ord = w.n_static_ordinals();
  v.resurface = w.resurface ? 1 : 0;
  v.ir_ord = w.infer_rest ? w.n_ordinals() : -1;
  v.ir_pause = 0;
  v.ord_off = w.ord_off.data();
  v.ord_mem = w.ord_mem.data();
}

bool finish_graph(HostGraph& g, LoadError& err) {
  try {
    check_graph(g);
    compile(g);
  } catch (const Bad& b) {
    err = b.e;
    return false;
  }
  return true;
}

bool load_graph(const char* text, size_t len, HostGraph& g, LoadError& err) {
  return read_pir(text, len, g, err) && finish_graph(g, err);
}

}  // namespace pe
