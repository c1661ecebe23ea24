// pe_graph.cc — `.pir` loader and graph compiler (host C++).
//
// Replaces REF parse_program (parser.cc:461-467) + validate
// (validate.cc:371-389) for the untiled programs the search starts from, and
// precompiles the per-op propagation rules of REF registry.cc:123-206 into
// flat tables.  The grammar follows SPEC tensor_ir "External Interfaces".
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

// ---------------------------------------------------------------- lexer
enum class Tok { kIdent, kValue, kAt, kString, kNumber, kLParen, kRParen, kLBrace,
                 kRBrace, kLBracket, kRBracket, kComma, kColon, kEquals, kArrow, kEnd };

struct Token {
  Tok tok = Tok::kEnd;
  std::string text;
  int line = 1, column = 1;
};

struct Fail {
  LoadError e;
};

[[noreturn]] void parse_fail(const Token& t, const std::string& msg) {
  Fail f;
  f.e.code = PE_ERR_PARSE;
  f.e.line = t.line;
  f.e.column = t.column;
  f.e.message = "parse error at " + std::to_string(t.line) + ":" + std::to_string(t.column) +
                ": " + msg;
  throw f;
}

[[noreturn]] void invalid(const std::string& msg, int code = PE_ERR_VALIDATION) {
  Fail f;
  f.e.code = code;
  f.e.message = msg;
  throw f;
}

class Lexer {
 public:
  Lexer(const char* s, size_t n) : s_(s), n_(n) {}
  Token next() {
    skip();
    Token t;
    t.line = line_;
    t.column = col_;
    if (p_ >= n_) return t;
    char c = s_[p_];
    auto single = [&](Tok k) {
      t.tok = k;
      adv();
      return t;
    };
    switch (c) {
      case '(': return single(Tok::kLParen);
      case ')': return single(Tok::kRParen);
      case '{': return single(Tok::kLBrace);
      case '}': return single(Tok::kRBrace);
      case '[': return single(Tok::kLBracket);
      case ']': return single(Tok::kRBracket);
      case ',': return single(Tok::kComma);
      case ':': return single(Tok::kColon);
      case '=': return single(Tok::kEquals);
      case '@': return single(Tok::kAt);
      default: break;
    }
    if (c == '%') {
      adv();
      t.tok = Tok::kValue;
      t.text = ident();
      if (t.text.empty()) parse_fail(t, "expected value name after '%'");
      return t;
    }
    if (c == '"') {
      adv();
      t.tok = Tok::kString;
      while (p_ < n_ && s_[p_] != '"') {
        t.text += s_[p_];
        adv();
      }
      if (p_ >= n_) parse_fail(t, "unterminated string");
      adv();
      return t;
    }
    if (c == '-' && p_ + 1 < n_ && s_[p_ + 1] == '>') {
      adv();
      adv();
      t.tok = Tok::kArrow;
      return t;
    }
    if (std::isdigit((unsigned char)c) || c == '-' || c == '+') {
      t.tok = Tok::kNumber;
      size_t b = p_;
      adv();
      while (p_ < n_ && (std::isdigit((unsigned char)s_[p_]) || s_[p_] == '.' || s_[p_] == 'e' ||
                         s_[p_] == 'E' ||
                         ((s_[p_] == '-' || s_[p_] == '+') && (s_[p_ - 1] == 'e' || s_[p_ - 1] == 'E'))))
        adv();
      t.text.assign(s_ + b, p_ - b);
      return t;
    }
    if (std::isalpha((unsigned char)c) || c == '_') {
      t.tok = Tok::kIdent;
      t.text = ident();
      return t;
    }
    parse_fail(t, std::string("unexpected character '") + c + "'");
  }

 private:
  void skip() {
    while (p_ < n_) {
      char c = s_[p_];
      if (c == '/' && p_ + 1 < n_ && s_[p_ + 1] == '/') {
        while (p_ < n_ && s_[p_] != '\n') adv();
      } else if (std::isspace((unsigned char)c)) {
        adv();
      } else {
        break;
      }
    }
  }
  std::string ident() {
    std::string o;
    while (p_ < n_ && (std::isalnum((unsigned char)s_[p_]) || s_[p_] == '_' || s_[p_] == '.' ||
                       s_[p_] == '/')) {
      o += s_[p_];
      adv();
    }
    return o;
  }
  void adv() {
    if (s_[p_] == '\n') {
      ++line_;
      col_ = 1;
    } else {
      ++col_;
    }
    ++p_;
  }
  const char* s_;
  size_t n_, p_ = 0;
  int line_ = 1, col_ = 1;
};

const std::map<std::string, Kind>& kind_names() {
  static const std::map<std::string, Kind> m = {
      {"constant", kConstant}, {"add", kAdd}, {"sub", kSub}, {"mul", kMul},
      {"div", kDiv}, {"neg", kNeg}, {"exp", kExp}, {"tanh", kTanh},
      {"rsqrt", kRsqrt}, {"maximum", kMaximum}, {"dot", kDot},
      {"reduce_sum", kReduceSum}, {"reduce_max", kReduceMax},
      {"transpose", kTranspose}, {"reshape", kReshape},
      {"broadcast_in_dim", kBroadcastInDim}, {"slice", kSlice},
      {"concatenate", kConcatenate}};
  return m;
}

// ---------------------------------------------------------------- parser
class Parser {
 public:
  Parser(const char* s, size_t n, HostGraph& g) : lx_(s, n), g_(g) { adv(); }

  void parse() {
    if (cur_.tok == Tok::kIdent && cur_.text == "mesh") {
      adv();
      expect(Tok::kLBrace, "'{'");
      while (cur_.tok != Tok::kRBrace) {
        g_.axis_names.push_back(expect(Tok::kString, "axis name string").text);
        expect(Tok::kEquals, "'='");
        g_.axis_sizes.push_back(expect_int("axis size"));
        if (cur_.tok == Tok::kComma) adv();
        else break;
      }
      expect(Tok::kRBrace, "'}'");
    }
    expect_ident("func");
    expect(Tok::kAt, "'@'");
    g_.name = expect(Tok::kIdent, "function name").text;
    expect(Tok::kLParen, "'('");
    while (cur_.tok != Tok::kRParen) {
      HostArg a;
      a.id = expect(Tok::kValue, "argument name").text;
      expect(Tok::kColon, "':'");
      a.shape = parse_type();
      if (cur_.tok == Tok::kLBrace) {
        adv();
        expect_ident("scope");
        expect(Tok::kEquals, "'='");
        a.scope = expect(Tok::kString, "scope string").text;
        expect(Tok::kRBrace, "'}'");
      }
      define(a.id);
      g_.args.push_back(std::move(a));
      if (cur_.tok == Tok::kComma) adv();
      else break;
    }
    expect(Tok::kRParen, "')'");
    expect(Tok::kArrow, "'->'");
    parse_type();
    expect(Tok::kLBrace, "'{'");
    for (;;) {
      if (cur_.tok == Tok::kIdent && cur_.text == "return") {
        adv();
        Token r = expect(Tok::kValue, "terminator value");
        auto it = ids_.find(r.text);
        if (it == ids_.end())
          invalid("returned value %" + r.text + " is not defined at top level");
        g_.result = it->second;
        expect(Tok::kRBrace, "'}'");
        break;
      }
      if (cur_.tok != Tok::kValue) parse_fail(cur_, "expected op definition or 'return'");
      HostOp op;
      op.id = cur_.text;
      adv();
      expect(Tok::kEquals, "'='");
      parse_op(op);
      define(op.id);
      g_.ops.push_back(std::move(op));
    }
    if (cur_.tok != Tok::kEnd) parse_fail(cur_, "trailing input after function body");
  }

 private:
  void define(const std::string& id) {
    int32_t idx = (int32_t)(g_.args.size() + g_.ops.size());
    if (id.empty() || !ids_.emplace(id, idx).second) invalid("redefinition of %" + id);
  }

  void parse_op(HostOp& op) {
    Token kt = expect(Tok::kIdent, "op kind");
    if (kt.text == "tile" || kt.text == "sum" || kt.text == "atomic" || kt.text == "slice_axis")
      invalid("op %" + op.id + ": tiled-dialect programs are not accepted as search roots; "
              "the engine starts from the untiled graph",
              PE_ERR_INVALID_ARGUMENT);
    if (kt.text == "all_reduce" || kt.text == "all_gather" || kt.text == "slice_by_coord")
      parse_fail(kt, "SPMD ops cannot appear in the textual input form");
    auto it = kind_names().find(kt.text);
    if (it == kind_names().end()) parse_fail(kt, "unknown op '" + kt.text + "'");
    op.kind = it->second;
    expect(Tok::kLParen, "'('");
    while (cur_.tok != Tok::kRParen) {
      Token v = expect(Tok::kValue, "operand");
      auto f = ids_.find(v.text);
      if (f == ids_.end())
        invalid("op %" + op.id + ": unknown or not-yet-defined value %" + v.text);
      op.operands.push_back(f->second);
      if (cur_.tok == Tok::kComma) adv();
      else break;
    }
    expect(Tok::kRParen, "')'");
    if (cur_.tok == Tok::kLBrace) parse_attrs(op);
    expect(Tok::kColon, "':'");
    op.shape = parse_type();
  }

  void parse_attrs(HostOp& op) {
    expect(Tok::kLBrace, "'{'");
    while (cur_.tok != Tok::kRBrace) {
      Token key = expect(Tok::kIdent, "attribute name");
      expect(Tok::kEquals, "'='");
      if (key.text == "contract") {
        int_pair(op.lhs_contract, op.rhs_contract);
      } else if (key.text == "batch") {
        int_pair(op.lhs_batch, op.rhs_batch);
      } else if (key.text == "dims" || key.text == "perm" || key.text == "map") {
        int_list(op.dims);
      } else if (key.text == "start") {
        i64_list(op.start);
      } else if (key.text == "limit") {
        i64_list(op.limit);
      } else if (key.text == "dim") {
        op.dim = (int)expect_int("dim");
      } else if (key.text == "value") {
        Token v = expect(Tok::kNumber, "number");
        char* end = nullptr;
        op.value = std::strtod(v.text.c_str(), &end);
        if (end != v.text.c_str() + v.text.size()) parse_fail(v, "malformed number");
      } else if (key.text == "scope") {
        op.scope = expect(Tok::kString, "scope string").text;
      } else {
        parse_fail(key, "unknown attribute '" + key.text + "'");
      }
      if (cur_.tok == Tok::kComma) adv();
      else break;
    }
    expect(Tok::kRBrace, "'}'");
  }

  std::vector<int64_t> parse_type() {
    Token t = expect(Tok::kIdent, "type");
    if (t.text != "f32") parse_fail(t, "unknown element type '" + t.text + "'");
    expect(Tok::kLBracket, "'['");
    std::vector<int64_t> s;
    while (cur_.tok != Tok::kRBracket) {
      s.push_back(expect_int("dimension"));
      if (cur_.tok == Tok::kComma) adv();
      else break;
    }
    expect(Tok::kRBracket, "']'");
    return s;
  }
  void int_list(std::vector<int>& o) {
    std::vector<int64_t> t;
    i64_list(t);
    for (int64_t v : t) o.push_back((int)v);
  }
  void i64_list(std::vector<int64_t>& o) {
    expect(Tok::kLBracket, "'['");
    while (cur_.tok != Tok::kRBracket) {
      o.push_back(expect_int("integer"));
      if (cur_.tok == Tok::kComma) adv();
      else break;
    }
    expect(Tok::kRBracket, "']'");
  }
  void int_pair(std::vector<int>& a, std::vector<int>& b) {
    expect(Tok::kLBracket, "'['");
    int_list(a);
    expect(Tok::kComma, "','");
    int_list(b);
    expect(Tok::kRBracket, "']'");
  }
  int64_t expect_int(const char* what) {
    Token t = expect(Tok::kNumber, what);
    const char* s = t.text.c_str();
    char* end = nullptr;
    long long v = std::strtoll(s, &end, 10);
    if (end != s + t.text.size() || t.text.empty() || t.text[0] == '+')
      parse_fail(t, std::string("expected integer ") + what);
    return v;
  }
  Token expect(Tok k, const char* what) {
    if (cur_.tok != k) parse_fail(cur_, std::string("expected ") + what);
    Token t = cur_;
    adv();
    return t;
  }
  void expect_ident(const char* name) {
    if (cur_.tok != Tok::kIdent || cur_.text != name)
      parse_fail(cur_, std::string("expected '") + name + "'");
    adv();
  }
  void adv() { cur_ = lx_.next(); }

  Lexer lx_;
  HostGraph& g_;
  Token cur_;
  std::map<std::string, int32_t> ids_;
};

// ---------------------------------------------------------------- validate
// Shape inference of the base dialect (REF validate.cc:161-225).
std::string shape_str(const std::vector<int64_t>& s) {
  std::string o = "f32[";
  for (size_t i = 0; i < s.size(); ++i) o += (i ? "," : "") + std::to_string(s[i]);
  return o + "]";
}

void validate(const HostGraph& g) {
  std::set<std::string> names;
  for (size_t a = 0; a < g.axis_names.size(); ++a) {
    if (g.axis_names[a].empty()) invalid("mesh axis with empty name");
    if (g.axis_sizes[a] < 1) invalid("mesh axis \"" + g.axis_names[a] + "\" has size < 1");
    if (g.axis_sizes[a] > kMaxDim)
      invalid("mesh axis \"" + g.axis_names[a] + "\" size exceeds 2^31-1",
              PE_ERR_INVALID_ARGUMENT);
    if (!names.insert(g.axis_names[a]).second)
      invalid("duplicate mesh axis \"" + g.axis_names[a] + "\"");
  }
  if ((int)g.axis_names.size() > kMaxAxes)
    invalid("more than 4 mesh axes", PE_ERR_INVALID_ARGUMENT);
  if (g.name.empty()) invalid("program without a name");
  for (const HostArg& a : g.args) {
    if ((int)a.shape.size() > kMaxRank) invalid("argument %" + a.id + " rank exceeds 4");
    for (int64_t d : a.shape) {
      if (d < 1) invalid("argument %" + a.id + " dimension < 1");
      if (d > kMaxDim)
        invalid("argument %" + a.id + " dimension exceeds 2^31-1", PE_ERR_INVALID_ARGUMENT);
    }
  }
  auto fail = [](const HostOp& op, const std::string& m, int code = PE_ERR_VALIDATION) {
    invalid("op %" + op.id + ": " + m, code);
  };
  auto in_rank = [&](const HostOp& op, int d, int r, const char* what) {
    if (d < 0 || d >= r) fail(op, std::string(what) + " " + std::to_string(d) + " out of range");
  };
  for (const HostOp& op : g.ops) {
    if ((int)op.shape.size() > kMaxRank) fail(op, "rank exceeds 4");
    for (int64_t d : op.shape) {
      if (d < 1) fail(op, "result dimension < 1");
      if (d > kMaxDim) fail(op, "result dimension exceeds 2^31-1", PE_ERR_INVALID_ARGUMENT);
    }
    std::vector<std::vector<int64_t>> in;
    for (int32_t v : op.operands) in.push_back(g.value_shape(v));
    auto arity = [&](size_t n) {
      if (in.size() != n)
        fail(op, "expects " + std::to_string(n) + " operand(s), got " + std::to_string(in.size()));
    };
    std::vector<int64_t> want;
    switch (op.kind) {
      case kConstant:
        arity(0);
        want = op.shape;
        break;
      case kAdd: case kSub: case kMul: case kDiv: case kMaximum:
        arity(2);
        if (in[0] != in[1]) fail(op, "operand shapes differ: " + shape_str(in[0]) + " vs " + shape_str(in[1]));
        want = in[0];
        break;
      case kNeg: case kExp: case kTanh: case kRsqrt:
        arity(1);
        want = in[0];
        break;
      case kDot: {
        arity(2);
        const auto& l = in[0];
        const auto& r = in[1];
        if (op.lhs_batch.size() != op.rhs_batch.size()) fail(op, "batch dimension lists differ in length");
        if (op.lhs_contract.size() != op.rhs_contract.size())
          fail(op, "contracting dimension lists differ in length");
        std::set<int> lu, ru;
        for (size_t i = 0; i < op.lhs_batch.size(); ++i) {
          in_rank(op, op.lhs_batch[i], (int)l.size(), "lhs batch dim");
          in_rank(op, op.rhs_batch[i], (int)r.size(), "rhs batch dim");
          if (l[op.lhs_batch[i]] != r[op.rhs_batch[i]]) fail(op, "batch dimension size mismatch");
          if (!lu.insert(op.lhs_batch[i]).second || !ru.insert(op.rhs_batch[i]).second)
            fail(op, "repeated batch dimension");
        }
        for (size_t i = 0; i < op.lhs_contract.size(); ++i) {
          in_rank(op, op.lhs_contract[i], (int)l.size(), "lhs contracting dim");
          in_rank(op, op.rhs_contract[i], (int)r.size(), "rhs contracting dim");
          if (l[op.lhs_contract[i]] != r[op.rhs_contract[i]])
            fail(op, "contracting dimension size mismatch");
          if (!lu.insert(op.lhs_contract[i]).second || !ru.insert(op.rhs_contract[i]).second)
            fail(op, "dimension both batch and contracting");
        }
        for (int b : op.lhs_batch) want.push_back(l[b]);
        for (int i = 0; i < (int)l.size(); ++i)
          if (!lu.count(i)) want.push_back(l[i]);
        for (int i = 0; i < (int)r.size(); ++i)
          if (!ru.count(i)) want.push_back(r[i]);
        if ((int)want.size() > kMaxRank) fail(op, "dot result rank exceeds 4");
        break;
      }
      case kReduceSum: case kReduceMax: {
        arity(1);
        std::set<int> red(op.dims.begin(), op.dims.end());
        if (red.size() != op.dims.size()) fail(op, "repeated reduce dim");
        for (int d : op.dims) in_rank(op, d, (int)in[0].size(), "reduce dim");
        for (int i = 0; i < (int)in[0].size(); ++i)
          if (!red.count(i)) want.push_back(in[0][i]);
        break;
      }
      case kTranspose: {
        arity(1);
        int r = (int)in[0].size();
        if ((int)op.dims.size() != r) fail(op, "permutation length does not match rank");
        std::set<int> seen(op.dims.begin(), op.dims.end());
        if ((int)seen.size() != r || (!seen.empty() && (*seen.begin() < 0 || *seen.rbegin() >= r)))
          fail(op, "permutation is not a bijection on dims");
        for (int d : op.dims) want.push_back(in[0][d]);
        break;
      }
      case kReshape: {
        arity(1);
        int64_t a = 1, b = 1;
        for (int64_t d : in[0]) a *= d;
        for (int64_t d : op.shape) b *= d;
        if (a != b) fail(op, "reshape changes element count");
        want = op.shape;
        break;
      }
      case kBroadcastInDim: {
        arity(1);
        if ((int)op.dims.size() != (int)in[0].size())
          fail(op, "broadcast dim map length does not match operand rank");
        int prev = -1;
        for (size_t i = 0; i < op.dims.size(); ++i) {
          int m = op.dims[i];
          in_rank(op, m, (int)op.shape.size(), "broadcast map entry");
          if (m <= prev) fail(op, "broadcast dim map must be strictly increasing");
          prev = m;
          if (in[0][i] != op.shape[m]) fail(op, "broadcast operand dim size mismatch");
        }
        want = op.shape;
        break;
      }
      case kSlice: {
        arity(1);
        int r = (int)in[0].size();
        if ((int)op.start.size() != r || (int)op.limit.size() != r)
          fail(op, "slice start/limit length does not match rank");
        for (int i = 0; i < r; ++i) {
          if (op.start[i] < 0 || op.limit[i] > in[0][i] || op.start[i] >= op.limit[i])
            fail(op, "slice bounds invalid for dim " + std::to_string(i));
          want.push_back(op.limit[i] - op.start[i]);
        }
        break;
      }
      case kConcatenate: {
        if (in.size() < 2) fail(op, "concatenate expects at least 2 operands");
        in_rank(op, op.dim, (int)in[0].size(), "concatenate dim");
        want = in[0];
        for (size_t i = 1; i < in.size(); ++i) {
          if (in[i].size() != in[0].size()) fail(op, "operand rank mismatch");
          for (int d = 0; d < (int)in[0].size(); ++d)
            if (d != op.dim && in[i][d] != in[0][d])
              fail(op, "non-concat dimension " + std::to_string(d) + " mismatch");
          want[op.dim] += in[i][op.dim];
        }
        if (in.size() > 8191) fail(op, "too many operands", PE_ERR_INVALID_ARGUMENT);
        break;
      }
      default:
        fail(op, "not a base-dialect op");
    }
    if (want != op.shape)
      fail(op, "declared type " + shape_str(op.shape) + " does not match inferred " + shape_str(want));
    for (int64_t d : op.shape)
      if (d > 0x7fffffff) fail(op, "dimension exceeds int32", PE_ERR_INVALID_ARGUMENT);
  }
  for (const HostArg& a : g.args)
    for (int64_t d : a.shape)
      if (d > 0x7fffffff) invalid("argument dimension exceeds int32", PE_ERR_INVALID_ARGUMENT);
  if (g.result < 0) invalid("program has no return");
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
  v.ord_off = w.ord_off.data();
  v.ord_mem = w.ord_mem.data();
}

bool load_graph(const char* text, size_t len, HostGraph& g, LoadError& err) {
  try {
    Parser p(text, len, g);
    p.parse();
    validate(g);
    compile(g);
  } catch (const Fail& f) {
    err = f.e;
    return false;
  }
  return true;
}

}  // namespace pe
