// pe_pir.cc — reader for the `.pir` text form of an untiled program.
//
// The text form is fixed by SPEC tensor_ir "External Interfaces"
// (SPEC.md:87-96):
//
//   program   := [mesh] func
//   mesh      := 'mesh' '{' [ STRING '=' INT { ',' STRING '=' INT } ] '}'
//   func      := 'func' '@' NAME '(' [ param { ',' param } ] ')' '->' type
//                '{' { stmt } 'return' VALUE '}'
//   param     := VALUE ':' type [ '{' 'scope' '=' STRING '}' ]
//   stmt      := VALUE '=' KIND '(' [ VALUE { ',' VALUE } ] ')' [ attrs ] ':' type
//   attrs     := '{' [ attr { ',' attr } ] '}'
//   type      := 'f32' '[' [ INT { ',' INT } ] ']'
//   VALUE     := '%' NAME      NAME := [A-Za-z0-9_./]+      // comments to EOL
//
// It fills a HostGraph (pe_graph.h); shape checking and rule compilation
// happen afterwards in pe_graph.cc, so every syntax error is reported before
// any semantic one (the reference's parse_program also parses the whole
// text before validate() runs, REF parser.h:28, validate.h).
//
// This is the engine's own reader: a character cursor with one function per
// grammar rule and a table of attribute readers.  Tiled-dialect statements
// (tile / sum / atomic / slice_axis) are refused with INVALID_ARGUMENT: the
// engine starts every search from the untiled graph.  SPMD-dialect kinds are
// syntax errors in this form.
#include <cerrno>
#include <cstdlib>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "pe.h"
#include "pe_graph.h"

namespace pe {
namespace {

// Carried out of the reader by exception; converted to a LoadError at the
// boundary (no exception crosses the C-ABI).
struct PirFault {
  int code;
  int line, col;
  std::string text;
};

bool name_char(char c) {
  return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || (c >= '0' && c <= '9') || c == '_' ||
         c == '.' || c == '/';
}
bool word_start(char c) { return (c >= 'a' && c <= 'z') || (c >= 'A' && c <= 'Z') || c == '_'; }

class Cursor {
 public:
  explicit Cursor(const std::string& s) : s_(s), i_(0) {}

  [[noreturn]] void syntax(const std::string& what) const {
    throw PirFault{PE_ERR_PARSE, line(), col(),
                   "line " + std::to_string(line()) + ", column " + std::to_string(col()) + ": " +
                       what + " (found " + found() + ")"};
  }
  [[noreturn]] void refuse(int code, const std::string& what) const {
    throw PirFault{code, 0, 0, what};
  }

  // whitespace and line comments
  void blank() {
    for (;;) {
      while (i_ < s_.size() && (s_[i_] == ' ' || s_[i_] == '\t' || s_[i_] == '\n' ||
                                s_[i_] == '\r' || s_[i_] == '\f' || s_[i_] == '\v'))
        ++i_;
      if (i_ + 1 < s_.size() && s_[i_] == '/' && s_[i_ + 1] == '/') {
        while (i_ < s_.size() && s_[i_] != '\n') ++i_;
        continue;
      }
      return;
    }
  }
  bool eof() {
    blank();
    return i_ >= s_.size();
  }
  char peek() {
    blank();
    return i_ < s_.size() ? s_[i_] : '\0';
  }
  bool take(char c) {
    if (peek() != c) return false;
    ++i_;
    return true;
  }
  void need(char c, const char* role) {
    if (!take(c)) syntax(std::string("'") + c + "' " + role);
  }
  void need_arrow() {
    blank();
    if (s_.compare(i_, 2, "->") != 0) syntax("'->' before the result type");
    i_ += 2;
  }
  // the next bare word without consuming it ("" when none)
  std::string look_word() {
    blank();
    size_t j = i_;
    if (j >= s_.size() || !word_start(s_[j])) return "";
    while (j < s_.size() && name_char(s_[j])) ++j;
    return s_.substr(i_, j - i_);
  }
  std::string word(const char* role) {
    std::string w = look_word();
    if (w.empty()) syntax(std::string("a keyword or kind name ") + role);
    i_ += w.size();
    return w;
  }
  void keyword(const char* kw) {
    if (look_word() != kw) syntax(std::string("keyword '") + kw + "'");
    i_ += std::strlen(kw);
  }
  // '%' NAME or '@' NAME
  std::string sigil_name(char sigil, const char* role) {
    if (!take(sigil)) syntax(std::string("'") + sigil + "' introducing " + role);
    size_t j = i_;
    while (j < s_.size() && name_char(s_[j])) ++j;
    if (j == i_) syntax(std::string("a name for ") + role);
    std::string n = s_.substr(i_, j - i_);
    i_ = j;
    return n;
  }
  std::string quoted(const char* role) {
    if (!take('"')) syntax(std::string("a quoted string for ") + role);
    size_t j = s_.find('"', i_);
    if (j == std::string::npos) syntax("a closing '\"'");
    std::string q = s_.substr(i_, j - i_);
    i_ = j + 1;
    return q;
  }
  int64_t integer(const char* role) {
    blank();
    const char* b = s_.c_str() + i_;
    if (!(*b == '-' || (*b >= '0' && *b <= '9'))) syntax(std::string("an integer for ") + role);
    char* e = nullptr;
    errno = 0;
    long long v = std::strtoll(b, &e, 10);
    if (errno == ERANGE) syntax(std::string("an integer in range for ") + role);
    if (*e == '.' || *e == 'e' || *e == 'E') syntax(std::string("an integer (not a real) for ") + role);
    i_ += (size_t)(e - b);
    return v;
  }
  double real(const char* role) {
    blank();
    const char* b = s_.c_str() + i_;
    char* e = nullptr;
    double v = std::strtod(b, &e);
    if (e == b || !(*b == '-' || *b == '+' || *b == '.' || (*b >= '0' && *b <= '9')))
      syntax(std::string("a number for ") + role);
    i_ += (size_t)(e - b);
    return v;
  }

  int line() const {
    int l = 1;
    for (size_t k = 0; k < i_ && k < s_.size(); ++k) l += s_[k] == '\n';
    return l;
  }
  int col() const {
    size_t k = i_;
    while (k > 0 && s_[k - 1] != '\n') --k;
    return (int)(i_ - k) + 1;
  }

 private:
  std::string found() const {
    if (i_ >= s_.size()) return "end of input";
    size_t j = i_;
    while (j < s_.size() && j < i_ + 12 && s_[j] != '\n') ++j;
    return "\"" + s_.substr(i_, j - i_) + "\"";
  }
  const std::string& s_;
  size_t i_;
};

// '[' elem { ',' elem } ']' (possibly empty)
template <typename F>
void bracketed(Cursor& c, F&& elem) {
  c.need('[', "opening a list");
  if (c.take(']')) return;
  do elem(); while (c.take(','));
  c.need(']', "closing a list");
}

std::vector<int64_t> read_type(Cursor& c) {
  if (c.look_word() != "f32") c.syntax("element type f32");
  c.word("naming the element type");
  std::vector<int64_t> dims;
  bracketed(c, [&] { dims.push_back(c.integer("a dimension")); });
  return dims;
}

std::vector<int> read_ints(Cursor& c, const char* role) {
  std::vector<int> v;
  bracketed(c, [&] { v.push_back((int)c.integer(role)); });
  return v;
}

// [[lhs...],[rhs...]]
void read_int_pair(Cursor& c, std::vector<int>& lhs, std::vector<int>& rhs, const char* role) {
  c.need('[', "opening a dimension-list pair");
  lhs = read_ints(c, role);
  c.need(',', "between the lhs and rhs lists");
  rhs = read_ints(c, role);
  c.need(']', "closing a dimension-list pair");
}

using AttrReader = void (*)(Cursor&, HostOp&);
const std::unordered_map<std::string, AttrReader>& attr_readers() {
  static const std::unordered_map<std::string, AttrReader> t = {
      {"contract", [](Cursor& c, HostOp& op) {
         read_int_pair(c, op.lhs_contract, op.rhs_contract, "a contracting dim");
       }},
      {"batch", [](Cursor& c, HostOp& op) {
         read_int_pair(c, op.lhs_batch, op.rhs_batch, "a batch dim");
       }},
      // reduce dims / transpose permutation / broadcast dimension map share
      // one field (at most one of them applies to a kind)
      {"dims", [](Cursor& c, HostOp& op) { op.dims = read_ints(c, "a reduced dim"); }},
      {"perm", [](Cursor& c, HostOp& op) { op.dims = read_ints(c, "a permutation entry"); }},
      {"map", [](Cursor& c, HostOp& op) { op.dims = read_ints(c, "a broadcast map entry"); }},
      {"start", [](Cursor& c, HostOp& op) {
         bracketed(c, [&] { op.start.push_back(c.integer("a slice start")); });
       }},
      {"limit", [](Cursor& c, HostOp& op) {
         bracketed(c, [&] { op.limit.push_back(c.integer("a slice limit")); });
       }},
      {"dim", [](Cursor& c, HostOp& op) { op.dim = (int)c.integer("the concatenation dim"); }},
      {"value", [](Cursor& c, HostOp& op) { op.value = c.real("a constant value"); }},
      {"scope", [](Cursor& c, HostOp& op) { op.scope = c.quoted("a scope"); }},
  };
  return t;
}

const std::unordered_map<std::string, Kind>& base_kinds() {
  static const std::unordered_map<std::string, Kind> t = {
      {"constant", kConstant}, {"add", kAdd}, {"sub", kSub}, {"mul", kMul}, {"div", kDiv},
      {"neg", kNeg}, {"exp", kExp}, {"tanh", kTanh}, {"rsqrt", kRsqrt}, {"maximum", kMaximum},
      {"dot", kDot}, {"reduce_sum", kReduceSum}, {"reduce_max", kReduceMax},
      {"transpose", kTranspose}, {"reshape", kReshape}, {"broadcast_in_dim", kBroadcastInDim},
      {"slice", kSlice}, {"concatenate", kConcatenate}};
  return t;
}

struct Reader {
  Cursor c;
  HostGraph& g;
  std::unordered_map<std::string, int32_t> scope;  // value name -> index

  Reader(const std::string& text, HostGraph& out) : c(text), g(out) {}

  int32_t bind(const std::string& name) {
    int32_t idx = g.num_values();
    if (!scope.emplace(name, idx).second)
      c.refuse(PE_ERR_VALIDATION, "value %" + name + " is defined twice");
    return idx;
  }
  int32_t use(const std::string& name, const std::string& user) {
    auto it = scope.find(name);
    if (it == scope.end())
      c.refuse(PE_ERR_VALIDATION, "%" + user + " uses %" + name + ", which has no earlier definition");
    return it->second;
  }

  void mesh() {
    c.keyword("mesh");
    c.need('{', "opening the mesh");
    if (c.take('}')) return;
    do {
      g.axis_names.push_back(c.quoted("an axis name"));
      c.need('=', "between an axis name and its size");
      g.axis_sizes.push_back(c.integer("an axis size"));
    } while (c.take(','));
    c.need('}', "closing the mesh");
  }

  void param() {
    HostArg a;
    a.id = c.sigil_name('%', "a parameter");
    c.need(':', "before a parameter type");
    a.shape = read_type(c);
    if (c.take('{')) {
      c.keyword("scope");
      c.need('=', "after 'scope'");
      a.scope = c.quoted("a scope");
      c.need('}', "closing the parameter attributes");
    }
    bind(a.id);
    g.args.push_back(std::move(a));
  }

  void statement(const std::string& id) {
    HostOp op;
    op.id = id;
    c.need('=', "after the defined value");
    std::string kind = c.look_word();
    if (kind == "tile" || kind == "sum" || kind == "atomic" || kind == "slice_axis")
      c.refuse(PE_ERR_INVALID_ARGUMENT,
               "%" + id + " is a tiled-dialect '" + kind +
                   "': search roots must be untiled programs");
    auto k = base_kinds().find(kind);
    if (k == base_kinds().end()) {
      if (kind == "all_reduce" || kind == "all_gather" || kind == "slice_by_coord")
        c.syntax("a base-dialect kind (SPMD collectives have no text form)");
      c.syntax("a known op kind");
    }
    op.kind = k->second;
    c.word("naming the op kind");
    c.need('(', "opening the operand list");
    if (!c.take(')')) {
      do op.operands.push_back(use(c.sigil_name('%', "an operand"), id));
      while (c.take(','));
      c.need(')', "closing the operand list");
    }
    if (c.take('{') && !c.take('}')) {
      do {
        auto r = attr_readers().find(c.look_word());
        if (r == attr_readers().end()) c.syntax("a known attribute name");
        c.word("naming an attribute");
        c.need('=', "after an attribute name");
        r->second(c, op);
      } while (c.take(','));
      c.need('}', "closing the attributes");
    }
    c.need(':', "before the result type");
    op.shape = read_type(c);
    bind(op.id);
    g.ops.push_back(std::move(op));
  }

  void program() {
    if (c.look_word() == "mesh") mesh();
    c.keyword("func");
    g.name = c.sigil_name('@', "the function");
    c.need('(', "opening the parameter list");
    if (!c.take(')')) {
      do param(); while (c.take(','));
      c.need(')', "closing the parameter list");
    }
    c.need_arrow();
    read_type(c);  // the declared result type is the returned value's type
    c.need('{', "opening the function body");
    while (c.look_word() != "return") {
      if (c.peek() != '%') c.syntax("a statement or 'return'");
      statement(c.sigil_name('%', "a defined value"));
    }
    c.keyword("return");
    std::string r = c.sigil_name('%', "the returned value");
    auto it = scope.find(r);
    if (it == scope.end()) c.refuse(PE_ERR_VALIDATION, "the returned value %" + r + " is undefined");
    g.result = it->second;
    c.need('}', "closing the function body");
    if (!c.eof()) c.syntax("end of input after the function");
  }
};

}  // namespace

bool read_pir(const char* text, size_t len, HostGraph& g, LoadError& err) {
  std::string src(text, len);  // NUL-terminated copy for the number readers
  try {
    Reader r(src, g);
    r.program();
  } catch (const PirFault& f) {
    err.code = f.code;
    err.line = f.line;
    err.column = f.col;
    err.message = f.text;
    return false;
  }
  return true;
}

}  // namespace pe
