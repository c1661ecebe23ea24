// binding_example.cc -- the reference-side binding INTEGRATION.md shows,
// compiled against the REFERENCE's own headers (partir::Program, REF
// ir.h:84-131) and linked with both the reference (oracle/_ref/liboracle.so,
// test infrastructure) and the engine library (libpe_b200.so).
//
// It builds the engine graph of a reference Program two ways -- by walking
// the Program into pe_graph_create_from_arrays, and by printing it with the
// reference's printer into pe_graph_create -- and checks they agree.  No GPU
// is needed (graph construction is host-side).  tests/test_binding.py
// builds and runs it.  TEST INFRASTRUCTURE.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "partir/error.h"
#include "partir/ir.h"
#include "partir/parser.h"
#include "partir/printer.h"
#include "pe.h"

// ---- the binding (INTEGRATION.md "Without the print / re-parse round trip")
pe_graph* graph_from_program(const partir::Program& p) {
  std::map<std::string, int32_t> idx;  // value id -> index
  std::vector<const char*> axn;
  std::vector<int64_t> axs;
  for (const auto& a : p.mesh.axes) {
    axn.push_back(a.name.c_str());
    axs.push_back(a.size);
  }
  std::vector<pe_arg_desc> args(p.args.size());
  for (size_t i = 0; i < p.args.size(); ++i) {
    const auto& a = p.args[i];
    args[i] = pe_arg_desc{a.id.c_str(), a.scope.c_str(), (int32_t)a.type.rank(), {}};
    for (int d = 0; d < a.type.rank(); ++d) args[i].shape[d] = a.type.shape[d];
    idx[a.id] = (int32_t)i;
  }
  std::vector<pe_op_desc> ops(p.ops.size());
  std::vector<std::vector<int32_t>> opnds(p.ops.size());
  for (size_t i = 0; i < p.ops.size(); ++i) {
    const partir::Operation& op = p.ops[i];  // base dialect only
    pe_op_desc& d = ops[i];
    d = pe_op_desc{};
    d.id = op.id.c_str();
    d.kind = (int32_t)op.kind;
    d.scope = op.scope.c_str();
    d.rank = (int32_t)op.result_type.rank();
    for (int k = 0; k < d.rank; ++k) d.shape[k] = op.result_type.shape[k];
    for (const auto& o : op.operands) opnds[i].push_back(idx.at(o));
    d.n_operands = (int32_t)opnds[i].size();
    d.operands = opnds[i].data();
    d.n_batch = (int32_t)op.dot.lhs_batch.size();
    d.n_contract = (int32_t)op.dot.lhs_contract.size();
    for (int k = 0; k < d.n_batch; ++k) {
      d.lhs_batch[k] = op.dot.lhs_batch[k];
      d.rhs_batch[k] = op.dot.rhs_batch[k];
    }
    for (int k = 0; k < d.n_contract; ++k) {
      d.lhs_contract[k] = op.dot.lhs_contract[k];
      d.rhs_contract[k] = op.dot.rhs_contract[k];
    }
    d.n_dims = (int32_t)op.dims.size();
    for (int k = 0; k < d.n_dims; ++k) d.dims[k] = op.dims[k];
    for (size_t k = 0; k < op.start.size(); ++k) {
      d.start[k] = op.start[k];
      d.limit[k] = op.limit[k];
    }
    d.dim = op.dim;
    d.value = op.value;
    idx[op.id] = (int32_t)(p.args.size() + i);
  }
  pe_graph* g = nullptr;
  pe_error err{};
  if (pe_graph_create_from_arrays(p.name.c_str(), (int32_t)axn.size(), axn.data(), axs.data(),
                                  (int32_t)args.size(), args.data(), (int32_t)ops.size(),
                                  ops.data(), idx.at(p.result_id), &g, &err) != PE_OK)
    throw partir::ValidationError(err.message);
  return g;
}

// ---- the check
int main(int argc, char** argv) {
  if (argc < 2) return 2;
  std::ifstream in(argv[1]);
  std::stringstream ss;
  ss << in.rdbuf();
  partir::Program p = partir::parse_program(ss.str());  // the reference's parser
  pe_graph* a = graph_from_program(p);
  std::string text = partir::print_program(p);          // the reference's printer
  pe_graph* b = nullptr;
  pe_error err{};
  if (pe_graph_create(text.data(), text.size(), &b, &err) != PE_OK) {
    std::fprintf(stderr, "pe_graph_create: %s\n", err.message);
    return 1;
  }
  int bad = 0;
  bad |= pe_graph_num_args(a) != pe_graph_num_args(b) || pe_graph_num_args(a) != (int)p.args.size();
  bad |= pe_graph_num_ops(a) != pe_graph_num_ops(b) || pe_graph_num_ops(a) != (int)p.ops.size();
  bad |= pe_graph_num_operands(a) != pe_graph_num_operands(b);
  bad |= pe_graph_num_groups(a) != pe_graph_num_groups(b);
  char n1[256], n2[256];
  int64_t s1[4], s2[4];
  for (int v = 0; v < pe_graph_num_args(a) + pe_graph_num_ops(a) && !bad; ++v) {
    pe_graph_value_name(a, v, n1, sizeof(n1));
    pe_graph_value_name(b, v, n2, sizeof(n2));
    int r1 = pe_graph_value_shape(a, v, s1), r2 = pe_graph_value_shape(b, v, s2);
    bad |= std::strcmp(n1, n2) != 0 || r1 != r2 || std::memcmp(s1, s2, 8 * r1) != 0;
  }
  std::printf("%s args=%d ops=%d operands=%d groups=%d\n", bad ? "MISMATCH" : "OK",
              pe_graph_num_args(a), pe_graph_num_ops(a), pe_graph_num_operands(a),
              pe_graph_num_groups(a));
  pe_graph_destroy(a);
  pe_graph_destroy(b);
  return bad ? 1 : 0;
}
