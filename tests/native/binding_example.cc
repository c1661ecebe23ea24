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
#include "partir/propagate.h"
#include "partir/rewrite.h"
#include "partir/spmd.h"
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

// ---- drop-in evaluation (needs a GPU): the reference's own apply_tile_action
// + propagate + lower_to_spmd + collective_stats next to pe_eval_batch on the
// same Program, in one process, through the C-ABI.  argv: file "eval" then
// action sequences "value:dim:axis[,value:dim:axis...]".
int eval_mode(const partir::Program& p, pe_graph* g, int n, char** seqs) {
  pe_engine* e = nullptr;
  pe_error err{};
  if (pe_engine_create(g, nullptr, nullptr, 0, &e, &err) != PE_OK) {
    std::fprintf(stderr, "pe_engine_create: %s\n", err.message);
    return 3;
  }
  std::vector<pe_action> acts;
  std::vector<uint32_t> off{0};
  std::vector<partir::CollectiveStats> ref;
  for (int c = 0; c < n; ++c) {
    partir::Program q = p;
    std::stringstream in(seqs[c]);
    std::string item;
    while (std::getline(in, item, ',')) {
      std::string v = item.substr(0, item.find(':'));
      std::string rest = item.substr(item.find(':') + 1);
      int dim = std::stoi(rest.substr(0, rest.find(':')));
      std::string axis = rest.substr(rest.find(':') + 1);
      q = partir::propagate(partir::apply_tile_action(q, v, dim, axis)).program;
      acts.push_back(pe_action{(uint32_t)pe_graph_value_index(g, v.c_str()), (uint8_t)dim,
                               (uint8_t)pe_graph_axis_index(g, axis.c_str()), PE_ACT_TILE, 0});
    }
    off.push_back((uint32_t)acts.size());
    ref.push_back(partir::collective_stats(partir::lower_to_spmd(q)));
  }
  std::vector<pe_result> out(n);
  if (pe_eval_batch(e, acts.data(), off.data(), (uint32_t)n, out.data(), nullptr, 0, 0, nullptr,
                    &err) != PE_OK) {
    std::fprintf(stderr, "pe_eval_batch: %s\n", err.message);
    return 3;
  }
  int bad = 0;
  for (int c = 0; c < n; ++c) {
    for (int a = 0; a < (int)p.mesh.axes.size(); ++a) {
      const std::string& ax = p.mesh.axes[a].name;
      auto get = [&](const std::map<std::string, partir::CollectiveStats::PerAxis>& m, bool bytes) {
        auto it = m.find(ax);
        return it == m.end() ? (int64_t)0 : (bytes ? it->second.bytes : it->second.count);
      };
      bad |= get(ref[c].all_reduce, false) != out[c].ar_cnt[a];
      bad |= get(ref[c].all_reduce, true) != out[c].ar_bytes[a];
      bad |= get(ref[c].all_gather, false) != out[c].ag_cnt[a];
      bad |= get(ref[c].all_gather, true) != out[c].ag_bytes[a];
      bad |= get(ref[c].slice_by_coord, false) != out[c].sbc_cnt[a];
    }
    std::printf("%s %s ar=%lld ag=%lld\n", seqs[c], out[c].status == 0 ? "ok" : "status!=0",
                (long long)ref[c].all_reduce_bytes(), (long long)ref[c].all_gather_bytes());
  }
  pe_engine_destroy(e);
  std::printf("%s\n", bad ? "MISMATCH" : "EVAL OK");
  return bad ? 1 : 0;
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
  if (!bad && argc > 3 && std::strcmp(argv[2], "eval") == 0) bad = eval_mode(p, a, argc - 3, argv + 3);
  pe_graph_destroy(a);
  pe_graph_destroy(b);
  return bad ? 1 : 0;
}
