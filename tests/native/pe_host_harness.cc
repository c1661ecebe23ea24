// pe_host_harness.cc — TEST HARNESS ONLY.
//
// Compiles the engine's per-candidate core (paper_2112_02958_b200/csrc/
// pe_core.cuh) with g++ so the CPU test suite can differential-fuzz the
// rewrite automaton against the oracle (the patched reference) on thousands
// of programs without a GPU.  The product library (libpe_b200.so) is built
// by nvcc only and contains no host copy of the core; this harness is never
// loaded by the product path.  GPU parity tests (tests/test_gpu_parity.py)
// check the device build against the same oracle.
#include <algorithm>
#include <cstring>
#include <vector>

#include "pe.h"
#include "pe_core.cuh"
#include "pe_graph.h"

namespace {

struct Harness {
  pe::HostGraph g;
  pe::GraphView v;
  pe::Layout L;
  pe::Worklist w;
  std::vector<uint8_t> arena;
  pe_search_config cfg;
  pe_cost_params cp;
  int64_t baseline = 1;
};

void defaults(pe_search_config* c, pe_cost_params* p) {
  std::memset(c, 0, sizeof(*c));
  c->auto_axes_mask = 0xffffffffu;
  c->max_decisions = 32;
  c->group_scopes = 1;
  c->uct_c = 1.414;
  p->memory_budget_bytes = 16ll << 30;
  p->flops_per_second = 1e14;
  p->bytes_per_second = 1e11;
  p->collective_latency_s = 1e-6;
  p->w_mem = 0.1;
  p->w_comm = 1.0;
  p->w_steps = 0.01;
}

int setup(Harness& h, const char* pir, size_t len, const pe_search_config* cfg,
          const pe_cost_params* cp, char* err, size_t errcap) {
  pe::LoadError le;
  if (!pe::load_graph(pir, len, h.g, le)) {
    if (err) std::snprintf(err, errcap, "%s", le.message.c_str());
    return le.code;
  }
  defaults(&h.cfg, &h.cp);
  if (cfg) h.cfg = *cfg;
  if (cp) h.cp = *cp;
  h.v = h.g.host_view();
  h.w = pe::build_worklist(h.g, h.cfg.auto_axes_mask, h.cfg.group_scopes != 0,
                           h.cfg.scoped_only != 0, h.cfg.resurface_stuck != 0,
                           pe::worklist_filter(h.g, h.cfg));
  h.cfg.worklist_args = nullptr;
  pe::attach_worklist(h.v, h.w);
  h.L = pe::make_layout(h.v);
  h.arena.assign(h.L.bytes, 0);
  pe::Cand c(h.v, h.L, h.arena.data());
  pe_result r;
  c.eval(nullptr, 0, h.cp, 1, r, nullptr, 0);
  h.baseline = std::max<int64_t>(1, r.peak_bytes);
  return 0;
}

}  // namespace

extern "C" {

int harness_eval_batch(const char* pir, size_t len, const pe_search_config* cfg,
                       const pe_cost_params* cp, const pe_action* acts, const uint32_t* off,
                       uint32_t n, pe_result* out, int32_t* trace, uint32_t trace_words,
                       char* err, size_t errcap) {
  Harness h;
  int rc = setup(h, pir, len, cfg, cp, err, errcap);
  if (rc) return rc;
  pe::Cand c(h.v, h.L, h.arena.data());
  for (uint32_t i = 0; i < n; ++i)
    c.eval(acts + off[i], (int32_t)(off[i + 1] - off[i]), h.cp, h.baseline, out[i],
           trace ? trace + (size_t)i * trace_words : nullptr, trace_words);
  return 0;
}

int harness_rollout_batch(const char* pir, size_t len, const pe_search_config* cfg,
                          const pe_cost_params* cp, const pe_action* prefix,
                          const uint32_t* poff, const uint64_t* seeds, uint32_t n,
                          pe_action* acts_out, uint32_t* n_out, pe_result* out,
                          uint64_t* legal_out, char* err, size_t errcap) {
  Harness h;
  int rc = setup(h, pir, len, cfg, cp, err, errcap);
  if (rc) return rc;
  pe::Cand c(h.v, h.L, h.arena.data());
  int32_t maxd = (int32_t)h.cfg.max_decisions;
  int32_t nord = h.w.n_ordinals();
  int32_t lw = (nord + 63) / 64;
  auto ro = h.v.resurface ? &pe::Cand::rollout<true> : &pe::Cand::rollout<false>;
  for (uint32_t i = 0; i < n; ++i)
    (c.*ro)(prefix + poff[i], (int32_t)(poff[i + 1] - poff[i]), seeds[i], maxd, h.cp,
            h.baseline, acts_out + (size_t)i * maxd, n_out + i, out[i],
            legal_out ? legal_out + (size_t)i * lw : nullptr, lw, pe::Resume());
  return 0;
}

// High-water marks of the arena counters over a batch of rollouts, relative
// to the graph size: {slots - (A+N), loops, front stack, spmd ops, operands}.
int harness_highwater(const char* pir, size_t len, const pe_search_config* cfg,
                      const uint64_t* seeds, uint32_t n, int64_t* out5) {
  Harness h;
  char err[256];
  if (setup(h, pir, len, cfg, nullptr, err, sizeof(err))) return 1;
  pe::Cand c(h.v, h.L, h.arena.data());
  int32_t maxd = (int32_t)h.cfg.max_decisions;
  std::vector<pe_action> acts(maxd);
  for (int k = 0; k < 5; ++k) out5[k] = 0;
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t na;
    pe_result r;
    c.rollout<false>(nullptr, 0, seeds[i], maxd, h.cp, h.baseline, acts.data(), &na, r, nullptr,
                     0);
    out5[0] = std::max<int64_t>(out5[0], c.nslots - (h.v.A + h.v.N));
    out5[1] = std::max<int64_t>(out5[1], c.nloops);
    out5[2] = std::max<int64_t>(out5[2], c.nfs);
    out5[3] = std::max<int64_t>(out5[3], c.nem);
    out5[4] = std::max<int64_t>(out5[4], c.neo);
  }
  return 0;
}

// Prefix-state reuse check: every seed's rollout is run,
// the state after its first min(d, decisions) decisions is saved from a
// second candidate, and the rollout is resumed from that snapshot; the
// resumed actions and results are returned (they must equal a rollout from
// the root).
int harness_resume_rollouts(const char* pir, size_t len, const pe_search_config* cfg,
                            const pe_cost_params* cp, const uint64_t* seeds, uint32_t n, int32_t d,
                            pe_action* acts_out, uint32_t* n_out, pe_result* out, char* err,
                            size_t errcap) {
  Harness h;
  int rc = setup(h, pir, len, cfg, cp, err, errcap);
  if (rc) return rc;
  std::vector<uint8_t> arena2(h.L.bytes, 0);
  pe::Cand c(h.v, h.L, h.arena.data()), c2(h.v, h.L, arena2.data());
  int32_t maxd = (int32_t)h.cfg.max_decisions;
  std::vector<pe_action> acts(maxd), tmp(maxd);
  std::vector<uint8_t> snap(pe::Cand::snap_bytes(h.v, h.L.caps));
  for (uint32_t i = 0; i < n; ++i) {
    uint32_t na = 0, nt = 0;
    pe_result r;
    c.rollout<false>(nullptr, 0, seeds[i], maxd, h.cp, h.baseline, acts.data(), &na, r, nullptr, 0);
    int32_t k = std::min<int32_t>(d, (int32_t)na);
    c2.rollout<false>(acts.data(), k, 0, k, h.cp, h.baseline, tmp.data(), &nt, r, nullptr, 0);
    c2.save(snap.data());
    pe::Resume rs;
    rs.snap = snap.data();
    rs.done = rs.draws = k;
    rs.path = acts.data();
    c.rollout<false>(nullptr, 0, seeds[i], maxd, h.cp, h.baseline, acts_out + (size_t)i * maxd,
                     n_out + i, out[i], nullptr, 0, rs);
  }
  return 0;
}

int64_t harness_arena_bytes(const char* pir, size_t len) {
  Harness h;
  char err[256];
  if (setup(h, pir, len, nullptr, nullptr, err, sizeof(err))) return -1;
  return (int64_t)h.L.bytes;
}

}  // extern "C"
