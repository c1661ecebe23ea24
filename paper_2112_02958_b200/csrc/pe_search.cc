// pe_search.cc — leaf-parallel, root-parallel MCTS over a batched evaluator.
//
// Restates SPEC search module (`mcts_search`, absent from the reference:
// REF CMakeLists.txt:26 lists src/search.cc, not shipped) with the choices
// declared in SURVEY.md Appendix B.5.6 / DESIGN.md §5:
//   * action ordinal = worklist entry x dim x auto axis, then Stop;
//   * selection: UCT  W/N + c*sqrt(ln N_parent / N), unvisited first,
//     ties -> lowest ordinal;
//   * expansion: lowest-ordinal untried action;
//   * rollout: uniform over legal TileValue actions, Stop weight 2 after the
//     first decision, <= max_decisions (done by the evaluator, on the GPU);
//   * backpropagation: N += 1, W += reward as 2^-32 fixed point (integer
//     sums keep the root-parallel merge bit-deterministic);
//   * leaf parallelism: `leaf_batch` leaves are selected with virtual loss
//     and evaluated in one batch (one GPU launch);
//   * root parallelism: every `merge_every` episodes the root children's
//     (N, W) deltas are all-reduced (SUM) through the merge hook, and the
//     other ranks' contributions shape this rank's root selection.
// Host C++; the evaluations it requests are the hot path.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "pe.h"

namespace {

constexpr double kFixed = 4294967296.0;  // 2^32

struct Node {
  int32_t parent = -1;
  uint32_t ord = 0;       // action ordinal that led here
  uint32_t depth = 0;     // decisions from the root
  bool terminal = false;  // Stop taken or decision cap reached
  bool known = false;     // legal actions known (node evaluated once)
  int64_t n = 0, w = 0;   // visits, fixed-point reward sum
  int64_t vn = 0;         // virtual visits of in-flight leaves
  std::vector<uint32_t> untried;  // legal ordinals + Stop, ascending
  uint32_t next_untried = 0;
  std::vector<std::pair<uint32_t, int32_t>> children;  // (ordinal, node), ascending
};

uint64_t splitmix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

void set_err(pe_error* err, int code, const std::string& m) {
  if (!err) return;
  err->code = code;
  err->line = err->column = 0;
  std::snprintf(err->message, sizeof(err->message), "%s", m.c_str());
}

struct Mcts {
  pe_mcts_params p;
  std::vector<Node> nodes;
  std::vector<int64_t> root_extra_n, root_extra_w;  // other ranks' root stats
  std::vector<int64_t> root_own_n, root_own_w;      // this rank, since last merge
  const pe_action* ord_actions;

  uint32_t stop() const { return p.n_ordinals; }

  int64_t child_n(const Node& parent, const Node& c) const {
    int64_t x = c.n + c.vn;
    if (parent.parent < 0) x += root_extra_n[c.ord];
    return x;
  }
  int64_t child_w(const Node& parent, const Node& c) const {
    int64_t x = c.w;
    if (parent.parent < 0) x += root_extra_w[c.ord];
    return x;
  }

  int32_t select_child(int32_t v) const {
    const Node& nd = nodes[v];
    int64_t pn = nd.n + nd.vn;
    if (nd.parent < 0)
      for (const auto& c : nd.children) pn += root_extra_n[nodes[c.second].ord];
    double lnp = std::log((double)std::max<int64_t>(pn, 1));
    int32_t best = -1;
    double best_v = 0;
    for (const auto& c : nd.children) {
      const Node& ch = nodes[c.second];
      int64_t cn = child_n(nd, ch);
      if (cn == 0) return c.second;  // unvisited first, lowest ordinal
      double q = ((double)child_w(nd, ch) / kFixed) / (double)cn;
      double u = q + p.uct_c * std::sqrt(lnp / (double)cn);
      if (best < 0 || u > best_v) {
        best = c.second;
        best_v = u;
      }
    }
    return best;
  }

  void prefix_of(int32_t v, std::vector<pe_action>& out) const {
    out.clear();
    for (int32_t x = v; nodes[x].parent >= 0; x = nodes[x].parent) {
      pe_action a = ord_actions[nodes[x].ord];
      out.push_back(a);
    }
    std::reverse(out.begin(), out.end());
  }
};

}  // namespace

extern "C" pe_status pe_mcts_run(const pe_mcts_params* prm, pe_rollout_fn eval, void* eval_user,
                                 pe_merge_fn merge, void* merge_user,
                                 const pe_action* ordinal_actions, pe_plan* out, pe_error* err) {
  if (!prm || !eval || !ordinal_actions || !out) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null argument");
    return PE_ERR_INVALID_ARGUMENT;
  }
  Mcts m;
  m.p = *prm;
  if (m.p.leaf_batch == 0) m.p.leaf_batch = 1;
  if (m.p.max_decisions == 0 || m.p.max_decisions > PE_PLAN_MAX_ACTIONS) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "max_decisions must be in [1, 64]");
    return PE_ERR_INVALID_ARGUMENT;
  }
  m.ord_actions = ordinal_actions;
  uint32_t n_ord1 = m.p.n_ordinals + 1;
  m.root_extra_n.assign(n_ord1, 0);
  m.root_extra_w.assign(n_ord1, 0);
  m.root_own_n.assign(n_ord1, 0);
  m.root_own_w.assign(n_ord1, 0);
  m.nodes.emplace_back();  // root
  uint32_t lw = (m.p.n_ordinals + 63) / 64;
  uint32_t maxd = m.p.max_decisions;
  uint64_t rank_seed = splitmix(m.p.seed ^ (0xD1B54A32D192ED03ull * (m.p.rank + 1)));

  std::memset(out, 0, sizeof(*out));
  out->seed = m.p.seed;
  double best_reward = -1.0;
  std::vector<pe_action> best_acts;
  pe_result best_res{};
  uint32_t best_ep = 0;

  std::vector<int32_t> leaves;
  std::vector<pe_action> pre, flat;
  std::vector<uint32_t> poff;
  std::vector<uint64_t> seeds;
  std::vector<pe_action> acts_out;
  std::vector<uint32_t> nacts;
  std::vector<pe_result> res;
  std::vector<uint64_t> legal;
  uint32_t done = 0;
  uint32_t merges_done = 0;
  while (done < m.p.episodes) {
    uint32_t B = std::min(m.p.leaf_batch, m.p.episodes - done);
    leaves.clear();
    for (uint32_t b = 0; b < B; ++b) {
      int32_t v = 0;
      for (;;) {
        Node& nd = m.nodes[v];
        if (nd.terminal || !nd.known) break;
        if (nd.next_untried < nd.untried.size()) {
          // expand the lowest-ordinal untried action
          uint32_t a = nd.untried[nd.next_untried++];
          Node c;
          c.parent = v;
          c.ord = a;
          c.depth = nd.depth + 1;
          c.terminal = a == m.stop() || c.depth >= maxd;
          int32_t ci = (int32_t)m.nodes.size();
          m.nodes[v].children.push_back({a, ci});
          m.nodes.push_back(std::move(c));
          v = ci;
          break;
        }
        if (nd.children.empty()) break;
        v = m.select_child(v);
      }
      for (int32_t x = v; x >= 0; x = m.nodes[x].parent) m.nodes[x].vn++;
      leaves.push_back(v);
    }
    // one batched evaluation (one launch on the GPU engine)
    flat.clear();
    poff.assign(1, 0);
    seeds.clear();
    for (uint32_t b = 0; b < B; ++b) {
      m.prefix_of(leaves[b], pre);
      flat.insert(flat.end(), pre.begin(), pre.end());
      poff.push_back((uint32_t)flat.size());
      seeds.push_back(splitmix(rank_seed + done + b));
    }
    if (flat.empty()) flat.push_back(pe_action{});
    acts_out.assign((size_t)B * maxd, pe_action{});
    nacts.assign(B, 0);
    res.assign(B, pe_result{});
    legal.assign((size_t)B * lw + 1, 0);
    int rc = eval(eval_user, flat.data(), poff.data(), seeds.data(), B, acts_out.data(),
                  nacts.data(), res.data(), legal.data());
    if (rc != 0) {
      set_err(err, PE_ERR_CUDA, "evaluator failed");
      return (pe_status)(rc > 0 ? rc : PE_ERR_INTERNAL);
    }
    for (uint32_t b = 0; b < B; ++b) {
      int32_t v = leaves[b];
      Node& nd = m.nodes[v];
      if (!nd.known) {
        nd.known = true;
        if (!nd.terminal && res[b].status == PE_CAND_OK) {
          for (uint32_t o = 0; o < m.p.n_ordinals; ++o)
            if ((legal[(size_t)b * lw + o / 64] >> (o % 64)) & 1ull) nd.untried.push_back(o);
          nd.untried.push_back(m.stop());
        } else {
          nd.terminal = true;
        }
      }
      double reward = res[b].status == PE_CAND_OK ? res[b].reward : 0.0;
      int64_t wf = (int64_t)std::llround(reward * kFixed);
      for (int32_t x = v; x >= 0; x = m.nodes[x].parent) {
        Node& y = m.nodes[x];
        y.vn--;
        y.n++;
        y.w += wf;
        if (y.parent == 0) {
          m.root_own_n[y.ord]++;
          m.root_own_w[y.ord] += wf;
        }
      }
      if (res[b].status == PE_CAND_OK && reward > best_reward) {
        best_reward = reward;
        best_acts.assign(acts_out.begin() + (size_t)b * maxd,
                         acts_out.begin() + (size_t)b * maxd + nacts[b]);
        best_res = res[b];
        best_ep = done + b;
      }
    }
    done += B;
    // root-parallel merge of root children statistics
    if (merge && m.p.merge_every && done / m.p.merge_every > merges_done) {
      merges_done = done / m.p.merge_every;
      std::vector<int64_t> buf(2 * (size_t)n_ord1);
      for (uint32_t o = 0; o < n_ord1; ++o) {
        buf[2 * o] = m.root_own_n[o];
        buf[2 * o + 1] = m.root_own_w[o];
      }
      if (merge(merge_user, buf.data(), (uint32_t)buf.size(), 0) != 0) {
        set_err(err, PE_ERR_INTERNAL, "merge hook failed");
        return PE_ERR_INTERNAL;
      }
      for (uint32_t o = 0; o < n_ord1; ++o) {
        m.root_extra_n[o] += buf[2 * o] - m.root_own_n[o];
        m.root_extra_w[o] += buf[2 * o + 1] - m.root_own_w[o];
        m.root_own_n[o] = 0;
        m.root_own_w[o] = 0;
      }
    }
  }
  // the best plan over all ranks: max reward, ties -> lowest rank
  uint32_t winner = m.p.rank;
  if (merge) {
    int64_t key[2] = {(int64_t)std::llround(std::max(best_reward, 0.0) * kFixed),
                      -(int64_t)m.p.rank};
    int64_t mx[1] = {key[0]};
    if (merge(merge_user, mx, 1, 1) != 0) {
      set_err(err, PE_ERR_INTERNAL, "merge hook failed");
      return PE_ERR_INTERNAL;
    }
    int64_t rk[1] = {key[0] == mx[0] ? key[1] : INT64_MIN / 2};
    if (merge(merge_user, rk, 1, 1) != 0) {
      set_err(err, PE_ERR_INTERNAL, "merge hook failed");
      return PE_ERR_INTERNAL;
    }
    winner = (uint32_t)(-rk[0]);
    std::vector<int64_t> plan(3 + PE_PLAN_MAX_ACTIONS, 0);
    if (winner == m.p.rank) {
      plan[0] = (int64_t)best_acts.size();
      plan[1] = best_ep;
      for (size_t k = 0; k < best_acts.size(); ++k) {
        int64_t x = 0;
        std::memcpy(&x, &best_acts[k], sizeof(pe_action));
        plan[3 + k] = x;
      }
    }
    if (merge(merge_user, plan.data(), (uint32_t)plan.size(), 0) != 0) {
      set_err(err, PE_ERR_INTERNAL, "merge hook failed");
      return PE_ERR_INTERNAL;
    }
    if (winner != m.p.rank) {
      best_acts.resize((size_t)plan[0]);
      for (size_t k = 0; k < best_acts.size(); ++k)
        std::memcpy(&best_acts[k], &plan[3 + k], sizeof(pe_action));
      best_ep = (uint32_t)plan[1];
      // re-evaluate the winning plan locally (deterministic)
      std::vector<pe_action> pfx = best_acts;
      pe_action stop{};
      stop.kind = PE_ACT_STOP;
      pfx.push_back(stop);
      uint32_t po[2] = {0, (uint32_t)pfx.size()};
      uint64_t sd = 0;
      std::vector<pe_action> ao(maxd);
      uint32_t na = 0;
      std::vector<uint64_t> lg(lw + 1);
      if (eval(eval_user, pfx.data(), po, &sd, 1, ao.data(), &na, &best_res, lg.data()) != 0) {
        set_err(err, PE_ERR_CUDA, "evaluator failed");
        return PE_ERR_CUDA;
      }
    }
  }
  out->n_actions = (uint32_t)std::min<size_t>(best_acts.size(), PE_PLAN_MAX_ACTIONS);
  for (uint32_t k = 0; k < out->n_actions; ++k) out->actions[k] = best_acts[k];
  out->episodes = done;
  out->found_at_episode = best_ep;
  out->winner_rank = winner;
  out->result = best_res;
  return PE_OK;
}
