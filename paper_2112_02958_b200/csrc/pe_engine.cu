// pe_engine.cu — CUDA engine and C-ABI (include/pe.h) for batched candidate
// evaluation on B200 (sm_100a).
//
// Device layout:
//   * the compiled graph (pe::GraphView tables) lives once in HBM;
//   * every in-flight candidate owns one arena (pe::Layout) in HBM, reused
//     across the candidates that slot processes;
//   * kernels: pe_eval_kernel (explicit action sequences) and
//     pe_rollout_kernel (MCTS leaf rollouts), one thread per candidate,
//     candidates claimed from a global work counter so long rollouts do not
//     stall a static partition.
// There is no CPU fallback: without a device every entry point fails with
// PE_ERR_NO_DEVICE.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <unordered_map>
#include <vector>

#include "pe.h"
#include "pe_core.cuh"
#include "pe_graph.h"

struct pe_graph {
  pe::HostGraph g;
};

struct pe_engine {
  const pe_graph* graph = nullptr;
  int device = 0;
  pe_search_config cfg{};
  pe_cost_params cp{};
  pe::GraphView dview{};  // device pointers
  pe::Layout layout{};      // tight arenas (main pass)
  pe::Layout big_layout{};  // full-size arenas (retry pass)
  uint8_t* d_graph = nullptr;
  uint8_t* d_arena = nullptr;
  uint8_t* d_big_arena = nullptr;
  uint32_t slots = 0;
  uint32_t big_slots = 0;
  int64_t baseline = 1;
  uint32_t n_ordinals = 0;
  pe::Worklist wl;
  uint64_t launches = 0;
  int64_t graph_bytes = 0;
  int sm_count = 148;
  bool l2_persist = false;  // experiment: graph image in the persisting L2 carve-out
  size_t l2_window = 0, l2_prev_limit = 0;
  // staging for host-pointer calls
  uint8_t* d_io = nullptr;
  size_t io_cap = 0;
  // work counters of the main-pass kernels (zeroed before each launch)
  uint32_t* d_ctr = nullptr;
  // prefix-trie scheduling: legal sets after short
  // decision prefixes (deterministic for the graph and config), per node:
  // legal-ordinal count, child offset, depth; children per legal index
  int sched_depth = 3;
  uint32_t sched_min_batch = 8192;
  int32_t sched_max_nodes = 1 << 16;
  std::vector<int32_t> t_nl, t_child_off, t_depth, t_parent, t_pick;
  std::vector<int32_t> t_legal_off, t_legal, t_child;
  bool t_dirty = true;
  int32_t* d_tnode = nullptr;  // int4 per node: nl, child offset, depth, 0
  int32_t* d_tchild = nullptr;
  uint32_t* d_tmiss = nullptr;
  size_t tnode_cap = 0, tchild_cap = 0;
  uint32_t* d_keys = nullptr;
  uint32_t* d_perm = nullptr;
  uint32_t* d_hist = nullptr;
  size_t sched_cap = 0, perm_cap = 0, hist_cap = 0;
  uint64_t sched_probes = 0;  // prefix states probed (diagnostic)
  // prefix-state reuse: per node its decision path and snapshot index
  int32_t path_cap = 3;
  std::vector<pe_action> t_path;
  std::vector<int32_t> t_snap;
  pe_action* d_tpath = nullptr;
  size_t tpath_cap = 0;
  uint8_t* d_snap = nullptr;
  uint64_t snap_stride = 0;
  int32_t snap_cap = 0, snap_used = 0;
  double snap_budget_gb = 0.0;  // prefix-state reuse: off unless enabled
  // Calls share the engine's arenas, work counters and staging buffers, so
  // calls on different streams are serialised on the device: each call's
  // stream waits for the previous call's last enqueued work.
  cudaEvent_t done = nullptr;
  // Prefix-state cache (pe_engine_set_prefix_cache): the post-prefix states
  // of host-mode rollout prefixes (MCTS leaves: the tree path), keyed by the
  // prefix's bytes.  A candidate starts from its longest cached prefix and
  // saves its own; slots are reused least-recently-used (clock hand).
  double pc_budget_gb = 0.0;
  uint8_t* d_pc = nullptr;
  uint64_t pc_stride = 0;
  int32_t pc_cap = 0, pc_hand = 0;
  std::unordered_map<std::string, int32_t> pc_map;
  std::vector<std::string> pc_key;
  std::vector<uint64_t> pc_used;
  uint64_t pc_clock = 0, pc_hits = 0, pc_saved = 0;
  std::vector<std::string> pc_pending;  // per candidate of the current call
  uint64_t* d_cv = nullptr;  // from | save addresses, from_len, saved flags
  size_t cv_cap = 0;
  // main rollout launch timing (pe_engine_set_kernel_timing): an event pair
  // around each main launch on its stream
  bool ktiming = false;
  uint32_t small_block = 32;  // block size of launches below full occupancy
  uint32_t cpw_force = 0;     // PE_CPW: cap on candidates per warp (experiments)
  bool coop = true;           // one-candidate-per-warp launches run warp-cooperatively
  std::vector<cudaEvent_t> kev, kev_free;
};

struct pe_state {
  pe_engine* e = nullptr;
  uint8_t* d_snap = nullptr;         // Cand::save image of the propagated state
  std::vector<pe_action> path;       // the decisions it covers
  pe_result result{};                // its evaluation (lowered + scored)
  std::vector<int32_t> trace;        // its parity trace (pe_state_specs)
};

namespace {

// NVTX range over an engine call (nsys / ncu timelines; header-only NVTX 3)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

void set_err(pe_error* err, int code, const std::string& msg, int line = 0, int col = 0) {
  if (!err) return;
  err->code = code;
  err->line = line;
  err->column = col;
  std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
}

bool cuda_ok(cudaError_t e, pe_error* err, const char* what) {
  if (e == cudaSuccess) return true;
  set_err(err, PE_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  return false;
}

// (round 1's PE_SOLO experiment -- one candidate per warp -- is now the
// runtime threads-per-slot choice of enqueue_rollouts)
constexpr uint32_t kThreadsPerSlot = 1;
#ifndef PE_MIN_BLOCKS
#define PE_MIN_BLOCKS 8
#endif
constexpr int kBlock = 128;
// resident blocks per SM the register allocation must allow: 8 -> 32 warps
// per SM (<= 64 registers / thread).  The per-thread work is a dependent
// chain of global-memory accesses, so resident warps = latency hiding:
// measured 342K vs 277K cand/s for 4 blocks (128 registers) at config 3
// despite the spills (profiles/r1_summary.md).
constexpr int kMinBlocks = PE_MIN_BLOCKS;
// The main rollout launch at full occupancy uses one block of all the SM's
// resident threads (same 64-register bound), so the first wave of an SM is
// kSmBlock consecutive positions of the trie-sorted order: neighbours share
// code paths (the kernel is instruction-fetch bound) and
// graph records.  Measured 3.05-3.09M vs 2.93-2.97M cand/s with 8 blocks of
// 128 (whose first waves interleave positions 148 x 128 apart on an SM).
// Smaller launches (fewer slots than the SMs' resident threads, e.g. a
// memory-budget-limited config 4) keep 128-thread blocks so every SM works.
constexpr int kSmBlock = kBlock * kMinBlocks;

#ifdef PE_PHASE_TIMERS
// profiling build only (tools/phase_profile.py): summed clock64 per phase
__device__ unsigned long long g_phase_cycles[9];
#endif
#ifdef PE_CAND_TIMES
// profiling build only (tools/tail_profile.py): per schedule position its
// start / end %globaltimer and SM
constexpr uint32_t kCandTimesCap = 1u << 20;
__device__ unsigned long long g_cand_times[kCandTimesCap * 2];
__device__ uint32_t g_cand_sm[kCandTimesCap];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

// resident rollout threads per SM (experiment knob; the product value is
// the 64-register limit's 1024)
#ifndef PE_SM_THREADS
#define PE_SM_THREADS (kBlock * kMinBlocks)
#endif
#ifndef PE_FW_GROUP
#define PE_FW_GROUP 1024
#endif
#ifndef PE_STATIC_SCHED
#define PE_STATIC_SCHED 0
#endif
// Next candidate of a thread.  Each thread starts on candidate `slot` (the
// 32 lanes of a warp start together); after that, the main pass hands out
// candidates from a work counter, so a batch that is not a multiple of the
// slot count does not leave threads idle while others run a second wave.
// RETRY launches (few candidates) keep the static stride.
template <bool RETRY>
__device__ __forceinline__ uint32_t next_cand(uint32_t i, uint32_t slots, uint32_t* ctr) {
  if (RETRY || PE_STATIC_SCHED) return i + slots;
  return slots + atomicAdd(ctr, 1u);
}

// One thread per candidate.  RETRY launches re-evaluate, in full-size
// arenas, exactly the candidates whose tight arena overflowed (status
// PE_CAND_CAPACITY).
template <bool RETRY>
__global__ void __launch_bounds__(kBlock, kMinBlocks)
pe_eval_kernel(const __grid_constant__ pe::GraphView g, const __grid_constant__ pe::Layout L,
               uint8_t* arena, uint32_t slots,
               const pe_action* acts, const uint32_t* off, uint32_t n, pe_cost_params cp,
               int64_t baseline, pe_result* out, int32_t* trace, uint32_t trace_words,
               uint8_t* argflags, uint32_t* ctr, uint32_t tps) {
  // tps = threads per slot (pe_rollout_kernel; threads_per_slot)
  if (threadIdx.x % tps) return;
  uint32_t slot = (blockIdx.x * blockDim.x + threadIdx.x) / tps;
  if (slot >= slots) return;
  pe::Cand c(g, L, arena + (uint64_t)(slot / pe::kLanes) * L.bytes, slot % pe::kLanes);
  for (uint32_t i = slot; i < n; i = next_cand<RETRY>(i, slots, ctr)) {
    if (RETRY && out[i].status != PE_CAND_CAPACITY) continue;
    pe_result r;
    c.eval(acts + off[i], (int32_t)(off[i + 1] - off[i]), cp, baseline, r,
           trace ? trace + (uint64_t)i * trace_words : nullptr, trace_words,
           argflags ? argflags + (uint64_t)i * g.A : nullptr);
    out[i] = r;
  }
}

// Prefix-state reuse: per candidate its trie key (2 * node,
// +1 when its next draw is Stop), per node {nl, child offset, depth,
// snapshot index or -1} and its decision path, and the snapshot pool.
struct SchedView {
  const uint32_t* keys = nullptr;
  const int4* tnode = nullptr;
  const pe_action* tpath = nullptr;
  int32_t path_cap = 0;
  const uint8_t* snap = nullptr;
  uint64_t stride = 0;
  uint32_t kstride = 1;  // keys are node * kstride + slot
};

// Per-candidate saved states (prefix-state cache, pe_state handles): start
// from the state at device address from[i] (0: none) covering the first
// from_len[i] prefix entries; save the post-prefix state to save[i] (0:
// none) and set saved[i] = 1 once written.
struct CacheView {
  const uint64_t* from = nullptr;
  const int32_t* from_len = nullptr;
  const uint64_t* save = nullptr;
  uint8_t* saved = nullptr;
};

template <bool RETRY, bool RS, int F>
__global__ void __launch_bounds__(kSmBlock, 1)
pe_rollout_kernel(const __grid_constant__ pe::GraphView g, const __grid_constant__ pe::Layout L,
                  uint8_t* arena, uint32_t slots,
                  const pe_action* prefix, const uint32_t* poff, const uint64_t* seeds,
                  uint32_t n, int32_t maxd, pe_cost_params cp, int64_t baseline,
                  pe_action* acts_out, uint32_t* n_out, pe_result* out, uint64_t* legal_out,
                  int32_t legal_words, uint32_t* ctr, const uint32_t* perm,
                  const __grid_constant__ SchedView sv, const __grid_constant__ CacheView cv,
                  uint32_t tps, uint32_t* max_acts) {
  // tps = threads per slot: one lane in every tps runs a candidate, so a
  // warp holds 32 / tps candidates (enqueue_rollouts picks it per launch:
  // the lanes of a warp serialise their divergent paths, so a batch that
  // does not need every lane runs with fewer candidates per warp)
  // (kFCoop: tps = 32 and every lane of the warp runs its one candidate)
  constexpr bool COOP = (F & pe::kFCoop) != 0;
  if (!COOP && threadIdx.x % tps) return;
  uint32_t slot = (blockIdx.x * blockDim.x + threadIdx.x) / tps;
  if (slot >= slots) return;
  const bool writer = !COOP || (threadIdx.x & 31) == 0;
  pe::Cand c(g, L, arena + (uint64_t)(slot / pe::kLanes) * L.bytes, slot % pe::kLanes);
  // k = schedule position; perm (prefix-trie scheduling) maps it to the
  // candidate, so lanes of a warp run candidates that share their first
  // decisions; results stay in candidate order.
  auto run = [&](uint32_t k) {
    uint32_t i = perm ? perm[k] : k;
    if (RETRY && out[i].status != PE_CAND_CAPACITY) return;
    // start from a saved state: the candidate's trie node's, or its longest
    // cached prefix's
    pe::Resume rs;
    if ((F & pe::kFResume) && sv.keys) {
      uint32_t key = sv.keys[i], node = key / sv.kstride;
      int4 nd = sv.tnode[node];
      if (nd.w >= 0) {
        rs.snap = sv.snap + sv.stride * (uint64_t)nd.w;
        rs.done = rs.draws = nd.z;
        rs.path = sv.tpath + (uint64_t)node * sv.path_cap;
        rs.stop = key % sv.kstride == 0;  // its next draw is Stop
      }
    }
    if ((F & pe::kFResume) && cv.from) {
      if (cv.from[i]) {
        rs.snap = reinterpret_cast<const uint8_t*>(cv.from[i]);
        rs.done = rs.k0 = cv.from_len[i];
        rs.path = prefix + poff[i];
      }
      if (cv.save[i]) {
        rs.save = reinterpret_cast<uint8_t*>(cv.save[i]);
        rs.saved = cv.saved + i;
      }
    }
#if defined(PE_CAND_TIMES) && defined(__CUDA_ARCH__)
    unsigned long long t_begin = gtimer();
#endif
    pe_result r;
    c.template rollout<RS, F>(prefix + poff[i], (int32_t)(poff[i + 1] - poff[i]), seeds[i], maxd,
                           cp, baseline, acts_out + (uint64_t)i * maxd, n_out + i, r,
                           legal_out ? legal_out + (uint64_t)i * legal_words : nullptr,
                           legal_words, rs);
    if (writer) out[i] = r;
#if defined(PE_CAND_TIMES) && defined(__CUDA_ARCH__)
    if (!RETRY && k < kCandTimesCap) {
      g_cand_times[2 * k] = t_begin;
      g_cand_times[2 * k + 1] = gtimer();
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      g_cand_sm[k] = smid;
    }
#endif
    // longest action list of the batch (host mode copies only that many
    // columns of acts_out back)
    if (max_acts && writer) atomicMax(max_acts, n_out[i]);
  };
  if (RETRY || COOP) {
    for (uint32_t k = slot; k < n; k += slots) run(k);
  } else {
    // Warp-chunked dynamic schedule: the first wave is position `slot`;
    // afterwards the warp's lanes take the next consecutive positions
    // together (lane 0 claims a chunk of the warp's width), so a warp keeps
    // running neighbours in the sorted order instead of scattering.
    const unsigned mask = __activemask();
    const uint32_t width = __popc(mask);
    const uint32_t rank = __popc(mask & ((1u << (threadIdx.x & 31)) - 1u));
    // (every lane of `mask` stays in the loop until the warp-uniform exit)
    uint32_t k = slot;
#if PE_FW_GROUP < 1024
    // experiment: an SM-wide block's first wave as 1024 / PE_FW_GROUP runs of
    // PE_FW_GROUP consecutive positions, spread over the order
    if (blockDim.x == PE_SM_THREADS && slots == gridDim.x * PE_SM_THREADS) {
      uint32_t t = threadIdx.x;
      k = ((t / PE_FW_GROUP) * gridDim.x + blockIdx.x) * PE_FW_GROUP + t % PE_FW_GROUP;
    }
#endif
    while (true) {
      if (k < n) run(k);
      __syncwarp(mask);
      uint32_t base = 0;
      if (rank == 0) base = slots + atomicAdd(ctr, width);
      base = __shfl_sync(mask, base, __ffs(mask) - 1);
      if (base >= n) break;
      k = base + rank;
    }
  }
#if defined(PE_PHASE_TIMERS) && defined(__CUDA_ARCH__)
  for (int k = 0; k < 9; ++k) atomicAdd(&g_phase_cycles[k], (unsigned long long)c.ph[k]);
#endif
}

// Arena calibration: root rollouts in full-size arenas, recording the
// largest value-slot, loop, front-stack, SPMD-op and operand-log counts.
__global__ void __launch_bounds__(kBlock, kMinBlocks)
pe_calib_kernel(const __grid_constant__ pe::GraphView g, const __grid_constant__ pe::Layout L,
                uint8_t* arena, uint32_t slots, uint32_t n, int32_t maxd, pe_cost_params cp,
                pe_action* acts, uint32_t* n_out, int32_t* hw) {
  uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= slots) return;
  pe::Cand c(g, L, arena + (uint64_t)(slot / pe::kLanes) * L.bytes, slot % pe::kLanes);
  for (uint32_t k = slot; k < n; k += slots) {
    pe_result r;
    c.template rollout<false, 0>(nullptr, 0, 0x5EEDull * (k + 1), maxd, cp, 1,
                              acts + (uint64_t)k * maxd, n_out + k, r, nullptr, 0);
    atomicMax(&hw[0], c.nslots);
    atomicMax(&hw[1], c.nloops);
    atomicMax(&hw[2], c.nfs);
    atomicMax(&hw[3], c.nem);
    atomicMax(&hw[4], c.neo);
  }
}

// ---- prefix-trie scheduling kernels ----
// Probe: evaluates each prefix (no decisions after it), records the legal
// set after it and saves the state after it as the node's snapshot.
__global__ void __launch_bounds__(kBlock, kMinBlocks)
pe_probe_kernel(const __grid_constant__ pe::GraphView g, const __grid_constant__ pe::Layout L,
                uint8_t* arena, uint32_t slots, const pe_action* prefix, const uint32_t* poff,
                uint32_t n, int32_t acts_stride, pe_cost_params cp, int64_t baseline,
                pe_action* acts_out, uint32_t* n_out, pe_result* out, uint64_t* legal_out,
                int32_t legal_words, uint8_t* snap, uint64_t stride, int32_t* snap_idx) {
  uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= slots) return;
  pe::Cand c(g, L, arena + (uint64_t)(slot / pe::kLanes) * L.bytes, slot % pe::kLanes);
  for (uint32_t k = slot; k < n; k += slots) {
    int32_t np = (int32_t)(poff[k + 1] - poff[k]);
    pe_result r;
    c.template rollout<false, 0>(prefix + poff[k], np, 0, np, cp, baseline,
                              acts_out + (uint64_t)k * acts_stride, n_out + k, r,
                              legal_out + (uint64_t)k * legal_words, legal_words);
    out[k] = r;
    // a probe that overflowed its tight arena saves nothing (the retry
    // launch re-derives its legal set only): report that to the host, which
    // attaches a snapshot to the trie node only when it was written
    if (snap_idx[k] >= 0) {
      if (r.status == PE_CAND_OK) c.save(snap + stride * (uint64_t)snap_idx[k]);
      else snap_idx[k] = -1;
    }
  }
}

// Walks candidate i's seed through the trie with exactly the rollout's
// draws (Cand::rollout: no draw when nothing is legal; Stop weight 1 before
// the first decision, 2 after) and keys it by the deepest known node (odd
// key: the rollout stops there).  Unprobed children that are reached are
// flagged for the host to probe.
__global__ void pe_sched_key_kernel(uint32_t n, const uint64_t* seeds, int32_t depth,
                                    int32_t maxd, uint32_t kstride, const int4* tnode,
                                    const int32_t* tchild, uint32_t* tmiss, uint32_t* nmiss,
                                    uint32_t* keys, uint32_t* hist) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t st = seeds[i];
  int32_t node = 0, steps = 0;
  uint32_t slot;  // 0: Stop drawn here, 1: the rollout ends here (nothing
                  // legal / decision cap), 2 + p: its next action is legal[p]
  while (true) {
    int4 nd = tnode[node];
    if (nd.x == 0 || steps >= maxd) {
      slot = 1;
      break;
    }
    uint64_t ws = steps >= 1 ? 2 : 1;
    uint64_t pick = pe::Cand::splitmix(st) % ((uint64_t)nd.x + ws);
    if (pick >= (uint64_t)nd.x) {
      slot = 0;
      break;
    }
    // at the trie's depth the next action is still known (the node's legal
    // set); below, an unprobed child is flagged for the host to probe
    if (steps >= depth) {
      slot = 2 + (uint32_t)pick;
      break;
    }
    int32_t c = tchild[nd.y + (int32_t)pick];
    if (c < 0) {
      tmiss[nd.y + (int32_t)pick] = 1u;
      atomicAdd(nmiss, 1u);  // candidates that would group deeper after a probe
      slot = 2 + (uint32_t)pick;
      break;
    }
    node = c;
    ++steps;
  }
  uint32_t key = (uint32_t)node * kstride + slot;
  keys[i] = key;
  atomicAdd(&hist[key], 1u);
}

// exclusive scan of hist[0, m) in place (one block)
__global__ void pe_sched_scan_kernel(uint32_t* hist, uint32_t m) {
  __shared__ uint32_t part[1024];
  uint32_t t = threadIdx.x, chunk = (m + blockDim.x - 1) / blockDim.x;
  uint32_t lo = min(m, t * chunk), hi = min(m, lo + chunk), sum = 0;
  for (uint32_t k = lo; k < hi; ++k) sum += hist[k];
  part[t] = sum;
  __syncthreads();
  if (t == 0) {
    uint32_t run = 0;
    for (uint32_t k = 0; k < blockDim.x; ++k) {
      uint32_t v = part[k];
      part[k] = run;
      run += v;
    }
  }
  __syncthreads();
  uint32_t run = part[t];
  for (uint32_t k = lo; k < hi; ++k) {
    uint32_t v = hist[k];
    hist[k] = run;
    run += v;
  }
}

__global__ void pe_sched_scatter_kernel(uint32_t n, const uint32_t* keys, uint32_t* offs,
                                        uint32_t* perm) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // reversed: deeper trie nodes (candidates with more decisions, the longer
  // rollouts) are handed out first, short ones fill the tail
  perm[n - 1 - atomicAdd(&offs[keys[i]], 1u)] = i;
}

// Append a host vector to the device image; returns its offset.
template <typename T>
size_t stage(std::vector<uint8_t>& img, const std::vector<T>& v) {
  size_t at = (img.size() + 15) & ~size_t(15);
  img.resize(at + std::max<size_t>(v.size() * sizeof(T), 16));
  if (!v.empty()) std::memcpy(img.data() + at, v.data(), v.size() * sizeof(T));
  return at;
}

bool ensure_io(pe_engine* e, size_t bytes, pe_error* err) {
  if (bytes <= e->io_cap) return true;
  if (e->d_io) cudaFree(e->d_io);
  e->d_io = nullptr;
  e->io_cap = 0;
  size_t cap = std::max<size_t>(bytes, 1 << 20);
  if (!cuda_ok(cudaMalloc(&e->d_io, cap), err, "cudaMalloc(io)")) return false;
  e->io_cap = cap;
  return true;
}

uint32_t launch_slots(const pe_engine* e, uint32_t n) { return std::min<uint32_t>(e->slots, n); }

// Candidates per warp of a launch, as threads per slot (32 / candidates per
// warp).  A lane's candidate waits for the other lanes' divergent paths
// (config 3: one candidate alone takes 7.5 ms, 1,024 candidates 46 ms at 32
// per warp but 11.4 ms at 1 per warp), so a launch that does not need every
// lane of the resident warps runs the fewest candidates per warp that still
// fit them in one wave: below 4 x the resident warps (the gain measured up
// to 3.5x; at 7x equal, at 14x 32 per warp wins by 5 %).  PE_CPW forces it.
uint32_t threads_per_slot(const pe_engine* e, uint32_t slots) {
  const uint32_t warps = (uint32_t)e->sm_count * PE_SM_THREADS / 32;
  uint32_t cpw = 32;
  if ((uint64_t)slots <= 4ull * warps)
    while (cpw > 1 && (uint64_t)(cpw / 2) * warps >= slots) cpw /= 2;
  if (e->cpw_force) cpw = std::min<uint32_t>(32, e->cpw_force);
  return 32 / cpw;
}

bool ir_expand_batch(pe_engine* e, std::vector<std::vector<pe_action>*>& seqs, cudaStream_t st,
                     pe_error* err);

// order this call after the engine's previous call (any stream)
bool call_begin(pe_engine* e, cudaStream_t st, pe_error* err) {
  return cuda_ok(cudaStreamWaitEvent(st, e->done, 0), err, "stream wait");
}
bool call_end(pe_engine* e, cudaStream_t st, pe_error* err) {
  return cuda_ok(cudaEventRecord(e->done, st), err, "event record");
}

}  // namespace

extern "C" {

void pe_default_cost_params(pe_cost_params* out) {
  out->memory_budget_bytes = 16ll << 30;
  out->flops_per_second = 1e14;
  out->bytes_per_second = 1e11;
  out->collective_latency_s = 1e-6;
  out->w_mem = 0.1;
  out->w_comm = 1.0;
  out->w_steps = 0.01;
}

void pe_default_search_config(pe_search_config* out) {
  std::memset(out, 0, sizeof(*out));
  out->auto_axes_mask = 0xffffffffu;
  out->max_decisions = 32;
  out->group_scopes = 1;
  out->episodes = 500;
  out->seed = 0;
  out->uct_c = 1.414;
  out->leaf_batch = 8192;  // one launch fills the GPU; DESIGN.md §5 (time-to-plan table)
}

// ------------------------------------------------------------------ graph
pe_status pe_graph_create(const char* pir, size_t len, pe_graph** out, pe_error* err) {
  if (!pir || !out) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null argument");
    return PE_ERR_INVALID_ARGUMENT;
  }
  pe_graph* g = new (std::nothrow) pe_graph();
  if (!g) {
    set_err(err, PE_ERR_INTERNAL, "out of memory");
    return PE_ERR_INTERNAL;
  }
  pe::LoadError le;
  if (!pe::load_graph(pir, len, g->g, le)) {
    set_err(err, le.code, le.message, le.line, le.column);
    delete g;
    return (pe_status)le.code;
  }
  *out = g;
  if (err) err->code = PE_OK;
  return PE_OK;
}

pe_status pe_graph_create_from_arrays(const char* name, int32_t n_axes,
                                      const char* const* axis_names, const int64_t* axis_sizes,
                                      int32_t n_args, const pe_arg_desc* args, int32_t n_ops,
                                      const pe_op_desc* ops, int32_t result, pe_graph** out,
                                      pe_error* err) {
  if (!out || n_axes < 0 || n_args < 0 || n_ops < 0 || (n_axes && (!axis_names || !axis_sizes)) ||
      (n_args && !args) || (n_ops && !ops)) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null argument or negative count");
    return PE_ERR_INVALID_ARGUMENT;
  }
  pe_graph* g = new (std::nothrow) pe_graph();
  if (!g) {
    set_err(err, PE_ERR_INTERNAL, "out of memory");
    return PE_ERR_INTERNAL;
  }
  pe::HostGraph& h = g->g;
  auto bad = [&](const std::string& m) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, m);
    delete g;
    return PE_ERR_INVALID_ARGUMENT;
  };
  h.name = name ? name : "";
  for (int32_t a = 0; a < n_axes; ++a) {
    h.axis_names.push_back(axis_names[a] ? axis_names[a] : "");
    h.axis_sizes.push_back(axis_sizes[a]);
  }
  auto dims_of = [](int32_t rank, const int64_t* sh) {
    return std::vector<int64_t>(sh, sh + std::max(0, std::min(rank, (int32_t)PE_MAX_RANK)));
  };
  for (int32_t a = 0; a < n_args; ++a) {
    const pe_arg_desc& d = args[a];
    if (d.rank < 0 || d.rank > PE_MAX_RANK) return bad("argument rank out of range");
    pe::HostArg x;
    x.id = d.id ? d.id : "a" + std::to_string(a);
    x.scope = d.scope ? d.scope : "";
    x.shape = dims_of(d.rank, d.shape);
    h.args.push_back(std::move(x));
  }
  for (int32_t o = 0; o < n_ops; ++o) {
    const pe_op_desc& d = ops[o];
    if (d.kind < 0 || d.kind >= pe::kNumBaseKinds) return bad("op kind outside the base dialect");
    if (d.rank < 0 || d.rank > PE_MAX_RANK || d.n_operands < 0 || (d.n_operands && !d.operands) ||
        d.n_batch < 0 || d.n_batch > PE_MAX_RANK || d.n_contract < 0 ||
        d.n_contract > PE_MAX_RANK || d.n_dims < 0 || d.n_dims > PE_MAX_RANK)
      return bad("op descriptor field out of range");
    pe::HostOp x;
    x.id = d.id ? d.id : std::to_string(o);
    x.kind = (pe::Kind)d.kind;
    x.shape = dims_of(d.rank, d.shape);
    for (int32_t k = 0; k < d.n_operands; ++k) {
      if (d.operands[k] < 0 || d.operands[k] >= n_args + o)
        return bad("op " + x.id + ": operand is not an earlier value");
      x.operands.push_back(d.operands[k]);
    }
    x.lhs_batch.assign(d.lhs_batch, d.lhs_batch + d.n_batch);
    x.rhs_batch.assign(d.rhs_batch, d.rhs_batch + d.n_batch);
    x.lhs_contract.assign(d.lhs_contract, d.lhs_contract + d.n_contract);
    x.rhs_contract.assign(d.rhs_contract, d.rhs_contract + d.n_contract);
    x.dims.assign(d.dims, d.dims + d.n_dims);
    if (x.kind == pe::kSlice && !x.operands.empty()) {
      int32_t r = (int32_t)h.value_shape(x.operands[0]).size();
      x.start.assign(d.start, d.start + r);
      x.limit.assign(d.limit, d.limit + r);
    }
    x.dim = d.dim;
    x.value = d.value;
    x.scope = d.scope ? d.scope : "";
    h.ops.push_back(std::move(x));
  }
  if (result < 0 || result >= n_args + n_ops) return bad("result is not a value index");
  h.result = result;
  std::vector<std::string> seen;
  for (int32_t v = 0; v < h.num_values(); ++v) {
    const std::string& id = v < n_args ? h.args[v].id : h.ops[v - n_args].id;
    seen.push_back(id);
  }
  std::sort(seen.begin(), seen.end());
  if (std::adjacent_find(seen.begin(), seen.end()) != seen.end()) return bad("duplicate value name");
  pe::LoadError le;
  if (!pe::finish_graph(h, le)) {
    set_err(err, le.code, le.message);
    delete g;
    return (pe_status)le.code;
  }
  *out = g;
  if (err) err->code = PE_OK;
  return PE_OK;
}

void pe_graph_destroy(pe_graph* g) { delete g; }
int32_t pe_graph_axis_name(const pe_graph* g, int32_t axis, char* buf, int32_t cap) {
  if (!g || axis < 0 || axis >= (int32_t)g->g.axis_names.size()) return -1;
  const std::string& s = g->g.axis_names[axis];
  if (buf && cap > 0) std::snprintf(buf, cap, "%s", s.c_str());
  return (int32_t)s.size();
}
int32_t pe_graph_num_args(const pe_graph* g) { return (int32_t)g->g.args.size(); }
int32_t pe_graph_num_ops(const pe_graph* g) { return (int32_t)g->g.ops.size(); }
int32_t pe_graph_num_axes(const pe_graph* g) { return (int32_t)g->g.axis_names.size(); }
int32_t pe_graph_num_operands(const pe_graph* g) { return (int32_t)g->g.oopnd.size(); }
int64_t pe_graph_axis_size(const pe_graph* g, int32_t axis) {
  if (axis < 0 || axis >= (int32_t)g->g.axis_sizes.size()) return -1;
  return g->g.axis_sizes[axis];
}
int32_t pe_graph_value_index(const pe_graph* g, const char* name) {
  return name ? g->g.value_index(name) : -1;
}
int32_t pe_graph_axis_index(const pe_graph* g, const char* name) {
  return name ? g->g.axis_index(name) : -1;
}
int32_t pe_graph_value_name(const pe_graph* g, int32_t v, char* buf, int32_t cap) {
  if (v < 0 || v >= g->g.num_values()) return -1;
  const std::string& s =
      v < (int32_t)g->g.args.size() ? g->g.args[v].id : g->g.ops[v - g->g.args.size()].id;
  if (buf && cap > 0) std::snprintf(buf, cap, "%s", s.c_str());
  return (int32_t)s.size();
}
int32_t pe_graph_value_shape(const pe_graph* g, int32_t v, int64_t* dims) {
  if (v < 0 || v >= g->g.num_values()) return -1;
  const auto& s = g->g.value_shape(v);
  for (size_t d = 0; d < s.size() && dims; ++d) dims[d] = s[d];
  return (int32_t)s.size();
}
int32_t pe_graph_arg_scope(const pe_graph* g, int32_t arg, char* buf, int32_t cap) {
  if (arg < 0 || arg >= (int32_t)g->g.args.size()) return -1;
  const std::string& s = g->g.args[arg].scope;
  if (buf && cap > 0) std::snprintf(buf, cap, "%s", s.c_str());
  return (int32_t)s.size();
}
int32_t pe_graph_num_groups(const pe_graph* g) { return (int32_t)g->g.groups.size(); }
int32_t pe_graph_group_size(const pe_graph* g, int32_t grp) {
  if (grp < 0 || grp >= (int32_t)g->g.groups.size()) return -1;
  return (int32_t)g->g.groups[grp].size();
}
int32_t pe_graph_group_member(const pe_graph* g, int32_t grp, int32_t i) {
  if (grp < 0 || grp >= (int32_t)g->g.groups.size()) return -1;
  if (i < 0 || i >= (int32_t)g->g.groups[grp].size()) return -1;
  return g->g.groups[grp][i];
}

// ------------------------------------------------------------------ engine
pe_status pe_engine_create(const pe_graph* graph, const pe_search_config* cfg,
                           const pe_cost_params* cp, int32_t device, pe_engine** out,
                           pe_error* err) {
  if (!graph || !out) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null argument");
    return PE_ERR_INVALID_ARGUMENT;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    set_err(err, PE_ERR_NO_DEVICE, "no CUDA device: the engine has no CPU fallback");
    return PE_ERR_NO_DEVICE;
  }
  if (device < 0 || device >= ndev) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "device index out of range");
    return PE_ERR_INVALID_ARGUMENT;
  }
  if (!cuda_ok(cudaSetDevice(device), err, "cudaSetDevice")) return PE_ERR_CUDA;
  pe_engine* e = new pe_engine();
  e->graph = graph;
  e->device = device;
  if (!cuda_ok(cudaEventCreateWithFlags(&e->done, cudaEventDisableTiming), err, "event")) {
    delete e;
    return PE_ERR_CUDA;
  }
  pe_default_search_config(&e->cfg);
  pe_default_cost_params(&e->cp);
  if (cfg) e->cfg = *cfg;
  if (cp) e->cp = *cp;
  if (e->cfg.max_decisions == 0) e->cfg.max_decisions = 32;
  cudaDeviceGetAttribute(&e->sm_count, cudaDevAttrMultiProcessorCount, device);
  const pe::HostGraph& g = graph->g;
  // worklist entries (SPEC build_worklist: arguments, optionally grouped)
  e->wl = pe::build_worklist(g, e->cfg.auto_axes_mask, e->cfg.group_scopes != 0,
                             e->cfg.scoped_only != 0, e->cfg.resurface_stuck != 0,
                             pe::worklist_filter(g, e->cfg));
  e->cfg.worklist_args = nullptr;  // read once; the caller's array may go away
  e->wl.infer_rest = e->cfg.infer_rest_action != 0;
  const pe::Worklist& w = e->wl;
  e->n_ordinals = (uint32_t)w.n_action_ordinals();

  // device image of the graph tables
  std::vector<uint8_t> img;
  size_t o_vshape = stage(img, g.vshape), o_vrank = stage(img, g.vrank);
  size_t o_okind = stage(img, g.okind), o_omask = stage(img, g.omask);
  size_t o_ooff = stage(img, g.oopnd_off), o_oopnd = stage(img, g.oopnd);
  size_t o_slotop = stage(img, g.slot_op), o_rerr = stage(img, g.orule_err);
  size_t o_cls = stage(img, g.ocls_off), o_crole = stage(img, g.cls_role);
  size_t o_crdim = stage(img, g.cls_rdim), o_cmoff = stage(img, g.cls_moff);
  size_t o_mem = stage(img, g.mem), o_scls = stage(img, g.slot_cls);
  size_t o_rcls = stage(img, g.op_rcls), o_uoff = stage(img, g.user_off);
  size_t o_users = stage(img, g.users), o_iu = stage(img, g.init_uses);
  size_t o_eoff = stage(img, w.ent_off), o_emem = stage(img, w.ent_mem);
  size_t o_goff = stage(img, w.grp_off), o_gmem = stage(img, w.grp_mem);
  size_t o_ooff2 = stage(img, w.ord_off), o_omem2 = stage(img, w.ord_mem);
  size_t o_eval = stage(img, w.ent_val);
  if (!cuda_ok(cudaMalloc(&e->d_graph, img.size()), err, "cudaMalloc(graph)") ||
      !cuda_ok(cudaMemcpy(e->d_graph, img.data(), img.size(), cudaMemcpyHostToDevice), err,
               "cudaMemcpy(graph)")) {
    pe_engine_destroy(e);
    return PE_ERR_CUDA;
  }
  e->graph_bytes = (int64_t)img.size();
  if (const char* lp = std::getenv("PE_L2_PERSIST")) {
    // experiment: the graph image as a persisting L2 window.  The carve-out
    // and the window are clamped to the device limits; a failure only turns
    // the hint off (and clears the pending error); destroy() gives the
    // carve-out back.
    if (std::atoi(lp) != 0) {
      int max_persist = 0, max_window = 0;
      cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, device);
      cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, device);
      size_t want = ((size_t)e->graph_bytes + (1 << 20)) & ~size_t((1 << 20) - 1);
      want = std::min<size_t>(want, (size_t)std::max(0, max_persist));
      e->l2_window = std::min<size_t>((size_t)e->graph_bytes, (size_t)std::max(0, max_window));
      if (want > 0 && e->l2_window > 0 &&
          cudaDeviceGetLimit(&e->l2_prev_limit, cudaLimitPersistingL2CacheSize) == cudaSuccess &&
          cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) == cudaSuccess) {
        e->l2_persist = true;
      } else {
        cudaGetLastError();
      }
    }
  }
  pe::GraphView v = g.host_view();
  uint8_t* b = e->d_graph;
  v.vshape = (const int32_t*)(b + o_vshape);
  v.vrank = b + o_vrank;
  v.okind = b + o_okind;
  v.omask = b + o_omask;
  v.oopnd_off = (const int32_t*)(b + o_ooff);
  v.oopnd = (const int32_t*)(b + o_oopnd);
  v.slot_op = (const int32_t*)(b + o_slotop);
  v.orule_err = b + o_rerr;
  v.ocls_off = (const int32_t*)(b + o_cls);
  v.cls_role = b + o_crole;
  v.cls_rdim = (const int8_t*)(b + o_crdim);
  v.cls_moff = (const int32_t*)(b + o_cmoff);
  v.mem = (const uint16_t*)(b + o_mem);
  v.slot_cls = (const int16_t*)(b + o_scls);
  v.op_rcls = (const int16_t*)(b + o_rcls);
  v.user_off = (const int32_t*)(b + o_uoff);
  v.users = (const int32_t*)(b + o_users);
  v.init_uses = (const int32_t*)(b + o_iu);
  pe::attach_worklist(v, w);  // scalars; pointers re-targeted to the device image
  v.ent_off = (const int32_t*)(b + o_eoff);
  v.ent_mem = (const int32_t*)(b + o_emem);
  v.grp_off = (const int32_t*)(b + o_goff);
  v.grp_mem = (const int32_t*)(b + o_gmem);
  v.ord_off = (const int32_t*)(b + o_ooff2);
  v.ord_mem = (const int32_t*)(b + o_omem2);
  v.ent_val = (const int32_t*)(b + o_eval);
  e->dview = v;

  // per-candidate arenas: one per thread slot, bounded by an HBM budget
  e->layout = pe::make_layout(v, /*tight=*/true);
  e->big_layout = pe::make_layout(v, /*tight=*/false);
  if (const char* sd = std::getenv("PE_SCHED_DEPTH")) e->sched_depth = std::atoi(sd);
  if (const char* co = std::getenv("PE_COOP")) e->coop = std::atoi(co) != 0;
  if (const char* cw = std::getenv("PE_CPW")) e->cpw_force = (uint32_t)std::max(0, std::atoi(cw));
  if (const char* sb = std::getenv("PE_SMALL_BLOCK"))  // experiment knob (32 .. 128)
    e->small_block = (uint32_t)std::min(128, std::max(32, std::atoi(sb) / 32 * 32));
  if (const char* sm = std::getenv("PE_SCHED_MIN_BATCH")) e->sched_min_batch = (uint32_t)std::atoi(sm);
  if (const char* sn = std::getenv("PE_SCHED_MAX_NODES")) e->sched_max_nodes = std::atoi(sn);
  if (const char* sg = std::getenv("PE_SCHED_SNAP_GB")) e->snap_budget_gb = std::atof(sg);
  e->path_cap = std::max(1, e->sched_depth);
  if (const char* dbg = std::getenv("PE_DEBUG_TIGHT_EM_CAP")) {
    // test hook: shrink the tight arena so candidates overflow and take the
    // retry path (tests/test_gpu_parity.py::test_capacity_retry_path)
    pe::Caps c = e->layout.caps;
    c.EM = std::max(4, std::atoi(dbg));
    e->layout = pe::relayout(v, c, false);
  }
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  // arena budget: up to 85 % of free HBM, at most 150 GiB (a second engine
  // created later sizes itself from what is then free; the rest -- >= 27 GB
  // on a 180 GB B200 -- is headroom for the caller's buffers and the prefix
  // cache); PE_ARENA_BUDGET_GB overrides.  Only large graphs are slot-limited
  // by it (config 4: 14.3 MB per candidate); 1/16 of it backs the full-size
  // retry arenas, which calibrated tight arenas rarely send work to.
  size_t budget = std::min<size_t>((size_t)(free_b * 0.85), (size_t)150 << 30);
  if (const char* gb = std::getenv("PE_ARENA_BUDGET_GB"))
    budget = std::min<size_t>(free_b, (size_t)(std::atof(gb) * (double)(1ull << 30)));
  // one resident thread per slot: kMinBlocks blocks of kBlock threads per SM;
  // arenas come in groups of kLanes interleaved candidates (one per warp)
  const uint64_t lanes = pe::kLanes;
  uint64_t want = (uint64_t)e->sm_count * PE_SM_THREADS / kThreadsPerSlot;
  uint64_t big_groups = std::min<uint64_t>(
      (uint64_t)e->sm_count * 8 / lanes,
      std::max<uint64_t>(1, (budget / 16) / std::max<uint64_t>(e->big_layout.bytes, 1)));
  e->big_slots = (uint32_t)(big_groups * lanes);
  // arenas start zeroed: the per-op `seen` marks of the stuck analysis are
  // cleared by each candidate after use, never wholesale
  if (!cuda_ok(cudaMalloc(&e->d_big_arena, (size_t)big_groups * e->big_layout.bytes), err,
               "cudaMalloc(big arena)") ||
      !cuda_ok(cudaMalloc(&e->d_ctr, 8 * sizeof(uint32_t)), err, "cudaMalloc(counters)") ||
      !cuda_ok(cudaMemset(e->d_big_arena, 0, (size_t)big_groups * e->big_layout.bytes), err,
               "zero arena")) {
    pe_engine_destroy(e);
    return PE_ERR_CUDA;
  }
  uint64_t fit_groups = (budget - big_groups * e->big_layout.bytes) /
                        std::max<uint64_t>(e->layout.bytes, 1);
  const char* calib_env = std::getenv("PE_CALIBRATE");
  bool calibrate = !(calib_env && std::atoi(calib_env) == 0) &&
                   !std::getenv("PE_DEBUG_TIGHT_EM_CAP") && !e->wl.auto_axes.empty();
  // (PE_CALIBRATE=2 forces it: tests exercise calibrated arenas on graphs
  // small enough for the oracle)
  bool force_calib = calib_env && std::atoi(calib_env) == 2;
  if ((fit_groups < want / lanes || force_calib) && calibrate) {
    // Slot-limited by the budget (large graphs): size the tight arena from
    // measured high-water marks of root rollouts (x1.3 + margin) instead of
    // the structural formula.  A candidate that still overflows takes the
    // full-size retry path, so calibration changes footprint, never results.
    const uint32_t nc = 2048;
    int32_t* d_hw = nullptr;
    pe_action* d_acts = nullptr;
    uint32_t* d_na = nullptr;
    int32_t hw[5] = {0, 0, 0, 0, 0};
    int32_t maxd = (int32_t)e->cfg.max_decisions;
    bool ok = cuda_ok(cudaMalloc(&d_hw, sizeof(hw)), err, "cudaMalloc(calibration)") &&
              cuda_ok(cudaMalloc(&d_acts, (size_t)nc * maxd * sizeof(pe_action)), err,
                      "cudaMalloc(calibration)") &&
              cuda_ok(cudaMalloc(&d_na, nc * 4), err, "cudaMalloc(calibration)") &&
              cuda_ok(cudaMemset(d_hw, 0, sizeof(hw)), err, "calibration");
    if (ok) {
      uint32_t bs = std::min<uint32_t>(e->big_slots, nc);
      pe_calib_kernel<<<(bs + kBlock - 1) / kBlock, kBlock>>>(
          v, e->big_layout, e->d_big_arena, bs, nc, maxd, e->cp, d_acts, d_na, d_hw);
      e->launches += 1;
      ok = cuda_ok(cudaGetLastError(), err, "calibration launch") &&
           cuda_ok(cudaMemcpy(hw, d_hw, sizeof(hw), cudaMemcpyDeviceToHost), err,
                   "calibration");
    }
    for (void* q : {(void*)d_hw, (void*)d_acts, (void*)d_na})
      if (q) cudaFree(q);
    if (!ok) {
      pe_engine_destroy(e);
      return PE_ERR_CUDA;
    }
    auto grow = [](int64_t x, int64_t pad) { return (int32_t)(x + x * 3 / 10 + pad); };
    pe::Caps c = e->layout.caps;
    const int32_t base_slots = v.A + v.N;
    c.V = std::min(c.V, base_slots + grow(std::max(0, hw[0] - base_slots), 128));
    c.L = std::min(c.L, grow(hw[1], 64));
    c.FS = std::min(c.FS, grow(hw[2], 16));
    c.EM = std::min(c.EM, grow(hw[3], 128));
    c.EO = std::min(c.EO, grow(hw[4], 128));
    e->layout = pe::relayout(v, c, false);
    fit_groups = (budget - big_groups * e->big_layout.bytes) /
                 std::max<uint64_t>(e->layout.bytes, 1);
  }
  uint64_t groups = std::max<uint64_t>(1, std::min(want / lanes, fit_groups));
  e->slots = (uint32_t)(groups * lanes);
  if (!cuda_ok(cudaMalloc(&e->d_arena, (size_t)groups * e->layout.bytes), err,
               "cudaMalloc(arena)") ||
      !cuda_ok(cudaMemset(e->d_arena, 0, (size_t)groups * e->layout.bytes), err, "zero arena")) {
    pe_engine_destroy(e);
    return PE_ERR_CUDA;
  }
  // replicated plan's peak (reward baseline)
  {
    uint32_t off[2] = {0, 0};
    pe_result r;
    e->baseline = 1;
    pe_status st = pe_eval_batch(e, nullptr, off, 1, &r, nullptr, 0, PE_SYNC, nullptr, err);
    if (st != PE_OK) {
      pe_engine_destroy(e);
      return st;
    }
    if (r.status != PE_CAND_OK) {
      set_err(err, PE_ERR_INTERNAL, "replicated plan failed to lower");
      pe_engine_destroy(e);
      return PE_ERR_INTERNAL;
    }
    e->baseline = std::max<int64_t>(1, r.peak_bytes);
  }
  *out = e;
  if (err) err->code = PE_OK;
  return PE_OK;
}

void pe_engine_destroy(pe_engine* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  if (e->l2_persist) {
    cudaCtxResetPersistingL2Cache();
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, e->l2_prev_limit);
    cudaGetLastError();
  }
  if (e->d_graph) cudaFree(e->d_graph);
  if (e->d_arena) cudaFree(e->d_arena);
  if (e->d_big_arena) cudaFree(e->d_big_arena);
  if (e->d_ctr) cudaFree(e->d_ctr);
  for (void* q : {(void*)e->d_tnode, (void*)e->d_tchild, (void*)e->d_tmiss, (void*)e->d_keys,
                  (void*)e->d_perm, (void*)e->d_hist, (void*)e->d_tpath, (void*)e->d_snap})
    if (q) cudaFree(q);
  if (e->d_io) cudaFree(e->d_io);
  if (e->d_pc) cudaFree(e->d_pc);
  if (e->d_cv) cudaFree(e->d_cv);
  if (e->done) cudaEventDestroy(e->done);
  for (cudaEvent_t k : e->kev) cudaEventDestroy(k);
  for (cudaEvent_t k : e->kev_free) cudaEventDestroy(k);
  delete e;
}

uint32_t pe_engine_num_ordinals(const pe_engine* e) { return e->n_ordinals; }
uint32_t pe_engine_legal_words(const pe_engine* e) { return (e->n_ordinals + 63) / 64; }
int64_t pe_engine_baseline_bytes(const pe_engine* e) { return e->baseline; }
int64_t pe_engine_arena_bytes(const pe_engine* e) {
  return (int64_t)(e->layout.bytes / pe::kLanes);  // per candidate
}
void pe_engine_set_kernel_timing(pe_engine* e, int32_t on) { e->ktiming = on != 0; }

uint32_t pe_engine_kernel_times(pe_engine* e, float* ms, uint32_t cap) {
  uint32_t n = 0;
  for (size_t k = 0; k + 1 < e->kev.size(); k += 2) {
    float t = 0;
    cudaEventSynchronize(e->kev[k + 1]);
    if (cudaEventElapsedTime(&t, e->kev[k], e->kev[k + 1]) != cudaSuccess) t = -1;
    if (ms && n < cap) ms[n] = t;
    ++n;
  }
  e->kev_free.insert(e->kev_free.end(), e->kev.begin(), e->kev.end());
  e->kev.clear();
  return n;
}

void pe_engine_arena_caps(const pe_engine* e, int32_t* caps5) {
  const pe::Caps& c = e->layout.caps;
  int32_t v[5] = {c.V, c.L, c.FS, c.EM, c.EO};
  for (int k = 0; k < 5; ++k) caps5[k] = v[k];
}
uint32_t pe_engine_slots(const pe_engine* e) { return e->slots; }
uint64_t pe_engine_launch_count(const pe_engine* e) { return e->launches; }
int64_t pe_engine_sched_nodes(const pe_engine* e) { return (int64_t)e->t_nl.size(); }

pe_status pe_engine_set_state_reuse(pe_engine* e, double budget_gb) {
  if (!e || budget_gb < 0) return PE_ERR_INVALID_ARGUMENT;
  if (e->d_snap) return e->snap_budget_gb == budget_gb ? PE_OK : PE_ERR_INVALID_ARGUMENT;
  e->snap_budget_gb = budget_gb;
  return PE_OK;
}
int64_t pe_engine_graph_bytes(const pe_engine* e) { return e->graph_bytes; }

pe_status pe_engine_ordinal_action(const pe_engine* e, uint32_t ord, pe_action* out) {
  if (!out || ord >= e->n_ordinals) return PE_ERR_INVALID_ARGUMENT;
  const pe::Worklist& w = e->wl;
  if (w.infer_rest && (int32_t)ord == w.n_ordinals()) {  // InferRest follows the TileValues
    *out = pe_action{0, 0, 0, PE_ACT_INFER_REST, 0};
    return PE_OK;
  }
  uint32_t na = (uint32_t)w.auto_axes.size();
  uint32_t ai = ord % na, d = (ord / na) % pe::kMaxRank, ent = ord / na / pe::kMaxRank;
  out->axis = (uint8_t)w.auto_axes[ai];
  out->dim = (uint8_t)d;
  out->pad = 0;
  if ((int32_t)ent >= w.n_entries()) {  // resurfaced stuck op: TileValue(op result)
    out->kind = PE_ACT_TILE;
    out->value = (uint32_t)(e->graph->g.args.size() + (ent - (uint32_t)w.n_entries()));
    return PE_OK;
  }
  out->kind = w.groups ? PE_ACT_TILE_GROUP : PE_ACT_TILE;
  out->value = (uint32_t)w.ent_val[ent];
  return PE_OK;
}

pe_status pe_infer_rest(pe_engine* e, const pe_action* prefix, uint32_t n_prefix, pe_action* out,
                        uint32_t cap, uint32_t* n_out, pe_error* err) {
  if (!e || (!prefix && n_prefix) || !out || !n_out) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null argument");
    return PE_ERR_INVALID_ARGUMENT;
  }
  std::vector<pe_action> cur(prefix, prefix + n_prefix);
  std::vector<std::vector<pe_action>*> one{&cur};
  if (!cuda_ok(cudaSetDevice(e->device), err, "cudaSetDevice") ||
      !ir_expand_batch(e, one, nullptr, err))
    return PE_ERR_CUDA;
  *n_out = (uint32_t)cur.size();
  if (cur.size() > cap) {
    set_err(err, PE_ERR_CAPACITY, "output buffer too small");
    return PE_ERR_CAPACITY;
  }
  std::copy(cur.begin(), cur.end(), out);
  return PE_OK;
}

pe_status pe_eval_batch(pe_engine* e, const pe_action* acts, const uint32_t* seq_off,
                        uint32_t n, pe_result* out, int32_t* trace, uint32_t trace_words,
                        uint32_t flags, void* stream, pe_error* err) {
  if (!e || !seq_off || !out) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null argument");
    return PE_ERR_INVALID_ARGUMENT;
  }
  if (!(flags & PE_MEM_DEVICE) && n > 0) {
    // Unexpanded INFER_REST decisions: expanded left to right, every
    // candidate's next one in the same batched expansion (ir_expand_batch).
    bool any = false;
    for (uint32_t k = 0; k < seq_off[n] && !any; ++k)
      any = acts[k].kind == PE_ACT_INFER_REST && !(acts[k].pad & PE_ACT_FLAG_EXPANDED);
    if (any) {
      if (!cuda_ok(cudaSetDevice(e->device), err, "cudaSetDevice")) return PE_ERR_CUDA;
      std::vector<std::vector<pe_action>> cur(n);
      std::vector<std::vector<int32_t>> orig(n);  // expanded index -> caller's index
      std::vector<uint32_t> pos(n);
      for (uint32_t c = 0; c < n; ++c) pos[c] = seq_off[c];
      for (;;) {
        std::vector<std::vector<pe_action>*> jobs;
        std::vector<uint32_t> who;
        for (uint32_t c = 0; c < n; ++c) {
          while (pos[c] < seq_off[c + 1]) {
            const pe_action& a = acts[pos[c]++];
            if (a.kind == PE_ACT_INFER_REST && !(a.pad & PE_ACT_FLAG_EXPANDED)) {
              jobs.push_back(&cur[c]);
              who.push_back(c);
              break;
            }
            cur[c].push_back(a);
            orig[c].push_back((int32_t)(pos[c] - 1 - seq_off[c]));
          }
        }
        if (jobs.empty()) break;
        std::vector<size_t> before(jobs.size());
        for (size_t j = 0; j < jobs.size(); ++j) before[j] = jobs[j]->size();
        if (!ir_expand_batch(e, jobs, (cudaStream_t)stream, err)) return PE_ERR_CUDA;
        for (size_t j = 0; j < jobs.size(); ++j)
          orig[who[j]].resize(jobs[j]->size(), (int32_t)(pos[who[j]] - 1 - seq_off[who[j]]));
      }
      std::vector<pe_action> flat;
      std::vector<uint32_t> off{0};
      for (uint32_t c = 0; c < n; ++c) {
        flat.insert(flat.end(), cur[c].begin(), cur[c].end());
        off.push_back((uint32_t)flat.size());
      }
      pe_status st = pe_eval_batch_ex(e, flat.data(), off.data(), n, out, trace, trace_words,
                                      nullptr, flags, stream, err);
      // an illegal action is named by its index in the caller's sequence
      for (uint32_t c = 0; st == PE_OK && c < n; ++c)
        if (out[c].status == PE_CAND_ILLEGAL && out[c].fail_step >= 0 &&
            out[c].fail_step < (int32_t)orig[c].size())
          out[c].fail_step = orig[c][out[c].fail_step];
      return st;
    }
  }
  return pe_eval_batch_ex(e, acts, seq_off, n, out, trace, trace_words, nullptr, flags, stream,
                          err);
}

pe_status pe_eval_batch_ex(pe_engine* e, const pe_action* acts, const uint32_t* seq_off,
                           uint32_t n, pe_result* out, int32_t* trace, uint32_t trace_words,
                           uint8_t* argflags, uint32_t flags, void* stream, pe_error* err) {
  NvtxRange nvtx_("pe_eval_batch");
  if (!e || !seq_off || !out) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null argument");
    return PE_ERR_INVALID_ARGUMENT;
  }
  if (n == 0) return PE_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (!cuda_ok(cudaSetDevice(e->device), err, "cudaSetDevice")) return PE_ERR_CUDA;
  if (!call_begin(e, st, err)) return PE_ERR_CUDA;
  const int32_t A = (int32_t)e->graph->g.args.size();
  const pe_action* d_acts = acts;
  const uint32_t* d_off = seq_off;
  pe_result* d_out = out;
  int32_t* d_trace = trace;
  uint8_t* d_flags = argflags;
  if (!(flags & PE_MEM_DEVICE)) {
    uint32_t n_acts = seq_off[n];
    size_t b_acts = ((size_t)n_acts * sizeof(pe_action) + 255) & ~size_t(255);
    size_t b_off = ((size_t)(n + 1) * 4 + 255) & ~size_t(255);
    size_t b_out = ((size_t)n * sizeof(pe_result) + 255) & ~size_t(255);
    size_t b_tr = trace ? (((size_t)n * trace_words * 4 + 255) & ~size_t(255)) : 0;
    size_t b_fl = argflags ? (size_t)n * A : 0;
    if (!ensure_io(e, b_acts + b_off + b_out + b_tr + b_fl + 256, err)) return PE_ERR_CUDA;
    uint8_t* p = e->d_io;
    d_acts = (const pe_action*)p;
    d_off = (const uint32_t*)(p + b_acts);
    d_out = (pe_result*)(p + b_acts + b_off);
    d_trace = trace ? (int32_t*)(p + b_acts + b_off + b_out) : nullptr;
    d_flags = argflags ? (p + b_acts + b_off + b_out + b_tr) : nullptr;
    if (n_acts && !cuda_ok(cudaMemcpyAsync((void*)d_acts, acts, (size_t)n_acts * sizeof(pe_action),
                                           cudaMemcpyHostToDevice, st), err, "H2D acts"))
      return PE_ERR_CUDA;
    if (!cuda_ok(cudaMemcpyAsync((void*)d_off, seq_off, (size_t)(n + 1) * 4,
                                 cudaMemcpyHostToDevice, st), err, "H2D offsets"))
      return PE_ERR_CUDA;
  }
  uint32_t slots = launch_slots(e, n);
  if (!cuda_ok(cudaMemsetAsync(e->d_ctr, 0, sizeof(uint32_t), st), err, "reset work counter"))
    return PE_ERR_CUDA;
  // parity traces need the SPMD operand log, which only the full-size
  // arenas keep: traced batches run there (the main pass has nothing to do)
  const bool full = d_trace != nullptr && trace_words > 0;
  uint32_t ms = full ? std::min<uint32_t>(e->big_slots, n) : slots;
  const uint32_t tps = threads_per_slot(e, ms);
  pe_eval_kernel<false><<<(ms * tps + e->small_block - 1) / e->small_block, e->small_block, 0,
                          st>>>(
      e->dview, full ? e->big_layout : e->layout, full ? e->d_big_arena : e->d_arena, ms, d_acts,
      d_off, n, e->cp, e->baseline, d_out, d_trace, trace_words, d_flags, e->d_ctr, tps);
  uint32_t bs = std::min<uint32_t>(e->big_slots, n);
  pe_eval_kernel<true><<<(bs + e->small_block - 1) / e->small_block, e->small_block, 0, st>>>(
      e->dview, e->big_layout, e->d_big_arena, bs, d_acts, d_off, n, e->cp, e->baseline, d_out,
      d_trace, trace_words, d_flags, nullptr, 1u);
  e->launches += 2;
  if (!cuda_ok(cudaGetLastError(), err, "pe_eval_kernel launch")) return PE_ERR_CUDA;
  if (!(flags & PE_MEM_DEVICE)) {
    if (!cuda_ok(cudaMemcpyAsync(out, d_out, (size_t)n * sizeof(pe_result),
                                 cudaMemcpyDeviceToHost, st), err, "D2H results"))
      return PE_ERR_CUDA;
    if (argflags && !cuda_ok(cudaMemcpyAsync(argflags, d_flags, (size_t)n * A,
                                             cudaMemcpyDeviceToHost, st), err, "D2H flags"))
      return PE_ERR_CUDA;
    if (trace && !cuda_ok(cudaMemcpyAsync(trace, d_trace, (size_t)n * trace_words * 4,
                                          cudaMemcpyDeviceToHost, st), err, "D2H trace"))
      return PE_ERR_CUDA;
    if (!call_end(e, st, err)) return PE_ERR_CUDA;
    if (!cuda_ok(cudaStreamSynchronize(st), err, "sync")) return PE_ERR_CUDA;
  } else if (!call_end(e, st, err)) {
    return PE_ERR_CUDA;
  } else if (flags & PE_SYNC) {
    if (!cuda_ok(cudaStreamSynchronize(st), err, "sync")) return PE_ERR_CUDA;
  }
  return PE_OK;
}

}  // extern "C"

// ---- prefix-trie scheduling, host side ----
namespace {


// Legal TileValue ordinals (ascending: the rollout's enumeration order
// without resurfacing) after each prefix: one rollout launch whose legal
// output is taken right after the prefix.  Own buffers: the caller's inputs
// may live in the staging buffer.
// snap_idx: per prefix the snapshot slot to save into, or -1; on return -1
// where no snapshot was written (the probe overflowed its tight arena).
bool sched_probe(pe_engine* e, const std::vector<std::vector<pe_action>>& prefixes,
                 std::vector<int32_t>& snap_idx, std::vector<std::vector<int32_t>>& legal,
                 std::vector<int32_t>& status, cudaStream_t st, pe_error* err) {
  uint32_t n = (uint32_t)prefixes.size();
  std::vector<pe_action> acts;
  std::vector<uint32_t> off{0};
  int32_t maxlen = 0;
  for (const auto& pr : prefixes) {
    acts.insert(acts.end(), pr.begin(), pr.end());
    off.push_back((uint32_t)acts.size());
    maxlen = std::max(maxlen, (int32_t)pr.size());
  }
  int32_t maxd = std::max(1, maxlen);
  int32_t lw = (int32_t)pe_engine_legal_words(e);
  size_t b_acts = std::max<size_t>(1, acts.size()) * sizeof(pe_action);
  size_t sizes[8] = {b_acts, (n + 1) * 4ull, n * 8ull, (size_t)n * maxd * sizeof(pe_action),
                     n * 4ull, n * sizeof(pe_result), (size_t)n * lw * 8, n * 4ull};
  void* buf[8] = {};
  bool ok = true;
  for (int k = 0; k < 8 && ok; ++k) ok = cuda_ok(cudaMalloc(&buf[k], sizes[k]), err, "cudaMalloc(probe)");
  std::vector<uint64_t> lg((size_t)n * lw);
  std::vector<pe_result> res(n);
  if (ok)
    ok = cuda_ok(cudaMemcpyAsync(buf[7], snap_idx.data(), n * 4ull, cudaMemcpyHostToDevice, st),
                 err, "H2D probe");
  if (ok) {
    ok = (acts.empty() || cuda_ok(cudaMemcpyAsync(buf[0], acts.data(), acts.size() * sizeof(pe_action),
                                                  cudaMemcpyHostToDevice, st), err, "H2D probe")) &&
         cuda_ok(cudaMemcpyAsync(buf[1], off.data(), off.size() * 4, cudaMemcpyHostToDevice, st),
                 err, "H2D probe") &&
         cuda_ok(cudaMemsetAsync(buf[2], 0, sizes[2], st), err, "probe seeds") &&
         cuda_ok(cudaMemsetAsync(e->d_ctr + 2, 0, 4, st), err, "probe counter");
  }
  if (ok) {
    uint32_t slots = launch_slots(e, n), bs = std::min<uint32_t>(e->big_slots, n);
    pe_probe_kernel<<<(slots + kBlock - 1) / kBlock, kBlock, 0, st>>>(
        e->dview, e->layout, e->d_arena, slots, (const pe_action*)buf[0], (const uint32_t*)buf[1],
        n, maxd, e->cp, e->baseline, (pe_action*)buf[3], (uint32_t*)buf[4], (pe_result*)buf[5],
        (uint64_t*)buf[6], lw, e->d_snap, e->snap_stride, (int32_t*)buf[7]);
    // overflowed probes: legal sets from full-size arenas (no snapshot); the
    // uniform maxd only adds draws after the prefix, its legal set is final
    pe_rollout_kernel<true, false, 0><<<(bs + kBlock - 1) / kBlock, kBlock, 0, st>>>(
        e->dview, e->big_layout, e->d_big_arena, bs, (const pe_action*)buf[0],
        (const uint32_t*)buf[1], (const uint64_t*)buf[2], n, maxd, e->cp, e->baseline,
        (pe_action*)buf[3], (uint32_t*)buf[4], (pe_result*)buf[5], (uint64_t*)buf[6], lw,
        nullptr, nullptr, SchedView(), CacheView(), 1u, nullptr);
    e->launches += 2;
    ok = cuda_ok(cudaGetLastError(), err, "probe launch") &&
         cuda_ok(cudaMemcpyAsync(lg.data(), buf[6], sizes[6], cudaMemcpyDeviceToHost, st), err,
                 "D2H probe") &&
         cuda_ok(cudaMemcpyAsync(res.data(), buf[5], sizes[5], cudaMemcpyDeviceToHost, st), err,
                 "D2H probe") &&
         cuda_ok(cudaMemcpyAsync(snap_idx.data(), buf[7], n * 4ull, cudaMemcpyDeviceToHost, st),
                 err, "D2H probe") &&
         cuda_ok(cudaStreamSynchronize(st), err, "probe sync");
  }
  for (int k = 0; k < 8; ++k)
    if (buf[k]) cudaFree(buf[k]);
  if (!ok) return false;
  status.assign(n, 0);
  for (uint32_t i = 0; i < n; ++i) status[i] = res[i].status;
  legal.assign(n, {});
  for (uint32_t i = 0; i < n; ++i)
    for (int32_t o = 0; o < (int32_t)e->n_ordinals; ++o)
      if ((lg[(size_t)i * lw + o / 64] >> (o % 64)) & 1ull) legal[i].push_back(o);
  e->sched_probes += n;
  return true;
}

int32_t sched_add_node(pe_engine* e, int32_t parent, int32_t pick,
                       const std::vector<int32_t>& legal) {
  int32_t id = (int32_t)e->t_nl.size();
  e->t_nl.push_back((int32_t)legal.size());
  e->t_legal_off.push_back((int32_t)e->t_legal.size());
  e->t_legal.insert(e->t_legal.end(), legal.begin(), legal.end());
  e->t_child_off.push_back((int32_t)e->t_child.size());
  e->t_child.insert(e->t_child.end(), legal.size(), -1);
  e->t_depth.push_back(parent < 0 ? 0 : e->t_depth[parent] + 1);
  e->t_parent.push_back(parent);
  e->t_pick.push_back(pick);
  e->t_snap.push_back(-1);
  e->t_path.resize((size_t)(id + 1) * e->path_cap, pe_action{0, 0, 0, PE_ACT_STOP, 0});
  if (parent >= 0) {
    e->t_child[e->t_child_off[parent] + pick] = id;
    for (int32_t k = 0; k < e->path_cap; ++k)
      e->t_path[(size_t)id * e->path_cap + k] = e->t_path[(size_t)parent * e->path_cap + k];
    int32_t d = e->t_depth[id];
    if (d <= e->path_cap)
      pe_engine_ordinal_action(e, (uint32_t)e->t_legal[e->t_legal_off[parent] + pick],
                               &e->t_path[(size_t)id * e->path_cap + d - 1]);
  }
  e->t_dirty = true;
  return id;
}

// decision path from the root to `node`
std::vector<pe_action> sched_path(pe_engine* e, int32_t node) {
  std::vector<pe_action> path;
  for (int32_t v = node; e->t_parent[v] >= 0; v = e->t_parent[v]) {
    int32_t par = e->t_parent[v];
    pe_action a;
    pe_engine_ordinal_action(e, (uint32_t)e->t_legal[e->t_legal_off[par] + e->t_pick[v]], &a);
    path.push_back(a);
  }
  std::reverse(path.begin(), path.end());
  return path;
}

template <typename T>
bool ensure_dev(T*& p, size_t& cap, size_t need, pe_error* err, const char* what) {
  if (need <= cap) return true;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  size_t c = std::max<size_t>(need, 1024);
  if (!cuda_ok(cudaMalloc(&p, c * sizeof(T)), err, what)) return false;
  cap = c;
  return true;
}

bool sched_upload(pe_engine* e, cudaStream_t st, pe_error* err) {
  if (!e->t_dirty) return true;
  size_t nodes = e->t_nl.size(), nch = std::max<size_t>(1, e->t_child.size());
  size_t tcap = e->tchild_cap;
  if (!ensure_dev(e->d_tnode, e->tnode_cap, nodes * 4, err, "cudaMalloc(trie)") ||
      !ensure_dev(e->d_tchild, e->tchild_cap, nch, err, "cudaMalloc(trie)"))
    return false;
  if (e->tchild_cap != tcap || !e->d_tmiss) {
    if (e->d_tmiss) cudaFree(e->d_tmiss);
    e->d_tmiss = nullptr;
    if (!cuda_ok(cudaMalloc(&e->d_tmiss, e->tchild_cap * 4), err, "cudaMalloc(trie)")) return false;
  }
  std::vector<int32_t> tn(nodes * 4, 0);
  for (size_t v = 0; v < nodes; ++v) {
    tn[4 * v] = e->t_nl[v];
    tn[4 * v + 1] = e->t_child_off[v];
    tn[4 * v + 2] = e->t_depth[v];
    tn[4 * v + 3] = e->t_snap[v];
  }
  if (!ensure_dev(e->d_tpath, e->tpath_cap, std::max<size_t>(1, e->t_path.size()), err,
                  "cudaMalloc(trie)") ||
      (!e->t_path.empty() &&
       !cuda_ok(cudaMemcpyAsync(e->d_tpath, e->t_path.data(), e->t_path.size() * sizeof(pe_action),
                                cudaMemcpyHostToDevice, st), err, "H2D trie")))
    return false;
  if (!cuda_ok(cudaMemcpyAsync(e->d_tnode, tn.data(), tn.size() * 4, cudaMemcpyHostToDevice, st),
               err, "H2D trie") ||
      (!e->t_child.empty() &&
       !cuda_ok(cudaMemcpyAsync(e->d_tchild, e->t_child.data(), e->t_child.size() * 4,
                                cudaMemcpyHostToDevice, st), err, "H2D trie")) ||
      !cuda_ok(cudaMemsetAsync(e->d_tmiss, 0, e->tchild_cap * 4, st), err, "trie misses"))
    return false;
  // (tn / t_child are read by the copies before this function returns)
  if (!cuda_ok(cudaStreamSynchronize(st), err, "trie sync")) return false;
  e->t_dirty = false;
  return true;
}

// Candidate order for a batch of root rollouts: grouped by the deepest trie
// node their first decisions reach.  Probes at most one new level per call
// (the prefix states the batch reached but the trie lacks).  Returns the
// device permutation, or nullptr (identity) when scheduling is off.
bool sched_perm(pe_engine* e, uint32_t n, const uint64_t* d_seeds, int32_t maxd,
                cudaStream_t st, const uint32_t** perm, SchedView* sv, pe_error* err) {
  NvtxRange nvtx_("sched_perm");
  *perm = nullptr;
  *sv = SchedView();
  int32_t depth = std::min(e->sched_depth, maxd);
  if (depth <= 0) return true;
  if (!e->d_snap && e->snap_budget_gb > 0) {
    // snapshot pool for prefix-state reuse: one slot per trie node while the
    // budget lasts (nodes without one fall back to the full computation)
    e->snap_stride = (pe::Cand::snap_bytes(e->dview, e->layout.caps) + 255) & ~uint64_t(255);
    uint64_t cap = (uint64_t)(e->snap_budget_gb * (double)(1ull << 30)) / e->snap_stride;
    e->snap_cap = (int32_t)std::min<uint64_t>(cap, (uint64_t)e->sched_max_nodes);
    if (e->snap_cap > 0 &&
        !cuda_ok(cudaMalloc(&e->d_snap, (size_t)e->snap_cap * e->snap_stride), err,
                 "cudaMalloc(snapshots)"))
      return false;
  }
  if (e->t_nl.empty()) {
    std::vector<std::vector<int32_t>> lg;
    std::vector<int32_t> stat, none{-1};
    if (!sched_probe(e, {{}}, none, lg, stat, st, err)) return false;  // root: init() state
    sched_add_node(e, -1, 0, lg[0]);
  }
  if (!ensure_dev(e->d_keys, e->sched_cap, n, err, "cudaMalloc(sched)") ||
      !ensure_dev(e->d_perm, e->perm_cap, n, err, "cudaMalloc(sched)"))
    return false;
  uint32_t m = 0, kstride = 1;
  for (int round = 0; round < 2; ++round) {
    if (!sched_upload(e, st, err)) return false;
    int32_t max_nl = 0;
    for (int32_t x : e->t_nl) max_nl = std::max(max_nl, x);
    kstride = (uint32_t)max_nl + 2;
    m = kstride * (uint32_t)e->t_nl.size();
    if (!ensure_dev(e->d_hist, e->hist_cap, m, err, "cudaMalloc(sched)") ||
        !cuda_ok(cudaMemsetAsync(e->d_hist, 0, (size_t)m * 4, st), err, "sched hist") ||
        !cuda_ok(cudaMemsetAsync(e->d_tmiss, 0, std::max<size_t>(1, e->t_child.size()) * 4, st),
                 err, "sched misses") ||
        !cuda_ok(cudaMemsetAsync(e->d_ctr + 3, 0, 4, st), err, "sched misses"))
      return false;
    pe_sched_key_kernel<<<(n + 255) / 256, 256, 0, st>>>(
        n, d_seeds, depth, maxd, kstride, (const int4*)e->d_tnode, e->d_tchild, e->d_tmiss,
        e->d_ctr + 3, e->d_keys, e->d_hist);
    e->launches += 1;
    if (!cuda_ok(cudaGetLastError(), err, "sched key launch")) return false;
    if (round == 1 || (int32_t)e->t_nl.size() >= e->sched_max_nodes) break;
    uint32_t nmiss = 0;
    if (!cuda_ok(cudaMemcpyAsync(&nmiss, e->d_ctr + 3, 4, cudaMemcpyDeviceToHost, st), err,
                 "D2H misses") ||
        !cuda_ok(cudaStreamSynchronize(st), err, "sched sync"))
      return false;
    // a probe launch costs about one candidate's latency: only worth it when
    // a noticeable share of the batch would group deeper
    if ((uint64_t)nmiss * 64 < n) break;
    std::vector<uint32_t> miss(e->t_child.size());
    if (!cuda_ok(cudaMemcpyAsync(miss.data(), e->d_tmiss, miss.size() * 4, cudaMemcpyDeviceToHost,
                                 st), err, "D2H misses") ||
        !cuda_ok(cudaStreamSynchronize(st), err, "sched sync"))
      return false;
    std::vector<std::pair<int32_t, int32_t>> want;  // (parent, pick)
    for (int32_t v = 0; v < (int32_t)e->t_nl.size(); ++v)
      for (int32_t k = 0; k < e->t_nl[v]; ++k)
        if (miss[e->t_child_off[v] + k] && e->t_child[e->t_child_off[v] + k] < 0)
          want.push_back({v, k});
    // deeper nodes only pay when they group enough candidates per warp:
    // skip a level whose new nodes would average fewer than 8 (e.g. an
    // ungrouped worklist with hundreds of root actions)
    if ((uint64_t)nmiss < 8ull * want.size()) break;
    if (want.size() + e->t_nl.size() > (size_t)e->sched_max_nodes)
      want.resize((size_t)e->sched_max_nodes - e->t_nl.size());
    std::vector<std::vector<pe_action>> prefixes;
    for (auto [v, k] : want) {
      std::vector<pe_action> pth = sched_path(e, v);
      pe_action a;
      pe_engine_ordinal_action(e, (uint32_t)e->t_legal[e->t_legal_off[v] + k], &a);
      pth.push_back(a);
      prefixes.push_back(std::move(pth));
    }
    std::vector<int32_t> sidx(want.size(), -1), stat;
    for (size_t q = 0; q < want.size() && e->snap_used < e->snap_cap; ++q) sidx[q] = e->snap_used++;
    std::vector<std::vector<int32_t>> lg;
    if (!sched_probe(e, prefixes, sidx, lg, stat, st, err)) return false;
    for (size_t q = 0; q < want.size(); ++q) {
      int32_t id = sched_add_node(e, want[q].first, want[q].second, lg[q]);
      e->t_snap[id] = sidx[q];  // -1 unless the probe wrote the snapshot
    }
  }
  pe_sched_scan_kernel<<<1, 1024, 0, st>>>(e->d_hist, m);
  pe_sched_scatter_kernel<<<(n + 255) / 256, 256, 0, st>>>(n, e->d_keys, e->d_hist, e->d_perm);
  e->launches += 2;
  if (!cuda_ok(cudaGetLastError(), err, "sched sort launch")) return false;
  *perm = e->d_perm;
  sv->keys = e->d_keys;
  sv->tnode = (const int4*)e->d_tnode;
  sv->tpath = e->d_tpath;
  sv->path_cap = e->path_cap;
  sv->snap = e->d_snap;
  sv->stride = e->snap_stride;
  sv->kstride = kstride;
  return true;
}

// Main + retry rollout launches over one batch (the caller has set up the
// schedule).  `gv` is the engine's graph view, possibly with ir_pause set.
cudaError_t enqueue_rollouts(pe_engine* e, const pe::GraphView& gv, const pe_action* d_prefix,
                             const uint32_t* d_poff, const uint64_t* d_seeds, uint32_t n,
                             pe_action* d_acts, uint32_t* d_nacts, pe_result* d_out,
                             uint64_t* d_legal, const uint32_t* perm, const SchedView& sv,
                             const CacheView& cv, uint32_t* max_acts, cudaStream_t st) {
  int32_t maxd = (int32_t)e->cfg.max_decisions;
  int32_t lw = (int32_t)pe_engine_legal_words(e);
  uint32_t slots = launch_slots(e, n);
  cudaError_t ce = cudaMemsetAsync(e->d_ctr + 1, 0, sizeof(uint32_t), st);
  if (ce != cudaSuccess) return ce;
  uint32_t bs = std::min<uint32_t>(e->big_slots, n);
  const uint32_t tps = threads_per_slot(e, slots);
  uint32_t threads = slots * tps;
  // a launch with fewer slots than the resident threads (small batches: MCTS
  // leaf batches, config 4's arena-limited slots) runs one-warp blocks, so
  // the block scheduler spreads its warps over every SM (128-thread blocks
  // left SMs idle: 8,192 candidates = 64 blocks on 148 SMs)
  uint32_t blk = threads % PE_SM_THREADS == 0 && threads >= (uint32_t)e->sm_count * PE_SM_THREADS
                     ? PE_SM_THREADS : e->small_block;
  uint32_t grid = (threads + blk - 1) / blk;
  uint32_t bgrid = (bs * kThreadsPerSlot + e->small_block - 1) / e->small_block;
  // (the stuck-resurfacing instantiation only when the worklist uses it)
  auto launch = [&](auto main_k, auto retry_k) {
    // (experiment PE_L2_PERSIST: the graph image as a persisting L2 window)
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeAccessPolicyWindow;
    at[0].val.accessPolicyWindow.base_ptr = e->d_graph;
    at[0].val.accessPolicyWindow.num_bytes = e->l2_window;
    at[0].val.accessPolicyWindow.hitRatio = 1.0f;
    at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(blk);
    lc.stream = st;
    lc.attrs = at;
    lc.numAttrs = e->l2_persist ? 1 : 0;
    cudaEvent_t k0 = nullptr, k1 = nullptr;
    if (e->ktiming) {
      for (cudaEvent_t* k : {&k0, &k1}) {
        if (!e->kev_free.empty()) {
          *k = e->kev_free.back();
          e->kev_free.pop_back();
        } else if (cudaEventCreate(k) != cudaSuccess) {
          *k = nullptr;
        }
      }
      if (k0 && k1) cudaEventRecord(k0, st);
    }
    cudaError_t le = cudaLaunchKernelEx(&lc, main_k, gv, e->layout, e->d_arena, slots, d_prefix,
                                        d_poff, d_seeds, n, maxd, e->cp, e->baseline, d_acts,
                                        d_nacts, d_out, d_legal, lw, e->d_ctr + 1, perm, sv,
                                        cv, tps, max_acts);
    if (e->ktiming && k0 && k1) {
      cudaEventRecord(k1, st);
      e->kev.push_back(k0);
      e->kev.push_back(k1);
    }
    // the retry launch reads the statuses the main launch writes: never
    // queue it behind a main launch that failed to start
    if (le != cudaSuccess) return le;
    retry_k<<<bgrid, e->small_block, 0, st>>>(gv, e->big_layout, e->d_big_arena, bs, d_prefix, d_poff,
                                      d_seeds, n, maxd, e->cp, e->baseline, d_acts, d_nacts,
                                      d_out, d_legal, lw, nullptr, nullptr, SchedView(),
                                      CacheView(), 1u, max_acts);
    return cudaGetLastError();
  };
  // the instantiation with only the features this launch needs (the
  // default -- root rollouts, no InferRest, no saved states -- has none);
  // resurfacing engines never use saved states
  const bool ir = gv.ir_ord >= 0 || gv.ir_pause;
  const bool res = (sv.keys && sv.snap) || cv.from;
  // one candidate per warp: the whole warp runs it (kFCoop)
  const bool coop = tps == 32 && e->coop && !ir && !e->wl.resurface;
  cudaError_t lerr;
  if (coop)
    lerr = res ? launch(pe_rollout_kernel<false, false, pe::kFCoop | pe::kFResume>,
                        pe_rollout_kernel<true, false, 0>)
               : launch(pe_rollout_kernel<false, false, pe::kFCoop>,
                        pe_rollout_kernel<true, false, 0>);
  else if (e->wl.resurface)
    lerr = ir ? launch(pe_rollout_kernel<false, true, pe::kFInferRest>,
                       pe_rollout_kernel<true, true, pe::kFInferRest>)
              : launch(pe_rollout_kernel<false, true, 0>, pe_rollout_kernel<true, true, 0>);
  else if (ir && res)
    lerr = launch(pe_rollout_kernel<false, false, pe::kFAll>,
                  pe_rollout_kernel<true, false, pe::kFInferRest>);
  else if (ir)
    lerr = launch(pe_rollout_kernel<false, false, pe::kFInferRest>,
                  pe_rollout_kernel<true, false, pe::kFInferRest>);
  else if (res)
    lerr = launch(pe_rollout_kernel<false, false, pe::kFResume>, pe_rollout_kernel<true, false, 0>);
  else
    lerr = launch(pe_rollout_kernel<false, false, 0>, pe_rollout_kernel<true, false, 0>);
  e->launches += 2;
  return lerr;
}

// ---- InferRest as a batched composite action (pe.h infer_rest_action) ----
// REF infer_rest (propagate.cc:484-544) from a state given as an action
// sequence: for every untiled (not sliced), non-atomic argument in order,
// each (dim x auto axis) that divides is a trial = the sequence + that tile,
// propagated and lowered; a trial is consistent when it evaluates and adds
// no all_gather bytes over the current state.  The first argument with
// exactly one consistent trial takes it, and the rounds repeat until none
// does.  Here ALL trials of ALL sequences being expanded run as one batched
// evaluation per round (chunked by size), so a batch of paused rollouts
// costs one launch per inference round, not one per candidate.

// Host sequences evaluated on the device through the engine's own eval
// kernels (private buffers: the caller's staging buffer may be in use).
bool eval_seqs(pe_engine* e, const std::vector<pe_action>& acts, const std::vector<uint32_t>& off,
               std::vector<pe_result>& res, std::vector<uint8_t>* argflags, cudaStream_t st,
               pe_error* err) {
  uint32_t n = (uint32_t)off.size() - 1;
  res.resize(n);
  if (n == 0) return true;
  const size_t A = e->graph->g.args.size();
  size_t b_acts = std::max<size_t>(1, acts.size()) * sizeof(pe_action);
  size_t b_fl = argflags ? (size_t)n * A : 0;
  void *d_acts = nullptr, *d_off = nullptr, *d_out = nullptr, *d_fl = nullptr;
  bool ok = cuda_ok(cudaMalloc(&d_acts, b_acts), err, "cudaMalloc(ir)") &&
            cuda_ok(cudaMalloc(&d_off, off.size() * 4), err, "cudaMalloc(ir)") &&
            cuda_ok(cudaMalloc(&d_out, (size_t)n * sizeof(pe_result)), err, "cudaMalloc(ir)") &&
            (!argflags || cuda_ok(cudaMalloc(&d_fl, std::max<size_t>(1, b_fl)), err, "cudaMalloc(ir)"));
  ok = ok && (acts.empty() || cuda_ok(cudaMemcpyAsync(d_acts, acts.data(), acts.size() * sizeof(pe_action),
                                                      cudaMemcpyHostToDevice, st), err, "H2D ir")) &&
       cuda_ok(cudaMemcpyAsync(d_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice, st), err,
               "H2D ir");
  ok = ok && pe_eval_batch_ex(e, (const pe_action*)d_acts, (const uint32_t*)d_off, n,
                              (pe_result*)d_out, nullptr, 0, (uint8_t*)d_fl, PE_MEM_DEVICE, st,
                              err) == PE_OK;
  ok = ok && cuda_ok(cudaMemcpyAsync(res.data(), d_out, (size_t)n * sizeof(pe_result),
                                     cudaMemcpyDeviceToHost, st), err, "D2H ir");
  if (ok && argflags) {
    argflags->resize(b_fl);
    ok = cuda_ok(cudaMemcpyAsync(argflags->data(), d_fl, b_fl, cudaMemcpyDeviceToHost, st), err,
                 "D2H ir");
  }
  ok = ok && cuda_ok(cudaStreamSynchronize(st), err, "ir sync");
  for (void* q : {d_acts, d_off, d_out, d_fl})
    if (q) cudaFree(q);
  return ok;
}

int64_t ag_total(const pe_result& r) {
  int64_t s = 0;
  for (int x = 0; x < PE_MAX_AXES; ++x) s += r.ag_bytes[x];
  return s;
}

// Appends [INFER_REST marker (expanded)] + the inferred tiles to every
// sequence of `seqs` (each = the state InferRest is applied to).
bool ir_expand_batch(pe_engine* e, std::vector<std::vector<pe_action>*>& seqs, cudaStream_t st,
                     pe_error* err) {
  NvtxRange nvtx_("ir_expand_batch");
  const pe::HostGraph& g = e->graph->g;
  const int32_t A = (int32_t)g.args.size();
  const pe_action marker{0, 0, 0, PE_ACT_INFER_REST, PE_ACT_FLAG_EXPANDED};
  struct Job {
    std::vector<pe_action>* seq;
    int64_t base_ag;
    std::vector<uint8_t> flags;  // bit 0 sliced, bit 1 atomic (arg_is_tiled / arg_is_atomic)
  };
  std::vector<Job> live;
  {
    std::vector<pe_action> flat;
    std::vector<uint32_t> off{0};
    for (auto* s : seqs) {
      s->push_back(marker);
      flat.insert(flat.end(), s->begin(), s->end());
      off.push_back((uint32_t)flat.size());
    }
    std::vector<pe_result> res;
    std::vector<uint8_t> fl;
    if (!eval_seqs(e, flat, off, res, &fl, st, err)) return false;
    for (size_t j = 0; j < seqs.size(); ++j) {
      if (res[j].status != PE_CAND_OK) continue;  // the candidate reports its own status
      Job jb{seqs[j], ag_total(res[j]), std::vector<uint8_t>(fl.begin() + j * A, fl.begin() + (j + 1) * A)};
      bool any_tiled = false;
      for (int32_t a = 0; a < A; ++a) any_tiled |= (jb.flags[a] & 1) != 0;
      if (any_tiled) live.push_back(std::move(jb));  // nothing tiled: a no-op
    }
  }
  const size_t kMaxTrialActs = (size_t)1 << 23;  // actions per trial launch
  while (!live.empty()) {
    // every trial of every live job, in (job, argument, dim, axis) order
    struct Trial {
      uint32_t job;
      int32_t arg;
      pe_action tile;
    };
    std::vector<Trial> trials;
    for (uint32_t j = 0; j < live.size(); ++j)
      for (int32_t a = 0; a < A; ++a) {
        if (live[j].flags[a] & 3) continue;
        const auto& sh = g.args[a].shape;
        for (int32_t d = 0; d < (int32_t)sh.size(); ++d)
          for (int32_t ax : e->wl.auto_axes)
            if (sh[d] % g.axis_sizes[ax] == 0)
              trials.push_back({j, a, pe_action{(uint32_t)a, (uint8_t)d, (uint8_t)ax, PE_ACT_TILE,
                                                PE_ACT_FLAG_INFERRED}});
      }
    std::vector<pe_result> tres(trials.size());
    for (size_t t0 = 0; t0 < trials.size();) {
      std::vector<pe_action> flat;
      std::vector<uint32_t> off{0};
      size_t t1 = t0;
      while (t1 < trials.size() && (t1 == t0 || flat.size() < kMaxTrialActs)) {
        const auto& s = *live[trials[t1].job].seq;
        flat.insert(flat.end(), s.begin(), s.end());
        flat.push_back(trials[t1].tile);
        off.push_back((uint32_t)flat.size());
        ++t1;
      }
      std::vector<pe_result> r;
      if (!eval_seqs(e, flat, off, r, nullptr, st, err)) return false;
      std::copy(r.begin(), r.end(), tres.begin() + t0);
      t0 = t1;
    }
    // per job: the first argument with exactly one consistent trial
    std::vector<int32_t> pick(live.size(), -1);
    for (size_t t = 0; t < trials.size();) {
      size_t u = t;
      int32_t hits = 0, hit = -1;
      for (; u < trials.size() && trials[u].job == trials[t].job && trials[u].arg == trials[t].arg; ++u)
        if (tres[u].status == PE_CAND_OK && ag_total(tres[u]) <= live[trials[t].job].base_ag) {
          if (hits++ == 0) hit = (int32_t)u;
        }
      if (hits == 1 && pick[trials[t].job] < 0) pick[trials[t].job] = hit;
      t = u;
    }
    std::vector<Job> next;
    std::vector<pe_action> flat;
    std::vector<uint32_t> off{0};
    for (uint32_t j = 0; j < live.size(); ++j) {
      if (pick[j] < 0) continue;  // no argument determined: this expansion is complete
      live[j].seq->push_back(trials[pick[j]].tile);
      flat.insert(flat.end(), live[j].seq->begin(), live[j].seq->end());
      off.push_back((uint32_t)flat.size());
      next.push_back(std::move(live[j]));
    }
    if (next.empty()) break;
    std::vector<pe_result> res;
    std::vector<uint8_t> fl;
    if (!eval_seqs(e, flat, off, res, &fl, st, err)) return false;
    live.clear();
    for (size_t j = 0; j < next.size(); ++j) {
      if (res[j].status != PE_CAND_OK) continue;
      next[j].base_ag = ag_total(res[j]);
      next[j].flags.assign(fl.begin() + j * A, fl.begin() + (j + 1) * A);
      live.push_back(std::move(next[j]));
    }
  }
  return true;
}

__global__ void pe_paused_kernel(const pe_result* out, uint32_t n, uint32_t* list, uint32_t* count) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && out[i].status == PE_CAND_PAUSED) list[atomicAdd(count, 1u)] = i;
}

// per paused candidate: pause position, draws consumed, recorded actions
__global__ void pe_ir_gather_kernel(const uint32_t* list, uint32_t m, const pe_result* out,
                                    const pe_action* acts, const uint32_t* nacts, int32_t maxd,
                                    int32_t* info, pe_action* acts_g) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  uint32_t i = list[j];
  info[3 * j] = out[i].fail_step;
  info[3 * j + 1] = out[i].reserved;
  info[3 * j + 2] = (int32_t)nacts[i];
  for (int32_t k = 0; k < maxd; ++k) acts_g[(uint64_t)j * maxd + k] = acts[(uint64_t)i * maxd + k];
}

// resumed results back into the caller's slots; legal rows only for
// candidates whose legal set is taken after the caller's prefix in this run
__global__ void pe_ir_scatter_kernel(const uint32_t* list, uint32_t m, const pe_result* out2,
                                     const pe_action* acts2, const uint32_t* nacts2,
                                     const uint64_t* legal2, const uint8_t* take_legal,
                                     int32_t maxd, int32_t lw, pe_result* out, pe_action* acts,
                                     uint32_t* nacts, uint64_t* legal) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  uint32_t i = list[j];
  out[i] = out2[j];
  nacts[i] = nacts2[j];
  for (int32_t k = 0; k < maxd; ++k) acts[(uint64_t)i * maxd + k] = acts2[(uint64_t)j * maxd + k];
  if (legal && take_legal[j])
    for (int32_t w = 0; w < lw; ++w) legal[(uint64_t)i * lw + w] = legal2[(uint64_t)j * lw + w];
}

struct RolloutIo {
  pe::GraphView gv;
  const pe_action* d_prefix;
  const uint32_t* d_poff;
  const uint64_t* d_seeds;
  uint32_t n;
  pe_action* d_acts;
  uint32_t* d_nacts;
  pe_result* d_out;
  uint64_t* d_legal;
  uint32_t* max_acts;
  const pe_action* h_prefix;  // host copies (host mode), else NULL
  const uint32_t* h_poff;
  const uint64_t* h_seeds;
};

// Resolves every paused candidate of a rollout batch: expand its InferRest
// decision (batched with all other paused candidates), then resume it from
// the expanded sequence with its RNG stream advanced past the draws it
// consumed (splitmix64 state = seed + draws * gamma); a resumed rollout may
// pause again.  The caller's outputs end up exactly as an uninterrupted
// rollout would have written them.
pe_status ir_resolve(pe_engine* e, const RolloutIo& io, cudaStream_t st, pe_error* err) {
  NvtxRange nvtx_("ir_resolve");
  const int32_t maxd = (int32_t)e->cfg.max_decisions;
  const int32_t lw = (int32_t)pe_engine_legal_words(e);
  const uint64_t kGamma = 0x9E3779B97F4A7C15ull;
  // host view of the caller's prefixes and seeds (device mode: fetched once)
  std::vector<pe_action> hp;
  std::vector<uint32_t> hpoff;
  std::vector<uint64_t> hseeds;
  bool have_host = io.h_poff != nullptr;
  struct Cur {
    std::vector<pe_action> prefix;
    uint64_t seed;
  };
  std::unordered_map<uint32_t, Cur> cur;  // candidates resumed at least once
  std::vector<void*> bufs;
  auto fail = [&](pe_status s) {
    cudaStreamSynchronize(st);
    for (void* q : bufs) cudaFree(q);
    return s;
  };
  auto dalloc = [&](size_t bytes) -> void* {
    void* q = nullptr;
    if (!cuda_ok(cudaMalloc(&q, std::max<size_t>(bytes, 16)), err, "cudaMalloc(ir)")) return nullptr;
    bufs.push_back(q);
    return q;
  };
  uint32_t* d_list = (uint32_t*)dalloc((size_t)io.n * 4 + 4);
  uint32_t* d_cnt = (uint32_t*)dalloc(4);
  if (!d_list || !d_cnt) return fail(PE_ERR_CUDA);
  for (int round = 0;; ++round) {
    uint32_t m = 0;
    if (!cuda_ok(cudaMemsetAsync(d_cnt, 0, 4, st), err, "ir count")) return fail(PE_ERR_CUDA);
    pe_paused_kernel<<<(io.n + 255) / 256, 256, 0, st>>>(io.d_out, io.n, d_list, d_cnt);
    e->launches += 1;
    if (!cuda_ok(cudaGetLastError(), err, "ir launch") ||
        !cuda_ok(cudaMemcpyAsync(&m, d_cnt, 4, cudaMemcpyDeviceToHost, st), err, "D2H ir") ||
        !cuda_ok(cudaStreamSynchronize(st), err, "ir sync"))
      return fail(PE_ERR_CUDA);
    if (m == 0) break;
    std::vector<uint32_t> list(m);
    // (all copies on the call's stream: a pageable cudaMemcpy may return
    // before its DMA lands, and a non-blocking stream does not wait for it)
    auto d2h = [&](void* dst, const void* src, size_t bytes) {
      return cuda_ok(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st), err, "D2H ir") &&
             cuda_ok(cudaStreamSynchronize(st), err, "ir sync");
    };
    if (!d2h(list.data(), d_list, (size_t)m * 4)) return fail(PE_ERR_CUDA);
    std::sort(list.begin(), list.end());
    if (!cuda_ok(cudaMemcpyAsync(d_list, list.data(), (size_t)m * 4, cudaMemcpyHostToDevice, st),
                 err, "H2D ir") ||
        !cuda_ok(cudaStreamSynchronize(st), err, "ir sync"))
      return fail(PE_ERR_CUDA);
    if (!have_host) {
      hpoff.assign(io.n + 1, 0);
      hseeds.assign(io.n, 0);
      bool ok = io.d_poff == nullptr || d2h(hpoff.data(), io.d_poff, (size_t)(io.n + 1) * 4);
      ok = ok && d2h(hseeds.data(), io.d_seeds, (size_t)io.n * 8);
      if (ok && io.d_prefix && hpoff[io.n]) {
        hp.resize(hpoff[io.n]);
        ok = d2h(hp.data(), io.d_prefix, hp.size() * sizeof(pe_action));
      }
      if (!io.d_prefix) std::fill(hpoff.begin(), hpoff.end(), 0u);
      if (!ok) return fail(PE_ERR_CUDA);
      have_host = true;
    }
    const pe_action* P = io.h_prefix ? io.h_prefix : hp.data();
    const uint32_t* PO = io.h_poff ? io.h_poff : hpoff.data();
    const uint64_t* SD = io.h_seeds ? io.h_seeds : hseeds.data();
    // pause position, draws and recorded actions of the paused candidates
    int32_t* d_info = (int32_t*)dalloc((size_t)m * 12);
    pe_action* d_ag = (pe_action*)dalloc((size_t)m * maxd * sizeof(pe_action));
    if (!d_info || !d_ag) return fail(PE_ERR_CUDA);
    pe_ir_gather_kernel<<<(m + 255) / 256, 256, 0, st>>>(d_list, m, io.d_out, io.d_acts, io.d_nacts,
                                                          maxd, d_info, d_ag);
    e->launches += 1;
    std::vector<int32_t> info((size_t)m * 3);
    std::vector<pe_action> ag((size_t)m * maxd);
    if (!cuda_ok(cudaGetLastError(), err, "ir launch") ||
        !cuda_ok(cudaMemcpyAsync(info.data(), d_info, info.size() * 4, cudaMemcpyDeviceToHost, st), err, "D2H ir") ||
        !cuda_ok(cudaMemcpyAsync(ag.data(), d_ag, ag.size() * sizeof(pe_action), cudaMemcpyDeviceToHost, st), err, "D2H ir") ||
        !cuda_ok(cudaStreamSynchronize(st), err, "ir sync"))
      return fail(PE_ERR_CUDA);
    // the state each InferRest applies to, and what follows it
    std::vector<std::vector<pe_action>> state(m), rest(m);
    std::vector<uint64_t> seed2(m);
    std::vector<uint8_t> take_legal(m, 0);
    for (uint32_t j = 0; j < m; ++j) {
      uint32_t i = list[j];
      auto it = cur.find(i);
      const pe_action* pb = it != cur.end() ? it->second.prefix.data() : P + PO[i];
      uint32_t pn = it != cur.end() ? (uint32_t)it->second.prefix.size() : PO[i + 1] - PO[i];
      uint64_t sd = it != cur.end() ? it->second.seed : SD[i];
      int32_t at = info[3 * j], draws = info[3 * j + 1], nrec = info[3 * j + 2];
      if (at >= 0) {  // an unexpanded marker in the prefix
        state[j].assign(pb, pb + at);
        rest[j].assign(pb + at + 1, pb + pn);
        // the legal set is taken after the caller's whole prefix, which
        // the resumed run reaches for the first time
        take_legal[j] = 1;
      } else {  // a drawn decision: the prefix, then the drawn tiles
        state[j].assign(pb, pb + pn);
        uint32_t rec = 0;
        for (uint32_t k = 0; k < pn; ++k) rec += (pb[k].pad & PE_ACT_FLAG_INFERRED) ? 0 : 1;
        if (nrec > maxd) return fail(PE_ERR_INTERNAL);
        for (int32_t k = (int32_t)rec; k < nrec - 1; ++k) state[j].push_back(ag[(size_t)j * maxd + k]);
      }
      seed2[j] = sd + (uint64_t)draws * kGamma;
    }
    std::vector<std::vector<pe_action>*> ptrs(m);
    for (uint32_t j = 0; j < m; ++j) ptrs[j] = &state[j];
    if (!ir_expand_batch(e, ptrs, st, err)) return fail(PE_ERR_CUDA);
    // resume: expanded state + the rest of the prefix, advanced seed
    std::vector<pe_action> flat;
    std::vector<uint32_t> off{0};
    for (uint32_t j = 0; j < m; ++j) {
      Cur c;
      c.prefix = std::move(state[j]);
      c.prefix.insert(c.prefix.end(), rest[j].begin(), rest[j].end());
      c.seed = seed2[j];
      flat.insert(flat.end(), c.prefix.begin(), c.prefix.end());
      off.push_back((uint32_t)flat.size());
      cur[list[j]] = std::move(c);
    }
    pe_action* d_p2 = (pe_action*)dalloc(std::max<size_t>(1, flat.size()) * sizeof(pe_action));
    uint32_t* d_o2 = (uint32_t*)dalloc(off.size() * 4);
    uint64_t* d_s2 = (uint64_t*)dalloc((size_t)m * 8);
    pe_action* d_a2 = (pe_action*)dalloc((size_t)m * maxd * sizeof(pe_action));
    uint32_t* d_n2 = (uint32_t*)dalloc((size_t)m * 4);
    pe_result* d_r2 = (pe_result*)dalloc((size_t)m * sizeof(pe_result));
    uint64_t* d_l2 = io.d_legal ? (uint64_t*)dalloc((size_t)m * lw * 8) : nullptr;
    uint8_t* d_tl = (uint8_t*)dalloc(m);
    if (!d_p2 || !d_o2 || !d_s2 || !d_a2 || !d_n2 || !d_r2 || (io.d_legal && !d_l2) || !d_tl)
      return fail(PE_ERR_CUDA);
    std::vector<uint64_t> s2h(seed2.begin(), seed2.end());
    bool ok = (flat.empty() || cuda_ok(cudaMemcpyAsync(d_p2, flat.data(), flat.size() * sizeof(pe_action),
                                                       cudaMemcpyHostToDevice, st), err, "H2D ir")) &&
              cuda_ok(cudaMemcpyAsync(d_o2, off.data(), off.size() * 4, cudaMemcpyHostToDevice, st), err, "H2D ir") &&
              cuda_ok(cudaMemcpyAsync(d_s2, s2h.data(), (size_t)m * 8, cudaMemcpyHostToDevice, st), err, "H2D ir") &&
              cuda_ok(cudaMemcpyAsync(d_tl, take_legal.data(), m, cudaMemcpyHostToDevice, st), err, "H2D ir");
    ok = ok && cuda_ok(enqueue_rollouts(e, io.gv, d_p2, d_o2, d_s2, m, d_a2, d_n2, d_r2, d_l2,
                                        nullptr, SchedView(), CacheView(), io.max_acts, st),
                       err, "pe_rollout_kernel launch (resume)");
    if (ok) {
      pe_ir_scatter_kernel<<<(m + 255) / 256, 256, 0, st>>>(d_list, m, d_r2, d_a2, d_n2, d_l2, d_tl,
                                                            maxd, lw, io.d_out, io.d_acts,
                                                            io.d_nacts, io.d_legal);
      e->launches += 1;
      ok = cuda_ok(cudaGetLastError(), err, "ir launch") &&
           cuda_ok(cudaStreamSynchronize(st), err, "ir sync");
    }
    // (flat / off / seeds are read by the async copies before this point)
    if (!ok) return fail(PE_ERR_CUDA);
    for (size_t k = 2; k < bufs.size(); ++k) cudaFree(bufs[k]);
    bufs.resize(2);
  }
  return fail(PE_OK);
}


uint64_t snapshot_stride(const pe_engine* e) {
  return (pe::Cand::snap_bytes(e->dview, e->big_layout.caps) + 255) & ~uint64_t(255);
}

// Per candidate: its longest cached prefix (start there) and, when its whole
// prefix is not cached yet, a slot to save the post-prefix state into.
bool pc_plan(pe_engine* e, const pe_action* prefix, const uint32_t* poff, uint32_t n,
             cudaStream_t st, CacheView* cv, std::vector<int32_t>& save_slot, pe_error* err) {
  if (!e->d_pc) {
    e->pc_stride = snapshot_stride(e);
    uint64_t cap = (uint64_t)(e->pc_budget_gb * (double)(1ull << 30)) / e->pc_stride;
    e->pc_cap = (int32_t)std::min<uint64_t>(cap, 1u << 20);
    if (e->pc_cap <= 0) return true;
    if (!cuda_ok(cudaMalloc(&e->d_pc, (size_t)e->pc_cap * e->pc_stride), err,
                 "cudaMalloc(prefix cache)"))
      return false;
    e->pc_key.assign(e->pc_cap, std::string());
    e->pc_used.assign(e->pc_cap, 0);
  }
  ++e->pc_clock;
  std::vector<uint64_t> from(n, 0), save(n, 0);
  std::vector<int32_t> from_len(n, 0);
  save_slot.assign(n, -1);
  std::unordered_map<std::string, int32_t> planned;  // full prefixes saved by this batch
  e->pc_pending.assign(n, std::string());
  for (uint32_t i = 0; i < n; ++i) {
    const char* b = reinterpret_cast<const char*>(prefix + poff[i]);
    uint32_t np = poff[i + 1] - poff[i];
    bool decisions = true;  // cache only plain decision prefixes
    for (uint32_t k = 0; k < np && decisions; ++k)
      decisions = prefix[poff[i] + k].kind <= PE_ACT_TILE_GROUP && prefix[poff[i] + k].pad == 0;
    if (!decisions || np == 0) continue;
    for (uint32_t k = np; k >= 1; --k) {
      auto it = e->pc_map.find(std::string(b, (size_t)k * sizeof(pe_action)));
      if (it == e->pc_map.end()) continue;
      from[i] = (uint64_t)(e->d_pc + e->pc_stride * (uint64_t)it->second);
      from_len[i] = (int32_t)k;
      e->pc_used[it->second] = e->pc_clock;
      ++e->pc_hits;
      break;
    }
    if (from_len[i] == (int32_t)np) continue;
    std::string key(b, (size_t)np * sizeof(pe_action));
    if (planned.count(key)) continue;
    // a slot not read by this batch: the clock hand's next
    int32_t slot = -1;
    for (int32_t tries = 0; tries < e->pc_cap && slot < 0; ++tries) {
      int32_t h = e->pc_hand;
      e->pc_hand = (e->pc_hand + 1) % e->pc_cap;
      if (e->pc_used[h] != e->pc_clock) slot = h;
    }
    if (slot < 0) continue;
    if (!e->pc_key[slot].empty()) e->pc_map.erase(e->pc_key[slot]);
    e->pc_key[slot].clear();
    e->pc_used[slot] = e->pc_clock;
    save[i] = (uint64_t)(e->d_pc + e->pc_stride * (uint64_t)slot);
    save_slot[i] = slot;
    e->pc_pending[i] = key;
    planned.emplace(std::move(key), slot);
  }
  // device arrays: from, save (u64), from_len (i32), saved flags (u8)
  size_t words = 2 * (size_t)n + ((size_t)n + 1) / 2 + ((size_t)n + 7) / 8 + 4;
  if (!ensure_dev(e->d_cv, e->cv_cap, words, err, "cudaMalloc(cache view)")) return false;
  uint64_t* d_from = e->d_cv;
  uint64_t* d_save = d_from + n;
  int32_t* d_len = reinterpret_cast<int32_t*>(d_save + n);
  uint8_t* d_saved = reinterpret_cast<uint8_t*>(d_len + ((n + 1) & ~1u));
  if (!cuda_ok(cudaMemcpyAsync(d_from, from.data(), (size_t)n * 8, cudaMemcpyHostToDevice, st), err, "H2D cache") ||
      !cuda_ok(cudaMemcpyAsync(d_save, save.data(), (size_t)n * 8, cudaMemcpyHostToDevice, st), err, "H2D cache") ||
      !cuda_ok(cudaMemcpyAsync(d_len, from_len.data(), (size_t)n * 4, cudaMemcpyHostToDevice, st), err, "H2D cache") ||
      !cuda_ok(cudaMemsetAsync(d_saved, 0, n, st), err, "cache flags") ||
      !cuda_ok(cudaStreamSynchronize(st), err, "cache sync"))  // (host vectors go away)
    return false;
  cv->from = d_from;
  cv->from_len = d_len;
  cv->save = d_save;
  cv->saved = d_saved;
  return true;
}

// After the launch: a slot becomes a cache entry only if its state was
// written (a candidate that overflowed its tight arena saves nothing).
bool pc_commit(pe_engine* e, uint32_t n, const std::vector<int32_t>& save_slot, cudaStream_t st,
               pe_error* err) {
  uint64_t* d_save = e->d_cv + n;
  uint8_t* d_saved = reinterpret_cast<uint8_t*>(reinterpret_cast<int32_t*>(d_save + n) +
                                                ((n + 1) & ~1u));
  std::vector<uint8_t> saved(n);
  if (!cuda_ok(cudaMemcpyAsync(saved.data(), d_saved, n, cudaMemcpyDeviceToHost, st), err, "D2H cache") ||
      !cuda_ok(cudaStreamSynchronize(st), err, "cache sync"))
    return false;
  for (uint32_t i = 0; i < n; ++i) {
    int32_t slot = save_slot[i];
    if (slot < 0 || !saved[i]) continue;
    e->pc_key[slot] = std::move(e->pc_pending[i]);
    e->pc_map[e->pc_key[slot]] = slot;
    ++e->pc_saved;
  }
  e->pc_pending.clear();
  return true;
}

// Candidates = prefix (host) from optional saved states, no draws (each
// prefix ends in Stop): the evaluation of prefix[c], optionally saving the
// post-prefix state (pe_state handles).
bool run_states(pe_engine* e, const std::vector<pe_action>& flat, const std::vector<uint32_t>& off,
                const std::vector<uint64_t>& from, const std::vector<int32_t>& from_len,
                const std::vector<uint64_t>& save, std::vector<uint8_t>& saved,
                std::vector<pe_result>& res, cudaStream_t st, pe_error* err) {
  uint32_t n = (uint32_t)off.size() - 1;
  const int32_t maxd = (int32_t)e->cfg.max_decisions;
  res.resize(n);
  saved.assign(n, 0);
  if (n == 0) return true;
  std::vector<void*> bufs;
  auto dal = [&](size_t b) {
    void* q = nullptr;
    if (cudaMalloc(&q, std::max<size_t>(b, 16)) != cudaSuccess) return (void*)nullptr;
    bufs.push_back(q);
    return q;
  };
  pe_action* d_p = (pe_action*)dal(std::max<size_t>(1, flat.size()) * sizeof(pe_action));
  uint32_t* d_o = (uint32_t*)dal(off.size() * 4);
  uint64_t* d_s = (uint64_t*)dal((size_t)n * 8);
  pe_action* d_a = (pe_action*)dal((size_t)n * maxd * sizeof(pe_action));
  uint32_t* d_n = (uint32_t*)dal((size_t)n * 4);
  pe_result* d_r = (pe_result*)dal((size_t)n * sizeof(pe_result));
  uint64_t* d_f = (uint64_t*)dal((size_t)n * 8);
  uint64_t* d_v = (uint64_t*)dal((size_t)n * 8);
  int32_t* d_l = (int32_t*)dal((size_t)n * 4);
  uint8_t* d_ok = (uint8_t*)dal(n);
  bool ok = bufs.size() == 10;
  if (!ok) set_err(err, PE_ERR_CUDA, "cudaMalloc(states)");
  ok = ok && (flat.empty() || cuda_ok(cudaMemcpyAsync(d_p, flat.data(), flat.size() * sizeof(pe_action),
                                                      cudaMemcpyHostToDevice, st), err, "H2D states")) &&
       cuda_ok(cudaMemcpyAsync(d_o, off.data(), off.size() * 4, cudaMemcpyHostToDevice, st), err, "H2D states") &&
       cuda_ok(cudaMemsetAsync(d_s, 0, (size_t)n * 8, st), err, "states") &&
       cuda_ok(cudaMemcpyAsync(d_f, from.data(), (size_t)n * 8, cudaMemcpyHostToDevice, st), err, "H2D states") &&
       cuda_ok(cudaMemcpyAsync(d_v, save.data(), (size_t)n * 8, cudaMemcpyHostToDevice, st), err, "H2D states") &&
       cuda_ok(cudaMemcpyAsync(d_l, from_len.data(), (size_t)n * 4, cudaMemcpyHostToDevice, st), err, "H2D states") &&
       cuda_ok(cudaMemsetAsync(d_ok, 0, n, st), err, "states");
  CacheView cv;
  cv.from = d_f;
  cv.from_len = d_l;
  cv.save = d_v;
  cv.saved = d_ok;
  ok = ok && cuda_ok(enqueue_rollouts(e, e->dview, d_p, d_o, d_s, n, d_a, d_n, d_r, nullptr,
                                      nullptr, SchedView(), cv, nullptr, st),
                     err, "pe_rollout_kernel launch (states)") &&
       cuda_ok(cudaMemcpyAsync(res.data(), d_r, (size_t)n * sizeof(pe_result), cudaMemcpyDeviceToHost, st),
               err, "D2H states") &&
       cuda_ok(cudaMemcpyAsync(saved.data(), d_ok, n, cudaMemcpyDeviceToHost, st), err, "D2H states") &&
       cuda_ok(cudaStreamSynchronize(st), err, "states sync");
  for (void* q : bufs) cudaFree(q);
  return ok;
}

bool plain_decisions(const pe_action* a, uint32_t n) {
  for (uint32_t k = 0; k < n; ++k)
    if (a[k].kind > PE_ACT_TILE_GROUP || a[k].pad != 0) return false;
  return true;
}

}  // namespace

extern "C" {

pe_status pe_rollout_batch(pe_engine* e, const pe_action* prefix, const uint32_t* prefix_off,
                           const uint64_t* seeds, uint32_t n, pe_action* acts_out,
                           uint32_t* n_acts_out, pe_result* out, uint64_t* legal_out,
                           uint32_t flags, void* stream, pe_error* err) {
  NvtxRange nvtx_("pe_rollout_batch");
  if (!e || !prefix_off || !seeds || !acts_out || !n_acts_out || !out) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null argument");
    return PE_ERR_INVALID_ARGUMENT;
  }
  if (n == 0) return PE_OK;
  if (e->wl.auto_axes.empty()) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "no auto axes selected");
    return PE_ERR_INVALID_ARGUMENT;
  }
  cudaStream_t st = (cudaStream_t)stream;
  if (!cuda_ok(cudaSetDevice(e->device), err, "cudaSetDevice")) return PE_ERR_CUDA;
  if (!call_begin(e, st, err)) return PE_ERR_CUDA;
  int32_t maxd = (int32_t)e->cfg.max_decisions;
  int32_t lw = (int32_t)pe_engine_legal_words(e);
  const pe_action* d_prefix = prefix;
  const uint32_t* d_poff = prefix_off;
  const uint64_t* d_seeds = seeds;
  pe_action* d_acts = acts_out;
  uint32_t* d_nacts = n_acts_out;
  pe_result* d_out = out;
  uint64_t* d_legal = legal_out;
  if (!(flags & PE_MEM_DEVICE)) {
    uint32_t np = prefix_off[n];
    auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
    size_t b_pre = al((size_t)np * sizeof(pe_action) + 8), b_poff = al((size_t)(n + 1) * 4);
    size_t b_seed = al((size_t)n * 8), b_acts = al((size_t)n * maxd * sizeof(pe_action));
    size_t b_nacts = al((size_t)n * 4), b_out = al((size_t)n * sizeof(pe_result));
    size_t b_legal = legal_out ? al((size_t)n * lw * 8) : 0;
    if (!ensure_io(e, b_pre + b_poff + b_seed + b_acts + b_nacts + b_out + b_legal, err))
      return PE_ERR_CUDA;
    uint8_t* p = e->d_io;
    d_prefix = (const pe_action*)p;
    p += b_pre;
    d_poff = (const uint32_t*)p;
    p += b_poff;
    d_seeds = (const uint64_t*)p;
    p += b_seed;
    d_acts = (pe_action*)p;
    p += b_acts;
    d_nacts = (uint32_t*)p;
    p += b_nacts;
    d_out = (pe_result*)p;
    p += b_out;
    d_legal = legal_out ? (uint64_t*)p : nullptr;
    if (np && !cuda_ok(cudaMemcpyAsync((void*)d_prefix, prefix, (size_t)np * sizeof(pe_action),
                                       cudaMemcpyHostToDevice, st), err, "H2D prefix"))
      return PE_ERR_CUDA;
    if (!cuda_ok(cudaMemcpyAsync((void*)d_poff, prefix_off, (size_t)(n + 1) * 4,
                                 cudaMemcpyHostToDevice, st), err, "H2D prefix_off") ||
        !cuda_ok(cudaMemcpyAsync((void*)d_seeds, seeds, (size_t)n * 8, cudaMemcpyHostToDevice,
                                 st), err, "H2D seeds"))
      return PE_ERR_CUDA;
  }
  // prefix-trie scheduling for batches of root rollouts (all prefixes
  // empty; a NULL prefix array in device mode), DESIGN.md §3.5
  const uint32_t* perm = nullptr;
  SchedView sv;
  bool roots = (flags & PE_MEM_DEVICE) ? prefix == nullptr : prefix_off[n] == 0;
  if (roots && e->sched_depth > 0 && !e->wl.resurface && !e->wl.infer_rest &&
      n >= e->sched_min_batch &&
      !sched_perm(e, n, d_seeds, maxd, st, &perm, &sv, err))
    return PE_ERR_CUDA;
  // candidates start from their node's saved state unless legal sets after
  // the (empty) prefix are requested
  if (d_legal || !sv.snap) sv.keys = nullptr;
  // host mode: the kernels record the longest action list so only that many
  // columns of acts_out travel back
  uint32_t* max_acts = (flags & PE_MEM_DEVICE) ? nullptr : e->d_ctr + 4;
  if (max_acts && !cuda_ok(cudaMemsetAsync(max_acts, 0, 4, st), err, "reset max acts"))
    return PE_ERR_CUDA;
  // InferRest decisions (pe.h infer_rest_action, or unexpanded markers in a
  // host prefix) pause their candidates for the batched expansion below
  bool ir = e->wl.infer_rest;
  if (!(flags & PE_MEM_DEVICE))
    for (uint32_t k = 0; k < prefix_off[n] && !ir; ++k)
      ir = prefix[k].kind == PE_ACT_INFER_REST && !(prefix[k].pad & PE_ACT_FLAG_EXPANDED);
  pe::GraphView gv = e->dview;
  gv.ir_pause = ir ? 1 : 0;
  // prefix-state cache (host mode, non-root prefixes)
  CacheView cv;
  std::vector<int32_t> pc_save;
  if (!(flags & PE_MEM_DEVICE) && e->pc_budget_gb > 0 && !roots && !ir && !e->wl.resurface &&
      !pc_plan(e, prefix, prefix_off, n, st, &cv, pc_save, err))
    return PE_ERR_CUDA;
  if (!cuda_ok(enqueue_rollouts(e, gv, d_prefix, d_poff, d_seeds, n, d_acts, d_nacts, d_out,
                                d_legal, perm, sv, cv, max_acts, st),
               err, "pe_rollout_kernel launch"))
    return PE_ERR_CUDA;
  if (cv.save && !pc_commit(e, n, pc_save, st, err)) return PE_ERR_CUDA;
  if (ir) {
    RolloutIo io{gv, d_prefix, d_poff, d_seeds, n, d_acts, d_nacts, d_out, d_legal, max_acts,
                 (flags & PE_MEM_DEVICE) ? nullptr : prefix,
                 (flags & PE_MEM_DEVICE) ? nullptr : prefix_off,
                 (flags & PE_MEM_DEVICE) ? nullptr : seeds};
    pe_status rs = ir_resolve(e, io, st, err);
    if (rs != PE_OK) return rs;
  }
  if (!(flags & PE_MEM_DEVICE)) {
    uint32_t kmax = 0;
    bool ok = cuda_ok(cudaMemcpyAsync(&kmax, max_acts, 4, cudaMemcpyDeviceToHost, st), err,
                      "D2H max acts") &&
              cuda_ok(cudaStreamSynchronize(st), err, "sync");
    kmax = std::min<uint32_t>(kmax, (uint32_t)maxd);
    ok = ok && (kmax == 0 ||
                cuda_ok(cudaMemcpy2DAsync(acts_out, (size_t)maxd * sizeof(pe_action), d_acts,
                                          (size_t)maxd * sizeof(pe_action),
                                          (size_t)kmax * sizeof(pe_action), n,
                                          cudaMemcpyDeviceToHost, st), err, "D2H acts")) &&
              cuda_ok(cudaMemcpyAsync(n_acts_out, d_nacts, (size_t)n * 4,
                                      cudaMemcpyDeviceToHost, st), err, "D2H n_acts") &&
              cuda_ok(cudaMemcpyAsync(out, d_out, (size_t)n * sizeof(pe_result),
                                      cudaMemcpyDeviceToHost, st), err, "D2H results");
    if (ok && legal_out)
      ok = cuda_ok(cudaMemcpyAsync(legal_out, d_legal, (size_t)n * lw * 8,
                                   cudaMemcpyDeviceToHost, st), err, "D2H legal");
    if (!ok || !call_end(e, st, err)) return PE_ERR_CUDA;
    if (!cuda_ok(cudaStreamSynchronize(st), err, "sync")) return PE_ERR_CUDA;
  } else if (!call_end(e, st, err)) {
    return PE_ERR_CUDA;
  } else if (flags & PE_SYNC) {
    if (!cuda_ok(cudaStreamSynchronize(st), err, "sync")) return PE_ERR_CUDA;
  }
  return PE_OK;
}

pe_status pe_engine_set_prefix_cache(pe_engine* e, double budget_gb) {
  if (!e || budget_gb < 0) return PE_ERR_INVALID_ARGUMENT;
  if (e->d_pc) return e->pc_budget_gb == budget_gb ? PE_OK : PE_ERR_INVALID_ARGUMENT;
  e->pc_budget_gb = budget_gb;
  return PE_OK;
}

void pe_engine_prefix_cache_stats(const pe_engine* e, uint64_t* hits, uint64_t* saved,
                                  int64_t* entries) {
  if (hits) *hits = e->pc_hits;
  if (saved) *saved = e->pc_saved;
  if (entries) *entries = (int64_t)e->pc_map.size();
}

pe_status pe_state_create(pe_engine* e, const pe_action* acts, uint32_t n, pe_state** out,
                          pe_error* err) {
  NvtxRange nvtx_("pe_state_create");
  if (!e || !out || (n && !acts)) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null argument");
    return PE_ERR_INVALID_ARGUMENT;
  }
  if (!plain_decisions(acts, n)) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "pe_state: TILE / TILE_GROUP decisions only");
    return PE_ERR_INVALID_ARGUMENT;
  }
  if (!cuda_ok(cudaSetDevice(e->device), err, "cudaSetDevice")) return PE_ERR_CUDA;
  pe_state* s = new pe_state();
  s->e = e;
  s->path.assign(acts, acts + n);
  // its evaluation and parity trace (arg / result specs, stuck list)
  const uint32_t tw = 8 + 2 * (uint32_t)e->graph->g.args.size() + 2 * (uint32_t)e->graph->g.ops.size();
  s->trace.assign(tw, 0);
  uint32_t off[2] = {0, n};
  pe_status ps = pe_eval_batch(e, n ? acts : nullptr, off, 1, &s->result, s->trace.data(), tw, 0,
                               nullptr, err);
  if (ps != PE_OK) {
    delete s;
    return ps;
  }
  if (s->result.status != PE_CAND_OK) {
    set_err(err, s->result.status == PE_CAND_ILLEGAL ? PE_ERR_ILLEGAL : PE_ERR_INTERNAL,
            "pe_state: the sequence does not evaluate (status " +
                std::to_string(s->result.status) + ")");
    pe_status code = s->result.status == PE_CAND_ILLEGAL ? PE_ERR_ILLEGAL : PE_ERR_INTERNAL;
    delete s;
    return code;
  }
  if (!cuda_ok(cudaMalloc(&s->d_snap, snapshot_stride(e)), err, "cudaMalloc(state)")) {
    delete s;
    return PE_ERR_CUDA;
  }
  std::vector<pe_action> flat(s->path);
  flat.push_back(pe_action{0, 0, 0, PE_ACT_STOP, 0});
  std::vector<uint8_t> saved;
  std::vector<pe_result> res;
  if (!run_states(e, flat, {0, (uint32_t)flat.size()}, {0}, {0}, {(uint64_t)s->d_snap}, saved, res,
                  nullptr, err)) {
    pe_state_destroy(s);
    return PE_ERR_CUDA;
  }
  if (!saved[0]) {  // (the full-size retry path saves nothing)
    set_err(err, PE_ERR_CAPACITY, "pe_state: state exceeds the engine's tight arena");
    pe_state_destroy(s);
    return PE_ERR_CAPACITY;
  }
  *out = s;
  if (err) err->code = PE_OK;
  return PE_OK;
}

void pe_state_destroy(pe_state* s) {
  if (!s) return;
  if (s->d_snap) cudaFree(s->d_snap);
  delete s;
}

uint32_t pe_state_num_decisions(const pe_state* s) { return (uint32_t)s->path.size(); }

pe_status pe_state_result(const pe_state* s, pe_result* out) {
  if (!s || !out) return PE_ERR_INVALID_ARGUMENT;
  *out = s->result;
  return PE_OK;
}

pe_status pe_state_specs(const pe_state* s, uint32_t* arg_specs, uint32_t* result_spec,
                         int32_t* stuck, uint32_t stuck_cap, uint32_t* n_stuck, pe_error* err) {
  if (!s) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null state");
    return PE_ERR_INVALID_ARGUMENT;
  }
  // the parity trace layout of pe.h: [0] words, [1] A, A arg specs, result
  // spec, n_stuck, (op, reason) pairs, ...
  const int32_t* t = s->trace.data();
  int32_t A = t[1];
  if (arg_specs)
    for (int32_t x = 0; x < A; ++x) arg_specs[x] = (uint32_t)t[2 + x];
  if (result_spec) *result_spec = (uint32_t)t[2 + A];
  int32_t ns = t[3 + A];
  if (n_stuck) *n_stuck = (uint32_t)ns;
  for (int32_t i = 0; stuck && i < ns && (uint32_t)i < stuck_cap; ++i) {
    stuck[2 * i] = t[4 + A + 2 * i];
    stuck[2 * i + 1] = t[5 + A + 2 * i];
  }
  return PE_OK;
}

pe_status pe_eval_from_states(pe_engine* e, const pe_state* const* parents, const pe_action* acts,
                              const uint32_t* seq_off, uint32_t n, pe_result* out, void* stream,
                              pe_error* err) {
  NvtxRange nvtx_("pe_eval_from_states");
  if (!e || !parents || !seq_off || !out || (seq_off[n] && !acts)) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null argument");
    return PE_ERR_INVALID_ARGUMENT;
  }
  if (n == 0) return PE_OK;
  if (!cuda_ok(cudaSetDevice(e->device), err, "cudaSetDevice")) return PE_ERR_CUDA;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<pe_action> flat;
  std::vector<uint32_t> off{0};
  std::vector<uint64_t> from(n, 0), save(n, 0);
  std::vector<int32_t> from_len(n, 0);
  for (uint32_t c = 0; c < n; ++c) {
    const pe_state* p = parents[c];
    if (p && p->e != e) {
      set_err(err, PE_ERR_INVALID_ARGUMENT, "state belongs to another engine");
      return PE_ERR_INVALID_ARGUMENT;
    }
    if (!plain_decisions(acts + seq_off[c], seq_off[c + 1] - seq_off[c])) {
      set_err(err, PE_ERR_INVALID_ARGUMENT, "pe_eval_from_states: TILE / TILE_GROUP actions only");
      return PE_ERR_INVALID_ARGUMENT;
    }
    if (p) {
      flat.insert(flat.end(), p->path.begin(), p->path.end());
      from[c] = (uint64_t)p->d_snap;
      from_len[c] = (int32_t)p->path.size();
    }
    flat.insert(flat.end(), acts + seq_off[c], acts + seq_off[c + 1]);
    flat.push_back(pe_action{0, 0, 0, PE_ACT_STOP, 0});
    off.push_back((uint32_t)flat.size());
  }
  std::vector<uint8_t> saved;
  std::vector<pe_result> res;
  if (!call_begin(e, st, err)) return PE_ERR_CUDA;
  if (!run_states(e, flat, off, from, from_len, save, saved, res, st, err)) return PE_ERR_CUDA;
  if (!call_end(e, st, err)) return PE_ERR_CUDA;
  std::copy(res.begin(), res.end(), out);
  return PE_OK;
}

}  // extern "C"

#ifdef PE_PHASE_TIMERS
extern "C" int pe_debug_phase_cycles(unsigned long long* out9, int reset) {
  if (cudaMemcpyFromSymbol(out9, g_phase_cycles, sizeof(unsigned long long) * 9) != cudaSuccess)
    return 1;
  if (reset) {
    unsigned long long z[9] = {0};
    cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z));
  }
  return 0;
}
#endif

#ifdef PE_CAND_TIMES
extern "C" int pe_debug_cand_times(unsigned long long* times, uint32_t* sms, uint32_t n) {
  n = n < kCandTimesCap ? n : kCandTimesCap;
  return cudaMemcpyFromSymbol(times, g_cand_times, sizeof(unsigned long long) * 2 * n) !=
             cudaSuccess ||
         cudaMemcpyFromSymbol(sms, g_cand_sm, sizeof(uint32_t) * n) != cudaSuccess;
}
#endif

// ------------------------------------------------------------------ search
namespace {
int engine_rollout_eval(void* user, const pe_action* prefix, const uint32_t* poff,
                        const uint64_t* seeds, uint32_t n, pe_action* acts_out,
                        uint32_t* n_acts_out, pe_result* out, uint64_t* legal_out) {
  pe_error err;
  return (int)pe_rollout_batch((pe_engine*)user, prefix, poff, seeds, n, acts_out, n_acts_out,
                               out, legal_out, 0, nullptr, &err);
}
}  // namespace

extern "C" pe_status pe_search(pe_engine* e, const pe_search_config* cfg, uint32_t merge_every,
                               uint32_t rank, pe_merge_fn merge, void* merge_user,
                               pe_plan* out, pe_error* err) {
  NvtxRange nvtx_("pe_search");
  if (!e || !out) {
    set_err(err, PE_ERR_INVALID_ARGUMENT, "null argument");
    return PE_ERR_INVALID_ARGUMENT;
  }
  const pe_search_config& c = cfg ? *cfg : e->cfg;
  // incremental leaf evaluation: a leaf starts from its parent's saved state
  if (e->pc_budget_gb == 0 && !e->d_pc) e->pc_budget_gb = 4.0;
  std::vector<pe_action> ords(e->n_ordinals + 1);
  for (uint32_t o = 0; o < e->n_ordinals; ++o) pe_engine_ordinal_action(e, o, &ords[o]);
  ords[e->n_ordinals] = pe_action{0, 0, 0, PE_ACT_STOP, 0};
  pe_mcts_params p;
  p.n_ordinals = e->n_ordinals;
  p.max_decisions = e->cfg.max_decisions;  // the rollout kernel's cap
  p.episodes = c.episodes;
  p.leaf_batch = c.leaf_batch ? c.leaf_batch : 8192;
  p.merge_every = merge_every;
  p.rank = rank;
  p.seed = c.seed;
  p.uct_c = c.uct_c;
  return pe_mcts_run(&p, engine_rollout_eval, e, merge, merge_user, ords.data(), out, err);
}
