// pe_core.cuh — per-candidate evaluation core of the engine.
//
// One candidate = one action sequence applied to the untiled graph, with
// `propagate` after every action, then `lower_to_spmd`, `collective_stats`
// and the SPEC cost model.  This file restates the reference's semantics
// (REF = /root/reference/proj) over flat, bounded per-candidate arrays so it
// runs inside a CUDA kernel with no allocation:
//
//   * the program is not copied per rewrite (REF rewrite.cc:78,
//     propagate.cc:461): a candidate owns an arena of value slots, loop
//     records and a top-level position table;
//   * `propagate`'s restart-after-every-rewrite loop (REF propagate.cc:465-471)
//     becomes ONE in-order forward sweep followed by ONE in-order backward
//     sweep (SURVEY.md Appendix B.2 phase structure; the argument is in
//     DESIGN.md §3.2), with `count_uses` (REF ir.cc:125-134) maintained
//     incrementally instead of by whole-program walks;
//   * lowering (REF spmd.cc:53-403, patch B) walks the same state in the
//     rewritten op order and accumulates collective bytes, liveness and flops.
//
// Compiled for the device by nvcc (the product path).  tests/native builds
// the same header with g++ purely as a test harness for differential fuzzing
// against the oracle; the product library never contains a host copy.
#pragma once
#include <stdint.h>

#include "pe.h"
#include "pe_graph_view.h"
#include "pe_rules.h"

namespace pe {

enum VKind : uint8_t {
  VK_FREE = 0,
  VK_ARG,     // function argument
  VK_TOP,     // original base op still at top level
  VK_LOOP,    // tile / sum loop result (REF ir.h kTile/kSum)
  VK_ATOMIC,  // atomic wrap of an argument (REF rewrite.cc:115-137)
  VK_SLICE,   // slice_axis in a loop body
  VK_LOCAL,   // per-iteration copy of an original op inside a loop body
  VK_DEAD     // erased (extended loop's old name, migrated producer)
};

enum LoopKind : uint8_t { LK_TILE = 0, LK_SUM = 1 };

// stuck reasons (REF propagate.h:28-32)
enum Reason : int32_t { R_INSUFFICIENT = 0, R_BLOCKED = 1, R_CONFLICT = 2, R_NONE = -1 };

// ---------------------------------------------------------------- arena
struct Caps {
  int32_t V;   // value slots
  int32_t L;   // loop records
  int32_t FS;  // front stack (arg action loops + atomics)
  int32_t EM;  // emitted SPMD ops
  int32_t EO;  // emitted operand references
};

// Per-candidate arenas, interleaved candidate-minor.
// The PE_LANES candidates of one warp share a group arena in which every
// field is stored as [index][lane]: lanes walking the graph in near-lockstep
// (same op index in init, the forward sweep and the lowering walk) touch the
// same cache lines, so their accesses coalesce.  The host test harness uses
// PE_LANES = 1 (plain structure of arrays).
//   value slots   vhdr (kind | tile flag | loop axis | loop dim), vref, vaux,
//                 uses, slcnt, body links, top-level position
//   lowering      lo_buf, lo_spec, lo_aux (acq | shape code), lo_gv (REF
//                 spmd.cc:42 `Lowered`; the global shape as a code, see Low)
//   arguments     direct-in-loop count, slice demand, atomic flag, SPMD arg
//                 type, final registered type of the argument buffer
//   loops         kind, axis, dim, body list, yield, result type
//   SPMD ops      head, first operand, last use, operand offset, local bytes,
//                 liveness delta, final registered type of the op's buffer
//   flat          operands, top-level positions, front stack, stuck list,
//                 carries bitmask, legal-ordinal list, operand log (trace)
#ifndef PE_LANES
#ifdef __CUDACC__
#define PE_LANES 32
#else
#define PE_LANES 1
#endif
#endif
constexpr int kLanes = PE_LANES;

// PE_BOUNDS_CHECK (debug builds, tests/test_gpu_bounds.py): every arena
// access must fall inside the candidate's group arena, else the kernel traps
// (the device-side stand-in for compute-sanitizer's memcheck on this path;
// overlaps between a lane's own arrays show up as parity failures).
#ifdef PE_BOUNDS_CHECK
PE_HD void pe_bounds_fail() {
#ifdef __CUDA_ARCH__
  __trap();
#else
  __builtin_trap();
#endif
}
template <typename T, int STRIDE>
struct Field {
  uint8_t* p;
  const uint8_t* lo;
  const uint8_t* hi;
  PE_HD T& operator[](int64_t i) const {
    uint8_t* q = p + i * STRIDE;
    if (q < lo || q + sizeof(T) > hi) pe_bounds_fail();
    return *reinterpret_cast<T*>(q);
  }
};
#else
template <typename T, int STRIDE>
struct Field {
  uint8_t* p;
  PE_HD T& operator[](int64_t i) const { return *reinterpret_cast<T*>(p + i * STRIDE); }
};
#endif
template <typename T>
using LF = Field<T, kLanes * (int)sizeof(T)>;

struct alignas(16) G4 {
  int32_t v[kMaxRank];
};
// a 32-byte record as two 16-byte halves (whole-record writes keep every
// L2 sector fully written: no partial-sector read-modify-write in DRAM)
struct alignas(16) V4 {
  int32_t x, y, z, w;
};
struct alignas(16) I64x2 {
  int64_t x, y;
};
// first half of a LowRec (buf, spec, acq, 0): written and read as one
// 16-byte access so the record's 32-byte sector is always written whole
struct alignas(16) LowHead {
  int32_t buf;
  uint32_t spec;
  uint32_t aux;  // acq | shape code << 4
  int32_t gv;
};

struct Layout {
  Caps caps;
  // byte offsets inside one group arena (kLanes candidates); record arrays
  // are interleaved [index][lane] at record granularity
  uint64_t vrec, lrec, arec, looprec, emrec;
  uint64_t rs, rsb;
  uint64_t opnd, fs, stk, seen, em_opnd, em_spec, carry, lg, dirty, st8, st4;
  uint32_t has_opnd;  // the SPMD operand log (parity traces) is allocated
  uint64_t bytes;  // one group arena
};

constexpr int kRec = 32;    // VRec, LowRec, LoopRec, ArgRec, EmRec

// A lane's view of its group arena: lane-adjusted base pointers (one per
// record / element size) and the layout's offsets, which live in the kernel
// parameter (constant) bank, so field views cost no registers.
//   VRec   [V]   0 vhdr (vk | tile flag | loop axis | loop dim) 4 vref 8 vaux
//                12 uses 16 slcnt 20 bnext 24 bprev 28 vpos
//   LowRec [V]   0 buf 4 spec 8 acq 16 g[4]            (REF spmd.cc:42 Lowered)
//   ArgRec [A]   0 direct-in-loop 4 slice demand 8 atomic 12 SPMD arg spec
//                16 arg local bytes 24 final registered spec (trace)
//   LoopRec[L]   0 kind 1 axis 2 dim 4 head 8 tail 12 yield 16 result type
//   EmRec  [EM]  0 head 4 first operand 8 last use 12 operand offset
//                16 local bytes 24 liveness delta
//   flat         collective_stats accumulators: st8 = all_reduce / all_gather
//                bytes per axis, st4 = their counts + slice_by_coord counts
struct Arena {
  const struct Layout* L;
  uint8_t *b1, *b4, *b8, *r16, *r32;
#ifdef PE_BOUNDS_CHECK
  const uint8_t *lo, *hi;  // the group arena
#define PE_REC(name, T, base, arr, off, STRIDE) \
  PE_HD Field<T, STRIDE> name() const { return {base + L->arr + (off), lo, hi}; }
#else
#define PE_REC(name, T, base, arr, off, STRIDE) \
  PE_HD Field<T, STRIDE> name() const { return {base + L->arr + (off)}; }
#endif
  PE_REC(vk, uint8_t, r32, vrec, 0, kLanes * kRec)
  PE_REC(vh, uint32_t, r32, vrec, 0, kLanes * kRec)
  PE_REC(vref, int32_t, r32, vrec, 4, kLanes * kRec)
  PE_REC(vaux, int32_t, r32, vrec, 8, kLanes * kRec)
  PE_REC(uses, int32_t, r32, vrec, 12, kLanes * kRec)
  PE_REC(slcnt, int32_t, r32, vrec, 16, kLanes * kRec)
  PE_REC(bnext, int32_t, r32, vrec, 20, kLanes * kRec)
  PE_REC(bprev, int32_t, r32, vrec, 24, kLanes * kRec)
  PE_REC(vpos, int32_t, r32, vrec, 28, kLanes * kRec)
  PE_REC(vr0, V4, r32, vrec, 0, kLanes * kRec)   // vhdr vref vaux uses
  PE_REC(vr1, V4, r32, vrec, 16, kLanes * kRec)  // slcnt bnext bprev vpos
  PE_REC(lo_buf, int32_t, r16, lrec, 0, kLanes * 16)
  PE_REC(lo_h, LowHead, r16, lrec, 0, kLanes * 16)
  PE_REC(adirect, int32_t, r32, arec, 0, kLanes * kRec)
  PE_REC(aslice, int32_t, r32, arec, 4, kLanes * kRec)
  PE_REC(awrapped, uint8_t, r32, arec, 8, kLanes * kRec)
  PE_REC(aspec0, uint32_t, r32, arec, 12, kLanes * kRec)
  PE_REC(alb0, int64_t, r32, arec, 16, kLanes * kRec)
  PE_REC(arg_spec, uint32_t, r32, arec, 24, kLanes * kRec)
  PE_REC(ar0, V4, r32, arec, 0, kLanes * kRec)
  PE_REC(lkind, uint8_t, r32, looprec, 0, kLanes * kRec)
  PE_REC(laxis, uint8_t, r32, looprec, 1, kLanes * kRec)
  PE_REC(ldim, int8_t, r32, looprec, 2, kLanes * kRec)
  PE_REC(lhead, int32_t, r32, looprec, 4, kLanes * kRec)
  PE_REC(ltail, int32_t, r32, looprec, 8, kLanes * kRec)
  PE_REC(lyield, int32_t, r32, looprec, 12, kLanes * kRec)
  PE_REC(ltype, int32_t, r32, looprec, 16, kLanes * kRec)
  PE_REC(lq0, V4, r32, looprec, 0, kLanes * kRec)   // kind|axis|dim, head, tail, yield
  PE_REC(lq1, V4, r32, looprec, 16, kLanes * kRec)  // result type
  PE_REC(em_head, int32_t, r32, emrec, 0, kLanes * kRec)
  PE_REC(em_op0, int32_t, r32, emrec, 4, kLanes * kRec)
  PE_REC(em_last, int32_t, r32, emrec, 8, kLanes * kRec)
  PE_REC(em_ooff, int32_t, r32, emrec, 12, kLanes * kRec)
  PE_REC(em_lb, int64_t, r32, emrec, 16, kLanes * kRec)
  PE_REC(delta, int64_t, r32, emrec, 24, kLanes * kRec)
  PE_REC(em_q0, V4, r32, emrec, 0, kLanes * kRec)      // head op0 last ooff
  PE_REC(em_q1, I64x2, r32, emrec, 16, kLanes * kRec)  // local bytes, delta
  PE_REC(em_spec, uint32_t, b4, em_spec, 0, kLanes * 4)  // final registered spec (trace)
  PE_REC(st8, int64_t, b8, st8, 0, kLanes * 8)
  PE_REC(st4, int32_t, b4, st4, 0, kLanes * 4)
  PE_REC(opnd, int32_t, b4, opnd, 0, kLanes * 4)
  PE_REC(fs, int32_t, b4, fs, 0, kLanes * 4)
  PE_REC(stk, int32_t, b4, stk, 0, kLanes * 4)
  PE_REC(em_opnd, int32_t, b4, em_opnd, 0, kLanes * 4)
  PE_REC(lg, int32_t, b4, lg, 0, kLanes * 4)
  PE_REC(carry, uint32_t, b4, carry, 0, kLanes * 4)
  PE_REC(dirty, uint32_t, b4, dirty, 0, kLanes * 4)
  PE_REC(rs, int32_t, b4, rs, 0, kLanes * 4)      // resurfaced ops, discovery order
  PE_REC(rsb, uint32_t, b4, rsb, 0, kLanes * 4)   // resurfaced-op bitmap
  PE_REC(seen, uint8_t, b1, seen, 0, kLanes * 1)
#undef PE_REC
};

#ifdef __CUDA_ARCH__
PE_HD int32_t pe_ctz(uint32_t x) { return __ffs((int)x) - 1; }
#else
PE_HD int32_t pe_ctz(uint32_t x) { return __builtin_ctz(x); }
#endif

PE_HD uint64_t align8(uint64_t x) { return (x + 7) & ~uint64_t(7); }
PE_HD uint64_t align128(uint64_t x) { return (x + 127) & ~uint64_t(127); }

inline Layout relayout(const GraphView& g, const Caps& caps, bool opnd_log);

// Host-side sizing.  The FULL layout's bounds are
// structural: every original op is pulled or migrated at most once, every
// value is tiled at most once.  The TIGHT layout is sized from measured
// high-water marks (slots ~ N+E, SPMD ops ~ 1.45 N on the 24-layer graph)
// with headroom; a candidate that overflows it reports PE_CAND_CAPACITY and
// is re-evaluated in a full-size arena by the retry kernel, so the tight
// layout changes memory footprint, never results.
inline Layout make_layout(const GraphView& g, bool tight = false) {
  Layout L{};
  int32_t A = g.A, N = g.N, E = g.E;
  int32_t K = A + N;               // action loops (each value tiled once)
  int32_t S = E + K;               // slices
  if (tight) {
    L.caps.V = A + 2 * N + E + 64;
    L.caps.L = N + 64;
    L.caps.FS = 2 * A + 4;
    L.caps.EM = (3 * (N + A)) / 2 + 256;
    L.caps.EO = E + L.caps.EM + 256;
  } else {
    L.caps.V = A + N + N + S + K + A + 8;
    L.caps.L = N + K + 4;
    L.caps.FS = 2 * A + 4;
    L.caps.EM = 3 * (N + S) + 2 * L.caps.L + A + 64;
    L.caps.EO = E + 2 * L.caps.EM + 64;
  }
  // (only the full-size arenas keep the SPMD operand log: parity traces run
  // in them)
  return relayout(g, L.caps, !tight);
}

// Byte offsets of every array of a group arena for the given capacities.
inline Layout relayout(const GraphView& g, const Caps& caps, bool opnd_log) {
  Layout L{};
  L.caps = caps;
  L.has_opnd = opnd_log ? 1u : 0u;
  int64_t A = g.A, N = g.N, E = g.E;
  uint64_t o = 0;
  auto take = [&](int64_t elems, int64_t elem_bytes) {
    uint64_t at = o;
    o = align128(o + (uint64_t)(elems + 1) * elem_bytes * kLanes);
    return at;
  };
  L.vrec = take(caps.V, kRec);
  L.lrec = take(caps.V, 16);
  L.arec = take(A, kRec);
  L.looprec = take(caps.L, kRec);
  L.emrec = take((int64_t)caps.EM + 1, kRec);
  L.opnd = take(E, 4);
  L.fs = take(caps.FS, 4);
  L.stk = take(2 * N, 4);
  L.seen = take(N, 1);
  L.em_opnd = take(opnd_log ? caps.EO : 0, 4);
  L.em_spec = take(opnd_log ? (int64_t)caps.EM + 1 : 0, 4);  // (trace only)
  L.st8 = take(2 * kMaxAxes, 8);
  L.st4 = take(3 * kMaxAxes, 4);
  L.carry = take(A / 32 + 1, 4);
  // legal list: static ordinals, plus every resurfaced op's when enabled
  L.lg = take(g.n_ord + (g.resurface ? N * kMaxRank * g.n_auto : 0), 4);
  L.dirty = take(N / 32 + 1, 4);
  L.rs = take(g.resurface ? N : 0, 4);
  L.rsb = take(g.resurface ? N / 32 + 1 : 0, 4);
  L.bytes = align128(o);
  return L;
}

// View of lane `lane` inside the group arena at `base`.
PE_HD Arena carve(const Layout& L, uint8_t* base, int lane = 0) {
  Arena a;
  a.L = &L;
  a.b1 = base + (uint64_t)lane;
  a.b4 = base + (uint64_t)lane * 4;
  a.b8 = base + (uint64_t)lane * 8;
  a.r16 = base + (uint64_t)lane * 16;
  a.r32 = base + (uint64_t)lane * kRec;
#ifdef PE_BOUNDS_CHECK
  a.lo = base;
  a.hi = base + L.bytes;
#endif
  return a;
}

// IEEE double helpers with explicit rounding (no FMA contraction) so the
// floating-point cost terms match the oracle bit-for-bit.
#ifdef __CUDA_ARCH__
PE_HD double dadd(double a, double b) { return __dadd_rn(a, b); }
PE_HD double dmul(double a, double b) { return __dmul_rn(a, b); }
PE_HD double ddiv(double a, double b) { return __ddiv_rn(a, b); }
#else
PE_HD double dadd(double a, double b) { volatile double r = a + b; return r; }
PE_HD double dmul(double a, double b) { volatile double r = a * b; return r; }
PE_HD double ddiv(double a, double b) { volatile double r = a / b; return r; }
#endif

// Lowered view of one value (REF spmd.cc:42-51 `Lowered`): buffer, spec
// word, acquired-in-loop mask (loops never nest, so acq is 0 or 1 per dim)
// and global shape.
//
// In the arena the global shape is not stored (16-byte records): it is the
// static shape of value gv with, per dim d, code (gx >> 2d) & 3 = 0 as is,
// 1 divided by, 2 multiplied by the size of axis (gx >> 8) & 3 -- a
// per-iteration copy divides its loop dim, an acquired sharded dim
// multiplies back (lower_base), and no other shapes arise.
struct Low {
  int32_t buf;
  uint32_t spec;
  uint32_t acq;
  int32_t gv;
  uint32_t gx;
};

struct Pull {
  int32_t ok;
  int32_t reason;
  int32_t cls;    // class index local to the op
  int32_t axis;
  int32_t drive;  // value slot of the driving loop
};

// Where a rollout starts: from init(), or from a saved
// propagated state (Cand::save) covering the first `done` decisions --
// `path`, recorded into the action output -- with the prefix applied from
// entry k0 on and `draws` RNG draws already consumed; the state after the
// whole prefix may be saved for later candidates (prefix-state cache,
// pe_state handles).
// Rollout features compiled into a kernel instantiation (the hot kernel's
// code size and register allocation bound its speed; the
// default launch carries neither): kFInferRest = InferRest actions / pauses,
// kFResume = start from / save saved states.
constexpr int kFInferRest = 1;
constexpr int kFResume = 2;
constexpr int kFAll = kFInferRest | kFResume;
// kFCoop: a whole warp runs ONE candidate (launches with one candidate per
// warp): every lane executes the sequential rewrite / lowering chain in
// lockstep on the same data (no divergence, broadcast loads, identical
// stores), and the data-parallel phases -- init(), the legal-set scan, the
// liveness sweep and its sums -- are split across the lanes (warp ballots,
// shuffle scans and reductions).
constexpr int kFCoop = 4;

PE_HD int32_t pe_lane() {
#ifdef __CUDA_ARCH__
  return (int32_t)(threadIdx.x & 31);
#else
  return 0;
#endif
}
PE_HD void pe_syncwarp() {
#ifdef __CUDA_ARCH__
  __syncwarp();
#endif
}

struct Resume {
  const uint8_t* snap = nullptr;
  int32_t done = 0;
  const pe_action* path = nullptr;
  int32_t k0 = 0;
  int32_t draws = 0;
  bool stop = false;       // (scheduling trie) its next draw is Stop
  uint8_t* save = nullptr;  // save the post-prefix state here ...
  uint8_t* saved = nullptr; // ... and set *saved = 1 once written
};

struct Cand {
  const GraphView& g;
  const Caps caps;
  Arena a;
  int32_t nslots, nloops, nfs, nem, neo, nstk;
  int32_t result_ref;
  int32_t pend;  // head of the pending-slice list (linked through vpos)
  int32_t nrs;   // resurfaced stuck ops (g.resurface)
  int32_t status;
  int64_t flops;
  int32_t result_buf;
  bool tracing = false;  // keep the full SPMD operand log (parity trace only)
#if defined(PE_PHASE_TIMERS) && defined(__CUDA_ARCH__)
  // profiling build only: clock64 cycles per phase
  // 0 init 1 apply 2 forward 3 backward 4 wrap 5 legal 6 analyze 7 lower 8 score
  long long ph[9];
  long long t_last;
  __device__ void tick_start() { t_last = clock64(); }
  __device__ void tick(int k) {
    long long t = clock64();
    ph[k] += t - t_last;
    t_last = t;
  }
#else
  PE_HD void tick_start() {}
  PE_HD void tick(int) {}
#endif

  PE_HD Cand(const GraphView& gv, const Layout& L, uint8_t* base, int lane = 0)
      : g(gv), caps(L.caps), a(carve(L, base, lane)) {
#if defined(PE_PHASE_TIMERS) && defined(__CUDA_ARCH__)
    for (int k = 0; k < 9; ++k) ph[k] = 0;
#endif
  }

  // ------------------------------------------------------------ helpers
  // (status codes are ordered: OK 0, ILLEGAL 1 < INTERNAL 2, CAPACITY 3)
  PE_HD void fail(int32_t st) {
    if (status < PE_CAND_INTERNAL) status = st;
  }
  PE_HD bool bad() const { return status >= PE_CAND_INTERNAL; }
  PE_HD int32_t NV() const { return g.A + g.N; }
  PE_HD int64_t asz(int32_t ax) const { return g.axis_size[ax]; }
  // VRec header word: vk | tile-loop flag << 8 | loop axis << 16 | loop dim << 24
  // (loop axis/dim denormalised into the value record so the sweeps test
  // "operand is a tile loop on (axis, dim)" with one load)
  PE_HD uint32_t vhdr(int32_t v) const { return a.vh()[v]; }
  PE_HD static bool hdr_tile(uint32_t h) { return (h & 0x1FFu) == (VK_LOOP | 0x100u); }
  PE_HD static int32_t hdr_axis(uint32_t h) { return (int32_t)((h >> 16) & 0xFFu); }
  PE_HD static int32_t hdr_dim(uint32_t h) { return (int32_t)(int8_t)(h >> 24); }
  PE_HD bool is_tile_loop(int32_t v) const { return hdr_tile(vhdr(v)); }
  // refresh the denormalised loop info of loop value v (loop record l)
  PE_HD void mark_loop_value(int32_t v, int32_t l) {
    uint32_t h = (uint32_t)VK_LOOP | ((a.lkind()[l] == LK_TILE ? 1u : 0u) << 8) |
                 ((uint32_t)a.laxis()[l] << 16) | ((uint32_t)(uint8_t)a.ldim()[l] << 24);
    a.vh()[v] = h;
  }
  // original value whose global shape a top-level value carries
  PE_HD int32_t shape_src(int32_t v) const {
    uint8_t k = a.vk()[v];
    if (k == VK_LOOP) return a.ltype()[a.vref()[v]];
    if (k == VK_ATOMIC) return a.vref()[v];
    return v;  // ARG / TOP
  }
  // a new value slot, written whole: header, vref, vaux, use count; no
  // slices, unlinked, no position
  PE_HD int32_t alloc_slot(uint32_t hdr, int32_t ref, int32_t aux, int32_t uses) {
    if (nslots >= caps.V) {
      fail(PE_CAND_CAPACITY);
      return -1;
    }
    int32_t s = nslots++;
    a.vr0()[s] = V4{(int32_t)hdr, ref, aux, uses};
    a.vr1()[s] = V4{0, -1, -1, 0};
    return s;
  }
  PE_HD static uint32_t loop_hdr(bool tile, int32_t axis, int32_t dim) {
    return (uint32_t)VK_LOOP | ((tile ? 1u : 0u) << 8) | ((uint32_t)(uint8_t)axis << 16) |
           ((uint32_t)(uint8_t)(int8_t)dim << 24);
  }
  // a new loop record, written whole: kind, axis, dim (-1 for sum loops),
  // empty body, no yield yet, result type
  PE_HD int32_t alloc_loop(int32_t kind, int32_t axis, int32_t dim, int32_t type) {
    if (nloops >= caps.L) {
      fail(PE_CAND_CAPACITY);
      return -1;
    }
    int32_t l = nloops++;
    a.lq0()[l] = V4{kind | (axis << 8) | ((int32_t)(uint8_t)(int8_t)dim << 16), -1, -1, -1};
    a.lq1()[l] = V4{type, 0, 0, 0};
    return l;
  }
  PE_HD void body_append(int32_t l, int32_t s) {
    a.bnext()[s] = -1;
    a.bprev()[s] = a.ltail()[l];
    if (a.ltail()[l] >= 0) a.bnext()[a.ltail()[l]] = s;
    else a.lhead()[l] = s;
    a.ltail()[l] = s;
  }
  PE_HD void body_insert_before(int32_t l, int32_t at, int32_t s) {
    int32_t p = a.bprev()[at];
    a.bprev()[s] = p;
    a.bnext()[s] = at;
    a.bprev()[at] = s;
    if (p >= 0) a.bnext()[p] = s;
    else a.lhead()[l] = s;
  }
  // Top-level order: even slot 2o is op o's own value
  // A+o (absent once DEAD), odd slot 2o+1 the action loop tiled right
  // after it, kept in vaux[A+o] (unused for top-level values; -1 = empty);
  // negative codes are front-stack entries.
  PE_HD void set_pos(int32_t v, int32_t code) {
    a.vpos()[v] = code;
    if (code >= 0) a.vaux()[g.A + (code >> 1)] = v;  // odd slots only
    else a.fs()[-code - 1] = v;
  }
  PE_HD void push_front(int32_t v) {
    if (nfs >= caps.FS) {
      fail(PE_CAND_CAPACITY);
      return;
    }
    set_pos(v, -(nfs + 1));
    nfs++;
  }
  // (callers mark v DEAD, which removes an even-slot value)
  PE_HD void clear_pos(int32_t v) {
    int32_t code = a.vpos()[v];
    if (code < 0) a.fs()[-code - 1] = -1;
    else if (code & 1) a.vaux()[g.A + (code >> 1)] = -1;
  }
  // REF rewrite.cc:27-38 replace_uses: every operand occurrence of an
  // original value lives in one of its original operand slots.
  PE_HD void replace_uses(int32_t v, int32_t t) {
    for (int32_t i = g.user_off[v]; i < g.user_off[v + 1]; ++i) {
      int32_t s = g.users[i];
      if (a.opnd()[s] == v) a.opnd()[s] = t;
    }
    if (result_ref == v) result_ref = t;
  }
  // Incremental sweeps.  A top-level op's pull decision
  // only changes when one of its operands becomes a tile loop, so forward()
  // visits just the ops marked here; a slice's migration check, once failed,
  // fails forever, so backward() checks each slice once, from the pending
  // list (slices are never top-level, so their vpos field is free for the
  // link).
  PE_HD void mark_users(int32_t v) {
    for (int32_t i = g.user_off[v]; i < g.user_off[v + 1]; ++i) {
      int32_t o = g.slot_op[g.users[i]];
      a.dirty()[o >> 5] |= 1u << (o & 31);
    }
  }
  PE_HD void push_pending(int32_t s) {
    a.vpos()[s] = pend;
    pend = s;
  }
  PE_HD void slice_created(int32_t u, int32_t d, int32_t axis) {
    a.slcnt()[u]++;
    if (u < g.A) {
      a.carry()[u >> 5] |= 1u << (u & 31);
      int32_t pair = d | (axis << 3);
      if (a.aslice()[u] == -1) a.aslice()[u] = pair;
      else if (a.aslice()[u] != pair) a.aslice()[u] = -2;
    }
  }
  PE_HD bool is_member(int32_t gc, int32_t k) const {
    for (int32_t m = g.cls_moff[gc]; m < g.cls_moff[gc + 1]; ++m)
      if ((g.mem[m] >> 2) == k) return true;
    return false;
  }

  // ------------------------------------------------------------ init
  // (ln, nl): this lane and the lanes sharing the candidate (kFCoop), or
  // (0, 1) for one lane per candidate
  PE_HD void init(int32_t ln = 0, int32_t nl = 1) {
    int32_t A = g.A, N = g.N;
    for (int32_t v = ln; v < A; v += nl) {
      a.vr0()[v] = V4{VK_ARG, v, 0, g.init_uses[v]};
      a.vr1()[v] = V4{0, -1, -1, 0};
      a.ar0()[v] = V4{0, -1, 0, 0};  // adirect, aslice, awrapped (+aspec0)
    }
    for (int32_t o = ln; o < N; o += nl) {
      int32_t v = A + o;
      a.vr0()[v] = V4{VK_TOP, o, -1, g.init_uses[v]};  // vaux: odd slot empty
      a.vr1()[v] = V4{0, -1, -1, 2 * o};
    }
    for (int32_t s = ln; s < g.E; s += nl) a.opnd()[s] = g.oopnd[s];
    for (int32_t w = ln; w <= (A >> 5); w += nl) a.carry()[w] = 0;
    for (int32_t w = ln; w <= (N >> 5); w += nl) a.dirty()[w] = 0;
    if (g.resurface)
      for (int32_t w = ln; w <= (N >> 5); w += nl) a.rsb()[w] = 0;
    if (nl > 1) pe_syncwarp();
    nrs = 0;
    pend = -1;
    nslots = A + N;
    nloops = 0;
    nfs = 0;
    nem = 0;
    neo = 0;
    nstk = 0;
    result_ref = g.result;
    status = PE_CAND_OK;
    flops = 0;
    result_buf = -1;
  }

  // ------------------------------------------------------------ snapshots
  // The state after a decision prefix (prefix-trie scheduling, DESIGN.md
  // §3.5), compact and lane-independent: what init() sets up and apply /
  // propagate write -- value, loop and argument records, operand slots,
  // front stack, carry bits, counters.  Lowering state is rebuilt by
  // lower(); after a whole propagate the dirty bits are clear and the
  // pending-slice list is empty.  (Engines with stuck resurfacing do not
  // schedule, so rs / rsb need no snapshot.)
  // A saved state is a DELTA against init(): the value records that
  // differ from their initial ones, every slot added after them, the loop
  // and argument records, the operand slots that were redirected, the front
  // stack and the carry bits.  Loading = init() + the delta, so starting
  // from a saved state never costs more than init() itself (a full copy of
  // a 52K-op state read ~3 MB per candidate and lost to replaying two
  // decisions).
  PE_HD static uint64_t snap_bytes(const GraphView& g, const Caps& caps) {
    return 16ull * (2 + 3ull * (uint64_t)(g.A + g.N) + 2ull * caps.V + 2ull * caps.L +
                    (uint64_t)g.A) +
           4ull * (2ull * (uint64_t)g.E + caps.FS + (uint64_t)(g.A >> 5) + 1);
  }
  PE_HD void init_records(int32_t v, V4& r0, V4& r1) const {
    if (v < g.A) {
      r0 = V4{VK_ARG, v, 0, g.init_uses[v]};
      r1 = V4{0, -1, -1, 0};
    } else {
      r0 = V4{VK_TOP, v - g.A, -1, g.init_uses[v]};
      r1 = V4{0, -1, -1, 2 * (v - g.A)};
    }
  }
  PE_HD static bool same(const V4& x, const V4& y) {
    return x.x == y.x && x.y == y.y && x.z == y.z && x.w == y.w;
  }
  PE_HD void save(uint8_t* dst) const {
    V4* p = reinterpret_cast<V4*>(dst);
    V4* head = p;
    p += 2;
    int32_t nch = 0;
    for (int32_t v = 0; v < g.A + g.N; ++v) {
      V4 r0 = a.vr0()[v], r1 = a.vr1()[v], i0, i1;
      init_records(v, i0, i1);
      if (same(r0, i0) && same(r1, i1)) continue;
      *p++ = V4{v, 0, 0, 0};
      *p++ = r0;
      *p++ = r1;
      ++nch;
    }
    for (int32_t v = g.A + g.N; v < nslots; ++v) {
      *p++ = a.vr0()[v];
      *p++ = a.vr1()[v];
    }
    for (int32_t l = 0; l < nloops; ++l) {
      *p++ = a.lq0()[l];
      *p++ = a.lq1()[l];
    }
    for (int32_t x = 0; x < g.A; ++x) *p++ = a.ar0()[x];
    int32_t* q = reinterpret_cast<int32_t*>(p);
    int32_t nop = 0;
    for (int32_t s = 0; s < g.E; ++s) {
      int32_t u = a.opnd()[s];
      if (u == g.oopnd[s]) continue;
      *q++ = s;
      *q++ = u;
      ++nop;
    }
    for (int32_t i = 0; i < nfs; ++i) *q++ = a.fs()[i];
    for (int32_t w = 0; w <= (g.A >> 5); ++w) *q++ = (int32_t)a.carry()[w];
    head[0] = V4{nslots, nloops, nfs, result_ref};
    head[1] = V4{nch, nop, 0, 0};
  }
  // init() for a candidate that starts from a saved prefix state; a state
  // saved from a full-size arena may not fit a tight one (CAPACITY: the
  // retry kernel loads it into a full-size arena)
  PE_HD void load(const uint8_t* src, int32_t ln = 0, int32_t nl = 1) {
    const V4* p = reinterpret_cast<const V4*>(src);
    V4 h = p[0], h2 = p[1];
    p += 2;
    init(ln, nl);
    if (h.x > caps.V || h.y > caps.L || h.z > caps.FS) {
      fail(PE_CAND_CAPACITY);
      return;
    }
    nslots = h.x;
    nloops = h.y;
    nfs = h.z;
    result_ref = h.w;
    for (int32_t k = 0; k < h2.x; ++k) {
      int32_t v = p->x;
      a.vr0()[v] = p[1];
      a.vr1()[v] = p[2];
      p += 3;
    }
    for (int32_t v = g.A + g.N; v < nslots; ++v) {
      a.vr0()[v] = *p++;
      a.vr1()[v] = *p++;
    }
    for (int32_t l = 0; l < nloops; ++l) {
      a.lq0()[l] = *p++;
      a.lq1()[l] = *p++;
    }
    for (int32_t x = 0; x < g.A; ++x) a.ar0()[x] = *p++;
    const int32_t* q = reinterpret_cast<const int32_t*>(p);
    for (int32_t k = 0; k < h2.y; ++k, q += 2) a.opnd()[q[0]] = q[1];
    for (int32_t i = 0; i < nfs; ++i) a.fs()[i] = *q++;
    for (int32_t w = 0; w <= (g.A >> 5); ++w) a.carry()[w] = (uint32_t)*q++;
    nrs = 0;
    pend = -1;
    nem = 0;
    neo = 0;
    nstk = 0;
    status = PE_CAND_OK;
    flops = 0;
    result_buf = -1;
  }

  // ------------------------------------------------------------ actions
  // carries_tiling (REF rewrite.cc:42-51) for an original value at top level
  PE_HD bool carries(int32_t v) const {
    if (a.vk()[v] == VK_LOOP) return true;
    if (a.slcnt()[v] > 0) return true;
    return v < g.A && a.awrapped()[v];
  }

  // apply_tile_action (REF rewrite.cc:61-113).  Returns false when illegal
  // (IllegalActionError); the state is untouched in that case.
  PE_HD bool apply_tile(int32_t v, int32_t dim, int32_t axis) {
    if (v < 0 || v >= NV()) return false;
    uint8_t k = a.vk()[v];
    if (k != VK_ARG && k != VK_TOP && k != VK_LOOP) return false;  // erased: does not exist
    if (axis < 0 || axis >= g.n_axes) return false;
    if (dim < 0 || dim >= g.vrank[v]) return false;
    if (g.amod((uint32_t)g.shape(v)[dim], axis) != 0) return false;
    if (carries(v)) return false;
    int32_t l = alloc_loop(LK_TILE, axis, dim, v);
    int32_t ls = l < 0 ? -1 : alloc_slot(loop_hdr(true, axis, dim), l, 0, a.uses()[v]);
    int32_t s = ls < 0 ? -1 : alloc_slot(VK_SLICE, v, dim | (l << 3), 1);  // used by the yield
    if (bad()) return false;
    a.lyield()[l] = s;
    body_append(l, s);
    push_pending(s);
    a.uses()[v] = 1;  // the slice
    slice_created(v, dim, axis);
    replace_uses(v, ls);
    mark_users(v);
    if (v < g.A) push_front(ls);
    else set_pos(ls, 2 * (v - g.A) + 1);
    return !bad();
  }

  PE_HD bool apply_action(const pe_action& act) {
    if (act.kind == PE_ACT_TILE) return apply_tile((int32_t)act.value, act.dim, act.axis);
    if (act.kind == PE_ACT_TILE_GROUP) {
      if ((int32_t)act.value >= g.n_groups) return false;
      int32_t applied = 0;
      for (int32_t i = g.grp_off[act.value]; i < g.grp_off[act.value + 1]; ++i) {
        if (apply_tile(g.grp_mem[i], act.dim, act.axis)) ++applied;
        if (bad()) return false;
      }
      return applied > 0;
    }
    return false;  // INFER_REST not supported by this engine version
  }

  // ------------------------------------------------------------ forward
  // plan_pull (REF propagate.cc:92-144) for a top-level base op.
  PE_HD Pull plan_pull(int32_t o) const {
    Pull p;
    p.ok = 0;
    p.reason = R_NONE;
    p.cls = -1;
    p.axis = -1;
    p.drive = -1;
    int32_t base = g.oopnd_off[o], n = g.oopnd_off[o + 1] - base;
    int32_t cbase = g.ocls_off[o];
    for (int32_t k = 0; k < n; ++k) {
      int32_t u = a.opnd()[base + k];
      uint32_t h = vhdr(u);
      if (!hdr_tile(h)) continue;
      int32_t c = g.slot_cls[(base + k) * 4 + hdr_dim(h)];
      if (c < 0 || g.cls_role[cbase + c] == kBlocked) {
        p.reason = R_BLOCKED;
        return p;
      }
      if (p.drive < 0) {
        p.drive = u;
        p.cls = c;
        p.axis = hdr_axis(h);
      }
    }
    if (p.drive < 0) return p;
    for (int32_t k = 0; k < n; ++k) {
      uint32_t h = vhdr(a.opnd()[base + k]);
      if (!hdr_tile(h)) continue;
      if (hdr_axis(h) == p.axis && g.slot_cls[(base + k) * 4 + hdr_dim(h)] != p.cls) {
        p.reason = R_CONFLICT;
        return p;
      }
    }
    int32_t gc = cbase + p.cls;
    for (int32_t m = g.cls_moff[gc]; m < g.cls_moff[gc + 1]; ++m) {
      int32_t k = g.mem[m] >> 2, d = g.mem[m] & 3;
      int32_t u = a.opnd()[base + k];
      if (g.amod((uint32_t)g.shape(shape_src(u))[d], p.axis) != 0) {
        p.reason = R_INSUFFICIENT;
        return p;
      }
      uint32_t h = vhdr(u);
      if (hdr_tile(h)) {
        bool sa = hdr_axis(h) == p.axis, sd = hdr_dim(h) == d;
        if (sa != sd) {
          p.reason = R_CONFLICT;
          return p;
        }
      }
    }
    p.ok = 1;
    return p;
  }

  PE_HD bool has_tiled_operand(int32_t o) const {
    for (int32_t s = g.oopnd_off[o]; s < g.oopnd_off[o + 1]; ++s)
      if (is_tile_loop(a.opnd()[s])) return true;
    return false;
  }

  // The rewrite of REF propagate.cc:194-247 (extend a single-use tile loop,
  // or a fresh tile / sum loop at X's slot) + build_sliced_consumer
  // (:149-180, slices deduplicated per (operand, dim)).
  PE_HD void pull(int32_t o, const Pull& p) {
    int32_t base = g.oopnd_off[o], n = g.oopnd_off[o + 1] - base;
    int32_t gc = g.ocls_off[o] + p.cls;
    bool contracting = g.cls_role[gc] == kContract;
    int32_t rd = g.cls_rdim[gc];
    int32_t lv0 = p.drive;
    bool extend = !contracting && a.uses()[lv0] == 1;
    int32_t l = extend ? a.vref()[lv0]
                       : alloc_loop(contracting ? LK_SUM : LK_TILE, p.axis, contracting ? -1 : rd,
                                    g.A + o);
    int32_t f = l < 0 ? -1 : alloc_slot(VK_LOCAL, o, (contracting ? 0 : rd + 1) | (l << 3), 1);
    if (bad()) return;
    // slice dedup per (operand, dim): a two-entry cache in registers, then
    // a search over this op's earlier members (already rewritten to slices)
    int32_t c0u = -1, c0d = 0, c0s = -1, c1u = -1, c1d = 0, c1s = -1;
    int32_t nc = 0;
    for (int32_t m = g.cls_moff[gc]; m < g.cls_moff[gc + 1]; ++m) {
      int32_t k = g.mem[m] >> 2, d = g.mem[m] & 3;
      int32_t ps = base + k;
      int32_t u = a.opnd()[ps];
      if (extend && u == lv0) {
        int32_t y = a.lyield()[l];
        a.opnd()[ps] = y;
        a.uses()[lv0]--;
        a.uses()[y]++;
        continue;
      }
      int32_t sl = c0u == u && c0d == d ? c0s : c1u == u && c1d == d ? c1s : -1;
      if (sl < 0) {
        // search fallback once the cache is full
        for (int32_t q = g.cls_moff[gc]; q < m && sl < 0 && nc >= 2; ++q) {
          int32_t k2 = g.mem[q] >> 2, d2 = g.mem[q] & 3;
          int32_t s2 = a.opnd()[base + k2];
          if (d2 == d && a.vk()[s2] == VK_SLICE && a.vref()[s2] == u &&
              (a.vaux()[s2] >> 3) == l && (a.vaux()[s2] & 7) == d)
            sl = s2;
        }
      }
      if (sl < 0) {
        // a new slice takes this operand's use of u: u's count is
        // unchanged (+1 slice, -1 operand slot), the slice has one use
        sl = alloc_slot(VK_SLICE, u, d | (l << 3), 1);
        if (bad()) return;
        body_append(l, sl);
        push_pending(sl);
        slice_created(u, d, p.axis);
        if (nc == 0) {
          c0u = u;
          c0d = d;
          c0s = sl;
          nc = 1;
        } else if (nc == 1) {
          c1u = u;
          c1d = d;
          c1s = sl;
          nc = 2;
        }
      } else {
        a.uses()[u]--;
        a.uses()[sl]++;
      }
      a.opnd()[ps] = sl;
    }
    for (int32_t k = 0; k < n; ++k) {
      int32_t u = a.opnd()[base + k];
      if (a.vk()[u] == VK_ARG && !is_member(gc, k)) a.adirect()[u]++;
    }
    if (extend) a.uses()[a.lyield()[l]]--;  // old yield is no longer yielded
    a.lyield()[l] = f;
    body_append(l, f);
    a.ltype()[l] = g.A + o;
    if (extend) {
      a.ldim()[l] = (int8_t)rd;
      clear_pos(lv0);
      a.vk()[lv0] = VK_DEAD;
    }
    int32_t xv = g.A + o;
    a.vref()[xv] = l;
    a.vh()[xv] = loop_hdr(!contracting, p.axis, contracting ? -1 : rd);
    mark_users(xv);
  }

  // REF propagate.cc:250-280: one in-order sweep over the top-level ops,
  // restricted to the ops whose operands changed (users are always later
  // in program order, so the sweep never has to look back).
  //
  // On the device the lanes that enter together step through the union of
  // their dirty ops in lockstep: each iteration takes the warp-wide
  // smallest next op, and the lanes holding it pull it together (same op,
  // same rule tables, one code path) while the others wait.  Each lane
  // still visits its own dirty ops in increasing order, so the result is
  // the sequential sweep's.  A lane that fails keeps taking part with no
  // op until every lane is done (the reduction needs all of them).
  PE_HD void forward() {
    int32_t nw = (g.N >> 5) + 1;
    int32_t w = 0;
    bool done = false;
#ifdef __CUDA_ARCH__
    const unsigned mask = __activemask();
#endif
    while (true) {
      int32_t mine = INT32_MAX;
      uint32_t bits = 0;
      if (!done) {
        while (w < nw && (bits = a.dirty()[w]) == 0) ++w;
        if (w < nw) mine = (w << 5) + pe_ctz(bits);
        else done = true;
      }
#ifdef __CUDA_ARCH__
      int32_t m = __reduce_min_sync(mask, mine);
#else
      int32_t m = mine;
#endif
      if (m == INT32_MAX) break;
      if (mine != m) continue;
      a.dirty()[w] = bits & (bits - 1);
      int32_t o = m;
      if (a.vk()[g.A + o] != VK_TOP) continue;
      // plan_pull sees every tiled operand: it either found a driving one
      // or stopped, blocked, at one -- no separate has_tiled_operand scan
      Pull p = plan_pull(o);
      if (p.drive < 0 && p.reason != R_BLOCKED) continue;  // no tiled operand
      if (g.orule_err[o]) {
        fail(PE_CAND_INTERNAL);
        done = true;
        continue;
      }
      if (!p.ok) continue;
      pull(o, p);
      if (bad()) done = true;
    }
  }

  // ------------------------------------------------------------ backward
  // REF propagate.cc:284-375: migrate the single-use producer of a sliced
  // value into the consuming loop.  The reference re-walks every loop body
  // each sweep; here each slice is checked once, when it is new.  Every
  // failure is permanent (the producer stays non-TOP, keeps >= 2 uses, or
  // keeps a non-divisible / conflicting member), and migrations of
  // different slices commute (each inserts at its own slice's position and
  // touches only its producer's operands), so the pending order is free.
  PE_HD void backward_slice(int32_t s) {
    {
      int32_t l = a.vaux()[s] >> 3;
      int32_t sz_axis = a.laxis()[l];
      {
        int32_t u = a.vref()[s];
        int32_t d = a.vaux()[s] & 7;
        if (a.vk()[u] == VK_TOP && a.uses()[u] == 1) {
          int32_t P = a.vref()[u];
          uint8_t kind = g.okind[P];
          int32_t pb = g.oopnd_off[P], pn = g.oopnd_off[P + 1] - pb;
          bool simple = kind == kConstant ||
                        (kind == kBroadcastInDim && !((g.omask[P] >> d) & 1));
          bool go = true;
          int32_t gc = -1;
          if (!simple) {
            if (g.orule_err[P]) {
              fail(PE_CAND_INTERNAL);
              return;
            }
            int32_t rc = g.op_rcls[P * 4 + d];
            if (rc < 0) {
              go = false;
            } else {
              gc = g.ocls_off[P] + rc;
              for (int32_t m = g.cls_moff[gc]; m < g.cls_moff[gc + 1]; ++m) {
                int32_t k = g.mem[m] >> 2, dd = g.mem[m] & 3;
                int32_t w = a.opnd()[pb + k];
                if (g.amod((uint32_t)g.shape(shape_src(w))[dd], sz_axis) != 0) go = false;
                uint32_t h = vhdr(w);
                if (hdr_tile(h)) {
                  bool sa = hdr_axis(h) == sz_axis, sd = hdr_dim(h) == dd;
                  if (sa != sd) go = false;
                }
              }
            }
          }
          if (go) {
            if (!simple) {
              int32_t c0u = -1, c0d = 0, c0s = -1, c1u = -1, c1d = 0, c1s = -1;
              int32_t nc = 0;
              for (int32_t m = g.cls_moff[gc]; m < g.cls_moff[gc + 1]; ++m) {
                int32_t k = g.mem[m] >> 2, dd = g.mem[m] & 3;
                int32_t w = a.opnd()[pb + k];
                int32_t sl = c0u == w && c0d == dd ? c0s : c1u == w && c1d == dd ? c1s : -1;
                if (sl < 0 && nc >= 2) {
                  for (int32_t q = g.cls_moff[gc]; q < m && sl < 0; ++q) {
                    int32_t k2 = g.mem[q] >> 2, d2 = g.mem[q] & 3;
                    int32_t s2 = a.opnd()[pb + k2];
                    if (d2 == dd && a.vk()[s2] == VK_SLICE && a.vref()[s2] == w &&
                        (a.vaux()[s2] >> 3) == l)
                      sl = s2;
                  }
                }
                if (sl < 0) {
                  // takes this operand's use of w (count unchanged)
                  sl = alloc_slot(VK_SLICE, w, dd | (l << 3), 1);
                  if (bad()) return;
                  body_insert_before(l, s, sl);
                  push_pending(sl);
                  slice_created(w, dd, sz_axis);
                  if (nc == 0) {
                    c0u = w;
                    c0d = dd;
                    c0s = sl;
                    nc = 1;
                  } else if (nc == 1) {
                    c1u = w;
                    c1d = dd;
                    c1s = sl;
                    nc = 2;
                  }
                } else {
                  a.uses()[w]--;
                  a.uses()[sl]++;
                }
                a.opnd()[pb + k] = sl;
              }
            }
            for (int32_t k = 0; k < pn; ++k) {
              int32_t w = a.opnd()[pb + k];
              if (a.vk()[w] == VK_ARG && (simple || !is_member(gc, k))) a.adirect()[w]++;
            }
            // the slice becomes P's per-iteration copy (it keeps S's name)
            a.vk()[s] = VK_LOCAL;
            a.vref()[s] = P;
            a.vaux()[s] = (d + 1) | (l << 3);
            a.slcnt()[u]--;
            clear_pos(u);
            a.vk()[u] = VK_DEAD;
          }
        }
      }
    }
  }

  // Visits the top-level values in program order: the front stack (most
  // recent first), then per op o its own value A+o (even slot, absent once
  // DEAD) and the action loop tiled right after it (odd slot).
  //
  // The op walk is a loop of its own, entered by all lanes together after
  // the front stack, so the lanes of a warp visit the same op in the same
  // iteration (same kind, same code path, same graph data): a single merged
  // loop over both sources offsets every lane by its front-stack length and
  // measured 1.14M -> 0.81M cand/s.  The even/odd pair is a
  // non-unrolled inner loop so f is inlined once for the op walk.
  template <typename F>
  PE_HD void for_top(F&& f) {
    for (int32_t i = nfs - 1; i >= 0; --i) {
      int32_t v = a.fs()[i];
      if (v >= 0) {
        f(v);
        if (bad()) return;
      }
    }
    for (int32_t o = 0; o < g.N; ++o) {
      V4 q = a.vr0()[g.A + o];  // header, vref, vaux = odd-slot occupant
      int32_t even = (q.x & 0xFF) != VK_DEAD ? g.A + o : -1;
#pragma unroll 1
      for (int32_t h = 0; h < 2; ++h) {
        int32_t v = h == 0 ? even : q.z;
        if (v < 0) continue;
        f(v);
        if (bad()) return;
      }
    }
  }

  PE_HD void backward() {
    while (pend >= 0) {
      int32_t s = pend;
      pend = a.vpos()[s];
      if (a.vk()[s] != VK_SLICE) continue;
      backward_slice(s);
      if (bad()) return;
    }
  }

  // wrap_replicated_args (REF propagate.cc:385-408): arguments used directly
  // inside a loop and never sliced are wrapped atomic, each at index 0.
  PE_HD void wrap() {
    for (int32_t x = 0; x < g.A; ++x) {
      if (a.adirect()[x] == 0 || a.slcnt()[x] != 0 || a.awrapped()[x]) continue;
      int32_t t = alloc_slot(VK_ATOMIC, x, 0, a.uses()[x]);
      if (bad()) return;
      replace_uses(x, t);
      a.uses()[x] = 1;
      a.awrapped()[x] = 1;
      a.carry()[x >> 5] |= 1u << (x & 31);
      push_front(t);
      if (bad()) return;
    }
  }

  PE_HD void propagate() {
    tick(1);
    forward();
    tick(2);
    if (bad()) return;
    backward();
    tick(3);
    if (bad()) return;
    wrap();
    tick(4);
  }

  // stuck analysis (REF propagate.cc:412-454), dedup by op id in discovery
  // order (:477-479).
  PE_HD void add_stuck(int32_t o, int32_t r) {
    if (a.seen()[o]) return;
    a.seen()[o] = 1;
    a.stk()[2 * nstk] = o;
    a.stk()[2 * nstk + 1] = r;
    nstk++;
  }
  // Stuck analysis (REF propagate.cc:412-454) of one loop-body slice:
  // a single-use TOP producer whose rule blocks the sliced dim.
  PE_HD void stuck_slice(int32_t s) {
    int32_t u = a.vref()[s], d = a.vaux()[s] & 7;
    if (a.vk()[u] != VK_TOP) return;
    int32_t P = a.vref()[u];
    uint8_t kind = g.okind[P];
    if (kind == kConstant) return;
    if (a.uses()[u] != 1) return;
    if (kind == kBroadcastInDim && !((g.omask[P] >> d) & 1)) return;
    if (g.orule_err[P]) {
      fail(PE_CAND_INTERNAL);
      return;
    }
    if (g.op_rcls[P * 4 + d] < 0) add_stuck(P, R_BLOCKED);
  }
  // ... and of one top-level op with a tiled operand that cannot be pulled
  PE_HD void stuck_top(int32_t v) {
    int32_t o = a.vref()[v];
    Pull p = plan_pull(o);
    if (p.drive < 0 && p.reason != R_BLOCKED) return;  // no tiled operand
    if (g.orule_err[o]) {
      fail(PE_CAND_INTERNAL);
      return;
    }
    if (p.ok) {
      fail(PE_CAND_INTERNAL);  // "pull available after fixpoint"
      return;
    }
    add_stuck(o, p.reason);
  }
  // The stuck list as its own walk (the resurfacing kernel; finish() folds
  // the same checks into lowering's walk).  `seen` is all-zero between uses
  // (arenas start zeroed; clear_seen() after the list is consumed).
  PE_HD void analyze() {
    nstk = 0;
    for_top([&](int32_t v) {
      uint8_t k = a.vk()[v];
      if (k == VK_LOOP) {
        int32_t l = a.vref()[v];
        for (int32_t s = a.lhead()[l]; s >= 0; s = a.bnext()[s]) {
          if (a.vk()[s] != VK_SLICE) continue;
          stuck_slice(s);
          if (bad()) return;
        }
      } else if (k == VK_TOP) {
        stuck_top(v);
      }
    });
  }
  PE_HD void clear_seen() {
    for (int32_t i = 0; i < nstk; ++i) a.seen()[a.stk()[2 * i]] = 0;
  }


  // ------------------------------------------------------------ lowering
  PE_HD int32_t rank_of_spec(uint32_t spec) const { return (spec >> 24) & 7; }
  // local_shape (REF mesh.cc:110-124): global dim / axis size, InternalError
  // when not divisible.  Branch-free (an unsharded dim divides by 1): after
  // a failure the candidate's outputs are discarded (finish), so only the
  // status matters, not the quotient returned alongside it.
  // global dim d of a record, from its shape code (Low)
  PE_HD uint32_t gdim(const Low& w, int d) const {
    uint32_t x = (uint32_t)g.shape(w.gv)[d], c = (w.gx >> (2 * d)) & 3u;
    uint32_t ax1 = ((w.gx >> 8) & 3u) + 1u;
    return c == 0 ? x : c == 1 ? g.quo1(x, ax1) : x * g.axis_sz32[ax1];
  }
  PE_HD int64_t local_dim(const Low& w, int d) {
    uint32_t ax1 = spec_axis(w.spec, d);
    uint32_t x = gdim(w, d);
    uint32_t q = g.quo1(x, ax1);
    if (x != q * g.axis_sz32[ax1]) fail(PE_CAND_INTERNAL);
    return q;
  }
  PE_HD int64_t local_elems(const Low& w) {
    int64_t e = 1;
    uint32_t rem = 0;
    int r = rank_of_spec(w.spec);
#pragma unroll
    for (int d = 0; d < kMaxRank; ++d) {
      uint32_t ax1 = spec_axis(w.spec, d);
      bool in = d < r;
      uint32_t x = in ? gdim(w, d) : 0u;
      uint32_t q = g.quo1(x, ax1);
      rem |= in ? x - q * g.axis_sz32[ax1] : 0u;
      e *= in ? (int64_t)q : 1;
    }
    if (rem) fail(PE_CAND_INTERNAL);
    return e;
  }
  PE_HD int64_t global_bytes(const Low& w) const {
    int64_t e = 4;
    int r = rank_of_spec(w.spec);
    for (int d = 0; d < r; ++d) e *= gdim(w, d);
    return e;
  }
  PE_HD Low load(int32_t v) const {
    Low w;
    LowHead h = a.lo_h()[v];
    w.buf = h.buf;
    w.spec = h.spec;
    w.acq = h.aux & 0xFu;
    w.gx = h.aux >> 4;
    w.gv = h.gv;
    return w;
  }
  PE_HD void store(int32_t v, const Low& w) {
    LowHead h;
    h.buf = w.buf;
    h.spec = w.spec;
    h.aux = w.acq | (w.gx << 4);
    h.gv = w.gv;
    a.lo_h()[v] = h;
  }
  // register_type (REF spmd.cc): the buffer's final DistType.  Only the
  // parity trace reads it: collective_stats takes each operand's type at
  // the collective's emission (emit_coll), which is its final one -- a
  // buffer is re-registered only by finish_loop for its loop's yield, the
  // last item of the body, so no collective consumed it earlier, or, when
  // the yield is a slice that kept its source's sharded buffer, with the
  // identical type.
  PE_HD void note_type(int32_t buf, uint32_t spec) {
    if (!tracing) return;
    if (buf < g.A) a.arg_spec()[buf] = spec;
    else a.em_spec()[buf - g.A] = spec;
  }
  // opens an SPMD op (first operand op0 or -1, local result bytes lb; the
  // record's first 32 bytes are written whole); operands are then appended
  // with add_operand
  PE_HD int32_t new_op(int32_t kind, int32_t axis, int32_t dim, int32_t nopnd, int32_t op0,
                       int64_t lb) {
    if (nem >= caps.EM || neo + nopnd > caps.EO) {
      fail(PE_CAND_CAPACITY);
      return -1;
    }
    int32_t j = nem++;
    a.em_q0()[j] = V4{kind | ((axis + 1) << 8) | ((dim + 1) << 12) | (nopnd << 16), op0, j, neo};
    a.em_q1()[j] = I64x2{lb, lb};  // liveness delta starts at +lb (def at j)
    return j;
  }
  PE_HD void add_operand(int32_t j, int32_t buf) {
    if (tracing) a.em_opnd()[neo] = buf;
    ++neo;
    // ops are emitted in order, so the current op is always the latest use
#ifndef PE_EXP_NO_LAST
    if (buf >= g.A) a.em_last()[buf - g.A] = j;
#endif
  }
  // pending_sum.front(): the pending axis with the smallest name (table
  // over the 4-bit pending mask, GraphView::pend_front)
  PE_HD int32_t pending_front(uint32_t spec) const { return g.pend_front[spec_pending(spec)]; }
  // emit_gather (REF spmd.cc:85-99) of dim d over axis ax,
  // emit_all_reduce (REF spmd.cc:102-114) over axis ax (d = -1), or the
  // slice_by_coord of lower_slice_axis (REF spmd.cc:240-252) of dim d by the
  // loop axis ax; updates the record in place.  One function for the three
  // so each emitting loop inlines a single copy (code size).
  PE_HD void emit_coll(Low& w, int32_t kind, int32_t ax, int d) {
    int32_t src = w.buf;
    // collective_stats (REF spmd.cc:405-434) on the operand's type, which
    // is final at emission (note_type): all_reduce bytes = its global
    // bytes, all_gather bytes = its local bytes x (axis size - 1)
    if (kind == kAllReduce) {
      a.st8()[ax] += global_bytes(w);
      a.st4()[ax]++;
    } else if (kind == kAllGather) {
      a.st8()[kMaxAxes + ax] += 4 * local_elems(w) * (asz(ax) - 1);
      a.st4()[kMaxAxes + ax]++;
    } else {
      a.st4()[2 * kMaxAxes + ax]++;
    }
    if (kind == kAllGather) {
      w.spec = spec_set_axis(w.spec, d, 0);
      w.acq &= ~(1u << d);
    } else if (kind == kAllReduce) {
      w.spec &= ~(1u << (16 + ax));
    } else {
      w.spec = spec_set_axis(w.spec, d, (uint32_t)(ax + 1));
      w.acq |= 1u << d;
    }
    int64_t lb = 4 * local_elems(w);
    int32_t j = new_op(kind, ax, d, 1, src, lb);
    if (j < 0) return;
    add_operand(j, src);
    w.buf = g.A + j;
    note_type(w.buf, w.spec);
  }
  PE_HD void emit_all_reduce(Low& w, int32_t ax) { emit_coll(w, kAllReduce, ax, -1); }
  // materialize_for_direct_use (REF spmd.cc:119-129); loop_axis = -1 at top.
  // Gathers every sharded dim in increasing order (a dim sharded by the
  // enclosing loop's axis and acquired in it stays), then all-reduces the
  // pending axes in name order -- one emission per iteration.
  PE_HD Low materialize(int32_t v, int32_t loop_axis) {
    Low w = load(v);
    if ((w.spec & 0x000FFFFFu) == 0) return w;  // replicated, nothing pending
    int32_t b0 = w.buf;
    int r = rank_of_spec(w.spec);
    while (true) {
      int32_t ax = -1, dd = -1;
#pragma unroll 1
      for (int d = 0; d < r; ++d) {
        uint32_t ax1 = spec_axis(w.spec, d);
        if (!ax1) continue;
        bool live = loop_axis >= 0 && (int32_t)ax1 - 1 == loop_axis && ((w.acq >> d) & 1);
        if (!live) {
          dd = d;
          ax = (int32_t)ax1 - 1;
          break;
        }
      }
      if (dd < 0) {
        if (!spec_pending(w.spec)) break;
        ax = pending_front(w.spec);
      }
      emit_coll(w, dd >= 0 ? kAllGather : kAllReduce, ax, dd);
      if (bad()) return w;
    }
    // every gather / all_reduce moves the record to a new buffer
    if (w.buf != b0) store(v, w);
    return w;
  }

  // lower_base (REF spmd.cc:256-323 with patch B) for a top-level op
  // (l = -1) or a per-iteration copy in loop l.  The first two operand
  // records are kept in registers after materialisation (every kind but
  // concatenate has <= 2 operands).
  PE_HD void lower_base(int32_t v, int32_t o, int32_t l) {
    int32_t base = g.oopnd_off[o], n = g.oopnd_off[o + 1] - base;
    int32_t lax = l >= 0 ? (int32_t)a.laxis()[l] : -1;
    uint8_t kind = g.okind[o];
    Low r;
    int32_t xv = g.A + o;
    int rank = g.vrank[xv];
    r.gv = xv;
    r.gx = 0;
    if (l >= 0) {
      int32_t dd = (a.vaux()[v] & 7) - 1;
      if (dd >= 0) r.gx = (1u << (2 * dd)) | ((uint32_t)lax << 8);
    }
    r.spec = (uint32_t)rank << 24;
    r.acq = 0;
    r.buf = -1;
    // Each operand is materialised and its sharding absorbed into the
    // result in one pass (the reference materialises all operands first;
    // a later operand's materialisation never changes an earlier operand's
    // record -- a repeated operand, mul(x, x), finds its record already
    // materialised -- so the order is immaterial).  The records stay in
    // their LowRecs; the operand buffers are re-read below.
    // flops on LOCAL operand shapes, taken from the
    // materialised records as they pass: dot = 2 * lhs elements * rhs free
    // dims (omask), reduce = input elements
    bool red = kind == kReduceSum || kind == kReduceMax;
    int64_t fl = kind == kDot ? 2 : 1;
#pragma unroll 1
    for (int32_t k = 0; k < n; ++k) {
      Low w = materialize(a.opnd()[base + k], lax);
      if (bad()) return;
      r.spec |= spec_pending(w.spec) << 16;
      if (kind == kConstant) continue;
      int wr = rank_of_spec(w.spec);
      if ((kind == kDot && k < 2) || (red && k == 0)) {
        uint32_t m = k == 0 ? 0xFu : g.omask[o];
#pragma unroll 1
        for (int d = 0; d < wr; ++d)
          if ((m >> d) & 1) fl *= local_dim(w, d);
      }
      if ((w.spec & 0xFFFFu) == 0) continue;  // no sharded dim
      ReshapeRule rr;
      if (kind == kReshape) {
        int64_t in[kMaxRank];
        for (int d = 0; d < wr; ++d) in[d] = local_dim(w, d);
        int32_t pit[kMaxRank];
        for (int d = 0; d < kMaxRank; ++d) pit[d] = (int32_t)gdim(r, d);
        rr = reshape_rule(in, wr, pit, rank);
        if (rr.error) {
          fail(PE_CAND_INTERNAL);
          return;
        }
      }
      for (int d = 0; d < wr; ++d) {
        uint32_t ax1 = spec_axis(w.spec, d);
        if (!ax1) continue;
        int role, rdim;
        if (kind == kReshape) {
          int c = rr.cls_of_dim[d];
          if (c < 0) {
            fail(PE_CAND_INTERNAL);
            return;
          }
          role = rr.role[c];
          rdim = rr.rdim[c];
        } else {
          int c = g.slot_cls[(base + k) * 4 + d];
          if (c < 0) {
            fail(PE_CAND_INTERNAL);
            return;
          }
          role = g.cls_role[g.ocls_off[o] + c];
          rdim = g.cls_rdim[g.ocls_off[o] + c];
        }
        if (role == kPass) {
          uint32_t cur = spec_axis(r.spec, rdim);
          if (cur && cur != ax1) {
            fail(PE_CAND_INTERNAL);
            return;
          }
          r.spec = spec_set_axis(r.spec, rdim, ax1);
          r.acq = (r.acq & ~(1u << rdim)) | (((w.acq >> d) & 1) << rdim);
        } else if (role == kBlocked) {
          fail(PE_CAND_INTERNAL);
          return;
        }
      }
    }
    // r.g holds the per-iteration (local) shape here; a sharded dim becomes
    // local * axis size.  So the local element count is the product of the
    // per-iteration dims (exact: no division, never a divisibility failure)
    // and the global bytes are 4 * local * the sharded dims' axis sizes.
    int64_t out_elems = 1, gmul = 1;
#pragma unroll
    for (int d = 0; d < kMaxRank; ++d) {
      if (d >= rank) break;
      out_elems *= gdim(r, d);
      uint32_t ax1 = spec_axis(r.spec, d);
      if (ax1) {
        int64_t sz = asz(ax1 - 1);
        gmul *= sz;
        // shape code: a divided dim is restored, any other multiplied; one
        // axis per code (inside a loop every sharded dim is by its axis)
        uint32_t c = (r.gx >> (2 * d)) & 3u;
        if ((r.gx & 0xFFu) != 0 && ((r.gx >> 8) & 3u) != ax1 - 1) fail(PE_CAND_CAPACITY);
        r.gx = (r.gx & ~(3u << (2 * d)) & 0xFFu) | ((c == 1 ? 0u : 2u) << (2 * d)) |
               ((ax1 - 1) << 8);
      }
    }
    int32_t j = new_op(kind, -1, -1, n, n > 0 ? a.lo_buf()[a.opnd()[base]] : -1, 4 * out_elems);
    if (j < 0) return;
#pragma unroll 1
    for (int32_t k = 0; k < n; ++k) add_operand(j, a.lo_buf()[a.opnd()[base + k]]);
    switch (kind) {
      case kDot: case kReduceSum: case kReduceMax:
        flops += fl;
        break;
      case kAdd: case kSub: case kMul: case kDiv: case kMaximum:
      case kNeg: case kExp: case kTanh: case kRsqrt:
        flops += out_elems;
        break;
      default:
        break;
    }
    r.buf = g.A + j;
    note_type(r.buf, r.spec);
    store(v, r);
  }

  // lower_slice_axis (REF spmd.cc:206-254)
  PE_HD void lower_slice(int32_t s, int32_t l) {
    int32_t lax = a.laxis()[l];
    int32_t u = a.vref()[s];
    int d = a.vaux()[s] & 7;
    Low src = load(u);
    if ((int32_t)spec_axis(src.spec, d) == lax + 1) {
      Low r = src;
      r.acq |= 1u << d;
      store(s, r);
      return;
    }
    // gather dim d if sharded (by another axis), then every dim sharded by
    // the loop axis in increasing order (InternalError if acquired), then
    // the slice itself -- one emission per iteration
    int rk = rank_of_spec(src.spec);
    while (true) {
      int32_t kind = kSliceByCoord, ax = lax, dd = d;
      if (spec_axis(src.spec, d) != 0) {
        kind = kAllGather;
        ax = (int32_t)spec_axis(src.spec, d) - 1;
      } else {
#pragma unroll 1
        for (int d2 = 0; d2 < rk; ++d2) {
          if ((int32_t)spec_axis(src.spec, d2) != lax + 1) continue;
          if ((src.acq >> d2) & 1) {
            fail(PE_CAND_INTERNAL);
            return;
          }
          kind = kAllGather;
          dd = d2;
          break;
        }
      }
      if (kind == kSliceByCoord) store(u, src);
      emit_coll(src, kind, ax, dd);
      if (bad()) return;
      if (kind == kSliceByCoord) break;
    }
    store(s, src);
  }

  PE_HD bool has_axis(uint32_t spec, int32_t ax) const {
    if ((spec_pending(spec) >> ax) & 1) return true;
    int r = rank_of_spec(spec);
    for (int d = 0; d < r; ++d)
      if ((int32_t)spec_axis(spec, d) == ax + 1) return true;
    return false;
  }

  // lower_loop (REF spmd.cc:157-204)
  // (the body is lowered by lower(); this is the loop's result from its
  // yield)
  PE_HD void finish_loop(int32_t v, int32_t l) {
    int32_t lax = a.laxis()[l];
    Low yv = load(a.lyield()[l]);
    int32_t lt = a.ltype()[l];
    bool tile = a.lkind()[l] == LK_TILE;
    Low w = yv;
    if (tile) {
      if (spec_pending(yv.spec)) {
        fail(PE_CAND_INTERNAL);
        return;
      }
      int dim = a.ldim()[l];
      uint32_t have = spec_axis(w.spec, dim);
      if ((int32_t)have == lax + 1) {
        w.acq &= ~(1u << dim);
      } else if (have == 0 && !has_axis(w.spec, lax)) {
        w.spec = spec_set_axis(w.spec, dim, (uint32_t)(lax + 1));
        w.acq &= ~(1u << dim);
      } else {
        fail(PE_CAND_INTERNAL);
        return;
      }
      w.gv = lt;
      w.gx = 0;
      int rk = rank_of_spec(w.spec);
      for (int d = 0; d < rk; ++d)
        if (local_dim(w, d) != local_dim(yv, d)) {
          fail(PE_CAND_INTERNAL);
          return;
        }
      if (bad()) return;
    } else {
      w.spec |= 1u << (16 + lax);
      int rk = rank_of_spec(w.spec);
      for (int d = 0; d < rk; ++d)
        if ((int32_t)spec_axis(w.spec, d) == lax + 1) {
          w.spec = spec_set_axis(w.spec, d, 0);
          w.acq &= ~(1u << d);
        }
      w.gv = lt;
      w.gx = 0;
    }
    // both kinds register the loop's result type (one inlined copy; its
    // local shape must exist, REF mesh.cc:110-124); a reduce loop then
    // all-reduces it over the loop axis
    local_elems(w);
    note_type(w.buf, w.spec);
    if (!tile) {
      emit_all_reduce(w, lax);
      if (bad()) return;
    }
    store(v, w);
  }

  // lower_to_spmd (REF spmd.cc:328-403).  stuck = also run the stuck
  // analysis (stuck_top / stuck_slice) on the way: it reads propagation
  // state only, which lowering never writes, and visits the same positions
  // and loop bodies in the same order as analyze() -- one walk instead of
  // two.
  PE_HD void lower(bool stuck) {
    nem = 0;
    neo = 0;
    flops = 0;
    for (int x = 0; x < 2 * kMaxAxes; ++x) a.st8()[x] = 0;
    for (int x = 0; x < 3 * kMaxAxes; ++x) a.st4()[x] = 0;
    for (int32_t x = 0; x < g.A; ++x) {
      Low w;
      int rank = g.vrank[x];
      w.gv = x;
      w.gx = 0;
      w.spec = (uint32_t)rank << 24;
      w.acq = 0;
      w.buf = x;
      int32_t direct = a.uses()[x] - a.slcnt()[x] - (result_ref == x ? 1 : 0);
      if (direct == 0 && a.aslice()[x] >= 0) {
        int d = a.aslice()[x] & 7, ax = a.aslice()[x] >> 3;
        if (g.amod((uint32_t)g.shape(x)[d], ax) == 0) w.spec = spec_set_axis(w.spec, d, (uint32_t)(ax + 1));
      }
      store(x, w);
      int64_t lb = 4 * local_elems(w);
      note_type(x, w.spec);
      a.aspec0()[x] = w.spec;
      a.alb0()[x] = lb;
    }
    for_top([&](int32_t v) {
      uint8_t k = a.vk()[v];
      if (k == VK_ATOMIC) {
        Low w = load(a.vref()[v]);
        int r = rank_of_spec(w.spec);
        bool rep = spec_pending(w.spec) == 0;
        for (int d = 0; d < r; ++d) rep = rep && spec_axis(w.spec, d) == 0;
        if (!rep) {
          fail(PE_CAND_INTERNAL);
          return;
        }
        store(v, w);
        return;
      }
      if (k != VK_TOP && k != VK_LOOP) return;
      if (stuck && k == VK_TOP) {
        stuck_top(v);
        if (bad()) return;
      }
      // A top-level op is lowered as a one-item body, so top-level and
      // per-iteration ops share one inlined lower_base (code size bounds
      // this kernel: instruction-cache stalls).
      int32_t l = k == VK_LOOP ? a.vref()[v] : -1;
      int32_t s = l >= 0 ? a.lhead()[l] : v;
      while (s >= 0) {
        int32_t next = l >= 0 ? a.bnext()[s] : -1;
        if (l >= 0 && a.vk()[s] == VK_SLICE) {
          if (stuck) {
            stuck_slice(s);
            if (bad()) return;
          }
          lower_slice(s, l);
        } else {
          lower_base(s, a.vref()[s], l);
        }
        if (bad()) return;
        s = next;
      }
      if (l >= 0) finish_loop(v, l);
    });
    if (bad()) return;
    Low res = load(result_ref);
    while (spec_pending(res.spec)) {
      emit_all_reduce(res, pending_front(res.spec));
      if (bad()) return;
    }
    store(result_ref, res);
    result_buf = res.buf;
  }

  // ------------------------------------------------------------ scoring
  PE_HD void score(const pe_cost_params& cp, int64_t baseline, int32_t steps,
                   pe_result& r, int32_t ln = 0, int32_t nl = 1) {
    // collective_stats (REF spmd.cc:405-434), accumulated at emission
    for (int x = 0; x < PE_MAX_AXES; ++x) {
      r.ar_bytes[x] = a.st8()[x];
      r.ag_bytes[x] = a.st8()[kMaxAxes + x];
      r.ar_cnt[x] = a.st4()[x];
      r.ag_cnt[x] = a.st4()[kMaxAxes + x];
      r.sbc_cnt[x] = a.st4()[2 * kMaxAxes + x];
    }
    // One pass over the SPMD ops, the liveness sweep:
    // new_op set delta[j] = +lb[j]; -lb[j] lands after the buffer's last
    // use (> j), so by the time the sweep reaches j every subtraction
    // landing there is already in delta[j] and the running sum is taken in
    // the same pass.
    if (result_buf >= g.A) a.em_last()[result_buf - g.A] = nem - 1;
    a.delta()[nem] = 0;
    int64_t run = 0, best = 0, base = 0;
#ifdef __CUDA_ARCH__
    if (nl > 1) {
      // the warp's lanes (kFCoop): every -lb[j] lands first (atomics: two
      // buffers may end at the same op), then a shuffle scan per 32 ops
      // carries the running sum and a warp max keeps its peak
      pe_syncwarp();
      for (int32_t j = ln; j < nem; j += nl) {
        V4 q = a.em_q0()[j];
        int64_t lb = a.em_q1()[j].x;
        atomicAdd(reinterpret_cast<unsigned long long*>(&a.delta()[q.z + 1]),
                  (unsigned long long)(-lb));
      }
      __syncwarp();
      int64_t carry = 0;
      for (int32_t c = 0; c < nem; c += 32) {
        int32_t j = c + ln;
        int64_t d = j < nem ? a.em_q1()[j].y : 0;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          int64_t t = __shfl_up_sync(0xFFFFFFFFu, d, off);
          if (ln >= off) d += t;
        }
        int64_t m = j < nem ? carry + d : 0;
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
          int64_t t = __shfl_xor_sync(0xFFFFFFFFu, m, off);
          m = t > m ? t : m;
        }
        best = m > best ? m : best;
        carry += __shfl_sync(0xFFFFFFFFu, d, 31);
      }
      for (int32_t x = ln; x < g.A; x += nl) base += a.alb0()[x];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) base += __shfl_xor_sync(0xFFFFFFFFu, base, off);
      __syncwarp();
    } else
#endif
    for (int32_t j = 0; j < nem; ++j) {
      V4 q = a.em_q0()[j];  // head, op0, last, operand offset
      I64x2 q1 = a.em_q1()[j];  // local bytes, liveness delta
      int64_t lb = q1.x;
      run += q1.y;
      if (run > best) best = run;
#ifndef PE_EXP_NO_DELTA
      a.delta()[q.z + 1] -= lb;
#endif
    }
    if (nl == 1)
      for (int32_t x = 0; x < g.A; ++x) base += a.alb0()[x];
    r.peak_bytes = base + best;
    r.flops = flops;
    r.n_spmd_ops = nem;
    r.n_steps = steps;
    int64_t ar = 0, ag = 0, arc = 0, agc = 0;
    for (int x = 0; x < PE_MAX_AXES; ++x) {
      ar += r.ar_bytes[x];
      ag += r.ag_bytes[x];
      arc += r.ar_cnt[x];
      agc += r.ag_cnt[x];
    }
    r.reduction_bytes = ar;
    r.baseline_bytes = baseline;
    double rt = ddiv((double)flops, cp.flops_per_second);
    rt = dadd(rt, ddiv((double)(ar + ag), cp.bytes_per_second));
    rt = dadd(rt, dmul(cp.collective_latency_s, (double)(arc + agc)));
    r.runtime_s = rt;
    r.feasible = r.peak_bytes <= cp.memory_budget_bytes ? 1 : 0;
    if (!r.feasible) {
      r.reward = 0.0;
    } else {
      double d = 1.0;
      d = dadd(d, dmul(cp.w_comm, ddiv((double)ar, (double)baseline)));
      d = dadd(d, dmul(cp.w_mem, ddiv((double)r.peak_bytes, (double)cp.memory_budget_bytes)));
      d = dadd(d, dmul(cp.w_steps, (double)steps));
      r.reward = ddiv(1.0, d);
    }
  }

  // parity trace (pe.h layout)
  PE_HD void write_trace(int32_t* t, uint32_t cap) {
    uint32_t n = 1;
    bool over = false;
    auto put = [&](int64_t v) {
      if (n < cap) t[n] = (int32_t)v;
      else over = true;
      ++n;
    };
    put(g.A);
    for (int32_t x = 0; x < g.A; ++x) put(a.aspec0()[x]);
    put(result_buf < g.A ? a.arg_spec()[result_buf] : a.em_spec()[result_buf - g.A]);
    put(nstk);
    for (int32_t i = 0; i < nstk; ++i) {
      put(a.stk()[2 * i]);
      put(a.stk()[2 * i + 1]);
    }
    put(nem);
    for (int32_t j = 0; j < nem; ++j) {
      int32_t h = a.em_head()[j];
      put(h);
      put(a.em_lb()[j] & 0xffffffff);
      put(a.em_lb()[j] >> 32);
      put(a.em_spec()[j]);
      int32_t no = (h >> 16) & 0xFFFF;
      for (int32_t q = 0; q < no; ++q) put(a.em_opnd()[a.em_ooff()[j] + q]);
    }
    if (cap > 0) t[0] = over ? -(int32_t)n : (int32_t)n;
  }

  // ------------------------------------------------------------ drivers
  // separate = run analyze() as its own walk before lowering (the
  // resurfacing kernel); otherwise the stuck analysis rides on lowering
  PE_HD void finish(const pe_cost_params& cp, int64_t baseline, int32_t steps,
                    bool propagated, pe_result& r, int32_t* trace, uint32_t trace_words,
                    bool separate = false, int32_t ln = 0, int32_t nl = 1) {
    tick(5);
    nstk = 0;
    if (separate && !bad() && propagated) analyze();
    tick(6);
    if (!bad()) lower(!separate && propagated);
    tick(7);
    finish_result(cp, baseline, steps, propagated, r, trace, trace_words, ln, nl);
    clear_seen();
    tick(8);
  }
  PE_HD void finish_result(const pe_cost_params& cp, int64_t baseline, int32_t steps,
                           bool propagated, pe_result& r, int32_t* trace, uint32_t trace_words,
                           int32_t ln = 0, int32_t nl = 1) {
    if (bad()) {
      int32_t st = status;
      for (int x = 0; x < PE_MAX_AXES; ++x) {
        r.ar_bytes[x] = r.ag_bytes[x] = 0;
        r.ar_cnt[x] = r.ag_cnt[x] = r.sbc_cnt[x] = 0;
      }
      r.peak_bytes = r.flops = r.reduction_bytes = r.baseline_bytes = 0;
      r.n_spmd_ops = 0;
      r.n_stuck = 0;
      r.feasible = 0;
      r.runtime_s = 0;
      r.reward = 0;
      r.n_steps = steps;
      r.status = st;
      r.fail_step = steps;
      if (trace && trace_words) trace[0] = 0;
      return;
    }
    int32_t fs = r.fail_step;
    score(cp, baseline, steps, r, ln, nl);
    r.n_stuck = propagated ? nstk : 0;
    r.status = status;
    r.fail_step = fs;
    if (trace && trace_words) write_trace(trace, trace_words);
  }

  // argflags (optional, A bytes): bit 0 = argument sliced, bit 1 = atomic
  // (infer_rest's arg_is_tiled / arg_is_atomic, REF propagate.cc:490-503)
  PE_HD void eval(const pe_action* acts, int32_t n, const pe_cost_params& cp,
                  int64_t baseline, pe_result& r, int32_t* trace, uint32_t trace_words,
                  uint8_t* argflags = nullptr) {
    // (traces are taken in full-size arenas, which keep the operand log)
    tracing = trace != nullptr && trace_words > 0 && a.L->has_opnd;
    tick_start();
    init();
    tick(0);
    r.fail_step = -1;
    r.reserved = 0;
    r.reserved2 = 0;
    int32_t steps = 0;
    bool propagated = false;
    for (int32_t k = 0; k < n; ++k) {
      if (acts[k].kind == PE_ACT_STOP) break;
      if (acts[k].kind == PE_ACT_INFER_REST) {
        // InferRest decision marker; the host expanded it into the inferred
        // tile actions that follow (pe_engine.cu infer_rest_expand), which
        // do not count as steps
        if (!(acts[k].pad & PE_ACT_FLAG_EXPANDED)) {
          status = PE_CAND_ILLEGAL;  // unexpanded: not executable on the device
          r.fail_step = k;
          break;
        }
        propagated = true;
        ++steps;
        continue;
      }
      bool ok = apply_action(acts[k]);
      if (bad()) break;
      if (!ok) {
        status = PE_CAND_ILLEGAL;
        r.fail_step = k;
        break;
      }
      propagate();
      propagated = true;
      if (bad()) break;
      if (!(acts[k].pad & PE_ACT_FLAG_INFERRED)) ++steps;
    }
    finish(cp, baseline, steps, propagated, r, trace, trace_words);
    if (argflags)
      for (int32_t x = 0; x < g.A; ++x)
        argflags[x] = (uint8_t)((a.slcnt()[x] > 0 ? 1 : 0) | (a.awrapped()[x] ? 2 : 0));
  }

  // ------------------------------------------------------------ rollouts
  // legal_actions (SPEC search module): a TileValue ordinal is legal when at
  // least one statically legal member does not carry tiling yet
  // (REF rewrite.cc:75-76).  Fills a.lg with the legal ordinals in order.
  // Stuck resurfacing (pe.h resurface_stuck; SPEC Worklist): the ops of
  // the current fixpoint's stuck list (REF propagate.cc:412-454, discovery
  // order) join the worklist once each.  Called at every decision boundary.
  PE_HD void resurface_update() {
    analyze();
    for (int32_t i = 0; i < nstk && !bad(); ++i) {
      int32_t o = a.stk()[2 * i];
      uint32_t bit = 1u << (o & 31);
      if (a.rsb()[o >> 5] & bit) continue;
      a.rsb()[o >> 5] |= bit;
      a.rs()[nrs++] = o;
    }
    clear_seen();
  }
  // Legal TileValue ordinals in worklist order (SPEC legal_actions): the
  // static entries, then the resurfaced ops in discovery order; a
  // resurfaced op is legal as apply_tile_action would accept it (still at
  // top level and carrying no tiling: TOP without slices; the dim divides).
  template <bool RS>
  PE_HD int32_t build_legal() {
    int32_t n = 0;
    for (int32_t o = 0; o < g.n_ord; ++o) {
      for (int32_t i = g.ord_off[o]; i < g.ord_off[o + 1]; ++i) {
        int32_t m = g.ord_mem[i];
        if (!((a.carry()[m >> 5] >> (m & 31)) & 1u)) {
          a.lg()[n++] = o;
          break;
        }
      }
    }
    for (int32_t i = 0; RS && i < nrs; ++i) {
      int32_t o = a.rs()[i], v = g.A + o;
      if (a.vk()[v] != VK_TOP || a.slcnt()[v] != 0) continue;
      int32_t rank = g.vrank[v];
      for (int32_t d = 0; d < rank; ++d)
        for (int32_t ai = 0; ai < g.n_auto; ++ai)
          if (g.amod((uint32_t)g.shape(v)[d], g.auto_axes[ai]) == 0)
            a.lg()[n++] = ((g.n_entries + o) * kMaxRank + d) * g.n_auto + ai;
    }
    return n;
  }
  // InferRest is legal when some argument neither carries a slice nor is
  // atomic-wrapped (SPEC legal_actions "if any argument untiled"; the carry
  // bits are exactly REF rewrite.cc:42-51 carries_tiling for arguments)
  PE_HD bool infer_rest_legal() const {
    for (int32_t w = 0; w <= (g.A >> 5); ++w) {
      int32_t bits = g.A - (w << 5);
      uint32_t all = bits >= 32 ? 0xFFFFFFFFu : ((1u << bits) - 1u);
      if ((a.carry()[w] & all) != all) return true;
    }
    return false;
  }
  // stop here for the host's batched InferRest expansion (pe_engine.cu
  // ir_resolve): record the (unexpanded) decision, report the position
  // (prefix index, or -1 for a drawn decision) and the draws consumed
  PE_HD void pause(pe_result& r, pe_action* acts_out, int32_t& nacts, int32_t maxd,
                   int32_t steps, int32_t at, int32_t draws) {
    if (nacts < maxd) acts_out[nacts] = pe_action{0, 0, 0, PE_ACT_INFER_REST, 0};
    ++nacts;
    r.status = PE_CAND_PAUSED;
    r.fail_step = at;
    r.reserved = draws;
    r.n_steps = steps;
  }
#ifdef __CUDA_ARCH__
  // build_legal<false> with the warp's lanes splitting the ordinals: a
  // ballot per 32 ordinals keeps the list in ordinal order (kFCoop)
  PE_HD int32_t build_legal_coop(int32_t ln) {
    int32_t n = 0;
    for (int32_t base = 0; base < g.n_ord; base += 32) {
      int32_t o = base + ln;
      bool ok = false;
      if (o < g.n_ord)
        for (int32_t i = g.ord_off[o]; i < g.ord_off[o + 1] && !ok; ++i) {
          int32_t m = g.ord_mem[i];
          ok = !((a.carry()[m >> 5] >> (m & 31)) & 1u);
        }
      unsigned b = __ballot_sync(0xFFFFFFFFu, ok);
      if (ok) a.lg()[n + __popc(b & ((1u << ln) - 1u))] = o;
      n += __popc(b);
    }
    __syncwarp();
    return n;
  }
#endif
  PE_HD pe_action ordinal_action(int32_t ord) const {
    pe_action x;
    int32_t na = g.n_auto;
    int32_t ai = ord % na, d = (ord / na) % kMaxRank, e = ord / na / kMaxRank;
    x.axis = (uint8_t)g.auto_axes[ai];
    x.dim = (uint8_t)d;
    x.pad = 0;
    if (e >= g.n_entries) {  // resurfaced stuck op: TileValue(op result)
      x.kind = PE_ACT_TILE;
      x.value = (uint32_t)(g.A + (e - g.n_entries));
      return x;
    }
    x.kind = g.entries_are_groups ? PE_ACT_TILE_GROUP : PE_ACT_TILE;
    x.value = (uint32_t)g.ent_val[e];
    return x;
  }
  PE_HD static uint64_t splitmix(uint64_t& st) {
    st += 0x9E3779B97F4A7C15ull;
    uint64_t z = st;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }

  // RS = stuck resurfacing compiled in (pe.h resurface_stuck); the engine
  // launches the RS instantiation only when the worklist asks for it, so
  // the default kernel carries none of its code (code size bounds this
  // kernel: instruction-cache stalls).
  template <bool RS, int F = kFAll>
  //
  // rs: start from a saved state instead of init() and
  // replaying the decisions it covers -- the scheduling trie's states of
  // root rollouts (their own seed draws the path; rs.stop: the next draw is
  // Stop) and the prefix-state cache / pe_state parents (the path is the
  // prefix's first rs.done entries).
  PE_HD void rollout(const pe_action* prefix, int32_t np, uint64_t seed, int32_t maxd,
                     const pe_cost_params& cp, int64_t baseline, pe_action* acts_out,
                     uint32_t* n_out, pe_result& r, uint64_t* legal_out, int32_t legal_words,
                     const Resume& rs = Resume()) {
    tracing = false;
    tick_start();
    int32_t steps = 0, nacts = 0;
    bool propagated = false, terminal = false;
    constexpr bool IR = (F & kFInferRest) != 0, RES = (F & kFResume) != 0;
    constexpr bool COOP = (F & kFCoop) != 0;
    const int32_t ln = COOP ? pe_lane() : 0, nln = COOP ? 32 : 1;
    if (RES && rs.snap) {
      load(rs.snap, ln, nln);
      for (int32_t k = 0; k < rs.done && k < maxd; ++k) acts_out[k] = rs.path[k];
      steps = nacts = rs.done;
      propagated = rs.done > 0;
      terminal = rs.stop;
    } else {
      init(ln, nln);
    }
    tick(0);
    r.fail_step = -1;
    r.reserved = 0;
    r.reserved2 = 0;
    if (legal_out)
      for (int32_t w = 0; w < legal_words; ++w) legal_out[w] = 0;
    // resurfacing runs at decision boundaries: before the next decision of
    // the prefix (tiles an INFER_REST expansion inferred belong to it) and
    // before enumerating legal actions -- i.e. after every whole decision,
    // as the oracle does after each apply_action
    bool rs_due = false;
    for (int32_t k = RES ? (bad() ? np : rs.k0) : 0; k < np; ++k) {
      if (RS && rs_due && !(prefix[k].pad & PE_ACT_FLAG_INFERRED)) {
        resurface_update();
        rs_due = false;
        if (bad()) break;
      }
      if (prefix[k].kind == PE_ACT_STOP) {
        terminal = true;
        break;
      }
      if (prefix[k].kind == PE_ACT_INFER_REST) {  // expanded by the host
        if (!(prefix[k].pad & PE_ACT_FLAG_EXPANDED)) {
          if (IR && g.ir_pause) {
            pause(r, acts_out, nacts, maxd, steps, k, 0);
            *n_out = (uint32_t)(nacts < maxd ? nacts : maxd);
            return;
          }
          status = PE_CAND_ILLEGAL;
          r.fail_step = k;
          terminal = true;
          break;
        }
        // recorded as the decision (unexpanded); its inferred tiles follow
        // in the prefix and are not recorded
        propagated = true;
        if (nacts < maxd) acts_out[nacts] = pe_action{0, 0, 0, PE_ACT_INFER_REST, 0};
        ++nacts;
        ++steps;
        continue;
      }
      bool ok = apply_action(prefix[k]);
      if (bad()) break;
      if (!ok) {
        status = PE_CAND_ILLEGAL;
        r.fail_step = k;
        terminal = true;
        break;
      }
      propagate();
      propagated = true;
      if (bad()) break;
      rs_due = RS;
      if (!(prefix[k].pad & PE_ACT_FLAG_INFERRED)) {  // decisions only
        if (nacts < maxd) acts_out[nacts] = prefix[k];
        ++nacts;
        ++steps;
      }
    }
    if (RS && rs_due && !bad() && status == PE_CAND_OK) resurface_update();
    if (RES && rs.save && !bad() && status == PE_CAND_OK) {
      save(rs.save);
      if (rs.saved) *rs.saved = 1;
    }
    if (!bad() && status == PE_CAND_OK) {
      if (legal_out) {
#ifdef __CUDA_ARCH__
        int32_t nl = COOP ? build_legal_coop(ln) : build_legal<RS>();
#else
        int32_t nl = build_legal<RS>();
#endif
        for (int32_t i = 0; i < nl; ++i) legal_out[a.lg()[i] >> 6] |= 1ull << (a.lg()[i] & 63);
        if (IR && g.ir_ord >= 0 && infer_rest_legal())
          legal_out[g.ir_ord >> 6] |= 1ull << (g.ir_ord & 63);
      }
      // (each decision draws once: splitmix adds the golden gamma per draw)
      uint64_t st = seed + (RES ? (uint64_t)rs.draws * 0x9E3779B97F4A7C15ull : 0);
      int32_t draws = RES ? rs.draws : 0;
      while (!terminal) {
        if (steps >= maxd) break;
        tick(4);
#ifdef __CUDA_ARCH__
        int32_t nl = COOP ? build_legal_coop(ln) : build_legal<RS>();
#else
        int32_t nl = build_legal<RS>();
#endif
        // InferRest follows the TileValue actions (SPEC legal_actions order)
        int32_t ir = IR && g.ir_ord >= 0 && infer_rest_legal() ? 1 : 0;
        if (nl + ir == 0) break;
        uint64_t ws = steps >= 1 ? 2 : 1;
        uint64_t pick = splitmix(st) % ((uint64_t)(nl + ir) + ws);
        ++draws;
        if (pick >= (uint64_t)(nl + ir)) break;
        if (IR && pick == (uint64_t)nl) {
          pause(r, acts_out, nacts, maxd, steps, -1, draws);
          *n_out = (uint32_t)(nacts < maxd ? nacts : maxd);
          return;
        }
        pe_action x = ordinal_action(a.lg()[pick]);
        tick(5);
        bool ok = apply_action(x);
        if (bad()) break;
        if (!ok) {
          status = PE_CAND_ILLEGAL;
          r.fail_step = nacts;
          break;
        }
        propagate();
        propagated = true;
        if (bad()) break;
        if (RS) {
          resurface_update();
          if (bad()) break;
        }
        if (nacts < maxd) acts_out[nacts] = x;
        ++nacts;
        ++steps;
      }
    }
    *n_out = (uint32_t)(nacts < maxd ? nacts : maxd);
    finish(cp, baseline, steps, propagated, r, nullptr, 0, false, ln, nln);
  }
};

}  // namespace pe
