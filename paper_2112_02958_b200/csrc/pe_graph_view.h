// pe_graph_view.h — the compiled, read-only graph as the kernels see it.
//
// Structure-of-arrays CSR resident in HBM (one copy per device, shared by all
// candidates).  Built once per program by the host graph compiler
// (pe_graph.cc) from the `.pir` text; it replaces the reference's AoS
// `Program` / `Operation` structs (REF ir.h:84-131) and the per-call rule
// instantiation of `rule_for` (REF registry.cc:123-206): every op's
// propagation rule is precomputed for its global operand shapes.
#pragma once
#include <stdint.h>

#ifdef __CUDACC__
#define PE_HD __host__ __device__ __forceinline__
#else
#define PE_HD inline
#endif

namespace pe {

// REF OpKind numbering (ir.h:31-62); only base kinds appear in a root graph.
enum Kind : uint8_t {
  kConstant = 0, kAdd, kSub, kMul, kDiv, kNeg, kExp, kTanh, kRsqrt, kMaximum,
  kDot, kReduceSum, kReduceMax, kTranspose, kReshape, kBroadcastInDim, kSlice,
  kConcatenate,
  kNumBaseKinds = 18,
  kAllReduce = 22, kAllGather = 23, kSliceByCoord = 24
};

// DimRole (REF registry.h:27-38)
enum Role : uint8_t { kPass = 0, kContract = 1, kBlocked = 2 };

constexpr int kMaxRank = 4;
constexpr int kMaxAxes = 4;
constexpr int64_t kMaxDim = 2147483647;  // dims and axis sizes fit int32

struct GraphView {
  int32_t A;        // arguments
  int32_t N;        // ops (top level, topologically ordered)
  int32_t E;        // operand slots
  int32_t n_axes;
  int64_t axis_size[kMaxAxes];
  // Division by an axis size d without a divide instruction sequence (the
  // inlined 32-bit divide is ~25 SASS instructions and local_dim is inlined
  // at many unrolled sites; code size is what bounds the rollout kernel --
  // instruction-cache stalls).  Dims and axis sizes are
  // validated to fit int32 (pe_graph.cc validate), so for 0 <= x < 2^31
  //   x / d == (x * m) >> s,  m = ceil(2^s / d),  s = 31 + ceil(log2 d)
  // exactly (Granlund & Montgomery 1994, Thm 4.2: the error m*d - 2^s < d
  // <= 2^(s-31)); m < 2^32 for every d >= 1.  These are the same integers
  // as the reference's int64 arithmetic (tests/test_semantics.py checks the
  // identity; the fuzz runs power-of-two and other meshes).
  // Tables are indexed by axis + 1 (the spec-word nibble); entry 0 is the
  // divisor 1 (m = 2^31, s = 31), so an unsharded dim divides by 1.
  uint32_t axis_sz32[kMaxAxes + 1];
  uint32_t axis_magic[kMaxAxes + 1];
  int32_t axis_mshift[kMaxAxes + 1];
  PE_HD uint32_t quo1(uint32_t x, uint32_t ax1) const {
    return (uint32_t)(((uint64_t)x * axis_magic[ax1]) >> axis_mshift[ax1]);
  }
  PE_HD uint32_t aquo(uint32_t x, int32_t ax) const { return quo1(x, (uint32_t)ax + 1); }
  PE_HD uint32_t amod(uint32_t x, int32_t ax) const {
    return x - aquo(x, ax) * axis_sz32[ax + 1];
  }
  // rank of each axis name in lexicographic order: ShardingSpec::pending_sum
  // is kept sorted by NAME (REF mesh.cc:74-77), so `pending_sum.front()` is
  // the axis with the smallest name rank.
  int32_t axis_name_rank[kMaxAxes];
  // pending mask (4 bits) -> its axis with the smallest name rank (-1 if 0)
  int8_t pend_front[16];
  int32_t result;   // returned value index

  // values [A+N]: args first, then op results
  const int32_t* vshape;  // [(A+N)*4] dims, 0-padded
  const uint8_t* vrank;   // [A+N]

  // ops [N]
  const uint8_t* okind;      // Kind
  const uint8_t* omask;      // dot: rhs free-dim mask; broadcast: mapped result-dim mask
  const int32_t* oopnd_off;  // [N+1] into oopnd / slot arrays
  const int32_t* oopnd;      // [E] original operand value index
  const int32_t* slot_op;    // [E] op owning operand slot
  const uint8_t* orule_err;  // [N] rule_for would throw (reshape factorisation)

  // propagation rules, per op: classes [ocls_off[o], ocls_off[o+1])
  const int32_t* ocls_off;   // [N+1]
  const uint8_t* cls_role;   // [C]
  const int8_t* cls_rdim;    // [C] result dim (pass-through) or -1
  const int32_t* cls_moff;   // [C+1] member range into mem
  const uint16_t* mem;       // member = operand << 2 | dim
  const int16_t* slot_cls;   // [E*4] (operand slot, dim) -> class index local to op, -1
  const int16_t* op_rcls;    // [N*4] result dim -> pass-through class (local) or -1

  // users CSR: value -> operand slots that originally read it
  const int32_t* user_off;   // [A+N+1]
  const int32_t* users;      // operand slot indices

  const int32_t* init_uses;  // [A+N] count_uses on the root (REF ir.cc:125-134)

  // worklist entries (scope groups or single arguments) for rollouts
  int32_t n_entries;
  int32_t n_auto;
  int32_t auto_axes[kMaxAxes];
  int32_t entries_are_groups;
  const int32_t* ent_off;    // [n_entries+1]
  const int32_t* ent_mem;    // arg indices
  const int32_t* ent_val;    // [n_entries] action value: group index / argument
  // scope groups (for PE_ACT_TILE_GROUP)
  int32_t n_groups;
  const int32_t* grp_off;    // [n_groups+1]
  const int32_t* grp_mem;
  // stuck resurfacing (pe.h resurface_stuck): resurfaced op o's ordinals
  // are ((n_entries + o) * kMaxRank + dim) * n_auto + ai
  int32_t resurface;
  // TileValue ordinals of the static entries: statically legal members
  int32_t n_ord;
  // InferRest as a rollout action (pe.h infer_rest_action): ir_ord = its
  // ordinal (after every TileValue ordinal), -1 when off.  A drawn InferRest
  // -- and, when ir_pause, an unexpanded InferRest in a prefix -- pauses the
  // candidate (PE_CAND_PAUSED) for the host's batched expansion.
  int32_t ir_ord;
  int32_t ir_pause;
  const int32_t* ord_off;    // [n_ord+1]
  const int32_t* ord_mem;

  PE_HD const int32_t* shape(int32_t v) const { return vshape + 4 * v; }
};

// spec word (pe.h trace layout): per dim (axis+1) in 4 bits, pending mask
// << 16, rank << 24
PE_HD uint32_t spec_axis(uint32_t spec, int d) { return (spec >> (4 * d)) & 0xFu; }
PE_HD uint32_t spec_set_axis(uint32_t spec, int d, uint32_t ax1) {
  return (spec & ~(0xFu << (4 * d))) | (ax1 << (4 * d));
}
PE_HD uint32_t spec_pending(uint32_t spec) { return (spec >> 16) & 0xFu; }

}  // namespace pe
