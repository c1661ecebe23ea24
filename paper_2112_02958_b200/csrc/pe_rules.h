// pe_rules.h — shape-dependent propagation rule pieces shared by the host
// graph compiler and the device lowering.
//
// Only `reshape` has a rule whose class structure depends on the concrete
// shapes (REF registry.cc:88-119, greedy factorisation into dim groups), and
// lowering instantiates rules on per-iteration LOCAL shapes (REF spmd.cc:270
// with patch B), so the device recomputes it there.  Every other kind's rule
// is shape-independent and lives in the precompiled per-op class table.
#pragma once
#include <stdint.h>

#include "pe_graph_view.h"

namespace pe {

struct ReshapeRule {
  int8_t cls_of_dim[kMaxRank];  // input dim -> class index
  uint8_t role[kMaxRank + kMaxRank];
  int8_t rdim[kMaxRank + kMaxRank];
  int8_t n_cls;
  int8_t error;  // factorisation failed (InternalError in the reference)
};

// Greedy factorisation of `a` -> `b` into groups with equal element products;
// 1:1 groups of equal size pass through, every other group (split / merge)
// is blocked.  Trailing 1-dims fold into the last group.
template <typename IA, typename IB>
PE_HD ReshapeRule reshape_rule(const IA* a, int ra, const IB* b, int rb) {
  ReshapeRule r;
  r.n_cls = 0;
  r.error = 0;
  for (int d = 0; d < kMaxRank; ++d) r.cls_of_dim[d] = -1;
  int i = 0, j = 0;
  while (i < ra || j < rb) {
    int i0 = i, j0 = j;
    int64_t pa = i < ra ? (int64_t)a[i++] : 1;
    int64_t pb = j < rb ? (int64_t)b[j++] : 1;
    while (pa != pb) {
      if (pa < pb && i < ra) pa *= a[i++];
      else if (pb < pa && j < rb) pb *= b[j++];
      else break;
    }
    while (i < ra && a[i] == 1 && j >= rb) ++i;
    while (j < rb && b[j] == 1 && i >= ra) ++j;
    if (pa != pb) {
      r.error = 1;
      return r;
    }
    if (i - i0 == 1 && j - j0 == 1 && (int64_t)a[i0] == (int64_t)b[j0]) {
      r.role[r.n_cls] = kPass;
      r.rdim[r.n_cls] = (int8_t)j0;
      r.cls_of_dim[i0] = r.n_cls;
      r.n_cls++;
    } else if (i > i0) {
      r.role[r.n_cls] = kBlocked;
      r.rdim[r.n_cls] = -1;
      for (int k = i0; k < i; ++k) r.cls_of_dim[k] = r.n_cls;
      r.n_cls++;
    }
  }
  return r;
}

}  // namespace pe
