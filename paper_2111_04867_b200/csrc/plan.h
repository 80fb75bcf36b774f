// Per-rank device plan built from a checked program (plan.cpp).
#pragma once
#include <vector>

#include "taccl_internal.h"

namespace taccl {

struct RankPlan {
  std::vector<KTB> tbs;
  std::vector<KStep> steps;
  std::vector<int32_t> deps;   // pairs (tb, step)
  std::vector<int32_t> fused;  // chain entries (kFuseStride ints), then forward entries (kFwdStride)
  int stage_chunks = 0;        // rrc staging this rank needs (chunk units)
  int stage2_chunks = 0;       // staged mode: every receive's slot (chunk units)
  int scratch_chunks = 0;      // EF scratch buffer (chunk units)
  int fused_chains = 0;
  bool partials = false;       // some step carries bf16 partial flags
  bool shadow = false;         // some step reads or writes the fp32 shadow of o / s (bf16 calls
                               // then need the shadow region: 2 x (o + s) bytes)
  std::vector<int32_t> order;  // merged execution: every step of the rank as tb << 16 | step, in
                               // global level order (plan.cpp merged_order); empty = not mergeable
};

// `fuse`: fuse rrc chains into multi-input reductions (env TACCL_NO_FUSE=1 disables);
// `fuse_rrcs`: fuse rrc + send-of-its-result into one pass (env TACCL_NO_RRCS=1 disables).
// `chain_sends`: fuse the sends of a chain's result into the chain (fuse_chain_sends).
// pull_kinds (pull mode): which receive-reduces may read their input in place —
// 1 plain rrc, 2 rrc fused with its send (K_RRCS), 4 fused chains
std::vector<RankPlan> build_plans(const Program& P, bool fuse, bool fuse_rrcs, bool chain_sends, int pull_kinds = 1);

}  // namespace taccl
