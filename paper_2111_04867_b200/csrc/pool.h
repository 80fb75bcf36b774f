// Symmetric multicast pool (pool.cpp).
#pragma once
#include <cuda.h>

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "taccl_internal.h"

namespace taccl {

// The pool's first bytes hold the multicast-reduce barrier flags (u32 per (phase, group,
// piece, rank)); allocations start after them.
constexpr int kMrGroups = 16;
TACCL_HD inline size_t mr_flag(int phase, int group, int piece, int rank) {
  return (((size_t)phase * kMrGroups + group) * kMaxSplit + piece) * kMaxRanks + rank;
}
constexpr size_t kPoolFlagBytes = ((2 * (size_t)kMrGroups * kMaxSplit * kMaxRanks * 4) + (1 << 21) - 1) & ~(size_t)((1 << 21) - 1);

struct Pool {
  bool up = false;
  int rank = 0, nranks = 0, dev = 0;
  size_t bytes = 0, align = 0, used = 0;
  CUmemGenericAllocationHandle phys = 0, mc = 0;
  std::vector<CUmemGenericAllocationHandle> peer_phys;
  char* uc = nullptr;      // this rank's allocation (local mapping)
  char* mcva = nullptr;    // the multicast mapping (multimem.* addresses)
  std::vector<char*> peer; // every rank's allocation mapped here (peer[rank] == uc)
  int fd_phys = -1, fd_mc = -1, listener = -1;
  uint64_t sock_id = 0;
};

// Collective, three phases with a host exchange/barrier between them (taccl.h):
// export (blob naming this rank's socket), connect (descriptor exchange, peers mapped, device
// added to the multicast object), bind (after every rank added its device).
bool pool_export(Pool& P, int rank, int nranks, int dev, size_t bytes, void* blob, size_t* len, std::string* err);
bool pool_connect(Pool& P, const void* all, size_t len_each, std::string* err);
bool pool_bind(Pool& P, std::string* err);
void pool_destroy(Pool& P);

}  // namespace taccl
