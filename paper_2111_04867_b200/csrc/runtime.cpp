// C ABI (include/taccl.h): communicator, IPC peer mappings, buffer registration, algorithm
// registry and the single-launch collective call.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "plan.h"
#include "pool.h"
#include "taccl_internal.h"

using namespace taccl;

namespace {

thread_local std::string g_err;

taccl_result_t fail(taccl_result_t code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CUDA_TRY(expr)                                                                  \
  do {                                                                                  \
    cudaError_t e_ = (expr);                                                            \
    if (e_ != cudaSuccess) return fail(TACCL_ERR_CUDA, std::string(#expr ": ") + cudaGetErrorString(e_)); \
  } while (0)

constexpr uint32_t kMagicArena = 0x7acc1a7e;
constexpr uint32_t kMagicBuf = 0x7acc1b0f;

struct HandleBlob {  // TACCL_HANDLE_BYTES
  uint32_t magic;
  int32_t rank;
  uint64_t offset;   // pointer - allocation base
  uint64_t bytes;
  cudaIpcMemHandle_t h;  // 64 bytes
  char pad[TACCL_HANDLE_BYTES - 24 - sizeof(cudaIpcMemHandle_t)];
};
static_assert(sizeof(HandleBlob) == TACCL_HANDLE_BYTES, "blob size");

struct DevPlan {  // one rank's plan blob in device memory
  void* mem = nullptr;
  int bytes = 0, steps_off = 0, deps_off = 0, fused_off = 0;
  int ntb = 0;
  int order_off = 0, norder = 0;  // merged execution order (norder 0: not mergeable)
};

struct Algo {
  std::string name;
  Coll coll;
  int nranks, p, instances;
  uint64_t min_bytes, max_bytes;
  uint32_t dtypes = 7;  // element types this algorithm is selected for (EF dtypes attribute)
  int max_scratch_chunks = 0, max_stage_chunks = 0, max_stage2_chunks = 0, max_steps_cnt = 1;
  // n = 1 plan that is one input -> output `cpy` (no deps): runs as the lean copy kernel
  bool lean_copy = false;
  // one `mr` step per rank, no dependencies (nvls template): the lean multicast-reduce kernel
  bool lean_mr = false;
  std::vector<int> mr_srcoff, mr_dstoff, mr_cnt;  // per rank
  int lean_srcoff = 0, lean_dstoff = 0, lean_cnt = 0;
  std::vector<DevPlan> plans;   // indexed by rank (only local ranks filled)
  std::vector<DevPlan> plans_ll;  // the same program planned for the LL kernel (chain sends fused)
  // the direct plan with fused chains also reading their peers' inputs in place (pull kinds
  // | 4): used for chunks >= TACCL_PULL_CHAIN_MIN (default 64 MiB), where the in-place loads
  // beat push + staging (profiles/r02_rs_scan_n4.txt: RS n=4 1 GiB 1373 vs 1470 us) — below,
  // the pushes overlap the reduction better (16 MiB: 51 vs 37 us). Empty if no chain pulls.
  std::vector<DevPlan> plans_pc;
  std::vector<int> ntb;         // per rank
  std::vector<std::vector<int>> weights;  // per rank, per tb
  std::vector<std::vector<int>> indep;    // per rank, per tb
  std::vector<int> wsum;        // per rank
  int fused_chains = 0;
  bool has_pull = false;  // some send of the direct plan is read in place (pull mode applies)
  bool has_prog = false;  // some message of the direct plan is streamed (plan.cpp mark_streamed)
  bool mergeable = false; // every rank's direct plans have a merged execution order (plan.cpp merged_order)
  bool has_mr = false;    // multicast reduce steps: needs the symmetric pool (NVLink SHARP)
  bool shadow = false;  // bf16 partials read/write the fp32 shadow (bf16 calls need its region)
  int max_o_chunks = 0, max_s_chunks = 0;
};

struct Reg {
  uintptr_t lo, hi;
  char* peer_base[kMaxRanks];  // peer's registered pointer (own rank: local pointer)
};

struct Comm {
  bool up = false, emulated = false, peers_set = false;
  int rank = 0, nranks = 0, device = 0;
  size_t arena_bytes = 0;
  std::vector<char*> arenas;           // local arenas (1, or nranks if emulated)
  char* peer_arena[kMaxRanks] = {};    // every rank's arena as seen by this process
  std::vector<Algo*> algos;
  std::vector<Reg> regs;
  std::map<std::string, char*> ipc_open;  // handle bytes -> mapped base
  int max_ctas = 0;
  uint64_t launches = 0;
  uint64_t timeout_ns = 0;
  unsigned long long* trace = nullptr;  // taccl_trace buffer (caller-owned)
  int trace_ctas = 0;
  int64_t staged_bytes = 0;  // one staged-mode parity region (identical on all ranks)
  // host-run pipeline (taccl_run_host): copy streams and events, created on first use
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_in[2] = {}, ev_k[2] = {}, ev_out[2] = {};
  Pool pool;  // symmetric multicast pool (taccl_pool_*), for multicast-reduce algorithms
};

Comm g;
uint64_t g_launches = 0;  // process lifetime (survives taccl_comm_destroy)

int elt_size(taccl_dtype_t d) { return d == TACCL_BFLOAT16 ? 2 : 4; }

size_t env_size(const char* name, size_t dflt) {
  const char* v = getenv(name);
  if (!v || !*v) return dflt;
  return (size_t)strtoull(v, nullptr, 10);
}

// Per-call knobs, read from the environment when a communicator is created and whenever an
// algorithm is loaded (taccl.h), not on every call: ~20 getenv scans of a 130-entry
// environment cost ~3.4 us of host time per eager call.
enum Knob {
  KN_LANES, KN_STAGED_MAX, KN_LL_MIN_PIECE, KN_MIN_PIECE, KN_TARGET_CTAS, KN_MERGED, KN_DEP_WEIGHTED,
  KN_PIECES_PER_CTA, KN_STRIPE, KN_LEAN_MAX, KN_MR_UNROLL, KN_COPY_VARIANT, KN_PULL, KN_PULL_CHAIN_MIN,
  KN_CTA_ORDER, KN_TMA, KN_READY_PER_PIECE, KN_PROG_STRIPES, KN_PAIR_SEND_WARPS, KN_COUNT
};
const char* const kKnobNames[KN_COUNT] = {
    "TACCL_LANES", "TACCL_STAGED_MAX", "TACCL_LL_MIN_PIECE", "TACCL_MIN_PIECE", "TACCL_TARGET_CTAS", "TACCL_MERGED",
    "TACCL_DEP_WEIGHTED", "TACCL_PIECES_PER_CTA", "TACCL_STRIPE", "TACCL_LEAN_MAX", "TACCL_MR_UNROLL",
    "TACCL_COPY_VARIANT", "TACCL_PULL", "TACCL_PULL_CHAIN_MIN", "TACCL_CTA_ORDER", "TACCL_TMA",
    "TACCL_READY_PER_PIECE", "TACCL_PROG_STRIPES", "TACCL_PAIR_SEND_WARPS"};
size_t g_knob_val[KN_COUNT];
bool g_knob_set[KN_COUNT];
void refresh_knobs() {
  for (int k = 0; k < KN_COUNT; ++k) {
    const char* v = getenv(kKnobNames[k]);
    g_knob_set[k] = v && *v;
    g_knob_val[k] = g_knob_set[k] ? (size_t)strtoull(v, nullptr, 10) : 0;
  }
}
inline size_t knob(Knob k, size_t dflt) { return g_knob_set[k] ? g_knob_val[k] : dflt; }

// one parity region of the staged (small-message) mode; both sit at the front of the arena's
// scratch area at a fixed place for the communicator's lifetime
int64_t staged_region_bytes() { return g.staged_bytes; }

taccl_result_t alloc_arena(char** out, size_t scratch) {
  char* p = nullptr;
  CUDA_TRY(cudaMalloc(&p, kOffScratch + scratch));
  CUDA_TRY(cudaMemset(p, 0, kOffScratch));
  Ctrl c{};
  c.epoch = 1;
  CUDA_TRY(cudaMemcpy(p + kOffCtrl, &c, sizeof(c), cudaMemcpyHostToDevice));
  *out = p;
  return TACCL_SUCCESS;
}

taccl_result_t comm_common_init(int nranks, int device, size_t scratch) {
  if (g.up) return fail(TACCL_ERR_INVALID_ARG, "communicator already initialized");
  refresh_knobs();
  if (nranks < 1 || nranks > kMaxRanks)
    return fail(TACCL_ERR_UNSUPPORTED, "nranks must be in [1, " + std::to_string(kMaxRanks) + "]");
  CUDA_TRY(cudaSetDevice(device));
  g.nranks = nranks;
  g.device = device;
  g.arena_bytes = kOffScratch + (scratch ? scratch : env_size("TACCL_SCRATCH_BYTES", 256ull << 20));
  g.timeout_ns = (uint64_t)(env_size("TACCL_TIMEOUT_S", 20) * 1000000000ull);
  g.staged_bytes = std::min<int64_t>((int64_t)env_size("TACCL_STAGED_REGION", 16 << 20),
                                     (int64_t)(g.arena_bytes - kOffScratch) / 8) & ~(int64_t)4095;
  std::string err;
  g.max_ctas = executor_max_ctas(device, &err);
  if (g.max_ctas <= 0) return fail(TACCL_ERR_CUDA, err);
  return TACCL_SUCCESS;
}

// allocation base of a device pointer via the driver entry point (no libcuda link dependency)
taccl_result_t alloc_base(const void* ptr, char** base, size_t* size) {
  typedef int (*GetRange)(unsigned long long*, size_t*, unsigned long long);
  static GetRange fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    CUDA_TRY(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
    if (!f || q != cudaDriverEntryPointSuccess) return fail(TACCL_ERR_CUDA, "cuMemGetAddressRange unavailable");
    fn = (GetRange)f;
  }
  unsigned long long b = 0;
  size_t s = 0;
  if (fn(&b, &s, (unsigned long long)(uintptr_t)ptr) != 0)
    return fail(TACCL_ERR_INVALID_ARG, "pointer is not device memory from cudaMalloc");
  *base = (char*)(uintptr_t)b;
  *size = s;
  return TACCL_SUCCESS;
}

taccl_result_t open_handle(const cudaIpcMemHandle_t& h, char** out) {
  std::string key((const char*)&h, sizeof(h));
  auto it = g.ipc_open.find(key);
  if (it != g.ipc_open.end()) {
    *out = it->second;
    return TACCL_SUCCESS;
  }
  void* p = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
  g.ipc_open[key] = (char*)p;
  *out = (char*)p;
  return TACCL_SUCCESS;
}

// message bytes S used for algorithm selection (SURVEY.md §8(b) convention 4, reading G8)
uint64_t select_bytes(taccl_coll_t coll, size_t count, int elt, int n) {
  if (coll == TACCL_ALLREDUCE) return (uint64_t)count * elt;
  // RS: nccl-tests convention, S = send bytes = n * recvcount * elt (like AG's output bytes)
  return (uint64_t)n * count * elt;
}

// mr_ok: the call may run multicast-reduce algorithms (both buffers in the symmetric pool,
// 16-byte aligned chunks); others are skipped so an ordinary algorithm for the range runs
Algo* select_algo(taccl_coll_t coll, uint64_t S, taccl_dtype_t dtype, bool mr_ok = false) {
  for (auto it = g.algos.rbegin(); it != g.algos.rend(); ++it) {  // latest load wins
    Algo* a = *it;
    if (a->has_mr && !mr_ok) continue;
    if ((int)a->coll == (int)coll && a->nranks == g.nranks && S >= a->min_bytes && ((a->dtypes >> dtype) & 1) &&
        (a->max_bytes == UINT64_MAX || S < a->max_bytes))
      return a;
  }
  return nullptr;
}

struct Geometry {
  int64_t ce = 0, chunk_bytes = 0, stripe = 0;
  int split = 1, grid = 0, budget = 0, dep_ctas = 1, staged = 0, indep_cap = 1;
  int merged = 0;  // merged execution: dep_ctas CTAs per rank, each running every threadblock
  int64_t scratch_off = 0, staging_off = 0, need = 0, shadow_off = 0, shadow_s = 0;
  std::vector<std::vector<int>> ct;  // [rank][tb] CTAs of the threadblock (0 for non-local ranks)
};

taccl_result_t geometry(const Algo* a, taccl_coll_t coll, size_t count, int elt, int nlocal_ranks,
                        int64_t base_off, Geometry* G) {
  int n_in, n_out;
  buffer_chunks(a->coll, a->nranks, a->p, &n_in, &n_out);
  const int64_t e_in = (coll == TACCL_ALLTOALL || coll == TACCL_REDUCESCATTER) ? (int64_t)a->nranks * count : (int64_t)count;
  if (e_in % n_in)
    return fail(TACCL_ERR_INVALID_ARG, "count " + std::to_string(count) + " does not split into " +
                                           std::to_string(n_in) + " equal chunks (reading G2)");
  G->ce = e_in / n_in;
  G->chunk_bytes = G->ce * elt;
  // lanes: extra CTAs per threadblock on top of the schedule's instances (same split rule)
  int total_tb = 0;
  for (int r = 0; r < a->nranks; ++r)
    if (a->plans[r].mem) total_tb += a->ntb[r];
  int lanes = 1;
  const size_t forced = knob(KN_LANES, 0);
  // staged (LL) mode for small messages: no entry handshake, no fences; sends write 16-byte
  // LL lines (8 payload bytes + flags) into the receiver's parity slot
  const int64_t sb = staged_region_bytes();
  const int64_t total_bytes = (int64_t)n_out * G->chunk_bytes;
  const int64_t ll_cb = 16 * ((G->chunk_bytes + 7) / 8);
  // LL up to 2 MiB of output for AG/A2A/AR and 4 MiB for RS (measured crossovers vs the
  // direct kernel at n=2 and n=4, profiles/r01_ll_threshold.txt); TACCL_STAGED_MAX overrides
  const int64_t ll_max = (int64_t)knob(KN_STAGED_MAX, coll == TACCL_REDUCESCATTER ? (4 << 20) : (2 << 20));
  G->staged = (int64_t)a->max_stage2_chunks * ll_cb <= sb && total_bytes <= ll_max && !a->has_mr ? 1 : 0;
  // bytes per CTA: LL lines are latency-bound, so LL pieces are small (4 KiB of payload per
  // CTA measured best at n=2 up to 1 MiB, profiles/r01_small_sweep_n2.txt)
  const int64_t min_piece = G->staged ? (int64_t)knob(KN_LL_MIN_PIECE, 4 << 10)
                                      : (int64_t)knob(KN_MIN_PIECE, 64 << 10);
  // 128 CTAs x 512 threads measured best for the HBM copy and 2-GPU pushes, 148 (one per SM)
  // for 4 ranks (AR ring +5%, AG/A2A equal; profiles/r01_scan.txt, r01_envscan_n4.txt)
  const int target = std::min(g.max_ctas, (int)knob(KN_TARGET_CTAS, g.nranks >= 4 ? 148 : 128));
  int nlocal = 0;
  for (int r = 0; r < a->nranks; ++r)
    if (a->plans[r].mem) ++nlocal;
  G->indep_cap = (int)std::max<int64_t>(1, std::min<int64_t>(kMaxSplit, (int64_t)a->max_steps_cnt * G->chunk_bytes / min_piece));
  G->budget = std::max(1, target / std::max(1, nlocal));
  // merged execution (TACCL_MERGED=1, A/B knob; plan.cpp merged_order): every CTA of a rank
  // runs all of its threadblocks, so each step gets the rank's whole CTA budget
  G->merged = !G->staged && a->mergeable && knob(KN_MERGED, 0) != 0 ? 1 : 0;
  // CTAs left for the dependent tbs once independent tbs took their weight share, shared
  // equally among the dependent tbs (TACCL_DEP_WEIGHTED=1: by data-volume weight — measured
  // slower for split send/reduce tbs, the reduce side needs its CTAs for HBM bandwidth);
  // per_dep = the largest share, which sets the piece count
  int per_dep = 1;
  const bool weighted = knob(KN_DEP_WEIGHTED, 0) != 0;
  std::vector<std::vector<int>> share(a->nranks);
  for (int r = 0; r < a->nranks; ++r) {
    if (!a->plans[r].mem) continue;
    int used = 0, ndep = 0;
    long long wdep = 0;
    for (int t = 0; t < a->ntb[r]; ++t) {
      if (a->indep[r][t]) used += tb_pieces(1, a->weights[r][t], a->wsum[r], G->budget, 1, G->indep_cap);
      else {
        ++ndep;
        wdep += std::max(1, a->weights[r][t]);
      }
    }
    const int avail = std::max(ndep, G->budget - used);
    share[r].assign(a->ntb[r], 0);
    for (int t = 0; t < a->ntb[r]; ++t)
      if (!a->indep[r][t]) {
        const int sh = weighted ? (int)std::max(1LL, (long long)avail * std::max(1, a->weights[r][t]) / std::max(1LL, wdep))
                                : std::max(1, avail / ndep);
        share[r][t] = sh;
        per_dep = std::max(per_dep, sh);
      }
  }
  if (G->merged) per_dep = G->budget;
  if (forced) {
    lanes = (int)forced;
    G->split = a->instances * lanes;
  } else {
    // pieces = CTAs of each dependent tb, each piece >= min_piece. The schedule's instances
    // (subchunks that follow the parent's path, run in parallel to fill a
    // link) set the MINIMUM piece count: the executor's pieces are already parallel lanes, so
    // when CTAs and bytes allow more pieces than m, m adds nothing (a multiple-of-m split
    // only cost CTAs: A2A n=4 1 GiB m=8 1284 vs 1197 us, profiles/r02_c3_grid_n4.txt)
    const int64_t step_bytes = (int64_t)a->max_steps_cnt * G->chunk_bytes;
    const int64_t ppc = std::max<int64_t>(1, (int64_t)knob(KN_PIECES_PER_CTA, 1));  // A/B knob
    const int64_t natural = std::max<int64_t>(1, std::min<int64_t>({step_bytes / min_piece, (int64_t)per_dep * ppc, (int64_t)kMaxSplit}));
    G->split = (int)std::min<int64_t>(kMaxSplit, std::max<int64_t>(a->instances, natural));
    lanes = (G->split + a->instances - 1) / a->instances;
  }
  // stripes: a power of two (<= TACCL_STRIPE, default 64 KiB) that also divides the chunk
  // when possible, so every stripe starts cache-line / page aligned
  int64_t gb = elt;
  while (gb < 4096 && G->chunk_bytes % (gb * 2) == 0) gb *= 2;
  // multicast reduces stream best in 16 KiB stripes (profiles/r02_nvls_scan_n4.txt: 64 MiB
  // 172 vs 183 us at 64 KiB)
  const int64_t smax = (int64_t)knob(KN_STRIPE, a->has_mr ? (16 << 10) : (64 << 10));
  int64_t st = gb;
  while (st * 2 <= smax && st * 2 * G->split <= G->chunk_bytes) st *= 2;
  G->stripe = st;
  if (G->split > kMaxSplit) return fail(TACCL_ERR_UNSUPPORTED, "instances x lanes exceeds TACCL_MAX_SPLIT");
  // every CTA of the launch must be co-resident (they wait on each other): pieces beyond the
  // device's capacity are run one after another by the same CTA
  G->dep_ctas = std::min(G->split, per_dep);
  G->grid = 0;
  G->ct.assign(a->nranks, {});
  if (G->merged) G->grid = nlocal * G->dep_ctas;
  for (int r = 0; r < a->nranks && !G->merged; ++r)
    if (a->plans[r].mem) {
      G->ct[r].assign(a->ntb[r], 0);
      for (int t = 0; t < a->ntb[r]; ++t) {
        G->ct[r][t] = a->indep[r][t] ? tb_pieces(1, a->weights[r][t], a->wsum[r], G->budget, G->split, G->indep_cap)
                                     : std::min(G->split, share[r][t]);
        G->grid += G->ct[r][t];
      }
    }
  if (G->grid > g.max_ctas)
    return fail(TACCL_ERR_UNSUPPORTED, "launch needs " + std::to_string(G->grid) + " co-resident CTAs, device holds " +
                                           std::to_string(g.max_ctas));
  G->scratch_off = kOffScratch + 2 * sb + base_off;
  G->staging_off = G->scratch_off + (((int64_t)a->max_scratch_chunks * G->chunk_bytes + 255) & ~(int64_t)255);
  G->need = G->staging_off + (int64_t)a->max_stage_chunks * G->chunk_bytes;
  // bf16 partials: the fp32 shadow of o and s (reading R6), after the staging
  G->shadow_off = G->shadow_s = 0;
  if (a->shadow && elt == 2) {
    G->shadow_off = (G->need + 255) & ~(int64_t)255;
    G->shadow_s = 2 * (int64_t)a->max_o_chunks * G->chunk_bytes;
    G->need = G->shadow_off + G->shadow_s + 2 * (int64_t)a->max_s_chunks * G->chunk_bytes;
  }
  if ((size_t)G->need > g.arena_bytes)
    return fail(TACCL_ERR_INVALID_ARG, "arena too small: need " + std::to_string(G->need) + " bytes, have " +
                                           std::to_string(g.arena_bytes) + " (raise scratch_bytes / TACCL_SCRATCH_BYTES)");
  (void)nlocal_ranks;
  return TACCL_SUCCESS;
}

// the lean copy kernel below 256 MiB: the interpreter's TMA bulk pipeline streams large copies
// faster (1 GiB: 6300 vs 6090 GB/s r+w), the lean kernel wins below (1 KB: 1.3 vs 3.2 us;
// 64 MiB: 22.3 vs 23.5 us; profiles/r01_lean_copy_n1.txt)
bool lean(const Algo* a, const Geometry& G) {
  return a->lean_copy && (int64_t)a->lean_cnt * G.chunk_bytes < (int64_t)knob(KN_LEAN_MAX, 256ull << 20);
}

taccl_result_t launch(const Algo* a, const Geometry& G, taccl_dtype_t dtype, int elt,
                      const std::vector<int>& ranks, const void* const* sends, void* const* recvs,
                      char* const (*peer_out)[kMaxRanks], void* stream,
                      const char* const (*peer_in)[kMaxRanks] = nullptr, bool mr = false) {
  if (lean(a, G)) {  // n = 1, one input -> output copy
    std::string err;
    const int64_t cb = G.chunk_bytes;
    if (launch_copy((char*)recvs[0] + a->lean_dstoff * cb, (const char*)sends[0] + a->lean_srcoff * cb,
                    a->lean_cnt * cb, stream, &err))
      return fail(TACCL_ERR_CUDA, err);
    ++g.launches;
    ++g_launches;
    return TACCL_SUCCESS;
  }
  if (mr && a->lean_mr && ranks.size() == 1) {  // one multicast reduce per rank
    KArgs M;
    memset(&M, 0, sizeof(M));
    const int r = ranks[0];
    KRank& R = M.r[0];
    R.arena = g.peer_arena[r];
    R.rank = r;
    R.mc_in = g.pool.mcva + ((const char*)sends[0] - g.pool.uc);
    R.mc_out = g.pool.mcva + ((char*)recvs[0] - g.pool.uc);
    R.nv_mc = g.pool.mcva;
    R.nv_uc = (unsigned*)g.pool.uc;
    M.nlocal = 1;
    M.nranks = g.nranks;
    M.dtype = dtype;
    M.elt = elt;
    M.timeout_ns = g.timeout_ns;
    std::string err;
    const int64_t cb = G.chunk_bytes;
    if (launch_mr(M, (int64_t)a->mr_srcoff[r] * cb, (int64_t)a->mr_dstoff[r] * cb, (int64_t)a->mr_cnt[r] * cb,
                  mr_grid(g.device), stream, &err))
      return fail(TACCL_ERR_CUDA, err);
    ++g.launches;
    ++g_launches;
    return TACCL_SUCCESS;
  }
  KArgs A;
  memset(&A, 0, sizeof(A));
  A.nlocal = (int)ranks.size();
  A.nranks = g.nranks;
  // one multimem.ld_reduce in flight per thread measured best (profiles/r02_nvls_scan_n4.txt:
  // 64 MiB 173 us at 1, 177 at 2, 183 at 4, 194 at 8)
  A.mr_unroll = (int)knob(KN_MR_UNROLL, 1);
  A.split = G.split;
  A.dep_ctas = G.dep_ctas;
  A.indep_cap = G.indep_cap;
  A.staged = G.staged;
  A.staged_bytes = staged_region_bytes();
  A.elt = elt;
  A.dtype = dtype;
  A.chunk_elems = G.ce;
  A.stripe = G.stripe;
  A.variant = (int)knob(KN_COPY_VARIANT, 0);
  A.scratch_off = G.scratch_off;
  A.staging_off = G.staging_off;
  A.shadow_off = G.shadow_off;
  A.shadow_s = G.shadow_s;
  A.timeout_ns = g.timeout_ns;
  A.trace = g.trace;
  A.trace_ctas = g.trace_ctas;
  const bool pull_on = peer_in && !G.staged && g.nranks > 1 && knob(KN_PULL, 1) != 0;
  // (not for schedules with streamed reduces: those already overlap the reduce with the
  // transfers and lose to in-place chain loads' slower peer reads — RS n=4 1 GiB 1264 vs
  // 1369 us, profiles/r02_knob_scan_prog_n4.txt)
  const bool pull_chains = pull_on && !a->plans_pc.empty() && !a->has_prog &&
                           G.chunk_bytes >= (int64_t)knob(KN_PULL_CHAIN_MIN, 64ull << 20);
  int cta = 0, smem = 0;
  for (size_t i = 0; i < ranks.size(); ++i) {
    const int r = ranks[i];
    KRank& R = A.r[i];
    const DevPlan& dp = G.staged ? a->plans_ll[r] : pull_chains ? a->plans_pc[r] : a->plans[r];
    R.plan = (const char*)dp.mem;
    R.plan_bytes = dp.bytes;
    R.steps_off = dp.steps_off;
    R.deps_off = dp.deps_off;
    R.fused_off = dp.fused_off;
    R.order_off = dp.order_off;
    R.norder = dp.norder;
    smem = std::max(smem, dp.bytes);
    R.in = (const char*)sends[i];
    R.out = (char*)recvs[i];
    R.arena = g.peer_arena[r];
    for (int q = 0; q < g.nranks; ++q) {
      R.peer_out[q] = peer_out[i][q];
      R.peer_arena[q] = g.peer_arena[q];
      R.peer_in[q] = peer_in ? peer_in[i][q] : nullptr;
    }
    if (mr) {  // multicast addresses of this call's buffers and the pool's barrier flags
      R.mc_in = g.pool.mcva + ((const char*)sends[i] - g.pool.uc);
      R.mc_out = g.pool.mcva + ((char*)recvs[i] - g.pool.uc);
      R.nv_mc = g.pool.mcva;
      R.nv_uc = (unsigned*)g.pool.uc;
    }
    R.rank = r;
    R.ntb = dp.ntb;
    R.budget = G.budget;
    R.wsum = a->wsum[r];
    const int first = cta;
    if (G.merged) {  // every CTA of the rank runs all its threadblocks (plan order)
      for (int c = 0; c < G.dep_ctas; ++c) {
        if (cta >= kMaxGrid) return fail(TACCL_ERR_UNSUPPORTED, "launch exceeds " + std::to_string(kMaxGrid) + " CTAs");
        A.cta_map[cta++] = cta_pack((int)i, 0, c, G.dep_ctas, 0) | kCtaMerged;
      }
    }
    // CTA order within the rank: round-robin over the threadblocks (CTA k of every tb, then
    // k + 1, ...), so every range of block indices — and with it every group of SMs the block
    // scheduler fills — mixes all connections (A2A n=4 1 GiB 1162 vs 1203 us, AR 64 MiB 176 vs
    // 180; profiles/r02_knob_scan_cta_order_n4.txt). TACCL_CTA_ORDER=0: tb by tb (A/B knob)
    const bool rr = knob(KN_CTA_ORDER, 1) == 1;
    int maxct = 0;
    for (int t = 0; t < dp.ntb && !G.merged; ++t) maxct = std::max(maxct, G.ct[r][t]);
    for (int o = 0; o < (rr ? maxct : dp.ntb) && !G.merged; ++o)
      for (int q = 0; q < (rr ? dp.ntb : G.ct[r][o]); ++q) {
        const int t = rr ? q : o, c = rr ? o : q;
        const int ct = G.ct[r][t];
        if (c >= ct) continue;
        if (cta >= kMaxGrid) return fail(TACCL_ERR_UNSUPPORTED, "launch exceeds " + std::to_string(kMaxGrid) + " CTAs");
        A.cta_map[cta++] = cta_pack((int)i, t, c, ct, a->indep[r][t]);
      }
    R.ncta = cta - first;
  }
  A.ncta = cta;
  A.plan_smem = smem <= kPlanSmemMax ? 1 : 0;
  A.tma = (int)knob(KN_TMA, 1);
  A.ready_per_piece = (int)knob(KN_READY_PER_PIECE, 0);
  // pull mode needs every peer's input mapped (registered, or in the symmetric arena) and
  // the direct kernel; TACCL_PULL=0 disables it
  // which receive-reduces pull is decided per step by the plan (TACCL_PULL_KINDS at load,
  // default plain rrcs only: plan.cpp); TACCL_PULL=0 turns the mode off
  // (only for plans with pulled steps: for the others the mode changes nothing, and a rank
  // running in place next to one that does not is legal)
  A.pull = (pull_on && (a->has_pull || pull_chains)) ? 1 : 0;
  // streamed messages (plan.cpp mark_streamed): progress published every TACCL_PROG_STRIPES
  // stripes (default 2; 0 = off, A/B knob — like every knob it must match on all ranks). Off in
  // pull mode (nothing is pushed) and with TMA pushes (their stores complete asynchronously)
  A.prog = (A.pull || A.tma == 2) ? 0 : (int)knob(KN_PROG_STRIPES, 2);
  // warp-specialised pairs: warps of the send part (of 16; A/B knob, default half)
  A.pair_send = 32 * (int)std::min<size_t>(15, std::max<size_t>(1, knob(KN_PAIR_SEND_WARPS, 8)));
  std::string err;
  const int dyn = (A.plan_smem ? smem : 0) + (A.staged || !A.tma ? 0 : kTmaBytes);
  if (launch_executor(A, cta, dyn, stream, &err)) return fail(TACCL_ERR_CUDA, err);
  ++g.launches;
  ++g_launches;
  return TACCL_SUCCESS;
}

taccl_result_t check_common(taccl_coll_t coll, size_t count, taccl_dtype_t dtype) {
  if (!g.up) return fail(TACCL_ERR_NOT_INITIALIZED, "no communicator");
  if (!g.emulated && !g.peers_set && g.nranks > 1) return fail(TACCL_ERR_NOT_INITIALIZED, "peers not set");
  if (coll < TACCL_ALLGATHER || coll > TACCL_REDUCESCATTER) return fail(TACCL_ERR_INVALID_ARG, "bad collective");
  if (dtype < TACCL_INT32 || dtype > TACCL_BFLOAT16) return fail(TACCL_ERR_INVALID_ARG, "bad dtype");
  (void)count;
  return TACCL_SUCCESS;
}

size_t in_bytes(taccl_coll_t coll, size_t count, int elt, int n) {
  return (coll == TACCL_ALLTOALL || coll == TACCL_REDUCESCATTER) ? (size_t)n * count * elt : count * elt;
}
size_t out_bytes(taccl_coll_t coll, size_t count, int elt, int n) {
  return (coll == TACCL_ALLREDUCE || coll == TACCL_REDUCESCATTER) ? count * elt : (size_t)n * count * elt;
}

taccl_result_t run_one(taccl_coll_t coll, const void* sendbuf, void* recvbuf, size_t count,
                       taccl_dtype_t dtype, void* stream, int64_t base_off, bool arena_out) {
  taccl_result_t rc = check_common(coll, count, dtype);
  if (rc) return rc;
  if (g.emulated) return fail(TACCL_ERR_INVALID_ARG, "emulated communicator: use taccl_run_emulated");
  if (count == 0) return TACCL_SUCCESS;
  const int elt = elt_size(dtype), n = g.nranks;
  if (!sendbuf || !recvbuf) return fail(TACCL_ERR_INVALID_ARG, "null buffer");
  const size_t ib = in_bytes(coll, count, elt, n), ob = out_bytes(coll, count, elt, n);
  const bool overlapping = (const char*)sendbuf < (const char*)recvbuf + ob && (const char*)recvbuf < (const char*)sendbuf + ib;
  // multicast-reduce algorithms need both buffers in the symmetric pool and whole 16-byte
  // vectors per chunk; an exactly in-place call is fine for them (each rank's multicast reduce
  // reads and writes only its own share, after every rank arrived)
  auto in_pool = [&](const void* p, size_t b) {
    return g.pool.up && (const char*)p >= g.pool.uc && (const char*)p + b <= g.pool.uc + g.pool.bytes;
  };
  const bool pooled = n > 1 && in_pool(sendbuf, ib) && in_pool(recvbuf, ob) && (!overlapping || sendbuf == recvbuf);
  Algo* a = select_algo(coll, select_bytes(coll, count, elt, n), dtype, pooled);
  if (a && a->has_mr) {  // chunk alignment decides too: fall back to an ordinary algorithm
    Geometry G0;
    if (geometry(a, coll, count, elt, 1, base_off, &G0) != TACCL_SUCCESS || G0.chunk_bytes % 16)
      a = select_algo(coll, select_bytes(coll, count, elt, n), dtype, false);
  }
  if (!a) return fail(TACCL_ERR_NO_ALGO, "no loaded algorithm for this collective, nranks and size");
  Geometry G;
  if ((rc = geometry(a, coll, count, elt, 1, base_off, &G))) return rc;
  if (overlapping && !a->has_mr) {
    // in-place / overlapping call (NCCL allows AG with sendbuf = recvbuf + rank*count and AR
    // with sendbuf = recvbuf; reading G10): the schedules read the input while peers write
    // the output, so the input is first copied (same stream, before the launch) to a private
    // region past this call's symmetric arena layout — private, so it need not be symmetric
    const int64_t priv = (G.need + 255) & ~(int64_t)255;
    if ((size_t)(priv + (int64_t)ib) > g.arena_bytes)
      return fail(TACCL_ERR_INVALID_ARG, "arena too small for an in-place call: need " + std::to_string(priv + ib) +
                                             " bytes (raise scratch_bytes / TACCL_SCRATCH_BYTES)");
    char* copy = g.arenas[0] + priv;
    CUDA_TRY(cudaMemcpyAsync(copy, sendbuf, ib, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    sendbuf = copy;
  }
  char* peer_out[1][kMaxRanks] = {};
  if (arena_out) {
    for (int q = 0; q < n; ++q) peer_out[0][q] = g.peer_arena[q] + ((char*)recvbuf - g.peer_arena[g.rank]);
  } else if (n > 1) {
    const Reg* hit = nullptr;
    for (const Reg& rg : g.regs)
      if ((uintptr_t)recvbuf >= rg.lo && (uintptr_t)recvbuf + ob <= rg.hi) hit = &rg;
    if (!hit) return fail(TACCL_ERR_NOT_REGISTERED, "recvbuf is not inside a registered buffer (taccl_register_buffer)");
    const uintptr_t off = (uintptr_t)recvbuf - hit->lo;
    for (int q = 0; q < n; ++q) peer_out[0][q] = hit->peer_base[q] + off;
  } else {
    peer_out[0][0] = (char*)recvbuf;
  }
  // pull mode: peers' inputs, when the input is inside a registered buffer or the arena
  // (host runs); an in-place call's private input copy is not symmetric -> no pull
  const char* peer_in[1][kMaxRanks] = {};
  bool have_in = false;
  if (n > 1 && !overlapping) {
    const char* sb = (const char*)sendbuf;
    if (sb >= g.peer_arena[g.rank] && sb + ib <= g.peer_arena[g.rank] + g.arena_bytes) {
      for (int q = 0; q < n; ++q) peer_in[0][q] = g.peer_arena[q] + (sb - g.peer_arena[g.rank]);
      have_in = true;
    } else {
      for (auto it = g.regs.rbegin(); it != g.regs.rend(); ++it)
        if (const Reg& rg = *it; (uintptr_t)sb >= rg.lo && (uintptr_t)sb + ib <= rg.hi) {
          for (int q = 0; q < n; ++q) peer_in[0][q] = rg.peer_base[q] + ((uintptr_t)sb - rg.lo);
          have_in = true;
          break;
        }
    }
  }
  std::vector<int> ranks{g.rank};
  const void* s[1] = {sendbuf};
  void* r[1] = {recvbuf};
  return launch(a, G, dtype, elt, ranks, s, r, peer_out, stream, have_in ? peer_in : nullptr, a->has_mr);
}

taccl_result_t upload(const RankPlan& rp, DevPlan* dp) {
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  const size_t b1 = al(rp.tbs.size() * sizeof(KTB)), b2 = al(rp.steps.size() * sizeof(KStep));
  const size_t b3 = al(rp.deps.size() * 4), b4 = al(rp.fused.size() * 4), b5 = al(rp.order.size() * 4);
  const size_t total = b1 + b2 + b3 + b4 + b5 + 16;
  std::vector<char> host(total, 0);
  if (!rp.tbs.empty()) memcpy(host.data(), rp.tbs.data(), rp.tbs.size() * sizeof(KTB));
  if (!rp.steps.empty()) memcpy(host.data() + b1, rp.steps.data(), rp.steps.size() * sizeof(KStep));
  if (!rp.deps.empty()) memcpy(host.data() + b1 + b2, rp.deps.data(), rp.deps.size() * 4);
  if (!rp.fused.empty()) memcpy(host.data() + b1 + b2 + b3, rp.fused.data(), rp.fused.size() * 4);
  if (!rp.order.empty()) memcpy(host.data() + b1 + b2 + b3 + b4, rp.order.data(), rp.order.size() * 4);
  char* m = nullptr;
  CUDA_TRY(cudaMalloc(&m, total));
  CUDA_TRY(cudaMemcpy(m, host.data(), total, cudaMemcpyHostToDevice));
  dp->mem = m;
  dp->bytes = (int)total;
  dp->steps_off = (int)b1;
  dp->deps_off = (int)(b1 + b2);
  dp->fused_off = (int)(b1 + b2 + b3);
  dp->order_off = (int)(b1 + b2 + b3 + b4);
  dp->norder = (int)rp.order.size();
  dp->ntb = (int)rp.tbs.size();
  return TACCL_SUCCESS;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

const char* taccl_last_error(void) { return g_err.c_str(); }

taccl_result_t taccl_check(void) {
  if (!g.up) return fail(TACCL_ERR_NOT_INITIALIZED, "no communicator");
  for (size_t i = 0; i < g.arenas.size(); ++i) {
    Ctrl c;
    CUDA_TRY(cudaMemcpy(&c, g.arenas[i] + kOffCtrl, sizeof(c), cudaMemcpyDeviceToHost));
    if (c.error && c.err_what == kErrPullMismatch)
      return fail(TACCL_ERR_INVALID_ARG, "rank " + std::to_string(c.err_rank) + " tb " + std::to_string(c.err_tb) +
                                             ": its receiver runs in the other pull mode (every rank's sendbuf must be"
                                             " registered, or none; in-place calls on all ranks or none)");
    if (c.error)
      return fail(TACCL_ERR_TIMEOUT, "device watchdog: rank " + std::to_string(c.err_rank) + " tb " +
                                         std::to_string(c.err_tb) + " step " + std::to_string(c.err_step) +
                                         " (op " + std::to_string(c.err_what) + ") waited longer than TACCL_TIMEOUT_S");
  }
  return TACCL_SUCCESS;
}

taccl_result_t taccl_validate(const char* text, size_t len, int direct_store) {
  if (!text) return fail(TACCL_ERR_INVALID_ARG, "null text");
  try {
    Program P = parse_ef(text, len);
    check_program(P, direct_store != 0);
  } catch (const SchedError& e) {
    return fail(TACCL_ERR_INVALID_SCHEDULE, e.kind + ": " + e.msg);
  }
  g_err.clear();
  return TACCL_SUCCESS;
}

taccl_result_t taccl_plan_dump(const char* text, size_t len, int rank, int ll, char* out, size_t cap,
                               size_t* needed) {
  if (!text || !needed) return fail(TACCL_ERR_INVALID_ARG, "null pointer");
  std::string d;
  try {
    Program P = parse_ef(text, len);
    check_program(P, true);
    if (rank < 0 || rank >= P.nranks) return fail(TACCL_ERR_INVALID_ARG, "rank out of range");
    const bool fuse = env_size("TACCL_NO_FUSE", 0) == 0, rrcs = env_size("TACCL_NO_RRCS", 0) == 0;
    std::vector<RankPlan> plans =
        ll ? build_plans(P, fuse, rrcs, env_size("TACCL_NO_CHAIN_SENDS_LL", 0) == 0)
           : build_plans(P, fuse, rrcs, env_size("TACCL_CHAIN_SENDS", 0) != 0, (int)env_size("TACCL_PULL_KINDS", 1));
    const RankPlan& rp = plans[rank];
    static const char* ops[] = {"SEND", "RECV", "RRC", "CPY", "NOP", "RRC_FUSED", "RRCS", "SENT", "PUB", "RCS", "MR"};
    static const char* bufs[] = {"i", "o", "s", "stage"};
    auto pairs = [&](int b, int c) {
      std::string x;
      for (int q = 0; q < c; ++q)
        x += (q ? "," : "") + std::to_string(rp.deps[2 * (b + q)]) + ":" + std::to_string(rp.deps[2 * (b + q) + 1]);
      return x;
    };
    for (size_t t = 0; t < rp.tbs.size(); ++t) {
      const KTB& kt = rp.tbs[t];
      d += "tb " + std::to_string(t) + " send=" + std::to_string(kt.send) + " recv=" + std::to_string(kt.recv) +
           " chan=" + std::to_string(kt.chan) + " indep=" + std::to_string(kt.indep) + "\n";
      for (int k = 0; k < kt.nsteps; ++k) {
        const KStep& x = rp.steps[kt.step_begin + k];
        d += "  " + std::to_string(k) + " " + ops[(int)x.op] + " src=" + bufs[(int)x.srcbuf] + ":" +
             std::to_string(x.srcoff) + " dst=" + bufs[(int)x.dstbuf] + ":" + std::to_string(x.dstoff) +
             " cnt=" + std::to_string(x.cnt) + " seq=" + std::to_string(x.seq) + " poff=" + std::to_string(x.poff) +
             " deps=" + pairs(x.dep_begin, x.dep_count) + " post=" + pairs(x.post_begin, x.post_count) +
             " part=" + std::to_string(x.part) + "/" + std::to_string(x.nparts) +
             " fuse=" + std::to_string(x.op == K_RRC_FUSED ? x.fuse_count : 0) + " fwd=" + std::to_string(x.fwd_count) +
             " pf=" + std::to_string(x.pflags) + (x.prog == 2 ? " prog2" : x.prog ? " prog" : "") + "\n";
      }
    }
    if (!rp.order.empty()) {  // merged execution order (plan.cpp merged_order): tb:step ...
      d += "order";
      for (int32_t o : rp.order) d += " " + std::to_string(o >> 16) + ":" + std::to_string(o & 0xFFFF);
      d += "\n";
    }
  } catch (const SchedError& e) {
    return fail(TACCL_ERR_INVALID_SCHEDULE, e.kind + ": " + e.msg);
  }
  *needed = d.size() + 1;
  if (out && cap) {
    const size_t m = std::min(cap - 1, d.size());
    memcpy(out, d.data(), m);
    out[m] = 0;
  }
  g_err.clear();
  return TACCL_SUCCESS;
}

taccl_result_t taccl_comm_init(int rank, int nranks, int cuda_device, size_t scratch_bytes) {
  if (rank < 0 || rank >= nranks) return fail(TACCL_ERR_INVALID_ARG, "rank out of range");
  taccl_result_t rc = comm_common_init(nranks, cuda_device, scratch_bytes);
  if (rc) return rc;
  char* a = nullptr;
  if ((rc = alloc_arena(&a, g.arena_bytes - kOffScratch))) return rc;
  g.arenas = {a};
  g.rank = rank;
  g.peer_arena[rank] = a;
  g.emulated = false;
  g.peers_set = (nranks == 1);
  g.up = true;
  return TACCL_SUCCESS;
}

taccl_result_t taccl_comm_init_emulated(int nranks, int cuda_device, size_t scratch_bytes) {
  taccl_result_t rc = comm_common_init(nranks, cuda_device, scratch_bytes);
  if (rc) return rc;
  g.arenas.clear();
  for (int r = 0; r < nranks; ++r) {
    char* a = nullptr;
    if ((rc = alloc_arena(&a, g.arena_bytes - kOffScratch))) return rc;
    g.arenas.push_back(a);
    g.peer_arena[r] = a;
  }
  g.rank = 0;
  g.emulated = true;
  g.peers_set = true;
  g.up = true;
  return TACCL_SUCCESS;
}

taccl_result_t taccl_comm_export_handle(void* out, size_t* len) {
  if (!g.up || g.emulated) return fail(TACCL_ERR_NOT_INITIALIZED, "no multi-process communicator");
  if (!out || !len) return fail(TACCL_ERR_INVALID_ARG, "null argument");
  HandleBlob b;
  memset(&b, 0, sizeof(b));
  b.magic = kMagicArena;
  b.rank = g.rank;
  b.bytes = g.arena_bytes;
  CUDA_TRY(cudaIpcGetMemHandle(&b.h, g.arenas[0]));
  memcpy(out, &b, sizeof(b));
  *len = sizeof(b);
  return TACCL_SUCCESS;
}

taccl_result_t taccl_comm_set_peers(const void* all, size_t len_each) {
  if (!g.up || g.emulated) return fail(TACCL_ERR_NOT_INITIALIZED, "no multi-process communicator");
  if (!all || len_each != sizeof(HandleBlob)) return fail(TACCL_ERR_INVALID_ARG, "bad handle blobs");
  for (int q = 0; q < g.nranks; ++q) {
    HandleBlob b;
    memcpy(&b, (const char*)all + q * len_each, sizeof(b));
    if (b.magic != kMagicArena || b.rank != q) return fail(TACCL_ERR_INVALID_ARG, "handle blob " + std::to_string(q) + " is not rank " + std::to_string(q) + "'s arena");
    if (b.bytes != g.arena_bytes) return fail(TACCL_ERR_INVALID_ARG, "ranks disagree on arena size");
    if (q == g.rank) continue;
    char* p = nullptr;
    taccl_result_t rc = open_handle(b.h, &p);
    if (rc) return rc;
    g.peer_arena[q] = p;
  }
  g.peers_set = true;
  return TACCL_SUCCESS;
}

taccl_result_t taccl_comm_destroy(void) {
  if (!g.up) return fail(TACCL_ERR_NOT_INITIALIZED, "no communicator");
  cudaDeviceSynchronize();
  for (Algo* a : g.algos) {
    for (auto& p : a->plans)
      if (p.mem) cudaFree(p.mem);
    for (auto& p : a->plans_ll)
      if (p.mem) cudaFree(p.mem);
    for (auto& p : a->plans_pc)
      if (p.mem) cudaFree(p.mem);
    delete a;
  }
  for (auto& kv : g.ipc_open) cudaIpcCloseMemHandle(kv.second);
  pool_destroy(g.pool);
  for (char* a : g.arenas) cudaFree(a);
  if (g.h2d) {
    cudaStreamDestroy(g.h2d);
    cudaStreamDestroy(g.d2h);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(g.ev_in[i]);
      cudaEventDestroy(g.ev_k[i]);
      cudaEventDestroy(g.ev_out[i]);
    }
  }
  g = Comm();
  return TACCL_SUCCESS;
}

taccl_result_t taccl_buffer_export(const void* ptr, size_t bytes, void* out, size_t* len) {
  if (!g.up || g.emulated) return fail(TACCL_ERR_NOT_INITIALIZED, "no multi-process communicator");
  if (!ptr || !out || !len) return fail(TACCL_ERR_INVALID_ARG, "null argument");
  char* base = nullptr;
  size_t size = 0;
  taccl_result_t rc = alloc_base(ptr, &base, &size);
  if (rc) return rc;
  if ((const char*)ptr + bytes > base + size) return fail(TACCL_ERR_INVALID_ARG, "range exceeds its allocation");
  HandleBlob b;
  memset(&b, 0, sizeof(b));
  b.magic = kMagicBuf;
  b.rank = g.rank;
  b.offset = (uint64_t)((const char*)ptr - base);
  b.bytes = bytes;
  CUDA_TRY(cudaIpcGetMemHandle(&b.h, base));
  memcpy(out, &b, sizeof(b));
  *len = sizeof(b);
  return TACCL_SUCCESS;
}

taccl_result_t taccl_register_buffer(const void* ptr, size_t bytes, const void* all, size_t len_each) {
  if (!g.up || g.emulated) return fail(TACCL_ERR_NOT_INITIALIZED, "no multi-process communicator");
  if (!ptr || !all || len_each != sizeof(HandleBlob)) return fail(TACCL_ERR_INVALID_ARG, "bad arguments");
  Reg rg;
  rg.lo = (uintptr_t)ptr;
  rg.hi = rg.lo + bytes;
  for (int q = 0; q < g.nranks; ++q) {
    HandleBlob b;
    memcpy(&b, (const char*)all + q * len_each, sizeof(b));
    if (b.magic != kMagicBuf || b.rank != q) return fail(TACCL_ERR_INVALID_ARG, "buffer blob " + std::to_string(q) + " invalid");
    if (b.bytes != bytes) return fail(TACCL_ERR_INVALID_ARG, "ranks registered buffers of different sizes");
    if (q == g.rank) {
      rg.peer_base[q] = (char*)ptr;
      continue;
    }
    char* base = nullptr;
    taccl_result_t rc = open_handle(b.h, &base);
    if (rc) return rc;
    rg.peer_base[q] = base + b.offset;
  }
  // the same range registered again (a freed buffer's address came back) replaces the old
  // mapping; lookups take the latest registration that covers a pointer
  g.regs.erase(std::remove_if(g.regs.begin(), g.regs.end(), [&](const Reg& o) { return o.lo == rg.lo && o.hi == rg.hi; }),
               g.regs.end());
  g.regs.push_back(rg);
  return TACCL_SUCCESS;
}

taccl_result_t taccl_unregister_buffer(const void* ptr) {
  if (!g.up || g.emulated) return fail(TACCL_ERR_NOT_INITIALIZED, "no multi-process communicator");
  const size_t before = g.regs.size();
  g.regs.erase(std::remove_if(g.regs.begin(), g.regs.end(), [&](const Reg& o) { return o.lo == (uintptr_t)ptr; }),
               g.regs.end());
  if (g.regs.size() == before) return fail(TACCL_ERR_NOT_REGISTERED, "no registration starts at this pointer");
  return TACCL_SUCCESS;
}

taccl_result_t taccl_pool_export(size_t bytes, void* out, size_t* len) {
  if (!g.up || g.emulated || g.nranks < 2) return fail(TACCL_ERR_NOT_INITIALIZED, "no multi-process communicator");
  if (g.pool.up || g.pool.phys) return fail(TACCL_ERR_INVALID_ARG, "pool already created");
  if (!out || !len || !bytes) return fail(TACCL_ERR_INVALID_ARG, "bad arguments");
  std::string err;
  if (!pool_export(g.pool, g.rank, g.nranks, g.device, bytes + kPoolFlagBytes, out, len, &err)) {
    pool_destroy(g.pool);
    return fail(TACCL_ERR_UNSUPPORTED, "pool: " + err);
  }
  return TACCL_SUCCESS;
}

taccl_result_t taccl_pool_connect(const void* all, size_t len_each) {
  if (!g.up || !g.pool.phys) return fail(TACCL_ERR_NOT_INITIALIZED, "taccl_pool_export first");
  std::string err;
  if (!pool_connect(g.pool, all, len_each, &err)) return fail(TACCL_ERR_CUDA, "pool: " + err);
  return TACCL_SUCCESS;
}

taccl_result_t taccl_pool_bind(void** base, size_t* bytes) {
  if (!g.up || !g.pool.uc) return fail(TACCL_ERR_NOT_INITIALIZED, "taccl_pool_connect first");
  std::string err;
  if (!pool_bind(g.pool, &err)) return fail(TACCL_ERR_CUDA, "pool: " + err);
  // ordinary algorithms reach pool buffers through the peers' unicast mappings
  Reg rg;
  rg.lo = (uintptr_t)g.pool.uc;
  rg.hi = rg.lo + g.pool.bytes;
  for (int q = 0; q < g.nranks; ++q) rg.peer_base[q] = g.pool.peer[q];
  g.regs.push_back(rg);
  if (base) *base = g.pool.uc + kPoolFlagBytes;
  if (bytes) *bytes = g.pool.bytes - kPoolFlagBytes;
  return TACCL_SUCCESS;
}

taccl_result_t taccl_pool_alloc(size_t bytes, void** ptr) {
  if (!g.up || !g.pool.up) return fail(TACCL_ERR_NOT_INITIALIZED, "no symmetric pool (taccl_pool_bind)");
  if (!ptr) return fail(TACCL_ERR_INVALID_ARG, "null pointer");
  const size_t at = (g.pool.used + 4095) & ~(size_t)4095;
  if (at + bytes > g.pool.bytes) return fail(TACCL_ERR_INVALID_ARG, "pool exhausted");
  g.pool.used = at + bytes;
  *ptr = g.pool.uc + at;
  return TACCL_SUCCESS;
}

taccl_result_t taccl_load_algo(const char* text, size_t len, taccl_algo_t* out) {
  if (!g.up) return fail(TACCL_ERR_NOT_INITIALIZED, "no communicator");
  refresh_knobs();
  if (!text) return fail(TACCL_ERR_INVALID_ARG, "null text");
  std::unique_ptr<Algo> a(new Algo);
  std::vector<RankPlan> plans, plans_ll, plans_pc;
  std::vector<int> P_o_chunks;
  try {
    Program P = parse_ef(text, len);
    check_program(P, true);
    if (P.nranks != g.nranks)
      return fail(TACCL_ERR_INVALID_ARG, "schedule has nranks=" + std::to_string(P.nranks) + ", communicator " + std::to_string(g.nranks));
    for (const Gpu& gp : P.gpus) {
      if ((int)gp.tbs.size() > kMaxTB) return fail(TACCL_ERR_UNSUPPORTED, "more than TACCL_MAX_TB threadblocks on a rank");
      for (const TB& tb : gp.tbs) {
        if (tb.chan >= kMaxChan) return fail(TACCL_ERR_UNSUPPORTED, "chan >= TACCL_MAX_CHAN");
        for (const Step& st : tb.steps) a->max_steps_cnt = std::max(a->max_steps_cnt, st.cnt);
      }
    }
    if (P.instances > kMaxSplit) return fail(TACCL_ERR_UNSUPPORTED, "instances > TACCL_MAX_SPLIT");
    const bool fuse = env_size("TACCL_NO_FUSE", 0) == 0, rrcs = env_size("TACCL_NO_RRCS", 0) == 0;
    // chain-send fusion pays off in the LL kernel (one step less per hop) but not in the
    // direct kernel (profiles/r01_chain_sends_ll_n4.txt): two plans, picked per call
    plans = build_plans(P, fuse, rrcs, env_size("TACCL_CHAIN_SENDS", 0) != 0, (int)env_size("TACCL_PULL_KINDS", 1));
    plans_ll = build_plans(P, fuse, rrcs, env_size("TACCL_NO_CHAIN_SENDS_LL", 0) == 0);
    const int pk = (int)env_size("TACCL_PULL_KINDS", 1);
    if (!(pk & 4)) plans_pc = build_plans(P, fuse, rrcs, env_size("TACCL_CHAIN_SENDS", 0) != 0, pk | 4);
    a->name = P.name;
    a->coll = P.coll;
    a->nranks = P.nranks;
    a->p = P.p;
    a->instances = P.instances;
    a->min_bytes = P.min_bytes;
    a->max_bytes = P.max_bytes;
    a->dtypes = P.dtypes;
    for (const Gpu& gp : P.gpus) P_o_chunks.push_back(gp.o_chunks);
  } catch (const SchedError& e) {
    return fail(TACCL_ERR_INVALID_SCHEDULE, e.kind + ": " + e.msg);
  }
  a->plans.assign(a->nranks, DevPlan());
  a->plans_ll.assign(a->nranks, DevPlan());
  // keep the pulled-chain plan only if it differs (some fused chain reads a peer's input)
  bool pc = false;
  for (const RankPlan& rp : plans_pc)
    for (size_t i = 0; i < rp.steps.size(); ++i)
      if (rp.steps[i].op == K_RRC_FUSED)
        for (int f = 0; f < rp.steps[i].fuse_count; ++f) pc = pc || rp.fused[kFuseStride * (rp.steps[i].fuse_begin + f) + 4] >= 0;
  if (pc) a->plans_pc.assign(a->nranks, DevPlan());
  a->ntb.assign(a->nranks, 0);
  for (int r = 0; r < a->nranks; ++r) {
    a->ntb[r] = (int)plans[r].tbs.size();
    a->weights.emplace_back();
    a->indep.emplace_back();
    long long ws = 0;
    for (const KTB& kt : plans[r].tbs) {
      a->weights.back().push_back(kt.weight);
      a->indep.back().push_back(kt.indep);
      ws += kt.weight;
    }
    a->wsum.push_back((int)std::min<long long>(ws, 1 << 30));
    a->max_scratch_chunks = std::max(a->max_scratch_chunks, plans[r].scratch_chunks);
    a->max_stage_chunks = std::max(a->max_stage_chunks, plans[r].stage_chunks);
    a->max_stage2_chunks = std::max(a->max_stage2_chunks, plans[r].stage2_chunks);
    a->shadow = a->shadow || plans[r].shadow || plans_ll[r].shadow;
    a->max_o_chunks = std::max(a->max_o_chunks, P_o_chunks[r]);
    a->max_s_chunks = std::max(a->max_s_chunks, plans[r].scratch_chunks);
    a->fused_chains += plans[r].fused_chains;
    for (const KStep& k : plans[r].steps) a->has_mr = a->has_mr || k.op == K_MR;
    for (const KStep& k : plans[r].steps) a->has_pull = a->has_pull || (k.op == K_SEND && k.poff >= 0);
    for (const KStep& k : plans[r].steps) a->has_prog = a->has_prog || k.prog;
    a->mergeable = (r == 0 || a->mergeable) && !plans[r].order.empty() && (!pc || !plans_pc[r].order.empty());
    {
      const RankPlan& rp = plans[r];
      const bool one_mr = rp.steps.size() == 1 && rp.steps[0].op == K_MR && rp.steps[0].dep_count == 0 &&
                          (rp.steps[0].srcbuf == KB_I || rp.steps[0].srcbuf == KB_O) && rp.steps[0].dstbuf == KB_O;
      if (r == 0) a->lean_mr = env_size("TACCL_NO_LEAN_MR", 0) == 0;
      a->lean_mr = a->lean_mr && one_mr;
      a->mr_srcoff.push_back(one_mr ? rp.steps[0].srcoff : 0);
      a->mr_dstoff.push_back(one_mr ? rp.steps[0].dstoff : 0);
      a->mr_cnt.push_back(one_mr ? rp.steps[0].cnt : 0);
      if (one_mr && rp.steps[0].srcbuf == KB_O) a->lean_mr = false;  // in-place-in-o forms: interpreter
    }
    if (a->nranks == 1 && plans[r].steps.size() == 1) {
      const KStep& k = plans[r].steps[0];
      if (k.op == K_CPY && k.srcbuf == KB_I && k.dstbuf == KB_O && k.dep_count == 0 &&
          env_size("TACCL_NO_LEAN_COPY", 0) == 0) {
        a->lean_copy = true;
        a->lean_srcoff = k.srcoff;
        a->lean_dstoff = k.dstoff;
        a->lean_cnt = k.cnt;
      }
    }
    if (g.emulated || r == g.rank) {
      taccl_result_t rc = upload(plans[r], &a->plans[r]);
      if (!rc) rc = upload(plans_ll[r], &a->plans_ll[r]);
      if (!rc && pc) rc = upload(plans_pc[r], &a->plans_pc[r]);
      if (rc) return rc;
    }
  }
  Algo* raw = a.release();
  g.algos.push_back(raw);
  if (out) *out = (taccl_algo_t)raw;
  return TACCL_SUCCESS;
}

taccl_result_t taccl_free(taccl_algo_t algo) {
  auto it = std::find(g.algos.begin(), g.algos.end(), (Algo*)algo);
  if (it == g.algos.end()) return fail(TACCL_ERR_INVALID_ARG, "unknown algorithm");
  for (auto& p : (*it)->plans)
    if (p.mem) cudaFree(p.mem);
  for (auto& p : (*it)->plans_ll)
    if (p.mem) cudaFree(p.mem);
  for (auto& p : (*it)->plans_pc)
    if (p.mem) cudaFree(p.mem);
  delete *it;
  g.algos.erase(it);
  return TACCL_SUCCESS;
}

taccl_result_t taccl_run(taccl_coll_t coll, const void* sendbuf, void* recvbuf, size_t count,
                         taccl_dtype_t dtype, void* stream) {
  return run_one(coll, sendbuf, recvbuf, count, dtype, stream, 0, false);
}

taccl_result_t taccl_run_emulated(taccl_coll_t coll, const void* const* sendbufs, void* const* recvbufs,
                                  size_t count, taccl_dtype_t dtype, void* stream) {
  taccl_result_t rc = check_common(coll, count, dtype);
  if (rc) return rc;
  if (!g.emulated) return fail(TACCL_ERR_INVALID_ARG, "not an emulated communicator");
  if (!sendbufs || !recvbufs) return fail(TACCL_ERR_INVALID_ARG, "null buffer array");
  if (count == 0) return TACCL_SUCCESS;
  const int elt = elt_size(dtype), n = g.nranks;
  Algo* a = select_algo(coll, select_bytes(coll, count, elt, n), dtype);
  if (!a) return fail(TACCL_ERR_NO_ALGO, "no loaded algorithm for this collective, nranks and size");
  Geometry G;
  if ((rc = geometry(a, coll, count, elt, n, 0, &G))) return rc;
  std::vector<int> ranks(n);
  char* peer_out[kMaxRanks][kMaxRanks] = {};
  const char* peer_in[kMaxRanks][kMaxRanks] = {};
  for (int r = 0; r < n; ++r) {
    ranks[r] = r;
    if (!sendbufs[r] || !recvbufs[r]) return fail(TACCL_ERR_INVALID_ARG, "null buffer");
    for (int q = 0; q < n; ++q) {
      peer_out[r][q] = (char*)recvbufs[q];
      peer_in[r][q] = (const char*)sendbufs[q];
    }
  }
  return launch(a, G, dtype, elt, ranks, sendbufs, recvbufs, peer_out, stream, peer_in);
}

taccl_result_t taccl_run_host(taccl_coll_t coll, const void* host_send, void* host_recv, size_t count,
                              taccl_dtype_t dtype, void* stream) {
  taccl_result_t rc = check_common(coll, count, dtype);
  if (rc) return rc;
  if (g.emulated) return fail(TACCL_ERR_INVALID_ARG, "emulated communicator: not supported for host runs");
  if (!host_send || !host_recv) return fail(TACCL_ERR_INVALID_ARG, "null buffer");
  if (count == 0) return TACCL_SUCCESS;
  const int elt = elt_size(dtype), n = g.nranks;
  // Pipelined over P pieces of the count axis: H2D of piece q+1, the collective on piece q
  // and D2H of piece q-1 overlap (PCIe is full duplex). Buffers are 1 or n rows of `count`
  // elements (rows_in / rows_out); piece q is the column range [q*cq, (q+1)*cq) of every
  // row, moved with 2-D copies into double-buffered device temps at the front of the
  // (symmetric) arena scratch, so every rank's temps sit at the same arena offset.
  const int rows_in = (coll == TACCL_ALLTOALL || coll == TACCL_REDUCESCATTER) ? n : 1;
  const int rows_out = (coll == TACCL_ALLGATHER || coll == TACCL_ALLTOALL) ? n : 1;
  const size_t piece_min = env_size("TACCL_HOST_PIECE_BYTES", 32 << 20);  // per row-set
  int P = (int)std::max<size_t>(1, std::min<size_t>(64, (size_t)rows_out * count * elt / piece_min));
  while (P > 1 && (count % P || (count / P) % (size_t)(8 * n))) --P;  // whole chunks per piece
  const size_t cq = count / P;
  const int64_t in_b = (int64_t)rows_in * cq * elt, out_b = (int64_t)rows_out * cq * elt;
  auto al = [](int64_t x) { return (x + 4095) & ~(int64_t)4095; };
  const int nb = P > 1 ? 2 : 1;
  const int64_t front = kOffScratch + 2 * staged_region_bytes();
  const int64_t base = nb * (al(in_b) + al(out_b));
  if ((size_t)(front + base) > g.arena_bytes) return fail(TACCL_ERR_INVALID_ARG, "arena too small for host run");
  char* dev_in[2] = {g.arenas[0] + front, g.arenas[0] + front + al(in_b)};
  char* dev_out[2] = {g.arenas[0] + front + nb * al(in_b), g.arenas[0] + front + nb * al(in_b) + al(out_b)};
  cudaStream_t s = (cudaStream_t)stream;
  if (P == 1) {
    CUDA_TRY(cudaMemcpyAsync(dev_in[0], host_send, (size_t)in_b, cudaMemcpyHostToDevice, s));
    if ((rc = run_one(coll, dev_in[0], dev_out[0], count, dtype, stream, base, true))) return rc;
    CUDA_TRY(cudaMemcpyAsync(host_recv, dev_out[0], (size_t)out_b, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return TACCL_SUCCESS;
  }
  if (!g.h2d) {
    CUDA_TRY(cudaStreamCreateWithFlags(&g.h2d, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&g.d2h, cudaStreamNonBlocking));
    for (int i = 0; i < 2; ++i) {
      CUDA_TRY(cudaEventCreateWithFlags(&g.ev_in[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&g.ev_k[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&g.ev_out[i], cudaEventDisableTiming));
    }
  }
  const size_t pitch = count * elt, w = cq * elt;
  // the copy streams start after everything already enqueued on the user's stream
  CUDA_TRY(cudaEventRecord(g.ev_k[0], s));
  CUDA_TRY(cudaStreamWaitEvent(g.h2d, g.ev_k[0], 0));
  CUDA_TRY(cudaStreamWaitEvent(g.d2h, g.ev_k[0], 0));
  for (int q = 0; q < P; ++q) {
    const int b = q & 1;
    if (q >= 2) CUDA_TRY(cudaStreamWaitEvent(g.h2d, g.ev_k[b], 0));  // kernel q-2 done with dev_in[b]
    CUDA_TRY(cudaMemcpy2DAsync(dev_in[b], w, (const char*)host_send + q * w, pitch, w, rows_in,
                               cudaMemcpyHostToDevice, g.h2d));
    CUDA_TRY(cudaEventRecord(g.ev_in[b], g.h2d));
    CUDA_TRY(cudaStreamWaitEvent(s, g.ev_in[b], 0));
    if (q >= 2) CUDA_TRY(cudaStreamWaitEvent(s, g.ev_out[b], 0));  // D2H q-2 done with dev_out[b]
    if ((rc = run_one(coll, dev_in[b], dev_out[b], cq, dtype, stream, base, true))) return rc;
    CUDA_TRY(cudaEventRecord(g.ev_k[b], s));
    CUDA_TRY(cudaStreamWaitEvent(g.d2h, g.ev_k[b], 0));
    CUDA_TRY(cudaMemcpy2DAsync((char*)host_recv + q * w, pitch, dev_out[b], w, w, rows_out,
                               cudaMemcpyDeviceToHost, g.d2h));
    CUDA_TRY(cudaEventRecord(g.ev_out[b], g.d2h));
  }
  CUDA_TRY(cudaStreamSynchronize(g.d2h));
  CUDA_TRY(cudaStreamSynchronize(s));
  return TACCL_SUCCESS;
}

taccl_result_t taccl_plan_info(taccl_coll_t coll, size_t count, taccl_dtype_t dtype, int* ctas, int* split,
                               int* threads) {
  taccl_result_t rc = check_common(coll, count, dtype);
  if (rc) return rc;
  const int elt = elt_size(dtype);
  Algo* a = select_algo(coll, select_bytes(coll, count, elt, g.nranks), dtype);
  if (!a) return fail(TACCL_ERR_NO_ALGO, "no loaded algorithm for this collective, nranks and size");
  Geometry G;
  if ((rc = geometry(a, coll, count, elt, 1, 0, &G))) return rc;
  if (lean(a, G)) {  // n = 1 single-copy plan: the lean copy kernel
    if (ctas) *ctas = copy_grid((int64_t)a->lean_cnt * G.chunk_bytes);
    if (split) *split = 1;
    if (threads) *threads = 256;
    return TACCL_SUCCESS;
  }
  if (ctas) *ctas = G.grid;
  if (split) *split = G.split;
  if (threads) *threads = G.staged ? kThreadsLL : kThreads;
  return TACCL_SUCCESS;
}

uint64_t taccl_launch_count(void) { return g_launches; }

taccl_result_t taccl_trace(void* dev_buf, size_t bytes) {
  if (!g.up) return fail(TACCL_ERR_NOT_INITIALIZED, "no communicator");
  if (!dev_buf) {
    g.trace = nullptr;
    g.trace_ctas = 0;
    return TACCL_SUCCESS;
  }
  const size_t per = sizeof(unsigned long long) * kTraceSlots;
  if (bytes < per) return fail(TACCL_ERR_INVALID_ARG, "trace buffer smaller than one CTA record");
  g.trace = (unsigned long long*)dev_buf;
  g.trace_ctas = (int)std::min<size_t>(bytes / per, 1 << 20);
  return TACCL_SUCCESS;
}

}  // extern "C"
