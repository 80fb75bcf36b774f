// Internal types shared by the loader/validator (host C++) and the executor (CUDA).
// The on-device plan layout and the arena layout are defined here once.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <utility>
#include <vector>

#include "../../include/taccl.h"

namespace taccl {

// ---------------------------------------------------------------- parsed program (host)
// ST_MR: multicast reduce (NVLink SHARP, reading N1): the k-th mr step of every rank
// forms group k; member r sums src[x_r..] over every rank and writes it to dst[y_r..] of every rank
enum StepType : int8_t { ST_S = 0, ST_R = 1, ST_RRC = 2, ST_CPY = 3, ST_NOP = 4, ST_MR = 5 };
enum BufId : int8_t { B_NONE = -1, B_I = 0, B_O = 1, B_S = 2 };
enum Coll : int8_t { C_AG = 0, C_A2A = 1, C_AR = 2, C_RS = 3 };

struct Step {
  int s = 0;
  StepType type = ST_NOP;
  BufId srcbuf = B_NONE;
  int srcoff = 0;
  BufId dstbuf = B_NONE;
  int dstoff = 0;
  int cnt = 0;
  std::vector<std::pair<int, int>> deps;  // (tb, step) on the same rank
};

struct TB {
  int id = 0, send = -1, recv = -1, chan = 0;
  std::vector<Step> steps;
};

struct Gpu {
  int id = 0, i_chunks = 0, o_chunks = 0, s_chunks = 0;
  std::vector<TB> tbs;
  int nchunks(BufId b) const { return b == B_I ? i_chunks : b == B_O ? o_chunks : s_chunks; }
};

struct Program {
  std::string name;
  Coll coll = C_AG;
  int nranks = 0, p = 1, instances = 1;
  uint64_t min_bytes = 0, max_bytes = 0;  // max_bytes == UINT64_MAX means inf
  uint32_t dtypes = 7;                    // bit taccl_dtype_t: element types it is selected for
  int overlap = 0;                        // execution hint: warp-specialised send + reduce pairs
  std::vector<Gpu> gpus;
};

// A check failure. kind is one of docs/SCHEDULE.md's classes.
struct SchedError {
  std::string kind, msg;
};

Program parse_ef(const char* text, size_t len);         // throws SchedError("syntax")
void check_program(const Program& prog, bool direct);   // throws SchedError
void buffer_chunks(Coll c, int n, int p, int* n_in, int* n_out);

// Happens-before over a checked program (program order + deps + send->recv matching).
class HB {
 public:
  explicit HB(const Program& P);  // throws SchedError on match / cycle errors
  ~HB();
  HB(const HB&) = delete;
  HB& operator=(const HB&) = delete;
  bool before(int r, int t, int k, int r2, int t2, int k2) const;  // strict reachability
 private:
  struct Impl;
  Impl* impl_;
};

// ---------------------------------------------------------------- device plan
// Step codes executed by the kernel.
enum KOp : int8_t {
  K_SEND = 0,      // copy local src -> peer (o / s / staging), then publish data flag
  K_RECV = 1,      // wait data flag (bytes already stored by the peer)
  K_RRC = 2,       // wait data flag, dst = src + staging
  K_CPY = 3,       // local copy
  K_NOP = 4,       // deps only
  K_RRC_FUSED = 5, // chain member: wait all chain flags, reduce its portion of
                   // dst = src + sum(staging_i) (fp32 accumulation for bf16)
  K_RRCS = 6,      // rrc fused with the next step's send of its result (recv-reduce-copy-send):
                   // one pass writes dst locally and the send's destination on the peer
  K_SENT = 7,      // a send already performed (and published) by the preceding K_RRCS
  K_PUB = 8,       // a send whose bytes the fused chain it follows already stored (fuse_chain_sends):
                   // publish the data flag only
  K_RCS = 9,       // recv fused with the next step's send of what it received (recv-copy-send,
                   // relays): LL: one pass over the lines; direct: wait, then push dst onward
  K_MR = 10        // multicast reduce (group seq): barrier, multimem.ld_reduce of src over every
                   // rank + multimem.st to every rank's dst (its pieces), barrier; direct kernel
};
enum KBuf : int8_t { KB_I = 0, KB_O = 1, KB_S = 2, KB_STAGE = 3 };

struct KStep {
  int8_t op;
  int8_t srcbuf, dstbuf;  // KBuf
  int8_t rbuf;            // K_SEND: destination buffer on the peer (KB_O / KB_S / KB_STAGE)
  int32_t srcoff, dstoff, cnt;  // chunk units
  int32_t roff;           // K_SEND/K_RRCS: destination offset on the peer (chunk units)
  int32_t fwd_seq;        // K_RRCS: message index of the fused send
  int32_t seq;            // message index on the tb's connection (K_SEND/K_RECV/K_RRC)
  int32_t soff;           // K_RRC: this rank's staging offset (chunk units)
  int32_t soff2;          // receives, staged mode: this rank's staged slot (chunk units)
  int32_t roff2;          // K_SEND/K_RRCS, staged mode: the peer's staged slot (chunk units)
  int32_t dep_begin, dep_count;  // into KRankPlan.deps (pairs tb, step)
  int32_t fuse_begin, fuse_count;  // K_RRC_FUSED: chain members' (tb, seq, soff), chain order
  int32_t part, nparts;   // K_RRC_FUSED: this member reduces portion `part` of `nparts`
  int32_t post_begin, post_count;  // deps waited AFTER the work, before publishing done
  int32_t need_done;      // some step depends on this one
  int32_t fwd_begin, fwd_count;  // K_RRC_FUSED: forward destinations (ints in the fused array:
                                 // peer, chan, rbuf, roff, roff2, seq per entry)
  int32_t poff;           // receive-reduces whose matched send reads the sender's input: that
                          // send's input offset (chunk units), else -1 (pull mode reads it in
                          // place); K_SEND: >= 0 iff its matched receive reads it in place
  int32_t pflags;         // bf16 partials (reading R6), bits P_*; bf16 calls only
  int32_t prog;           // streamed message (direct kernel): K_SEND publishes its progress every
                          // KArgs.prog stripes; K_RRC / K_RRC_FUSED reduce each stripe group as
                          // soon as every input message published it (plan.cpp mark_streamed)
};
// bf16 partials: an rrc's result keeps its fp32 accumulator in the rank's shadow region (one
// fp32 per element of o and s) when a later reduction reads it; such reads and the sends that
// feed an rrc move fp32 (2x the bf16 bytes; staging slots of fp32 messages are 2x as large)
constexpr int P_SRC = 1;   // receive-reduce: its local source is read as fp32 from the shadow
constexpr int P_IN = 2;    // receive-reduce: the matched send's message is fp32
constexpr int P_KEEP = 4;  // receive-reduce: also write the fp32 result to the destination's shadow
constexpr int P_OUT = 8;   // send (or the forward of K_RRCS): transmit fp32 (from the shadow / acc)
constexpr int P_MIX = 16;  // K_RRC_FUSED: some member message or forward is fp32 (fused array bits)
// K_RRC_FUSED member entries in the fused array: tb, seq, soff, soff2, poff, P_IN of its message
constexpr int kFuseStride = 6;
// streamed messages: the progress word carries the message index in 12 bits (executor.cu)
constexpr int kProgSeqMax = 4094;
// forward entries (fuse_chain_sends): peer, chan, rbuf, roff, roff2, seq, P_OUT
constexpr int kFwdStride = 7;

struct KTB {
  int32_t send, recv, chan;
  int32_t step_begin, nsteps;
  int32_t weight;  // data volume weight used to share the rank's CTAs among its tbs
  int32_t indep;   // no peers and no dependencies in or out: may use its own piece count
};

// ---------------------------------------------------------------- arena layout (bytes)
// Identical on every rank so peers can compute addresses in each other's arenas.
constexpr int kMaxRanks = TACCL_MAX_RANKS;
constexpr int kMaxChan = TACCL_MAX_CHAN;
constexpr int kMaxSplit = TACCL_MAX_SPLIT;
constexpr int kMaxTB = TACCL_MAX_TB;
constexpr size_t kFlagSlots = (size_t)kMaxRanks * kMaxChan * kMaxSplit;
constexpr size_t kOffData = 0;                                   // u64[kFlagSlots], written by senders
constexpr size_t kOffReady = kOffData + kFlagSlots * 8;          // u64[kFlagSlots], written by receivers
constexpr size_t kOffDone = kOffReady + kFlagSlots * 8;          // u64[kMaxTB*kMaxSplit], local
constexpr size_t kOffAck = kOffDone + (size_t)kMaxTB * kMaxSplit * 8;  // u64[kFlagSlots], pull mode:
                                                                  // written by readers of our input
constexpr size_t kOffProg = kOffAck + kFlagSlots * 8;          // u64[kFlagSlots], written by senders
                                                                  // of streamed messages (KStep.prog)
constexpr size_t kOffCtrl = kOffProg + kFlagSlots * 8;
constexpr size_t kCtrlBytes = 256;   // epoch (u64), finished (u32), error (u32), err detail
constexpr size_t kOffScratch = (kOffCtrl + kCtrlBytes + 4095) & ~(size_t)4095;

#ifdef __CUDACC__
#define TACCL_HD __host__ __device__
#else
#define TACCL_HD
#endif

TACCL_HD inline size_t flag_slot(int peer, int chan, int j) {
  return ((size_t)peer * kMaxChan + chan) * kMaxSplit + j;
}

constexpr int kErrPullMismatch = 100;  // Ctrl.err_what: ranks disagree on pull mode

struct Ctrl {
  unsigned long long epoch;
  unsigned int finished;
  unsigned int error;       // 0 ok, 1 timeout
  int err_rank, err_tb, err_step, err_what;
};

}  // namespace taccl

namespace taccl {

// ---------------------------------------------------------------- kernel arguments
// Per local rank (one in multi-process mode, all ranks when emulated). Passed by value.
struct KRank {
  const char* plan;        // the rank's plan blob: [KTB...][KStep...][deps][fused], 16-B aligned
  int32_t plan_bytes, steps_off, deps_off, fused_off;  // blob size and section offsets
  const char* in;
  char* out;
  char* arena;
  char* peer_out[kMaxRanks];    // peer's output buffer (this call's recvbuf on the peer)
  char* peer_arena[kMaxRanks];  // peer's arena (flags, scratch, staging)
  const char* peer_in[kMaxRanks];  // pull mode: peer's input buffer (this call's sendbuf on the peer)
  char* mc_in;             // multicast reduce: this call's sendbuf / recvbuf at their multicast
  char* mc_out;            // addresses (symmetric pool), else null
  char* nv_mc;             // the pool's barrier flags: multicast address ...
  unsigned* nv_uc;         // ... and this rank's local copy
  int32_t rank, ntb, ncta;  // ncta: CTAs of this rank in the launch
  int32_t budget;          // CTAs of this rank: tb t gets tb_ctas(weight_t, wsum, ...)
  int32_t wsum, pad;
  int32_t order_off, norder;  // merged execution: the plan blob's step order (tb << 16 | step)
};

struct KArgs {
  KRank r[kMaxRanks];
  int32_t nlocal;          // local ranks in this launch
  int32_t nranks;          // ranks of the communicator (multicast-reduce barriers)
  int32_t mr_unroll;       // multicast reduce: 16-byte vectors in flight per thread
  int32_t split;           // pieces per chunk (instances x lanes); flags are per piece
  int32_t variant;         // data-movement variant (env TACCL_COPY_VARIANT); timing probes
                           // only, results invalid: 9 = no fence before data flags, 20 = LL
                           // kernel returns after its prologue, 21 = no arrival wait at exit,
                           // 22 = LL sends skip their source load (send zeros)
  int32_t dep_ctas;        // CTAs per dependent tb (<= split; CTA c runs pieces c, c+dep_ctas, ...)
  int32_t plan_smem;       // copy the rank's plan blob into shared memory at kernel start
  int32_t indep_cap;       // max pieces of an independent tb (bytes / min piece)
  int32_t staged;          // staged mode: sends land in the receiver's parity staging slot,
                           // receivers copy/reduce from it; no entry handshake
  int32_t tma;             // TMA bulk copies: 0 off, 1 local copies (default), 2 + peer pushes
  int64_t staged_bytes;    // size of one parity region (at kOffScratch + parity * staged_bytes)
  int32_t elt;             // element bytes
  int32_t dtype;           // taccl_dtype_t
  int64_t chunk_elems;     // c_e
  int64_t stripe;          // bytes per stripe of a chunk (pieces own every split-th stripe)
  int64_t scratch_off;     // byte offset of the EF scratch buffer inside every arena
  int64_t staging_off;     // byte offset of the rrc staging area inside every arena
  int64_t shadow_off;      // bf16 partials: byte offset of the fp32 shadow of o inside every arena
  int64_t shadow_s;        // ... and of the shadow of s, relative to shadow_off
  uint64_t timeout_ns;
  unsigned long long* trace;  // optional %globaltimer stamps, kTraceSlots per CTA (taccl_trace)
  int32_t trace_ctas;         // CTAs that fit in the trace buffer
  int32_t ncta;               // grid size
  int32_t ready_per_piece;    // A/B knob (TACCL_READY_PER_PIECE): entry handshake per piece start
  int32_t pair_send;          // warp-specialised pairs: threads of the send part (TACCL_PAIR_SEND_WARPS)
  int32_t prog;               // streamed messages: stripes per published group (0 = off; every
                              // rank of a call agrees: off in pull mode and with TMA pushes)
  int32_t pull;               // pull mode (direct kernel): a receive-reduce whose matched send
                              // reads the sender's input loads it from the peer (no push, no
                              // staging); the reader acks, the sender's CTAs wait for the acks
                              // before they exit (its input may be reused after the call)
  uint32_t cta_map[256];      // per CTA: local rank, tb, first piece, CTAs of the tb (cta_pack)
};
constexpr int kMaxGrid = 256;

// CTA map word: tb (6 bits), first piece (9), CTAs of the tb (10), local rank (3), indep (1)
TACCL_HD inline uint32_t cta_pack(int lr, int t, int c0, int ct, int indep) {
  return (uint32_t)t | ((uint32_t)c0 << 6) | ((uint32_t)ct << 15) | ((uint32_t)lr << 25) | ((uint32_t)indep << 28);
}
TACCL_HD inline int cta_tb(uint32_t m) { return (int)(m & 63); }
TACCL_HD inline int cta_c0(uint32_t m) { return (int)((m >> 6) & 511); }
TACCL_HD inline int cta_ct(uint32_t m) { return (int)((m >> 15) & 1023); }
TACCL_HD inline int cta_lr(uint32_t m) { return (int)((m >> 25) & 7); }
TACCL_HD inline int cta_indep(uint32_t m) { return (int)((m >> 28) & 1); }
// merged execution (plan.cpp merged_order): the CTA runs every threadblock's steps of its
// pieces in the plan's level order (tb field 0, CTAs of the tb = the rank's CTAs)
constexpr uint32_t kCtaMerged = 1u << 29;
TACCL_HD inline int cta_merged(uint32_t m) { return (int)((m >> 29) & 1); }

// Trace record of one CTA (TACCL_TRACE_SLOTS u64 per CTA; first piece only):
// [0] entry, [1] prologue done (plan + epoch), then per step k < kTraceSteps:
// [2+4k] step start, [3+4k] waits satisfied, [4+4k] thread 0's own data work done (LL
// kernel only), [5+4k] step done (flag published),
// [kTraceSlots-2] identity (rank << 32 | tb << 16 | first piece), [kTraceSlots-1] exit.
constexpr int kTraceSlots = TACCL_TRACE_SLOTS;
constexpr int kTraceSteps = (kTraceSlots - 4) / 4;

#ifndef TACCL_DIRECT_THREADS
#define TACCL_DIRECT_THREADS 512
#endif
constexpr int kThreads = TACCL_DIRECT_THREADS;  // direct (bulk) kernel; 512/kThreads CTAs per SM
constexpr int kDirectPerSM = 512 / kThreads;    // (512 threads: one CTA per SM, 128 registers)
constexpr int kThreadsLL = 256;  // LL (small-message) kernel: 255 registers/thread, no spills
constexpr int kTmaStages = 4, kTmaStage = (32 << 10) / kDirectPerSM;
constexpr int kTmaBytes = kTmaStages * kTmaStage;  // dynamic smem of the direct kernel

// Pieces of one threadblock = its CTAs (same rule on host and device). Dependent tbs share
// the launch-wide split (a dependency or a connection pairs piece j with piece j); an
// independent tb (e.g. the own-chunk copy) gets its own count from its data-volume share
// of the rank's CTA budget.
TACCL_HD inline int tb_pieces(int indep, int weight, int wsum, int budget, int split, int cap) {
  if (!indep) return split;  // (run by min(split, KArgs.dep_ctas) CTAs)
  long long c = wsum > 0 ? (long long)budget * weight / wsum : 1;
  if (c > cap) c = cap;
  return c < 1 ? 1 : c > kMaxSplit ? kMaxSplit : (int)c;
}

// executor.cu
int launch_executor(const KArgs& a, int grid, int smem, void* stream, std::string* err);
// single-step local-copy plans (n = 1): dst[0, bytes) = src[0, bytes) in one lean kernel
int launch_copy(char* dst, const char* src, int64_t bytes, void* stream, std::string* err);
int copy_grid(int64_t bytes);  // its grid size
// single-step multicast-reduce plans (the nvls Allreduce): every CTA of every rank reduces the
// same grid-stride vectors of [src_off, src_off + bytes) of its share (16-byte multiple)
int launch_mr(const KArgs& a, int64_t src_off, int64_t dst_off, int64_t bytes, int grid, void* stream, std::string* err);
int mr_grid(int device);
constexpr int kPlanSmemMax = (48 << 10) / kDirectPerSM;  // plans up to this size are staged in smem
int executor_max_ctas(int device, std::string* err);  // co-resident CTA capacity

}  // namespace taccl
