/*
 * taccl.h — C ABI of the B200 executor for TACCL-EF chunk schedules (arXiv 2111.04867).
 *
 * The library runs synthesized collective algorithms (Allgather, Alltoall, Allreduce,
 * ReduceScatter):
 * every GPU executes per-threadblock programs of send / recv / recvReduceCopy / copy steps
 * over chunk indices with cross-step dependencies, the paper's runtime model
 * (§6.1), in ONE kernel launch per collective call. Bytes
 * move by direct loads/stores into peer HBM over NVLink/NVSwitch (CUDA IPC mappings); no
 * NCCL call is on the path. Schedule syntax: docs/SCHEDULE.md (EF v1).
 *
 * Threading: one communicator per process (global state). Calls are not thread-safe. As in
 * NCCL, every rank must issue the same sequence of collective calls on one stream.
 *
 * Errors: every call returns taccl_result_t. On failure taccl_last_error() returns a
 * thread-local message naming the failing check (e.g. "postcondition: (chunk 5, rank 3)
 * missing"). Device-side failures (a spin wait that exceeded TACCL_TIMEOUT_S seconds) are
 * recorded in the communicator's error word and surface from taccl_check() as
 * TACCL_ERR_TIMEOUT; the communicator must then be destroyed.
 */
#ifndef TACCL_H
#define TACCL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  TACCL_SUCCESS = 0,
  TACCL_ERR_INVALID_ARG = 1,      /* bad pointer/size/count, count not divisible into chunks */
  TACCL_ERR_INVALID_SCHEDULE = 2, /* schedule failed a check (last_error names it)          */
  TACCL_ERR_NO_ALGO = 3,          /* no loaded algorithm matches (coll, nranks, bytes)        */
  TACCL_ERR_CUDA = 4,             /* a CUDA runtime call failed (last_error has the string)   */
  TACCL_ERR_UNSUPPORTED = 5,      /* e.g. in-place call, too many ranks/threadblocks          */
  TACCL_ERR_TIMEOUT = 6,          /* device watchdog fired (see taccl_check)                  */
  TACCL_ERR_NOT_INITIALIZED = 7,  /* no communicator, or peers not set                        */
  TACCL_ERR_NOT_REGISTERED = 8    /* buffer not registered with taccl_register_buffer         */
} taccl_result_t;

/* ReduceScatter ("an inverse of Allgather"): rank r receives the
 * element-wise sum over ranks of elements [r*count, (r+1)*count) of every sendbuf. */
typedef enum {
  TACCL_ALLGATHER = 0,
  TACCL_ALLTOALL = 1,
  TACCL_ALLREDUCE = 2,
  TACCL_REDUCESCATTER = 3
} taccl_coll_t;

/* Element types. AG/A2A move raw bytes (dtype only sets the element size); AR sums:
 * INT32 wraps mod 2^32, FLOAT32 is IEEE binary32 round-to-nearest-even, BFLOAT16
 * accumulates in fp32 and rounds to nearest even once per reduction (chains of rrc into one
 * destination are fused). */
typedef enum { TACCL_INT32 = 0, TACCL_FLOAT32 = 1, TACCL_BFLOAT16 = 2 } taccl_dtype_t;

typedef struct taccl_algo* taccl_algo_t;

/* Hard limits of this build (taccl_load_algo rejects larger programs with UNSUPPORTED). */
#define TACCL_MAX_RANKS 8    /* one NVSwitch domain of 8 B200s                        */
#define TACCL_MAX_CHAN 16    /* channels per (peer, direction)                         */
#define TACCL_MAX_SPLIT 512  /* pieces per chunk (instances x lanes)                   */
#define TACCL_MAX_TB 64      /* threadblocks per rank in one schedule                  */
#define TACCL_HANDLE_BYTES 128 /* size of one exported handle blob                     */

/* ---- diagnostics ----------------------------------------------------------------------- */

/* Message for the last failing call on this thread ("" if none). Never NULL. */
const char* taccl_last_error(void);

/* Non-blocking check of the device error word; TACCL_ERR_TIMEOUT if a watchdog fired. */
taccl_result_t taccl_check(void);

/* ---- schedule checks (host only; usable without a GPU) -------------------------------- */

/* Parse and check EF v1 text (docs/SCHEDULE.md) in the documented order: syntax,
 * structure, match, cycle, race (direct_store != 0: the executor's single-assignment rule;
 * 0: queue semantics), uninit, postcondition (collective pre/postcondition over chunks,
 * App. B). `text` need not be NUL-terminated; it is not retained.
 * Returns SUCCESS or INVALID_SCHEDULE; last_error is "<class>: <message>". */
taccl_result_t taccl_validate(const char* text, size_t len, int direct_store);

/* Host-only, no communicator or GPU: check `text` (direct-store mode) and write rank `rank`'s
 * executable plan as text into out[0, cap) (NUL-terminated, truncated if cap is too small;
 * *needed = full length + 1). ll = 0: the direct kernel's plan, 1: the LL kernel's. One line
 * per threadblock ("tb <t> send=<p> recv=<p> chan=<c> indep=<0|1>") followed by one line per
 * step: "  <k> <OP> src=<buf>:<off> dst=<buf>:<off> cnt=<n> seq=<s> poff=<o> deps=<t:k,...>
 * post=<t:k,...> part=<i>/<n> fuse=<count> fwd=<count>". For tests and inspection of the
 * plan transformations (chain fusion, rrc+send fusion, pull-mode marking).
 * Env knobs that shape plans at load (TACCL_NO_FUSE, TACCL_PULL_KINDS, ...) apply; the
 * per-call knobs (TACCL_STAGED_MAX, TACCL_MIN_PIECE, TACCL_PROG_STRIPES, ...) are also re-read
 * here (and at communicator creation), not on every taccl_run.
 * Errors: INVALID_ARG (null pointers, rank out of range), INVALID_SCHEDULE. */
taccl_result_t taccl_plan_dump(const char* text, size_t len, int rank, int ll, char* out, size_t cap,
                               size_t* needed);

/* ---- communicator (one per process) ---------------------------------------------------- */
/* The paper's runtime reuses NCCL's communicator and transports (§6); this
 * build replaces them with one arena per rank that peers map over NVLink (CUDA IPC), so the
 * "connections" between threadblocks of different GPUs are plain loads and
 * stores into peer HBM plus flag words. The library owns the arena: the paper's runtime
 * "allocates ... scratch buffers" while the user preallocates input/output. */

/* One rank per process on `cuda_device`. Allocates the rank's arena in device memory:
 * flags plus `scratch_bytes` of scratch/staging (0 = default 256 MiB, env
 * TACCL_SCRATCH_BYTES overrides). Peers are unusable until taccl_comm_set_peers.
 * Errors: INVALID_ARG (rank out of range, already initialized), UNSUPPORTED (nranks outside
 * [1, TACCL_MAX_RANKS]), CUDA (allocation). */
taccl_result_t taccl_comm_init(int rank, int nranks, int cuda_device, size_t scratch_bytes);

/* All `nranks` ranks emulated in this process on one device (tests and single-GPU runs of
 * multi-rank schedules): one launch runs every rank's threadblocks, peers are the other
 * ranks' arenas in the same HBM. Use taccl_run_emulated. Errors as taccl_comm_init. */
taccl_result_t taccl_comm_init_emulated(int nranks, int cuda_device, size_t scratch_bytes);

/* Writes this rank's arena IPC handle blob (TACCL_HANDLE_BYTES) to `out`; *len = size.
 * Errors: NOT_INITIALIZED (no multi-process communicator), INVALID_ARG (null). */
taccl_result_t taccl_comm_export_handle(void* out, size_t* len);

/* `all_handles` = nranks blobs of `len_each` bytes in rank order (from an all-gather of
 * taccl_comm_export_handle). Opens the peers' arenas. Errors: INVALID_ARG (a blob is not
 * rank q's arena, arena sizes differ), CUDA (IPC open). */
taccl_result_t taccl_comm_set_peers(const void* all_handles, size_t len_each);

/* Frees algorithms, buffers registrations, peer mappings and the arena (synchronizes the
 * device first). */
taccl_result_t taccl_comm_destroy(void);

/* ---- user buffer registration (zero-copy direct stores) -------------------------------- */

/* The user preallocates the input and output buffers; a send stores
 * straight into the matched receive's destination on the peer, so the
 * peer's output must be mapped here first.
 * Collective, like NCCL window registration: every rank registers its own buffer of the
 * same role in the same order. Step 1: export a blob for [ptr, ptr+bytes) (any pointer
 * inside a cudaMalloc'd allocation). Step 2: pass all ranks' blobs (rank order) to
 * taccl_register_buffer. Afterwards a taccl_run whose recvbuf lies inside [ptr, ptr+bytes)
 * stores into the peers' registered buffers at the same offset, and one whose sendbuf lies
 * inside a registered buffer runs in pull mode (receive-reduces fed by a peer's input load it
 * in place over NVLink; the call then completes only after every reader is done with this
 * rank's sendbuf). An unregistered sendbuf is pushed (no pull mode).
 * Registering the same range again replaces the earlier mapping; lookups use the latest
 * registration covering a pointer. All ranks of a call must agree on pull mode: either every
 * rank's sendbuf lies in a registered buffer (and no rank runs in place) or none does. A
 * disagreement is detected by the entry handshake before any data moves: the sender aborts
 * and taccl_check returns INVALID_ARG naming it (its receiver then surfaces TIMEOUT).
 * Errors: NOT_INITIALIZED, INVALID_ARG (not device memory, range beyond its allocation,
 * blob mismatch, sizes differ across ranks), CUDA (IPC). */
taccl_result_t taccl_buffer_export(const void* ptr, size_t bytes, void* out, size_t* len);
taccl_result_t taccl_register_buffer(const void* ptr, size_t bytes, const void* all_blobs,
                                     size_t len_each);
/* Local: drop the registration that starts at `ptr` (before the buffer is freed).
 * Errors: NOT_INITIALIZED, NOT_REGISTERED (no registration starts at ptr). */
taccl_result_t taccl_unregister_buffer(const void* ptr);

/* ---- symmetric multicast pool (NVLink SHARP) ------------------------------------------ */

/* B200 extension (reading N1, §5 "pool"): the NVSwitch can reduce in the switch —
 * multimem.ld_reduce returns the sum of every GPU's copy of an address, multimem.st writes all
 * copies — which needs memory bound to a multicast object. The pool is that memory: one
 * cuMemCreate allocation of the same size per rank, every peer's mapped here (so ordinary
 * schedules reach pool buffers too), and one multicast object bound over all of them.
 * Collective, in three phases with a host exchange between them (the Python binding's
 * Comm.create_pool drives them over torch.distributed):
 *   1. taccl_pool_export(bytes): allocate, and for rank 0 create the multicast object; writes a
 *      TACCL_HANDLE_BYTES blob naming this rank's descriptor socket.
 *   2. taccl_pool_connect(all blobs, rank order): exchange the allocation/multicast handles as
 *      POSIX file descriptors over Unix domain sockets, map every peer, add this device to the
 *      multicast object.
 *   3. (after every rank finished phase 2) taccl_pool_bind: bind this rank's memory to the
 *      multicast object, map it, clear the barrier flags; *base / *bytes = the allocatable
 *      range. Every rank must then pass a host barrier before any collective uses the pool.
 * taccl_pool_alloc: symmetric bump allocation (call in the same order with the same sizes on
 * every rank; 4 KiB aligned). A taccl_run whose sendbuf and recvbuf both lie in the pool may
 * select multicast-reduce algorithms (EF step `mr`); other calls skip them. The choice is
 * local, so every rank of a call must agree: either all ranks' buffers lie in the pool at the
 * same offsets (the symmetric allocation order above gives that) or none does. A disagreement
 * is not detected before data moves; it surfaces as TIMEOUT from taccl_check.
 * Errors: NOT_INITIALIZED (no multi-process communicator / wrong phase order), UNSUPPORTED (no
 * multicast support), CUDA (driver calls, descriptor exchange), INVALID_ARG (pool exhausted).
 * The pool lives until taccl_comm_destroy. */
taccl_result_t taccl_pool_export(size_t bytes, void* blob, size_t* len);
taccl_result_t taccl_pool_connect(const void* all_blobs, size_t len_each);
taccl_result_t taccl_pool_bind(void** base, size_t* bytes);
taccl_result_t taccl_pool_alloc(size_t bytes, void** ptr);

/* ---- north-star calls ------------------------------------------------------------------ */

/* taccl_load_algo: the paper's lowered TACCL-EF program (§6.1: buffers,
 * threadblocks with one send and one receive peer, steps with dependencies) arrives as
 * text (EF v1, docs/SCHEDULE.md). It is parsed, checked in direct-store mode (structure,
 * matching, acyclicity, races, and the collective's postcondition "each chunk reaches its
 * destination GPUs as specified by the collective"; App. B
 * PAPER.md:1324-1330) and planned for the device. The algorithm is registered under
 * (coll, nranks, [minBytes, maxBytes), dtypes) for selection by taccl_run — the paper keeps
 * size-specialised algorithms per collective; the optional dtypes
 * attribute restricts the element types (docs/SCHEDULE.md). `*out` may be NULL.
 * Ownership: the text is copied (not retained); the library owns the device plan until
 * taccl_free or taccl_comm_destroy. Requires an initialized communicator whose nranks
 * matches. Errors: INVALID_SCHEDULE ("<class>: <message>", first failing check),
 * INVALID_ARG (nranks mismatch, null), UNSUPPORTED (limits above), CUDA. */
taccl_result_t taccl_load_algo(const char* schedule_text, size_t len, taccl_algo_t* out);

/* taccl_run: one collective call with NCCL-compatible semantics ("the
 * same API as NCCL"), executed "in a single kernel launch" with the loaded
 * algorithm selected by (coll, nranks, S) where S =
 * output bytes (AG), per-rank send bytes (A2A), buffer bytes (AR), send bytes (RS). NCCL
 * count convention: AG count = elements per rank (recvbuf holds nranks*count), A2A count =
 * elements per peer (both buffers hold nranks*count), AR count = total elements, RS count =
 * elements per rank (sendbuf holds nranks*count, recvbuf count). Chunks are equal-sized
 * (PAPER.md:742-744): the input splits into N_in chunks of c_e = E_in / N_in elements.
 * sendbuf/recvbuf are user-owned device pointers; recvbuf must be
 * registered (taccl_register_buffer) unless emulated or nranks == 1; a registered sendbuf
 * enables pull mode (TACCL_PULL=0 disables it). sendbuf is read-only for the call; recvbuf
 * is valid once `stream` passes the call.
 * In-place / overlapping buffers are accepted (the input is first copied, on `stream`, to a
 * private arena region; INVALID_ARG if the arena is too small). Enqueues ONE kernel on `stream`
 * (a cudaStream_t; NULL = legacy default stream); returns without synchronizing. The
 * call is CUDA-graph capturable (epochs live on the device).
 * Errors: NOT_INITIALIZED, INVALID_ARG (null buffer, count not divisible into N_in chunks
 * (reading G2), arena too small), NO_ALGO (no loaded algorithm for (coll, nranks, S)),
 * NOT_REGISTERED (recvbuf), UNSUPPORTED (launch needs more co-resident CTAs than the device
 * holds), CUDA (launch). Device-side failures surface later through taccl_check. */
taccl_result_t taccl_run(taccl_coll_t coll, const void* sendbuf, void* recvbuf, size_t count,
                         taccl_dtype_t dtype, void* stream);

/* Emulated communicator: sendbufs[r]/recvbufs[r] are rank r's device buffers. */
taccl_result_t taccl_run_emulated(taccl_coll_t coll, const void* const* sendbufs,
                                  void* const* recvbufs, size_t count, taccl_dtype_t dtype,
                                  void* stream);

/* Same as taccl_run with HOST buffers: copies sendbuf H2D, runs, copies recvbuf D2H on
 * `stream` through library-owned device buffers, and synchronizes the stream. For
 * end-to-end measurements; pinned host memory gives full PCIe bandwidth. */
taccl_result_t taccl_run_host(taccl_coll_t coll, const void* host_send, void* host_recv,
                              size_t count, taccl_dtype_t dtype, void* stream);

/* taccl_free: release an algorithm and its device plan (the runtime-owned half of the
 * paper's buffer split). Invalid while a run using it is in flight
 * (synchronize the stream first). Errors: INVALID_ARG (unknown or already freed handle). */
taccl_result_t taccl_free(taccl_algo_t algo);

/* ---- introspection (tests, bench) ----------------------------------------------------- */

/* Launch geometry taccl_run would use: CTAs of the single launch and split factor
 * (instances x lanes). */
taccl_result_t taccl_plan_info(taccl_coll_t coll, size_t count, taccl_dtype_t dtype,
                               int* ctas, int* split, int* threads);

/* Number of executor kernel launches issued by this process so far. */
uint64_t taccl_launch_count(void);

/* Device-side step timeline (SURVEY.md §5 tracing). `dev_buf` is a device buffer of `bytes`
 * bytes owned by the caller; while set, every launch overwrites it with TACCL_TRACE_SLOTS
 * u64 %globaltimer stamps (ns) per CTA, CTA-major (layout in taccl_internal.h): entry,
 * prologue end, then per step start / waits satisfied / done, identity word, exit. CTAs
 * beyond bytes / (8 * TACCL_TRACE_SLOTS) are not traced. NULL disables (the default).
 * Returns INVALID_ARG if bytes is smaller than one CTA's record. */
#define TACCL_TRACE_SLOTS 64
taccl_result_t taccl_trace(void* dev_buf, size_t bytes);

#ifdef __cplusplus
}
#endif
#endif /* TACCL_H */
