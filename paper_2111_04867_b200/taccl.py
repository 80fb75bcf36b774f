"""Thin Python binding of the C ABI (include/taccl.h): argument marshalling only.

Every step of a collective runs inside libtaccl.so (one sm_100a kernel launch per call);
this module converts torch tensors to pointers/counts/streams and, for multi-process
communicators, drives the one-time handle exchange through torch.distributed (CS3 in
SURVEY.md §3). There is no fallback: if the in-tree library is missing, import fails.
"""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TACCL_LIB") or os.path.join(HERE, "libtaccl.so")  # TACCL_LIB: experiment variants

ALLGATHER, ALLTOALL, ALLREDUCE, REDUCESCATTER = 0, 1, 2, 3
INT32, FLOAT32, BFLOAT16 = 0, 1, 2
COLLS = {"allgather": ALLGATHER, "alltoall": ALLTOALL, "allreduce": ALLREDUCE, "reducescatter": REDUCESCATTER}
REDUCING = (ALLREDUCE, REDUCESCATTER)
ERRORS = {0: "SUCCESS", 1: "INVALID_ARG", 2: "INVALID_SCHEDULE", 3: "NO_ALGO", 4: "CUDA",
          5: "UNSUPPORTED", 6: "TIMEOUT", 7: "NOT_INITIALIZED", 8: "NOT_REGISTERED"}
HANDLE_BYTES = 128
TRACE_SLOTS = 64  # TACCL_TRACE_SLOTS

_lib = None


class TacclError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"taccl {ERRORS.get(code, code)}: {msg}")
        self.code = code
        self.msg = msg


def lib():
    """Load the in-tree libtaccl.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        c_int, c_size, c_vp, c_cp = ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_char_p
        sig = {
            "taccl_last_error": ([], c_cp),
            "taccl_check": ([], c_int),
            "taccl_validate": ([c_cp, c_size, c_int], c_int),
            "taccl_plan_dump": ([c_cp, c_size, c_int, c_int, c_vp, c_size, ctypes.POINTER(c_size)], c_int),
            "taccl_comm_init": ([c_int, c_int, c_int, c_size], c_int),
            "taccl_comm_init_emulated": ([c_int, c_int, c_size], c_int),
            "taccl_comm_export_handle": ([c_vp, ctypes.POINTER(c_size)], c_int),
            "taccl_comm_set_peers": ([c_vp, c_size], c_int),
            "taccl_comm_destroy": ([], c_int),
            "taccl_buffer_export": ([c_vp, c_size, c_vp, ctypes.POINTER(c_size)], c_int),
            "taccl_register_buffer": ([c_vp, c_size, c_vp, c_size], c_int),
            "taccl_unregister_buffer": ([c_vp], c_int),
            "taccl_pool_export": ([c_size, c_vp, ctypes.POINTER(c_size)], c_int),
            "taccl_pool_connect": ([c_vp, c_size], c_int),
            "taccl_pool_bind": ([ctypes.POINTER(c_vp), ctypes.POINTER(c_size)], c_int),
            "taccl_pool_alloc": ([c_size, ctypes.POINTER(c_vp)], c_int),
            "taccl_load_algo": ([c_cp, c_size, ctypes.POINTER(c_vp)], c_int),
            "taccl_run": ([c_int, c_vp, c_vp, c_size, c_int, c_vp], c_int),
            "taccl_run_emulated": ([c_int, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_size, c_int, c_vp], c_int),
            "taccl_run_host": ([c_int, c_vp, c_vp, c_size, c_int, c_vp], c_int),
            "taccl_free": ([c_vp], c_int),
            "taccl_plan_info": ([c_int, c_size, c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_int),
                                 ctypes.POINTER(c_int)], c_int),
            "taccl_launch_count": ([], ctypes.c_uint64),
            "taccl_trace": ([c_vp, c_size], c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise TacclError(rc, lib().taccl_last_error().decode())


def last_error() -> str:
    return lib().taccl_last_error().decode()


def plan_dump(text: str, rank: int, ll: bool = False) -> str:
    """Rank `rank`'s executable plan as text (host only; include/taccl.h taccl_plan_dump)."""
    b = text.encode()
    need = ctypes.c_size_t(0)
    _check(lib().taccl_plan_dump(b, len(b), rank, int(ll), None, 0, ctypes.byref(need)))
    buf = ctypes.create_string_buffer(need.value)
    _check(lib().taccl_plan_dump(b, len(b), rank, int(ll), buf, need.value, ctypes.byref(need)))
    return buf.value.decode()


def validate(text: str, direct: bool = True):
    """(ok, kind, message) from the C++ validator (host only; no GPU needed)."""
    b = text.encode()
    rc = lib().taccl_validate(b, len(b), 1 if direct else 0)
    if rc == 0:
        return True, None, ""
    msg = last_error()
    kind, _, rest = msg.partition(": ")
    return False, kind, rest


def dtype_code(t, coll):
    import torch
    if coll in REDUCING:
        m = {torch.int32: INT32, torch.float32: FLOAT32, torch.bfloat16: BFLOAT16}
        if t.dtype not in m:
            raise TypeError(f"allreduce/reducescatter support int32/float32/bfloat16, got {t.dtype}")
        return m[t.dtype]
    # AG / A2A move raw bytes: only the element size matters
    es = t.element_size()
    if es == 4:
        return INT32
    if es == 2:
        return BFLOAT16
    raise TypeError(f"allgather/alltoall support 2- and 4-byte elements, got {t.dtype}")


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


class Comm:
    """One communicator per process (the C library holds global state)."""

    def __init__(self, rank=0, nranks=1, device=0, scratch_bytes=0, emulated=False, group=None):
        self.rank, self.nranks, self.device, self.emulated = rank, nranks, device, emulated
        self.group = group
        if emulated:
            _check(lib().taccl_comm_init_emulated(nranks, device, scratch_bytes))
        else:
            _check(lib().taccl_comm_init(rank, nranks, device, scratch_bytes))
            if nranks > 1:
                blob = ctypes.create_string_buffer(HANDLE_BYTES)
                n = ctypes.c_size_t(0)
                _check(lib().taccl_comm_export_handle(blob, ctypes.byref(n)))
                allb = self._all_gather_bytes(blob.raw[:n.value])
                _check(lib().taccl_comm_set_peers(allb, HANDLE_BYTES))

    def _all_gather_bytes(self, b: bytes) -> bytes:
        return all_gather_blobs(b, self.nranks, self.group)

    def load(self, text: str):
        b = text.encode()
        h = ctypes.c_void_p()
        _check(lib().taccl_load_algo(b, len(b), ctypes.byref(h)))
        return h

    def load_defaults(self, colls=("allgather", "alltoall", "allreduce", "reducescatter")):
        """Load the size-specialised default schedule set of every collective in `colls`
        (generator/tuned.py); returns the algorithm handles."""
        from .generator.tuned import default_schedules
        return [self.load(t) for c in colls for t in default_schedules(c, self.nranks)]

    def free(self, h):
        _check(lib().taccl_free(h))

    def register(self, t):
        """Collective (every rank, same role, same order — like NCCL window registration): map
        tensor `t`'s storage on every rank, as a zero-copy receive target (outputs) or an
        in-place pull source (inputs, pull mode). Explicit: run() never registers, so no rank
        can enter the exchange while another skips it. Registering a storage range again
        replaces the earlier mapping (a freed tensor's address may come back with different
        peer addresses)."""
        if self.emulated or self.nranks == 1:
            return
        ptr, nbytes = t.untyped_storage().data_ptr(), t.untyped_storage().nbytes()
        if self._in_pool(ptr, nbytes):  # pool tensors are mapped on every rank already
            return
        blob = ctypes.create_string_buffer(HANDLE_BYTES)
        n = ctypes.c_size_t(0)
        _check(lib().taccl_buffer_export(ctypes.c_void_p(ptr), nbytes, blob, ctypes.byref(n)))
        allb = self._all_gather_bytes(blob.raw[:n.value])
        _check(lib().taccl_register_buffer(ctypes.c_void_p(ptr), nbytes, allb, HANDLE_BYTES))

    def create_pool(self, nbytes):
        """Collective: the symmetric multicast pool (include/taccl.h taccl_pool_*), so
        multicast-reduce (NVLink SHARP) algorithms can run on tensors from pool_tensor()."""
        blob = ctypes.create_string_buffer(HANDLE_BYTES)
        n = ctypes.c_size_t(0)
        rc = lib().taccl_pool_export(nbytes, blob, ctypes.byref(n))
        err = last_error() if rc else ""
        allb = self._all_gather_bytes(blob.raw if rc == 0 else b"\0" * HANDLE_BYTES)  # every rank joins
        if rc:
            raise TacclError(rc, err)
        if any(int.from_bytes(allb[q * HANDLE_BYTES:q * HANDLE_BYTES + 4], "little") != 0x7acc1c0d
               for q in range(self.nranks)):
            raise TacclError(5, "a peer could not create its pool")
        _check(lib().taccl_pool_connect(allb, HANDLE_BYTES))
        self._barrier()  # every device added to the multicast object before anyone binds
        base, size = ctypes.c_void_p(), ctypes.c_size_t()
        _check(lib().taccl_pool_bind(ctypes.byref(base), ctypes.byref(size)))
        self._pool = (base.value, size.value)
        self._barrier()  # flags cleared everywhere before any collective uses them
        return size.value

    def pool_tensor(self, numel, dtype):
        """A tensor in the symmetric pool (same offset on every rank: allocate in the same order
        with the same sizes everywhere)."""
        import torch
        nbytes = numel * torch.empty((), dtype=dtype).element_size()
        p = ctypes.c_void_p()
        _check(lib().taccl_pool_alloc(nbytes, ctypes.byref(p)))

        class _Mem:  # zero-copy view (CUDA array interface); the pool owns the memory
            __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (p.value, False), "version": 3}
        return torch.as_tensor(_Mem(), device="cuda").view(dtype)

    def _barrier(self):
        import torch.distributed as dist
        dist.barrier(group=self.group)

    def _in_pool(self, ptr, nbytes):
        base, size = getattr(self, "_pool", (0, 0))
        return base <= ptr and ptr + nbytes <= base + size

    def unregister(self, t):
        """Local: forget the mapping of `t`'s storage (call before the tensor is freed)."""
        if self.emulated or self.nranks == 1:
            return
        if self._in_pool(t.untyped_storage().data_ptr(), t.untyped_storage().nbytes()):
            return
        _check(lib().taccl_unregister_buffer(ctypes.c_void_p(t.untyped_storage().data_ptr())))

    def run(self, coll, out, inp, stream=None):
        """One collective call; `coll` in COLLS. Tensors are contiguous CUDA tensors. With
        nranks > 1, `out` must lie in a registered storage (register(); NOT_REGISTERED
        otherwise); a registered `inp` enables pull mode (every rank's, or none)."""
        c = COLLS[coll] if isinstance(coll, str) else coll
        n = self.nranks
        count = inp.numel() // n if c in (ALLTOALL, REDUCESCATTER) else inp.numel()
        _check(lib().taccl_run(c, ctypes.c_void_p(inp.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                               count, dtype_code(inp, c), _stream(stream)))

    def run_emulated(self, coll, outs, inps, stream=None):
        c = COLLS[coll] if isinstance(coll, str) else coll
        n = self.nranks
        count = inps[0].numel() // n if c in (ALLTOALL, REDUCESCATTER) else inps[0].numel()
        S = (ctypes.c_void_p * n)(*[x.data_ptr() for x in inps])
        R = (ctypes.c_void_p * n)(*[x.data_ptr() for x in outs])
        _check(lib().taccl_run_emulated(c, S, R, count, dtype_code(inps[0], c), _stream(stream)))

    def run_host(self, coll, host_out, host_in, stream=None):
        """End-to-end: host input -> device -> collective -> host output (numpy or pinned torch)."""
        c = COLLS[coll] if isinstance(coll, str) else coll
        n = self.nranks
        count = host_in.numel() // n if c in (ALLTOALL, REDUCESCATTER) else host_in.numel()
        _check(lib().taccl_run_host(c, ctypes.c_void_p(host_in.data_ptr()), ctypes.c_void_p(host_out.data_ptr()),
                                    count, dtype_code(host_in, c), _stream(stream)))

    def plan_info(self, coll, count, dtype_c):
        c = COLLS[coll] if isinstance(coll, str) else coll
        a, b, t = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().taccl_plan_info(c, count, dtype_c, ctypes.byref(a), ctypes.byref(b), ctypes.byref(t)))
        return {"ctas": a.value, "split": b.value, "threads": t.value}

    def trace(self, buf):
        """Per-step %globaltimer timeline of the following launches into device tensor `buf`
        (TRACE_SLOTS u64 per CTA); None disables."""
        if buf is None:
            _check(lib().taccl_trace(None, 0))
        else:
            _check(lib().taccl_trace(ctypes.c_void_p(buf.data_ptr()), buf.numel() * buf.element_size()))

    def check(self):
        _check(lib().taccl_check())

    def destroy(self):
        _check(lib().taccl_comm_destroy())

    # NCCL-style conveniences (PAPER.md:755-757 API compatibility, reading M20)
    def all_gather(self, out, inp, stream=None):
        self.run(ALLGATHER, out, inp, stream)

    def all_to_all(self, out, inp, stream=None):
        self.run(ALLTOALL, out, inp, stream)

    def all_reduce(self, out, inp, stream=None):
        self.run(ALLREDUCE, out, inp, stream)

    def reduce_scatter(self, out, inp, stream=None):
        self.run(REDUCESCATTER, out, inp, stream)


def all_gather_blobs(b: bytes, nranks: int, group=None) -> bytes:
    """The one-time handle exchange: every rank's fixed-size blob, in rank
    order, concatenated — the layout taccl_comm_set_peers / taccl_register_buffer expect.
    Works on any torch.distributed backend (gloo in the CPU tests, nccl in the bench)."""
    import torch.distributed as dist
    if len(b) != HANDLE_BYTES:
        raise ValueError(f"handle blobs are {HANDLE_BYTES} bytes, got {len(b)}")
    out = [None] * nranks
    dist.all_gather_object(out, b, group=group)
    return b"".join(out)


def launch_count() -> int:
    return int(lib().taccl_launch_count())
