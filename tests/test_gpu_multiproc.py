"""Multi-process parity (one process per GPU, peers mapped with CUDA IPC over NVLink):
every rank's output vs the oracle, bit-exact for AG/A2A/int32-AR and integer-valued float
AR. Skipped when fewer than 2 GPUs are visible (the round-end box may have one; the
emulated tests in test_gpu_parity.py cover the same schedules on one GPU)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.gpu2]

NGPU = torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, n, port, cases, q):
    import torch.distributed as dist

    import oracle
    from paper_2111_04867_b200 import taccl
    from paper_2111_04867_b200.generator import generate
    from paper_2111_04867_b200.inputs import allreduce_input, random_bits
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    try:
        comm = taccl.Comm(rank=rank, nranks=n, device=rank, scratch_bytes=64 << 20)
        tdt = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}
        view = {"int32": np.int32, "float32": np.int32, "bfloat16": np.int16}
        results = []
        for (coll, algo, p, m, dtype, count, kind) in cases:
            text = generate(coll, algo, n, p, m)
            h = comm.load(text)
            e_in = n * count if coll in ("alltoall", "reducescatter") else count
            if coll in ("allreduce", "reducescatter"):
                ins = [allreduce_input(e_in, dtype, kind, 21, r) for r in range(n)]
            else:
                ins = [random_bits(e_in, dtype, 22, r) for r in range(n)]
            x = torch.from_numpy(ins[rank].view(view[dtype])).view(tdt[dtype]).cuda()
            e_out = count if coll in ("allreduce", "reducescatter") else n * count
            out = torch.empty(e_out, dtype=tdt[dtype], device="cuda")
            comm.register(out)  # collective, explicit (run() never registers)
            comm.register(x)    # pull mode for receive-reduces fed by a peer's input
            for _ in range(3):  # repeated calls exercise epochs / entry handshakes
                out.view(torch.uint8).fill_(0xA5)
                comm.run(coll, out, x)
            torch.cuda.synchronize()
            comm.check()
            got = out.cpu().view({"int32": torch.int32, "float32": torch.int32, "bfloat16": torch.int16}[dtype]).numpy()
            want = oracle.run(oracle.parse(text), ins, dtype)[rank]
            ok = bool(np.array_equal(got.view(want.dtype), want))
            # the same call through host buffers, pipelined in several pieces (e2e path)
            os.environ["TACCL_HOST_PIECE_BYTES"] = str(1 << 14)
            h_in = torch.from_numpy(ins[rank].view(view[dtype])).view(tdt[dtype]).pin_memory()
            h_out = torch.empty(e_out, dtype=tdt[dtype]).pin_memory()
            comm.run_host(coll, h_out, h_in)
            os.environ.pop("TACCL_HOST_PIECE_BYTES")
            vt = {"int32": torch.int32, "float32": torch.int32, "bfloat16": torch.int16}[dtype]
            ok = ok and bool(np.array_equal(h_out.view(vt).numpy().view(want.dtype), want))
            # NCCL's in-place forms (reading G10): AR sendbuf == recvbuf, AG sendbuf = own slot
            if coll in ("allreduce", "allgather"):
                buf = torch.empty(e_out, dtype=tdt[dtype], device="cuda")
                comm.register(buf)
                if coll == "allreduce":
                    buf.copy_(x)
                    comm.run(coll, buf, buf)
                else:
                    buf[rank * count:(rank + 1) * count].copy_(x)
                    comm.run(coll, buf, buf[rank * count:(rank + 1) * count])
                torch.cuda.synchronize()
                ok = ok and bool(np.array_equal(buf.cpu().view(vt).numpy().view(want.dtype), want))
                comm.unregister(buf)
            results.append(ok)
            comm.unregister(out)
            comm.unregister(x)
            comm.free(h)
        comm.destroy()
        q.put((rank, results, None))
    except Exception as e:  # report to the parent instead of hanging it
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


CASES = [
    ("allgather", "direct", 1, 1, "bfloat16", 1 << 16, None),
    ("allgather", "ring", 2, 2, "int32", 2 * 50001, None),
    ("alltoall", "direct", 2, 4, "bfloat16", 2 * 7777, None),
    ("allreduce", "direct", 1, 1, "int32", 4 * 300001, "bits"),
    ("allreduce", "ring", 2, 1, "bfloat16", 8 * 4099, "intval"),
    ("allreduce", "direct", 1, 2, "float32", 2 * (1 << 18), "intval"),
    ("allgather", "direct", 1, 1, "bfloat16", 3, None),
    ("reducescatter", "direct", 1, 1, "float32", 1 << 17, "intval"),
    ("reducescatter", "ring", 2, 2, "int32", 2 * 3001, "bits"),
    # above the LL threshold: the direct kernel in pull mode (inputs registered by comm.run)
    ("reducescatter", "direct", 1, 1, "bfloat16", 3 << 20, "intval"),
    ("reducescatter", "direct", 2, 2, "int32", 2 * 600007, "bits"),
]


@pytest.mark.parametrize("n", [2, 4])
def test_multiprocess_parity(n):
    if NGPU < n:
        pytest.skip(f"needs {n} GPUs, have {NGPU}")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, n, port, CASES, q)) for r in range(n)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(n)]
    for p in procs:
        p.join(timeout=60)
    for rank, results, err in sorted(res, key=lambda x: x[0]):
        assert err is None, f"rank {rank}: {err}"
        assert all(results), f"rank {rank}: failing cases {[c for c, ok in zip(CASES, results) if not ok]}"


def _timeout_worker(rank, n, port, q):
    import torch.distributed as dist
    from paper_2111_04867_b200 import taccl
    from paper_2111_04867_b200.generator import generate
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), TACCL_TIMEOUT_S="1")
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    try:
        comm = taccl.Comm(rank=rank, nranks=n, device=rank, scratch_bytes=16 << 20)
        comm.load(generate("allgather", "direct", n, 1, 1))
        x = torch.ones(1 << 16, dtype=torch.int32, device="cuda")
        out = torch.empty(n << 16, dtype=torch.int32, device="cuda")
        comm.register(out)
        comm.register(x)  # registration is collective and explicit
        code = None
        if rank == 0:  # rank 1 never joins the call: rank 0's waits must time out, not hang
            comm.run("allgather", out, x)
            torch.cuda.synchronize()
            try:
                comm.check()
            except taccl.TacclError as e:
                code = e.code
        dist.barrier()
        comm.destroy()
        q.put((rank, code, None))
    except Exception as e:
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


def test_watchdog_timeout_surfaces():
    # a peer that never issues the call: the device watchdog (%globaltimer, TACCL_TIMEOUT_S)
    # ends every spin and taccl_check reports TACCL_ERR_TIMEOUT (6)
    if NGPU < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_timeout_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    assert res[0][2] is None and res[1][2] is None, res
    assert res[0][1] == 6


# ---------------------------------------------------------------- full sizes, real peers, every element

FULL_CASES = [  # (coll, dtype, total bytes, input kind); bench.py's workload is the first
    ("allgather", "bfloat16", 1 << 30, "bits"),
    ("alltoall", "bfloat16", 1 << 30, "bits"),
    ("allreduce", "int32", 1 << 28, "bits"),
    ("allreduce", "bfloat16", 1 << 28, "uniform"),
    ("reducescatter", "int32", 1 << 30, "bits"),
    ("allreduce", "float32", 1 << 28, "uniform"),
    ("reducescatter", "bfloat16", 1 << 30, "uniform"),
]


def _full_worker(rank, n, port, q):
    import torch.distributed as dist

    from paper_2111_04867_b200 import taccl
    from paper_2111_04867_b200.generator import default_schedules
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    try:
        comm = taccl.Comm(rank=rank, nranks=n, device=rank, scratch_bytes=2 * (1 << 30) + (64 << 20))
        results = []
        for coll, dtype, total, kind in FULL_CASES:
            hs = [comm.load(t) for t in default_schedules(coll, n)]
            tdt = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}[dtype]
            es = 2 if dtype == "bfloat16" else 4
            count = total // es if coll == "allreduce" else total // es // n
            rows_in = n if coll in ("alltoall", "reducescatter") else 1
            rows_out = n if coll in ("allgather", "alltoall") else 1
            def make_input(src):  # rank src's seeded input (regenerated identically on any B200)
                g = torch.Generator(device="cuda").manual_seed(211104867 + 1000 * 3 + src)
                if kind == "uniform":  # U[1,2) (bf16: rounded)
                    return (torch.rand(rows_in * count, device="cuda", generator=g) + 1.0).to(tdt)
                if dtype == "int32":
                    return torch.randint(-2**31, 2**31 - 1, (rows_in * count,), dtype=torch.int32, device="cuda", generator=g)
                return torch.randint(-2**15, 2**15, (rows_in * count,), dtype=torch.int16, device="cuda", generator=g).view(tdt)

            x = make_input(rank)
            out = torch.empty(rows_out * count, dtype=tdt, device="cuda")
            out.view(torch.uint8).fill_(0xA5)
            comm.register(out)
            comm.register(x)
            comm.run(coll, out, x)  # the bench's call: registered user buffers, size-selected schedule
            torch.cuda.synchronize()
            comm.check()
            # EVERY element of this rank's output vs the oracle's definition on all ranks' inputs
            # (regenerated here from their seeds), column block by column block (tests/fullsize.py)
            from fullsize import check_blocked
            ins = [x if src == rank else make_input(src) for src in range(n)]
            ok, detail = check_blocked(coll, n, count, dtype, kind != "uniform", ins, {rank: out})
            if not ok:
                print(f"rank {rank} {coll} {dtype}: {detail}", flush=True)
            del ins
            comm.unregister(out)
            comm.unregister(x)
            results.append(ok)
            for h in hs:
                comm.free(h)
            del x, out
        comm.destroy()
        q.put((rank, results, None))
    except Exception as e:
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [2, 4])
def test_full_size_multiprocess(n):
    # BASELINE.json's 1 GiB sizes through the real multi-process path (CUDA IPC peers, the
    # default size-specialised sets, the launch configuration bench.py times), every output
    # element checked against the oracle's definition on all ranks' inputs
    if NGPU < n:
        pytest.skip(f"needs {n} GPUs, have {NGPU}")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_full_worker, args=(r, n, port, q)) for r in range(n)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(n)]
    for p in procs:
        p.join(timeout=60)
    for rank, results, err in sorted(res, key=lambda x: x[0]):
        assert err is None, f"rank {rank}: {err}"
        assert all(results), f"rank {rank}: failing cases {[c for c, ok in zip(FULL_CASES, results) if not ok]}"


# ---------------------------------------------------------------- multicast reduce (NVLink SHARP)

NVLS_CASES = [  # (dtype, count, kind, in_place); counts keep 16-byte chunks
    ("bfloat16", 8 * 4096, "uniform", False),
    ("bfloat16", 8 * (1 << 18), "normal", False),
    ("bfloat16", 8 * 4096, "intval", False),
    ("float32", 8 * 4096, "intval", False),
    ("float32", 8 * 4096, "uniform", False),
    ("int32", 8 * 1024, "bits", False),
    ("bfloat16", 8 * 4096, "uniform", True),
    ("bfloat16", 8 * (3 << 20), "uniform", False),  # 48 MiB of bf16: many pieces per CTA
]


def _nvls_worker(rank, n, port, q, lean=True):
    import torch.distributed as dist

    import oracle
    from paper_2111_04867_b200 import taccl
    from paper_2111_04867_b200.generator import generate
    from paper_2111_04867_b200.inputs import allreduce_input
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if not lean:  # the interpreter's K_MR step instead of the lean multicast-reduce kernel
        os.environ["TACCL_NO_LEAN_MR"] = "1"
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    tdt = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}
    view = {"int32": np.int32, "float32": np.int32, "bfloat16": np.int16}
    tview = {"int32": torch.int32, "float32": torch.int32, "bfloat16": torch.int16}
    try:
        comm = taccl.Comm(rank=rank, nranks=n, device=rank, scratch_bytes=64 << 20)
        comm.create_pool(1 << 30)
        nv = generate("allreduce", "nvls", n, 1, 1)
        comm.load(generate("allreduce", "direct", n, 1, 1))  # the fallback for non-pool calls
        comm.load(nv)
        results = []
        for dtype, count, kind, in_place in NVLS_CASES:
            ins = [allreduce_input(count, dtype, kind, 23, r) for r in range(n)]
            x = comm.pool_tensor(count, tdt[dtype])
            x.view(tview[dtype]).copy_(torch.from_numpy(ins[rank].view(view[dtype])).view(tview[dtype]))
            out = x if in_place else comm.pool_tensor(count, tdt[dtype])
            for _ in range(3):  # repeated calls: epochs of the multicast barriers
                if not in_place:
                    out.view(torch.uint8).fill_(0xA5)
                else:
                    x.view(tview[dtype]).copy_(torch.from_numpy(ins[rank].view(view[dtype])).view(tview[dtype]))
                comm.run("allreduce", out, x)
            torch.cuda.synchronize()
            comm.check()
            got = out.view(tview[dtype]).cpu().numpy().view(ins[0].dtype)
            want = oracle.run(oracle.parse(nv), ins, dtype)[rank]
            tol = 1e-2 if dtype == "bfloat16" else 1e-6
            if kind == "normal":  # the switch's accumulation and rounding are its own: norm-wise bound
                ref = oracle.expected_allreduce_f64(ins, dtype)
                scale = sum(np.abs(oracle.collectives.to_f64(v, dtype)) for v in ins)
                ok = bool((np.abs(oracle.collectives.to_f64(got, dtype) - ref) / scale).max() <= tol)
            elif kind == "uniform":  # north star: within 1e-2 / 1e-6 of the fp64 sum (the switch
                # rounds bf16 its own way, profiles/r02_nvls_rounding.txt: not bit-exact vs RNE)
                ref = oracle.expected_allreduce_f64(ins, dtype)
                ok = bool((np.abs(oracle.collectives.to_f64(got, dtype) - ref) / np.abs(ref)).max() <= tol)
            else:  # integers wrap exactly; integer-valued floats: every partial sum is exact
                ok = bool(np.array_equal(got, want))
            results.append(ok)
        # ordinary schedules on pool tensors: peers reached through the pool's unicast mappings
        for coll, algo in (("allgather", "ring"), ("alltoall", "direct"), ("reducescatter", "direct")):
            comm.load(generate(coll, algo, n, 1, 1))
            cnt = 3 << 18  # 0.75 Mi elements: the zero-copy kernel
            e_in = n * cnt if coll in ("alltoall", "reducescatter") else cnt
            e_out = cnt if coll == "reducescatter" else n * cnt
            ins = [allreduce_input(e_in, "int32", "bits", 26, r) for r in range(n)]
            xi = comm.pool_tensor(e_in, torch.int32)
            xi.copy_(torch.from_numpy(ins[rank]))
            xo = comm.pool_tensor(e_out, torch.int32)
            comm.register(xo)  # a no-op for pool tensors (every rank maps the pool already)
            comm.run(coll, xo, xi)
            torch.cuda.synchronize()
            comm.check()
            results.append(bool(np.array_equal(xo.cpu().numpy(), oracle.expected_outputs(coll, ins, "int32")[rank])))
        # not in the pool -> the multicast algorithm is skipped, the direct one runs
        xs = torch.from_numpy(allreduce_input(n * 1024, "int32", "bits", 24, rank)).cuda()
        os_ = torch.empty_like(xs)
        comm.register(os_)
        comm.run("allreduce", os_, xs)
        torch.cuda.synchronize()
        alls = [allreduce_input(n * 1024, "int32", "bits", 24, r) for r in range(n)]
        results.append(bool(np.array_equal(os_.cpu().numpy(), oracle.expected_outputs("allreduce", alls, "int32")[rank])))
        comm.destroy()
        q.put((rank, results, None))
    except Exception as e:
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("lean", [True, False])
@pytest.mark.parametrize("n", [2, 4])
def test_multicast_reduce_parity(n, lean):
    # the EF multicast-reduce step through the symmetric pool: multimem.ld_reduce/st over the
    # NVSwitch between processes (POSIX-fd handle exchange), vs the oracle
    if NGPU < n:
        pytest.skip(f"needs {n} GPUs, have {NGPU}")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nvls_worker, args=(r, n, port, q, lean)) for r in range(n)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(n)]
    for p in procs:
        p.join(timeout=60)
    for rank, results, err in sorted(res, key=lambda x: x[0]):
        assert err is None, f"rank {rank}: {err}"
        assert all(results), f"rank {rank}: {results}"


def _mismatch_worker(rank, n, port, q):
    import torch.distributed as dist
    from paper_2111_04867_b200 import taccl
    from paper_2111_04867_b200.generator import generate
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), TACCL_TIMEOUT_S="2")
    torch.cuda.set_device(rank)
    dist.init_process_group("gloo", rank=rank, world_size=n)
    try:
        comm = taccl.Comm(rank=rank, nranks=n, device=rank, scratch_bytes=64 << 20)
        comm.load(generate("reducescatter", "direct", n, 1, 1))
        count = 3 << 20  # above the LL threshold: the zero-copy kernel, where pull mode applies
        x = torch.ones(n * count, dtype=torch.bfloat16, device="cuda")
        out = torch.empty(count, dtype=torch.bfloat16, device="cuda")
        comm.register(out)
        comm.register(x)
        if rank == 0:  # registered input, out of place: pull mode
            comm.run("reducescatter", out, x)
        else:  # NCCL's in-place form: the input is copied privately, so this rank pushes
            comm.run("reducescatter", x[rank * count:(rank + 1) * count], x)
        torch.cuda.synchronize()
        code = None
        try:
            comm.check()
        except taccl.TacclError as e:
            code = e.code
        q.put((rank, code, None))
    except Exception as e:
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


def test_pull_mode_disagreement_is_detected():
    # one rank in pull mode, its peer not: the entry handshake carries the mode,
    # the senders abort before moving data, taccl_check reports it — no silent corruption, no hang
    if NGPU < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_mismatch_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(2)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
    assert res[0][2] is None and res[1][2] is None, res
    assert res[0][1] == 1 and res[1][1] == 1, res  # INVALID_ARG naming the disagreement, both ranks
