#!/usr/bin/env python
"""1 KB - 1 GB sweep of our executor vs NCCL (via torch.distributed) on the same box.

  torchrun --nproc-per-node N tools/sweep.py [--colls allgather,alltoall,allreduce]
           [--size-lo 10 --size-hi 30] [--out gpurun_out/sweep_nN.jsonl]

Per size: barrier, 5 warm-up calls, I = max(20, ~50 ms worth) calls between CUDA events on
the launching stream; t = elapsed / I; max over ranks (SURVEY.md §8(d) timing protocol).
S convention (reading G8): AG output bytes, A2A per-rank send bytes, AR buffer bytes.
busbw = S/t x (n-1)/n (AG, A2A) or 2(n-1)/n (AR); at n = 1 we report 2S/t (copy path).
Every our-side result is checked (bit-exact for AG/A2A, int-valued AR) once per size.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2111_04867_b200 import taccl  # noqa: E402
from paper_2111_04867_b200.generator import generate  # noqa: E402

ALGOS = {"allgather": ["direct", "ring", "auto"], "alltoall": ["direct"],
         "allreduce": ["direct", "ring", "oneshot", "nvls", "auto"],
         "reducescatter": ["direct", "ring", "auto"]}


def gen(coll, al, n):
    if al == "auto":  # the size-specialised default set (generator/tuned.py)
        from paper_2111_04867_b200.generator.tuned import default_schedules
        return default_schedules(coll, n)
    """algorithm name -> EF text. name[_pP][_mM][_split|_peer][_ovl]: chunks per rank P, instances M
    (PAPER.md:702-711, 785-789); _split = sends and receives in separate threadblocks;
    _peer = same-peer threadblock pairing only (no relay-first pairing); _ovl = the overlap="1"
    execution hint (warp-specialised send + receive-reduce pairs)"""
    parts = al.split("_")
    p = next((int(x[1:]) for x in parts[1:] if x[:1] == "p" and x[1:].isdigit()), 1)
    m = next((int(x[1:]) for x in parts[1:] if x[:1] == "m" and x[1:].isdigit()), 1)
    pair = False if "split" in parts[1:] else "peer" if "peer" in parts[1:] else True
    return generate(coll, parts[0], n, p, m, pair=pair, overlap="ovl" in parts[1:])


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_gbs(coll, text, n, S, es, cap):
    """The oracle (test infrastructure, oracle/) timed on this host, single thread, on the
    point's own schedule: S / t at S <= cap, else on a cap-byte sample of the same workload
    (count scaled down). Returns (GB/s, sample bytes, seconds)."""
    import time

    import numpy as np

    import oracle
    from paper_2111_04867_b200.inputs import allreduce_input, random_bits
    Ss = min(S, cap)
    dtn = "bfloat16" if es == 2 else "float32"
    count = Ss // es if coll == "allreduce" else Ss // es // n
    e_in = n * count if coll in ("alltoall", "reducescatter") else count
    texts = text if isinstance(text, list) else [text]
    prog = None
    for t in texts:  # the default set's member for this size
        p = oracle.parse(t)
        if p.min_bytes <= S < p.max_bytes:
            prog = p
    prog = prog or oracle.parse(texts[-1])
    if coll in ("allreduce", "reducescatter"):
        ins = [allreduce_input(e_in, dtn, "intval", 50, r) for r in range(n)]
    else:
        ins = [random_bits(e_in, dtn, 50, r) for r in range(n)]
    from oracle.validate import build_graph, topo_order
    graph = build_graph(prog)  # parse + happens-before graph outside the timed execution
    order = topo_order(graph)
    t0 = time.perf_counter()
    oracle.run(prog, ins, dtn, graph=graph, order=order)
    t = time.perf_counter() - t0
    return Ss / t / 1e9, Ss, t


def factor(coll, n):
    if n == 1:
        return 2.0
    return 2.0 * (n - 1) / n if coll == "allreduce" else (n - 1) / n


def timeit_graph(fn, stream, world, iters=200):
    """Capture `iters` calls into one CUDA graph and time its replay: per-call device time
    without host launch overhead (both our executor and NCCL are capturable)."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for _ in range(iters):
            fn()
    g.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    g.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    del g
    return ms, iters


def timeit(fn, stream, world, target_ms=50.0):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(5):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    est = max(e0.elapsed_time(e1) / 5, 1e-3)
    iters = int(max(20, min(2000, target_ms / est)))
    if world > 1:
        t = torch.tensor([iters], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        iters = int(t.item())
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(iters):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return ms, iters


HBM_PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6549.8
CPU = cpu_model()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--colls", default="allgather,alltoall,allreduce,reducescatter")
    ap.add_argument("--size-lo", type=int, default=10, help="smallest size 2^lo bytes")
    ap.add_argument("--size-hi", type=int, default=30, help="largest size 2^hi bytes")
    ap.add_argument("--sizes", default=None, help="comma list of sizes in MiB (overrides --size-lo/--size-hi)")
    ap.add_argument("--dtype", default="bfloat16")
    ap.add_argument("--out", default=None)
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays (no host overhead)")
    ap.add_argument("--algos", default=None, help="comma list overriding the per-collective defaults")
    ap.add_argument("--pool", action="store_true", help="buffers in the symmetric multicast pool (NVLS eligible)")
    ap.add_argument("--oracle-cap", type=int, default=0,
                    help="time the CPU oracle per point on rank 0 (sample <= this many bytes; 0 = off)")
    ap.add_argument("--peak-nvlink", type=float, default=705.0,
                    help="measured per-direction NVLink ceiling for roofline fractions (profiles/r01_p2p_probe.txt)")
    a = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = world
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    sizes = [int(float(x) * (1 << 20)) for x in a.sizes.split(",")] if a.sizes else [1 << k for k in range(a.size_lo, a.size_hi + 1)]
    S_max = max(sizes)
    comm = taccl.Comm(rank=rank, nranks=n, device=local, scratch_bytes=2 * S_max + (64 << 20))
    dt = torch.bfloat16 if a.dtype == "bfloat16" else torch.float32
    es = 2 if dt == torch.bfloat16 else 4
    # buffers sized for the largest message; registered once (zero-copy); --pool: both in the
    # symmetric multicast pool (multicast-reduce algorithms eligible; peers mapped by the pool)
    if a.pool and n > 1:
        comm.create_pool(2 * S_max + (8 << 20))
        big_in = comm.pool_tensor(S_max // es + 64, dt)
        big_out = comm.pool_tensor(S_max // es + 64, dt)
    else:
        big_in = torch.empty(S_max // es + 64, dtype=dt, device="cuda")
        big_out = torch.empty(S_max // es + 64, dtype=dt, device="cuda")
        comm.register(big_out)
        comm.register(big_in)  # pull mode (receive-reduce reads peers' inputs in place)
    stream = torch.cuda.Stream() if a.graph else torch.cuda.current_stream()
    torch.cuda.set_stream(stream)
    tf = (lambda f, st, w: timeit_graph(f, st, w)) if a.graph else timeit

    def load(t):  # one EF text or a list of them (a size-ranged set)
        if world > 1:  # every rank runs rank 0's text (a solver need not be bit-deterministic)
            obj = [t]
            dist.broadcast_object_list(obj, src=0)
            t = obj[0]
        return [comm.load(x) for x in t] if isinstance(t, list) else [comm.load(t)]

    def free(hs):
        for h in hs:
            comm.free(h)
    out_f = open(a.out or os.path.join(ROOT, "gpurun_out", f"sweep_n{n}.jsonl"), "a") if rank == 0 else None
    for coll in a.colls.split(","):
        algos = (a.algos.split(",") if a.algos else ALGOS[coll]) if n > 1 else ["direct"]
        handles = {al: load(gen(coll, al, n)) for al in algos}
        for S in sizes:
            if coll == "allgather":
                count = S // es // n
                inp, out = big_in[:count], big_out[:n * count]
            elif coll == "alltoall":
                count = S // es // n
                inp, out = big_in[:n * count], big_out[:n * count]
            elif coll == "reducescatter":  # S = send bytes (nccl-tests)
                count = S // es // n
                inp, out = big_in[:n * count], big_out[:count]
            else:
                count = S // es
                inp, out = big_in[:count], big_out[:count]
            if count == 0 or (coll in ("alltoall", "allreduce") and count % n):
                continue
            inp.copy_(torch.randint(-8, 8, inp.shape, device="cuda").to(dt))
            rec = {"coll": coll, "n": n, "S": S, "dtype": a.dtype, "graph": a.graph}
            for al in algos:
                if al == "oneshot" and S * (n - 1) > (64 << 20):
                    continue  # (n-1) x S of staging: a small-message schedule
                # select this algorithm: load order decides (latest wins) -> reload on top
                free(handles[al])
                handles[al] = load(gen(coll, al, n))
                ms, it = tf(lambda: comm.run(coll, out, inp, stream), stream, world)
                rec[f"taccl_{al}_us"] = round(ms * 1e3, 3)
                rec[f"taccl_{al}_busbw"] = round(S / (ms / 1e3) * factor(coll, n) / 1e9, 2)
                # check once (bits for AG/A2A, int-valued sum for AR)
                if coll == "allgather" and n > 1:
                    ok = torch.equal(out[rank * count:(rank + 1) * count].view(torch.int16 if es == 2 else torch.int32),
                                     inp.view(torch.int16 if es == 2 else torch.int32))
                    rec[f"taccl_{al}_ok"] = bool(ok)
            comm.check()
            if n > 1 and not a.no_nccl:
                if coll == "allgather":
                    f = lambda: dist.all_gather_into_tensor(out, inp)  # noqa: E731
                elif coll == "alltoall":
                    f = lambda: dist.all_to_all_single(out, inp)  # noqa: E731
                elif coll == "reducescatter":
                    f = lambda: dist.reduce_scatter_tensor(out, inp)  # noqa: E731
                else:
                    f = lambda: dist.all_reduce(out, op=dist.ReduceOp.SUM)  # noqa: E731
                ms, it = tf(f, stream, world)
                rec["nccl_us"] = round(ms * 1e3, 3)
                rec["nccl_busbw"] = round(S / (ms / 1e3) * factor(coll, n) / 1e9, 2)
            elif n == 1:
                ms, it = tf(lambda: out.copy_(inp), stream, world)
                rec["torch_copy_us"] = round(ms * 1e3, 3)
                rec["torch_copy_gbs"] = round(S / (ms / 1e3) * 2 / 1e9, 2)
            best = min((rec[f"taccl_{al}_us"], al) for al in algos if f"taccl_{al}_us" in rec)
            rec["taccl_best"] = best[1]
            rec["taccl_best_us"] = best[0]
            rec["taccl_best_busbw"] = rec[f"taccl_{best[1]}_busbw"]
            # the library's own choice: the size-specialised default set when it was run
            dflt = "auto" if "taccl_auto_us" in rec else best[1]
            rec["taccl_default"] = dflt
            bw = rec[f"taccl_{dflt}_busbw"]
            if n == 1:  # copy path: read+write bytes vs the measured HBM copy peak
                rec["roofline_frac"] = round(bw / HBM_PEAK, 4)
            else:  # busbw vs the measured NVLink ceiling per direction, and vs the nominal 900
                rec["roofline_frac"] = round(bw / a.peak_nvlink, 4)
                rec["frac_of_900"] = round(bw / 900.0, 4)
            if "nccl_us" in rec:
                rec["speedup_vs_nccl"] = round(rec["nccl_us"] / rec[f"taccl_{dflt}_us"], 3)
                rec["speedup_vs_nccl_best_variant"] = round(rec["nccl_us"] / best[0], 3)
            if a.oracle_cap:
                if rank == 0:
                    gbs, ss, sec = oracle_gbs(coll, gen(coll, dflt, n), n, S, es, a.oracle_cap)
                    rec["oracle_gbs"] = round(gbs, 4)
                    rec["oracle_sample_bytes"] = ss
                    rec["oracle_s"] = round(sec, 4)
                    rec["oracle_cores"] = f"1 of {len(os.sched_getaffinity(0))} ({CPU})"
                if world > 1:
                    dist.barrier()
            if rank == 0:
                print(json.dumps(rec), flush=True)
                out_f.write(json.dumps(rec) + "\n")
        for h in handles.values():
            free(h)
    comm.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
