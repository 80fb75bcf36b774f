#!/usr/bin/env python
"""Benchmark of the TACCL-schedule executor (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl taccl|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...     (N > 1, one rank per GPU)

A step is one collective call = one launch of the whole hot path (SURVEY.md §8(a) a0–a8).
  N = 1: Allgather with one rank = the local copy path, 1 GiB bf16 output (north star
         "1 GPU (local copy path vs HBM roofline)"); value = read+write bytes / time.
  N > 1: Allgather, the size-specialised default schedule set, 1 GiB bf16 output, one process
         per GPU, peers' HBM mapped with CUDA IPC; value = the metric, bus bandwidth per GPU
         (nccl-tests busbw = S/t x (N-1)/N, t = max over ranks); its fraction of 900 GB/s
         NVLink and the whole-job aggregate (N x busbw) are reported beside it.
Inputs are resident in HBM before the timed region and larger than L2 (126 MB), so no
flush is needed. Timing: W warm-up calls, barrier + synchronize, K calls between CUDA
events on the launching stream, synchronize, max over ranks.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import nvlink_counters  # noqa: E402  (NVML only; no GPU work)

GIB = 1 << 30
MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
NVLINK_NOMINAL = 900.0     # GB/s per direction per GPU (NVLink 5)
NVLINK_MEASURED_REF = 770.0  # peer copy per direction, /opt/skills/guides/B200_PROFILING.md
HBM_FALLBACK = 6650.0      # B200_PROFILING.md fallback when MEASURED_PEAKS.json is absent


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="taccl", choices=["taccl", "reference"])
    ap.add_argument("--size", type=int, default=GIB, help="S: Allgather output bytes")
    ap.add_argument("--algo", default="auto", help="auto = the size-specialised default set (generator/tuned.py)")
    ap.add_argument("--chunks", type=int, default=1)
    ap.add_argument("--instances", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


def hbm_peak():
    try:
        with open(MEASURED) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return HBM_FALLBACK, "fallback (B200_PROFILING.md)"


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_gpu{index}.csv")

    def __enter__(self):
        os.makedirs(os.path.dirname(self.path), exist_ok=True)
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            self.p.wait()
            self.f.close()

    def summary(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 8 and parts[1].replace(".", "").isdigit():
                    rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows)}


def busbw_factor(coll, n):
    return 2.0 * (n - 1) / n if coll == "allreduce" else (n - 1) / n


def resolve_algo(algo, n, S):
    """the schedule the run uses: `auto` = the default set's member for this size"""
    if n == 1:
        return "direct"
    if algo != "auto":
        return algo
    from paper_2111_04867_b200.generator.tuned import ranges
    return next(r[0] for r in ranges("allgather", n) if r[1] <= S < r[2] and (len(r) == 3 or "bfloat16" in r[3]))


def cpu_oracle_baseline(size_bytes, n, algo, seconds=10.0):
    """The oracle (test infrastructure) as it stands, on a bounded sample of the workload."""
    import numpy as np

    import oracle
    from paper_2111_04867_b200.generator import generate
    from paper_2111_04867_b200.inputs import random_bits
    sample = min(size_bytes, 256 << 20)
    count = sample // 2 // n
    prog = oracle.parse(generate("allgather", algo, n, 1, 1))
    ins = [random_bits(count, "bfloat16", 2, r) for r in range(n)]
    times = []
    t_end = time.perf_counter() + seconds
    while time.perf_counter() < t_end or len(times) < 2:
        t0 = time.perf_counter()
        outs = oracle.run(prog, ins, "bfloat16")
        times.append(time.perf_counter() - t0)
    assert np.array_equal(outs[0][:count], ins[0])
    t = statistics.median(times)
    per_rank_bytes = (2 * sample) if n == 1 else sample * busbw_factor("allgather", n)
    value = per_rank_bytes * n / t / 1e9
    return {"value": round(value, 3), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"Allgather n={n} {algo} schedule, {sample >> 20} MiB output bf16 (of {size_bytes >> 20} MiB), "
                      f"median of {len(times)} runs of oracle.run (NumPy, single thread)",
            "host_cores_available": len(os.sched_getaffinity(0))}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def c1_oracle_timing(reps=21):
    """BASELINE.json configs[0] (C1): the Allgather ring schedule, 2 ranks, 2 chunks per rank,
    4 KB int32 output (tests/golden/c1_ag_ring_n2_p2.xml), through the CPU oracle: parse +
    validate and execute timed separately, median of `reps` runs each."""
    import numpy as np

    import oracle
    from oracle.validate import build_graph, topo_order
    text = open(os.path.join(ROOT, "tests", "golden", "c1_ag_ring_n2_p2.xml")).read()
    ins = [((r << 16) + np.arange(512)).astype(np.int32) for r in range(2)]
    tv, tx = [], []
    for _ in range(reps):
        t0 = time.perf_counter()
        prog = oracle.parse(text)
        ok = oracle.validate(prog).ok
        t1 = time.perf_counter()
        graph = build_graph(prog)
        order = topo_order(graph)
        outs = oracle.run(prog, ins, "int32", graph=graph, order=order)
        t2 = time.perf_counter()
        tv.append(t1 - t0)
        tx.append(t2 - t1)
    j = np.arange(1024)
    exact = ok and all(np.array_equal(o, ((j >> 9) << 16) + (j & 511)) for o in outs)  # the worked example
    return {"config": "C1: Allgather ring, 2 ranks, 2 chunks/rank, 4 KB int32 output (CPU oracle)",
            "parse_validate_ms": round(statistics.median(tv) * 1e3, 4),
            "execute_ms": round(statistics.median(tx) * 1e3, 4),
            "runs": reps, "statistic": "median", "bit_exact_vs_worked_example": bool(exact),
            "cores": f"1 of {len(os.sched_getaffinity(0))}", "cpu_model": cpu_model(),
            "execute_gbs": round(4096 / statistics.median(tx) / 1e9, 6)}


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n = world if world > 1 else a.gpus
    if n != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE {world}")
    coll = "allgather"
    S = a.size
    workload = (f"allgather n=1 local copy path, {S >> 20} MiB bf16" if n == 1 else
                f"allgather n={n}, {S >> 20} MiB output bf16, schedule {a.algo}")
    metric = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]

    if a.impl == "reference":
        # reference arm = the oracle (no runnable reference exists: /root/reference is a paper)
        if rank != 0:
            return
        steps = a.steps or 3
        cpu = cpu_oracle_baseline(S, n, resolve_algo(a.algo, n, S), seconds=max(2.0, 2.0 * (steps + a.warmup)))
        line = {"impl": "reference", "metric": metric, "value": cpu["value"], "unit": "GB/s", "n_gpus": n,
                "steps": steps, "warmup": a.warmup, "ms_per_step": None, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": workload + " (oracle, bounded sample)", "l2": "inputs > L2"},
                "cpu_baseline": cpu, "e2e": {"value": cpu["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                                             "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch
    import torch.distributed as dist

    from paper_2111_04867_b200 import taccl
    from paper_2111_04867_b200.generator import generate

    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    count = S // 2 // n  # bf16 elements per rank
    scratch = (2 * S + (64 << 20)) if not a.no_e2e else (64 << 20)
    comm = taccl.Comm(rank=rank, nranks=n, device=local_rank, scratch_bytes=scratch)
    algo_used = resolve_algo(a.algo, n, S)
    if a.algo == "auto":
        comm.load_defaults(("allgather",))
    else:
        comm.load(generate(coll, algo_used, n, a.chunks, a.instances))
    g = torch.Generator(device="cuda").manual_seed(211104867 + rank)
    inp = torch.randint(-32768, 32767, (count,), dtype=torch.int16, device="cuda", generator=g).view(torch.bfloat16)
    out = torch.empty(n * count, dtype=torch.bfloat16, device="cuda")
    comm.register(out)
    comm.register(inp)
    stream = torch.cuda.current_stream()
    steps = a.steps or (6000 if n == 1 else 2500)  # timed region >= ~2 s for the clock samples

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(max(3, a.warmup)):
        comm.all_gather(out, inp)
    barrier()
    comm.check()
    # correctness of what we time, every element: out chunk s must be rank s's input (the
    # Allgather definition), regenerated here from rank s's seed
    ob = out.view(torch.int16)  # compare raw bits (random patterns include NaNs)
    for src in range(n):
        ref = torch.randint(-32768, 32767, (count,), dtype=torch.int16, device="cuda",
                            generator=torch.Generator(device="cuda").manual_seed(211104867 + src))
        assert torch.equal(ob[src * count:(src + 1) * count], ref), f"rank {rank}: chunk {src} differs"
        del ref

    launches0 = taccl.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    phys = local_rank  # NVML index of this rank's GPU
    vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
    if vis and all(x.strip().isdigit() for x in vis.split(",")):
        phys = int(vis.split(",")[local_rank])
    nvl0 = nvlink_counters.read(phys) if n > 1 else None
    with Clocks(local_rank) as clk:
        barrier()
        e0.record(stream)
        for _ in range(steps):
            comm.all_gather(out, inp)
        e1.record(stream)
        torch.cuda.synchronize()
    nvl1 = nvlink_counters.read(phys) if n > 1 else None
    launches = taccl.launch_count() - launches0
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    comm.check()
    t_step = ms / 1e3 / steps
    if n == 1:
        per_rank_bytes = 2.0 * S
        value = per_rank_bytes / t_step / 1e9
        peak, src = hbm_peak()
        roof = {"bound": "hbm", "achieved": round(value, 1), "peak": peak, "unit": "GB/s",
                "frac": round(value / peak, 4), "peak_source": src}
        busbw = None
    else:
        busbw = S / t_step * busbw_factor(coll, n) / 1e9
        value = busbw  # the metric: bus GB/s per GPU (nccl-tests busbw; the aggregate is beside it)
        egress = S * (n - 1) / n  # algorithmic NVLink bytes per launch per GPU
        ach = egress / t_step / 1e9
        roof = {"bound": "nvlink", "achieved": round(ach, 1), "peak": NVLINK_MEASURED_REF, "unit": "GB/s",
                "frac": round(ach / NVLINK_MEASURED_REF, 4), "frac_of_nominal_900": round(ach / NVLINK_NOMINAL, 4),
                "peak_source": "measured peer copy per direction per GPU (B200_PROFILING.md fallback; "
                               "MEASURED_PEAKS.json has no NVLink figure); nominal 900 for context"}
    roof["traffic"] = None
    tr_path = os.path.join(ROOT, "profiles", "traffic.json")
    if n == 1 and os.path.exists(tr_path):  # ncu DRAM bytes per launch (tools/ncu_round.sh)
        roof["traffic"] = json.load(open(tr_path)).get(f"n{n}_{S}")
    if n > 1 and nvl0 and nvl1:
        # NVLink payload bytes this GPU transmitted per launch (NVML counters around the timed
        # region; the ncu recipe cannot capture a multi-rank kernel), max over ranks
        tx = torch.tensor([(nvl1["tx"] - nvl0["tx"]) / steps, (nvl1["rx"] - nvl0["rx"]) / steps],
                          dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tx, op=dist.ReduceOp.MAX)
        roof["traffic"] = round(float(tx[0]))
        roof["traffic_rx"] = round(float(tx[1]))
        roof["traffic_source"] = f"NVML NVLink {nvl0['field']} tx/rx bytes per launch, max over ranks (algorithmic {int(S * (n - 1) / n)})"
    # n = 1: the schedule is one input -> output copy (the lean copy kernel below 256 MiB)
    roof["kernel"] = "taccl_copy_kernel" if n == 1 and S < (256 << 20) else "taccl_exec_kernel"

    # e2e: same metric through the C ABI with HOST buffers (pinned), copies inside the timed region
    e2e = None
    if not a.no_e2e:
        h_in = inp.cpu().pin_memory()
        h_out = torch.empty(n * count, dtype=torch.bfloat16).pin_memory()
        comm.run_host("allgather", h_out, h_in)  # warm
        barrier()
        t0 = time.perf_counter()
        for _ in range(a.e2e_steps):
            comm.run_host("allgather", h_out, h_in)
        barrier()
        te = (time.perf_counter() - t0) / a.e2e_steps
        if world > 1:
            t = torch.tensor([te], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            te = float(t.item())
        assert torch.equal(h_out.view(torch.int16)[rank * count:(rank + 1) * count], h_in.view(torch.int16))
        ev = (2.0 * S if n == 1 else S * busbw_factor(coll, n)) / te / 1e9
        e2e = {"value": round(ev, 2), "unit": "GB/s", "h2d_bytes_per_step": count * 2,
               "d2h_bytes_per_step": n * count * 2, "ms_per_step": round(te * 1e3, 3),
               "timing": "host wall clock around taccl_run_host (H2D + kernel + D2H + stream sync), max over ranks"}

    if rank == 0:
        line = {"metric": metric, "value": round(value, 2), "unit": "GB/s", "n_gpus": n, "steps": steps,
                "warmup": a.warmup, "ms_per_step": round(t_step * 1e3, 4), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": {"workload": workload, "size_bytes": S, "algo": algo_used if n > 1 else "copy",
                           "algo_choice": a.algo,
                           "chunks_per_rank": a.chunks, "instances": a.instances,
                           "plan": comm.plan_info("allgather", count, taccl.BFLOAT16),
                           "l2": "inputs and outputs > 126 MB L2 (no flush needed)",
                           "value_definition": ("read+write bytes / t (local copy path)" if n == 1 else
                                                "busbw per GPU = S/t * (N-1)/N (nccl-tests; max-over-ranks t)")},
                "roofline": roof, "gpu_launches": launches, "clocks": clk.summary(), "e2e": e2e}
        if busbw is not None:
            line["busbw_per_gpu"] = round(busbw, 2)
            line["busbw_frac_of_900"] = round(busbw / NVLINK_NOMINAL, 4)
            line["aggregate_busbw"] = round(n * busbw, 2)  # whole job: N x busbw
        if n == 1 and not a.no_cpu:
            line["cpu_baseline"] = cpu_oracle_baseline(S, n, algo_used)
            line["cpu_baseline"]["cpu_model"] = cpu_model()
            line["c1_oracle"] = c1_oracle_timing()
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
    comm.destroy()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
