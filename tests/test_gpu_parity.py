"""GPU parity: the sm_100a executor (through the C ABI) vs the oracle, element by element.

All ranks of a schedule are emulated on cuda:0 in ONE launch (taccl_run_emulated), so every
multi-rank path — sends into peer buffers, flags, dependencies, rrc staging and fused
chains — runs on a single B200. Bars (BASELINE.json north star): Allgather, Alltoall and
int32 Allreduce bit-exact; float Allreduce bit-exact on integer-valued inputs (every
summation order is exact there), and within 1e-6 (fp32) / 1e-2 (bf16) relative of the
fp64 sum on U[1,2) inputs.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2111_04867_b200 import taccl  # noqa: E402
from paper_2111_04867_b200.generator import generate  # noqa: E402
from paper_2111_04867_b200.inputs import allreduce_input, random_bits  # noqa: E402
from conftest import golden  # noqa: E402

TDT = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}
VIEW = {"int32": (torch.int32, np.int32), "float32": (torch.int32, np.int32), "bfloat16": (torch.int16, np.int16)}


def to_dev(x, dtype):
    tv, nv = VIEW[dtype]
    return torch.from_numpy(np.ascontiguousarray(x).view(nv)).view(TDT[dtype]).cuda()


def to_host(t, dtype, like):
    tv, nv = VIEW[dtype]
    return t.cpu().view(tv).numpy().view(like.dtype)


MODES = {"direct": "0", "staged": str(1 << 40)}  # TACCL_STAGED_MAX: zero-copy vs staged mode


def run_gpu(text, coll, n, dtype, ins, lanes=None, scratch=64 << 20, mode=None, pull=None):
    if pull is not None:  # pull mode: receive-reduces load peers' inputs in place; the tests
        os.environ["TACCL_PULL"] = str(int(pull))  # pull every kind (plain rrc, rrc+send, chains)
        os.environ["TACCL_PULL_KINDS"] = "7"
    if lanes:
        os.environ["TACCL_LANES"] = str(lanes)
    if mode:
        os.environ["TACCL_STAGED_MAX"] = MODES[mode]
    comm = taccl.Comm(nranks=n, device=0, emulated=True, scratch_bytes=scratch)
    try:
        comm.load(text)
        dev_in = [to_dev(x, dtype) for x in ins]
        e_out = {"allgather": ins[0].size * n, "reducescatter": ins[0].size // n}.get(coll, ins[0].size)
        dev_out = [torch.full((e_out,), 0, dtype=TDT[dtype], device="cuda") for _ in range(n)]
        for o in dev_out:  # poison, like the oracle's 0xA5 output
            o.view(torch.uint8).fill_(0xA5)
        comm.run_emulated(coll, dev_out, dev_in)
        torch.cuda.synchronize()
        comm.check()
        return [to_host(o, dtype, ins[0]) for o in dev_out]
    finally:
        comm.destroy()
        os.environ.pop("TACCL_LANES", None)
        os.environ.pop("TACCL_STAGED_MAX", None)
        os.environ.pop("TACCL_PULL", None)
        os.environ.pop("TACCL_PULL_KINDS", None)


def bits_inputs(coll, n, count, dtype, cfg):
    e_in = n * count if coll == "alltoall" else count
    return [random_bits(e_in, dtype, cfg, r) for r in range(n)]


def assert_bits_equal(got, want):
    for r, (g, w) in enumerate(zip(got, want)):
        if not np.array_equal(g, w):
            bad = np.nonzero(g != w)[0]
            raise AssertionError(f"rank {r}: {bad.size} mismatches, first at {bad[:8]}")


# ---------------------------------------------------------------- golden C1 (config C1)

def test_c1_worked_example():
    text = golden("c1_ag_ring_n2_p2.xml")
    ins = [((r << 16) + np.arange(512)).astype(np.int32) for r in range(2)]
    got = run_gpu(text, "allgather", 2, "int32", ins)
    j = np.arange(1024)
    for g in got:
        assert g.tolist() == (((j >> 9) << 16) + (j & 511)).tolist()


def test_gar_golden_allreduce():
    text = golden("ar_rsag_n2_p1.xml")
    ins = [allreduce_input(2 * 777, "int32", "bits", 5, r) for r in range(2)]
    got = run_gpu(text, "allreduce", 2, "int32", ins)
    assert_bits_equal(got, oracle.run(oracle.parse(text), ins, "int32"))


@pytest.mark.parametrize("count", [1, 1000, 4099, 1 << 16])
@pytest.mark.parametrize("lanes,mode", [(None, "staged"), (4, "staged"), (3, "staged"), (None, "direct"), (4, "direct")])
def test_copy_transfer_dependencies(count, lanes, mode):
    # copies that depend on transfers and transfers that depend on copies, with several pieces
    # per chunk (lanes): the LL kernel's copy must cover exactly the bytes its transfers'
    # piece j covers (executor.cu LL K_CPY)
    text = golden("ag_relay_cpy_n2.xml")
    ins = [random_bits(count, "int32", 19, r) for r in range(2)]
    got = run_gpu(text, "allgather", 2, "int32", ins, lanes=lanes, mode=mode)
    assert_bits_equal(got, oracle.expected_outputs("allgather", ins, "int32"))


# ---------------------------------------------------------------- AG / A2A bit-exact

AGA2A = [
    # coll, algo, n, p, m, dtype, count (elements per rank / per peer)
    ("allgather", "ring", 2, 1, 1, "bfloat16", 1),          # 2-byte chunks
    ("allgather", "ring", 4, 2, 1, "bfloat16", 2 * 1001),   # ragged chunk (not 16B multiple)
    ("allgather", "direct", 8, 1, 1, "bfloat16", 4096),
    ("allgather", "direct", 8, 2, 4, "int32", 8 * 3000),
    ("allgather", "ring", 8, 2, 8, "bfloat16", 2 * 8 * 4099),
    ("allgather", "hier", 8, 1, 1, "bfloat16", 5000),
    ("allgather", "hier", 4, 2, 2, "int32", 4 * 333),
    ("alltoall", "direct", 2, 1, 1, "bfloat16", 3),
    ("alltoall", "direct", 4, 4, 1, "bfloat16", 4 * 257),
    ("alltoall", "direct", 8, 1, 8, "int32", 8 * 1024),
    ("alltoall", "direct", 8, 4, 4, "bfloat16", 4 * 4 * 512),
    ("alltoall", "hier", 8, 1, 1, "bfloat16", 4096),
    ("alltoall", "hier", 8, 2, 4, "int32", 2 * 4 * 97),
]


@pytest.mark.parametrize("coll,algo,n,p,m,dtype,count", AGA2A)
@pytest.mark.parametrize("lanes,mode", [(None, "direct"), (4, "direct"), (None, "staged"), (2, "staged")])
def test_allgather_alltoall_bit_exact(coll, algo, n, p, m, dtype, count, lanes, mode):
    text = generate(coll, algo, n, p, m)
    ins = bits_inputs(coll, n, count, dtype, cfg=2 if coll == "allgather" else 3)
    got = run_gpu(text, coll, n, dtype, ins, lanes=lanes, mode=mode)
    assert_bits_equal(got, oracle.run(oracle.parse(text), ins, dtype))
    assert_bits_equal(got, oracle.expected_outputs(coll, ins, dtype))


@pytest.mark.parametrize("coll,algo,n,p,m,count", [
    ("allgather", "ring", 4, 1, 3, 4099), ("allgather", "direct", 8, 2, 8, 2 * 1001),
    ("alltoall", "direct", 4, 2, 4, 2 * 517), ("allreduce", "ring", 4, 1, 3, 4 * 1001),
    ("allreduce", "direct", 8, 1, 8, 8 * 1003), ("reducescatter", "ring", 4, 2, 2, 2 * 999)])
@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_instances_ragged_vs_expanded_oracle(coll, algo, n, p, m, count, mode):
    # instances with c_e not a multiple of m: the oracle runs the literally
    # expanded program (reading G3's floor split, oracle/instances.py); the executor runs its
    # own piece split. Same bits (int32, so reductions are exact in any order).
    text = generate(coll, algo, n, p, m)
    prog = oracle.parse(text)
    assert oracle.chunk_elems(coll, n, p, count) % m != 0
    e_in = n * count if coll in ("alltoall", "reducescatter") else count
    ins = [allreduce_input(e_in, "int32", "bits", 18, r) for r in range(n)]
    got = run_gpu(text, coll, n, "int32", ins, mode=mode)
    assert_bits_equal(got, oracle.run(oracle.expand_instances(prog), ins, "int32"))


GREEDY = [("allgather", 8, 2, {"policy": "uc-max"}), ("allgather", 8, 1, {"policy": "uc-min"}),
          ("alltoall", 8, 2, {"topology": "2x4"}), ("allreduce", 8, 1, {"policy": "uc-min"}),
          ("allreduce", 4, 2, {"policy": "uc-max"}), ("allgather", 8, 2, {"topology": "2x4"})]


@pytest.mark.parametrize("coll,n,p,kw", GREEDY)
@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_greedy_schedules_bit_exact(coll, n, p, kw, mode):
    text = generate(coll, "greedy", n, p, 1, **kw)
    count = n * p * 997 if coll != "allgather" else p * 997
    if coll == "allreduce":
        ins = [allreduce_input(count, "int32", "bits", 10, r) for r in range(n)]
        got = run_gpu(text, coll, n, "int32", ins, mode=mode)
        assert_bits_equal(got, oracle.expected_outputs(coll, ins, "int32"))
    else:
        ins = bits_inputs(coll, n, count, "bfloat16", 11)
        got = run_gpu(text, coll, n, "bfloat16", ins, mode=mode)
        assert_bits_equal(got, oracle.expected_outputs(coll, ins, "bfloat16"))


MILP = [("allgather", 8, 2, {}), ("alltoall", 8, 2, {}), ("allgather", 8, 2, {"topology": "2x4", "size": 1 << 16}),
        ("alltoall", 8, 1, {"topology": "2x4", "size": 1 << 16}), ("allreduce", 4, 2, {}),
        ("reducescatter", 8, 1, {"topology": "2x4", "size": 1 << 16})]


@pytest.mark.parametrize("coll,n,p,kw", MILP)
@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_milp_schedules_bit_exact(coll, n, p, kw, mode):
    """The three-stage MILP synthesizer's schedules (generator/milp.py; chunks the Stage-3
    MILP sends together become cnt > 1 steps) run bit-exactly."""
    text = generate(coll, "milp", n, p, 1, **kw)
    count = p * 997 if coll == "allgather" else n * p * 997
    if coll in ("allreduce", "reducescatter"):
        ins = [allreduce_input(count, "int32", "bits", 12, r) for r in range(n)]
        got = run_gpu(text, coll, n, "int32", ins, mode=mode)
        assert_bits_equal(got, oracle.expected_outputs(coll, ins, "int32"))
    else:
        ins = bits_inputs(coll, n, count, "bfloat16", 13)
        got = run_gpu(text, coll, n, "bfloat16", ins, mode=mode)
        assert_bits_equal(got, oracle.expected_outputs(coll, ins, "bfloat16"))


# ---------------------------------------------------------------- AR

AR = [
    ("ring", 2, 1, 1), ("ring", 4, 2, 2), ("ring", 8, 1, 4),
    ("direct", 2, 1, 1), ("direct", 4, 1, 2), ("direct", 8, 2, 1), ("direct", 8, 1, 8),
    ("oneshot", 2, 1, 1), ("oneshot", 4, 2, 1), ("oneshot", 8, 1, 2),
    ("dring", 4, 1, 1), ("dring", 8, 2, 2),
]


@pytest.mark.parametrize("algo,n,p,m", AR)
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("mode", ["direct", "staged", "push"])
def test_allreduce_exact(algo, n, p, m, dtype, mode):
    # direct = zero-copy kernel (pull mode on: rrcs fed by a peer's input load it in place);
    # push = the same kernel with pull off (sends push into the receiver's rrc staging)
    count = n * p * 1013 if dtype == "bfloat16" else n * p * 2051
    text = generate("allreduce", algo, n, p, m)
    kind = "bits" if dtype == "int32" else "intval"
    ins = [allreduce_input(count, dtype, kind, 4, r) for r in range(n)]
    got = run_gpu(text, "allreduce", n, dtype, ins, mode="direct" if mode == "push" else mode, pull=mode != "push")
    if dtype == "int32":
        assert_bits_equal(got, oracle.expected_outputs("allreduce", ins, "int32"))
    # integer-valued floats: every order is exact, so the oracle's schedule result is the answer
    assert_bits_equal(got, oracle.run(oracle.parse(text), ins, dtype))


@pytest.mark.parametrize("n,p,m", [(3, 1, 1), (4, 1, 2), (8, 2, 1)])
@pytest.mark.parametrize("dtype", ["int32", "bfloat16"])
@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_allreduce_chain_sends_fusion(n, p, m, dtype, mode):
    # TACCL_CHAIN_SENDS=1: the AG-phase sends of a direct AR are performed by the RS-phase
    # chain members as they reduce (plan.cpp fuse_chain_sends); same bits as the oracle
    os.environ["TACCL_CHAIN_SENDS"] = "1"
    try:
        count = n * p * 1013 if dtype == "bfloat16" else n * p * 2051
        text = generate("allreduce", "direct", n, p, m)
        kind = "bits" if dtype == "int32" else "intval"
        ins = [allreduce_input(count, dtype, kind, 16, r) for r in range(n)]
        got = run_gpu(text, "allreduce", n, dtype, ins, mode=mode)
        assert_bits_equal(got, oracle.run(oracle.parse(text), ins, dtype))
    finally:
        os.environ.pop("TACCL_CHAIN_SENDS", None)


BF16_TOL_SCHEDS = [  # every generator family's bf16 Allreduce, including multi-hop reduction chains
    ("allreduce", "ring", 8, 1, {}), ("allreduce", "direct", 8, 1, {}), ("allreduce", "oneshot", 8, 1, {}),
    ("allreduce", "greedy", 8, 1, {"policy": "uc-min"}), ("allreduce", "greedy", 8, 2, {"policy": "uc-max"}),
    ("allreduce", "milp", 8, 1, {}), ("allreduce", "ring", 4, 1, {}), ("allreduce", "direct", 4, 1, {}),
    ("reducescatter", "ring", 8, 1, {}), ("reducescatter", "greedy", 8, 2, {}),
    ("reducescatter", "milp", 8, 1, {"topology": "2x4", "size": 1 << 16})]


@pytest.mark.parametrize("algo,n,dtype,tol", [
    ("ring", 8, "float32", 1e-6), ("direct", 8, "float32", 1e-6), ("direct", 4, "float32", 1e-6),
    ("oneshot", 8, "float32", 1e-6)])
def test_allreduce_tolerance_uniform_fp32(algo, n, dtype, tol):
    count = n * 40000
    text = generate("allreduce", algo, n, 1, 1)
    ins = [allreduce_input(count, dtype, "uniform", 6, r) for r in range(n)]
    ref = oracle.expected_allreduce_f64(ins, dtype)
    got = run_gpu(text, "allreduce", n, dtype, ins)
    for g in got:
        rel = np.abs(oracle.collectives.to_f64(g, dtype) - ref) / np.abs(ref)
        assert rel.max() <= tol, rel.max()


@pytest.mark.parametrize("coll,algo,n,p,kw", BF16_TOL_SCHEDS)
@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_bf16_tolerance_uniform(coll, algo, n, p, kw, mode):
    # north star: bf16 Allreduce within 1e-2 relative of the fp64 sum, for EVERY schedule the
    # generator makes (ring / greedy / MILP chains hop rank to rank: fp32 partials, reading R6)
    text = generate(coll, algo, n, p, 1, **kw)
    count = n * p * 40000 if coll == "allreduce" else p * 40000
    e_in = n * count if coll == "reducescatter" else count
    ins = [allreduce_input(e_in, "bfloat16", "uniform", 6, r) for r in range(n)]
    got = run_gpu(text, coll, n, "bfloat16", ins, mode=mode)
    ref = oracle.expected_allreduce_f64(ins, "bfloat16")
    for r, g in enumerate(got):
        want = ref if coll == "allreduce" else ref[r * count:(r + 1) * count]
        rel = np.abs(oracle.collectives.to_f64(g, "bfloat16") - want) / np.abs(want)
        assert rel.max() <= 1e-2, (r, rel.max())


BF16_EXACT_SCHEDS = BF16_TOL_SCHEDS + [("allreduce", "ring", 4, 2, {"m": 2}), ("allreduce", "milp", 4, 2, {}),
                                       ("allreduce", "dring", 4, 1, {}),
                                       ("reducescatter", "direct", 8, 1, {}), ("reducescatter", "ring", 4, 2, {"m": 2})]


@pytest.mark.parametrize("coll,algo,n,p,kw", BF16_EXACT_SCHEDS)
@pytest.mark.parametrize("kind", ["uniform", "normal"])
@pytest.mark.parametrize("mode", ["direct", "staged", "push"])
def test_bf16_partials_bit_exact(coll, algo, n, p, kw, kind, mode):
    # the executor's bf16 reductions are deterministic: fp32 partials along every reduction
    # chain, one RNE where a value leaves it (reading R6). Bit-exact against the oracle's
    # partials mode on non-integer inputs (U[1,2) and N(0,1)), in the zero-copy kernel (pull
    # and push) and the LL kernel
    kw = dict(kw)
    m = kw.pop("m", 1)
    text = generate(coll, algo, n, p, m, **kw)
    count = n * p * 1003 if coll == "allreduce" else p * 1003
    e_in = n * count if coll == "reducescatter" else count
    ins = [allreduce_input(e_in, "bfloat16", kind, 8, r) for r in range(n)]
    got = run_gpu(text, coll, n, "bfloat16", ins, mode="direct" if mode == "push" else mode, pull=mode != "push")
    assert_bits_equal(got, oracle.run(oracle.parse(text), ins, "bfloat16", bf16="partials"))


@pytest.mark.parametrize("mode", ["direct", "staged"])
@pytest.mark.parametrize("kind", ["uniform", "normal"])
def test_bf16_partials_relay_golden(mode, kind):
    # rs_relay_n4: a partial sum relayed through a plain receive is rounded there (reading R6)
    text = golden("rs_relay_n4.xml")
    ins = [allreduce_input(4 * 2053, "bfloat16", kind, 9, r) for r in range(4)]
    got = run_gpu(text, "reducescatter", 4, "bfloat16", ins, mode=mode)
    assert_bits_equal(got, oracle.run(oracle.parse(text), ins, "bfloat16", bf16="partials"))


@pytest.mark.parametrize("dtype,tol", [("float32", 1e-6), ("bfloat16", 1e-2)])
def test_allreduce_tolerance_normal_normwise(dtype, tol):
    n, count = 8, 8 * 30000
    text = generate("allreduce", "direct", n, 1, 1)
    ins = [allreduce_input(count, dtype, "normal", 7, r) for r in range(n)]
    ref = oracle.expected_allreduce_f64(ins, dtype)
    scale = sum(np.abs(oracle.collectives.to_f64(x, dtype)) for x in ins)
    got = run_gpu(text, "allreduce", n, dtype, ins)
    for g in got:
        assert (np.abs(oracle.collectives.to_f64(g, dtype) - ref) / scale).max() <= tol


# ---------------------------------------------------------------- ReduceScatter

RS = [("ring", 2, 1, 1), ("ring", 4, 2, 2), ("ring", 8, 1, 4), ("direct", 2, 1, 1), ("direct", 4, 2, 1),
      ("direct", 8, 1, 8), ("direct", 1, 1, 1), ("greedy", 8, 2, 1)]


@pytest.mark.parametrize("algo,n,p,m", RS)
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("mode", ["direct", "staged", "push"])
def test_reducescatter_exact(algo, n, p, m, dtype, mode):
    # ReduceScatter as the inverse of an Allgather; count = elements per rank
    count = p * 1013 if dtype == "bfloat16" else p * 2051
    text = generate("reducescatter", algo, n, p, m)
    kind = "bits" if dtype == "int32" else "intval"
    ins = [allreduce_input(n * count, dtype, kind, 12, r) for r in range(n)]
    got = run_gpu(text, "reducescatter", n, dtype, ins, mode="direct" if mode == "push" else mode, pull=mode != "push")
    if dtype == "int32":
        assert_bits_equal(got, oracle.expected_outputs("reducescatter", ins, "int32"))
    assert_bits_equal(got, oracle.run(oracle.parse(text), ins, dtype))


@pytest.mark.parametrize("coll,n,p", [("reducescatter", 4, 1), ("reducescatter", 8, 2), ("allreduce", 4, 1)])
@pytest.mark.parametrize("dtype", ["int32", "bfloat16"])
def test_pulled_chain_plan(coll, n, p, dtype):
    # the large-chunk plan whose fused chains load every peer's input in place
    # (TACCL_PULL_CHAIN_MIN=0 selects it at any size): same bits as the oracle
    os.environ["TACCL_PULL_CHAIN_MIN"] = "0"
    try:
        count = p * 1013 * (n if coll == "allreduce" else 1)
        text = generate(coll, "direct", n, p, 1)
        e_in = n * count if coll == "reducescatter" else count
        kind = "bits" if dtype == "int32" else "uniform"
        ins = [allreduce_input(e_in, dtype, kind, 25, r) for r in range(n)]
        got = run_gpu(text, coll, n, dtype, ins, mode="direct")
        assert_bits_equal(got, oracle.run(oracle.parse(text), ins, dtype))
    finally:
        os.environ.pop("TACCL_PULL_CHAIN_MIN", None)


@pytest.mark.parametrize("algo,n,dtype,tol", [("direct", 8, "float32", 1e-6), ("ring", 4, "float32", 1e-6),
                                              ("direct", 8, "bfloat16", 1e-2), ("ring", 4, "bfloat16", 1e-2)])
def test_reducescatter_tolerance_uniform(algo, n, dtype, tol):
    count = 30000
    text = generate("reducescatter", algo, n, 1, 1)
    ins = [allreduce_input(n * count, dtype, "uniform", 13, r) for r in range(n)]
    ref = oracle.expected_reducescatter_f64(ins, dtype)
    got = run_gpu(text, "reducescatter", n, dtype, ins)
    for g, w in zip(got, ref):
        rel = np.abs(oracle.collectives.to_f64(g, dtype) - w) / np.abs(w)
        assert rel.max() <= tol, rel.max()


# ---------------------------------------------------------------- size-specialised sets

@pytest.mark.parametrize("coll,n,counts", [
    ("allreduce", 4, [4 * 1000, 4 * 65536, 4 * 262144]),        # oneshot below 512 KiB, direct above
    ("allreduce", 2, [2 * 1000, 2 * (8 << 20) + 2 * 1024]),       # oneshot below 16 MiB, direct above
    ("reducescatter", 4, [1000, 5 << 20]),                        # direct below 32 MiB, ring above
    ("allgather", 4, [1000, 17 << 20])])                          # direct below 128 MiB, ring above
def test_default_set_selects_by_size(coll, n, counts):
    from paper_2111_04867_b200.generator import default_schedules
    comm = taccl.Comm(nranks=n, device=0, emulated=True, scratch_bytes=1 << 30)
    try:
        for t in default_schedules(coll, n):
            comm.load(t)
        for count in counts:
            e_in = n * count if coll == "reducescatter" else count
            ins = [allreduce_input(e_in, "int32", "bits", 14, r) for r in range(n)]
            dev_in = [to_dev(x, "int32") for x in ins]
            e_out = {"allgather": n * count}.get(coll, count)
            dev_out = [torch.empty(e_out, dtype=torch.int32, device="cuda") for _ in range(n)]
            comm.run_emulated(coll, dev_out, dev_in)
            torch.cuda.synchronize()
            comm.check()
            got = [to_host(o, "int32", ins[0]) for o in dev_out]
            assert_bits_equal(got, oracle.expected_outputs(coll, ins, "int32"))
    finally:
        comm.destroy()


def test_dtypes_attribute_restricts_selection():
    # EF dtypes="...": an algorithm is selected only for the listed element types
    n, count = 2, 2 * 1024
    comm = taccl.Comm(nranks=n, device=0, emulated=True, scratch_bytes=16 << 20)
    try:
        comm.load(generate("allreduce", "direct", n, 1, 1, dtypes=("bfloat16",)))
        ins = [allreduce_input(count, "int32", "bits", 20, r) for r in range(n)]
        dev_in = [to_dev(x, "int32") for x in ins]
        dev_out = [torch.empty(count, dtype=torch.int32, device="cuda") for _ in range(n)]
        with pytest.raises(taccl.TacclError) as e:
            comm.run_emulated("allreduce", dev_out, dev_in)
        assert e.value.code == 3  # NO_ALGO
        comm.load(generate("allreduce", "ring", n, 1, 1, dtypes=("int32", "float32")))
        comm.run_emulated("allreduce", dev_out, dev_in)
        torch.cuda.synchronize()
        assert_bits_equal([to_host(o, "int32", ins[0]) for o in dev_out], oracle.expected_outputs("allreduce", ins, "int32"))
    finally:
        comm.destroy()


# ---------------------------------------------------------------- host-buffer runs (e2e path)

@pytest.mark.parametrize("coll,count,piece", [("allgather", 1 << 16, 1 << 12), ("allgather", 1000, 0),
                                              ("allreduce", 3 << 16, 1 << 14), ("reducescatter", 1 << 15, 1 << 12)])
def test_run_host_pipelined_single_rank(coll, count, piece):
    # taccl_run_host splits the count axis into pieces (2-D copies, double-buffered temps,
    # H2D / kernel / D2H overlapped); TACCL_HOST_PIECE_BYTES forces several pieces here
    from paper_2111_04867_b200.generator import generate
    os.environ["TACCL_HOST_PIECE_BYTES"] = str(piece or (1 << 30))
    comm = taccl.Comm(rank=0, nranks=1, device=0, scratch_bytes=64 << 20)
    try:
        comm.load(generate(coll, "direct", 1, 1, 1))
        x = allreduce_input(count, "int32", "bits", 15, 0)
        h_in = torch.from_numpy(x).pin_memory()
        h_out = torch.empty(count, dtype=torch.int32).pin_memory()
        for _ in range(2):
            h_out.fill_(0)
            comm.run_host(coll, h_out, h_in)
            assert np.array_equal(h_out.numpy(), oracle.expected_outputs(coll, [x], "int32")[0])
        comm.check()
    finally:
        comm.destroy()
        os.environ.pop("TACCL_HOST_PIECE_BYTES", None)


# ---------------------------------------------------------------- full sizes, every element

@pytest.mark.parametrize("coll,n,total_bytes,dtype,kind", [
    ("allgather", 1, 1 << 30, "bfloat16", "bits"), ("allgather", 4, 1 << 30, "bfloat16", "bits"),
    ("alltoall", 4, 1 << 30, "bfloat16", "bits"), ("allreduce", 4, 1 << 28, "int32", "bits"),
    ("reducescatter", 4, 1 << 30, "int32", "bits"), ("allreduce", 4, 1 << 28, "bfloat16", "uniform"),
    ("allreduce", 4, 1 << 28, "float32", "uniform"), ("reducescatter", 4, 1 << 30, "bfloat16", "uniform")])
def test_full_size_against_oracle(coll, n, total_bytes, dtype, kind):
    # BASELINE.json sizes (up to 1 GiB), the default schedule sets the bench uses; inputs
    # generated on the device (seeded); EVERY output element compared with the oracle's
    # definition, column block by column block (tests/fullsize.py): bit-exact for AG/A2A and
    # int32 AR/RS, within 1e-6 / 1e-2 of the fp64 sum for float AR/RS on U[1,2)
    from fullsize import check_blocked, rows
    from paper_2111_04867_b200.generator import default_schedules
    tdt = TDT[dtype]
    es = 2 if dtype == "bfloat16" else 4
    count = total_bytes // es if coll == "allreduce" else total_bytes // es // n
    rows_in, rows_out = rows(coll, n)
    comm = taccl.Comm(nranks=n, device=0, emulated=n > 1, scratch_bytes=3 * total_bytes + (64 << 20)) if n > 1 else \
        taccl.Comm(rank=0, nranks=1, device=0, scratch_bytes=64 << 20)
    try:
        for t in default_schedules(coll, n):
            comm.load(t)
        g = torch.Generator(device="cuda").manual_seed(211104867 + 1000 * 2)
        if kind == "uniform":  # U[1,2) (bf16: rounded)
            ins = [(torch.rand(rows_in * count, device="cuda", generator=g) + 1.0).to(tdt) for _ in range(n)]
        elif dtype == "int32":
            ins = [torch.randint(-2**31, 2**31 - 1, (rows_in * count,), dtype=tdt, device="cuda", generator=g) for _ in range(n)]
        else:  # random 16-bit patterns (NaN payloads included), compared as raw bits
            ins = [torch.randint(-2**15, 2**15, (rows_in * count,), dtype=torch.int16, device="cuda",
                                 generator=g).view(tdt) for _ in range(n)]
        outs = [torch.empty(rows_out * count, dtype=tdt, device="cuda") for _ in range(n)]
        for o in outs:
            o.view(torch.uint8).fill_(0xA5)
        if n > 1:
            comm.run_emulated(coll, outs, ins)
        else:
            comm.run(coll, outs[0], ins[0])
        torch.cuda.synchronize()
        comm.check()
        ok, detail = check_blocked(coll, n, count, dtype, kind == "bits", ins, dict(enumerate(outs)))
        assert ok, detail
    finally:
        comm.destroy()


# ---------------------------------------------------------------- device tracing

@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_trace_timeline_is_consistent(mode):
    # taccl_trace: per CTA entry <= prologue <= step start <= waits <= done <= exit, identity
    # words name (rank, tb, piece) of every CTA of the launch
    os.environ["TACCL_STAGED_MAX"] = MODES[mode]
    n, count = 4, 4 * 8192
    comm = taccl.Comm(nranks=n, device=0, emulated=True, scratch_bytes=64 << 20)
    try:
        text = generate("allreduce", "direct", n, 1, 1)
        comm.load(text)
        ins = [to_dev(allreduce_input(count, "int32", "bits", 17, r), "int32") for r in range(n)]
        outs = [torch.empty(count, dtype=torch.int32, device="cuda") for _ in range(n)]
        comm.run_emulated("allreduce", outs, ins)
        buf = torch.zeros(1024 * taccl.TRACE_SLOTS, dtype=torch.int64, device="cuda")
        comm.trace(buf)
        comm.run_emulated("allreduce", outs, ins)
        torch.cuda.synchronize()
        comm.trace(None)
        comm.check()
        grid = comm.plan_info("allreduce", count, taccl.INT32)["ctas"]  # all emulated ranks' CTAs
        T = buf[:grid * taccl.TRACE_SLOTS].view(grid, taccl.TRACE_SLOTS).cpu().tolist()
        prog = oracle.parse(text)
        seen = set()
        for row in T:
            ident = row[-2]
            r, tb = ident >> 32, (ident >> 16) & 0xFFFF
            seen.add((r, tb))
            assert 0 < row[0] <= row[1] <= row[-1], row[:2] + row[-2:]
            nsteps = len(prog.gpus[r].tbs[tb].steps)
            last = row[1]
            for k in range(nsteps):
                s0, s1, s3 = row[2 + 4 * k], row[3 + 4 * k], row[5 + 4 * k]
                assert last <= s0 <= s1 <= s3 <= row[-1], (r, tb, k, last, s0, s1, s3, row[-1])
                last = s3
        assert seen == {(r, t) for r in range(n) for t in range(len(prog.gpus[r].tbs))}
    finally:
        comm.destroy()
        os.environ.pop("TACCL_STAGED_MAX", None)


# ---------------------------------------------------------------- edge cases

@pytest.mark.parametrize("lean_max", [None, "0"])
def test_single_rank_copy_path(lean_max):
    # n = 1 schedules are one input -> output copy: the lean copy kernel below TACCL_LEAN_MAX
    # (default 256 MiB), the interpreter above; "0" forces the interpreter at every size
    text = generate("allgather", "direct", 1, 1, 1)
    if lean_max is not None:
        os.environ["TACCL_LEAN_MAX"] = lean_max
    try:
        for count in (1, 7, 4096, (1 << 20) + 3, (3 << 20) + 1):
            ins = bits_inputs("allgather", 1, count, "bfloat16", 8)
            got = run_gpu(text, "allgather", 1, "bfloat16", ins)
            assert_bits_equal(got, ins)
    finally:
        os.environ.pop("TACCL_LEAN_MAX", None)


def test_lean_copy_geometry():
    comm = taccl.Comm(rank=0, nranks=1, device=0, scratch_bytes=8 << 20)
    try:
        comm.load(generate("allgather", "direct", 1, 1, 1))
        assert comm.plan_info("allgather", 1 << 20, taccl.BFLOAT16)["threads"] == 256      # lean kernel
        assert comm.plan_info("allgather", 1 << 28, taccl.BFLOAT16)["threads"] == 512      # 512 MiB: interpreter
    finally:
        comm.destroy()


@pytest.mark.parametrize("coll", ["allgather", "allreduce"])
def test_in_place_single_rank(coll):
    # NCCL's in-place forms (reading G10): the input is copied to a private arena region first
    comm = taccl.Comm(rank=0, nranks=1, device=0, scratch_bytes=8 << 20)
    try:
        comm.load(generate(coll, "direct", 1, 1, 1))
        x = to_dev(allreduce_input(12345, "int32", "bits", 18, 0), "int32")
        buf = x.clone()
        comm.run(coll, buf, buf)
        torch.cuda.synchronize()
        comm.check()
        assert torch.equal(buf, x)
    finally:
        comm.destroy()


def test_count_not_divisible_is_rejected():
    comm = taccl.Comm(nranks=2, device=0, emulated=True, scratch_bytes=1 << 20)
    try:
        comm.load(generate("allreduce", "direct", 2, 1, 1))
        x = [torch.zeros(3, dtype=torch.float32, device="cuda") for _ in range(2)]
        with pytest.raises(taccl.TacclError) as e:
            comm.run_emulated("allreduce", x, x)
        assert e.value.code == 1
    finally:
        comm.destroy()


def test_invalid_schedule_rejected_at_load():
    comm = taccl.Comm(nranks=2, device=0, emulated=True, scratch_bytes=1 << 20)
    try:
        bad = golden("c1_ag_ring_n2_p2.xml").replace('dstoff="2" cnt="2" deps=""/>\n  </tb>\n  <tb id="1"', 'dstoff="0" cnt="2" deps=""/>\n  </tb>\n  <tb id="1"', 1)
        with pytest.raises(taccl.TacclError) as e:
            comm.load(bad)
        assert e.value.code == 2
    finally:
        comm.destroy()


@pytest.mark.parametrize("sizes", [[4096, 1 << 20, 4096, 8, 1 << 22, 4096], [64, 64, 1 << 21, 64]])
def test_mode_and_size_changes_between_calls(sizes):
    # consecutive calls alternate between staged and zero-copy mode and between sizes (the
    # staged parity regions have a fixed place; flags are epoch-monotone)
    n = 4
    text = generate("allreduce", "direct", n, 1, 1)
    comm = taccl.Comm(nranks=n, device=0, emulated=True, scratch_bytes=64 << 20)
    try:
        comm.load(text)
        for it, count in enumerate(sizes * 3):
            count = n * max(1, count // n)
            ins = [allreduce_input(count, "int32", "bits", 30 + it, r) for r in range(n)]
            dev_in = [to_dev(x, "int32") for x in ins]
            dev_out = [torch.empty(count, dtype=torch.int32, device="cuda") for _ in range(n)]
            comm.run_emulated("allreduce", dev_out, dev_in)
            torch.cuda.synchronize()
            assert_bits_equal([to_host(o, "int32", ins[0]) for o in dev_out], oracle.expected_outputs("allreduce", ins, "int32"))
        comm.check()
    finally:
        comm.destroy()


def test_cuda_graph_capture_replays_correctly():
    # taccl_run is capturable: epochs live on the device, so graph replays advance them
    n, count = 4, 4 * 8192
    comm = taccl.Comm(nranks=n, device=0, emulated=True, scratch_bytes=16 << 20)
    try:
        comm.load(generate("allgather", "direct", n, 1, 1))
        ins = bits_inputs("allgather", n, count, "bfloat16", 12)
        dev_in = [to_dev(x, "bfloat16") for x in ins]
        dev_out = [torch.empty(n * count, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            comm.run_emulated("allgather", dev_out, dev_in, stream=s)  # warm
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            comm.run_emulated("allgather", dev_out, dev_in, stream=s)
        for it in range(5):
            for o in dev_out:
                o.zero_()
            g.replay()
            torch.cuda.synchronize()
            assert_bits_equal([to_host(o, "bfloat16", ins[0]) for o in dev_out],
                              oracle.expected_outputs("allgather", ins, "bfloat16"))
        comm.check()
    finally:
        comm.destroy()


def test_repeated_calls_reuse_flags_and_epochs():
    # 50 back-to-back calls on one stream: epochs advance on the device, results stay exact
    n, count = 4, 4 * 4096
    text = generate("allreduce", "ring", n, 1, 2)
    comm = taccl.Comm(nranks=n, device=0, emulated=True, scratch_bytes=16 << 20)
    try:
        comm.load(text)
        ins = [allreduce_input(count, "int32", "bits", 9, r) for r in range(n)]
        dev_in = [to_dev(x, "int32") for x in ins]
        dev_out = [torch.empty(count, dtype=torch.int32, device="cuda") for _ in range(n)]
        want = oracle.expected_outputs("allreduce", ins, "int32")
        for it in range(50):
            comm.run_emulated("allreduce", dev_out, dev_in)
        torch.cuda.synchronize()
        comm.check()
        assert_bits_equal([to_host(o, "int32", ins[0]) for o in dev_out], want)
    finally:
        comm.destroy()
