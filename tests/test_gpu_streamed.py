"""GPU parity of streamed messages (KStep.prog, plan.cpp mark_streamed; DESIGN.md §6 "streamed
reduces"): a receive-reduce whose threadblock does nothing before it reduces each group of
stripes as soon as every input message published it. The result must equal the oracle's run of
the same schedule (PAPER.md:223-225 Allreduce, 722-727 ReduceScatter) for every group size,
stripe size, piece count and ragged tail — and, since the receiver skips the whole-message
flag, a sender that failed to publish would surface as a timeout in comm.check()."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_2111_04867_b200 import taccl  # noqa: E402
from paper_2111_04867_b200.generator import generate  # noqa: E402
from paper_2111_04867_b200.inputs import allreduce_input  # noqa: E402
from test_gpu_parity import assert_bits_equal, run_gpu  # noqa: E402


def _run(text, coll, n, dtype, ins, env, mode="direct"):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return run_gpu(text, coll, n, dtype, ins, mode=mode, pull=False)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


SCHEDS = [("reducescatter", "direct", 2, 1), ("reducescatter", "direct", 4, 1), ("reducescatter", "direct", 8, 2),
          ("allreduce", "direct", 2, 1), ("allreduce", "direct", 4, 1), ("allreduce", "direct", 8, 1),
          ("allreduce", "ring", 4, 1), ("reducescatter", "ring", 4, 2)]
KNOBS = [{"TACCL_PROG_STRIPES": "1", "TACCL_STRIPE": "4096"},
         {"TACCL_PROG_STRIPES": "2", "TACCL_STRIPE": "4096", "TACCL_LANES": "3"},
         {"TACCL_PROG_STRIPES": "3", "TACCL_STRIPE": "8192"},
         {"TACCL_PROG_STRIPES": "2"},
         {"TACCL_PROG_STRIPES": "0"}]  # off: the whole-message flags alone


@pytest.mark.parametrize("coll,algo,n,p", SCHEDS)
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("knob", range(len(KNOBS)))
def test_streamed_split_schedules_exact(coll, algo, n, p, dtype, knob):
    text = generate(coll, algo, n, p, 1, pair=False)
    if algo == "direct":  # the split direct schedules stream every reduce
        assert " prog" in taccl.plan_dump(text, 0)
    # chunks of 50-70 KiB: 13-18 stripes of 4 KiB, a ragged last stripe, several groups per piece
    c_e = 12289 if dtype == "bfloat16" else 6151
    count = p * c_e * (n if coll == "allreduce" else 1)
    kind = "bits" if dtype == "int32" else "intval"
    e_in = n * count if coll == "reducescatter" else count
    ins = [allreduce_input(e_in, dtype, kind, 31, r) for r in range(n)]
    got = _run(text, coll, n, dtype, ins, KNOBS[knob])
    if dtype == "int32":
        assert_bits_equal(got, oracle.expected_outputs(coll, ins, "int32"))
    assert_bits_equal(got, oracle.run(oracle.parse(text), ins, dtype))


@pytest.mark.parametrize("coll,n", [("reducescatter", 4), ("allreduce", 4), ("reducescatter", 8)])
@pytest.mark.parametrize("kind", ["uniform", "normal"])
@pytest.mark.parametrize("form", ["split", "overlap"])
def test_streamed_bf16_fused_rounding_bit_exact(coll, n, kind, form):
    # non-integer bf16: the fused chain's fp32 sum in chain order, rounded once (reading R3), is
    # the same whether the stripes are reduced as they land (split lowering, or beside the send
    # on half the warps: overlap="1") or after the whole message
    text = generate(coll, "direct", n, 1, 1, pair=form != "split", overlap=form == "overlap")
    count = 40000 if coll == "allreduce" else 10000
    e_in = n * count if coll == "reducescatter" else count
    ins = [allreduce_input(e_in, "bfloat16", kind, 33, r) for r in range(n)]
    got = _run(text, coll, n, "bfloat16", ins, {"TACCL_PROG_STRIPES": "1", "TACCL_STRIPE": "4096"})
    assert_bits_equal(got, oracle.run(oracle.parse(text), ins, "bfloat16"))


def test_streamed_repeated_calls_and_epochs():
    # progress words are keyed by (epoch, message): back-to-back calls on the same slots must
    # never take an earlier call's word for this one's
    n, count = 4, 4 * 24593
    text = generate("allreduce", "direct", n, 1, 1, pair=False)
    os.environ.update({"TACCL_PULL": "0", "TACCL_STAGED_MAX": "0", "TACCL_PROG_STRIPES": "1", "TACCL_STRIPE": "4096"})
    comm = taccl.Comm(nranks=n, device=0, emulated=True, scratch_bytes=64 << 20)
    try:
        comm.load(text)
        for it in range(6):
            ins = [allreduce_input(count, "int32", "bits", 40 + it, r) for r in range(n)]
            dev_in = [torch.from_numpy(x).cuda() for x in ins]
            dev_out = [torch.empty(count, dtype=torch.int32, device="cuda") for _ in range(n)]
            comm.run_emulated("allreduce", dev_out, dev_in)
            torch.cuda.synchronize()
            comm.check()
            want = oracle.expected_outputs("allreduce", ins, "int32")
            assert all(np.array_equal(o.cpu().numpy(), w) for o, w in zip(dev_out, want)), it
    finally:
        comm.destroy()
        for k in ("TACCL_PULL", "TACCL_STAGED_MAX", "TACCL_PROG_STRIPES", "TACCL_STRIPE"):
            os.environ.pop(k, None)


@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("dtype", ["int32", "bfloat16"])
@pytest.mark.parametrize("mode", ["direct", "staged"])
def test_split_allreduce_chain_sends(n, dtype, mode):
    # split lowering + chain sends (plan.cpp fuse_chain_sends: the Allgather phase's sends,
    # in other threadblocks, become K_PUB and the streamed chain members store the reduced
    # groups to the peers as they compute them); LL plans fuse them by default
    text = generate("allreduce", "direct", n, 1, 1, pair=False)
    count = n * 6151 if dtype == "int32" else n * 12289
    kind = "bits" if dtype == "int32" else "uniform"
    ins = [allreduce_input(count, dtype, kind, 35, r) for r in range(n)]
    env = {"TACCL_CHAIN_SENDS": "1", "TACCL_PROG_STRIPES": "1", "TACCL_STRIPE": "4096"}
    got = _run(text, "allreduce", n, dtype, ins, env, mode=mode)
    if dtype == "int32":
        assert_bits_equal(got, oracle.expected_outputs("allreduce", ins, "int32"))
    assert_bits_equal(got, oracle.run(oracle.parse(text), ins, dtype))


def test_streamed_piece_with_more_groups_than_the_word_holds():
    # 16 MiB chunks, 1 KiB stripes, 2 pieces: 8192 stripes per piece at one stripe per group —
    # more than the progress word's 4095 groups, so both ends widen the groups to 3 stripes
    n, count = 2, 4 << 20
    text = generate("reducescatter", "direct", n, 1, 1, pair=False)
    ins = [allreduce_input(n * count, "int32", "bits", 39, r) for r in range(n)]
    env = {"TACCL_PROG_STRIPES": "1", "TACCL_STRIPE": "1024", "TACCL_LANES": "2"}
    got = _run(text, "reducescatter", n, "int32", ins, env)
    assert_bits_equal(got, oracle.expected_outputs("reducescatter", ins, "int32"))


@pytest.mark.parametrize("coll,n,p", [("reducescatter", 2, 1), ("reducescatter", 4, 1), ("reducescatter", 4, 2),
                                      ("reducescatter", 8, 1), ("allreduce", 4, 1), ("allreduce", 8, 1)])
@pytest.mark.parametrize("dtype", ["int32", "bfloat16"])
@pytest.mark.parametrize("knob", [{}, {"TACCL_PROG_STRIPES": "1", "TACCL_STRIPE": "4096"},
                                  {"TACCL_LANES": "3", "TACCL_STRIPE": "8192"},
                                  {"TACCL_PAIR_SEND_WARPS": "12"}, {"TACCL_PAIR_SEND_WARPS": "3"}])
def test_warp_specialised_pairs(coll, n, p, dtype, knob):
    # overlap="1": the paired lowering's send + receive-reduce threadblocks run both steps at
    # once on the two halves of each CTA (streamed_pair, prog 2)
    text = generate(coll, "direct", n, p, 1, overlap=True)
    assert " prog2" in taccl.plan_dump(text, 0)
    env = dict(knob)
    c_e = 12289 if dtype == "bfloat16" else 6151
    count = p * c_e * (n if coll == "allreduce" else 1)
    kind = "bits" if dtype == "int32" else "intval"
    e_in = n * count if coll == "reducescatter" else count
    ins = [allreduce_input(e_in, dtype, kind, 41, r) for r in range(n)]
    got = _run(text, coll, n, dtype, ins, env)
    if dtype == "int32":
        assert_bits_equal(got, oracle.expected_outputs(coll, ins, "int32"))
    assert_bits_equal(got, oracle.run(oracle.parse(text), ins, dtype))
