"""GPU parity of merged execution (TACCL_MERGED=1; plan.cpp merged_order, DESIGN.md §6
"merged threadblocks"): every CTA of a rank runs all of its threadblocks' steps in the plan's
level order. Results must equal the oracle's run of the same schedule bit for bit (int32 and
integer-valued floats: PAPER.md:218-225 definitions), and a wrong order would deadlock and
surface as a watchdog timeout in comm.check()."""
import os

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_2111_04867_b200.generator import generate  # noqa: E402
from paper_2111_04867_b200.inputs import allreduce_input, random_bits  # noqa: E402
from test_gpu_parity import assert_bits_equal, run_gpu  # noqa: E402

SCHEDS = [("allgather", "direct", 4, 1, {}), ("allgather", "ring", 4, 2, {}), ("allgather", "ring", 8, 1, {}),
          ("alltoall", "direct", 4, 1, {}), ("alltoall", "direct", 8, 2, {}), ("alltoall", "hier", 4, 1, {}),
          ("allgather", "greedy", 8, 1, {}), ("alltoall", "greedy", 4, 2, {}),
          ("allreduce", "direct", 4, 1, {}), ("allreduce", "direct", 8, 1, {}), ("allreduce", "ring", 4, 1, {}),
          ("allreduce", "dring", 4, 1, {}), ("allreduce", "oneshot", 4, 1, {}), ("allreduce", "direct", 4, 1, {"pair": False}),
          ("reducescatter", "direct", 4, 1, {}), ("reducescatter", "direct", 4, 1, {"pair": False}),
          ("reducescatter", "ring", 4, 2, {}), ("reducescatter", "direct", 2, 1, {}),
          ("alltoall", "rounds", 4, 1, {}), ("allgather", "rounds", 8, 1, {}), ("alltoall", "rounds", 3, 2, {})]


def _inputs(coll, n, p, dtype, seed):
    c_e = 6151
    if coll in ("allgather",):
        return [random_bits(p * c_e, dtype, seed, r) for r in range(n)]
    if coll == "alltoall":
        return [random_bits(n * p * c_e, dtype, seed, r) for r in range(n)]
    kind = "bits" if dtype == "int32" else "intval"
    e = n * p * c_e
    return [allreduce_input(e, dtype, kind, seed, r) for r in range(n)]


@pytest.mark.parametrize("coll,algo,n,p,kw", SCHEDS)
@pytest.mark.parametrize("dtype", ["int32", "bfloat16"])
@pytest.mark.parametrize("pull", [False, True])
@pytest.mark.parametrize("lanes", [None, 3])
def test_merged_execution_exact(coll, algo, n, p, kw, dtype, pull, lanes):
    text = generate(coll, algo, n, p, 1, **kw)
    ins = _inputs(coll, n, p, dtype, 51)
    os.environ["TACCL_MERGED"] = "1"
    try:
        got = run_gpu(text, coll, n, dtype, ins, lanes=lanes, mode="direct", pull=pull)
    finally:
        os.environ.pop("TACCL_MERGED", None)
    if dtype == "int32":
        assert_bits_equal(got, oracle.expected_outputs(coll, ins, "int32"))
    assert_bits_equal(got, oracle.run(oracle.parse(text), ins, dtype))
