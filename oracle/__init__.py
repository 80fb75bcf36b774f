"""CPU oracle for TACCL-EF chunk schedules (arXiv 2111.04867).

TEST INFRASTRUCTURE, NOT PRODUCT CODE. Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import anything under `oracle/`.
The product path (`paper_2111_04867_b200`) never imports it, and the oracle imports nothing
from the product: the two share no parser, validator, geometry or arithmetic.

It is a plain, slow, obviously-correct restatement of what the paper says a schedule
computes:

* `collectives` — the collectives' definitions (§2; ReduceScatter 722–727) and their chunk
  pre/postconditions (App. B).
* `ef` — an independent parser for the EF v1 text (docs/SCHEDULE.md).
* `validate` — structure, send/recv matching, the happens-before DAG, races.
* `simulate` — executes the program step by step on host buffers, symbolically (chunk
  tokens / reduction multisets) or numerically (NumPy), in any topological order.
* `instances` — literal instance expansion.

Pins (tests/test_oracle_*.py, `-m "not gpu"`): closed-form definitions, the C1 worked
example, brute force over all linearisations on tiny programs, symbolic/numeric agreement,
the instance invariant, involution of Alltoall, library bf16 rounding, mutation verdicts.
Parity unpinned: nothing in this package — see DESIGN.md §"Oracle pins".
"""
from .ef import Program, ScheduleError, parse  # noqa: F401
from .collectives import chunk_elems, expected_outputs, expected_allreduce_f64, expected_reducescatter_f64  # noqa: F401
from .validate import validate, Verdict  # noqa: F401
from .simulate import run, run_symbolic  # noqa: F401
from .instances import expand_instances  # noqa: F401
