"""CPU pins of the alpha-beta profiler's solver (generator/profiler.py):
synthetic measurements with known alpha, beta and per-call cost are recovered; the paper's
own worked example (Table 1 InfiniBand constants, two 32 KB chunks: 10.025 us one after the
other, 8.325 us together) solves back to Table 1's alpha and beta."""
import numpy as np
import pytest

from paper_2111_04867_b200.generator.profiler import connection_table, solve_alpha_beta


def _synthetic(alpha, beta, c, noise, seed):
    rng = np.random.default_rng(seed)
    out = []
    for k in (2, 4, 8):
        for s in (2.0 ** e for e in range(-10, 7)):  # 1 KiB .. 64 MiB chunks, in MB
            for mode in ("seq", "tog"):
                t = c + (k * (alpha + beta * s) if mode == "seq" else alpha + k * beta * s)
                out.append((mode, k, s, t * (1 + noise * rng.standard_normal())))
    return out


@pytest.mark.parametrize("alpha,beta,c", [(2.6, 1.42, 3.1), (0.7, 8.0, 0.0), (1.7, 106.0, 5.0)])
def test_recovers_known_alpha_beta(alpha, beta, c):
    fit = solve_alpha_beta(_synthetic(alpha, beta, c, 0.0, 1))
    assert fit["alpha_us"] == pytest.approx(alpha, rel=1e-9, abs=1e-9)
    assert fit["beta_us_per_MB"] == pytest.approx(beta, rel=1e-9)
    assert fit["c_us"] == pytest.approx(c, abs=1e-9)
    noisy = solve_alpha_beta(_synthetic(alpha, beta, c, 0.002, 2))
    assert noisy["beta_us_per_MB"] == pytest.approx(beta, rel=0.01)


def test_alpha_is_what_separates_seq_from_tog():
    # with beta = 0 the difference between k one-after-another transfers and one k-chunk
    # transfer is exactly (k - 1) * alpha; a solver that swapped the models would get -alpha
    meas = [("seq", 4, 1.0, 10 + 4 * 2.0), ("tog", 4, 1.0, 10 + 2.0), ("seq", 2, 1.0, 10 + 2 * 2.0),
            ("tog", 2, 1.0, 10 + 2.0), ("seq", 8, 0.5, 10 + 8 * 2.0)]
    fit = solve_alpha_beta(meas)
    assert fit["alpha_us"] == pytest.approx(2.0) and fit["beta_us_per_MB"] == pytest.approx(0.0, abs=1e-9)


def test_paper_infiniband_example_solves_to_table_1():
    # with Table 1's IB alpha = 1.7 us, beta = 106 us/MB, two 32 KB chunks take
    # 2 * (1.7 + 106 * 0.03125) = 10.025 us apart and 1.7 + 2 * 106 * 0.03125 = 8.325 us together
    s = 32 / 1024
    meas = [("seq", 2, s, 10.025), ("tog", 2, s, 8.325)]
    fit = solve_alpha_beta(meas, fit_c=False)
    assert fit["alpha_us"] == pytest.approx(1.7) and fit["beta_us_per_MB"] == pytest.approx(106.0)
    assert 1 - 8.325 / 10.025 == pytest.approx(0.1696, abs=1e-4)  # the paper's "17% faster"


def test_too_few_measurements_rejected():
    with pytest.raises(ValueError):
        solve_alpha_beta([("seq", 2, 1.0, 5.0), ("tog", 2, 1.0, 4.0)])


def test_connection_table():
    rows = [{"probe": "connections", "connections": c, "volume_bytes": v, "egress_GBps": bw}
            for c, v, bw in [(1, 1 << 30, 700.0), (2, 1 << 30, 690.0), (3, 1 << 30, 680.0), (1, 1 << 20, 300.0)]]
    t = connection_table(rows)
    assert [r["connections"] for r in t] == [1, 2, 3]
    assert [r["vs_one_connection"] for r in t] == [1.0, round(690 / 700, 4), round(680 / 700, 4)]
