"""Pins for the byte/speedup model (CPU only): the paper's printed numbers
(tests/golden/paper_numbers.json) and the formulas of Tables 1/2 and
Eqs. 6, 9, 10."""
import json
import math
import os
from fractions import Fraction

import pytest

from paper_2605_19049_b200 import cost

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))
D = GOLD["head_dim_d"]["value"]


def test_state_size_and_384mb():
    st = cost.LayerBytes.make().st
    assert st == GOLD["state_bytes_per_layer_request"]["value_mb"] * 2 ** 20
    assert 4 * 48 * st == GOLD["verify_4_drafts_extra_memory"]["value_mb"] * 2 ** 20


def test_optimal_chunk_is_2_sqrt_d():
    assert abs(2 * math.sqrt(D) - GOLD["optimal_buffer_2sqrt_d"]["value"]) < 5e-3
    m_star = cost.paper_optimal_chunk(D)
    assert m_star in (22, 23)
    # Eq. 6 is symmetric in the sense f(m) = f(4d/m): the maximum sits at sqrt(4d)
    assert cost.paper_speedup_chunkwise(D, 16) == cost.paper_speedup_chunkwise(D, 32)


def test_table1_recurrent_and_chunkwise_consistency():
    _, rd, wr = cost.paper_table1("recurrent", D)
    assert (rd, wr) == (66304, 65792)
    # Eq. 6 is the ratio of total recurrent to total chunkwise access (Table 1)
    for m in (1, 4, 16, 23, 64):
        _, cr, cw = cost.paper_table1("chunkwise", D, m=m)
        assert Fraction(rd + wr) / (cr + cw) == cost.paper_speedup_chunkwise(D, m)


def test_table2_gdn_exact_speedups():
    _, rd, wr = cost.paper_table2("recurrent", D)
    for m in (1, 8, 23, 32):
        _, cr, cw = cost.paper_table2("chunkwise", D, m=m)
        assert Fraction(rd + wr) / (cr + cw) == cost.paper_speedup_chunkwise_gdn(D, m)
        # the GDN exact form is close to the vanilla approximation
        assert abs(cost.paper_speedup_chunkwise_gdn(D, m) / cost.paper_speedup_chunkwise(D, m) - 1) < 1e-3
    for L in (16, 64, 128):
        _, pr, pw = cost.paper_table2("parallel", D, L=L)
        _, cr, cw = cost.paper_table2("chunkwise", D, m=23)
        assert Fraction(cr + cw) / (pr + pw) == cost.paper_speedup_kv_only_gdn(D, 23, L)


def test_verify_speedup_numbers():
    s8 = float(cost.paper_speedup_verify(D, 8))
    assert abs(s8 - GOLD["verify_speedup_8_drafts_model"]["value"]) < 0.25     # "approximately 3x"
    assert abs(float(cost.paper_speedup_verify(D, 2)) - GOLD["verify_m2_parity"]["value"]) < 0.02
    # -> (m+1)/3 as d >> m
    assert abs(float(cost.paper_speedup_verify(10 ** 7, 5)) - 2.0) < 1e-5
    for m in (1, 2, 4, 8):
        assert abs(float(cost.paper_speedup_verify_gdn(D, m)) - float(cost.paper_speedup_verify(D, m))) < 1e-2


def test_kv_only_simplification_at_2_sqrt_d():
    """with m = 2 sqrt(d), Eq. 10 becomes (d + 2 sqrt(d) + 7/2) / (L + 2)."""
    m = 2 * math.sqrt(D)
    for L in (8, 64, 128):
        eq10 = (D + 2 * D / m + m / 2 + 3.5) / (L + 2)
        assert abs(eq10 - (D + 2 * math.sqrt(D) + 3.5) / (L + 2)) < 1e-12
    # monotonically decreasing in L; crossover (speedup 1) just above d
    vals = [cost.paper_speedup_kv_only(D, 23, L) for L in range(1, 200)]
    assert all(a > b for a, b in zip(vals, vals[1:]))
    L_star = next(L for L in range(1, 400) if cost.paper_speedup_kv_only(D, 23, L) < 1)
    assert D < L_star < 160


def test_capacity_ratio():
    assert cost.paper_capacity_ratio(4) == GOLD["capacity_ratio_4_drafts"]["value"]
    r = float(cost.paper_capacity_ratio(4, record_bytes_per_token=4 * D + 2, d=D))
    assert 4.8 < r < 5


def test_layer_bytes_appendix_b():
    b = cost.LayerBytes.make()
    assert (b.st, b.inp, b.rec, b.o) == (2097152, 16640, 20608, 16384)
    assert cost.LayerBytes.make(u_bytes=2).rec == 12416
    assert cost.LayerBytes.make(in_bytes=4).rec == 24704
    assert b.recurrent() == 4227328
    # cycle-average buffered bytes per token beat recurrent for C >= 8
    ratios = {C: b.recurrent() / float(b.cycle_avg(C)) for C in (1, 8, 16, 22, 32)}
    assert ratios[1] < 1 < ratios[8] < ratios[16]
    assert abs(ratios[16] - 1.633) < 2e-3
    assert abs(b.verify(4) + b.commit(0, 4) - 6.588e6) < 2e3
    assert abs(b.recurrent_verify(4) - 10.618e6) < 2e3
