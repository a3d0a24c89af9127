"""CPU: the C-ABI library loads, exports every symbol include/cpdb.h declares,
and its host-only scheduler matches the reference plans (no GPU needed)."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "cpdb.h")).read()
    return sorted(set(re.findall(r"\b(cpdb_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2503_18759_b200 import _cpdb
    lib = _cpdb.load()
    decl = declared_symbols()
    assert len(decl) >= 30
    for name in decl:
        assert hasattr(lib, name), name
    assert set(decl) == set(_cpdb.exported_symbols())


def test_version_and_no_gpu_fails_loudly():
    import paper_2503_18759_b200 as cpd
    from paper_2503_18759_b200 import _cpdb
    lib = _cpdb.load()
    assert b"sm_100a" in lib.cpdb_version()
    if lib.cpdb_device_ok(0):
        pytest.skip("a B200 is present")
    with pytest.raises(cpd.CpdError):
        cpd.Context(0)


@pytest.mark.parametrize("order", [3, 4])
@pytest.mark.parametrize("strategy", ["naive", "dim-tree", "branch-reuse"])
def test_scheduler_matches_reference(golden, order, strategy):
    import paper_2503_18759_b200 as cpd
    s = cpd.build_schedule(order, strategy, 7)
    assert np.array_equal(s.flat(), golden[f"sched_{order}_{strategy}"])
    assert [s.cycle_start, s.cycle_length] == list(golden[f"sched_{order}_{strategy}_cycle"])
    cpd.validate_schedule(s)


def test_retained_keys_match_oracle(port):
    import paper_2503_18759_b200 as cpd
    for order in (3, 4):
        for strategy in ("naive", "dim-tree", "branch-reuse"):
            s = cpd.build_schedule(order, strategy, 7)
            for it in range(7):
                for b in range(order):
                    assert cpd.retained_keys(s, it, b) == port.retained_keys(order, strategy, 7,
                                                                             it, b)


def test_root_counts_and_costs():
    """dim_tree_test.cpp:107-123 (9/6/4, 12/6/4), :154-162, :164-200."""
    import paper_2503_18759_b200 as cpd
    for order, expect in ((3, (9, 6, 4)), (4, (12, 6, 4))):
        dims = [5, 6, 7, 8][:order]
        got = tuple(cpd.measured_cost(order, s, dims, 3, 3)[1]
                    for s in ("naive", "dim-tree", "branch-reuse"))
        assert got == expect
        for s in ("naive", "dim-tree", "branch-reuse"):
            assert cpd.measured_cost(order, s, dims, 3, 3)[0] == cpd.closed_form_cost(order, s,
                                                                                       dims, 3)
    # steady state: one root TTM per sweep
    for order in (3, 4):
        s_roots = [cpd.measured_cost(order, "branch-reuse", [6] * order, 2, i)[1] for i in
                   range(1, 10)]
        assert np.all(np.diff(s_roots)[2:] == 1)
    # hand-evaluated closed form at 100^3 R=10 (dim_tree_test.cpp:177-187)
    assert cpd.closed_form_cost(3, "branch-reuse", [100] * 3, 10) == (
        8 * 100 ** 3 * 10 + 4 * 100 ** 2 * 100 + 8 * 100 ** 2 * 100 + 6 * 100 ** 2 * 100)
    assert [cpd.leading_flop_coefficient(3, s) for s in ("naive", "dim-tree", "branch-reuse")] \
        == [18, 12, 8]
    assert [cpd.leading_flop_coefficient(4, s) for s in ("naive", "dim-tree", "branch-reuse")] \
        == [24, 12, 8]


def test_branch_reuse_update_orders():
    """Appendix A / solver_test.cpp:208-218: 123, 132, 231, 132, 231."""
    import paper_2503_18759_b200 as cpd
    s = cpd.build_schedule(3, "branch-reuse", 5)
    assert [s.update_order(i) for i in range(5)] == [[0, 1, 2], [0, 2, 1], [1, 2, 0], [0, 2, 1],
                                                    [1, 2, 0]]
    s4 = cpd.build_schedule(4, "branch-reuse", 8)
    assert s4.update_order(1) == [2, 3, 1, 0] and s4.update_order(2) == [0, 2, 3, 1]
    assert s4.update_order(5) == s4.update_order(2)


def test_stale_schedule_rejected():
    """dim_tree_test.cpp:275-307: a plan that reads an intermediate after one
    of its absorbed factors changed is rejected at build/validate time."""
    import paper_2503_18759_b200 as cpd
    S, step = cpd.Schedule, cpd.step
    bad = S(3, 1, [[cpd.ModeUpdate(0, [step(0b111, 2), step(0b011, 1)]),
                    cpd.ModeUpdate(2, [step(0b111, 1), step(0b101, 0)]),
                    cpd.ModeUpdate(1, [step(0b011, 0)])]], 0, 1)
    with pytest.raises(cpd.StaleIntermediateError):
        cpd.validate_schedule(bad)
    missing = S(3, 1, [[cpd.ModeUpdate(0, [step(0b011, 1)]),
                        cpd.ModeUpdate(1, [step(0b111, 0), step(0b110, 2)]),
                        cpd.ModeUpdate(2, [step(0b111, 0), step(0b110, 1)])]], 0, 1)
    with pytest.raises(cpd.CpdError):
        cpd.validate_schedule(missing)
    with pytest.raises(ValueError):
        cpd.build_schedule(5, "dim-tree", 2)
    with pytest.raises(ValueError):
        cpd.build_schedule(3, "naive", 0)


def test_select_beta_table():
    """solver_test.cpp:88-99"""
    import paper_2503_18759_b200 as cpd
    assert cpd.select_beta(0.95, 0.955, 0.03) == 1.0 / 2000.0
    assert cpd.select_beta(0.60, 0.80, 0.03) is None
    assert cpd.select_beta(0.50, 0.51, 0.03) == 1.0 / 250.0
    assert cpd.select_beta(0.79, 0.80, 0.03) == 1.0 / 500.0
    assert cpd.select_beta(0.90, 0.90, 0.03) == 1.0 / 500.0
    assert cpd.select_beta(0.905, 0.905, 0.03) == 1.0 / 2000.0
    assert cpd.select_beta(0.70, 0.70, 0.03) == 1.0 / 500.0
    assert cpd.select_beta(-0.5, -0.49, 0.03) == 1.0 / 250.0


def test_init_state_checked_before_the_abi():
    """a given model / sweep state must match the tensor and
    the config before Context.solve hands raw buffers to the C ABI
    (solvers.hpp:105-112 messages)."""
    import paper_2503_18759_b200 as cpd
    dims, R = (5, 4, 3), 2
    good = cpd.SweepState(0, np.ones(R), [np.zeros((d, R)) for d in dims])
    cpd.check_init_state(good, dims, R)
    cases = [
        (cpd.SweepState(0, np.ones(R), [np.zeros((d, R)) for d in dims[:2]]), "tensor/config"),
        (cpd.SweepState(0, np.ones(R + 1), [np.zeros((d, R)) for d in dims]), "tensor/config"),
        (cpd.SweepState(0, np.ones(R), [np.zeros((d, R + 1)) for d in dims]), "tensor/config"),
        (cpd.SweepState(0, np.ones(R), [np.zeros((d + 1, R)) for d in dims]), "rows"),
        (cpd.SweepState(0, np.ones(R), [np.zeros((d, R)) for d in dims],
                        q0_history=[np.zeros((R * R + 1, R)), None, None]), "Q0 history"),
    ]
    for st, what in cases:
        with pytest.raises(cpd.CpdInvalidArgument, match=what):
            cpd.check_init_state(st, dims, R)
