"""The reference's own hot-path unit tests (dim_tree_test, linalg_test,
tensor_test, kruskal_test, solver_test, io_test, synth_test, cli_test and the
acceptance criteria C01-C12 of acceptance_test from /root/reference/proj/tests),
compiled UNCHANGED against the drop-in `cpd::` headers (include/cpd) and
libcpdb.so by oracle/conformance/Makefile, run on the B200.

The binaries are built in the container (where the reference sources are)
and travel to the GPU box in oracle/_ref/conformance/.  Every case runs on the
library, including the CP-ALS normal-equation ones (cp_als, mttkrp,
solve_spd, fitness_fast_als: SURVEY.md 8f row 4).
"""
import os
import re
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "oracle", "_ref", "conformance")
SUITES = ["dim_tree_test", "linalg_test", "tensor_test", "kruskal_test", "solver_test", "io_test",
          "synth_test", "cli_test", "acceptance_test"]


def run_suite(name):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (needs /root/reference at build time)")
    p = subprocess.run([exe], capture_output=True, text=True, timeout=900)
    m = re.search(r"\[==========\] (\d+) passed, (\d+) failed", p.stdout)
    assert m, p.stdout[-2000:] + p.stderr[-4000:]
    failed = re.findall(r"^\[  FAILED  \] (\S+)$", p.stdout, re.M)
    return int(m.group(1)), failed, p


@pytest.mark.gpu
@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_on_device(suite):
    passed, failed, p = run_suite(suite)
    assert passed > 0
    assert not failed, "\n".join(failed) + "\n" + p.stderr[-6000:]


@pytest.mark.gpu
def test_acceptance_criteria_all_pass():
    """acceptance_test.cpp prints one line per criterion: C01-C12 all PASS on
    the device path (C08 runs the CLI through cpd::run_command, cli.hpp)."""
    passed, failed, p = run_suite("acceptance_test")
    crit = re.findall(r"^\[criterion +(\d+)\] (.*): (PASS|FAIL)$", p.stdout, re.M)
    assert len(crit) == 12, p.stdout[-3000:]
    assert all(r == "PASS" for _, _, r in crit), crit
