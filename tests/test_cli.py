"""the `cpd` command-line front end (cli.hpp:72-252) on
the device path -- bin/cpd-b200.  Output formats (trace CSV, .cpdf model,
.cpdt tensor, `counts` report) follow io.hpp / cli.hpp; exit codes 0/1/2/3/4
as cli.hpp:230-250."""
import os
import struct
import subprocess

import numpy as np
import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "paper_2503_18759_b200", "bin", "cpd-b200")


def cli(*args, check=None):
    if not os.path.exists(BIN):
        pytest.fail(f"{BIN} not built")
    p = subprocess.run([BIN, *map(str, args)], capture_output=True, text=True, timeout=600)
    if check is not None:
        assert p.returncode == check, (p.returncode, p.stdout, p.stderr)
    return p


def read_cpdf(path):
    b = open(path, "rb").read()
    assert b[:4] == b"CPDF" and b[4] == 1
    order, rank = b[5], struct.unpack("<I", b[6:10])[0]
    dims = struct.unpack("<%dQ" % order, b[10:10 + 8 * order])
    v = np.frombuffer(b[10 + 8 * order:], dtype="<f8")
    lam, off, fs = v[:rank], rank, []
    for d in dims:
        fs.append(v[off:off + d * rank].reshape(d, rank))
        off += d * rank
    assert off == v.size
    return lam, fs


def parse_trace(path):
    lines = open(path).read().splitlines()
    assert lines[0] == "iter,order,fitness,raw_radicand,seconds,root_ttms,flops,beta,regularized"
    rows = []
    for ln in lines[1:]:
        f = ln.split(",")
        rows.append(dict(iteration=int(f[0]), order=[int(c) - 1 for c in f[1]],
                         fitness=float(f[2]), raw=float(f[3]), root=int(f[5]), flops=int(f[6]),
                         beta=float(f[7]), regularized=f[8] == "1"))
    return rows


@pytest.mark.parametrize("order,dims,rank", [(3, "512,512,512", 32), (4, "128,128,128,128", 16),
                                             (3, "9,8,7", 3)])
def test_counts_report(order, dims, rank):
    import paper_2503_18759_b200 as cpd
    out = cli("counts", "--order", order, "--dims", dims, "--rank", rank, check=0).stdout
    d = [int(v) for v in dims.split(",")]
    expected = (9, 6, 4) if order == 3 else (12, 6, 4)
    for name, want in zip(("naive", "dim-tree", "branch-reuse"), expected):
        line = next(ln for ln in out.splitlines() if ln.startswith(name + ":"))
        fl, roots = cpd.measured_cost(order, name, d, rank, 3)
        assert f"root_ttms={want} " in line and f"measured_flops={fl} " in line
        assert line.endswith(f"closed_form_flops={cpd.closed_form_cost(order, name, d, rank)}")


def test_exit_codes(tmp_path, ref):
    assert cli("decompose", "-i", tmp_path / "missing.cpdt", "--alg", "qr-bre", "--rank", 2).returncode == 2
    bad = tmp_path / "bad.cpdt"
    bad.write_bytes(b"CPDT\x02\x01" + b"\x00" * 8)
    assert cli("decompose", "-i", bad, "--alg", "qr-bre", "--rank", 2).returncode == 3
    assert cli("info", "-i", bad).returncode == 3
    # --alg als runs CP-ALS on the device: a malformed file
    # is a format error for it too, as in the reference
    assert cli("decompose", "-i", bad, "--alg", "als", "--rank", 2).returncode == 3
    assert cli("decompose", "-i", bad, "--alg", "bogus", "--rank", 2).returncode == 1
    assert cli("decompose", "-i", bad, "--alg", "qr", "--rank", 2, "--bogus", 1).returncode == 1
    assert cli("counts", "--order", 5, "--dims", "2,2,2,2,2", "--rank", 1).returncode == 1
    good = tmp_path / "g.cpdt"
    ref.write_tensor_file(str(good), np.ones((3, 4, 5)))
    out = cli("info", "-i", good, check=0).stdout
    assert out == "tensor file, version 1, order 3, dims 3x4x5, 60 values\n"


@pytest.mark.gpu
def test_decompose_end_to_end(tmp_path, port, ref):
    x = port.synth_baseline(0, (40, 36, 32), 5, 1e-2, 20250001)
    xin = tmp_path / "x.cpdt"
    ref.write_tensor_file(str(xin), x)
    trace, model = tmp_path / "t.csv", tmp_path / "m.cpdf"
    out = cli("decompose", "-i", xin, "--alg", "qr-bre", "--rank", 5, "--iters", 15, "--seed", 7,
              "--trace", trace, "-o", model, check=0).stdout
    o = port.solve(x, 5, 15, extrapolate=True, seed=7)
    rows = parse_trace(trace)
    assert len(rows) == len(o.trace)
    for r, w in zip(rows, o.trace):
        assert r["iteration"] == w["iteration"] and r["order"] == w["update_order"]
        assert r["flops"] == w["flops"] and r["root"] == w["root_ttm_count"]
        assert r["beta"] == w["beta_used"]
        assert abs(r["fitness"] - w["fitness"]) <= 1e-10 * w["fitness"]
    assert out.startswith("final_fitness ")
    assert abs(float(out.split()[1]) - o.trace[-1]["fitness"]) <= 1e-10
    lam, fs = read_cpdf(model)
    for f, w in zip(fs, o.factors):
        assert np.linalg.norm(f - w) / np.linalg.norm(w) <= 1e-10
    assert cli("info", "-i", model, check=0).stdout == \
        "model file, version 1, order 3, rank 5, dims 40x36x32\n"


@pytest.mark.gpu
def test_synth_matches_reference_generator(tmp_path, ref):
    out = tmp_path / "s.cpdt"
    cli("synth", "--dims", "12,10,8", "--rank", 3, "--collinearity", "0.5", "--l1", 5,
        "--l2", 2, "--seed", 17, "-o", out, check=0)
    rc, got = ref.read_tensor_file(str(out))
    assert rc == 0
    want = ref.assemble_noisy((12, 10, 8), 3, [0.5, 0.5, 0.5], 5.0, 2.0, 17)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-12


@pytest.mark.gpu
def test_synth_baseline_device_generator(tmp_path):
    import paper_2503_18759_b200 as cpd
    out = tmp_path / "c1.cpdt"
    cli("synth", "--baseline", "c1", "-o", out, check=0)
    ctx = cpd.Context(0)
    ctx.synth_tensor(0, [100, 100, 100], 10, 1e-2, 20250001)
    x = ctx.get_tensor([100, 100, 100])
    ctx.load_tensor(str(out))
    assert np.array_equal(ctx.get_tensor([100, 100, 100]), x)


@pytest.mark.gpu
def test_decompose_als_end_to_end(tmp_path, port, ref):
    """cpd-b200 decompose --alg als (cli.hpp:86-88: cp_als) with X streamed to
    HBM, trace and final fitness vs the reference's cp_als."""
    x = ref.synth_baseline(0, (30, 28, 26), 4, 1e-2, 777)
    xin = tmp_path / "x.cpdt"
    ref.write_tensor_file(str(xin), x)
    trace = tmp_path / "t.csv"
    out = cli("decompose", "-i", xin, "--alg", "als", "--rank", 4, "--iters", 12, "--seed", 9,
              "--trace", trace, check=0).stdout
    o = ref.cp_als(x, 4, 12, seed=9)
    rows = parse_trace(trace)
    assert len(rows) == len(o.trace)
    for r, w in zip(rows, o.trace):
        assert abs(r["fitness"] - w["fitness"]) <= 1e-10 * abs(w["fitness"])
    assert out.startswith("final_fitness ")
