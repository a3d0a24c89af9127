""".cpdt tensor files (io.hpp:93-121) streamed straight
into HBM.  Pinned against the reference's own codec (oracle/_ref: cpd::
write_tensor_file / read_tensor_file): files it writes load bit-exactly, files
we write it reads back bit-exactly, and the malformed files it rejects we
reject (format_error <-> FormatError, file_error <-> FileError)."""
import os
import struct

import numpy as np
import pytest

import paper_2503_18759_b200 as cpd


def header(dims, magic=b"CPDT", version=1):
    return magic + bytes([version, len(dims)]) + b"".join(struct.pack("<Q", d) for d in dims)


MALFORMED = {
    "bad_magic": lambda: header((2, 3), magic=b"CPDX") + np.zeros(6).tobytes(),
    "bad_version": lambda: header((2, 3), version=2) + np.zeros(6).tobytes(),
    "zero_order": lambda: b"CPDT" + bytes([1, 0]),
    "zero_extent": lambda: header((2, 0, 3)),
    "truncated": lambda: header((2, 3)) + np.zeros(5).tobytes(),
    "trailing": lambda: header((2, 3)) + np.zeros(6).tobytes() + b"\x00",
    "short_header": lambda: b"CPD",
}


@pytest.fixture()
def tmpfile(tmp_path):
    return lambda name: str(tmp_path / name)


def test_info_of_reference_written_file(ref, tmpfile):
    x = np.arange(4 * 5 * 6, dtype=np.float64).reshape(4, 5, 6) * 0.25 - 3.0
    p = tmpfile("x.cpdt")
    ref.write_tensor_file(p, x)
    assert os.path.getsize(p) == 6 + 8 * 3 + 8 * x.size
    assert cpd.cpdt_info(p) == [4, 5, 6]
    # our reading of the bytes == the reference's
    rc, back = ref.read_tensor_file(p)
    assert rc == 0 and np.array_equal(back, x)


@pytest.mark.parametrize("case", sorted(MALFORMED))
def test_malformed_rejected_like_reference(ref, tmpfile, case):
    p = tmpfile(case + ".cpdt")
    with open(p, "wb") as f:
        f.write(MALFORMED[case]())
    rc, _ = ref.read_tensor_file(p)
    assert rc == 9, (case, rc)  # reference: format_error
    with pytest.raises(cpd.FormatError):
        cpd.cpdt_info(p)


def test_missing_file(ref, tmpfile):
    p = tmpfile("nope.cpdt")
    assert ref.read_tensor_file(p)[0] == 8  # file_error
    with pytest.raises(cpd.FileError):
        cpd.cpdt_info(p)


@pytest.mark.gpu
def test_load_save_roundtrip_bit_exact(ctx, ref, tmpfile):
    rng = np.random.default_rng(5)
    x = rng.standard_normal((33, 17, 9))
    p = tmpfile("in.cpdt")
    ref.write_tensor_file(p, x)
    ctx.load_tensor(p)
    assert ctx.dims == [33, 17, 9]
    assert np.array_equal(ctx.get_tensor([33, 17, 9]), x)
    q = tmpfile("out.cpdt")
    ctx.save_tensor(q)
    rc, back = ref.read_tensor_file(q)
    assert rc == 0 and np.array_equal(back, x)
    with open(p, "rb") as a, open(q, "rb") as b:
        assert a.read() == b.read()


@pytest.mark.gpu
def test_load_large_multichunk(ctx, tmpfile):
    """> 2 staging chunks (64 MiB each): 160 MiB tensor."""
    dims = (320, 256, 256)
    x = np.random.default_rng(9).standard_normal(dims)
    p = tmpfile("big.cpdt")
    with open(p, "wb") as f:
        f.write(header(dims))
        f.write(x.tobytes())
    ctx.load_tensor(p)
    assert np.array_equal(ctx.get_tensor(list(dims)), x)


@pytest.mark.gpu
def test_nonfinite_payload_rejected(ctx, ref, tmpfile):
    x = np.ones((4, 4, 4))
    x[1, 2, 3] = np.nan
    p = tmpfile("nan.cpdt")
    with open(p, "wb") as f:
        f.write(header(x.shape) + x.tobytes())
    assert ref.read_tensor_file(p)[0] == 9
    with pytest.raises(cpd.FormatError):
        ctx.load_tensor(p)


@pytest.mark.gpu
def test_solve_from_loaded_file_matches_in_memory(ctx, port, ref, tmpfile):
    x = port.rng_normals(41, 12 * 10 * 8).reshape(12, 10, 8)
    p = tmpfile("s.cpdt")
    ref.write_tensor_file(p, x)
    cfg = cpd.SolverConfig(rank=3, max_iterations=6, seed=2)
    ctx.load_tensor(p)
    a = ctx.solve(cfg, extrapolate=True)
    b = cpd.als_qr_bre(x, cfg, ctx=ctx)
    assert [t.fitness for t in a.trace] == [t.fitness for t in b.trace]
