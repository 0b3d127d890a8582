"""FKT tensor files (tensor_io.hpp:13-18, tensor_io.cpp:12-117).

The product library, the C oracle and the unmodified reference (behind its
shim, using its own tensor_write_file / tensor_read_file) write byte-identical
files for the same planes, read each other's files, and fail with the same
Errc on malformed ones. The GPU case round-trips device planes.
"""
import struct

import numpy as np
import pytest

from paper_2508_07071_b200._ffi import F32, F64X3, U8, U8X3
from paper_2508_07071_b200.opfuse import OpfuseError

KINDS = [(U8, np.uint8, ()), (F32, np.float32, ()), (F64X3, np.float64, (3,)), (U8X3, np.uint8, (3,))]


def planes_of(lib, kind, dtype, tail, n=3, seed=0):
    rng = np.random.default_rng(seed)
    arrs = []
    for i in range(n):
        h, w = 5 + i, 7 + 2 * i
        a = rng.integers(0, 256, (h, w) + tail).astype(dtype) if dtype == np.uint8 else \
            rng.standard_normal((h, w) + tail).astype(dtype)
        arrs.append(a)
    return arrs, [lib.plane_from_numpy(a) for a in arrs]


@pytest.mark.parametrize("kind,dtype,tail", KINDS)
def test_files_identical_and_cross_readable(tmp_path, oracle, reference, kind, dtype, tail):
    arrs, po = planes_of(oracle, kind, dtype, tail)
    _, pr = planes_of(reference, kind, dtype, tail)
    oracle.tensor_write_file(po, tmp_path / "o.fkt")
    reference.tensor_write_file(pr, tmp_path / "r.fkt")
    raw = (tmp_path / "o.fkt").read_bytes()
    assert raw == (tmp_path / "r.fkt").read_bytes()
    assert raw[:4] == b"FKT1" and struct.unpack_from("<I", raw, 4)[0] == len(arrs)
    for lib, path in ((oracle, "r.fkt"), (reference, "o.fkt")):
        got = lib.tensor_read_file(tmp_path / path)
        assert len(got) == len(arrs)
        for g, a in zip(got, arrs):
            assert g.kind == kind and (g.height, g.width) == a.shape[:2]
            assert np.array_equal(lib.download(g).view(np.uint8), a.view(np.uint8))


def test_error_codes_match_reference(tmp_path, oracle, reference):
    cases = {"missing": None, "short": b"FK", "magic": b"FKT2\x01\x00\x00\x00",
             "empty": b"FKT1\x00\x00\x00\x00", "tag": b"FKT1\x01\x00\x00\x00\x09\x00\x00\x00\x01\x00\x00\x00\x01\x00\x00\x00",
             "trunc": b"FKT1\x01\x00\x00\x00\x00\x00\x00\x00\x04\x00\x00\x00\x04\x00\x00\x00\x01\x02",
             "mixed": b"FKT1\x02\x00\x00\x00" + b"\x00\x00\x00\x00\x01\x00\x00\x00\x01\x00\x00\x00\x07" +
                      b"\x01\x00\x00\x00\x01\x00\x00\x00\x01\x00\x00\x00\x00\x00\x80\x3f"}
    for name, blob in cases.items():
        path = tmp_path / f"{name}.fkt"
        if blob is not None:
            path.write_bytes(blob)
        codes = []
        for lib in (oracle, reference):
            with pytest.raises(OpfuseError) as e:
                lib.tensor_read_file(path)
            codes.append(e.value.code)
        assert codes[0] == codes[1], (name, codes)
    assert codes[0] == "InnerKindMismatch"
    for lib in (oracle, reference):
        with pytest.raises(OpfuseError) as e:
            lib.tensor_write_file([], tmp_path / "x.fkt")
        assert e.value.code == "EmptyBatch"


def test_ppm_matches_reference(tmp_path, oracle, reference):
    rng = np.random.default_rng(4)
    a = rng.integers(0, 256, (6, 9, 3), dtype=np.uint8)
    oracle.write_ppm(oracle.plane_from_numpy(a), tmp_path / "o.ppm")
    reference.write_ppm(reference.plane_from_numpy(a), tmp_path / "r.ppm")
    assert (tmp_path / "o.ppm").read_bytes() == (tmp_path / "r.ppm").read_bytes() == b"P6\n9 6\n255\n" + a.tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("kind,dtype,tail", KINDS)
def test_device_planes_round_trip(tmp_path, cuda, oracle, kind, dtype, tail):
    arrs, pc = planes_of(cuda, kind, dtype, tail)
    _, po = planes_of(oracle, kind, dtype, tail)
    cuda.tensor_write_file(pc, tmp_path / "c.fkt")
    oracle.tensor_write_file(po, tmp_path / "o.fkt")
    assert (tmp_path / "c.fkt").read_bytes() == (tmp_path / "o.fkt").read_bytes()
    got = cuda.tensor_read_file(tmp_path / "o.fkt")
    for g, a in zip(got, arrs):
        assert np.array_equal(cuda.download(g).view(np.uint8), a.view(np.uint8))
