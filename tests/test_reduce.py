"""ReduceDPP (dpp.hpp:32-53, dpp.cpp:46-246): multi_reduce_plane on the C oracle,
the unmodified reference, and the CUDA product.

CPU: the oracle restatement equals the reference bit for bit (same worker
count), on the SPEC.md examples (:366-383) and on random reads / specs; error
codes match. GPU: the CUDA fold equals the oracle exactly for u8 sums and every
Max / Min (ties between +0 and -0 resolved to the earliest element, NaNs never
adopted), and float sums (accumulated in double, in a different order) within
the 2^-20 relative tolerance SPEC.md:388 declares.
"""
import math

import numpy as np
import pytest

from fkchains import _rand_compute, make_compute, make_read, random_chain
from paper_2508_07071_b200 import opfuse as of
from paper_2508_07071_b200._ffi import F32, F32X3, F64, F64X3, LANES, REDUCE_MAX, REDUCE_MIN, REDUCE_SUM, U8, U8X3
from paper_2508_07071_b200.opfuse import Library, OpfuseError


def lk(kind):
    return kind - 3 if kind >= U8X3 else kind


def random_specs(rng, lib, read, spec):
    """1-5 (combine, transform, identity) specs over `read`'s output kind."""
    out = []
    k = read.output_kind
    for _ in range(int(rng.integers(1, 6))):
        combine = int(rng.integers(0, 3))
        transform, vk = None, k
        if rng.random() < 0.5:
            c, vk = _rand_compute(rng, k, max(1, len(spec.reads)), False)
            transform = make_compute(lib, c)
        ident = None
        if rng.random() < 0.3:
            vals = [float(rng.choice([0.0, -0.0, 1.0, 7.5, -3.0, np.nan])) for _ in range(LANES[vk])]
            if lk(vk) == U8:
                vals = [int(v) % 256 if not math.isnan(v) else 5 for v in vals]
            ident = of.const_of(vk, *vals)
        out.append((combine, transform, ident))
    return out


def reduce_on(lib, spec, rng_seed, workers):
    rng = np.random.default_rng(rng_seed)
    read, planes = make_read(lib, spec)
    specs = random_specs(rng, lib, read, spec)
    res, reads = lib.multi_reduce_plane(read, specs, workers)
    return res, reads, [(c, read.output_kind if t is None else (t.output_kind or t.input_kind)) for c, t, _ in specs]


def same_bits(a, b):
    return all((x == y) or (isinstance(x, float) and math.isnan(x) and math.isnan(y)) or
               (x == 0 and y == 0 and math.copysign(1, x) == math.copysign(1, y)) for x, y in zip(a, b)) and \
        all(not (isinstance(x, float) and x == 0 and math.copysign(1, x) != math.copysign(1, y)) for x, y in zip(a, b))


@pytest.fixture(scope="module")
def oracle():
    return Library("oracle")


@pytest.fixture(scope="module")
def reference():
    try:
        return Library("reference")
    except FileNotFoundError:
        pytest.skip("reference shim not built (oracle/_ref)")


def test_spec_examples(oracle, reference):
    for lib in (oracle, reference):
        r = lib.op_read_per_thread(lib.plane_from_numpy(np.array([[3, 1, 2]], dtype=np.uint8)))
        res, reads = lib.multi_reduce_plane(r, [(REDUCE_SUM, None, None), (REDUCE_MAX, None, None),
                                                (REDUCE_MIN, None, None)])
        assert res == [(6,), (3,), (1,)] and reads == 3
        r = lib.op_read_per_thread(lib.plane_from_numpy(np.full((5, 6), 7.0, dtype=np.float32)))
        assert lib.reduce_plane(r, REDUCE_MAX) == (7.0,)
        r = lib.op_read_per_thread(lib.plane_from_numpy(np.arange(64, dtype=np.float64).reshape(8, 8)))
        res, reads = lib.multi_reduce_plane(r, [(REDUCE_SUM, None, None)] * 3)
        assert reads == 64 and res[0] == (2016.0,)


def test_errors_match_reference(oracle, reference):
    for lib in (oracle, reference):
        p = lib.plane_from_numpy(np.zeros((4, 4), dtype=np.float32))
        r = lib.op_read_per_thread(p)
        with pytest.raises(OpfuseError) as e:
            lib.multi_reduce_plane(r, [])
        assert e.value.code == "EmptyIterSpace"
        with pytest.raises(OpfuseError) as e:
            lib.multi_reduce_plane(r, [(REDUCE_SUM, lib.op_cast(U8, F32), None)])
        assert e.value.code == "KindMismatch"
        with pytest.raises(OpfuseError) as e:
            lib.multi_reduce_plane(r, [(REDUCE_SUM, lib.op_read_per_thread(p), None)])
        assert e.value.code == "InvalidConfig"


@pytest.mark.parametrize("seed", range(4))
def test_oracle_equals_reference(oracle, reference, seed):
    rng = np.random.default_rng(500 + seed)
    for i in range(40):
        spec = random_chain(rng, max_dim=20)
        w = int(rng.choice([1, 2, 4]))
        a, ra, kinds = reduce_on(oracle, spec, 9000 + 100 * seed + i, w)
        b, rb, _ = reduce_on(reference, spec, 9000 + 100 * seed + i, w)
        assert ra == rb
        for x, y in zip(a, b):
            assert same_bits(x, y), (x, y, kinds)


# ------------------------------------------------------------------- GPU --

def close(x, y, combine, kind):
    if combine == REDUCE_SUM and lk(kind) != U8:
        for a, b in zip(x, y):
            if math.isnan(a) or math.isnan(b):
                assert math.isnan(a) and math.isnan(b)
            elif math.isinf(a) or math.isinf(b):
                assert a == b
            else:
                assert abs(a - b) <= abs(b) * 2.0 ** -20 + 1e-300, (a, b)
        return
    assert same_bits(x, y), (x, y, combine, kind)


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4))
def test_cuda_equals_oracle(oracle, seed):
    cuda = Library("cuda")
    rng = np.random.default_rng(700 + seed)
    for i in range(40):
        spec = random_chain(rng, max_dim=40, max_batch=5)
        a, ra, kinds = reduce_on(cuda, spec, 7000 + 100 * seed + i, 0)
        b, rb, _ = reduce_on(oracle, spec, 7000 + 100 * seed + i, 1)
        assert ra == rb
        for x, y, (c, k) in zip(a, b, kinds):
            close(x, y, c, k)


@pytest.mark.gpu
def test_cuda_signed_zero_ties_and_nans(oracle):
    """Max/Min over values equal as numbers but not as bits (+0/-0): the earliest
    element in (z, y, x) order wins, as in the reference's sequential fold; NaNs
    are never adopted; a NaN identity survives. Large planes exercise the
    cross-CTA combine."""
    cuda = Library("cuda")
    rng = np.random.default_rng(3)
    for dt, kind in ((np.float32, F32), (np.float64, F64)):
        for first in (0.0, -0.0):
            a = np.zeros((700, 900), dtype=dt)
            a[rng.random(a.shape) < 0.5] = -0.0
            a.flat[0] = first
            a[rng.random(a.shape) < 0.01] = np.nan
            for libs in ((cuda, oracle),):
                got = [lib.multi_reduce_plane(lib.op_read_per_thread(lib.plane_from_numpy(a)),
                                              [(REDUCE_MAX, None, None), (REDUCE_MIN, None, None),
                                               (REDUCE_MAX, None, of.const_of(kind, float("nan"))),
                                               (REDUCE_SUM, None, None)])[0] for lib in libs]
                for x, y in zip(got[0][:3], got[1][:3]):
                    assert same_bits(x, y), (x, y)


@pytest.mark.gpu
def test_cuda_large_u8x3_and_many_specs(oracle):
    """A 4K u8x3 plane with 6 specs (two traversals of 4 specs on the device)."""
    cuda = Library("cuda")
    rng = np.random.default_rng(11)
    a = rng.integers(0, 256, (1080, 1920, 3), dtype=np.uint8)
    specs_of = lambda lib: [(REDUCE_SUM, None, None), (REDUCE_MAX, None, None), (REDUCE_MIN, None, None),  # noqa: E731
                            (REDUCE_SUM, lib.op_cast(U8X3, F64X3), None),
                            (REDUCE_MAX, lib.make_arith(7, of.const_of(U8X3, 3, 5, 7)), None),
                            (REDUCE_SUM, lib.make_arith(8, of.const_of(U8X3, 1, 2, 3)), of.const_of(U8X3, 9, 9, 9))]
    res = [lib.multi_reduce_plane(lib.op_read_per_thread(lib.plane_from_numpy(a)), specs_of(lib), 16)
           for lib in (cuda, oracle)]
    assert res[0][1] == res[1][1]
    kinds = [U8X3, U8X3, U8X3, F64X3, U8X3, U8X3]
    for x, y, (c, _, _), k in zip(res[0][0], res[1][0], specs_of(oracle), kinds):
        close(x, y, c, k)


@pytest.mark.gpu
@pytest.mark.parametrize("dt,kind", [(np.uint8, U8), (np.float32, F32), (np.uint8, U8X3)])
def test_cuda_plain_rows(oracle, dt, kind):
    """One plane of 16-byte aligned u8 / f32 / u8x3 rows: the vector kernels
    (fk_reduce_plain, fk_reduce_plain3). Crops whose width is not a multiple of
    the vector leave a partial last vector per row; transforms run per spec;
    -0 / NaN included; an unaligned crop takes the per-tile kernel."""
    cuda = Library("cuda")
    rng = np.random.default_rng(21)
    shape = (517, 1024, 3) if kind == U8X3 else (517, 1024)
    big = (rng.integers(0, 256, shape, dtype=np.uint8) if dt == np.uint8
           else rng.standard_normal(shape).astype(np.float32))
    if dt == np.float32:
        big[rng.random(big.shape) < 0.001] = np.nan
    cast_to = {U8: F32, F32: U8, U8X3: F32X3}[kind]
    vals = (3, 4, 5) if kind == U8X3 else (3,)
    crops = [(0, 0, 1024, 517), (16, 3, 37, 200), (16, 0, 1000, 1), (0, 1, 5, 516), (64, 5, 960, 511), (3, 2, 50, 50)]
    for x0, y0, w, h in crops:
        specs_of = lambda lib: [(REDUCE_SUM, None, None), (REDUCE_MAX, None, None), (REDUCE_MIN, None, None),  # noqa
                                (REDUCE_SUM, lib.make_arith(8, of.const_of(kind, *vals)), None),
                                (REDUCE_MAX, lib.op_cast(kind, cast_to), of.const_of(cast_to, *([7] * len(vals))))]
        res = []
        for lib in (cuda, oracle):
            p = lib.plane_from_numpy(big, kind)
            r = lib.op_crop(p, x0, y0, w, h) if (w, h) != (1024, 517) else lib.op_read_per_thread(p)
            res.append(lib.multi_reduce_plane(r, specs_of(lib)))
        assert res[0][1] == res[1][1] == w * h
        if x0 % 16 == 0:
            assert cuda.last_kernel().startswith("fk_reduce_plain"), cuda.last_kernel()
        kinds = [kind, kind, kind, kind, cast_to]
        for x, y, (c, _, _), k in zip(res[0][0], res[1][0], specs_of(oracle), kinds):
            close(x, y, c, k)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", [U8, U8X3])
def test_cuda_plain_rows_mixed_value_kinds(oracle, kind):
    """Plain u8 rows folded by u8-valued Max/Min specs (packed 16x2 lanes) next
    to f32-valued Max/Min specs (cast transforms) in the same traversal, on data
    whose extrema are non-zero (10..255): the packed lanes must only join the
    specs that fed them (an f32 Min returned 0.0 instead of 10.0)."""
    cuda = Library("cuda")
    rng = np.random.default_rng(5)
    shape = (300, 1024, 3) if kind == U8X3 else (300, 1024)
    big = rng.integers(10, 256, shape, dtype=np.uint8)
    to = F32X3 if kind == U8X3 else F32
    n = 3 if kind == U8X3 else 1
    spec_sets = [
        lambda lib: [(REDUCE_MIN, lib.op_cast(kind, to), None), (REDUCE_MIN, None, None),
                     (REDUCE_MAX, lib.op_cast(kind, to), None), (REDUCE_MAX, None, None)],
        lambda lib: [(REDUCE_MIN, lib.op_cast(kind, to), of.const_of(to, *([300.0] * n))),
                     (REDUCE_MIN, None, of.const_of(kind, *([200] * n))),
                     (REDUCE_SUM, None, None), (REDUCE_MAX, lib.op_cast(kind, to), None)],
    ]
    for specs_of in spec_sets:
        res = []
        for lib in (cuda, oracle):
            p = lib.plane_from_numpy(big, kind)
            res.append(lib.multi_reduce_plane(lib.op_read_per_thread(p), specs_of(lib)))
        assert cuda.last_kernel().startswith("fk_reduce_plain"), cuda.last_kernel()
        for x, y, (c, t, _) in zip(res[0][0], res[1][0], specs_of(oracle)):
            close(x, y, c, kind if t is None else to)
        mins = [v for (c, t, _), v in zip(specs_of(oracle), res[0][0]) if c == REDUCE_MIN]
        assert all(min(v) >= 10 for v in mins), mins
