"""The lazy facade (paper_2508_07071_b200.api, mirroring api.cpp) on the C oracle
and the reference: SPEC acceptance #2/#4/#8 through execute_operations /
execute_batch, provenance-annotated errors, the uid-keyed cache."""
import numpy as np
import pytest

from paper_2508_07071_b200 import api
from paper_2508_07071_b200._ffi import BILINEAR, F32, F32X3, SWAP_RB, U8, U8X3
from paper_2508_07071_b200.opfuse import Library, OpfuseError, f32, f32x3, u8

from fkchains import outputs_equal


@pytest.fixture(params=["oracle", "reference"])
def lib(request):
    return Library(request.param)


def _memory_pipeline(lib):
    """SPEC §6.10 / bench.cpp:414-430 (with the 256x512 source; 256x256 crops out of bounds)."""
    rng = np.random.default_rng(42)
    source = lib.plane_from_numpy(rng.random((512, 256, 3)).astype(np.float32))
    out = [lib.plane_alloc(60, 120, F32) for _ in range(3)]
    handles = [api.resize(api.crop(source, 10, 20, 120, 240, lib=lib), 60, 120, BILINEAR),
               api.cvt_color(SWAP_RB), api.multiply(f32x3(255, 255, 255), lib=lib),
               api.subtract(f32x3(0.485, 0.456, 0.406), lib=lib), api.divide(f32x3(0.229, 0.224, 0.225), lib=lib),
               api.split(out, lib=lib)]
    return handles, out


def test_facade_memory_pipeline_and_single_validation(lib):
    handles, out = _memory_pipeline(lib)
    p = api.build_pipeline(handles)
    assert p.n_compute == 3                      # SwapRB folded into the read
    assert lib.plan_memory_savings(p) == 259200  # SPEC acceptance #2
    before = api.validations()
    r1 = api.execute_operations(handles)
    first = [o.to_numpy().copy() for o in out]
    r2 = api.execute_operations(handles)
    assert api.validations() == before + 1       # SPEC acceptance #8: one validation for two calls
    assert r1.passes == r2.passes == 1
    assert all(np.array_equal(a, o.to_numpy()) for a, o in zip(first, out))


def test_facade_matches_reference_bit_for_bit():
    outs = []
    for backend in ("oracle", "reference"):
        L = Library(backend)
        handles, out = _memory_pipeline(L)
        api.execute_operations(handles)
        outs.append([[o.to_numpy() for o in out]])
    assert outputs_equal(outs[0], outs[1])


def test_facade_errors_name_the_handle(lib):
    a = lib.plane_alloc(8, 8, U8X3)
    b = lib.plane_alloc(8, 8, F32X3)
    with pytest.raises(OpfuseError) as e:
        api.build_pipeline([api.read(a, lib=lib), api.cvt_color(SWAP_RB), api.subtract(f32x3(1, 2, 3), lib=lib),
                            api.write(b, lib=lib)])
    assert e.value.code == "KindMismatch" and e.value.provenance == "subtract (handle #3)"
    with pytest.raises(OpfuseError) as e:
        api.divide(f32(0.0), lib=lib)
    assert e.value.code == "DivByZeroParam" and e.value.provenance == "divide"
    with pytest.raises(OpfuseError) as e:
        api.build_pipeline([api.cvt_color(SWAP_RB), api.write(b, lib=lib)])
    assert e.value.provenance == "cvt_color"


def test_execute_batch_50_planes(lib):
    """SPEC acceptance #4: execute_batch over N=50 planes -> one execution visiting 50*w*h points."""
    rng = np.random.default_rng(1)
    srcs = [lib.plane_from_numpy(rng.integers(0, 256, (12, 10), dtype=np.uint8)) for _ in range(50)]
    dsts = [lib.plane_alloc(10, 12, U8) for _ in range(50)]
    rep = api.execute_batch([api.read(s, lib=lib) for s in srcs], [api.multiply(u8(3), lib=lib)],
                            [api.write(d, lib=lib) for d in dsts])
    assert rep.passes == 1 and rep.points_visited == 50 * 10 * 12
    for s, d in zip(srcs, dsts):
        assert np.array_equal(d.to_numpy(), (s.to_numpy().astype(np.uint32) * 3 % 256).astype(np.uint8))


def test_execute_batch_heterogeneous_counts(lib):
    a = lib.plane_alloc(4, 4, U8)
    with pytest.raises(OpfuseError) as e:
        api.execute_batch([api.read(a, lib=lib)], [], [])
    assert e.value.code == "HeterogeneousBatch"


def test_cast_handle(lib):
    """The facade's cast handle (absent from the reference api.hpp):
    u8x3 frame -> cvt -> cast f32x3 -> subtract, built from handles only."""
    if lib.name.startswith("reference"):
        pytest.skip("the reference facade has no cast handle; checked on the oracle")
    rng = np.random.default_rng(3)
    frame = lib.plane_from_numpy(rng.integers(0, 256, (20, 30, 3), dtype=np.uint8))
    out = [lib.plane_alloc(10, 8, F32) for _ in range(3)]
    handles = [api.resize(api.crop(frame, 2, 3, 20, 16, lib=lib), 10, 8, BILINEAR, lib=lib),
               api.cvt_color(SWAP_RB), api.cast(F32X3), api.subtract(f32x3(1, 2, 3), lib=lib),
               api.split(out, lib=lib)]
    p = api.build_pipeline(handles)
    assert p.n_compute == 1       # swap and cast folded into the read
    api.execute_operations(handles)
    ref = Library("oracle")
    want = [ref.plane_alloc(10, 8, F32) for _ in range(3)]
    src = ref.plane_from_numpy(frame.to_numpy())
    rd = ref.fold_unary_into_read(ref.fold_unary_into_read(
        ref.op_resize(ref.op_crop(src, 2, 3, 20, 16), 10, 8, BILINEAR), ref.op_color_convert(SWAP_RB, U8X3)),
        ref.op_cast(U8X3, F32X3))
    ref.execute_fused(ref.validate_chain([rd, ref.op_sub(f32x3(1, 2, 3)), ref.op_split_write(want)]))
    for a, b in zip(out, want):
        assert np.array_equal(a.to_numpy(), b.to_numpy())
    with pytest.raises(OpfuseError) as e:
        api.build_pipeline([api.cast(F32), api.write(out[0], lib=lib)])
    assert e.value.provenance == "cast"
