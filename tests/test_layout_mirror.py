"""Layout mirror: PhysiCell's vector-of-vectors density
(NestedDensity, mesh.hpp:93-100) <-> the flat voxel-major layout the
kernels use (translate_vector_to_array / translate_array_to_vector,
mesh.cpp:101-136) and DensityField::all_finite (mesh.cpp:95-99). The host
translation is checked against the reference's own functions (oracle/_ref)
on CPU; the device upload/download of nested fields on the GPU."""
import ctypes

import numpy as np
import pytest

import paper_2110_13368_b200 as B
from oracle import RefError, ref_lib, reference_available
from paper_2110_13368_b200 import workloads as W
from tests.helpers import bits_equal, make_session

_d = ctypes.c_double


def _ref_translate(nested):
    arrs = [np.ascontiguousarray(np.asarray(v, dtype=np.float64)) for v in nested]
    ptrs = (ctypes.POINTER(_d) * max(1, len(arrs)))(*[a.ctypes.data_as(ctypes.POINTER(_d)) for a in arrs])
    counts = np.array([a.size for a in arrs] or [0], dtype=np.int64)
    S = ctypes.c_int()
    L = ref_lib()
    cp = counts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))
    rc = L.ref_translate_vector_to_array(ptrs, cp, len(arrs), None, ctypes.byref(S))
    if rc:
        raise RefError(rc, L.ref_last_error().decode())
    out = np.empty(len(arrs) * S.value)
    rc = L.ref_translate_vector_to_array(ptrs, cp, len(arrs), out.ctypes.data_as(ctypes.POINTER(_d)),
                                         ctypes.byref(S))
    assert rc == 0
    return out, S.value


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("nvox,S", [(0, 0), (1, 1), (7, 3), (1000, 4)])
def test_translate_matches_reference(nvox, S):
    rng = np.random.default_rng(nvox + S)
    nested = [rng.standard_normal(S) * 10.0 ** rng.integers(-300, 300) for _ in range(nvox)]
    got = B.translate_vector_to_array(nested)
    want = _ref_translate(nested)
    assert got[1] == want[1] and bits_equal(got[0], want[0])
    if nvox:  # translate_array_to_vector inverts it (the reference's round trip)
        back = np.empty(got[0].size)
        L = ref_lib()
        assert L.ref_translate_round_trip(got[0].ctypes.data_as(ctypes.POINTER(_d)), got[0].size, S,
                                          back.ctypes.data_as(ctypes.POINTER(_d))) == 0
        assert bits_equal(back, got[0])


@pytest.mark.skipif(not reference_available(), reason="oracle/_ref not built")
def test_ragged_error_matches_reference():
    nested = [np.ones(3), np.ones(3), np.ones(2), np.ones(3)]
    with pytest.raises(RefError) as er:
        _ref_translate(nested)
    with pytest.raises(B.StateError) as eg:  # std::invalid_argument -> status 2
        B.translate_vector_to_array(nested)
    assert er.value.code == 2 and str(eg.value) == str(er.value)[len("[2] "):]
    assert "ragged nested density: voxel 2 holds 2 substrates, expected 3" in str(eg.value)


@pytest.mark.gpu
def test_nested_upload_download_and_all_finite():
    if B.device_count() == 0:
        pytest.fail("no sm_100 device visible")
    w = W.make("t", (20, 16, 12), 3, 100, 1, seed=4)
    a = make_session(w)
    b = make_session(w)
    rng = np.random.default_rng(2)
    flat = rng.random(w.voxels * w.S) * 40
    nested = [flat[v * w.S:(v + 1) * w.S] for v in range(w.voxels)]
    a.upload_field(flat)
    b.upload_field_nested(nested)
    a.advance(11, w.dt)
    b.advance(11, w.dt)
    got = b.download_field_nested()
    assert len(got) == w.voxels and all(g.size == w.S for g in got)
    assert bits_equal(np.concatenate(got), a.download_field())
    assert b.all_finite()
    flat[5] = np.nan
    b.upload_field(flat)
    assert not b.all_finite()
    flat[5] = np.inf
    b.upload_field(flat)
    assert not b.all_finite()
    bad = list(nested)
    bad[3] = np.ones(w.S + 1)
    with pytest.raises(B.StateError, match="ragged nested density: voxel 3"):
        b.upload_field_nested(bad)
    a.close()
    b.close()
