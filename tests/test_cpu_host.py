"""CPU-only checks: host-side API mirror (params, quadrature, ordering logic)
against the reference's golden vectors, and the C ABI library loading with
every symbol include/feast_b200.h declares (no compute without a GPU)."""

import os
import re

import numpy as np
import pytest

import paper_1203_4031_b200 as fb
from paper_1203_4031_b200 import _lib
from paper_1203_4031_b200.kernel import _ordering, filter_sort_flag, random_uniform, trace_error

from conftest import ROOT


def test_feastinit_defaults():
    f = fb.feastinit()
    assert [f.slot(i) for i in (1, 2, 3, 4, 5, 6, 7, 14)] == [0, 8, 12, 20, 0, 0, 5, 0]
    assert fb.validate_params(f) == 0
    assert f[1] == 8 and len(f) == 64


@pytest.mark.parametrize("slot,bad", [(1, 5), (2, 7), (3, 0), (4, -1), (5, 2), (6, 3), (7, 0), (14, 2)])
def test_validate_params_codes(slot, bad):
    f = fb.feastinit()
    f.set_slot(slot, bad)
    assert fb.validate_params(f) == 100 + slot


def test_check_problem_precedence():
    assert fb.check_problem(2, 2, -5.0, 5.0) == 0
    assert fb.check_problem(0, 1, 0.0, 1.0) == 202
    assert fb.check_problem(4, 9, 0.0, 1.0) == 201
    assert fb.check_problem(4, 2, 1.0, -1.0) == 200


def test_info_descriptions():
    assert fb.info_classification(0) == "success"
    assert fb.info_classification(3) == "warning"
    assert fb.info_classification(-2) == "error"
    assert "fpm(2)" in fb.info_description(102)
    assert "3-th argument" in fb.info_description(-103)


def test_fpm_coerce_from_foreign_object():
    class Foreign:
        def slot(self, i):
            return {2: 16}.get(i, 0)
    f = fb.FeastParams.coerce(Foreign())
    assert f.slot(2) == 16


@pytest.mark.parametrize("ne", fb.ALLOWED_CONTOUR_POINTS)
def test_quadrature_bitexact_vs_reference(unit_golden, ne):
    r = fb.gauss_legendre(ne)
    assert r.nodes.tobytes() == unit_golden[f"gl_nodes_{ne}"].tobytes()
    assert r.weights.tobytes() == unit_golden[f"gl_weights_{ne}"].tobytes()
    c = fb.build_contour(r, -0.7, 1.3)
    assert c.z.tobytes() == unit_golden[f"contour_z_{ne}"].tobytes()


def test_host_random_uniform_bitexact(unit_golden):
    for key in unit_golden.files:
        if key.startswith("rng_"):
            _, seed, off, cnt = key.split("_")
            assert random_uniform(int(seed), int(off), int(cnt)).tobytes() == unit_golden[key].tobytes()


def test_trace_error_golden():
    assert trace_error(4.0, np.nextafter(4.0, 5.0), -5.0, 5.0) == pytest.approx(1.776356839400251e-16, rel=1e-12)


def test_filter_sort_flag_cases():
    e = np.array([1.0, 2.0, 9.0])
    x = np.array([[10.0, 20.0, 90.0]])
    res = np.array([1e-12, -1.0, 1e-11])
    assert filter_sort_flag(e, x, res, 0.0, 5.0) == 1
    assert np.array_equal(e, [1.0, 9.0, 2.0]) and res[2] == -1.0
    e = np.array([1.0, 2.0])
    res = np.array([np.inf, 1e-12])
    order, m, nsp = _ordering(e, res, 0.0, 5.0)
    assert m == 1 and nsp == 1 and list(order) == [1, 0]


def test_library_exports_every_header_symbol():
    hdr = open(os.path.join(ROOT, "include", "feast_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|int64_t|size_t|const char\*)\s+(fb_\w+)\(", hdr, re.M))
    assert len(declared) >= 20
    lib = _lib.load()
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)
    assert lib.fb_abi_version() == 1
    assert lib.fb_zgetrf_dinv_doubles(64) >= 2 * 4 * 32 * 32


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.FeastB200Unavailable):
        fb.feast_sy(np.eye(4), 0.0, 2.0, 4)


def test_validation_errors_need_no_gpu():
    # argument checks happen before any device work (kernel.py:220-227)
    assert fb.SymmetricRci(0, 1, 0.0, 1.0).info == 202
    assert fb.SymmetricRci(4, 9, 0.0, 1.0).step() == fb.RciTask.DONE
    f = fb.feastinit()
    f.set_slot(2, 9)
    assert fb.SymmetricRci(4, 2, -1.0, 1.0, fpm=f).info == 102
