"""CPU tests of the product's host side: the plan layer behind the C-ABI and the library
exports.  No device calls (sfc_plan_* / sfc_catalog_json are host-only)."""
import ctypes
import json
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2407_02913_b200 as sfc
from paper_2407_02913_b200 import _lib

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CAT = json.load(open(os.path.join(HERE, "golden", "catalog_3x3.json")))
CAT_R = json.load(open(os.path.join(HERE, "golden", "catalog_large_r.json")))
VARIANTS = ["sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3", "sfc6-6x6-5x5", "sfc6-4x4-7x7"]


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "sfc_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(sfc_\w+)\s*\(", header, re.M))
    assert declared == set(_lib.EXPORTED)
    L = _lib.lib()
    for name in declared:
        assert getattr(L, name) is not None
    nm = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (sfc_\w+)", nm))
    assert declared <= exported


def test_catalog_json_matches_reference_export_text():
    js, h = sfc.catalog_export_json()
    mine = json.loads(js)["algorithms"]
    assert [a["name"] for a in mine] == VARIANTS
    exact = dict(CAT["exact_text"], **CAT_R["exact_text"])
    for a in mine:
        text = json.dumps(a, separators=(",", ":"))
        assert text == exact[a["name"]]      # byte-identical to the reference's export


def test_fnv_hash_of_export():
    js, h = sfc.catalog_export_json()
    x = 0xCBF29CE484222325
    for c in js.encode():
        x ^= c
        x = (x * 0x100000001B3) & 0xFFFFFFFFFFFFFFFF
    assert h == x


@pytest.mark.parametrize("name,K,full,reduced,pct", [("sfc4-4x4-3x3", 7, 49, 46, 31.94),
                                                      ("sfc6-6x6-3x3", 10, 100, 88, 27.16),
                                                      ("sfc6-7x7-3x3", 12, 144, 132, 29.93)])
def test_channel_and_product_counts(name, K, full, reduced, pct):
    # test_catalog.cpp:101-126
    s = sfc.catalog_algorithm(name)
    assert s.K == K and s.mults_full() == full and s.mults_reduced() == reduced
    assert s.complexity_pct() == pytest.approx(pct, rel=1e-3)


def test_correction_schedules():
    # test_catalog.cpp:128-144
    def corr(n):
        return [(c.out, c.desired, c.wrapped, c.tap) for c in sfc.catalog_algorithm(n).corrections]
    assert corr("sfc6-6x6-3x3") == [(0, 0, 6, 0), (5, 7, 1, 2)]
    assert corr("sfc4-4x4-3x3") == [(0, 0, 4, 0), (3, 5, 1, 2)]
    assert corr("sfc6-7x7-3x3") == [(0, 0, 6, 0), (6, 7, 1, 1), (5, 7, 1, 2), (6, 8, 2, 2)]


def test_sfc6_rows_documented_arrangement():
    # test_catalog.cpp:165-187
    s = sfc.catalog_algorithm("sfc6-6x6-3x3")
    assert s.offset == 1 and s.a_denom == 6
    bt = [[1, 1, 1, 1, 1, 1], [1, 1, 0, -1, -1, 0], [0, -1, -1, 0, 1, 1], [1, 0, -1, -1, 0, 1],
          [1, 0, -1, 1, 0, -1], [0, -1, 1, 0, -1, 1], [1, -1, 0, 1, -1, 0], [1, -1, 1, -1, 1, -1]]
    g = [[1, 1, 1], [0, 1, 1], [-1, -1, 0], [-1, 0, 1], [-1, 0, 1], [1, -1, 0], [0, -1, 1], [1, -1, 1]]
    assert np.array_equal(s.BT[:8, 1:7], bt) and np.all(s.BT[:8, 0] == 0) and np.all(s.BT[:8, 7] == 0)
    assert np.array_equal(s.G[:8], g)


@pytest.mark.parametrize("name", VARIANTS)
def test_triples_and_exact_identity(name):
    s = sfc.catalog_algorithm(name)
    K, n, M, R = s.K, s.n_in, s.M, s.R
    # exhaustive per-axis identity: sum_k A[k,t] BT[k,i] G[k,j] = a_denom [i == t + j]
    lhs = np.einsum("kt,ki,kj->tij", s.A, s.BT, s.G)
    rhs = np.zeros((M, n, R), np.int64)
    for t in range(M):
        for j in range(R):
            rhs[t, t + j, j] = s.a_denom
    assert np.array_equal(lhs, rhs)
    # Karatsuba sum rows (test_catalog.cpp:80-99)
    trip = {"sfc4-4x4-3x3": [(4, 3, 2)]}.get(name, [(1, 2, 3), (4, 5, 6)])
    for a, b, c in trip:
        assert np.array_equal(s.BT[c], s.BT[a] + s.BT[b]) and np.array_equal(s.G[c], s.G[a] + s.G[b])


def test_unknown_algorithm_raises_value_error():
    with pytest.raises(ValueError, match="unknown algorithm"):
        sfc.catalog_algorithm.__wrapped__("wino-4x4-3x3")


def test_error_codes_map_to_reference_exceptions():
    h = ctypes.c_void_p()
    rc = _lib.lib().sfc_plan_create(b"nope", ctypes.byref(h))
    assert rc == _lib.SFC_ERR_INVALID
    assert b"unknown algorithm: nope" == _lib.lib().sfc_last_error()
    with pytest.raises(_lib.SfcInvalidArgument):
        _lib.check(rc)


def test_scalar_helpers_match_reference_kats():
    g = np.load(os.path.join(HERE, "golden", "qconv_cases.npz"))
    for (v, s, b), (q, sat) in zip(g["kat/quantize_in"], g["kat/quantize_out"]):
        cnt = [0]
        assert sfc.quantize_value(v, s, int(b), cnt) == q and cnt[0] == sat
    grp = g["kat/scale_group"]
    got = [sfc.scale_minmax([-3.0, 1.0, 2.0], 8), sfc.scale_minmax([-3.0, 1.0, 2.0], 4),
           sfc.scale_minmax(np.zeros(10), 8), sfc.scale_minmax(grp, 8), sfc.scale_mse_grid(grp, 8),
           sfc.scale_mse_grid(grp, 4)]
    assert np.array_equal(np.array(got).view(np.int64), g["kat/scale_out"].view(np.int64))


def test_workload_seeds_are_deterministic():
    from paper_2407_02913_b200 import workloads as wl
    L = wl.WORKLOADS[2].layers[0]
    a, b = wl.activations(2, 0, L), wl.activations(2, 0, L)
    assert a.dtype == np.int8 and a.shape == (8, 128, 28, 28) and np.array_equal(a, b)
    assert a.min() >= 0 and a.max() <= 127
    w = wl.weights(2, 0, L)
    assert w.dtype == np.int8 and np.abs(w.astype(int)).max() == 127
    assert len(wl.WORKLOADS[3].layers) == 13 and len(wl.WORKLOADS[4].layers) == 13
    assert wl.direct_equivalent_ops(L) == 18 * 8 * 128 * 128 * 28 * 28
