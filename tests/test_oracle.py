"""Pin the CPU oracle (oracle/sfc_oracle.c) before trusting it.

* against the committed golden fixtures produced by the reference itself
  (tests/golden/make_golden.py) -- runs everywhere;
* against the live compiled reference (oracle/_ref) on fresh seeded inputs when it
  was built (this container) -- bitwise equality of the fp64 output.
Mirrors proj/tests/test_quant.cpp / test_catalog.cpp known answers.
"""
import json
import os

import numpy as np
import pytest

from oracle import bindings as ob

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "qconv_cases.npz"))
VARIANTS = ["sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3"]
TAGS = sorted({k.split("/")[0] for k in GOLD.files if "/" in k and not k.startswith("kat")})
needs_ref = pytest.mark.skipif(not ob.ref_available(), reason="oracle/_ref not built (no /root/reference)")


def bits_equal(a, b):
    return np.array_equal(np.asarray(a, np.float64).view(np.int64), np.asarray(b, np.float64).view(np.int64))


# ------------------------------------------------------------------------------ specs
@pytest.mark.parametrize("name", VARIANTS)
def test_oracle_spec_matches_reference_export(name):
    cat = json.load(open(os.path.join(HERE, "golden", "catalog_3x3.json")))
    ref = next(a for a in cat["algorithms"] if a["name"] == name)
    s = ob.spec(name)
    assert s["N"] == ref["N"] and s["M"] == ref["tile"] and s["R"] == ref["kernel"]
    assert s["offset"] == ref["offset"] and s["a_denom"] == ref["denominator"]
    assert s["mults_full"] == ref["mults_full"] and s["mults_reduced"] == ref["mults_reduced"]
    for key in ("BT", "G", "A"):
        assert np.array_equal(s[key], np.array(ref[key], dtype=np.int64)), key
    assert s["n_corrections"] == len(ref["corrections"])


@pytest.mark.parametrize("name", VARIANTS)
def test_oracle_spec_is_exact(name):
    # sum_k A[k,t] BT[k,i] G[k,j] == a_denom [i == t + j] for every (t, i, j)
    assert ob.check_identity(name) == 0


@pytest.mark.parametrize("name", VARIANTS)
def test_execute_tile_matches_direct_correlation(name):
    # catalog.cpp:410-450 gate; test_catalog.cpp:189-206 (large values)
    s = ob.spec(name)
    rng = np.random.default_rng(77)
    n, R, M = s["n"], s["R"], s["M"]
    for trial in range(40):
        hi = 2000 if trial % 2 else 8
        x = rng.integers(-hi, hi + 1, size=(n, n))
        f = rng.integers(-hi, hi + 1, size=(R, R))
        want = np.array([[np.sum(x[i:i + R, j:j + R] * f) for j in range(M)] for i in range(M)])
        assert np.array_equal(ob.execute_tile(name, x, f), want)


# ------------------------------------------------------------------------------ scalar KATs
def test_quantize_value_known_answers():
    ins, outs = GOLD["kat/quantize_in"], GOLD["kat/quantize_out"]
    for (v, s, b), (q, sat) in zip(ins, outs):
        assert ob.quantize_value(v, s, int(b)) == (q, sat)
    # test_quant.cpp:34-58
    assert ob.quantize_value(2.5, 1.0, 8)[0] == 2
    assert ob.quantize_value(3.5, 1.0, 8)[0] == 4
    assert ob.quantize_value(-2.5, 1.0, 8)[0] == -2
    assert ob.quantize_value(0.26, 0.1, 8)[0] == 3
    assert ob.quantize_value(127.6, 1.0, 8) == (127, 1)
    assert ob.quantize_value(-130.0, 1.0, 8) == (-128, 1)
    assert ob.quantize_value(9.0, 1.0, 4) == (7, 1)


def test_scale_known_answers():
    g = GOLD["kat/scale_group"]
    got = [ob.scale_minmax([-3.0, 1.0, 2.0], 8), ob.scale_minmax([-3.0, 1.0, 2.0], 4), ob.scale_minmax(np.zeros(10), 8),
           ob.scale_minmax(g, 8), ob.scale_mse_grid(g, 8), ob.scale_mse_grid(g, 4)]
    assert bits_equal(got, GOLD["kat/scale_out"])
    assert ob.scale_minmax(np.zeros(10), 8) == 1e-8


# ------------------------------------------------------------------------------ golden convs
@pytest.mark.parametrize("tag", TAGS)
@pytest.mark.parametrize("variant", VARIANTS)
def test_oracle_matches_reference_golden(tag, variant):
    x, w = GOLD[f"{tag}/x"], GOLD[f"{tag}/w"]
    pad, bits, asc, fsc, srch = (int(v) for v in GOLD[f"{tag}/meta"])
    r = ob.quantized_conv(x, w, variant, pad, bits, asc, fsc, srch, threads=2, want=("out",), report=True)
    assert bits_equal(r["out"], GOLD[f"{tag}/{variant}/out"])
    rep = GOLD[f"{tag}/{variant}/report"]
    assert r["report"]["saturations"] == rep[3]
    assert r["report"]["values_quantized"] == rep[4]
    assert r["report"]["mse"] == pytest.approx(rep[0], rel=1e-12, abs=0)
    assert r["report"]["snr_db"] == pytest.approx(rep[2], rel=1e-12)


@pytest.mark.parametrize("tag", TAGS)
def test_oracle_direct_conv_matches_reference_golden(tag):
    x, w = GOLD[f"{tag}/x"], GOLD[f"{tag}/w"]
    pad = int(GOLD[f"{tag}/meta"][0])
    assert bits_equal(ob.direct_conv(x, w, pad), GOLD[f"{tag}/direct"])


def test_oracle_y_int_consistent_with_output():
    # per-oc-uniform scales: y_int = llround(out * N^2 / (sa * sf[oc]))
    x, w = GOLD["small_p1/x"], GOLD["small_p1/w"]
    for v in VARIANTS:
        r = ob.quantized_conv(x, w, v, 1, want=("out", "y_int", "pacc"))
        d2 = r["spec"]["a_denom"] ** 2
        rec = np.rint(r["out"] * d2 / (r["act_scale"][0] * r["fil_scale"][None, :, None, None]))
        assert np.array_equal(rec.astype(np.int64), r["y_int"])


def test_values_quantized_formula():
    # test_quant.cpp:121-124: OC*IC*K^2 + tiles*C*K^2
    x, w = GOLD["ragged_p1/x"], GOLD["ragged_p1/w"]
    for v in VARIANTS:
        r = ob.quantized_conv(x, w, v, 1, want=())
        K = r["spec"]["K"]
        assert r["report"]["values_quantized"] == w.shape[0] * w.shape[1] * K * K + r["report"]["tiles"] * x.shape[1] * K * K
        assert r["report"]["saturations"] == 0


def test_thread_count_independence():
    x, w = GOLD["small_p1/x"], GOLD["small_p1/w"]
    a = ob.quantized_conv(x, w, "sfc6-6x6-3x3", 1, threads=1, want=("out", "y_int"))
    b = ob.quantized_conv(x, w, "sfc6-6x6-3x3", 1, threads=5, want=("out", "y_int"))
    assert bits_equal(a["out"], b["out"]) and np.array_equal(a["y_int"], b["y_int"])


def test_invalid_bits_raise():
    x = np.zeros((1, 1, 8, 8), np.int8)
    w = np.zeros((1, 1, 3, 3), np.int8)
    for bits in (1, 17):
        with pytest.raises(ValueError):
            ob.quantized_conv(x, w, "sfc4-4x4-3x3", 1, bits)


# ------------------------------------------------------------------------------ live reference
@needs_ref
@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_bitwise_vs_live_reference(variant, seed):
    rng = np.random.default_rng(seed)
    B, C, OC = int(rng.integers(1, 3)), int(rng.integers(1, 12)), int(rng.integers(1, 9))
    H, W = int(rng.integers(3, 20)), int(rng.integers(3, 20))
    pad = int(rng.integers(0, 3))
    if H + 2 * pad < 3 or W + 2 * pad < 3:
        pad = 1
    lo = -128 if seed % 2 else 0
    x = rng.integers(lo, 128, size=(B, C, H, W), dtype=np.int8)
    w = rng.integers(-127, 128, size=(OC, C, 3, 3), dtype=np.int8)
    bits = int(rng.integers(2, 17))
    out, rep = ob.ref_quantized_fast_conv2d(x, w, variant, pad, bits)
    r = ob.quantized_conv(x, w, variant, pad, bits, want=("out",), report=True)
    assert bits_equal(r["out"], out)
    assert r["report"]["saturations"] == rep["saturations"]
    assert r["report"]["values_quantized"] == rep["values_quantized"]


@needs_ref
def test_oracle_bitwise_vs_live_reference_config1():
    from paper_2407_02913_b200 import workloads as wl
    L = wl.WORKLOADS[1].layers[0]
    x, w = wl.activations(1, 0, L), wl.weights(1, 0, L)
    out, rep = ob.ref_quantized_fast_conv2d(x, w, "sfc6-6x6-3x3", 1)
    r = ob.quantized_conv(x, w, "sfc6-6x6-3x3", 1, want=("out",), report=True)
    assert bits_equal(r["out"], out)
    assert r["report"]["mse"] == rep["mse"] and r["report"]["snr_db"] == rep["snr_db"]


@needs_ref
def test_frequency_energy_reference_dc():
    # test_quant.cpp:97-107: constant input, padding 0 -> DC energy 36^2, every other bin 0
    e = ob.ref_frequency_energy(np.ones((1, 1, 14, 14)), "sfc6-6x6-3x3", 0)
    assert e[0] == 1296.0 and np.all(e[1:] == 0.0)


# ------------------------------------------------------------------------------ 5x5 / 7x7 variants
LARGE_R = ["sfc6-6x6-5x5", "sfc6-4x4-7x7"]  # catalog.cpp:249-250
GOLD_R = np.load(os.path.join(HERE, "golden", "qconv_large_r.npz"))
TAGS_R = sorted({k.split("/")[0] for k in GOLD_R.files})


@pytest.mark.parametrize("name", LARGE_R)
def test_oracle_large_r_spec_matches_reference_export(name):
    cat = json.load(open(os.path.join(HERE, "golden", "catalog_large_r.json")))
    ref = next(a for a in cat["algorithms"] if a["name"] == name)
    s = ob.spec(name)
    assert s["N"] == ref["N"] and s["M"] == ref["tile"] and s["R"] == ref["kernel"]
    assert s["offset"] == ref["offset"] and s["a_denom"] == ref["denominator"]
    assert s["mults_full"] == ref["mults_full"] and s["mults_reduced"] == ref["mults_reduced"]
    for key in ("BT", "G", "A"):
        assert np.array_equal(s[key], np.array(ref[key], dtype=np.int64)), key
    assert s["n_corrections"] == len(ref["corrections"])
    assert ob.check_identity(name) == 0


@pytest.mark.parametrize("name", LARGE_R)
def test_oracle_large_r_execute_tile(name):
    s = ob.spec(name)
    rng = np.random.default_rng(78)
    n, R, M = s["n"], s["R"], s["M"]
    for trial in range(20):
        hi = 2000 if trial % 2 else 8
        x = rng.integers(-hi, hi + 1, size=(n, n))
        f = rng.integers(-hi, hi + 1, size=(R, R))
        want = np.array([[np.sum(x[i:i + R, j:j + R] * f) for j in range(M)] for i in range(M)])
        assert np.array_equal(ob.execute_tile(name, x, f), want)


@pytest.mark.parametrize("variant", LARGE_R)
@pytest.mark.parametrize("tag", TAGS_R)
def test_oracle_large_r_matches_reference_golden(tag, variant):
    x, (pad, bits) = GOLD_R[f"{tag}/x"], GOLD_R[f"{tag}/meta"]
    w = GOLD_R[f"{tag}/{variant}/w"]
    r = ob.quantized_conv(x, w, variant, int(pad), int(bits), want=("out",), report=True)
    assert bits_equal(r["out"], GOLD_R[f"{tag}/{variant}/out"])
    rep = GOLD_R[f"{tag}/{variant}/report"]
    assert r["report"]["saturations"] == rep[3] and r["report"]["values_quantized"] == rep[4]
    assert np.array_equal(ob.direct_conv(x, w, int(pad)), GOLD_R[f"{tag}/{variant}/direct"])


@needs_ref
@pytest.mark.parametrize("variant", LARGE_R)
@pytest.mark.parametrize("seed", [4, 5])
def test_oracle_large_r_bitwise_vs_live_reference(variant, seed):
    rng = np.random.default_rng(seed)
    R = ob.spec(variant)["R"]
    B, C, OC = 1, int(rng.integers(1, 6)), int(rng.integers(1, 5))
    H, W = int(rng.integers(R, 18)), int(rng.integers(R, 18))
    pad = int(rng.integers(0, R))
    x = rng.integers(-128, 128, size=(B, C, H, W), dtype=np.int8)
    w = rng.integers(-127, 128, size=(OC, C, R, R), dtype=np.int8)
    out, rep = ob.ref_quantized_fast_conv2d(x, w, variant, pad, 8)
    r = ob.quantized_conv(x, w, variant, pad, 8, want=("out",), report=True)
    assert bits_equal(r["out"], out)
    assert r["report"]["values_quantized"] == rep["values_quantized"]
