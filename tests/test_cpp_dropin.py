"""The C++ sfconv:: drop-in (include/sfconv/*.hpp over libsfc_b200.so), exercised by a C++
program written against the reference's own API (tests/cpp/test_dropin.cpp)."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import bindings as ob

HERE = os.path.dirname(os.path.abspath(__file__))
BIN = os.path.join(HERE, "cpp", "test_dropin")


def _build():
    subprocess.run(["make", "-s", "-C", os.path.join(HERE, "cpp")], check=True)


def test_dropin_host_side():
    """Catalog, exact tile execution, validation gate and scalar quantizer KATs (no GPU needed)."""
    _build()
    r = subprocess.run([BIN, "--host-only"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout


@pytest.mark.gpu
def test_dropin_full_suite(cuda):
    _build()
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[SKIP]" not in r.stdout and "[FAIL]" not in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3"])
@pytest.mark.parametrize("shape", [(2, 5, 13, 11, 7, 1, 8), (1, 64, 28, 28, 32, 1, 8), (1, 9, 10, 12, 4, 0, 5)])
def test_dropin_quantized_fast_conv2d_matches_oracle(cuda, variant, shape):
    """quantized_fast_conv2d through the C++ API vs the oracle: fp64 output within 1e-6 (the
    dequantisation runs in fp64 on the device from the bit-exact integer accumulator), the
    report and the counters."""
    _build()
    B, C, H, W, OC, pad, bits = shape
    rng = np.random.default_rng(sum(shape))
    x = rng.integers(-128, 128, size=(B, C, H, W), dtype=np.int8)
    w = rng.integers(-127, 128, size=(OC, C, 3, 3), dtype=np.int8)
    with tempfile.TemporaryDirectory() as d:
        xp, wp, op = (os.path.join(d, n) for n in ("x.bin", "w.bin", "o.bin"))
        x.tofile(xp)
        w.tofile(wp)
        r = subprocess.run([BIN, "run", variant, str(pad), str(bits), str(B), str(C), str(H), str(W), str(OC), xp, wp,
                            op], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        raw = np.fromfile(op, np.float64)
    HO, WO = H + 2 * pad - 2, W + 2 * pad - 2
    out, tail = raw[:-5].reshape(B, OC, HO, WO), raw[-5:]
    ref = ob.quantized_conv(x, w, variant, pad, bits, want=("out",), report=True)
    err = np.abs(out - ref["out"]).max() / np.abs(ref["out"]).max()
    assert err <= 1e-12   # fp64 from the exact y_int: only the last-bit rounding differs
    assert tail[0] == pytest.approx(ref["report"]["mse"], rel=1e-9)
    assert tail[2] == pytest.approx(ref["report"]["snr_db"], rel=1e-9)
    assert tail[3] == ref["report"]["saturations"] and tail[4] == ref["report"]["values_quantized"]


@pytest.mark.gpu
@pytest.mark.parametrize("variant,cfg", [("sfc6-6x6-3x3", (1, 2, 0)), ("sfc4-4x4-3x3", (0, 0, 1)),
                                         ("sfc6-6x6-5x5", (0, 0, 0)), ("sfc6-4x4-7x7", (1, 1, 1))])
def test_dropin_quant_config_and_large_filters(cuda, variant, cfg):
    """The full QuantConfig (per-frequency scopes, MseGrid) and the 5x5 / 7x7 algorithms through
    the C++ API: fp64 output vs the oracle (<= 1e-12 relative), counters equal."""
    _build()
    R = ob.spec(variant)["R"]
    B, C, H, W, OC, pad, bits = 1, 6, 14, 13, 5, R // 2, 8
    rng = np.random.default_rng(R * 7 + sum(cfg))
    x = rng.integers(-128, 128, size=(B, C, H, W), dtype=np.int8)
    w = rng.integers(-127, 128, size=(OC, C, R, R), dtype=np.int8)
    with tempfile.TemporaryDirectory() as d:
        xp, wp, op = (os.path.join(d, n) for n in ("x.bin", "w.bin", "o.bin"))
        x.tofile(xp)
        w.tofile(wp)
        r = subprocess.run([BIN, "run", variant, str(pad), str(bits), str(B), str(C), str(H), str(W), str(OC),
                            *(str(v) for v in cfg), xp, wp, op], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr
        raw = np.fromfile(op, np.float64)
    HO, WO = H + 2 * pad - R + 1, W + 2 * pad - R + 1
    out, tail = raw[:-5].reshape(B, OC, HO, WO), raw[-5:]
    ref = ob.quantized_conv(x, w, variant, pad, bits, *cfg, want=("out",), report=True)
    assert np.abs(out - ref["out"]).max() / np.abs(ref["out"]).max() <= 1e-12
    assert tail[3] == ref["report"]["saturations"] and tail[4] == ref["report"]["values_quantized"]


@pytest.mark.gpu
@pytest.mark.parametrize("variant,cfg", [("sfc6-6x6-3x3", (0, 0, 0)), ("sfc6-7x7-3x3", (1, 2, 1)),
                                         ("sfc6-4x4-7x7", (0, 1, 0))])
def test_dropin_real_valued_tensors(cuda, variant, cfg):
    """Real-valued DenseTensors through the C++ API (the reference's own use, e.g. quantsim's
    N(0,1) data): fp64 output vs the reference's golden output (<= 1e-12), counters equal."""
    _build()
    gold = np.load(os.path.join(HERE, "golden", "qconv_real.npz"))
    tag = {(0, 0, 0): "real_default", (1, 2, 1): None, (0, 1, 0): None}[cfg]
    R = ob.spec(variant)["R"]
    rng = np.random.default_rng(R + sum(cfg))
    if tag:
        x, w = gold[f"{tag}/x"], gold[f"{tag}/{variant}/w"]
        want, rep = gold[f"{tag}/{variant}/out"], gold[f"{tag}/{variant}/report"]
        bits, pad = 8, int(rep[5])
    else:
        x = rng.normal(size=(1, 4, 11, 12))
        w = rng.normal(size=(3, 4, R, R))
        bits, pad = 8, R // 2
        want = rep = None
    B, C, H, W = x.shape
    OC = w.shape[0]
    with tempfile.TemporaryDirectory() as d:
        xp, wp, op = (os.path.join(d, n) for n in ("x.bin", "w.bin", "o.bin"))
        np.ascontiguousarray(x, np.float64).tofile(xp)
        np.ascontiguousarray(w, np.float64).tofile(wp)
        r = subprocess.run([BIN, "run", variant, str(pad), str(bits), str(B), str(C), str(H), str(W), str(OC),
                            *(str(v) for v in cfg), xp, wp, op], capture_output=True, text=True, timeout=300,
                           env=dict(os.environ, SFC_TEST_F64="1"))
        assert r.returncode == 0, r.stderr
        raw = np.fromfile(op, np.float64)
    HO, WO = H + 2 * pad - R + 1, W + 2 * pad - R + 1
    out, tail = raw[:-5].reshape(B, OC, HO, WO), raw[-5:]
    if want is not None:
        assert np.abs(out - want).max() / np.abs(want).max() <= 1e-12
        assert tail[3] == rep[3] and tail[4] == rep[4]
    else:  # the Python mirror of the same real-valued path must agree bit for bit
        import torch
        from paper_2407_02913_b200 import sfconv as sc
        py = sc.quantized_fast_conv2d(torch.from_numpy(x), torch.from_numpy(w), sc.catalog_algorithm(variant), pad,
                                      sc.QuantConfig(bits, *cfg))
        assert np.array_equal(out, py.output.cpu().numpy())
