"""GPU parity of the B200 path (libsfc_b200.so via the C-ABI) against the oracle and the
reference's golden fixtures.

Bar (BASELINE.json north_star): integer transform-domain values (vq, uq), per-frequency
contractions (pacc) and the output accumulator y_int bit-exact; the dequantised fp32
output within max|got - want| / max|want| <= 1e-6 (the reference's own error metric,
proj/tests/test_conv.cpp:47-55).
"""
import ctypes
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import bindings as ob  # noqa: E402
from paper_2407_02913_b200 import _lib, sfconv as sc, workloads as wl  # noqa: E402

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "qconv_cases.npz"))
VARIANTS = ["sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3"]
LARGE_R = ["sfc6-6x6-5x5", "sfc6-4x4-7x7"]  # catalog.cpp:249-250
TOL = 1e-6


def maxrel(got, want):
    want = np.asarray(want, np.float64)
    den = np.abs(want).max()
    return np.abs(np.asarray(got, np.float64) - want).max() / (den if den > 0 else 1.0)


def run_gpu(x, w, variant, pad=1, bits=8, outs=("y", "f32"), requant=0.0, vmax=None, views=True):
    dev = torch.device("cuda", 0)
    layer = sc.SfcLayer(variant, torch.from_numpy(w).to(dev), bits=bits)
    xt = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    B, C, H, W = x.shape
    R = w.shape[2]
    HO, WO = H + 2 * pad - R + 1, W + 2 * pad - R + 1
    ws = layer.workspace(B, H, W, pad)
    res = {}
    kw = {}
    if "y" in outs:
        kw["y_int32"] = res["y"] = torch.empty((B, w.shape[0], HO, WO), dtype=torch.int32, device=dev)
    if "f32" in outs:
        kw["out_f32"] = res["f32"] = torch.empty((B, w.shape[0], HO, WO), dtype=torch.float32, device=dev)
    if "i8" in outs:
        kw["out_i8"] = res["i8"] = torch.empty((B, w.shape[0], HO, WO), dtype=torch.int8, device=dev)
    if vmax is None:  # the product path: absmax keeps V, quantization fused into the GEMM
        layer.forward(xt, ws, pad, requant_scale=requant, **kw)
    else:
        vm = torch.tensor([vmax], dtype=torch.int32, device=dev)
        layer.conv(xt, vm, ws, pad, requant_scale=requant, **kw)
    torch.cuda.synchronize()
    out = {k: v.cpu().numpy() for k, v in res.items()}
    out["stats"] = layer.stats(B, H, W, pad, ws)
    out["sf"], out["umax"] = layer.filter_scales()
    if views:
        # forward never materialises vq: take it from the recompute path (absmax, then a
        # quantize pass that re-derives V from x) on its own workspace, whose y must match.
        _, pacc = layer.views(B, H, W, pad, ws)
        out["pacc"] = None if pacc is None else pacc.cpu().numpy()  # (Cin <= 4: fused dp4a, no P)
        ws2 = layer.workspace(B, H, W, pad)
        y2 = torch.empty_like(res["y"]) if "y" in res else None
        vm = torch.zeros(1, dtype=torch.int32, device=dev)
        if vmax is None:
            layer.absmax(xt, vm, pad)
        else:
            vm.fill_(vmax)
        layer.conv(xt, vm, ws2, pad, y_int32=y2)
        vq, pacc2 = layer.views(B, H, W, pad, ws2)
        out["vq"] = vq.cpu().numpy()
        if pacc2 is not None:
            assert np.array_equal(pacc2.cpu().numpy(), out["pacc"]), "pacc: recompute path vs product path"
        if y2 is not None:
            assert torch.equal(y2, res["y"]), "y: recompute path vs product path"
        out["uq"] = layer.uq().cpu().numpy()
    out["filter_sat"] = layer.filter_saturations()
    return out


def check_against_oracle(x, w, variant, pad=1, bits=8, intermediates=True):
    want = ("out", "y_int", "pacc", "vq", "uq") if intermediates else ("out", "y_int")
    r = ob.quantized_conv(x, w, variant, pad, bits, want=want)
    g = run_gpu(x, w, variant, pad, bits, views=intermediates)
    assert np.array_equal(g["sf"], r["fil_scale"]), "filter scales"
    assert g["stats"]["act_scale"] == r["act_scale"][0], "activation scale"
    if intermediates:
        assert np.array_equal(g["uq"], r["uq"].transpose(2, 0, 1)), "uq"
        assert np.array_equal(g["vq"], r["vq"].transpose(2, 0, 1)), "vq"
        if g["pacc"] is not None:
            assert np.array_equal(g["pacc"].astype(np.int64), r["pacc"].transpose(2, 0, 1)), "pacc"
    assert np.array_equal(g["y"].astype(np.int64), r["y_int"]), "y_int"
    assert maxrel(g["f32"], r["out"]) <= TOL
    assert g["stats"]["saturations"] + g["filter_sat"] == 0
    return g, r


# ------------------------------------------------------------------------------ small seeded cases
CASES = [  # (B, C, OC, H, W, pad, lo)
    (1, 8, 8, 14, 14, 1, -128),
    (2, 5, 3, 13, 11, 1, -128),
    (1, 3, 17, 9, 23, 0, 0),
    (3, 64, 64, 12, 12, 1, 0),
    (1, 65, 130, 10, 10, 2, -128),
    (2, 130, 33, 7, 7, 1, -128),
    (1, 17, 257, 6, 6, 1, -128),
    (1, 1, 1, 1, 1, 1, -128),
    (1, 2, 2, 3, 3, 0, -128),
    # wide rows (> 10 tiles, >= 64 channels): the row-chunk CTAs of the register transform
    (1, 64, 16, 9, 130, 1, -128),
    (2, 70, 8, 7, 100, 2, 0),
    (1, 128, 12, 13, 71, 0, -128),
]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("case", CASES, ids=[f"b{c[0]}c{c[1]}o{c[2]}h{c[3]}w{c[4]}p{c[5]}" for c in CASES])
def test_small_cases_bit_exact(cuda, variant, case):
    B, C, OC, H, W, pad, lo = case
    rng = np.random.default_rng(hash(case) & 0xFFFF)
    x = rng.integers(lo, 128, size=(B, C, H, W), dtype=np.int8)
    w = rng.integers(-127, 128, size=(OC, C, 3, 3), dtype=np.int8)
    check_against_oracle(x, w, variant, pad)


SWAR_CASES = [  # (B, C, OC, H, W, pad): odd / small / non-multiple-of-64 channel counts, border tiles
    (2, 5, 3, 13, 11, 1), (1, 64, 8, 14, 14, 1), (3, 130, 9, 9, 17, 0), (1, 1, 2, 7, 7, 1), (2, 67, 16, 20, 6, 2),
    (1, 128, 32, 29, 31, 1),
]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("case", SWAR_CASES, ids=[f"b{c[0]}c{c[1]}o{c[2]}h{c[3]}w{c[4]}p{c[5]}" for c in SWAR_CASES])
def test_swar_absmax_kernel_bit_exact(cuda, variant, case, monkeypatch):
    """The two-channel SWAR absmax / keep-V kernel (k_act_pair, used for large layers) forced on
    small ragged cases: vmax, vq, uq, pacc and y_int bit-exact against the oracle."""
    monkeypatch.setenv("SFC_ACT_PAIR", "1")
    B, C, OC, H, W, pad = case
    rng = np.random.default_rng(sum(case) + len(variant))
    x = rng.integers(-128, 128, size=(B, C, H, W), dtype=np.int8)
    w = rng.integers(-127, 128, size=(OC, C, 3, 3), dtype=np.int8)
    g, r = check_against_oracle(x, w, variant, pad)
    assert g["stats"]["vmax"] == r["report"]["vmax"]


@pytest.mark.parametrize("qfuse", ["0", "1"])
def test_padding_channels_never_count_as_saturations(cuda, qfuse, monkeypatch):
    """Kept-V channels past C are not defined (the workspace is reused, not cleared): the
    quantizers zero them before quantizing, so with the exact-fallback quantizer (bits 5 here:
    no proven multiplier) a workspace full of garbage still reports 0 saturations and the
    oracle's y."""
    monkeypatch.setenv("SFC_QFUSE", qfuse)
    rng = np.random.default_rng(5)
    x = rng.integers(-128, 128, size=(2, 9, 15, 13), dtype=np.int8)
    w = rng.integers(-127, 128, size=(6, 9, 3, 3), dtype=np.int8)
    layer = sc.SfcLayer("sfc6-6x6-3x3", torch.from_numpy(w).cuda(), 5)
    ws = layer.workspace(2, 15, 13, 1)
    ws.fill_(0x7F)
    y = torch.empty((2, 6, 15, 13), dtype=torch.int32, device="cuda")
    layer.forward(torch.from_numpy(x).cuda(), ws, 1, y_int32=y)
    st = layer.stats(2, 15, 13, 1, ws)
    assert not st["fast_quantizer_exact"] and st["saturations"] == 0
    assert np.array_equal(y.cpu().numpy().astype(np.int64), ob.quantized_conv(x, w, "sfc6-6x6-3x3", 1, 5)["y_int"])


@pytest.mark.parametrize("bits", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("variant", VARIANTS)
def test_bit_widths(cuda, variant, bits):
    rng = np.random.default_rng(bits)
    x = rng.integers(-128, 128, size=(2, 9, 15, 13), dtype=np.int8)
    w = rng.integers(-127, 128, size=(6, 9, 3, 3), dtype=np.int8)
    check_against_oracle(x, w, variant, 1, bits)


WIDE_CASES = [  # (bits, act_scope, filter_scope, search)
    (9, 0, 0, 0), (10, 0, 0, 0), (12, 0, 0, 0), (13, 1, 0, 0), (14, 0, 2, 0), (15, 0, 1, 1), (16, 0, 0, 0),
    (16, 1, 2, 1),
]


@pytest.mark.parametrize("variant", VARIANTS + LARGE_R)
@pytest.mark.parametrize("wide", WIDE_CASES, ids=[f"b{c[0]}a{c[1]}f{c[2]}s{c[3]}" for c in WIDE_CASES])
def test_wide_bit_widths(cuda, variant, wide):
    """bits 9-16 (quant.cpp:155-156 accepts 2..16): integer-valued fp64 operands contracted by an
    exact fp64 GEMM (|P| <= C * 2^30 < 2^53), then the reference-order fp64 epilogue.  Output
    vs the oracle (fp32 output of the int8 API; the fp64 output through the report's mse at
    1e-9), scales and counters exactly."""
    bits, asc, fsc, srch = wide
    R = sc.catalog_algorithm(variant).R
    rng = np.random.default_rng(bits * 7 + asc + 3 * fsc + 11 * srch)
    x = rng.integers(-128, 128, size=(2, 7, 13, 11), dtype=np.int8)
    w = rng.integers(-127, 128, size=(5, 7, R, R), dtype=np.int8)
    pad = R // 2
    r = ob.quantized_conv(x, w, variant, pad, bits, asc, fsc, srch, want=("out",), report=True)
    rep = sc.quantized_fast_conv2d(torch.from_numpy(x), torch.from_numpy(w), sc.catalog_algorithm(variant), pad,
                                   sc.QuantConfig(bits, asc, fsc, srch))
    assert rep.y_int is None
    assert maxrel(rep.output.cpu().numpy(), r["out"]) <= TOL  # fp32 output; the fp64 one is pinned via mse
    assert np.array_equal(np.atleast_1d(rep.act_scale), r["act_scale"][: np.atleast_1d(rep.act_scale).size])
    assert rep.saturations == r["report"]["saturations"]
    assert rep.values_quantized == r["report"]["values_quantized"]
    assert rep.mse == pytest.approx(r["report"]["mse"], rel=1e-9)


# ------------------------------------------------------------------------------ golden fixtures
GOLD_TAGS = sorted({k.split("/")[0] for k in GOLD.files if k.endswith("/meta")})


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("tag", GOLD_TAGS)
def test_golden_reference_outputs(cuda, tag, variant):
    pad, bits, asc, fsc, srch = (int(v) for v in GOLD[f"{tag}/meta"])
    x, w = GOLD[f"{tag}/x"], GOLD[f"{tag}/w"]
    if asc or fsc or srch or bits > 8:  # the general QuantConfig / wide path (fp64 epilogue, no y_int)
        rep = sc.quantized_fast_conv2d(torch.from_numpy(x), torch.from_numpy(w), sc.catalog_algorithm(variant), pad,
                                       sc.QuantConfig(bits, asc, fsc, srch))
        assert maxrel(rep.output.cpu().numpy(), GOLD[f"{tag}/{variant}/out"]) <= TOL
        r = GOLD[f"{tag}/{variant}/report"]
        assert rep.saturations == r[3] and rep.values_quantized == r[4]
        assert rep.mse == pytest.approx(r[0], rel=1e-6) and rep.snr_db == pytest.approx(r[2], rel=1e-6)
        return
    ref = GOLD[f"{tag}/{variant}/out"]
    g = run_gpu(x, w, variant, pad, bits)
    assert maxrel(g["f32"], ref) <= TOL
    d2 = sc.catalog_algorithm(variant).a_denom ** 2
    rec = np.rint(ref * d2 / (g["stats"]["act_scale"] * g["sf"][None, :, None, None])).astype(np.int64)
    assert np.array_equal(rec, g["y"].astype(np.int64))


@pytest.mark.parametrize("variant", VARIANTS)
def test_golden_report_via_public_api(cuda, variant):
    tag = "small_p1"
    x, w = GOLD[f"{tag}/x"], GOLD[f"{tag}/w"]
    rep_ref = GOLD[f"{tag}/{variant}/report"]
    rep = sc.quantized_fast_conv2d(torch.from_numpy(x), torch.from_numpy(w), sc.catalog_algorithm(variant), 1)
    assert rep.mse == pytest.approx(rep_ref[0], rel=1e-9)
    assert rep.signal_energy == pytest.approx(rep_ref[1], rel=1e-12)
    assert rep.snr_db == pytest.approx(rep_ref[2], rel=1e-9)
    assert rep.saturations == rep_ref[3] and rep.values_quantized == rep_ref[4]
    assert maxrel(rep.output.cpu().numpy(), GOLD[f"{tag}/{variant}/out"]) <= TOL
    # the rest of the reference API on the device
    u = sc.transform_filters(torch.from_numpy(w), sc.catalog_algorithm(variant)).cpu().numpy()
    assert np.array_equal(u, GOLD[f"{tag}/{variant}/u"])
    e = sc.frequency_energy(torch.from_numpy(GOLD[f"{tag}/{variant}/energy_x"]), sc.catalog_algorithm(variant), 1)
    assert np.array_equal(e, GOLD[f"{tag}/{variant}/energy"])


def test_golden_direct_conv(cuda):
    for tag in GOLD_TAGS:
        x, w = GOLD[f"{tag}/x"], GOLD[f"{tag}/w"]
        pad = int(GOLD[f"{tag}/meta"][0])
        got = sc.direct_conv2d(torch.from_numpy(x), torch.from_numpy(w), 1, pad).cpu().numpy()
        assert np.array_equal(got, GOLD[f"{tag}/direct"])


def test_frequency_energy_dc(cuda):
    # test_quant.cpp:97-107
    e = sc.frequency_energy(torch.ones((1, 1, 14, 14), dtype=torch.int8), sc.catalog_algorithm("sfc6-6x6-3x3"), 0)
    assert e[0] == 1296.0 and np.all(e[1:] == 0.0)


# ------------------------------------------------------------------------------ BASELINE configs
@pytest.mark.parametrize("variant", ["sfc6-6x6-3x3"])
def test_config1_bit_exact(cuda, variant):
    L = wl.WORKLOADS[1].layers[0]
    check_against_oracle(wl.activations(1, 0, L), wl.weights(1, 0, L), variant)


@pytest.mark.parametrize("variant", VARIANTS)
def test_config2_bit_exact(cuda, variant):
    L = wl.WORKLOADS[2].layers[0]
    check_against_oracle(wl.activations(2, 0, L), wl.weights(2, 0, L), variant)


@pytest.mark.slow
def test_config5_bit_exact(cuda):
    L = wl.WORKLOADS[5].layers[0]
    x, w = wl.activations(5, 0, L), wl.weights(5, 0, L)
    check_against_oracle(x, w, "sfc6-6x6-3x3", intermediates=False)


@pytest.mark.parametrize("cfg,idx", [(3, 0), (3, 4), (3, 7), (3, 10), (4, 0), (4, 2), (4, 8), (4, 12)])
def test_stack_layers_shard_properties(cuda, cfg, idx):
    """Full-size ResNet-18 / VGG-16 layers: the GPU global absmax equals the oracle's, and a
    2-image shard of the full-batch output (y_int and harness int8 requant) is bit-exact against
    the oracle run on those images with the full-batch scale (size-independent check)."""
    work = wl.WORKLOADS[cfg]
    L = work.layers[idx]
    x, w = wl.activations(cfg, idx, L), wl.weights(cfg, idx, L)
    s_l = float(wl.requant_scales(cfg, len(work.layers))[idx])
    g = run_gpu(x, w, "sfc6-6x6-3x3", L.pad, outs=("y", "i8"), requant=s_l, views=False)
    full = ob.quantized_conv(x, w, "sfc6-6x6-3x3", L.pad, want=())
    assert g["stats"]["vmax"] == full["report"]["vmax"]
    pick = np.random.default_rng(idx).choice(L.batch, size=2, replace=False)
    part = ob.quantized_conv(x[pick], w, "sfc6-6x6-3x3", L.pad, want=("y_int",), vmax_override=full["report"]["vmax"])
    assert np.array_equal(g["y"][pick].astype(np.int64), part["y_int"])
    # harness requant: clamp(rint(y * (sa * sf / 36) * s), 0, 127) in fp64
    scale = (g["stats"]["act_scale"] * g["sf"]) / 36.0
    want8 = np.clip(np.rint(g["y"].astype(np.float64) * scale[None, :, None, None] * s_l), 0, 127).astype(np.int8)
    assert np.array_equal(g["i8"], want8)


# ------------------------------------------------------------------------------ quantizer exactness
@pytest.mark.parametrize("bits", [2, 4, 8])
def test_device_quantizer_exhaustive(cuda, bits):
    """Every integer v in [-vmax, vmax] for many vmax (incl. tie-prone multiples of 127 and 254):
    device q(v) == rint(v / sa) with sa = max(vmax / qmax, 1e-8) in fp64 (quant.cpp:102-120)."""
    qmax = (1 << (bits - 1)) - 1
    vmaxes = sorted(set(list(range(0, 300)) + list(range(300, 4609, 37)) + [127 * k for k in range(1, 37)] +
                        [254 * k for k in range(1, 19)] + [1020, 2040, 2041, 3084, 3164, 4064, 4572, 4607, 4608]))
    n_fast = 0
    for vmax in vmaxes:
        d = torch.empty(2 * vmax + 1, dtype=torch.int32, device="cuda")
        info = np.zeros(4, np.int64)
        _lib.check(_lib.lib().sfc_debug_quantizer(vmax, bits, ctypes.c_void_p(d.data_ptr()),
                                                  info.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), None))
        sa = max(vmax / qmax, 1e-8)
        assert info[3:4].view(np.float64)[0] == sa
        v = np.arange(-vmax, vmax + 1, dtype=np.float64)
        want = np.clip(np.rint(v / sa), -qmax - 1, qmax).astype(np.int32)
        assert np.array_equal(d.cpu().numpy(), want), f"vmax={vmax} bits={bits} fast={info[0]}"
        n_fast += int(info[0])
    assert n_fast >= 0.9 * len(vmaxes)   # the verified multiply-shift path is the common case


# ------------------------------------------------------------------------------ edge cases / errors
def test_zero_and_constant_inputs(cuda):
    w = np.random.default_rng(5).integers(-127, 128, size=(4, 3, 3, 3), dtype=np.int8)
    for x in (np.zeros((1, 3, 10, 10), np.int8), np.full((1, 3, 10, 10), 7, np.int8),
              np.full((2, 3, 5, 9), -128, np.int8)):
        for v in VARIANTS:
            check_against_oracle(x, w, v)
    g = run_gpu(np.zeros((1, 3, 10, 10), np.int8), w, "sfc6-6x6-3x3")
    assert g["stats"]["act_scale"] == 1e-8 and g["stats"]["vmax"] == 0 and not g["y"].any()


def test_zero_filters(cuda):
    x = np.random.default_rng(6).integers(-128, 128, size=(1, 4, 8, 8), dtype=np.int8)
    w = np.zeros((3, 4, 3, 3), np.int8)
    g, r = check_against_oracle(x, w, "sfc6-7x7-3x3")
    assert np.all(g["sf"] == 1e-8) and not g["y"].any()


def test_errors_like_reference(cuda):
    spec = sc.catalog_algorithm("sfc4-4x4-3x3")
    x = torch.zeros((1, 1, 8, 8), dtype=torch.int8)
    f = torch.zeros((1, 1, 3, 3), dtype=torch.int8)
    for bits in (1, 17):   # test_quant.cpp:190-199
        with pytest.raises(ValueError, match="between 2 and 16 bits"):
            sc.quantized_fast_conv2d(x, f, spec, 1, sc.QuantConfig(bits=bits))
    with pytest.raises(ValueError, match="filter shape does not match"):
        sc.transform_filters(torch.zeros((1, 1, 5, 5)), spec)
    with pytest.raises(ValueError, match="input channel count"):
        sc.quantized_fast_conv2d(torch.zeros((1, 2, 8, 8), dtype=torch.int8), f, spec, 1)
    with pytest.raises(ValueError, match="filter larger than padded input"):
        sc.quantized_fast_conv2d(torch.zeros((1, 1, 2, 2), dtype=torch.int8), f, spec, 0)
    # fractional values take the real-valued path (no longer refused); the reference's output
    # for a constant 0.5 input and a zero filter is exactly 0
    rep = sc.quantized_fast_conv2d(torch.full((1, 1, 8, 8), 0.5), f, spec, 1)
    assert rep.output.dtype == torch.float64 and float(rep.output.abs().max()) == 0.0
    # bits 9-16 are accepted like the reference (the wide fp64-GEMM path)
    rep = sc.quantized_fast_conv2d(x, f, spec, 1, sc.QuantConfig(bits=12))
    assert float(rep.output.abs().max()) == 0.0 and rep.saturations == 0


def test_concurrent_streams_match(cuda):
    """Layers are immutable; two calls on two streams with distinct workspaces agree."""
    L = wl.WORKLOADS[2].layers[0]
    x = torch.from_numpy(wl.activations(2, 0, L)).cuda()
    w = torch.from_numpy(wl.weights(2, 0, L)).cuda()
    layer = sc.SfcLayer("sfc6-6x6-3x3", w)
    outs = []
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for s in streams:
        with torch.cuda.stream(s):
            ws = layer.workspace(8, 28, 28, 1)
            y = torch.empty((8, 128, 28, 28), dtype=torch.int32, device="cuda")
            layer.forward(x, ws, 1, y_int32=y, stream=s)
            outs.append(y)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1])


@pytest.mark.parametrize("variant", VARIANTS)
def test_repeated_forwards_are_deterministic(cuda, variant):
    """Races show up as run-to-run differences long before they hit a fixed oracle case:
    ten forwards of the config-2 layer (fresh workspaces) must agree bit for bit."""
    L = wl.WORKLOADS[2].layers[0]
    x = torch.from_numpy(wl.activations(2, 0, L)).cuda()
    w = torch.from_numpy(wl.weights(2, 0, L)).cuda()
    ho = L.hw + 2 * L.pad - L.r + 1
    first = None
    for _ in range(10):
        layer = sc.SfcLayer(variant, w)
        ws = layer.workspace(L.batch, L.hw, L.hw, L.pad)
        y = torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int32, device="cuda")
        layer.forward(x, ws, L.pad, y_int32=y)
        _, p = layer.views(L.batch, L.hw, L.hw, L.pad, ws)
        cur = (y.clone(), p.clone())
        if first is None:
            first = cur
        else:
            for a, b in zip(first, cur):
                assert torch.equal(a, b)


@pytest.mark.parametrize("variant", VARIANTS)
def test_kept_and_recompute_paths_agree(cuda, variant, monkeypatch):
    """forward (absmax keeps V; quantization in the GEMM when V is L2-sized, else streaming)
    == transform + conv_kept (the multi-GPU entry points) with the streaming quantizer
    (SFC_QFUSE=0) and with quantization fused into the GEMM (SFC_QFUSE=1) == absmax + conv
    (quantize recomputes the transform from x): y, P and stats bit for bit, and vq where it
    is materialised."""
    for cfg, li in ((2, 0), (1, 0), (3, 0)):
        L = wl.WORKLOADS[cfg].layers[li]
        x = torch.from_numpy(wl.activations(cfg, li, L)).cuda()
        w = torch.from_numpy(wl.weights(cfg, li, L)).cuda()
        layer = sc.SfcLayer(variant, w)
        ho = L.hw + 2 * L.pad - L.r + 1
        res = {}
        for mode in ("forward", "kept", "kept-qfused", "kept-qtma", "recompute"):
            ws = layer.workspace(L.batch, L.hw, L.hw, L.pad)
            y = torch.empty((L.batch, L.cout, ho, ho), dtype=torch.int64, device="cuda")
            if mode == "kept-qfused":
                monkeypatch.setenv("SFC_QFUSE", "1")
            elif mode == "kept-qtma":
                monkeypatch.setenv("SFC_QFUSE", "2")
            elif mode == "kept":
                monkeypatch.setenv("SFC_QFUSE", "0")  # streaming quantizer materialises vq
            else:
                monkeypatch.delenv("SFC_QFUSE", raising=False)
            if mode.startswith("forward"):
                layer.forward(x, ws, L.pad, y_int64=y)
            else:
                vmax = torch.zeros(1, dtype=torch.int32, device="cuda")
                if mode.startswith("kept"):
                    layer.transform(x, vmax, ws, L.pad)
                    layer.conv_kept(tuple(x.shape), vmax, ws, L.pad, y_int64=y)
                else:
                    layer.absmax(x, vmax, L.pad)
                    layer.conv(x, vmax, ws, L.pad, y_int64=y)
            vq, p = layer.views(L.batch, L.hw, L.hw, L.pad, ws)
            res[mode] = (y.clone(), None if p is None else p.clone(), vq.clone(),
                         layer.stats(L.batch, L.hw, L.hw, L.pad, ws))
        monkeypatch.delenv("SFC_QFUSE", raising=False)
        ref = res["recompute"]
        for mode, r in res.items():
            assert torch.equal(ref[0], r[0]), (cfg, mode, "y")
            if ref[1] is not None:  # (chunked P is consumed from L2 and never materialised)
                assert torch.equal(ref[1], r[1]), (cfg, mode, "P")
            assert ref[3] == r[3], (cfg, mode, "stats")
        assert torch.equal(ref[2], res["kept"][2]), (cfg, "vq")


@pytest.mark.parametrize("variant", VARIANTS + LARGE_R)
@pytest.mark.parametrize("budget_mb", [2])
def test_chunked_p_matches_whole(cuda, variant, budget_mb, monkeypatch):
    """P chunking (GEMM -> output transform per chunk of image tile rows, each chunk's P
    consumed from L2 and discarded): a small budget forces 2..many chunks, ragged last chunk
    included; y, fp32 out and stats equal the unchunked run bit for bit and y the oracle's.
    The general QuantConfig path chunks the same way."""
    R = sc.catalog_algorithm(variant).R
    rng = np.random.default_rng(budget_mb * 31 + R)
    B, C, OC, H = 20, 40, 96, 22
    x = rng.integers(-128, 128, size=(B, C, H, H), dtype=np.int8)
    w = rng.integers(-127, 128, size=(OC, C, R, R), dtype=np.int8)
    pad = R // 2
    xt, wt = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    res = {}
    for mode in ("whole", "chunked"):
        if mode == "chunked":
            monkeypatch.setenv("SFC_PCHUNK_MB", str(budget_mb))
        else:
            monkeypatch.setenv("SFC_PCHUNK_MB", "0")
        layer = sc.SfcLayer(variant, wt)
        ws = layer.workspace(B, H, H, pad)
        y = torch.empty((B, OC, H, H), dtype=torch.int64, device="cuda")
        out = torch.empty((B, OC, H, H), dtype=torch.float32, device="cuda")
        layer.forward(xt, ws, pad, y_int64=y, out_f32=out)
        _, pacc = layer.views(B, H, H, pad, ws)
        gen = sc.quantized_fast_conv2d(xt, wt, sc.catalog_algorithm(variant), pad, sc.QuantConfig(8, 1, 2, 0))
        res[mode] = (y.cpu(), out.cpu(), layer.stats(B, H, H, pad, ws), pacc is None, gen.output.cpu(), gen.mse)
    monkeypatch.delenv("SFC_PCHUNK_MB")
    whole, chunked = res["whole"], res["chunked"]
    assert not whole[3] and chunked[3]  # the budget really chunked P
    assert torch.equal(whole[0], chunked[0]) and torch.equal(whole[1], chunked[1]) and whole[2] == chunked[2]
    assert torch.equal(whole[4], chunked[4]) and whole[5] == chunked[5]
    r = ob.quantized_conv(x, w, variant, pad, want=("y_int",))
    assert np.array_equal(chunked[0].numpy(), r["y_int"])


GENERAL_SHARD_CFGS = [(8, 1, 0, 0), (8, 0, 2, 1), (6, 1, 1, 1), (12, 1, 2, 1), (8, 0, 1, 0)]


@pytest.mark.parametrize("variant", ["sfc6-6x6-3x3", "sfc4-4x4-3x3", "sfc6-6x6-5x5"])
@pytest.mark.parametrize("cfg", GENERAL_SHARD_CFGS, ids=[f"b{c[0]}a{c[1]}f{c[2]}s{c[3]}" for c in GENERAL_SHARD_CFGS])
def test_general_quantconfig_shard_protocol(cuda, variant, cfg):
    """The multi-GPU steps of a non-default QuantConfig (sfc_general_prepare / _mse_partial /
    _conv, distributed.CudaEngine) run shard by shard on one device, exactly as the ranks run
    them: maxima max-reduced, MseGrid sums chained in batch order.  Output, scales and counts
    equal the whole-batch forward bit for bit."""
    from paper_2407_02913_b200.distributed import CudaEngine, shard_bounds
    bits, asc, fsc, srch = cfg
    R = sc.catalog_algorithm(variant).R
    rng = np.random.default_rng(sum(cfg) + R)
    B, C, OC, H = 5, 6, 7, 12
    x = rng.integers(-128, 128, size=(B, C, H, H), dtype=np.int8)
    x[3:] //= 4
    w = rng.integers(-127, 128, size=(OC, C, R, R), dtype=np.int8)
    pad = R // 2
    xt = torch.from_numpy(x).cuda()
    layer = sc.SfcLayer(variant, torch.from_numpy(w).cuda(), bits, fsc, srch, act_scope=asc)
    ws = layer.workspace(B, H, H, pad)
    full = torch.empty((B, OC, H, H), dtype=torch.float64, device="cuda")
    layer.forward(xt, ws, pad, out_f64=full)
    full_scales = layer.act_scales(B, H, H, pad, ws)
    full_stats = layer.stats(B, H, H, pad, ws)
    world = 3
    engines = [CudaEngine(layer, pad) for _ in range(world)]
    shards = [xt[lo:hi] for lo, hi in (shard_bounds(B, r, world) for r in range(world))]
    maxima = [e.general_prepare(xs) for e, xs in zip(engines, shards)]
    glob = torch.stack(maxima).max(0).values  # the all-reduce(MAX)
    for m in maxima:
        m.copy_(glob)
    err = None
    if srch:
        for e, xs in zip(engines, shards):  # rank order = batch order
            err = e.general_mse(xs, err)
    outs, sat = [], 0
    for e, xs in zip(engines, shards):
        o = torch.empty((xs.shape[0], OC, H, H), dtype=torch.float64, device="cuda")
        e.general_conv(xs, err, out_f64=o)
        outs.append(o)
        n = xs.shape[0]
        assert np.array_equal(layer.act_scales(n, H, H, pad, e._workspace(xs)), full_scales)
        sat += layer.stats(n, H, H, pad, e._workspace(xs))["saturations"]
    assert torch.equal(torch.cat(outs), full)
    assert sat == full_stats["saturations"]


# ------------------------------------------------------------------------------ 5x5 / 7x7 variants
GOLD_R = np.load(os.path.join(HERE, "golden", "qconv_large_r.npz"))
TAGS_R = sorted({k.split("/")[0] for k in GOLD_R.files})
CASES_R = [  # (B, C, OC, H, W, pad, lo)
    (1, 8, 8, 16, 16, 2, -128),
    (2, 5, 3, 13, 11, 3, -128),
    (1, 70, 33, 12, 12, 1, 0),
    (1, 3, 130, 9, 9, 0, -128),
    (1, 2, 2, 7, 7, 3, -128),
]


@pytest.mark.parametrize("variant", LARGE_R)
@pytest.mark.parametrize("case", CASES_R, ids=[f"b{c[0]}c{c[1]}o{c[2]}h{c[3]}w{c[4]}p{c[5]}" for c in CASES_R])
def test_large_r_bit_exact(cuda, variant, case):
    B, C, OC, H, W, pad, lo = case
    R = ob.spec(variant)["R"]
    rng = np.random.default_rng(hash(case) & 0xFFFF)
    x = rng.integers(lo, 128, size=(B, C, H, W), dtype=np.int8)
    w = rng.integers(-127, 128, size=(OC, C, R, R), dtype=np.int8)
    check_against_oracle(x, w, variant, pad)


@pytest.mark.parametrize("variant", LARGE_R)
@pytest.mark.parametrize("tag", TAGS_R)
def test_large_r_golden_reference_outputs(cuda, tag, variant):
    """fp32 output vs the reference's own quantized_fast_conv2d (fp64), max-normalised <= 1e-6."""
    x, (pad, bits) = GOLD_R[f"{tag}/x"], GOLD_R[f"{tag}/meta"]
    w = GOLD_R[f"{tag}/{variant}/w"]
    g = run_gpu(x, w, variant, int(pad), int(bits), views=False)
    assert maxrel(g["f32"], GOLD_R[f"{tag}/{variant}/out"]) <= TOL
    assert g["stats"]["saturations"] + g["filter_sat"] == 0


@pytest.mark.parametrize("variant", LARGE_R)
def test_large_r_layer_size(cuda, variant):
    """A 56x56, 64-channel, batch-4 layer against the oracle (y_int bit-exact, fp32 <= 1e-6)."""
    R = ob.spec(variant)["R"]
    rng = np.random.default_rng(91)
    x = rng.integers(0, 128, size=(4, 64, 56, 56), dtype=np.int8)
    w = rng.integers(-127, 128, size=(64, 64, R, R), dtype=np.int8)
    check_against_oracle(x, w, variant, R // 2, intermediates=False)


# ------------------------------------------------------------------------------ general QuantConfig
GENERAL_CONFIGS = [  # (act_scope, filter_scope, search, bits)
    (1, 0, 0, 8), (0, 1, 0, 8), (0, 2, 0, 8), (1, 2, 0, 8), (0, 0, 1, 8), (1, 1, 1, 6), (0, 2, 1, 4), (1, 0, 0, 3),
]


@pytest.mark.parametrize("variant", VARIANTS + ["sfc6-6x6-5x5"])
@pytest.mark.parametrize("cfg", GENERAL_CONFIGS, ids=[f"a{c[0]}f{c[1]}s{c[2]}b{c[3]}" for c in GENERAL_CONFIGS])
def test_general_quant_config_vs_oracle(cuda, variant, cfg):
    """Per-frequency activation scales, per-frequency / per-(oc, f) filter scales, MseGrid:
    the scales are exactly the oracle's (same fp64 search order), vq / uq / pacc bit-exact,
    fp32 output within 1e-6 (fp64 epilogue, dequantised before A as quant.cpp:258-263)."""
    asc, fsc, srch, bits = cfg
    R = ob.spec(variant)["R"]
    rng = np.random.default_rng(sum(cfg) * 31 + R)
    B, C, OC, H, W, pad = 2, 6, 5, 13, 12, R // 2
    x = rng.integers(-128, 128, size=(B, C, H, W), dtype=np.int8)
    w = rng.integers(-127, 128, size=(OC, C, R, R), dtype=np.int8)
    r = ob.quantized_conv(x, w, variant, pad, bits, asc, fsc, srch, want=("out", "pacc", "vq", "uq"), report=True)
    dev = torch.device("cuda", 0)
    layer = sc.SfcLayer(variant, torch.from_numpy(w).to(dev), bits=bits, filter_scope=fsc, search=srch, act_scope=asc)
    xt = torch.from_numpy(x).to(dev)
    HO, WO = H + 2 * pad - R + 1, W + 2 * pad - R + 1
    ws = layer.workspace(B, H, W, pad)
    out = torch.empty((B, OC, HO, WO), dtype=torch.float32, device=dev)
    out64 = torch.empty((B, OC, HO, WO), dtype=torch.float64, device=dev)
    layer.forward(xt, ws, pad, out_f32=out, out_f64=out64)
    torch.cuda.synchronize()
    assert np.array_equal(layer.act_scales(B, H, W, pad, ws), r["act_scale"]), "activation scales"
    assert np.array_equal(layer.filter_scales_native(), r["fil_scale"]), "filter scales"
    assert np.array_equal(layer.uq().cpu().numpy(), r["uq"].transpose(2, 0, 1)), "uq"
    vq, pacc = layer.views(B, H, W, pad, ws)
    assert np.array_equal(vq.cpu().numpy(), r["vq"].transpose(2, 0, 1)), "vq"
    assert np.array_equal(pacc.cpu().numpy().astype(np.int64), r["pacc"].transpose(2, 0, 1)), "pacc"
    assert maxrel(out.cpu().numpy(), r["out"]) <= TOL
    assert maxrel(out64.cpu().numpy(), r["out"]) <= 1e-12
    st = layer.stats(B, H, W, pad, ws)
    assert st["saturations"] + layer.filter_saturations() == r["report"]["saturations"]
    with pytest.raises(_lib.SfcUnsupported):  # y_int is not defined for these configurations
        layer.forward(xt, ws, pad, y_int32=torch.empty((B, OC, HO, WO), dtype=torch.int32, device=dev))


# ------------------------------------------------------------------------------ real-valued tensors
GOLD_REAL = np.load(os.path.join(HERE, "golden", "qconv_real.npz"))
TAGS_REAL = sorted({k.split("/")[0] for k in GOLD_REAL.files})


@pytest.mark.parametrize("variant", VARIANTS + LARGE_R)
@pytest.mark.parametrize("tag", TAGS_REAL)
def test_real_valued_tensors_vs_reference_golden(cuda, tag, variant):
    """The reference API's doubles (N(0,1) inputs and filters, as the reference CLI's quantsim
    feeds): V and U in the reference's arithmetic order, so scales / vq / uq / pacc are the
    reference's and the fp64 output agrees to the epilogue's rounding (<= 1e-12)."""
    x = GOLD_REAL[f"{tag}/x"]
    asc, fsc, srch, bits = (int(v) for v in GOLD_REAL[f"{tag}/meta"])
    w = GOLD_REAL[f"{tag}/{variant}/w"]
    r = GOLD_REAL[f"{tag}/{variant}/report"]
    pad = int(r[5])
    rep = sc.quantized_fast_conv2d(torch.from_numpy(x), torch.from_numpy(w), sc.catalog_algorithm(variant), pad,
                                   sc.QuantConfig(bits, asc, fsc, srch))
    assert rep.output.dtype == torch.float64
    assert maxrel(rep.output.cpu().numpy(), GOLD_REAL[f"{tag}/{variant}/out"]) <= 1e-12
    assert rep.saturations == r[3] and rep.values_quantized == r[4]
    assert rep.mse == pytest.approx(r[0], rel=1e-9) and rep.snr_db == pytest.approx(r[2], rel=1e-9)
    # the fp64 direct conv in the reference's summation order is bitwise the reference's
    B, C, H, W = x.shape
    OC, R = w.shape[0], w.shape[2]
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    out = torch.empty((B, OC, H + 2 * pad - R + 1, W + 2 * pad - R + 1), dtype=torch.float64, device="cuda")
    _lib.check(_lib.lib().sfc_direct_conv_f64(ctypes.c_void_p(xd.data_ptr()), B, C, H, W,
                                              ctypes.c_void_p(wd.data_ptr()), OC, R, 1, pad,
                                              ctypes.c_void_p(out.data_ptr()), None))
    assert np.array_equal(out.cpu().numpy(), GOLD_REAL[f"{tag}/{variant}/direct"])



@pytest.mark.parametrize("variant", VARIANTS + LARGE_R)
@pytest.mark.parametrize("tag", TAGS_REAL)
def test_fast_conv2d_float_path(cuda, tag, variant):
    """fast_conv2d (conv.cpp:384-553) on the device: vs the reference's own float-path output
    (<= 1e-12) and vs the fp64 direct conv at the reference's bar (<= 1e-10, test_conv.cpp:78-90);
    the product / tile counters equal the reference's full-schedule counts."""
    x, w = GOLD_REAL[f"{tag}/x"], GOLD_REAL[f"{tag}/{variant}/w"]
    pad = int(GOLD_REAL[f"{tag}/{variant}/report"][5])
    out, cnt = sc.fast_conv2d_counters(torch.from_numpy(x), torch.from_numpy(w), sc.catalog_algorithm(variant), pad)
    got = out.cpu().numpy()
    assert maxrel(got, GOLD_REAL[f"{tag}/{variant}/fast"]) <= 1e-12
    assert maxrel(got, GOLD_REAL[f"{tag}/{variant}/direct"]) <= 1e-10
    assert [cnt["multiplications"], cnt["tiles"]] == list(GOLD_REAL[f"{tag}/{variant}/fast_counts"])


@pytest.mark.parametrize("variant", VARIANTS + LARGE_R)
@pytest.mark.parametrize("tag", TAGS_REAL)
def test_fast_conv2d_paired_schedule(cuda, tag, variant):
    """reduced_products (conv.cpp:466-509): six evaluation products per (triple x triple) block
    folded onto its corners.  Matches the reference's own paired output (<= 1e-12), the full
    schedule (<= 1e-12, test_conv.cpp:140-162) and the reference's paired product count."""
    x, w = GOLD_REAL[f"{tag}/x"], GOLD_REAL[f"{tag}/{variant}/w"]
    pad = int(GOLD_REAL[f"{tag}/{variant}/report"][5])
    spec = sc.catalog_algorithm(variant)
    out, cnt = sc.fast_conv2d_counters(torch.from_numpy(x), torch.from_numpy(w), spec, pad, reduced_products=True)
    got = out.cpu().numpy()
    assert maxrel(got, GOLD_REAL[f"{tag}/{variant}/fast_red"]) <= 1e-12
    assert maxrel(got, GOLD_REAL[f"{tag}/{variant}/fast"]) <= 1e-12
    assert [cnt["multiplications"], cnt["tiles"]] == list(GOLD_REAL[f"{tag}/{variant}/fast_red_counts"])
    B, C = x.shape[:2]
    assert cnt["multiplications"] == spec.mults_reduced() * cnt["tiles"] * w.shape[0] * C


SMALL_C_CASES = [  # (B, C, OC, H, W, pad): Cin <= 4 takes the fused dp4a path by default
    (2, 3, 64, 30, 26, 1), (1, 1, 5, 9, 9, 1), (3, 2, 33, 14, 14, 0), (1, 4, 40, 13, 19, 2), (2, 3, 70, 57, 57, 1),
]


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("case", SMALL_C_CASES)
def test_small_channel_fused_path(cuda, variant, case, monkeypatch):
    """Cin <= 4: the dp4a contraction fused into the output transform (no P) gives the
    oracle's y_int / fp32 / int8 bit for bit, and equals the tensor-core GEMM path
    (SFC_SMALLC=0, whose pacc is also checked against the oracle)."""
    B, C, OC, H, W, pad = case
    rng = np.random.default_rng(B * 1000 + C * 100 + OC)
    x = rng.integers(-128, 128, size=(B, C, H, W), dtype=np.int8)
    w = rng.integers(-127, 128, size=(OC, C, 3, 3), dtype=np.int8)
    dev = torch.device("cuda", 0)
    layer = sc.SfcLayer(variant, torch.from_numpy(w).to(dev))
    assert layer.schedule(B, H, W, pad)["p_layout"] == 3
    g, r = check_against_oracle(x, w, variant, pad, intermediates=True)
    assert g["pacc"] is None
    ga = run_gpu(x, w, variant, pad, outs=("y", "f32", "i8"), requant=0.02, views=False)
    monkeypatch.setenv("SFC_SMALLC", "0")
    gb = run_gpu(x, w, variant, pad, outs=("y", "f32", "i8"), requant=0.02, views=False)
    g0, _ = check_against_oracle(x, w, variant, pad, intermediates=True)
    assert g0["pacc"] is not None
    for k in ("y", "f32", "i8"):
        assert np.array_equal(ga[k], gb[k]), k


@pytest.mark.parametrize("variant", VARIANTS)
def test_p24_and_output_kernels_agree(cuda, variant, monkeypatch):
    """The output-transform paths agree bit for bit: unit-major 24-bit P with the tensor-core
    output transform (default, out_mma.cu), 24-bit P rows with the CUDA-core kernels
    (SFC_OUT_MMA=0: persistent kernel on 512-channel layers, one-block kernel with
    SFC_OUT_PERS=0) and int32 P (SFC_P24=0): y, fp32, int8 requant and pacc on a 512-channel
    layer, a 64-channel layer and a small ragged one."""
    rng = np.random.default_rng(11)
    for (B, C, OC, H, W, pad) in ((26, 64, 512, 14, 14, 1), (40, 64, 64, 30, 26, 1), (2, 40, 70, 11, 9, 1)):
        x = rng.integers(-128, 128, size=(B, C, H, W), dtype=np.int8)
        w = rng.integers(-127, 128, size=(OC, C, 3, 3), dtype=np.int8)
        dev = torch.device("cuda", 0)
        layer = sc.SfcLayer(variant, torch.from_numpy(w).to(dev))
        for k in ("SFC_P24", "SFC_OUT_PERS", "SFC_OUT_MMA"):
            monkeypatch.delenv(k, raising=False)
        # (small grids keep the 24-bit rows and the one-block kernels)
        assert layer.schedule(B, H, W, pad)["p_layout"] == (1 if B == 2 else 2)
        res = {}
        for name, env in (("default", {}), ("rows", {"SFC_OUT_MMA": "0"}), ("p32", {"SFC_P24": "0"}),
                          ("one-block", {"SFC_OUT_MMA": "0", "SFC_OUT_PERS": "0"})):
            for k in ("SFC_P24", "SFC_OUT_PERS", "SFC_OUT_MMA"):
                monkeypatch.delenv(k, raising=False)
            for k, v in env.items():
                monkeypatch.setenv(k, v)
            res[name] = run_gpu(x, w, variant, pad, outs=("y", "f32", "i8"), requant=0.003, views=True)
        for name in ("rows", "p32", "one-block"):
            for k in ("y", "f32", "i8", "pacc", "vq"):
                assert np.array_equal(res["default"][k], res[name][k]), (name, k)

@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("outs", [("y32",), ("i8",), ("y32", "f32"), ("y64", "f64", "i8"), ("f32", "i8")],
                         ids=lambda o: "+".join(o))
def test_tensor_core_output_transform_every_output_set(cuda, variant, outs, monkeypatch):
    """k_out_mma (unit-major P) against the CUDA-core output kernels (SFC_OUT_MMA=0) for every
    output set it specialises or reads at run time, on shapes whose unit tiles cross image rows
    (tw = 3, 5), leave partial output tiles (odd and even WO), and partial channel blocks
    (OC = 70): every output bit for bit."""
    rng = np.random.default_rng(21)
    dev = torch.device("cuda", 0)
    for (B, C, OC, H, W) in ((64, 48, 70, 17, 15), (80, 64, 96, 14, 20)):
        x = torch.from_numpy(rng.integers(-128, 128, size=(B, C, H, W), dtype=np.int8)).to(dev)
        w = torch.from_numpy(rng.integers(-127, 128, size=(OC, C, 3, 3), dtype=np.int8)).to(dev)
        layer = sc.SfcLayer(variant, w)
        res = {}
        for name, env in (("mma", {}), ("cuda-core", {"SFC_OUT_MMA": "0"})):
            monkeypatch.delenv("SFC_OUT_MMA", raising=False)
            for k, v in env.items():
                monkeypatch.setenv(k, v)
            assert layer.schedule(B, H, W, 1)["p_layout"] == (2 if name == "mma" else 1)
            ws = layer.workspace(B, H, W, 1)
            kinds = {"y32": torch.int32, "y64": torch.int64, "f32": torch.float32, "f64": torch.float64,
                     "i8": torch.int8}
            t = {k: torch.full((B, OC, H, W), 77, dtype=kinds[k], device=dev) for k in outs}
            layer.forward(x, ws, 1, y_int32=t.get("y32"), y_int64=t.get("y64"), out_f32=t.get("f32"),
                          out_f64=t.get("f64"), out_i8=t.get("i8"), requant_scale=0.0021)
            torch.cuda.synchronize()
            res[name] = {k: v.cpu().numpy() for k, v in t.items()}
        for k in outs:
            assert np.array_equal(res["mma"][k], res["cuda-core"][k]), k


def _p2_flag_fraction(layer, B, H, W, pad, ws):
    """Fraction of (unit, f) rows of plane 2 the GEMM flagged (sparse plane 2 of unit-major P)."""
    import ctypes
    vq, pa = ctypes.c_void_p(), ctypes.c_void_p()
    geom = np.zeros(6, np.int64)
    sc.check(sc.lib().sfc_conv_views(layer._h, B, H, W, pad, sc._ptr(ws), ws.numel(), ctypes.byref(vq), ctypes.byref(pa),
                                     geom.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    T, Tpad, _, OCpad = (int(v) for v in geom[:4])
    F = layer.spec.K ** 2
    n_ob, n_tg = OCpad // 32, Tpad // 4
    fl = sc._wrap_device(pa.value + 3 * F * Tpad * OCpad, (n_ob, n_tg // 8, F, 8), torch.uint8, ws.device)
    return float((fl != 0).float().mean())


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("kind", ["relu-dc-only", "signed-mixed", "huge-all-flagged", "tiny-none"])
def test_sparse_plane2_of_unit_major_p(cuda, variant, kind, monkeypatch):
    """Sparse plane 2 (the GEMM stores P + 2^15 and writes a plane-2 row only when one of its
    values leaves 16 bits): every flag regime -- post-ReLU inputs (the DC frequency only: rows
    loaded one by one), signed inputs at 256 channels (many rows: the box + fix-up path),
    large operands (most rows) and few channels (hardly any row) -- gives the
    dense layout's (SFC_P2_DENSE=1) and the oracle's pacc / y_int / int8 / fp32 bit for bit."""
    rng = np.random.default_rng({"relu-dc-only": 5, "signed-mixed": 6, "huge-all-flagged": 7, "tiny-none": 8}[kind])
    if kind == "relu-dc-only":
        B, C, OC, H, W = 40, 64, 64, 26, 22
        x = rng.integers(0, 128, size=(B, C, H, W), dtype=np.int8)
        w = np.clip(np.rint(rng.normal(0, 40, size=(OC, C, 3, 3))), -127, 127).astype(np.int8)
    elif kind == "signed-mixed":
        B, C, OC, H, W = 96, 256, 128, 14, 14  # (256 channels: int32-exact y for every variant)
        x = rng.integers(-128, 128, size=(B, C, H, W), dtype=np.int8)
        w = np.clip(np.rint(rng.normal(0, 45, size=(OC, C, 3, 3))), -127, 127).astype(np.int8)
    elif kind == "huge-all-flagged":
        B, C, OC, H, W = 96, 256, 128, 14, 14
        x = np.full((B, C, H, W), 127, dtype=np.int8)
        x[:, ::2] = -128
        w = np.full((OC, C, 3, 3), 127, dtype=np.int8)
        w[:, ::2] = -127
        x[rng.random(x.shape) < 0.3] = 90
    else:
        B, C, OC, H, W = 40, 8, 64, 26, 22
        x = rng.integers(-128, 128, size=(B, C, H, W), dtype=np.int8)
        w = rng.integers(-2, 3, size=(OC, C, 3, 3)).astype(np.int8)
    dev = torch.device("cuda", 0)
    layer = sc.SfcLayer(variant, torch.from_numpy(w).to(dev))
    monkeypatch.delenv("SFC_P2_DENSE", raising=False)
    assert layer.schedule(B, H, W, 1)["p_layout"] == 2
    res = {}
    for name in ("sparse", "dense"):
        if name == "dense":
            monkeypatch.setenv("SFC_P2_DENSE", "1")
        res[name] = run_gpu(x, w, variant, 1, outs=("y", "f32", "i8"), requant=0.0017, views=True)
    monkeypatch.delenv("SFC_P2_DENSE")
    for k in ("y", "f32", "i8", "pacc", "vq"):
        assert np.array_equal(res["sparse"][k], res["dense"][k]), k
    check_against_oracle(x, w, variant, 1, intermediates=True)
    xt = torch.from_numpy(x).to(dev)
    ws = layer.workspace(B, H, W, 1)
    y = torch.empty((B, OC, H, W), dtype=torch.int32, device=dev)
    layer.forward(xt, ws, 1, y_int32=y)
    torch.cuda.synchronize()
    frac = _p2_flag_fraction(layer, B, H, W, 1, ws)
    if kind == "relu-dc-only":
        assert 0.0 < frac < 0.08, frac
    elif kind == "tiny-none":
        assert frac < 0.01, frac
    elif kind == "huge-all-flagged":
        assert frac > 0.01, frac
    else:
        assert 0.005 < frac < 0.98, frac
