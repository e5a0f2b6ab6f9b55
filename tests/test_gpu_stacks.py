"""Configs 3 and 4 (BASELINE.json): every layer of the ResNet-18 (batch 64) and VGG-16 (batch 128)
stacks at full size through the product forward (int32 y_int and the harness int8 requant in one
call), checked against the oracle (oracle/sfc_oracle.c, pinned to the compiled reference):

* the activation absmax over the WHOLE batch (quant.cpp:171-172) equals the oracle's;
* y_int of 8 images spread over the batch (first and last included) equals the oracle's int64
  y_int for those images quantized with the full batch's scale (quant.cpp:239-279);
* the int8 requant clamp(rint(y * (sa * sf[oc] / N^2) * s_l), 0, 127) (harness-defined, fp64)
  recomputed from the ORACLE's y_int and the oracle's scales equals the GPU's int8 output on
  those images, and the GPU's int8 output over the whole batch equals the requant of its own
  y_int.

The oracle runs on every host thread.  Its full-batch absmax pass is run with a one-filter slice
of the weights (the activation scale depends on x only), so the contraction it performs is a
1/OC sliver of the layer's.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import bindings as ob  # noqa: E402
from paper_2407_02913_b200 import sfconv as sc, workloads as wl  # noqa: E402

pytestmark = pytest.mark.gpu
CASES = [(3, i) for i in range(13)] + [(4, i) for i in range(13)]


@pytest.mark.parametrize("cfg,idx", CASES, ids=[f"cfg{c}_layer{i}" for c, i in CASES])
def test_stack_layer_full_batch(cuda, cfg, idx):
    work = wl.WORKLOADS[cfg]
    L = work.layers[idx]
    variant = work.variants[0]
    x, w = wl.activations(cfg, idx, L), wl.weights(cfg, idx, L)
    s_l = float(wl.requant_scales(cfg, len(work.layers))[idx])
    B, ho = L.batch, L.hw + 2 * L.pad - L.r + 1

    layer = sc.SfcLayer(variant, torch.from_numpy(w).to(cuda))
    xt = torch.from_numpy(x).to(cuda)
    ws = layer.workspace(B, L.hw, L.hw, L.pad)
    y = torch.empty((B, L.cout, ho, ho), dtype=torch.int32, device=cuda)
    q8 = torch.empty((B, L.cout, ho, ho), dtype=torch.int8, device=cuda)
    layer.forward(xt, ws, L.pad, requant_scale=s_l, y_int32=y, out_i8=q8)
    torch.cuda.synchronize()
    st = layer.stats(B, L.hw, L.hw, L.pad, ws)
    sf_gpu, _ = layer.filter_scales()
    y, q8 = y.cpu().numpy(), q8.cpu().numpy()
    del ws, xt

    # full-batch activation absmax and scale
    full = ob.quantized_conv(x, w[:1], variant, L.pad, want=())
    vmax = full["report"]["vmax"]
    assert st["vmax"] == vmax
    assert st["act_scale"] == full["act_scale"][0]

    # 8 images spread over the batch, quantized with the full batch's scale
    pick = np.unique(np.linspace(0, B - 1, 8).round().astype(int))
    part = ob.quantized_conv(x[pick], w, variant, L.pad, want=("y_int",), vmax_override=vmax)
    assert np.array_equal(y[pick].astype(np.int64), part["y_int"]), "y_int differs from the oracle"
    assert np.array_equal(sf_gpu, part["fil_scale"])

    # harness int8 requant from the oracle's y_int and scales
    den = float(part["spec"]["a_denom"]) ** 2
    scale = (part["act_scale"][0] * part["fil_scale"]) / den
    want8 = np.clip(np.rint(part["y_int"].astype(np.float64) * scale[None, :, None, None] * s_l), 0, 127)
    assert np.array_equal(q8[pick], want8.astype(np.int8)), "int8 requant differs from the oracle's"
    # and over the whole batch, from the GPU's own y_int (same fp64 formula)
    own = np.clip(np.rint(y.astype(np.float64) * scale[None, :, None, None] * s_l), 0, 127).astype(np.int8)
    assert np.array_equal(q8, own)
