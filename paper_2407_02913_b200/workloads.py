"""Seeded synthetic workloads for the five BASELINE.json configurations (1-5) and the
5x5 / 7x7 SFC variants at config 2's shape (6, 7, not BASELINE configs).

No public dataset is involved: ImageNet is only cited by the
paper for accuracy numbers.  Inputs are generated on the host with numpy's
PCG64 (platform independent) and the *same int8 bytes* are fed to the GPU path,
the C oracle and the compiled reference (the latter as doubles), so every arm
sees identical data.

Seed scheme: base = 0x5fc07751 (the reference CLI default,
proj/tools/sfconv_cli.cpp:30); for config c and layer L
    activations  seed base + 1000*c + 2*L       uniform int in [lo, 127]
    weights      seed base + 1000*c + 2*L + 1   N(0, sigma), per-oc symmetric int8
    requant      seed base + 1000*c + 999       U[1e-3, 1e-2] per layer
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 0x5FC07751
SFC_3x3_VARIANTS = ("sfc4-4x4-3x3", "sfc6-6x6-3x3", "sfc6-7x7-3x3")


@dataclass(frozen=True)
class Layer:
    name: str
    batch: int
    cin: int
    cout: int
    hw: int
    act_lo: int = 0          # activations uniform in [act_lo, 127]
    sigma: float = 1.0       # weight N(0, sigma) before per-oc int8 quantization
    pad: int = 1
    r: int = 3               # filter size (R x R)


@dataclass(frozen=True)
class Workload:
    config: int
    name: str
    layers: tuple
    variants: tuple = ("sfc6-6x6-3x3",)
    requant: bool = False    # int8 output clamp(rint(out * s_l), 0, 127) (harness-defined)
    description: str = ""
    extra: dict = field(default_factory=dict)


def _resnet18_layers(batch: int):
    out = []
    for c, hw, n in ((64, 56, 4), (128, 28, 3), (256, 14, 3), (512, 7, 3)):
        for i in range(n):
            out.append(Layer(f"res{c}_{hw}_{i}", batch, c, c, hw))
    return tuple(out)


def _vgg16_layers(batch: int):
    spec = [(3, 64, 224), (64, 64, 224), (64, 128, 112), (128, 128, 112), (128, 256, 56),
            (256, 256, 56), (256, 256, 56), (256, 512, 28), (512, 512, 28), (512, 512, 28),
            (512, 512, 14), (512, 512, 14), (512, 512, 14)]
    return tuple(Layer(f"vgg{i}_{ci}_{co}_{hw}", batch, ci, co, hw) for i, (ci, co, hw) in enumerate(spec))


WORKLOADS = {
    1: Workload(1, "cfg1_n1_c64_56", (Layer("conv", 1, 64, 64, 56, act_lo=-128),),
                description="single conv N=1 64->64 56x56, x~U[-128,127], sfc6-6x6-3x3"),
    2: Workload(2, "cfg2_n8_c128_28_sweep", (Layer("conv", 8, 128, 128, 28),),
                variants=SFC_3x3_VARIANTS,
                description="N=8 128->128 28x28, x~U[0,127], every 3x3 SFC variant"),
    3: Workload(3, "cfg3_resnet18_b64", _resnet18_layers(64), requant=True,
                description="ResNet-18 13 stride-1 3x3 convs, batch 64, int8 requant"),
    4: Workload(4, "cfg4_vgg16_b128", _vgg16_layers(128), requant=True,
                description="VGG-16 13 convs, batch 128, int8 requant"),
    5: Workload(5, "cfg5_n256_c512_14", (Layer("conv", 256, 512, 512, 14, act_lo=-128, sigma=0.5),),
                description="N=256 512->512 14x14, x~U[-128,127], w~N(0,0.5)"),
    6: Workload(6, "cfg6_n8_c128_28_r5", (Layer("conv", 8, 128, 128, 28, pad=2, r=5),),
                variants=("sfc6-6x6-5x5",),
                description="config 2's shape with 5x5 filters (pad 2), sfc6-6x6-5x5"),
    7: Workload(7, "cfg7_n8_c128_28_r7", (Layer("conv", 8, 128, 128, 28, pad=3, r=7),),
                variants=("sfc6-4x4-7x7",),
                description="config 2's shape with 7x7 filters (pad 3), sfc6-4x4-7x7"),
}


def activations(cfg: int, layer_idx: int, layer: Layer, batch: int | None = None) -> np.ndarray:
    """int8 NCHW activations, uniform integers in [layer.act_lo, 127]."""
    rng = np.random.default_rng(BASE_SEED + 1000 * cfg + 2 * layer_idx)
    b = layer.batch if batch is None else batch
    return rng.integers(layer.act_lo, 128, size=(b, layer.cin, layer.hw, layer.hw), dtype=np.int8)


def quantize_weights_per_oc(w: np.ndarray) -> np.ndarray:
    """Symmetric per-output-channel int8: s_oc = max|w_oc|/127, q = clip(rint(w/s_oc), -127, 127)."""
    amax = np.abs(w).reshape(w.shape[0], -1).max(axis=1)
    s = np.where(amax > 0, amax / 127.0, 1.0)
    q = np.rint(w / s[:, None, None, None])
    return np.clip(q, -127, 127).astype(np.int8)


def weights(cfg: int, layer_idx: int, layer: Layer) -> np.ndarray:
    rng = np.random.default_rng(BASE_SEED + 1000 * cfg + 2 * layer_idx + 1)
    w = rng.normal(0.0, layer.sigma, size=(layer.cout, layer.cin, layer.r, layer.r))
    return quantize_weights_per_oc(w)


def requant_scales(cfg: int, n_layers: int) -> np.ndarray:
    rng = np.random.default_rng(BASE_SEED + 1000 * cfg + 999)
    return rng.uniform(1e-3, 1e-2, size=n_layers)


def direct_equivalent_ops(layer: Layer, batch: int | None = None) -> int:
    """2 R^2 * N * Cout * Cin * HO * WO (2 ops per MAC of a direct R x R conv; 18 for 3x3)."""
    b = layer.batch if batch is None else batch
    ho = layer.hw + 2 * layer.pad - layer.r + 1
    return 2 * layer.r * layer.r * b * layer.cout * layer.cin * ho * ho


def tile_grid(layer: Layer, m: int, batch: int | None = None):
    b = layer.batch if batch is None else batch
    ho = layer.hw + 2 * layer.pad - layer.r + 1
    th = -(-ho // m)
    return b * th * th, th, ho
