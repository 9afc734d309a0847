"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method: only shapes and random
draws.  Recipes follow BASELINE.json ``configs`` (restated in DESIGN.md
"Input recipe"); the paper's own workloads (ILSVRC-12 activations through
Inception V3 / ResNet V2 50) are not available, and these VGG/ResNet
3x3 stride-1 shapes stand in for them.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

NCHW, NHWC = 0, 1
BASE_SEED = 190101965


@dataclasses.dataclass(frozen=True)
class LayerCfg:
    n: int
    h: int
    w: int
    c_in: int
    c_out: int
    pad: int = 1
    x_dist: str = "uniform"      # uniform int8 | relu (max(U{-127..127},0)) | uniform_pos
    w_dist: str = "uniform"      # uniform int8 | normal (clamp(round(N(0,sigma)), +-127))
    w_sigma: float = 0.0
    scaling: bool = True


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    index: int
    layers: tuple          # tuple[LayerCfg]; C5 has 13, the rest 1
    pools_after: tuple = ()  # layer indices followed by a 2x2/2 max pool (C5)
    description: str = ""


def _vgg16_layers(n=256):
    chans = [(3, 64), (64, 64), (64, 128), (128, 128), (128, 256), (256, 256), (256, 256),
             (256, 512), (512, 512), (512, 512), (512, 512), (512, 512), (512, 512)]
    sizes = [224, 224, 112, 112, 56, 56, 56, 28, 28, 28, 14, 14, 14]
    return tuple(LayerCfg(n, s, s, ci, co, 1, "uniform", "normal", 24.0, True)
                 for (ci, co), s in zip(chans, sizes))


CONFIGS = {
    "C1": Config("C1", 0, (LayerCfg(1, 8, 8, 4, 4, 1, "uniform", "uniform", 0.0, True),),
                 description="batch 1, 8x8, 4->4, int8 uniform x and w; scaling off then on"),
    "C2": Config("C2", 1, (LayerCfg(32, 56, 56, 64, 64, 1, "uniform", "normal", 32.0, True),),
                 description="VGG-style layer: batch 32, 56x56, 64->64, w ~ round(N(0,32))"),
    "C3": Config("C3", 2, (LayerCfg(64, 28, 28, 128, 128, 1, "relu", "normal", 24.0, True),),
                 description="ResNet-style: batch 64, 28x28, 128->128, post-ReLU x, w ~ round(N(0,24))"),
    "C4": Config("C4", 3, (LayerCfg(128, 14, 14, 256, 256, 1, "relu", "normal", 24.0, True),),
                 description="ResNet-style: batch 128, 14x14, 256->256, post-ReLU x, w ~ round(N(0,24))"),
    "C5": Config("C5", 4, _vgg16_layers(), pools_after=(1, 3, 6, 9),
                 description="VGG-16 13-layer 3x3 stack at 224x224, batch 256, requantised, max-pool"),
}


def generator(seed: int) -> torch.Generator:
    g = torch.Generator()
    g.manual_seed(int(seed))
    return g


def draw_x(shape_nhwc, dist: str, g: torch.Generator) -> np.ndarray:
    if dist == "uniform":
        t = torch.randint(-128, 128, shape_nhwc, generator=g, dtype=torch.int16)
    elif dist == "relu":
        t = torch.randint(-127, 128, shape_nhwc, generator=g, dtype=torch.int16).clamp_(min=0)
    elif dist == "extreme_neg":
        t = torch.full(shape_nhwc, -128, dtype=torch.int16)
    elif dist == "extreme_pos":
        t = torch.full(shape_nhwc, 127, dtype=torch.int16)
    else:
        raise ValueError(dist)
    return t.to(torch.int8).numpy()


def draw_w(shape_ohwi, dist: str, sigma: float, g: torch.Generator) -> np.ndarray:
    if dist == "uniform":
        t = torch.randint(-128, 128, shape_ohwi, generator=g, dtype=torch.int16)
    elif dist == "normal":
        t = torch.round(torch.randn(shape_ohwi, generator=g, dtype=torch.float64) * sigma)
        t = t.clamp_(-127, 127).to(torch.int16)
    elif dist == "extreme_neg":
        t = torch.full(shape_ohwi, -128, dtype=torch.int16)
    elif dist == "extreme_pos":
        t = torch.full(shape_ohwi, 127, dtype=torch.int16)
    else:
        raise ValueError(dist)
    return t.to(torch.int8).numpy()


def layer_inputs(layer: LayerCfg, seed: int, layout: int = NHWC, n: int | None = None):
    """(x, w) int8 numpy arrays for one layer; x drawn first, then w."""
    g = generator(seed)
    nn = layer.n if n is None else n
    x = draw_x((nn, layer.h, layer.w, layer.c_in), layer.x_dist, g)
    w = draw_w((layer.c_out, 3, 3, layer.c_in), layer.w_dist, layer.w_sigma, g)
    if layout == NCHW:
        x = np.ascontiguousarray(x.transpose(0, 3, 1, 2))
        w = np.ascontiguousarray(w.transpose(0, 3, 1, 2))
    return x, w


def config_inputs(name: str, layout: int = NHWC, rank: int = 0, layer: int = 0, n: int | None = None):
    cfg = CONFIGS[name]
    seed = BASE_SEED + 1000 * cfg.index + 17 * layer + 100003 * rank
    return layer_inputs(cfg.layers[layer], seed, layout, n)


def random_layer(rng: np.random.Generator, n, h, w, c_in, c_out, layout=NHWC, lo=-128, hi=127):
    """Small random layer for sweeps (tests)."""
    x = rng.integers(lo, hi + 1, size=(n, h, w, c_in), dtype=np.int64).astype(np.int8)
    wt = rng.integers(lo, hi + 1, size=(c_out, 3, 3, c_in), dtype=np.int64).astype(np.int8)
    if layout == NCHW:
        x = np.ascontiguousarray(x.transpose(0, 3, 1, 2))
        wt = np.ascontiguousarray(wt.transpose(0, 3, 1, 2))
    return x, wt


def requant_shift(layer: LayerCfg, sigma_in: float | None = None) -> int:
    """Fixed requantisation shift S (M0 = 1) chosen from shapes only
    (A14): S = round(log2(sigma_w sqrt(9 Cin) sigma_in / 32))."""
    sw = layer.w_sigma if layer.w_dist == "normal" else 73.9
    if sigma_in is None:
        sigma_in = 73.9 if layer.x_dist == "uniform" else 52.0
    v = sw * math.sqrt(9 * layer.c_in) * sigma_in / 32.0
    return max(0, int(round(math.log2(v))))


def direct_ops(layer: LayerCfg, n: int | None = None) -> int:
    """Direct-convolution int ops 2*N*Ho*Wo*Cin*Cout*9 (the metric's numerator)."""
    nn = layer.n if n is None else n
    ho, wo = layer.h + 2 * layer.pad - 2, layer.w + 2 * layer.pad - 2
    return 2 * nn * ho * wo * layer.c_in * layer.c_out * 9


def stack_shifts(name: str = "C5"):
    """Requantisation shift per layer of a stack config (A14): sigma_in
    = 73.9 (uniform int8) into layer 1, 32 into every later layer."""
    cfg = CONFIGS[name]
    return [requant_shift(l, 73.9 if i == 0 else 32.0) for i, l in enumerate(cfg.layers)]


def stack_inputs(name: str = "C5", n: int | None = None, layout: int = NHWC, rank: int = 0):
    """(x, [w_l]) for a layer stack: x from layer 0's seed, each layer's w from its own seed."""
    cfg = CONFIGS[name]
    x, _ = config_inputs(name, layout, rank=rank, layer=0, n=n)
    ws = [config_inputs(name, layout, rank=rank, layer=i, n=1)[1] for i in range(len(cfg.layers))]
    return x, ws
