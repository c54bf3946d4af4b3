"""Seeded synthetic workloads shared by the tests, bench.py and the oracle harness.

This module holds NO arithmetic of the method (no mask predicate, no ACSR, no
softmax): it only names the BASELINE.json configurations as pattern descriptors
plus shapes, and draws the Q/K/V inputs from a seeded generator.  Both the CUDA
path and the oracle receive the arrays it produces; neither imports the other.

Input recipe:
  * Q, K, V are [B, H, N, d], d innermost, values uniform in [-1, 1)
    (SPEC.md S:602), drawn per (tensor, b*H+h) slice from
    ``torch.Generator('cpu').manual_seed(slice_seed(cfg, t, bh))`` with
    ``torch.rand(N, d, dtype=float32) * 2 - 1``;
  * bf16 configurations round that fp32 draw to bf16 (round-to-nearest-even,
    ``Tensor.to``) and the oracle reads the ROUNDED values (SURVEY A-13);
  * scale = 1/sqrt(d) (SURVEY A-1);
  * the mask is the config's descriptor, identical for every (b, h).
Per-slice seeding lets the oracle regenerate any (b, h) slice by itself, which
is how the full-size parity tests sample Mistral-sized heads.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

# Pattern kinds, named as in SURVEY.md §8(b)/§8(c) C-2.
KINDS = ("window", "blocked", "strided", "dilated", "global_local", "bigbird",
         "strided_local")


@dataclass(frozen=True)
class Pattern:
    """Pattern descriptor (parameters only; the semantics live on each side).

    Fields mirror ``splat_pattern`` in include/splat.h; unused fields are 0.
    """
    kind: str
    seq_len: int
    lo: int = 0
    hi: int = 0
    block: int = 0
    n_global: int = 0
    stride: int = 0
    radius: int = 0
    causal: int = 0

    def __post_init__(self):
        if self.kind not in KINDS:
            raise ValueError(f"unknown pattern kind {self.kind!r}")

    def with_seq_len(self, n: int) -> "Pattern":
        d = dict(self.__dict__)
        d["seq_len"] = n
        return Pattern(**d)


@dataclass(frozen=True)
class Config:
    name: str
    pattern: Pattern
    B: int
    H: int
    d: int
    dtype: str           # "bf16" or "fp32"
    index: int           # position in BASELINE.json configs (seed base)
    baseline_text: str = field(default="", compare=False)

    @property
    def N(self) -> int:
        return self.pattern.seq_len

    @property
    def BH(self) -> int:
        return self.B * self.H

    @property
    def scale(self) -> float:
        return 1.0 / math.sqrt(self.d)

    @property
    def torch_dtype(self):
        return torch.bfloat16 if self.dtype == "bf16" else torch.float32


# BASELINE.json "configs", in order, with the readings of SURVEY.md §8(c) C-2/A-2.
CONFIGS = [
    Config("tiny", Pattern("window", 256, lo=32, hi=32), 1, 1, 64, "fp32", 0,
           "sliding-window attention, batch 1, 1 head, seq 256, d 64, window 32, fp32"),
    Config("longformer", Pattern("global_local", 4096, lo=256, hi=256, n_global=32),
           8, 12, 64, "bf16", 1,
           "Longformer window(512)+global(32 tokens), batch 8, 12 heads, seq 4096, d 64, bf16"),
    Config("bigbird", Pattern("bigbird", 4096, block=64, radius=1), 8, 12, 64, "bf16", 2,
           "BigBird-style blocked (block 64, 3 sliding + 2 global blocks), batch 8, 12 heads, seq 4096, d 64, bf16"),
    Config("sparse_transformer", Pattern("strided_local", 8192, stride=128, causal=1),
           4, 16, 128, "bf16", 3,
           "Sparse-Transformer strided + dilated (stride 128), batch 4, 16 heads, seq 8192, d 128, bf16"),
    Config("mistral", Pattern("window", 32768, lo=4095, hi=0), 4, 32, 128, "bf16", 4,
           "Mistral-style sliding window 4096, batch 4, 32 heads, seq 32768, d 128, bf16"),
]
CONFIG_BY_NAME = {c.name: c for c in CONFIGS}

TENSORS = {"q": 0, "k": 1, "v": 2}


def slice_seed(cfg_index: int, tensor: int, bh: int) -> int:
    """Seed of one [N, d] slice: config index, tensor (0=Q,1=K,2=V), b*H+h."""
    return 1_000_003 * (cfg_index + 1) + 7_919 * tensor + bh


def make_slice(cfg_index: int, tensor: int, bh: int, N: int, d: int,
               dtype=torch.float32) -> torch.Tensor:
    """One seeded [N, d] slice, uniform in [-1, 1), rounded to ``dtype``."""
    g = torch.Generator(device="cpu")
    g.manual_seed(slice_seed(cfg_index, tensor, bh))
    x = torch.rand(N, d, generator=g, dtype=torch.float32) * 2.0 - 1.0
    return x.to(dtype)


def make_tensor(cfg_index: int, tensor: int, B: int, H: int, N: int, d: int,
                dtype=torch.float32, bh_range=None) -> torch.Tensor:
    """[B*H (or len(bh_range)), N, d] stack of seeded slices (CPU)."""
    rng = range(B * H) if bh_range is None else bh_range
    out = torch.empty((len(rng), N, d), dtype=dtype)
    for i, bh in enumerate(rng):
        out[i] = make_slice(cfg_index, tensor, bh, N, d, dtype)
    return out


def make_qkv(cfg: Config, bh_range=None, N: int | None = None):
    """Q, K, V for ``cfg`` as CPU tensors of shape [B, H, N, d] (or [len(bh_range), N, d]).

    ``N`` overrides the sequence length (small parity variants of a config)."""
    n = cfg.N if N is None else N
    outs = []
    for t in (0, 1, 2):
        x = make_tensor(cfg.index, t, cfg.B, cfg.H, n, cfg.d, cfg.torch_dtype, bh_range)
        if bh_range is None:
            x = x.view(cfg.B, cfg.H, n, cfg.d)
        outs.append(x)
    return tuple(outs)


def make_random(shape, seed: int, dtype=torch.float32, scale: float = 1.0) -> torch.Tensor:
    """Generic seeded uniform [-scale, scale) tensor for ad-hoc parity cases."""
    g = torch.Generator(device="cpu")
    g.manual_seed(seed)
    x = (torch.rand(*shape, generator=g, dtype=torch.float32) * 2.0 - 1.0) * scale
    return x.to(dtype)
