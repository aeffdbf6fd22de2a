"""Seeded synthetic inputs for the MH-LatentMoE layer - shared by the oracle
tests and the CUDA path, and holding NONE of the method's arithmetic.

Every tensor is drawn from ``np.random.Generator(PCG64(SeedSequence([seed,
tid] + extra)))`` with a fixed tensor id (x=0, W_in=1, W_r=2, b=3, W1=4, W2=5,
W_out=6, dout=7), so any subset can be regenerated independently.  Values are
rounded to bfloat16 (RNE, via float32 bit arithmetic) for bf16 storage; W_r and
b are always float32 (the router computes in FP32).

Value distributions:
  conf   variance-preserving: x,dout ~ N(0,1); W_in ~ N(0,1/d); W_r,W1 ~ N(0,1/d_h);
         W2 ~ N(0,1/d_e); W_out ~ N(0,1/D); b ~ N(0, 0.1^2)
  paper  the paper's init (P:1995-P:1996): all weights N(0, 0.02^2), output
         projections (W_out, W2) further x 1/sqrt(2L), L = 12 (R18); b = 0
  skew   as paper, plus b[h,e] = -s * sigma_S * ln(1+e)   (expert-load imbalance)
  exact  as conf, but every sub-token is EXACT in fp32 whatever the summation order: W_in has
         EXACT_NNZ = 8 nonzeros per row, each +-2^-j (j in {1,2,3}), and x is bf16 with
         |x| >= 2^-6 (smaller values flushed to 0).  Every product is then a multiple of 2^-16
         below 2^3 in magnitude and every partial sum of a row a multiple of 2^-16 below 2^7,
         i.e. representable in fp32's 24-bit significand, so the GPU's fp32-accumulated Xs is the
         exact value and rounds to bf16 exactly as the oracle's fp64 value does (no R22 budget:
         the router sees identical sub-tokens on both sides and north_star's margin rule applies
         as stated).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, asdict

import numpy as np

TID = dict(x=0, W_in=1, W_r=2, b=3, W1=4, W2=5, W_out=6, dout=7)


@dataclass(frozen=True)
class LayerConfig:
    """One BASELINE.json config.  T is the GLOBAL token count of the layer step."""
    name: str
    T: int
    d: int
    N_h: int
    d_h: int
    N_e: int
    k: int
    d_e: int
    dtype: str          # "bf16" or "fp32" (storage/compute mode of the CUDA path)
    fwd_only: bool = False
    routing_tokens: bool = False   # separate routing sub-tokens (P:1565-P:1570): W_in is [2D, d]

    @property
    def D(self) -> int:
        return self.N_h * self.d_h

    def replace(self, **kw) -> "LayerConfig":
        d = asdict(self)
        d.update(kw)
        return LayerConfig(**d)


# BASELINE.json "configs" (global T; per-GPU T_loc = T under weak scaling at N=1)
PRESETS = {
    "tiny": LayerConfig("tiny", T=256, d=64, N_h=4, d_h=16, N_e=8, k=2, d_e=16, dtype="fp32"),
    "small": LayerConfig("small", T=8192, d=768, N_h=4, d_h=192, N_e=64, k=8, d_e=64, dtype="bf16",
                         fwd_only=True),
    "paper": LayerConfig("paper", T=65536, d=2048, N_h=8, d_h=256, N_e=64, k=8, d_e=128, dtype="bf16"),
    "g2x": LayerConfig("g2x", T=65536, d=2048, N_h=8, d_h=256, N_e=128, k=16, d_e=64, dtype="bf16"),
}
for _k in (2, 4, 16):
    PRESETS[f"paper_k{_k}"] = PRESETS["paper"].replace(name=f"paper_k{_k}", k=_k)
# separate routing sub-tokens (ablation P:1565-P:1570), supplementary: W_in [2D, d], the HP scatter doubles
PRESETS["paper_rtok"] = PRESETS["paper"].replace(name="paper_rtok", routing_tokens=True)
# paper's own Table-5 shape (P:2070-P:2080), supplementary (multi-block online top-k, N_e > 256)
PRESETS["table5"] = LayerConfig("table5", T=16384, d=1024, N_h=8, d_h=128, N_e=768, k=4, d_e=256, dtype="bf16")


def to_bf16_exact(a: np.ndarray) -> np.ndarray:
    """Round float32 values to bfloat16 (round-to-nearest-even) and return them
    as float32 (exactly representable).  Input-generation helper only."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return (rounded & 0xFFFFFFFF).astype(np.uint32).view(np.float32)


def _rng(seed: int, tid: int, extra=()) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, tid, *extra])))


def _normal(seed, tid, shape, std, extra=()):
    a = _rng(seed, tid, extra).standard_normal(size=shape, dtype=np.float32)
    if std != 1.0:
        a *= np.float32(std)
    return a


EXACT_NNZ = 8


def _sparse_pow2(seed, tid, shape):
    """EXACT_NNZ nonzeros per row at distinct random columns, values +-2^-j, j uniform in {1,2,3}."""
    rng = _rng(seed, tid)
    rows, cols = shape
    nnz = min(EXACT_NNZ, cols)
    a = np.zeros(shape, np.float32)
    for r in range(rows):
        c = rng.choice(cols, nnz, replace=False)
        a[r, c] = rng.choice([-1.0, 1.0], nnz) * np.exp2(-rng.integers(1, 4, nnz).astype(np.float32))
    return a


def quantize_exact_tokens(a: np.ndarray) -> np.ndarray:
    """bf16 values with |x| >= 2^-6 (smaller ones flushed to 0): the token side of `exact`."""
    q = to_bf16_exact(a)
    q[np.abs(q) < 2.0 ** -6] = 0.0
    return q


def make_weights(cfg: LayerConfig, seed: int = 0, dist: str = "conf", skew: float = 0.0) -> dict:
    """Layer parameters as float32 arrays (bf16-exact where stored in bf16)."""
    d, D, N_h, d_h, N_e, d_e = cfg.d, cfg.D, cfg.N_h, cfg.d_h, cfg.N_e, cfg.d_e
    if dist == "conf":
        std = dict(W_in=1 / math.sqrt(d), W_r=1 / math.sqrt(d_h), W1=1 / math.sqrt(d_h),
                   W2=1 / math.sqrt(d_e), W_out=1 / math.sqrt(D), b=0.1)
    elif dist == "exact":
        std = dict(W_in=None, W_r=1 / math.sqrt(d_h), W1=1 / math.sqrt(d_h),
                   W2=1 / math.sqrt(d_e), W_out=1 / math.sqrt(D), b=0.1)
    elif dist in ("paper", "skew"):
        o = 0.02 / math.sqrt(2 * 12)
        std = dict(W_in=0.02, W_r=0.02, W1=0.02, W2=o, W_out=o, b=0.0)
    else:
        raise ValueError(dist)
    rows_in = (2 if cfg.routing_tokens else 1) * D
    W = dict(
        W_in=(_sparse_pow2(seed, TID["W_in"], (rows_in, d)) if dist == "exact"
              else _normal(seed, TID["W_in"], (rows_in, d), std["W_in"])),
        W_out=_normal(seed, TID["W_out"], (d, D), std["W_out"]),
        W_r=_normal(seed, TID["W_r"], (N_h, d_h, N_e), std["W_r"]),
        W1=_normal(seed, TID["W1"], (N_h, N_e, d_e, d_h), std["W1"]),
        W2=_normal(seed, TID["W2"], (N_h, N_e, d_e, d_h), std["W2"]),
    )
    if std["b"] > 0:
        W["b"] = _normal(seed, TID["b"], (N_h, N_e), std["b"])
    else:
        W["b"] = np.zeros((N_h, N_e), np.float32)
    if dist == "skew" and skew:
        sigma_s = 0.02 * math.sqrt(d) * 0.02 * math.sqrt(d_h)  # score std under the paper init
        W["b"] = (-skew * sigma_s * np.log1p(np.arange(N_e, dtype=np.float64)))[None, :].repeat(N_h, 0).astype(np.float32)
    if cfg.dtype == "bf16":
        for name in ("W_in", "W_out", "W1", "W2"):
            W[name] = to_bf16_exact(W[name])
    return W


def make_tokens(cfg: LayerConfig, seed: int = 0, T: int | None = None, rank: int = 0, which: str = "x") -> np.ndarray:
    """x or dout [T, d] ~ N(0,1) for one token shard (rank-seeded)."""
    T = cfg.T if T is None else T
    a = _normal(seed, TID[which], (T, cfg.d), 1.0, extra=(rank,))
    return to_bf16_exact(a) if cfg.dtype == "bf16" else a


def make_problem(cfg: LayerConfig, seed: int = 0, dist: str = "conf", T: int | None = None, skew: float = 0.0):
    """(weights, x, dout) of the global problem."""
    W = make_weights(cfg, seed, dist, skew)
    x = make_tokens(cfg, seed, T, which="x")
    if dist == "exact":
        x = quantize_exact_tokens(x)
    dout = make_tokens(cfg, seed, T, which="dout")
    return W, x, dout
