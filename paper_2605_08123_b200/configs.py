"""The five BASELINE.json configurations and their seeded synthetic inputs.

Recipe (restated here; seed 0 is the reference CLI
default, proj/tools/sinktail_main.cpp:34):
  * every tensor [B, H, L', d] is one counter-RNG stream (inc/rng.hpp:38-56)
    indexed by its flat row-major position, tags "Q", "K", "V", "G" (dO);
    head (b, h) is rows [(b*H+h)*L', ...) -- draw-order independent.
  * c2: Q and K scaled by 0.5 (normal_matrix(..., scale), rng.hpp:47);
    valid length l_b = 1024 + floor(U_b * 1025), U_b = counter_uniform(fold_tag(seed,"len") + b),
    i.e. uniform in [L/2, L]; rows and cols >= l_b are masked.
  * c3: l_b = clip(round(300 * exp(0.6 z_b)), 64, 1024), z_b = counter_normal(seed,"len",b);
    symbols s_{b,i} = floor(20 * counter_uniform(fold_tag(seed,"sym") + b*L + i));
    table = normal(seed,"table",20x64); q/k/v = table[s] + 0.1 * normal(seed,"noise_q|k|v")
    (q, k and v share the symbol embedding, each with its own noise stream);
    one dustbin token per side at index L with constant cost 1.0; its V row is
    normal(seed,"dustbin_v") (reference convention, inc/problem.hpp:72); its
    Q/K rows are zero (unused under the constant cost).
  * c4/c5: N(0,1)/sqrt(d) generated in double, rounded once to bf16 (RNE via
    f32); dO is N(0,1) rounded to bf16.  The oracle consumes the same rounded values.
No external dataset is used: config 3 stands in for the paper's Pfam/ESM-2
workload with seeded synthetic tokens of that shape.
"""
from __future__ import annotations

import ctypes
import dataclasses
import importlib
import math
from typing import Callable, Dict, Optional

import numpy as np

# The counter RNG backend (bit-exact restatements of inc/rng.hpp:38-56): by default the
# product library's st_normal_fill / st_uniform_fill, loaded lazily.  bench.py's reference arm
# loads this file by path and installs the oracle's stoc_* fills instead, so that arm never
# maps libsinkattn.so (set_rng_backend).
_BACKEND: Dict[str, Callable] = {}


def set_rng_backend(normal: Callable, uniform: Callable) -> None:
    _BACKEND["normal"], _BACKEND["uniform"] = normal, uniform


def _product_lib():
    return importlib.import_module("paper_2605_08123_b200._lib").lib


@dataclasses.dataclass(frozen=True)
class Config:
    cid: int
    B: int
    H: int
    L: int
    d: int
    w: int          # reference half band; metric uses the full width Wf = 2w+1
    eps: float
    T: int
    R: int
    dtype: str      # "f32" | "bf16"
    mask: str = "none"      # "none" | "uniform_len" | "lognormal_len"
    dustbin: int = 0
    dustbin_cost: float = 1.0
    qk_scale: float = 1.0
    in_scale: float = 1.0   # applied to Q, K, V (c4/c5: 1/sqrt(d))
    embed: str = "normal"   # "normal" | "alphabet"

    @property
    def Wf(self) -> int:
        return 2 * self.w + 1

    @property
    def rows(self) -> int:
        return self.L + self.dustbin

    def nominal_cells(self) -> int:
        """B*H*L*Wf -- the metric's band cells per Sinkhorn step."""
        return self.B * self.H * self.L * self.Wf

    def nominal_cell_steps(self) -> int:
        return self.nominal_cells() * (self.T + self.R)

    def replace(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


CONFIGS: Dict[int, Config] = {
    1: Config(1, B=1, H=1, L=256, d=32, w=16, eps=0.1, T=20, R=2, dtype="f32"),
    2: Config(2, B=8, H=4, L=2048, d=64, w=64, eps=0.05, T=50, R=2, dtype="f32", mask="uniform_len", qk_scale=0.5),
    3: Config(3, B=16, H=8, L=1024, d=64, w=32, eps=0.1, T=30, R=2, dtype="f32", mask="lognormal_len", dustbin=1,
              dustbin_cost=1.0, embed="alphabet"),
    4: Config(4, B=4, H=8, L=32768, d=128, w=128, eps=0.05, T=100, R=2, dtype="bf16", in_scale=1 / math.sqrt(128)),
    5: Config(5, B=1, H=16, L=131072, d=64, w=256, eps=0.05, T=50, R=2, dtype="bf16", in_scale=1 / math.sqrt(64)),
}


def normal_fill(seed: int, tag: str, start: int, n: int, scale: float = 1.0) -> np.ndarray:
    if "normal" in _BACKEND:
        return _BACKEND["normal"](seed, tag, start, n, scale)
    out = np.empty(n, dtype=np.float64)
    _product_lib().st_normal_fill(seed, tag.encode(), start, n, scale,
                                  out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


def uniform_fill(seed: int, tag: str, start: int, n: int) -> np.ndarray:
    if "uniform" in _BACKEND:
        return _BACKEND["uniform"](seed, tag, start, n)
    out = np.empty(n, dtype=np.float64)
    _product_lib().st_uniform_fill(seed, tag.encode(), start, n, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
    return out


def to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round (double -> f32 -> bf16, RNE each) and return the bf16 bit patterns."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    r = ((b + np.uint32(0x7FFF) + ((b >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)).astype(np.uint16)
    return r


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


def lengths(cfg: Config, seed: int = 0) -> Optional[np.ndarray]:
    if cfg.mask == "none":
        return None
    if cfg.mask == "uniform_len":
        u = uniform_fill(seed, "len", 0, cfg.B)
        lo = cfg.L // 2
        return (lo + np.floor(u * (cfg.L - lo + 1))).astype(np.int64)
    if cfg.mask == "lognormal_len":
        z = normal_fill(seed, "len", 0, cfg.B)
        return np.clip(np.round(300.0 * np.exp(0.6 * z)), 64, cfg.L).astype(np.int64)
    raise ValueError(cfg.mask)


def masks(cfg: Config, seed: int = 0):
    ls = lengths(cfg, seed)
    if ls is None:
        return None, None, None
    m = (np.arange(cfg.L)[None, :] < ls[:, None]).astype(np.uint8)
    return m, m.copy(), ls


@dataclasses.dataclass
class Inputs:
    cfg: Config
    heads: range           # flat (b*H+h) head range generated
    Q: np.ndarray          # float32 [nh, L', d] (bf16-rounded values for bf16 configs)
    K: np.ndarray
    V: np.ndarray
    G: np.ndarray
    row_mask: Optional[np.ndarray]  # uint8 [B, L] (all examples)
    col_mask: Optional[np.ndarray]
    lengths: Optional[np.ndarray]
    bits: Optional[dict] = None     # bf16 bit patterns (uint16) per tensor for bf16 configs


def _conv(cfg: Config, x: np.ndarray) -> np.ndarray:
    """Round one head's double values to the storage dtype (f32, or bf16 bit patterns)."""
    return to_bf16_bits(x) if cfg.dtype == "bf16" else x.astype(np.float32)


def _tensor(cfg: Config, seed: int, tag: str, heads: range, scale: float) -> np.ndarray:
    Lr, d = cfg.rows, cfg.d
    per = Lr * d
    out = np.empty((len(heads), Lr, d), dtype=np.uint16 if cfg.dtype == "bf16" else np.float32)
    for n, bh in enumerate(heads):
        out[n] = _conv(cfg, normal_fill(seed, tag, bh * per, per, scale).reshape(Lr, d))
    return out


def _alphabet_tensor(cfg: Config, seed: int, which: str, heads: range) -> np.ndarray:
    L, d, Lr = cfg.L, cfg.d, cfg.rows
    table = normal_fill(seed, "table", 0, 20 * d).reshape(20, d)
    out = np.empty((len(heads), Lr, d), dtype=np.uint16 if cfg.dtype == "bf16" else np.float32)
    for n, bh in enumerate(heads):
        b = bh // cfg.H
        sym = np.floor(uniform_fill(seed, "sym", b * L, L) * 20).astype(np.int64)
        x = np.zeros((Lr, d), dtype=np.float64)
        x[:L] = table[sym] + normal_fill(seed, "noise_" + which, bh * L * d, L * d, 0.1).reshape(L, d)
        if which == "v" and cfg.dustbin:
            x[L] = normal_fill(seed, "dustbin_v", bh * d, d)
        out[n] = _conv(cfg, x)
    return out


def make_inputs(cfg: Config, seed: int = 0, heads: Optional[range] = None) -> Inputs:
    if heads is None:
        heads = range(cfg.B * cfg.H)
    rm, cm, ls = masks(cfg, seed)
    if cfg.embed == "alphabet":
        Q = _alphabet_tensor(cfg, seed, "q", heads)
        K = _alphabet_tensor(cfg, seed, "k", heads)
        V = _alphabet_tensor(cfg, seed, "v", heads)
    else:
        Q = _tensor(cfg, seed, "Q", heads, cfg.in_scale * cfg.qk_scale)
        K = _tensor(cfg, seed, "K", heads, cfg.in_scale * cfg.qk_scale)
        V = _tensor(cfg, seed, "V", heads, cfg.in_scale)
    G = _tensor(cfg, seed, "G", heads, 1.0)
    bits = None
    if cfg.dtype == "bf16":
        bits = {"Q": Q, "K": K, "V": V, "G": G}
        Q, K, V, G = (bf16_bits_to_f32(bits[k]) for k in ("Q", "K", "V", "G"))
    return Inputs(cfg, heads, Q, K, V, G, rm, cm, ls, bits)


def active_cells(cfg: Config, seed: int = 0) -> int:
    """Exact active edges of the support over all heads (masks and dustbin spokes included)."""
    _, _, ls = masks(cfg, seed)
    Ls = [cfg.L] * cfg.B if ls is None else list(ls)
    tot = 0
    for l in Ls:
        w = min(cfg.w, l - 1)
        band = l * (2 * w + 1) - w * (w + 1)
        spokes = (2 * l + 1) if cfg.dustbin else 0
        tot += (band + spokes) * cfg.H
    return int(tot)
