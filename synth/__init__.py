"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no dedup, no scatter, no
sums): it only draws the inputs of one exchange step --

* token ids J_g: i.i.d. Zipf(s) over a frequency-ordered vocabulary, rank r ->
  id r-1 ("inversely proportional to its rank"; reading R7),
  by inverse CDF from numpy's Philox stream keyed by (seed, rank, step);
* gradient rows Delta_g and the table E0: a counter-based hash of
  (seed, stream, rank, step, element index) mapped to fp32.  The hash is
  written once with torch integer ops, so the CPU (oracle) and the GPU
  (inputs resident in HBM) produce bit-identical values.

Value modes:
  INT    Delta in {-8..7}, E0 in {-16..15}/16, lr = 2^-4 -> every partial sum is
         an exact fp32 integer, so results are bit-exact in any order.
  POS    Delta ~ U[0.5, 1.5), E0 ~ U[-1, 1)
  SIGNED Delta ~ U[-1, 1),    E0 ~ U[-1, 1)   (timing default, lr = 0.1)
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

MASTER_SEED = 181010045

MODES = ("int", "pos", "signed")

# Stream tags for the counter hash (any distinct 32-bit constants).
_TAG_IDS, _TAG_GRAD, _TAG_TABLE = 0x1D5, 0x6AD, 0x7AB


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json workload (configs[0..4]); SURVEY.md Sec. 8(d)."""
    name: str
    V: int          # vocabulary |V|
    K: int          # tokens per GPU
    D: int          # embedding dim
    s: float = 1.0  # Zipf exponent (R7)
    G: int = 1      # ranks (the tiny config is G=2 emulated)

    def with_(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)


CONFIGS = {
    "tiny": Config("tiny", V=10_000, K=4096, D=64, G=2),
    "1b": Config("1b", V=793_000, K=32_768, D=512),
    "char": Config("char", V=256, K=131_072, D=1024),
    "amazon": Config("amazon", V=2_000_000, K=131_072, D=1024),
    "tieba": Config("tieba", V=500_000, K=262_144, D=2048),
}


# ------------------------------------------------------------------ Zipf ids

_cdf_cache: dict = {}


def zipf_pmf(V: int, s: float) -> np.ndarray:
    """P(rank r) = r^-s / H_{V,s}, r = 1..V (fp64)."""
    w = np.arange(1, V + 1, dtype=np.float64) ** (-float(s))
    return w / w.sum()


def _zipf_cdf(V: int, s: float) -> np.ndarray:
    key = (V, float(s))
    if key not in _cdf_cache:
        c = np.cumsum(zipf_pmf(V, s))
        c[-1] = 1.0
        _cdf_cache[key] = c
    return _cdf_cache[key]


def _rng(seed: int, rank: int, step: int, tag: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(np.random.SeedSequence([seed, rank, step, tag])))


def zipf_ids(V: int, s: float, n: int, seed: int = MASTER_SEED, rank: int = 0,
             step: int = 0) -> np.ndarray:
    """n i.i.d. Zipf(s) ids over 0..V-1 (rank r -> id r-1), inverse CDF."""
    u = _rng(seed, rank, step, _TAG_IDS).random(n)
    ids = np.searchsorted(_zipf_cdf(V, s), u, side="right")
    return np.minimum(ids, V - 1).astype(np.uint32)


def expected_unique(V: int, s: float, N: int) -> float:
    """Closed form E[U](N) = sum_r 1 - (1 - p_r)^N for N i.i.d. Zipf draws."""
    p = zipf_pmf(V, s)
    return float(np.sum(-np.expm1(N * np.log1p(-p))))


def ids_for(cfg: Config, rank: int, step: int = 0, seed: int = MASTER_SEED) -> np.ndarray:
    return zipf_ids(cfg.V, cfg.s, cfg.K, seed=seed, rank=rank, step=step)


# ------------------------------------------------------------ counter values

def _mul32(x: torch.Tensor, c: int) -> torch.Tensor:
    """(x * c) mod 2^32 for 0 <= x < 2^32 without int64 overflow."""
    lo, hi = c & 0xFFFF, c >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & 0xFFFFFFFF


def _mix32(x: torch.Tensor) -> torch.Tensor:
    """lowbias32 integer hash (32-bit in, 32-bit out), on int64 tensors."""
    x = x ^ (x >> 16)
    x = _mul32(x, 0x7FEB352D)
    x = x ^ (x >> 15)
    x = _mul32(x, 0x846CA68B)
    x = x ^ (x >> 16)
    return x


def _key(seed: int, tag: int, rank: int, step: int) -> int:
    h = (seed * 0x9E3779B1 + tag * 0x85EBCA77 + rank * 0xC2B2AE3D + step * 0x27D4EB2F) & 0xFFFFFFFF
    return h


def counter_bits(n: int, key: int, device="cpu", offset: int = 0) -> torch.Tensor:
    """32-bit hash of element indices offset..offset+n-1 under ``key`` (int64)."""
    return hash_index(torch.arange(offset, offset + n, dtype=torch.int64, device=device), key)


def hash_index(idx: torch.Tensor, key: int) -> torch.Tensor:
    """32-bit hash of int64 element indices under ``key``."""
    lo = idx & 0xFFFFFFFF
    hi = idx >> 32
    x = _mix32(lo ^ key)
    x = _mix32(x ^ ((hi * 0x9E37 + 0x632B) & 0xFFFFFFFF) ^ ((key >> 7) & 0xFFFFFFFF))
    return x


def _to_value(bits: torch.Tensor, kind: str) -> torch.Tensor:
    if kind == "int_grad":          # {-8..7}
        return ((bits >> 28) - 8).to(torch.float32)
    if kind == "int_table":         # {-16..15}/16
        return ((bits >> 27) - 16).to(torch.float32) * (1.0 / 16.0)
    u = (bits >> 8).to(torch.float32) * (1.0 / 16777216.0)   # 24-bit uniform, exact
    if kind == "pos":
        return u + 0.5
    if kind == "signed":
        return u * 2.0 - 1.0
    raise ValueError(kind)


def _fill(out: torch.Tensor, key: int, kind: str, row0: int) -> torch.Tensor:
    rows, D = out.shape
    chunk = max(1, (1 << 26) // max(D, 1))          # bound the int64 temporaries
    for r in range(0, rows, chunk):
        n = min(chunk, rows - r)
        bits = counter_bits(n * D, key, out.device, offset=(row0 + r) * D)
        out[r:r + n] = _to_value(bits, kind).view(n, D)
    return out


def _rows(D: int, positions, key: int, kind: str) -> torch.Tensor:
    pos = torch.as_tensor(np.asarray(positions, np.int64)).reshape(-1)
    idx = (pos[:, None] * D + torch.arange(D, dtype=torch.int64)[None, :]).reshape(-1)
    return _to_value(hash_index(idx, key), kind).view(len(pos), D)


_GKIND = {"int": "int_grad", "pos": "pos", "signed": "signed"}


def grad_values(K: int, D: int, mode: str, rank: int = 0, step: int = 0,
                seed: int = MASTER_SEED, device="cpu", row0: int = 0,
                rows: int | None = None) -> torch.Tensor:
    """Delta_g (K x D fp32) or rows row0..row0+rows-1 of it."""
    rows = K - row0 if rows is None else rows
    out = torch.empty(rows, D, dtype=torch.float32, device=device)
    return _fill(out, _key(seed, _TAG_GRAD, rank, step), _GKIND[mode], row0)


def grad_rows(D: int, mode: str, positions, rank: int = 0, step: int = 0,
              seed: int = MASTER_SEED) -> torch.Tensor:
    """Rows ``positions`` of Delta_g (len(positions) x D) without drawing the rest."""
    return _rows(D, positions, _key(seed, _TAG_GRAD, rank, step), _GKIND[mode])


def _tkind(mode: str) -> str:
    return "int_table" if mode == "int" else "signed"


def table_values(V: int, D: int, mode: str, seed: int = MASTER_SEED, device="cpu",
                 row0: int = 0, rows: int | None = None) -> torch.Tensor:
    """E0 (V x D fp32) or rows row0..row0+rows-1 of it; identical on every rank."""
    rows = V - row0 if rows is None else rows
    out = torch.empty(rows, D, dtype=torch.float32, device=device)
    return _fill(out, _key(seed, _TAG_TABLE, 0, 0), _tkind(mode), row0)


def table_rows(V: int, D: int, mode: str, ids, seed: int = MASTER_SEED) -> torch.Tensor:
    """E0[ids] on the CPU without materialising the V x D table."""
    return _rows(D, ids, _key(seed, _TAG_TABLE, 0, 0), _tkind(mode))


def default_lr(mode: str) -> float:
    return 2.0 ** -4 if mode == "int" else 0.1


def heaps_fit(ns, us):
    """Unweighted least squares of log U on log N: returns (alpha, c)."""
    x = np.log(np.asarray(ns, np.float64))
    y = np.log(np.asarray(us, np.float64))
    A = np.vstack([x, np.ones_like(x)]).T
    slope, icpt = np.linalg.lstsq(A, y, rcond=None)[0]
    return float(slope), float(math.exp(icpt))
