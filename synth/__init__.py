"""Seeded synthetic inputs shaped like the paper's workloads.

Shared by the oracle side (tests, cpu_baseline) and the CUDA side (tests,
bench, smoke).  This module holds NONE of the method's arithmetic: it only
draws random numbers and names the configurations of BASELINE.json.

Every (b, h) slice has its own ``torch.Generator`` (CPU) seeded from
``250114577 + config index`` and the slice number, so one slice can be
regenerated without the others (sampled oracle checks at full size).
Draw order per slice: Q[N, d_k], K[N, d_k], V[N, d_v], dO[N, d_v], all
N(0, 1) float32 ("iid").  The "tokens" variants reproduce the structure of
the paper's token workloads (repeated tokens => identical keys, code ties,
distance ties and hub keys); see DESIGN.md.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace

import numpy as np
import torch

SEED_BASE = 250114577
EPS = float(np.float32(0.5))          # eps = sigmoid(theta = 0) (reading D14)


@dataclass(frozen=True)
class Config:
    name: str
    cfg_index: int          # index into BASELINE.json "configs"
    B: int
    H: int
    N: int
    d_k: int
    d_v: int
    k: int
    window: int
    chunk: int
    causal: int
    mean_slot: int = 1
    bits: int = 0
    inputs: str = "iid"     # "iid" | "tokens"
    vocab: int = 0
    zipf: float = 0.0
    ar_layout: bool = False

    @property
    def BH(self) -> int:
        return self.B * self.H

    def problem_kwargs(self) -> dict:
        return dict(B=self.B, H=self.H, N=self.N, d_k=self.d_k, d_v=self.d_v, k=self.k, window=self.window,
                    chunk=self.chunk, bits=self.bits, causal=self.causal, mean_slot=self.mean_slot)

    def with_(self, **kw) -> "Config":
        return replace(self, **kw)


def _long(n: int) -> Config:
    return Config(f"long{n // 1024}k", 4, 8, 12, n, 3, 64, 64, 128, n // 32, 1)


# BASELINE.json "configs" with the chunk counts of SURVEY 8 (reading D18)
CONFIGS = {
    "tiny": Config("tiny", 0, 1, 1, 256, 2, 16, 8, 16, 32, 1),
    "ar": Config("ar", 1, 64, 4, 2048, 3, 64, 32, 64, 256, 1),
    "ar_tokens": Config("ar_tokens", 1, 64, 4, 2048, 3, 64, 32, 64, 256, 1, inputs="tokens", vocab=8192,
                        ar_layout=True),
    "lra_nc": Config("lra_nc", 2, 32, 8, 4096, 3, 64, 64, 128, 4096, 0),
    "lra_c": Config("lra_c", 2, 32, 8, 4096, 3, 64, 64, 128, 256, 1),
    "lra_tokens": Config("lra_tokens", 2, 32, 8, 4096, 3, 64, 64, 128, 256, 1, inputs="tokens", vocab=256,
                         zipf=1.1),
    "wiki": Config("wiki", 3, 16, 12, 8192, 4, 64, 64, 128, 256, 1),
    "wiki_tokens": Config("wiki_tokens", 3, 16, 12, 8192, 4, 64, 64, 128, 256, 1, inputs="tokens", vocab=32768,
                          zipf=1.0),
    "long64k": _long(65536),
    "long128k": _long(131072),
    "long256k": _long(262144),
    "long512k": _long(524288),
    "long1m": _long(1048576),
}


def slice_seed(cfg: Config, bh: int) -> int:
    return ((SEED_BASE + cfg.cfg_index) * 1_000_003 + 7919 * bh + (17 if cfg.inputs == "tokens" else 0)) % (2**62)


def _tokens(cfg: Config, g: torch.Generator) -> torch.Tensor:
    N, V = cfg.N, cfg.vocab
    if cfg.ar_layout:
        # MQAR-like: first 25% key/value pairs, then filler where half the
        # positions are probes repeating an earlier key token.
        nkv = N // 4
        t = torch.randint(0, V, (N,), generator=g)
        probe = torch.rand(N, generator=g) < 0.5
        src = torch.randint(0, max(nkv, 1), (N,), generator=g)
        t[nkv:] = torch.where(probe[nkv:], t[src[nkv:]], t[nkv:])
        return t
    # Zipf(s) over the vocabulary by inverse-CDF sampling
    ranks = torch.arange(1, V + 1, dtype=torch.float64)
    w = ranks.pow(-cfg.zipf)
    cdf = torch.cumsum(w / w.sum(), 0)
    u = torch.rand(N, generator=g, dtype=torch.float64)
    return torch.searchsorted(cdf, u).clamp_(max=V - 1)


def make_slice(cfg: Config, bh: int):
    """One (b,h) slice: dict of float32 numpy arrays Q,K [N,d_k], V,dO [N,d_v]."""
    g = torch.Generator().manual_seed(slice_seed(cfg, bh))
    N = cfg.N
    if cfg.inputs == "iid":
        Q = torch.randn(N, cfg.d_k, generator=g)
        K = torch.randn(N, cfg.d_k, generator=g)
    else:
        emb = torch.randn(cfg.vocab, cfg.d_k, generator=g)
        t = _tokens(cfg, g)
        K = emb[t].contiguous()                         # identical rows for repeated tokens
        Q = (emb[t] + 0.05 * torch.randn(N, cfg.d_k, generator=g)).contiguous()
    V = torch.randn(N, cfg.d_v, generator=g)
    dO = torch.randn(N, cfg.d_v, generator=g)
    return dict(Q=Q.numpy(), K=K.numpy(), V=V.numpy(), dO=dO.numpy())


def make_inputs(cfg: Config, bh_range=None):
    """Stacked slices [B*H or len(bh_range)] -> arrays shaped [B', H', N, .] (B'=1 when a range is given)."""
    bhs = list(range(cfg.BH)) if bh_range is None else list(bh_range)
    out = {name: [] for name in ("Q", "K", "V", "dO")}
    for bh in bhs:
        s = make_slice(cfg, bh)
        for name in out:
            out[name].append(s[name])
    lead = (cfg.B, cfg.H) if bh_range is None else (1, len(bhs))
    return {name: np.stack(v).reshape(*lead, *v[0].shape) for name, v in out.items()}


def sample_queries(cfg: Config, n: int, bh_range=None, seed: int = 0) -> np.ndarray:
    """Seeded uniform sample of flat query ids (bh_local*N + i), sorted."""
    nbh = cfg.BH if bh_range is None else len(list(bh_range))
    rng = np.random.default_rng(SEED_BASE + cfg.cfg_index + 1000 * seed)
    flat = rng.choice(nbh * cfg.N, size=min(n, nbh * cfg.N), replace=False)
    return np.sort(flat).astype(np.int64)
