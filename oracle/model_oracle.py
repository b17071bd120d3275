"""CPU restatement of the reference decoder (numpy, fp64) — test
infrastructure, never the product.

Restates /root/reference/proj/core/src/model.cpp:
  init_model :82-102 (SplitMix64 draws, rng.hpp:10-29), weight_sum :52-67,
  embed :104-129, layer_norm :131-150, transformer_layer :152-209,
  prefill :211-236, unembed_logits :238-246, argmax_token :248-255,
  decode_step :257-283, decode_greedy :285-297, generate_monolithic :299-305,
  generate_split :307-316.
The attention block is the monolithic causal softmax over the concatenated
cache (full_attention, attention.cpp:45-78), which the reference's spliced
per-segment form equals (SPEC: split == monolithic). Pinned against the
unmodified reference (oracle/_ref) by tests/test_model_oracle.py and against
the committed reference goldens (tests/golden/model_golden.json).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

M64 = (1 << 64) - 1
GAMMA = np.uint64(0x9E3779B97F4A7C15)
LN_EPS = 1e-5  # model.cpp:14


def splitmix_uniform(seed: int, first: int, n: int, lo: float, hi: float) -> np.ndarray:
    """Draws first .. first+n-1 of SplitMix64(seed), uniform(lo, hi)
    (rng.hpp:15-27: state += gamma; mix; (z >> 11) * 2^-53; lo + (hi-lo)*u)."""
    with np.errstate(over="ignore"):
        i = np.arange(first + 1, first + n + 1, dtype=np.uint64)
        z = np.uint64(seed & M64) + i * GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return lo + (hi - lo) * u


@dataclass
class Config:
    n_layers: int = 2
    n_heads: int = 2
    d_model: int = 8
    vocab_size: int = 32
    max_positions: int = 512
    init_seed: int = 1

    @property
    def d_head(self) -> int:
        return self.d_model // self.n_heads


@dataclass
class Layer:
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: np.ndarray


class Model:
    """init_model (model.cpp:82-102): one SplitMix64 stream, uniform(-0.1, 0.1),
    embedding, per layer wq wk wv wo w1 b1 w2 b2, unembedding."""

    def __init__(self, cfg: Config):
        if min(cfg.n_layers, cfg.n_heads, cfg.d_model, cfg.vocab_size, cfg.max_positions) <= 0:
            raise ValueError("ModelConfig: all dimensions must be positive")
        if cfg.d_model % cfg.n_heads:
            raise ValueError("ModelConfig: d_model not divisible by n_heads")
        self.cfg = cfg
        D, V, F = cfg.d_model, cfg.vocab_size, 4 * cfg.d_model
        sizes = [V * D] + [D * D] * 4 + [D * F, F, F * D, D]
        total = V * D + cfg.n_layers * (4 * D * D + 2 * D * F + F + D) + D * V
        self.draws = splitmix_uniform(cfg.init_seed, 0, total, -0.1, 0.1)
        off = 0

        def take(n, shape):
            nonlocal off
            a = self.draws[off:off + n].reshape(shape)
            off += n
            return a
        self.embedding = take(V * D, (V, D))
        self.layers = []
        for _ in range(cfg.n_layers):
            self.layers.append(Layer(take(D * D, (D, D)), take(D * D, (D, D)), take(D * D, (D, D)),
                                     take(D * D, (D, D)), take(D * F, (D, F)), take(F, (F,)),
                                     take(F * D, (F, D)), take(D, (D,))))
        self.unembed = take(D * V, (D, V))
        assert off == total and sizes

    def weight_sum(self) -> float:
        """model.cpp:52-67: sequential sum in generation order."""
        return float(np.cumsum(self.draws)[-1]) if self.draws.size else 0.0

    # ------------------------------------------------------------ blocks --
    def embed(self, tokens, pos_offset: int) -> np.ndarray:
        D = self.cfg.d_model
        if pos_offset + len(tokens) > self.cfg.max_positions:
            raise IndexError("embed: positions overflow max_positions")
        c = np.arange(D)
        pair = (c - c % 2).astype(np.float64)
        freq = np.power(10000.0, -pair / D)
        out = np.empty((len(tokens), D))
        for i, t in enumerate(tokens):
            if not 0 <= t < self.cfg.vocab_size:
                raise IndexError(f"embed: unknown token id {t}")
            ang = float(pos_offset + i) * freq
            out[i] = self.embedding[t] + np.where(c % 2 == 0, np.sin(ang), np.cos(ang))
        return out

    @staticmethod
    def layer_norm(x: np.ndarray) -> np.ndarray:
        mean = x.mean(axis=1, keepdims=True)
        var = ((x - mean) ** 2).mean(axis=1, keepdims=True)
        return (x - mean) / np.sqrt(var + LN_EPS)

    def layer(self, l: int, hidden: np.ndarray, pos_offset: int, k_cache: np.ndarray,
              v_cache: np.ndarray):
        """transformer_layer (model.cpp:152-209); k_cache/v_cache = the
        concatenated visible segments (positions 0 .. pos_offset-1)."""
        lw = self.layers[l]
        H, dh = self.cfg.n_heads, self.cfg.d_head
        n = hidden.shape[0]
        normed = self.layer_norm(hidden)
        q, k, v = normed @ lw.wq, normed @ lw.wk, normed @ lw.wv
        K = np.concatenate([k_cache, k]) if k_cache is not None else k
        Vv = np.concatenate([v_cache, v]) if v_cache is not None else v
        base = K.shape[0] - n  # keys before the new rows
        attn = np.empty_like(q)
        scale = 1.0 / np.sqrt(float(dh))
        for h in range(H):
            sl = slice(h * dh, (h + 1) * dh)
            s = (q[:, sl] @ K[:, sl].T) * scale
            vis = np.arange(K.shape[0])[None, :] <= (base + np.arange(n))[:, None]
            s = np.where(vis, s, -np.inf)
            m = s.max(axis=1, keepdims=True)
            w = np.exp(s - m)
            attn[:, sl] = (w @ Vv[:, sl]) / w.sum(axis=1, keepdims=True)
        x = hidden + attn @ lw.wo
        h1 = self.layer_norm(x) @ lw.w1 + lw.b1
        h1 = np.where(h1 < 0.0, 0.0, h1)
        out = x + h1 @ lw.w2 + lw.b2
        return out, k, v

    def unembed_logits(self, row: np.ndarray) -> np.ndarray:
        return (self.layer_norm(row[None, :]) @ self.unembed)[0]

    @staticmethod
    def argmax_token(logits) -> int:
        return int(np.argmax(np.asarray(logits)))  # first index of the maximum


@dataclass
class Session:
    """SegmentedCache of one session as concatenated per-layer K/V (positions
    0 .. end-1) — the monolithic view the spliced cache must equal."""
    model: Model
    k: list = field(default_factory=list)
    v: list = field(default_factory=list)

    @property
    def end_position(self) -> int:
        return 0 if not self.k else self.k[0].shape[0]

    def prefill(self, tokens):
        """prefill (model.cpp:211-236) + cache.append: returns the final
        hidden rows of the new tokens."""
        m = self.model
        pos = self.end_position
        hidden = m.embed(tokens, pos)
        new_k, new_v = [], []
        for l in range(m.cfg.n_layers):
            kc = self.k[l] if self.k else None
            vc = self.v[l] if self.v else None
            hidden, k, v = m.layer(l, hidden, pos, kc, vc)
            new_k.append(k)
            new_v.append(v)
        if self.k:
            self.k = [np.concatenate([a, b]) for a, b in zip(self.k, new_k)]
            self.v = [np.concatenate([a, b]) for a, b in zip(self.v, new_v)]
        else:
            self.k, self.v = new_k, new_v
        return hidden

    def decode_step(self, last: int):
        """decode_step (model.cpp:257-283): (next token, logits)."""
        hidden = self.prefill([last])
        logits = self.model.unembed_logits(hidden[-1])
        return Model.argmax_token(logits), logits


def generate_split(model: Model, cloud, edge, n_steps: int):
    s = Session(model)
    s.prefill(cloud)
    hidden = s.prefill(edge)
    return _greedy(model, s, hidden, n_steps)


def generate_monolithic(model: Model, prompt, n_steps: int):
    s = Session(model)
    hidden = s.prefill(prompt)
    return _greedy(model, s, hidden, n_steps)


def _greedy(model: Model, s: Session, hidden, n_steps: int):
    """decode_greedy (model.cpp:285-297)."""
    out = []
    if n_steps == 0:
        return out
    out.append(Model.argmax_token(model.unembed_logits(hidden[-1])))
    while len(out) < n_steps:
        out.append(s.decode_step(out[-1])[0])
    return out
