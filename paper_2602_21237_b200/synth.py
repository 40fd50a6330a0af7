"""Seeded synthetic relations: the reference generator and the BASELINE configs.

``GenSpec`` / ``generate_relation`` restate the reference's documented
sampling procedure (relation.py:234-295) so identical specs give
bit-identical relations on a box without ``relab``:

    rng = np.random.default_rng(seed)
    uniform:  keys = rng.integers(0, key_domain, n, dtype=int64)
    zipf(s):  u = rng.random(n); c = cumsum(r ** -s, r = 1..key_domain)
              keys = searchsorted(c, u * c[-1], side="right")
    payload = rng.integers(0, 256, (n, payload_width), dtype=uint8)

The ``cfgN_*`` builders follow SURVEY.md §8(d) for BASELINE.json configs 1-5
(all inputs synthetic; no public dataset is involved).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Union

import numpy as np

from .records import Bytes, Int64, Relation, Schema


@dataclass(frozen=True)
class Uniform:
    """Keys uniform over [0, key_domain)."""


@dataclass(frozen=True)
class Zipf:
    """Keys Zipf(s) over ranks [0, key_domain)."""

    s: float

    def __post_init__(self) -> None:
        if not self.s > 0:
            raise ValueError(f"zipf exponent must be > 0, got {self.s}")


@dataclass(frozen=True)
class GenSpec:
    n: int
    key_domain: int
    distribution: Union[Uniform, Zipf] = Uniform()
    payload_width: int = 8
    seed: int = 0
    clustered: bool = False

    def __post_init__(self) -> None:
        if self.n < 0:
            raise ValueError("n must be >= 0")
        if self.key_domain < 1:
            raise ValueError("key_domain must be >= 1")
        if self.payload_width < 0:
            raise ValueError("payload_width must be >= 0")


def zipf_ranks(rng: np.random.Generator, n: int, domain: int, s: float) -> np.ndarray:
    weights = np.cumsum(np.arange(1, domain + 1, dtype=np.float64) ** -s)
    return np.searchsorted(weights, rng.random(n) * weights[-1], side="right").astype(np.int64)


def generate_relation(spec: GenSpec) -> Relation:
    rng = np.random.default_rng(spec.seed)
    if isinstance(spec.distribution, Zipf):
        keys = zipf_ranks(rng, spec.n, spec.key_domain, spec.distribution.s)
    else:
        keys = rng.integers(0, spec.key_domain, spec.n, dtype=np.int64)
    if spec.clustered:
        keys = np.sort(keys)
    payload = rng.integers(0, 256, (spec.n, spec.payload_width), dtype=np.uint8)
    return Relation(Schema((("key", Int64()), ("payload", Bytes(spec.payload_width)))), (keys, payload))


KEY_PAYLOAD = Schema((("key", Int64()), ("payload", Int64())))


def uniform_keys(n: int, domain: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).integers(0, domain, n, dtype=np.int64)


def cfg1_relations(n: int = 1_000_000, domain: int = 1_000_000, seed: int = 0):
    """BASELINE cfg1 (and cfg5 with domain = n): R seed s, S seed s+1
    (bench.py:163-166 convention), int64 payload = row index."""
    pay = np.arange(n, dtype=np.int64)
    r = Relation(KEY_PAYLOAD, (uniform_keys(n, domain, seed), pay))
    s = Relation(KEY_PAYLOAD, (uniform_keys(n, domain, seed + 1), pay))
    return r, s


def cfg2_relation(n: int = 10_000_000, seed: int = 0) -> Relation:
    """BASELINE cfg2: full-range int64 keys, ~1% duplicates copied from random
    earlier rows, int32 payload carried as Bytes(4) little-endian."""
    rng = np.random.default_rng(seed)
    keys = rng.integers(np.iinfo(np.int64).min, np.iinfo(np.int64).max, n, dtype=np.int64, endpoint=True)
    n_dup = n // 100
    if n_dup and n > 1:
        dst = rng.choice(np.arange(1, n), n_dup, replace=False)
        src = (rng.random(n_dup) * dst).astype(np.int64)
        keys[dst] = keys[src]
    payload = rng.integers(0, 2**32, n, dtype=np.uint32).view(np.int32)
    schema = Schema((("key", Int64()), ("payload", Bytes(4))))
    return Relation(schema, (keys, payload.view(np.uint8).reshape(n, 4)))


def cfg3_relations(n: int = 10_000_000, domain: int = 1_000_000, s: float = 1.1, seed: int = 0,
                   perm_seed: int = 1000):
    """BASELINE cfg3: Zipf(s) ranks from the reference sampler, mapped to key
    ids through one shared permutation (default_rng(perm_seed))."""
    ids = np.random.default_rng(perm_seed).permutation(domain).astype(np.int64)
    pay = np.arange(n, dtype=np.int64)
    out = []
    for sd in (seed, seed + 1):
        ranks = zipf_ranks(np.random.default_rng(sd), n, domain, s)
        out.append(Relation(KEY_PAYLOAD, (ids[ranks], pay)))
    return tuple(out)


def cfg4_relations(n: int = 100_000_000, seed: int = 0):
    """BASELINE cfg4: key = (a << 32) | b with a, b uniform int32 in [0, 2^16)
    (the composite key packed into one int64; the reference has only
    single-attribute Int64 join keys), 16-byte payload."""
    schema = Schema((("key", Int64()), ("payload", Bytes(16))))
    out = []
    for sd in (seed, seed + 1):
        rng = np.random.default_rng(sd)
        a = rng.integers(0, 2**16, n, dtype=np.int32)
        b = rng.integers(0, 2**16, n, dtype=np.int32)
        key = (a.astype(np.int64) << 32) | b.astype(np.int64)
        payload = rng.integers(0, 256, (n, 16), dtype=np.uint8)
        out.append(Relation(schema, (key, payload)))
    return tuple(out)
