"""Seeding: per-filter Philox4x32-10 keys derived from numpy SeedSequences.

The reference gives filter m the stream ``default_rng(SeedSequence(master)
.spawn(M)[m])`` (ensemble.py:56-60, filters.py:177).  The GPU bank keeps the
same seed tree but turns each child SeedSequence into a 64-bit Philox key
(``generate_state(2, uint32)``); every draw is then a pure function of
(key, counter), counters being built from (particle, time, draw, purpose).
Consequences, mirroring the reference's guarantees:

* ``run_ensemble(M=1, master)`` equals ``run_filter(filter_seeds(master,1)[0])``
  bit for bit (test_ensemble.py:24-29 analogue);
* results are independent of how filters are sharded across GPUs
  (the reference's workers-independence, test_ensemble.py:59-65).

``philox4x32_10`` is a numpy mirror of the device function used by the
known-answer tests.
"""

from __future__ import annotations

import functools

import numpy as np

M0, M1 = 0xD2511F53, 0xCD9E8D57
W0, W1 = 0x9E3779B9, 0xBB67AE85
MASK = 0xFFFFFFFF


def as_seed_sequence(seed):
    if isinstance(seed, np.random.SeedSequence):
        return seed
    if isinstance(seed, np.random.Generator):
        # a Generator passed as seed: derive a child sequence from its stream
        return np.random.SeedSequence(seed.integers(0, 2**63, size=4, dtype=np.uint64).tolist())
    return np.random.SeedSequence(seed)


def seed_key(seed) -> np.ndarray:
    """64-bit Philox key (2 x uint32) of one filter's seed."""
    return as_seed_sequence(seed).generate_state(2, dtype=np.uint32)


def filter_seeds(master_seed, n_filters):
    """Per-filter seed sequences: children spawn(n_filters) of the master
    (ensemble.py:56-60)."""
    return as_seed_sequence(master_seed).spawn(n_filters)


def filter_keys(master_seed, n_filters) -> np.ndarray:
    """(n_filters, 2) uint32 keys for the bank (cached for int seeds: the
    SeedSequence tree is deterministic and spawning is ~15 us per filter)."""
    if isinstance(master_seed, (int, np.integer)) and not isinstance(master_seed, bool):
        return _filter_keys_cached(int(master_seed), int(n_filters)).copy()
    return np.stack([seed_key(s) for s in filter_seeds(master_seed, n_filters)]).astype(np.uint32)


@functools.lru_cache(maxsize=32)
def _filter_keys_cached(master_seed: int, n_filters: int) -> np.ndarray:
    return np.stack([seed_key(s) for s in filter_seeds(master_seed, n_filters)]).astype(np.uint32)


def philox4x32_10(ctr, key):
    """numpy mirror: ctr (n,4) uint32, key (n,2) uint32 -> (n,4) uint32."""
    c = np.asarray(ctr, dtype=np.uint64).reshape(-1, 4).copy()
    k = np.asarray(key, dtype=np.uint64).reshape(-1, 2).copy()
    for _ in range(10):
        p0 = c[:, 0] * M0
        p1 = c[:, 2] * M1
        hi0, lo0 = p0 >> 32, p0 & MASK
        hi1, lo1 = p1 >> 32, p1 & MASK
        c = np.stack([hi1 ^ c[:, 1] ^ k[:, 0], lo1, hi0 ^ c[:, 3] ^ k[:, 1], lo0], axis=1)
        k = np.stack([(k[:, 0] + W0) & MASK, (k[:, 1] + W1) & MASK], axis=1)
    return c.astype(np.uint32)
