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


# numpy SeedSequence constants (numpy/random/bit_generator.pyx: hashmix, mix,
# mix_entropy, generate_state); restated vectorised over many sequences so a
# bank of thousands of filters derives its keys in one numpy pass instead of
# one SeedSequence object per filter (~6 us spawn + ~2 us generate_state each)
_INIT_A, _MULT_A = 0x43B0D7E5, 0x931E8875
_INIT_B, _MULT_B = 0x8B51F9DD, 0x58F38DED
_MIX_L, _MIX_R = 0xCA01F9DD, 0x4973F715
_POOL = 4


def _words(x) -> list[int]:
    """numpy's _coerce_to_uint32_array for ints and (nested) int sequences."""
    if isinstance(x, (int, np.integer)):
        x = int(x)
        if x < 0:
            raise ValueError("SeedSequence entropy must be non-negative")
        out = [x & MASK]
        x >>= 32
        while x:
            out.append(x & MASK)
            x >>= 32
        return out
    out: list[int] = []
    for e in x:
        out += _words(e)
    return out


def _keys_from_words(cols: list[np.ndarray]) -> np.ndarray:
    """generate_state(2, uint32) of SeedSequences whose assembled entropy
    words are the columns ``cols`` (each a (n,) uint64 array)."""
    n = cols[0].shape[0]
    u = np.uint64
    hc = _INIT_A

    def hashmix(v):
        nonlocal hc
        v = (v ^ u(hc)) & u(MASK)
        hc = (hc * _MULT_A) & MASK
        v = (v * u(hc)) & u(MASK)
        return v ^ (v >> u(16))

    def mix(x, y):
        r = (u(_MIX_L) * x - u(_MIX_R) * y) & u(MASK)
        return r ^ (r >> u(16))

    zero = np.zeros(n, dtype=np.uint64)
    mixer = [hashmix(cols[i] if i < len(cols) else zero) for i in range(_POOL)]
    for s in range(_POOL):
        for d in range(_POOL):
            if s != d:
                mixer[d] = mix(mixer[d], hashmix(mixer[s]))
    for s in range(_POOL, len(cols)):
        for d in range(_POOL):
            mixer[d] = mix(mixer[d], hashmix(cols[s]))
    h = _INIT_B
    out = np.empty((n, 2), dtype=np.uint32)
    for i in range(2):
        v = mixer[i] ^ u(h)
        h = (h * _MULT_B) & MASK
        v = (v * u(h)) & u(MASK)
        out[:, i] = (v ^ (v >> u(16))).astype(np.uint32)
    return out


def _run_words(ss: np.random.SeedSequence, spawned: bool) -> list[int]:
    run = _words(ss.entropy)
    if spawned and len(run) < _POOL:
        run += [0] * (_POOL - len(run))
    return run


def child_keys(parent: np.random.SeedSequence, start: int, n: int) -> np.ndarray:
    """Keys of the children ``start .. start+n-1`` of ``parent`` (the
    sequences ``parent.spawn`` creates, spawn_key + (index,)), vectorised."""
    if parent.pool_size != _POOL or start + n > MASK:
        kids = [np.random.SeedSequence(parent.entropy,
                                       spawn_key=tuple(parent.spawn_key) + (start + i,),
                                       pool_size=parent.pool_size) for i in range(n)]
        return np.stack([k.generate_state(2, dtype=np.uint32) for k in kids]).astype(np.uint32)
    head = _run_words(parent, True) + _words(parent.spawn_key)
    cols = [np.full(n, w, dtype=np.uint64) for w in head]
    cols.append(np.arange(start, start + n, dtype=np.uint64))
    return _keys_from_words(cols)


def seed_keys(seeds) -> np.ndarray:
    """(len(seeds), 2) uint32 keys, one per seed, vectorised over seeds whose
    assembled entropy has the same length (e.g. spawn_child siblings)."""
    seqs = [as_seed_sequence(s) for s in seeds]
    out = np.empty((len(seqs), 2), dtype=np.uint32)
    groups: dict[int, list[tuple[int, list[int]]]] = {}
    for i, ss in enumerate(seqs):
        if ss.pool_size != _POOL:
            out[i] = ss.generate_state(2, dtype=np.uint32)
            continue
        spawn = _words(ss.spawn_key)
        w = _run_words(ss, len(spawn) > 0) + spawn
        groups.setdefault(len(w), []).append((i, w))
    for rows in groups.values():
        idx = np.array([i for i, _ in rows])
        mat = np.array([w for _, w in rows], dtype=np.uint64)
        out[idx] = _keys_from_words([mat[:, j].copy() for j in range(mat.shape[1])])
    return out


def seed_key(seed) -> np.ndarray:
    """64-bit Philox key (2 x uint32) of one filter's seed."""
    return as_seed_sequence(seed).generate_state(2, dtype=np.uint32)


def filter_seeds(master_seed, n_filters):
    """Per-filter seed sequences: children spawn(n_filters) of the master
    (ensemble.py:56-60; a SeedSequence master is advanced like the
    reference's)."""
    return as_seed_sequence(master_seed).spawn(n_filters)


class FilterSeeds:
    """The children ``start .. start+n-1`` of a master SeedSequence, built on
    first access (the keys do not need the objects)."""

    def __init__(self, parent, start, n, children=None):
        self.parent, self.start, self.n, self._kids = parent, start, n, children

    def __len__(self):
        return self.n

    def __getitem__(self, f):
        if self._kids is None:
            p = self.parent
            self._kids = [np.random.SeedSequence(p.entropy,
                                                 spawn_key=tuple(p.spawn_key) + (self.start + i,),
                                                 pool_size=p.pool_size)
                          for i in range(self.n)]
        return self._kids[f]


def filter_keys_and_seeds(master_seed, n_filters):
    """(keys (n_filters, 2) uint32, FilterSeeds) for an ensemble.  A
    SeedSequence master is advanced by n_filters spawns, exactly like the
    reference's ``filter_seeds`` (ensemble.py:56-60); an int master is not
    an object the caller holds, so nothing is spawned."""
    n_filters = int(n_filters)
    if isinstance(master_seed, np.random.SeedSequence):
        start = master_seed.n_children_spawned
        keys = child_keys(master_seed, start, n_filters)
        kids = master_seed.spawn(n_filters)  # the reference's side effect
        return keys, FilterSeeds(master_seed, start, n_filters, kids)
    ss = as_seed_sequence(master_seed)
    return child_keys(ss, 0, n_filters), FilterSeeds(ss, 0, n_filters)


def filter_keys(master_seed, n_filters) -> np.ndarray:
    """(n_filters, 2) uint32 keys for the bank."""
    return filter_keys_and_seeds(master_seed, n_filters)[0]


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
