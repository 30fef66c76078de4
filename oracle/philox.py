"""Counter-based Philox4x64-10 restated in numpy uint64 arithmetic (oracle only).

numpy's ``np.random.Philox`` (the generator the reference draws every sample
key from, ``sampler.py:105,125`` and ``trainer.py:40-42``) is a Random123
Philox4x64 with 10 rounds.  Its stream contract, verified against numpy 2.3.5:

* key   = ``SeedSequence(seed).generate_state(2, uint64)``
* draw j (0-based, per generator) = word ``j % 4`` of
  ``philox(counter=(j // 4 + 1, 0, 0, 0), key)`` -- numpy increments the
  counter *before* the first block, so block 0 uses counter 1;
* ``Generator.random()`` returns ``(word >> 11) * 2**-53``; comparing the
  53-bit integer ``word >> 11`` orders draws identically, including ties.
"""

from __future__ import annotations

import numpy as np

M0 = np.uint64(0xD2E7470EE14C6C93)
M1 = np.uint64(0xCA5A826395121157)
W0 = np.uint64(0x9E3779B97F4A7C15)
W1 = np.uint64(0xBB67AE8584CAA73B)
_LO32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)
_S11 = np.uint64(11)


def _mul_hi_lo(a: np.ndarray, m: np.uint64):
    """128-bit product of uint64 arrays with a constant, as (hi, lo)."""
    a_lo, a_hi = a & _LO32, a >> _S32
    m_lo, m_hi = m & _LO32, m >> _S32
    ll, lh, hl, hh = a_lo * m_lo, a_lo * m_hi, a_hi * m_lo, a_hi * m_hi
    carry = ((ll >> _S32) + (lh & _LO32) + (hl & _LO32)) >> _S32
    return hh + (lh >> _S32) + (hl >> _S32) + carry, a * m


def philox4x64_10(c0, c1, c2, c3, k0, k1):
    """Ten Philox rounds on counter words (arrays) under key (k0, k1)."""
    c0, c1, c2, c3 = (np.asarray(c, dtype=np.uint64) for c in (c0, c1, c2, c3))
    k0, k1 = np.uint64(k0), np.uint64(k1)
    with np.errstate(over="ignore"):
        for _ in range(10):
            h0, l0 = _mul_hi_lo(c0, M0)
            h1, l1 = _mul_hi_lo(c2, M1)
            c0, c1, c2, c3 = h1 ^ c1 ^ k0, l1, h0 ^ c3 ^ k1, l0
            k0 = k0 + W0
            k1 = k1 + W1
    return c0, c1, c2, c3


def key_for_seed(seed: int) -> tuple[int, int]:
    """Philox key of ``np.random.Philox(seed)`` (SeedSequence-derived)."""
    k = np.random.SeedSequence(int(seed)).generate_state(2, np.uint64)
    return int(k[0]), int(k[1])


def raw_words(key: tuple[int, int], start: int, count: int) -> np.ndarray:
    """uint64 stream words at absolute draw positions [start, start+count)."""
    if count <= 0:
        return np.empty(0, dtype=np.uint64)
    b0 = start // 4
    b1 = (start + count - 1) // 4 + 1
    ctr = np.arange(b0 + 1, b1 + 1, dtype=np.uint64)
    zero = np.zeros_like(ctr)
    words = np.stack(philox4x64_10(ctr, zero, zero, zero, key[0], key[1]), axis=1).reshape(-1)
    off = start - 4 * b0
    return words[off : off + count]


def keys53(key: tuple[int, int], start: int, count: int) -> np.ndarray:
    """The 53-bit integer behind ``Generator.random()`` at each position."""
    return raw_words(key, start, count) >> _S11


def uniform(key: tuple[int, int], start: int, count: int) -> np.ndarray:
    """float64 uniforms identical to ``Generator(Philox(seed)).random``."""
    return keys53(key, start, count).astype(np.float64) * (2.0 ** -53)
