"""Pure-Python restatement of numpy's seeding + PCG64 + 3-of-n choice stream.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Third-party algorithm: numpy 2.3.5 (not vendored under /root/reference; the
reference pins only ``numpy>=1.24`` at ``pkg/pyproject.toml:11``).  Call sites
in the reference: ``np.random.default_rng(cfg.seed)`` (``posest.py:243``) and
``rng.choice(n, size=3, replace=False)`` once per minimal sample
(``posest.py:252``).  Restated from numpy's published algorithm:

* ``SeedSequence(seed).generate_state(4, uint64)``: 4-word entropy pool mixed
  with the hashmix/mix constants, then words drawn with a second hash chain.
* ``PCG64``: 128-bit LCG, ``state = state * M + inc``; output XSL-RR
  ``rotr64(hi ^ lo, state >> 122)``.  Seeding: ``state = 0; inc = (seq<<1)|1;
  step; state += initstate; step``.
* ``next_uint32`` buffers the high half of a 64-bit output.
* bounded draw in ``[0, j]``: ``j == 0`` → 0 without a draw; else Lemire's
  multiply-shift with rejection while ``lo32(m) < (2^32-1-j) % (j+1)``.
* ``choice(n, 3, replace=False)``: Floyd's algorithm over j = n-3..n-1
  (use j when the drawn value is already taken), then a tail shuffle
  (i = 2, 1: swap(out[bounded(i)], out[i])).

Pinned against golden sample sets produced by numpy itself
(``tests/golden/rng.npz``).
"""

from __future__ import annotations

MASK32 = (1 << 32) - 1
MASK64 = (1 << 64) - 1
MASK128 = (1 << 128) - 1
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645

# SeedSequence constants (numpy/random/bit_generator.pyx)
_INIT_A = 0x43B0D7E5
_MULT_A = 0x931E8875
_INIT_B = 0x8B51F9DD
_MULT_B = 0x58F38DED
_MIX_MULT_L = 0xCA01F9DD
_MIX_MULT_R = 0x4973F715
_XSHIFT = 16
_POOL = 4


def _entropy_words(seed: int) -> list[int]:
    if seed < 0:
        raise ValueError("seed must be non-negative")
    words = []
    while True:
        words.append(seed & MASK32)
        seed >>= 32
        if seed == 0:
            break
    return words


def seed_sequence_pool(seed: int) -> list[int]:
    """Mixed entropy pool of ``SeedSequence(seed)``."""
    entropy = _entropy_words(seed)
    hc = [_INIT_A]

    def hashmix(v):
        v = (v ^ hc[0]) & MASK32
        hc[0] = (hc[0] * _MULT_A) & MASK32
        v = (v * hc[0]) & MASK32
        return v ^ (v >> _XSHIFT)

    def mix(x, y):
        r = (_MIX_MULT_L * x - _MIX_MULT_R * y) & MASK32
        return r ^ (r >> _XSHIFT)

    pool = [hashmix(entropy[i] if i < len(entropy) else 0) for i in range(_POOL)]
    for src in range(_POOL):
        for dst in range(_POOL):
            if src != dst:
                pool[dst] = mix(pool[dst], hashmix(pool[src]))
    for src in range(_POOL, len(entropy)):
        for dst in range(_POOL):
            pool[dst] = mix(pool[dst], hashmix(entropy[src]))
    return pool


def seed_sequence_state64(seed: int, n_words: int = 4) -> list[int]:
    pool = seed_sequence_pool(seed)
    hc = _INIT_B
    w32 = []
    for i in range(2 * n_words):
        v = pool[i % _POOL] ^ hc
        hc = (hc * _MULT_B) & MASK32
        v = (v * hc) & MASK32
        w32.append(v ^ (v >> _XSHIFT))
    return [w32[2 * i] | (w32[2 * i + 1] << 32) for i in range(n_words)]


class PCG64Stream:
    """numpy ``PCG64`` with the ``next_uint32`` half-word buffer."""

    def __init__(self, state: int, inc: int, has_uint32: int = 0, uinteger: int = 0):
        self.state = state & MASK128
        self.inc = inc & MASK128
        self.has_uint32 = int(has_uint32)
        self.uinteger = uinteger & MASK32

    @classmethod
    def from_seed(cls, seed: int) -> "PCG64Stream":
        v = seed_sequence_state64(seed, 4)
        initstate = (v[0] << 64) | v[1]
        initseq = (v[2] << 64) | v[3]
        inc = ((initseq << 1) | 1) & MASK128
        s = (0 * PCG_MULT + inc) & MASK128
        s = (s + initstate) & MASK128
        s = (s * PCG_MULT + inc) & MASK128
        return cls(s, inc)

    def next64(self) -> int:
        self.state = (self.state * PCG_MULT + self.inc) & MASK128
        hi = self.state >> 64
        lo = self.state & MASK64
        x = hi ^ lo
        rot = self.state >> 122
        return ((x >> rot) | (x << ((64 - rot) & 63))) & MASK64

    def next32(self) -> int:
        if self.has_uint32:
            self.has_uint32 = 0
            return self.uinteger
        v = self.next64()
        self.has_uint32 = 1
        self.uinteger = v >> 32
        return v & MASK32

    def bounded(self, j: int) -> int:
        """Uniform integer in [0, j] (numpy ``random_bounded_uint64``, 32-bit range)."""
        if j == 0:
            return 0
        if j > MASK32 - 1:
            raise NotImplementedError("populations above 2^32-1 are not on the path")
        excl = j + 1
        m = self.next32() * excl
        left = m & MASK32
        if left < excl:
            thr = (MASK32 - j) % excl
            while left < thr:
                m = self.next32() * excl
                left = m & MASK32
        return m >> 32

    def choice3(self, n: int) -> list[int]:
        """``Generator.choice(n, 3, replace=False)``."""
        if n < 3:
            raise ValueError("population smaller than the sample")
        out = []
        for j in range(n - 3, n):
            v = self.bounded(j)
            out.append(j if v in out else v)
        for i in (2, 1):
            k = self.bounded(i)
            out[k], out[i] = out[i], out[k]
        return out

    def state_dict(self) -> dict:
        return {"state": self.state, "inc": self.inc,
                "has_uint32": self.has_uint32, "uinteger": self.uinteger}


def sample_batches(seed: int, n: int, batch_sizes) -> list[list[list[int]]]:
    """Minimal sample sets in the order ``ransac_pnp`` draws them."""
    g = PCG64Stream.from_seed(seed)
    return [[g.choice3(n) for _ in range(b)] for b in batch_sizes]
