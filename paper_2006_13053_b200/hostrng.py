"""Seed streams of the sfft driver: numpy's PCG64/SeedSequence, natively.

The reference derives every per-iteration stream as
``default_rng(SeedSequence((master, tag, t, i)))`` (latfft/dimincr.py:99-100)
and draws coordinate-line nodes (``uniform(size=d)``, :137-141), fixed tails
(``uniform(size=d-t-1)``, :231-232) and lattice generators
(``integers(0, M, size=(L, d))``, lattice.py:225-227) from it.  ``Streams``
holds a batch of such generators as one (rows, 6) uint64 state array and
draws from all of them in one call into csrc/hostrng.cpp -- the same numbers
numpy produces (tests/test_host.py pins this against numpy), without ~25 us
of Python per stream on the driver's critical path.

Any draw outside these three forms goes through ``Stream.numpy()``, a real
numpy Generator carrying the identical state.
"""

from __future__ import annotations

import numpy as np

from . import _native


def _words(x):
    """SeedSequence's uint32 words of one non-negative int (bit_generator.pyx
    _int_to_uint32_array)."""
    x = int(x)
    if x < 0:
        raise ValueError("expected non-negative integer")
    if x == 0:
        return [0]
    out = []
    while x > 0:
        out.append(x & 0xFFFFFFFF)
        x >>= 32
    return out


def _ptr(a):
    return a.ctypes.data


class Streams:
    """rows independent PCG64 generators seeded from entropy tuples."""

    __slots__ = ("state",)

    def __init__(self, entropies):
        words = [sum((_words(v) for v in e), []) for e in entropies]
        nw = {len(w) for w in words}
        self.state = np.zeros((len(words), 6), dtype=np.uint64)
        if not words:
            return
        if len(nw) == 1:
            arr = np.ascontiguousarray(words, dtype=np.uint32)
            _native.check(_native.lib().sfftb_pcg64_seed(_ptr(arr), len(words), nw.pop(),
                                                         _ptr(self.state)), "pcg64_seed")
        else:
            for r, w in enumerate(words):
                arr = np.ascontiguousarray(w, dtype=np.uint32)
                _native.check(_native.lib().sfftb_pcg64_seed(
                    _ptr(arr), 1, len(w), _ptr(self.state[r:r + 1])), "pcg64_seed")

    def __len__(self):
        return self.state.shape[0]

    def __getitem__(self, r):
        return Stream(self, r)

    def uniform_each(self, k):
        """(rows, k) float64: ``uniform(size=k)`` from every stream."""
        out = np.empty((len(self), int(k)), dtype=np.float64)
        if out.size:
            _native.check(_native.lib().sfftb_pcg64_random(_ptr(self.state), len(self), int(k),
                                                           _ptr(out)), "pcg64_random")
        return out

    def integers_each(self, low, high, shape):
        """(rows, *shape) int64: ``integers(low, high, size=shape)`` per stream."""
        shape = tuple(int(v) for v in np.atleast_1d(shape))
        cnt = int(np.prod(shape)) if shape else 1
        out = np.empty((len(self), cnt), dtype=np.int64)
        if cnt and len(self):
            if int(high) <= int(low):
                raise ValueError("low >= high")
            _native.check(_native.lib().sfftb_pcg64_integers(
                _ptr(self.state), len(self), int(low), int(high) - 1, cnt, _ptr(out)),
                "pcg64_integers")
        return out.reshape((len(self),) + shape)


class Stream:
    """One row of a Streams batch with the Generator methods the driver uses."""

    __slots__ = ("_b", "_r")

    def __init__(self, batch, r):
        self._b, self._r = batch, r

    def _one(self):
        sub = Streams.__new__(Streams)
        sub.state = self._b.state[self._r:self._r + 1]
        return sub

    def uniform(self, low=0.0, high=1.0, size=None):
        if low != 0.0 or high != 1.0 or size is None or np.ndim(size) > 0:
            return self._via_numpy("uniform", low, high, size)
        return self._one().uniform_each(size)[0]

    def integers(self, low, high=None, size=None, dtype=np.int64, endpoint=False):
        if high is None or endpoint or np.dtype(dtype) != np.int64 or size is None:
            return self._via_numpy("integers", low, high, size, dtype=dtype, endpoint=endpoint)
        shape = (size,) if np.ndim(size) == 0 else tuple(size)
        return self._one().integers_each(low, high, shape)[0]

    def numpy(self):
        """A numpy Generator with this stream's exact state (advances separately)."""
        s = [int(v) for v in self._b.state[self._r]]
        g = np.random.Generator(np.random.PCG64())
        g.bit_generator.state = {"bit_generator": "PCG64",
                                 "state": {"state": (s[0] << 64) | s[1],
                                           "inc": (s[2] << 64) | s[3]},
                                 "has_uint32": s[4], "uinteger": s[5]}
        return g

    def _via_numpy(self, name, *args, **kw):
        g = self.numpy()
        out = getattr(g, name)(*args, **kw)
        st = g.bit_generator.state
        self._b.state[self._r] = [st["state"]["state"] >> 64,
                                  st["state"]["state"] & 0xFFFFFFFFFFFFFFFF,
                                  st["state"]["inc"] >> 64,
                                  st["state"]["inc"] & 0xFFFFFFFFFFFFFFFF,
                                  st["has_uint32"], st["uinteger"]]
        return out


def _small(v):
    return 0 <= v < (1 << 32)


def grid(master, tag, ts, indices):
    """Streams for SeedSequence((master, tag, t, i)) over t in ts (outer), i in
    indices (inner) -- the entropy words assembled with numpy in one go when
    tag, t and i are single words (always, for the driver)."""
    ts, indices = list(ts), list(indices)
    if not (_small(tag) and all(_small(v) for v in ts) and all(_small(v) for v in indices)):
        return Streams([(master, tag, t, i) for t in ts for i in indices])
    mw = _words(master)
    rows = len(ts) * len(indices)
    arr = np.empty((rows, len(mw) + 3), dtype=np.uint32)
    arr[:, :len(mw)] = mw
    arr[:, len(mw)] = tag
    arr[:, len(mw) + 1] = np.repeat(np.asarray(ts, dtype=np.uint32), len(indices))
    arr[:, len(mw) + 2] = np.tile(np.asarray(indices, dtype=np.uint32), len(ts))
    out = Streams.__new__(Streams)
    out.state = np.zeros((rows, 6), dtype=np.uint64)
    if rows:
        _native.check(_native.lib().sfftb_pcg64_seed(_ptr(arr), rows, arr.shape[1],
                                                     _ptr(out.state)), "pcg64_seed")
    return out


def streams(master, tag, t, indices):
    """Streams for SeedSequence((master, tag, t, i)), i in indices."""
    return grid(master, tag, [t], indices)


# ---------------------------------------------------------------------------
# one numpy Generator's state as the 6-word layout of csrc/hostrng.cpp
# ---------------------------------------------------------------------------

def state6(g):
    """np.uint64[6] of a numpy Generator(PCG64)."""
    st = g.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("only PCG64 generators are restated natively")
    s, inc = st["state"]["state"], st["state"]["inc"]
    return np.array([s >> 64, s & 0xFFFFFFFFFFFFFFFF, inc >> 64, inc & 0xFFFFFFFFFFFFFFFF,
                     st["has_uint32"], st["uinteger"]], dtype=np.uint64)


def set_state6(g, st):
    """Write a 6-word state back into the numpy Generator (numpy continues
    exactly where the native draws stopped)."""
    s = [int(v) for v in st]
    g.bit_generator.state = {"bit_generator": "PCG64",
                             "state": {"state": (s[0] << 64) | s[1],
                                       "inc": (s[2] << 64) | s[3]},
                             "has_uint32": s[4], "uinteger": s[5]}


def advance(st, delta):
    """Advance st (6 words, in place) by delta 64-bit outputs."""
    _native.check(_native.lib().sfftb_pcg64_advance(_ptr(st), int(delta), None), "pcg64_advance")


def jump_tables(st):
    """(256,) uint64: the jump-by-2^i maps of st's LCG (sfftb_box_integers)."""
    tab = np.zeros(256, dtype=np.uint64)
    tmp = st.copy()
    _native.check(_native.lib().sfftb_pcg64_advance(_ptr(tmp), 0, _ptr(tab)), "pcg64_advance")
    return tab


def after_words(st, words_used, last_hi):
    """The state after `words_used` buffered 32-bit words were drawn from st
    (numpy's next_uint32 buffering); last_hi = the high half of the 64-bit
    output holding the last word."""
    out = st.copy()
    j = int(words_used)
    if j <= 0:
        return out
    if out[4]:
        out[4] = 0  # the buffered high half went first
        j -= 1
        if j == 0:
            return out
    advance(out, (j + 1) // 2)
    out[4] = j & 1
    out[5] = int(last_hi)
    return out


def choice_no_replace(g, pop, size):
    """Generator.choice(pop, size, replace=False) with g advanced exactly as
    numpy advances it: numpy's tail-shuffle regime (pop > 10000 and
    size > pop // 50) natively (csrc/hostrng.cpp), Floyd's regime by numpy."""
    pop, size = int(pop), int(size)
    if not (pop > 10000 and size > pop // 50):
        return g.choice(pop, size=size, replace=False)
    st = state6(g)
    out = np.empty(size, dtype=np.int64)
    _native.check(_native.lib().sfftb_pcg64_choice_tail(_ptr(st), pop, size, 0, _ptr(out)),
                  "pcg64_choice_tail")
    set_state6(g, st)
    return out
