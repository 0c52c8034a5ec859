"""Counter-based noise (drop-in for ``sdebatch.rng``,
/root/reference/pkg/src/sdebatch/rng.py).

Array generation runs on the GPU with the same device functions the fused
stepper uses, so ``normals_for_orbits`` returns exactly the draws the stepper
consumes.  Philox words are bit-exact with the reference; normals match to
the last few ulps (device log/sqrt/sincos vs numpy).  The scalar helpers
(``to_uniform``, ``box_muller``, ``counter_key``) are plain host arithmetic,
as in the reference.

Additional streams (not in the reference):
``sfc64`` and ``xoshiro256pp``, one stream per (orbit, 4-normal block)
seeded by SplitMix64 from (seed, global orbit, block), consumed at two 64-bit
outputs per block per step.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _native as nat

PHILOX_M0 = 0xD2511F53
PHILOX_M1 = 0xCD9E8D57
PHILOX_W0 = 0x9E3779B9
PHILOX_W1 = 0xBB67AE85
PHILOX_ROUNDS = 10

_MASK32 = 0xFFFFFFFF
_MASK64 = 0xFFFFFFFFFFFFFFFF

#: counter word reserved for parameter-sampling streams (rng.py:41-42)
SAMPLING_TAG = 0xFFFFFFFF

_TWO_NEG_32 = 2.0 ** -32
_TWO_PI = 2.0 * math.pi

STREAMS = tuple(nat.STREAM_IDS)


@dataclass(frozen=True)
class CounterKey:
    """Address of one Philox block (rng.py:48-53)."""

    key: tuple[int, int]
    counter: tuple[int, int, int, int]


def counter_key(seed: int, orbit: int, chunk: int, step: int, block: int) -> CounterKey:
    """Injective packing of a draw address (rng.py:56-71)."""
    if not 0 <= orbit <= _MASK32:
        raise ValueError("orbit index must fit in 32 bits, got %r" % (orbit,))
    if not 0 <= chunk <= _MASK32 or not 0 <= step <= _MASK32 or not 0 <= block <= _MASK32:
        raise ValueError("counter words must fit in 32 bits")
    seed &= _MASK64
    return CounterKey(key=(seed & _MASK32, orbit), counter=(seed >> 32, chunk, step, block))


def _philox_words(k0, k1, c0, c1, c2, c3):
    """Philox-4x32-10 over broadcast uint32 arrays, on the device (rng.py:93-118)."""
    arrs = np.broadcast_arrays(*(np.asarray(x, dtype=np.uint32) for x in (k0, k1, c0, c1, c2, c3)))
    shape = arrs[0].shape
    packed = np.ascontiguousarray(np.stack([a.reshape(-1) for a in arrs], axis=-1), dtype=np.uint32)
    out = np.empty((packed.shape[0], 4), dtype=np.uint32)
    if packed.shape[0]:
        ctx = nat.context()
        nat.check(nat.lib().sdb_philox_words(ctx, nat.u32ptr(packed), packed.shape[0],
                                             nat.u32ptr(out)), ctx, "sdb_philox_words")
    return tuple(out[:, k].reshape(shape) for k in range(4))


def philox_block(ck: CounterKey) -> tuple[int, int, int, int]:
    """One Philox block (rng.py:74-90)."""
    words = _philox_words(ck.key[0], ck.key[1], *ck.counter)
    return tuple(int(w) for w in words)


def to_uniform(word):
    """(word + 1) / 2**32 on (0, 1] (rng.py:121-129).

    Like ``box_muller`` below, a scalar helper of the reference's public API
    (its tests use them as the scalar oracle of the normal transform), kept
    on the host: one exact addition and scaling, never on the run path --
    the stepper forms the same uniform on the device (csrc/sdeb_math.cuh)."""
    if isinstance(word, np.ndarray):
        return (word.astype(np.float64) + 1.0) * _TWO_NEG_32
    return (float(word) + 1.0) * _TWO_NEG_32


def box_muller(u1: float, u2: float) -> tuple[float, float]:
    """Scalar Box-Muller (rng.py:132-142); host scalar helper (see to_uniform).
    Batched normals come from the device (``normals_for_orbits``)."""
    if u1 <= 0.0:
        raise ValueError("box_muller requires u1 > 0, got %r" % (u1,))
    r = math.sqrt(-2.0 * math.log(u1))
    a = _TWO_PI * u2
    return (r * math.cos(a), r * math.sin(a))


def _seed_words(seed: int) -> tuple[int, int]:
    seed &= _MASK64
    return seed & _MASK32, seed >> 32


def normals_for_orbits(seed: int, orbits: np.ndarray, chunk: int, step: int, m: int,
                       stream: str = "philox") -> np.ndarray:
    """Standard normals for one step of a group of orbits, shape (len(orbits), m)
    (rng.py:150-188), generated on the device."""
    orbits = np.ascontiguousarray(np.asarray(orbits, dtype=np.uint32).reshape(-1))
    if m < 0:
        raise ValueError("noise count must be >= 0")
    if m == 0:
        return np.empty((orbits.size, 0), dtype=np.float64)
    if stream == "philox" and chunk == SAMPLING_TAG:
        raise ValueError("counter word 0x%08X is reserved for sampling streams" % SAMPLING_TAG)
    out = np.empty((orbits.size, m), dtype=np.float64)
    if orbits.size:
        ctx = nat.context()
        nat.check(nat.lib().sdb_normals(ctx, nat.STREAM_IDS[stream], int(seed) & _MASK64,
                                        nat.u32ptr(orbits), orbits.size, int(chunk) & _MASK32,
                                        int(step) & _MASK32, int(m), nat.dptr(out)),
                  ctx, "sdb_normals")
    return out


def normals_for_step(seed: int, orbit: int, chunk: int, step: int, m: int,
                     stream: str = "philox") -> np.ndarray:
    """rng.py:191-197."""
    return normals_for_orbits(seed, np.array([orbit], dtype=np.uint32), chunk, step, m, stream)[0]


def sampling_uniforms(seed: int, orbits: np.ndarray, count: int) -> np.ndarray:
    """Reserved-tag uniforms on [0, 1), shape (len(orbits), count) (rng.py:200-222)."""
    orbits = np.ascontiguousarray(np.asarray(orbits, dtype=np.uint32).reshape(-1))
    if count < 0:
        raise ValueError("count must be >= 0")
    if count == 0:
        return np.empty((orbits.size, 0), dtype=np.float64)
    out = np.empty((orbits.size, count), dtype=np.float64)
    if orbits.size:
        ctx = nat.context()
        nat.check(nat.lib().sdb_sampling_uniforms(ctx, int(seed) & _MASK64, nat.u32ptr(orbits),
                                                  orbits.size, int(count), nat.dptr(out)),
                  ctx, "sdb_sampling_uniforms")
    return out


def stream_raw(stream: str, seed: int, orbit: int, block: int, count: int) -> np.ndarray:
    """First ``count`` raw 64-bit outputs of one sfc64/xoshiro256pp stream."""
    out = np.empty(count, dtype=np.uint64)
    if count:
        ctx = nat.context()
        nat.check(nat.lib().sdb_stream_raw(ctx, nat.STREAM_IDS[stream], int(seed) & _MASK64,
                                           int(orbit), int(block), int(count), nat.u64ptr(out)),
                  ctx, "sdb_stream_raw")
    return out
