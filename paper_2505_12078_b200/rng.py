"""Philox4x32-10 stream, bit-compatible with the reference generator.

Restates ``spock::Philox`` (proj/src/rng.cpp:10-131): key/counter schedule,
53-bit uniforms, Box-Muller normals with one cached spare, exponential-spacing
simplex draws and the row-major ``normal_matrix`` fill order.  The block
function is evaluated with numpy over many counters at once; the consumed
stream is identical to the scalar reference because Philox is counter based.
"""
from __future__ import annotations

import math

import numpy as np

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = 0x9E3779B9
_W1 = 0xBB67AE85
_MASK32 = np.uint64(0xFFFFFFFF)


def _philox_blocks(key0: int, key1: int, ctr: int, count: int) -> np.ndarray:
    """Philox4x32-10 output words for counters ctr..ctr+count-1 (rng.cpp:32-59)."""
    c = np.arange(count, dtype=object) + ctr  # 128-bit counters
    c = np.array([int(v) for v in c], dtype=object)
    w = [np.array([(int(v) >> (32 * k)) & 0xFFFFFFFF for v in c], dtype=np.uint64) for k in range(4)]
    c0, c1, c2, c3 = w
    k0, k1 = key0, key1
    for _ in range(10):
        p0 = _M0 * c0
        p1 = _M1 * c2
        n0 = (p1 >> np.uint64(32)) ^ c1 ^ np.uint64(k0)
        n1 = p1 & _MASK32
        n2 = (p0 >> np.uint64(32)) ^ c3 ^ np.uint64(k1)
        n3 = p0 & _MASK32
        c0, c1, c2, c3 = n0, n1, n2, n3
        k0 = (k0 + _W0) & 0xFFFFFFFF
        k1 = (k1 + _W1) & 0xFFFFFFFF
    out = np.empty((count, 4), dtype=np.uint64)
    out[:, 0], out[:, 1], out[:, 2], out[:, 3] = c0, c1, c2, c3
    return out.reshape(-1)


class Philox:
    """spock::Philox (proj/include/spock/rng.hpp:12-42)."""

    _CHUNK = 4096

    def __init__(self, seed: int, stream: int = 0):
        seed &= (1 << 64) - 1
        self._k0 = seed & 0xFFFFFFFF
        self._k1 = (seed >> 32) & 0xFFFFFFFF
        self._ctr = (stream & ((1 << 64) - 1)) << 64  # counter words 2,3 hold the stream
        self._buf = np.empty(0, dtype=np.uint64)
        self._pos = 0
        self.have_spare = False
        self.spare = 0.0

    def _need(self, n32: int) -> None:
        avail = self._buf.size - self._pos
        if avail >= n32:
            return
        blocks = max(self._CHUNK, (n32 - avail + 3) // 4)
        new = _philox_blocks(self._k0, self._k1, self._ctr, blocks)
        self._ctr = (self._ctr + blocks) & ((1 << 128) - 1)
        self._buf = np.concatenate([self._buf[self._pos:], new])
        self._pos = 0

    def next_u32_array(self, n: int) -> np.ndarray:
        self._need(n)
        out = self._buf[self._pos:self._pos + n]
        self._pos += n
        return out

    def next_u32(self) -> int:
        return int(self.next_u32_array(1)[0])

    def next_u64_array(self, n: int) -> np.ndarray:
        w = self.next_u32_array(2 * n)
        return w[0::2] | (w[1::2] << np.uint64(32))

    def next_u64(self) -> int:
        return int(self.next_u64_array(1)[0])

    def uniform_array(self, n: int) -> np.ndarray:
        return (self.next_u64_array(n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53

    def uniform(self, lo: float = 0.0, hi: float | None = None) -> float:
        u = float(self.uniform_array(1)[0])
        if hi is None:
            return u
        return lo + (hi - lo) * u

    def uniform_int(self, lo: int, hi: int) -> int:
        """Unbiased integer on [lo, hi] by rejection (rng.cpp:78-88)."""
        if hi < lo:
            raise ValueError("uniform_int: empty range")
        rng = (hi - lo) + 1
        if rng == 1 << 64:
            return self.next_u64()
        limit = (2 ** 64 - 1) - (2 ** 64 - 1) % rng
        while True:
            u = self.next_u64()
            if u < limit:
                return lo + u % rng

    def normal_array(self, n: int) -> np.ndarray:
        """n successive normal() draws (rng.cpp:90-103)."""
        out = np.empty(n, dtype=np.float64)
        k = 0
        if n > 0 and self.have_spare:
            out[0] = self.spare
            self.have_spare = False
            k = 1
        rem = n - k
        if rem <= 0:
            return out
        pairs = (rem + 1) // 2
        # peek: a pair consumes two u64 unless u1 == 0 (probability 2^-53)
        self._need(4 * pairs)
        w = self._buf[self._pos:self._pos + 4 * pairs]
        u64 = w[0::2] | (w[1::2] << np.uint64(32))
        u = (u64 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        u1, u2 = u[0::2], u[1::2]
        if np.any(u1 <= 0.0):  # exact scalar fallback, never hit in practice
            for i in range(rem):
                out[k + i] = self.normal()
            return out
        self._pos += 4 * pairs
        mag = np.sqrt(-2.0 * np.log(u1))
        ang = 2.0 * math.pi * u2
        z = np.empty(2 * pairs)
        z[0::2] = mag * np.cos(ang)
        z[1::2] = mag * np.sin(ang)
        out[k:] = z[:rem]
        if rem % 2 == 1:
            self.have_spare = True
            self.spare = float(z[-1])
        return out

    def normal(self, mean: float = 0.0, std: float = 1.0) -> float:
        if self.have_spare:
            self.have_spare = False
            return mean + std * self.spare
        u1 = self.uniform()
        while u1 <= 0.0:
            u1 = self.uniform()
        u2 = self.uniform()
        mag = math.sqrt(-2.0 * math.log(u1))
        ang = 2.0 * math.pi * u2
        self.spare = mag * math.sin(ang)
        self.have_spare = True
        return mean + std * mag * math.cos(ang)

    def simplex(self, n: int) -> np.ndarray:
        """Normalized exponential spacings (rng.cpp:107-117)."""
        v = np.empty(n)
        for i in range(n):
            u = self.uniform()
            while u <= 0.0:
                u = self.uniform()
            v[i] = -math.log(u)
        return v / v.sum()

    def uniform_vector(self, n: int, lo: float, hi: float) -> np.ndarray:
        return lo + (hi - lo) * self.uniform_array(n)

    def normal_matrix(self, rows: int, cols: int, mean: float, std: float) -> np.ndarray:
        """Row-major fill order (rng.cpp:125-131)."""
        return mean + std * self.normal_array(rows * cols).reshape(rows, cols)
