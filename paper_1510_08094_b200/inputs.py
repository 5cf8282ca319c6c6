"""Seeded synthetic inputs and the BASELINE.json configurations.

* ``sh_coeffs``: coefficients c_lm = z_lm / (1+l)^p of a real spherical-
  harmonic sum (BASELINE.json configs), z_lm ~ N(0,1) from a counter-based
  generator keyed by (seed, l, m) (SplitMix64 + Box-Muller), so any (l, m)
  can be drawn independently and reproducibly.  l >= 1: the surface mean is
  zero.  ``solution=True`` returns the analytic solution's coefficients
  -c_lm / (l(l+1)) (u = Lap^-1 f on the sphere).  The grid values are then
  synthesised on the device by ``Plan.shgen``.
* ``bench_problem`` / ``random_mean_zero_problem``: the reference's two
  coefficient-space workload generators (poisson.cpp:190-216 and
  tests/support/poisson_oracle.hpp:119-154), same std::mt19937_64 stream and
  libstdc++ uniform_real_distribution<double>(-1, 1) draws.
"""
from __future__ import annotations

import dataclasses

import numpy as np

M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    M: int        # doubled theta count (reference pb.m)
    N: int        # lambda count (reference pb.n)
    L: int        # max spherical-harmonic degree
    p: float      # coefficient decay exponent
    nrhs: int
    note: str

    @property
    def dof(self) -> int:  # per RHS, PAPER.md:1207-1208 convention (M N / 2)
        return self.M * self.N // 2


CONFIGS = {
    "C1": Config("C1", 512, 256, 32, 2.0, 1, "n=m=256, CPU reference case"),
    "C2": Config("C2", 4096, 2048, 512, 2.0, 1, "n=m=2048, ~4.2M DOF, 1 GPU"),
    "C3": Config("C3", 20000, 10000, 2000, 2.0, 1, "paper scale n=m=10000, ~1e8 DOF"),
    "C4": Config("C4", 2048, 1024, 256, 1.5, 64, "64 independent RHS at n=m=1024"),
    "C5": Config("C5", 65536, 32768, 8192, 2.0, 1, "n=m=32768, ~1.07e9 DOF"),
}


def _splitmix64(z: np.ndarray) -> np.ndarray:
    z = (z + np.uint64(0x9E3779B97F4A7C15)) & M64
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & M64
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & M64
    return z ^ (z >> np.uint64(31))


def normals(seed: int, idx: np.ndarray) -> np.ndarray:
    """z_i ~ N(0,1) for integer counters idx (Box-Muller on two SplitMix64 draws)."""
    with np.errstate(over="ignore"):
        base = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        golden = np.uint64(0x9E3779B97F4A7C15)
        i = idx.astype(np.uint64)
        x1 = _splitmix64(base ^ ((np.uint64(2) * i) * golden & M64))
        x2 = _splitmix64(base ^ ((np.uint64(2) * i + np.uint64(1)) * golden & M64))
    u1 = ((x1 >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53
    u2 = (x2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)


def sh_coeffs(seed: int, L: int, p: float, solution: bool = False) -> np.ndarray:
    """(L+1)^2 coefficients indexed l*l + l + m (m = -l..l); entry 0 (l = 0) is 0."""
    n = (L + 1) ** 2
    idx = np.arange(n, dtype=np.int64)
    l = np.floor(np.sqrt(idx)).astype(np.int64)
    l = np.where((l + 1) ** 2 <= idx, l + 1, l)
    l = np.where(l * l > idx, l - 1, l)
    c = normals(seed, idx) / (1.0 + l) ** p
    c[0] = 0.0
    if solution:
        ll = l.astype(np.float64)
        with np.errstate(divide="ignore", invalid="ignore"):
            c = np.where(l > 0, -c / (ll * (ll + 1.0)), 0.0)
    return c


# ----------------------------------------------------- std::mt19937_64 (libstdc++)
class MT19937_64:
    NN, MM = 312, 156
    A = np.uint64(0xB5026F5AA96619E9)
    UM = np.uint64(0xFFFFFFFF80000000)
    LM = np.uint64(0x7FFFFFFF)

    def __init__(self, seed: int):
        mt = np.zeros(self.NN, np.uint64)
        mt[0] = np.uint64(seed & 0xFFFFFFFFFFFFFFFF)
        x = int(mt[0])
        for i in range(1, self.NN):
            x = (6364136223846793005 * (x ^ (x >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
            mt[i] = np.uint64(x)
        self.mt = mt
        self.buf = np.zeros(0, np.uint64)
        self.pos = 0

    def _twist(self):
        mt, NN, MM = self.mt, self.NN, self.MM
        one = np.uint64(1)

        def mix(hi, lo, far):
            x = (hi & self.UM) | (lo & self.LM)
            return far ^ (x >> one) ^ np.where((x & one) == one, self.A, np.uint64(0))

        mt[: NN - MM] = mix(mt[: NN - MM], mt[1 : NN - MM + 1], mt[MM:NN])
        mt[NN - MM : NN - 1] = mix(mt[NN - MM : NN - 1], mt[NN - MM + 1 : NN], mt[0 : MM - 1])
        mt[NN - 1] = mix(mt[NN - 1 : NN], mt[0:1], mt[MM - 1 : MM])[0]
        x = mt.copy()
        x ^= (x >> np.uint64(29)) & np.uint64(0x5555555555555555)
        x ^= (x << np.uint64(17)) & np.uint64(0x71D67FFFEDA60000)
        x ^= (x << np.uint64(37)) & np.uint64(0xFFF7EEE000000000)
        x ^= x >> np.uint64(43)
        self.buf = x
        self.pos = 0

    def next_u64(self, count: int) -> np.ndarray:
        out = np.empty(count, np.uint64)
        k = 0
        while k < count:
            if self.pos >= self.NN:
                self._twist()
            if self.buf.size == 0:
                self._twist()
            take = min(count - k, self.NN - self.pos)
            out[k : k + take] = self.buf[self.pos : self.pos + take]
            self.pos += take
            k += take
        return out

    def uniform_pm1(self, count: int) -> np.ndarray:
        """uniform_real_distribution<double>(-1, 1): -1 + 2 * generate_canonical."""
        u = self.next_u64(count).astype(np.float64) / 18446744073709551616.0
        u = np.where(u >= 1.0, np.nextafter(1.0, 0.0), u)
        return -1.0 + 2.0 * u


def _msin2_apply(col: np.ndarray) -> np.ndarray:
    """Msin^2 column apply in the reference's accumulation order (banded.cpp:8-19)."""
    m = col.shape[0]
    y = np.zeros_like(col)
    d = np.full(m, 0.5)
    d[0] = d[-1] = 0.25
    y[:] = d * col
    y[2:] = -0.25 * col[:-2] + y[2:]          # acc = (-1/4) x_{i-2}, then + diag x_i
    y[:-2] = y[:-2] + (-0.25) * col[2:]       # then + (-1/4) x_{i+2}
    return y


def _weights(m: int) -> np.ndarray:
    k = np.arange(m) - m // 2
    w = np.zeros(m)
    even = (k % 2) == 0
    w[even] = 2.0 / (1.0 - k[even].astype(np.float64) ** 2)
    return w


def _remove_mean(col: np.ndarray, w: np.ndarray) -> None:
    m = col.shape[0]
    prod = w * col.real + 1j * (w * col.imag)
    mean = complex(np.cumsum(prod.real)[-1], np.cumsum(prod.imag)[-1])
    col[m // 2] -= mean / w[m // 2]


def bench_problem(sizes) -> np.ndarray:
    """bench_poisson's F for the last of `sizes` (poisson.cpp:190-216)."""
    rng = MT19937_64(0x5EED)
    F = None
    for s in sizes:
        F = np.zeros((s, s), np.complex128)
        w = _weights(s)
        band = max(2, s // 8)
        for kc in range(s):
            k = kc - s // 2
            col = np.zeros(s, np.complex128)
            if abs(k) <= band:
                lo, hi = s // 2 - band, s // 2 + band
                lo, hi = max(lo, 0), min(hi, s - 1)
                u = rng.uniform_pm1(2 * (hi - lo + 1))
                col[lo : hi + 1] = u[1::2] + 1j * u[0::2]  # GCC evaluates complex(unit(rng), unit(rng)) right to left
            if k == 0:
                _remove_mean(col, w)
            F[:, kc] = _msin2_apply(col)
    return F


def random_mean_zero_problem(m: int, n: int, seed: int) -> np.ndarray:
    """tests/support/poisson_oracle.hpp:119-154."""
    rng = MT19937_64(seed)
    w = _weights(m)
    F = np.zeros((m, n), np.complex128)
    bt, bl = m // 4, n // 4
    for kc in range(n):
        k = kc - n // 2
        col = np.zeros(m, np.complex128)
        if abs(k) <= bl:
            sign = 1.0 if k % 2 == 0 else -1.0
            u = rng.uniform_pm1(2 * bt)
            v = u[1::2] + 1j * u[0::2]  # (imaginary part drawn first, as compiled by GCC)
            j = np.arange(1, bt + 1)
            col[m // 2 + j] = v
            col[m // 2 - j] = sign * v
            if k % 2 == 0:
                u = rng.uniform_pm1(2)
                col[m // 2] = u[1] + 1j * u[0]
        if k == 0:
            _remove_mean(col, w)
        F[:, kc] = _msin2_apply(col)
    return F
