"""Synthetic M-step inputs, identical for every backend.

Every value is a pure function of (seed, flat index) or of the reference's own
sequential generator, so the CUDA solver, the oracle and the reference CPU
solver are all fed the same bytes:

* ``Rng`` restates the reference splitmix64 stream (rng.hpp:10-58).
* ``counter_uniform(seed, idx)`` is the first ``Rng(seed, idx).uniform()``;
  ``counter_gaussian`` the first ``Rng(seed, idx).gaussian()`` — counter-based,
  vectorised over numpy uint64 arrays.
* ``random_phantom_spec`` / ``generate_phantom`` restate phantom.cpp:11-63
  (isotropic Gaussian blobs truncated at 4 sigma).

Problem definition (`synthetic_problem`):
  truth t   = generate_phantom(random_phantom_spec(B, N, 77), N), B = round(0.05 N^3/270)
  weight W  = 1 + (u(5, n) + u(5, -n)) / 2                      (centrosymmetric, U[1,2])
  x0        = t + 0.5 RMS(t) g(501, i)                           (white Gaussian noise)
  numerator Y = W * fft3_centered(x0)                             (Hermitian, finalized)
  x_init = anchor = x0  (the naive solve Re ifft3_centered(Y/W), test_regularizer.cpp:376)
  eps = 0.1 max|t|, eps' = eps/3, (alpha, beta, gamma, mu) = derive_config(scale_data(acc))
White real-space noise is the same as one Hermitian complex Gaussian draw per
Friedel orbit in Fourier space (simulate.cpp:31-49), which keeps Y exactly
Hermitian and the accumulator exactly finalized.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_GOLDEN = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1


def _mix(z):
    """splitmix64 output function (rng.hpp:11-14) on uint64 arrays."""
    z = (z ^ (z >> np.uint64(30))) * np.uint64(_M1)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(_M2)
    return z ^ (z >> np.uint64(31))


class Rng:
    """Scalar restatement of cryomap::Rng (rng.hpp:25-58)."""

    def __init__(self, seed: int, stream: int = 0):
        s = (seed ^ ((_GOLDEN + (stream << 1)) & _MASK)) & _MASK
        self.state = (s + 2 * _GOLDEN) & _MASK  # mix_seed: two discarded draws

    def next_u64(self) -> int:
        self.state = (self.state + _GOLDEN) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * _M1) & _MASK
        z = ((z ^ (z >> 27)) * _M2) & _MASK
        return z ^ (z >> 31)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        u = float(self.next_u64() >> 11) * 2.0**-53
        return lo + (hi - lo) * u

    def gaussian(self) -> float:
        u1 = self.uniform()
        u2 = self.uniform()
        if u1 <= 0.0:
            u1 = 2.0**-53
        return math.sqrt(-2.0 * math.log(u1)) * math.cos(6.283185307179586476925286766559 * u2)


def _stream_states(seed: int, idx: np.ndarray) -> np.ndarray:
    idx = idx.astype(np.uint64)
    with np.errstate(over="ignore"):
        s = np.uint64(seed) ^ (np.uint64(_GOLDEN) + (idx << np.uint64(1)))
        return s + np.uint64((2 * _GOLDEN) & _MASK)


def counter_uniform(seed: int, idx: np.ndarray, draw: int = 0) -> np.ndarray:
    """The (draw+1)-th ``Rng(seed, idx).uniform()`` for every idx (float64)."""
    with np.errstate(over="ignore"):
        s = _stream_states(seed, idx) + np.uint64(((draw + 1) * _GOLDEN) & _MASK)
        z = _mix(s)
    return (z >> np.uint64(11)).astype(np.float64) * 2.0**-53


def counter_gaussian(seed: int, idx: np.ndarray) -> np.ndarray:
    """First ``Rng(seed, idx).gaussian()`` for every idx (rng.hpp:47-52)."""
    u1 = counter_uniform(seed, idx, 0)
    u2 = counter_uniform(seed, idx, 1)
    u1 = np.where(u1 <= 0.0, 2.0**-53, u1)
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586476925286766559 * u2)


@dataclass
class Blob:
    cx: float
    cy: float
    cz: float
    amplitude: float
    sigma: float


def random_phantom_spec(n_blobs: int, side_n: int, seed: int) -> list[Blob]:
    """phantom.cpp:40-63."""
    rng = Rng(seed, 0xB10B)
    c = (side_n - 1) / 2.0
    radius = 0.27 * side_n
    blobs = []
    for _ in range(n_blobs):
        while True:
            x = rng.uniform(-1.0, 1.0)
            y = rng.uniform(-1.0, 1.0)
            z = rng.uniform(-1.0, 1.0)
            if x * x + y * y + z * z <= 1.0:
                break
        sigma = rng.uniform(1.6, 2.8)
        amp = rng.uniform(0.6, 1.4)
        blobs.append(Blob(c + radius * x, c + radius * y, c + radius * z, amp, sigma))
    return blobs


def bond_phantom_spec(n_chains: int, side_n: int, seed: int) -> list[Blob]:
    """BASELINE config 2: anisotropic, bond-like structure as a plain
    blob list (phantom.hpp:10-18) - chains of 6-12 blobs spaced 0.75 sigma along a
    random direction, starts in the same ball as random_phantom_spec."""
    rng = Rng(seed, 0xB0D5)
    c = (side_n - 1) / 2.0
    radius = 0.27 * side_n
    blobs = []
    for _ in range(n_chains):
        while True:
            x, y, z = rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-1, 1)
            if x * x + y * y + z * z <= 1.0:
                break
        while True:
            dx, dy, dz = rng.uniform(-1, 1), rng.uniform(-1, 1), rng.uniform(-1, 1)
            r = math.sqrt(dx * dx + dy * dy + dz * dz)
            if 1e-3 < r <= 1.0:
                break
        dx, dy, dz = dx / r, dy / r, dz / r
        sigma = rng.uniform(1.6, 2.8)
        amp = rng.uniform(0.6, 1.4)
        length = 6 + int(rng.uniform(0.0, 7.0))  # 6 .. 12 blobs
        step = 0.75 * sigma
        for b in range(length):
            blobs.append(Blob(c + radius * x + b * step * dx, c + radius * y + b * step * dy,
                              c + radius * z + b * step * dz, amp, sigma))
    return blobs


def generate_phantom(blobs: list[Blob], side_n: int) -> np.ndarray:
    """phantom.cpp:11-38; returns float64 [k][j][i] (x fastest)."""
    n = side_n
    v = np.zeros((n, n, n), dtype=np.float64)
    for b in blobs:
        cut = 4.0 * b.sigma
        ilo, ihi = max(0, math.ceil(b.cx - cut)), min(n - 1, math.floor(b.cx + cut))
        jlo, jhi = max(0, math.ceil(b.cy - cut)), min(n - 1, math.floor(b.cy + cut))
        klo, khi = max(0, math.ceil(b.cz - cut)), min(n - 1, math.floor(b.cz + cut))
        di = np.arange(ilo, ihi + 1, dtype=np.float64) - b.cx
        dj = np.arange(jlo, jhi + 1, dtype=np.float64) - b.cy
        dk = np.arange(klo, khi + 1, dtype=np.float64) - b.cz
        d2 = dk[:, None, None] ** 2 + dj[None, :, None] ** 2 + di[None, None, :] ** 2
        inv2s2 = 1.0 / (2.0 * b.sigma * b.sigma)
        val = np.where(d2 > cut * cut, 0.0, b.amplitude * np.exp(-d2 * inv2s2))
        v[klo:khi + 1, jlo:jhi + 1, ilo:ihi + 1] += val
    return v


def mate_flat(n: int) -> np.ndarray:
    """Flat index of the Friedel mate of every storage index (volume.hpp:37)."""
    r = (-np.arange(n)) % n
    return ((r[:, None, None] * n + r[None, :, None]) * n + r[None, None, :]).reshape(-1)


def symmetric_weight(n: int, seed: int = 5, lo: float = 1.0, hi: float = 2.0) -> np.ndarray:
    idx = np.arange(n ** 3, dtype=np.uint64)
    u = counter_uniform(seed, idx)
    w = lo + (hi - lo) * 0.5 * (u + u[mate_flat(n)])
    return w.reshape(n, n, n)


def halfshift3(x: np.ndarray) -> np.ndarray:
    """fourier.cpp:88-97: out[i] = x[(i + n/2) % n] on every axis."""
    h = x.shape[0] // 2
    return np.roll(x, shift=(-h, -h, -h), axis=(0, 1, 2))


def fft3_centered(x: np.ndarray, workers: int = -1) -> np.ndarray:
    """fourier.cpp:109 (host helper for input generation)."""
    import scipy.fft

    return scipy.fft.fftn(halfshift3(x).astype(np.complex128), workers=workers)


def n_blobs_for(n: int) -> int:
    return int(round(0.05 * n ** 3 / 270.0))


@dataclass
class Problem:
    n: int
    truth: np.ndarray      # float64 [n,n,n]
    weight: np.ndarray     # float64 [n,n,n] full grid
    numerator: np.ndarray  # complex128 [n,n,n] full grid, Hermitian
    x0: np.ndarray         # float64 [n,n,n]
    eps: float
    eps_prime: float


def synthetic_problem(n: int, n_blobs: int | None = None, phantom_seed: int = 77,
                      weight_seed: int = 5, noise_seed: int = 501,
                      noise_frac: float = 0.5, kind: str = "blobs") -> Problem:
    """kind "blobs": BASELINE configs 1/3 (isotropic blobs); "bonds": config 2
    (chains, about the same occupancy: n_blobs / 9 chains of ~9 blobs)."""
    if n_blobs is None:
        n_blobs = max(1, n_blobs_for(n))
    if kind == "bonds":
        spec = bond_phantom_spec(max(1, n_blobs // 9), n, phantom_seed)
    elif kind == "blobs":
        spec = random_phantom_spec(n_blobs, n, phantom_seed)
    else:
        raise ValueError(f"unknown phantom kind {kind!r}")
    t = generate_phantom(spec, n)
    w = symmetric_weight(n, weight_seed)
    rms = math.sqrt(float(np.mean(t * t)))
    nu = counter_gaussian(noise_seed, np.arange(n ** 3, dtype=np.uint64)).reshape(n, n, n)
    x0 = t + noise_frac * rms * nu
    y = w * fft3_centered(x0)
    eps = 0.1 * float(np.max(np.abs(t)))
    return Problem(n, t, w, y, x0, eps, eps / 3.0)


def synthetic_backprojection(n: int, n_images: int, n_poses: int = 12, trans_radius: int = 1,
                             entries_per_image: int = 3, kernel_kind: int = 0,
                             radius_cutoff: float = -1.0, seed: int = 0,
                             grid_angles: bool = True, identity_ctf: bool = False):
    """Backprojection inputs of the reference's shapes (ParticleSet, posterior
    rows, OrientationGrid): random Fourier images, realistic CTFs
    (ctf.hpp:9-14 defaults, defocus varied per image), poses on a 15-degree
    lattice (grid_angles; exercises exact-.5 rotated points) or uniform, the
    integer shift disc of radius trans_radius (orientation.hpp:17), and a few
    candidates per image with random posteriors, one of them 0 (skipped,
    backproject.cpp:43)."""
    from .backproject import BackprojectInput
    rng = np.random.default_rng(seed)
    images = (rng.standard_normal((n_images, n, n)) + 1j * rng.standard_normal((n_images, n, n)))
    params = np.zeros((n_images, 6))
    params[:, 0] = 300.0
    params[:, 1] = rng.uniform(8000.0, 25000.0, n_images)
    params[:, 2] = 2.0
    params[:, 3] = 0.07
    params[:, 4] = 1.0 if identity_ctf else 0.0
    params[:, 5] = 1.2
    if grid_angles:
        poses = np.stack([rng.integers(0, 24, n_poses) * 15.0, rng.integers(0, 13, n_poses) * 15.0,
                          rng.integers(0, 24, n_poses) * 15.0], axis=1)
    else:
        poses = np.stack([rng.uniform(0, 360, n_poses), rng.uniform(0, 180, n_poses),
                          rng.uniform(0, 360, n_poses)], axis=1)
    r = trans_radius
    shifts = np.array([(dx, dy) for dy in range(-r, r + 1) for dx in range(-r, r + 1)
                       if dx * dx + dy * dy <= r * r], np.int32)
    ncand = n_poses * len(shifts)
    ep, ec, epost = [], [], []
    for i in range(n_images):
        cands = rng.choice(ncand, size=min(entries_per_image, ncand), replace=False)
        post = rng.dirichlet(np.ones(len(cands)))
        post[-1] = 0.0
        ep += [i] * len(cands)
        ec += list(cands)
        epost += list(post)
    return BackprojectInput(images, params, poses, shifts, np.array(ep), np.array(ec),
                            np.array(epost), kernel_kind, 2.0, radius_cutoff)
