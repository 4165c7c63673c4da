"""Synthetic input volumes (benchmark and test data, not the hot path).

Restates the reference test phantoms (``/root/reference/pkg/tests/
phantoms.py``) so that the GPU box -- where the reference does not exist --
can regenerate exactly the inputs the golden vectors were made from.  The
generators are bit-identical to the reference ones for the same numpy build;
``tests/golden`` stores the sha256 of every generated input to prove it.

All arrays use the reference convention ``[x, y, z]`` (z fastest).
"""

from __future__ import annotations

import numpy as np

BRAIN_DIMS = (145, 174, 145)        # BASELINE.json configs[0]
BRAIN_SEED = 20240817               # reference tests/conftest.py:10-12


def _lattice(dims):
    return np.meshgrid(*(np.arange(n, dtype=np.float64) for n in dims), indexing="ij")


def blob_field(dims, centers, sigmas, amplitudes) -> np.ndarray:
    """Sum of isotropic Gaussians on the lattice (phantoms.py:16-33)."""
    gx, gy, gz = _lattice(dims)
    acc = np.zeros(dims, dtype=np.float64)
    for c, s, a in zip(centers, sigmas, amplitudes):
        acc += a * np.exp(-((gx - c[0]) ** 2 + (gy - c[1]) ** 2 + (gz - c[2]) ** 2) / (2.0 * s * s))
    return acc.astype(np.float32)


def random_blob_phantom(dims, rng, n_blobs=12, margin=10, sigma_range=(2.0, 5.0),
                        amplitude_range=(0.4, 1.0), signed=True, noise=0.0) -> np.ndarray:
    """phantoms.py:36-52 (returns the float32 array, not a Volume)."""
    centers = [[rng.uniform(margin, d - 1 - margin) for d in dims] for _ in range(n_blobs)]
    sig = rng.uniform(*sigma_range, size=n_blobs)
    amp = rng.uniform(*amplitude_range, size=n_blobs)
    if signed:
        amp *= rng.choice([-1.0, 1.0], size=n_blobs)
    f = blob_field(dims, centers, sig, amp)
    if noise > 0:
        f = f + rng.normal(0.0, noise, size=dims).astype(np.float32)
    return f


def kernel_soup_field(dims, centers, sigmas, amplitudes, cutoff=5.0) -> np.ndarray:
    """Locally rendered Gaussian-kernel soup (phantoms.py:83-109)."""
    acc = np.zeros(dims, dtype=np.float64)
    hi_lim = np.array(dims)
    for c, s, a in zip(centers, sigmas, amplitudes):
        r = cutoff * s
        lo = np.maximum(np.ceil(np.asarray(c) - r).astype(int), 0)
        hi = np.minimum(np.floor(np.asarray(c) + r).astype(int) + 1, hi_lim)
        if np.any(lo >= hi):
            continue
        x, y, z = np.ogrid[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]]
        d2 = (x - c[0]) ** 2 + (y - c[1]) ** 2 + (z - c[2]) ** 2
        acc[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]] += a * np.exp(-d2 / (2.0 * s * s))
    return acc.astype(np.float32)


def soup_params(dims, rng, density=1 / 900.0, sigma_range=(2.2, 4.5), margin=4):
    """phantoms.py:112-121."""
    n = max(8, int(np.prod(dims) * density))
    centers = np.column_stack([rng.uniform(margin, d - 1 - margin, size=n) for d in dims])
    sigmas = np.exp(rng.uniform(np.log(sigma_range[0]), np.log(sigma_range[1]), size=n))
    amps = rng.uniform(0.35, 1.0, size=n) * rng.choice([-1.0, 1.0], size=n)
    return centers, sigmas, amps


def soup_volume(dims, rng, noise=0.0) -> np.ndarray:
    """Soup phantom plus optional N(0, noise) (reference tests/test_detect.py:221-233)."""
    field = kernel_soup_field(dims, *soup_params(dims, rng))
    if noise > 0:
        field = field + rng.normal(0.0, noise, size=dims).astype(np.float32)
    return field


def brain_volume(seed: int = BRAIN_SEED, dims=BRAIN_DIMS) -> np.ndarray:
    """The configs[0] volume: 145x174x145 soup + N(0, 0.01), seed 20240817."""
    return soup_volume(dims, np.random.default_rng(seed), noise=0.01)


def rotation_from_axis_angle(axis, angle_deg: float) -> np.ndarray:
    """phantoms.py:170-184."""
    k = np.asarray(axis, dtype=np.float64)
    k = k / np.linalg.norm(k)
    t = np.deg2rad(angle_deg)
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    return np.eye(3) + np.sin(t) * K + (1 - np.cos(t)) * (K @ K)


def transformed_pair(dims, rng, scale, rotation, translation, density=1 / 900.0,
                     sigma_range=(2.2, 4.5), noise=0.0):
    """Phantom pair related exactly by x -> scale*R x + t (phantoms.py:124-141;
    the transform application mirrors match.py:48-51)."""
    centers, sigmas, amps = soup_params(dims, rng, density, sigma_range)
    moved = scale * (centers @ np.asarray(rotation, dtype=np.float64).T) + np.asarray(translation, dtype=np.float64)
    keep = np.all((moved > 2.0) & (moved < np.array(dims) - 3.0), axis=1)
    a = kernel_soup_field(dims, centers[keep], sigmas[keep], amps[keep])
    b = kernel_soup_field(dims, moved[keep], scale * sigmas[keep], amps[keep])
    if noise > 0:
        a = a + rng.normal(0.0, noise, size=dims).astype(np.float32)
        b = b + rng.normal(0.0, noise, size=dims).astype(np.float32)
    return a, b


def match_pair(dims=BRAIN_DIMS, seed: int = BRAIN_SEED):
    """The configs[1] two-volume matching pair:
    10 degrees about (0.3, 1, 0.2), t = (2, -1, 1.5), noise 0.01."""
    rot = rotation_from_axis_angle((0.3, 1.0, 0.2), 10.0)
    return transformed_pair(dims, np.random.default_rng(seed), 1.0, rot, (2.0, -1.0, 1.5), noise=0.01)


def batch_from(base: np.ndarray, count: int, seed: int = 0, noise: float = 0.01) -> np.ndarray:
    """``count`` distinct volumes derived cheaply from one phantom (flips,
    cyclic shifts and fresh N(0, noise)); used to fill large benchmark batches
    without paying the phantom renderer per volume.  Returns (count, nx, ny, nz)."""
    rng = np.random.default_rng(seed)
    out = np.empty((count,) + base.shape, dtype=np.float32)
    for i in range(count):
        v = base
        for ax in range(3):
            if rng.random() < 0.5:
                v = np.flip(v, axis=ax)
        v = np.roll(v, tuple(int(s) for s in rng.integers(0, 16, size=3)), axis=(0, 1, 2))
        out[i] = v + rng.normal(0.0, noise, size=base.shape).astype(np.float32)
    return out


def zero_background_volume(dims, seed: int, radius_frac: float = 0.42, scale: float = 1.0) -> np.ndarray:
    """Soup phantom + N(0, 0.01) set to exactly 0 outside a centred sphere of
    radius ``radius_frac * min(dims)`` (a skull-stripped-MRI-like background),
    then multiplied by ``scale`` in float32 (scale = 1e-22 makes every fp32 sum
    of squared gradient components underflow).  Golden: tests/golden/zeroback.npz."""
    v = soup_volume(dims, np.random.default_rng(seed), noise=0.01)
    c = (np.array(dims) - 1) / 2.0
    g = np.meshgrid(*[np.arange(d) for d in dims], indexing="ij")
    r2 = sum((gi - ci) ** 2 for gi, ci in zip(g, c))
    v = np.where(r2 <= (radius_frac * min(dims)) ** 2, v, 0.0).astype(np.float32)
    return (v * np.float32(scale)).astype(np.float32)
