"""Seeded magnetisation inputs m (unit vectors, [n,3] float64)."""
import numpy as np


def m_uniform(n, direction=(0.0, 0.0, 1.0)):
    d = np.asarray(direction, dtype=np.float64)
    d = d / np.linalg.norm(d)
    return np.tile(d, (n, 1))


def m_random(n, seed=0):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=(n, 3))
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def m_smooth(xyz, period, theta=0.3):
    """m = (cos th, sin th cos kx, sin th sin kx), k = 2 pi / period."""
    k = 2.0 * np.pi / period
    ph = k * xyz[:, 0]
    return np.stack([np.full_like(ph, np.cos(theta)), np.sin(theta) * np.cos(ph),
                     np.sin(theta) * np.sin(ph)], axis=1)
