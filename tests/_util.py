"""Shared helpers for the parity tests: seeded synthetic inputs (SURVEY 8d
generator, following gallery.py:59-60's numpy default_rng) and the
normwise tolerance c*n*u_work of acceptance.py:197 / harness.py:151."""
import numpy as np


def synth(n, target, seed, cos=False):
    """X = G * (target / ||G||_1), G ~ N(0,1) from default_rng(seed); the
    cosine config first divides by sqrt(n)."""
    G = np.random.default_rng(seed).standard_normal((n, n))
    if cos:
        G = G / np.sqrt(n)
    return G * (target / np.abs(G).sum(axis=0).max())


def tol(r, n, d):
    """10 r n 10^-d (the reference's mixed-vs-fixed slack)."""
    return 10.0 * r * n * 10.0 ** (-d)


def words_of(report, b=None):
    """Result words (W, n, n) of one matrix of a report / batch report."""
    res = report.result
    idx = 0 if b is None else b
    return res.data[:, idx].double().cpu().numpy()
