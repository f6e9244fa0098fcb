"""Seeded synthetic inputs for the five BASELINE.json configurations.

The paper's trained Netflix / KDD / R2 models are not available, so each
configuration is a seeded synthetic model with the shapes, sizes and value
distributions BASELINE.json states.  Pinned choices:

* one ``numpy.random.default_rng(seed)`` per config, draws in the order
  written below, generated in float64 and cast to float32 (the reference
  then upcasts to float64 exactly, model_io.py:37-48);
* "N(0, 1/sqrt(32))" is read as standard deviation 1/sqrt(32);
* "item norms rescaled by log-normal" multiplies each item row by a
  log-normal draw (cfg5); "item directions normalised, norms log-normal"
  (cfg2/cfg4) builds unit directions times a log-normal norm.

The same arrays feed the GPU path, the CPU oracle and the reference arm.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    users: np.ndarray          # float32 [U, f]
    items: np.ndarray          # float32 [I, f]
    k: int
    ks: tuple
    clusters: int | None       # k-means clusters for the index path
    max_iters: int
    seed: int
    expected_path: str         # what BASELINE.json says the optimizer picks


def _unit_rows(a):
    n = np.linalg.norm(a, axis=1, keepdims=True)
    n[n == 0.0] = 1.0
    return a / n


def cfg1(scale: float = 1.0) -> Workload:
    """8192 x 2048, f=32, N(0, 1/sqrt(32)) entries, K=10, seed 0."""
    rng = np.random.default_rng(0)
    nu, ni = int(8192 * scale), int(2048 * scale)
    users = rng.normal(0.0, 1.0 / np.sqrt(32.0), (nu, 32))
    items = rng.normal(0.0, 1.0 / np.sqrt(32.0), (ni, 32))
    return Workload("cfg1", users.astype(np.float32), items.astype(np.float32), 10, (10,), 8, 100, 0, "matmul")


def _mixture(seed, nu, ni, f, centers, sigma, ln_sigma, name, ks, k, scale):
    rng = np.random.default_rng(seed)
    nu, ni = int(nu * scale), int(ni * scale)
    cen = rng.normal(0.0, 1.0, (centers, f))
    comp = rng.integers(0, centers, nu)
    users = cen[comp] + rng.normal(0.0, sigma, (nu, f))
    d = _unit_rows(rng.normal(0.0, 1.0, (ni, f)))
    items = d * rng.lognormal(0.0, ln_sigma, ni)[:, None]
    return Workload(name, users.astype(np.float32), items.astype(np.float32), k, ks, centers, 3, seed, "index")


def cfg2(scale: float = 1.0) -> Workload:
    """Netflix shape 480,189 x 17,770, f=50: 256-Gaussian user mixture
    (centers N(0,1), sigma 0.3), unit item directions x lognormal(0, 0.5)
    norms; k-means C=256, 3 iterations; K in {1,5,10,50}; seed 1."""
    return _mixture(1, 480_189, 17_770, 50, 256, 0.3, 0.5, "cfg2", (1, 5, 10, 50), 10, scale)


def cfg3(scale: float = 1.0) -> Workload:
    """480,189 x 17,770, f=100, i.i.d. N(0,1), K=10, seed 2 (optimizer must
    pick blocked MM); k-means with the default C=8, 100 iterations."""
    rng = np.random.default_rng(2)
    nu, ni = int(480_189 * scale), int(17_770 * scale)
    users = rng.normal(0.0, 1.0, (nu, 100))
    items = rng.normal(0.0, 1.0, (ni, 100))
    return Workload("cfg3", users.astype(np.float32), items.astype(np.float32), 10, (10,), 8, 100, 2, "matmul")


def cfg4(scale: float = 1.0) -> Workload:
    """R2 shape 1,823,179 x 136,736, f=50: 1024-Gaussian mixture, sigma 0.05,
    lognormal(0, 1.0) item norms, C=1024, 3 iterations, K in {1,10}; seed 3."""
    return _mixture(3, 1_823_179, 136_736, 50, 1024, 0.05, 1.0, "cfg4", (1, 10), 10, scale)


def cfg5(scale: float = 1.0) -> Workload:
    """1M x 1M, f=128: items N(0,1) rows x lognormal(0, 0.7), users N(0,1);
    K=100; catalog sharded across GPUs; seed 4."""
    rng = np.random.default_rng(4)
    nu, ni = int(1_000_000 * scale), int(1_000_000 * scale)
    items = rng.normal(0.0, 1.0, (ni, 128)) * rng.lognormal(0.0, 0.7, ni)[:, None]
    users = rng.normal(0.0, 1.0, (nu, 128))
    return Workload("cfg5", users.astype(np.float32), items.astype(np.float32), 100, (100,), None, 3, 4, "matmul")


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}
