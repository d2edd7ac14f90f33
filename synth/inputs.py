"""Seeded synthetic inputs, drawn in the fixed order of SURVEY.md §8(d) ("Synthetic inputs").

The paper's own workloads (UCI tables through DKL features, the airline series, BayesOpt
traces; §4, lines 481-569 and 619-670) are not in the container.  These draws are
stand-ins with the shapes of BASELINE.json's configs; every value is fp64.
"""
from __future__ import annotations

import dataclasses

import numpy as np

from .configs import Problem


@dataclasses.dataclass
class Inputs:
    X: np.ndarray      # (n, d) fp64 training inputs, row-major
    y: np.ndarray      # (n,)  fp64 training targets
    Xs: np.ndarray     # (t, d) fp64 test inputs


def _draw(p: Problem, rng: np.random.Generator, n: int, t: int) -> Inputs:
    if p.data == "sin6pi":            # configs 1 and 5
        x = rng.uniform(0.0, 1.0, n)
        y = np.sin(6.0 * np.pi * x) + rng.normal(0.0, p.noise_sd, n)
        xs = rng.uniform(0.0, 1.0, t)
        return Inputs(x[:, None], y, xs[:, None])
    if p.data == "sum5sin":           # config 2: frequencies in cycles per unit
        x = rng.uniform(0.0, 1.0, n)
        f = rng.uniform(1.0, 20.0, 5)
        a = rng.normal(0.0, 1.0, 5)
        y = (a[None, :] * np.sin(2.0 * np.pi * f[None, :] * x[:, None])).sum(1)
        y = y + rng.normal(0.0, p.noise_sd, n)
        xs = rng.uniform(0.0, 1.0, t)
        return Inputs(x[:, None], y, xs[:, None])
    if p.data == "sincos2d":          # config 3
        X = rng.uniform(-1.0, 1.0, (n, 2))
        y = np.sin(3.0 * X[:, 0]) * np.cos(3.0 * X[:, 1]) + rng.normal(0.0, p.noise_sd, n)
        Xs = rng.uniform(-1.0, 1.0, (t, 2))
        return Inputs(X, y, Xs)
    if p.data == "rsinr3d":           # config 4
        X = np.clip(rng.normal(0.0, 1.0, (n, 3)), -3.0, 3.0)
        r = np.sqrt((X * X).sum(1))
        y = r * np.sin(r) + rng.normal(0.0, p.noise_sd, n)
        Xs = np.clip(rng.normal(0.0, 1.0, (t, 3)), -3.0, 3.0)
        return Inputs(X, y, Xs)
    if p.data == "styblinski_tang":   # config 6 (additive): 0.5 sum_i (x_i^4 - 16 x_i^2 + 5 x_i), / 100
        X = rng.uniform(-5.0, 5.0, (n, p.d))
        y = 0.5 * (X ** 4 - 16.0 * X ** 2 + 5.0 * X).sum(1) / 100.0 + rng.normal(0.0, p.noise_sd, n)
        Xs = rng.uniform(-5.0, 5.0, (t, p.d))
        return Inputs(X, y, Xs)
    raise ValueError(f"unknown data recipe {p.data}")


def make_inputs(p: Problem, seed: int | None = None) -> Inputs:
    """X, y, X* for problem p, from numpy default_rng(seed) (seed 0 unless given)."""
    rng = np.random.default_rng(p.seed if seed is None else seed)
    return _draw(p, rng, p.n, p.t)


def make_zeta(k_sample: int, s: int, seed: int = 1) -> np.ndarray:
    """Shared standard-normal draws zeta (k' x s, fp64, column j = sample j), config 5's
    `default_rng(1).normal((k', s))`."""
    return np.random.default_rng(seed).normal(0.0, 1.0, (k_sample, s))


def tiny_problem(kind: str, seed: int = 0):
    """Tiny problems for the dense-bridge pins: returns
    (Problem, Inputs).  All use sigma^2 = 0.01 and are run to breakdown by the tests."""
    import dataclasses as _dc
    from .configs import CONFIGS
    if kind == "1d_n40":
        p = _dc.replace(CONFIGS[1], name="tiny_1d_n40", n=40, m=(64,), t=50, k=200)
    elif kind == "1d_n200":
        p = _dc.replace(CONFIGS[1], name="tiny_1d_n200", n=200, m=(64,), t=50, k=200)
    elif kind == "2d":
        # 16 nodes per axis on [-1.3, 1.3] keep every x in [-1, 1] one cell inside the grid
        p = _dc.replace(CONFIGS[3], name="tiny_2d", n=300, m=(16, 16), lo=(-1.3, -1.3),
                        hi=(1.3, 1.3), t=50, k=400, sigma2=0.01, lengthscale=(0.3, 0.3),
                        precision="fp64")
    elif kind == "3d":
        # 8 nodes per axis on [-4.5, 4.5] keep every clipped x in [-3, 3] inside the grid
        p = _dc.replace(CONFIGS[4], name="tiny_3d", n=500, m=(8, 8, 8), lo=(-4.5,) * 3,
                        hi=(4.5,) * 3, t=50, k=600, sigma2=0.01, lengthscale=(1.0, 1.0, 1.0),
                        precision="fp64")
    elif kind == "additive3":
        # 3 additive components, 15 nodes per axis on [-7, 7] (x in [-5, 5] stays 2 cells inside)
        p = _dc.replace(CONFIGS[6], name="tiny_additive3", d=3, n=200, m=(15,) * 3, lo=(-7.0,) * 3,
                        hi=(7.0,) * 3, lengthscale=(1.5, 1.0, 2.0), t=50, k=400, precision="fp64")
    else:
        raise ValueError(kind)
    return p, make_inputs(p, seed)
