"""Workload definitions (BASELINE.json `configs`, readings from SURVEY.md §8(c) A5-A7).

Grid bounds for configs 2-4 are not in BASELINE.json: reading A5 (5% margin on each side
of the data range) is used.  sigma^2 for configs 3/4 follows reading A7 (equal to the
data-noise variance).  Outputscale s^2 = 1 everywhere (reading A6).
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Tuple


@dataclasses.dataclass(frozen=True)
class Problem:
    name: str
    d: int
    n: int                       # training points
    m: Tuple[int, ...]           # grid points per dimension
    lo: Tuple[float, ...]        # grid start per dimension  (u_{d,i} = lo_d + i*h_d)
    hi: Tuple[float, ...]        # grid end per dimension
    lengthscale: Tuple[float, ...]
    outputscale: float
    sigma2: float
    k: int                       # Lanczos steps
    t: int                       # test points
    precision: str               # "fp32" | "fp64"
    data: str                    # generator name in synth.inputs
    noise_sd: float
    k_sample: int = 0            # k' of the sampling cache (config 5)
    s: int = 0                   # samples drawn (config 5)
    seed: int = 0
    kind: str = "product"        # "product" (Kronecker grid) | "additive" (Eq. 16)
    # fp32 outputs from an fp64-built cache (love_opts.cache_fp64, reading A12b): config 5 is
    # converged (var << prior) and an fp32 Lanczos breaks down before the fp64 oracle does
    cache_fp64: bool = False

    @property
    def h(self) -> Tuple[float, ...]:
        return tuple((b - a) / (mm - 1) for a, b, mm in zip(self.lo, self.hi, self.m))

    @property
    def m_total(self) -> int:
        if self.kind == "additive":
            return sum(self.m)
        out = 1
        for mm in self.m:
            out *= mm
        return out


CONFIGS = {
    1: Problem("cfg1_1d_fp64", 1, 1000, (256,), (-0.05,), (1.05,), (0.05,), 1.0, 0.01,
               50, 1000, "fp64", "sin6pi", 0.1),
    2: Problem("cfg2_1d_fp32", 1, 1_000_000, (100_000,), (-0.05,), (1.05,), (0.01,), 1.0, 0.01,
               100, 1_000_000, "fp32", "sum5sin", 0.1),
    3: Problem("cfg3_2d_kron", 2, 500_000, (256, 256), (-1.1, -1.1), (1.1, 1.1), (0.1, 0.1),
               1.0, 0.05 ** 2, 100, 1_000_000, "fp32", "sincos2d", 0.05),
    4: Problem("cfg4_3d_kron", 3, 2_000_000, (64, 64, 64), (-3.3, -3.3, -3.3), (3.3, 3.3, 3.3),
               (0.5, 0.5, 0.5), 1.0, 0.1 ** 2, 100, 4_000_000, "fp32", "rsinr3d", 0.1),
    5: Problem("cfg5_sampling", 1, 100_000, (10_000,), (-0.05,), (1.05,), (0.05,), 1.0, 0.01,
               100, 10_000, "fp32", "sin6pi", 0.1, k_sample=100, s=1000, cache_fp64=True),
    # SURVEY 8(f) NEXT #2 (not a BASELINE config): additive composition of 10 1-D RBF kernels
    # with m = 100 inducing points each, the paper's Styblinski-Tang model;
    # x ~ U(-5, 5)^10, grid [-5.5, 5.5] per axis (reading A5), y a scaled Styblinski-Tang
    # function + N(0, 0.1^2).
    6: Problem("cfg6_additive10", 10, 100_000, (100,) * 10, (-5.5,) * 10, (5.5,) * 10, (1.0,) * 10, 1.0, 0.01,
               100, 100_000, "fp32", "styblinski_tang", 0.1, kind="additive"),
}


def get_config(i: int) -> Problem:
    return CONFIGS[i]


def scaled_config(i: int, n: Optional[int] = None, m: Optional[Tuple[int, ...]] = None,
                  k: Optional[int] = None, t: Optional[int] = None,
                  precision: Optional[str] = None, k_sample: Optional[int] = None,
                  s: Optional[int] = None, cache_fp64: bool = False) -> Problem:
    """A smaller problem with the same data distribution, kernel and grid bounds as config i
    (used for parity at sizes the oracle finishes in seconds).  cache_fp64 is not inherited:
    a scaled problem runs the precision path it names."""
    p = CONFIGS[i]
    return dataclasses.replace(
        p,
        name=p.name + "_scaled",
        n=p.n if n is None else n,
        m=p.m if m is None else tuple(m),
        k=p.k if k is None else k,
        t=p.t if t is None else t,
        precision=p.precision if precision is None else precision,
        k_sample=p.k_sample if k_sample is None else k_sample,
        s=p.s if s is None else s,
        cache_fp64=cache_fp64,
    )
