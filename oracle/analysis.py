"""Closed forms from the paper's analysis (§5) — TEST INFRASTRUCTURE ONLY (oracle pins O7/O8).

* ``p_error_general``  — Theorem "Probability of Error of the Upper-Bound Sketch", Eq. at P:520:
      P[Xbar_i > X_i] ~= ∫ [1 - exp(-(h/m)(1 - Φ(α)) Σ_{j≠i} p_j)]^h φ(α) dα
  evaluated by numerical quadrature for a given density φ / CDF Φ.
* ``p_error_gaussian`` — Corollary, Eq. at P:572 (proof Appendix A):
      1 + Σ_{k=1}^{h} C(h,k) (-1)^k m / (k h (n-1) p) (1 - exp(-k h (n-1) p / m))
* ``expected_error_general`` — Lemma "Expected Value of Error", P:636-640:
      E[Zbar_i] ~= ∫_0^∞ ∫ [1 - exp(-(h/m)(1 - Φ(α+δ)) Σ p_j)]^h φ(α) dα dδ
"""
from __future__ import annotations

import math

import numpy as np
from scipy import integrate, stats


def p_error_gaussian(m: float, h: int, others: float) -> float:
    """Eq. at P:572 with (n-1)p = ``others`` (expected number of other active coordinates)."""
    acc = 1.0
    for k in range(1, h + 1):
        x = k * h * others / m
        acc += math.comb(h, k) * (-1) ** k * (1.0 - math.exp(-x)) / x
    return acc


def p_error_general(m: float, h: int, others: float, pdf, cdf, lo: float, hi: float) -> float:
    """Eq. at P:520 by quadrature over the support [lo, hi] of φ."""
    f = lambda a: (1.0 - math.exp(-(h / m) * (1.0 - cdf(a)) * others)) ** h * pdf(a)
    v, _ = integrate.quad(f, lo, hi, limit=400)
    return v


def expected_error_general(m: float, h: int, others: float, pdf, cdf, lo: float, hi: float) -> float:
    """Lemma at: E[Zbar] = ∫_0^∞ P[Zbar >= δ] dδ (support [lo, hi] bounds δ by hi - lo)."""
    def tail(d):
        f = lambda a: (1.0 - math.exp(-(h / m) * (1.0 - min(1.0, cdf(a + d))) * others)) ** h * pdf(a)
        v, _ = integrate.quad(f, lo, hi, limit=200)
        return v
    v, _ = integrate.quad(tail, 0.0, hi - lo, limit=200)
    return v


def uniform_pm1():
    """Uniform over [-1, 1] (Table 1/2 row 'Uniform[-1,1]')."""
    return (lambda a: 0.5 if -1.0 <= a <= 1.0 else 0.0), (lambda a: min(1.0, max(0.0, (a + 1.0) / 2.0))), -1.0, 1.0


def gaussian(sigma: float):
    d = stats.norm(0.0, sigma)
    return d.pdf, d.cdf, -12.0 * sigma, 12.0 * sigma


def p_error_mixture(m: float, h: int, nnz: np.ndarray) -> float:
    """Over-estimation rate of a collection whose documents have ``nnz`` active coordinates each:
    every active coordinate of a document with ψ actives sees ψ-1 others, so the rate is the
    nnz-weighted mean of Eq. at (n-1)p = ψ-1 (O7)."""
    nnz = np.asarray(nnz, dtype=np.int64)
    vals, counts = np.unique(nnz[nnz >= 2], return_counts=True)
    w = vals * counts
    rates = np.array([p_error_gaussian(m, h, float(v - 1)) for v in vals])
    total = float((nnz[nnz >= 1]).sum())
    # documents with a single active coordinate are never over-estimated
    return float((rates * w).sum() / total) if total > 0 else 0.0
