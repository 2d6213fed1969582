"""Gauss-Legendre nodes/weights and the half-circle contour (host constants).

Mirrors quadrature.py:12-95: the kernel receives z_e, w_e, theta_e and the
radius as scalars, so these stay on the host.  Nodes come from Newton's
method on P_Ne started at cos(pi (k - 1/4) / (Ne + 1/2)) for the positive
roots, which are then mirrored so paired nodes are exact negations.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .params import ALLOWED_CONTOUR_POINTS


@dataclass(frozen=True)
class QuadratureRule:
    order: int
    nodes: np.ndarray
    weights: np.ndarray


@dataclass(frozen=True)
class Contour:
    theta: np.ndarray
    z: np.ndarray
    weights: np.ndarray
    radius: float
    center: float

    def __len__(self) -> int:
        return len(self.z)


def _pn(order, x):
    """(P_order(x), P'_order(x)) by the three-term recurrence."""
    prev, cur = np.ones_like(x), x.copy()
    for j in range(2, order + 1):
        prev, cur = cur, ((2 * j - 1) * x * cur - (j - 1) * prev) / j
    return cur, order * (x * cur - prev) / (x * x - 1.0)


def gauss_legendre(ne: int) -> QuadratureRule:
    if ne not in ALLOWED_CONTOUR_POINTS:
        raise ValueError(f"unsupported quadrature order {ne}; allowed: {ALLOWED_CONTOUR_POINTS}")
    half = ne // 2
    x = np.cos(math.pi * (np.arange(1, half + 1) - 0.25) / (ne + 0.5))
    for _ in range(100):
        p, dp = _pn(ne, x)
        step = p / dp
        x = x - step
        if np.max(np.abs(step)) < 1e-16:
            break
    _, dp = _pn(ne, x)
    w = 2.0 / ((1.0 - x * x) * dp * dp)
    pos_x, pos_w = x[::-1], w[::-1]
    if ne % 2:
        _, d0 = _pn(ne, np.zeros(1))
        nodes = np.concatenate([-pos_x[::-1], [0.0], pos_x])
        weights = np.concatenate([pos_w[::-1], 2.0 / (d0 * d0), pos_w])
    else:
        nodes = np.concatenate([-pos_x[::-1], pos_x])
        weights = np.concatenate([pos_w[::-1], pos_w])
    return QuadratureRule(ne, nodes, weights)


def build_contour(rule: QuadratureRule, emin: float, emax: float) -> Contour:
    if not emin < emax:
        raise ValueError(f"invalid interval: emin={emin} >= emax={emax}")
    radius = (emax - emin) / 2.0
    center = (emax + emin) / 2.0
    theta = -(np.pi / 2.0) * (rule.nodes - 1.0)
    return Contour(theta, center + radius * np.exp(1j * theta), rule.weights.copy(), radius, center)
