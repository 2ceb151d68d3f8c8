"""The paper's own q-domain spectral factor (TEST INFRASTRUCTURE).

Used only to pin the oracle's energy-domain discretisation against the
paper's continuous form (reading R2):

  g(r') = int int C G_so G_od T dtheta S(theta, q) f(r, q) dr dq     (Eq. 1)
  S(theta, q) = q (1 + cos^2 theta) cos(theta/2) / sin^2(theta/2)
                * Phi(hc q / sin(theta/2))

Integrating the energy-integrated model over q first (instead of E, with the
scaled delta of PAPER.md:599-608) gives the energy form the oracle sums:

  int Phi(E) E f(E sin(theta/2)/hc) dE (1 + cos^2 theta) cos(theta/2)
      = hc^2 int S(theta, q) f(q) dq,

so the oracle's  sum_k phi_k E_k f~(u_k) (1+cos^2) cos(theta/2), with
phi_k = Phi(E_k) dE, converges to hc^2 int S f dq as the grids refine.
"""
from __future__ import annotations

import math

HC = 12.3984193  # keV Angstrom


def bragg_energy(q: float, theta: float) -> float:
    """E = hc q / sin(theta/2)  (Eq. bragg)."""
    return HC * q / math.sin(0.5 * theta)


def spectral_factor(theta: float, q: float, Phi) -> float:
    """S(theta, q) of PAPER.md:661."""
    sh = math.sin(0.5 * theta)
    return q * (1.0 + math.cos(theta) ** 2) * math.cos(0.5 * theta) / sh ** 2 * Phi(HC * q / sh)
