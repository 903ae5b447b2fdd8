"""Numerical check of the spherical-harmonic factorisation used by the linear-in-degree
triplet kernels (csrc/triplet_sh.cu), in fp64 numpy/torch on the CPU.

Per centre j with out-edges p, q (unit vectors u), the reference's triplet sum
(egn/engine.py:136-148, cos(l alpha) = T_l(u_p . u_q)) is

    S[p, c] = sum_{q != p} sum_l T_l(u_p . u_q) Q[q, l, c].

Write T_l in the Legendre basis, T_l = sum_j a_lj P_j, and use the addition theorem
P_j(u_p . u_q) = 4 pi / (2j+1) sum_m Y_jm(u_p) Y_jm(u_q) (real orthonormal harmonics):

    S[p, c] = sum_{j,m} Y_jm(u_p) M[jm, c] - self[p, c],
    M[jm, c] = sum_q Y_jm(u_q) Q'[q, j, c],   Q'[q, j, c] = 4 pi / (2j+1) sum_l a_lj Q[q, l, c],
    self[p, c] = sum_j (2j+1) / (4 pi) Q'[p, j, c]      (the q = p term, T_l(1) = 1)

-- O(n L^2) per centre instead of O(n^2 L).  Run: python tools/sh_triplet_check.py
"""

from __future__ import annotations

import math

import numpy as np
import torch


def legendre_of_chebyshev(L: int) -> np.ndarray:
    """a[l, j]: T_l(x) = sum_j a[l, j] P_j(x), l, j < L."""
    from numpy.polynomial import chebyshev as C, legendre as Lg

    a = np.zeros((L, L))
    for l in range(L):
        e = np.zeros(l + 1)
        e[l] = 1.0
        leg = Lg.poly2leg(C.cheb2poly(e))
        a[l, : leg.size] = leg
    return a


def real_sh(u: torch.Tensor, L: int) -> torch.Tensor:
    """Real orthonormal spherical harmonics Y_jm(u), j < L, index j*j + j + m, for unit u [n, 3]
    (Cartesian recurrences of the kernel: C_m + i S_m = (x + i y)^m, Q_j^m(z) associated
    Legendre without the (1 - z^2)^(m/2) factor)."""
    x, y, z = u[:, 0], u[:, 1], u[:, 2]
    n = u.shape[0]
    out = torch.zeros((n, L * L), dtype=u.dtype)
    Cm = [torch.ones_like(x)]
    Sm = [torch.zeros_like(x)]
    for m in range(1, L):
        c_prev, s_prev = Cm[m - 1], Sm[m - 1]
        Cm.append(x * c_prev - y * s_prev)
        Sm.append(x * s_prev + y * c_prev)
    for m in range(L):
        # Q_m^m = (2m-1)!!  (Condon-Shortley phase dropped: any consistent real basis works)
        qmm = float(np.prod(np.arange(1, 2 * m, 2))) if m else 1.0
        q_prev2, q_prev = None, torch.full_like(z, qmm)
        for j in range(m, L):
            if j == m:
                q = q_prev
            elif j == m + 1:
                q = (2 * m + 1) * z * q_prev
                q_prev2, q_prev = q_prev, q
            else:
                q = ((2 * j - 1) * z * q_prev - (j + m - 1) * q_prev2) / (j - m)
                q_prev2, q_prev = q_prev, q
            norm = math.sqrt((2 * j + 1) / (4 * math.pi) * math.factorial(j - m) / math.factorial(j + m))
            if m == 0:
                out[:, j * j + j] = norm * q
            else:
                out[:, j * j + j + m] = math.sqrt(2.0) * norm * q * Cm[m]
                out[:, j * j + j - m] = math.sqrt(2.0) * norm * q * Sm[m]
    return out


def direct(u, Q):
    """S[p, c] = sum_{q != p} sum_l T_l(u_p . u_q) Q[q, l, c]."""
    n, L, _ = Q.shape
    x = (u @ u.T).clamp(-1, 1)
    T = [torch.ones_like(x), x]
    for _ in range(2, L):
        T.append(2 * x * T[-1] - T[-2])
    T = torch.stack(T[:L], dim=-1)  # [p, q, l]
    T = T * (1 - torch.eye(n, dtype=u.dtype))[:, :, None]
    return torch.einsum("pql,qlc->pc", T, Q)


def factorised(u, Q):
    n, L, C = Q.shape
    a = torch.as_tensor(legendre_of_chebyshev(L), dtype=u.dtype)
    js = torch.arange(L, dtype=u.dtype)
    Qp = torch.einsum("lj,qlc->qjc", a, Q) * (4 * math.pi / (2 * js + 1))[None, :, None]
    Y = real_sh(u, L)  # [n, L*L]
    jidx = torch.tensor([j for j in range(L) for _ in range(2 * j + 1)])
    M = torch.einsum("qa,qac->ac", Y, Qp[:, jidx, :])
    self_t = torch.einsum("j,qjc->qc", (2 * js + 1) / (4 * math.pi), Qp)
    return Y @ M - self_t


def main():
    torch.manual_seed(0)
    for n, L, C in ((2, 7, 3), (23, 7, 64), (64, 7, 16), (500, 7, 8), (37, 4, 5)):
        u = torch.randn(n, 3, dtype=torch.float64)
        u = u / u.norm(dim=1, keepdim=True)
        Q = torch.randn(n, L, C, dtype=torch.float64)
        d = direct(u, Q)
        f = factorised(u, Q)
        err = (d - f).abs().max() / d.abs().max()
        # gradients w.r.t. the unit vectors and Q through both formulations
        u1 = u.clone().requires_grad_(True)
        q1 = Q.clone().requires_grad_(True)
        w = torch.randn(n, C, dtype=torch.float64)
        (direct(u1, q1) * w).sum().backward()
        u2 = u.clone().requires_grad_(True)
        q2 = Q.clone().requires_grad_(True)
        (factorised(u2, q2) * w).sum().backward()
        # the direct form is only defined on the sphere: compare tangential gradients
        tan = lambda g: g - (g * u).sum(1, keepdim=True) * u  # noqa: E731
        gu = (tan(u1.grad) - tan(u2.grad)).abs().max() / tan(u1.grad).abs().max()
        gq = (q1.grad - q2.grad).abs().max() / q1.grad.abs().max()
        print(f"n={n:4d} L={L} C={C:3d}: S rel err {err:.2e}, dS/du rel err {gu:.2e}, dS/dQ rel err {gq:.2e}")
        assert err < 1e-12 and gu < 1e-10 and gq < 1e-12


if __name__ == "__main__":
    main()
