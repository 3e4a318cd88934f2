"""Restarted GMRES(m) and flexible right-preconditioned FGMRES(m) — oracle.

PAPER.md:236  "...or omitting it entirely as GMRES is the default choice
within the DD-CPM software."  PAPER.md:244-250: GMRES preconditioned by the
DD-CPM (R)AS preconditioner.

Textbook algorithm (Saad, Iterative Methods for Sparse Linear Systems,
Alg. 6.9 GMRES with modified Gram-Schmidt and Givens rotations, §6.5.5;
restarts §6.5.5; flexible variant Alg. 9.6 FGMRES).  Reading R5
fixes the conventions the CUDA path shares:
  * x0 = 0 unless given; r0 = b - A x0 recomputed at every restart;
  * convergence when the Givens residual estimate |g_{j+1}| <= rtol * ||b||_2,
    checked after every Arnoldi step (PETSc's default test);
  * iteration count = number of Arnoldi steps (= operator applications
    inside cycles); happy breakdown (h_{j+1,j} == 0) ends the cycle;
  * preconditioning is on the right: A M z = b, x = x0 + Z y (flexible form,
    Z_j = M(v_j) stored), so the monitored residual is the true one.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass
class SolveStats:
    iterations: int
    converged: bool
    resid_est: float      # last Givens estimate |g_{j+1}|
    resid_true: float     # ||b - A x||_2 at return
    bnorm: float
    cycles: int


def gmres(A, b, x0=None, restart=30, rtol=1e-10, maxiter=20000, M=None):
    """(F)GMRES(restart). A, M: callables v -> A v / M v.  Returns (x, SolveStats)."""
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    x = np.zeros(n) if x0 is None else np.array(x0, dtype=np.float64)
    bnorm = float(np.linalg.norm(b))
    target = rtol * bnorm
    its = 0
    cycles = 0
    est = np.inf
    converged = False
    if bnorm == 0.0:
        return np.zeros(n), SolveStats(0, True, 0.0, 0.0, 0.0, 0)
    while True:
        r = b - A(x)
        beta = float(np.linalg.norm(r))
        if beta <= target:
            converged = True
            est = beta
            break
        if its >= maxiter:
            break
        cycles += 1
        m = restart
        V = np.zeros((m + 1, n))
        Z = np.zeros((m, n))
        H = np.zeros((m + 1, m))
        cs = np.zeros(m)
        sn = np.zeros(m)
        g = np.zeros(m + 1)
        g[0] = beta
        V[0] = r / beta
        k = 0
        for j in range(m):
            Z[j] = V[j] if M is None else M(V[j])
            w = A(Z[j])
            its += 1
            for i in range(j + 1):          # modified Gram-Schmidt
                H[i, j] = float(np.dot(V[i], w))
                w = w - H[i, j] * V[i]
            H[j + 1, j] = float(np.linalg.norm(w))
            for i in range(j):              # apply previous Givens rotations
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            den = np.hypot(H[j, j], H[j + 1, j])
            breakdown = H[j + 1, j] == 0.0
            if den == 0.0:
                cs[j], sn[j] = 1.0, 0.0
            else:
                cs[j], sn[j] = H[j, j] / den, H[j + 1, j] / den
            vnext = H[j + 1, j]
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = cs[j] * g[j]
            est = abs(g[j + 1])
            k = j + 1
            if est <= target or breakdown or its >= maxiter:
                break
            V[j + 1] = w / vnext
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):      # back substitution
            y[i] = (g[i] - np.dot(H[i, i + 1:k], y[i + 1:k])) / H[i, i]
        x = x + Z[:k].T @ y
        if est <= target:
            converged = True
            break
        if its >= maxiter:
            break
    rt = float(np.linalg.norm(b - A(x)))
    return x, SolveStats(its, converged, float(est), rt, bnorm, cycles)


def arnoldi_fixed(A, b, k: int):
    """Exactly k GMRES steps from x0 = 0 (no restart, no tolerance): z = V_k y_k.

    The inexact local solver of the RAS preconditioner (reading R6).
    Stops early only on happy breakdown.
    """
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    beta = float(np.linalg.norm(b))
    if beta == 0.0 or k == 0:
        return np.zeros(n)
    V = np.zeros((k + 1, n))
    H = np.zeros((k + 1, k))
    V[0] = b / beta
    kk = k
    for j in range(k):
        w = A(V[j])
        for i in range(j + 1):
            H[i, j] = float(np.dot(V[i], w))
            w = w - H[i, j] * V[i]
        H[j + 1, j] = float(np.linalg.norm(w))
        if H[j + 1, j] == 0.0:
            kk = j + 1
            break
        V[j + 1] = w / H[j + 1, j]
    e1 = np.zeros(kk + 1)
    e1[0] = beta
    y, *_ = np.linalg.lstsq(H[: kk + 1, :kk], e1, rcond=None)
    return V[:kk].T @ y
