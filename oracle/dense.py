"""Dense-matrix numpy oracle for tiny problems (TEST INFRASTRUCTURE ONLY).

An independent second restatement used to pin the C++ oracle: every operator
is materialised entry by entry as a dense matrix, following the reference's
own test oracles (/root/reference/proj/tests/oracles.hpp:28-66) -- dense
Kronecker A = K_tau (x) M_h + M_tau (x) K_h, B = -N_tau (x) M_h and the
block lower-bidiagonal space-time matrix -- plus dense transfer matrices
built from the stencil definitions (transfer.cpp:22-46, 75-96, 138-158) and a
dense two-level / multilevel cycle (mg.cpp:96-166) using numpy.linalg.solve
for the exact block inverses.  DG blocks come from numpy's Gauss-Legendre
rule, not from the C++ code.
"""
from __future__ import annotations

import numpy as np
from numpy.polynomial import legendre as npleg


def leg(l, x):
    c = np.zeros(l + 1)
    c[l] = 1.0
    return npleg.legval(x, c)


def dleg(l, x):
    c = np.zeros(l + 1)
    c[l] = 1.0
    return npleg.legval(x, npleg.legder(c))


def dg_block(p, tau):
    """K[k,l] = -int psi_l psi_k' + psi_l(tau)psi_k(tau); M = int psi_l psi_k;
    N[k,l] = psi_l(tau) psi_k(0)  (dg_time.hpp:14-19)."""
    n = p + 1
    x, w = npleg.leggauss(n + 1)
    t = 0.5 * tau * (x + 1.0)
    w = 0.5 * tau * w
    K = np.zeros((n, n))
    M = np.zeros((n, n))
    N = np.zeros((n, n))
    for k in range(n):
        for l in range(n):
            vl = leg(l, 2 * t / tau - 1)
            dk = dleg(k, 2 * t / tau - 1) * 2.0 / tau
            K[k, l] = -np.sum(w * vl * dk) + leg(l, 1.0) * leg(k, 1.0)
            M[k, l] = np.sum(w * vl * leg(k, 2 * t / tau - 1))
            N[k, l] = leg(l, 1.0) * leg(k, -1.0)
    return K, M, N


def time_transfer(p, tau):
    n = p + 1
    x, w = npleg.leggauss(n + 1)
    s = 0.5 * tau * (x + 1.0)
    w = 0.5 * tau * w
    _, M, _ = dg_block(p, tau)
    Mt1 = np.zeros((n, n))
    Mt2 = np.zeros((n, n))
    for k in range(n):
        fk = leg(k, 2 * s / tau - 1)
        for l in range(n):
            Mt1[k, l] = np.sum(w * leg(l, s / tau - 1) * fk)
            Mt2[k, l] = np.sum(w * leg(l, (s + tau) / tau - 1) * fk)
    R1 = np.linalg.solve(M, Mt1).T
    R2 = np.linalg.solve(M, Mt2).T
    return R1, R2


def tri(n, off, diag):
    return np.diag(np.full(n, diag)) + np.diag(np.full(n - 1, off), 1) + np.diag(np.full(n - 1, off), -1)


def space_mats(dim, level):
    n1 = 2 ** (level + 1) - 1
    h = 2.0 ** -(level + 1)
    M1 = tri(n1, h / 6, 4 * h / 6)
    K1 = tri(n1, -1 / h, 2 / h)
    if dim == 1:
        return M1, K1
    if dim == 2:
        return np.kron(M1, M1), np.kron(K1, M1) + np.kron(M1, K1)
    M = np.kron(np.kron(M1, M1), M1)
    K = np.kron(np.kron(K1, M1), M1) + np.kron(np.kron(M1, K1), M1) + np.kron(np.kron(M1, M1), K1)
    return M, K


def dense_block(K, M, Mh, Kh):
    """A(l*nx+i, k*nx+j) = K(l,k) Mh(i,j) + M(l,k) Kh(i,j) (oracles.hpp:28-40)."""
    return np.kron(K, Mh) + np.kron(M, Kh)


def dense_space_time(K, M, N, Mh, Kh, n_t):
    A = dense_block(K, M, Mh, Kh)
    B = -np.kron(N, Mh)
    b = A.shape[0]
    L = np.zeros((n_t * b, n_t * b))
    for n in range(n_t):
        L[n * b:(n + 1) * b, n * b:(n + 1) * b] = A
        if n > 0:
            L[n * b:(n + 1) * b, (n - 1) * b:n * b] = B
    return L


def restrict_line_matrix(n1):
    m = (n1 - 1) // 2
    R = np.zeros((m, n1))
    for j in range(m):
        R[j, 2 * j] = 0.5
        R[j, 2 * j + 1] = 1.0
        R[j, 2 * j + 2] = 0.5
    return R


def space_restriction(dim, level):
    R1 = restrict_line_matrix(2 ** (level + 1) - 1)
    R = R1
    for _ in range(dim - 1):
        R = np.kron(R1, R)  # x fastest: kron(y-op, x-op)
    return R


def time_restriction(R1, R2, n_t, nx):
    """Semi restriction matrix: coarse step n <- R1 fine_2n + R2 fine_2n+1."""
    nl = R1.shape[0]
    b = nl * nx
    T = np.zeros((n_t // 2 * b, n_t * b))
    I = np.eye(nx)
    for n in range(n_t // 2):
        T[n * b:(n + 1) * b, 2 * n * b:(2 * n + 1) * b] = np.kron(R1, I)
        T[n * b:(n + 1) * b, (2 * n + 1) * b:(2 * n + 2) * b] = np.kron(R2, I)
    return T


def spatial_vcycle(p, tau, dim, level, b, x0=None, omega_x=2.0 / 3.0, nu1_x=2, nu2_x=2,
                   gamma_x=1):
    """Dense restatement of SpatialVCycleSolver::cycle (smoother.cpp:8-78) on one
    slab b (DG-major, length (p+1) * n1^dim): damped point-block Jacobi with
    D = K diag(M_h) + M diag(K_h), full weighting / its transpose per DG
    component, numpy.linalg.solve on the 1-node grid."""
    K, M, _ = dg_block(p, tau)
    nl = p + 1

    def rec(s, x, rhs):
        Mh, Kh = space_mats(dim, s)
        A = dense_block(K, M, Mh, Kh)
        if s == 0:
            return np.linalg.solve(A, rhs)
        D = np.kron(K * Mh[0, 0] + M * Kh[0, 0], np.eye(Mh.shape[0]))
        for _ in range(nu1_x):
            x = x + omega_x * np.linalg.solve(D, rhs - A @ x)
        r = rhs - A @ x
        Rf = np.kron(np.eye(nl), space_restriction(dim, s))
        rc = Rf @ r
        ec = np.zeros_like(rc)
        for _ in range(gamma_x):
            ec = rec(s - 1, ec, rc)
        x = x + Rf.T @ ec
        for _ in range(nu2_x):
            x = x + omega_x * np.linalg.solve(D, rhs - A @ x)
        return x

    x = np.zeros_like(b) if x0 is None else np.array(x0, dtype=np.float64)
    return rec(level, x, b)


class DenseHierarchy:
    """Dense restatement of build_hierarchy + mg_cycle (mg.cpp:10-132)."""

    def __init__(self, p_t, dim, space_level, time_level, t_final=1.0, mu_star=0.3, policy=0,
                 block_solver="exact", spatial=None):
        self.levels = []
        self.p_t, self.dim = p_t, dim
        self.block_solver = block_solver  # "exact" | "vcycle" (smoother.cpp:82-92)
        self.spatial = dict(spatial or {})
        n_t = 2 ** time_level
        tau = t_final / n_t
        s = space_level
        while True:
            K, M, N = dg_block(p_t, tau)
            Mh, Kh = space_mats(dim, s)
            h = 2.0 ** -(s + 1)
            lev = dict(n_t=n_t, s=s, tau=tau, mu=tau / h ** 2, K=K, M=M, N=N,
                       A=dense_block(K, M, Mh, Kh),
                       L=dense_space_time(K, M, N, Mh, Kh, n_t), nx=Mh.shape[0],
                       coarsen=0)
            self.levels.append(lev)
            if n_t == 1:
                break
            full = (lev["mu"] >= mu_star and s > 0) if policy == 0 else (s > 0 if policy == 2 else False)
            lev["coarsen"] = 2 if full else 1
            R1, R2 = time_transfer(p_t, tau)
            T = time_restriction(R1, R2, n_t, lev["nx"])
            if full:
                Rs = space_restriction(dim, s)
                nl = p_t + 1
                Rs_full = np.kron(np.eye(n_t // 2 * nl), Rs)
                lev["R"] = Rs_full @ T
            else:
                lev["R"] = T
            n_t //= 2
            tau *= 2
            if full:
                s -= 1

    def smooth(self, lev, u, f, omega, nu):
        L = self.levels[lev]
        b = L["A"].shape[0]
        for _ in range(nu):
            r = f - L["L"] @ u
            if self.block_solver == "vcycle":
                rs = r.reshape(L["n_t"], b)
                x = np.concatenate([spatial_vcycle(self.p_t, L["tau"], self.dim, L["s"], rs[n],
                                                   **self.spatial) for n in range(L["n_t"])])
            else:
                x = np.linalg.solve(L["A"], r.reshape(L["n_t"], b).T).T.reshape(-1)
            u = u + omega * x
        return u

    def cycle(self, lev, u, f, nu1=1, nu2=1, gamma=1, omega=0.5):
        L = self.levels[lev]
        if lev + 1 == len(self.levels):
            return np.linalg.solve(L["L"], f)
        u = self.smooth(lev, u, f, omega, nu1)
        r = f - L["L"] @ u
        rc = L["R"] @ r
        ec = np.zeros_like(rc)
        for _ in range(gamma):
            ec = self.cycle(lev + 1, ec, rc, nu1, nu2, gamma, omega)
        u = u + L["R"].T @ ec
        return self.smooth(lev, u, f, omega, nu2)
