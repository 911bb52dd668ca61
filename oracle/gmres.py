"""ORACLE — TEST INFRASTRUCTURE ONLY.  Restarted GMRES (Saad & Schultz 1986, cited at P:778)
with modified Gram-Schmidt Arnoldi and complex Givens rotations.

Reading R14: zero initial guess; restart m = 50; stop when the implicit
residual |g_{j+1}| / ||f|| <= tol (the relative residual of P:821) or after maxit inner
iterations; the returned relres is recomputed as ||f - A psi|| / ||f|| with the same
operator.
"""
import numpy as np


def givens(a, b):
    """(c, s) with c real such that [c s; -conj(s) c] [a; b] = [rho; 0]."""
    if b == 0:
        return 1.0, 0.0
    if a == 0:
        return 0.0, 1.0
    rho = np.sqrt(abs(a) ** 2 + abs(b) ** 2)
    c = abs(a) / rho
    s = (a / abs(a)) * np.conj(b) / rho
    return c, s


def gmres(matvec, f, tol, restart=50, maxit=1000):
    """Solve A psi = f.  Returns (psi, iterations, relres_true, history, converged)."""
    f = np.asarray(f, dtype=np.complex128)
    n = f.size
    bnorm = np.linalg.norm(f)
    psi = np.zeros(n, dtype=np.complex128)
    history = [1.0]
    if bnorm == 0.0:
        return psi, 0, 0.0, history, True
    iters = 0
    converged = False
    r = f.copy()  # psi0 = 0
    while iters < maxit and not converged:
        beta = np.linalg.norm(r)
        if beta / bnorm <= tol:
            converged = True
            break
        m = restart
        V = np.zeros((m + 1, n), dtype=np.complex128)
        H = np.zeros((m + 1, m), dtype=np.complex128)
        cs = np.zeros(m)
        sn = np.zeros(m, dtype=np.complex128)
        g = np.zeros(m + 1, dtype=np.complex128)
        g[0] = beta
        V[0] = r / beta
        k = 0
        for j in range(m):
            w = matvec(V[j])
            iters += 1
            for i in range(j + 1):  # modified Gram-Schmidt
                H[i, j] = np.vdot(V[i], w)
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] != 0:
                V[j + 1] = w / H[j + 1, j]
            for i in range(j):  # previous rotations
                hi, hi1 = H[i, j], H[i + 1, j]
                H[i, j] = cs[i] * hi + sn[i] * hi1
                H[i + 1, j] = -np.conj(sn[i]) * hi + cs[i] * hi1
            cs[j], sn[j] = givens(H[j, j], H[j + 1, j])
            H[j, j] = cs[j] * H[j, j] + sn[j] * H[j + 1, j]
            H[j + 1, j] = 0.0
            g[j + 1] = -np.conj(sn[j]) * g[j]
            g[j] = cs[j] * g[j]
            k = j + 1
            history.append(abs(g[j + 1]) / bnorm)
            if abs(g[j + 1]) / bnorm <= tol:
                converged = True
                break
            if iters >= maxit:
                break
        y = np.zeros(k, dtype=np.complex128)  # back substitution H[:k,:k] y = g[:k]
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - np.dot(H[i, i + 1:k], y[i + 1:k])) / H[i, i]
        psi = psi + V[:k].T @ y
        r = f - matvec(psi)
    relres = np.linalg.norm(f - matvec(psi)) / bnorm
    return psi, iters, relres, history, converged
