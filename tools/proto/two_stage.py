"""numpy prototype of the two-stage symmetric eigensolver (design aid for
csrc/syev2.cu): dense -> band (panel QR + two-sided compact-WY update),
band -> tridiagonal (Householder bulge chasing), top-k eigenvalues of T,
eigenvectors by inverse iteration on the band matrix, back-transform Q1."""
import numpy as np
import scipy.linalg as sl


def house(x):
    alpha = x[0]
    xn2 = float(x[1:] @ x[1:])
    v = x.copy()
    v[0] = 1.0
    if xn2 == 0.0:
        return v * 0 + np.eye(len(x))[0], 0.0, alpha
    nrm = np.sqrt(alpha * alpha + xn2)
    beta = -nrm if alpha >= 0 else nrm
    tau = (beta - alpha) / beta
    v[1:] = x[1:] / (alpha - beta)
    return v, tau, beta


def panel_qr(P):
    m, b = P.shape
    P = P.copy()
    V = np.zeros((m, b))
    taus = np.zeros(b)
    for t in range(b):
        if t >= m:
            break
        v, tau, beta = house(P[t:, t])
        V[t:, t] = v
        taus[t] = tau
        P[t:, t:] -= tau * np.outer(v, v @ P[t:, t:])
    T = np.zeros((b, b))
    for t in range(b):
        T[t, t] = taus[t]
        if t:
            T[:t, t] = -taus[t] * T[:t, :t] @ (V[:, :t].T @ V[:, t])
    R = np.triu(P[:b, :])
    return V, T, R


def sy2sb(A, b):
    A = A.copy()
    n = A.shape[0]
    refl = []
    for j0 in range(0, n - b - 1, b):
        r0 = j0 + b
        P = A[r0:, j0:j0 + b]
        V, T, R = panel_qr(P)
        m = n - r0
        A[r0:, j0:j0 + b] = 0.0
        A[r0:r0 + min(b, m), j0:j0 + b] = R[:min(b, m)]
        A[j0:j0 + b, r0:] = A[r0:, j0:j0 + b].T
        A22 = A[r0:, r0:]
        X = A22 @ V @ T
        M = T.T @ (V.T @ X)
        W = X - 0.5 * V @ M
        A[r0:, r0:] = A22 - V @ W.T - W @ V.T
        refl.append((r0, V, T))
    return A, refl


def sb2st(B, b):
    B = B.copy()
    n = B.shape[0]
    for j in range(n - 2):
        k = 0
        while True:
            r0 = j + 1 + k * b
            c = j if k == 0 else j + 1 + (k - 1) * b
            r1 = min(n, r0 + b)
            if r1 - r0 < 2:
                break
            x = B[r0:r1, c]
            if np.abs(x[1:]).max() == 0.0:
                break
            v, tau, beta = house(x)
            B[r0:r1, :] -= tau * np.outer(v, v @ B[r0:r1, :])
            B[:, r0:r1] -= tau * np.outer(B[:, r0:r1] @ v, v)
            k += 1
    return B


def band_invit(B, b, lam, iters=3):
    n = B.shape[0]
    ab = np.zeros((2 * b + 1, n))
    rng = np.random.default_rng(0)
    Z = np.zeros((n, len(lam)))
    for t, l in enumerate(lam):
        M = B - l * np.eye(n) + 1e-300
        for i in range(2 * b + 1):
            off = b - i
            ab[i] = 0
            if off >= 0:
                ab[i, off:] = np.diagonal(M, off)
            else:
                ab[i, :n + off] = np.diagonal(M, off)
        x = rng.uniform(-1, 1, n)
        for _ in range(iters):
            x = sl.solve_banded((b, b), ab, x)
            x /= np.linalg.norm(x)
        Z[:, t] = x
    return Z


if __name__ == "__main__":
    rng = np.random.default_rng(1)
    n, b, k = 300, 16, 40
    X = rng.standard_normal((400, n)) * np.exp(-np.linspace(0, 6, n))
    A = X.T @ X
    Bd, refl = sy2sb(A, b)
    i, j = np.indices(Bd.shape)
    print("band defect", np.abs(Bd[np.abs(i - j) > b]).max() / np.abs(A).max())
    ev = np.linalg.eigvalsh(A)[::-1]
    print("band eig err", np.abs(np.linalg.eigvalsh(Bd)[::-1] - ev).max() / ev[0])
    T = sb2st(Bd, b)
    print("tridiag defect", np.abs(T[np.abs(i - j) > 1]).max() / ev[0])
    print("fill max bandwidth during chase ok")
    d, e = np.diagonal(T).copy(), np.diagonal(T, -1).copy()
    lt = sl.eigvalsh_tridiagonal(d, e)[::-1][:k]
    print("tridiag eig err", np.abs(lt - ev[:k]).max() / ev[0])
    Zb = band_invit(Bd, b, lt)
    # back-transform: Z <- Q1 Z, Q1 = Q_0 Q_1 ... (apply last first)
    Z = Zb.copy()
    for r0, V, Tm in reversed(refl):
        Z[r0:] -= V @ (Tm @ (V.T @ Z[r0:]))
    w, U = np.linalg.eigh(A)
    U = U[:, ::-1][:, :k]
    print("vector residual", np.abs(A @ Z - Z * lt).max() / ev[0])
    print("subspace sin", np.linalg.norm(U - Z @ (Z.T @ U), 2))


def sb2st_instrumented(B, b):
    B = B.copy()
    n = B.shape[0]
    maxbw = 0
    cols_touched = 0
    for j in range(n - 2):
        k = 0
        while True:
            r0 = j + 1 + k * b
            c = j if k == 0 else j + 1 + (k - 1) * b
            r1 = min(n, r0 + b)
            if r1 - r0 < 2:
                break
            x = B[r0:r1, c]
            if np.abs(x[1:]).max() == 0.0:
                break
            # nonzero column extent of rows r0..r1
            nz = np.nonzero(np.abs(B[r0:r1, :]).max(axis=0) > 0)[0]
            cols_touched = max(cols_touched, nz.max() - c + 1)
            assert nz.min() >= c, (nz.min(), c)
            v, tau, beta = house(x)
            B[r0:r1, :] -= tau * np.outer(v, v @ B[r0:r1, :])
            B[:, r0:r1] -= tau * np.outer(B[:, r0:r1] @ v, v)
            ii, jj = np.nonzero(np.abs(B) > 1e-300)
            maxbw = max(maxbw, (ii - jj).max())
            k += 1
    return maxbw, cols_touched


if __name__ == "__main__":
    for (n, b) in [(120, 8), (130, 16), (97, 4)]:
        A = rng.standard_normal((n, n))
        A = A + A.T
        Bd, _ = sy2sb(A, b)
        print(n, b, "max bandwidth during chase", sb2st_instrumented(Bd, b))
