"""numpy prototype of the blocked Q2 back-transform (design aid for
csrc/syev_band.cu k_q2_tbuild / k_q2_wy).

The bulge chase of a bandwidth-b band leaves reflectors H(s, k) (sweep s,
step k) acting on rows s+1+b*k .. s+b+b*k; Q2 = prod_s prod_k H(s, k) in chase
order.  Blocked form: groups of nb consecutive sweeps (group a = sweeps
nb*a-1 .. nb*a+nb-2, so that a group's window starts on an nb-aligned row),
block (a, k) = H(s0, k) H(s0+1, k) ... H(s0+nb-1, k) = I - V T V^T
(V: (b+nb-1) x nb parallelogram, T upper, dlarft 'F'), and a super-group of
G groups is applied in one downward pass: for k ascending, groups
descending.  Super-groups are applied last first.  Checks the result
against the reflector-by-reflector application."""
import numpy as np

from two_stage import house


def chase_reflectors(B, b):
    B = B.copy()
    n = B.shape[0]
    refl = {}
    for s in range(n - 2):
        k = 0
        while True:
            r0 = s + 1 + k * b
            c = s if k == 0 else s + 1 + (k - 1) * b
            r1 = min(n, r0 + b)
            if r1 - r0 < 2:
                break
            x = B[r0:r1, c]
            if np.abs(x[1:]).max() == 0.0:
                break
            v, tau, beta = house(x)
            B[r0:r1, :] -= tau * np.outer(v, v @ B[r0:r1, :])
            B[:, r0:r1] -= tau * np.outer(B[:, r0:r1] @ v, v)
            vv = np.zeros(b)
            vv[:r1 - r0] = v
            refl[(s, k)] = (vv, tau)
            k += 1
    return B, refl


def q2_sequential(refl, n, b, Z):
    Z = Z.copy()
    for (s, k) in sorted(refl, reverse=True):  # last sweep first
        v, tau = refl[(s, k)]
        r0 = s + 1 + k * b
        L = min(b, n - r0)
        Z[r0:r0 + L] -= tau * np.outer(v[:L], v[:L] @ Z[r0:r0 + L])
    return Z


def q2_blocked(refl, n, b, Z, nb=8, G=8):
    Z = Z.copy()
    W = b + nb - 1
    ngroups = (n - 2) // nb + 1
    nsg = (ngroups + G - 1) // G
    for sg in reversed(range(nsg)):
        k = 0
        while True:
            active = False
            for g in reversed(range(G)):
                a = sg * G + g
                s0 = nb * a - 1
                base = s0 + 1 + b * k
                V = np.zeros((W, nb))
                taus = np.zeros(nb)
                for j in range(nb):
                    if (s0 + j, k) in refl:
                        v, tau = refl[(s0 + j, k)]
                        V[j:j + b, j] = v
                        taus[j] = tau
                if not taus.any():
                    continue
                active = True
                T = np.zeros((nb, nb))
                for j in range(nb):
                    T[j, j] = taus[j]
                    if j:
                        T[:j, j] = -taus[j] * T[:j, :j] @ (V[:, :j].T @ V[:, j])
                rows = slice(base, min(n, base + W))
                Vr = V[:rows.stop - base]
                Z[rows] -= Vr @ (T @ (Vr.T @ Z[rows]))
            k += 1
            if not active and b * k > n:
                break
    return Z


if __name__ == "__main__":
    rng = np.random.default_rng(3)
    b = 32
    for n in (70, 129, 300):
        A = rng.standard_normal((n, n))
        A = A + A.T
        B = np.triu(np.tril(A, b), -b)
        Bt, refl = chase_reflectors(B, b)
        Z = rng.standard_normal((n, 5))
        z1 = q2_sequential(refl, n, b, Z)
        z2 = q2_blocked(refl, n, b, Z)
        # Q2^T B Q2 is the tridiagonal
        Q = q2_sequential(refl, n, b, np.eye(n))
        tri_err = np.abs(Q.T @ B @ Q - Bt).max()
        print(n, len(refl), np.abs(z1 - z2).max(), tri_err)
