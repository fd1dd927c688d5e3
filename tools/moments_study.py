# FP32 error of the "row-moment" exact-tracker extraction vs the FP64 reference.
#   PYTHONPATH=. python tools/moments_study.py
# L_K and B = L_K G are real-coefficient polynomials in A, expanded in the
# Chebyshev basis T_m(Ahat): L = sum_n l_n T_n, B = sum_m g_m T_m.  With
#   D_m[i]    = Re T_m[i,i]                                (T_0 = I -> D_0 = 1)
#   Q_mn[i]   = Re sum_{j != i} T_m[i,j] conj(T_n[i,j])    (Q_0n = 0)
# the reference's extraction (detect.cpp:375-395) is, per row i,
#   mu_i  = sum_m g_m D_m[i]
#   sum_{j!=i} |B_ij|^2        = sum_{m,n>=1} g_m g_n Q_mn[i]
#   Re sum_j B_ij conj(L_ij)   = mu_i L_ii + sum_{m,n>=1} g_m l_n Q_mn[i]
# so per vector the extraction is O(K^2 U) instead of O(K U^2).
import sys
import numpy as np
sys.argv = [sys.argv[0], 'none']
import tools.fp32_tracker_study as st  # noqa: E402

f32, c64 = np.float32, np.complex64
QST = np.float32
DONLY = False
ref = st.ref


def run(B, U, S, K, snr_db, bits, nsc=20, corr=0.0, seed=0, accum=np.float32, tdt=c64):
    rng = np.random.default_rng(seed)
    n0 = U / 10 ** (snr_db / 10); rho_u = 1 / n0
    H, Y = st.gen(B, U, nsc, S, n0, bits, rng)
    if corr:
        idx = np.arange(B); Rm = corr ** np.abs(idx[:, None] - idx[None, :])
        w, V = np.linalg.eigh(Rm); Rs = (V * np.sqrt(np.clip(w, 0, None))) @ V.T
        H = np.einsum('bc,ncu->nbu', Rs, H.astype(np.complex128)).astype(c64)
        pts, _, _ = ref.constellation(bits)
        X = pts[rng.integers(0, 1 << bits, (nsc, S, U))]
        N = (rng.standard_normal((nsc, B, S)) + 1j * rng.standard_normal((nsc, B, S))) * np.sqrt(n0 / 2)
        Y = (np.einsum('nbu,nsu->nbs', H.astype(np.complex128), X) + N).astype(c64)
    R = ref.detect(H, Y, rho_u, n0, 1.0, bits, K, 'exact')
    _, a0, a1 = ref.constellation(bits)
    e = dict(x=0.0, mu=0.0, rho=0.0); lf = lt = hard = 0
    for n in range(nsc):
        Hn = H[n]; A = (Hn.conj().T @ Hn).astype(c64); A[np.diag_indices(U)] += f32(1 / rho_u)
        lo = f32(1 / rho_u)
        x = np.ones(U, c64)
        for _ in range(7):
            x = (A @ x).astype(c64); x /= np.linalg.norm(x)
        hi = f32(np.vdot(x, A @ x).real * 1.1)
        c = f32((lo + hi) / 2); d = f32((hi - lo) / 2)
        Ah = ((A - c * np.eye(U, dtype=c64)) / d).astype(c64)
        T = [np.eye(U, dtype=tdt), Ah.astype(tdt)]
        for m in range(2, K + 1):
            T.append((2 * (Ah @ T[-1]) - T[-2]).astype(tdt))
        D = np.array([T[m].diagonal().real for m in range(K + 1)], dtype=QST)
        Q = np.zeros((K + 1, K + 1, U), accum)
        if DONLY:
            # diagonals of T_k, k <= 2K, from row products of T_a, T_{a-1} only
            Dk = np.zeros((2 * K + 1, U), accum); Dk[0] = 1; Dk[1] = T[1].diagonal().real
            for a in range(1, K + 1):
                Dk[2 * a] = 2 * (T[a] * T[a].conj()).real.astype(accum).sum(1, dtype=accum) - 1
                if a >= 2:
                    Dk[2 * a - 1] = 2 * (T[a] * T[a - 1].conj()).real.astype(accum).sum(1, dtype=accum) - Dk[1]
            Dk = Dk.astype(QST)
            for m in range(1, K + 1):
                for q in range(1, K + 1):
                    Q[m, q] = (Dk[m + q] + Dk[abs(m - q)]) / 2 - Dk[m] * Dk[q]
            D = Dk[:K + 1]
        else:
          for m in range(1, K + 1):
            for q in range(m, K + 1):
                P = (T[m] * T[q].conj()).real.astype(accum)
                np.fill_diagonal(P, 0)
                Q[m, q] = Q[q, m] = P.sum(1, dtype=accum)
        Q = Q.astype(QST)

        def mulA(co):
            out = c * co.copy(); sh = np.zeros_like(co); sh[1] += co[0]
            for m in range(1, len(co) - 1):
                sh[m + 1] += co[m] / 2; sh[m - 1] += co[m] / 2
            return out + d * sh
        for s in range(S):
            b = (Hn.conj().T @ Y[n, :, s]).astype(c64)
            v, al, be = st.cg32(A, b, K)
            lc = st.coeff_L(al, be, K, mulA)
            gc = mulA(lc) - (1 / rho_u) * lc
            mu = gc[0] + sum(gc[m] * D[m] for m in range(1, K + 1))
            Lii = lc[0] + sum(lc[m] * D[m] for m in range(1, K + 1))
            inter = sum(gc[m] * gc[q] * Q[m, q] for m in range(1, K + 1) for q in range(1, K + 1))
            cross = mu * Lii + sum(gc[m] * lc[q] * Q[m, q] for m in range(1, K + 1) for q in range(1, K + 1))
            nu2 = inter + n0 * cross
            rho = (mu * mu / nu2).astype(f32); mu = mu.astype(f32)
            llr = st.llr_np(v / mu, rho, bits, (a0, a1))
            rx = R['xhat'][n, s]; rmu = R['mu'][n, s]; rrho = R['rho'][n, s]; rl = R['llr'][n, s].reshape(llr.shape)
            e['x'] = max(e['x'], np.max(np.abs(v - rx) / np.abs(rx)))
            e['mu'] = max(e['mu'], np.max(np.abs(mu - rmu) / np.abs(rmu)))
            e['rho'] = max(e['rho'], np.max(np.abs(rho - rrho) / np.abs(rrho)))
            bad = np.abs(llr - rl) > 1e-3 * np.abs(rl) + 1e-4
            lf += bad.sum(); lt += bad.size
            hard += np.sum(((llr > 0) != (rl > 0)) & (np.abs(rl) >= 1e-4))
    print(f"B={B} U={U} K={K} snr={snr_db} corr={corr} moments: x {e['x']:.1e} mu {e['mu']:.1e} "
          f"rho {e['rho']:.1e} llr_fail {lf}/{lt} hard {hard}", flush=True)


if __name__ == '__main__':
    run(128, 8, 1, 3, 10, 4, 60)
    for K in (2, 4, 8):
        run(64, 32, 2, K, 20, 6, 20)
    run(128, 64, 1, 8, 20, 6, 6)
    run(256, 32, 4, 4, 15, 6, 10, corr=0.5)
    run(128, 64, 2, 8, 28, 6, 6)
    run(128, 64, 2, 16, 28, 6, 6)
