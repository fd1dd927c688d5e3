# FP32 error of exact-tracker formulations vs the FP64 reference.
#   PYTHONPATH=. python tools/fp32_tracker_study.py literal cheb mono
# numpy complex64 emulation of: the literal Eq.(10) recursion (detect.cpp:350-358),
# the Chebyshev-basis coefficient recursion used by the kernels, and the monomial
# basis; compared with the reference library (oracle/_ref) on random channels.
import numpy as np, oracle, sys
ref = oracle.Oracle('ref')
import os
PIT = int(os.environ.get('PIT', 12)); PMARGIN = float(os.environ.get('PMARGIN', 1.05))
f32, c64 = np.float32, np.complex64

def gen(B, U, n, S, n0, bits, rng, corr=False):
    H = ((rng.standard_normal((n, B, U)) + 1j*rng.standard_normal((n, B, U)))/np.sqrt(2)).astype(c64)
    pts, _, _ = ref.constellation(bits)
    X = pts[rng.integers(0, 1 << bits, (n, S, U))]
    N = (rng.standard_normal((n, S, B)) + 1j*rng.standard_normal((n, S, B)))*np.sqrt(n0/2)
    Y = (np.einsum('nbu,nsu->nbs', H.astype(np.complex128), X) + N.transpose(0, 2, 1)).astype(c64)
    return H, Y

def llr_np(z, rho, bits, pts_axes):
    a0, a1 = pts_axes
    out = []
    for comp in (z.real, z.imag):
        for p in range(bits//2):
            d0 = np.min((comp[..., None]-a0[p])**2, -1); d1 = np.min((comp[..., None]-a1[p])**2, -1)
            out.append(np.clip(rho*(d0-d1), -64, 64))
    return np.stack(out, -1)

def cg32(A, b, K):
    U = A.shape[0]
    v = np.zeros(U, c64); r = b.copy(); p = b.copy(); rn = f32(np.vdot(r, r).real); rn0 = rn
    al, be = [], []
    for k in range(K):
        a, bb = f32(1), f32(0)
        if not rn <= 1e-28*rn0:
            e = A @ p; curv = f32(np.vdot(p, e).real)
            a = f32(rn/curv); v = v + a*p; r = r - a*e; rn2 = f32(np.vdot(r, r).real); bb = f32(rn2/rn); rn = rn2; p = r + bb*p
        al.append(a); be.append(bb)
    return v, al, be

def literal_L(A, al, be):
    U = A.shape[0]; I = np.eye(U, dtype=c64)
    L = np.zeros_like(A); L1 = np.zeros_like(A); L2 = np.zeros_like(A)
    am1 = am2 = f32(1); bm1 = bm2 = f32(0)
    for k, (a, b) in enumerate(zip(al, be)):
        if k == 0: L2, L1, L = L1, L, a*I
        else:
            c1 = f32(a*(1+bm1)/am1); c2 = f32(a*bm2/am2)
            D1 = L-L1; D2 = L1-L2
            N = L + c1*D1 - a*(A@D1) - c2*D2
            L2, L1, L = L1, L, N
        am2, am1, bm2, bm1 = am1, a, bm1, b
    return L

def coeff_L(al, be, K, mulA):
    # three-term recursion on coefficient vectors (length K+1), mulA maps coeffs of p(A) to coeffs of A p(A)
    n = K+2
    L = np.zeros(n); L1 = np.zeros(n); L2 = np.zeros(n)
    am1 = am2 = 1.0; bm1 = bm2 = 0.0
    for k, (a, b) in enumerate(zip(al, be)):
        a = float(a); b = float(b)
        if k == 0: L2, L1, L = L1, L, a*np.eye(n)[0]
        else:
            c1 = a*(1+bm1)/am1; c2 = a*bm2/am2
            D1 = L-L1; D2 = L1-L2
            N = L + c1*D1 - a*mulA(D1) - c2*D2
            L2, L1, L = L1, L, N
        am2, am1, bm2, bm1 = am1, a, bm1, b
    return L

def run(B, U, S, K, snr_db, bits, nsc=40, mode='literal', seed=0):
    rng = np.random.default_rng(seed)
    n0 = U/10**(snr_db/10); rho_u = 1/n0
    H, Y = gen(B, U, nsc, S, n0, bits, rng)
    R = ref.detect(H, Y, rho_u, n0, 1.0, bits, K, 'exact')
    _, a0, a1 = ref.constellation(bits)
    errs = dict(x=[], mu=[], rho=[]); llr_fail = 0; llr_tot = 0; hard = 0
    for n in range(nsc):
        Hn = H[n]; A = (Hn.conj().T @ Hn).astype(c64); A[np.diag_indices(U)] += f32(1/rho_u)
        G = A.copy(); G[np.diag_indices(U)] -= f32(1/rho_u)
        if mode != 'literal':
            c = f32(np.trace(A).real/U)
            dev = A - c*np.eye(U, dtype=c64)
            # half-width from Gershgorin-like radius or frobenius
            if mode == 'cheb':
                d = f32(np.sqrt(np.sum(np.abs(dev)**2)/U)*2.5)
            elif mode == 'chebk':  # the kernels' round-1 choice
                d = f32(np.sqrt(np.sum(np.abs(dev)**2)/U)*2.0)
            elif mode in ('chebpos', 'chebrow'):
                # positive interval [rho^-1, lambda_max]: A = G + rho^-1 I >= rho^-1 I
                lo = f32(1/rho_u)
                if mode == 'chebpos':  # power-iteration estimate of lambda_max, margin
                    x = np.ones(U, c64)
                    for _ in range(PIT):
                        x = (A @ x).astype(c64); x /= np.linalg.norm(x)
                    hi = f32(np.vdot(x, A @ x).real * PMARGIN)
                else:  # Gershgorin row-sum bound
                    hi = f32(np.max(np.sum(np.abs(A), 1)))
                c = f32((lo + hi) / 2); d = f32((hi - lo) / 2)
            else:
                d = f32(1.0); c = f32(0.0)
            Ah = ((A - c*np.eye(U, dtype=c64))/d).astype(c64)
            T = [np.eye(U, dtype=c64), Ah]
            for m in range(2, K+2):
                T.append((2*(Ah@T[-1]) - T[-2]).astype(c64) if mode.startswith('cheb') else (Ah@T[-1]).astype(c64))
            def mulA(co):
                out = c*co.copy()
                if mode.startswith('cheb'):
                    sh = np.zeros_like(co)
                    sh[1] += co[0]
                    for m in range(1, len(co)-1):
                        sh[m+1] += co[m]/2; sh[m-1] += co[m]/2
                    return out + d*sh
                else:
                    sh = np.zeros_like(co); sh[1:] = co[:-1]; return out + d*sh
        for s in range(S):
            b = (Hn.conj().T @ Y[n, :, s]).astype(c64)
            v, al, be = cg32(A, b, K)
            if mode == 'literal':
                L = literal_L(A, al, be); Bm = L @ G
            else:
                lc = coeff_L(al, be, K, mulA)
                bc = mulA(lc) - (1/rho_u)*lc
                L = sum(f32(lc[m])*T[m] for m in range(K+1)).astype(c64)
                Bm = sum(f32(bc[m])*T[m] for m in range(K+2)).astype(c64)
            mu = Bm.diagonal().real
            offd = np.abs(Bm)**2; np.fill_diagonal(offd, 0)
            nu2 = offd.sum(1) + n0*(np.sum(Bm*L.conj(), 1)).real
            rho = mu*mu/nu2
            llr = llr_np(v/mu, rho, bits, (a0, a1))
            rx = R['xhat'][n, s]; rmu = R['mu'][n, s]; rrho = R['rho'][n, s]; rl = R['llr'][n, s]
            errs['x'].append(np.max(np.abs(v-rx)/np.abs(rx)))
            errs['mu'].append(np.max(np.abs(mu-rmu)/np.abs(rmu)))
            errs['rho'].append(np.max(np.abs(rho-rrho)/np.abs(rrho)))
            rl = rl.reshape(llr.shape)
            bad = np.abs(llr-rl) > 1e-3*np.abs(rl) + 1e-4
            llr_fail += bad.sum(); llr_tot += bad.size
            hard += np.sum(((llr > 0) != (rl > 0)) & (np.abs(rl) >= 1e-4))
    print(f"B={B} U={U} K={K} {mode:8s} x {np.max(errs['x']):.1e} mu {np.max(errs['mu']):.1e} rho {np.max(errs['rho']):.1e} llr_fail {llr_fail}/{llr_tot} hard {hard}")

if sys.argv[1] == 'weak':  # U = 64 weakly regularised (rho_u ~ 10), K = 8 / 16
    for mode in sys.argv[2:]:
        run(128, 64, 2, 8, 28, 6, 6, mode)
        run(128, 64, 2, 16, 28, 6, 6, mode)
    sys.exit(0)
for mode in sys.argv[1:]:
    run(128, 8, 1, 3, 10, 4, 60, mode)
    run(64, 32, 2, 2, 20, 6, 20, mode)
    run(64, 32, 2, 8, 20, 6, 20, mode)
    run(128, 64, 1, 8, 20, 6, 6, mode)
    run(256, 32, 4, 4, 15, 6, 10, mode)
