"""numpy checker for b2l_rayleigh_ritz (test infrastructure only).

The Rayleigh-Ritz step of one iteration on the projected Gram blocks, with
the reference's repair ladders (lobpcg.py:475-519, b_orthonormalize
:147-200), written with numpy / scipy LAPACK exactly as the host solver did
before the step moved into the native library.  Same inputs and outputs as
small.NativeRitz.
"""

import numpy as np

from paper_0705_2626_b200.small import NotSPD, gen_sym_eig, scaled_cholesky


class Degenerate(Exception):
    def __init__(self, fallbacks):
        super().__init__("BasisDegeneracy")
        self.fallbacks = fallbacks


def rayleigh_ritz_ref(m, kst, have_p, G1, G2, lam, J, sel, floor):
    rW, rP = m, m + kst
    cW, cP, cAP = m, m + kst, 2 * m + kst
    pending = 0
    keep = list(range(J.size))
    mw = None
    while keep:
        ks = sel[keep]
        try:
            _, mw = scaled_cholesky(G1[rW + ks][:, cW + ks], floor)
            break
        except NotSPD as err:
            del keep[err.pivot]
    pending += J.size - len(keep)
    if not keep:
        raise Degenerate(pending)
    wcols = sel[keep]
    mp = None
    if have_p:
        try:
            _, mp = scaled_cholesky(G1[rP + J][:, cP + J], floor)
        except NotSPD:
            pending += 1
    gXAW = G2[:m][:, wcols]
    gWAW = G2[m + wcols][:, wcols]
    gXBW = G1[:m][:, cW + wcols]
    if have_p:
        gXAP = G1[:m][:, cAP + J]
        gWAP = G1[rW + wcols][:, cAP + J]
        gXBP = G1[:m][:, cP + J]
        gWBP = G1[rW + wcols][:, cP + J]
        gPAP = G1[rP + J][:, cAP + J]
    use_p = mp is not None
    while True:
        kw = mw.shape[1]
        kp = J.size if use_p else 0
        d = m + kw + kp
        ga = np.zeros((d, d))
        gb = np.zeros((d, d))
        sx, sw, sp = slice(0, m), slice(m, m + kw), slice(m + kw, d)
        ga[sx, sx] = np.diag(lam)
        gb[sx, sx] = np.eye(m)
        ga[sw, sw] = mw.T @ gWAW @ mw
        gb[sw, sw] = np.eye(kw)
        ga[sx, sw] = gXAW @ mw
        gb[sx, sw] = gXBW @ mw
        if kp:
            ga[sx, sp] = gXAP @ mp
            ga[sw, sp] = mw.T @ gWAP @ mp
            gb[sx, sp] = gXBP @ mp
            gb[sw, sp] = mw.T @ gWBP @ mp
            ga[sp, sp] = mp.T @ gPAP @ mp
            gb[sp, sp] = np.eye(kp)
        try:
            lam_new, c = gen_sym_eig(ga, gb, m, floor)
            break
        except NotSPD as err:
            pending += 1
            if use_p:
                use_p = False
            elif m <= err.pivot < m + kw and kw > 1:
                mw = mw[:, np.arange(kw) != err.pivot - m]
            else:
                raise Degenerate(pending)
    kw = mw.shape[1]
    cx, cw, cp = c[:m], c[m:m + kw], c[m + kw:]
    cw_raw = np.zeros((kst, m))
    cw_raw[wcols] = mw @ cw
    if use_p:
        cp_raw = mp @ cp
        pcols = J.astype(np.int32)
    else:
        cp_raw = np.zeros((0, m))
        pcols = np.zeros(0, dtype=np.int32)
    coef = np.concatenate([cx.ravel(), cw_raw.ravel(), cp_raw.ravel()])
    return lam_new, coef, pcols, pending
