"""Float64 oracle for Algorithm 3 (RPCA+UOT-DF ADMM).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): only tests/, __graft_entry__
and bench.py's CPU legs may import it; it shares no code with the CUDA path.

Problem (eq:RPCA_UOTDF), frames t = 0..T-1 (the paper's 1..T):
    min_{S, L >= 0}  1/2 sum_t ||y_t - Phi_t (s_t + l_t)||^2 + lambda ||S||_1
                     + gamma ||L||_* + kappa sum_{t<T-1} V_mu(s_t, s_{t+1})
with Phi_t DIAGONAL (per-pixel weights phi_t; Phi = I by default) -- the case the
paper calls O(TN); dense Phi is out of scope.

The ADMM of the split problem follows Algorithm 3 line by
line, in its order, with plain numpy in float64:
  line 5  k_t = (x_t - l_t + a_t) + wz_t (z_t + b_t) + ww_t (w_t + c_t)
  line 6  sigma_t = 1 + wz_t + ww_t          (wz_t = 1 for t < T-1, ww_t = 1 for t > 0)
  line 7  s_t = max(k_t/sigma_t - lambda/(rho sigma_t), 0)                       (L25)
  line 8  L = Pi_+((T - D + X - S + A)/2)
  line 9  x_t = (Phi_t^T Phi_t + rho I)^{-1}(Phi_t^T y_t + rho (s_t + l_t - a_t))   (L26)
  line 10 T = svt_{gamma/rho}(L + D)         (numpy SVD: a library primitive)
  line 11 (z_t, w_{t+1}) = prox^mu_{kappa/rho V}(s_t - b_t, s_{t+1} - c_{t+1}):
          inner_iters warm-started iterations of Algorithm 1 (oracle.iterate) on the
          T-1 independent pairs, prox weight rho/kappa in the L2 convention
  line 12 A = A + X - S - L                                                      (L27)
  line 13 D = D + L - T
  line 14 b_t = b_t + z_t - s_t ;  line 15 c_{t+1} = c_{t+1} + w_{t+1} - s_{t+1}
Readings:
  L25 line 7 prints the two-sided shrink^{l1}; the argmin it solves has
      s >= 0, whose exact minimiser is the one-sided max(. - lambda/(rho sigma), 0).
  L26 line 9 prints (Phi^T y + k); the displayed minimiser of
      ||y - Phi x||^2 + rho ||x - k||^2 is (Phi^T Phi + rho I)^{-1}(Phi^T y + rho k).
  L27 line 12 prints A + X - S + L; the augmented Lagrangian has the
      term ||X - S - L + A||^2, whose scaled dual ascent is A + X - S - L.
  L28 residuals (P:905 cites Boyd S3.3): primal ||[X-S-L; L-T; z-s; w-s]||_F,
      dual rho ||[X - X_prev; T - T_prev; z - z_prev; w - w_prev]||_F.
``literal`` takes any of {"L25", "L26", "L27"} to apply the PRINTED line instead of
the reading -- used only by the pin tests to show that each reading is needed.

Layouts: frames [T][ny][nx]; per-pair arrays [T-1][ny][nx] with z_t, b_t (left
frame of pair t) and w_{t+1}, c_{t+1} (right frame) stored at index t.

Pins: tests/test_rpca_pins.py (R1..R7).
"""
from __future__ import annotations

import math

import numpy as np

from . import iterate, State

STATE = ("S", "L", "X", "Tm", "A", "D", "Z", "W", "Bd", "Cd", "mx", "my", "r", "ain")


def svt(M, sigma):
    """shrink^*_sigma(M) = U shrink^{l1}_sigma(Sigma) V^T for a 2-D matrix."""
    U, sv, Vt = np.linalg.svd(np.asarray(M, dtype=np.float64), full_matrices=False)
    return (U * np.maximum(sv - sigma, 0.0)) @ Vt


def nuclear_norm(M):
    return float(np.linalg.svd(np.asarray(M, dtype=np.float64), compute_uv=False).sum())


def zero_state(T, ny, nx):
    """Algorithm 3 line 2: every variable 0; inner prox states 0."""
    st = {k: np.zeros((T, ny, nx)) for k in ("S", "L", "X", "Tm", "A", "D")}
    for k in ("Z", "W", "Bd", "Cd", "mx", "my", "r", "ain"):
        st[k] = np.zeros((T - 1, ny, nx))
    return st


def objective(Y, S, L, lam, gamma, kappa, mu, phi=None, v_pairs=None):
    """eq:RPCA_UOTDF.  v_pairs: per-pair V_mu(s_t, s_{t+1}) values if known
    (else the OT term is omitted and only the other terms are returned)."""
    phi = np.ones_like(Y) if phi is None else phi
    T = Y.shape[0]
    data = 0.5 * float(((Y - phi * (S + L)) ** 2).sum())
    nuc = nuclear_norm(L.reshape(T, -1).T)
    ot = 0.0 if v_pairs is None else kappa * float(np.sum(v_pairs))
    return data + lam * float(np.abs(S).sum()) + gamma * nuc + ot


def admm(Y, lam, gamma, kappa, mu, rho, tau1, tau2, n_outer, inner_iters=1, phi=None, state=None,
         literal=()):
    """Run n_outer iterations of Algorithm 3 on Y [T][ny][nx] (float64 copy).

    Returns (state dict (STATE keys), res [n_outer][2] = primal, dual residuals of L28,
    nuc [n_outer] = ||T||_* after line 10)."""
    Y = np.asarray(Y, dtype=np.float64)
    T, ny, nx = Y.shape
    if T < 2:
        raise ValueError("Algorithm 3 needs T >= 2 frames")
    P = T - 1
    phi = np.ones_like(Y) if phi is None else np.asarray(phi, dtype=np.float64)
    st = {k: np.array(v, dtype=np.float64, copy=True) for k, v in (state or zero_state(T, ny, nx)).items()}
    S, L, X, Tm, A, D = (st[k] for k in ("S", "L", "X", "Tm", "A", "D"))
    Z, W, Bd, Cd = st["Z"], st["W"], st["Bd"], st["Cd"]
    res = np.zeros((n_outer, 2))
    nuc = np.zeros(n_outer)
    wz = np.array([1.0 if t < T - 1 else 0.0 for t in range(T)])       # line 4
    ww = np.array([1.0 if t > 0 else 0.0 for t in range(T)])
    for it in range(n_outer):
        # line 5: k_t (z_t/b_t exist for t < T-1, w_t/c_t for t > 0)
        K = X - L + A
        for t in range(T):
            if wz[t]:
                K[t] += Z[t] + Bd[t]
            if ww[t]:
                K[t] += W[t - 1] + Cd[t - 1]
        sig = 1.0 + wz + ww                                             # line 6
        Snew = np.empty_like(S)
        for t in range(T):                                              # line 7
            q = K[t] / sig[t]
            thr = lam / (rho * sig[t])
            if "L25" in literal:
                Snew[t] = np.sign(q) * np.maximum(np.abs(q) - thr, 0.0)
            else:
                Snew[t] = np.maximum(q - thr, 0.0)
        Lnew = np.maximum(0.5 * (Tm - D + X - Snew + A), 0.0)         # line 8
        if "L26" in literal:                                            # line 9
            Xnew = (phi * Y + Snew + Lnew - A) / (phi * phi + rho)
        else:
            Xnew = (phi * Y + rho * (Snew + Lnew - A)) / (phi * phi + rho)
        Mmat = (Lnew + D).reshape(T, -1).T                              # N x T, columns = frames
        Tnew = svt(Mmat, gamma / rho).T.reshape(T, ny, nx)              # line 10
        nuc[it] = nuclear_norm(Tnew.reshape(T, -1).T)
        # line 11: per-pair prox, centres (s_t - b_t, s_{t+1} - c_{t+1}), warm-started
        centres = np.stack([Snew[:-1] - Bd, Snew[1:] - Cd], axis=1)     # [P][2][ny][nx]
        inner = State(st["mx"], st["my"], st["r"], st["ain"], np.stack([Z, W], axis=1))
        inner, _ = iterate(centres, mu, rho / kappa, tau1, tau2, inner_iters, inner)
        Znew, Wnew = inner.x[:, 0].copy(), inner.x[:, 1].copy()
        st["mx"], st["my"], st["r"], st["ain"] = inner.mx, inner.my, inner.r, inner.a
        if "L27" in literal:                                            # line 12
            Anew = A + Xnew - Snew + Lnew
        else:
            Anew = A + Xnew - Snew - Lnew
        Dnew = D + Lnew - Tnew                                          # line 13
        Bnew = Bd + Znew - Snew[:-1]                                    # line 14
        Cnew = Cd + Wnew - Snew[1:]                                     # line 15
        # L28 residuals
        pr = ((Xnew - Snew - Lnew) ** 2).sum() + ((Lnew - Tnew) ** 2).sum() \
            + ((Znew - Snew[:-1]) ** 2).sum() + ((Wnew - Snew[1:]) ** 2).sum()
        du = ((Xnew - X) ** 2).sum() + ((Tnew - Tm) ** 2).sum() + ((Znew - Z) ** 2).sum() + ((Wnew - W) ** 2).sum()
        res[it] = (math.sqrt(pr), rho * math.sqrt(du))
        S, L, X, Tm, A, D, Z, W, Bd, Cd = Snew, Lnew, Xnew, Tnew, Anew, Dnew, Znew, Wnew, Bnew, Cnew
        if not all(np.isfinite(v).all() for v in (S, L, X, Tm, A, D, Z, W)):
            raise FloatingPointError("non-finite iterate")
    st.update(S=S, L=L, X=X, Tm=Tm, A=A, D=D, Z=Z, W=W, Bd=Bd, Cd=Cd)
    return st, res, nuc


# ----------------------------------------------------------------------------- signed split
SIGNED_STATE = ("Sp", "Sm", "L", "X", "Tm", "A", "D", "Zp", "Wp", "Bp", "Cp", "Zm", "Wm", "Bm", "Cm",
                "mx", "my", "r", "ain")


def zero_state_signed(T, ny, nx):
    """Cold start of the signed split (eq:RPCA_UOTDF_PN): every variable 0; the
    inner prox states cover 2(T-1) pairs (the S+ chain's pairs, then the S- chain's)."""
    st = {k: np.zeros((T, ny, nx)) for k in ("Sp", "Sm", "L", "X", "Tm", "A", "D")}
    for k in ("Zp", "Wp", "Bp", "Cp", "Zm", "Wm", "Bm", "Cm"):
        st[k] = np.zeros((T - 1, ny, nx))
    for k in ("mx", "my", "r", "ain"):
        st[k] = np.zeros((2 * (T - 1), ny, nx))
    return st


def signed_s_update(u, kp, km, m, lam_rho):
    """Exact joint minimiser over s+, s- >= 0 (reading L30) of
        lam_rho (s+ + s-) + 1/2 (u - s+ + s-)^2 + 1/2 (m s+^2 - 2 kp s+) + 1/2 (m s-^2 - 2 km s-),
    the s-block of the split augmented Lagrangian divided by rho (u = x - l + a; kp, km the
    summed z + b / w + c targets of each sign; m = number of those terms, >= 1).  A strictly
    convex quadratic on the quadrant: the minimiser is the best of the face minimisers
    (interior stationary point, the two clipped edge minimisers, the origin)."""
    def F(sp, sm):
        return lam_rho * (sp + sm) + 0.5 * (u - sp + sm) ** 2 + 0.5 * (m * sp * sp - 2 * kp * sp) \
            + 0.5 * (m * sm * sm - 2 * km * sm)
    r1 = u + kp - lam_rho
    r2 = -u + km - lam_rho
    det = (1.0 + m) ** 2 - 1.0
    ip = ((1.0 + m) * r1 + r2) / det                       # interior: [[1+m, -1], [-1, 1+m]] s = r
    im = (r1 + (1.0 + m) * r2) / det
    cands = [(np.maximum(r1 / (1.0 + m), 0.0), np.zeros_like(u)),      # s- = 0 edge
             (np.zeros_like(u), np.maximum(r2 / (1.0 + m), 0.0)),      # s+ = 0 edge
             (np.zeros_like(u), np.zeros_like(u))]
    best_p, best_m = cands[0]
    best = F(best_p, best_m)
    for cp, cm in cands[1:] + [(ip, im)]:
        ok = (cp >= 0) & (cm >= 0)
        val = np.where(ok, F(cp, cm), np.inf)
        take = val < best
        best_p = np.where(take, cp, best_p)
        best_m = np.where(take, cm, best_m)
        best = np.where(take, val, best)
    return best_p, best_m


def admm_signed(Y, lam, gamma, kappa, mu, rho, tau1, tau2, n_outer, inner_iters=1, phi=None, state=None):
    """Signed split of Algorithm 3 for eq:RPCA_UOTDF_PN: S = S+ - S-, S+/- >= 0,
    each with its own l1 weight lambda and its own chain of UOT terms; L >= 0.  The split
    (not printed; reading L30) extends Algorithm 3's: X = S+ - S- + L, T = L, z+/-_t = s+/-_t,
    w+/-_{t+1} = s+/-_{t+1}; per iteration, in Algorithm 3's order:
      s+, s- jointly (signed_s_update) with u = x - l + a and the z/w targets of each sign;
      L = Pi_+((T - D + X - (S+ - S-) + A)/2);  x = (phi y + rho(s+ - s- + l - a))/(phi^2 + rho);
      T = svt_{gamma/rho}(L + D);  the 2(T-1) pair proxes of the S+ and S- chains;
      A += X - (S+ - S-) - L;  D += L - T;  b/c of each sign += z/w - s.
    Returns (state dict, res [n_outer][2] (L28 with both signs' terms), nuc)."""
    Y = np.asarray(Y, dtype=np.float64)
    T, ny, nx = Y.shape
    if T < 2:
        raise ValueError("Algorithm 3 needs T >= 2 frames")
    P = T - 1
    phi = np.ones_like(Y) if phi is None else np.asarray(phi, dtype=np.float64)
    st = {k: np.array(v, dtype=np.float64, copy=True) for k, v in (state or zero_state_signed(T, ny, nx)).items()}
    res = np.zeros((n_outer, 2))
    nuc = np.zeros(n_outer)
    wz = np.array([1.0 if t < T - 1 else 0.0 for t in range(T)])
    ww = np.array([1.0 if t > 0 else 0.0 for t in range(T)])
    m = (wz + ww)[:, None, None]
    for it in range(n_outer):
        Sp, Sm, L, X, Tm, A, D = (st[k] for k in ("Sp", "Sm", "L", "X", "Tm", "A", "D"))
        u = X - L + A
        kp, km = np.zeros_like(Y), np.zeros_like(Y)
        for t in range(T):
            if wz[t]:
                kp[t] += st["Zp"][t] + st["Bp"][t]
                km[t] += st["Zm"][t] + st["Bm"][t]
            if ww[t]:
                kp[t] += st["Wp"][t - 1] + st["Cp"][t - 1]
                km[t] += st["Wm"][t - 1] + st["Cm"][t - 1]
        Spn, Smn = signed_s_update(u, kp, km, m, lam / rho)
        Sn = Spn - Smn
        Ln = np.maximum(0.5 * (Tm - D + X - Sn + A), 0.0)
        Xn = (phi * Y + rho * (Sn + Ln - A)) / (phi * phi + rho)
        Tn = svt((Ln + D).reshape(T, -1).T, gamma / rho).T.reshape(T, ny, nx)
        nuc[it] = nuclear_norm(Tn.reshape(T, -1).T)
        centres = np.concatenate([np.stack([Spn[:-1] - st["Bp"], Spn[1:] - st["Cp"]], axis=1),
                                  np.stack([Smn[:-1] - st["Bm"], Smn[1:] - st["Cm"]], axis=1)])   # [2P][2]
        zw = np.concatenate([np.stack([st["Zp"], st["Wp"]], axis=1), np.stack([st["Zm"], st["Wm"]], axis=1)])
        inner = State(st["mx"], st["my"], st["r"], st["ain"], zw)
        inner, _ = iterate(centres, mu, rho / kappa, tau1, tau2, inner_iters, inner)
        Zp, Wp, Zm, Wm = inner.x[:P, 0], inner.x[:P, 1], inner.x[P:, 0], inner.x[P:, 1]
        pr = ((Xn - Sn - Ln) ** 2).sum() + ((Ln - Tn) ** 2).sum()
        du = ((Xn - X) ** 2).sum() + ((Tn - Tm) ** 2).sum()
        for (z, w, s_new, zo, wo) in ((Zp, Wp, Spn, st["Zp"], st["Wp"]), (Zm, Wm, Smn, st["Zm"], st["Wm"])):
            pr += ((z - s_new[:-1]) ** 2).sum() + ((w - s_new[1:]) ** 2).sum()
            du += ((z - zo) ** 2).sum() + ((w - wo) ** 2).sum()
        res[it] = (math.sqrt(pr), rho * math.sqrt(du))
        st.update(Bp=st["Bp"] + Zp - Spn[:-1], Cp=st["Cp"] + Wp - Spn[1:],
                  Bm=st["Bm"] + Zm - Smn[:-1], Cm=st["Cm"] + Wm - Smn[1:])
        st.update(Sp=Spn, Sm=Smn, L=Ln, X=Xn, Tm=Tn, A=A + Xn - Sn - Ln, D=D + Ln - Tn,
                  Zp=Zp.copy(), Wp=Wp.copy(), Zm=Zm.copy(), Wm=Wm.copy(),
                  mx=inner.mx, my=inner.my, r=inner.r, ain=inner.a)
        if not all(np.isfinite(st[k]).all() for k in ("Sp", "Sm", "L", "X", "A", "D")):
            raise FloatingPointError("non-finite iterate")
    return st, res, nuc
