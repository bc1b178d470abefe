"""Independent pin of the plastic return mappings (snow, sand): golden vectors from numpy's SVD.

    python tests/golden/make_plastic_golden.py        # writes tests/golden/plastic.npz

The reference package has no plastic model, so there is nothing of the reference
to run.  What pins `orc_snow_project` / `orc_sand_project` / `orc_sand_tau` (oracle/mpm_oracle.c)
instead is a restatement of the PUBLISHED closed forms on top of LAPACK's SVD (`numpy.linalg.svd`)
-- the way the reference's own tests pin its fixed-corotated stress and its Jacobi SVD against
scipy (tests/test_domain.py:111-124, 175-186 of the reference).  Nothing here shares code with the
oracle: different SVD (LAPACK gesdd vs Jacobi on F^T F), different language, written from the
papers:

  snow   Stomakhin, Schroeder, Chai, Teran, Selle 2013, "A material point method for snow
         simulation", section 7: F = U S V^T (rotation variant), S' = clamp(S, 1-theta_c, 1+theta_s),
         F_E = U S' V^T, F_P' = V S'^-1 U^T F F_P  =>  J_P' = J_P det(S) / det(S');
         hardening mu(F_P) = mu0 exp(xi (1 - J_P)), same for lambda; fixed-corotated stress
         tau = 2 mu (F_E - R_E) F_E^T + lam (J_E - 1) J_E I  (their eq. 1-2, Kirchhoff form).
         J_P is kept in [0.1, 10] (this repository's guard against runaway hardening).
  sand   Klar, Gast, Pradhana, Fu, Schroeder, Jiang, Teran 2016, "Drucker-Prager elastoplasticity
         for sand animation", section 6 + Algorithm "Project": e = log S, e_hat = e - tr(e)/3,
         tr(e) > 0 -> S' = I (tip); dg = |e_hat| + (3 lam + 2 mu)/(2 mu) tr(e) alpha,
         dg <= 0 -> S' = S; else S' = exp(e - dg e_hat/|e_hat|).  (The paper's listing also sends
         e_hat = 0 to the tip; with tr <= 0 that state is inside the cone, dg <= 0, and it is left
         unchanged here so that the map is continuous -- see oracle/mpm_oracle.c.)  alpha = sqrt(2/3) 2 sin(phi) /
         (3 - sin(phi)).  Energy: St. Venant-Kirchhoff with Hencky strain, Kirchhoff stress
         tau = U (2 mu e + lam tr(e) I) U^T.  Singular values are taken in magnitude and floored
         at 1e-6 before the logarithm (this repository's guard).  The volume-correction scalar
         accumulates tr(e) of the tip projections.

Inputs: a few hundred random deformation gradients (perturbations 1e-3 .. 0.5 of the identity,
random rotations applied left and right) plus adversarial cases: inverted (det < 0), nearly
singular, exactly ON the yield limits (a singular value equal to 1 - theta_c / 1 + theta_s; Hencky
strains with dg = 0 up to rounding), pure rotations (S = I, repeated singular values), isotropic
stretch / compression (e_hat = 0).
"""
import os

import numpy as np

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "plastic.npz")

THETA_C, THETA_S, XI = 2.5e-2, 7.5e-3, 10.0
MU, LAM = 1.0e5 / 2.6, 1.0e5 * 0.3 / (1.3 * 0.4)     # Lame parameters of E = 1e5, nu = 0.3
PHI = 30.0
ALPHA = np.sqrt(2.0 / 3.0) * 2.0 * np.sin(np.radians(PHI)) / (3.0 - np.sin(np.radians(PHI)))


def rot_svd(F):
    """LAPACK SVD turned into the rotation variant: det U = det V = +1, the sign of det F carried
    by the LAST (smallest) singular value."""
    U, s, Vt = np.linalg.svd(F)
    s = s.copy()
    if np.linalg.det(U) < 0.0:
        U = U.copy(); U[:, 2] *= -1.0; s[2] *= -1.0
    if np.linalg.det(Vt) < 0.0:
        Vt = Vt.copy(); Vt[2, :] *= -1.0; s[2] *= -1.0
    return U, s, Vt


def snow_project(F, Jp):
    U, s, Vt = rot_svd(F)
    sc = np.clip(s, 1.0 - THETA_C, 1.0 + THETA_S)
    FE = (U * sc) @ Vt
    j = Jp * np.prod(s) / np.prod(sc)
    j = 0.1 if not (j > 0.1) else min(j, 10.0)
    return FE, j


def corotated_tau(F, mu, lam):
    """tau = 2 mu (F - R) F^T + lam (J - 1) J I with R = U V^T from the rotation-variant SVD."""
    U, s, Vt = rot_svd(F)
    R = U @ Vt
    J = np.prod(s)
    return 2.0 * mu * (F - R) @ F.T + lam * (J - 1.0) * J * np.eye(3)


def snow_tau(FE, Jp):
    h = np.exp(XI * (1.0 - Jp))
    return corotated_tau(FE, MU * h, LAM * h)


def sand_project(F, vc):
    U, s, Vt = rot_svd(F)
    a = np.maximum(np.abs(s), 1e-6)
    e = np.log(a)
    tr = e.sum()
    dev = e - tr / 3.0
    dn = np.sqrt((dev * dev).sum())
    if tr > 0.0:
        sc = np.ones(3)
        vc = vc + tr
    else:
        dg = dn + (3.0 * LAM + 2.0 * MU) / (2.0 * MU) * tr * ALPHA
        sc = a if dg <= 0.0 else np.exp(e - dg * dev / dn)
    return (U * sc) @ Vt, vc


def sand_tau(F):
    U, s, _ = rot_svd(F)
    e = np.log(np.maximum(np.abs(s), 1e-6))
    d = 2.0 * MU * e + LAM * e.sum()
    return (U * d) @ U.T


def random_rotation(rng):
    q, r = np.linalg.qr(rng.normal(size=(3, 3)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0.0:
        q[:, 0] *= -1.0
    return q


def from_singular_values(rng, s):
    return (random_rotation(rng) * np.asarray(s, dtype=np.float64)) @ random_rotation(rng).T


def cases():
    rng = np.random.default_rng(20211100699)
    F, tag = [], []
    for amp in (1e-3, 1e-2, 3e-2, 0.1, 0.3, 0.5):          # 300 random states
        for _ in range(50):
            G = np.eye(3) + amp * rng.normal(size=(3, 3))
            F.append(random_rotation(rng) @ G)
            tag.append(0)
    for _ in range(20):                                     # inverted
        s = 1.0 + 0.2 * rng.normal(size=3)
        s = np.sort(np.abs(s))[::-1]
        s[2] = -s[2]
        F.append(from_singular_values(rng, s)); tag.append(1)
    for eps in (1e-3, 1e-5, 1e-7, 1e-9, 0.0):               # nearly singular / singular
        for _ in range(4):
            F.append(from_singular_values(rng, [1.0 + 0.1 * rng.random(), 0.9, eps])); tag.append(2)
    for _ in range(10):                                     # ON the snow yield limits
        F.append(from_singular_values(rng, [1.0 + THETA_S, 1.0, 1.0 - THETA_C])); tag.append(3)
        F.append(from_singular_values(rng, [1.0 + THETA_S, 1.0 + THETA_S, 1.0 + THETA_S])); tag.append(3)
    for _ in range(20):                                     # on the Drucker-Prager cone: dg = 0
        dev = rng.normal(size=3)
        dev -= dev.mean()
        dev *= 0.05 / np.linalg.norm(dev)
        tr = -0.05 / ((3.0 * LAM + 2.0 * MU) / (2.0 * MU) * ALPHA)
        F.append(from_singular_values(rng, np.exp(dev + tr / 3.0))); tag.append(4)
    for _ in range(10):                                     # pure rotations, isotropic states
        F.append(random_rotation(rng)); tag.append(5)
        F.append(from_singular_values(rng, [0.97] * 3)); tag.append(5)
        F.append(from_singular_values(rng, [1.02] * 3)); tag.append(5)
    F = np.asarray(F)
    Jp = np.where(np.arange(len(F)) % 3 == 0, 1.0, 0.6 + 0.8 * rng.random(len(F)))
    vc = 0.01 * rng.normal(size=len(F))
    return F, np.asarray(tag), Jp, vc


def main():
    F, tag, Jp, vc = cases()
    n = len(F)
    snow_FE, snow_Jp, snow_t = np.empty((n, 3, 3)), np.empty(n), np.empty((n, 3, 3))
    sand_FE, sand_vc, sand_t = np.empty((n, 3, 3)), np.empty(n), np.empty((n, 3, 3))
    for k in range(n):
        snow_FE[k], snow_Jp[k] = snow_project(F[k], Jp[k])
        snow_t[k] = snow_tau(snow_FE[k], snow_Jp[k])
        sand_FE[k], sand_vc[k] = sand_project(F[k], vc[k])
        sand_t[k] = sand_tau(sand_FE[k])
    np.savez_compressed(OUT, F=F, tag=tag, Jp=Jp, vc=vc, theta_c=THETA_C, theta_s=THETA_S, xi=XI,
                        mu=MU, lam=LAM, alpha=ALPHA, snow_FE=snow_FE, snow_Jp=snow_Jp, snow_tau=snow_t,
                        sand_FE=sand_FE, sand_vc=sand_vc, sand_tau=sand_t)
    print("wrote", OUT, n, "states;", {int(t): int((tag == t).sum()) for t in np.unique(tag)})


if __name__ == "__main__":
    main()
