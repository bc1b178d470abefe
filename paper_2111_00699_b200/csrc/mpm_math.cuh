// Constitutive math of the transfer kernels in fp32 (sm_100a).
// Restates, in single precision, the scalar routines of the reference:
//   _svd3_scalars   domain.py:195-379   (Jacobi on F^T F, descending order, det(V)=+1,
//                                        Gram-Schmidt U, sign carried by the last value)
//   _corotated_tau  domain.py:383-441   tau = 2 mu (F - R) F^T + lam (J-1) J I
//   _fluid_tau      pipeline.py:151-156 tau = -kappa (J^-gamma - 1)
// The convergence thresholds are the fp32 counterparts of the reference's fp64 ones.
#pragma once

#include "mpm_common.cuh"

namespace mpm {

__device__ __forceinline__ float det3(const float *f)
{
    return f[0] * (f[4] * f[8] - f[5] * f[7]) - f[1] * (f[3] * f[8] - f[5] * f[6]) +
           f[2] * (f[3] * f[7] - f[4] * f[6]);
}

// One Jacobi rotation zeroing a_pq (domain.py:232-303).  P, Q: columns of V it mixes
// (compile-time so that V stays in registers).
template <int P, int Q>
__device__ __forceinline__ void jacobi_rotate(float &app, float &aqq, float &apq, float &arp,
                                              float &arq, float *v)
{
    const float a_pq = apq;
    // rotation angle from approximate (2 ulp) reciprocal / square root: c^2 + s^2 = 1 holds to
    // rounding whatever t is, so V stays orthogonal; accuracy of t only affects convergence
    const float theta = __fdividef(0.5f * (aqq - app), a_pq);
    const float r = __fsqrt_rn(1.0f + theta * theta);
    const float t = theta >= 0.0f ? __fdividef(1.0f, theta + r) : -__fdividef(1.0f, r - theta);
    const float c = rsqrtf(1.0f + t * t);
    const float s = t * c;
    const float pp = app, qq = aqq;
    app = c * c * pp - 2.0f * s * c * a_pq + s * s * qq;
    aqq = s * s * pp + 2.0f * s * c * a_pq + c * c * qq;
    apq = 0.0f;
    const float rp = arp, rq = arq;
    arp = c * rp - s * rq;
    arq = s * rp + c * rq;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float tmp = v[3 * k + P];
        v[3 * k + P] = c * tmp - s * v[3 * k + Q];
        v[3 * k + Q] = s * tmp + c * v[3 * k + Q];
    }
}

// f = u diag(s) v^T, row-major 3x3.  s[0] >= s[1] >= |s[2]|, det(u) = det(v) = +1.
__device__ __forceinline__ void svd3(const float *f, float *u, float *s, float *v)
{
    float a00 = f[0] * f[0] + f[3] * f[3] + f[6] * f[6];
    float a01 = f[0] * f[1] + f[3] * f[4] + f[6] * f[7];
    float a02 = f[0] * f[2] + f[3] * f[5] + f[6] * f[8];
    float a11 = f[1] * f[1] + f[4] * f[4] + f[7] * f[7];
    float a12 = f[1] * f[2] + f[4] * f[5] + f[7] * f[8];
    float a22 = f[2] * f[2] + f[5] * f[5] + f[8] * f[8];
    v[0] = 1.f; v[1] = 0.f; v[2] = 0.f; v[3] = 0.f; v[4] = 1.f; v[5] = 0.f; v[6] = 0.f; v[7] = 0.f; v[8] = 1.f;
    const float tol = 3e-8f * (fabsf(a00) + fabsf(a11) + fabsf(a22)) + 1e-37f;
    for (int it = 0; it < 15; ++it) {
        const float m01 = fabsf(a01), m02 = fabsf(a02), m12 = fabsf(a12);
        float big = m01;
        int pair = 0;
        if (m02 > big) { big = m02; pair = 1; }
        if (m12 > big) { big = m12; pair = 2; }
        if (big <= tol) break;
        if (pair == 0) jacobi_rotate<0, 1>(a00, a11, a01, a02, a12, v);
        else if (pair == 1) jacobi_rotate<0, 2>(a00, a22, a02, a01, a12, v);
        else jacobi_rotate<1, 2>(a11, a22, a12, a01, a02, v);
    }
    float w0 = a00, w1 = a11, w2 = a22, tmp;
#define MPM_SWAPCOL(p, q)                                                                   \
    {                                                                                       \
        tmp = v[p]; v[p] = v[q]; v[q] = tmp;                                                \
        tmp = v[3 + p]; v[3 + p] = v[3 + q]; v[3 + q] = tmp;                                \
        tmp = v[6 + p]; v[6 + p] = v[6 + q]; v[6 + q] = tmp;                                \
    }
    if (w0 < w1) { tmp = w0; w0 = w1; w1 = tmp; MPM_SWAPCOL(0, 1) }
    if (w1 < w2) { tmp = w1; w1 = w2; w2 = tmp; MPM_SWAPCOL(1, 2) }
    if (w0 < w1) { tmp = w0; w0 = w1; w1 = tmp; MPM_SWAPCOL(0, 1) }
#undef MPM_SWAPCOL
    if (det3(v) < 0.0f) { v[2] = -v[2]; v[5] = -v[5]; v[8] = -v[8]; }
    const float s0 = w0 > 0.0f ? sqrtf(w0) : 0.0f;
    const float s1 = w1 > 0.0f ? sqrtf(w1) : 0.0f;
    float s2 = w2 > 0.0f ? sqrtf(w2) : 0.0f;
    float u00 = f[0] * v[0] + f[1] * v[3] + f[2] * v[6];
    float u10 = f[3] * v[0] + f[4] * v[3] + f[5] * v[6];
    float u20 = f[6] * v[0] + f[7] * v[3] + f[8] * v[6];
    float n = sqrtf(u00 * u00 + u10 * u10 + u20 * u20);
    if (n < 1e-30f) { u00 = 1.0f; u10 = 0.0f; u20 = 0.0f; }
    else { const float inv = 1.0f / n; u00 *= inv; u10 *= inv; u20 *= inv; }
    float u01 = f[0] * v[1] + f[1] * v[4] + f[2] * v[7];
    float u11 = f[3] * v[1] + f[4] * v[4] + f[5] * v[7];
    float u21 = f[6] * v[1] + f[7] * v[4] + f[8] * v[7];
    const float d = u01 * u00 + u11 * u10 + u21 * u20;
    u01 -= d * u00; u11 -= d * u10; u21 -= d * u20;
    n = sqrtf(u01 * u01 + u11 * u11 + u21 * u21);
    if (n < 1e-30f) {
        u01 = -u10; u11 = u00; u21 = 0.0f;
        const float n2 = sqrtf(u01 * u01 + u11 * u11);
        if (n2 < 1e-30f) { u01 = 0.0f; u11 = 1.0f; u21 = 0.0f; }
        else { u01 /= n2; u11 /= n2; }
    } else { const float inv = 1.0f / n; u01 *= inv; u11 *= inv; u21 *= inv; }
    const float u02 = u10 * u21 - u20 * u11;
    const float u12 = u20 * u01 - u00 * u21;
    const float u22 = u00 * u11 - u10 * u01;
    const float fv0 = f[0] * v[2] + f[1] * v[5] + f[2] * v[8];
    const float fv1 = f[3] * v[2] + f[4] * v[5] + f[5] * v[8];
    const float fv2 = f[6] * v[2] + f[7] * v[5] + f[8] * v[8];
    if (fv0 * u02 + fv1 * u12 + fv2 * u22 < 0.0f) s2 = -s2;
    u[0] = u00; u[1] = u01; u[2] = u02; u[3] = u10; u[4] = u11; u[5] = u12;
    u[6] = u20; u[7] = u21; u[8] = u22;
    s[0] = s0; s[1] = s1; s[2] = s2;
}

// Rotation factor R of the polar decomposition F = R S by Newton's iteration
// R <- (R + R^-T) / 2 (Higham 1986), R^-T = cof(R) / det(R).  Quadratic convergence; after the
// first update every singular value is >= 1, so det(R) - 1 bounds the distance to
// orthogonality and one more update after det - 1 < 1e-3 reaches fp32 resolution.
// Returns false when F is too close to singular / inverted for the iteration (the caller
// then takes the reference's SVD route, which also handles reflections and the clamp).
__device__ __forceinline__ bool polar_rotation(const float *f, float J, float *r)
{
    if (!(J > 0.02f)) return false;
#pragma unroll
    for (int k = 0; k < 9; ++k) r[k] = f[k];
    float det = J;
    for (int it = 0; it < 14; ++it) {
        const float c00 = r[4] * r[8] - r[5] * r[7], c01 = r[5] * r[6] - r[3] * r[8], c02 = r[3] * r[7] - r[4] * r[6];
        const float c10 = r[2] * r[7] - r[1] * r[8], c11 = r[0] * r[8] - r[2] * r[6], c12 = r[1] * r[6] - r[0] * r[7];
        const float c20 = r[1] * r[5] - r[2] * r[4], c21 = r[2] * r[3] - r[0] * r[5], c22 = r[0] * r[4] - r[1] * r[3];
        if (it > 0) det = r[0] * c00 + r[1] * c01 + r[2] * c02;
        const bool last = it > 0 && det - 1.0f < 1e-3f;
        const float h = __fdividef(0.5f, det);
        r[0] = 0.5f * r[0] + h * c00; r[1] = 0.5f * r[1] + h * c01; r[2] = 0.5f * r[2] + h * c02;
        r[3] = 0.5f * r[3] + h * c10; r[4] = 0.5f * r[4] + h * c11; r[5] = 0.5f * r[5] + h * c12;
        r[6] = 0.5f * r[6] + h * c20; r[7] = 0.5f * r[7] + h * c21; r[8] = 0.5f * r[8] + h * c22;
        if (last) return true;
    }
    return false;
}

// Fixed-corotated Kirchhoff stress (domain.py:383-441): tau = 2 mu (F - R) F^T + lam (J-1) J I.
// Regular states use the Newton polar factor; near-singular or inverted F takes the
// reference's route (Jacobi SVD, reflection handling, singular values floored at 1e-4 when
// J <= 1e-10).  Returns 1 when the floor was applied, as the reference's clamp flag.
// the rare route is kept out of line so that its registers do not weigh on the hot path
__device__ __noinline__ int corotated_parts_svd(const float *f, float *w, float *dm, float *Jout)
{
    float J = *Jout;
    int clamped = 0;
    {
        float u[9], s[3], v[9];
        svd3(f, u, s, v);
        if (J <= 1e-10f) {
#pragma unroll
            for (int k = 0; k < 3; ++k) if (s[k] < 1e-4f) s[k] = 1e-4f;
            J = s[0] * s[1] * s[2];
            clamped = 1;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b)
                    w[3 * a + b] = s[0] * u[3 * a] * v[3 * b] + s[1] * u[3 * a + 1] * v[3 * b + 1] +
                                   s[2] * u[3 * a + 2] * v[3 * b + 2];
        } else {
#pragma unroll
            for (int k = 0; k < 9; ++k) w[k] = f[k];   // U S V^T == F: skip the lossy reconstruction
        }
#pragma unroll
        for (int a = 0; a < 3; ++a)
#pragma unroll
            for (int b = 0; b < 3; ++b)
                dm[3 * a + b] = w[3 * a + b] - (u[3 * a] * v[3 * b] + u[3 * a + 1] * v[3 * b + 1] +
                                                u[3 * a + 2] * v[3 * b + 2]);
    }
    *Jout = J;
    return clamped;
}

__device__ __forceinline__ int corotated_tau(const float *f, float mu, float lam, float *t)
{
    float J = det3(f);
    int clamped = 0;
    float w[9], dm[9];
    if (polar_rotation(f, J, dm)) {
#pragma unroll
        for (int k = 0; k < 9; ++k) { w[k] = f[k]; dm[k] = f[k] - dm[k]; }
    } else {
        // The out-of-line route takes addresses: it works on private copies so that f, w, dm and J
        // of the regular route stay in registers (arrays whose address escapes to a call live on
        // the stack for the whole kernel, ~20 local stores per warp on the hot path before).
        float ft[9], wt[9], dt[9], Jt = J;
#pragma unroll
        for (int k = 0; k < 9; ++k) ft[k] = f[k];
        clamped = corotated_parts_svd(ft, wt, dt, &Jt);
#pragma unroll
        for (int k = 0; k < 9; ++k) { w[k] = wt[k]; dm[k] = dt[k]; }
        J = Jt;
    }
    const float two_mu = 2.0f * mu;
    const float diag = lam * (J - 1.0f) * J;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b) {
            const float acc = two_mu * (dm[3 * a] * w[3 * b] + dm[3 * a + 1] * w[3 * b + 1] +
                                        dm[3 * a + 2] * w[3 * b + 2]);
            t[3 * a + b] = (a == b) ? acc + diag : acc;
        }
    return clamped;
}

// ---- plastic models (not in the reference; float64 definition in oracle/mpm_oracle.c) -------
// Both return the Kirchhoff stress of the projected elastic state from its SVD:
//   tau = U diag(d) U^T.
struct PlasticParams {
    float mu, lam, theta_c, theta_s, hardening, sand_alpha;
};

__device__ __forceinline__ void tau_from_principal(const float *u, const float *d, float *t)
{
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            t[3 * a + b] = d[0] * u[3 * a] * u[3 * b] + d[1] * u[3 * a + 1] * u[3 * b + 1] +
                           d[2] * u[3 * a + 2] * u[3 * b + 2];
}

__device__ __forceinline__ void rebuild_from_svd(const float *u, const float *sc, const float *v, float *f)
{
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            f[3 * a + b] = sc[0] * u[3 * a] * v[3 * b] + sc[1] * u[3 * a + 1] * v[3 * b + 1] +
                           sc[2] * u[3 * a + 2] * v[3 * b + 2];
}

// snow: fixed-corotated on F_E = U S' V^T with hardened moduli:
//   (F_E - R) F_E^T = U (S' - I) S' U^T  =>  d_k = 2 mu_h (s_k - 1) s_k + lam_h (J - 1) J
__device__ __forceinline__ void snow_principal(const float *sc, float jp, const PlasticParams &p, float *d)
{
    const float h = expf(p.hardening * (1.0f - jp));
    const float J = sc[0] * sc[1] * sc[2];
    const float diag = p.lam * h * (J - 1.0f) * J;
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] = 2.0f * p.mu * h * (sc[k] - 1.0f) * sc[k] + diag;
}

// sand: Hencky strain e = log S, d_k = 2 mu e_k + lam tr(e)
__device__ __forceinline__ void sand_principal(const float *e, const PlasticParams &p, float *d)
{
    const float tr = e[0] + e[1] + e[2];
#pragma unroll
    for (int k = 0; k < 3; ++k) d[k] = 2.0f * p.mu * e[k] + p.lam * tr;
}

// Return mapping on the singular values s of the trial elastic deformation: projected values sc,
// plastic scalar update, principal Kirchhoff stresses d of the projected state.  Elementwise in
// s, so neither the order nor (for sand, which takes |s|) the sign convention of the
// decomposition matters.  MAT: 2 snow, 3 sand.
template <int MAT>
__device__ __forceinline__ void plastic_return(const float *s, float &plastic, const PlasticParams &p,
                                               float *sc, float *d)
{
    if (MAT == MPM_MAT_SNOW) {
        const float num = s[0] * s[1] * s[2];
        float den = 1.0f;
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            sc[k] = fminf(fmaxf(s[k], 1.0f - p.theta_c), 1.0f + p.theta_s);
            den *= sc[k];
        }
        float j = plastic * num / den;
        j = j > 0.1f ? j : 0.1f;
        plastic = fminf(j, 10.0f);
        snow_principal(sc, plastic, p, d);
    } else {
        float e[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) e[k] = logf(fmaxf(fabsf(s[k]), 1e-6f));
        const float tr = e[0] + e[1] + e[2];
        const float d0 = e[0] - tr * (1.0f / 3.0f), d1 = e[1] - tr * (1.0f / 3.0f), d2 = e[2] - tr * (1.0f / 3.0f);
        const float dn = sqrtf(d0 * d0 + d1 * d1 + d2 * d2);
        if (tr > 0.0f) {   // tip of the cone; dg > 0 below implies dn > 0 (see orc_sand_project)
            e[0] = e[1] = e[2] = 0.0f;
            plastic += tr;
        } else {
            const float dg = dn + (3.0f * p.lam + 2.0f * p.mu) / (2.0f * p.mu) * tr * p.sand_alpha;
            if (dg > 0.0f) {
                const float k = dg / dn;
                e[0] -= k * d0; e[1] -= k * d1; e[2] -= k * d2;
            }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) sc[k] = expf(e[k]);
        sand_principal(e, p, d);
    }
}

// General route: Jacobi SVD of F itself (reflections, near-singular states).  Out of line: only
// states the Newton polar iteration refuses (J <= 0.02) come here.
template <int MAT>
__device__ __noinline__ void plastic_project_svd(float *f, float *plastic, PlasticParams p, float *tau)
{
    float u[9], s[3], v[9], sc[3], d[3];
    svd3(f, u, s, v);
    plastic_return<MAT>(s, *plastic, p, sc, d);
    rebuild_from_svd(u, sc, v, f);
    tau_from_principal(u, d, tau);
}

// One rotation of the cyclic Jacobi eigen-solver of a symmetric 3x3 matrix (Rutishauser's update:
// a_pp -= t a_pq, a_qq += t a_pq).  No pivot search and no branch: every lane of the warp walks
// the same three rotations per sweep; an already negligible a_pq gets the identity (t = 0, which
// also absorbs the 0/0 of a_pp == a_qq, a_pq == 0).
template <int P, int Q>
__device__ __forceinline__ void sym_rotate(float &app, float &aqq, float &apq, float &arp, float &arq,
                                           float *v, float eps)
{
    const float theta = __fdividef(aqq - app, 2.0f * apq);
    float t = copysignf(__fdividef(1.0f, fabsf(theta) + sqrtf(fmaf(theta, theta, 1.0f))), theta);
    t = fabsf(apq) > eps ? t : 0.0f;
    const float c = rsqrtf(fmaf(t, t, 1.0f)), s = t * c;
    app = fmaf(-t, apq, app);
    aqq = fmaf(t, apq, aqq);
    apq = t != 0.0f ? 0.0f : apq;
    const float rp = arp, rq = arq;
    arp = c * rp - s * rq;
    arq = s * rp + c * rq;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float vp = v[3 * k + P], vq = v[3 * k + Q];
        v[3 * k + P] = c * vp - s * vq;
        v[3 * k + Q] = s * vp + c * vq;
    }
}

// S = V diag(lam) V^T for symmetric S (upper triangle given), V orthogonal, eigenvalues unordered.
__device__ __forceinline__ void sym_eig3(float a00, float a11, float a22, float a01, float a02, float a12,
                                         float *lam, float *v)
{
    v[0] = 1.f; v[1] = 0.f; v[2] = 0.f; v[3] = 0.f; v[4] = 1.f; v[5] = 0.f; v[6] = 0.f; v[7] = 0.f; v[8] = 1.f;
    const float scale = fabsf(a00) + fabsf(a11) + fabsf(a22);
    const float tol = 2e-8f * scale + 1e-37f, eps = 1e-9f * scale + 1e-38f;
#pragma unroll 1
    for (int sweep = 0; sweep < 6; ++sweep) {
        if (fmaxf(fmaxf(fabsf(a01), fabsf(a02)), fabsf(a12)) <= tol) break;
        sym_rotate<0, 1>(a00, a11, a01, a02, a12, v, eps);
        sym_rotate<0, 2>(a00, a22, a02, a01, a12, v, eps);
        sym_rotate<1, 2>(a11, a22, a12, a01, a02, v, eps);
    }
    lam[0] = a00; lam[1] = a11; lam[2] = a22;
}

// Return mapping of the trial elastic deformation (in place), plastic scalar update, and the
// stress of the projected state.  With the polar factor F = R S at hand (Newton iteration, also
// what the fixed-corotated stress uses) the SVD is the eigen-decomposition of the symmetric
// stretch: S = R^T F = V diag(s) V^T, U = R V.  Working on S instead of F^T F does not square the
// condition number, and S is positive definite, so there is no reflection / sign handling.
template <int MAT>
__device__ __forceinline__ void plastic_project(float *f, float &plastic, const PlasticParams &p, float *tau)
{
    float r[9];
    const float J = det3(f);
    if (!polar_rotation(f, J, r)) {
        // private copies for the out-of-line route (see corotated_tau): f, tau, the plastic scalar
        // and the parameters of the regular route never have their address taken
        float ft[9], tt[9], pl = plastic;
#pragma unroll
        for (int k = 0; k < 9; ++k) ft[k] = f[k];
        plastic_project_svd<MAT>(ft, &pl, p, tt);
#pragma unroll
        for (int k = 0; k < 9; ++k) { f[k] = ft[k]; tau[k] = tt[k]; }
        plastic = pl;
        return;
    }
    const float s00 = r[0] * f[0] + r[3] * f[3] + r[6] * f[6];
    const float s11 = r[1] * f[1] + r[4] * f[4] + r[7] * f[7];
    const float s22 = r[2] * f[2] + r[5] * f[5] + r[8] * f[8];
    // S is symmetric up to the residual of the polar iteration: average the two triangles
    const float s01 = 0.5f * (r[0] * f[1] + r[3] * f[4] + r[6] * f[7] + r[1] * f[0] + r[4] * f[3] + r[7] * f[6]);
    const float s02 = 0.5f * (r[0] * f[2] + r[3] * f[5] + r[6] * f[8] + r[2] * f[0] + r[5] * f[3] + r[8] * f[6]);
    const float s12 = 0.5f * (r[1] * f[2] + r[4] * f[5] + r[7] * f[8] + r[2] * f[1] + r[5] * f[4] + r[8] * f[7]);
    if (MAT == MPM_MAT_SNOW) {
        // Elastic fast path: when every singular value lies inside the yield interval nothing is
        // clamped and the projection is the identity.  Gershgorin discs of S bound them without
        // an eigen-solve; the stress is then the fixed-corotated form with hardened moduli.
        const float o01 = fabsf(s01), o02 = fabsf(s02), o12 = fabsf(s12);
        const float lo = fminf(fminf(s00 - o01 - o02, s11 - o01 - o12), s22 - o02 - o12);
        const float hi = fmaxf(fmaxf(s00 + o01 + o02, s11 + o01 + o12), s22 + o02 + o12);
        if (lo >= 1.0f - p.theta_c && hi <= 1.0f + p.theta_s) {
            plastic = fminf(plastic > 0.1f ? plastic : 0.1f, 10.0f);
            const float h = expf(p.hardening * (1.0f - plastic));
            const float two_mu = 2.0f * p.mu * h, diag = p.lam * h * (J - 1.0f) * J;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    const float acc = two_mu * ((f[3 * a] - r[3 * a]) * f[3 * b] +
                                                (f[3 * a + 1] - r[3 * a + 1]) * f[3 * b + 1] +
                                                (f[3 * a + 2] - r[3 * a + 2]) * f[3 * b + 2]);
                    tau[3 * a + b] = (a == b) ? acc + diag : acc;
                }
            return;
        }
    }
    float lam[3], v[9], u[9], sc[3], d[3];
    sym_eig3(s00, s11, s22, s01, s02, s12, lam, v);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int b = 0; b < 3; ++b)
            u[3 * a + b] = r[3 * a] * v[b] + r[3 * a + 1] * v[3 + b] + r[3 * a + 2] * v[6 + b];
    plastic_return<MAT>(lam, plastic, p, sc, d);
    rebuild_from_svd(u, sc, v, f);
    tau_from_principal(u, d, tau);
}

// Stress of an already projected state (split P2G): one SVD of the stored F_E.
template <int MAT>
__device__ __forceinline__ void plastic_tau(const float *f, float plastic, const PlasticParams &p, float *tau)
{
    if (MAT == MPM_MAT_SNOW) {
        // The stored F_E is already projected, so its stress is the fixed-corotated form with
        // hardened moduli, tau = 2 mu_h (F - R) F^T + lam_h (J - 1) J I (= U (2 mu_h (S - I) S + ...) U^T):
        // the polar factor is all it takes.  States the Newton iteration refuses go through the SVD.
        float r[9];
        const float J = det3(f);
        if (polar_rotation(f, J, r)) {
            const float h = expf(p.hardening * (1.0f - plastic));
            const float two_mu = 2.0f * p.mu * h, diag = p.lam * h * (J - 1.0f) * J;
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    const float acc = two_mu * ((f[3 * a] - r[3 * a]) * f[3 * b] +
                                                (f[3 * a + 1] - r[3 * a + 1]) * f[3 * b + 1] +
                                                (f[3 * a + 2] - r[3 * a + 2]) * f[3 * b + 2]);
                    tau[3 * a + b] = (a == b) ? acc + diag : acc;
                }
            return;
        }
    }
    float u[9], s[3], v[9], d[3];
    svd3(f, u, s, v);
    if (MAT == MPM_MAT_SNOW) {
        snow_principal(s, plastic, p, d);
    } else {
        float e[3];
#pragma unroll
        for (int k = 0; k < 3; ++k) e[k] = logf(fmaxf(fabsf(s[k]), 1e-6f));
        sand_principal(e, p, d);
    }
    tau_from_principal(u, d, tau);
}

__device__ __forceinline__ float fluid_tau(float J, float kappa, float gamma, int clamp_tension)
{
    float p = kappa * (powf(J, -gamma) - 1.0f);
    if (clamp_tension && p < 0.0f) p = 0.0f;
    return -p;
}

}  // namespace mpm
