// model_dev.cuh — per-step discretisation of the state-space models on the device.
//
// Replaces the reference's per-step `discretize` / `discretize_with_grad`
// (kernels.hpp:392-443), which run a Padé expm and one 2b x 2b Van Loan
// exponential per hyperparameter per step.  Here every leaf uses its exact
// closed form:
//   Matérn-ν (b = ν + 1/2):  F + λI is nilpotent, so
//       Φ = e^{-λΔt} Σ_{k<b} (F+λI)^k Δt^k / k!,
//       dΦ/dℓ = -(1/ℓ)[K, Φ] - (Δt/ℓ) F Φ   with K = diag(0, 1, ..., b-1)
//       (F(λ) = λ T F(1) T^{-1}, T = diag(1, λ, λ², ...)).
//   EQ order J (modal 2x2 rotation blocks, kernels.hpp:286-306):
//       Φ_p = e^{aΔt/ℓ} R(cΔt/ℓ),  dΦ/dℓ = -(Δt/ℓ) F Φ.
//   Quasi-periodic harmonic j:  Φ_j = e^{-Δt/env} R(j ω0 Δt),
//       Q_j = var q_j² (1 - e^{-2Δt/env}) I₂.
// Q = Pinf - Φ Pinf Φ^T symmetrised exactly as the reference (:402-403), and
// dQ by the reference's product rule (:419-423).  Step 0 (the anchor,
// SPEC.md:326) is encoded as dt < 0: Φ := 0, so Q = Pinf and dQ = dPinf.
//
// Per-series parameters live in a flat record (built on the host, capi.cpp):
//   rec[0] = sigma, rec[1] = jitter, rec[2 .. 2+nt) = d jitter / d theta,
//   then one sub-record per leaf at desc.rec[l]:
//     Matérn: var, len, lam
//     EQ    : var, len                     (+ shared constants in desc.eqconst)
//     QP    : var, len, period, env, w0, q2[0..J], dq2/dlen[0..J]
#pragma once

#include "devmat.cuh"
#include "model_desc.h"

namespace spingp_dev {

// ------------------------------------------------------------ accurate Q --
// The reference evaluates Q = Pinf - Φ Pinf Φ^T (kernels.hpp:402), which cancels
// catastrophically when Δt is small against the lengthscale (Q ~ Δt^{2b-1} while
// Pinf ~ 1): its fp64 error is ~eps·|Pinf|, far above the small eigenvalues of Q
// (SURVEY.md App. A).  The device evaluates the SAME matrix through its integral
// form Q(Δt) = ∫_0^Δt e^{Fs} L q L^T e^{F^T s} ds in closed form, entry by entry,
// with no cancellation; its θ-derivatives follow from the same form.

// 1/j for the runtime-length tail series (constant memory: warp-uniform index).
#ifdef SPINGP_HOST_EMU
static const double kRecip[96] = {
#else
static __constant__ double kRecip[96] = {
#endif
    0.0, 1.0 / 1, 1.0 / 2, 1.0 / 3, 1.0 / 4, 1.0 / 5, 1.0 / 6, 1.0 / 7, 1.0 / 8, 1.0 / 9, 1.0 / 10, 1.0 / 11,
    1.0 / 12, 1.0 / 13, 1.0 / 14, 1.0 / 15, 1.0 / 16, 1.0 / 17, 1.0 / 18, 1.0 / 19, 1.0 / 20, 1.0 / 21, 1.0 / 22,
    1.0 / 23, 1.0 / 24, 1.0 / 25, 1.0 / 26, 1.0 / 27, 1.0 / 28, 1.0 / 29, 1.0 / 30, 1.0 / 31, 1.0 / 32, 1.0 / 33,
    1.0 / 34, 1.0 / 35, 1.0 / 36, 1.0 / 37, 1.0 / 38, 1.0 / 39, 1.0 / 40, 1.0 / 41, 1.0 / 42, 1.0 / 43, 1.0 / 44,
    1.0 / 45, 1.0 / 46, 1.0 / 47, 1.0 / 48, 1.0 / 49, 1.0 / 50, 1.0 / 51, 1.0 / 52, 1.0 / 53, 1.0 / 54, 1.0 / 55,
    1.0 / 56, 1.0 / 57, 1.0 / 58, 1.0 / 59, 1.0 / 60, 1.0 / 61, 1.0 / 62, 1.0 / 63, 1.0 / 64, 1.0 / 65, 1.0 / 66,
    1.0 / 67, 1.0 / 68, 1.0 / 69, 1.0 / 70, 1.0 / 71, 1.0 / 72, 1.0 / 73, 1.0 / 74, 1.0 / 75, 1.0 / 76, 1.0 / 77,
    1.0 / 78, 1.0 / 79, 1.0 / 80, 1.0 / 81, 1.0 / 82, 1.0 / 83, 1.0 / 84, 1.0 / 85, 1.0 / 86, 1.0 / 87, 1.0 / 88,
    1.0 / 89, 1.0 / 90, 1.0 / 91, 1.0 / 92, 1.0 / 93, 1.0 / 94, 1.0 / 95};

// R_m(x) = e^{-x} Σ_{j>m} x^j / j!  (= 1 - e^{-x} Σ_{j<=m} x^j/j!), m = 0..M, x >= 0.
// No divisions: reciprocals are compile-time constants (unrolled tiers) or a table.
// x < 0.25: 14 tail terms by Horner; x < 6: terms until they stop contributing;
// else the direct form (no cancellation there).
template <int K, int M>
SP_DEV double tail_horner(double x) {  // Σ_{k<K} x^k (M+1)!/(M+1+k)!  (nested, smallest term first)
    double h = 1.0;
#pragma unroll
    for (int k = K - 2; k >= 0; --k) h = fma(h, x * (1.0 / double(M + 2 + k)), 1.0);
    return h;
}
template <int M>
SP_DEV void exp_tails(double x, double ex, double* R) {  // ex = e^{-x}
    double pw[M + 1];  // x^m / m!
    pw[0] = 1.0;
#pragma unroll
    for (int m = 1; m <= M; ++m) pw[m] = pw[m - 1] * (x * (1.0 / double(m)));
    if (x < 6.0) {
        const double t0 = pw[M] * (x * (1.0 / double(M + 1)));
        double s;
        if (x < 0.25) {
            s = t0 * tail_horner<14, M>(x);  // remainder < 0.25^14/14! relative
        } else {
            double term = t0;
            s = 0.0;
            for (int k = 0; k < 90 - M; ++k) {  // terms decrease monotonically once j > x
                s += term;
                term *= x * kRecip[M + 2 + k];
                if (term <= 1e-17 * s) break;
            }
        }
        R[M] = ex * s;
#pragma unroll
        for (int m = M; m >= 1; --m) R[m - 1] = R[m] + ex * pw[m];
    } else {
        double acc = 0.0;
#pragma unroll
        for (int m = 0; m <= M; ++m) {
            acc += pw[m];
            R[m] = 1.0 - ex * acc;
        }
    }
}

// ------------------------------------------------------------------ Matérn --
// Unit-λ companion model F1 = F(λ=1) (kernels.hpp:137-200) with F(λ) = λ T F1 T^{-1},
// T = diag(1, λ, λ², ...).  The noise column e^{F1 s} e_b = e^{-s} Σ_k c_k s^k and the
// unit spectral density q1 (F1 P1 + P1 F1^T + q1 e_b e_b^T = 0 with the unit-variance Pinf):
//   Matérn-1/2: c0 = [1];                                   q1 = 2
//   Matérn-3/2: c0 = [0,1], c1 = [1,-1];                    q1 = 4
//   Matérn-5/2: c0 = [0,0,1], c1 = [0,1,-2], c2 = ½[1,-1,1];  q1 = 16/3
// Then Q(Δt) = var T Q1(λΔt) T,  Q1(u)_ij = q1 Σ_kl c_k[i] c_l[j] I_{k+l}(u),
// I_m(u) = ∫_0^u s^m e^{-2s} ds = m!/2^{m+1} R_m(2u),
// and dQ/dλ = ((i+j)/λ) Q_ij + var Δt q1 (T v(u))(T v(u))^T, v(u) = e^{-u} Σ_k c_k u^k.
template <int D>
SP_DEV double matern_c(int k, int i) {
    if constexpr (D == 1) {
        return 1.0;
    } else if constexpr (D == 2) {
        return k == 0 ? (i == 1 ? 1.0 : 0.0) : (i == 0 ? 1.0 : -1.0);
    } else {
        if (k == 0) return i == 2 ? 1.0 : 0.0;
        if (k == 1) return i == 0 ? 0.0 : (i == 1 ? 1.0 : -2.0);
        return i == 1 ? -0.5 : 0.5;
    }
}
template <int D>
SP_DEV double matern_q1() {
    if constexpr (D == 1) return 2.0;
    else if constexpr (D == 2) return 4.0;
    else return 16.0 / 3.0;
}

// Block of dimension D at offset o inside LD x LD arrays.
template <int D, int LD>
SP_DEV void matern_block(const double* lr, double dt, int o, double* Phi, double* Q) {
    const double var = lr[0], lam = lr[2];
    double P[D * D];
    // Pinf (kernels.hpp:137-200)
    if constexpr (D == 1) {
        P[0] = var;
    } else if constexpr (D == 2) {
        P[0] = var; P[1] = 0.0; P[2] = 0.0; P[3] = var * lam * lam;
    } else {
        const double kap = lam * lam * (1.0 / 3.0);
        P[0] = var; P[1] = 0.0; P[2] = -var * kap;
        P[3] = 0.0; P[4] = var * kap; P[5] = 0.0;
        P[6] = -var * kap; P[7] = 0.0; P[8] = var * lam * lam * lam * lam;
    }
    if (dt < 0.0) {
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) {
                Phi[(o + i) * LD + o + j] = 0.0;
                Q[(o + i) * LD + o + j] = P[i * D + j];
            }
        return;
    }
    // Φ = e^{-λΔt} (I + NΔt + N²Δt²/2), N = F + λI nilpotent
    const double e = exp(-lam * dt);
    double ph[D * D];
    if constexpr (D == 1) {
        ph[0] = e;
    } else if constexpr (D == 2) {
        const double x = lam * dt;
        ph[0] = e * (1.0 + x); ph[1] = e * dt;
        ph[2] = -e * lam * x; ph[3] = e * (1.0 - x);
    } else {
        const double l2 = lam * lam, l3 = l2 * lam;
        const double N[9] = {lam, 1.0, 0.0, 0.0, lam, 1.0, -l3, -3.0 * l2, -2.0 * lam};
        double N2[9];
        mm<3>(N2, N, N);
        const double h = 0.5 * dt * dt;
#pragma unroll
        for (int k = 0; k < 9; ++k) ph[k] = e * ((k % 4 == 0 ? 1.0 : 0.0) + dt * N[k] + h * N2[k]);
    }
    // Q = var T Q1(λΔt) T (cancellation-free integral form)
    constexpr int M = 2 * (D - 1);
    double R[M + 1];
    const double u = lam * dt;
    exp_tails<M>(2.0 * u, e * e, R);  // e^{-2λΔt} = (e^{-λΔt})²
    double I[M + 1];
    {
        double f = 0.5;  // m! / 2^{m+1}
#pragma unroll
        for (int m = 0; m <= M; ++m) {
            I[m] = f * R[m];
            f *= double(m + 1) * 0.5;
        }
    }
    double tp[D];
    tp[0] = 1.0;
#pragma unroll
    for (int i = 1; i < D; ++i) tp[i] = tp[i - 1] * lam;
    const double q1 = matern_q1<D>();
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j <= i; ++j) {
            double s = 0.0;
#pragma unroll
            for (int k = 0; k < D; ++k)
#pragma unroll
                for (int l = 0; l < D; ++l) s += matern_c<D>(k, i) * matern_c<D>(l, j) * I[k + l];
            const double v = var * q1 * s * tp[i] * tp[j];
            Q[(o + i) * LD + o + j] = v;
            Q[(o + j) * LD + o + i] = v;
        }
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) Phi[(o + i) * LD + o + j] = ph[i * D + j];
}

// g[var] += ½Tr(M dQ̃_var) ; g[len] += ½Tr(M dQ̃_len) + Tr(dΦ_len Bm)
// (the jitter-derivative part ½ djit Tr(M) is added by the caller for every θ).
template <int D, int LD>
SP_DEV void matern_grad(const double* lr, double dt, int o, const double* Phi, const double* Q,
                        const double* M, const double* Bm, double& gvar, double& glen) {
    const double var = lr[0], len = lr[1], lam = lr[2];
    double ph[D * D], Mb[D * D], Bb[D * D], Qb[D * D];
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) {
            ph[i * D + j] = Phi[(o + i) * LD + o + j];
            Mb[i * D + j] = M[(o + i) * LD + o + j];
            Bb[i * D + j] = Bm[(o + i) * LD + o + j];
            Qb[i * D + j] = Q[(o + i) * LD + o + j];
        }
    // d/dvar: dΦ = 0, dQ = Q / var (also at the anchor, where Q = Pinf)
    (void)len;
    const double ilen = lr[3];  // 1/ℓ and 1/var come with the record (no per-step division)
    gvar += 0.5 * mtrprod<D>(Mb, Qb) * lr[4];
    // d/dℓ = -(λ/ℓ) d/dλ.  dQ/dλ_ij = ((i+j)/λ) Q_ij + var Δt q1 (T v)_i (T v)_j
    double dQ[D * D];
    const double c = -lam * ilen;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j) dQ[i * D + j] = -double(i + j) * ilen * Qb[i * D + j];
    if (dt < 0.0) {  // anchor: dPinf/dℓ_ij = -(i+j)/ℓ Pinf_ij
        glen += 0.5 * mtrprod<D>(Mb, dQ);
        return;
    }
    {
        const double u = lam * dt, eu = exp(-u);
        double v[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            double s = 0.0, pw = 1.0;
#pragma unroll
            for (int k = 0; k < D; ++k) {
                s += matern_c<D>(k, i) * pw;  // c_k already carries the 1/k!
                pw *= u;
            }
            v[i] = eu * s;
        }
        double tp = 1.0, tv[D];
#pragma unroll
        for (int i = 0; i < D; ++i) {
            tv[i] = tp * v[i];
            tp *= lam;
        }
        const double w = c * var * dt * matern_q1<D>();
#pragma unroll
        for (int i = 0; i < D; ++i)
#pragma unroll
            for (int j = 0; j < D; ++j) dQ[i * D + j] += w * tv[i] * tv[j];
    }
    // dΦ = -(1/ℓ)[K, Φ] - (Δt/ℓ) F Φ
    double F[D * D];
    if constexpr (D == 1) {
        F[0] = -lam;
    } else if constexpr (D == 2) {
        F[0] = 0.0; F[1] = 1.0; F[2] = -lam * lam; F[3] = -2.0 * lam;
    } else {
        F[0] = 0.0; F[1] = 1.0; F[2] = 0.0; F[3] = 0.0; F[4] = 0.0; F[5] = 1.0;
        F[6] = -lam * lam * lam; F[7] = -3.0 * lam * lam; F[8] = -3.0 * lam;
    }
    double FP[D * D], dph[D * D];
    mm<D>(FP, F, ph);
    const double c1 = -ilen, c2 = -dt * ilen;
#pragma unroll
    for (int i = 0; i < D; ++i)
#pragma unroll
        for (int j = 0; j < D; ++j)
            dph[i * D + j] = c1 * double(i - j) * ph[i * D + j] + c2 * FP[i * D + j];
    glen += 0.5 * mtrprod<D>(Mb, dQ) + mtrprod<D>(dph, Bb);
}

// ---------------------------------------------------------------------- EQ --
// Modal EQ (kernels.hpp:286-306): F = A/ℓ with 2x2 blocks A_p = [[a_p, c_p], [-c_p, a_p]],
// noise gain g = e_first of every pair, Pinf = var s0 p1 (s0 = 1/k0, kernels.hpp:310-315).
// Q(Δt) = var s0 G(Δt/ℓ),  G(τ) = ∫_0^τ e^{Au} g g^T e^{A^T u} du, block (p,q):
//   ½ [[C- + C+, S- - S+], [-(S+ + S-), C- - C+]],  C± + i S± = ∫_0^τ e^{(α + iβ±)u} du,
//   α = a_p + a_q, β± = c_p ± c_q  — evaluated with a complex expm1 (no cancellation).
// dQ/dℓ = -var s0 (Δt/ℓ²) e^{Aτ} g g^T e^{A^T τ}; dQ/dvar = Q/var.
// Constants at desc.eqconst + eqc[l]: (a_p, c_p) pairs, P1 = s0 p1 (J*J), s0.
SP_DEV void phi1_int(double a, double b, double tau, double& re, double& im) {
    // (e^{(a+ib)τ} - 1) / (a + ib)
    const double x = a * tau, y = b * tau;
    double sy, cy;
    sincos(y, &sy, &cy);
    const double sh = sin(0.5 * y);
    const double er = expm1(x) * cy - 2.0 * sh * sh;  // Re(e^w - 1)
    const double ei = exp(x) * sy;                     // Im(e^w - 1)
    const double den = a * a + b * b;
    re = (er * a + ei * b) / den;
    im = (ei * a - er * b) / den;
}

template <int LD>
SP_DEV void eq_block(int o, int J, const double* ac, const double* lr, double dt, double* Phi,
                     double* Q) {
    const double var = lr[0], len = lr[1];
    const double* P1 = ac + J;  // J/2 pairs of (a, c), then P1, then s0
    const double s0 = P1[J * J];
    if (dt < 0.0) {
        for (int i = 0; i < J; ++i)
            for (int j = 0; j < J; ++j) {
                Phi[(o + i) * LD + o + j] = 0.0;
                Q[(o + i) * LD + o + j] = var * P1[i * J + j];
            }
        return;
    }
    for (int i = 0; i < J; ++i)
        for (int j = 0; j < J; ++j) Phi[(o + i) * LD + o + j] = 0.0;
    const double tau = dt * lr[2];  // dt / len
    for (int p = 0; p < J / 2; ++p) {
        const double a = ac[2 * p], c = ac[2 * p + 1];
        const double rho = exp(a * tau);
        double sn, cs;
        sincos(c * tau, &sn, &cs);
        const int k = o + 2 * p;
        Phi[k * LD + k] = rho * cs;
        Phi[k * LD + k + 1] = rho * sn;
        Phi[(k + 1) * LD + k] = -rho * sn;
        Phi[(k + 1) * LD + k + 1] = rho * cs;
    }
    const double w = 0.5 * var * s0;
    for (int p = 0; p < J / 2; ++p)
        for (int q = 0; q <= p; ++q) {
            const double al = ac[2 * p] + ac[2 * q];
            double cm, sm, cp, sp;
            phi1_int(al, ac[2 * p + 1] - ac[2 * q + 1], tau, cm, sm);
            phi1_int(al, ac[2 * p + 1] + ac[2 * q + 1], tau, cp, sp);
            const double g00 = w * (cm + cp), g01 = w * (sm - sp), g10 = -w * (sp + sm), g11 = w * (cm - cp);
            const int r = o + 2 * p, s = o + 2 * q;
            Q[r * LD + s] = g00;
            Q[r * LD + s + 1] = g01;
            Q[(r + 1) * LD + s] = g10;
            Q[(r + 1) * LD + s + 1] = g11;
            Q[s * LD + r] = g00;
            Q[(s + 1) * LD + r] = g01;
            Q[s * LD + r + 1] = g10;
            Q[(s + 1) * LD + r + 1] = g11;
        }
}

template <int LD>
SP_DEV void eq_grad(int o, int J, const double* ac, const double* lr, double dt, const double* Phi,
                    const double* Q, const double* M, const double* Bm, double& gvar,
                    double& glen) {
    const double var = lr[0], len = lr[1];
    const double s0 = ac[J + J * J];
    // var: dQ = Q / var
    double s = 0.0;
    for (int i = 0; i < J; ++i)
        for (int k = 0; k < J; ++k) s += M[(o + i) * LD + o + k] * Q[(o + k) * LD + o + i];
    const double ilen = lr[2], ivar = lr[3];
    gvar += 0.5 * s * ivar;
    if (dt < 0.0) return;  // dPinf/dℓ = 0 and dΦ = 0 at the anchor
    const double tau = dt * ilen;
    // dQ/dℓ = -var s0 (Δt/ℓ²) z z^T with z = e^{Aτ} g: pair p -> e^{a τ} [cos(cτ), -sin(cτ)]
    double z0[kMaxB / 2], z1[kMaxB / 2];
    for (int p = 0; p < J / 2; ++p) {
        const double rho = exp(ac[2 * p] * tau);
        double sn, cs;
        sincos(ac[2 * p + 1] * tau, &sn, &cs);
        z0[p] = rho * cs;
        z1[p] = -rho * sn;
    }
    double tq = 0.0, tb = 0.0;
    const double cdt = -dt * ilen;
    for (int p = 0; p < J / 2; ++p) {
        const double a = ac[2 * p], c = ac[2 * p + 1];
        const int k = o + 2 * p;
        const double zp0 = z0[p], zp1 = z1[p];
        for (int q = 0; q < J / 2; ++q) {
            const int kq = o + 2 * q;
            const double zq0 = z0[q], zq1 = z1[q];
            tq += M[kq * LD + k] * zp0 * zq0 + M[(kq + 1) * LD + k] * zp0 * zq1 +
                  M[kq * LD + k + 1] * zp1 * zq0 + M[(kq + 1) * LD + k + 1] * zp1 * zq1;
        }
        // dΦ = -(Δt/ℓ) F Φ on the 2x2 block
        const double f00 = a * ilen, f01 = c * ilen, f10 = -c * ilen, f11 = a * ilen;
        const double p00 = Phi[k * LD + k], p01 = Phi[k * LD + k + 1];
        const double p10 = Phi[(k + 1) * LD + k], p11 = Phi[(k + 1) * LD + k + 1];
        const double d00 = cdt * (f00 * p00 + f01 * p10), d01 = cdt * (f00 * p01 + f01 * p11);
        const double d10 = cdt * (f10 * p00 + f11 * p10), d11 = cdt * (f10 * p01 + f11 * p11);
        tb += d00 * Bm[k * LD + k] + d01 * Bm[(k + 1) * LD + k] + d10 * Bm[k * LD + k + 1] +
              d11 * Bm[(k + 1) * LD + k + 1];
    }
    glen += 0.5 * (-var * s0 * dt * ilen * ilen) * tq + tb;
}

// ---------------------------------------------------------------------- QP --
template <int LD>
SP_DEV void qp_block(int o, int J, const double* lr, double dt, double* Phi, double* Q) {
    const int d = 2 * (J + 1);
    const double var = lr[0], env = lr[3], w0 = lr[4];
    const double* q2 = lr + 5;
    for (int i = 0; i < d; ++i)
        for (int j = 0; j < d; ++j) {
            Phi[(o + i) * LD + o + j] = 0.0;
            Q[(o + i) * LD + o + j] = 0.0;
        }
    (void)env;
    const double ienv = lr[5 + 2 * (J + 1)];
    const double rho = dt < 0.0 ? 0.0 : exp(-dt * ienv);
    const double one_m = dt < 0.0 ? 1.0 : -expm1(-2.0 * dt * ienv);
    // harmonics by the angle-addition recurrence from one sincos (error ~ j ulp, j <= 15)
    double s1 = 0.0, c1 = 1.0, sn = 0.0, cs = 1.0;
    if (dt >= 0.0) sincos(w0 * dt, &s1, &c1);
    for (int j = 0; j <= J; ++j) {
        const int k = o + 2 * j;
        if (j > 0) {
            const double cn = cs * c1 - sn * s1;
            sn = sn * c1 + cs * s1;
            cs = cn;
        }
        if (dt >= 0.0) {
            Phi[k * LD + k] = rho * cs;
            Phi[k * LD + k + 1] = -rho * sn;
            Phi[(k + 1) * LD + k] = rho * sn;
            Phi[(k + 1) * LD + k + 1] = rho * cs;
        }
        const double qv = var * q2[j] * one_m;
        Q[k * LD + k] = qv;
        Q[(k + 1) * LD + k + 1] = qv;
    }
}

// gradients w.r.t. (var, len, period, env) of one QP leaf
template <int LD>
SP_DEV void qp_grad(int o, int J, const double* lr, double dt, const double* Phi, const double* M,
                    const double* Bm, double* g4) {
    const double var = lr[0];
    const double* q2 = lr + 5;
    const double* dq2 = lr + 5 + (J + 1);
    const double ienv = lr[5 + 2 * (J + 1)], dwp = lr[5 + 2 * (J + 1) + 1];  // 1/env, w0/period
    const double rho2 = dt < 0.0 ? 0.0 : exp(-2.0 * dt * ienv);
    const double one_m = dt < 0.0 ? 1.0 : -expm1(-2.0 * dt * ienv);
    for (int j = 0; j <= J; ++j) {
        const int k = o + 2 * j;
        const double trM = M[k * LD + k] + M[(k + 1) * LD + k + 1];
        g4[0] += 0.5 * trM * q2[j] * one_m;         // dQ/dvar = q2 (1 - ρ²) I
        g4[1] += 0.5 * trM * var * dq2[j] * one_m;  // dQ/dlen = var dq2 (1 - ρ²) I
        if (dt < 0.0) continue;
        // env: dΦ = (Δt/env²) Φ ; dQ = -2 var q2 (Δt/env²) ρ² I
        const double ce = dt * ienv * ienv;
        const double trPB = Phi[k * LD + k] * Bm[k * LD + k] + Phi[k * LD + k + 1] * Bm[(k + 1) * LD + k] +
                            Phi[(k + 1) * LD + k] * Bm[k * LD + k + 1] +
                            Phi[(k + 1) * LD + k + 1] * Bm[(k + 1) * LD + k + 1];
        g4[3] += 0.5 * trM * (-2.0 * var * q2[j] * ce * rho2) + ce * trPB;
        // period: dF = j dω [[0,-1],[1,0]], dω = -ω0/period; dΦ = Δt dF Φ; dQ = 0
        const double s = double(j) * (-dwp) * dt;
        // dΦ = s * [[-Φ10, -Φ11], [Φ00, Φ01]]
        const double d00 = -s * Phi[(k + 1) * LD + k], d01 = -s * Phi[(k + 1) * LD + k + 1];
        const double d10 = s * Phi[k * LD + k], d11 = s * Phi[k * LD + k + 1];
        g4[2] += d00 * Bm[k * LD + k] + d01 * Bm[(k + 1) * LD + k] + d10 * Bm[k * LD + k + 1] +
                 d11 * Bm[(k + 1) * LD + k + 1];
    }
}


#ifndef SPINGP_HOST_EMU
// ---------------------------------------------------- team-parallel leaves --
// The same closed forms, with the independent pieces of one leaf (EQ rotation blocks and
// (p, q) covariance pairs, QP harmonics) spread over the `nl` lanes of a team (team.cuh):
// lane `ln` computes pieces ln, ln + nl, ...  The block has been zero-filled by the team.
template <int LD>
SP_DEV void eq_block_team(int o, int J, const double* ac, const double* lr, double dt, double* Phi, double* Q,
                          int ln, int nl) {
    const double var = lr[0];
    const double* P1 = ac + J;
    const double s0 = P1[J * J];
    if (dt < 0.0) {
        for (int k = ln; k < J * J; k += nl) Q[(o + k / J) * LD + o + k % J] = var * P1[k];
        return;
    }
    const double tau = dt * lr[2];
    for (int p = ln; p < J / 2; p += nl) {
        const double a = ac[2 * p], c = ac[2 * p + 1];
        const double rho = exp(a * tau);
        double sn, cs;
        sincos(c * tau, &sn, &cs);
        const int k = o + 2 * p;
        Phi[k * LD + k] = rho * cs;
        Phi[k * LD + k + 1] = rho * sn;
        Phi[(k + 1) * LD + k] = -rho * sn;
        Phi[(k + 1) * LD + k + 1] = rho * cs;
    }
    const double w = 0.5 * var * s0;
    const int np = (J / 2) * (J / 2 + 1) / 2;
    for (int k = ln; k < np; k += nl) {
        int p = 0;
        while ((p + 1) * (p + 2) / 2 <= k) ++p;
        const int q = k - p * (p + 1) / 2;
        const double al = ac[2 * p] + ac[2 * q];
        double cm, sm, cp, sp;
        phi1_int(al, ac[2 * p + 1] - ac[2 * q + 1], tau, cm, sm);
        phi1_int(al, ac[2 * p + 1] + ac[2 * q + 1], tau, cp, sp);
        const double g00 = w * (cm + cp), g01 = w * (sm - sp), g10 = -w * (sp + sm), g11 = w * (cm - cp);
        const int r = o + 2 * p, s = o + 2 * q;
        Q[r * LD + s] = g00;
        Q[r * LD + s + 1] = g01;
        Q[(r + 1) * LD + s] = g10;
        Q[(r + 1) * LD + s + 1] = g11;
        Q[s * LD + r] = g00;
        Q[(s + 1) * LD + r] = g01;
        Q[s * LD + r + 1] = g10;
        Q[(s + 1) * LD + r + 1] = g11;
    }
}

template <int LD>
SP_DEV void eq_grad_team(int o, int J, const double* ac, const double* lr, double dt, const double* Phi,
                         const double* Q, const double* M, const double* Bm, double& gvar, double& glen, int ln,
                         int nl) {
    const double var = lr[0];
    const double s0 = ac[J + J * J];
    double s = 0.0;
    for (int i = ln; i < J; i += nl)
        for (int k = 0; k < J; ++k) s += M[(o + i) * LD + o + k] * Q[(o + k) * LD + o + i];
    const double ilen = lr[2], ivar = lr[3];
    gvar += 0.5 * s * ivar;
    if (dt < 0.0) return;
    // z = e^{Aτ} g: pair p -> e^{a τ} [cos(cτ), -sin(cτ)] = (Φ_kk, -Φ_{k,k+1}) of the
    // rotation block eq_block_team wrote (same expressions: no second exp / sincos)
    double z0[kMaxB / 2], z1[kMaxB / 2];
    for (int p = 0; p < J / 2; ++p) {
        const int k = o + 2 * p;
        z0[p] = Phi[k * LD + k];
        z1[p] = -Phi[k * LD + k + 1];
    }
    double tq = 0.0, tb = 0.0;
    const double cdt = -dt * ilen;
    for (int p = ln; p < J / 2; p += nl) {
        const double a = ac[2 * p], c = ac[2 * p + 1];
        const int k = o + 2 * p;
        const double zp0 = z0[p], zp1 = z1[p];
        for (int q = 0; q < J / 2; ++q) {
            const int kq = o + 2 * q;
            const double zq0 = z0[q], zq1 = z1[q];
            tq += M[kq * LD + k] * zp0 * zq0 + M[(kq + 1) * LD + k] * zp0 * zq1 +
                  M[kq * LD + k + 1] * zp1 * zq0 + M[(kq + 1) * LD + k + 1] * zp1 * zq1;
        }
        const double f00 = a * ilen, f01 = c * ilen, f10 = -c * ilen, f11 = a * ilen;
        const double p00 = Phi[k * LD + k], p01 = Phi[k * LD + k + 1];
        const double p10 = Phi[(k + 1) * LD + k], p11 = Phi[(k + 1) * LD + k + 1];
        const double d00 = cdt * (f00 * p00 + f01 * p10), d01 = cdt * (f00 * p01 + f01 * p11);
        const double d10 = cdt * (f10 * p00 + f11 * p10), d11 = cdt * (f10 * p01 + f11 * p11);
        tb += d00 * Bm[k * LD + k] + d01 * Bm[(k + 1) * LD + k] + d10 * Bm[k * LD + k + 1] +
              d11 * Bm[(k + 1) * LD + k + 1];
    }
    glen += 0.5 * (-var * s0 * dt * ilen * ilen) * tq + tb;
}

// harmonic j by its own sincos (the thread-per-chunk qp_block uses the angle-addition
// recurrence from one sincos; the two agree to a few ulp)
template <int LD>
SP_DEV void qp_block_team(int o, int J, const double* lr, double dt, double* Phi, double* Q, int ln, int nl) {
    const double var = lr[0], w0 = lr[4];
    const double* q2 = lr + 5;
    const double ienv = lr[5 + 2 * (J + 1)];
    const double rho = dt < 0.0 ? 0.0 : exp(-dt * ienv);
    const double one_m = dt < 0.0 ? 1.0 : -expm1(-2.0 * dt * ienv);
    for (int j = ln; j <= J; j += nl) {
        const int k = o + 2 * j;
        if (dt >= 0.0) {
            double sn = 0.0, cs = 1.0;
            if (j > 0) sincos(double(j) * (w0 * dt), &sn, &cs);
            Phi[k * LD + k] = rho * cs;
            Phi[k * LD + k + 1] = -rho * sn;
            Phi[(k + 1) * LD + k] = rho * sn;
            Phi[(k + 1) * LD + k + 1] = rho * cs;
        }
        const double qv = var * q2[j] * one_m;
        Q[k * LD + k] = qv;
        Q[(k + 1) * LD + k + 1] = qv;
    }
}

template <int LD>
SP_DEV void qp_grad_team(int o, int J, const double* lr, double dt, const double* Phi, const double* M,
                         const double* Bm, double* g4, int ln, int nl) {
    const double var = lr[0];
    const double* q2 = lr + 5;
    const double* dq2 = lr + 5 + (J + 1);
    const double ienv = lr[5 + 2 * (J + 1)], dwp = lr[5 + 2 * (J + 1) + 1];
    const double rho2 = dt < 0.0 ? 0.0 : exp(-2.0 * dt * ienv);
    const double one_m = dt < 0.0 ? 1.0 : -expm1(-2.0 * dt * ienv);
    for (int j = ln; j <= J; j += nl) {
        const int k = o + 2 * j;
        const double trM = M[k * LD + k] + M[(k + 1) * LD + k + 1];
        g4[0] += 0.5 * trM * q2[j] * one_m;
        g4[1] += 0.5 * trM * var * dq2[j] * one_m;
        if (dt < 0.0) continue;
        const double ce = dt * ienv * ienv;
        const double trPB = Phi[k * LD + k] * Bm[k * LD + k] + Phi[k * LD + k + 1] * Bm[(k + 1) * LD + k] +
                            Phi[(k + 1) * LD + k] * Bm[k * LD + k + 1] +
                            Phi[(k + 1) * LD + k + 1] * Bm[(k + 1) * LD + k + 1];
        g4[3] += 0.5 * trM * (-2.0 * var * q2[j] * ce * rho2) + ce * trPB;
        const double sj = double(j) * (-dwp) * dt;
        const double d00 = -sj * Phi[(k + 1) * LD + k], d01 = -sj * Phi[(k + 1) * LD + k + 1];
        const double d10 = sj * Phi[k * LD + k], d11 = sj * Phi[k * LD + k + 1];
        g4[2] += d00 * Bm[k * LD + k] + d01 * Bm[(k + 1) * LD + k] + d10 * Bm[k * LD + k + 1] +
                 d11 * Bm[(k + 1) * LD + k + 1];
    }
}
#endif

// ------------------------------------------------------------------ traits --
// A Traits type provides B (block size of the instantiation), the emission row
// and the two per-step model functions used by the elimination kernels.

// Single Matérn leaf: everything in registers.
template <int D>
struct MaternTraits {
    static constexpr int B = D;
    SP_DEV static double H(const ModelDesc&, int i) { return i == 0 ? 1.0 : 0.0; }
    SP_DEV static void step(const ModelDesc& md, const double* rec, double dt, double* Phi,
                            double* Q) {
        matern_block<D, D>(rec + md.rec[0], dt, 0, Phi, Q);
    }
    SP_DEV static void grad(const ModelDesc& md, const double* rec, double dt, const double* Phi,
                            const double* Q, const double* M, const double* Bm, double* g) {
        double gv = 0.0, gl = 0.0;
        matern_grad<D, D>(rec + md.rec[0], dt, 0, Phi, Q, M, Bm, gv, gl);
        const double hm = 0.5 * mtrace<D>(M);
        g[0] += gv + hm * rec[2];
        g[1] += gl + hm * rec[3];
    }
};

// Any sum of leaves, padded to B (padding states: Φ = 0, Q = 1, H = 0 — exactly
// decoupled, so results are identical to the unpadded system).
template <int BB>
struct GenericTraits {
    static constexpr int B = BB;
    static constexpr int NP = kMaxTheta;  // gradient slots of the team reduction
    static constexpr bool kDiag2 = false;
    SP_DEV static double H(const ModelDesc& md, int i) { return i < md.b ? md.H[i] : 0.0; }
    template <int LD = BB>  // row stride of Phi, Q (the team kernels use an odd one)
    SP_DEV static void step(const ModelDesc& md, const double* rec, double dt, double* Phi,
                            double* Q) {
        // Zero-fill with a rolled loop: statically unrolled (vectorised) zero stores
        // followed by the leaves' dynamically offset stores into the same local array
        // were reordered by nvcc 12.9 / sm_100a (lost Q[0..1]; tools/dbg/dbg_generic.cu).
#pragma unroll 1
        for (int i = 0; i < BB * BB; ++i) {
            Phi[(i / BB) * LD + i % BB] = 0.0;
            Q[(i / BB) * LD + i % BB] = 0.0;
        }
        for (int i = md.b; i < BB; ++i) Q[i * LD + i] = 1.0;  // padding
        SP_MEMFENCE();
        for (int l = 0; l < md.nleaves; ++l) {
            const double* lr = rec + md.rec[l];
            SP_MEMFENCE();
            switch (md.type[l]) {
                case MATERN12: matern_block<1, LD>(lr, dt, md.off[l], Phi, Q); break;
                case MATERN32: matern_block<2, LD>(lr, dt, md.off[l], Phi, Q); break;
                case MATERN52: matern_block<3, LD>(lr, dt, md.off[l], Phi, Q); break;
                case EQ: eq_block<LD>(md.off[l], md.dim[l], md.eqconst + md.eqc[l], lr, dt, Phi, Q); break;
                case QP: qp_block<LD>(md.off[l], md.order[l], lr, dt, Phi, Q); break;
            }
        }
        SP_MEMFENCE();
    }
    template <int LD = BB>
    SP_DEV static void grad(const ModelDesc& md, const double* rec, double dt, const double* Phi,
                            const double* Q, const double* M, const double* Bm, double* g) {
        double hm = 0.0;
        for (int i = 0; i < md.b; ++i) hm += M[i * LD + i];
        hm *= 0.5;
        SP_MEMFENCE();
        for (int l = 0; l < md.nleaves; ++l) {
            const double* lr = rec + md.rec[l];
            const int t0 = md.th[l];
            SP_MEMFENCE();
            double gv = 0.0, gl = 0.0;
            switch (md.type[l]) {
                case MATERN12: matern_grad<1, LD>(lr, dt, md.off[l], Phi, Q, M, Bm, gv, gl); break;
                case MATERN32: matern_grad<2, LD>(lr, dt, md.off[l], Phi, Q, M, Bm, gv, gl); break;
                case MATERN52: matern_grad<3, LD>(lr, dt, md.off[l], Phi, Q, M, Bm, gv, gl); break;
                case EQ:
                    eq_grad<LD>(md.off[l], md.dim[l], md.eqconst + md.eqc[l], lr, dt, Phi, Q, M, Bm, gv, gl);
                    break;
                case QP: {
                    double g4[4] = {0.0, 0.0, 0.0, 0.0};
                    qp_grad<LD>(md.off[l], md.order[l], lr, dt, Phi, M, Bm, g4);
                    g[t0 + 2] += g4[2];
                    g[t0 + 3] += g4[3];
                    gv = g4[0];
                    gl = g4[1];
                    break;
                }
            }
            g[t0] += gv;
            g[t0 + 1] += gl;
        }
        for (int p = 0; p < md.nt; ++p) g[p] += hm * rec[2 + p];
    }
#ifndef SPINGP_HOST_EMU
    // team versions (team.cuh): the dynamically offset leaves run on lane 0
    template <int LD>
    SP_DEV static void step_team(const ModelDesc& md, const double* rec, double dt, double* Phi, double* Q, int ln,
                                 int, unsigned) {
        if (ln == 0) step<LD>(md, rec, dt, Phi, Q);
    }
    template <int LD>
    SP_DEV static void grad_team(const ModelDesc& md, const double* rec, double dt, const double* Phi,
                                 const double* Q, const double* M, const double* Bm, int ln, int, double* g) {
        if (ln == 0) grad<LD>(md, rec, dt, Phi, Q, M, Bm, g);
    }
#endif
};

// Static-structure models: leaf types and offsets are template constants, so every
// block index is a compile-time constant after inlining (the fast, fully optimised
// path for the BASELINE models; GenericTraits above is the any-sum fallback).
template <int D>
struct SMatern {
    static constexpr int dim = D, np = 2;
    // Φ, Q block diagonal in aligned 2 x 2 blocks (the team kernels' fast path)
    static constexpr bool kDiag2 = D == 2;
    template <int O, int LD>
    SP_DEV static void step(const ModelDesc&, int, const double* lr, double dt, double* Phi, double* Q) {
        matern_block<D, LD>(lr, dt, O, Phi, Q);
    }
    template <int O, int LD>
    SP_DEV static void grad(const ModelDesc&, int, const double* lr, double dt, const double* Phi,
                            const double* Q, const double* M, const double* Bm, double* g) {
        matern_grad<D, LD>(lr, dt, O, Phi, Q, M, Bm, g[0], g[1]);
    }
#ifndef SPINGP_HOST_EMU
    // the last lane of the team (the other leaf's pieces start at lane 0)
    template <int O, int LD>
    SP_DEV static void step_team(const ModelDesc& md, int l, const double* lr, double dt, double* Phi, double* Q,
                                 int ln, int nl) {
        if (ln == nl - 1) matern_block<D, LD>(lr, dt, O, Phi, Q);
    }
    template <int O, int LD>
    SP_DEV static void grad_team(const ModelDesc& md, int l, const double* lr, double dt, const double* Phi,
                                 const double* Q, const double* M, const double* Bm, double* g, int ln, int nl) {
        if (ln == nl - 1) matern_grad<D, LD>(lr, dt, O, Phi, Q, M, Bm, g[0], g[1]);
    }
#endif
};
template <int J>
struct SEQ {
    static constexpr int dim = J, np = 2;
    static constexpr bool kDiag2 = false;  // Q couples every modal pair
    template <int O, int LD>
    SP_DEV static void step(const ModelDesc& md, int l, const double* lr, double dt, double* Phi, double* Q) {
        eq_block<LD>(O, J, md.eqconst + md.eqc[l], lr, dt, Phi, Q);
    }
    template <int O, int LD>
    SP_DEV static void grad(const ModelDesc& md, int l, const double* lr, double dt, const double* Phi,
                            const double* Q, const double* M, const double* Bm, double* g) {
        eq_grad<LD>(O, J, md.eqconst + md.eqc[l], lr, dt, Phi, Q, M, Bm, g[0], g[1]);
    }
#ifndef SPINGP_HOST_EMU
    template <int O, int LD>
    SP_DEV static void step_team(const ModelDesc& md, int l, const double* lr, double dt, double* Phi, double* Q,
                                 int ln, int nl) {
        eq_block_team<LD>(O, J, md.eqconst + md.eqc[l], lr, dt, Phi, Q, ln, nl);
    }
    template <int O, int LD>
    SP_DEV static void grad_team(const ModelDesc& md, int l, const double* lr, double dt, const double* Phi,
                                 const double* Q, const double* M, const double* Bm, double* g, int ln, int nl) {
        eq_grad_team<LD>(O, J, md.eqconst + md.eqc[l], lr, dt, Phi, Q, M, Bm, g[0], g[1], ln, nl);
    }
#endif
};
template <int J>
struct SQP {
    static constexpr int dim = 2 * (J + 1), np = 4;
    static constexpr bool kDiag2 = true;  // one 2 x 2 rotation block per harmonic
    template <int O, int LD>
    SP_DEV static void step(const ModelDesc&, int, const double* lr, double dt, double* Phi, double* Q) {
        qp_block<LD>(O, J, lr, dt, Phi, Q);
    }
    template <int O, int LD>
    SP_DEV static void grad(const ModelDesc&, int, const double* lr, double dt, const double* Phi,
                            const double*, const double* M, const double* Bm, double* g) {
        qp_grad<LD>(O, J, lr, dt, Phi, M, Bm, g);
    }
#ifndef SPINGP_HOST_EMU
    template <int O, int LD>
    SP_DEV static void step_team(const ModelDesc&, int, const double* lr, double dt, double* Phi, double* Q, int ln,
                                 int nl) {
        qp_block_team<LD>(O, J, lr, dt, Phi, Q, ln, nl);
    }
    template <int O, int LD>
    SP_DEV static void grad_team(const ModelDesc&, int, const double* lr, double dt, const double* Phi,
                                 const double*, const double* M, const double* Bm, double* g, int ln, int nl) {
        qp_grad_team<LD>(O, J, lr, dt, Phi, M, Bm, g, ln, nl);
    }
#endif
};

// One or two static leaves (the second at offset dim of the first).
template <class L0, class L1 = void>
struct StaticTraits {
    static constexpr int B = L0::dim + L1::dim;
    static constexpr int NP = L0::np + L1::np;
    static constexpr bool kDiag2 = L0::kDiag2 && L1::kDiag2 && (L0::dim % 2 == 0);
    SP_DEV static double H(const ModelDesc& md, int i) { return md.H[i]; }
    SP_DEV static void step(const ModelDesc& md, const double* rec, double dt, double* Phi, double* Q) {
        mzero<B>(Phi);
        mzero<B>(Q);
        SP_MEMFENCE();
        L0::template step<0, B>(md, 0, rec + md.rec[0], dt, Phi, Q);
        SP_MEMFENCE();
        L1::template step<L0::dim, B>(md, 1, rec + md.rec[1], dt, Phi, Q);
        SP_MEMFENCE();
    }
    SP_DEV static void grad(const ModelDesc& md, const double* rec, double dt, const double* Phi,
                            const double* Q, const double* M, const double* Bm, double* g) {
        double g0[4] = {0.0, 0.0, 0.0, 0.0}, g1[4] = {0.0, 0.0, 0.0, 0.0};
        SP_MEMFENCE();
        L0::template grad<0, B>(md, 0, rec + md.rec[0], dt, Phi, Q, M, Bm, g0);
        SP_MEMFENCE();
        L1::template grad<L0::dim, B>(md, 1, rec + md.rec[1], dt, Phi, Q, M, Bm, g1);
        SP_MEMFENCE();
        const double hm = 0.5 * mtrace<B>(M);
#pragma unroll
        for (int p = 0; p < L0::np; ++p) g[p] += g0[p] + hm * rec[2 + p];
#pragma unroll
        for (int p = 0; p < L1::np; ++p) g[L0::np + p] += g1[p] + hm * rec[2 + L0::np + p];
    }
#ifndef SPINGP_HOST_EMU
    // team versions (team.cuh): zero-fill spread over the lanes, a team barrier, then
    // every leaf's pieces spread over the lanes; gradient partials per lane in g[NP]
    template <int LD>
    SP_DEV static void step_team(const ModelDesc& md, const double* rec, double dt, double* Phi, double* Q, int ln,
                                 int nl, unsigned mask) {
        for (int i = ln; i < B * B; i += nl) {
            Phi[(i / B) * LD + i % B] = 0.0;
            Q[(i / B) * LD + i % B] = 0.0;
        }
        __syncwarp(mask);
        L0::template step_team<0, LD>(md, 0, rec + md.rec[0], dt, Phi, Q, ln, nl);
        L1::template step_team<L0::dim, LD>(md, 1, rec + md.rec[1], dt, Phi, Q, ln, nl);
    }
    template <int LD>
    SP_DEV static void grad_team(const ModelDesc& md, const double* rec, double dt, const double* Phi,
                                 const double* Q, const double* M, const double* Bm, int ln, int nl, double* g) {
        double g0[4] = {0.0, 0.0, 0.0, 0.0}, g1[4] = {0.0, 0.0, 0.0, 0.0};
        L0::template grad_team<0, LD>(md, 0, rec + md.rec[0], dt, Phi, Q, M, Bm, g0, ln, nl);
        L1::template grad_team<L0::dim, LD>(md, 1, rec + md.rec[1], dt, Phi, Q, M, Bm, g1, ln, nl);
        const double hm = ln < B ? 0.5 * M[ln * LD + ln] : 0.0;  // lane ln's share of ½Tr(M)
#pragma unroll
        for (int p = 0; p < L0::np; ++p) g[p] += g0[p] + hm * rec[2 + p];
#pragma unroll
        for (int p = 0; p < L1::np; ++p) g[L0::np + p] += g1[p] + hm * rec[2 + L0::np + p];
    }
#endif
};
template <class L0>
struct StaticTraits<L0, void> {
    static constexpr int B = L0::dim;
    static constexpr int NP = L0::np;
    static constexpr bool kDiag2 = L0::kDiag2;
    SP_DEV static double H(const ModelDesc& md, int i) { return md.H[i]; }
    SP_DEV static void step(const ModelDesc& md, const double* rec, double dt, double* Phi, double* Q) {
        mzero<B>(Phi);
        mzero<B>(Q);
        SP_MEMFENCE();
        L0::template step<0, B>(md, 0, rec + md.rec[0], dt, Phi, Q);
        SP_MEMFENCE();
    }
    SP_DEV static void grad(const ModelDesc& md, const double* rec, double dt, const double* Phi,
                            const double* Q, const double* M, const double* Bm, double* g) {
        double g0[4] = {0.0, 0.0, 0.0, 0.0};
        SP_MEMFENCE();
        L0::template grad<0, B>(md, 0, rec + md.rec[0], dt, Phi, Q, M, Bm, g0);
        SP_MEMFENCE();
        const double hm = 0.5 * mtrace<B>(M);
#pragma unroll
        for (int p = 0; p < L0::np; ++p) g[p] += g0[p] + hm * rec[2 + p];
    }
#ifndef SPINGP_HOST_EMU
    template <int LD>
    SP_DEV static void step_team(const ModelDesc& md, const double* rec, double dt, double* Phi, double* Q, int ln,
                                 int nl, unsigned mask) {
        for (int i = ln; i < B * B; i += nl) {
            Phi[(i / B) * LD + i % B] = 0.0;
            Q[(i / B) * LD + i % B] = 0.0;
        }
        __syncwarp(mask);
        L0::template step_team<0, LD>(md, 0, rec + md.rec[0], dt, Phi, Q, ln, nl);
    }
    template <int LD>
    SP_DEV static void grad_team(const ModelDesc& md, const double* rec, double dt, const double* Phi,
                                 const double* Q, const double* M, const double* Bm, int ln, int nl, double* g) {
        double g0[4] = {0.0, 0.0, 0.0, 0.0};
        L0::template grad_team<0, LD>(md, 0, rec + md.rec[0], dt, Phi, Q, M, Bm, g0, ln, nl);
        const double hm = ln < B ? 0.5 * M[ln * LD + ln] : 0.0;
#pragma unroll
        for (int p = 0; p < L0::np; ++p) g[p] += g0[p] + hm * rec[2 + p];
    }
#endif
};

}  // namespace spingp_dev
