// host_model.cpp — host-side model setup (g++, C++20): kernel leaves -> device
// model description and per-series parameter records, plus the host-only C ABI
// entry points (spingp_kernel_dims, spingp_state_space).  Uses the drop-in
// C++ API of include/spingp/kernels.hpp for the reference's state_space_of.
#include <atomic>
#include <cstdlib>
#include "host_model.hpp"

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <numbers>
#include <stdexcept>

#include "spingp/kernels.hpp"

using namespace spingp_dev;

namespace spingp_host {

namespace {
// Device constants of the modal EQ realisation (kernels.hpp:202-321), computed in
// x87 long double and rounded once: the spectral-factor roots (a_p, c_p) at unit
// lengthscale, the unit-variance Pinf = s0 G(inf) and s0 = 1/k0.  G(inf) =
// ∫_0^inf e^{Au} g g^T e^{A^T u} du in closed form (2x2 blocks
// ½ [[C- + C+, S- - S+], [-(S+ + S-), C- - C+]], C± + i S± = -1/(α + iβ±),
// α = a_p + a_q, β± = c_p ± c_q) — the exact solution of the reference's Lyapunov
// equation (matexp.hpp:37-52).  The EQ Pinf is ill-conditioned (cond ~1e6 at order 6)
// and k0 = H G H^T cancels by ~1e4, so double-precision constants would perturb the
// small eigen-directions of every Q̃ well above the fp64 floor of the reference.
struct EqConst {
    std::vector<double> H;   // emission row (partial-fraction residues)
    std::vector<double> ac;  // a_0, c_0, a_1, c_1, ...
    std::vector<double> P1;  // J x J
    double s0 = 0.0;
};
EqConst eq_constants(int J) {
    using R = long double;
    using C = std::complex<R>;
    // roots of T_J(J z) J!/J^J (Weierstrass iteration), then 4+ Newton steps on T_J
    std::vector<R> c(J);
    for (int k = 0; k < J; ++k) {
        R v = 1;
        for (int i = k + 1; i <= J; ++i) v *= R(i);
        c[k] = v / std::pow(R(J), R(J - k));
    }
    auto poly = [&](C z) {
        C s = 1;
        for (int k = J - 1; k >= 0; --k) s = s * z + c[k];
        return s;
    };
    std::vector<C> z(J);
    for (int k = 0; k < J; ++k) z[k] = std::pow(C(0.4L, 0.9L), k);
    for (int it = 0; it < 2000; ++it) {
        R ch = 0;
        for (int k = 0; k < J; ++k) {
            C den = 1;
            for (int m = 0; m < J; ++m)
                if (m != k) den *= (z[k] - z[m]);
            const C st = poly(z[k]) / den;
            z[k] -= st;
            ch = std::max(ch, std::abs(st));
        }
        if (ch < 1e-19L) break;
    }
    std::vector<C> roots;
    for (int k = 0; k < J; ++k) {
        C y = z[k] * R(J);
        for (int it = 0; it < 8; ++it) {
            C t = 1, tp = 0, term = 1;
            for (int i = 1; i <= J; ++i) {
                tp += term;
                term *= y / R(i);
                t += term;
            }
            if (std::abs(tp) == 0) break;
            y -= t / tp;
        }
        C r = std::sqrt(R(-2) * y);
        if (r.real() > 0) r = -r;
        roots.push_back(r);
    }
    std::vector<C> up;
    for (C r : roots)
        if (r.imag() > 0) up.push_back(r);
    if (2 * up.size() != roots.size()) throw std::runtime_error("eq kernel: roots did not split into conjugate pairs");
    std::sort(up.begin(), up.end(),
              [](C a, C b) { return a.real() != b.real() ? a.real() < b.real() : a.imag() < b.imag(); });
    std::vector<R> H(J), G(static_cast<size_t>(J) * J);
    for (size_t p = 0; p < up.size(); ++p) {
        C den = 1;
        for (C o : roots)
            if (std::abs(o - up[p]) > 1e-12L) den *= (up[p] - o);
        const C res = C(1) / den;
        H[2 * p] = 2 * res.real();
        H[2 * p + 1] = 2 * res.imag();
    }
    auto inv = [](R a, R b, R& re, R& im) {
        const R d = a * a + b * b;
        re = -a / d;
        im = b / d;
    };
    for (int p = 0; p < J / 2; ++p)
        for (int q = 0; q < J / 2; ++q) {
            const R al = up[p].real() + up[q].real();
            R cm, sm, cp, sp;
            inv(al, up[p].imag() - up[q].imag(), cm, sm);
            inv(al, up[p].imag() + up[q].imag(), cp, sp);
            G[(2 * p) * J + 2 * q] = (cm + cp) / 2;
            G[(2 * p) * J + 2 * q + 1] = (sm - sp) / 2;
            G[(2 * p + 1) * J + 2 * q] = -(sp + sm) / 2;
            G[(2 * p + 1) * J + 2 * q + 1] = (cm - cp) / 2;
        }
    R k0 = 0;
    for (int i = 0; i < J; ++i)
        for (int j = 0; j < J; ++j) k0 += H[i] * G[i * J + j] * H[j];
    EqConst out;
    for (R v : H) out.H.push_back(static_cast<double>(v));
    for (const C& r : up) {
        out.ac.push_back(static_cast<double>(r.real()));
        out.ac.push_back(static_cast<double>(r.imag()));
    }
    const R s0 = R(1) / k0;
    for (R v : G) out.P1.push_back(static_cast<double>(v * s0));
    out.s0 = static_cast<double>(s0);
    return out;
}

int leaf_dim(const spingp_leaf& l) {
    switch (l.type) {
        case SPINGP_MATERN12: return 1;
        case SPINGP_MATERN32: return 2;
        case SPINGP_MATERN52: return 3;
        case SPINGP_EQ: return l.order;
        case SPINGP_QP: return 2 * (l.order + 1);
    }
    throw std::invalid_argument("unknown kernel leaf type");
}
int leaf_np(const spingp_leaf& l) { return l.type == SPINGP_QP ? 4 : 2; }

spingp::KernelSpec spec_of(const spingp_leaf* leaves, int32_t n_leaves) {
    std::vector<spingp::KernelSpec> parts;
    for (int i = 0; i < n_leaves; ++i) {
        const spingp_leaf& l = leaves[i];
        switch (l.type) {
            case SPINGP_MATERN12: parts.push_back(spingp::KernelSpec::matern12()); break;
            case SPINGP_MATERN32: parts.push_back(spingp::KernelSpec::matern32()); break;
            case SPINGP_MATERN52: parts.push_back(spingp::KernelSpec::matern52()); break;
            case SPINGP_EQ: parts.push_back(spingp::KernelSpec::eq(1.0, 1.0, l.order)); break;
            case SPINGP_QP: parts.push_back(spingp::KernelSpec::quasi_periodic(1.0, 1.0, 1.0, 1.0, l.order)); break;
            default: throw std::invalid_argument("unknown kernel leaf type");
        }
    }
    if (parts.empty()) throw std::invalid_argument("kernel has no leaves");
    if (parts.size() == 1) return parts[0];
    return spingp::KernelSpec::sum(parts);
}

}  // namespace

HostModel build_model(const spingp_leaf* leaves, int32_t n_leaves, int32_t n_theta) {
    if (!leaves || n_leaves < 1) throw std::invalid_argument("kernel has no leaves");
    if (n_leaves > kMaxLeaves) throw ApiError{SPINGP_UNSUPPORTED, -1, "too many kernel leaves"};
    HostModel hm;
    ModelDesc& d = hm.desc;
    int off = 0, th = 0, rec = 0;
    for (int l = 0; l < n_leaves; ++l) {
        const spingp_leaf& lf = leaves[l];
        if (lf.type == SPINGP_EQ && (lf.order < 2 || lf.order % 2 || lf.order > 16))
            throw std::invalid_argument("eq approximation order must be even and in [2, 16]");
        if (lf.type == SPINGP_QP && (lf.order < 0 || lf.order > 15))
            throw std::invalid_argument("qp harmonics must be in [0, 15]");
        d.type[l] = lf.type;
        d.off[l] = off;
        d.dim[l] = leaf_dim(lf);
        d.order[l] = lf.order;
        d.th[l] = th;
        off += d.dim[l];
        th += leaf_np(lf);
    }
    if (n_theta != th) throw std::invalid_argument("theta size does not match kernel parameter count");
    if (off > kMaxB) throw ApiError{SPINGP_UNSUPPORTED, -1, "state dimension above 16 is not built"};
    hm.b = off;
    hm.nt = th;
    d.b = off;
    d.nleaves = n_leaves;
    d.nt = th;
    std::vector<std::pair<int, std::vector<double>>> eq_h;
    rec = 2 + th;
    for (int l = 0; l < n_leaves; ++l) {
        d.rec[l] = rec;
        switch (leaves[l].type) {
            case SPINGP_MATERN12: case SPINGP_MATERN32: case SPINGP_MATERN52: rec += 5; break;  // var, len, lam, 1/len, 1/var
            case SPINGP_EQ: rec += 4; break;  // var, len, 1/len, 1/var
            case SPINGP_QP: rec += 7 + 2 * (leaves[l].order + 1); break;  // + 1/env, w0/period
        }
        d.eqc[l] = 0;
        if (leaves[l].type == SPINGP_EQ) {
            // unit variance / unit lengthscale model: roots (a, c) and P1
            const int J = leaves[l].order;
            const EqConst ec = eq_constants(J);
            eq_h.emplace_back(l, ec.H);
            d.eqc[l] = static_cast<int>(hm.eqconst.size());
            hm.eqconst.insert(hm.eqconst.end(), ec.ac.begin(), ec.ac.end());
            hm.eqconst.insert(hm.eqconst.end(), ec.P1.begin(), ec.P1.end());
            hm.eqconst.push_back(ec.s0);
        }
    }
    hm.rec_stride = rec;
    d.rec_stride = rec;
    // emission row
    const auto ssm = spingp::state_space_of(spec_of(leaves, n_leaves), spingp::default_theta(spec_of(leaves, n_leaves)));
    for (int i = 0; i < kMaxB; ++i) d.H[i] = i < hm.b ? ssm.H(i) : 0.0;
    for (const auto& [l, Hl] : eq_h)  // EQ emission rows from the extended-precision constants
        for (size_t i = 0; i < Hl.size(); ++i) d.H[d.off[l] + i] = Hl[i];
    hm.single_matern = n_leaves == 1 && leaves[0].type <= SPINGP_MATERN52;
    return hm;
}

// Per-series record (see model_dev.cuh): sigma, jitter, d jitter/dθ, leaf records.
void fill_record(const HostModel& hm, const double* theta, double sigma, double* r) {
    if (!(sigma > 0.0)) throw std::invalid_argument("sigma must be positive");  // +inf: no observation term
    const ModelDesc& d = hm.desc;
    const double b = hm.b;
    double tr = 0.0;
    std::vector<double> dtr(hm.nt, 0.0);
    for (int l = 0; l < d.nleaves; ++l) {
        const double* th = theta + d.th[l];
        const char* nm[4] = {"var", "len", "period", "env"};
        for (int p = 0; p < (d.type[l] == QP ? 4 : 2); ++p)
            if (!(th[p] > 0.0) || !std::isfinite(th[p]))
                throw std::invalid_argument(std::string("hyperparameter must be positive: ") + nm[p]);
        const double var = th[0], len = th[1];
        double* lr = r + d.rec[l];
        switch (d.type[l]) {
            case MATERN12: case MATERN32: case MATERN52: {
                const double lam = d.type[l] == MATERN12 ? 1.0 / len
                                   : d.type[l] == MATERN32 ? std::sqrt(3.0) / len
                                                           : std::sqrt(5.0) / len;
                lr[0] = var; lr[1] = len; lr[2] = lam;
                lr[3] = 1.0 / len; lr[4] = 1.0 / var;  // the per-step gradient needs no division
                // Pinf diagonal: var * (1, lam^2, lam^4 / ...) as in kernels.hpp:137-200
                double pd[3] = {var, 0.0, 0.0};
                if (d.type[l] == MATERN32) pd[1] = var * lam * lam;
                if (d.type[l] == MATERN52) {
                    pd[1] = var * lam * lam / 3.0;
                    pd[2] = var * lam * lam * lam * lam;
                }
                for (int i = 0; i < d.dim[l]; ++i) {
                    tr += pd[i];
                    dtr[d.th[l]] += pd[i] / var;
                    dtr[d.th[l] + 1] += -(2.0 * i) / len * pd[i];
                }
                break;
            }
            case EQ: {
                lr[0] = var; lr[1] = len;
                lr[2] = 1.0 / len; lr[3] = 1.0 / var;
                const int J = d.dim[l];
                const double* P1 = hm.eqconst.data() + d.eqc[l] + J;
                for (int i = 0; i < J; ++i) {
                    tr += var * P1[i * J + i];
                    dtr[d.th[l]] += P1[i * J + i];
                }
                break;
            }
            case QP: {
                const double period = th[2], env = th[3];
                const int J = d.order[l];
                lr[0] = var; lr[1] = len; lr[2] = period; lr[3] = env;
                lr[4] = 2.0 * std::numbers::pi / period;
                lr[5 + 2 * (J + 1)] = 1.0 / env;        // per-step code multiplies, never divides
                lr[5 + 2 * (J + 1) + 1] = lr[4] / period;
                const double x = 1.0 / (len * len), ex = std::exp(-x);
                for (int j = 0; j <= J; ++j) {
                    const double cj = j == 0 ? 1.0 : 2.0;
                    const double ij = std::cyl_bessel_i(double(j), x);
                    const double ip = j == 0 ? std::cyl_bessel_i(1.0, x)
                                             : 0.5 * (std::cyl_bessel_i(double(j - 1), x) +
                                                      std::cyl_bessel_i(double(j + 1), x));
                    const double q2 = cj * ij * ex;
                    const double dq2 = cj * ex * (ip - ij) * (-2.0 / (len * len * len));
                    lr[5 + j] = q2;
                    lr[5 + J + 1 + j] = dq2;
                    tr += 2.0 * var * q2;
                    dtr[d.th[l]] += 2.0 * q2;
                    dtr[d.th[l] + 1] += 2.0 * var * dq2;
                }
                break;
            }
        }
    }
    r[0] = sigma;
    r[1] = 1e-10 * tr / b;
    for (int p = 0; p < hm.nt; ++p) r[2 + p] = 1e-10 * dtr[p] / b;
}

// Padded block sizes with kernel instantiations (padding states are exactly
// decoupled, see model_dev.cuh GenericTraits).
int pad_b(int b) {
    static const int sizes[] = {1, 2, 3, 4, 6, 8, 12, 16};
    for (int s : sizes)
        if (b <= s) return s;
    throw ApiError{SPINGP_UNSUPPORTED, -1, "state dimension above 16 is not built"};
}

// Level 0: enough chunks to give every one of the 148 SMs ~256 resident threads
// (b <= 3) or ~128 (larger blocks); upper levels: chunks of 8 blocks until one
// block is left.
StaticModel static_model(const HostModel& hm) {
    const spingp_dev::ModelDesc& d = hm.desc;
    if (d.nleaves == 1 && d.type[0] == EQ && d.order[0] == 6) return SM_EQ6;
    if (d.nleaves == 1 && d.type[0] == EQ && d.order[0] == 10) return SM_EQ10;
    if (d.nleaves == 2 && d.type[0] == MATERN32 && d.type[1] == QP && d.order[1] == 6) return SM_M32_QP6;
    if (d.nleaves == 2 && d.type[0] == MATERN32 && d.type[1] == EQ && d.order[1] == 10) return SM_M32_EQ10;
    return SM_NONE;
}

PredictGrid predict_grid(const double* t, const double* y, int64_t n, const double* test_t, int64_t m) {
    if (n < 1 || m < 0 || !t || !y || (m > 0 && !test_t)) throw std::invalid_argument("bad predict arguments");
    for (int64_t k = 0; k < m; ++k)
        if (!std::isfinite(test_t[k])) throw std::invalid_argument("test times must be finite");
    std::vector<int64_t> ord(static_cast<size_t>(m));
    for (int64_t k = 0; k < m; ++k) ord[static_cast<size_t>(k)] = k;
    std::stable_sort(ord.begin(), ord.end(), [&](int64_t a, int64_t b) { return test_t[a] < test_t[b]; });
    double lo = t[0], hi = t[n - 1];
    if (m) {
        lo = std::min(lo, test_t[ord.front()]);
        hi = std::max(hi, test_t[ord.back()]);
    }
    const double eps = 1e-9 * (hi > lo ? hi - lo : 1.0);
    PredictGrid g;
    const size_t L = static_cast<size_t>(n + m);
    g.t.reserve(L);
    g.y.reserve(L);
    g.obs.reserve(L);
    g.test_pos.assign(static_cast<size_t>(m), -1);
    int64_t i = 0, k = 0;
    while (i < n || k < m) {
        // training point first on ties: the test point is then nudged past it
        const bool take_train = k >= m || (i < n && t[i] <= test_t[ord[static_cast<size_t>(k)]]);
        if (take_train) {
            if (!g.t.empty() && !(t[i] > g.t.back()))
                throw std::invalid_argument("a test time nudged by 1e-9 x span reaches the next training time");
            g.t.push_back(t[i]);
            g.y.push_back(y[i]);
            g.obs.push_back(1);
            ++i;
        } else {
            const int64_t kk = ord[static_cast<size_t>(k)];
            double tt = test_t[kk];
            if (!g.t.empty() && !(tt > g.t.back())) tt = g.t.back() + eps;
            g.test_pos[static_cast<size_t>(kk)] = static_cast<int64_t>(g.t.size());
            g.t.push_back(tt);
            g.y.push_back(0.0);
            g.obs.push_back(0);
            ++k;
        }
    }
    return g;
}

bool upper_tree() {
    static const bool t = [] {
        const char* e = std::getenv("SPINGP_UPPER");
        return !(e && (std::strcmp(e, "coop") == 0 || std::strcmp(e, "levels") == 0));
    }();
    return t;
}

namespace {
// resident threads of one k_rev0 wave at b = 3 (set from an occupancy query when a context
// is created, spingp_ctx_create -> set_plan_wave; 296 x 128 = 2 CTAs x 148 SMs on a B200)
std::atomic<int64_t> g_wave{296 * 128};
}  // namespace

void set_plan_wave(int64_t threads) {
    if (threads > 0) g_wave.store(threads);
}

Plan make_plan(int64_t n, int64_t S, int Bsz, int64_t m0_override, int tree, int64_t g_override) {
    if (n < 1 || S < 1) throw std::invalid_argument("need at least one point and one series");
    Plan p;
    // b >= 6: one thread per b x b merge is too long a chain for the tree's single-thread
    // top rounds (measured on B200: cfg4 45.9 vs 33.9 ms, cfg5 811 vs 385 ms per 1M/200k
    // points); those sizes keep the cooperative per-thread levels
    // (measured with the tree built for b >= 6 too: cfg4 17.6 vs 15.7 ms, cfg5 737 vs
    // 337 ms at 1 M points; the tree kernels are now only instantiated for b <= 4)
    p.tree = (tree < 0 ? upper_tree() : tree != 0) && Bsz <= 4;
    Geom& g = p.geo;
    g.S = static_cast<int>(S);
    // level-0 chunk count: enough threads to fill every SM (tuned on B200);
    // SPINGP_CHUNKS overrides it for tuning experiments
    static const int64_t env_target = [] {
        const char* e = std::getenv("SPINGP_CHUNKS");
        return e ? std::atoll(e) : 0LL;
    }();
    const int64_t target = env_target > 0 ? env_target : 75776;
    int64_t m0 = m0_override > 0 ? m0_override : std::max<int64_t>(8, (n * S + target - 1) / target);
    m0 = std::max<int64_t>(1, std::min<int64_t>(m0, n));
    // Wave quantisation of k_rev0 (b = 3: 2 CTAs of 128 threads per SM, 296 resident on
    // a B200): a plan a few CTAs past a full wave pays a whole extra wave, so lengthen the
    // chunks until the last wave is full (cfg3: 608 -> 576 CTAs, 2.26 -> 1.81 ms per step).
    if (m0_override <= 0 && env_target <= 0 && Bsz == 3) {
        const int64_t kWave = g_wave.load();
        const auto chunks = [&](int64_t m) { return S * ((n + m - 1) / m); };
        const int64_t w = chunks(m0) / kWave, rem = chunks(m0) % kWave;
        if (w >= 1 && rem > 0 && rem < kWave / 4)
            while (m0 < n && chunks(m0) > w * kWave) ++m0;
    }
    const int64_t G = g_override >= 2 ? std::min<int64_t>(g_override, tree_group_size(Bsz)) : tree_group_size(Bsz);
    int lev = 0;
    int64_t cur = n, m = m0;
    while (true) {
        if (lev >= kMaxLev) throw ApiError{SPINGP_UNSUPPORTED, -1, "too many reduction levels"};
        if (lev > 0) m = p.tree ? std::min(cur, G) : (cur <= 8 ? cur : 4);
        if (m < 2 && cur > 1) m = 2;
        g.n[lev] = cur;
        g.m[lev] = static_cast<int>(m);
        g.K[lev] = (cur + m - 1) / m;
        cur = g.K[lev];
        ++lev;
        // the tree path always ends with a tree level (its top group holds the inverse)
        if (cur == 1 && (!p.tree || lev > 1)) break;
    }
    g.nlev = lev;
    g.n[lev] = 1;
    return p;
}

}  // namespace spingp_host

using namespace spingp_host;

namespace {
thread_local std::string g_host_error;
template <class F>
int host_guarded(F&& body) {
    try {
        return body();
    } catch (const ApiError& e) {
        g_host_error = e.what;
        return e.status;
    } catch (const std::invalid_argument& e) {
        g_host_error = e.what();
        return SPINGP_BAD_ARG;
    } catch (const std::exception& e) {
        g_host_error = e.what();
        return SPINGP_UNSUPPORTED;
    }
}
}  // namespace

extern "C" {

int spingp_kernel_dims(const spingp_leaf* leaves, int32_t n_leaves, int32_t* b, int32_t* n_theta) {
    return host_guarded([&] {
        if (!leaves || n_leaves < 1) throw std::invalid_argument("kernel has no leaves");
        int bb = 0, nt = 0;
        for (int i = 0; i < n_leaves; ++i) {
            bb += leaf_dim(leaves[i]);
            nt += leaf_np(leaves[i]);
        }
        if (b) *b = bb;
        if (n_theta) *n_theta = nt;
        return SPINGP_OK;
    });
}

int spingp_state_space(const spingp_leaf* leaves, int32_t n_leaves, const double* theta,
                       int32_t n_theta, double* F, double* H, double* Pinf, double* dF,
                       double* dPinf, int32_t* f_constant) {
    return host_guarded([&] {
        const auto spec = spec_of(leaves, n_leaves);
        if (static_cast<size_t>(n_theta) != spingp::param_count(spec))
            throw std::invalid_argument("theta size does not match kernel parameter count");
        const auto m = spingp::state_space_of(spec, std::vector<double>(theta, theta + n_theta));
        const auto b = m.dim();
        if (F) std::memcpy(F, m.F.data(), sizeof(double) * b * b);
        if (H) std::memcpy(H, m.H.data(), sizeof(double) * b);
        if (Pinf) std::memcpy(Pinf, m.Pinf.data(), sizeof(double) * b * b);
        for (size_t p = 0; p < m.theta.size(); ++p) {
            if (dF) std::memcpy(dF + p * b * b, m.theta[p].dF.data(), sizeof(double) * b * b);
            if (dPinf) std::memcpy(dPinf + p * b * b, m.theta[p].dPinf.data(), sizeof(double) * b * b);
            if (f_constant) f_constant[p] = m.theta[p].f_constant ? 1 : 0;
        }
        return SPINGP_OK;
    });
}

}  // extern "C"
