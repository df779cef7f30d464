// emu.cpp — host emulation of the product's evaluation and btd_core pipelines,
// running the SAME kernel code (engine.cuh) on the CPU thread by thread.
// TEST INFRASTRUCTURE ONLY: lets the CPU test suite check the device algorithm
// (partitioned elimination, selected inverse, fused gradient) against the oracle
// without a GPU.  The product never links this.
#include "cuda_host_emu.h"

#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../paper_1610_08035_b200/csrc/engine.cuh"
#include "../../paper_1610_08035_b200/csrc/tree.cuh"
#include "../../paper_1610_08035_b200/csrc/host_model.hpp"

using namespace spingp_dev;
using namespace spingp_host;

namespace {

std::string g_err;
int64_t g_tree_group = 0;  // emu_set_tree_group
const unsigned char* g_obs = nullptr;  // emu_set_obs: observation mask of the next eval (S = 1)
unsigned long long g_status;
double g_diag[4];  // logdetP, logdetQ, fit_y, fit_e of the last series evaluated

unsigned nblocks(long long n, int tpb) { return static_cast<unsigned>((n + tpb - 1) / tpb); }

// ------------------------------------------------------------ tree levels (tree.cuh) --
// The CTA of k_tree_fwd / k_tree_rev / k_tree_one emulated phase by phase: every
// emulated thread runs a phase before any runs the next (the kernel's barriers).
enum EmuTree { EMU_FWD = 0, EMU_REV = 1, EMU_ONE = 2 };

template <int B>
TreeArgs emu_tree_args(const Geom& g, int l, std::vector<std::vector<double>>& rec, std::vector<std::vector<double>>& fac,
                       std::vector<std::vector<double>>& sol, std::vector<double>& top, bool needC) {
    TreeArgs ta{};
    ta.rec_in = rec[l - 1].data();
    ta.SKin = g.K[l - 1] * g.S;
    ta.nin = g.n[l];
    ta.rec_out = rec[l].data();
    ta.fac = fac[l].data();
    ta.solU = sol[l + 1].data();
    ta.sol = sol[l].data();
    ta.toplogdet = top.data();
    ta.status = &g_status;
    ta.G = g.m[l];
    ta.nG = static_cast<int>(g.K[l]);
    ta.S = g.S;
    ta.segL = g.segL;
    ta.needC = needC ? 1 : 0;
    const long long gcap = std::min<long long>(g.m[l], g.n[l]);
    ta.RS = static_cast<int>(tree_row(gcap));
    ta.ES = static_cast<int>(tree_row(gcap + 1));
    ta.span = 1;
    for (int i = 1; i < l; ++i) ta.span *= g.m[i];
    ta.K0 = g.K[0];
    ta.n0 = g.n[0];
    ta.m0 = g.m[0];
    return ta;
}

template <int B>
void emu_tree(EmuTree kind, const TreeArgs& ta) {
    using TR = Tree<B>;
    std::vector<double> sm(static_cast<size_t>(TR::NR) * ta.RS + static_cast<size_t>(TR::NS) * ta.ES, std::nan(""));
    double* R = sm.data();
    double* E = R + static_cast<size_t>(TR::NR) * ta.RS;
    const int nt = std::max(1, (std::min(ta.G, ta.RS) + 1) / 2);  // one node per thread per round
    std::vector<TreeFwdScratch<B>> fs(nt);
    std::vector<TreeRevScratch<B>> rs(nt);
    const bool needC = ta.needC != 0;
    for (long long gidx = 0; gidx < static_cast<long long>(ta.S) * ta.nG; ++gidx) {
        const TreeGroup t = tree_group(ta, gidx);
        auto all = [&](auto&& f) {
            for (int tid = 0; tid < nt; ++tid) f(tid);
        };
        const int J = tree_levels(t.cnt);
        if (kind != EMU_REV) {
            all([&](int tid) { tree_load_recs<B>(ta, t, R, tid, nt); });
            for (int j = 0; j < J; ++j) {
                const int n = tree_width(t.cnt, j);
                all([&](int tid) {
                    tree_fwd_compute<B>(R, ta.RS, n, tid, fs[tid]);
                    if (!fs[tid].ok) report(ta.status, tree_point(ta, t, t.k0 + std::min(t.cnt, (2 * tid + 1) << j) - 1), ST_NOT_PD);
                });
                all([&](int tid) { tree_fwd_store<B>(R, ta.RS, n, tid, fs[tid]); });
            }
        }
        if (kind == EMU_FWD) {
            all([&](int tid) { tree_store_fwd<B>(ta, t, R, tid, nt); });
            continue;
        }
        if (kind == EMU_ONE) tree_top<B>(ta, t, R, E);
        else all([&](int tid) { tree_load_rev<B>(ta, t, R, E, tid, nt); });
        for (int j = J - 1; j >= 0; --j) {
            const int n = tree_width(t.cnt, j);
            all([&](int tid) { tree_rev_compute<B>(R, E, ta.RS, ta.ES, n, tid, needC, rs[tid]); });
            all([&](int tid) { tree_rev_store<B>(E, ta.ES, n, tid, needC, rs[tid]); });
        }
        all([&](int tid) { tree_store_rev<B>(ta, t, E, tid, nt); });
    }
}

// fac[l] sized for the tree factors at levels >= 1
template <int B>
size_t emu_fac_size(const Geom& g, int l) {
    return static_cast<size_t>(g.m[l]) * (l ? Tree<B>::NF : Fac<B>::N) * g.K[l] * g.S;
}

template <class T>
void emu_eval(const HostModel& hm, const Plan& plan, std::vector<double>& params, const double* t,
              const double* y, uint32_t flags, double* loglik, double* grad, double* mean, double* var) {
    constexpr int B = T::B;
    const Geom& g = plan.geo;
    const int nt = hm.nt;
    std::vector<double> eqc = hm.eqconst;
    ModelDesc md = hm.desc;
    md.eqconst = eqc.data();
    std::vector<std::vector<double>> fac(g.nlev), rec(g.nlev), sol(g.nlev + 1);
    for (int l = 0; l < g.nlev; ++l) {
        const size_t SK = static_cast<size_t>(g.K[l]) * g.S;
        fac[l].assign(emu_fac_size<B>(g, l), 0.0);
        rec[l].assign(Rec<B>::N * SK, 0.0);
    }
    for (int l = 1; l <= g.nlev; ++l) sol[l].assign(Sol<B>::N * static_cast<size_t>(g.n[l]) * g.S, 0.0);
    std::vector<double> top(g.S, 0.0);
    const long long SK0 = g.K[0] * g.S;
    std::vector<double> part(static_cast<size_t>(P_GRAD + nt) * SK0, 0.0);
    const int tpb = 32;
    unsigned long long* st = &g_status;
    emu_launch(nblocks(SK0, tpb), tpb, [&] {
        k_fwd0<T>(md, params.data(), t, y, g, fac[0].data(), rec[0].data(), part.data(), st, nullptr, 0, SK0, g_obs);
    });
    const bool gr = flags & 1u, needC = gr || (flags & 4u);
    if (plan.tree) {
        for (int l = 1; l + 1 < g.nlev; ++l) emu_tree<B>(EMU_FWD, emu_tree_args<B>(g, l, rec, fac, sol, top, needC));
        emu_tree<B>(EMU_ONE, emu_tree_args<B>(g, g.nlev - 1, rec, fac, sol, top, needC));
        for (int l = g.nlev - 2; l >= 1; --l) emu_tree<B>(EMU_REV, emu_tree_args<B>(g, l, rec, fac, sol, top, needC));
    } else {
    for (int l = 1; l < g.nlev; ++l) {
        RecSource<B> src{rec[l - 1].data(), g.K[l - 1] * g.S, g.n[l]};
        emu_launch(nblocks(g.K[l] * g.S, tpb), tpb,
                   [&] { k_fwdL<B, RecSource<B>>(src, g, l, fac[l].data(), rec[l].data(), st); });
    }
    emu_launch(nblocks(g.S, tpb), tpb, [&] { k_top<B>(g, rec[g.nlev - 1].data(), sol[g.nlev].data(), top.data(), st); });
    for (int l = g.nlev - 1; l >= 1; --l) {
        RecSource<B> src{rec[l - 1].data(), g.K[l - 1] * g.S, g.n[l]};
        SolSink<B> sink{sol[l].data(), g.n[l] * g.S, g.n[l], 0};
        emu_launch(nblocks(g.K[l] * g.S, tpb), tpb, [&] {
            k_revL<B, RecSource<B>, SolSink<B>>(src, sink, g, l, fac[l].data(), sol[l + 1].data(), needC ? 1 : 0);
        });
    }
    }
    Outs outs{(flags & 2u) ? mean : nullptr, (flags & 4u) ? var : nullptr, (flags & 8u) ? 1 : 0, gr ? 1 : 0,
              needC ? 1 : 0};
    emu_launch(nblocks(SK0, tpb), tpb, [&] {
        k_rev0<T>(md, params.data(), t, y, g, fac[0].data(), sol[1].data(), part.data(), outs, st, nullptr, 0, SK0, g_obs);
    });
    for (int s = 0; s < g.S; ++s) {
        double acc[P_GRAD + kMaxTheta] = {};
        for (int c = 0; c < P_GRAD + nt; ++c)
            for (long long k = 0; k < g.K[0]; ++k) acc[c] += part[c * SK0 + s * g.K[0] + k];
        const double ld = top[s];  // cumulative records: the whole log-determinant
        g_diag[0] = ld;
        g_diag[1] = acc[P_LDQ];
        g_diag[2] = acc[P_FITY];
        g_diag[3] = acc[P_FITE];
        const double* rp = params.data() + static_cast<size_t>(s) * hm.rec_stride;
        long long nobs = g.n[0];
        if (g_obs) {
            nobs = 0;
            for (long long i = 0; i < g.n[0]; ++i) nobs += g_obs[s * g.n[0] + i] ? 1 : 0;
        }
        const double sig = rp[0], s2 = sig * sig, nn = static_cast<double>(nobs);
        loglik[s] = -0.5 * (acc[P_FITY] + acc[P_FITE]) - 0.5 * (ld + acc[P_LDQ] + nn * std::log(s2)) -
                    0.5 * nn * 1.8378770664093454835606594728112;
        if (gr) {
            for (int p = 0; p < nt; ++p) grad[s * (nt + 1) + p] = acc[P_GRAD + p];
            grad[s * (nt + 1) + nt] = 2.0 * sig * (-0.5 * nn / s2 + acc[P_NOISE] / (2.0 * s2 * s2));
        }
    }
}

template <int B>
void emu_btd(int64_t n, int b, const double* diag, const double* upper, const double* rhs, int k, int col,
             double* x, double* cdiag, double* cupper, double* logdet, bool needC, int64_t m0) {
    const Plan plan = make_plan(n, 1, B, m0, 0);
    const Geom& g = plan.geo;
    std::vector<std::vector<double>> fac(g.nlev), rec(g.nlev), sol(g.nlev + 1);
    for (int l = 0; l < g.nlev; ++l) {
        fac[l].assign(static_cast<size_t>(g.m[l]) * Fac<B>::N * g.K[l], 0.0);
        rec[l].assign(Rec<B>::N * g.K[l], 0.0);
    }
    for (int l = 1; l <= g.nlev; ++l) sol[l].assign(Sol<B>::N * static_cast<size_t>(g.n[l]), 0.0);
    std::vector<double> top(1, 0.0);
    unsigned long long* st = &g_status;
    const int tpb = 32;
    UserSource<B> usrc{diag, upper, rhs, n, b, k, col};
    emu_launch(nblocks(g.K[0], tpb), tpb, [&] { k_fwdL<B, UserSource<B>>(usrc, g, 0, fac[0].data(), rec[0].data(), st); });
    for (int l = 1; l < g.nlev; ++l) {
        RecSource<B> src{rec[l - 1].data(), g.K[l - 1], g.n[l]};
        emu_launch(nblocks(g.K[l], tpb), tpb, [&] { k_fwdL<B, RecSource<B>>(src, g, l, fac[l].data(), rec[l].data(), st); });
    }
    emu_launch(1, 1, [&] { k_top<B>(g, rec[g.nlev - 1].data(), sol[g.nlev].data(), top.data(), st); });
    for (int l = g.nlev - 1; l >= 1; --l) {
        RecSource<B> src{rec[l - 1].data(), g.K[l - 1], g.n[l]};
        SolSink<B> sink{sol[l].data(), g.n[l], g.n[l], 0};
        emu_launch(nblocks(g.K[l], tpb), tpb, [&] {
            k_revL<B, RecSource<B>, SolSink<B>>(src, sink, g, l, fac[l].data(), sol[l + 1].data(), needC ? 1 : 0);
        });
    }
    UserSink<B> usink{x, cdiag, cupper, b, k, col};
    emu_launch(nblocks(g.K[0], tpb), tpb, [&] {
        k_revL<B, UserSource<B>, UserSink<B>>(usrc, usink, g, 0, fac[0].data(), sol[1].data(), needC ? 1 : 0);
    });
    if (logdet) *logdet = top[0];  // cumulative records
}

// ---------------------------------------------------------------- segment mode ----
// Multi-rank partition of one series (one rank per process or emulated in turn).
struct SegStateBase {
    virtual ~SegStateBase() = default;
    virtual void forward(double* record) = 0;
    virtual void reverse(const double* records, double* partials, double* mean, double* var) = 0;
};

template <class T>
struct SegState : SegStateBase {
    static constexpr int B = T::B;
    HostModel hm;
    Plan plan;
    std::vector<double> params, eqc;
    const double* t;
    const double* y;
    uint32_t flags;
    int rank, nranks;
    ModelDesc md;
    std::vector<std::vector<double>> fac, rec, sol;
    std::vector<double> part, top;
    SegState(const HostModel& h, const Plan& p, std::vector<double> prm, const double* tt, const double* yy,
             uint32_t fl, int r, int P)
        : hm(h), plan(p), params(std::move(prm)), t(tt), y(yy), flags(fl), rank(r), nranks(P) {
        eqc = hm.eqconst;
        md = hm.desc;
        md.eqconst = eqc.data();
        const Geom& g = plan.geo;
        fac.resize(g.nlev);
        rec.resize(g.nlev);
        sol.resize(g.nlev + 1);
        for (int l = 0; l < g.nlev; ++l) {
            fac[l].assign(emu_fac_size<B>(g, l), 0.0);
            rec[l].assign(Rec<B>::N * g.K[l], 0.0);
        }
        for (int l = 1; l <= g.nlev; ++l) sol[l].assign(Sol<B>::N * static_cast<size_t>(g.n[l] + g.segL), 0.0);
        part.assign(static_cast<size_t>(P_GRAD + hm.nt) * g.K[0], 0.0);
        top.assign(1, 0.0);
    }
    const double* halo() const { return params.data() + hm.rec_stride; }
    void forward(double* record) override {
        const Geom& g = plan.geo;
        unsigned long long* st = &g_status;
        emu_launch(nblocks(g.K[0], 32), 32, [&] {
            k_fwd0<T>(md, params.data(), t, y, g, fac[0].data(), rec[0].data(), part.data(), st, halo(), 0, g.K[0], nullptr);
        });
        for (int l = 1; l < g.nlev; ++l) {
            if (plan.tree) {
                emu_tree<B>(EMU_FWD, emu_tree_args<B>(g, l, rec, fac, sol, top, false));
                continue;
            }
            RecSource<B> src{rec[l - 1].data(), g.K[l - 1], g.n[l]};
            emu_launch(nblocks(g.K[l], 32), 32, [&] { k_fwdL<B, RecSource<B>>(src, g, l, fac[l].data(), rec[l].data(), st); });
        }
        std::copy(rec[g.nlev - 1].begin(), rec[g.nlev - 1].begin() + Rec<B>::N, record);
    }
    void reverse(const double* records, double* partials, double* mean, double* var) override {
        const Geom& g = plan.geo;
        unsigned long long* st = &g_status;
        std::vector<double> scratch(64 * (2 * B * B + B));
        emu_launch(1, 1, [&] { k_seg_solve<B>(nranks, rank, records, sol[g.nlev].data(), top.data(), st, 0, scratch.data()); });
        const bool gr = flags & 1u, needC = gr || (flags & 4u);
        for (int l = g.nlev - 1; l >= 1; --l) {
            if (plan.tree) {
                emu_tree<B>(EMU_REV, emu_tree_args<B>(g, l, rec, fac, sol, top, needC));
                continue;
            }
            RecSource<B> src{rec[l - 1].data(), g.K[l - 1], g.n[l]};
            SolSink<B> sink{sol[l].data(), g.n[l] + g.segL, g.n[l], g.segL};
            emu_launch(nblocks(g.K[l], 32), 32, [&] {
                k_revL<B, RecSource<B>, SolSink<B>>(src, sink, g, l, fac[l].data(), sol[l + 1].data(), needC ? 1 : 0);
            });
        }
        Outs outs{(flags & 2u) ? mean : nullptr, (flags & 4u) ? var : nullptr, (flags & 8u) ? 1 : 0, gr ? 1 : 0,
                  needC ? 1 : 0};
        emu_launch(nblocks(g.K[0], 32), 32, [&] {
            k_rev0<T>(md, params.data(), t, y, g, fac[0].data(), sol[1].data(), part.data(), outs, st, halo(), 0, g.K[0], nullptr);
        });
        const int NC = P_GRAD + hm.nt;
        for (int c = 0; c < NC; ++c) {
            double acc = 0.0;
            for (long long k = 0; k < g.K[0]; ++k) acc += part[c * g.K[0] + k];
            partials[c] = acc;
        }
        partials[P_LOGDET] = top[0];
    }
};

std::unique_ptr<SegStateBase> g_seg;

int finish() {
    if (g_status == ~0ULL) return SPINGP_OK;
    return static_cast<int>(g_status & 15ULL);
}

}  // namespace

extern "C" {

const char* emu_last_error(void) { return g_err.c_str(); }
void emu_set_tree_group(int64_t g) { g_tree_group = g; }
void emu_set_obs(const unsigned char* obs) { g_obs = obs; }

// The level structure make_plan gives (host logic shared with the library): nlev, tree
// flag, then per level n, m, K.
int emu_plan(int64_t n, int64_t S, int32_t Bsz, int64_t m0, int64_t* out, int32_t cap) {
    try {
        const Plan p = make_plan(n, S, Bsz, m0);
        const Geom& g = p.geo;
        if (cap < 2 + 3 * g.nlev) return SPINGP_BAD_ARG;
        out[0] = g.nlev;
        out[1] = p.tree ? 1 : 0;
        for (int l = 0; l < g.nlev; ++l) {
            out[2 + 3 * l] = g.n[l];
            out[3 + 3 * l] = g.m[l];
            out[4 + 3 * l] = g.K[l];
        }
        return SPINGP_OK;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SPINGP_BAD_ARG;
    }
}
void emu_last_diag(double* out) {
    for (int i = 0; i < 4; ++i) out[i] = g_diag[i];
}

int emu_eval_batched(const spingp_leaf* leaves, int32_t n_leaves, const double* theta, int32_t n_theta,
                     int64_t S, int64_t n, const double* t, const double* y, const double* sigma,
                     uint32_t flags, double* loglik, double* grad, double* mean, double* var,
                     int64_t* fail_block, int64_t m0, int force_generic) {
    g_status = ~0ULL;
    try {
        const HostModel hm = build_model(leaves, n_leaves, n_theta);
        const bool matern = hm.single_matern && !force_generic;
        const StaticModel sm = force_generic ? SM_NONE : static_model(hm);
        const int Bsz = (matern || sm != SM_NONE) ? hm.b : std::max(3, pad_b(hm.b));
        const Plan plan = make_plan(n, S, Bsz, m0, -1, g_tree_group);
        std::vector<double> params(static_cast<size_t>(S) * hm.rec_stride, 0.0);
        for (int64_t s = 0; s < S; ++s) fill_record(hm, theta + s * n_theta, sigma[s], params.data() + s * hm.rec_stride);
#define E(...) emu_eval<__VA_ARGS__>(hm, plan, params, t, y, flags, loglik, grad, mean, var)
        if (sm == SM_EQ6) E(StaticTraits<SEQ<6>>);
        else if (sm == SM_EQ10) E(StaticTraits<SEQ<10>>);
        else if (sm == SM_M32_QP6) E(StaticTraits<SMatern<2>, SQP<6>>);
        else if (sm == SM_M32_EQ10) E(StaticTraits<SMatern<2>, SEQ<10>>);
        else if (matern) {
            if (hm.b == 1) E(MaternTraits<1>);
            else if (hm.b == 2) E(MaternTraits<2>);
            else E(MaternTraits<3>);
        } else {
            switch (Bsz) {
                case 3: E(GenericTraits<3>); break;
                case 4: E(GenericTraits<4>); break;
                case 6: E(GenericTraits<6>); break;
                case 8: E(GenericTraits<8>); break;
                case 12: E(GenericTraits<12>); break;
                case 16: E(GenericTraits<16>); break;
            }
        }
#undef E
    } catch (const ApiError& e) {
        g_err = e.what;
        return e.status;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SPINGP_BAD_ARG;
    }
    if (fail_block) *fail_block = g_status == ~0ULL ? -1 : static_cast<int64_t>((g_status >> 4) & ((1ULL << 56) - 1));
    return finish();
}

// spingp_predict (capi.cu) on the host emulation: same grid merge, masked evaluation
int emu_predict(const spingp_leaf* leaves, int32_t n_leaves, const double* theta, int32_t n_theta, int64_t n,
                const double* t, const double* y, const double* test_t, int64_t m, double sigma, uint32_t flags,
                double* loglik, double* grad, double* mean, double* var, int64_t* fail_block, int64_t m0) {
    PredictGrid pg;
    try {
        pg = predict_grid(t, y, n, test_t, m);
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SPINGP_BAD_ARG;
    }
    const int64_t L = n + m;
    std::vector<double> mu(static_cast<size_t>(L)), v(static_cast<size_t>(L));
    g_obs = pg.obs.data();
    const uint32_t f = (flags & 9u) | 2u | 4u;
    const int st = emu_eval_batched(leaves, n_leaves, theta, n_theta, 1, L, pg.t.data(), pg.y.data(), &sigma, f, loglik,
                                    grad, mu.data(), v.data(), fail_block, m0, 0);
    g_obs = nullptr;
    for (int64_t k = 0; k < m; ++k) {
        mean[k] = mu[static_cast<size_t>(pg.test_pos[static_cast<size_t>(k)])];
        var[k] = v[static_cast<size_t>(pg.test_pos[static_cast<size_t>(k)])];
    }
    return st;
}

int emu_btd(int64_t n, int32_t b, const double* diag, const double* upper, const double* rhs, int32_t k,
            double* x, double* cdiag, double* cupper, double* logdet, int64_t* fail_block, int64_t m0) {
    g_status = ~0ULL;
    const bool needC = cdiag != nullptr;
    const int B = pad_b(b);
    for (int col = 0; col < (k > 0 ? k : 1); ++col) {
        double* ld = col == 0 ? logdet : nullptr;
        const double* r = k > 0 ? rhs : nullptr;
        double* xx = k > 0 ? x : nullptr;
        switch (B) {
            case 1: emu_btd<1>(n, b, diag, upper, r, k, col, xx, cdiag, cupper, ld, needC, m0); break;
            case 2: emu_btd<2>(n, b, diag, upper, r, k, col, xx, cdiag, cupper, ld, needC, m0); break;
            case 3: emu_btd<3>(n, b, diag, upper, r, k, col, xx, cdiag, cupper, ld, needC, m0); break;
            case 4: emu_btd<4>(n, b, diag, upper, r, k, col, xx, cdiag, cupper, ld, needC, m0); break;
            case 6: emu_btd<6>(n, b, diag, upper, r, k, col, xx, cdiag, cupper, ld, needC, m0); break;
            case 8: emu_btd<8>(n, b, diag, upper, r, k, col, xx, cdiag, cupper, ld, needC, m0); break;
            case 12: emu_btd<12>(n, b, diag, upper, r, k, col, xx, cdiag, cupper, ld, needC, m0); break;
            case 16: emu_btd<16>(n, b, diag, upper, r, k, col, xx, cdiag, cupper, ld, needC, m0); break;
        }
    }
    if (fail_block) *fail_block = g_status == ~0ULL ? -1 : static_cast<int64_t>(g_status >> 4);
    return finish();
}

// One step of the device discretisation (T::step) and its θ-derivatives (read
// back through T::grad with unit M / Bm probes):  Phi, Q (raw, no jitter),
// dPhi[nt][b][b], dQt[nt][b][b] (with the jitter derivative).  dt < 0 = anchor.
int emu_discretize(const spingp_leaf* leaves, int32_t n_leaves, const double* theta, int32_t n_theta,
                   double sigma, double dt, double* Phi, double* Q, double* dPhi, double* dQt, double* jit) {
    try {
        const HostModel hm = build_model(leaves, n_leaves, n_theta);
        std::vector<double> rec(hm.rec_stride);
        fill_record(hm, theta, sigma, rec.data());
        std::vector<double> eqc = hm.eqconst;
        ModelDesc md = hm.desc;
        md.eqconst = eqc.data();
        const int b = hm.b, nt = hm.nt;
        if (jit) *jit = rec[1];
        auto run = [&](auto tag) {
            using T = decltype(tag);
            constexpr int B = T::B;
            double P[B * B], Qq[B * B];
            T::step(md, rec.data(), dt, P, Qq);
            for (int i = 0; i < b; ++i)
                for (int j = 0; j < b; ++j) {
                    Phi[i * b + j] = P[i * B + j];
                    Q[i * b + j] = Qq[i * B + j];
                }
            if (!dPhi) return;
            for (int a = 0; a < b; ++a)
                for (int c = 0; c < b; ++c) {
                    double M[B * B] = {}, Bm[B * B] = {}, g[kMaxTheta] = {};
                    Bm[c * B + a] = 1.0;  // g = Tr(dPhi Bm) = dPhi[a][c]
                    T::grad(md, rec.data(), dt, P, Qq, M, Bm, g);
                    for (int p = 0; p < nt; ++p) dPhi[(p * b + a) * b + c] = g[p];
                    double M2[B * B] = {}, B2[B * B] = {}, g2[kMaxTheta] = {};
                    M2[a * B + c] += 1.0;
                    M2[c * B + a] += 1.0;  // g = ½Tr(M dQ) = dQ[a][c] (a != c) or dQ[a][a]
                    T::grad(md, rec.data(), dt, P, Qq, M2, B2, g2);
                    for (int p = 0; p < nt; ++p) dQt[(p * b + a) * b + c] = g2[p];
                }
        };
        if (hm.single_matern) {
            if (hm.b == 1) run(MaternTraits<1>{});
            else if (hm.b == 2) run(MaternTraits<2>{});
            else run(MaternTraits<3>{});
        } else {
            switch (std::max(3, pad_b(hm.b))) {
                case 3: run(GenericTraits<3>{}); break;
                case 4: run(GenericTraits<4>{}); break;
                case 6: run(GenericTraits<6>{}); break;
                case 8: run(GenericTraits<8>{}); break;
                case 12: run(GenericTraits<12>{}); break;
                case 16: run(GenericTraits<16>{}); break;
            }
        }
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return SPINGP_BAD_ARG;
    }
    return 0;
}

int emu_seg_forward(const spingp_leaf* leaves, int32_t n_leaves, const double* theta, int32_t n_theta,
                    const double* t, const double* y, int64_t n_local, double t_left, double t_right, int32_t rank,
                    int32_t nranks, double sigma, uint32_t flags, int64_t m0, double* record) {
    g_status = ~0ULL;
    try {
        const HostModel hm = build_model(leaves, n_leaves, n_theta);
        const StaticModel sm = static_model(hm);
        const int Bsz = (hm.single_matern || sm != SM_NONE) ? hm.b : std::max(3, pad_b(hm.b));
        Plan plan = make_plan(n_local, 1, Bsz, m0, -1, g_tree_group);
        plan.geo.segL = rank > 0;
        plan.geo.segR = rank + 1 < nranks;
        std::vector<double> params(hm.rec_stride + 2, 0.0);
        fill_record(hm, theta, sigma, params.data());
        params[hm.rec_stride] = t_left;
        params[hm.rec_stride + 1] = t_right;
#define MK(...) g_seg.reset(new SegState<__VA_ARGS__>(hm, plan, params, t, y, flags, rank, nranks))
        if (sm == SM_EQ6) MK(StaticTraits<SEQ<6>>);
        else if (sm == SM_M32_QP6) MK(StaticTraits<SMatern<2>, SQP<6>>);
        else if (hm.single_matern && hm.b == 1) MK(MaternTraits<1>);
        else if (hm.single_matern && hm.b == 2) MK(MaternTraits<2>);
        else if (hm.single_matern && hm.b == 3) MK(MaternTraits<3>);
        else if (Bsz == 3) MK(GenericTraits<3>);
        else if (Bsz == 4) MK(GenericTraits<4>);
        else if (Bsz == 6) MK(GenericTraits<6>);
        else if (Bsz == 8) MK(GenericTraits<8>);
        else if (Bsz == 12) MK(GenericTraits<12>);
        else MK(GenericTraits<16>);
#undef MK
        g_seg->forward(record);
    } catch (const std::exception& e) {
        g_err = e.what();
        return SPINGP_BAD_ARG;
    }
    return finish();
}

int emu_seg_sizes(const spingp_leaf* leaves, int32_t n_leaves, int32_t n_theta, int32_t* nrec, int32_t* npart) {
    try {
        const HostModel hm = build_model(leaves, n_leaves, n_theta);
        const int B = (hm.single_matern || static_model(hm) != SM_NONE) ? hm.b : std::max(3, pad_b(hm.b));
        *nrec = 3 * B * B + 2 * B + 1;
        *npart = 5 + hm.nt;
    } catch (const std::exception& e) {
        g_err = e.what();
        return SPINGP_BAD_ARG;
    }
    return 0;
}

int emu_seg_reverse(const double* records, double* partials, double* mean, double* var) {
    if (!g_seg) return SPINGP_BAD_ARG;
    g_seg->reverse(records, partials, mean, var);
    return finish();
}

}  // extern "C"
