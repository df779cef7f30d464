// spingp — the bench CLI of SPEC.md:417-503 (module bench_cli) over the B200 library.
//
// The reference ships this executable as a stub (proj/tools/spingp_cli.cpp, built as
// `spingp`, proj/tools/CMakeLists.txt:1-3); the SPEC defines its behaviour.  Host C++
// on the drop-in API (include/spingp/*.hpp -> libspingp_b200.so):
//
//   gen-data   --n N --seed S [--noise 0.2] --out DIR            SPEC.md:431-438 generate_sinusoid_data
//   fit        --kernel EXPR --data FILE [--budget 200] --out DIR     optimize_hyperparameters
//   predict    --kernel EXPR --data FILE --grid a:b:m --out DIR       predict at test times
//   scaling-n  --kernel EXPR --ns 1000,2000,... [--method spingp|kf|dense] [--repetitions 5] --out DIR
//   scaling-b  --bs 2,4,8,12,16 --n 1000 [--method ...] --out DIR     SPEC.md:462-468 (Σ Matérn-3/2 leaves, b = 2k)
//   co2        --data NOAA_FILE [--budget 200] --out DIR              SPEC.md:469-475 ingest + fit + 8-year forecast
//
// Kernel grammar: `matern32(var=1.0, len=2.5) + eq(var=1.0, len=100, order=10)`;
// leaves matern12|matern32|matern52|eq|qp (qp: var, len, period, env, order).
// Methods: spingp (the GPU path), kf (Kalman prediction-error decomposition)
// and dense (Cholesky of K + σ²I) — both host C++ here, MLL only.
// Outputs: report.csv (RFC-4180, header row), metrics.json (schema_version 1),
// forecast.csv.  Timing: median of >= 5 repetitions after 1 warm-up, steady_clock; slopes
// by least squares on (ln x, ln seconds).  Exit code nonzero iff a
// sub-run failed; partial results are still written.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <map>
#include <memory>
#include <random>
#include <sstream>
#include <string>
#include <sys/stat.h>
#include <vector>

#include "spingp/engine.hpp"
#include "spingp/optimize.hpp"

using namespace spingp;

namespace {

using Args = std::map<std::string, std::string>;

std::string arg(const Args& a, const std::string& k, const std::string& def = "") {
    auto it = a.find(k);
    if (it != a.end()) return it->second;
    if (def.empty()) throw std::invalid_argument("missing --" + k);
    return def;
}

std::vector<double> list_of(const std::string& s) {
    std::vector<double> v;
    std::stringstream ss(s);
    std::string tok;
    while (std::getline(ss, tok, ',')) v.push_back(std::stod(tok));
    return v;
}

// ------------------------------------------------------------------ grammar --
struct Parsed {
    KernelSpec spec;
    HyperparameterSet theta;
};

KernelSpec parse_leaf(const std::string& txt) {
    const auto lp = txt.find('('), rp = txt.rfind(')');
    std::string name = txt.substr(0, lp);
    name.erase(std::remove_if(name.begin(), name.end(), ::isspace), name.end());
    std::map<std::string, double> kv;
    if (lp != std::string::npos) {
        if (rp == std::string::npos || rp < lp) throw std::invalid_argument("unbalanced parentheses in '" + txt + "'");
        std::stringstream ss(txt.substr(lp + 1, rp - lp - 1));
        std::string item;
        while (std::getline(ss, item, ',')) {
            const auto eq = item.find('=');
            if (eq == std::string::npos) {
                if (item.find_first_not_of(" \t") == std::string::npos) continue;
                throw std::invalid_argument("expected key=value in '" + item + "'");
            }
            std::string k = item.substr(0, eq);
            k.erase(std::remove_if(k.begin(), k.end(), ::isspace), k.end());
            kv[k] = std::stod(item.substr(eq + 1));
        }
    }
    auto get = [&](const char* k, double d) { return kv.count(k) ? kv[k] : d; };
    if (name == "matern12") return KernelSpec::matern12(get("var", 1), get("len", 1));
    if (name == "matern32") return KernelSpec::matern32(get("var", 1), get("len", 1));
    if (name == "matern52") return KernelSpec::matern52(get("var", 1), get("len", 1));
    if (name == "eq") return KernelSpec::eq(get("var", 1), get("len", 1), static_cast<int>(get("order", 10)));
    if (name == "qp")
        return KernelSpec::quasi_periodic(get("var", 1), get("len", 1), get("period", 1), get("env", 1),
                                          static_cast<int>(get("order", 6)));
    throw std::invalid_argument("unknown kernel '" + name + "'");
}

Parsed parse_kernel(const std::string& expr) {
    std::vector<KernelSpec> parts;
    int depth = 0;
    std::string cur;
    for (char c : expr) {
        if (c == '(') ++depth;
        if (c == ')') --depth;
        if (c == '+' && depth == 0) {
            parts.push_back(parse_leaf(cur));
            cur.clear();
        } else {
            cur += c;
        }
    }
    parts.push_back(parse_leaf(cur));
    Parsed p;
    p.spec = parts.size() == 1 ? parts[0] : KernelSpec::sum(parts);
    p.theta = default_theta(p.spec);
    return p;
}

// ------------------------------------------------------------------- data --
Dataset read_csv(const std::string& path) {
    std::ifstream f(path);
    if (!f) throw std::runtime_error("cannot read " + path);
    Dataset d;
    std::string line;
    while (std::getline(f, line)) {
        if (line.empty() || line[0] == '#' || std::isalpha(static_cast<unsigned char>(line[0]))) continue;
        std::replace(line.begin(), line.end(), ',', ' ');
        std::stringstream ss(line);
        double t, y;
        if (ss >> t >> y) {
            d.times.push_back(t);
            d.values.push_back(y);
        }
    }
    return d;
}

void write_data(const std::string& path, const Dataset& d) {
    std::ofstream f(path);
    f << "t,y\n";
    f.precision(17);
    for (size_t i = 0; i < d.times.size(); ++i) f << d.times[i] << "," << d.values[i] << "\n";
}

// y = sin(2π f1 t) + 0.6 sin(2π f2 t) + η, η ~ N(0, noise²), t = i h;
// f1 = 0.04, f2 = 0.17, h = 1 (SPEC.md:485 defaults).  mt19937_64, explicit transforms.
Dataset sinusoids(int64_t n, uint64_t seed, double noise) {
    std::mt19937_64 g(seed);
    auto u01 = [&] { return (static_cast<double>(g() >> 11) + 0.5) * 0x1.0p-53; };
    Dataset d;
    const double pi = 3.14159265358979323846;
    for (int64_t i = 0; i < n; ++i) {
        const double t = static_cast<double>(i);
        const double z = std::sqrt(-2.0 * std::log(u01())) * std::cos(2.0 * pi * u01());  // Box-Muller
        d.times.push_back(t);
        d.values.push_back(std::sin(2 * pi * 0.04 * t) + 0.6 * std::sin(2 * pi * 0.17 * t) + noise * z);
    }
    return d;
}

// ------------------------------------------------- comparison methods (host) --
double kf_mll(const Dataset& d, const KernelSpec& spec, const HyperparameterSet& th, double s2) {
    const StateSpaceModel ssm = state_space_of(spec, th);
    const Index b = ssm.dim();
    std::vector<double> m(b, 0.0), P(ssm.Pinf.data(), ssm.Pinf.data() + b * b), tmp(b * b);
    double ll = 0.0;
    const double l2pi = std::log(2.0 * 3.14159265358979323846);
    for (size_t i = 0; i < d.times.size(); ++i) {
        if (i > 0) {
            const DiscreteStep st = discretize(ssm, d.times[i] - d.times[i - 1]);
            std::vector<double> mn(b, 0.0);
            for (Index a = 0; a < b; ++a)
                for (Index c = 0; c < b; ++c) mn[a] += st.Phi(a, c) * m[c];
            m = mn;
            for (Index a = 0; a < b; ++a)
                for (Index c = 0; c < b; ++c) {
                    double s = 0.0;
                    for (Index k = 0; k < b; ++k) s += st.Phi(a, k) * P[k * b + c];
                    tmp[a * b + c] = s;
                }
            for (Index a = 0; a < b; ++a)
                for (Index c = 0; c < b; ++c) {
                    double s = st.Q(a, c);
                    for (Index k = 0; k < b; ++k) s += tmp[a * b + k] * st.Phi(c, k);
                    P[a * b + c] = s;
                }
        }
        std::vector<double> PH(b, 0.0);
        double hm = 0.0, S = s2;
        for (Index a = 0; a < b; ++a) {
            for (Index c = 0; c < b; ++c) PH[a] += P[a * b + c] * ssm.H(c);
            hm += ssm.H(a) * m[a];
        }
        for (Index a = 0; a < b; ++a) S += ssm.H(a) * PH[a];
        if (!(S > 0.0)) throw NotPositiveDefinite("kf: innovation variance <= 0", static_cast<std::ptrdiff_t>(i));
        const double v = d.values[i] - hm;
        ll += -0.5 * (l2pi + std::log(S) + v * v / S);
        for (Index a = 0; a < b; ++a) {
            m[a] += PH[a] * v / S;
            for (Index c = 0; c < b; ++c) P[a * b + c] -= PH[a] * PH[c] / S;
        }
    }
    return ll;
}

double dense_mll(const Dataset& d, const KernelSpec& spec, const HyperparameterSet& th, double s2) {
    const size_t n = d.times.size();
    if (n > 20000) throw std::invalid_argument("dense: N above the dense cap");
    std::vector<double> K(n * n);
    std::map<double, double> kcache;  // k(|τ|): on a regular grid only N distinct lags
    for (size_t i = 0; i < n; ++i)
        for (size_t j = 0; j <= i; ++j) {
            const double tau = d.times[i] - d.times[j];
            auto it = kcache.find(tau);
            if (it == kcache.end()) it = kcache.emplace(tau, kernel_eval(spec, th, tau, 0.0)).first;
            K[i * n + j] = it->second + (i == j ? s2 : 0.0);
        }
    double logdet = 0.0;
    for (size_t j = 0; j < n; ++j) {  // in-place lower Cholesky
        double s = K[j * n + j];
        for (size_t k = 0; k < j; ++k) s -= K[j * n + k] * K[j * n + k];
        if (!(s > 0.0)) throw NotPositiveDefinite("dense: K + s2 I not PD", static_cast<std::ptrdiff_t>(j));
        const double l = std::sqrt(s);
        K[j * n + j] = l;
        logdet += 2.0 * std::log(l);
        for (size_t i = j + 1; i < n; ++i) {
            double v = K[i * n + j];
            for (size_t k = 0; k < j; ++k) v -= K[i * n + k] * K[j * n + k];
            K[i * n + j] = v / l;
        }
    }
    std::vector<double> z(d.values);
    for (size_t i = 0; i < n; ++i) {
        for (size_t k = 0; k < i; ++k) z[i] -= K[i * n + k] * z[k];
        z[i] /= K[i * n + i];
    }
    double fit = 0.0;
    for (double v : z) fit += v * v;
    return -0.5 * fit - 0.5 * logdet - 0.5 * static_cast<double>(n) * std::log(2.0 * 3.14159265358979323846);
}

// one MLL(+gradient for spingp) evaluation by `method`
double evaluate(const std::string& method, const Dataset& d, const Parsed& k, double s2, Device* devp) {
    if (method == "spingp") {
        Device& dev = *devp;
        mll_gradient(d, k.spec, k.theta, NoiseModel{s2}, dev);
        return log_marginal_likelihood(d, k.spec, k.theta, NoiseModel{s2}, dev);
    }
    if (method == "kf") return kf_mll(d, k.spec, k.theta, s2);
    if (method == "dense") return dense_mll(d, k.spec, k.theta, s2);
    throw std::invalid_argument("unknown method " + method);
}

// ---------------------------------------------------------------- reports --
struct Row {
    std::string method;
    double x;
    double seconds;
    double mll;
    std::string error;
};

double slope(const std::vector<Row>& rows, const std::string& method) {
    double sx = 0, sy = 0, sxx = 0, sxy = 0;
    int n = 0;
    for (const Row& r : rows)
        if (r.method == method && r.error.empty() && r.seconds > 0) {
            const double lx = std::log(r.x), ly = std::log(r.seconds);
            sx += lx, sy += ly, sxx += lx * lx, sxy += lx * ly, ++n;
        }
    if (n < 2) return std::nan("");
    return (n * sxy - sx * sy) / (n * sxx - sx * sx);
}

std::string csv_quote(const std::string& s) {
    if (s.find_first_of(",\"\n") == std::string::npos) return s;
    std::string o = "\"";
    for (char c : s) o += (c == '"') ? std::string("\"\"") : std::string(1, c);
    return o + "\"";
}

std::string json_str(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}

void write_report(const std::string& dir, const std::string& xname, const std::vector<Row>& rows,
                  const std::vector<std::string>& methods, const std::string& extra_json) {
    std::ofstream c(dir + "/report.csv");
    c.precision(17);
    c << "method," << xname << ",median_seconds,mll,error\n";
    for (const Row& r : rows)
        c << r.method << "," << r.x << "," << r.seconds << "," << r.mll << "," << csv_quote(r.error) << "\n";
    std::ofstream j(dir + "/metrics.json");
    j.precision(17);
    j << "{\"schema_version\": 1, \"sweep\": " << json_str(xname) << ", \"slopes\": {";
    for (size_t i = 0; i < methods.size(); ++i) {
        const double s = slope(rows, methods[i]);
        j << (i ? ", " : "") << json_str(methods[i]) << ": " << (std::isnan(s) ? std::string("null") : std::to_string(s));
    }
    j << "}, \"rows\": " << rows.size() << extra_json << "}\n";
}

template <class F>
double median_seconds(int reps, F&& f) {
    f();  // warm-up
    std::vector<double> t;
    for (int r = 0; r < reps; ++r) {
        const auto a = std::chrono::steady_clock::now();
        f();
        t.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - a).count());
    }
    std::sort(t.begin(), t.end());
    return t[t.size() / 2];
}

std::vector<std::string> methods_of(const Args& a) {
    std::vector<std::string> m;
    std::stringstream ss(arg(a, "method", "spingp"));
    std::string tok;
    while (std::getline(ss, tok, ',')) m.push_back(tok);
    return m;
}

int sweep(const Args& a, bool over_b) {
    const std::string dir = arg(a, "out");
    mkdir(dir.c_str(), 0755);
    const int reps = std::max(5, std::stoi(arg(a, "repetitions", "5")));
    const uint64_t seed = std::stoull(arg(a, "seed", "1"));
    const double s2 = 0.04;  // noise σ = 0.2
    const auto methods = methods_of(a);
    std::unique_ptr<Device> dev;  // the GPU context only when the spingp method runs
    if (std::find(methods.begin(), methods.end(), "spingp") != methods.end()) dev = std::make_unique<Device>(0);
    std::vector<Row> rows;
    int failed = 0;
    std::vector<double> xs = list_of(arg(a, over_b ? "bs" : "ns", over_b ? "2,4,8,12,16" : "1000,2000,4000,8000"));
    std::string kexpr = arg(a, "kernel", "matern32(len=5) + eq(len=20, order=10)");  // b = 12
    for (const std::string& m : methods)
        for (double x : xs) {
            Row r{m, x, 0.0, std::nan(""), ""};
            try {
                Parsed k;
                Dataset d;
                if (over_b) {
                    // b = 2 k: a sum of k Matérn-3/2 leaves with distinct lengthscales
                    const int kk = static_cast<int>(x) / 2;
                    if (kk < 1 || 2 * kk != static_cast<int>(x)) throw std::invalid_argument("b must be even");
                    std::string e;
                    for (int i = 0; i < kk; ++i) e += (i ? " + " : "") + std::string("matern32(len=") + std::to_string(2.0 + 3.0 * i) + ")";
                    k = parse_kernel(e);
                    d = sinusoids(std::stoll(arg(a, "n", "1000")), seed, 0.2);
                } else {
                    k = parse_kernel(kexpr);
                    d = sinusoids(static_cast<int64_t>(x), seed, 0.2);
                }
                r.seconds = median_seconds(reps, [&] { r.mll = evaluate(m, d, k, s2, dev.get()); });
            } catch (const std::exception& e) {
                r.error = e.what();
                ++failed;
            }
            std::cerr << m << " " << x << " " << r.seconds << " s " << r.mll << (r.error.empty() ? "" : " " + r.error) << "\n";
            rows.push_back(r);
        }
    write_report(dir, over_b ? "b" : "N", rows, methods,
                 ", \"kernel\": " + json_str(over_b ? std::string("sum of b/2 matern32 leaves") : kexpr) +
                     ", \"repetitions\": " + std::to_string(reps) + ", \"seed\": " + std::to_string(seed) +
                     ", \"data\": \"sinusoids f1=0.04 f2=0.17 amplitudes 1/0.6 noise 0.2 h=1\"");
    return failed ? 1 : 0;
}

void write_fit(const std::string& dir, const Parsed& k, const OptimizeResult& r, const std::string& extra) {
    std::ofstream j(dir + "/metrics.json");
    j.precision(17);
    const auto names = hyperparameter_names(k.spec);
    j << "{\"schema_version\": 1, \"theta\": {";
    for (size_t i = 0; i < r.theta.size(); ++i) j << (i ? ", " : "") << json_str(names[i]) << ": " << r.theta[i];
    j << "}, \"sigma_n2\": " << r.noise.sigma_n2 << ", \"mll\": " << (r.trace.empty() ? std::nan("") : r.trace.back())
      << ", \"iterations\": " << r.iterations << ", \"line_search_failed\": " << (r.line_search_failed ? "true" : "false")
      << extra << "}\n";
}

int cmd_fit(const Args& a) {
    const std::string dir = arg(a, "out");
    mkdir(dir.c_str(), 0755);
    Parsed k = parse_kernel(arg(a, "kernel"));
    const Dataset d = read_csv(arg(a, "data"));
    const auto r = optimize_hyperparameters(d, k.spec, k.theta, NoiseModel{std::stod(arg(a, "noise2", "0.1"))},
                                            std::stoi(arg(a, "budget", "200")));
    write_fit(dir, k, r, "");
    return 0;
}

void write_forecast(const std::string& path, const PosteriorSummary& p) {
    std::ofstream f(path);
    f.precision(17);
    f << "t,mean,variance\n";
    for (size_t i = 0; i < p.times.size(); ++i) f << p.times[i] << "," << p.mean[i] << "," << p.variance[i] << "\n";
}

int cmd_predict(const Args& a) {
    const std::string dir = arg(a, "out");
    mkdir(dir.c_str(), 0755);
    Parsed k = parse_kernel(arg(a, "kernel"));
    const Dataset d = read_csv(arg(a, "data"));
    const auto g = list_of([&] { std::string s = arg(a, "grid"); std::replace(s.begin(), s.end(), ':', ','); return s; }());
    if (g.size() != 3 || g[2] < 1) throw std::invalid_argument("--grid a:b:m");
    std::vector<double> ts;
    for (int i = 0; i < static_cast<int>(g[2]); ++i) ts.push_back(g[0] + (g[1] - g[0]) * i / std::max(1.0, g[2] - 1));
    const auto p = predict(d, k.spec, k.theta, NoiseModel{std::stod(arg(a, "noise2", "0.04"))}, ts, false);
    write_forecast(dir + "/forecast.csv", p);
    return 0;
}

// NOAA weekly file: '#' comments; columns yr mon day decimal ppm ...; -999.99 = missing
// (SPEC.md:440-447).  Values are mean-centred (the mean is recorded).
Dataset ingest_co2(const std::string& path, double& mean_out) {
    std::ifstream f(path);
    if (!f) throw std::runtime_error("cannot read " + path);
    Dataset d;
    std::string line;
    while (std::getline(f, line)) {
        if (line.empty() || line[0] == '#') continue;
        std::replace(line.begin(), line.end(), ',', ' ');
        std::stringstream ss(line);
        double c[5];
        int k = 0;
        while (k < 5 && ss >> c[k]) ++k;
        if (k < 5 || c[4] <= -999.0) continue;
        if (!d.times.empty() && !(c[3] > d.times.back())) throw std::runtime_error("non-increasing timestamps");
        d.times.push_back(c[3]);
        d.values.push_back(c[4]);
    }
    if (d.times.empty()) throw std::runtime_error("NoValidRows: no valid rows in " + path);
    double m = 0.0;
    for (double v : d.values) m += v;
    m /= static_cast<double>(d.values.size());
    for (double& v : d.values) v -= m;
    mean_out = m;
    return d;
}

int cmd_co2(const Args& a) {
    const std::string dir = arg(a, "out");
    mkdir(dir.c_str(), 0755);
    double mean = 0.0;
    const Dataset all = ingest_co2(arg(a, "data"), mean);
    Parsed k = parse_kernel(arg(a, "kernel", "matern32(var=10, len=20) + eq(var=1, len=1, order=10)"));
    const double hold = all.times.back() - 8.0;  // hold out the final 8 years
    Dataset train, test;
    for (size_t i = 0; i < all.times.size(); ++i) {
        Dataset& dst = all.times[i] <= hold ? train : test;
        dst.times.push_back(all.times[i]);
        dst.values.push_back(all.values[i]);
    }
    if (train.times.size() < 2 || test.times.empty()) throw std::invalid_argument("co2: too few rows to hold out 8 years");
    const auto r = optimize_hyperparameters(train, k.spec, k.theta, NoiseModel{0.1}, std::stoi(arg(a, "budget", "200")));
    std::vector<double> ts = test.times;
    for (int w = 1; w <= 8 * 52; ++w) ts.push_back(all.times.back() + w / 52.0);
    const auto p = predict(train, k.spec, r.theta, r.noise, ts, false);
    PosteriorSummary out = p;
    for (double& m : out.mean) m += mean;
    write_forecast(dir + "/forecast.csv", out);
    double se = 0.0, se0 = 0.0, tmean = 0.0;
    for (double v : train.values) tmean += v;
    tmean /= static_cast<double>(train.values.size());
    for (size_t i = 0; i < test.times.size(); ++i) {
        se += (p.mean[i] - test.values[i]) * (p.mean[i] - test.values[i]);
        se0 += (tmean - test.values[i]) * (tmean - test.values[i]);
    }
    const double n = static_cast<double>(test.times.size());
    std::ostringstream ex;
    ex.precision(17);
    ex << ", \"rows\": " << all.times.size() << ", \"heldout_rows\": " << test.times.size()
       << ", \"heldout_rmse\": " << std::sqrt(se / n) << ", \"constant_mean_rmse\": " << std::sqrt(se0 / n)
       << ", \"mean_ppm\": " << mean;
    write_fit(dir, k, r, ex.str());
    return 0;
}

int cmd_gen(const Args& a) {
    const std::string dir = arg(a, "out");
    mkdir(dir.c_str(), 0755);
    write_data(dir + "/data.csv", sinusoids(std::stoll(arg(a, "n")), std::stoull(arg(a, "seed", "1")),
                                            std::stod(arg(a, "noise", "0.2"))));
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::cerr << "usage: spingp gen-data|fit|predict|scaling-n|scaling-b|co2 [--key value ...]\n";
        return 2;
    }
    const std::string cmd = argv[1];
    Args a;
    for (int i = 2; i + 1 < argc; i += 2) {
        std::string k = argv[i];
        if (k.rfind("--", 0) != 0) {
            std::cerr << "expected --key, got " << k << "\n";
            return 2;
        }
        a[k.substr(2)] = argv[i + 1];
    }
    try {
        if (cmd == "gen-data") return cmd_gen(a);
        if (cmd == "fit") return cmd_fit(a);
        if (cmd == "predict") return cmd_predict(a);
        if (cmd == "scaling-n") return sweep(a, false);
        if (cmd == "scaling-b") return sweep(a, true);
        if (cmd == "co2") return cmd_co2(a);
        std::cerr << "unknown subcommand " << cmd << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
