// calibration.cpp — host side of the threshold calibration loop (SURVEY.md §8
// f1): score-population statistics, the cubic fit and profile JSON I/O, as the
// C-ABI of include/sinkr_cuda.h.  Restates calibration.cpp of the reference
// (calibration.cpp:14-243) with its expression order; this file is built with
// -ffp-contract=off like the reference (no FMA), so every double it returns
// is bit-identical to the reference's (tests/test_calibration.py).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "host_util.hpp"
#include "json_lite.hpp"

using sinkr::host::fail;
using sinkr::host::guard;

namespace {

// fraction of the sorted population strictly above t (calibration.cpp:16-19)
double frac_above(const std::vector<double>& sorted, double t) {
    const auto first_above = std::upper_bound(sorted.begin(), sorted.end(), t);
    return static_cast<double>(sorted.end() - first_above) / static_cast<double>(sorted.size());
}

std::vector<double> sorted_copy(const double* s, size_t n) {
    std::vector<double> v(s, s + n);
    std::sort(v.begin(), v.end());
    return v;
}

// solve_threshold (calibration.cpp:58-71): the lower (1 - target) empirical
// quantile, index floor((1 - target) * n + 1e-9) clamped to [1, n].
double quantile_threshold(const std::vector<double>& sorted, double target) {
    const size_t n = sorted.size();
    size_t k = static_cast<size_t>(std::floor((1.0 - target) * static_cast<double>(n) + 1e-9));
    if (k < 1) k = 1;
    if (k > n) k = n;
    return sorted[k - 1];
}

// fit_cubic (calibration.cpp:73-117): normal equations over {x^3, x^2, x, 1},
// Gaussian elimination with partial pivoting over a row permutation, back
// substitution, then the residual sum of squares under Horner evaluation.
void cubic_fit(const double* xs, const double* ys, size_t n, double coeffs[4], double* residual) {
    std::set<double> distinct(xs, xs + n);
    if (n < 4 || distinct.size() < 4)
        fail(SINKR_INVALID_ARGUMENT, "cubic fit needs at least 4 points with 4 distinct x values");
    double A[4][4] = {};
    double rhs[4] = {};
    for (size_t p = 0; p < n; ++p) {
        const double x = xs[p], y = ys[p];
        const double phi[4] = {x * x * x, x * x, x, 1.0};
        for (int i = 0; i < 4; ++i) {
            for (int j = 0; j < 4; ++j) A[i][j] += phi[i] * phi[j];
            rhs[i] += phi[i] * y;
        }
    }
    int row_of[4] = {0, 1, 2, 3};
    for (int c = 0; c < 4; ++c) {
        int best = c;
        for (int i = c + 1; i < 4; ++i)
            if (std::fabs(A[row_of[i]][c]) > std::fabs(A[row_of[best]][c])) best = i;
        std::swap(row_of[c], row_of[best]);
        const double piv = A[row_of[c]][c];
        if (std::fabs(piv) < 1e-30) fail(SINKR_INVALID_ARGUMENT, "cubic fit design matrix is rank deficient");
        for (int i = c + 1; i < 4; ++i) {
            const double f = A[row_of[i]][c] / piv;
            for (int j = c; j < 4; ++j) A[row_of[i]][j] -= f * A[row_of[c]][j];
            rhs[row_of[i]] -= f * rhs[row_of[c]];
        }
    }
    double sol[4] = {0.0, 0.0, 0.0, 0.0};
    for (int i = 3; i >= 0; --i) {
        double acc = rhs[row_of[i]];
        for (int j = i + 1; j < 4; ++j) acc -= A[row_of[i]][j] * sol[j];
        sol[i] = acc / A[row_of[i]][i];
    }
    double ss = 0.0;
    for (size_t p = 0; p < n; ++p) {
        const double x = xs[p];
        const double pred = ((sol[0] * x + sol[1]) * x + sol[2]) * x + sol[3];
        ss += (ys[p] - pred) * (ys[p] - pred);
    }
    for (int i = 0; i < 4; ++i) coeffs[i] = sol[i];
    if (residual) *residual = ss;
}

void set_default(sinkr_profile* p) {
    std::memset(p, 0, sizeof(*p));
    p->threshold.length_normalizer = 1.0;
    p->threshold.clamp_lo = 0.0;
    p->threshold.clamp_hi = 1.0;
    p->target_skip = 0.60;
    p->gamma = 0.65;
    p->excluded_layers[0] = 0;
    p->excluded_layers[1] = 1;
    p->num_excluded_layers = 2;
}

std::string read_file(const char* path, const char* what) {
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(SINKR_RUNTIME_ERROR, std::string("cannot open '") + path + "' for reading");
    std::stringstream ss;
    ss << in.rdbuf();
    (void)what;
    return ss.str();
}

}  // namespace

extern "C" {

void sinkr_profile_default(sinkr_profile* out) {
    if (out) set_default(out);
}

void sinkr_profile_constant(double tau, sinkr_profile* out) {
    if (!out) return;
    set_default(out);
    out->threshold.coeffs[3] = tau;
    out->threshold.clamp_lo = std::min(tau, 0.0);
    out->threshold.clamp_hi = std::max(tau, 1.0);
}

sinkr_status sinkr_sweep(const double* scores, size_t n, const double* thresholds, size_t m,
                         double* skip_ratios) {
    return guard([&] {
        if (n == 0) fail(SINKR_INVALID_ARGUMENT, "sweep over empty score population");
        if (m && (!thresholds || !skip_ratios)) fail(SINKR_INVALID_ARGUMENT, "null argument");
        const auto s = sorted_copy(scores, n);
        for (size_t i = 0; i < m; ++i) skip_ratios[i] = frac_above(s, thresholds[i]);
    });
}

sinkr_status sinkr_skip_ratio_at(const double* scores, size_t n, double threshold, double* out) {
    return guard([&] {
        if (n == 0) fail(SINKR_INVALID_ARGUMENT, "skip ratio over empty score population");
        if (!out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        *out = frac_above(sorted_copy(scores, n), threshold);
    });
}

sinkr_status sinkr_solve_threshold(const double* scores, size_t n, double target_skip,
                                   double* out) {
    return guard([&] {
        if (n == 0) fail(SINKR_INVALID_ARGUMENT, "solve_threshold over empty score population");
        if (target_skip < 0.0 || target_skip >= 1.0)
            fail(SINKR_INVALID_ARGUMENT, "target_skip must be in [0, 1)");
        if (!out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        *out = quantile_threshold(sorted_copy(scores, n), target_skip);
    });
}

sinkr_status sinkr_fit_cubic(const double* x, const double* y, size_t n, double* coeffs,
                             double* residual) {
    return guard([&] {
        if (!coeffs || (n && (!x || !y))) fail(SINKR_INVALID_ARGUMENT, "null argument");
        cubic_fit(x, y, n, coeffs, residual);
    });
}

// calibrate (calibration.cpp:119-172)
sinkr_status sinkr_calibrate(const size_t* lengths, size_t n_lengths, const double* scores,
                             const size_t* sample_layers, const size_t* offsets,
                             double target_skip, double gamma, const size_t* excluded_layers,
                             size_t num_excluded_layers, sinkr_profile* out) {
    return guard([&] {
        if (!out || (n_lengths && (!lengths || !offsets)))
            fail(SINKR_INVALID_ARGUMENT, "null argument");
        if (num_excluded_layers > SINKR_MAX_EXCLUDED_LAYERS)
            fail(SINKR_INVALID_ARGUMENT, "too many excluded layers");
        std::set<size_t> distinct(lengths, lengths + n_lengths);
        if (distinct.size() < 4) fail(SINKR_INVALID_ARGUMENT, "calibration needs at least 4 distinct lengths");
        if (distinct.size() > SINKR_MAX_CALIBRATION_POINTS)
            fail(SINKR_INVALID_ARGUMENT, "too many calibration lengths");
        const size_t normalizer = *std::max_element(lengths, lengths + n_lengths);
        sinkr_profile p;
        set_default(&p);
        p.target_skip = target_skip;
        p.gamma = gamma;
        p.num_excluded_layers = num_excluded_layers;
        for (size_t i = 0; i < num_excluded_layers; ++i) p.excluded_layers[i] = excluded_layers[i];
        p.threshold.length_normalizer = static_cast<double>(normalizer);
        std::vector<double> fx, fy;
        for (size_t len : distinct) {
            size_t idx = 0;
            while (lengths[idx] != len) ++idx;  // the population of its first occurrence
            std::vector<double> routable;
            for (size_t s = offsets[idx]; s < offsets[idx + 1]; ++s) {
                const size_t layer = sample_layers ? sample_layers[s] : 0;
                bool excl = false;
                for (size_t k = 0; k < num_excluded_layers; ++k) excl |= excluded_layers[k] == layer;
                if (!excl) routable.push_back(scores[s]);
            }
            if (routable.empty())
                fail(SINKR_RUNTIME_ERROR, "calibration population is empty after layer exclusion");
            if (target_skip < 0.0 || target_skip >= 1.0)
                fail(SINKR_INVALID_ARGUMENT, "target_skip must be in [0, 1)");
            std::sort(routable.begin(), routable.end());
            const double tau = quantile_threshold(routable, target_skip);
            const double realized = frac_above(routable, tau);
            p.points[p.num_points++] = sinkr_calibration_point{len, tau, realized};
            fx.push_back(static_cast<double>(len) / p.threshold.length_normalizer);
            fy.push_back(tau);
        }
        cubic_fit(fx.data(), fy.data(), fx.size(), p.threshold.coeffs, nullptr);
        double lo = p.points[0].tau, hi = lo;
        for (size_t i = 0; i < p.num_points; ++i) {
            lo = std::min(lo, p.points[i].tau);
            hi = std::max(hi, p.points[i].tau);
        }
        // clamp headroom around the solved range (calibration.cpp:166-170)
        p.threshold.clamp_lo = std::max(-1.0, lo - 0.1);
        p.threshold.clamp_hi = std::min(1.0, hi + 0.1);
        *out = p;
    });
}

// save_profile (calibration.cpp:174-195): the reference's key order.
sinkr_status sinkr_save_profile(const char* path, const sinkr_profile* p) {
    return guard([&] {
        if (!path || !p) fail(SINKR_INVALID_ARGUMENT, "null argument");
        using sinkr::json::num;
        std::string j = "{\n";
        j += "  \"version\": 1,\n";
        j += "  \"gamma\": " + num(p->gamma) + ",\n";
        j += "  \"target_skip\": " + num(p->target_skip) + ",\n";
        j += "  \"length_normalizer\": " + num(p->threshold.length_normalizer) + ",\n";
        j += "  \"coefficients\": [";
        for (int i = 0; i < 4; ++i) j += (i ? ", " : "") + num(p->threshold.coeffs[i]);
        j += "],\n";
        j += "  \"clamp\": [" + num(p->threshold.clamp_lo) + ", " + num(p->threshold.clamp_hi) + "],\n";
        j += "  \"excluded_layers\": [";
        for (size_t i = 0; i < p->num_excluded_layers; ++i)
            j += (i ? ", " : "") + num((unsigned long long)p->excluded_layers[i]);
        j += "],\n";
        j += "  \"calibration_points\": [";
        for (size_t i = 0; i < p->num_points; ++i) {
            j += i ? ",\n" : "\n";
            j += "    {\"length\": " + num((unsigned long long)p->points[i].length) +
                 ", \"tau\": " + num(p->points[i].tau) + ", \"skip\": " + num(p->points[i].skip) + "}";
        }
        j += p->num_points ? "\n  ]\n}\n" : "]\n}\n";
        std::ofstream out(path, std::ios::binary | std::ios::trunc);
        if (!out) fail(SINKR_RUNTIME_ERROR, std::string("cannot open '") + path + "' for writing");
        out << j;
        if (!out) fail(SINKR_RUNTIME_ERROR, std::string("write failed for '") + path + "'");
    });
}

// load_profile (calibration.cpp:197-243): required keys, version 1, array
// shapes; unknown keys are ignored with a warning on stderr.
sinkr_status sinkr_load_profile(const char* path, sinkr_profile* out) {
    return guard([&] {
        if (!path || !out) fail(SINKR_INVALID_ARGUMENT, "null argument");
        const std::string text = read_file(path, "profile");
        sinkr::json::Value j;
        try {
            j = sinkr::json::parse(text);
        } catch (const std::runtime_error& e) {
            fail(SINKR_RUNTIME_ERROR,
                 std::string("profile JSON parse error in '") + path + "': " + e.what());
        }
        if (!j.is_object()) fail(SINKR_RUNTIME_ERROR, "profile JSON must be an object");
        static const char* known[] = {"version", "gamma", "target_skip", "length_normalizer",
                                      "coefficients", "clamp", "excluded_layers",
                                      "calibration_points"};
        for (const auto& kv : j.obj) {
            bool k = false;
            for (const char* n : known) k |= kv.first == n;
            if (!k) std::fprintf(stderr, "profile: ignoring unknown key \"%s\"\n", kv.first.c_str());
        }
        for (const char* key : known)
            if (!j.contains(key))
                fail(SINKR_RUNTIME_ERROR, std::string("profile JSON missing key \"") + key + "\"");
        try {
            if (j.at("version").as_i64() != 1)
                fail(SINKR_RUNTIME_ERROR, "unsupported profile version " + j.at("version").str);
            sinkr_profile p;
            set_default(&p);
            p.gamma = j.at("gamma").as_double();
            p.target_skip = j.at("target_skip").as_double();
            p.threshold.length_normalizer = j.at("length_normalizer").as_double();
            const auto& co = j.at("coefficients");
            if (!co.is_array() || co.arr.size() != 4)
                fail(SINKR_RUNTIME_ERROR, "profile JSON key \"coefficients\" must be a 4-element array");
            for (int i = 0; i < 4; ++i) p.threshold.coeffs[i] = co.arr[i].as_double();
            const auto& cl = j.at("clamp");
            if (!cl.is_array() || cl.arr.size() != 2)
                fail(SINKR_RUNTIME_ERROR, "profile JSON key \"clamp\" must be a 2-element array");
            p.threshold.clamp_lo = cl.arr[0].as_double();
            p.threshold.clamp_hi = cl.arr[1].as_double();
            const auto& ex = j.at("excluded_layers");
            if (!ex.is_array()) fail(SINKR_RUNTIME_ERROR, "profile JSON key \"excluded_layers\" must be an array");
            if (ex.arr.size() > SINKR_MAX_EXCLUDED_LAYERS)
                fail(SINKR_RUNTIME_ERROR, "profile has too many excluded layers");
            p.num_excluded_layers = ex.arr.size();
            for (size_t i = 0; i < ex.arr.size(); ++i) p.excluded_layers[i] = ex.arr[i].as_u64();
            const auto& pts = j.at("calibration_points");
            if (!pts.is_array()) fail(SINKR_RUNTIME_ERROR, "profile JSON key \"calibration_points\" must be an array");
            if (pts.arr.size() > SINKR_MAX_CALIBRATION_POINTS)
                fail(SINKR_RUNTIME_ERROR, "profile has too many calibration points");
            p.num_points = 0;
            for (const auto& q : pts.arr) {
                for (const char* key : {"length", "tau", "skip"})
                    if (!q.contains(key))
                        fail(SINKR_RUNTIME_ERROR, std::string("profile JSON missing key \"") + key + "\"");
                p.points[p.num_points++] = sinkr_calibration_point{
                    (size_t)q.at("length").as_u64(), q.at("tau").as_double(), q.at("skip").as_double()};
            }
            *out = p;
        } catch (const std::runtime_error& e) {
            fail(SINKR_RUNTIME_ERROR, std::string("profile JSON in '") + path + "': " + e.what());
        }
    });
}

}  // extern "C"
