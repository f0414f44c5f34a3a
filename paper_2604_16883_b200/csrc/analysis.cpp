// analysis.cpp — proxy-reliability scoring on the host:
// oracle sink labels from full-attention BOS masses and the precision-recall
// curve of the routing proxy against them.  The reference declares these in
// analysis.hpp:12-39 without shipping an implementation; the semantics follow
// SPEC.md (analysis-oracle module): strict alpha0 > gamma, group label from
// the mean alpha0 of the group's heads, operating points at every distinct
// score (positive iff score >= threshold) in descending order, AUPRC by
// average-precision step summation sum_i (R_i - R_{i-1}) * P_i.
#include <algorithm>
#include <cstring>
#include <numeric>
#include <vector>

#include "host_util.hpp"

using sinkr::host::fail;
using sinkr::host::guard;

extern "C" {

sinkr_status sinkr_oracle_labels(const double* alpha0, size_t n_heads, size_t group,
                                 double gamma, int mode, double* label_alpha0,
                                 uint8_t* is_sink) {
    return guard([&] {
        if (!alpha0 || !label_alpha0 || !is_sink) fail(SINKR_INVALID_ARGUMENT, "null argument");
        if (mode != 0 && mode != 1) fail(SINKR_INVALID_ARGUMENT, "mode must be 0 (head) or 1 (group mean)");
        for (size_t i = 0; i < n_heads; ++i)
            if (!(alpha0[i] >= 0.0 && alpha0[i] <= 1.0 + 1e-4))
                fail(SINKR_INVALID_ARGUMENT, "alpha0 outside [0, 1]");
        if (mode == 0) {
            for (size_t i = 0; i < n_heads; ++i) {
                label_alpha0[i] = alpha0[i];
                is_sink[i] = alpha0[i] > gamma ? 1 : 0;
            }
            return;
        }
        if (group == 0 || n_heads % group != 0)
            fail(SINKR_INVALID_ARGUMENT, "n_heads must be a multiple of the group width");
        for (size_t g = 0; g < n_heads / group; ++g) {
            double s = 0.0;
            for (size_t i = 0; i < group; ++i) s += alpha0[g * group + i];
            const double mean = s / static_cast<double>(group);
            label_alpha0[g] = mean;
            is_sink[g] = mean > gamma ? 1 : 0;
        }
    });
}

sinkr_status sinkr_pr_curve(const double* scores, const uint8_t* labels, size_t n,
                            double* points, size_t* num_points, double* auprc) {
    return guard([&] {
        if ((n && (!scores || !labels)) || !num_points || !auprc)
            fail(SINKR_INVALID_ARGUMENT, "null argument");
        size_t positives = 0;
        for (size_t i = 0; i < n; ++i) positives += labels[i] ? 1 : 0;
        if (positives == 0) fail(SINKR_INVALID_ARGUMENT, "pr_curve needs at least one positive label");
        std::vector<size_t> order(n);
        std::iota(order.begin(), order.end(), size_t{0});
        std::stable_sort(order.begin(), order.end(),
                         [&](size_t a, size_t b) { return scores[a] > scores[b]; });
        size_t tp = 0, fp = 0, np = 0;
        double prev_recall = 0.0, ap = 0.0;
        for (size_t i = 0; i < n;) {
            const double thr = scores[order[i]];
            while (i < n && scores[order[i]] == thr) {  // all ties enter together
                if (labels[order[i]]) ++tp; else ++fp;
                ++i;
            }
            const double precision = static_cast<double>(tp) / static_cast<double>(tp + fp);
            const double recall = static_cast<double>(tp) / static_cast<double>(positives);
            const double f1 = (precision + recall) > 0.0 ? 2.0 * precision * recall / (precision + recall) : 0.0;
            ap += (recall - prev_recall) * precision;
            prev_recall = recall;
            if (points) {
                points[4 * np + 0] = thr;
                points[4 * np + 1] = precision;
                points[4 * np + 2] = recall;
                points[4 * np + 3] = f1;
            }
            ++np;
        }
        *num_points = np;
        *auprc = ap;
    });
}

}  // extern "C"
