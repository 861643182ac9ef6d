// a6: lightweight sample reallocation policy (§6.1), host C++.
//   threshold = knee of the throughput-vs-sample-count curve (reading Z13)
//   Eq. 6: maximise samples received by d-instances subject to
//     s_next >= thr, d_next <= thr, each instance migrates at most once;
//   greedy: pair the most-loaded source with the least-loaded destination, repeatedly;
//     move min(s_cur - thr, thr - d_cur); prefer shorter sequences, then lower avg accepted.
#include <algorithm>
#include <numeric>
#include <vector>

#include "common.cuh"

extern "C" rs_status rs_knee_threshold(const double* counts, const double* tput, int32_t n, double frac,
                                       int32_t* threshold) {
    RS_REQUIRE(counts && tput && threshold && n >= 3, RS_ERR_INVALID_ARG, "rs_knee_threshold: need >= 3 points");
    for (int i = 1; i < n; ++i)
        RS_REQUIRE(counts[i] > counts[i - 1], RS_ERR_INVALID_ARG, "rs_knee_threshold: counts must increase");
    const double g0 = (tput[1] - tput[0]) / (counts[1] - counts[0]);
    if (g0 <= 0.0) {
        *threshold = (int32_t)counts[0];
        return RS_OK;
    }
    for (int i = 1; i < n; ++i) {
        const double g = (tput[i] - tput[i - 1]) / (counts[i] - counts[i - 1]);
        if (g < frac * g0) {
            *threshold = (int32_t)counts[i];
            return RS_OK;
        }
    }
    *threshold = (int32_t)counts[n - 1];
    return RS_OK;
}

extern "C" rs_status rs_plan_reallocation(const int32_t* loads, int32_t G, int32_t thr, int32_t* src, int32_t* dst,
                                          int32_t* count, int32_t* n_transfers) {
    RS_REQUIRE(loads && src && dst && count && n_transfers && G >= 0 && thr >= 0, RS_ERR_INVALID_ARG,
               "rs_plan_reallocation: bad args");
    std::vector<int> srcs, dsts;
    for (int i = 0; i < G; ++i) {
        if (loads[i] > thr) srcs.push_back(i);
        if (loads[i] < thr) dsts.push_back(i);
    }
    std::sort(srcs.begin(), srcs.end(), [&](int a, int b) { return loads[a] != loads[b] ? loads[a] > loads[b] : a < b; });
    std::sort(dsts.begin(), dsts.end(), [&](int a, int b) { return loads[a] != loads[b] ? loads[a] < loads[b] : a < b; });
    int m = 0;
    for (size_t k = 0; k < srcs.size() && k < dsts.size(); ++k) {
        const int s = srcs[k], d = dsts[k];
        const int c = std::min(loads[s] - thr, thr - loads[d]);
        if (c <= 0) break;
        src[m] = s;
        dst[m] = d;
        count[m] = c;
        ++m;
    }
    *n_transfers = m;
    return RS_OK;
}

extern "C" rs_status rs_choose_samples(const int64_t* gid, const int32_t* seq_len, const double* avg_accepted,
                                       int32_t n, int32_t k, int64_t* chosen) {
    RS_REQUIRE(gid && seq_len && avg_accepted && chosen && n >= 0 && k >= 0 && k <= n, RS_ERR_INVALID_ARG,
               "rs_choose_samples: bad args");
    std::vector<int> idx(n);
    std::iota(idx.begin(), idx.end(), 0);
    std::sort(idx.begin(), idx.end(), [&](int a, int b) {
        if (seq_len[a] != seq_len[b]) return seq_len[a] < seq_len[b];
        if (avg_accepted[a] != avg_accepted[b]) return avg_accepted[a] < avg_accepted[b];
        return gid[a] < gid[b];
    });
    for (int i = 0; i < k; ++i) chosen[i] = gid[idx[i]];
    return RS_OK;
}

// the decision is taken every `cooldown` steps and a reallocation is triggered only if the
// inefficiency is present: some instance is below the threshold (it could take samples without
// losing throughput) while another is above it (reading Z13).
extern "C" rs_status rs_realloc_should_trigger(const int32_t* loads, int32_t G, int32_t thr, int32_t steps_since_last,
                                               int32_t cooldown, int32_t* trigger) {
    RS_REQUIRE(loads && trigger && G >= 0 && thr >= 0 && cooldown >= 0, RS_ERR_INVALID_ARG,
               "rs_realloc_should_trigger: bad args");
    bool below = false, above = false;
    for (int i = 0; i < G; ++i) {
        below = below || loads[i] < thr;
        above = above || loads[i] > thr;
    }
    *trigger = (steps_since_last >= cooldown && below && above) ? 1 : 0;
    return RS_OK;
}
