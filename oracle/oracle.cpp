// ============================================================================
// O1 -- the CPU ORACLE for the PM4Py-GPU hot path (arXiv 2204.04898).
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load this library.  The
// product path (paper_2204_04898_b200/, libpm4g) never links, loads or calls
// it, and it shares no code, header, table or helper with that path.
//
// What it computes is the plain definition of every output, written out in the
// paper's order (§3) with no blocking, fusion or
// reordering:
//   step 1  "The dataframe is ordered based on three criteria (in order, case
//           identifier, the timestamp, and the absolute index of the event)"
//             -> std::stable_sort of row indices by (case, ts); the
//           stability realises the third criterion.
//   step 2  "the timestamp and the activity of the previous event"
//           -> in one loop, each event with a predecessor in its case forms
//           the directly-follows pair (prev_act, act) with duration
//           ts - prev_ts  (frequency/performance DFG)
//   step 3  "A cases dataframe ... number of events for the case, the
//           throughput time of the case, and some numerical features that
//           uniquely identify the case's variant" -> per case
//           n_events, duration = last ts - first ts, start / end
//           activity, and the variant = the exact activity
//           sequence ("double aggregation"), keyed here by
//           the sequence itself in a std::map (no hashing at all).
// Filters (P:126 timestamp.py, P:128 attributes.py) are plain
// per-row / per-case predicates evaluated on the definition; the NEXT rows of
// SURVEY.md 8(f) add whole-case filters (start / end activity, case size,
// throughput, paths, variants: P:98-103) and
// the per-edge min / max pair duration.
//
// Readings where the paper is silent are the ones listed in DESIGN.md
// "Readings" (R1..R19, = SURVEY.md §8(c) table); each is cited at its use.
// Integer sums are int64 two's complement defined modulo 2^64 (R8); an
// __int128 shadow records whether any sum wrapped.
// ============================================================================
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <numeric>
#include <vector>

namespace {

struct Variant {
    uint64_t count = 0;
    uint32_t rep = 0;  // smallest case code with this sequence (R11)
};

template <class T>
void copy_out(const std::vector<T>& v, T* dst) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(T));
}

}  // namespace

struct orc_result {
    uint32_t A = 0;
    int64_t n = 0;
    // formatted log (step 1)
    std::vector<uint32_t> s_case, s_act;
    std::vector<int64_t> s_ts, perm;
    // DFG (step 2)
    std::vector<uint64_t> cnt;
    std::vector<int64_t> sum;       // modulo 2^64 (R8)
    std::vector<__int128> sum_wide; // shadow, to detect wrap-around
    std::vector<double> mean;
    // performance DFG min / max of the pair durations (NEXT-2, S:281, S:306,
    // S:339): over the u64 difference ts_{i+1} - ts_i, which is exact because
    // 0 <= ts_{i+1} - ts_i < 2^64 after the sort (R20); 0 where cnt == 0
    std::vector<uint64_t> dmin, dmax;
    // cases dataframe (step 3)
    std::vector<uint64_t> start, end;
    std::vector<uint32_t> case_code, n_events;
    std::vector<int64_t> dur, first_row;
    // variants
    std::vector<uint64_t> v_count;
    std::vector<uint32_t> v_len, v_rep;
    std::vector<uint64_t> v_off;
    std::vector<uint32_t> v_act;
    std::vector<uint32_t> case_variant;  // per case (ascending code): output index
    int overflow = 0;
    double t_sort = 0, t_loop = 0;       // wall seconds of step 1 / steps 2 + 3 (timing only)
};

extern "C" {

// S:59-67 validate(): the first violated invariant.  Returns 0 (ok) or
// 2 (code out of range: case >= n_case_codes or act >= n_act); *bad = row.
int orc_validate(int64_t n, const uint32_t* case_, const uint32_t* act,
                 uint64_t n_case_codes, uint32_t n_act, int64_t* bad) {
    for (int64_t i = 0; i < n; ++i) {
        if ((uint64_t)case_[i] >= n_case_codes || act[i] >= n_act) {
            if (bad) *bad = i;
            return 2;
        }
    }
    if (bad) *bad = -1;
    return 0;
}

orc_result* orc_run(int64_t n, const uint32_t* case_, const uint32_t* act,
                    const int64_t* ts, uint32_t A) {
    orc_result* r = new orc_result();
    r->A = A;
    r->n = n;
    const auto t0 = std::chrono::steady_clock::now();

    // ---- step 1: stable sort of row indices by (case, ts)  (R1, R2)
    std::vector<int64_t> idx(n);
    std::iota(idx.begin(), idx.end(), (int64_t)0);
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t i, int64_t j) {
        if (case_[i] != case_[j]) return case_[i] < case_[j];
        return ts[i] < ts[j];
    });
    r->perm = idx;
    r->s_case.resize(n);
    r->s_act.resize(n);
    r->s_ts.resize(n);
    for (int64_t k = 0; k < n; ++k) {
        r->s_case[k] = case_[idx[k]];
        r->s_act[k] = act[idx[k]];
        r->s_ts[k] = ts[idx[k]];
    }

    const auto t1 = std::chrono::steady_clock::now();
    r->t_sort = std::chrono::duration<double>(t1 - t0).count();

    // ---- steps 2 + 3: one loop over the formatted log
    const size_t AA = (size_t)A * A;
    r->cnt.assign(AA, 0);
    r->sum.assign(AA, 0);
    r->sum_wide.assign(AA, 0);
    r->dmin.assign(AA, 0);
    r->dmax.assign(AA, 0);
    r->start.assign(A, 0);
    r->end.assign(A, 0);

    std::map<std::vector<uint32_t>, Variant> variants;
    std::vector<std::vector<uint32_t>> case_seq;  // per case, for case_variant

    std::vector<uint32_t> seq;       // activity sequence of the open case
    int64_t first_k = 0;             // formatted-log row of the open case's first event
    auto close_case = [&](int64_t last_k) {
        uint32_t code = r->s_case[first_k];
        r->end[r->s_act[last_k]] += 1;
        r->case_code.push_back(code);
        r->n_events.push_back((uint32_t)(last_k - first_k + 1));
        r->dur.push_back(r->s_ts[last_k] - r->s_ts[first_k]);            // R9: last - first
        r->first_row.push_back(first_k);
        Variant& v = variants[seq];
        if (v.count == 0) v.rep = code;   // cases arrive in ascending code: first = min
        v.count += 1;
        case_seq.push_back(seq);
    };
    for (int64_t k = 0; k < n; ++k) {
        bool new_case = (k == 0) || (r->s_case[k] != r->s_case[k - 1]);
        if (new_case) {
            if (k > 0) close_case(k - 1);
            first_k = k;
            seq.clear();
            r->start[r->s_act[k]] += 1;
        } else {
            // directly-follows pair (previous event of the same case, this event)
            uint32_t a = r->s_act[k - 1], b = r->s_act[k];
            int64_t d = r->s_ts[k] - r->s_ts[k - 1];
            size_t e = (size_t)a * A + b;
            r->cnt[e] += 1;                                              // R5: occurrences
            r->sum[e] = (int64_t)((uint64_t)r->sum[e] + (uint64_t)d);    // R8: mod 2^64
            r->sum_wide[e] += (__int128)d;
            const uint64_t du = (uint64_t)r->s_ts[k] - (uint64_t)r->s_ts[k - 1];  // R20
            if (r->cnt[e] == 1 || du < r->dmin[e]) r->dmin[e] = du;
            if (r->cnt[e] == 1 || du > r->dmax[e]) r->dmax[e] = du;
        }
        seq.push_back(r->s_act[k]);
    }
    if (n > 0) close_case(n - 1);

    r->mean.assign(AA, 0.0);
    for (size_t e = 0; e < AA; ++e) {
        if (r->sum_wide[e] != (__int128)r->sum[e]) r->overflow = 1;
        if (r->cnt[e] > 0) r->mean[e] = (double)r->sum[e] / (double)r->cnt[e];  // R6
    }

    // variants in output order: count desc, then representative case asc (R11)
    std::vector<std::pair<const std::vector<uint32_t>*, Variant>> vs;
    for (auto& kv : variants) vs.push_back({&kv.first, kv.second});
    std::sort(vs.begin(), vs.end(), [](const auto& x, const auto& y) {
        if (x.second.count != y.second.count) return x.second.count > y.second.count;
        return x.second.rep < y.second.rep;
    });
    std::map<std::vector<uint32_t>, uint32_t> out_index;
    r->v_off.push_back(0);
    for (size_t i = 0; i < vs.size(); ++i) {
        const auto& s = *vs[i].first;
        r->v_count.push_back(vs[i].second.count);
        r->v_len.push_back((uint32_t)s.size());
        r->v_rep.push_back(vs[i].second.rep);
        r->v_act.insert(r->v_act.end(), s.begin(), s.end());
        r->v_off.push_back(r->v_act.size());
        out_index[s] = (uint32_t)i;
    }
    for (auto& s : case_seq) r->case_variant.push_back(out_index[s]);
    r->t_loop = std::chrono::duration<double>(std::chrono::steady_clock::now() - t1).count();
    return r;
}

// per-stage wall time of the last orc_run on r (timing instrumentation only)
void orc_timing(const orc_result* r, double* sort_s, double* loop_s) {
    *sort_s = r->t_sort;
    *loop_s = r->t_loop;
}

void orc_free(orc_result* r) { delete r; }
int64_t orc_n_cases(const orc_result* r) { return (int64_t)r->case_code.size(); }
int64_t orc_n_variants(const orc_result* r) { return (int64_t)r->v_count.size(); }
int64_t orc_variants_total_len(const orc_result* r) { return (int64_t)r->v_act.size(); }
int orc_overflow(const orc_result* r) { return r->overflow; }


void orc_get_sorted(const orc_result* r, uint32_t* s_case, uint32_t* s_act, int64_t* s_ts,
                    int64_t* perm) {
    copy_out(r->s_case, s_case);
    copy_out(r->s_act, s_act);
    copy_out(r->s_ts, s_ts);
    copy_out(r->perm, perm);
}
void orc_get_dfg(const orc_result* r, uint64_t* cnt, int64_t* sum, double* mean) {
    copy_out(r->cnt, cnt);
    copy_out(r->sum, sum);
    copy_out(r->mean, mean);
}
void orc_get_dfg_minmax(const orc_result* r, uint64_t* dmin, uint64_t* dmax) {
    copy_out(r->dmin, dmin);
    copy_out(r->dmax, dmax);
}
void orc_get_start_end(const orc_result* r, uint64_t* start, uint64_t* end) {
    copy_out(r->start, start);
    copy_out(r->end, end);
}
void orc_get_cases(const orc_result* r, uint32_t* case_code, uint32_t* n_events, int64_t* dur,
                   int64_t* first_row, uint32_t* case_variant) {
    copy_out(r->case_code, case_code);
    copy_out(r->n_events, n_events);
    copy_out(r->dur, dur);
    copy_out(r->first_row, first_row);
    copy_out(r->case_variant, case_variant);
}
void orc_get_variants(const orc_result* r, uint64_t* count, uint32_t* len, uint32_t* rep,
                      uint64_t* seq_off, uint32_t* seq_act) {
    copy_out(r->v_count, count);
    copy_out(r->v_len, len);
    copy_out(r->v_rep, rep);
    copy_out(r->v_off, seq_off);
    copy_out(r->v_act, seq_act);
}

// ---------------------------------------------------------------- filters
// P:126 "three different types of timestamp filtering (events, cases
// contained, cases intersecting)".  Bounds inclusive (R12).
// mode 0 = events: keep rows with t1 <= ts <= t2.
// mode 1 = cases contained: keep every row of cases with start >= t1 and end <= t2.
// mode 2 = cases intersecting: keep every row of cases with start <= t2 and end >= t1.
// start / end are the case's first / last timestamp in the formatted log
// (S:179).  Output: keep[i] in input order.  Returns 1 (EINVAL) if t1 > t2.
int orc_filter_time(int64_t n, const uint32_t* case_, const int64_t* ts, int64_t t1, int64_t t2,
                    int mode, uint8_t* keep) {
    if (t1 > t2 || mode < 0 || mode > 2) return 1;
    if (mode == 0) {
        for (int64_t i = 0; i < n; ++i) keep[i] = (ts[i] >= t1 && ts[i] <= t2) ? 1 : 0;
        return 0;
    }
    std::vector<int64_t> idx(n);
    std::iota(idx.begin(), idx.end(), (int64_t)0);
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t i, int64_t j) {
        if (case_[i] != case_[j]) return case_[i] < case_[j];
        return ts[i] < ts[j];
    });
    std::map<uint32_t, bool> case_keep;
    for (int64_t k = 0; k < n;) {
        int64_t e = k;
        while (e + 1 < n && case_[idx[e + 1]] == case_[idx[k]]) ++e;
        int64_t start = ts[idx[k]], end = ts[idx[e]];
        bool ok = (mode == 1) ? (start >= t1 && end <= t2) : (start <= t2 && end >= t1);
        case_keep[case_[idx[k]]] = ok;
        k = e + 1;
    }
    for (int64_t i = 0; i < n; ++i) keep[i] = case_keep[case_[i]] ? 1 : 0;
    return 0;
}

// P:96-97.  Predicate on one attribute column:
//   kind 0: u32 codes, match = value in set[0..nset)
//   kind 1: i64,       match = lo_i <= value <= hi_i
//   kind 2: f64,       match = lo_f <= value <= hi_f
// valid (nullable): valid[i] == 0 means null, which never matches.
// level 0 = events: row kept iff match == keep_matching.
// level 1 = cases: row kept iff (its case has >= 1 matching row) == keep_matching
//          ("filtering the cases with at least one event with activity ...").
int orc_filter_attr(int64_t n, const uint32_t* case_, int kind, const void* col,
                    const uint8_t* valid, const uint32_t* set, int64_t nset, int64_t lo_i,
                    int64_t hi_i, double lo_f, double hi_f, int level, int keep_matching,
                    uint8_t* keep) {
    if (kind < 0 || kind > 2 || level < 0 || level > 1) return 1;
    if (kind == 1 && lo_i > hi_i) return 1;
    if (kind == 2 && !(lo_f <= hi_f)) return 1;
    std::vector<uint8_t> match(n, 0);
    for (int64_t i = 0; i < n; ++i) {
        if (valid && !valid[i]) continue;
        bool m = false;
        if (kind == 0) {
            uint32_t v = ((const uint32_t*)col)[i];
            for (int64_t s = 0; s < nset; ++s)
                if (set[s] == v) { m = true; break; }
        } else if (kind == 1) {
            int64_t v = ((const int64_t*)col)[i];
            m = (v >= lo_i && v <= hi_i);
        } else {
            double v = ((const double*)col)[i];
            m = (v >= lo_f && v <= hi_f);
        }
        match[i] = m ? 1 : 0;
    }
    if (level == 0) {
        for (int64_t i = 0; i < n; ++i) keep[i] = (match[i] == (keep_matching ? 1 : 0)) ? 1 : 0;
        return 0;
    }
    std::map<uint32_t, bool> any;
    for (int64_t i = 0; i < n; ++i) {
        bool& a = any[case_[i]];
        a = a || match[i];
    }
    for (int64_t i = 0; i < n; ++i)
        keep[i] = (any[case_[i]] == (keep_matching != 0)) ? 1 : 0;
    return 0;
}

// ---------------------------------------------------------------- case-level filters (NEXT-1)
// Whole-case filters on the formatted log (S:372-380,
// S:428-435).  The case's rows are its rows in (case, ts, ingest)
// order (step 1); match(case) is:
//   kind 0 START_IN:   first activity in codes[0..ncodes)
//   kind 1 END_IN:     last activity in codes
//   kind 2 SIZE:       lo <= n_events <= hi
//   kind 3 THROUGHPUT: lo <= last ts - first ts <= hi
//   kind 4 PATHS:      some consecutive pair (a_k, a_{k+1}) equals one of the
//                      pairs (codes[2j], codes[2j+1])
// and every row of the case is kept iff match(case) == keep_matching (keep /
// remove mode).  Returns 1 (EINVAL) on lo > hi or an odd
// number of path codes; keep[] is in input order.
int orc_filter_cases(int64_t n, const uint32_t* case_, const uint32_t* act, const int64_t* ts,
                     int kind, const uint32_t* codes, int64_t ncodes, int64_t lo, int64_t hi,
                     int keep_matching, uint8_t* keep) {
    if (kind < 0 || kind > 4) return 1;
    if ((kind == 2 || kind == 3) && lo > hi) return 1;
    if (kind == 4 && (ncodes % 2) != 0) return 1;
    std::vector<int64_t> idx(n);
    std::iota(idx.begin(), idx.end(), (int64_t)0);
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t i, int64_t j) {
        if (case_[i] != case_[j]) return case_[i] < case_[j];
        return ts[i] < ts[j];
    });
    auto in_codes = [&](uint32_t a) {
        for (int64_t s = 0; s < ncodes; ++s)
            if (codes[s] == a) return true;
        return false;
    };
    std::map<uint32_t, bool> case_keep;
    for (int64_t k = 0; k < n;) {
        int64_t e = k;
        while (e + 1 < n && case_[idx[e + 1]] == case_[idx[k]]) ++e;
        bool m = false;
        if (kind == 0) m = in_codes(act[idx[k]]);
        if (kind == 1) m = in_codes(act[idx[e]]);
        if (kind == 2) m = (e - k + 1) >= lo && (e - k + 1) <= hi;
        if (kind == 3) m = (ts[idx[e]] - ts[idx[k]]) >= lo && (ts[idx[e]] - ts[idx[k]]) <= hi;
        if (kind == 4)
            for (int64_t q = k; q < e && !m; ++q)
                for (int64_t j = 0; j + 1 < ncodes; j += 2)
                    if (act[idx[q]] == codes[j] && act[idx[q + 1]] == codes[j + 1]) m = true;
        case_keep[case_[idx[k]]] = (m == (keep_matching != 0));
        k = e + 1;
    }
    for (int64_t i = 0; i < n; ++i) keep[i] = case_keep[case_[i]] ? 1 : 0;
    return 0;
}

// filter_by_variants ("keeps/remove all the cases whose variant fall
// inside the collection"): match(case) = its exact activity
// sequence equals one of the given sequences (CSR seq_off[0..nseq], seq_act).
int orc_filter_variants(int64_t n, const uint32_t* case_, const uint32_t* act, const int64_t* ts,
                        const uint64_t* seq_off, const uint32_t* seq_act, int64_t nseq,
                        int keep_matching, uint8_t* keep) {
    std::map<std::vector<uint32_t>, bool> wanted;
    for (int64_t s = 0; s < nseq; ++s)
        wanted[std::vector<uint32_t>(seq_act + seq_off[s], seq_act + seq_off[s + 1])] = true;
    std::vector<int64_t> idx(n);
    std::iota(idx.begin(), idx.end(), (int64_t)0);
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t i, int64_t j) {
        if (case_[i] != case_[j]) return case_[i] < case_[j];
        return ts[i] < ts[j];
    });
    std::map<uint32_t, bool> case_keep;
    for (int64_t k = 0; k < n;) {
        int64_t e = k;
        std::vector<uint32_t> seq;
        seq.push_back(act[idx[k]]);
        while (e + 1 < n && case_[idx[e + 1]] == case_[idx[k]]) seq.push_back(act[idx[++e]]);
        const bool m = wanted.count(seq) > 0;
        case_keep[case_[idx[k]]] = (m == (keep_matching != 0));
        k = e + 1;
    }
    for (int64_t i = 0; i < n; ++i) keep[i] = case_keep[case_[i]] ? 1 : 0;
    return 0;
}

// ---------------------------------------------------------------- EFG + temporal profile (NEXT-3)
// P:122 "EFG retrieval / Temporal Profile (efg.py): discovers the
// eventually-follows graphs or the temporal profile".
// For every case of the formatted log (step 1) and every ordered index pair
// i < j inside it: edge (act_i, act_j) gets count += 1, sum += d and
// sumsq += d^2 with d = ts_j - ts_i >= 0 taken as u64 (R20); sum modulo 2^64
// (R8), sumsq as an exact unsigned 128-bit value ("unsigned 128-bit"),
// returned as lo / hi u64 words.  Temporal profile (reading R22): with
// m = (double)count, mean = (double)sum / m; s2 = (double)sumsq_hi * 2^64 +
// (double)sumsq_lo; V = (s2 - (double)sum * mean) / m; stdev = V > 0 ?
// sqrt(V) : 0 -- IEEE fp64 round-to-nearest, no contraction (ISO C++ mode);
// mean = stdev = 0 where count = 0.
void orc_efg(int64_t n, const uint32_t* case_, const uint32_t* act, const int64_t* ts, uint32_t A,
             uint64_t* cnt, uint64_t* sum, uint64_t* sq_lo, uint64_t* sq_hi, double* mean, double* stdev) {
    const size_t AA = (size_t)A * A;
    std::vector<uint64_t> c(AA, 0), sm(AA, 0);
    std::vector<unsigned __int128> q(AA, 0);
    std::vector<int64_t> idx(n);
    std::iota(idx.begin(), idx.end(), (int64_t)0);
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t i, int64_t j) {
        if (case_[i] != case_[j]) return case_[i] < case_[j];
        return ts[i] < ts[j];
    });
    for (int64_t k = 0; k < n;) {
        int64_t e = k;
        while (e + 1 < n && case_[idx[e + 1]] == case_[idx[k]]) ++e;
        for (int64_t x = k; x <= e; ++x)
            for (int64_t y = x + 1; y <= e; ++y) {
                const size_t ed = (size_t)act[idx[x]] * A + act[idx[y]];
                const uint64_t d = (uint64_t)ts[idx[y]] - (uint64_t)ts[idx[x]];
                c[ed] += 1;
                sm[ed] += d;
                q[ed] += (unsigned __int128)d * d;
            }
        k = e + 1;
    }
    for (size_t ed = 0; ed < AA; ++ed) {
        if (cnt) cnt[ed] = c[ed];
        if (sum) sum[ed] = sm[ed];
        if (sq_lo) sq_lo[ed] = (uint64_t)q[ed];
        if (sq_hi) sq_hi[ed] = (uint64_t)(q[ed] >> 64);
        double mu = 0.0, sd = 0.0;
        if (c[ed] > 0) {
            const double m = (double)c[ed];
            mu = (double)sm[ed] / m;
            const double s2 = (double)(uint64_t)(q[ed] >> 64) * 18446744073709551616.0 + (double)(uint64_t)q[ed];
            const double V = (s2 - (double)sm[ed] * mu) / m;
            sd = V > 0.0 ? std::sqrt(V) : 0.0;
        }
        if (mean) mean[ed] = mu;
        if (stdev) stdev[ed] = sd;
    }
}

}  // extern "C"
