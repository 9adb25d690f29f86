// Host-side trace validation and packing.
//
// Validation restates RoutingTrace.validate / AccessEvent.validate /
// TraceHeader.validate (pkg/src/moecache/trace.py:57-137): the same checks in
// the same event order, reported as MCB_ERR_INVALID (InvalidConfigError).
// Packing restates layer_schedules (pkg/src/moecache/replay.py:44-81): per
// layer stream, new_sequence on a seq_id change of that layer, prefill
// load-once dedup per (sequence, layer), positions counted per layer.
// The result is the chain-major layout of mcb.h (uniform when the trace is
// decode-only with a single sequence).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <set>
#include <string>
#include <vector>

#include "mcb_internal.h"

struct mcb_packed {
    mcb_trace view{};
    std::vector<uint8_t> acc;
    std::vector<int64_t> chain_acc_off, chain_ev_off, chain_rt_off;
    std::vector<uint32_t> ev_info;
    std::vector<uint8_t> routed;
    int64_t num_decode_steps = 0;
};

namespace {

int fail(const std::string &msg) { return mcb_set_error(MCB_ERR_INVALID, msg.c_str()); }

}  // namespace

// RoutingTrace.validate (trace.py:115-137) with TraceHeader.validate and
// AccessEvent.validate (trace.py:57-107): the same checks, the same order of
// reporting (every event's own checks and the ordering first, the
// decode-step completeness last) and the same messages.  No engine limits
// (num_experts may exceed 128 here).  Outputs the trace's shape.
static int validate_events(int32_t L, int32_t E, int32_t K, int64_t n, const int64_t *seq, const uint8_t *phase,
                           const int64_t *step, const int32_t *layer, const int64_t *off, const int32_t *experts,
                           int64_t *decode_steps_out, bool *decode_only_out, bool *single_seq_out) {
    if (L < 1) return fail("num_layers must be >= 1, got " + std::to_string(L));
    if (E < 1) return fail("num_experts must be >= 1, got " + std::to_string(E));
    if (K < 1 || K > E)
        return fail("top_k must satisfy 1 <= top_k <= num_experts, got top_k=" + std::to_string(K) +
                    " with num_experts=" + std::to_string(E));
    if (n > 0 && (!seq || !phase || !step || !layer || !off || !experts))
        return mcb_set_error(MCB_ERR_INVALID, "NULL event array");
    std::vector<uint8_t> mark(E, 0);
    std::vector<uint8_t> present(L, 0);
    bool decode_only = true, single_seq = true;
    int64_t grp_seq = -1, grp_step = -1, grp_count = 0;
    bool in_grp = false;
    std::string missing_msg;   // the first incomplete decode step, reported after every event checked
    auto close_group = [&]() {
        if (in_grp && grp_count != L && missing_msg.empty()) {
            std::string m;
            for (int32_t l = 0; l < L; ++l)
                if (!present[l]) m += (m.empty() ? "" : ", ") + std::to_string(l);
            missing_msg = "decode step (seq " + std::to_string(grp_seq) + ", step " + std::to_string(grp_step) +
                          ") missing events for layers [" + m + "]";
        }
    };
    int64_t decode_steps = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (seq[i] < 0) return fail("seq_id must be >= 0, got " + std::to_string(seq[i]));
        if (step[i] < 0) return fail("step must be >= 0, got " + std::to_string(step[i]));
        if (layer[i] < 0 || layer[i] >= L)
            return fail("layer " + std::to_string(layer[i]) + " out of range [0, " + std::to_string(L) + ")");
        if (phase[i] > 1) return fail("phase must be 0 (prefill) or 1 (decode)");
        const int64_t len = off[i + 1] - off[i];
        if (len < 0) return fail("negative expert count");
        // duplicates (set(experts) smaller than the list), any value
        bool dup = false;
        for (int64_t j = 0; j < len && !dup; ++j) {
            const int32_t e = experts[off[i] + j];
            if (e >= 0 && e < E) {
                if (mark[e]) dup = true;
                mark[e] = 1;
            } else {
                for (int64_t jj = 0; jj < j; ++jj)
                    if (experts[off[i] + jj] == e) dup = true;
            }
        }
        for (int64_t j = 0; j < len; ++j) {
            const int32_t e = experts[off[i] + j];
            if (e >= 0 && e < E) mark[e] = 0;
        }
        if (dup) {
            std::string m;
            for (int64_t j = 0; j < len; ++j) m += (j ? ", " : "") + std::to_string(experts[off[i] + j]);
            return fail("experts contain duplicates: [" + m + "]");
        }
        for (int64_t j = 0; j < len; ++j) {
            const int32_t e = experts[off[i] + j];
            if (e < 0 || e >= E)
                return fail("expert " + std::to_string(e) + " out of range [0, " + std::to_string(E) + ")");
        }
        if (phase[i] == 1) {
            if (len != K)
                return fail("decode event must route exactly top_k=" + std::to_string(K) + " experts, got " +
                            std::to_string(len));
        } else if (len < 1 || len > E) {
            return fail("prefill event must route between 1 and " + std::to_string(E) + " experts, got " +
                        std::to_string(len));
        }
        if (i > 0) {   // strict (seq, phase, step, layer) order
            const int64_t a[4] = {seq[i - 1], phase[i - 1], step[i - 1], layer[i - 1]};
            const int64_t b[4] = {seq[i], phase[i], step[i], layer[i]};
            if (!std::lexicographical_compare(a, a + 4, b, b + 4))
                return fail("events out of order at (" + std::to_string(seq[i]) + ", " + std::to_string(phase[i]) +
                            ", " + std::to_string(step[i]) + ", " + std::to_string(layer[i]) +
                            "); must be strictly increasing by (seq_id, phase, step, layer)");
        }
        if (phase[i] == 1) {
            if (!in_grp || grp_seq != seq[i] || grp_step != step[i]) {
                close_group();
                in_grp = true;
                grp_seq = seq[i];
                grp_step = step[i];
                grp_count = 0;
                std::fill(present.begin(), present.end(), 0);
                ++decode_steps;  // num_decode_steps (trace.py:139-141): distinct (seq, step)
            }
            ++grp_count;
            present[layer[i]] = 1;
        } else {
            decode_only = false;
        }
        if (seq[i] != seq[0]) single_seq = false;
    }
    close_group();
    if (!missing_msg.empty()) return fail(missing_msg);
    *decode_steps_out = decode_steps;
    *decode_only_out = decode_only;
    *single_seq_out = single_seq;
    return MCB_OK;
}

extern "C" int mcb_validate_trace(int32_t L, int32_t E, int32_t K, int64_t n, const int64_t *seq,
                                  const uint8_t *phase, const int64_t *step, const int32_t *layer,
                                  const int64_t *off, const int32_t *experts) {
    mcb_clear_error();
    int64_t d;
    bool a, b;
    return validate_events(L, E, K, n, seq, phase, step, layer, off, experts, &d, &a, &b);
}

extern "C" int mcb_pack_trace(int32_t L, int32_t E, int32_t K, int64_t n, const int64_t *seq,
                              const uint8_t *phase, const int64_t *step, const int32_t *layer,
                              const int64_t *off, const int32_t *experts, mcb_packed **out) {
    mcb_clear_error();
    if (!out) return mcb_set_error(MCB_ERR_INVALID, "out is NULL");
    *out = nullptr;
    int64_t decode_steps = 0;
    bool decode_only = true, single_seq = true;
    if (int rc = validate_events(L, E, K, n, seq, phase, step, layer, off, experts, &decode_steps, &decode_only,
                                 &single_seq))
        return rc;
    if (E > MCB_MAX_EXPERTS)
        return mcb_set_error(MCB_ERR_UNSUPPORTED, "num_experts > 128 is not supported by the B200 engine");

    auto *p = new (std::nothrow) mcb_packed();
    if (!p) return mcb_set_error(MCB_ERR_NOMEM, "out of host memory");
    p->num_decode_steps = decode_steps;
    mcb_trace &v = p->view;
    v.num_layers = L;
    v.num_experts = E;
    v.top_k = K;
    v.num_traces = 1;

    if (decode_only && single_seq) {
        // uniform: every layer has decode_steps events of K accesses; events
        // are stored (step, layer) so layer l's t-th event is event t*L + l.
        const int64_t T = decode_steps;
        v.uniform = 1;
        v.events_per_chain = T;
        p->acc.assign(((size_t)L * T * K + 127) / 128 * 128 + 128, 0);  // padded for chunked loads
        v.total_acc = (int64_t)L * T * K;
        v.total_events = (int64_t)L * T;
        for (int64_t t = 0; t < T; ++t)
            for (int32_t l = 0; l < L; ++l) {
                const int64_t i = t * L + l;
                for (int32_t k = 0; k < K; ++k)
                    p->acc[((size_t)l * T + t) * K + k] = (uint8_t)experts[off[i] + k];
            }
        v.acc = p->acc.data();
        *out = p;
        return MCB_OK;
    }

    // general layout: bucket events per layer, keeping stored order
    std::vector<int64_t> ev_count(L, 0);
    for (int64_t i = 0; i < n; ++i) ev_count[layer[i]]++;
    p->chain_ev_off.assign(L + 1, 0);
    for (int32_t l = 0; l < L; ++l) p->chain_ev_off[l + 1] = p->chain_ev_off[l] + ev_count[l];
    std::vector<int64_t> ev_idx(n);
    {
        std::vector<int64_t> fill(L, 0);
        for (int64_t i = 0; i < n; ++i) ev_idx[p->chain_ev_off[layer[i]] + fill[layer[i]]++] = i;
    }
    p->ev_info.resize(n);
    p->chain_acc_off.assign(L + 1, 0);
    p->chain_rt_off.assign(L + 1, 0);
    std::vector<uint8_t> seen(E, 0);
    for (int32_t l = 0; l < L; ++l) {
        bool have_last = false;
        int64_t last_seq = 0;
        std::fill(seen.begin(), seen.end(), 0);
        for (int64_t q = p->chain_ev_off[l]; q < p->chain_ev_off[l + 1]; ++q) {
            const int64_t i = ev_idx[q];
            const bool new_seq = !have_last || last_seq != seq[i];
            if (new_seq) {
                have_last = true;
                last_seq = seq[i];
                std::fill(seen.begin(), seen.end(), 0);
            }
            const int64_t len = off[i + 1] - off[i];
            uint32_t n_acc = 0;
            for (int64_t j = 0; j < len; ++j) {
                const int32_t e = experts[off[i] + j];
                p->routed.push_back((uint8_t)e);
                if (phase[i] == 1) {
                    p->acc.push_back((uint8_t)e);
                    ++n_acc;
                } else if (!seen[e]) {
                    p->acc.push_back((uint8_t)e);
                    ++n_acc;
                }
            }
            if (phase[i] == 0)
                for (int64_t j = 0; j < len; ++j) seen[experts[off[i] + j]] = 1;
            p->ev_info[q] = mcb_ev_pack(n_acc, (uint32_t)len, phase[i] == 1, new_seq);
        }
        p->chain_acc_off[l + 1] = (int64_t)p->acc.size();
        p->chain_rt_off[l + 1] = (int64_t)p->routed.size();
    }
    p->acc.resize(((p->acc.size() + 127) / 128 + 1) * 128, 0);  // padded for chunked loads
    if (p->routed.empty()) p->routed.push_back(0);
    if (p->ev_info.empty()) p->ev_info.push_back(0);
    v.uniform = 0;
    v.total_acc = p->chain_acc_off[L];
    v.total_events = p->chain_ev_off[L];
    v.acc = p->acc.data();
    v.chain_acc_off = p->chain_acc_off.data();
    v.chain_ev_off = p->chain_ev_off.data();
    v.chain_rt_off = p->chain_rt_off.data();
    v.ev_info = p->ev_info.data();
    v.routed = p->routed.data();
    *out = p;
    return MCB_OK;
}

extern "C" int mcb_packed_view(const mcb_packed *p, mcb_trace *view, int64_t *total_acc, int64_t *total_events,
                               int64_t *total_routed, int64_t *num_decode_steps) {
    mcb_clear_error();
    if (!p) return mcb_set_error(MCB_ERR_INVALID, "packed trace is NULL");
    if (view) *view = p->view;
    const mcb_trace &v = p->view;
    const int64_t chains = (int64_t)v.num_layers * v.num_traces;
    if (total_acc) *total_acc = v.uniform ? chains * v.events_per_chain * v.top_k : p->chain_acc_off[chains];
    if (total_events) *total_events = v.uniform ? chains * v.events_per_chain : p->chain_ev_off[chains];
    if (total_routed) *total_routed = v.uniform ? chains * v.events_per_chain * v.top_k : p->chain_rt_off[chains];
    if (num_decode_steps) *num_decode_steps = p->num_decode_steps;
    return MCB_OK;
}

extern "C" int mcb_packed_positions(const mcb_packed *p, int64_t chain, int64_t *tick, int64_t *decode_index) {
    mcb_clear_error();
    if (!p) return mcb_set_error(MCB_ERR_INVALID, "packed trace is NULL");
    const mcb_trace &v = p->view;
    const int64_t chains = (int64_t)v.num_layers * v.num_traces;
    if (chain < 0 || chain >= chains) return mcb_set_error(MCB_ERR_INVALID, "chain out of range");
    if (v.uniform) {
        for (int64_t t = 0, q = 0; t < v.events_per_chain; ++t)
            for (int32_t k = 0; k < v.top_k; ++k, ++q) {
                tick[q] = t;
                decode_index[q] = t;
            }
        return MCB_OK;
    }
    int64_t q = 0, dec = 0;
    for (int64_t e = p->chain_ev_off[chain]; e < p->chain_ev_off[chain + 1]; ++e) {
        const uint32_t info = p->ev_info[e];
        const int64_t tk = e - p->chain_ev_off[chain];
        for (uint32_t j = 0; j < mcb_ev_nacc(info); ++j, ++q) {
            tick[q] = tk;
            decode_index[q] = dec;
        }
        if (mcb_ev_decode(info)) ++dec;
    }
    return MCB_OK;
}

extern "C" int mcb_packed_free(mcb_packed *p) {
    delete p;
    return MCB_OK;
}
