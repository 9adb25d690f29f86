/*
 * oracle.c -- CPU restatement of the reference replay path.  TEST
 * INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py as the CHECKER.  The
 * product path (paper_2601_17063_b200) never links or calls this file.
 *
 * It restates, literally and in plain C, the reference algorithm of
 * FlashMoE's simulation lab (moecache 0.1.0, /root/reference/pkg/src):
 *
 *   layer_schedules          replay.py:44-81   (prefill load-once dedup,
 *                                                position0, tick, decode_index)
 *   OracleIndex.next_use     policies.py:57-76 (per-(layer,expert) sorted
 *                                                positions + bisect_right)
 *   CachePolicy.access       policies.py:95-107
 *   LRU / LFU / Belady       policies.py:132-149, 171-214
 *   FIFO / ARC / LeCaR       policies.py:152-168, 217-302, 305-395
 *   FeatureTracker           features.py:34-52
 *   EvictionNet.forward      net.py:43-53, 88-105 (float64)
 *   ml_policy_evict          mlpolicy.py:15-26
 *   MLEvictionPolicy         mlpolicy.py:47-62
 *   _replay_layer            engine.py:205-263
 *   _refetch_rate            engine.py:266-297
 *   step_latency_s           engine.py:58-62
 *
 * Victims are chosen by scanning the resident experts in ascending id order
 * with the reference's comparison (min of (key, id) / first strictly greater
 * next-use / first strictly greater score), NOT with the key reformulation
 * the CUDA engine uses -- so agreement between the two is evidence.
 *
 * Parity of this file is pinned against fixtures produced by the reference
 * itself (tests/golden/make_golden.py writes the fixtures).
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off; no FMA contraction so
 * the float64 latency sums and forward pass are plain IEEE mul/add).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_ERR_INVALID 1
#define ORC_ERR_NO_EVICTABLE 3
#define ORC_ERR_NOMEM 6

enum { ORC_LRU = 0, ORC_LFU = 1, ORC_BELADY = 2, ORC_ML = 3, ORC_FIFO = 4, ORC_ARC = 5, ORC_LECAR = 6 };
/* FIFO: policies.py:152-168; ARC: policies.py:217-302; LeCaR: policies.py:305-395 */

/* LeCaR parameters (LeCaRPolicy.__init__, policies.py:333-349) and the
 * random.Random(seed).random() stream every per-layer instance draws from
 * (one draw per eviction; produced by the caller with Python's own random
 * module).  Set with orc_set_lecar before a replay. */
static double g_lecar_lr = 0.45, g_lecar_base = 0.005;
static const double *g_lecar_u = NULL;
static int64_t g_lecar_n = 0;

void orc_set_lecar(double learning_rate, double discount_base, const double *u, int64_t n) {
    g_lecar_lr = learning_rate;
    g_lecar_base = discount_base;
    g_lecar_u = u;
    g_lecar_n = n;
}

#define OUT_HIT 0xFFFFu
#define OUT_MISS 0xFFFEu

/* per-layer counter slots (mirrors engine.py:213-217 + _refetch_rate) */
enum { C_PH = 0, C_PM, C_DH, C_DM, C_COMP, C_EVICT, C_REFETCH, C_N };

typedef struct {
    int phase;        /* 0 prefill, 1 decode */
    int new_seq;
    int n_routed;
    const int32_t *routed;
    int n_acc;
    int32_t *acc;     /* owned copy (prefill dedup) */
    int64_t position0;
    int64_t tick;
    int64_t decode_index;
} orc_step;

typedef struct {
    int64_t n_steps;
    orc_step *steps;
    int64_t n_acc;    /* total accesses = stream length */
    int32_t *stream;  /* flattened accesses (build_oracle_index, replay.py:84-89) */
    int64_t *dec_of;  /* decode index of each position (engine.py:278-288) */
} orc_layer;

/* ------------------------------------------------------------------ */
/* layer_schedules (replay.py:44-81)                                    */
/* ------------------------------------------------------------------ */

static void free_layers(orc_layer *ls, int L) {
    if (!ls) return;
    for (int l = 0; l < L; ++l) {
        for (int64_t s = 0; s < ls[l].n_steps; ++s) free(ls[l].steps[s].acc);
        free(ls[l].steps);
        free(ls[l].stream);
        free(ls[l].dec_of);
    }
    free(ls);
}

static orc_layer *build_layers(int L, int E, int64_t n_events, const int64_t *seq,
                               const uint8_t *phase, const int32_t *layer,
                               const int64_t *exp_off, const int32_t *experts) {
    orc_layer *ls = (orc_layer *)calloc((size_t)L, sizeof(orc_layer));
    int64_t *cap = (int64_t *)calloc((size_t)L, sizeof(int64_t));
    int64_t *pos = (int64_t *)calloc((size_t)L, sizeof(int64_t));
    int64_t *dcount = (int64_t *)calloc((size_t)L, sizeof(int64_t));
    int64_t *last_seq = (int64_t *)malloc((size_t)L * sizeof(int64_t));
    int *has_last = (int *)calloc((size_t)L, sizeof(int));
    uint8_t *seen = (uint8_t *)calloc((size_t)L * (size_t)E, 1);
    if (!ls || !cap || !pos || !dcount || !last_seq || !has_last || !seen) goto fail;

    for (int64_t i = 0; i < n_events; ++i) {
        int l = layer[i];
        orc_layer *ly = &ls[l];
        if (ly->n_steps == cap[l]) {
            cap[l] = cap[l] ? cap[l] * 2 : 64;
            orc_step *ns = (orc_step *)realloc(ly->steps, (size_t)cap[l] * sizeof(orc_step));
            if (!ns) goto fail;
            ly->steps = ns;
        }
        orc_step *st = &ly->steps[ly->n_steps];
        memset(st, 0, sizeof(*st));
        int new_seq = !has_last[l] || last_seq[l] != seq[i];
        if (new_seq) {
            has_last[l] = 1;
            last_seq[l] = seq[i];
            memset(seen + (size_t)l * E, 0, (size_t)E);
        }
        int n = (int)(exp_off[i + 1] - exp_off[i]);
        const int32_t *ex = experts + exp_off[i];
        st->acc = (int32_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int32_t));
        if (!st->acc) goto fail;
        int na = 0;
        if (phase[i] == 0) {
            /* prefill: drop experts already seen in this (seq, layer) prefill */
            uint8_t *sn = seen + (size_t)l * E;
            for (int j = 0; j < n; ++j)
                if (!sn[ex[j]]) st->acc[na++] = ex[j];
            for (int j = 0; j < n; ++j) sn[ex[j]] = 1;
        } else {
            for (int j = 0; j < n; ++j) st->acc[na++] = ex[j];
        }
        st->phase = phase[i];
        st->new_seq = new_seq;
        st->n_routed = n;
        st->routed = ex;
        st->n_acc = na;
        st->position0 = pos[l];
        st->tick = ly->n_steps;
        st->decode_index = dcount[l];
        ly->n_steps++;
        pos[l] += na;
        if (phase[i] == 1) dcount[l]++;
    }
    for (int l = 0; l < L; ++l) {
        orc_layer *ly = &ls[l];
        ly->n_acc = pos[l];
        ly->stream = (int32_t *)malloc((size_t)(pos[l] > 0 ? pos[l] : 1) * sizeof(int32_t));
        ly->dec_of = (int64_t *)malloc((size_t)(pos[l] > 0 ? pos[l] : 1) * sizeof(int64_t));
        if (!ly->stream || !ly->dec_of) goto fail;
        int64_t p = 0;
        for (int64_t s = 0; s < ly->n_steps; ++s)
            for (int j = 0; j < ly->steps[s].n_acc; ++j) {
                ly->stream[p] = ly->steps[s].acc[j];
                ly->dec_of[p] = ly->steps[s].decode_index;
                ++p;
            }
    }
    free(cap); free(pos); free(dcount); free(last_seq); free(has_last); free(seen);
    return ls;
fail:
    free(cap); free(pos); free(dcount); free(last_seq); free(has_last); free(seen);
    free_layers(ls, L);
    return NULL;
}

/* ------------------------------------------------------------------ */
/* OracleIndex (policies.py:51-76): positions per expert + bisect_right */
/* ------------------------------------------------------------------ */

typedef struct {
    int E;
    int64_t *off;   /* [E+1] */
    int64_t *pos;   /* positions grouped by expert, ascending */
} orc_index;

static int index_build(orc_index *ix, const orc_layer *ly, int E) {
    ix->E = E;
    ix->off = (int64_t *)calloc((size_t)E + 1, sizeof(int64_t));
    ix->pos = (int64_t *)malloc((size_t)(ly->n_acc > 0 ? ly->n_acc : 1) * sizeof(int64_t));
    int64_t *fill = (int64_t *)calloc((size_t)E, sizeof(int64_t));
    if (!ix->off || !ix->pos || !fill) { free(fill); return -1; }
    for (int64_t p = 0; p < ly->n_acc; ++p) ix->off[ly->stream[p] + 1]++;
    for (int e = 0; e < E; ++e) ix->off[e + 1] += ix->off[e];
    for (int64_t p = 0; p < ly->n_acc; ++p) {
        int e = ly->stream[p];
        ix->pos[ix->off[e] + fill[e]++] = p;
    }
    free(fill);
    return 0;
}

static void index_free(orc_index *ix) { free(ix->off); free(ix->pos); }

/* index of the first stored position > p (bisect_right) */
static int64_t bisect_right(const int64_t *a, int64_t n, int64_t p) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
        int64_t mid = (lo + hi) / 2;
        if (p < a[mid]) hi = mid; else lo = mid + 1;
    }
    return lo;
}

/* next_use distance; returns -1 for math.inf */
static int64_t next_use(const orc_index *ix, int e, int64_t p) {
    const int64_t *a = ix->pos + ix->off[e];
    int64_t n = ix->off[e + 1] - ix->off[e];
    if (n == 0) return -1;
    int64_t i = bisect_right(a, n, p);
    if (i == n) return -1;
    return a[i] - p;
}

/* ------------------------------------------------------------------ */
/* EvictionNet.forward, float64 (net.py:43-53, 88-105)                  */
/* ------------------------------------------------------------------ */

static double sigmoid_ref(double z) {
    if (z >= 0) return 1.0 / (1.0 + exp(-z));
    double ez = exp(z);
    return ez / (1.0 + ez);
}

/* params: w1[H][2E] b1[H] w2[H][H] b2[H] w3[E][H] b3[E], row-major */
void orc_net_forward(const double *params, int E, int H, const double *x, double *out,
                     double *h1, double *h2) {
    const int D = 2 * E;
    const double *w1 = params, *b1 = w1 + (size_t)H * D, *w2 = b1 + H, *b2 = w2 + (size_t)H * H,
                 *w3 = b2 + H, *b3 = w3 + (size_t)E * H;
    for (int i = 0; i < H; ++i) {
        double s = 0.0;
        for (int j = 0; j < D; ++j) s += w1[(size_t)i * D + j] * x[j];
        double z = s + b1[i];
        h1[i] = z * sigmoid_ref(z);
    }
    for (int i = 0; i < H; ++i) {
        double s = 0.0;
        for (int j = 0; j < H; ++j) s += w2[(size_t)i * H + j] * h1[j];
        double z = s + b2[i];
        h2[i] = z * sigmoid_ref(z);
    }
    for (int i = 0; i < E; ++i) {
        double s = 0.0;
        for (int j = 0; j < H; ++j) s += w3[(size_t)i * H + j] * h2[j];
        out[i] = s + b3[i];
    }
}

size_t orc_net_param_count(int E, int H) {
    return (size_t)H * 2 * E + H + (size_t)H * H + H + (size_t)E * H + E;
}

/* ------------------------------------------------------------------ */
/* one layer replay (engine.py:205-263 with policies.py / mlpolicy.py)  */
/* ------------------------------------------------------------------ */

typedef struct {
    int policy;
    int include_prefill;
    int capacity;
    double t_load, t_compute, ml_cost;
    int loads_serial;
    int window;
    int E, H;
    const double *net;          /* this layer's params (ML only) */
} orc_cfg;

#define FNV_OFF 0xCBF29CE484222325ull
#define FNV_PRIME 0x100000001B3ull

static inline uint64_t fnv16(uint64_t h, uint16_t c) {
    h ^= (uint64_t)(c & 0xFF); h *= FNV_PRIME;
    h ^= (uint64_t)(c >> 8);   h *= FNV_PRIME;
    return h;
}

/* Spliceable decision hash used by the CUDA engine: h = h * P + (code + 1)
 * mod 2^64 over the per-access outcome codes, so h(AB) = h(A) * P^|B| + h(B).
 * (FNV-1a above is the hash stored in the reference-made fixtures.) */
static inline uint64_t poly16(uint64_t h, uint16_t c) { return h * FNV_PRIME + (uint64_t)c + 1u; }

/* evictions list for _refetch_rate (engine.py:266-297) */
typedef struct { int64_t pos, decode_index; int victim; } evrec;

/* ---- ARC (policies.py:217-302): T1/T2 resident, B1/B2 ghosts, each an LRU-
 * ordered list; list membership per expert plus an insertion clock gives the
 * OrderedDict order (LRU end = smallest clock). */
enum { ARC_NONE = 0, ARC_T1 = 1, ARC_T2 = 2, ARC_B1 = 3, ARC_B2 = 4 };
typedef struct {
    int E, C;
    uint8_t *lst;
    int64_t *ord;
    int64_t clock;
    int n[5];
    double p;
} arc_state;

static void arc_put(arc_state *a, int e, int l) {   /* append at the MRU end of list l */
    if (a->lst[e]) a->n[a->lst[e]]--;
    a->lst[e] = (uint8_t)l;
    a->ord[e] = a->clock++;
    a->n[l]++;
}
static void arc_del(arc_state *a, int e) {
    if (a->lst[e]) a->n[a->lst[e]]--;
    a->lst[e] = ARC_NONE;
}
/* LRU end of list l, skipping pinned experts when pinned != NULL; -1 if none */
static int arc_lru(const arc_state *a, int l, const uint8_t *pinned) {
    int best = -1;
    for (int e = 0; e < a->E; ++e)
        if (a->lst[e] == l && !(pinned && pinned[e]) && (best < 0 || a->ord[e] < a->ord[best])) best = e;
    return best;
}
/* _replace (policies.py:236-254): returns the victim or -1 (NoEvictableError) */
static int arc_replace(arc_state *a, int in_b2, const uint8_t *pinned) {
    const int use_t1 = a->n[ARC_T1] >= 1 &&
                       ((double)a->n[ARC_T1] > a->p || (in_b2 && (double)a->n[ARC_T1] == a->p));
    const int src[2] = {use_t1 ? ARC_T1 : ARC_T2, use_t1 ? ARC_T2 : ARC_T1};
    for (int i = 0; i < 2; ++i) {
        const int v = arc_lru(a, src[i], pinned);
        if (v >= 0) {
            arc_put(a, v, src[i] == ARC_T1 ? ARC_B1 : ARC_B2);
            return v;
        }
    }
    return -1;
}
/* ARCPolicy.access (policies.py:256-302): *victim = evicted expert or -1;
 * returns 0, or -1 for NoEvictableError */
static int arc_access(arc_state *a, int x, const uint8_t *pinned, int *victim) {
    *victim = -1;
    if (a->lst[x] == ARC_T1 || a->lst[x] == ARC_T2) {
        arc_put(a, x, ARC_T2);
        return 0;
    }
    const int c = a->C;
    const int full = a->n[ARC_T1] + a->n[ARC_T2] >= c;
    if (a->lst[x] == ARC_B1) {
        double q = (double)a->n[ARC_B2] / (double)a->n[ARC_B1];
        if (q < 1.0) q = 1.0;
        const double np = a->p + q;
        a->p = (double)c <= np ? (double)c : np;
        if (full && (*victim = arc_replace(a, 0, pinned)) < 0) return -1;
        arc_put(a, x, ARC_T2);
    } else if (a->lst[x] == ARC_B2) {
        double q = (double)a->n[ARC_B1] / (double)a->n[ARC_B2];
        if (q < 1.0) q = 1.0;
        const double np = a->p - q;
        a->p = 0.0 >= np ? 0.0 : np;
        if (full && (*victim = arc_replace(a, 1, pinned)) < 0) return -1;
        arc_put(a, x, ARC_T2);
    } else {
        const int l1 = a->n[ARC_T1] + a->n[ARC_B1];
        if (l1 == c) {
            if (a->n[ARC_T1] < c) {
                arc_del(a, arc_lru(a, ARC_B1, NULL));
                if (a->n[ARC_T1] + a->n[ARC_T2] >= c && (*victim = arc_replace(a, 0, pinned)) < 0) return -1;
            } else {
                const int v = arc_lru(a, ARC_T1, pinned);   /* T1's LRU, no ghost entry */
                if (v < 0) return -1;
                arc_del(a, v);
                *victim = v;
            }
        } else if (l1 < c) {
            const int total = l1 + a->n[ARC_T2] + a->n[ARC_B2];
            if (total >= c) {
                if (total == 2 * c) arc_del(a, arc_lru(a, ARC_B2, NULL));
                if (a->n[ARC_T1] + a->n[ARC_T2] >= c && (*victim = arc_replace(a, 0, pinned)) < 0) return -1;
            }
        }
        arc_put(a, x, ARC_T1);
    }
    return 0;
}

static int replay_layer(const orc_layer *ly, const orc_cfg *cfg, int64_t *cnt, double *lat,
                        uint16_t *outcomes, uint64_t *hash /* [2]: fnv, poly */) {
    const int E = cfg->E, C = cfg->capacity;
    int rc = ORC_OK;
    uint8_t *res = (uint8_t *)calloc((size_t)E, 1);
    uint8_t *pinned = (uint8_t *)calloc((size_t)E, 1);
    uint8_t *seen = (uint8_t *)calloc((size_t)E, 1);
    int64_t *stamp = (int64_t *)calloc((size_t)E, sizeof(int64_t));
    int64_t *freq = (int64_t *)calloc((size_t)E, sizeof(int64_t));
    double *rec = (double *)malloc((size_t)E * sizeof(double));
    int64_t *fr = (int64_t *)calloc((size_t)E, sizeof(int64_t));
    double *x = (double *)malloc((size_t)2 * E * sizeof(double));
    double *scores = (double *)calloc((size_t)E, sizeof(double));
    double *h1 = (double *)malloc((size_t)(cfg->H > 0 ? cfg->H : 1) * sizeof(double));
    double *h2 = (double *)malloc((size_t)(cfg->H > 0 ? cfg->H : 1) * sizeof(double));
    int64_t ev_cap = 1024, n_ev = 0;
    evrec *evs = (evrec *)malloc((size_t)ev_cap * sizeof(evrec));
    orc_index ix = {0};
    int have_ix = 0;
    arc_state arc = {E, C, NULL, NULL, 0, {0, 0, 0, 0, 0}, 0.0};
    uint8_t *ghost = (uint8_t *)calloc((size_t)E, 1);
    int64_t *gpos = (int64_t *)calloc((size_t)E, sizeof(int64_t));
    if (!res || !pinned || !seen || !stamp || !freq || !rec || !fr || !x || !scores || !h1 || !h2 || !evs || !ghost ||
        !gpos) {
        rc = ORC_ERR_NOMEM; goto done;
    }
    if (index_build(&ix, ly, E) != 0) { rc = ORC_ERR_NOMEM; goto done; }
    have_ix = 1;
    for (int e = 0; e < E; ++e) rec[e] = INFINITY;

    int n_res = 0;
    int64_t fifo_clock = 0;
    /* LeCaR: ghost membership (1 lru, 2 lfu) + eviction position, weights, draws */
    int n_ghost[3] = {0, 0, 0};
    double w_lru = 0.5, w_lfu = 0.5;
    const double discount = pow(g_lecar_base, 1.0 / (double)C);   /* discount_base ** (1.0 / capacity) */
    int64_t n_draw = 0;
    if (cfg->policy == ORC_ARC) {
        arc.lst = (uint8_t *)calloc((size_t)E, 1);
        arc.ord = (int64_t *)calloc((size_t)E, sizeof(int64_t));
        if (!arc.lst || !arc.ord) { rc = ORC_ERR_NOMEM; goto done; }
    }
    uint64_t h = FNV_OFF, hp = 0;
    double dlat = 0.0, plat = 0.0;
    for (int k = 0; k < C_N; ++k) cnt[k] = 0;

    for (int64_t s = 0; s < ly->n_steps; ++s) {
        const orc_step *st = &ly->steps[s];
        if (st->new_seq) {
            /* start_sequence: LFU counts (policies.py:184-185), ML tracker (mlpolicy.py:56-57) */
            if (cfg->policy == ORC_LFU || cfg->policy == ORC_LECAR) memset(freq, 0, (size_t)E * sizeof(int64_t));
            if (cfg->policy == ORC_ML) {
                for (int e = 0; e < E; ++e) { rec[e] = INFINITY; fr[e] = 0; }
            }
        }
        if (cfg->policy == ORC_ML) {
            /* begin_event (mlpolicy.py:59-62) */
            if (st->phase == 1 || cfg->include_prefill) {
                for (int e = 0; e < E; ++e) rec[e] += 1.0;
                for (int j = 0; j < st->n_routed; ++j) { rec[st->routed[j]] = 1.0; fr[st->routed[j]] += 1; }
            }
            int64_t maxf = 0;
            for (int e = 0; e < E; ++e) if (fr[e] > maxf) maxf = fr[e];
            for (int e = 0; e < E; ++e) {
                x[e] = 1.0 / rec[e];
                x[E + e] = maxf > 0 ? (double)fr[e] / (double)maxf : 0.0;
            }
            orc_net_forward(cfg->net, E, cfg->H, x, scores, h1, h2);
        }
        const int decode = st->phase == 1;
        memset(pinned, 0, (size_t)E);
        int64_t step_misses = 0;
        int64_t pos = st->position0;
        for (int j = 0; j < st->n_acc; ++j, ++pos) {
            const int xe = st->acc[j];
            int hit = res[xe];
            int victim = -1;
            if (cfg->policy == ORC_ARC) {
                /* ARC overrides access() entirely; the resident set is T1 u T2 */
                if (arc_access(&arc, xe, decode ? pinned : NULL, &victim) != 0) { rc = ORC_ERR_NO_EVICTABLE; goto done; }
                if (!hit) {
                    if (victim >= 0) { res[victim] = 0; n_res--; }
                    res[xe] = 1;
                    n_res++;
                }
            } else if (hit) {
                if (cfg->policy == ORC_LRU || cfg->policy == ORC_LECAR) stamp[xe] = pos;
                if (cfg->policy == ORC_LFU || cfg->policy == ORC_LECAR) freq[xe] += 1;
            } else {
                if (cfg->policy == ORC_LFU || cfg->policy == ORC_LECAR) freq[xe] += 1;   /* _on_miss */
                if (cfg->policy == ORC_LECAR && ghost[xe]) {
                    /* ghost hit: lecar_update (policies.py:305-327, 358-367) */
                    const double reward = pow(discount, (double)(pos - gpos[xe]));
                    if (ghost[xe] == 1) w_lfu *= exp(g_lecar_lr * reward);
                    else w_lru *= exp(g_lecar_lr * reward);
                    const double total = w_lru + w_lfu;
                    w_lru = w_lru / total;
                    w_lfu = w_lfu / total;
                    n_ghost[ghost[xe]]--;
                    ghost[xe] = 0;
                }
                if (n_res >= C && cfg->policy == ORC_LECAR) {
                    /* _choose_victim (policies.py:379-395) */
                    int any = 0;
                    for (int e = 0; e < E; ++e) any |= res[e] && !(decode && pinned[e]);
                    if (!any) { rc = ORC_ERR_NO_EVICTABLE; goto done; }
                    if (n_draw >= g_lecar_n) { rc = ORC_ERR_INVALID; goto done; }
                    const int use_lru = g_lecar_u[n_draw++] < w_lru;
                    int64_t bk = 0;
                    for (int e = 0; e < E; ++e) {
                        if (!res[e] || (decode && pinned[e])) continue;
                        const int64_t kk = use_lru ? stamp[e] : freq[e];
                        if (victim < 0 || kk < bk) { victim = e; bk = kk; }
                    }
                    const int g = use_lru ? 1 : 2;
                    ghost[victim] = (uint8_t)g;
                    gpos[victim] = pos;
                    if (++n_ghost[g] > C) {   /* popitem(last=False): the oldest entry */
                        int o = -1;
                        for (int e = 0; e < E; ++e)
                            if (ghost[e] == g && (o < 0 || gpos[e] < gpos[o])) o = e;
                        ghost[o] = 0;
                        n_ghost[g]--;
                    }
                    res[victim] = 0;
                    n_res--;
                } else if (n_res >= C) {
                    if (cfg->policy == ORC_LRU || cfg->policy == ORC_LFU || cfg->policy == ORC_FIFO) {
                        int64_t bk = 0;
                        for (int e = 0; e < E; ++e) {
                            if (!res[e] || (decode && pinned[e])) continue;
                            /* FIFO: min (arrival clock, id) (policies.py:168); arrival
                             * is kept in stamp[] (written at insertion only) */
                            int64_t kk = (cfg->policy == ORC_LRU || cfg->policy == ORC_FIFO) ? stamp[e] : freq[e];
                            if (victim < 0 || kk < bk) { victim = e; bk = kk; }
                        }
                    } else if (cfg->policy == ORC_BELADY) {
                        /* best_dist = -1.0; d > best_dist over sorted ids; inf > finite */
                        int best_inf = 0;
                        int64_t best = -1;
                        int any = 0;
                        for (int e = 0; e < E; ++e) {
                            if (!res[e] || (decode && pinned[e])) continue;
                            any = 1;
                            int64_t d = next_use(&ix, e, pos);
                            if (best_inf) continue;
                            if (d < 0) { victim = e; best_inf = 1; }
                            else if (d > best) { victim = e; best = d; }
                        }
                        if (!any) victim = -1;
                    } else {
                        double best = -INFINITY;
                        for (int e = 0; e < E; ++e) {
                            if (!res[e] || (decode && pinned[e])) continue;
                            if (scores[e] > best) { victim = e; best = scores[e]; }
                        }
                    }
                    if (victim < 0) { rc = ORC_ERR_NO_EVICTABLE; goto done; }
                    res[victim] = 0;
                    n_res--;
                }
                res[xe] = 1;
                n_res++;
                if (cfg->policy == ORC_LRU || cfg->policy == ORC_LECAR) stamp[xe] = pos;   /* _on_insert */
                if (cfg->policy == ORC_FIFO) stamp[xe] = fifo_clock++;   /* FIFOPolicy._on_insert */
            }
            /* engine-side accounting (engine.py:243-257) */
            if (hit) {
                cnt[decode ? C_DH : C_PH]++;
            } else {
                cnt[decode ? C_DM : C_PM]++;
                step_misses++;
                if (!seen[xe]) cnt[C_COMP]++;
            }
            seen[xe] = 1;
            uint16_t code = hit ? OUT_HIT : (victim < 0 ? OUT_MISS : (uint16_t)victim);
            if (victim >= 0) {
                if (n_ev == ev_cap) {
                    ev_cap *= 2;
                    evrec *ne = (evrec *)realloc(evs, (size_t)ev_cap * sizeof(evrec));
                    if (!ne) { rc = ORC_ERR_NOMEM; goto done; }
                    evs = ne;
                }
                evs[n_ev].pos = pos;
                evs[n_ev].decode_index = st->decode_index;
                evs[n_ev].victim = victim;
                n_ev++;
            }
            if (outcomes) outcomes[pos] = code;
            h = fnv16(h, code);
            hp = poly16(hp, code);
            if (decode) pinned[xe] = 1;
        }
        /* step_latency_s (engine.py:58-62) and accumulation (engine.py:258-262) */
        double latency;
        if (step_misses > 0)
            latency = (double)(cfg->loads_serial ? step_misses : 1) * cfg->t_load;
        else
            latency = (double)st->n_acc * cfg->t_compute;
        if (decode)
            dlat += latency + (cfg->policy == ORC_ML ? cfg->ml_cost : 0.0);
        else
            plat += latency;
    }
    cnt[C_EVICT] = n_ev;
    /* _refetch_rate numerator (engine.py:289-296) */
    for (int64_t i = 0; i < n_ev; ++i) {
        const int64_t *a = ix.pos + ix.off[evs[i].victim];
        int64_t n = ix.off[evs[i].victim + 1] - ix.off[evs[i].victim];
        int64_t j = bisect_right(a, n, evs[i].pos);
        if (j < n && ly->dec_of[a[j]] - evs[i].decode_index <= cfg->window) cnt[C_REFETCH]++;
    }
    lat[0] = dlat;
    lat[1] = plat;
    if (hash) { hash[0] = h; hash[1] = hp; }
done:
    if (have_ix) index_free(&ix);
    free(res); free(pinned); free(seen); free(stamp); free(freq); free(rec); free(fr);
    free(x); free(scores); free(h1); free(h2); free(evs);
    free(arc.lst); free(arc.ord); free(ghost); free(gpos);
    return rc;
}

/* ------------------------------------------------------------------ */
/* public entry points                                                  */
/* ------------------------------------------------------------------ */

/*
 * Simulate one trace under one (policy, capacity).  The trace is flat:
 * events in stored order with seq/phase/layer and CSR experts.
 * Outputs per layer: cnt[L][C_N], lat[L][2] (decode, prefill), hashes[L][2] (fnv, poly);
 * outcomes (optional) are written at outcome_off[l] + position.
 * The caller folds layers in layer order (engine.py:330-343).
 */
int orc_simulate(int L, int E, int64_t n_events, const int64_t *seq, const uint8_t *phase,
                 const int32_t *layer, const int64_t *exp_off, const int32_t *experts,
                 int policy, int include_prefill, int capacity, double t_load, double t_compute,
                 int loads_serial, double ml_cost, int window, int H, int n_nets,
                 const double *nets, int64_t *cnt, double *lat, uint64_t *hashes,
                 uint16_t *outcomes, const int64_t *outcome_off, int64_t *layer_len) {
    orc_layer *ls = build_layers(L, E, n_events, seq, phase, layer, exp_off, experts);
    if (!ls) return ORC_ERR_NOMEM;
    int rc = ORC_OK;
    size_t np = orc_net_param_count(E, H);
    for (int l = 0; l < L && rc == ORC_OK; ++l) {
        orc_cfg cfg = {policy, include_prefill, capacity, t_load, t_compute, ml_cost, loads_serial,
                       window, E, H, NULL};
        if (policy == ORC_ML) cfg.net = nets + (n_nets == 1 ? 0 : (size_t)l * np);
        if (layer_len) layer_len[l] = ls[l].n_acc;
        rc = replay_layer(&ls[l], &cfg, cnt + (size_t)l * C_N, lat + 2 * l,
                          outcomes ? outcomes + outcome_off[l] : NULL, hashes ? hashes + 2 * l : NULL);
    }
    free_layers(ls, L);
    return rc;
}

/* Per-layer access-stream lengths (for sizing the outcomes buffer). */
int orc_layer_lengths(int L, int E, int64_t n_events, const int64_t *seq, const uint8_t *phase,
                      const int32_t *layer, const int64_t *exp_off, const int32_t *experts,
                      int64_t *layer_len) {
    orc_layer *ls = build_layers(L, E, n_events, seq, phase, layer, exp_off, experts);
    if (!ls) return ORC_ERR_NOMEM;
    for (int l = 0; l < L; ++l) layer_len[l] = ls[l].n_acc;
    free_layers(ls, L);
    return ORC_OK;
}

/* --------------- batched decode-only chains (CPU baseline) --------------- */

/*
 * A "uniform" workload: n_chains independent decode-only single-sequence
 * layer streams of T events x K experts (ids[chain][T][K], uint8), each
 * replayed under every (policy, capacity) job.  This is exactly what
 * simulate() does per layer for a decode-only trace; it is split into jobs
 * so the host baseline can use every core (the reference's sweep(jobs) is
 * thread-based and GIL-bound).
 */
typedef struct {
    const uint8_t *ids;
    int T, K, E, H;
    int64_t n_chains;
    const int32_t *job_policy, *job_cap;   /* per job */
    int n_jobs;                             /* jobs per chain */
    const double *nets;                     /* per chain layer: nets[chain % n_nets] */
    int n_nets;
    int layers_per_trace;
    double t_load, t_compute, ml_cost;
    int loads_serial, window;
    int64_t *cnt;     /* [chain][job][C_N] */
    double *lat;      /* [chain][job][2] */
    uint64_t *hash;   /* [chain][job][2] (fnv, poly) */
    int64_t next;     /* work counter */
    pthread_mutex_t mu;
    int rc;
} batch_t;

static void *batch_worker(void *arg) {
    batch_t *b = (batch_t *)arg;
    const int T = b->T, K = b->K;
    int64_t n_acc = (int64_t)T * K;
    orc_layer ly;
    memset(&ly, 0, sizeof(ly));
    ly.n_steps = T;
    ly.n_acc = n_acc;
    ly.steps = (orc_step *)calloc((size_t)T, sizeof(orc_step));
    ly.stream = (int32_t *)malloc((size_t)(n_acc > 0 ? n_acc : 1) * sizeof(int32_t));
    ly.dec_of = (int64_t *)malloc((size_t)(n_acc > 0 ? n_acc : 1) * sizeof(int64_t));
    if (!ly.steps || !ly.stream || !ly.dec_of) { b->rc = ORC_ERR_NOMEM; goto out; }
    size_t np = orc_net_param_count(b->E, b->H);
    for (;;) {
        pthread_mutex_lock(&b->mu);
        int64_t w = b->next++;
        pthread_mutex_unlock(&b->mu);
        if (w >= b->n_chains * b->n_jobs) break;
        int64_t c = w / b->n_jobs;
        int j = (int)(w % b->n_jobs);
        const uint8_t *src = b->ids + (size_t)c * n_acc;
        for (int64_t p = 0; p < n_acc; ++p) { ly.stream[p] = src[p]; ly.dec_of[p] = p / K; }
        for (int t = 0; t < T; ++t) {
            orc_step *st = &ly.steps[t];
            st->phase = 1; st->new_seq = (t == 0); st->n_routed = K;
            st->routed = ly.stream + (size_t)t * K;
            st->acc = ly.stream + (size_t)t * K;
            st->n_acc = K; st->position0 = (int64_t)t * K; st->tick = t; st->decode_index = t;
        }
        int layer = (int)(c % b->layers_per_trace);
        orc_cfg cfg = {b->job_policy[j], 1, b->job_cap[j], b->t_load, b->t_compute, b->ml_cost,
                       b->loads_serial, b->window, b->E, b->H,
                       b->nets ? b->nets + (size_t)(layer % b->n_nets) * np : NULL};
        int rc = replay_layer(&ly, &cfg, b->cnt + ((size_t)c * b->n_jobs + j) * C_N,
                              b->lat + ((size_t)c * b->n_jobs + j) * 2, NULL,
                              b->hash + ((size_t)c * b->n_jobs + j) * 2);
        if (rc) b->rc = rc;
    }
out:
    free(ly.steps); free(ly.stream); free(ly.dec_of);
    return NULL;
}

int orc_replay_uniform(const uint8_t *ids, int64_t n_chains, int layers_per_trace, int T, int K,
                       int E, int n_jobs, const int32_t *job_policy, const int32_t *job_cap,
                       double t_load, double t_compute, int loads_serial, double ml_cost,
                       int window, int H, int n_nets, const double *nets, int n_threads,
                       int64_t *cnt, double *lat, uint64_t *hash) {
    batch_t b;
    memset(&b, 0, sizeof(b));
    b.ids = ids; b.T = T; b.K = K; b.E = E; b.H = H; b.n_chains = n_chains;
    b.job_policy = job_policy; b.job_cap = job_cap; b.n_jobs = n_jobs;
    b.nets = nets; b.n_nets = n_nets > 0 ? n_nets : 1; b.layers_per_trace = layers_per_trace;
    b.t_load = t_load; b.t_compute = t_compute; b.ml_cost = ml_cost;
    b.loads_serial = loads_serial; b.window = window;
    b.cnt = cnt; b.lat = lat; b.hash = hash;
    pthread_mutex_init(&b.mu, NULL);
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = (pthread_t *)malloc((size_t)n_threads * sizeof(pthread_t));
    if (!th) return ORC_ERR_NOMEM;
    for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, batch_worker, &b);
    for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&b.mu);
    return b.rc;
}

/* Per-event fp64 scores of one decode-only chain (tests of the GPU scorer). */
int orc_score_chain(const uint8_t *ids, int T, int K, int E, int H, const double *net,
                    double *scores /* [T][E] */) {
    double *rec = (double *)malloc((size_t)E * sizeof(double));
    int64_t *fr = (int64_t *)calloc((size_t)E, sizeof(int64_t));
    double *x = (double *)malloc((size_t)2 * E * sizeof(double));
    double *h1 = (double *)malloc((size_t)H * sizeof(double));
    double *h2 = (double *)malloc((size_t)H * sizeof(double));
    if (!rec || !fr || !x || !h1 || !h2) { free(rec); free(fr); free(x); free(h1); free(h2); return ORC_ERR_NOMEM; }
    for (int e = 0; e < E; ++e) rec[e] = INFINITY;
    for (int t = 0; t < T; ++t) {
        for (int e = 0; e < E; ++e) rec[e] += 1.0;
        for (int j = 0; j < K; ++j) { int e = ids[(size_t)t * K + j]; rec[e] = 1.0; fr[e] += 1; }
        int64_t maxf = 0;
        for (int e = 0; e < E; ++e) if (fr[e] > maxf) maxf = fr[e];
        for (int e = 0; e < E; ++e) {
            x[e] = 1.0 / rec[e];
            x[E + e] = maxf > 0 ? (double)fr[e] / (double)maxf : 0.0;
        }
        orc_net_forward(net, E, H, x, scores + (size_t)t * E, h1, h2);
    }
    free(rec); free(fr); free(x); free(h1); free(h2);
    return ORC_OK;
}

/* ------------------- the reference's synthetic generator ------------------ */

/*
 * generate_trace / _draw_routed (trace.py:212-287), restated for decode-only
 * single-sequence traces (the bench workloads): per (token, layer) K draws
 * without replacement from (1 - b) * pop + b * uniform(hot set of the last
 * w_hot events of the layer), one numpy Generator.choice per draw.  numpy's
 * own arithmetic, op by op: PCG64 (128-bit LCG, XSL-RR output) stepped once
 * per choice, random() = (u64 >> 11) * 2^-53, p.sum() as numpy's pairwise
 * sum (8 accumulators for 8 <= n <= 128), p /= total, cumsum, cdf /= cdf[-1],
 * searchsorted(side='right').  The popularity table (trace.py:186-202) and
 * the stream's initial state (default_rng([seed, 1]).bit_generator.state)
 * come from numpy in the caller.  The stream is consumed token -> layer ->
 * slot (trace.py:265-283), so layers are interleaved: this restatement walks
 * the stream in that order, unlike the GPU kernel which jumps per chain.
 */
typedef unsigned __int128 orc_u128;

static uint64_t orc_pcg_out(orc_u128 s) {
    uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    unsigned r = (unsigned)(s >> 122);
    return (x >> r) | (x << ((64u - r) & 63u));
}

static double orc_np_sum(const double *a, int n) {
    if (n < 8) {
        double r = 0.0;
        for (int i = 0; i < n; ++i) r += a[i];
        return r;
    }
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
        for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
}

/* One trace: out[T][L][K] (the reference's event order). */
int orc_gen_decode(int L, int E, int K, int64_t T, int w_hot, double boost, const double *pop,
                   const uint64_t *state /* hi, lo, inc_hi, inc_lo */, uint8_t *out) {
    if (E > 128 || E < 1 || K < 1 || K > E || w_hot < 1 || w_hot > 64) return ORC_ERR_INVALID;
    const orc_u128 mult = ((orc_u128)0x2360ED051FC65DA4ull << 64) | (orc_u128)0x4385DF649FCCF645ull;
    const orc_u128 inc = ((orc_u128)state[2] << 64) | state[3];
    orc_u128 st = ((orc_u128)state[0] << 64) | state[1];
    uint8_t *ring = (uint8_t *)calloc((size_t)L * 64 * 128, 1);   /* [layer][w][E] routed flags */
    int *n_recent = (int *)calloc((size_t)L, sizeof(int));
    int *head = (int *)calloc((size_t)L, sizeof(int));
    if (!ring || !n_recent || !head) { free(ring); free(n_recent); free(head); return ORC_ERR_NOMEM; }
    const double omb = 1.0 - boost;
    double p[128];
    for (int64_t t = 0; t < T; ++t) {
        for (int l = 0; l < L; ++l) {
            uint8_t hot[128], chosen[128];
            memset(hot, 0, sizeof hot);
            memset(chosen, 0, sizeof chosen);
            for (int i = 0; i < n_recent[l]; ++i)
                for (int e = 0; e < E; ++e) hot[e] |= ring[((size_t)l * 64 + i) * 128 + e];
            int nh = 0;
            for (int e = 0; e < E; ++e) nh += hot[e];
            const int mix = nh > 0 && boost > 0.0;
            const double hm = mix ? 1.0 / (double)nh : 0.0;
            uint8_t *o = out + ((size_t)t * L + l) * K;
            for (int k = 0; k < K; ++k) {
                for (int e = 0; e < E; ++e) {
                    double v = pop[(size_t)l * E + e];
                    if (mix) v = omb * v + boost * (hot[e] ? hm : 0.0);
                    if (chosen[e]) v = 0.0;
                    p[e] = v;
                }
                double total = orc_np_sum(p, E);
                if (!(total > 0.0)) {
                    for (int e = 0; e < E; ++e) p[e] = chosen[e] ? 0.0 : 1.0;
                    total = orc_np_sum(p, E);
                }
                st = st * mult + inc;
                const double u = (double)(orc_pcg_out(st) >> 11) * (1.0 / 9007199254740992.0);
                double c = 0.0;
                for (int e = 0; e < E; ++e) { c += p[e] / total; p[e] = c; }
                const double last = p[E - 1];
                int idx = 0;
                for (int e = 0; e < E; ++e) idx += (p[e] / last <= u) ? 1 : 0;
                chosen[idx] = 1;
                o[k] = (uint8_t)idx;
            }
            uint8_t *slot = ring + ((size_t)l * 64 + head[l]) * 128;
            memcpy(slot, chosen, 128);
            head[l] = head[l] + 1 == w_hot ? 0 : head[l] + 1;
            if (n_recent[l] < w_hot) n_recent[l]++;
        }
    }
    free(ring); free(n_recent); free(head);
    return ORC_OK;
}

typedef struct {
    int L, E, K, w_hot;
    int64_t T, n;
    double boost;
    const double *pop;
    const uint64_t *states;
    uint8_t *out;
    int64_t next;
    pthread_mutex_t mu;
    int rc;
} genb_t;

static void *gen_worker(void *arg) {
    genb_t *g = (genb_t *)arg;
    for (;;) {
        pthread_mutex_lock(&g->mu);
        int64_t i = g->next++;
        pthread_mutex_unlock(&g->mu);
        if (i >= g->n) break;
        int rc = orc_gen_decode(g->L, g->E, g->K, g->T, g->w_hot, g->boost, g->pop, g->states + 4 * i,
                                g->out + (size_t)i * g->T * g->L * g->K);
        if (rc) g->rc = rc;
    }
    return NULL;
}

/* n independent traces (one state each, one shared popularity table) on
 * n_threads host threads: out[trace][T][L][K]. */
int orc_gen_decode_batch(int L, int E, int K, int64_t T, int w_hot, double boost, const double *pop,
                         int64_t n, const uint64_t *states, int n_threads, uint8_t *out) {
    genb_t g;
    memset(&g, 0, sizeof g);
    g.L = L; g.E = E; g.K = K; g.w_hot = w_hot; g.T = T; g.n = n; g.boost = boost;
    g.pop = pop; g.states = states; g.out = out;
    pthread_mutex_init(&g.mu, NULL);
    if (n_threads < 1) n_threads = 1;
    pthread_t *th = (pthread_t *)malloc((size_t)n_threads * sizeof(pthread_t));
    if (!th) return ORC_ERR_NOMEM;
    for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, gen_worker, &g);
    for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&g.mu);
    return g.rc;
}
