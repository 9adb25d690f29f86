/*
 * mcb.h -- C ABI of the B200 expert-cache replay engine (libmcb.so).
 *
 * The reference (FlashMoE simulation lab, moecache 0.1.0) is pure Python;
 * its hot path is reached through engine.run_simulation / simulate / sweep
 * (pkg/src/moecache/engine.py:300-391, 439-465).  The per-access
 * CachePolicy.access protocol (policies.py:95-113) is far too fine-grained
 * to cross an FFI, so this ABI sits at run_simulation/sweep granularity: one
 * call replays a packed trace under a policy list x capacity list and
 * returns the per-(trace, policy, capacity) counters from which SimReport
 * (engine.py:95-122) is assembled.  The binding a maintainer would add on the
 * reference side is a ctypes stub; see INTEGRATION.md.
 *
 * Conventions: extern "C", plain pointers and sizes, no exceptions cross the
 * boundary; every entry point returns an mcb_status and records a message
 * retrievable with mcb_last_error() (thread-local).  Device entry points take
 * device pointers and a cudaStream_t passed as void*; they enqueue work and
 * do not synchronise.  Host entry points take host pointers, copy in, run and
 * copy out (synchronously).  The caller owns every buffer it passes; the
 * context owns only its device scratch.
 *
 * Supported: num_experts <= 128, top_k <= num_experts, chains of < 2^32
 * accesses, policies LRU / LFU / Belady / ML (the north star's four) and the
 * state-dependent FIFO, ARC and LeCaR (whole-chain kernels).  Anything else
 * (custom per-access policy objects, > 128 experts) is rejected with
 * MCB_ERR_UNSUPPORTED rather than falling back to a CPU path.
 */
#ifndef MCB_H_
#define MCB_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCB_ABI_VERSION 1

/* ---- status codes (mapped by the Python shim onto the reference's exceptions) ---- */
typedef enum {
    MCB_OK = 0,
    MCB_ERR_INVALID = 1,       /* InvalidConfigError (trace.py:23) / SimulationError (engine.py:30) */
    MCB_ERR_CAPACITY = 2,      /* CapacityTooSmallError (engine.py:34, 312-316, 449-453) */
    MCB_ERR_NO_EVICTABLE = 3,  /* NoEvictableError (policies.py:24, mlpolicy.py:24-25) */
    MCB_ERR_CUDA = 4,          /* CUDA runtime failure */
    MCB_ERR_UNSUPPORTED = 5,   /* policy / shape outside the B200 engine */
    MCB_ERR_NOMEM = 6,
    MCB_ERR_SHAPE = 7          /* ValueError: net E mismatch (mlpolicy.py:47-50) */
} mcb_status;

/* ---- policies (engine.py:150 names) ---- */
typedef enum {
    MCB_LRU = 0,               /* policies.py:132-149 */
    MCB_LFU = 1,               /* policies.py:171-197 */
    MCB_BELADY = 2,            /* policies.py:200-214 */
    MCB_ML = 3,                /* mlpolicy.py:33-65, include_prefill=True */
    MCB_ML_NO_PREFILL = 4,     /* mlpolicy.py, {"name": "ml", "include_prefill": False} */
    MCB_FIFO = 5,              /* policies.py:152-168 (whole-chain replay kernels only) */
    MCB_ARC = 6,               /* policies.py:217-302 (whole-chain replay kernels only) */
    MCB_LECAR = 7              /* policies.py:305-395, parameters from mcb_set_lecar (whole-chain kernels only) */
} mcb_policy;

/* ---- per-(trace, policy, capacity) report slots ---- */
enum {
    MCB_R_PREFILL_HITS = 0,
    MCB_R_PREFILL_MISSES = 1,
    MCB_R_DECODE_HITS = 2,
    MCB_R_DECODE_MISSES = 3,
    MCB_R_COMPULSORY = 4,
    MCB_R_EVICTIONS = 5,
    MCB_R_REFETCHED = 6,       /* numerator of refetch_within_w (engine.py:266-297) */
    MCB_R_STATUS = 7,          /* mcb_status of this cell (NO_EVICTABLE possible for ML) */
    MCB_R_N = 8
};

/* outcome codes written per access when outcomes are requested */
#define MCB_OUT_HIT 0xFFFFu
#define MCB_OUT_MISS 0xFFFEu   /* miss without eviction; otherwise the victim id */

/*
 * Packed trace.  A trace unrolls into one access stream per layer
 * (replay.py:44-81); a "chain" is one (trace, layer) stream, chain index
 * c = trace * num_layers + layer.  Streams are stored chain-major so a chain
 * is contiguous in HBM.
 *
 * uniform = 1: decode-only, one sequence per trace, every chain has
 *   events_per_chain events of top_k accesses; acc[c][t][k] (uint8).  The
 *   chain_* / ev_info / routed pointers are ignored.
 * uniform = 0: general (prefill + several sequences):
 *   chain_acc_off[c]..[c+1]  accesses of chain c in acc (after prefill
 *                            load-once dedup, replay.py:54-71)
 *   chain_ev_off[c]..[c+1]   events of chain c in ev_info
 *   chain_rt_off[c]..[c+1]   routed ids of chain c in routed (the full stored
 *                            expert list; feature updates use it)
 *   ev_info[e] = n_acc | n_routed << 9 | is_decode << 30 | new_sequence << 31
 */
typedef struct {
    int32_t num_layers;
    int32_t num_experts;
    int32_t top_k;
    int32_t num_traces;
    int32_t uniform;
    int32_t reserved;
    int64_t events_per_chain;          /* uniform only */
    int64_t total_acc;                 /* general only: chain_acc_off[n_chains] */
    int64_t total_events;              /* general only: chain_ev_off[n_chains] */
    const uint8_t *acc;                /* readable up to round_up(total, 128) bytes */
    const int64_t *chain_acc_off;      /* [n_chains + 1] */
    const int64_t *chain_ev_off;       /* [n_chains + 1] */
    const int64_t *chain_rt_off;       /* [n_chains + 1] */
    const uint32_t *ev_info;           /* [n_events] */
    const uint8_t *routed;             /* [n_routed] */
} mcb_trace;

/* CostModel (engine.py:38-55) */
typedef struct {
    double t_load_s;
    double t_compute_s;
    double ml_score_cost_s;
    int32_t loads_serial;
    int32_t window;                    /* refetch window w (engine.py:266-297) */
} mcb_cost;

/*
 * EvictionNet parameters (net.py:61-86), float64, in .evnet order
 * (net.py:282-305): per net w1[H][2E] b1[H] w2[H][H] b2[H] w3[E][H] b3[E].
 * num_nets = 1 (one shared net) or num_layers (net for layer l at index l).
 */
typedef struct {
    int32_t num_experts;
    int32_t hidden;
    int32_t num_nets;
    int32_t reserved;
    const double *params;
} mcb_nets;

/*
 * Outputs.  reports[trace][pol][cap][MCB_R_N] int64 and
 * latency[trace][pol][cap][2] float64 (decode, prefill) are summed over
 * layers in layer order exactly like engine.py:330-343 (float64, no FMA).
 * Optional (NULL to skip): chain_reports[c][pol][cap][MCB_R_N],
 * hashes[c][pol][cap] (polynomial hash h = h * 0x100000001B3 + code + 1 mod
 * 2^64 over the u16 outcome codes of the chain, in access order -- spliceable
 * across the segmented replay's segments),
 * outcomes[pol][cap][total_acc] u16 (record_decisions, small traces),
 * chain_latency[c][pol][cap][2] float64 (the per-layer decode / prefill
 * latency sums of _replay_layer, engine.py:258-263, before the layer fold --
 * what a layer-sharded multi-GPU run gathers to fold in layer order).
 */
typedef struct {
    int64_t *reports;
    double *latency;
    int64_t *chain_reports;
    uint64_t *hashes;
    uint16_t *outcomes;
    double *chain_latency;
} mcb_outputs;

typedef struct mcb_ctx mcb_ctx;

/* ---- lifecycle / errors ----
 * Threading model: a context owns device scratch buffers (next-use, ranks,
 * segment records, duel and training workspaces) that its asynchronous
 * entry points reuse, plus per-context settings (tuning knobs, LeCaR
 * parameters).  Calls on one context are serialised by an internal mutex,
 * but their device work is only ordered on the stream passed in: issue the
 * asynchronous calls of one context on one stream (or synchronise between
 * streams), and give each host thread that changes settings its own
 * context.  mcb_last_error is thread-local. */
int mcb_abi_version(void);
int mcb_ctx_create(int device, mcb_ctx **out);
int mcb_ctx_destroy(mcb_ctx *ctx);

/* ---- Multi-GPU: the context's NCCL communicator ----
 * The sharded engine (one process per GPU, traces or layers per rank) needs
 * one collective: an in-place int64 sum of the per-(trace, policy, capacity)
 * counters and float64 latency bit patterns, every slot written by exactly
 * one rank (paper_2601_17063_b200/distributed.py).  These entry points give a
 * non-Python caller that collective; the reference's counterpart is the
 * thread pool of sweep(jobs) (engine.py:456-464).  NCCL is loaded at run
 * time (MCB_ERR_UNSUPPORTED without it).
 * mcb_comm_unique_id: rank 0 creates the 128-byte id and shares it;
 * mcb_comm_init: every rank joins with it (the context then owns the
 * communicator until mcb_comm_destroy / mcb_ctx_destroy);
 * mcb_comm_allreduce_i64: in-place sum of count int64 on a device buffer. */
int mcb_comm_unique_id(uint8_t *out, int32_t n);
int mcb_comm_init(mcb_ctx *ctx, int32_t nranks, int32_t rank, const uint8_t *unique_id);
int mcb_comm_allreduce_i64(mcb_ctx *ctx, int64_t *buf, int64_t count, void *stream);
int mcb_comm_destroy(mcb_ctx *ctx);
int mcb_last_error(char *buf, size_t n);
/* Launch statistics of the last mcb_replay on this context: number of kernels
 * launched, and the uncertain-rank counter of the ML scorer (events whose
 * float64 scores had two values closer than 1e-12 relative). */
int mcb_last_stats(mcb_ctx *ctx, int64_t *kernels_launched, int64_t *uncertain_events);
/* Trace ranges the last mcb_replay / mcb_replay_host was split into to stay
 * within the scratch budget (MCB_TUNE_SCRATCH_BYTES); 1 = one range. */
int mcb_last_chunks(mcb_ctx *ctx, int64_t *chunks);
/* Stage timing: when enabled, mcb_replay records CUDA events on its stream
 * around each stage; mcb_last_timings returns the stage durations in ms of
 * the last call (after the stream has been synchronised):
 * [0] K2 next-use scan, [1] K3 scorer, [2] K4 replay, [3] K5 fold. */
int mcb_set_timing(mcb_ctx *ctx, int32_t enable);
/* Device-side counters of the last mcb_replay (synchronises the device):
 * [0] uncertain scorer events (float64 near ties), [1] segmented replay:
 * events replayed by the fix-up walk, [2] segments whose speculative state
 * never converged, [3] segments walked, [4] latency folds done event by
 * event, [5] events the tensor-core scorer re-scored in float64. */
int mcb_read_stats(mcb_ctx *ctx, int64_t *out, int32_t n);
/* Tuning knobs (results never depend on them):
 * MCB_TUNE_SOLO_MIN: minimum instance count for the thread-per-instance
 * replay kernel (num_experts <= 16); below it one warp replays one instance. */
#define MCB_TUNE_SOLO_MIN 0
/* MCB_TUNE_SEG_EV: segmented speculative replay of uniform traces with
 * num_experts <= 16 (mcb_segment.cu): 0 = automatic (used when the instances
 * are too few to fill the GPU), < 0 = off, > 0 = events per segment. */
#define MCB_TUNE_SEG_EV 1
/* MCB_TUNE_SEG_NW: warm-up events replayed before each speculative segment
 * (0 = automatic). */
#define MCB_TUNE_SEG_NW 2
/* MCB_TUNE_SEG_PASSES: speculation passes of the segmented replay (0 = auto,
 * else 1..8; pass p > 0 restarts every segment from pass p-1's end state of
 * its predecessor; num_experts <= 16 uses at most 2). */
#define MCB_TUNE_SEG_PASSES 3
/* MCB_TUNE_GROUP_LANES: lanes per cache instance of the num_experts > 16
 * replay (0 = automatic, 8, 16 or 32). */
#define MCB_TUNE_GROUP_LANES 4
/* MCB_TUNE_SERIAL: 1 = run every stage on the caller's stream (no concurrent
 * side stream), so mcb_last_timings attributes time to each stage alone. */
#define MCB_TUNE_SERIAL 5
/* MCB_TUNE_K3_CTAS: scorer grid -- < 0 (default) = one CTA per 32-event tile;
 * 0 = persistent, every CTA that fits; k > 0 = persistent, at most k per SM. */
#define MCB_TUNE_K3_CTAS 6
/* MCB_TUNE_ML_CHUNKS: the K3 -> ML replay pipeline depth (chain ranges whose
 * ML replay overlaps the scoring of the next range); 1 = no pipelining. */
#define MCB_TUNE_ML_CHUNKS 7
/* MCB_TUNE_OVERLAP: where the non-ML replay runs concurrently -- 0 (default)
 * after the scorer, next to the ML replay; 1 during the scorer. */
#define MCB_TUNE_OVERLAP 8
/* MCB_TUNE_WIDE_MIN: minimum instance count (per launch) for the
 * thread-per-instance replay of 16 < num_experts <= 128 (default 8192: e.g.
 * C4's ML replay at 8 GPUs, 13,824 instances per rank, 26 -> 20 ms); below it
 * one warp replays one instance. */
#define MCB_TUNE_WIDE_MIN 9
/* MCB_TUNE_SEG_TSPEC: speculation of the segmented replay for num_experts
 * > 16 -- 0 automatic (one thread per (instance, segment) for chains of
 * >= 65,536 events, else one warp), 1 thread, -1 warp. */
#define MCB_TUNE_SEG_TSPEC 10
/* MCB_TUNE_SCRATCH_BYTES: device scratch budget of one mcb_replay call
 * (next-use positions, ML rank rows, feature snapshots, per-instance
 * outputs).  A uniform multi-trace batch whose scratch would exceed it is
 * replayed in consecutive trace ranges that reuse the same scratch (results
 * are identical; outcomes are not supported then).  0 (default) = 40% of
 * the device memory free at the call. */
#define MCB_TUNE_SCRATCH_BYTES 11
/* MCB_TUNE_K3_TC: 1 (default) = the tensor-core scorer (fp16 x 2 split on
 * tcgen05, certified ranks, float64 re-score of uncertified events) for
 * uniform traces with hidden 128 and num_experts in {8, 16, 32, 64, 128};
 * 0 = the float64 DMMA scorer for every event.  Ranks are identical. */
#define MCB_TUNE_K3_TC 12
/* MCB_TUNE_K3_TAU_PPB: the tensor-core scorer certifies an event's order when
 * every two adjacent scores differ by more than 2 * tau * max|s|; tau in units
 * of 1e-9 (default 4000 = 4e-6).  Larger = more events re-scored in float64. */
#define MCB_TUNE_K3_TAU_PPB 13
/* MCB_TUNE_K3_GROUPS: layout of the tensor-core scorer for num_experts <= 64:
 * 3 (default) or 2 epilogue groups (128-event tiles in flight per SM) with
 * the MMA operands in shared memory, or 1 = two groups with the operands in
 * TMEM and a deep weight ring.  num_experts = 128 always runs 2 groups, with
 * the operands in TMEM unless the knob is 2.  Ranks are identical. */
#define MCB_TUNE_K3_GROUPS 14
/* MCB_TUNE_UPLOAD_PIECES: mcb_replay_host copies a uniform batch of >= 16
 * traces in this many trace-range pieces (default 8, at most 16; 0/1 = one
 * copy) and starts the trace-only stages (K2, K3) of each piece as soon as
 * it has landed, so the host-to-device copy overlaps the scorer. */
#define MCB_TUNE_UPLOAD_PIECES 16
int mcb_set_tuning(mcb_ctx *ctx, int32_t knob, int64_t value);
/* LeCaR parameters used by the MCB_LECAR cells of later mcb_replay calls on
 * this context (LeCaRPolicy.__init__, policies.py:333-349; defaults 0.45,
 * 0.005, 0).  Every per-layer policy object of the reference seeds its own
 * random.Random(seed), so each cache instance consumes the same stream of
 * random() draws, one per eviction; the engine materialises that stream
 * (CPython's MT19937 seeding and genrand_res53) and the per-capacity
 * regret factors exp(learning_rate * discount**elapsed) with the host libm,
 * so the device only multiplies, adds and divides.  seed >= 0 (an int seed;
 * negative values seed like their absolute value in CPython). */
int mcb_set_lecar(mcb_ctx *ctx, double learning_rate, double discount_base, int64_t seed);
/* Host-only: the first n values of CPython's random.Random(seed).random()
 * (the stream mcb_set_lecar's seed selects), into out[n]. */
int mcb_lecar_random(int64_t seed, int64_t n, double *out);
int mcb_last_timings(mcb_ctx *ctx, float *ms, int32_t n);

/* ---- K10: EvictionNet training (net.py:107-279) ----
 * All nets of one call train together (the reference trains one net per
 * layer, cli.py:253-283).  Device pointers, asynchronous on `stream`.
 * params / adam_m / adam_v: float64 [num_nets][P] in .evnet order (w1, b1,
 * w2, b2, w3, b3; P = H*2E + H + H*H + H + E*H + E). */
typedef struct {
    int32_t num_nets, num_experts, hidden, reserved;
    int64_t num_samples;          /* rows per net */
    const double *features;       /* [net][num_samples][2E] */
    const double *targets;        /* [net][num_samples][E] */
    const uint8_t *masks;         /* [net][num_samples][E] (0 / 1) */
} mcb_train_data;
typedef struct {
    double learning_rate, weight_decay, beta1, beta2, eps;   /* AdamW (net.py:159-170) */
    int64_t batch_size;
    int64_t n_train;              /* the first n_train rows train (net.py:219-226) */
} mcb_train_cfg;
/* One epoch (net.py:245-256): mini-batches of rows order[start : start + batch]
 * (order: device int32 [n_train], the epoch's permutation), forward, masked
 * MSE gradient, backward, AdamW step (optimizer step count before the epoch =
 * step0).  bad: device float64 [num_nets][4] = {flag, loss, batch offset, epoch}
 * of the first non-finite batch loss (NonFiniteLossError, net.py:250-254);
 * zero it before the first epoch. */
int mcb_train_epoch(mcb_ctx *ctx, const mcb_train_data *data, const mcb_train_cfg *cfg, double *params,
                    double *adam_m, double *adam_v, int64_t step0, int64_t epoch, const int32_t *order, double *bad,
                    void *stream);
/* Masked-MSE sums over rows [row0, row0 + rows) of every net (evaluate,
 * net.py:236-239): sums: device float64 [num_nets][2] = {sum m (pred - y)^2,
 * sum m}. */
int mcb_train_eval(mcb_ctx *ctx, const mcb_train_data *data, const double *params, int64_t row0, int64_t rows,
                   double *sums, void *stream);

/* ---- K8: eviction_quality_duel (engine.py:404-436) ----
 * outcomes_a / outcomes_b: two policies' per-access outcome codes of the
 * same trace and capacity (mcb_outputs.outcomes rows: victim id,
 * MCB_OUT_HIT, MCB_OUT_MISS), next_pos: K2's output for the trace.  At every
 * access where both evict, the victim with the strictly larger next use
 * wins.  wins: device int64[2] = {A wins, B wins}; the reference's result is
 * A / (A + B), or 0.5 when both are 0.  Device pointers, asynchronous. */
int mcb_eviction_duel(mcb_ctx *ctx, const mcb_trace *trace, const uint16_t *outcomes_a,
                      const uint16_t *outcomes_b, const uint32_t *next_pos, int64_t *wins, void *stream);

/* ---- K7: GPU validate + pack of a decode-only batch (batch-kind .mcbt) ----
 * ids: device uint8 [num_traces][decode_steps][num_layers][top_k] in the
 * reference's event order (trace.py:121-127, one sequence per trace).
 * acc: device uint8, >= num_traces * num_layers * decode_steps * top_k bytes:
 * the chain-major uniform layout of mcb_trace.  first_bad: device int64,
 * receives the event-order index (trace * T + step) * L + layer of the first
 * event AccessEvent.validate rejects (trace.py:80-106: expert outside
 * [0, num_experts) or a duplicate), or -1.  Asynchronous on `stream`.
 * Replaces parse_trace / RoutingTrace.validate + layer_schedules for this
 * layout (trace.py:350-412, replay.py:44-81). */
int mcb_pack_decode_ids(mcb_ctx *ctx, const uint8_t *ids, int64_t num_traces, int64_t decode_steps,
                        int32_t num_layers, int32_t top_k, int32_t num_experts, uint8_t *acc, int64_t *first_bad,
                        void *stream);

/* ---- host-side trace validation + packing (trace.py:57-141, replay.py:44-81) ----
 * Input: one trace as flat events in stored order: seq_id, phase (0 prefill,
 * 1 decode), step, layer, CSR experts.  Validates exactly what
 * RoutingTrace.validate() checks (MCB_ERR_INVALID + message on failure) and
 * produces an owned packed trace (uniform layout when the trace is
 * decode-only with one sequence); num_experts > 128 is MCB_ERR_UNSUPPORTED
 * (after validation). */
typedef struct mcb_packed mcb_packed;
int mcb_pack_trace(int32_t num_layers, int32_t num_experts, int32_t top_k, int64_t num_events,
                   const int64_t *seq_id, const uint8_t *phase, const int64_t *step,
                   const int32_t *layer, const int64_t *expert_off, const int32_t *experts,
                   mcb_packed **out);
/* Validation only (RoutingTrace.validate, trace.py:115-137, with the
 * reference's messages): no engine limits, nothing allocated. */
int mcb_validate_trace(int32_t num_layers, int32_t num_experts, int32_t top_k, int64_t num_events,
                       const int64_t *seq_id, const uint8_t *phase, const int64_t *step, const int32_t *layer,
                       const int64_t *expert_off, const int32_t *experts);
/* Host view of a packed trace, sizes, and num_decode_steps() (trace.py:139-141). */
int mcb_packed_view(const mcb_packed *p, mcb_trace *view, int64_t *total_acc, int64_t *total_events,
                    int64_t *total_routed, int64_t *num_decode_steps);
/* Per-access (tick, decode_index) of chain c (for EvictionRecord assembly). */
int mcb_packed_positions(const mcb_packed *p, int64_t chain, int64_t *tick, int64_t *decode_index);
int mcb_packed_free(mcb_packed *p);

/* ---- the hot path ----
 * Replays every chain of `trace` under every policy in `policies` and every
 * capacity in `capacities` (engine.py:439-465 cross product).  Belady
 * next-use positions (K2) and ML ranks (K3) are computed once per chain and
 * shared by every capacity.  `nets` may be NULL when no ML policy is listed.
 * mcb_replay: device pointers, asynchronous on `stream`.
 * mcb_replay_host: host pointers (pinned or pageable), synchronous; the
 * host<->device copies are part of the call. */
int mcb_replay(mcb_ctx *ctx, const mcb_trace *trace, const int32_t *policies, int32_t n_policies,
               const int32_t *capacities, int32_t n_capacities, const mcb_cost *cost,
               const mcb_nets *nets, const mcb_outputs *out, void *stream);
int mcb_replay_host(mcb_ctx *ctx, const mcb_trace *trace, const int32_t *policies,
                    int32_t n_policies, const int32_t *capacities, int32_t n_capacities,
                    const mcb_cost *cost, const mcb_nets *nets, const mcb_outputs *out,
                    void *stream /* NULL: the context's own stream */);

/* ---- individual kernels (exposed for tests and benchmarks) ---- */
/* K2: next_pos[i] = chain-relative position of the next access of the same
 * expert after access i of its chain, 0xFFFFFFFF if none
 * (OracleIndex.next_use, policies.py:65-76).  Device pointers. */
int mcb_next_use(mcb_ctx *ctx, const mcb_trace *trace, uint32_t *next_pos, void *stream);
/* K3: per event, rank[e] in 0..E of expert e's float64 score
 * (0 = never selectable: NaN or -inf, mlpolicy.py:15-26); optional float64
 * scores[event][E].  Device pointers. */
int mcb_score(mcb_ctx *ctx, const mcb_trace *trace, const mcb_nets *nets, int32_t include_prefill,
              uint8_t *ranks, double *scores, void *stream);

/* K3-TC alone (tests and calibration): the tensor-core scorer's ranks (after
 * the float64 re-score of uncertified events, identical to mcb_score's) and
 * its fp32 scores[event][E] before certification.  Uniform traces, hidden
 * 128, num_experts in {8, 16, 32, 64, 128}.  Device pointers. */
int mcb_score_tc_scores(mcb_ctx *ctx, const mcb_trace *trace, const mcb_nets *nets, uint8_t *ranks,
                        float *scores, void *stream);

/* ---- K1: router-logits GEMM + top-k trace generator (tcgen05 / TMA) ----
 * hidden[T][d] bf16 (shared by all layers), weight[L*E][d] bf16 (router
 * gate rows of every layer, layer-major).  Writes acc[l][t][k] (uint8,
 * chain-major uniform layout for trace 0) with the K largest logits of
 * layer l per token, sorted descending, ties to the lower expert id
 * (torch.topk semantics used by the HF routers the extractor hooks,
 * extractor.py:162-183).  Optional fp32 logits[t][L*E].  Device pointers. */
int mcb_router_topk(mcb_ctx *ctx, const void *hidden_bf16, const void *weight_bf16, int64_t T,
                    int32_t d, int32_t num_layers, int32_t num_experts, int32_t top_k,
                    uint8_t *acc, float *logits, void *stream);

/* K1's input: AR(1) hidden states over tokens, out[T][d_pad] bf16 with
 * h[0] ~ N(0, 1), h[t] = rho h[t-1] + sqrt(1 - rho^2) n(t) per column j < d
 * (n: a counter-based normal of (seed, t, j)), column d = 1 (the bias input
 * of the gate rows), columns > d = 0.  Device pointer. */
int mcb_ar1_hidden(mcb_ctx *ctx, int64_t T, int32_t d, int32_t d_pad, double rho, uint64_t seed, void *out_bf16,
                   void *stream);

/* ---- Belady-labelled training data ----
 * Replaces build_training_data (pkg/src/moecache/dataset.py:35-96) for any
 * packed trace (prefill and several sequences included): for every event of
 * every chain the float64 feature vector [1/r || f / max_f] after the
 * event's tracker update (features.py:34-52; prefill events update it only
 * with include_prefill), float64 targets min(d, distance_cap) / distance_cap
 * with d the events until the expert is next routed (replay.py:92-109; never
 * -> 1.0), and the Belady residency mask at `capacity` before the event's
 * accesses.  Outputs features[event][2E], targets[event][E], masks[event][E]
 * (bytes), events in mcb_trace order (chain-major); the reference's samples
 * are the decode events.  Device pointers, asynchronous on `stream`. */
int mcb_training_data(mcb_ctx *ctx, const mcb_trace *trace, int32_t capacity, int32_t distance_cap,
                      int32_t include_prefill, double *features, double *targets, uint8_t *masks, void *stream);

/* ---- bit-exact reference generator ----
 * Replaces generate_trace / _draw_routed (pkg/src/moecache/trace.py:212-287):
 * the same routing as the reference's numpy generator, bit for bit.  The
 * host supplies the per-layer popularity (trace.py:186-202, float64 [L][E])
 * and the initial PCG64 state of default_rng([rng_seed, 1]) as
 * {state_hi, state_lo, inc_hi, inc_lo} (a HOST array of 4).  Writes
 * experts[seq][token][layer][K] (tokens: prefill then decode; the
 * reference's event order).  popularity / experts are device pointers; the
 * call is asynchronous on `stream`. */
int mcb_gen_reference(mcb_ctx *ctx, int32_t num_layers, int32_t num_experts, int32_t top_k, int64_t num_seqs,
                      int64_t prefill_tokens, int64_t decode_steps, int32_t w_hot, double recency_boost,
                      const double *popularity, const uint64_t *pcg_state, uint8_t *experts, void *stream);
/* Batch form for decode-only single-sequence traces (generate_trace with
 * num_seqs = 1, prefill_tokens = 0, one rng_seed per trace and a shared
 * popularity table, e.g. popularity_seed fixed): pcg_states is a DEVICE
 * array [num_traces][4] (the initial state of default_rng([rng_seed_i, 1])),
 * experts a device uint8 [trace][layer][token][K] -- the chain-major uniform
 * layout of mcb_trace, ready to replay. */
int mcb_gen_reference_batch(mcb_ctx *ctx, int32_t num_layers, int32_t num_experts, int32_t top_k,
                            int64_t num_traces, int64_t decode_steps, int32_t w_hot, double recency_boost,
                            const double *popularity, const uint64_t *pcg_states, uint8_t *experts, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* MCB_H_ */
