// Device-side views and kernel launch declarations (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "mcb_internal.h"

#define MCB_MAX_POL 8
#define MCB_MAX_CAP 64
#define MCB_TILE_EV 32          // events per scorer tile (K3)

// Chain-major trace view usable on the device (mcb.h mcb_trace, device pointers).
struct DevTrace {
    int L, E, K;
    int uniform;
    int64_t T;                  // uniform: events per chain
    int64_t n_chains;
    int64_t total_acc, total_events;
    const uint8_t *acc;
    const int64_t *acc_off, *ev_off, *rt_off;
    const uint32_t *ev_info;
    const uint8_t *routed;

    __device__ __forceinline__ int64_t acc_begin(int64_t c) const { return uniform ? c * T * K : acc_off[c]; }
    __device__ __forceinline__ int64_t acc_end(int64_t c) const { return uniform ? (c + 1) * T * K : acc_off[c + 1]; }
    __device__ __forceinline__ int64_t ev_begin(int64_t c) const { return uniform ? c * T : ev_off[c]; }
    __device__ __forceinline__ int64_t ev_end(int64_t c) const { return uniform ? (c + 1) * T : ev_off[c + 1]; }
    __device__ __forceinline__ int64_t rt_begin(int64_t c) const { return uniform ? c * T * K : rt_off[c]; }
    __device__ __forceinline__ const uint8_t *routed_ptr() const { return uniform ? acc : routed; }
    __device__ __forceinline__ uint32_t info(int64_t c, int64_t global_ev) const {
        return uniform ? mcb_ev_pack((uint32_t)K, (uint32_t)K, true, global_ev == c * T) : ev_info[global_ev];
    }
};

struct ReplayParams {
    DevTrace tr;
    int n_pol, n_cap;                   // totals (output indexing)
    int n_pol_launch;                   // policies replayed by this launch ...
    int32_t pol_map[MCB_MAX_POL];       // ... and their indices in pol[]
    int32_t pol[MCB_MAX_POL];
    int32_t cap[MCB_MAX_CAP];
    const uint32_t *next_pos;           // K2 output (Belady)
    const uint8_t *rank[2];             // K3 output: [0] include_prefill, [1] decode-only features
    double t_load, t_compute, ml_cost;
    int loads_serial, window;
    int64_t *inst_out;                  // [chain][pol][cap][MCB_R_N]
    double *inst_lat;                   // [chain][pol][cap][2]
    uint64_t *hashes;                   // optional [chain][pol][cap]
    uint16_t *outcomes;                 // optional [pol][cap][total_acc]
    int64_t solo_min_instances;         // thread-per-instance kernel threshold (E <= 16)
    int64_t wide_min_instances;         // thread-per-instance kernel threshold (16 < E <= 64)
    int64_t chain_lo, chain_hi;         // chains [lo, hi) replayed by this launch (outputs stay global)
    int group_lanes;                    // lane-group size of k_replay (0 = automatic)
    uint8_t *res_masks;                 // optional [chain][T][E]: resident set at each event start
    const double *lecar_u;              // LeCaR: random() stream, one draw per eviction (policies.py:381)
    const double *lecar_f;              // LeCaR: [cap][lecar_tlen] regret factors exp(lr * discount**elapsed)
    int64_t lecar_tlen;                 //   elapsed >= lecar_tlen has factor 1.0
                                        // (uniform traces, one policy x capacity; dataset.py masks)
    // segmented speculative replay (mcb_segment.cu); seg.n_seg == 0: whole-chain kernels
    struct Seg {
        int SE;                         // events per segment (multiple of MCB_SNAP_EV)
        int n_seg;                      // segments per chain
        int NW;                         // warm-up events before each segment (multiple of MCB_SNAP_EV)
        int passes;                     // speculation passes (1 or 2; LRU always 1)
        int n_snap;                     // snapshots per chain (every MCB_SNAP_EV events)
        int snap_e;                     // experts per snapshot record (16, or E rounded up to 32)
        int thread_spec;                // E > 16: speculation by one thread per (instance, segment)
        int64_t Tpad;                   // row stride of codes (events, multiple of 16)
        int2 *snap;                     // [chain][n_snap][16] (last position before, count before)
        int2 *summ;                     // scratch [chain][n_snap][16]
        struct SegOut *out[2];          // [inst][seg] of speculation pass 0 and pass 1
        uint8_t *codes;                 // [inst][Tpad] per-event miss counts
    } seg;
    unsigned long long *stats;          // device counters (mcb_read_stats): [1] fix-up events,
                                        // [2] unconverged segments, [3] segments walked
};

#define MCB_SNAP_EV 32           // key-snapshot granularity of the segmented replay (events)
#define MCB_SEG_BINS 18          // miss-count histogram bins (K <= 16 -> 17 used)

// Per (instance, segment) result of the speculative pass (mcb_segment.cu).
struct SegOut {
    uint32_t misses, nev, refc, comp;   // counters of the segment (speculative run)
    uint32_t res_end;                   // state at the segment end ...
    int32_t stuck_ev;                   // first event (chain-relative) with no evictable expert, -1 none
    uint32_t res_start;                 // ... and at the segment start (after the warm-up)
    uint32_t pad0;
    uint64_t hash;                      // poly hash of the segment's outcome codes (from 0)
    uint32_t ring_end[4];               // refetch rings, 8 x 16-bit slots
    uint32_t ring_start[4];
    uint32_t pk_start[16];              // packed policy keys at the segment start (non-ML)
    uint16_t hist[MCB_SEG_BINS];        // events per miss count
    uint32_t pad1[5];                   // 192 bytes
};

// launchers (mcb_kernels.cu); return the number of kernels launched or <0 on error
int launch_next_use(const DevTrace &tr, uint32_t *next_pos, uint32_t *scratch, cudaStream_t s);
size_t next_use_scratch_words(const DevTrace &tr);   // scratch for the blocked walk (0: not used)
int launch_replay(const ReplayParams &p, cudaStream_t s);
int launch_replay_wide(const ReplayParams &p, cudaStream_t s);   // mcb_wide.cu; 0 = not applicable
int preload_wide_kernels();
void prepare_launch_attributes(const DevTrace &tr, int H);
int preload_kernels();   // force module loading + smem attributes (call at context creation)
// segmented replay (uniform traces, num_experts <= 16); seg_* are host helpers
bool seg_eligible(const ReplayParams &p);
int seg_events_per_segment(int64_t T, int64_t n_inst_launch, int64_t override_se, int E, bool paired);
size_t seg_snap_bytes(int64_t n_chains, int n_snap, int E);
int seg_snap_stride(int E);
int preload_segment_warp_kernels();
int seg_warmup_events(int se, int64_t override_nw, int E);
size_t seg_out_bytes(int64_t n_inst, int n_seg, int E);
size_t seg_codes_bytes(int64_t n_inst, int64_t Tpad);
int launch_seg_snapshot(const ReplayParams &p, cudaStream_t s);
enum { SEG_ALL = 0, SEG_SPEC = 1, SEG_FINISH = 2 };   // launch_replay_segmented phases
int launch_replay_segmented(const ReplayParams &p, cudaStream_t s, int phase = SEG_ALL);
int preload_segment_kernels();
int launch_fold(const ReplayParams &p, int num_traces, int64_t *reports, double *latency, cudaStream_t s);
int launch_prepare_nets(const double *params, int E, int H, int num_nets, double *wt, cudaStream_t s);
__host__ __device__ size_t prepared_net_doubles(int E, int H);
__host__ __device__ size_t net_param_doubles(int E, int H);
// K3: snapshot scan + tile scorer. snaps scratch: n_tiles_total * (2E+1) int32; tile_off: n_chains+1 int64
int launch_score_prep(const DevTrace &tr, int include_prefill, int32_t *snaps, int64_t *tile_off, int64_t max_tiles,
                      cudaStream_t s);
// k3_ctas: grid mode of the tile scorer (mcb.h MCB_TUNE_K3_CTAS)
int launch_score_tiles(const DevTrace &tr, const double *wt, int H, int num_nets, int include_prefill,
                       uint8_t *ranks, double *scores, const int32_t *snaps, const int64_t *tile_off,
                       int64_t tile_lo, int64_t tile_hi, unsigned long long *uncertain, int k3_ctas, cudaStream_t s);
int launch_train_features(const DevTrace &tr, const int32_t *snaps, const int64_t *tile_off, int64_t max_tiles,
                          int include_prefill, double *features, cudaStream_t s);
int launch_train_targets(const DevTrace &tr, int distance_cap, double *targets, cudaStream_t s);
// K3-TC (mcb_score_tc.cu): fp16x2 tcgen05 scorer with certified ranks; flagged
// events go to per-net lists that launch_rescore re-scores in float64.
bool score_tc_eligible(const DevTrace &tr, int H);
size_t score_tc_net_bytes(int E);
int score_tc_bias_stride(int E);
int preload_score_tc();
int launch_score_tc(const DevTrace &tr, const double *params, int num_nets, const int32_t *snaps, uint8_t *wimg,
                    float *bias, uint8_t *ranks, float tau, int32_t *flag_cnt, int32_t *flag_list, int64_t bucket_cap,
                    unsigned long long *stats, float *dbg_scores, int groups, cudaStream_t s, bool prep = true,
                    int64_t ev_base = 0);
int launch_rescore(const DevTrace &tr, const double *wt, int H, int num_nets, const int32_t *snaps,
                   const int32_t *flag_cnt, const int32_t *flag_list, int64_t bucket_cap, uint8_t *ranks,
                   unsigned long long *uncertain, cudaStream_t s);
int launch_score(const DevTrace &tr, const double *wt, int H, int num_nets, int include_prefill,
                 uint8_t *ranks, double *scores, int32_t *snaps, int64_t *tile_off, int64_t max_tiles,
                 unsigned long long *uncertain, int k3_ctas, cudaStream_t s);
