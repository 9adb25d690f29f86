// Internal declarations shared by the libmcb translation units.
#pragma once

#include <stdint.h>

#include "../../include/mcb.h"

#define MCB_MAX_EXPERTS 128
#define MCB_NEXT_INF 0xFFFFFFFFu

// ev_info bit layout (mcb.h): n_acc | n_routed << 9 | decode << 30 | new_seq << 31
#ifdef __CUDACC__
#define MCB_HD __host__ __device__ __forceinline__
#else
#define MCB_HD inline
#endif
MCB_HD uint32_t mcb_ev_pack(uint32_t n_acc, uint32_t n_rt, bool decode, bool new_seq) {
    return (n_acc & 0x1FFu) | ((n_rt & 0x1FFu) << 9) | ((uint32_t)decode << 30) | ((uint32_t)new_seq << 31);
}
MCB_HD uint32_t mcb_ev_nacc(uint32_t info) { return info & 0x1FFu; }
MCB_HD uint32_t mcb_ev_nrt(uint32_t info) { return (info >> 9) & 0x1FFu; }
MCB_HD bool mcb_ev_decode(uint32_t info) { return (info >> 30) & 1u; }
MCB_HD bool mcb_ev_newseq(uint32_t info) { return (info >> 31) & 1u; }

int mcb_set_error(int code, const char *msg);
void mcb_clear_error();

// LeCaR host inputs (mcb_lecar.cpp)
void mcb_lecar_stream(int64_t seed, int64_t n, double *out);
int64_t mcb_lecar_factor_len(const int32_t *caps, int n_cap, double lr, double base, int64_t max_elapsed);
void mcb_lecar_factors(const int32_t *caps, int n_cap, double lr, double base, int64_t tlen, double *f);
