// Host-side inputs of the LeCaR replay (policies.py:305-395).
//
// The reference gives every per-layer LeCaRPolicy its own random.Random(seed)
// (policies.py:347), so every cache instance draws the SAME stream of
// random() values, one per eviction (policies.py:381).  The stream is
// materialised here with CPython's MT19937 (init_by_array seeding from the
// integer's 32-bit digits, genrand_res53 doubles) and handed to the device
// as a table indexed by the instance's eviction count.
//
// The regret update (lecar_update, policies.py:305-327) multiplies one weight
// by exp(learning_rate * discount**elapsed), discount = discount_base **
// (1 / capacity).  Those factors depend only on (capacity, elapsed), so they
// are evaluated here with the host libm -- the pow / exp the reference's
// float ** int and math.exp call -- and the device only multiplies, adds and
// divides (IEEE-exact, so the weights match the reference bit for bit).
#include <math.h>
#include <stdint.h>
#include <string.h>

#include <vector>

#include "mcb_internal.h"

namespace {

// MT19937 as CPython's _randommodule.c uses it (Matsumoto & Nishimura's
// reference algorithm).
struct MT {
    static const int N = 624, M = 397;
    uint32_t mt[N];
    int mti = N + 1;

    void init_genrand(uint32_t s) {
        mt[0] = s;
        for (mti = 1; mti < N; ++mti) mt[mti] = 1812433253u * (mt[mti - 1] ^ (mt[mti - 1] >> 30)) + (uint32_t)mti;
    }
    void init_by_array(const uint32_t *key, size_t len) {
        init_genrand(19650218u);
        size_t i = 1, j = 0;
        for (size_t k = (N > len ? N : len); k; --k) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
            ++i;
            ++j;
            if (i >= (size_t)N) { mt[0] = mt[N - 1]; i = 1; }
            if (j >= len) j = 0;
        }
        for (size_t k = N - 1; k; --k) {
            mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
            ++i;
            if (i >= (size_t)N) { mt[0] = mt[N - 1]; i = 1; }
        }
        mt[0] = 0x80000000u;
        mti = N;
    }
    uint32_t next() {
        static const uint32_t mag01[2] = {0u, 0x9908b0dfu};
        if (mti >= N) {
            int kk = 0;
            uint32_t y;
            for (; kk < N - M; ++kk) {
                y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
                mt[kk] = mt[kk + M] ^ (y >> 1) ^ mag01[y & 1u];
            }
            for (; kk < N - 1; ++kk) {
                y = (mt[kk] & 0x80000000u) | (mt[kk + 1] & 0x7fffffffu);
                mt[kk] = mt[kk + (M - N)] ^ (y >> 1) ^ mag01[y & 1u];
            }
            y = (mt[N - 1] & 0x80000000u) | (mt[0] & 0x7fffffffu);
            mt[N - 1] = mt[M - 1] ^ (y >> 1) ^ mag01[y & 1u];
            mti = 0;
        }
        uint32_t y = mt[mti++];
        y ^= y >> 11;
        y ^= (y << 7) & 0x9d2c5680u;
        y ^= (y << 15) & 0xefc60000u;
        y ^= y >> 18;
        return y;
    }
    double random() {   // genrand_res53
        const uint32_t a = next() >> 5, b = next() >> 6;
        return ((double)a * 67108864.0 + (double)b) * (1.0 / 9007199254740992.0);
    }
};

void seed_python(MT &g, int64_t seed) {
    // random.seed(int): abs(n) split into 32-bit digits, least significant first (at least one)
    uint64_t n = seed < 0 ? (uint64_t)0 - (uint64_t)seed : (uint64_t)seed;
    uint32_t key[2] = {(uint32_t)n, (uint32_t)(n >> 32)};
    g.init_by_array(key, key[1] ? 2 : 1);
}

}  // namespace

extern "C" int mcb_lecar_random(int64_t seed, int64_t n, double *out) {
    mcb_clear_error();
    if (n < 0 || (n > 0 && !out)) return mcb_set_error(MCB_ERR_INVALID, "invalid output");
    MT g;
    seed_python(g, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = g.random();
    return MCB_OK;
}

// Regret factors per capacity: f[c][e] = exp(lr * pow(discount_base ** (1/cap_c), e))
// for e < tlen, and every elapsed >= tlen has factor exactly 1.0.  tlen is the
// first elapsed whose argument lr * discount**e is below 2^-54 (exp rounds to
// 1.0 there and for every larger e, the sequence being non-increasing), else
// max_elapsed + 1.  Returns tlen; fills f (n_cap * tlen) when f != nullptr.
int64_t mcb_lecar_factor_len(const int32_t *caps, int n_cap, double lr, double base, int64_t max_elapsed) {
    int64_t tlen = 1;
    for (int c = 0; c < n_cap; ++c) {
        const double d = pow(base, 1.0 / (double)caps[c]);
        int64_t e = 0;
        const bool decays = lr >= 0.0 && d >= 0.0 && d < 1.0;
        if (!decays) {
            e = max_elapsed + 1;
        } else {
            while (e <= max_elapsed && !(lr * pow(d, (double)e) < 0x1p-54)) ++e;
        }
        if (e + 1 > tlen) tlen = e + 1;
    }
    if (tlen > max_elapsed + 1) tlen = max_elapsed + 1;
    return tlen;
}

void mcb_lecar_factors(const int32_t *caps, int n_cap, double lr, double base, int64_t tlen, double *f) {
    for (int c = 0; c < n_cap; ++c) {
        const double d = pow(base, 1.0 / (double)caps[c]);   // discount_base ** (1.0 / capacity)
        for (int64_t e = 0; e < tlen; ++e) {
            const double reward = pow(d, (double)e);         // discount ** elapsed
            f[(int64_t)c * tlen + e] = exp(lr * reward);     // math.exp(learning_rate * reward)
        }
    }
}

void mcb_lecar_stream(int64_t seed, int64_t n, double *out) {
    MT g;
    seed_python(g, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = g.random();
}
