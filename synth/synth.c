/*
 * synth.c -- seeded synthetic inputs for the PaREM hot path.
 *
 * This module is the ONLY code shared by the oracle (oracle/) and the CUDA
 * path (paper_1412_1741_b200/): it produces input byte strings and DFA
 * transition tables.  It contains none of the method's arithmetic (no chunking,
 * no S/L/R speculation, no route walks, no composition, no DFA execution).
 *
 * RNG: a counter-based SplitMix64 finalizer over (seed, stream, index), so any
 * index range can be generated independently and in parallel, bit-reproducibly.
 *   key(seed, stream)      = fmix(seed * GOLDEN ^ fmix(stream + 1))
 *   draw(seed, stream, i)  = fmix(key + (i + 1) * GOLDEN)
 * Uniform symbol in [0, A):   floor(u * A / 2^64)  (128-bit multiply-high)
 * Bernoulli(p):               u < floor(p * 2^64)
 *
 * Streams: 0 = input bytes, 1 = table targets, 2 = accept bits, 3 = pattern P,
 *          4 = sparse selectors, 5 = Markov-source permutations.
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <math.h>
#include <stdlib.h>

#define GOLDEN 0x9E3779B97F4A7C15ull

static inline uint64_t fmix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline uint64_t key_of(uint64_t seed, uint64_t stream) {
    return fmix(seed * GOLDEN ^ fmix(stream + 1));
}

static inline uint64_t draw_k(uint64_t key, uint64_t i) { return fmix(key + (i + 1) * GOLDEN); }

static inline uint32_t below(uint64_t u, uint32_t A) {
    return (uint32_t)(((unsigned __int128)u * A) >> 64);
}

uint64_t synth_draw(uint64_t seed, uint64_t stream, uint64_t index) {
    return draw_k(key_of(seed, stream), index);
}

uint32_t synth_below(uint64_t seed, uint64_t stream, uint64_t index, uint32_t A) {
    return below(synth_draw(seed, stream, index), A);
}

uint64_t synth_bernoulli_threshold(double p) {
    if (p <= 0.0) return 0;
    if (p >= 1.0) return UINT64_MAX;
    return (uint64_t)ldexp(p, 64);
}

/* out[k] = uniform symbol in [0, A) for absolute index (offset + k). */
void synth_uniform_symbols(uint8_t* out, uint64_t n, uint32_t A, uint64_t seed,
                           uint64_t stream, uint64_t offset) {
    const uint64_t key = key_of(seed, stream);
    int64_t nn = (int64_t)n;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < nn; ++k)
        out[k] = (uint8_t)below(draw_k(key, offset + (uint64_t)k), A);
}

/* out[s] = 1 with probability p (stream 2 by convention). */
void synth_bernoulli(uint8_t* out, uint64_t n, double p, uint64_t seed, uint64_t stream) {
    const uint64_t key = key_of(seed, stream);
    const uint64_t thr = synth_bernoulli_threshold(p);
    for (uint64_t k = 0; k < n; ++k) out[k] = draw_k(key, k) < thr ? 1 : 0;
}

/* ---- DFA tables (row-major table[s*A + c], element width 2 or 4 bytes) ---- */

static inline void put(void* table, uint32_t eb, uint64_t idx, uint32_t v) {
    if (eb == 2) ((uint16_t*)table)[idx] = (uint16_t)v;
    else ((uint32_t*)table)[idx] = v;
}

/* Dense uniform random DFA: delta(s,c) uniform over Q (stream 1, index s*A+c). */
void synth_random_dfa(void* table, uint32_t eb, uint32_t Q, uint32_t A, uint64_t seed) {
    const uint64_t key = key_of(seed, 1);
    for (uint64_t i = 0; i < (uint64_t)Q * A; ++i) put(table, eb, i, below(draw_k(key, i), Q));
}

/* Sparse-adjacency DFA: each state has T distinct-draw targets t[s][j] (stream 1,
 * index T*s+j); delta(s,c) = t[s][sel(s,c)], sel uniform in [0,T) (stream 4, index A*s+c). */
void synth_sparse_dfa(void* table, uint32_t eb, uint32_t Q, uint32_t A, uint32_t T, uint64_t seed) {
    const uint64_t kt = key_of(seed, 1), ks = key_of(seed, 4);
    for (uint64_t s = 0; s < Q; ++s)
        for (uint64_t c = 0; c < A; ++c) {
            uint32_t j = below(draw_k(ks, A * s + c), T);
            put(table, eb, s * A + c, below(draw_k(kt, T * s + j), Q));
        }
}

/* Random partial DFA: like synth_random_dfa but each entry is DEAD (all-ones of the
 * element width) with probability p_dead (stream 4, index s*A+c). */
void synth_partial_dfa(void* table, uint32_t eb, uint32_t Q, uint32_t A, double p_dead, uint64_t seed) {
    const uint64_t kt = key_of(seed, 1), kd = key_of(seed, 4);
    const uint64_t thr = synth_bernoulli_threshold(p_dead);
    const uint32_t dead = eb == 2 ? 0xFFFFu : 0xFFFFFFFFu;
    for (uint64_t i = 0; i < (uint64_t)Q * A; ++i)
        put(table, eb, i, draw_k(kd, i) < thr ? dead : below(draw_k(kt, i), Q));
}

/* Literal-search DFA for Sigma* P (failure-function / KMP automaton).
 * State j = length of the longest prefix of P that is a suffix of the text read so far.
 * States 0..m; the only accepting state is m.  Row m continues like row fail(m).
 * Building the searched automaton is input preparation, not PaREM's method. */
int synth_kmp_dfa(void* table, uint32_t eb, const uint8_t* P, uint32_t m, uint32_t A) {
    if (m == 0) return -1;
    for (uint32_t k = 0; k < m; ++k) if (P[k] >= A) return -1;
    /* fail[] via the classic prefix function */
    uint32_t* pi = (uint32_t*)malloc(sizeof(uint32_t) * (m + 1));
    if (!pi) return -2;
    pi[0] = 0;
    for (uint32_t i = 1, k = 0; i < m; ++i) {
        while (k > 0 && P[i] != P[k]) k = pi[k - 1];
        if (P[i] == P[k]) ++k;
        pi[i] = k;
    }
    for (uint32_t s = 0; s <= m; ++s)
        for (uint32_t c = 0; c < A; ++c) {
            uint32_t v;
            if (s < m && P[s] == c) v = s + 1;
            else if (s == 0) v = 0;
            else {
                uint32_t f = pi[s - 1]; /* fall back to the longest proper border */
                /* the row of state f has already been filled (f < s) */
                v = eb == 2 ? ((uint16_t*)table)[(uint64_t)f * A + c]
                            : ((uint32_t*)table)[(uint64_t)f * A + c];
            }
            put(table, eb, (uint64_t)s * A + c, v);
        }
    free(pi);
    return 0;
}

/* ---- cfg5: order-1 Markov source with a skewed (Zipf 1.1) symbol distribution ----
 * Row a in 0..255 (and an extra initial row 256) has a random permutation pi_a of the
 * 256 symbols (Fisher-Yates; stream 5, index 256*a + k).  All rows share the rank
 * weights (r+1)^-1.1; next symbol x_k = pi_{x_{k-1}}[F^-1(u_k)], u_k = draw(seed, 0, k).
 * The first byte of every 2^20-byte block uses row 256, so blocks are independent. */
#define MARKOV_BLOCK (1ull << 20)

static void markov_tables(uint64_t seed, uint8_t perm[257][256], uint64_t thr[256]) {
    const uint64_t kp = key_of(seed, 5);
    for (uint32_t a = 0; a < 257; ++a) {
        for (uint32_t k = 0; k < 256; ++k) perm[a][k] = (uint8_t)k;
        for (uint32_t k = 255; k > 0; --k) {
            uint32_t j = below(draw_k(kp, 256ull * a + k), k + 1);
            uint8_t t = perm[a][k]; perm[a][k] = perm[a][j]; perm[a][j] = t;
        }
    }
    double w[256], tot = 0.0;
    for (int r = 0; r < 256; ++r) { w[r] = pow((double)(r + 1), -1.1); tot += w[r]; }
    double cum = 0.0;
    for (int r = 0; r < 256; ++r) {
        cum += w[r];
        double f = cum / tot;
        thr[r] = r == 255 ? UINT64_MAX : (uint64_t)ldexp(f, 64);
    }
}

static inline uint32_t rank_of(const uint64_t thr[256], uint64_t u) {
    uint32_t lo = 0, hi = 255; /* first r with u < thr[r] (thr[255] = max) */
    while (lo < hi) { uint32_t mid = (lo + hi) >> 1; if (u < thr[mid]) hi = mid; else lo = mid + 1; }
    return lo;
}

void synth_markov_bytes(uint8_t* out, uint64_t n, uint64_t seed) {
    static uint8_t perm[257][256];
    uint64_t thr[256];
    markov_tables(seed, perm, thr);
    const uint64_t key = key_of(seed, 0);
    int64_t nblocks = (int64_t)((n + MARKOV_BLOCK - 1) / MARKOV_BLOCK);
#pragma omp parallel for schedule(static)
    for (int64_t b = 0; b < nblocks; ++b) {
        uint64_t lo = (uint64_t)b * MARKOV_BLOCK, hi = lo + MARKOV_BLOCK;
        if (hi > n) hi = n;
        uint32_t prev = 256;
        for (uint64_t k = lo; k < hi; ++k) {
            uint32_t r = rank_of(thr, draw_k(key, k));
            uint8_t x = perm[prev][r];
            out[k] = x;
            prev = x;
        }
    }
}
