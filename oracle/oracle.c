/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously correct CPU
 * definition of what the PaREM hot path computes.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.  It shares
 * no code with the CUDA path (paper_1412_1741_b200/) and imports nothing from it.
 *
 * Sources (/root/reference/PAPER.md = "P:line"):
 *   DFA semantics  (Q, Sigma, delta, q0, F), acceptance iff the last state is in F  -- P:58
 *   sequential REM: start from q0, n steps                                        -- P:65
 *   what is counted: Alg. 1 "if Tt[r][char] in F: found++" tests the DESTINATION  -- P:104-107
 *   S(c) = {q : delta(q,c) defined}, L(c) = {delta(q,c)}, R = S n L, R_0 = {q0}     -- P:67-68
 * Readings taken where the paper is silent:
 *   C3  count = #{k in 1..n : q_k in F}; the empty prefix is never counted.
 *   C9  DEAD (missing entry = all-ones of the element width) ends the walk: final = DEAD,
 *       accept = false, count = hits before death.
 *   C11 any byte >= A is a hard error ESYMBOL at the SMALLEST offending offset, checked
 *       over all n bytes before matching, regardless of death.
 *   C12 n = 0 gives (q0, q0 in F, 0).
 * Pins (tests/test_oracle*.py): Table I / Table II values, (a|b)*abb hand strings,
 * exhaustive regex fullmatch on short strings, naive substring counts, one-hot x 0/1
 * transition-matrix products, partition invariants.
 */
#include <stdint.h>
#include <stddef.h>

#define ORACLE_OK 0
#define ORACLE_EINVAL (-1)
#define ORACLE_ESYMBOL (-2)
#define ORACLE_DEAD 0xFFFFFFFFu

typedef struct {
    uint64_t match_count;
    uint32_t final_state;   /* ORACLE_DEAD if the walk died */
    uint32_t accepted;
    uint64_t bad_offset;    /* valid iff status == ORACLE_ESYMBOL */
    int32_t status;
    uint32_t reserved;
} oracle_result;

static inline uint32_t entry(const void* table, uint32_t eb, uint64_t idx) {
    return eb == 2 ? ((const uint16_t*)table)[idx] : ((const uint32_t*)table)[idx];
}

static inline int in_F(const uint8_t* acc_bitmap, uint32_t s) {
    return (acc_bitmap[s >> 3] >> (s & 7)) & 1;   /* LSB-first bitmap */
}

/* delta as an all-ones-means-DEAD table, normalised to ORACLE_DEAD */
static inline uint32_t delta(const void* table, uint32_t eb, uint32_t A, uint32_t s, uint32_t c) {
    uint32_t v = entry(table, eb, (uint64_t)s * A + c);
    if ((eb == 2 && v == 0xFFFFu) || (eb == 4 && v == 0xFFFFFFFFu)) return ORACLE_DEAD;
    return v;
}

/* Sequential DFA walk. */
int oracle_walk(uint32_t Q, uint32_t A, const void* table, uint32_t eb, uint32_t q0,
                const uint8_t* acc_bitmap, const uint8_t* T, uint64_t n, oracle_result* out) {
    out->match_count = 0; out->final_state = ORACLE_DEAD; out->accepted = 0;
    out->bad_offset = 0; out->status = ORACLE_OK; out->reserved = 0;
    if (Q == 0 || A == 0 || A > 256 || q0 >= Q || (eb != 2 && eb != 4)) {
        out->status = ORACLE_EINVAL; return ORACLE_EINVAL;
    }
    /* C11: validate every byte first, smallest offending offset wins */
    for (uint64_t k = 0; k < n; ++k)
        if (T[k] >= A) { out->status = ORACLE_ESYMBOL; out->bad_offset = k; return ORACLE_ESYMBOL; }
    uint32_t s = q0;
    uint64_t count = 0;
    for (uint64_t k = 0; k < n; ++k) {
        uint32_t e = delta(table, eb, A, s, T[k]);
        if (e == ORACLE_DEAD) {            /* C9 */
            out->match_count = count; out->final_state = ORACLE_DEAD; out->accepted = 0;
            return ORACLE_OK;
        }
        if (e >= Q) { out->status = ORACLE_EINVAL; return ORACLE_EINVAL; }
        s = e;
        if (in_F(acc_bitmap, s)) count += 1;   /* destination tested, C3 */
    }
    out->match_count = count;
    out->final_state = s;
    out->accepted = (uint32_t)in_F(acc_bitmap, s);
    return ORACLE_OK;
}

/* NEXT-2 (i): the k-symbol look-back candidate rule, a generalisation of L (
 * related work P:529): for i >= 1
 *   R_i^(k) = delta*(Q, T[max(0, b_i - k), b_i)) n S(T[b_i]),
 * the states some start can be in after the k symbols before the boundary (DEAD removed),
 * restricted to those with a transition on the chunk's first symbol; k = 1 is the paper's
 * R = S n L.  |R_0| = 1.  Direct set iteration, O(p * k * Q). */
int oracle_lookback_stats(uint32_t Q, uint32_t A, const void* table, uint32_t eb, const uint8_t* T, uint64_t n,
                          const uint64_t* b, uint64_t p, uint64_t k, uint64_t* routes, uint64_t* route_steps,
                          uint8_t* scratch /* 2 Q bytes */) {
    if (p == 0 || b[0] != 0 || b[p] != n || k == 0) return ORACLE_EINVAL;
    uint8_t* cur = scratch;
    uint8_t* nxt = scratch + Q;
    uint64_t r_total = 1, steps = b[1] - b[0];
    for (uint64_t i = 1; i < p; ++i) {
        if (b[i] <= b[i - 1] || b[i] >= n) return ORACLE_EINVAL;
        for (uint32_t q = 0; q < Q; ++q) cur[q] = 1;   /* all of Q */
        const uint64_t a = b[i] > k ? b[i] - k : 0;
        for (uint64_t j = a; j < b[i]; ++j) {           /* the image under T[j] */
            if (T[j] >= A) return ORACLE_ESYMBOL;
            for (uint32_t q = 0; q < Q; ++q) nxt[q] = 0;
            for (uint32_t q = 0; q < Q; ++q)
                if (cur[q]) {
                    uint32_t d = delta(table, eb, A, q, T[j]);
                    if (d != ORACLE_DEAD) nxt[d] = 1;
                }
            uint8_t* t = cur; cur = nxt; nxt = t;
        }
        if (T[b[i]] >= A) return ORACLE_ESYMBOL;
        uint64_t r = 0;
        for (uint32_t q = 0; q < Q; ++q)
            if (cur[q] && delta(table, eb, A, q, T[b[i]]) != ORACLE_DEAD) ++r;
        r_total += r;
        steps += r * (b[i + 1] - b[i]);
    }
    *routes = r_total;
    *route_steps = steps;
    return ORACLE_OK;
}

/* Match end positions (NEXT-4; Alg. 1's visited-state vector Rr, reduced to the
 * steps whose destination is in F): every k in [0, n) with q_{k+1} in F, ascending, i.e.
 * the 0-based offset of the symbol that completes an occurrence.  Writes min(count, cap)
 * offsets; *count = all of them (= oracle_walk's match_count).  Stops at DEAD (C9);
 * ESYMBOL as oracle_walk (C11). */
int oracle_positions(uint32_t Q, uint32_t A, const void* table, uint32_t eb, uint32_t q0,
                     const uint8_t* acc_bitmap, const uint8_t* T, uint64_t n, uint64_t* pos, uint64_t cap,
                     uint64_t* count) {
    *count = 0;
    if (Q == 0 || A == 0 || A > 256 || q0 >= Q || (eb != 2 && eb != 4)) return ORACLE_EINVAL;
    for (uint64_t k = 0; k < n; ++k)
        if (T[k] >= A) return ORACLE_ESYMBOL;
    uint32_t s = q0;
    uint64_t c = 0;
    for (uint64_t k = 0; k < n; ++k) {
        uint32_t e = delta(table, eb, A, s, T[k]);
        if (e == ORACLE_DEAD) break;
        if (e >= Q) return ORACLE_EINVAL;
        s = e;
        if (in_F(acc_bitmap, s)) {
            if (c < cap) pos[c] = k;
            ++c;
        }
    }
    *count = c;
    return ORACLE_OK;
}

/* State after consuming T[0..offsets[j]) for ascending offsets (ORACLE_DEAD once dead).
 * Used for the speculation-soundness checks: the true boundary state lies in R_i. */
int oracle_states_at(uint32_t Q, uint32_t A, const void* table, uint32_t eb, uint32_t q0,
                     const uint8_t* T, uint64_t n, const uint64_t* offsets, uint64_t m,
                     uint32_t* states) {
    if (Q == 0 || A == 0 || A > 256 || q0 >= Q) return ORACLE_EINVAL;
    uint32_t s = q0;
    uint64_t k = 0;
    for (uint64_t j = 0; j < m; ++j) {
        uint64_t target = offsets[j];
        if (target > n || (j > 0 && target < offsets[j - 1])) return ORACLE_EINVAL;
        for (; k < target; ++k) {
            if (T[k] >= A) return ORACLE_ESYMBOL;
            if (s != ORACLE_DEAD) s = delta(table, eb, A, s, T[k]);
        }
        states[j] = s;
    }
    return ORACLE_OK;
}

/* The paper's speculation counts for a given partition b[0]=0 < b[1] < ... < b[p]=n
 * (P:67-68): |R_0| = 1 and, for i >= 1,
 *   R_i = S(T[b_i]) n L(T[b_i - 1]),  S(c) = {q : delta(q,c) != DEAD},
 *   L(c) = {delta(q,c) : q in Q} \ {DEAD}.
 * routes = sum_i |R_i|  ("calculations"),  route_steps = sum_i |R_i| * (b_{i+1}-b_i).
 * Computed by direct set construction per boundary (O(p*Q)). */
int oracle_route_stats(uint32_t Q, uint32_t A, const void* table, uint32_t eb,
                       const uint8_t* T, uint64_t n, const uint64_t* b, uint64_t p,
                       uint64_t* routes, uint64_t* route_steps, uint8_t* scratch /* Q bytes */) {
    if (p == 0 || b[0] != 0 || b[p] != n) return ORACLE_EINVAL;
    uint64_t r_total = 1, steps = b[1] - b[0];
    for (uint64_t i = 1; i < p; ++i) {
        if (b[i] <= b[i - 1] || b[i] >= n) return ORACLE_EINVAL;
        uint32_t c_last = T[b[i] - 1], c_first = T[b[i]];
        if (c_last >= A || c_first >= A) return ORACLE_ESYMBOL;
        for (uint32_t q = 0; q < Q; ++q) scratch[q] = 0;
        for (uint32_t q = 0; q < Q; ++q) {            /* L(c_last) */
            uint32_t d = delta(table, eb, A, q, c_last);
            if (d != ORACLE_DEAD) scratch[d] = 1;
        }
        uint64_t r = 0;
        for (uint32_t q = 0; q < Q; ++q)              /* intersect with S(c_first) */
            if (scratch[q] && delta(table, eb, A, q, c_first) != ORACLE_DEAD) ++r;
        r_total += r;
        steps += r * (b[i + 1] - b[i]);
    }
    *routes = r_total;
    *route_steps = steps;
    return ORACLE_OK;
}
