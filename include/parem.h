/*
 * parem.h -- C ABI of the B200-native PaREM hot path: chunked, speculative DFA matching.
 *
 * Method (PAPER.md = /root/reference/PAPER.md, cited "P:line"):
 *   * DFA (Q, Sigma, delta, q0, F); a string is accepted iff the last state is in F.
 *   * The input T is split into p chunks (domain decomposition, Alg. 1 lines 3-4
 *     P:81-82).  Chunk i >= 1 is run from every state of R_i = S(c_first) n L(c_last)
 *     (P:67): S(c) = states with a transition on the chunk's first symbol,
 *     L(c) = distinct destinations on the previous chunk's last symbol (reading C1).
 *     Chunk 0 starts from q0 only.
 *   * Each route counts the positions whose destination state is in F (Alg. 1 P:104-107,
 *     reading C3/C4: per-route counts), giving a per-chunk map start -> (end, hits).
 *   * The maps are joined by start state (reading C5) -- an associative function
 *     composition -- into (final state, accept flag, match count).
 *
 * Result semantics (identical to the sequential walk, readings C3, C9, C11, C12 of DESIGN.md):
 *   final_state  = q_n, or PAREM_DEAD if a missing transition was taken;
 *   accepted     = final_state in F (0 if DEAD);
 *   match_count  = #{k in [1, n] : q_k in F} (u64; the start state is never counted;
 *                  hits before a death are kept);
 *   n = 0        -> (q0, q0 in F, 0);
 *   any byte >= alphabet_size -> status PAREM_ESYMBOL, bad_offset = smallest such offset
 *                  (all n bytes are checked, regardless of death); other fields undefined.
 *
 * Threading: a parem_dfa handle is immutable after creation; concurrent matches on
 * different streams are safe as long as each in-flight call has its own workspace.
 * No function aborts or exits; errors are status codes with a thread-local message.
 */
#ifndef PAREM_H
#define PAREM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ---- */
#define PAREM_OK 0
#define PAREM_EINVAL (-1)     /* bad argument (host-detectable)                          */
#define PAREM_ESYMBOL (-2)    /* input byte >= alphabet_size (device-detected)           */
#define PAREM_ECUDA (-3)      /* CUDA runtime error (message via parem_last_error)       */
#define PAREM_ENOMEM (-4)     /* allocation failed / workspace too small                 */
#define PAREM_EINTERNAL (-5)  /* internal invariant violated (e.g. speculation unsound)  */

/* Output sentinel for a dead walk.  On INPUT, a DEAD (missing) transition is the
 * all-ones value of the table element width (0xFFFF for uint16, 0xFFFFFFFF for uint32);
 * the paper treats tables as possibly sparse. */
#define PAREM_DEAD 0xFFFFFFFFu

/* boundary_policy */
#define PAREM_BOUNDARY_GRID 0u   /* b_i = i * chunk_len, remainder to the last chunk (C7)   */
#define PAREM_BOUNDARY_SNAP 1u   /* planner: move b_i forward (<= window) to minimise |L(T[b_i-1])| */
#define PAREM_BOUNDARY_AUTO 2u   /* planner picks GRID or SNAP (GRID when every |L(c)| is small and the
                                    thread-per-chunk kernel merges converged routes, else SNAP)   */
/* candidates */
#define PAREM_CANDIDATES_PAREM 0u  /* R_i = S n L (the paper's rule)                        */
#define PAREM_CANDIDATES_ENUM 1u   /* every chunk i >= 1 starts from all of Q (Enum) */
#define PAREM_CANDIDATES_LOOKBACK 2u /* R_i = delta*(Q, T[b_i - k, b_i)) n S(T[b_i]), k = options.lookback
                                        (NEXT-2 (i); k = 1 is the paper's rule); tiny kernel only */

/* Result of one match (56 bytes).  routes = sum_i |R_i| ("calculations"; with
 * |R_0| = 1), route_steps = sum_i |R_i| * len_i (candidate-steps, the lookup roofline's
 * work), num_chunks = p.  lookups_k reports what the converging path actually executed after
 * merging routes that met (set walk: the deduplicated set per step; follow and head walks: the
 * live routes), for the lookup roofline of DESIGN.md section 7. */
typedef struct parem_result {
    uint64_t match_count;
    uint32_t final_state;
    uint32_t accepted;
    uint64_t bad_offset;
    uint64_t num_chunks;
    uint64_t routes;
    uint64_t route_steps;
    int32_t status;
    uint32_t lookups_k;   /* diagnostic: table lookups issued at distinct states by the converging
                             path's kernels, in units of 1024 (0 on the other paths) */
} parem_result;

/* Options (NULL = defaults: planner-chosen chunk length, AUTO boundaries, PaREM candidates).
 * chunk_len forces the nominal chunk length (bytes, >= 1): p = max(1, floor(n / chunk_len))
 * chunks; with GRID the remainder goes to the last chunk.  Results are independent of all
 * options (only the stats routes/route_steps/num_chunks change). */
typedef struct parem_options {
    uint64_t chunk_len;
    uint32_t boundary_policy;
    uint32_t candidates;
    uint32_t kernel;       /* 0 = auto; 1 = tiny (thread per chunk); 2 = lanes (group per chunk); 3 = conv (converging: set walk + follow + join) */
    uint32_t flags;        /* PAREM_FLAG_* */
    uint32_t lookback;     /* k for PAREM_CANDIDATES_LOOKBACK (>= 1) */
    uint32_t reserved;
} parem_options;

/* flags: the workspace's 64-byte header is already zero -- freshly zero-filled by the
 * caller, or left so by a previous call on it that completed (every completed call leaves
 * it zeroed, ESYMBOL and EINTERNAL results included).  The library then skips its per-call
 * header reset (one cudaMemsetAsync), so a match is exactly its kernel launches.  Without
 * the flag the header is reset on `stream` before the kernels. */
#define PAREM_FLAG_WS_CLEAN 1u

typedef struct parem_dfa parem_dfa;

/* Create a DFA handle (P:58 quintuple; the table is the paper's adjacency matrix Tt,
 * P:76).
 *   num_states     1 <= Q <= 4194304 (Q <= 65535 for 2-byte tables); larger -> PAREM_EINVAL
 *                  (device table offsets are 32-bit).
 *   alphabet_size  A in [1, 256]; symbols are raw byte values 0..A-1 (mapping characters
 *                  to symbols is the caller's job).
 *   table          host pointer, row-major Q x A, table[s*A + c] = delta(s, c), elements of
 *                  elem_bytes (2 or 4) bytes; an entry is < Q or DEAD (all-ones).
 *   start_state    q0 < Q.
 *   accept_bitmap  host pointer, ceil(Q/8) bytes, LSB-first: s in F iff bit (s & 7) of byte s>>3.
 * The library copies table and bitmap (the caller keeps ownership) and uploads device
 * copies to the current CUDA device.  Returns PAREM_EINVAL on a bad argument, PAREM_ECUDA /
 * PAREM_ENOMEM on device failure; *out is set only on success. */
int parem_dfa_create(uint32_t num_states, uint32_t alphabet_size, const void* table, uint32_t elem_bytes,
                     uint32_t start_state, const uint8_t* accept_bitmap, parem_dfa** out);

/* Destroy a handle.  The caller guarantees no in-flight match uses it.  NULL is a no-op. */
int parem_dfa_destroy(parem_dfa* dfa);

/* Workspace bytes needed by parem_match_async for an n-byte input with these options
 * (0 on bad arguments).  The caller allocates device memory of at least this size
 * (e.g. torch.empty(ws, dtype=torch.uint8, device="cuda")); one per in-flight call. */
size_t parem_workspace_bytes(const parem_dfa* dfa, uint64_t n, const parem_options* opts);

/* Enqueue one match on `stream` (graph-capturable; no host synchronisation).
 *   d_input    device pointer to n bytes, any alignment, caller-owned, valid until the
 *              stream work completes.
 *   d_ws       device workspace of ws_bytes >= parem_workspace_bytes(...).
 *   d_result   device pointer to one parem_result, written by the last kernel.
 * Host-detectable errors return immediately (nothing enqueued); device-side errors
 * (PAREM_ESYMBOL with the smallest bad_offset) land in d_result->status. */
int parem_match_async(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, void* d_ws, size_t ws_bytes,
                      const parem_options* opts, parem_result* d_result, void* stream /* cudaStream_t */);

/* Batched matching: `count` INDEPENDENT inputs of n bytes each, laid out back to back at
 * d_input (input i = d_input[i*n .. (i+1)*n)), each matched from q0 exactly as
 * parem_match_async would (the paper's method per input: P:65-70), results to
 * d_results[0 .. count) (device, caller-owned).  When every input is a whole number of
 * the tiny kernel's 1024-chunk tiles (DFAs with <= 32 internal states, n a multiple of
 * 64 KiB, 16-byte aligned input, no SNAP/look-back options) all inputs run in ONE launch
 * -- the throughput path for many small inputs (packets, reads): a single 1 MiB match is
 * launch- and drain-bound.  Otherwise the inputs are matched one after another on the
 * stream (same workspace).  Workspace: parem_batch_workspace_bytes(dfa, n, count, opts).
 * Per-input status/bad_offset as in parem_match_async (offsets local to the input). */
size_t parem_batch_workspace_bytes(const parem_dfa* dfa, uint64_t n, uint64_t count, const parem_options* opts);
int parem_match_batch_async(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, uint64_t count, void* d_ws,
                            size_t ws_bytes, const parem_options* opts, parem_result* d_results,
                            void* stream /* cudaStream_t */);

/* ---- one input sharded over G GPUs ----
 * The paper splits T into parts matched independently and joins their routes (P:67, P:70,
 * P:114-115).  GPU g holds segment g (bytes [o_g, o_g + n_g) of T) and computes its
 * SEGMENT MAP over the paper's candidate set for the segment's first position,
 * R = L(last byte of segment g-1) ({q0} for segment 0): map[r] =
 * (state after the segment, matches in it) for every r in R.  The G maps (Q entries of
 * 16 bytes each) are exchanged with one all-gather and folded along q0's path.
 *
 * parem_segment_map (synchronous): prev_symbol = the last byte of the previous segment
 * (-1 for segment 0); h_map: host array of num_states entries (entries outside R have
 * valid = 0); *status / *bad_offset: PAREM_OK or PAREM_ESYMBOL with the smallest bad
 * offset LOCAL to the segment.  Routes from R merge (Table II): every candidate
 * walks a head of X bytes on the device, each distinct state reached is finished with one
 * ordinary match; a segment on which routes never merge is walked whole from every
 * candidate (correct, slow).  Allocates its own device scratch. */
typedef struct parem_segmap_entry {
    uint64_t match_count;     /* matches inside the segment from this entering state */
    uint32_t end_state;       /* state after the segment, PAREM_DEAD if the walk died */
    uint32_t valid;           /* 1: the entering state is a candidate (in R)          */
} parem_segmap_entry;
int parem_segment_map(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, int32_t prev_symbol,
                      const parem_options* opts, parem_segmap_entry* h_map, int32_t* status, uint64_t* bad_offset,
                      void* stream /* cudaStream_t */);

/* Fold G segment maps (host memory, G x num_states entries, segment-major) along q0's path:
 * the join of P:70 over segments.  statuses/bad_offsets: per segment (as returned by
 * parem_segment_map), seg_offsets: o_g (global offset of each segment's first byte).
 * Writes final state, accept flag, match count and the earliest ESYMBOL (global offset) to
 * *out (num_chunks = G, routes / route_steps = 0).  Host-only, no device needed.  Returns
 * PAREM_EINTERNAL if the path enters a state that is not a candidate of the next segment
 * (cannot happen for maps built from the paper's rule: it is sound, reading C1). */
int parem_fold_segment_maps(uint32_t num_states, uint32_t start_state, const uint8_t* accept_bitmap,
                            const parem_segmap_entry* maps, uint32_t G, const int32_t* statuses,
                            const uint64_t* bad_offsets, const uint64_t* seg_offsets, parem_result* out);

/* Like parem_match_async, but the walk continues from a previous segment's result:
 * the start state is d_carry->final_state (PAREM_DEAD stays dead), counts add to
 * d_carry->match_count and bad offsets are reported as offset_base + local offset
 * (an earlier ESYMBOL in d_carry wins).  d_carry may equal d_result.  This is the
 * associativity of the composition exposed at the ABI: segments can be streamed. */
int parem_match_continue_async(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, uint64_t offset_base,
                               void* d_ws, size_t ws_bytes, const parem_options* opts,
                               const parem_result* d_carry, parem_result* d_result, void* stream);

/* Convenience: internal workspace, D2H copy of the result and a stream sync.
 * Returns the result's status (PAREM_OK, PAREM_ESYMBOL, ...). */
int parem_match(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, const parem_options* opts,
                parem_result* h_result, void* stream);

/* End to end from HOST memory: pipelines host->device copies of h_input (pinned memory
 * recommended) in segments with matching (parem_match_continue_async) on `stream`, then
 * copies the result back and synchronises.  Internal device buffers are allocated per
 * call.  Returns the result's status. */
int parem_match_host(const parem_dfa* dfa, const uint8_t* h_input, uint64_t n, const parem_options* opts,
                     parem_result* h_result, void* stream);

/* Introspection (tests, bench, DESIGN.md numbers). */
typedef struct parem_dfa_info {
    uint32_t num_states;      /* Q as given                                  */
    uint32_t internal_states; /* Q + 1 if a DEAD sink was added, else Q      */
    uint32_t alphabet_size;
    uint32_t has_sink;
    uint32_t min_L;           /* min_c |L(c)| over c < A                     */
    uint32_t max_L;           /* max_c |L(c)|                                */
    uint64_t sum_L;           /* sum_c |L(c)|                                */
    uint32_t start_state;
    uint32_t table_class;     /* 1 = tiny (<= 32 states), 2 = lanes/smem, 3 = lanes/L2 */
    uint64_t device_bytes;    /* device memory held by the handle            */
} parem_dfa_info;
int parem_dfa_get_info(const parem_dfa* dfa, parem_dfa_info* info);

typedef struct parem_plan_info {
    uint32_t kernel;          /* 1 tiny, 2 lanes, 3 conv                          */
    uint32_t block_threads;
    uint64_t grid_blocks;
    uint64_t num_chunks;      /* p                                                */
    uint64_t chunk_len;       /* nominal chunk length                             */
    uint32_t boundary_policy;
    uint32_t candidates;
    uint32_t slots;           /* candidate registers/lanes per chunk per pass     */
    uint32_t symbols_per_lookup;
    size_t smem_bytes;
    size_t workspace_bytes;
    uint32_t snap_window;
    uint32_t reserved;
} parem_plan_info;
int parem_plan(const parem_dfa* dfa, uint64_t n, const parem_options* opts, parem_plan_info* out);

/* Message of the last error on this thread ("" if none). */
const char* parem_last_error(void);

/* Version string. */
const char* parem_version(void);

/* ---- match positions (Alg. 1's visited states Rr) ----
 * parem_find_async runs the match of parem_match_async (same d_result) and then writes the
 * offsets k, ascending, of every step whose state is in F (k = 0-based offset of the symbol
 * that completes an occurrence; their number is d_result->match_count) to d_positions
 * (device, caller-owned, max_positions u64 entries; only the first max_positions are
 * written).  Every chunk's true entering state is resolved from the composition, the hit
 * counts are exclusive-scanned into output offsets and each chunk is walked once more from
 * its true state.  Workspace: parem_find_workspace_bytes (>= parem_workspace_bytes).  On an
 * ESYMBOL result the positions are unspecified.  n = 0 writes nothing. */
size_t parem_find_workspace_bytes(const parem_dfa* dfa, uint64_t n, const parem_options* opts);
int parem_find_async(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, void* d_ws, size_t ws_bytes,
                     const parem_options* opts, uint64_t* d_positions, uint64_t max_positions,
                     parem_result* d_result, void* stream);

/* ---- route trace (Alg. 1's visited-state vector Rr; Table II
 * "Visited states") ----
 * parem_trace_async runs the match (same d_result) and writes the states VISITED by the routes the
 * join selects -- the concatenation of the Rr vectors of the true route of every chunk, which
 * is the sequential run q_1 .. q_n -- for the window lo <= k < hi <= n:
 *     d_states[k - lo] = state after symbol k   (uint32; PAREM_DEAD once the walk has died).
 * d_states is device memory, caller-owned, hi - lo entries; lo == hi writes nothing.  Every
 * chunk's true entering state is resolved as for parem_find_async and the chunks that meet the
 * window are walked once more from it.  Workspace: parem_find_workspace_bytes.  On an ESYMBOL
 * result the trace is unspecified.  EINVAL if lo > hi or hi > n. */
int parem_trace_async(const parem_dfa* dfa, const uint8_t* d_input, uint64_t n, void* d_ws, size_t ws_bytes,
                      const parem_options* opts, uint64_t lo, uint64_t hi, uint32_t* d_states,
                      parem_result* d_result, void* stream);

/* ---- regular-expression front end (host) ----
 * Compiles a pattern of the paper's language (Table III): concatenation `ab`,
 * Kleene star `a*`, union `a|b`, positive closure `a+`, range `[x..y]` (every alphabet
 * byte with x <= byte <= y), optionality `a?`, groups `( )`; `\` quotes an operator byte.
 * AST -> McNaughton-Yamada-Thompson NFA -> subset construction -> minimal DFA (Moore
 * refinement), states numbered breadth-first from the start state (start = 0), complete
 * table (an unmatched suffix leads to an explicit non-accepting trap state).
 *   alphabet       NUL-terminated string of distinct bytes: symbol i is alphabet[i]; NULL or
 *                  "" = the distinct bytes of the pattern in increasing order.  The input
 *                  of a match is the symbol ids (mapping bytes to ids is the caller's job).
 *   flags          PAREM_REGEX_SEARCH: compile Sigma* R, whose match count is the number
 *                  of positions where an occurrence of R ends (the paper's "parallel"
 *                  automaton, Table I); 0: the anchored language R.
 *   max_states     capacity of `table` rows / `accept_bitmap` bits (0 = 65536).
 *   table          host, row-major max_states x A uint32 (parem_dfa_create's layout), or
 *                  NULL together with accept_bitmap for a size query (info only).
 *   accept_bitmap  host, ceil(max_states / 8) bytes, LSB-first.
 * Returns PAREM_OK, PAREM_EINVAL (syntax error / byte outside the alphabet / subset
 * explosion; parem_last_error() names the offset) or PAREM_ENOMEM (max_states too small;
 * info->num_states says how many are needed). */
#define PAREM_REGEX_SEARCH 1u
typedef struct parem_regex_info {
    uint32_t num_states;
    uint32_t alphabet_size;
    uint32_t start_state;
    uint32_t reserved;
    char alphabet[256];   /* symbol i = alphabet[i] (alphabet_size bytes, not NUL-terminated) */
} parem_regex_info;
int parem_regex_compile(const char* pattern, const char* alphabet, uint32_t flags, uint32_t max_states,
                        uint32_t* table, uint8_t* accept_bitmap, parem_regex_info* info);

/* ---- transition-table text I/O ("the PaREM creates a log file with the
 * transition table"; format S:184-188).  Host only.  UTF-8 / LF text:
 *     symbols<TAB>s1<TAB>s2...        one character per symbol (\xHH for a byte that is not a
 *                                     printable ASCII character other than backslash)
 *     start<TAB><id>
 *     finals[<TAB><id>...]            zero or more ids
 *     <state-id><TAB><dest or ->...   one row per state in id order, '-' = DEAD
 * parem_table_write_text: row-major uint32 table (PAREM_DEAD = missing), LSB-first accept bitmap,
 * alphabet_size symbol bytes; *needed = bytes of text (no NUL); out == NULL is a size query;
 * ENOMEM if cap < *needed.  parem_table_read_text: the inverse (read(write(d)) == d exactly);
 * table / accept_bitmap == NULL is a size query (info->num_states, alphabet_size, start_state,
 * alphabet); EINVAL on malformed text with "line N: reason" in parem_last_error(); ENOMEM if
 * the table has more than max_states states. */
int parem_table_write_text(uint32_t num_states, uint32_t alphabet_size, const uint32_t* table, uint32_t start_state,
                           const uint8_t* accept_bitmap, const char* alphabet, char* out, size_t cap, size_t* needed);
int parem_table_read_text(const char* text, size_t len, uint32_t max_states, uint32_t* table, uint8_t* accept_bitmap,
                          parem_regex_info* info);

/* ---- per-kernel timing (bench.py; off by default) ----
 * parem_profile(1) clears the record and makes every later match issued by this host
 * thread record CUDA events on its stream around each kernel it launches (not while the
 * stream is being captured into a graph); parem_profile(0) stops recording.
 * parem_profile_read() waits for the events and returns one entry per recorded kernel
 * launch, in launch order: kernel name, device duration (ms) and the index of its match
 * since parem_profile(1); *count = number of entries (<= max are written).
 * Returns PAREM_OK or PAREM_ECUDA. */
typedef struct parem_kernel_time {
    char name[40];
    float ms;
    uint32_t match;
} parem_kernel_time;
int parem_profile(int enable);
int parem_profile_read(parem_kernel_time* out, int max, int* count);

/* ---- roofline micro-benchmarks (bench.py; not part of the matching path) ----
 * Each returns the device time in milliseconds of `reps` back-to-back launches measured
 * with CUDA events on `stream` (or a negative status).
 *   read_stream: 16-B vector loads over n bytes, grid-stride, reduced to *d_sink.
 *   gather:      every thread performs `steps` dependent random lookups into a table of
 *                table_bytes (uint16 entries) held in shared memory (where=0) or global /
 *                L2 (where=1; indices scattered over the whole table) or in shared memory,
 *                lane-private (where=2); every chain mixes its own pseudo-random stream into
 *                the next index (chains never coalesce, as routes under different inputs do
 *                not); lookups_out = total lookups per launch.  d_sink[0..1]:
 *                the kernels write d_sink[0] only if their result equals d_sink[1] (pass
 *                0xFFFFFFFF there), which keeps the loads alive. */
float parem_bench_read_stream(const uint8_t* d_input, uint64_t n, uint32_t* d_sink, int reps, void* stream);
float parem_bench_gather(uint32_t where, const uint16_t* d_table, uint32_t table_entries, uint32_t steps,
                         uint32_t* d_sink, uint64_t* lookups_out, int reps, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PAREM_H */
