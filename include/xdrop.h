/*
 * include/xdrop.h -- C ABI of the B200-native batched X-drop seed-and-extend
 * library (libxdrop.so, built from paper_2309_07270_b200/csrc/).
 *
 * What the library computes
 * -------------------------
 * For each candidate read pair with a shared k-mer seed it runs ALIGN:
 *   seed  = sum_{t<k} s(A[a_pos+t], B[b_pos+t])
 *   R     = EXTEND(A[a_pos+k:], B[b_pos+k:])                 (right extension)
 *   L     = EXTEND(reverse(A[:a_pos]), reverse(B[:b_pos]))   (left extension)
 * where EXTEND is the anti-diagonal X-drop dynamic program: cells of one
 * anti-diagonal d = i + j are independent (§II on LOGAN), a cell
 * is dead when its value falls below (best over anti-diagonals < d) - X
 * ("X-drop"; "--ga 15"), and the
 * recurrence is Needleman-Wunsch with linear gaps ("essentially
 * Needleman-Wunsch or Smith-Waterman algorithm with X-Drop").
 * Every detail the paper leaves open (tie-breaks, hull, termination, seed
 * score, coordinates) is fixed in DESIGN.md "Readings"; the
 * CPU oracle in oracle/ implements the same reading independently.
 *
 * Conventions
 * -----------
 * - Every function returns XDROP_OK (0) or a negative xdrop_status; nothing
 *   throws across the ABI.  xdrop_strerror() names a status.
 * - Ownership: the caller owns every buffer it passes (host or device) and
 *   every output buffer; the library owns its device workspaces and streams.
 *   xdrop_align_batch is synchronous: inputs may be freed on return and `out`
 *   is complete.
 * - On error the outputs are unspecified and xdrop_last_error_index() returns
 *   the offending pair index (EINVAL/ESEED/ELENGTH) or pool base index
 *   (EALPHABET), else -1.
 * - Determinism: results are bit-identical across runs, policies, device
 *   counts and kernel paths (the result never depends on the band window).
 * - Thread safety: one context per host thread, or serialise calls.
 */
#ifndef XDROP_H_
#define XDROP_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  XDROP_OK = 0,
  XDROP_EINVAL = -1,     /* bad argument (null pointer, bad params, bad id) */
  XDROP_ENOMEM = -2,     /* host or device allocation failed */
  XDROP_ECUDA = -3,      /* CUDA runtime error */
  XDROP_EALPHABET = -4,  /* a base outside {A,C,G,T,a,c,g,t} ("--alph dna") */
  XDROP_ESEED = -5,      /* seed out of range: a_pos<0, a_pos+k>|A| (same for B) */
  XDROP_ELENGTH = -6,    /* a read longer than XDROP_MAX_READ_LEN, or score range exceeded */
  XDROP_ESTATE = -7,     /* call on a finalized / null context */
  XDROP_ENODEV = -8      /* no usable CUDA device */
} xdrop_status;

/* Rank->GPU mapping policies.  CELLS is the default sharding by estimated cell
 * count; the other three re-create the paper's schedulers (§III-B..D,
 * Alg. 1 l.5-30): ONE2ALL = one logical rank at a time drives all GPUs,
 * ONE2ONE = rank r drives GPU r mod m with per-pipeline token rings (token per
 * sub-batch), OPT_ONE2ONE = as ONE2ONE with the token held per batch
 * (BASELINE.json's "mixed scheme").  Results never depend on the policy. */
typedef enum {
  XDROP_POLICY_CELLS = 0,
  XDROP_POLICY_ONE2ALL = 1,
  XDROP_POLICY_ONE2ONE = 2,
  XDROP_POLICY_OPT_ONE2ONE = 3
} xdrop_policy;

#define XDROP_MAX_READ_LEN (1 << 18) /* bases per read (fast-path key range) */

/* Scoring and X-drop parameters.  Valid ranges: 1 <= match <= 32,
 * -64 <= mismatch <= -1, -64 <= gap <= -1, 0 <= xdrop <= 2^20,
 * 1 <= k <= 1024.  BASELINE: {+1, -1, -1, 15, 17}; the paper ran k=31, X=15
 * (PAPER.md:221, 224). */
typedef struct {
  int32_t match, mismatch, gap, xdrop, k;
} xdrop_params;

typedef struct {
  const int* devices;   /* CUDA device ordinals; NULL -> device 0 .. n_devices-1 */
  int n_devices;        /* >= 1 */
  int policy;           /* xdrop_policy */
  int n_ranks;          /* logical ranks for ONE2ALL/ONE2ONE/OPT (>= 1); ignored by CELLS */
  int batch_size;       /* pairs per batch, PAPER.md:100 ("batches of size 10,000"); 0 -> 10000 */
  int subbatches;       /* c sub-batches per batch; 0 -> 1 */
  int flags;            /* XDROP_FLAG_* */
} xdrop_init_opts;

#define XDROP_FLAG_FORCE_WIDE 1    /* skip the lane-per-extension path (tests; ignored with SEQAN_COMPAT) */
#define XDROP_FLAG_FORCE_GENERAL 2 /* send every extension to the unbounded fallback (tests) */
#define XDROP_FLAG_NO_SORT 4       /* do not length-sort the work queue (tests) */
/* Packed-mode band kernel (X + M <= 510).  Default: chosen per batch on the device by
 * a probe (up to 4096 evenly spaced extensions of the batch run for <= 128 anti-diagonals in the T0
 * window; the shared kernel when the predicted T0 -> T1 escalations reach 1024, else the tiered
 * one); results are identical either way. */
#define XDROP_FLAG_TIERED 8        /* always the tiered kernel (small per-tier loops, short tails) */
#define XDROP_FLAG_SHARED 16       /* always the shared kernel (one loop for every tier, no I$ thrash) */
/* SeqAn/LOGAN-style conventions (readings Q28-Q30; LOGAN is the
 * aligner PAPER.md:85-89 names, the conventions themselves are not in the paper): a pure-gap cell
 * (i = 0 or j = 0) is live only if H > best - X (strict), and each extension reports its "longest
 * extension" -- the largest-H live cell of the last anti-diagonal holding a live cell, smallest i on
 * ties -- and H at that cell instead of the maximum (xdrop_result.score = seed + both such H;
 * begin / end = those cells).  Thresholds, hull, `cells` and termination are the default mode's.
 * Packed mode (X + M <= 510): the default mode's packed tiers in compat instances up to S = 2,048,
 * wider extensions restart in shared-memory-ring / global-memory general-path kernels; 32-bit mode
 * (or env XDROP_COMPAT_GENERAL=1): the general path only.  All entry points honour it. */
#define XDROP_FLAG_SEQAN_COMPAT 32

/* A read pool in HOST memory: ASCII bases, read r = seq[offsets[r] .. offsets[r+1]). */
typedef struct {
  const char* seq;
  const int64_t* offsets; /* n + 1 entries, non-decreasing, offsets[0] >= 0 */
  int64_t n;              /* number of reads */
} xdrop_seqs;

/* One candidate pair: seed A[a_pos, a_pos+k) ~ B'[b_pos, b_pos+k).  16 bytes.
 * B' = B, or reverse(complement(B)) when b_id has bit 31 set (b_id | XDROP_PAIR_RC: the
 * reads come from opposite strands); b_pos, b_begin and b_end are then positions in B'
 * (reading Q16). */
typedef struct {
  int32_t a_id, b_id, a_pos, b_pos;
} xdrop_pair;
#define XDROP_PAIR_RC ((int32_t)0x80000000)

/* Result of ALIGN, 0-based half-open coordinates [begin, end).  20 bytes. */
typedef struct {
  int32_t score, a_begin, a_end, b_begin, b_end;
} xdrop_result;

typedef struct xdrop_ctx xdrop_ctx;

/* Create a context over opts->n_devices GPUs (NULL opts: 1 GPU, CELLS). */
int xdrop_init(const xdrop_init_opts* opts, xdrop_ctx** out_ctx);

/* Align n_pairs pairs (host buffers).  B may equal A (same pool).  out has
 * n_pairs entries; cells_out (nullable) receives per-pair DP cell counts
 * (hull cells of the left + right extensions). */
int xdrop_align_batch(xdrop_ctx* ctx, const xdrop_seqs* A, const xdrop_seqs* B,
                      const xdrop_pair* pairs, int64_t n_pairs, const xdrop_params* p,
                      xdrop_result* out, int64_t* cells_out);

/* Device-resident variant on the context's first device: every pointer is
 * device memory (e.g. torch tensors' data_ptr()).  seqA/offA describe an ASCII
 * pool of nA reads with total length lenA (= offA[nA], passed so no D2H read
 * is needed); seqB may equal seqA.  Work is enqueued on `stream`
 * (cudaStream_t, NULL = the context's stream); the call returns after the
 * stream has completed so it can report validation errors.
 * Validation happens on the device (prep_kernel) before any extension runs: a
 * pair whose read id is out of range, whose read's offsets leave the pool
 * (off[r] < 0, off[r+1] < off[r] or off[r+1] > len), whose read exceeds
 * XDROP_MAX_READ_LEN or whose seed leaves a read returns XDROP_ESEED with
 * xdrop_last_error_index() = the smallest such pair index.  The work queue is
 * emptied on the device first, so no band kernel dereferences an unvalidated
 * id or position, and the context stays usable.  A base outside the alphabet
 * returns XDROP_EALPHABET (checked first) with the pool base index. */
int xdrop_align_batch_device(xdrop_ctx* ctx,
                             const char* seqA, const int64_t* offA, int64_t nA, int64_t lenA,
                             const char* seqB, const int64_t* offB, int64_t nB, int64_t lenB,
                             const xdrop_pair* pairs, int64_t n_pairs, const xdrop_params* p,
                             xdrop_result* out, int64_t* cells_out, void* stream);

/* ---- registered read pools (the pool is replicated once, not per call) ----
 * ELBA aligns many batches ("batches of size 10,000") against the same reads.
 * xdrop_pool_register uploads a host pool ONCE: the ASCII bases go to the context's first device and
 * are 2-bit packed there (alphabet check: XDROP_EALPHABET + base index), the packed words (0.25 B
 * per base) are copied device-to-device to every other device of the context (cudaMemcpyPeer: NVLink
 * on a multi-GPU node), and the offsets are kept on every device plus a host copy (validation and
 * cost estimates).  *pool_id receives a handle >= 0; the caller's buffers may be freed on return.
 * xdrop_align_pooled is xdrop_align_batch on registered pools (poolB may equal poolA): only the pairs
 * (16 B) go to the devices and only the results come back; same validation, scheduling policies,
 * results and statistics.  xdrop_pool_release frees a pool (XDROP_EINVAL for an unknown id);
 * xdrop_finalize frees every pool still registered. */
int xdrop_pool_register(xdrop_ctx* ctx, const xdrop_seqs* S, int32_t* pool_id);
int xdrop_align_pooled(xdrop_ctx* ctx, int32_t poolA, int32_t poolB, const xdrop_pair* pairs, int64_t n_pairs,
                       const xdrop_params* p, xdrop_result* out, int64_t* cells_out);
int xdrop_pool_release(xdrop_ctx* ctx, int32_t pool_id);

/* ---- candidate-pair filters (device pointers, work on `stream`, the call
 * returns after the stream completed).  Neither needs a context.  On an invalid pair (read id out
 * of range, seed outside its read, a non-ACGT base in a seed) they return XDROP_ESEED and set
 * *err_index (nullable) to the smallest such pair index; XDROP_EINVAL on bad sizes or parameters.
 *
 * f2, BELLA's adaptive threshold ("An adaptive threshold is used to perform the X-drop alignment",
 * PAPER.md:74; the formula is DESIGN.md reading Q12, not the paper's): for each pair with result
 * res[p] (e.g. the `out` of xdrop_align_batch_device), ov = min(a_pos, b_pos) + min(|A| - a_pos,
 * |B'| - b_pos) (the overlap the seed's diagonal implies), mu = phi * ov, and
 *   keep[p] = 1  iff  res[p].score >= mu - sqrt(c * mu)     (IEEE fp64, round to nearest, no FMA)
 * -- a Chernoff lower bound of the score a true overlap of that length reaches (c = 2 ln(1/gamma)).
 * 0 < phi <= 1e6, 0 <= c <= 1e12.  offA / offB: n+1 int64 offsets of the pools (B may equal A). */
int xdrop_adaptive_filter_device(const int64_t* offA, int64_t nA, const int64_t* offB, int64_t nB,
                                 const xdrop_pair* pairs, const xdrop_result* res, int64_t n,
                                 double phi, double c, uint8_t* keep, int64_t* err_index, void* stream);
/* f4, the k-mer frequency band of ELBA's seeds (LOWER_KMER_FREQ, UPPER_KMER_FREQ):
 * freq[p] = the number of positions of the ASCII pool (seq, off: n_reads reads, len bases) whose k-mer
 * equals pair p's seed k-mer A[a_pos, a_pos + k) on either strand (canonical k-mers, A0 C1 G2 T3,
 * first base most significant; k-mers containing a non-ACGT base or crossing a read boundary do not
 * count), 1 <= k <= 31; keep[p] = lower <= freq[p] <= upper.  freq or keep may be NULL (not both). */
int xdrop_seed_kmer_freq_device(const char* seq, const int64_t* off, int64_t n_reads, int64_t len,
                                const xdrop_pair* pairs, int64_t n, int k, int lower, int upper,
                                int32_t* freq, uint8_t* keep, int64_t* err_index, void* stream);

/* ---- several seeds per candidate pair (reading Q26) ----
 * Seed-and-extend tools extend every seed a candidate pair shares and keep the best alignment
 * ("seed-and-extend").  A candidate is a maximal run of ADJACENT rows
 * of `pairs` with equal a_id and equal b_id (the strand bit XDROP_PAIR_RC included); non-adjacent
 * repeats are separate candidates.  best[i] = the index of the row of i's candidate with the
 * highest score, ties to the lowest index.
 *
 * Device form: pairs (n x 16 B), res (n x 20 B, e.g. the `out` of xdrop_align_batch_device) and
 * best (n x int64) are device pointers; work is enqueued on `stream` (NULL = the context's
 * stream) and the call returns after the stream has completed.  n = 0 is a no-op; n < 0 or a NULL
 * pointer with n > 0 -> XDROP_EINVAL. */
int xdrop_best_seed_device(xdrop_ctx* ctx, const xdrop_pair* pairs, const xdrop_result* res, int64_t n,
                           int64_t* best, void* stream);
/* Host form: xdrop_align_batch (out, cells_out as there) + the selection above into best
 * (n_pairs x int64, caller-owned host memory). */
int xdrop_align_multiseed(xdrop_ctx* ctx, const xdrop_seqs* A, const xdrop_seqs* B,
                          const xdrop_pair* pairs, int64_t n_pairs, const xdrop_params* p,
                          xdrop_result* out, int64_t* best, int64_t* cells_out);

/* Counters of the last call on this context: summed over every device and sub-batch turn of the
 * call (the *_ms fields: the maximum over devices and turns). */
typedef struct {
  int64_t items;          /* extensions (2 per pair) */
  int64_t escalated[4];   /* extensions that reached path level 1, 2, 3 (general); with
                             XDROP_FLAG_SEQAN_COMPAT in the general path only: [0] all,
                             [1] hulls wider than 256 cells (warp ring), [2] wider than 1,024
                             (8-warp ring), [3] wider than 8,192 (global-memory kernel) */
  int64_t cells;          /* total DP cells */
  float kernel_ms;        /* CUDA-event time of the alignment kernels (all levels) */
  float total_ms;         /* CUDA-event time of the whole device pipeline */
  float pack_ms;          /* ASCII -> 2-bit pack kernel */
  int64_t launches;       /* kernels launched by the last call */
  float level_ms[4];      /* CUDA-event time of each band level (0: lane/extension, 1-2: warp/extension, 3: general) */
  int64_t level_cells[4]; /* DP cells of the extensions completed at each level */
  int64_t level_items[4]; /* extensions completed at each level */
  int64_t long_items;     /* extensions run in the multi-lane "long" mode of level 0 */
  int64_t stolen;         /* lane-mode extensions checkpointed at the tail and resumed 4 lanes wide */
  int64_t band_kernel;    /* band kernel of the call: 0 32-bit merged, 1 packed tiered, 2 packed shared */
  int64_t cta_items;      /* extensions checkpointed into the S = 2048 thread-block level */
  int64_t cta4k_items;    /* extensions checkpointed into the S = 4096 thread-block level */
  int64_t endgame_stolen; /* shared kernel: T1/T2 extensions moved to the 32 x 8 shape at the tail */
  int64_t probe_overflows; /* per-batch kernel probe: sampled extensions that outgrew the T0 window */
} xdrop_stats;
int xdrop_last_stats(const xdrop_ctx* ctx, xdrop_stats* st);

/* ---- scheduler observability (§III; SPEC.md verify semantics) ---- */
typedef struct {
  int32_t rank, gpu, batch, sub;  /* logical rank, device slot, 1-based batch / sub-batch (0 for CELLS) */
  int64_t n_pairs;
  double t0_ms, t1_ms;            /* host wall clock relative to the call start */
} xdrop_trace_event;

typedef struct {
  int64_t handoffs;       /* token messages (Alg. 1 l.30 MPI_Send(True,[right])) */
  int64_t exchange_msgs;  /* batch-count exchange messages (Alg. 1 l.5-11) */
  int64_t turns;          /* sub-batch executions (events in the trace) */
  double span_ms;         /* first turn start to last turn end ("alignment time", Table I) */
  double busy_ms[16];     /* per device slot */
  int32_t max_concurrent; /* most turns running at one instant */
  int32_t n_events;       /* events recorded for xdrop_last_trace */
} xdrop_sched_stats;

int xdrop_last_sched_stats(const xdrop_ctx* ctx, xdrop_sched_stats* st);
/* Copy up to cap events of the last call's trace; returns the number available. */
int64_t xdrop_last_trace(const xdrop_ctx* ctx, xdrop_trace_event* buf, int64_t cap);

/* Host-only dry run of a policy (no GPU needed): every turn "runs" for
 * ns_per_unit * sum(w) nanoseconds of sleep.  gpu_of_pair (nullable, n
 * entries) receives the device slot that ran each pair.  Returns the number of
 * trace events (<= cap copied to trace) or a negative status. */
int64_t xdrop_sched_simulate(int m, int policy, int n_ranks, int batch_size, int subbatches,
                             const int64_t* w, int64_t n, double ns_per_unit, xdrop_sched_stats* st,
                             xdrop_trace_event* trace, int64_t cap, int32_t* gpu_of_pair);

/* Work-unit timeline of the last call's band kernel (only when the environment variable
 * XDROP_TIMELINE is set at xdrop_init): records of 3 x uint64 {type | warp << 8, start_ns,
 * end_ns}; type 0 lane batch, 1 long batch, 2 stolen batch, 3 lane-pair tier, 4 warp tier.
 * Returns the number of records (<= cap copied). */
int64_t xdrop_last_timeline(const xdrop_ctx* ctx, uint64_t* buf, int64_t cap);

/* Alg. 1 ring search over ranks 0..n-1: first rank r,
 * walking down (left) / up (right) from `rank` with wrap-around, with
 * batch <= counts[r]; -1 when the walk returns to `rank`. */
int xdrop_ring_left(int rank, int batch, const int* counts, int n);
int xdrop_ring_right(int rank, int batch, const int* counts, int n);
/* Reading Q21's token order over one ring of n members (member v has counts[v] batches, each of
 * turns_per_batch turns): the member index owning the turn after (batch b, iteration it) of member u,
 * with that turn's batch / iteration in *next_b / *next_it (nullable), or -1 if none; _prev: the member
 * owning the turn before, or -1.  The scheduler and the multi-process rank mode both use these. */
int xdrop_ring_turn_next(int u, int b, int it, const int* counts, int n, int turns_per_batch,
                         int* next_b, int* next_it);
int xdrop_ring_turn_prev(int u, int b, int it, const int* counts, int n, int turns_per_batch);

int xdrop_finalize(xdrop_ctx* ctx);
const char* xdrop_strerror(int status);
int64_t xdrop_last_error_index(const xdrop_ctx* ctx);

/* Measured single-pipe integer issue rates of CUDA device `device` (the roofline denominators;
 * SURVEY.md §8(d) P_int).  Six probes, each a loop of ONE SASS instruction kind in 8 independent
 * chains per thread (csrc/xdrop_peaks.cu; tests/test_capi_host.py checks the SASS):
 *   0 VIMNMX3.S16x2 (ALU pipe, two 16-bit lanes)  1 VIMNMX3 (ALU, 32-bit)  2 LOP3 (ALU)
 *   3 IADD3 (ALU)  4 IMAD (FMA pipe)  5 VIMNMX3.S16x2 and IMAD alternating (both pipes).
 * out[2p] = thread-instructions per second (CUDA events, best of 3), out[2p+1] = warp-instructions
 * per SM per SM clock (clock64).  n_out >= 12, else XDROP_EINVAL.  Allocates and frees its own
 * scratch; no context needed. */
int xdrop_alu_peaks(int device, double* out, int n_out);

#ifdef __cplusplus
}
#endif
#endif /* XDROP_H_ */
