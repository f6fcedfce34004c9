/*
 * oracle/xdrop_oracle.c -- CPU oracle for batched X-drop seed-and-extend.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this file's
 * library.  The product path (paper_2309_07270_b200/) never links, imports or
 * executes it, and this file shares no code, header, table or constant with
 * the CUDA path.
 *
 * What it computes (the reading is DESIGN.md "Readings" / SURVEY.md §8(c)):
 *
 *   The paper names the method but prints no recurrence.  Its anchors are
 *     - PAPER.md:73-74 (§II, BELLA): "seed-and-extend algorithm ... X-drop"
 *     - PAPER.md:81   (§II, diBELLA 2D): "an algorithm similar to X-Drop"
 *     - PAPER.md:85-89 (§II, LOGAN): X-drop is a DP; "each cell on the same
 *       anti-diagonal of the DP table is independent of the other and can be
 *       processed concurrently" (l.87)
 *     - PAPER.md:224 (§IV-A): "--ga (GPU-based x-drop alignment): 15"
 *     - PAPER.md:327 (§IV-E): "essentially Needleman-Wunsch or Smith-Waterman
 *       algorithm with X-Drop"
 *
 *   EXTEND(a[0:m], b[0:n]) walks anti-diagonals d = i + j in order.  The
 *   pruning threshold of anti-diagonal d is (best over anti-diagonals < d) - X,
 *   which is what makes the cells of one anti-diagonal independent (l.87).
 *   Written out step by step below, in the notation of DESIGN.md:
 *     H(0,0)=0, best=0, (i*,j*)=(0,0), L_0={0}, L_{-1}={}, cells=1
 *     for d = 1 .. m+n:
 *       stop if L_{d-1} and L_{d-2} are both empty
 *       hull  lo = max(0, d-n, min(min L_{d-1}, min L_{d-2}+1))
 *             hi = min(m, d,   max(max L_{d-1}+1, max L_{d-2}+1))
 *       cells += max(0, hi-lo+1)
 *       for i in [lo,hi], j=d-i: candidates from LIVE predecessors only
 *             H(i-1,j)+g   if i-1 in L_{d-1}
 *             H(i,j-1)+g   if i   in L_{d-1}
 *             H(i-1,j-1)+s(a[i-1],b[j-1])  if i-1 in L_{d-2}
 *         no candidate -> dead; else v=max, live iff v >= best - X
 *       if L_d nonempty and max_{L_d} H > best (strict):
 *             best = that max, i* = smallest live i attaining it, j* = d-i*
 *
 *   ALIGN(A,B,a_pos,b_pos,k): seed = sum_{t<k} s(A[a_pos+t],B[b_pos+t]);
 *     R = EXTEND(A[a_pos+k:], B[b_pos+k:]);
 *     L = EXTEND(reverse(A[:a_pos]), reverse(B[:b_pos]));
 *     score = L.best + seed + R.best; a_begin = a_pos - L.i*,
 *     b_begin = b_pos - L.j*, a_end = a_pos+k+R.i*, b_end = b_pos+k+R.j*,
 *     cells = L.cells + R.cells.
 *
 *   SeqAn/LOGAN-style mode (compat = 1, DESIGN.md readings
 *   Q28-Q30; the conventions are LOGAN's/SeqAn's, PAPER.md:85-89 names LOGAN
 *   but prints none of them):
 *     Q28  a pure-gap cell (i = 0 or j = 0, d >= 1) is live iff v > best - X
 *          (strict); interior cells keep v >= best - X
 *     Q29  the reported end is the "longest extension": the live cell of the
 *          LAST anti-diagonal with a live cell, largest H there, ties to the
 *          smallest i; the extension's score is H at that cell (Q30), not best
 *     best, the thresholds, the hull, the cell count and the termination are
 *     the same as above.
 *
 * Storage: the values of an anti-diagonal are kept in an array indexed by i
 * (three such arrays, for d, d-1, d-2).  A slot outside the recorded hull
 * [lo,hi] of its anti-diagonal is "not live"; that is the whole bookkeeping.
 * No blocking, no banding beyond the hull, no vectorisation.
 *
 * Threads: oracle_align_batch runs pairs on a plain pthread pool (pairs are
 * independent; each pair is computed by exactly the code above).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  int32_t best, istar, jstar;
  int64_t cells;
} oracle_ext;

typedef struct {
  int32_t score, a_begin, a_end, b_begin, b_end;
} oracle_result;

static int up(int c) { return (c >= 'a' && c <= 'z') ? c - 32 : c; }

/* Watson-Crick complement of a base (reading Q16: strand) */
static unsigned char complement(unsigned char c) {
  switch (up(c)) {
    case 'A': return 'T';
    case 'C': return 'G';
    case 'G': return 'C';
    case 'T': return 'A';
    default: return c;
  }
}

/* s(x,y) = M if x == y (case-insensitive), else mu  (reading Q10) */
static int sub_score(unsigned char x, unsigned char y, int M, int mu) {
  return up(x) == up(y) ? M : mu;
}

/* One anti-diagonal: values by i, live flags by i, and its hull/live extent. */
typedef struct {
  int32_t *H;
  unsigned char *live;
  int64_t lo, hi;       /* hull computed for this anti-diagonal (lo>hi: empty) */
  int64_t minL, maxL;   /* extent of the live set (minL > maxL: empty) */
} diag_t;

static int is_live(const diag_t *D, int64_t i) {
  if (i < D->lo || i > D->hi) return 0;
  return D->live[i];
}

int oracle_extend_mode(const unsigned char *a, int64_t m, const unsigned char *b, int64_t n,
                       int M, int mu, int g, int X, int compat, oracle_ext *out) {
  diag_t D[3];
  for (int t = 0; t < 3; ++t) {
    D[t].H = (int32_t *)calloc((size_t)(m + 1), sizeof(int32_t));
    D[t].live = (unsigned char *)calloc((size_t)(m + 1), 1);
    if (!D[t].H || !D[t].live) return -2;
  }
  /* d = 0: only the origin, live with H = 0. */
  diag_t *d0 = &D[0];
  d0->lo = 0; d0->hi = 0; d0->H[0] = 0; d0->live[0] = 1; d0->minL = 0; d0->maxL = 0;
  /* d = -1: empty. */
  diag_t *dm1 = &D[2];
  dm1->lo = 1; dm1->hi = 0; dm1->minL = 1; dm1->maxL = 0;

  int64_t best = 0, istar = 0, jstar = 0, cells = 1;
  int64_t lastv = 0, lasti = 0, lastd = 0;   /* compat: max cell of the last live anti-diagonal */
  for (int64_t d = 1; d <= m + n; ++d) {
    diag_t *P1 = &D[(d - 1) % 3];   /* anti-diagonal d-1 */
    diag_t *P2 = &D[(d + 1) % 3];   /* anti-diagonal d-2  ((d-2) mod 3) */
    diag_t *C = &D[d % 3];          /* anti-diagonal d (overwrites d-3) */
    int e1 = P1->minL > P1->maxL, e2 = P2->minL > P2->maxL;
    if (e1 && e2) break;            /* two consecutive empty anti-diagonals */

    int64_t lo, hi;
    if (!e1 && !e2) {
      lo = P1->minL < P2->minL + 1 ? P1->minL : P2->minL + 1;
      hi = P1->maxL + 1 > P2->maxL + 1 ? P1->maxL + 1 : P2->maxL + 1;
    } else if (!e1) {
      lo = P1->minL; hi = P1->maxL + 1;
    } else {
      lo = P2->minL + 1; hi = P2->maxL + 1;
    }
    if (lo < 0) lo = 0;
    if (lo < d - n) lo = d - n;
    if (hi > m) hi = m;
    if (hi > d) hi = d;
    if (hi >= lo) cells += hi - lo + 1;

    int64_t thr = best - X;  /* best over anti-diagonals < d */
    int64_t vstar = 0, istar_d = -1;
    C->minL = 1; C->maxL = 0;
    for (int64_t i = lo; i <= hi; ++i) {
      int64_t j = d - i;
      int have = 0;
      int64_t v = 0;
      if (i >= 1 && is_live(P1, i - 1)) {            /* H(i-1,j) + g */
        int64_t c = (int64_t)P1->H[i - 1] + g;
        if (!have || c > v) v = c;
        have = 1;
      }
      if (j >= 1 && is_live(P1, i)) {                /* H(i,j-1) + g */
        int64_t c = (int64_t)P1->H[i] + g;
        if (!have || c > v) v = c;
        have = 1;
      }
      if (i >= 1 && j >= 1 && is_live(P2, i - 1)) {  /* H(i-1,j-1) + s */
        int64_t c = (int64_t)P2->H[i - 1] + sub_score(a[i - 1], b[j - 1], M, mu);
        if (!have || c > v) v = c;
        have = 1;
      }
      int lv = have && v >= thr;
      if (compat && (i == 0 || j == 0)) lv = have && v > thr;   /* Q28: strict on the boundary */
      C->live[i] = (unsigned char)lv;
      C->H[i] = (int32_t)v;
      if (lv) {
        if (C->minL > C->maxL) { C->minL = i; C->maxL = i; }
        else { if (i < C->minL) C->minL = i; if (i > C->maxL) C->maxL = i; }
        if (istar_d < 0 || v > vstar) { vstar = v; istar_d = i; }  /* smallest i on ties */
      }
    }
    C->lo = lo; C->hi = hi;
    if (istar_d >= 0 && vstar > best) {
      best = vstar; istar = istar_d; jstar = d - istar_d;
    }
    if (istar_d >= 0) { lastv = vstar; lasti = istar_d; lastd = d; }   /* Q29 */
  }
  if (compat) { best = lastv; istar = lasti; jstar = lastd - lasti; }  /* Q29, Q30 */
  out->best = (int32_t)best; out->istar = (int32_t)istar; out->jstar = (int32_t)jstar;
  out->cells = cells;
  for (int t = 0; t < 3; ++t) { free(D[t].H); free(D[t].live); }
  return 0;
}

int oracle_extend(const unsigned char *a, int64_t m, const unsigned char *b, int64_t n,
                  int M, int mu, int g, int X, oracle_ext *out) {
  return oracle_extend_mode(a, m, b, n, M, mu, g, X, 0, out);
}

/* ALIGN for one pair; A, B are whole reads (ASCII).  compat: Q28-Q30 in both extensions. */
int oracle_align_mode(const unsigned char *A, int64_t lenA, const unsigned char *B, int64_t lenB,
                      int64_t a_pos, int64_t b_pos, int k, int M, int mu, int g, int X, int compat,
                      oracle_result *res, int64_t *cells, oracle_ext *left, oracle_ext *right) {
  if (a_pos < 0 || b_pos < 0 || a_pos + k > lenA || b_pos + k > lenB || k < 1) return -5;
  int64_t seed = 0;
  for (int t = 0; t < k; ++t) seed += sub_score(A[a_pos + t], B[b_pos + t], M, mu);

  oracle_ext R, L;
  int rc = oracle_extend_mode(A + a_pos + k, lenA - a_pos - k, B + b_pos + k, lenB - b_pos - k,
                              M, mu, g, X, compat, &R);
  if (rc) return rc;
  unsigned char *ra = (unsigned char *)malloc((size_t)a_pos + 1);
  unsigned char *rb = (unsigned char *)malloc((size_t)b_pos + 1);
  if (!ra || !rb) { free(ra); free(rb); return -2; }
  for (int64_t t = 0; t < a_pos; ++t) ra[t] = A[a_pos - 1 - t];
  for (int64_t t = 0; t < b_pos; ++t) rb[t] = B[b_pos - 1 - t];
  rc = oracle_extend_mode(ra, a_pos, rb, b_pos, M, mu, g, X, compat, &L);
  free(ra); free(rb);
  if (rc) return rc;

  res->score = (int32_t)(L.best + seed + R.best);
  res->a_begin = (int32_t)(a_pos - L.istar);
  res->b_begin = (int32_t)(b_pos - L.jstar);
  res->a_end = (int32_t)(a_pos + k + R.istar);
  res->b_end = (int32_t)(b_pos + k + R.jstar);
  if (cells) *cells = L.cells + R.cells;
  if (left) *left = L;
  if (right) *right = R;
  return 0;
}

int oracle_align(const unsigned char *A, int64_t lenA, const unsigned char *B, int64_t lenB,
                 int64_t a_pos, int64_t b_pos, int k, int M, int mu, int g, int X,
                 oracle_result *res, int64_t *cells, oracle_ext *left, oracle_ext *right) {
  return oracle_align_mode(A, lenA, B, lenB, a_pos, b_pos, k, M, mu, g, X, 0, res, cells, left, right);
}

/* ---- batch over a read pool, plain thread pool ------------------------- */
typedef struct {
  const unsigned char *seqA; const int64_t *offA;
  const unsigned char *seqB; const int64_t *offB;
  const int32_t *pairs;      /* 4 per pair: a_id, b_id, a_pos, b_pos */
  const int64_t *order;      /* optional processing order (NULL: 0..n-1) */
  int64_t n;
  int k, M, mu, g, X, compat;
  oracle_result *out; int64_t *cells;
  volatile int64_t next;
  volatile int err; volatile int64_t err_index;
  pthread_mutex_t mu_lock;
} batch_t;

static void *worker(void *arg) {
  batch_t *B = (batch_t *)arg;
  for (;;) {
    int64_t t = __atomic_fetch_add(&B->next, 1, __ATOMIC_RELAXED);
    if (t >= B->n) break;
    int64_t p = B->order ? B->order[t] : t;
    const int32_t *q = B->pairs + 4 * p;
    const unsigned char *A = B->seqA + B->offA[q[0]];
    int64_t lenA = B->offA[q[0] + 1] - B->offA[q[0]];
    const int32_t bid = q[1] & 0x7fffffff;               /* bit 31: use reverse(complement(B)) */
    const unsigned char *Bs = B->seqB + B->offB[bid];
    int64_t lenB = B->offB[bid + 1] - B->offB[bid];
    unsigned char *rcb = NULL;
    if (q[1] & (int32_t)0x80000000) {
      rcb = (unsigned char *)malloc((size_t)lenB + 1);
      for (int64_t u = 0; u < lenB; ++u) rcb[u] = complement(Bs[lenB - 1 - u]);
      Bs = rcb;
    }
    int64_t c = 0;
    int rc = oracle_align_mode(A, lenA, Bs, lenB, q[2], q[3], B->k, B->M, B->mu, B->g, B->X,
                               B->compat, &B->out[p], &c, NULL, NULL);
    free(rcb);
    if (B->cells) B->cells[p] = c;
    if (rc) {
      pthread_mutex_lock(&B->mu_lock);
      if (!B->err || p < B->err_index) { B->err = rc; B->err_index = p; }
      pthread_mutex_unlock(&B->mu_lock);
    }
  }
  return NULL;
}

/* Returns 0, or the first error code; *err_index receives the smallest failing pair. */
int oracle_align_batch_mode(const unsigned char *seqA, const int64_t *offA,
                            const unsigned char *seqB, const int64_t *offB,
                            const int32_t *pairs, const int64_t *order, int64_t n,
                            int k, int M, int mu, int g, int X, int compat,
                            oracle_result *out, int64_t *cells, int nthreads, int64_t *err_index) {
  batch_t B;
  memset(&B, 0, sizeof(B));
  B.seqA = seqA; B.offA = offA; B.seqB = seqB; B.offB = offB; B.pairs = pairs;
  B.order = order; B.n = n; B.k = k; B.M = M; B.mu = mu; B.g = g; B.X = X; B.compat = compat;
  B.out = out; B.cells = cells; B.next = 0; B.err = 0; B.err_index = -1;
  pthread_mutex_init(&B.mu_lock, NULL);
  if (nthreads < 1) nthreads = 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  for (int t = 0; t < nthreads; ++t) pthread_create(&th[t], NULL, worker, &B);
  for (int t = 0; t < nthreads; ++t) pthread_join(th[t], NULL);
  free(th);
  pthread_mutex_destroy(&B.mu_lock);
  if (err_index) *err_index = B.err_index;
  return B.err;
}

int oracle_align_batch(const unsigned char *seqA, const int64_t *offA,
                       const unsigned char *seqB, const int64_t *offB,
                       const int32_t *pairs, const int64_t *order, int64_t n,
                       int k, int M, int mu, int g, int X,
                       oracle_result *out, int64_t *cells, int nthreads, int64_t *err_index) {
  return oracle_align_batch_mode(seqA, offA, seqB, offB, pairs, order, n, k, M, mu, g, X, 0,
                                 out, cells, nthreads, err_index);
}
