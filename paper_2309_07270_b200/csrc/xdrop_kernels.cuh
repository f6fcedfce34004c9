// xdrop_kernels.cuh -- sm_100a kernels of the batched X-drop hot path.
//
// Operation (include/xdrop.h): EXTEND is the anti-diagonal
// X-drop DP; cells of one anti-diagonal are independent, the
// threshold of anti-diagonal d is (best over anti-diagonals < d) - X
// (PAPER.md:73-74, 224), the recurrence is NW with linear gaps.
//
// B200 design:
//  * Bases are 2-bit packed (16 per u32) once per call by pack_kernel; every
//    extension streams its two segments through 64-bit register windows
//    (chars are compared 32 at a time with one 64-bit XOR).
//  * Cells are held in DIAGONAL coordinates k = i - j: register R[q] holds
//    diagonal K0 + q, so a band that follows the alignment does not drift
//    through registers (only net indels move it).  Anti-diagonal d updates the
//    slots of parity d in place: R[q] <- max(R[q] + s, max(R[q-1], R[q+1]) + g).
//  * band_kernel<G, C>: G lanes per extension, C cells per lane per
//    anti-diagonal (window S = G*C cells = 2S diagonals).  G = 1 is the
//    lane-per-extension path (no cross-lane traffic at all: 32 extensions per
//    warp, integer-ALU bound); G = 32 is warp-per-extension for wide bands
//    (one shuffle + CREDUX reductions per anti-diagonal).
//  * An extension whose live band leaves its window is re-queued to the next
//    (wider) level; the result never depends on the window (cells outside the
//    hull are dead by construction), so escalation is exact.
//  * general_kernel is the unbounded fallback (anti-diagonals in global
//    scratch), used only beyond S = 1024.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace xk {

constexpr unsigned FULL = 0xffffffffu;
constexpr int NEGV = -(1 << 23);   // value of a dead cell (biased domain); NEGV * 128 fits int32
constexpr int BIAS = 1 << 21;      // stored value = H + BIAS; live values are > 0
constexpr int GUARD = 2048;        // bases of padding before/after the packed pool
constexpr int EMIN = 1 << 29;      // extent of an empty live set: [EMIN, EMAX]
constexpr int EMAX = -(1 << 29);
constexpr int NBUCKET = 16384;     // cost buckets for the length-sorted queue
constexpr int BUCKET_SHIFT = 4;

struct ExtOut {          // one extension result (32 B)
  int32_t best, istar, jstar, level;
  int64_t cells;
  int64_t pad;
};

struct PairDesc { int32_t a_id, b_id, a_pos, b_pos; };

struct Problem {
  const uint32_t* PA; const int64_t* offA; int64_t nA;
  const uint32_t* PB; const int64_t* offB; int64_t nB;
  int64_t lenA, lenB;  // bases in each pool (prep_kernel checks every read's offsets against them)
  const PairDesc* pairs; int64_t n_pairs;
  int M, mu, g, X, k;
  int keym;          // 128: argmax key multiplier, passed at run time so ptxas keeps it an IMAD (FMA pipe)
  int pkM, pkU;      // packed lane mode: 32 * (M - 2g), 32 * (mu - 2g)
  ExtOut* ext;
};

// ------------------------------------------------------------ packed streams
#ifdef XDROP_CHECKED
// Checked build (libxdrop_checked.so, tests only): every packed-pool word a kernel reads must lie
// inside one of the two pools the host registered for this call (g_chk_base / g_chk_words, set by
// dev_pipeline); anything else traps, so a guard-band or coordinate bug that leaves the pools fails
// the call with XDROP_ECUDA.  The check is against POOL bounds: a coordinate bug that reads another
// read of the same pool is caught by the oracle parity of the tests, not here.  The bounds are
// per-module device globals, so the checked build supports one context per device at a time.
__device__ const uint32_t* g_chk_base[2];
__device__ int64_t g_chk_words[2];
__device__ __forceinline__ void chk_word(const uint32_t* q) {
  for (int b = 0; b < 2; ++b)
    if (q >= g_chk_base[b] && q < g_chk_base[b] + g_chk_words[b]) return;
  __trap();
}
#define XDROP_CHK(q) chk_word(q)
// every extension result written must belong to an item of this call
#define XDROP_CHK_ITEM(P, it) do { if ((it) < 0 || (int64_t)(it) >= 2 * (P).n_pairs) __trap(); } while (0)
#else
#define XDROP_CHK(q) ((void)0)
#define XDROP_CHK_ITEM(P, it) ((void)0)
#endif
__device__ __forceinline__ uint32_t fwd16(const uint32_t* __restrict__ P, int64_t x) {
  const int64_t w = x >> 4;
  const int sh = (int)(x & 15) << 1;
  XDROP_CHK(P + w);
  XDROP_CHK(P + w + 1);
  const uint32_t lo = __ldg(P + w), hi = __ldg(P + w + 1);
  return __funnelshift_r(lo, hi, sh);
}
// swap the two bits of every 2-bit field (undoes __brev's per-field bit reversal)
__device__ __forceinline__ uint32_t swap_pairs(uint32_t y) {
  return ((y >> 1) & 0x55555555u) | ((y & 0x55555555u) << 1);
}
// chars t .. t+15 of a stream (start, dir) as true 2-bit codes; dir < 0 reads backwards
// (the two streams of an RC pair run in opposite directions, so codes must be exact)
__device__ __forceinline__ uint32_t load16(const uint32_t* __restrict__ P, int64_t start, int dir, int64_t t) {
  return dir > 0 ? fwd16(P, start + t) : swap_pairs(__brev(fwd16(P, start - t - 15)));
}
__device__ __forceinline__ uint64_t load32c(const uint32_t* __restrict__ P, int64_t start, int dir, int64_t t) {
  return (uint64_t)load16(P, start, dir, t) | ((uint64_t)load16(P, start, dir, t + 16) << 32);
}
// reverse the order of the 32 2-bit fields of x, keeping each field's bits
__device__ __forceinline__ uint64_t rev_fields(uint64_t x) {
  uint64_t y = __brevll(x);
  return ((y >> 1) & 0x5555555555555555ull) | ((y & 0x5555555555555555ull) << 1);
}
__device__ __forceinline__ int char_at(const uint32_t* __restrict__ P, int64_t start, int dir, int64_t t) {
  const int64_t x = start + (dir > 0 ? t : -t);
  XDROP_CHK(P + (x >> 4));
  return (int)((__ldg(P + (x >> 4)) >> ((int)(x & 15) << 1)) & 3u);
}

// b_id bit 31 (XDROP_PAIR_RC): the pair uses reverse(complement(B)); b_pos and the
// reported B coordinates are positions in revcomp(B) (reading Q16)
constexpr int32_t PAIR_RC = (int32_t)0x80000000;

struct Geom { int64_t sa, sb; int da, db; int m, n; uint64_t bmask; };

__device__ __forceinline__ Geom item_geom(const Problem& P, int item) {
  const int p = item >> 1;
  const PairDesc pd = P.pairs[p];
  const bool rc = (pd.b_id & PAIR_RC) != 0;
  const int bid = pd.b_id & 0x7fffffff;
  const int64_t a0 = P.offA[pd.a_id] + GUARD, b0 = P.offB[bid] + GUARD;
  const int lenA = (int)(P.offA[pd.a_id + 1] - P.offA[pd.a_id]);
  const int lenB = (int)(P.offB[bid + 1] - P.offB[bid]);
  Geom G;
  G.bmask = rc ? ~0ull : 0ull;       // complemented codes: XOR every field with 3
  if (item & 1) {   // right extension: A[a_pos+k:], B'[b_pos+k:]
    G.sa = a0 + pd.a_pos + P.k; G.da = 1; G.m = lenA - pd.a_pos - P.k;
    G.n = lenB - pd.b_pos - P.k;
    if (!rc) { G.sb = b0 + pd.b_pos + P.k; G.db = 1; }
    else { G.sb = b0 + lenB - 1 - pd.b_pos - P.k; G.db = -1; }   // B'[t] = comp(B[lenB-1-t])
  } else {          // left extension: reverse(A[:a_pos]), reverse(B'[:b_pos])
    G.sa = a0 + pd.a_pos - 1; G.da = -1; G.m = pd.a_pos;
    G.n = pd.b_pos;
    if (!rc) { G.sb = b0 + pd.b_pos - 1; G.db = -1; }
    else { G.sb = b0 + lenB - pd.b_pos; G.db = 1; }
  }
  return G;
}

// ---------------------------------------------------------- group reductions
template <int G> __device__ __forceinline__ int gmax(int v) {
  if constexpr (G == 1) return v;
  else if constexpr (G == 32) return __reduce_max_sync(FULL, v);
  else {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
    return v;
  }
}
template <int G> __device__ __forceinline__ int gmin(int v) {
  if constexpr (G == 1) return v;
  else if constexpr (G == 32) return __reduce_min_sync(FULL, v);
  else {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(FULL, v, o));
    return v;
  }
}

// ------------------------------------------------------------ band kernel
// argmax key = v * 128 + (127 - t): formed with IMAD (FMA pipe; P.keym), decoded with one shift
constexpr int KEYSH = 7;

// max over k[0..N) as a tree of 3-input VIMNMX3 (depth log3 N, not N/2)
template <int N>
__device__ __forceinline__ int tree_max3(int (&k)[N]) {
  if constexpr (N == 1) {
    return k[0];
  } else {
    constexpr int M = (N + 2) / 3;
    int t[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      if (3 * i + 2 < N) t[i] = __vimax3_s32(k[3 * i], k[3 * i + 1], k[3 * i + 2]);
      else if (3 * i + 1 < N) t[i] = max(k[3 * i], k[3 * i + 1]);
      else t[i] = k[3 * i];
    }
    return tree_max3<M>(t);
  }
}

// State of one extension as seen by one lane of its group.
template <int C> struct Band {
  int R[2 * C];                 // diagonals K0 + 2C*gl + r, r in [0, 2C)
  uint64_t Aw, Bw;              // a[ia0_l + t], b[jb0_l - t] for t = 0..31
  uint64_t bmask;               // ~0 when b is complemented (reverse-complement pairs)
  uint32_t An, An2, Bn, Bn2;    // stream reservoirs (next chars in stream order)
  int64_t sa, sb; int da, db;
  int m, n, K0, ia0, jb0;       // ia0/jb0: char index of global cell t = 0
  int best, istar, jstar;       // best is biased (H + BIAS)
  int dbase;                    // R holds W = H + BIAS + |g| (d - dbase)  (offset space, see band_diag)
  int thrW;                     // pruning threshold of the next anti-diagonal, in W space
  int minL1, maxL1, minL2, maxL2;   // live extents (in i) of d-1 and d-2
  long long cells;
  int item;
  bool active;
};

template <int G, int C>
__device__ __forceinline__ void band_reload(Band<C>& B, int gl, int rem, const Problem& P) {
  const int ia = B.ia0 + C * gl, jb = B.jb0 - C * gl;
  B.Aw = load32c(P.PA, B.sa, B.da, ia);
  B.An = load16(P.PA, B.sa, B.da, ia + 32);
  B.An2 = load16(P.PA, B.sa, B.da, ia + 32 + rem);
  B.Bw = rev_fields(load32c(P.PB, B.sb, B.db, jb - 31));
  B.Bn = load16(P.PB, B.sb, B.db, jb + 1);
  B.Bn2 = load16(P.PB, B.sb, B.db, jb + 1 + rem);
}

// One anti-diagonal d of parity PAR: the C cells of this lane, the group
// reductions (live extent, best and its smallest i), the hull count, and the
// stream advance to d+1.
//
// Offset space: registers hold W_d = H_d + BIAS - g (d - dbase).  Then
//   H_d(k) = max(H_{d-1}(k-1) + g, H_{d-1}(k+1) + g, H_{d-2}(k) + s)
// becomes
//   W_d(k) = max3(W_{d-1}(k-1), W_{d-1}(k+1), W_{d-2}(k) + s - 2g),
// one VIMNMX3 instead of VIMNMX + VIADDMNMX.  The threshold is carried in W
// space: thrW_{d+1} = max(thrW_d, vmaxW_d - X) - g, the only bookkeeping on
// the anti-diagonal-to-anti-diagonal critical path; the live mask and the
// argmax key are reduced as trees so a lone warp's step is issue-bound.
template <int G, int C, int PAR, bool CHECK>
__device__ __forceinline__ void band_diag(Band<C>& B, int gl, int d, int qlo, int qhi, const Problem& P) {
  constexpr int NR = 2 * C;
  constexpr int NCH = (C % 4 == 0 && C >= 8) ? 4 : 1;   // live-mask chains
  constexpr int CL = C / NCH;                            // cells per chain
  static_assert(C % NCH == 0, "chain split");
  const int thr = B.thrW;
  const int M = P.M - 2 * P.g, mu = P.mu - 2 * P.g;
  const int keym = P.keym;
  const uint64_t x = B.Aw ^ B.Bw ^ B.bmask;
  int nb = NEGV;
  if constexpr (G > 1) {
    if constexpr (PAR == 0) {
      nb = __shfl_up_sync(FULL, B.R[NR - 1], 1, G);
      if (gl == 0) nb = NEGV;
    } else {
      nb = __shfl_down_sync(FULL, B.R[0], 1, G);
      if (gl == G - 1) nb = NEGV;
    }
  }
  const int two = keym >> (KEYSH - 1);  // 2, opaque: keeps ch * two + s an IMAD
  int kacc[NCH];                        // running argmax keys, one per chain (max3 of pairs)
  int kpend[NCH];                       // a key waiting for its partner
  int ch[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) { ch[c] = 0; kacc[c] = NEGV * 128; kpend[c] = NEGV * 128; }
#pragma unroll
  for (int tt = 0; tt < C; ++tt) {
    const int r = 2 * tt + PAR;
    const int lft = (r == 0) ? nb : B.R[r == 0 ? 0 : r - 1];
    const int rgt = (r == NR - 1) ? nb : B.R[r == NR - 1 ? 0 : r + 1];
    const bool mis = ((x >> (2 * tt)) & 3ull) != 0ull;
    const int dg = B.R[r] + (mis ? mu : M);
    int v = __vimax3_s32(lft, rgt, dg);
    // prune on the FMA pipe: s = -1 if v < thr (dead) else 0; a dead value is
    // forced negative (v | 0xFF800000), below every threshold (> 2^20) for good
    int sd = __mulhi(v - thr, 2);
    if constexpr (CHECK) {
      const int q = 2 * C * gl + r;
      sd = (q >= qlo && q <= qhi) ? sd : -1;
    }
    v = v | (sd & (int)0xFF800000);
    B.R[r] = v;
    const int key = v * keym + (127 - tt);
    if ((tt % CL) % 2 == 0) kpend[tt / CL] = key;
    else kacc[tt / CL] = __vimax3_s32(kacc[tt / CL], kpend[tt / CL], key);
    ch[tt / CL] = ch[tt / CL] * two + sd;  // accumulates -(dead bits)
  }
  unsigned dbits = 0;                   // cell tt at bit C-1-tt
#pragma unroll
  for (int c = 0; c < NCH; ++c) dbits = (dbits << CL) + (unsigned)(-ch[c]);
  int mk;
  if constexpr (CL % 2 == 1) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) kacc[c] = max(kacc[c], kpend[c]);
  }
  if constexpr (NCH == 4) mk = max(__vimax3_s32(kacc[0], kacc[1], kacc[2]), kacc[3]);
  else mk = kacc[0];
  // ---- critical path: next threshold
  const int vl = mk >> KEYSH;           // best W value of this lane (NEGV if none live)
  int gv, gt;
  if constexpr (G == 1) {
    gv = vl; gt = 127 - (mk & 127);
  } else {
    gv = gmax<G>(vl);
    const unsigned ball = __ballot_sync(FULL, vl == gv);
    const int grp = (threadIdx.x & 31) / G;
    const unsigned gb = (G == 32) ? ball : ((ball >> (grp * G)) & ((1u << G) - 1u));
    const int first = __ffs(gb) - 1;
    gt = __shfl_sync(FULL, C * gl + 127 - (mk & 127), first, G);
  }
  B.thrW = max(thr, gv - P.X) - P.g;
  // ---- off the critical path: live extent, best / argmax, hull count
  const unsigned lb = ~dbits & (C == 32 ? 0xffffffffu : ((1u << C) - 1u));
  int tmin = (__clz(lb) - (32 - C)) + C * gl;
  int tmax = (C - __ffs(lb)) + C * gl;
  tmin = lb ? tmin : EMIN;
  tmax = lb ? tmax : EMAX;
  tmin = gmin<G>(tmin);
  tmax = gmax<G>(tmax);
  const int ibase = (d + B.K0 + PAR) >> 1;
  const int woff = -P.g * (d - B.dbase);
  const bool up = B.active && (gv - woff > B.best);
  B.best = up ? gv - woff : B.best;
  B.istar = up ? ibase + gt : B.istar;
  B.jstar = up ? d - ibase - gt : B.jstar;
  // hull of anti-diagonal d (from the live sets of d-1 and d-2)
  const int lo = max(max(0, d - B.n), min(B.minL1, B.minL2 + 1));
  const int hi = min(min(B.m, d), max(B.maxL1, B.maxL2) + 1);
  B.cells += (B.active && hi >= lo) ? (long long)(hi - lo + 1) : 0ll;
  B.minL2 = B.minL1; B.maxL2 = B.maxL1;
  B.minL1 = (tmin == EMIN) ? EMIN : ibase + tmin;
  B.maxL1 = (tmax == EMAX) ? EMAX : ibase + tmax;
  // stream advance for anti-diagonal d+1
  if constexpr (PAR == 0) {       // even -> odd: a advances (ia0 += 1)
    B.Aw = (B.Aw >> 2) | ((uint64_t)(B.An & 3u) << 62);
    B.An >>= 2;
    B.ia0 += 1;
  } else {                        // odd -> even: b advances (jb0 += 1)
    B.Bw = (B.Bw << 2) | (uint64_t)(B.Bn & 3u);
    B.Bn >>= 2;
    B.jb0 += 1;
  }
}

// lanes of this lane's group (shifts are taken by one group while the other
// groups of the warp may not take them)
template <int G> __device__ __forceinline__ unsigned group_mask() {
  if constexpr (G == 32) return FULL;
  else return ((1u << G) - 1u) << (((threadIdx.x & 31) / G) * G);
}

template <int G, int C>
__device__ __forceinline__ void band_shift(Band<C>& B, int gl, int dir) {
  constexpr int NR = 2 * C;
  const unsigned gm = group_mask<G>();
  if (dir > 0) {            // K0 += 2: R[r] <- R[r+2]
    int n0 = NEGV, n1 = NEGV;
    if constexpr (G > 1) {
      n0 = __shfl_down_sync(gm, B.R[0], 1, G);
      n1 = __shfl_down_sync(gm, B.R[1], 1, G);
      if (gl == G - 1) { n0 = NEGV; n1 = NEGV; }
    }
#pragma unroll
    for (int r = 0; r < NR - 2; ++r) B.R[r] = B.R[r + 2];
    B.R[NR - 2] = n0; B.R[NR - 1] = n1;
  } else {                  // K0 -= 2: R[r] <- R[r-2]
    int n0 = NEGV, n1 = NEGV;
    if constexpr (G > 1) {
      n0 = __shfl_up_sync(gm, B.R[NR - 2], 1, G);
      n1 = __shfl_up_sync(gm, B.R[NR - 1], 1, G);
      if (gl == 0) { n0 = NEGV; n1 = NEGV; }
    }
#pragma unroll
    for (int r = NR - 1; r >= 2; --r) B.R[r] = B.R[r - 2];
    B.R[0] = n0; B.R[1] = n1;
  }
}

// lane mode: shift the register window by 2*K diagonals (R[r] <- R[r + 2K])
template <int C, int K>
__device__ __forceinline__ void shift_regs(int (&R)[2 * C]) {
  if constexpr (K > 0) {
#pragma unroll
    for (int r = 0; r < 2 * C; ++r) R[r] = (r + 2 * K < 2 * C) ? R[(r + 2 * K) % (2 * C)] : NEGV;
  } else {
#pragma unroll
    for (int r = 2 * C - 1; r >= 0; --r) R[r] = (r + 2 * K >= 0) ? R[(r + 2 * K + 2 * C) % (2 * C)] : NEGV;
  }
}
template <int C>
__device__ __forceinline__ void band_shift_n(Band<C>& B, int s) {
  switch (s) {
    case 1: shift_regs<C, 1>(B.R); break;   case -1: shift_regs<C, -1>(B.R); break;
    case 2: shift_regs<C, 2>(B.R); break;   case -2: shift_regs<C, -2>(B.R); break;
    case 3: shift_regs<C, 3>(B.R); break;   case -3: shift_regs<C, -3>(B.R); break;
    case 4: shift_regs<C, 4>(B.R); break;   case -4: shift_regs<C, -4>(B.R); break;
    case 5: shift_regs<C, 5>(B.R); break;   case -5: shift_regs<C, -5>(B.R); break;
    case 6: shift_regs<C, 6>(B.R); break;   case -6: shift_regs<C, -6>(B.R); break;
    case 7: shift_regs<C, 7>(B.R); break;   case -7: shift_regs<C, -7>(B.R); break;
    case 8: shift_regs<C, 8>(B.R); break;   case -8: shift_regs<C, -8>(B.R); break;
    default: break;
  }
}

// ---------------------------------------------------------------- escalation
// An extension whose live band outgrows its window is CHECKPOINTED, not
// restarted: the group writes a record (scalars + the two live anti-diagonals
// of its window) to a pool and publishes the record slot on a queue; the next
// tier resumes it at the same anti-diagonal in a wider window.  The record
// holds everything the recurrence reads, so resumption is exact.
__device__ __forceinline__ int ld_volatile(const int* p) { return *((const volatile int*)p); }

struct Esc {
  int* pool;        // records of rec_ints ints (HDR header ints + 2*S_src cells)
  int rec_ints;
  int cap;          // records available in the pool (0: always fall back)
  int* pool_tail;   // records allocated
  int* q;           // published record slots (pre-set to -1)
  int* q_tail;
  int* fb_items;    // pool full: the item restarts in the unbounded kernel
  int* fb_tail;
};
constexpr int HDR = 32;
constexpr int REC_T = 17;          // header int: publication time (globaltimer >> 10, ~us) of the record
constexpr int REC_LAST = 18;       // header ints 18-20: compat mode's last-anti-diagonal maximum (packed tiers)
__device__ __forceinline__ int rec_stamp() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return (int)(unsigned)(t >> 10);
}

// queue push: slot = atomicAdd(tail); store; fence (consumers may be running)
__device__ __forceinline__ void push_item(int* items, int* tail, int item) {
  const int pos = atomicAdd(tail, 1);
  *((volatile int*)items + pos) = item;
  __threadfence();
}

template <int G, int C>
__device__ __forceinline__ void band_save(const Band<C>& B, int gl, int d, const Esc& e) {
  constexpr int S = G * C;
  const unsigned gm = group_mask<G>();
  int slot = 0;
  if (gl == 0) slot = atomicAdd(e.pool_tail, 1);
  if constexpr (G > 1) slot = __shfl_sync(gm, slot, 0, G);
  if (slot >= e.cap) {
    if (gl == 0) push_item(e.fb_items, e.fb_tail, B.item);
    return;
  }
  int* rec = e.pool + (size_t)slot * e.rec_ints;
  if (gl == 0) {
    rec[0] = B.item; rec[1] = d; rec[2] = B.K0; rec[3] = B.dbase; rec[4] = B.thrW; rec[5] = B.best;
    rec[6] = B.istar; rec[7] = B.jstar; rec[8] = B.minL1; rec[9] = B.maxL1; rec[10] = B.minL2;
    rec[11] = B.maxL2; rec[12] = B.ia0; rec[13] = B.jb0; rec[14] = S;
    rec[15] = (int)(B.cells & 0xffffffffll); rec[16] = (int)(B.cells >> 32);
    rec[REC_T] = rec_stamp();
  }
#pragma unroll
  for (int r = 0; r < 2 * C; ++r) rec[HDR + 2 * C * gl + r] = B.R[r];
  __threadfence();
  if constexpr (G > 1) __syncwarp(gm);
  if (gl == 0) push_item(e.q, e.q_tail, slot);
}

// End of a block of two anti-diagonals (d-1 odd, d even): termination,
// reservoir refill, window management.  The window is checked every two
// anti-diagonals, so it keeps the live cells of d-1 and d inside [2, 2S-3]
// (the band grows by at most one diagonal per side per anti-diagonal).
template <int G, int C>
__device__ __forceinline__ void band_block_end(Band<C>& B, int gl, int d, int& rem, const Problem& P, int level,
                                               const Esc& esc) {
  constexpr int S = G * C;
  if (d - B.dbase >= 1024) {      // keep the offset space bounded (|g| * 1024 <= 2^16)
    const int woff = -P.g * (d - B.dbase);
#pragma unroll
    for (int r = 0; r < 2 * C; ++r) B.R[r] -= woff;
    B.thrW -= woff;
    B.dbase = d;
  }
  if (--rem == 0) {
    rem = 16;
    B.An = B.An2; B.Bn = B.Bn2;
    if (B.active) {
      B.An2 = load16(P.PA, B.sa, B.da, B.ia0 + C * gl + 48);
      B.Bn2 = load16(P.PB, B.sb, B.db, B.jb0 - C * gl + 17);
    }
  }
  if (!B.active) return;
  const bool e0 = (B.minL1 == EMIN), e1 = (B.minL2 == EMIN);
  if ((e0 && e1) || d >= B.m + B.n) {
    if (gl == 0) {
      ExtOut o; o.best = B.best - BIAS; o.istar = B.istar; o.jstar = B.jstar; o.level = level;
      o.cells = B.cells; o.pad = 0;
      XDROP_CHK_ITEM(P, B.item);
      P.ext[B.item] = o;
    }
    B.active = false;
    return;
  }
  int qmn = 1 << 30, qmx = -(1 << 30);
  if (!e0) { qmn = 2 * B.minL1 - d - B.K0; qmx = 2 * B.maxL1 - d - B.K0; }
  if (!e1) { qmn = min(qmn, 2 * B.minL2 - (d - 1) - B.K0); qmx = max(qmx, 2 * B.maxL2 - (d - 1) - B.K0); }
  if constexpr (G == 1) {
    // lane mode: when the live band nears an edge, re-centre it in one move
    // (shift by 2s diagonals, |s| <= 8) so shifts stay rare.
    if (qmx >= 2 * S - 2 || qmn <= 1) {
      const int s_lo = (qmx - 2 * S + 4) >> 1;            // ceil((qmx - 2S + 3) / 2)
      const int s_hi = (qmn - 2) >> 1;                     // floor((qmn - 2) / 2)
      if (s_lo > s_hi) {
        band_save<G, C>(B, gl, d, esc);
        B.active = false;
        return;
      }
      int sh = (((qmn + qmx) >> 1) - S) >> 1;              // centre of the band -> centre of the window
      sh = min(max(sh, s_lo), s_hi);
      sh = min(max(sh, -8), 8);
      if (sh == 0) sh = s_lo > 0 ? s_lo : s_hi;
      band_shift_n<C>(B, sh);
      B.K0 += 2 * sh; B.ia0 += sh; B.jb0 -= sh;
      band_reload<G, C>(B, gl, rem, P);
    }
  } else {
    int dir = 0;
    bool ovf = false;
    if (qmx >= 2 * S - 2) { if (qmn >= 4) dir = 1; else ovf = true; }
    else if (qmn <= 1) { if (qmx <= 2 * S - 5) dir = -1; else ovf = true; }
    if (ovf) {
      band_save<G, C>(B, gl, d, esc);
      B.active = false;
      return;
    }
    if (dir != 0) {
      band_shift<G, C>(B, gl, dir);
      B.K0 += 2 * dir; B.ia0 += dir; B.jb0 -= dir;
      band_reload<G, C>(B, gl, rem, P);
    }
  }
}

// anti-diagonal loop from each group's own B.d (resumed groups of a warp may sit
// at different anti-diagonals; all are even at block boundaries)
// Tail stealing: once `thresh` warps sit idle, a lane-mode warp checkpoints every extension
// that still has >= min_rem anti-diagonals to go, so idle warps resume it with 4 lanes.
struct Steal { const int* idle; int thresh; int min_rem; Esc es; };

template <int G, int C>
__device__ __forceinline__ void band_loop(Band<C>& B, int gl, int& d, int& rem, const Problem& P, int level,
                                          const Esc& esc, const Steal* st = nullptr) {
  constexpr int S = G * C;
  int blk = 0;
  while (__any_sync(FULL, B.active)) {
    if (st != nullptr && ((++blk & 31) == 0)) {
      int go = 0;
      if ((threadIdx.x & 31) == 0) go = ld_volatile(st->idle) >= st->thresh;
      go = __shfl_sync(FULL, go, 0);
      if (go && B.active) {
        const int ic = (B.minL1 == EMIN) ? B.minL2 : (B.minL1 >> 1) + (B.maxL1 >> 1);
        const int left = 2 * min(B.m - ic, B.n - (d - ic));   // anti-diagonals still ahead (estimate)
        if (left >= st->min_rem) {
          band_save<G, C>(B, gl, d, st->es);
          B.active = false;
        }
      }
      if (!__any_sync(FULL, B.active)) break;
    }
    // boundary (i > m or j > n) enters the window?  checked for the later step
    const int d2 = d + 2;
    const bool need = B.active && (d2 - B.K0 - 2 * B.n > 0 || 2 * B.m - d2 - B.K0 < 2 * S - 1);
    if (__any_sync(FULL, need)) {
      band_diag<G, C, 1, true>(B, gl, d + 1, d + 1 - B.K0 - 2 * B.n, 2 * B.m - (d + 1) - B.K0, P);
      band_diag<G, C, 0, true>(B, gl, d2, d2 - B.K0 - 2 * B.n, 2 * B.m - d2 - B.K0, P);
    } else {
      band_diag<G, C, 1, false>(B, gl, d + 1, 0, 0, P);
      band_diag<G, C, 0, false>(B, gl, d2, 0, 0, P);
    }
    d = d2;
    band_block_end<G, C>(B, gl, d, rem, P, level, esc);
  }
}

template <int C>
__device__ __forceinline__ void band_idle(Band<C>& B) {
  B.active = false; B.item = 0;
  B.sa = GUARD; B.sb = GUARD; B.da = 1; B.db = 1; B.m = 0; B.n = 0; B.bmask = 0;
}

// Run one extension from its seed per group of G lanes (item < 0: idle group).  Warp-collective.
template <int G, int C>
__device__ __forceinline__ void band_run(const Problem& P, int item, int level, const Esc& esc,
                                         const Steal* st = nullptr) {
  constexpr int S = G * C;
  const int gl = (threadIdx.x & 31) % G;
  Band<C> B;
  if (item >= 0) {
    B.active = true; B.item = item;
    const Geom gm = item_geom(P, B.item);
    B.sa = gm.sa; B.sb = gm.sb; B.da = gm.da; B.db = gm.db; B.m = gm.m; B.n = gm.n; B.bmask = gm.bmask;
  } else {
    band_idle(B);
  }
  B.K0 = -S;
  B.ia0 = -S / 2;          // window chars for d = 1 (odd): ia0 = (1+K0+1)/2 - 1
  B.jb0 = S / 2 - 1;       //                               jb0 = (1-K0-1)/2 - 1
#pragma unroll
  for (int r = 0; r < 2 * C; ++r) B.R[r] = NEGV;
  // origin: d = 0, k = 0 -> q = S -> lane G/2 (r = 0), or lane 0 r = C when G = 1
  if constexpr (G == 1) B.R[C] = BIAS;
  else if (gl == G / 2) B.R[0] = BIAS;
  B.best = BIAS; B.istar = 0; B.jstar = 0; B.cells = 1; B.dbase = 0;
  B.thrW = BIAS - P.X - P.g;     // threshold of anti-diagonal 1 in W space (woff_1 = -g)
  B.minL1 = 0; B.maxL1 = 0; B.minL2 = EMIN; B.maxL2 = EMAX;
  int rem = 16;
  band_reload<G, C>(B, gl, rem, P);
  if (B.active && B.m + B.n == 0) {
    if (gl == 0) {
      ExtOut o; o.best = 0; o.istar = 0; o.jstar = 0; o.level = level; o.cells = 1; o.pad = 0;
      XDROP_CHK_ITEM(P, B.item);
      P.ext[B.item] = o;
    }
    B.active = false;
  }
  int d = 0;
  band_loop<G, C>(B, gl, d, rem, P, level, esc, st);
}

// Resume one checkpointed extension per group (rec == nullptr: idle group) in a
// window of S = G*C >= the record's; the old window lands in the middle.
template <int G, int C>
__device__ __forceinline__ void band_resume(const Problem& P, const int* rec, int level, const Esc& esc) {
  constexpr int S = G * C;
  const int gl = (threadIdx.x & 31) % G;
  Band<C> B;
  int d = 0;
  if (rec) {
    B.active = true; B.item = rec[0];
    const Geom gm = item_geom(P, B.item);
    B.sa = gm.sa; B.sb = gm.sb; B.da = gm.da; B.db = gm.db; B.m = gm.m; B.n = gm.n; B.bmask = gm.bmask;
    d = rec[1];
    const int s_src = rec[14];
    const int sh = S - s_src;                      // K0' = K0 - sh (sh >= 0, even)
    B.K0 = rec[2] - sh; B.dbase = rec[3]; B.thrW = rec[4]; B.best = rec[5];
    B.istar = rec[6]; B.jstar = rec[7]; B.minL1 = rec[8]; B.maxL1 = rec[9]; B.minL2 = rec[10];
    B.maxL2 = rec[11]; B.ia0 = rec[12] - sh / 2; B.jb0 = rec[13] + sh / 2;
    B.cells = (long long)(unsigned)rec[15] | ((long long)rec[16] << 32);
#pragma unroll
    for (int r = 0; r < 2 * C; ++r) {
      const int q = 2 * C * gl + r - sh;
      B.R[r] = (q >= 0 && q < 2 * s_src) ? rec[HDR + q] : NEGV;
    }
  } else {
    band_idle(B);
    B.K0 = -S; B.ia0 = -S / 2; B.jb0 = S / 2 - 1; B.dbase = 0; B.thrW = 0; B.best = 0;
    B.istar = 0; B.jstar = 0; B.cells = 0; B.minL1 = EMIN; B.maxL1 = EMAX; B.minL2 = EMIN; B.maxL2 = EMAX;
#pragma unroll
    for (int r = 0; r < 2 * C; ++r) B.R[r] = NEGV;
  }
  int rem = 16;
  band_reload<G, C>(B, gl, rem, P);
  band_loop<G, C>(B, gl, d, rem, P, level, esc);
}

// Standalone kernel, fresh extensions: persistent warps, 32/G per warp batch.
template <int G, int C>
__global__ void __launch_bounds__(128)
band_kernel(Problem P, const int* __restrict__ items, const int* __restrict__ n_items_ptr, int* queue_head,
            Esc esc, int level) {
  constexpr int IPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int n_items = *n_items_ptr;
  for (;;) {
    int base = 0;
    if (lane == 0) base = atomicAdd(queue_head, IPW);
    base = __shfl_sync(FULL, base, 0);
    if (base >= n_items) break;
    const int slot = base + grp;
    band_run<G, C>(P, slot < n_items ? items[slot] : -1, level, esc);
  }
}

// Standalone kernel resuming checkpointed extensions (records of `src`).
template <int G, int C>
__global__ void __launch_bounds__(128)
band_resume_kernel(Problem P, Esc src, int* queue_head, Esc esc, int level) {
  constexpr int IPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int n = *src.q_tail;
  for (;;) {
    int base = 0;
    if (lane == 0) base = atomicAdd(queue_head, IPW);
    base = __shfl_sync(FULL, base, 0);
    if (base >= n) break;
    const int slot = base + grp;
    const int* rec = slot < n ? src.pool + (size_t)src.q[slot] * src.rec_ints : nullptr;
    band_resume<G, C>(P, rec, level, esc);
  }
}

// claim up to `want` published entries of a queue (lane 0 only); returns the
// first claimed index and sets k (0: nothing claimed)
__device__ __forceinline__ int claim(int* head, const int* tail, int want, bool partial, int& k) {
  k = 0;
  int h = ld_volatile(head);
  int t = ld_volatile(tail);
  bool fresh = true;                    // t was read after h
  for (;;) {
    // the tail only grows, so a stale t under-estimates what is available: a failed CAS retries
    // with it (one L2 round trip per attempt under contention, not two); re-read it only when it
    // seems to leave nothing to claim
    int avail = t - h;
    if (avail <= 0 || (avail < want && !partial)) {
      if (fresh) return 0;
      t = ld_volatile(tail);
      fresh = true;
      avail = t - h;
      if (avail <= 0 || (avail < want && !partial)) return 0;
    }
    const int kk = min(want, avail);
    const int old = atomicCAS(head, h, h + kk);
    if (old == h) { k = kk; return h; }
    h = old;
    fresh = false;
  }
}
// claim for a batch consumer: up to `want` entries, fewer only when `partial` or the oldest unclaimed
// record has waited >= age_us (lane 0 only)
__device__ __forceinline__ int claim_batch(int* head, const Esc& e, int want, bool partial, int age_us, int& k) {
  k = 0;
  const int h = ld_volatile(head), t = ld_volatile(e.q_tail);
  if (t <= h) return 0;
  if (!partial && t - h < want) {
    const int slot = ld_volatile(e.q + h);
    if (slot < 0) return 0;
    const int st = ld_volatile(e.pool + (size_t)slot * e.rec_ints + REC_T);
    if ((int)((unsigned)rec_stamp() - (unsigned)st) < age_us) return 0;
  }
  return claim(head, e.q_tail, want, true, k);
}
__device__ __forceinline__ int wait_entry(const int* q, int i) {
  int v;
  do { v = ld_volatile(q + i); } while (v < 0);
  return v;
}
// the one claimed entry h of a warp-wide consumer (lane 0 waits, all lanes get it)
__device__ __forceinline__ int wait_entry_w(const int* q, int h, int lane) {
  int slot = -1;
  if (lane == 0) slot = wait_entry(q, h);
  return __shfl_sync(FULL, slot, 0);
}

#include "xdrop_pk16.cuh"
#include "xdrop_pkwide.cuh"

// Standalone kernel resuming checkpointed extensions in the packed 16-bit mode (X + M <= 510).
#ifndef XDROP_PKR_MINBLOCKS
#define XDROP_PKR_MINBLOCKS 3
#endif
template <int G, int C, bool CP = false>
__global__ void __launch_bounds__(128, XDROP_PKR_MINBLOCKS)
pk_resume_kernel(Problem P, Esc src, int* queue_head, Esc esc, int level) {
  constexpr int IPW = 32 / G;
  const int lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int n = *src.q_tail;
  for (;;) {
    int base = 0;
    if (lane == 0) base = atomicAdd(queue_head, IPW);
    base = __shfl_sync(FULL, base, 0);
    if (base >= n) break;
    const int slot = base + grp;
    const int* rec = slot < n ? src.pool + (size_t)src.q[slot] * src.rec_ints : nullptr;
    pk_resume<G, C, CP>(P, rec, level, esc);
  }
}

// Counters of the merged kernel (ints): see xdrop_capi.cu
struct MergedCtr { int* head0; int* done0; int* head_long; int* n_long; int* q1_head; int* done1; int* q2_head;
                   int* idle; int* qs_head; int* dones;
                   unsigned long long* tl; int* tl_n; int tl_cap;     // optional work-unit timeline
                   int endgame;                                       // T0 items left -> 4-lane dispatch
                   int* smcnt; int t0_per_sm; int idle_ns;
                   int age_us;                        // batch claims of T1/T2 go partial after this wait
                   const int* probe_cnt; int probe_thr; };  // packed kernels: the shared one runs iff
                                                             // *probe_cnt >= probe_thr, the tiered one iff not

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// timeline record: [type | warp << 8, start_ns, end_ns]
__device__ __forceinline__ void tl_rec(const MergedCtr& c, int type, unsigned long long t0) {
  if (c.tl == nullptr || (threadIdx.x & 31) != 0) return;
  const int i = atomicAdd(c.tl_n, 1);
  if (i >= c.tl_cap) return;
  const unsigned long long w = (blockIdx.x * (blockDim.x >> 5)) + (threadIdx.x >> 5);
  c.tl[3 * i] = (unsigned long long)type | (w << 8); c.tl[3 * i + 1] = t0; c.tl[3 * i + 2] = gtimer();
}

// Tiers 0-2 in ONE persistent kernel (32-bit cells; the packed mode is pk_merged_kernel below).
//  T0  fresh extensions: the longest (the first n_long of the length-sorted
//      queue; n_long is set on the device from the batch's total work per
//      resident lane, see scan_kernel) run GL lanes per extension (CL cells,
//      same 32-cell window) so their anti-diagonal chain -- the launch's
//      critical path -- is GL times shorter per step; the rest run one lane
//      per extension (C0 = 32 cells).
//  T1  checkpointed T0 extensions resume 8 lanes x 8 cells per extension (S = 64),
//      claimed as soon as they appear.
//  T2  checkpointed T1 extensions resume one warp per extension (S = 256).
//  T2 overflows are checkpointed for the separate S = 1024 launch.
// Escalated work takes priority, so it runs while T0 drains, not as a tail.
#ifndef XDROP_MERGED_MINBLOCKS
#define XDROP_MERGED_MINBLOCKS 3
#endif
// packed escalation tiers (pk_merged_kernel): T1 = XDROP_T1_G lanes x 32 cells, T2 = XDROP_T2_G x 32
#ifndef XDROP_T1_G
#define XDROP_T1_G 4
#endif
#ifndef XDROP_T2_G
#define XDROP_T2_G 8
#endif
// resident 4-warp blocks per SM requested from ptxas: the tiered kernel's loops fit 128 registers
// (4 blocks, 16 warps per SM; measured faster than 3 on the throughput-bound E. coli batch), the shared
// kernel's single run-time-G loop needs its 168 (4 blocks slowed its S = 1024 tier: X-sweep X = 50
// 51.6 -> 74.2 ms)
#ifndef XDROP_PKT_MINBLOCKS
#define XDROP_PKT_MINBLOCKS 4
#endif
#ifndef XDROP_PKM_MINBLOCKS
#define XDROP_PKM_MINBLOCKS 3
#endif
#ifndef XDROP_PK_C
#define XDROP_PK_C 32          // cells per lane of the tiered kernel's packed lane mode (T0)
#endif

// the first t0_per_sm resident blocks of each SM take fresh (T0) extensions; the others serve
// only escalated / stolen work
__device__ __forceinline__ bool t0_block(const MergedCtr& c) {
  __shared__ int s_t0;
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    s_t0 = (c.t0_per_sm <= 0) || atomicAdd(c.smcnt + (smid & 1023), 1) < c.t0_per_sm;
  }
  __syncthreads();
  return s_t0 != 0;
}

// no work visible: finished once T0 is done (=> T1's queue is final), T1 is done (=> T2's queue is
// final) and T2's queue is drained (stolen records come only from T0 batches, before their done0 add)
__device__ __forceinline__ bool merged_finished(const MergedCtr& c, int n_items, const Esc& e1, const Esc& e2,
                                                const Steal& st) {
  if (ld_volatile(c.done0) < n_items) return false;
  const int ts = ld_volatile(st.es.q_tail);
  if (ld_volatile(c.dones) < ts || ld_volatile(c.qs_head) < ts) return false;
  const int t1 = ld_volatile(e1.q_tail);
  if (ld_volatile(c.done1) < t1 || ld_volatile(c.q1_head) < t1) return false;
  return ld_volatile(c.q2_head) >= ld_volatile(e2.q_tail);
}

template <int C0, int GL, int CL>
__global__ void __launch_bounds__(128, XDROP_MERGED_MINBLOCKS)
band_merged_kernel(Problem P, const int* __restrict__ items, const int* __restrict__ n_items_ptr, MergedCtr c,
                   Esc e1, Esc e2, Esc e3, Steal st) {
  const int lane = threadIdx.x & 31;
  const int n_items = *n_items_ptr;
  const int n_long = min(*c.n_long, n_items);
  const int first = (GL > 1) ? n_long : 0;
  const bool t0ok = t0_block(c);
  bool idle = false;                    // this warp is counted in *c.idle
  unsigned nap = 1000;                  // current poll period of an escalation-only warp (ns)
  auto busy = [&]() { if (idle && lane == 0) atomicSub(c.idle, 1); idle = false; nap = 1000; };
  for (;;) {
    // T2 (S = 256): one extension per warp
    {
      int k = 0, h = 0;
      if (lane == 0) h = claim(c.q2_head, e2.q_tail, 1, true, k);
      k = __shfl_sync(FULL, k, 0);
      if (k) {
        h = __shfl_sync(FULL, h, 0);
        busy();
        const unsigned long long t0 = c.tl ? gtimer() : 0;
        const int slot = wait_entry_w(e2.q, h, lane);
        band_resume<32, 8>(P, e2.pool + (size_t)slot * e2.rec_ints, 1, e3);
        tl_rec(c, 4, t0);
        continue;
      }
    }
    // T1: up to 4 checkpointed extensions per warp, eight lanes x 8 cells (S = 64)
    {
      int k = 0, h = 0;
      if (lane == 0) h = claim(c.q1_head, e1.q_tail, 4, true, k);
      k = __shfl_sync(FULL, k, 0);
      if (k) {
        h = __shfl_sync(FULL, h, 0);
        const int g = lane >> 3;
        int slot = -1;
        if (g < k && (lane & 7) == 0) slot = wait_entry(e1.q, h + g);
        slot = __shfl_sync(FULL, slot, lane & ~7);
        busy();
        const unsigned long long t0 = c.tl ? gtimer() : 0;
        band_resume<8, 8>(P, slot >= 0 ? e1.pool + (size_t)slot * e1.rec_ints : nullptr, 1, e2);
        tl_rec(c, 3, t0);
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(c.done1, k);
        continue;
      }
    }
    // stolen lane-mode extensions: 8 per warp, 4 lanes each (same 32-cell window)
    {
      int k = 0, h = 0;
      if (lane == 0) h = claim(c.qs_head, st.es.q_tail, 8, true, k);
      k = __shfl_sync(FULL, k, 0);
      if (k) {
        h = __shfl_sync(FULL, h, 0);
        const int g = lane >> 2;
        int slot = -1;
        if (g < k && (lane & 3) == 0) slot = wait_entry(st.es.q, h + g);
        slot = __shfl_sync(FULL, slot, lane & ~3);
        busy();
        const unsigned long long t0 = c.tl ? gtimer() : 0;
        band_resume<4, 8>(P, slot >= 0 ? st.es.pool + (size_t)slot * st.es.rec_ints : nullptr, 0, e1);
        tl_rec(c, 2, t0);
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(c.dones, k);
        continue;
      }
    }
    // T0: long extensions, 32/GL per warp
    if (GL > 1 && t0ok) {
      int base = n_long;
      if (lane == 0 && ld_volatile(c.head_long) < n_long) base = atomicAdd(c.head_long, 32 / GL);
      base = __shfl_sync(FULL, base, 0);
      if (base < n_long) {
        const int slot = base + lane / GL;
        busy();
        const unsigned long long t0 = c.tl ? gtimer() : 0;
        band_run<GL, CL>(P, slot < n_long ? items[slot] : -1, 0, e1);
        tl_rec(c, 1, t0);
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(c.done0, min(32 / GL, n_long - base));
        continue;
      }
    }
    // T0: the rest, 32 per warp (lane per extension); in the endgame (less than `endgame`
    // extensions left in the queue) 8 per warp with 4 lanes each, to shorten the tail
    int base = n_items, take = 32;
    if (lane == 0 && t0ok) {
      const int h0 = first + ld_volatile(c.head0);
      if (h0 < n_items) {
        take = (n_items - h0 < c.endgame) ? 8 : 32;
        base = first + atomicAdd(c.head0, take);
      }
    }
    base = __shfl_sync(FULL, base, 0);
    take = __shfl_sync(FULL, take, 0);
    if (base < n_items) {
      busy();
      const unsigned long long t0 = c.tl ? gtimer() : 0;
      if (take == 32) {
        const int slot = base + lane;
        band_run<1, C0>(P, slot < n_items ? items[slot] : -1, 0, e1, &st);
        tl_rec(c, 0, t0);
      } else {
        const int slot = base + (lane >> 2);
        band_run<4, 8>(P, slot < min(base + 8, n_items) ? items[slot] : -1, 0, e1);
        tl_rec(c, 5, t0);
      }
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicAdd(c.done0, min(take, n_items - base));
      continue;
    }
    int fin = 0;
    if (lane == 0) {
      fin = merged_finished(c, n_items, e1, e2, st);
      if (!fin && !idle && t0ok) { atomicAdd(c.idle, 1); idle = true; }
    }
    fin = __shfl_sync(FULL, fin, 0);
    if (fin) break;
    // escalation-only warps back off exponentially while their queues stay empty (their polling
    // of the hot queue counters otherwise slows the T0 warps measurably)
    __nanosleep(t0ok ? 1000 : nap);
    if (!t0ok) nap = min(2 * nap, c.idle_ns);
  }
}

// The packed-mode merged kernel (X + M <= 510): the same tiers and queues as band_merged_kernel,
// with two loop instances, each at one call site, so the hot code stays in the instruction cache
// (a loop per tier did not fit: DESIGN.md §7):
//   pk_unit<32> with a run-time G: T0 lane mode G = 1 (S = 32, 32 fresh extensions per warp),
//                 T1 G = XDROP_T1_G (S = 128) and T2 G = XDROP_T2_G (S = 256), 32/G extensions
//                 per warp, refilling
//   long T0 extensions from their seed and stolen lane-mode extensions: one GL x CL instance.  T1/T2 wait for a full batch of records
// unless the oldest queued one has waited age_us or T0 has been fully claimed.
template <int GL, int CL, bool CP = false>
__global__ void __launch_bounds__(128, XDROP_PKM_MINBLOCKS)
pk_merged_kernel(Problem P, const int* __restrict__ items, const int* __restrict__ n_items_ptr, MergedCtr c,
                 const PkTier* tiers, Steal st) {
  static_assert(GL * CL == 32, "4-lane units keep the lane window");
  if (*c.probe_cnt < c.probe_thr) return;            // the batch's probe chose the tiered kernel
  enum { NONE = 0, FRESH, T1, T2, T3, STOLEN, LONG, WIDE };
  const int lane = threadIdx.x & 31;
  const int n_items = *n_items_ptr;
  const int n_long = min(*c.n_long, n_items);
  const int first = n_long;
  const bool t0ok = t0_block(c);
  bool idle = false;
  unsigned nap = 1000;
  for (;;) {
    // lane 0 picks the unit: T3, T2, T1, stolen, long, fresh (escalated work first)
    int kind = NONE, h = 0, k = 0, base = 0;
    if (lane == 0) {
      const bool t0_over = ld_volatile(c.head0) + first >= n_items;
      h = claim(tiers[4].head, tiers[4].src.q_tail, 1, true, k);
      if (k) kind = WIDE;
      if (!kind) { h = claim(tiers[3].head, tiers[3].src.q_tail, 1, true, k); if (k) kind = T3; }
      if (!kind) { h = claim_batch(c.q2_head, tiers[2].src, 32 / XDROP_T2_G, t0_over, c.age_us, k); if (k) kind = T2; }
      if (!kind) { h = claim_batch(c.q1_head, tiers[1].src, 32 / XDROP_T1_G, t0_over, c.age_us, k); if (k) kind = T1; }
      if (!kind) { h = claim(c.qs_head, st.es.q_tail, 32 / GL, true, k); if (k) kind = STOLEN; }
      if (!kind && t0ok && ld_volatile(c.head_long) < n_long) {
        base = atomicAdd(c.head_long, 32 / GL);
        if (base < n_long) kind = LONG;
      }
      if (!kind && t0ok && !t0_over) {
        base = first + atomicAdd(c.head0, 32);
        if (base < n_items) kind = FRESH;
      }
      if (kind && idle) { atomicSub(c.idle, 1); idle = false; }
      if (!kind) {
        // T2 done (=> T3's queue is final), the endgame steals done (they may push S1024 records) and
        // T3 drained, besides the lower tiers
        const int t2 = ld_volatile(tiers[2].src.q_tail), tw = ld_volatile(tiers[4].src.q_tail);
        if (merged_finished(c, n_items, tiers[1].src, tiers[2].src, st) && ld_volatile(tiers[2].done) >= t2 &&
            ld_volatile(tiers[4].done) >= tw && ld_volatile(tiers[4].head) >= tw &&
            ld_volatile(tiers[3].head) >= ld_volatile(tiers[3].src.q_tail))
          kind = -1;
        else if (!idle && t0ok) { atomicAdd(c.idle, 1); idle = true; }
      } else {
        nap = 1000;
      }
    }
    kind = __shfl_sync(FULL, kind, 0);
    if (kind < 0) break;
    if (kind == NONE) {
      // escalation-only warps back off exponentially while their queues stay empty
      __nanosleep(t0ok ? 1000 : nap);
      if (!t0ok) nap = min(2 * nap, c.idle_ns);
      continue;
    }
    h = __shfl_sync(FULL, h, 0);
    k = __shfl_sync(FULL, k, 0);
    base = __shfl_sync(FULL, base, 0);
    const unsigned long long t0 = c.tl ? gtimer() : 0;
    if (kind == WIDE) {
      // endgame steal of a T1/T2 extension: one per warp, 32 lanes x 8 cells (S = 256), overflow to T3
      const int slot = wait_entry_w(tiers[4].src.q, h, lane);
      pk_resume<32, 8, CP>(P, tiers[4].src.pool + (size_t)slot * tiers[4].src.rec_ints, 1, tiers[4].esc);
      tl_rec(c, 7, t0);
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicAdd(tiers[4].done, 1);
    } else if (kind == STOLEN || kind == LONG) {
      // one GL x CL instance for both: fresh from the seed (long) or from a stolen record
      const int g = lane / GL, gl = lane % GL;
      Band16<CL> B;
      int d = 0;
      pk_keys<CL>(B, GL, gl, P.keym >> 8);
      if (kind == LONG) {
        const int slot = base + g;
        pk_init_seed<CL, CP>(B, GL, gl, slot < n_long ? items[slot] : -1, P);
      } else {
        int slot = -1;
        if (g < k && gl == 0) slot = wait_entry(st.es.q, h + g);
        slot = __shfl_sync(FULL, slot, lane & ~(GL - 1));
        pk_resume_init<CL, CP>(B, GL, gl, d, slot >= 0 ? st.es.pool + (size_t)slot * st.es.rec_ints : nullptr, P);
      }
      pk_loop<CL, CP>(B, GL, gl, d, P, 0, tiers[0].esc, nullptr);
      tl_rec(c, kind == LONG ? 1 : 2, t0);
      __threadfence();
      __syncwarp();
      if (lane == 0) {
        if (kind == LONG) atomicAdd(c.done0, min(32 / GL, n_long - base));
        else atomicAdd(c.dones, k);
      }
    } else {
      // T0 lane mode (G = 1), T1 (G = XDROP_T1_G), T2 (G = XDROP_T2_G), T3 (G = 32, S = 1024): one
      // loop instance
      const int t = kind == FRESH ? 0 : kind == T1 ? 1 : kind == T2 ? 2 : 3;
      pk_unit<32, CP>(P, t == 0 ? 1 : t == 1 ? XDROP_T1_G : t == 2 ? XDROP_T2_G : 32, t, tiers, items, base, n_items,
                  h, k, st);
      tl_rec(c, t == 0 ? 0 : t == 1 ? 3 : t == 2 ? 4 : 6, t0);
      if (t == 0) {
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(c.done0, min(32, n_items - base));
      }
    }
  }
}

// The packed-mode TIERED kernel: a compile-time loop instance per tier with few cells per lane in
// the escalation tiers (T1 = 8 lanes x 8 cells, S = 64, claimed as soon as records appear;
// T2 = 32 lanes x 8 cells, S = 256, one per warp; 4-lane units for long / stolen extensions).
// Short anti-diagonal latency for the escalated extensions, so they never become the launch's
// tail; but with several hot loops on an SM it stalls on instruction fetch once escalated work
// is a large share of the batch.  xdrop_capi.cu picks it or pk_merged_kernel per call (§7).
template <int GL, int CL, bool CP = false>
__global__ void __launch_bounds__(128, XDROP_PKT_MINBLOCKS)
pk_tiered_kernel(Problem P, const int* __restrict__ items, const int* __restrict__ n_items_ptr, MergedCtr c,
                 Esc e1, Esc e2, Esc e3, Steal st) {
  if (*c.probe_cnt >= c.probe_thr) return;           // the batch's probe chose the shared kernel
  const int lane = threadIdx.x & 31;
  const int n_items = *n_items_ptr;
  const int n_long = min(*c.n_long, n_items);
  const int first = n_long;
  const bool t0ok = t0_block(c);
  bool idle = false;
  unsigned nap = 1000;
  auto busy = [&]() { if (idle && lane == 0) atomicSub(c.idle, 1); idle = false; nap = 1000; };
  for (;;) {
    // T2 (S = 256): one extension per warp, 32 lanes x 8 cells
    {
      int k = 0, h = 0;
      if (lane == 0) h = claim(c.q2_head, e2.q_tail, 1, true, k);
      k = __shfl_sync(FULL, k, 0);
      if (k) {
        h = __shfl_sync(FULL, h, 0);
        busy();
        const unsigned long long t0 = c.tl ? gtimer() : 0;
        const int slot = wait_entry_w(e2.q, h, lane);
        pk_resume<32, 8, CP>(P, e2.pool + (size_t)slot * e2.rec_ints, 1, e3);
        tl_rec(c, 4, t0);
        continue;
      }
    }
    // T1: up to 4 checkpointed extensions per warp, 8 lanes x 8 cells (S = 64)
    {
      int k = 0, h = 0;
      if (lane == 0) h = claim(c.q1_head, e1.q_tail, 4, true, k);
      k = __shfl_sync(FULL, k, 0);
      if (k) {
        h = __shfl_sync(FULL, h, 0);
        const int g = lane >> 3;
        int slot = -1;
        if (g < k && (lane & 7) == 0) slot = wait_entry(e1.q, h + g);
        slot = __shfl_sync(FULL, slot, lane & ~7);
        busy();
        const unsigned long long t0 = c.tl ? gtimer() : 0;
        pk_resume<8, 8, CP>(P, slot >= 0 ? e1.pool + (size_t)slot * e1.rec_ints : nullptr, 1, e2);
        tl_rec(c, 3, t0);
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(c.done1, k);
        continue;
      }
    }
    // stolen lane-mode extensions: 32/GL per warp, GL lanes each (same 32-cell window)
    {
      int k = 0, h = 0;
      if (lane == 0) h = claim(c.qs_head, st.es.q_tail, 32 / GL, true, k);
      k = __shfl_sync(FULL, k, 0);
      if (k) {
        h = __shfl_sync(FULL, h, 0);
        const int g = lane / GL;
        int slot = -1;
        if (g < k && (lane % GL) == 0) slot = wait_entry(st.es.q, h + g);
        slot = __shfl_sync(FULL, slot, lane & ~(GL - 1));
        busy();
        const unsigned long long t0 = c.tl ? gtimer() : 0;
        pk_resume<GL, CL, CP>(P, slot >= 0 ? st.es.pool + (size_t)slot * st.es.rec_ints : nullptr, 0, e1);
        tl_rec(c, 2, t0);
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(c.dones, k);
        continue;
      }
    }
    // T0: long extensions, 32/GL per warp
    if (t0ok) {
      int base = n_long;
      if (lane == 0 && ld_volatile(c.head_long) < n_long) base = atomicAdd(c.head_long, 32 / GL);
      base = __shfl_sync(FULL, base, 0);
      if (base < n_long) {
        const int slot = base + lane / GL;
        busy();
        const unsigned long long t0 = c.tl ? gtimer() : 0;
        pk_run<GL, CL, CP>(P, slot < n_long ? items[slot] : -1, 0, e1);
        tl_rec(c, 1, t0);
        __threadfence();
        __syncwarp();
        if (lane == 0) atomicAdd(c.done0, min(32 / GL, n_long - base));
        continue;
      }
    }
    // T0: the rest, 32 per warp (lane per extension)
    int base = n_items;
    if (lane == 0 && t0ok) {
      const int h0 = first + ld_volatile(c.head0);
      if (h0 < n_items) base = first + atomicAdd(c.head0, 32);
    }
    base = __shfl_sync(FULL, base, 0);
    if (base < n_items) {
      busy();
      const unsigned long long t0 = c.tl ? gtimer() : 0;
      const int slot = base + lane;
      pk_run<1, XDROP_PK_C, CP>(P, slot < n_items ? items[slot] : -1, 0, e1, &st);
      tl_rec(c, 0, t0);
      __threadfence();
      __syncwarp();
      if (lane == 0) atomicAdd(c.done0, min(32, n_items - base));
      continue;
    }
    int fin = 0;
    if (lane == 0) {
      fin = merged_finished(c, n_items, e1, e2, st);
      if (!fin && !idle && t0ok) { atomicAdd(c.idle, 1); idle = true; }
    }
    fin = __shfl_sync(FULL, fin, 0);
    if (fin) break;
    __nanosleep(t0ok ? 1000 : nap);
    if (!t0ok) nap = min(2 * nap, c.idle_ns);
  }
}

// Per-batch choice of the packed band kernel: a probe runs an evenly spaced sample of
// n_probe extensions of the length-sorted queue in the T0 lane mode (one lane each, the T0 window)
// for at most 2 * cap_half anti-diagonals (m, n capped; results it writes are overwritten by the
// band kernel that follows) and counts the extensions whose band outgrows the window (cnt: an Esc
// with no record pool, so pk_save only counts).  The two packed kernels launched after it read the
// count and all but one exit at once: escalated work is then predicted from the batch itself, not
// from the previous call.
template <int C>
__global__ void __launch_bounds__(128)
pk_probe_kernel(Problem P, const int* __restrict__ items, const int* __restrict__ n_items_ptr, int n_probe,
                int stride, int cap_half, Esc cnt) {
  const int n_items = *n_items_ptr;
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  int item = -1;
  if (gid < n_probe && (int64_t)gid * stride < n_items) item = items[(int64_t)gid * stride];
  Band16<C> B;
  pk_keys<C>(B, 1, 0, P.keym >> 8);
  pk_init_seed<C>(B, 1, 0, item, P);
  B.m = min(B.m, cap_half);
  B.n = min(B.n, cap_half);
  pk_loop<C>(B, 1, 0, 0, P, 0, cnt, nullptr);
}

// ------------------------------------------------------------ CTA path
// One extension per thread block ("CTA per pair" for the widest bands): NT
// threads x CC cells = S cells (2S diagonals) in registers, the same cell update
// as band_diag; neighbours across warp boundaries and the per-anti-diagonal
// reductions go through shared memory, one barrier per anti-diagonal (buffers
// double-buffered by anti-diagonal parity).  <256, 16> (S = 4096) resumes the S = 1024 level's
// checkpoints; an extension wider than that restarts in the unbounded kernel.  <128, 8> (S = 1024,
// checkpointing into the <256, 16> queue) can replace the warp-per-extension S = 1024 level
// (XDROP_S1024=1); measured slower.
#ifndef XDROP_CTA_MINB
#define XDROP_CTA_MINB 3       // resident 4-warp CTA blocks per SM requested from ptxas
#endif
template <int NT, int CC>
__global__ void __launch_bounds__(NT, NT == 128 ? XDROP_CTA_MINB : 1)
band_cta_kernel(Problem P, Esc src, int* queue_head, Esc esc, int level) {
  constexpr int S = NT * CC, NR = 2 * CC, NW = NT / 32;
  constexpr int NCH = 4, CL = CC / NCH;
  static_assert(CC % 4 == 0 && CC <= 32, "CC");
  __shared__ int edgeL[2][NW], edgeR[2][NW];   // lane 0's R[0], lane 31's R[NR-1] per warp
  __shared__ int red[2][NW][4];                // tmin, tmax, vmax, t* per warp
  __shared__ int sh_next[NW][2];               // window shift hand-over across warps
  __shared__ int s_q;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int n = *src.q_tail;
  const int keym = P.keym, two = keym >> (KEYSH - 1);
  for (;;) {
    if (t == 0) s_q = atomicAdd(queue_head, 1);
    __syncthreads();
    const int qi = s_q;
    __syncthreads();
    if (qi >= n) return;
    const int* rec = src.pool + (size_t)src.q[qi] * src.rec_ints;
    // ---- resume (as band_resume with G = NT)
    const int item = rec[0];
    const Geom gm = item_geom(P, item);
    int d = rec[1];
    const int s_src = rec[14], shv = S - s_src;
    int K0 = rec[2] - shv, dbase = rec[3], thrW = rec[4], best = rec[5], istar = rec[6], jstar = rec[7];
    int minL1 = rec[8], maxL1 = rec[9], minL2 = rec[10], maxL2 = rec[11];
    int ia0 = rec[12] - shv / 2, jb0 = rec[13] + shv / 2;
    long long cells = (long long)(unsigned)rec[15] | ((long long)rec[16] << 32);
    int R[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
      const int q = NR * t + r - shv;
      R[r] = (q >= 0 && q < 2 * s_src) ? rec[HDR + q] : NEGV;
    }
    uint64_t Aw, Bw;
    uint32_t An, An2, Bn, Bn2;
    int rem = 16;
    auto reload = [&]() {
      const int ia = ia0 + CC * t, jb = jb0 - CC * t;
      Aw = load32c(P.PA, gm.sa, gm.da, ia);
      An = load16(P.PA, gm.sa, gm.da, ia + 32);
      An2 = load16(P.PA, gm.sa, gm.da, ia + 32 + rem);
      Bw = rev_fields(load32c(P.PB, gm.sb, gm.db, jb - 31));
      Bn = load16(P.PB, gm.sb, gm.db, jb + 1);
      Bn2 = load16(P.PB, gm.sb, gm.db, jb + 1 + rem);
    };
    reload();
    if (lane == 0) edgeL[d & 1][w] = R[0];        // read by anti-diagonal d+1
    if (lane == 31) edgeR[d & 1][w] = R[NR - 1];
    __syncthreads();
    bool active = true;
    while (active) {
#pragma unroll
      for (int par = 1; par >= 0; --par) {         // odd anti-diagonal, then even
        ++d;
        const int pb = (d - 1) & 1, cb = d & 1;      // previous / current buffers
        const int M2 = P.M - 2 * P.g, mu2 = P.mu - 2 * P.g;
        const int qlo = d - K0 - 2 * gm.n, qhi = 2 * gm.m - d - K0;
        const uint64_t x = Aw ^ Bw ^ gm.bmask;
        int nb;
        if (par == 0) { nb = __shfl_up_sync(FULL, R[NR - 1], 1); if (lane == 0) nb = w > 0 ? edgeR[pb][w - 1] : NEGV; }
        else { nb = __shfl_down_sync(FULL, R[0], 1); if (lane == 31) nb = w < NW - 1 ? edgeL[pb][w + 1] : NEGV; }
        int key[CC];
        int ch[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) ch[c] = 0;
#pragma unroll
        for (int tt = 0; tt < CC; ++tt) {
          const int r = 2 * tt + par;
          const int lft = (r == 0) ? nb : R[r == 0 ? 0 : r - 1];
          const int rgt = (r == NR - 1) ? nb : R[r >= NR - 1 ? 0 : r + 1];
          const bool mis = ((x >> (2 * tt)) & 3ull) != 0ull;
          int v = __vimax3_s32(lft, rgt, R[r] + (mis ? mu2 : M2));
          const int q = NR * t + r;
          int sd = __mulhi(v - thrW, 2);
          sd = (q >= qlo && q <= qhi) ? sd : -1;
          v = v | (sd & (int)0xFF800000);
          R[r] = v;
          key[tt] = v * keym + (127 - tt);
          ch[tt / CL] = ch[tt / CL] * two + sd;
        }
        unsigned dbits = 0;
#pragma unroll
        for (int c = 0; c < NCH; ++c) dbits = (dbits << CL) + (unsigned)(-ch[c]);
        const int mk = tree_max3<CC>(key);
        const int vl = mk >> KEYSH;
        const unsigned lb = ~dbits & (CC == 32 ? 0xffffffffu : ((1u << CC) - 1u));
        const int tmin = lb ? (__clz(lb) - (32 - CC)) + CC * t : EMIN;
        const int tmax = lb ? (CC - __ffs(lb)) + CC * t : EMAX;
        // warp reductions, then across warps through shared memory
        const int wv = __reduce_max_sync(FULL, vl);
        const unsigned ball = __ballot_sync(FULL, vl == wv);
        const int wgt = __shfl_sync(FULL, CC * t + 127 - (mk & 127), __ffs(ball) - 1);
        const int wmin = __reduce_min_sync(FULL, tmin), wmax = __reduce_max_sync(FULL, tmax);
        if (lane == 0) { red[cb][w][0] = wmin; red[cb][w][1] = wmax; red[cb][w][2] = wv; red[cb][w][3] = wgt;
                         edgeL[cb][w] = R[0]; }
        if (lane == 31) edgeR[cb][w] = R[NR - 1];
        // stream advance for d+1
        if (par == 0) { Aw = (Aw >> 2) | ((uint64_t)(An & 3u) << 62); An >>= 2; ia0 += 1; }
        else { Bw = (Bw << 2) | (uint64_t)(Bn & 3u); Bn >>= 2; jb0 += 1; }
        __syncthreads();
        int gv = NEGV, gt = 0, gmn = EMIN, gmx = EMAX;
#pragma unroll
        for (int k = 0; k < NW; ++k) {
          const int v = red[cb][k][2];
          if (v > gv) { gv = v; gt = red[cb][k][3]; }
          gmn = min(gmn, red[cb][k][0]); gmx = max(gmx, red[cb][k][1]);
        }
        thrW = max(thrW, gv - P.X) - P.g;
        const int ibase = (d + K0 + par) >> 1;
        const int woff = -P.g * (d - dbase);
        if (gv - woff > best) { best = gv - woff; istar = ibase + gt; jstar = d - istar; }
        const int lo = max(max(0, d - gm.n), min(minL1, minL2 + 1));
        const int hi = min(min(gm.m, d), max(maxL1, maxL2) + 1);
        cells += hi >= lo ? (long long)(hi - lo + 1) : 0ll;
        minL2 = minL1; maxL2 = maxL1;
        minL1 = gmn == EMIN ? EMIN : ibase + gmn;
        maxL1 = gmx == EMAX ? EMAX : ibase + gmx;
      }
      // ---- block end (uniform over the block)
      if (d - dbase >= 1024) {
        const int woff = -P.g * (d - dbase);
#pragma unroll
        for (int r = 0; r < NR; ++r) R[r] -= woff;
        thrW -= woff; dbase = d;
        // the edge copies for anti-diagonal d+1 are in shared memory: rebase them too
        __syncthreads();
        if (lane == 0) edgeL[d & 1][w] = R[0];
        if (lane == 31) edgeR[d & 1][w] = R[NR - 1];
        __syncthreads();
      }
      if (--rem == 0) {
        rem = 16; An = An2; Bn = Bn2;
        An2 = load16(P.PA, gm.sa, gm.da, ia0 + CC * t + 48);
        Bn2 = load16(P.PB, gm.sb, gm.db, jb0 - CC * t + 17);
      }
      const bool e0 = minL1 == EMIN, e1 = minL2 == EMIN;
      if ((e0 && e1) || d >= gm.m + gm.n) {
        if (t == 0) {
          ExtOut o; o.best = best - BIAS; o.istar = istar; o.jstar = jstar; o.level = level; o.cells = cells; o.pad = 0;
          XDROP_CHK_ITEM(P, item);
          P.ext[item] = o;
        }
        active = false;
        break;
      }
      int qmn = 1 << 30, qmx = -(1 << 30);
      if (!e0) { qmn = 2 * minL1 - d - K0; qmx = 2 * maxL1 - d - K0; }
      if (!e1) { qmn = min(qmn, 2 * minL2 - (d - 1) - K0); qmx = max(qmx, 2 * maxL2 - (d - 1) - K0); }
      int dir = 0;
      if (qmx >= 2 * S - 2) dir = qmn >= 4 ? 1 : 2;
      else if (qmn <= 1) dir = qmx <= 2 * S - 5 ? -1 : 2;
      if (dir == 2) {
        // wider than the block window: checkpoint for the next (wider) CTA level when `esc` has a
        // record pool, else restart in the unbounded kernel
        if (t == 0) s_q = esc.cap > 0 ? atomicAdd(esc.pool_tail, 1) : esc.cap;
        __syncthreads();
        const int slot = s_q;
        if (slot < esc.cap) {
          int* out = esc.pool + (size_t)slot * esc.rec_ints;
          if (t == 0) {
            out[0] = item; out[1] = d; out[2] = K0; out[3] = dbase; out[4] = thrW; out[5] = best;
            out[6] = istar; out[7] = jstar; out[8] = minL1; out[9] = maxL1; out[10] = minL2; out[11] = maxL2;
            out[12] = ia0; out[13] = jb0; out[14] = S;
            out[15] = (int)(cells & 0xffffffffll); out[16] = (int)(cells >> 32); out[REC_T] = rec_stamp();
          }
#pragma unroll
          for (int r = 0; r < NR; ++r) out[HDR + NR * t + r] = R[r];
          __threadfence();
          __syncthreads();
          if (t == 0) push_item(esc.q, esc.q_tail, slot);
        } else if (t == 0) {
          push_item(esc.fb_items, esc.fb_tail, item);
        }
        active = false;
        break;
      }
      if (dir != 0) {
        // shift by 2 diagonals across the block: R[r] <- R[r + 2 dir]
        int n0, n1;
        if (dir > 0) {
          if (lane == 0) { sh_next[w][0] = R[0]; sh_next[w][1] = R[1]; }
          __syncthreads();
          n0 = __shfl_down_sync(FULL, R[0], 1); n1 = __shfl_down_sync(FULL, R[1], 1);
          if (lane == 31) { n0 = w < NW - 1 ? sh_next[w + 1][0] : NEGV; n1 = w < NW - 1 ? sh_next[w + 1][1] : NEGV; }
#pragma unroll
          for (int r = 0; r < NR - 2; ++r) R[r] = R[r + 2];
          R[NR - 2] = n0; R[NR - 1] = n1;
        } else {
          if (lane == 31) { sh_next[w][0] = R[NR - 2]; sh_next[w][1] = R[NR - 1]; }
          __syncthreads();
          n0 = __shfl_up_sync(FULL, R[NR - 2], 1); n1 = __shfl_up_sync(FULL, R[NR - 1], 1);
          if (lane == 0) { n0 = w > 0 ? sh_next[w - 1][0] : NEGV; n1 = w > 0 ? sh_next[w - 1][1] : NEGV; }
#pragma unroll
          for (int r = NR - 1; r >= 2; --r) R[r] = R[r - 2];
          R[0] = n0; R[1] = n1;
        }
        K0 += 2 * dir; ia0 += dir; jb0 -= dir;
        reload();
        // refresh the edges of the current buffer (read by the next anti-diagonal)
        if (lane == 0) edgeL[d & 1][w] = R[0];
        if (lane == 31) edgeR[d & 1][w] = R[NR - 1];
        __syncthreads();
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------ general path
// Warp per extension, one anti-diagonal's values indexed by i; the hull of each anti-diagonal
// bounds what is valid.  compat != 0: the SeqAn/LOGAN-style mode (XDROP_FLAG_SEQAN_COMPAT,
// DESIGN.md Q28-Q30): a pure-gap cell (i = 0 or j = 0) lives only if v > best - X, and the
// extension reports its "longest extension" -- the largest-H live cell of the last anti-diagonal
// with a live cell (smallest i on ties) -- with H there instead of best.  Thresholds, hull, cells
// and termination are unchanged.
// CAP = 0: three arrays of m + 1 values in global scratch (unbounded band width).  CAP > 0: three
// rings of CAP values in shared memory, slot i mod CAP (exact while every hull is at most CAP
// wide); returns false, with nothing written, as soon as a hull is wider.  NW warps work on the
// extension (NW > 1: the whole thread block; per anti-diagonal one barrier, which also publishes
// the per-warp reductions `red`, double-buffered by parity).
// NW == 1 and G < 32: G lanes of the warp per extension (group-local shuffle reductions; the groups
// of a warp run their extensions independently).
template <int CAP, int NW, int G = 32>
__device__ __forceinline__ bool gen_extend(const Problem& P, int item, int* Hc, int* H1, int* H2, int level,
                                           int compat, int (*red)[NW][4]) {
  static_assert(NW == 1 || G == 32, "multi-warp extensions use whole warps");
  constexpr int T = NW == 1 ? G : 32 * NW;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int t = NW == 1 ? (lane & (G - 1)) : (int)threadIdx.x;
  const unsigned gmk = gmask(G);
  auto sync = [gmk]() { if constexpr (NW == 1) __syncwarp(gmk); else __syncthreads(); };
  auto rmax = [gmk](int v) {
    if constexpr (G == 32) return __reduce_max_sync(FULL, v);
    else {
#pragma unroll
      for (int o = 1; o < G; o <<= 1) v = max(v, __shfl_xor_sync(gmk, v, o));
      return v;
    }
  };
  auto rmin = [gmk](int v) {
    if constexpr (G == 32) return __reduce_min_sync(FULL, v);
    else {
#pragma unroll
      for (int o = 1; o < G; o <<= 1) v = min(v, __shfl_xor_sync(gmk, v, o));
      return v;
    }
  };
  const Geom gm = item_geom(P, item);
  const int m = gm.m, n = gm.n;
  auto ix = [](int i) { return CAP ? (i & (CAP - 1)) : i; };
  // anti-diagonals d (Hc), d-1 (H1), d-2 (H2), rotated in registers: values by i, the hull
  // [lo, hi] computed and the live extent [mn, mx] (EMIN/EMAX: empty)
  if (t == 0) H1[0] = BIAS;                     // d = 0: the origin; d = -1: empty
  int lo1 = 0, hi1 = 0, mn1 = 0, mx1 = 0;
  int lo2 = 1, hi2 = 0, mn2 = EMIN, mx2 = EMAX;
  int best = BIAS, istar = 0, jstar = 0;
  int lastv = BIAS, lasti = 0, lastd = 0;      // compat: max cell of the last live anti-diagonal
  long long cells = 1;
  const int cm = (int)(gm.bmask & 3ull);
  sync();
  for (int d = 1; d <= m + n; ++d) {
    if (mn1 == EMIN && mn2 == EMIN) break;
    const int lo = max(max(0, d - n), min(mn1, mn2 == EMIN ? EMIN : mn2 + 1));
    const int hi = min(min(m, d), max(mx1, mx2 == EMAX ? EMAX : mx2) + 1);
    if (CAP && hi - lo + 1 > CAP) return false;   // uniform over the working threads
    if (hi >= lo) cells += hi - lo + 1;
    const int thr = best - P.X;
    int kbest = NEGV, ibest = 0x7fffffff, lmn = EMIN, lmx = EMAX;
    for (int i = lo + t; i <= hi; i += T) {
      const int j = d - i;
      int v = NEGV;
      if (i >= 1 && i - 1 >= lo1 && i - 1 <= hi1) v = max(v, H1[ix(i - 1)] + P.g);
      if (j >= 1 && i >= lo1 && i <= hi1) v = max(v, H1[ix(i)] + P.g);
      if (i >= 1 && j >= 1 && i - 1 >= lo2 && i - 1 <= hi2) {
        const int ca = char_at(P.PA, gm.sa, gm.da, i - 1);
        const int cb = char_at(P.PB, gm.sb, gm.db, j - 1) ^ cm;
        v = max(v, H2[ix(i - 1)] + (ca == cb ? P.M : P.mu));
      }
      const bool live = (compat && (i == 0 || j == 0)) ? v > thr : v >= thr;   // Q28: strict edge
      v = live ? v : NEGV;
      Hc[ix(i)] = v;
      if (live) {
        if (v > kbest) { kbest = v; ibest = i; }
        lmn = min(lmn, i); lmx = max(lmx, i);
      }
    }
    int gv = rmax(kbest);
    int gi = rmin((kbest == gv) ? ibest : 0x7fffffff);
    lmn = rmin(lmn);
    lmx = rmax(lmx);
    if constexpr (NW > 1) {
      int* r = red[d & 1][w];
      if (lane == 0) { r[0] = gv; r[1] = gi; r[2] = lmn; r[3] = lmx; }
      __syncthreads();
      gv = NEGV; gi = 0x7fffffff; lmn = EMIN; lmx = EMAX;
#pragma unroll
      for (int u = 0; u < NW; ++u) {
        const int* q = red[d & 1][u];
        if (q[0] > gv || (q[0] == gv && q[1] < gi)) { gv = q[0]; gi = q[1]; }
        lmn = min(lmn, q[2]); lmx = max(lmx, q[3]);
      }
    }
    if (lmn != EMIN && gv > best) { best = gv; istar = gi; jstar = d - gi; }
    if (lmn != EMIN) { lastv = gv; lasti = gi; lastd = d; }                        // Q29
    int* const tmp = H2; H2 = H1; H1 = Hc; Hc = tmp;
    lo2 = lo1; hi2 = hi1; mn2 = mn1; mx2 = mx1;
    lo1 = lo; hi1 = hi; mn1 = lmn; mx1 = lmx;
    if constexpr (NW == 1) __syncwarp(gmk);
  }
  if (compat) { best = lastv; istar = lasti; jstar = lastd - lasti; }              // Q29, Q30
  if (t == 0) {
    ExtOut o; o.best = best - BIAS; o.istar = istar; o.jstar = jstar; o.level = level;
    o.cells = cells; o.pad = 0;
    XDROP_CHK_ITEM(P, item);
    P.ext[item] = o;
  }
  sync();
  return true;
}

// The unbounded fallback: global scratch of 3 x stride values per warp (stride > longest m).
__global__ void __launch_bounds__(128)
general_kernel(Problem P, const int* __restrict__ items, const int* __restrict__ n_items_ptr,
               int* queue_head, int* scratch, int64_t stride, int level, int compat) {
  const int lane = threadIdx.x & 31;
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int* const base = scratch + (int64_t)warp_global * 3 * stride;
  const int n_items = *n_items_ptr;
  for (;;) {
    int slot = 0;
    if (lane == 0) slot = atomicAdd(queue_head, 1);
    slot = __shfl_sync(FULL, slot, 0);
    if (slot >= n_items) break;
    gen_extend<0, 1>(P, items[slot], base, base + stride, base + 2 * stride, level, compat, nullptr);
  }
}

// The compat mode's kernels: the general path with its anti-diagonals in shared-memory rings.
// general_group_kernel: 8 lanes per extension, 4 per warp, three 256-value rings each (48 KB per
// 4-warp block) -- most hulls are a few dozen cells wide; wider ones are queued (ovf) for
// general_ring_kernel: one warp per extension, 3 x 1,024 values per warp (48 KB per 4-warp block,
// 4 blocks per SM); an extension whose hull outgrows its ring is queued (ovf) for
// general_wide_kernel: one 8-warp block per extension, 3 x 8,192 values (96 KB, 2 blocks per SM),
// which redoes it from the seed and queues the still wider ones for general_kernel.
constexpr int kGenRing = 1024, kGenRingWide = 8192, kGenGroup = 8, kGenGroupRing = 256;
// Which compat kernel takes the batch first: the group kernel unless a probe of the batch counted
// >= thr extensions whose band outgrows 32 cells early (wide hulls: the group shape's per-anti-
// diagonal chain would be the launch's tail), then the warp-ring kernel takes the queue directly.
struct GenChoice { const int* cnt; int thr; };
__global__ void __launch_bounds__(128, 4)
general_group_kernel(Problem P, const int* __restrict__ items, const int* __restrict__ n_items_ptr,
                     int* queue_head, int* ovf_items, int* ovf_count, int level, int compat, GenChoice ch) {
  if (*ch.cnt >= ch.thr) return;
  constexpr int NG = 32 / kGenGroup;
  __shared__ int ring[4][NG][3][kGenGroupRing];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, g = lane / kGenGroup;
  const int n_items = *n_items_ptr;
  for (;;) {
    int base = 0;
    if (lane == 0) base = atomicAdd(queue_head, NG);
    base = __shfl_sync(FULL, base, 0);
    if (base >= n_items) break;
    const int slot = base + g;
    if (slot < n_items) {                                // group-uniform
      const int item = items[slot];
      if (!gen_extend<kGenGroupRing, 1, kGenGroup>(P, item, ring[w][g][0], ring[w][g][1], ring[w][g][2], level,
                                                   compat, nullptr) &&
          (lane & (kGenGroup - 1)) == 0)
        ovf_items[atomicAdd(ovf_count, 1)] = item;
    }
    __syncwarp();
  }
}
__global__ void __launch_bounds__(128, 4)
general_ring_kernel(Problem P, const int* __restrict__ items, const int* __restrict__ n_items_ptr,
                    int* queue_head, int* ovf_items, int* ovf_count, int level, int compat, GenChoice ch,
                    const int* __restrict__ items0, const int* __restrict__ n_items0_ptr) {
  __shared__ int ring[4][3][kGenRing];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (*ch.cnt >= ch.thr) { items = items0; n_items_ptr = n_items0_ptr; }   // the group kernel stood aside
  const int n_items = *n_items_ptr;
  for (;;) {
    int slot = 0;
    if (lane == 0) slot = atomicAdd(queue_head, 1);
    slot = __shfl_sync(FULL, slot, 0);
    if (slot >= n_items) break;
    const int item = items[slot];
    if (!gen_extend<kGenRing, 1>(P, item, ring[w][0], ring[w][1], ring[w][2], level, compat, nullptr) &&
        lane == 0)
      ovf_items[atomicAdd(ovf_count, 1)] = item;
    __syncwarp();
  }
}

__global__ void __launch_bounds__(256, 2)
general_wide_kernel(Problem P, const int* __restrict__ items, const int* __restrict__ n_items_ptr,
                    int* queue_head, int* ovf_items, int* ovf_count, int level, int compat) {
  extern __shared__ int ring_w[];                 // 3 x kGenRingWide
  __shared__ int red[2][8][4];
  __shared__ int s_slot;
  const int n_items = *n_items_ptr;
  for (;;) {
    if (threadIdx.x == 0) s_slot = atomicAdd(queue_head, 1);
    __syncthreads();
    const int slot = s_slot;
    __syncthreads();
    if (slot >= n_items) break;
    const int item = items[slot];
    if (!gen_extend<kGenRingWide, 8>(P, item, ring_w, ring_w + kGenRingWide, ring_w + 2 * kGenRingWide, level,
                                     compat, red) && threadIdx.x == 0)
      ovf_items[atomicAdd(ovf_count, 1)] = item;
    __syncthreads();
  }
}

// ----------------------------------------------------------- pack / prepare
// ASCII -> 2-bit (A0 C1 G2 T3, base t at bits 2(t mod 16) of word t/16),
// written at pool index + GUARD.  Any other byte sets *bad to its index.
__device__ __forceinline__ uint32_t code_of(unsigned ch, int64_t t, unsigned long long* bad) {
  const unsigned u = ch & 0xDFu;   // upper case
  if (!(u == 'A' || u == 'C' || u == 'G' || u == 'T')) atomicMin(bad, (unsigned long long)t);
  return ((ch >> 1) ^ (ch >> 2)) & 3u;   // A/a 0, C/c 1, G/g 2, T/t 3
}
// 16 ASCII bases (one aligned uint4) -> one 2-bit word, four bases per 32-bit SIMD step:
// ((c >> 1) ^ (c >> 2)) & 3 is A0 C1 G2 T3 (either case) for each byte at once; returns false if any
// byte is outside {A,C,G,T,a,c,g,t}
__device__ __forceinline__ bool pack16(const uint4 q, uint32_t& word) {
  const uint32_t v[4] = {q.x, q.y, q.z, q.w};
  uint32_t ok = 0xffffffffu;
  word = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const uint32_t u = v[k] & 0xDFDFDFDFu;          // upper case
    ok &= __vcmpeq4(u, 0x41414141u) | __vcmpeq4(u, 0x43434343u) | __vcmpeq4(u, 0x47474747u) |
          __vcmpeq4(u, 0x54545454u);
    const uint32_t c = ((v[k] >> 1) ^ (v[k] >> 2)) & 0x03030303u;
    word |= ((c | (c >> 6) | (c >> 12) | (c >> 18)) & 0xFFu) << (8 * k);
  }
  return ok == 0xffffffffu;
}
// Every word of the packed pool (guards included: their bases are 0), four words per thread from four
// 16-byte loads when the ASCII pool is 16-byte aligned and the words are inside it; the per-byte path
// handles the pool's ends and records the index of a bad base.
__global__ void pack_kernel(const char* __restrict__ seq, int64_t len, uint32_t* __restrict__ out,
                            int64_t nwords, unsigned long long* bad) {
  const int64_t w0 = 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x);   // first output word
  if (w0 >= nwords) return;
  const bool al = (reinterpret_cast<uintptr_t>(seq) & 15) == 0;
  uint32_t words[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int64_t w = w0 + k;
    const int64_t t0 = w * 16 - GUARD;   // pool index of the first base in this word (GUARD % 16 == 0)
    uint32_t word = 0;
    bool done = false;
    if (al && t0 >= 0 && t0 + 16 <= len) done = pack16(__ldg(reinterpret_cast<const uint4*>(seq + t0)), word);
    if (!done && w < nwords) {
      word = 0;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int64_t t = t0 + u;
        if (t >= 0 && t < len) word |= code_of((unsigned char)seq[t], t, bad) << (2 * u);
      }
    }
    words[k] = word;
  }
  if (w0 + 4 <= nwords) {
    *reinterpret_cast<uint4*>(out + w0) = make_uint4(words[0], words[1], words[2], words[3]);
  } else {
    for (int k = 0; k < 4 && w0 + k < nwords; ++k) out[w0 + k] = words[k];
  }
}

// validate pairs, estimate costs, histogram of cost buckets.  A pair is valid when its read ids are
// in range, both reads' offsets lie inside their pool (0 <= off[r] <= off[r+1] <= len), both reads
// are at most max_len bases and the seed lies inside both reads (include/xdrop.h, XDROP_ESEED).
// An invalid pair sets *bad_pair to (the minimum of) its index; scan_kernel then empties the
// queue, so no band kernel ever dereferences an unvalidated id or position (device API).
__device__ __forceinline__ bool read_ok(const int64_t* off, int64_t n, int64_t len, int64_t r, int64_t& L) {
  if (r < 0 || r >= n) return false;
  const int64_t o0 = off[r], o1 = off[r + 1];
  L = o1 - o0;
  return o0 >= 0 && o1 >= o0 && o1 <= len;
}
__global__ void prep_kernel(Problem P, int* __restrict__ wcost, int* __restrict__ hist,
                            unsigned long long* bad_pair, int max_len, int* __restrict__ max_m) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P.n_pairs) return;
  const PairDesc pd = P.pairs[p];
  const int bid = pd.b_id & 0x7fffffff;
  int64_t lenA = 0, lenB = 0;
  bool ok = read_ok(P.offA, P.nA, P.lenA, pd.a_id, lenA) && read_ok(P.offB, P.nB, P.lenB, bid, lenB);
  int wl = 0, wr = 0;
  if (ok) {
    ok = pd.a_pos >= 0 && pd.b_pos >= 0 && pd.a_pos + (int64_t)P.k <= lenA &&
         pd.b_pos + (int64_t)P.k <= lenB && lenA <= max_len && lenB <= max_len;
    if (ok) {
      wl = min(pd.a_pos, pd.b_pos);
      wr = (int)min(lenA - pd.a_pos - P.k, lenB - pd.b_pos - P.k);
      // the unbounded path indexes an anti-diagonal by i in [0, m]: its scratch stride
      atomicMax(max_m, max(pd.a_pos, (int)(lenA - pd.a_pos - P.k)));
    }
  }
  if (!ok) atomicMin(bad_pair, (unsigned long long)p);
  wcost[2 * p] = wl;
  wcost[2 * p + 1] = wr;
  atomicAdd(&hist[min(wl >> BUCKET_SHIFT, NBUCKET - 1)], 1);
  atomicAdd(&hist[min(wr >> BUCKET_SHIFT, NBUCKET - 1)], 1);
}

// exclusive scan of the histogram in DESCENDING bucket order (one block of
// 1024), plus the long-extension cut: extensions whose cost w exceeds
// alpha * (total w / resident lanes) -- i.e. whose own anti-diagonal chain is
// a sizeable fraction of the whole launch's per-lane work -- form the prefix
// [0, n_long) of the sorted queue (alpha <= 0 disables the long mode).
__global__ void scan_kernel(const int* __restrict__ hist, int* __restrict__ cursor, int* __restrict__ n_long,
                            long long lanes, float alpha, const unsigned long long* __restrict__ bad_pair,
                            int* __restrict__ n_items) {
  __shared__ int part[1024];
  __shared__ unsigned long long wsum[32];
  constexpr int PER = NBUCKET / 1024;
  const int t = threadIdx.x;
  int local[PER];
  int s = 0;
  unsigned long long ws = 0;
#pragma unroll
  for (int u = 0; u < PER; ++u) {       // thread t owns descending ranks t*PER .. t*PER+PER-1
    const int b = NBUCKET - 1 - (t * PER + u);
    const int h = hist[b];
    local[u] = s; s += h;
    ws += (unsigned long long)h * (unsigned long long)((b << BUCKET_SHIFT) + (1 << (BUCKET_SHIFT - 1)));
  }
  part[t] = s;
  for (int o = 16; o > 0; o >>= 1) ws += __shfl_xor_sync(FULL, ws, o);
  if ((t & 31) == 0) wsum[t >> 5] = ws;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  const int base = part[t] - s;
#pragma unroll
  for (int u = 0; u < PER; ++u) cursor[NBUCKET - 1 - (t * PER + u)] = base + local[u];
  __syncthreads();
  if (t == 0) {
    unsigned long long tot = 0;
    for (int w = 0; w < 32; ++w) tot += wsum[w];
    int nl = 0;
    if (alpha > 0.f && lanes > 0) {
      const double thr_w = (double)alpha * (double)tot / (double)lanes;
      const long long tb = (long long)(thr_w / (double)(1 << BUCKET_SHIFT)) + 1;   // buckets fully above
      if (tb < NBUCKET) nl = cursor[tb] + hist[tb];   // items in buckets >= tb
    }
    *n_long = nl;
    // a pair failed validation (prep_kernel): no extension is queued, every band kernel finds an
    // empty queue (the force-general path reads the same count), and the host returns XDROP_ESEED
    if (*bad_pair != ~0ull) { *n_items = 0; *n_long = 0; }
  }
}

__global__ void scatter_kernel(const int* __restrict__ wcost, int64_t n_items, int* __restrict__ cursor,
                               int* __restrict__ items, int nosort) {
  const int64_t it = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (it >= n_items) return;
  if (nosort) { items[it] = (int)it; return; }
  const int b = min(wcost[it] >> BUCKET_SHIFT, NBUCKET - 1);
  const int pos = atomicAdd(&cursor[b], 1);
  items[pos] = (int)it;
}

// combine: seed score + left/right results -> per-pair result
__global__ void combine_kernel(Problem P, int* __restrict__ out5, long long* __restrict__ cells_out,
                               unsigned long long* __restrict__ level_acc) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // per-level [cells x4, items x4]
  if (p < P.n_pairs) {
    const PairDesc pd = P.pairs[p];
    const bool rc = (pd.b_id & PAIR_RC) != 0;
    const int bid = pd.b_id & 0x7fffffff;
    const int64_t xa = P.offA[pd.a_id] + GUARD + pd.a_pos;
    const int64_t lenB = P.offB[bid + 1] - P.offB[bid];
    // seed columns of B' = B (forward) or revcomp(B) (backward, complemented)
    const int64_t xb = P.offB[bid] + GUARD + (rc ? lenB - 1 - pd.b_pos : pd.b_pos);
    int mism = 0;
    for (int t = 0; t < P.k; t += 16) {
      const uint32_t bw = rc ? ~load16(P.PB, xb, -1, t) : fwd16(P.PB, xb + t);
      const uint32_t x = fwd16(P.PA, xa + t) ^ bw;
      uint32_t f = (x | (x >> 1)) & 0x55555555u;
      const int rem = P.k - t;
      if (rem < 16) f &= (1u << (2 * rem)) - 1u;
      mism += __popc(f);
    }
    const int seed = (P.k - mism) * P.M + mism * P.mu;
    const ExtOut L = P.ext[2 * p], R = P.ext[2 * p + 1];
    int* o = out5 + 5 * p;
    o[0] = L.best + seed + R.best;
    o[1] = pd.a_pos - L.istar;
    o[2] = pd.a_pos + P.k + R.istar;
    o[3] = pd.b_pos - L.jstar;
    o[4] = pd.b_pos + P.k + R.jstar;
    if (cells_out) cells_out[p] = L.cells + R.cells;
    acc[L.level & 3] += (unsigned long long)L.cells; acc[R.level & 3] += (unsigned long long)R.cells;
    acc[4 + (L.level & 3)] += 1; acc[4 + (R.level & 3)] += 1;
  }
  // reduce per warp (every lane reaches here), one atomic per counter per warp
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    unsigned long long v = acc[i];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    if ((threadIdx.x & 31) == 0 && v) atomicAdd(&level_acc[i], v);
  }
}

// f4: best seed per candidate (adjacent rows with equal a_id, b_id); the thread of a candidate's
// first row scans the run once (O(n) total), ties to the lowest row
__global__ void best_seed_kernel(const PairDesc* __restrict__ pairs, const int* __restrict__ res5, int64_t n,
                                 long long* __restrict__ best) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const PairDesc p = pairs[i];
  if (i > 0) {
    const PairDesc q = pairs[i - 1];
    if (q.a_id == p.a_id && q.b_id == p.b_id) return;      // not the first row of its candidate
  }
  int64_t j = i, bi = i;
  int bs = res5[5 * i];
  while (j + 1 < n) {
    const PairDesc q = pairs[j + 1];
    if (q.a_id != p.a_id || q.b_id != p.b_id) break;
    ++j;
    const int s = res5[5 * j];
    if (s > bs) { bs = s; bi = j; }
  }
  for (int64_t t = i; t <= j; ++t) best[t] = bi;
}

}  // namespace xk
