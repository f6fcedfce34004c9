// xdrop_pk16.cuh -- packed 16-bit band mode (included by xdrop_kernels.cuh).
//
// Same operation as band_run<G, C> (G lanes per extension, a window of S = G*C
// cells per anti-diagonal = 2S diagonals, exact checkpoints to the 32-bit
// record format), but the cells of an anti-diagonal are held as PAIRS of 16-bit
// values and updated with the sm_100a dynamic-programming instructions
// (VIMNMX.S16x2 / VIADDMNMX.S16x2), two cells per instruction.
//
// G is a plain function argument (every function is force-inlined): a constant
// G folds to the specialised code (pk_tiered_kernel: one instance per tier), and
// pk_merged_kernel ("shared") runs ONE instance of the C = 32 loop with a
// run-time G for the lane tier (G = 1, S = 32) and the escalation tiers
// (G = 4, S = 128; G = 8, S = 256).  One hot loop instead of one per tier keeps
// the kernel's hot code inside the SM's instruction cache (with a
// loop per tier the C. elegans-shaped batch stalled on instruction fetch).
//
// Layout.  Cell t of parity p sits on diagonal K0 + 2t + p; lane gl of a group
// owns cells t = gl*C + tl, tl < C.  Pair u of a parity array holds local cells
// (u, u + NP), NP = C/2 -- lo and hi half.  With this strided pairing the two
// neighbours of every pair are again whole pairs (for even cells: odd pairs u-1
// and u; for odd cells: even pairs u and u+1); only the pair at the seam needs
// one PRMT (and one shuffle from the next lane).
//
// Values.  A cell of anti-diagonal d is stored RELATIVE to the pruning
// threshold of d and scaled by 32:  v = 32 * (W - thrW_d) + (31 - t), W the
// offset-space value of band_diag.  So  live <=> v >= 0  (sign bit clear), the
// low 5 bits make v its own argmax key (larger value first, then smaller t =
// smaller i), and the recurrence
//   W_d(k) = max(W_{d-1}(k -+ 1), W_{d-2}(k) + s - 2g)
// becomes, per pair,
//   v = max(max(L, R) + D1, V2 + s' + D2)          D1 = 32 (thrW_{d-1} - thrW_d)
//     = VIADDMNMX(VIADDMNMX(V2, s' + D2 - D1, VIMNMX(L, R)), D1, -)
// Dead cells are forced to 0xC0xx (below any value a live predecessor can
// give) by one PRMT (sign of each half replicated into a byte mask, with the
// 31 - t key bytes inserted) and one LOP3.  The PRMT masks of 8 pairs are also
// accumulated by one IMAD each into a word from which the dead bits of the
// anti-diagonal are decoded exactly (live extent, hull count).
//
// Range: live values are < 32 (X + M) + 32, so this mode requires X + M <= 510
// (xdrop_capi.cu falls back to the 32-bit kernels otherwise).
#pragma once

#ifndef XDROP_PK_FMA
#define XDROP_PK_FMA 1           // cell adds on the FMA pipe (see pk_cells)
#endif

namespace pk {
constexpr uint32_t DEAD2 = 0xC000C000u;    // a pair of dead cells
constexpr uint32_t KILLC = 0xC01FC01Fu;    // LOP3 constant: bits taken from the PRMT mask
constexpr uint32_t NOFLOOR = 0x80008000u;  // no-op third operand of VIADDMNMX
constexpr uint32_t INV255 = 0xFEFEFFu;     // 255^-1 mod 2^24
}  // namespace pk

// prmt.b32 with sign-replicating selectors (__byte_perm drops selector bit 3)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
  return d;
}
// out = c ? b : (a & ~b) bitwise, as ONE LOP3 (the compiler splits the C form in two)
__device__ __forceinline__ uint32_t lop_kill(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0x98;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}
// an opaque copy (keeps a loop-invariant constant in a register instead of rematerialising it)
__device__ __forceinline__ uint32_t opaque(uint32_t x) {
  uint32_t d;
  asm volatile("mov.b32 %0, %1;" : "=r"(d) : "r"(x));
  return d;
}
// bits 0, 2, .., 30 of x -> bits 0..15
__device__ __forceinline__ uint32_t even_bits16(uint32_t x) {
  x &= 0x55555555u;
  x = (x | (x >> 1)) & 0x33333333u;
  x = (x | (x >> 2)) & 0x0F0F0F0Fu;
  x = (x | (x >> 4)) & 0x00FF00FFu;
  return __byte_perm(x, 0u, 0x4420);
}
// bit planes of 32 2-bit codes (code t at bits 2t..2t+1): plane b bit t = bit b of code t
__device__ __forceinline__ uint32_t plane32(uint64_t w, int b) {
  return even_bits16((uint32_t)(w >> b)) | (even_bits16((uint32_t)(w >> 32 >> b)) << 16);
}

// lanes of this lane's group of G (G a power of two <= 32)
__device__ __forceinline__ unsigned gmask(int G) {
  if (G == 32) return FULL;
  const int lane = threadIdx.x & 31;
  return ((1u << G) - 1u) << (lane & ~(G - 1));
}
// max / min over the lanes of each group of G (all 32 lanes converged; xor partners stay in the group)
__device__ __forceinline__ int gmax_rt(int v, int G) {
  if (G == 32) return __reduce_max_sync(FULL, v);
  for (int o = 1; o < G; o <<= 1) v = max(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ int gmin_rt(int v, int G) {
  if (G == 32) return __reduce_min_sync(FULL, v);
  for (int o = 1; o < G; o <<= 1) v = min(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
// min over this group's lanes only (callable from group-divergent code)
__device__ __forceinline__ int gmin_grp(int v, int G) {
  const unsigned gm = gmask(G);
  for (int o = 1; o < G; o <<= 1) v = min(v, __shfl_xor_sync(gm, v, o));
  return v;
}

template <int C> struct Band16 {
  static constexpr int NP = C / 2;
  uint32_t E[NP], O[NP];          // even / odd cells, pair u = (local cell u, local cell u + NP)
  uint32_t TC[NP / 2];            // key bytes 31 - t of pairs 2j, 2j+1: [lo(2j), hi(2j), lo(2j+1), hi(2j+1)]
  uint32_t A0, A1, B0, B1;        // bit planes: bit tl <-> a[ia0 + C gl + tl], b[jb0 - C gl - tl] (b ^ cm)
  uint32_t An0, An1, Bn0, Bn1;    // reservoir planes: next a at bit 0 (>>), next b at bit 31 (<<)
  uint32_t Anr, Bnr;              // raw codes of the next reservoir refill (16 bases each)
  uint32_t cm;                    // ~0: b complemented
  int64_t sa, sb; int da, db;
  int m, n, K0, ia0, jb0;
  int istar, dstar, dbase;        // argmax cell (istar, dstar - istar); best is derived from thrN (pk_best)
  int dneed;                      // the window can hold cells beyond the matrix from anti-diagonal dneed + 1
  int thrD1, thrD, thrN;          // W-space thresholds of anti-diagonals d-1, d and d+1
  int minL1, maxL1, minL2, maxL2;
  int cells;                      // < 2^19 anti-diagonals x 32 cells
  int item;
  bool active;
  int lastH, lasti, lastd;        // compat mode (Q29): H + BIAS, i and d of the last live anti-diagonal's maximum
};

// key bits of a cell: 31 - t with t the cell's index in the whole window when the window has at
// most 32 cells (then the key maximum over the group is also the argmax), else its index in the
// lane (wider groups extend the key with the lane: see pk_diag)
__device__ __forceinline__ bool pk_global_keys(int G, int C) { return G * C <= 32; }
__device__ __forceinline__ int pk_key_base(int G, int C, int gl) { return pk_global_keys(G, C) ? 31 - C * gl : 31; }

// best (H + BIAS) after anti-diagonal d from the threshold of d + 1: the X-drop threshold IS the best
// score so far minus X (reading Q2: thr_{d+1} = best_{<=d} - X), and thrN holds it in W space,
// W = H + BIAS - g (d + 1 - dbase); so no separate best needs tracking per anti-diagonal
template <int C>
__device__ __forceinline__ int pk_best(const Band16<C>& B, int d, const Problem& P) {
  return B.thrN + P.g * (d + 1 - B.dbase) + P.X;
}
// first anti-diagonal pair (d + 1, d + 2) whose window can reach cells beyond the matrix (i > m at
// q > 2m - d - K0, j > n at q < d - K0 - 2n, q = 2t + parity in [0, 2S)): pk_step masks them then
template <int C>
__device__ __forceinline__ void pk_set_dneed(Band16<C>& B, int S) {
  B.dneed = min(B.K0 + 2 * B.n, 2 * B.m - B.K0 - 2 * S + 1);
}

// key bytes 31 - t; `zero` is an opaque 0 so the words stay in registers (PRMT operand c)
template <int C>
__device__ __forceinline__ void pk_keys(Band16<C>& B, int G, int gl, int zero) {
  constexpr int NP = C / 2;
  const int tb = pk_key_base(G, C, gl) + zero;
#pragma unroll
  for (int j = 0; j < NP / 2; ++j)
    B.TC[j] = opaque((uint32_t)(tb - 2 * j) | ((uint32_t)(tb - 2 * j - NP) << 8) |
                     ((uint32_t)(tb - 2 * j - 1) << 16) | ((uint32_t)(tb - 2 * j - 1 - NP) << 24));
}

// window + reservoirs at (ia0, jb0); `rem` blocks until the next refill
template <int C>
__device__ __forceinline__ void pk_reload(Band16<C>& B, int gl, int rem, const Problem& P) {
  const int ia = B.ia0 + C * gl, jb = B.jb0 - C * gl;
  const uint64_t aw = load32c(P.PA, B.sa, B.da, ia);
  B.A0 = plane32(aw, 0); B.A1 = plane32(aw, 1);
  const uint64_t ar = load32c(P.PA, B.sa, B.da, ia + 32);
  const uint32_t keep = (rem >= 16) ? 0xffffffffu : ((1u << (16 + rem)) - 1u);
  B.An0 = plane32(ar, 0) & keep; B.An1 = plane32(ar, 1) & keep;
  B.Anr = load16(P.PA, B.sa, B.da, ia + 48 + rem);
  const uint64_t bw = load32c(P.PB, B.sb, B.db, jb - 31);
  B.B0 = __brev(plane32(bw, 0)) ^ B.cm; B.B1 = __brev(plane32(bw, 1)) ^ B.cm;
  const uint64_t br = load32c(P.PB, B.sb, B.db, jb + 1);
  const uint32_t keepb = (rem >= 16) ? 0xffffffffu : ~((1u << (16 - rem)) - 1u);
  B.Bn0 = (__brev(plane32(br, 0)) ^ B.cm) & keepb; B.Bn1 = (__brev(plane32(br, 1)) ^ B.cm) & keepb;
  B.Bnr = load16(P.PB, B.sb, B.db, jb + 17 + rem);
}

// max over k[0..N) of packed 16-bit keys (tree of VIMNMX3.S16x2)
template <int N>
__device__ __forceinline__ uint32_t tree16(const uint32_t (&k)[N]) {
  if constexpr (N == 1) {
    return k[0];
  } else {
    constexpr int M = (N + 2) / 3;
    uint32_t t[M];
#pragma unroll
    for (int i = 0; i < M; ++i) {
      if (3 * i + 2 < N) t[i] = __vimax3_s16x2(k[3 * i], k[(3 * i + 1) % N], k[(3 * i + 2) % N]);
      else if (3 * i + 1 < N) t[i] = __vmaxs2(k[3 * i], k[(3 * i + 1) % N]);
      else t[i] = k[3 * i];
    }
    return tree16<M>(t);
  }
}

// One anti-diagonal d of parity PAR: V (parity PAR, holds d-2) is updated in place from
// N (holds d-1).  by: local cells (bit tl) beyond the matrix (i > m or j > n; 0 away from the
// edges): they compare as mismatches, so their values only fall along any path (pk_diag shows why
// they then never matter).  Returns the lane's packed key maximum; ch[] are the PRMT-mask chains.
// XW (pk_wide_kernel, G = 64 lanes over two warps): the seam of the warp's boundary lane comes from
// the other warp through shared memory (xseam; DEAD2 at the group's own edges)
template <int C, int PAR, bool FMA = (XDROP_PK_FMA != 0), bool XW = false>
__device__ __forceinline__ uint32_t pk_cells(uint32_t (&V)[C / 2], const uint32_t (&N)[C / 2], const Band16<C>& B,
                                             int G, int gl, uint32_t by, const Problem& P,
                                             uint32_t (&ch)[C > 16 ? 2 : 1], uint32_t xseam = 0) {
  constexpr int NP = C / 2, NCH = C > 16 ? 2 : 1, NPC = NP / NCH;
  const int thr_d = B.thrN;
  const uint32_t two = (uint32_t)P.keym >> (KEYSH - 1);  // 2, opaque: keeps the chains on IMAD
  const uint32_t one = two >> 1;                          // 1, opaque: keeps the adds on IMAD
  (void)one;
  // per-anti-diagonal scalars on the FMA pipe (IMAD with opaque constants; the ALU pipe is the
  // binding one): D1 = 32 (thrD - thr_d) < 0, Ev = 32 (thrD1 - thrD), s' + D2 - D1 = pk + Ev
  const int k32 = (int)(two << 4), k65536 = (int)(two << 15), k65537 = k65536 + (int)one;
  const int D1 = B.thrD * k32 - thr_d * k32;
  const int Ev = B.thrD1 * k32 - B.thrD * k32;
  const int sM = Ev * (int)one + P.pkM, sU = Ev * (int)one + P.pkU;   // match / mismatch
  // packed pairs: (x, x) = x * 65537 (+ 2^16 when x < 0: the borrow of the low half)
  const int negM = (int)__umulhi((uint32_t)sM, two), negU = (int)__umulhi((uint32_t)sU, two);
  const uint32_t base = (uint32_t)(sM * k65537 + negM * k65536);
  // sE = base + bits * kk, bits = (mismatch(lo), mismatch(hi) << 16); the 2^16 terms undo the
  // borrows of negative low halves (the hi-half product drops them mod 2^32)
  const uint32_t kk = (uint32_t)((negU - negM) * k65536 + (P.pkU - P.pkM));
  const uint32_t D1p = (uint32_t)(D1 * k65537 + k65536);
  uint32_t mis = (B.A0 ^ B.B0) | ((B.A1 ^ B.B1) | by);   // bit tl: local cell tl compares unequal bases
  if constexpr (NP < 16) {                                // hi cells (tl >= NP) to bits 16..
    constexpr uint32_t LO = (1u << NP) - 1u;
    mis = (mis & LO) | ((mis << (16 - NP)) & (LO << 16));
  }
  // seam pair: the neighbour cell beyond the lane's last (first) cell
  uint32_t seam;
  if constexpr (PAR == 0) {
    uint32_t x = pk::DEAD2;
    if constexpr (XW) { x = __shfl_up_sync(FULL, N[NP - 1], 1); if ((gl & 31) == 0) x = xseam; }
    else if (G > 1) { x = __shfl_up_sync(FULL, N[NP - 1], 1, G); if (gl == 0) x = pk::DEAD2; }
    seam = __byte_perm(N[NP - 1], x, 0x1076);            // (left lane's last odd cell, own odd cell NP-1)
  } else {
    uint32_t x = pk::DEAD2;
    if constexpr (XW) { x = __shfl_down_sync(FULL, N[0], 1); if ((gl & 31) == 31) x = xseam; }
    else if (G > 1) { x = __shfl_down_sync(FULL, N[0], 1, G); if (gl == G - 1) x = pk::DEAD2; }
    seam = __byte_perm(N[0], x, 0x5432);                 // (own even cell NP, right lane's even cell 0)
  }
  // the hi half of a seam pair may hold a cell with key bits up to 31 (the next lane's cell 0);
  // clear them so the FMA-pipe adds' carries (see below) cannot reach its value bits
  if (G > 1 && FMA) seam &= 0xFFE0FFFFu;
#pragma unroll
  for (int c = 0; c < NCH; ++c) ch[c] = 0;
#pragma unroll
  for (int u = 0; u < NP; ++u) {
    uint32_t L, R;
    if constexpr (PAR == 0) {
      L = (u == 0) ? seam : N[u == 0 ? 0 : u - 1];
      R = N[u];
    } else {
      L = N[u];
      R = (u == NP - 1) ? seam : N[u == NP - 1 ? 0 : u + 1];
    }
    const uint32_t sh = (u == 0) ? mis : __umulhi(mis, 1u << (32 - u));
    const uint32_t sE = (sh & 0x00010001u) * kk + base;
    uint32_t v;
    if constexpr (FMA) {
    // the two adds as 32-bit IMADs (FMA pipe) instead of 16x2 ALU ops: a carry out of the low
    // half adds 1 to the high half, i.e. to the key bits of a hi cell (31 - t <= 31 - NP <= 27),
    // at most +2 over both adds, so it never reaches the value bits; the kill rewrites the keys
    const uint32_t X2 = V[u] * one + sE;
    v = __vimax3_s16x2(L, R, X2);
    v = v * one + D1p;
    } else {
    const uint32_t nb = __vmaxs2(L, R);
    v = __viaddmax_s16x2(V[u], sE, nb);
    v = __viaddmax_s16x2(v, D1p, pk::NOFLOOR);
    }
    // [31-t(lo), sign(lo) x 8, 31-t(hi), sign(hi) x 8]
    const uint32_t m = prmt(v, B.TC[u >> 1], (u & 1) ? 0xB796u : 0xB594u);
    v = lop_kill(v, m, pk::KILLC);
    V[u] = v;
    ch[u / NPC] = ch[u / NPC] * two + m;
  }
  return tree16<NP>(V);
}

// dead bits of the lane (local cell tl at bit C-1-tl) from the mask chains
template <int C>
__device__ __forceinline__ uint32_t pk_dead(const uint32_t (&ch)[C > 16 ? 2 : 1], const uint32_t (&chc)[C > 16 ? 2 : 1]) {
  constexpr int NP = C / 2, NPC = C > 16 ? NP / 2 : NP;
  if constexpr (C == 32) {
    const uint32_t y0 = ((ch[0] - chc[0]) >> 8) * pk::INV255;   // [A8, 0, B8, -]: cells 0-7, 16-23
    const uint32_t y1 = ((ch[1] - chc[1]) >> 8) * pk::INV255;   //                 cells 8-15, 24-31
    return __byte_perm(y0, y1, 0x0426);
  } else if constexpr (C > 16) {
    const uint32_t y0 = ((ch[0] - chc[0]) >> 8) * pk::INV255;
    const uint32_t y1 = ((ch[1] - chc[1]) >> 8) * pk::INV255;
    return ((y0 & 0xffu) << (C - NPC)) | ((y1 & 0xffu) << (C - 2 * NPC)) | (((y0 >> 16) & 0xffu) << NPC) |
           ((y1 >> 16) & 0xffu);
  } else {
    const uint32_t y = ((ch[0] - chc[0]) >> 8) * pk::INV255;    // [A, 0, B, -]: A bit NP-1-u: cell u
    return ((y & 0xffu) << NP) | ((y >> 16) & 0xffu);
  }
}

// REDUX: G = 32 groups reduce with CREDUX (one instruction each); the shared kernel's run-time-G
// loop passes false so that its single instance carries no second reduction path (code size, I$).
// by / byr: the cells beyond the matrix, bit tl / bit C-1-tl (pk_beyond; 0 away from the edges).
// A cell beyond the matrix never feeds a cell inside it (its predecessors have i' <= i, j' <= j) and,
// comparing as a mismatch, lies below the real cell it descends from, hence below best_{<d}: it can
// neither raise the threshold nor become the argmax, and byr drops it from the live extents -- the
// same result as masking it dead, for a few instructions per anti-diagonal near the edges only.
// CP (compat mode, XDROP_FLAG_SEQAN_COMPAT; Q28-Q30): (a) a pure-gap cell lives only
// strictly above the threshold.  Its W is the constant BIAS + g dbase (H = d g), the threshold in W
// space rises by >= |g| per anti-diagonal, so the rules differ on at most the one anti-diagonal whose
// threshold equals that constant: there the edge cells (value bits 0) are killed and the lane's key
// maximum and live bits are recomputed from its cells.  (b) the last live anti-diagonal's maximum
// is kept (lastH / lasti / lastd) and reported instead of the best cell.
template <int C, int PAR, bool REDUX = true, bool CP = false>
__device__ __forceinline__ void pk_diag(Band16<C>& B, int G, int gl, int d, uint32_t by, uint32_t byr,
                                        const Problem& P, const uint32_t (&chc)[C > 16 ? 2 : 1]) {
  constexpr int NP = C / 2;
  uint32_t ch[C > 16 ? 2 : 1];
  uint32_t kk;
  if constexpr (PAR == 0) kk = pk_cells<C, 0>(B.E, B.O, B, G, gl, by, P, ch);
  else kk = pk_cells<C, 1>(B.O, B.E, B, G, gl, by, P, ch);
  const int thr_d = B.thrN;
  bool fixed = false;
  uint32_t lbfix = 0;
  if constexpr (CP) {
    if (__any_sync(FULL, B.active && thr_d == BIAS + P.g * B.dbase)) {
      fixed = true;
      uint32_t (&V)[NP] = PAR == 0 ? B.E : B.O;
      const int kb = pk_key_base(G, C, gl);
      const int ib = (d + B.K0 + PAR) >> 1;
      const int e0 = -ib - C * gl, e1 = d - ib - C * gl;         // local cells of i = 0 and j = 0
      int km = -32768;
#pragma unroll
      for (int u = 0; u < NP; ++u) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int tl = u + NP * h;
          int v = h ? ((int)V[u] >> 16) : (int)(int16_t)(V[u] & 0xffffu);
          if (B.active && (tl == e0 || tl == e1) && v >= 0 && (v >> 5) == 0) {
            const uint32_t dead = 0xC000u | (uint32_t)(kb - tl);
            V[u] = h ? ((V[u] & 0xffffu) | (dead << 16)) : ((V[u] & 0xffff0000u) | dead);
            v = (int)(int16_t)dead;
          }
          km = max(km, v);
          if (v >= 0) lbfix |= 1u << (C - 1 - tl);
        }
      }
      kk = ((uint32_t)km << 16) | ((uint32_t)km & 0xffffu);
    }
  }
  // key maximum over both halves: both halves of kk2 hold it; the hi half sign-extends
  const uint32_t kk2 = __vmaxs2(kk, __byte_perm(kk, 0u, 0x1032));
  const int kl = ((int)kk2) >> 16;                        // lane key: 32 * value + 31 - (local cell)
  // no live cell: kmax is a dead key (< -16128), so vrel <= -505 and neither the threshold nor best
  // can move (thrH_d = best_{<d} - X, so gv <= best - 505); no separate liveness test is needed
  const uint32_t dl = pk_dead<C>(ch, chc);
  unsigned lb = ~(dl | byr) & (C == 32 ? 0xffffffffu : ((1u << C) - 1u));
  if constexpr (CP) { if (fixed) lb = lbfix & ~byr & (C == 32 ? 0xffffffffu : ((1u << C) - 1u)); }
  const int tmin_l = (__clz(lb) - (32 - C)) + C * gl;
  const int tmax_l = (C - __ffs(lb)) + C * gl;
  const int ibase = (d + B.K0 + PAR) >> 1;
  int vrel, tst, mn, mx;
  if (G == 1) {
    vrel = kl >> 5;
    tst = 31 - (kl & 31);
    mn = lb ? ibase + tmin_l : EMIN;
    mx = lb ? ibase + tmax_l : EMAX;
  } else {
    int tmin, tmax;
    if (pk_global_keys(G, C)) {                           // window-wide keys: the max is the argmax
      const int km = gmax_rt(kl, G);
      vrel = km >> 5;
      tst = 31 - (km & 31);
      tmin = gmin_rt(lb ? tmin_l : EMIN, G);
      tmax = gmax_rt(lb ? tmax_l : EMAX, G);
    } else {
      // 32-bit group key: value, then the lowest lane, then the lowest local cell (reading Q8:
      // smallest i); the live extents travel as one 16x2 word (tmax, 0x7FFF - tmin; -1 = none)
      int K = (int)((uint32_t)(kl >> 5) << 10) | ((31 - gl) << 5) | (kl & 31);
      if (REDUX && G == 32) {                             // CREDUX: one instruction per reduction
        K = __reduce_max_sync(FULL, K);
        tmin = __reduce_min_sync(FULL, lb ? tmin_l : EMIN);
        tmax = __reduce_max_sync(FULL, lb ? tmax_l : EMAX);
      } else {
        uint32_t ex = lb ? (((uint32_t)tmax_l << 16) | (uint32_t)(0x7FFF - tmin_l)) : 0xFFFFFFFFu;
        for (int o = 1; o < G; o <<= 1) {
          K = max(K, __shfl_xor_sync(FULL, K, o));
          ex = __vmaxs2(ex, __shfl_xor_sync(FULL, ex, o));
        }
        const int hx = ((int)ex) >> 16, lx = (int)(int16_t)(ex & 0xffffu);
        tmax = hx < 0 ? EMAX : hx;
        tmin = lx < 0 ? EMIN : 0x7FFF - lx;
      }
      vrel = K >> 10;
      tst = C * (31 - ((K >> 5) & 31)) + 31 - (K & 31);
    }
    mn = (tmin == EMIN) ? EMIN : ibase + tmin;
    mx = (tmax == EMAX) ? EMAX : ibase + tmax;
  }
  // ---- critical path: next threshold
  B.thrD1 = B.thrD; B.thrD = thr_d;
  B.thrN = thr_d + max(0, vrel - P.X) - P.g;
  // ---- off the critical path: argmax, hull count (garbage in inactive lanes is harmless: their
  // state is never written out).  best improves iff the anti-diagonal's maximum exceeds
  // thr_d + X = best_{<d} (strictly: reading Q8, the earliest anti-diagonal keeps a tie)
  const bool up = vrel > P.X;
  B.istar = up ? ibase + tst : B.istar;
  B.dstar = up ? d : B.dstar;
  if constexpr (CP) {
    // the maximum over REAL cells: a cell beyond the matrix (by) cannot be best but may top an
    // anti-diagonal, so where some lane has one the key maximum is redone without them
    int vr = vrel, ts = tst;
    if (__any_sync(FULL, by != 0)) {
      const uint32_t (&V)[NP] = PAR == 0 ? B.E : B.O;
      int kr = -32768;                                   // below any 16-bit key; packs into K below
#pragma unroll
      for (int u = 0; u < NP; ++u) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int tl = u + NP * h;
          const int v = h ? ((int)V[u] >> 16) : (int)(int16_t)(V[u] & 0xffffu);
          if (!((by >> tl) & 1u)) kr = max(kr, v);
        }
      }
      if (G == 1) {
        vr = kr >> 5; ts = 31 - (kr & 31);
      } else if (pk_global_keys(G, C)) {
        const int km = gmax_rt(kr, G);
        vr = km >> 5; ts = 31 - (km & 31);
      } else {
        int K = (int)((uint32_t)(kr >> 5) << 10) | ((31 - gl) << 5) | (kr & 31);
        for (int o = 1; o < G; o <<= 1) K = max(K, __shfl_xor_sync(FULL, K, o));
        vr = K >> 10; ts = C * (31 - ((K >> 5) & 31)) + 31 - (K & 31);
      }
    }
    if (mn != EMIN) { B.lastH = thr_d + vr + P.g * (d - B.dbase); B.lasti = ibase + ts; B.lastd = d; }
  }
  // hull of anti-diagonal d (reading Q5), clamped to the matrix: lo >= 0 and hi <= d hold already
  // (live cells of d-1, d-2 are inside it), lo >= d - n and hi <= m are applied here
  const int lo = max(min(B.minL1, B.minL2 + 1), d - B.n);
  const int hi = min(max(B.maxL1, B.maxL2) + 1, B.m);
  B.cells += max(0, hi - lo + 1);
  B.minL2 = B.minL1; B.maxL2 = B.maxL1;
  B.minL1 = mn; B.maxL1 = mx;
  if constexpr (PAR == 0) {       // even -> odd: a advances
    B.A0 = __funnelshift_r(B.A0, B.An0, 1); B.A1 = __funnelshift_r(B.A1, B.An1, 1);
    B.An0 >>= 1; B.An1 >>= 1;
    B.ia0 += 1;
  } else {                        // odd -> even: b advances
    B.B0 = __funnelshift_l(B.Bn0, B.B0, 1); B.B1 = __funnelshift_l(B.Bn1, B.B1, 1);
    B.Bn0 <<= 1; B.Bn1 <<= 1;
    B.jb0 += 1;
  }
}

// cells of anti-diagonal dd beyond the matrix, for this lane: by (bit tl), byr (bit C-1-tl).
// Cell tl has i = ibase + C gl + tl: i > m for tl >= s1, j = dd - i > n for tl < s2.
template <int C>
__device__ __forceinline__ void pk_beyond(const Band16<C>& B, int gl, int dd, int par, uint32_t& by, uint32_t& byr) {
  const int ibase = ((dd + B.K0 + par) >> 1) + C * gl;
  const int s1 = min(max(B.m - ibase + 1, 0), C), s2 = min(max(dd - ibase - B.n, 0), C);
  const uint32_t ge1 = __funnelshift_lc(0u, 0xffffffffu, s1);          // bits >= s1
  const uint32_t ge2 = __funnelshift_lc(0u, 0xffffffffu, s2);          // bits >= s2
  by = ge1 | ~ge2;
  byr = ~__funnelshift_lc(0u, 0xffffffffu, C - s1) | __funnelshift_lc(0u, 0xffffffffu, C - s2);
}

// lane mode: shift the window by 2K diagonals: cell t <- cell t + K (both parities)
template <int NP, int K>
__device__ __forceinline__ void pk_shift_arr(uint32_t (&A)[NP]) {
  uint32_t T[NP];
#pragma unroll
  for (int u = 0; u < NP; ++u) {
    if constexpr (K > 0) {
      if (u + K < NP) T[u] = A[(u + K) % NP];
      else T[u] = __byte_perm(A[(u + K - NP + NP) % NP], pk::DEAD2, 0x7632);   // (old hi, dead)
    } else {
      if (u + K >= 0) T[u] = A[(u + K + NP) % NP];
      else T[u] = __byte_perm(A[(u + K + NP) % NP], pk::DEAD2, 0x1054);        // (dead, old lo)
    }
  }
#pragma unroll
  for (int u = 0; u < NP; ++u) A[u] = T[u];
}
template <int C, int K>
__device__ __forceinline__ void pk_shift_k(Band16<C>& B) {
  pk_shift_arr<C / 2, K>(B.E); pk_shift_arr<C / 2, K>(B.O);
}
template <int C>
__device__ __forceinline__ void pk_shift_n(Band16<C>& B, int s) {
  switch (s) {
    case 1: pk_shift_k<C, 1>(B); break;   case -1: pk_shift_k<C, -1>(B); break;
    case 2: pk_shift_k<C, 2>(B); break;   case -2: pk_shift_k<C, -2>(B); break;
    case 3: pk_shift_k<C, 3>(B); break;   case -3: pk_shift_k<C, -3>(B); break;
    case 4: pk_shift_k<C, 4>(B); break;   case -4: pk_shift_k<C, -4>(B); break;
    case 5: pk_shift_k<C, 5>(B); break;   case -5: pk_shift_k<C, -5>(B); break;
    case 6: pk_shift_k<C, 6>(B); break;   case -6: pk_shift_k<C, -6>(B); break;
    case 7: pk_shift_k<C, 7>(B); break;   case -7: pk_shift_k<C, -7>(B); break;
    case 8: pk_shift_k<C, 8>(B); break;   case -8: pk_shift_k<C, -8>(B); break;
    default: break;
  }
}
// group mode: shift by one cell (dir = +1: cell t <- t + 1), across the group's lanes
template <int NP>
__device__ __forceinline__ void pk_shift1(uint32_t (&A)[NP], int G, int gl, int dir) {
  const unsigned gm = gmask(G);
  if (dir > 0) {
    uint32_t x = __shfl_down_sync(gm, A[0], 1, G);
    if (gl == G - 1) x = pk::DEAD2;
    const uint32_t last = __byte_perm(A[0], x, 0x5432);
#pragma unroll
    for (int u = 0; u < NP - 1; ++u) A[u] = A[u + 1];
    A[NP - 1] = last;
  } else {
    uint32_t x = __shfl_up_sync(gm, A[NP - 1], 1, G);
    if (gl == 0) x = pk::DEAD2;
    const uint32_t first = __byte_perm(A[NP - 1], x, 0x1076);
#pragma unroll
    for (int u = NP - 1; u >= 1; --u) A[u] = A[u - 1];
    A[0] = first;
  }
}

// after a window shift: restore the key bits 31 - (local cell) of every pair (a shift moves lo
// cells, whose keys reach 31, into hi halves, where the FMA-pipe adds may carry into the keys)
template <int NP>
__device__ __forceinline__ void pk_rekey(uint32_t (&A)[NP], int kb) {
#pragma unroll
  for (int u = 0; u < NP; ++u)
    A[u] = (A[u] & 0xFFE0FFE0u) | (uint32_t)(kb - u) | ((uint32_t)(kb - u - NP) << 16);
}

// checkpoint in the 32-bit record format of band_save (S = G*C; d even: E holds d, O holds d-1)
template <int C, bool CP = false>
__device__ __forceinline__ void pk_save(const Band16<C>& B, int G, int gl, int d, const Esc& e, const Problem& P) {
  constexpr int NP = C / 2;
  int slot = 0;
  if (gl == 0) slot = atomicAdd(e.pool_tail, 1);
  if (G > 1) slot = __shfl_sync(gmask(G), slot, 0, G);
  if (slot >= e.cap) {
    if (gl == 0) push_item(e.fb_items, e.fb_tail, B.item);
    return;
  }
  int* rec = e.pool + (size_t)slot * e.rec_ints;
  if (gl == 0) {
    rec[0] = B.item; rec[1] = d; rec[2] = B.K0; rec[3] = B.dbase; rec[4] = B.thrN; rec[5] = pk_best(B, d, P);
    rec[6] = B.istar; rec[7] = B.dstar - B.istar; rec[8] = B.minL1; rec[9] = B.maxL1; rec[10] = B.minL2;
    rec[11] = B.maxL2; rec[12] = B.ia0; rec[13] = B.jb0; rec[14] = G * C;
    rec[15] = B.cells; rec[16] = 0; rec[REC_T] = rec_stamp();
    if constexpr (CP) { rec[REC_LAST] = B.lastH; rec[REC_LAST + 1] = B.lasti; rec[REC_LAST + 2] = B.lastd; }
  }
#pragma unroll
  for (int u = 0; u < NP; ++u) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = C * gl + u + NP * h;
      const int ve = h ? ((int)B.E[u] >> 16) : (int)(int16_t)(B.E[u] & 0xffffu);
      const int vo = h ? ((int)B.O[u] >> 16) : (int)(int16_t)(B.O[u] & 0xffffu);
      rec[HDR + 2 * t] = ve >= 0 ? B.thrD + (ve >> 5) : NEGV;
      rec[HDR + 2 * t + 1] = vo >= 0 ? B.thrD1 + (vo >> 5) : NEGV;
    }
  }
  __threadfence();
  if (G > 1) __syncwarp(gmask(G));
  if (gl == 0) push_item(e.q, e.q_tail, slot);
}

// end of a block of two anti-diagonals (as band_block_end<G, C>)
template <int C, bool CP = false>
__device__ __forceinline__ void pk_block_end(Band16<C>& B, int G, int gl, int d, int& rem, const Problem& P,
                                             int level, const Esc& esc) {
  const int S = G * C;
  if (--rem == 0) {
    rem = 16;
    if (B.active) {
      B.An0 |= even_bits16(B.Anr) << 16; B.An1 |= even_bits16(B.Anr >> 1) << 16;
      B.Bn0 |= ((__brev(even_bits16(B.Bnr)) ^ B.cm) >> 16);
      B.Bn1 |= ((__brev(even_bits16(B.Bnr >> 1)) ^ B.cm) >> 16);
      B.Anr = load16(P.PA, B.sa, B.da, B.ia0 + C * gl + 64);
      B.Bnr = load16(P.PB, B.sb, B.db, B.jb0 - C * gl + 33);
    }
  }
  if (!B.active) return;
  const bool e0 = (B.minL1 == EMIN), e1 = (B.minL2 == EMIN);
  if ((e0 && e1) || d >= B.m + B.n) {
    if (gl == 0) {
      ExtOut o; o.best = pk_best(B, d, P) - BIAS; o.istar = B.istar; o.jstar = B.dstar - B.istar; o.level = level;
      if constexpr (CP) { o.best = B.lastH - BIAS; o.istar = B.lasti; o.jstar = B.lastd - B.lasti; }   // Q29, Q30
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
  if (G == 1) {
    if (qmx >= 2 * S - 2 || qmn <= 1) {
      const int s_lo = (qmx - 2 * S + 4) >> 1;
      const int s_hi = (qmn - 2) >> 1;
      if (s_lo > s_hi) {
        pk_save<C, CP>(B, G, gl, d, esc, P);
        B.active = false;
        return;
      }
      int sh = (((qmn + qmx) >> 1) - S) >> 1;
      sh = min(max(sh, s_lo), s_hi);
      sh = min(max(sh, -8), 8);
      if (sh == 0) sh = s_lo > 0 ? s_lo : s_hi;
      pk_shift_n<C>(B, sh);
      pk_rekey<C / 2>(B.E, pk_key_base(G, C, gl)); pk_rekey<C / 2>(B.O, pk_key_base(G, C, gl));
      B.K0 += 2 * sh; B.ia0 += sh; B.jb0 -= sh;
      pk_set_dneed<C>(B, S);
      pk_reload<C>(B, gl, rem, P);
    }
  } else {
    int dir = 0;
    bool ovf = false;
    if (qmx >= 2 * S - 2) { if (qmn >= 4) dir = 1; else ovf = true; }
    else if (qmn <= 1) { if (qmx <= 2 * S - 5) dir = -1; else ovf = true; }
    if (ovf) {
      pk_save<C, CP>(B, G, gl, d, esc, P);
      B.active = false;
      return;
    }
    if (dir != 0) {
      pk_shift1<C / 2>(B.E, G, gl, dir); pk_shift1<C / 2>(B.O, G, gl, dir);
      pk_rekey<C / 2>(B.E, pk_key_base(G, C, gl)); pk_rekey<C / 2>(B.O, pk_key_base(G, C, gl));
      B.K0 += 2 * dir; B.ia0 += dir; B.jb0 -= dir;
      pk_set_dneed<C>(B, S);
      pk_reload<C>(B, gl, rem, P);
    }
  }
}

// keep W (= offset-space values of the 32-bit record format) bounded: rebase every >= 1024
// anti-diagonals.  Called from the loops' every-32-blocks branch (warp-uniform), so d - dbase stays
// below 1024 + 64: |W| and the 32-bit tiers' argmax keys W * 128 stay far inside int32.
template <int C>
__device__ __forceinline__ void pk_rebase(Band16<C>& B, int d, const Problem& P) {
  if (d - B.dbase >= 1024) {
    const int woff = -P.g * (d - B.dbase);
    B.thrD1 -= woff; B.thrD -= woff; B.thrN -= woff;
    B.dbase = d;
  }
}

// key-byte part of the PRMT-mask chains (pk_dead subtracts it)
template <int C>
__device__ __forceinline__ void pk_chain_consts(const Band16<C>& B, uint32_t (&chc)[C > 16 ? 2 : 1]) {
  constexpr int NP = C / 2, NCH = C > 16 ? 2 : 1, NPC = NP / NCH;
#pragma unroll
  for (int c = 0; c < NCH; ++c) {
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < NPC; ++j) {
      const int u = c * NPC + j;
      const uint32_t w = B.TC[u >> 1];
      s = s * 2u + ((u & 1) ? ((w >> 16) & 0xffu) | (((w >> 24) & 0xffu) << 16) : (w & 0xffu) | (((w >> 8) & 0xffu) << 16));
    }
    chc[c] = s;
  }
}

// two anti-diagonals (d+1, d+2) and the block end; the cells beyond the matrix are flagged (pk_beyond)
// only when some lane's window can reach them (d + 2 > dneed), else the masks are 0
template <int C, bool REDUX = true, bool CP = false>
__device__ __forceinline__ void pk_step(Band16<C>& B, int G, int gl, int& d, int& rem, const Problem& P, int level,
                                        const Esc& esc, const uint32_t (&chc)[C > 16 ? 2 : 1]) {
  const int d2 = d + 2;
  uint32_t by1 = 0, byr1 = 0, by2 = 0, byr2 = 0;
  if (__any_sync(FULL, B.active && d2 > B.dneed)) {
    pk_beyond<C>(B, gl, d + 1, 1, by1, byr1);
    pk_beyond<C>(B, gl, d2, 0, by2, byr2);
  }
  pk_diag<C, 1, REDUX, CP>(B, G, gl, d + 1, by1, byr1, P, chc);
  pk_diag<C, 0, REDUX, CP>(B, G, gl, d2, by2, byr2, P, chc);
  d = d2;
  pk_block_end<C, CP>(B, G, gl, d, rem, P, level, esc);
}

// tail stealing check (lane mode): once enough warps idle, checkpoint this lane's extension to
// the steal queue if it still has >= min_rem anti-diagonals ahead
template <int C, bool CP = false>
__device__ __forceinline__ void pk_steal(Band16<C>& B, int G, int gl, int d, const Steal& st, const Esc& to,
                                         const Problem& P) {
  // (the group-uniform `left` test keeps pk_save's group shuffles converged for G > 1)
  int go = 0;
  if ((threadIdx.x & 31) == 0) go = ld_volatile(st.idle) >= st.thresh;
  go = __shfl_sync(FULL, go, 0);
  if (go && B.active) {
    const int ic = (B.minL1 == EMIN) ? B.minL2 : (B.minL1 >> 1) + (B.maxL1 >> 1);
    const int left = 2 * min(B.m - ic, B.n - (d - ic));
    if (left >= st.min_rem) {
      pk_save<C, CP>(B, G, gl, d, to, P);
      B.active = false;
    }
  }
}

// anti-diagonal loop (from an even d; groups of a warp may sit at different d)
template <int C, bool CP = false>
__device__ __forceinline__ void pk_loop(Band16<C>& B, int G, int gl, int d, const Problem& P, int level,
                                        const Esc& esc, const Steal* st) {
  uint32_t chc[C > 16 ? 2 : 1];
  pk_chain_consts<C>(B, chc);
  int rem = 16, blk = 0;
  pk_reload<C>(B, gl, rem, P);
  while (__any_sync(FULL, B.active)) {
    if ((++blk & 31) == 0) {
      pk_rebase<C>(B, d, P);
      if (G == 1 && st != nullptr) {
        pk_steal<C, CP>(B, G, gl, d, *st, st->es, P);
        if (!__any_sync(FULL, B.active)) break;
      }
    }
    pk_step<C, true, CP>(B, G, gl, d, rem, P, level, esc, chc);
  }
}

template <int C>
__device__ __forceinline__ void pk_geom(Band16<C>& B, const Problem& P, int item) {
  if (item >= 0) {
    B.active = true; B.item = item;
    const Geom gm = item_geom(P, B.item);
    B.sa = gm.sa; B.sb = gm.sb; B.da = gm.da; B.db = gm.db; B.m = gm.m; B.n = gm.n;
    B.cm = (uint32_t)gm.bmask;
  } else {
    B.active = false; B.item = 0;
    B.sa = GUARD; B.sb = GUARD; B.da = 1; B.db = 1; B.m = 0; B.n = 0; B.cm = 0;
  }
}

// Group state of a fresh extension at its seed (item < 0: idle group); window S = G*C <= 32.
template <int C, bool CP = false>
__device__ __forceinline__ void pk_init_seed(Band16<C>& B, int G, int gl, int item, const Problem& P) {
  constexpr int NP = C / 2;
  const int S = G * C;
  pk_geom<C>(B, P, item);
  B.K0 = -S; B.ia0 = -S / 2; B.jb0 = S / 2 - 1;
#pragma unroll
  for (int u = 0; u < NP; ++u) { B.E[u] = pk::DEAD2; B.O[u] = pk::DEAD2; }
  // origin: d = 0, k = 0 -> even cell S/2 (lane (S/2) / C, local cell tl), relative to thrW_0 = BIAS - X
  {
    const int tl = (S / 2) % C, u0 = tl % NP, h0 = tl / NP;
    if (gl == (S / 2) / C) {
      const uint32_t v0 = (uint32_t)(32 * P.X + pk_key_base(G, C, gl) - tl) & 0xffffu;
#pragma unroll
      for (int u = 0; u < NP; ++u)
        if (u == u0) B.E[u] = h0 ? ((pk::DEAD2 & 0xffffu) | (v0 << 16)) : ((pk::DEAD2 & 0xffff0000u) | v0);
    }
  }
  B.istar = 0; B.dstar = 0; B.cells = 1; B.dbase = 0;
  if constexpr (CP) { B.lastH = BIAS; B.lasti = 0; B.lastd = 0; }
  B.thrD = BIAS - P.X; B.thrD1 = B.thrD; B.thrN = BIAS - P.X - P.g;     // best = BIAS (pk_best)
  B.minL1 = 0; B.maxL1 = 0; B.minL2 = EMIN; B.maxL2 = EMAX;
  pk_set_dneed<C>(B, S);
  if (B.active && B.m + B.n == 0) {
    if (gl == 0) {
      ExtOut o; o.best = 0; o.istar = 0; o.jstar = 0; o.level = 0; o.cells = 1; o.pad = 0;
      XDROP_CHK_ITEM(P, B.item);
      P.ext[B.item] = o;
    }
    B.active = false;
  }
}

// Run one extension per group of G lanes from its seed (item < 0: idle group).  Warp-collective.
template <int G, int C, bool CP = false>
__device__ __forceinline__ void pk_run(const Problem& P, int item, int level, const Esc& esc,
                                       const Steal* st = nullptr) {
  static_assert(G * C <= 32 && C % 4 == 0 && C / 2 <= 16, "packed window from a seed");
  const int gl = (threadIdx.x & 31) % G;
  Band16<C> B;
  pk_keys<C>(B, G, gl, P.keym >> 8);
  pk_init_seed<C, CP>(B, G, gl, item, P);
  pk_loop<C, CP>(B, G, gl, 0, P, level, esc, st);
}

// Group state from a checkpoint record (rec == nullptr: idle group) in a window of S = G*C >= the
// record's; the old window lands in the middle.  Stored values become relative to a reference T per
// anti-diagonal with every live W >= T and W - T <= X + M:  T_d = min(thrW_{d+1} + g, min live W_d),
// T_{d-1} = min(thrW_{d+1} + 2g, min live W_{d-1}) (the true thresholds satisfy
// thr_d <= thrW_{d+1} + g, thr_{d-1} <= thr_d + g, and live values exceed their threshold by at
// most X + M).  The recurrence only needs differences of the references, so any such T is exact.
// Group-local: only the lanes of this group take part (a refilling pool calls it for some groups).
template <int C, bool CP = false>
__device__ __forceinline__ void pk_resume_init(Band16<C>& B, int G, int gl, int& d, const int* rec,
                                               const Problem& P) {
  constexpr int NP = C / 2;
  const int S = G * C;
  d = 0;
  pk_geom<C>(B, P, rec ? rec[0] : -1);
  int w_e[C], w_o[C];                                    // this lane's cells: even (d), odd (d-1)
  if (rec) {
    d = rec[1];
    const int s_src = rec[14];
    const int sh = S - s_src;                            // K0' = K0 - sh (sh >= 0, even)
    B.K0 = rec[2] - sh; B.dbase = rec[3]; B.thrN = rec[4];      // rec[5] (best) follows from thrN
    B.istar = rec[6]; B.dstar = rec[6] + rec[7]; B.minL1 = rec[8]; B.maxL1 = rec[9]; B.minL2 = rec[10];
    B.maxL2 = rec[11]; B.ia0 = rec[12] - sh / 2; B.jb0 = rec[13] + sh / 2;
    B.cells = rec[15];
    if constexpr (CP) { B.lastH = rec[REC_LAST]; B.lasti = rec[REC_LAST + 1]; B.lastd = rec[REC_LAST + 2]; }
#pragma unroll
    for (int t = 0; t < C; ++t) {
      const int qe = 2 * (C * gl + t) - sh, qo = qe + 1;
      w_e[t] = (qe >= 0 && qe < 2 * s_src) ? rec[HDR + qe] : NEGV;
      w_o[t] = (qo >= 0 && qo < 2 * s_src) ? rec[HDR + qo] : NEGV;
    }
  } else {
    B.K0 = -S; B.ia0 = -S / 2; B.jb0 = S / 2 - 1; B.dbase = 0; B.thrN = 0;
    B.istar = 0; B.dstar = 0; B.cells = 0; B.minL1 = EMIN; B.maxL1 = EMAX; B.minL2 = EMIN; B.maxL2 = EMAX;
    if constexpr (CP) { B.lastH = BIAS; B.lasti = 0; B.lastd = 0; }
#pragma unroll
    for (int t = 0; t < C; ++t) { w_e[t] = NEGV; w_o[t] = NEGV; }
  }
  int me = 1 << 30, mo = 1 << 30;                        // live W > 0 (biased); dead cells are negative
#pragma unroll
  for (int t = 0; t < C; ++t) {
    if (w_e[t] > 0) me = min(me, w_e[t]);
    if (w_o[t] > 0) mo = min(mo, w_o[t]);
  }
  me = gmin_grp(me, G); mo = gmin_grp(mo, G);
  B.thrD = min(B.thrN + P.g, me);
  B.thrD1 = min(B.thrN + 2 * P.g, mo);
  pk_set_dneed<C>(B, S);
  const int kb = pk_key_base(G, C, gl);
#pragma unroll
  for (int u = 0; u < NP; ++u) {
    uint32_t e = 0, o = 0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = u + NP * h;
      const uint32_t tc = kb - t;
      const uint32_t ve = w_e[t] > 0 ? ((uint32_t)(32 * (w_e[t] - B.thrD)) | tc) & 0xffffu : 0xC000u | tc;
      const uint32_t vo = w_o[t] > 0 ? ((uint32_t)(32 * (w_o[t] - B.thrD1)) | tc) & 0xffffu : 0xC000u | tc;
      e |= ve << (16 * h); o |= vo << (16 * h);
    }
    B.E[u] = e; B.O[u] = o;
  }
}

// Resume one checkpointed extension per group (rec == nullptr: idle group).  Warp-collective.
template <int G, int C, bool CP = false>
__device__ __forceinline__ void pk_resume(const Problem& P, const int* rec, int level, const Esc& esc) {
  const int gl = (threadIdx.x & 31) % G;
  Band16<C> B;
  int d = 0;
  pk_keys<C>(B, G, gl, P.keym >> 8);
  pk_resume_init<C, CP>(B, G, gl, d, rec, P);
  pk_loop<C, CP>(B, G, gl, d, P, level, esc, nullptr);
}

// A tier of pk_merged_kernel's shared loop, read from device memory where used (rare paths), so
// the queue descriptors take no registers in the loop.
struct PkTier {
  Esc src;          // records this tier resumes (pool tiers); tier 0: the lane-steal queue
  Esc esc;          // where its extensions that outgrow the window are checkpointed
  int* head;        // claim head of src's queue
  int* done;        // ended extensions of this tier (nullptr: not counted)
  int level;        // reported level of extensions that end here
};

// take up to k claimed records (queue index h..) into the idle groups of the warp (warp-collective)
template <int C, bool CP = false>
__device__ __forceinline__ void pk_take(Band16<C>& B, int G, int gl, int& d, int& rem, const Esc& src, int h, int k,
                                        const Problem& P) {
  const int lane = threadIdx.x & 31;
  const unsigned idle = __ballot_sync(FULL, !B.active && gl == 0);
  const int rank = __popc(idle & ((1u << (lane & ~(G - 1))) - 1u));
  if (!B.active && rank < k) {                           // group-uniform
    int slot = -1;
    if (gl == 0) slot = wait_entry(src.q, h + rank);
    slot = __shfl_sync(gmask(G), slot, 0, G);
    pk_resume_init<C, CP>(B, G, gl, d, src.pool + (size_t)slot * src.rec_ints, P);
    rem = 16;
    pk_reload<C>(B, gl, rem, P);
  }
}

// One work unit of pk_merged_kernel's shared C = 32 loop, with the lanes per extension G chosen at
// run time (one instance serves every tier, so the hot code stays in the instruction cache):
//  tier 0 (fresh): 32 fresh extensions, G = 1, items[base + lane]; lane-mode tail stealing
//  tier 1, 2 (pool): a refilling resume pool (T1: G = 4, T2: G = 8): the 32/G groups start with the
//        k records of tiers[t].src at queue index h; a group whose extension ends (result written,
//        or checkpointed to tiers[t].esc) takes the next queued record at the next refill point
//        (every 8 blocks; at once when the whole warp is idle).  The records taken are added to
//        *tiers[t].done when the unit returns (after every checkpoint it wrote is published).
// Loop-carried state beyond the extension's is kept to a few registers (the loop runs at the
// 168-register cap of 3 blocks per SM, where every extra live value costs instructions).
template <int C, bool CP = false>
__device__ __forceinline__ void pk_unit(const Problem& P, int G, int t, const PkTier* tiers, const int* items,
                                        int base, int n_items, int h, int k, const Steal& st) {
  const int lane = threadIdx.x & 31, gl = lane & (G - 1);
  Band16<C> B;
  pk_keys<C>(B, G, gl, P.keym >> 8);
  uint32_t chc[C > 16 ? 2 : 1];
  pk_chain_consts<C>(B, chc);
  int d = 0, rem = 16;
  int taken = k;                                         // pool: records claimed (lane 0)
  if (t == 0) {
    const int slot = base + lane;
    pk_init_seed<C, CP>(B, 1, 0, slot < n_items ? items[slot] : -1, P);
    pk_reload<C>(B, gl, rem, P);
  } else {
    pk_resume_init<C, CP>(B, G, gl, d, nullptr, P);
    pk_take<C, CP>(B, G, gl, d, rem, tiers[t].src, h, k, P);
  }
  for (int blk = 1;; ++blk) {
    if (t != 0) {
      const bool any = __any_sync(FULL, B.active);
      if (!any || (blk & 7) == 0) {
        const unsigned idle = __ballot_sync(FULL, !B.active && gl == 0);
        int kk = 0;
        if (idle) {
          int hh = 0;
          if (lane == 0) hh = claim(tiers[t].head, tiers[t].src.q_tail, __popc(idle), true, kk);
          kk = __shfl_sync(FULL, kk, 0);
          if (kk) {
            hh = __shfl_sync(FULL, hh, 0);
            taken += kk;
            pk_take<C, CP>(B, G, gl, d, rem, tiers[t].src, hh, kk, P);
          }
        }
        if (!any && kk == 0) {
          int* done = tiers[t].done;
          if (done != nullptr) {
            __syncwarp();
            if (lane == 0) { __threadfence(); atomicAdd(done, taken); }
          }
          return;
        }
      }
    }
    if ((blk & 31) == 0) {
      pk_rebase<C>(B, d, P);
      // tail stealing: lane extensions to the 4-lane queue (tiers[0].src); endgame: a T1/T2 extension
      // with a long way to go leaves the wide C = 32 shape for the latency shape (32 lanes x 8 cells,
      // tiers[4].src) once enough warps idle.  One call site (pk_save is large)
      if (t <= 2) pk_steal<C, CP>(B, G, gl, d, st, tiers[t == 0 ? 0 : 4].src, P);
    }
    if (!__any_sync(FULL, B.active)) {
      if (t != 0) continue;                              // report and refill (or return) above
      return;
    }
    pk_step<C, true, CP>(B, G, gl, d, rem, P, tiers[t].level, tiers[t].esc, chc);
  }
}
