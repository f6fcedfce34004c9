// xdrop_pk16.cuh -- packed 16-bit lane mode of tier T0 (included by xdrop_kernels.cuh).
//
// Same operation as band_run<1, 32> (one extension per lane, a window of 32
// cells per anti-diagonal = 64 diagonals, re-centred by band shifts, exact
// checkpoints to the 32-bit tiers), but the cells of an anti-diagonal are held
// as 16 PAIRS of 16-bit values and updated with the sm_100a dynamic-programming
// instructions (VIMNMX.S16x2 / VIADDMNMX.S16x2), two cells per instruction.
//
// Layout.  Cell t (0..31) of parity p sits on diagonal K0 + 2t + p.  Pair u of
// a parity array holds cells (u, u + 16) -- lo and hi half.  With this strided
// pairing the two neighbours of every pair are again whole pairs (for even
// cells: odd pairs u-1 and u; for odd cells: even pairs u and u+1); only the
// pair at the seam needs one PRMT.
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
// accumulated by one IMAD each into a word from which the 32 dead bits of the
// anti-diagonal are decoded exactly (live extent, hull count).
//
// Range: live values are < 32 (X + M) + 32, so this mode requires X + M <= 510
// (xdrop_capi.cu falls back to the 32-bit lane mode otherwise).
#pragma once

namespace pk {
constexpr uint32_t DEAD2 = 0xC000C000u;    // a pair of dead cells
constexpr uint32_t KILLC = 0xC01FC01Fu;    // LOP3 constant: bits taken from the PRMT mask
constexpr uint32_t NOFLOOR = 0x80008000u;  // no-op third operand of VIADDMNMX
// 31 - t key bytes: TCW(j) = [31-2j, 15-2j, 30-2j, 14-2j] (pairs 2j and 2j+1, lo / hi cell)
__host__ __device__ constexpr uint32_t TCW(int j) {
  return (uint32_t)(31 - 2 * j) | ((uint32_t)(15 - 2 * j) << 8) | ((uint32_t)(30 - 2 * j) << 16) |
         ((uint32_t)(14 - 2 * j) << 24);
}
// PRMT mask of pair u with no dead cell: [31-u, 0, 15-u, 0]
__host__ __device__ constexpr uint32_t MTC(int u) { return (uint32_t)(31 - u) | ((uint32_t)(15 - u) << 16); }
// chain c (pairs 8c .. 8c+7) accumulates sum_j 2^(7-j) m(8c+j); its key-byte part:
__host__ __device__ constexpr uint32_t CHC(int c) {
  uint32_t s = 0;
  for (int j = 0; j < 8; ++j) s = s * 2u + MTC(8 * c + j);
  return s;
}
constexpr uint32_t INV255 = 0xFEFEFFu;     // 255^-1 mod 2^24
}  // namespace pk

// prmt.b32 with sign-replicating selectors (__byte_perm drops selector bit 3)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t d;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(sel));
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

struct Band16 {
  uint32_t E[16], O[16];          // even / odd cells, pair u = (cell u, cell u + 16)
  uint32_t A0, A1, B0, B1;        // bit planes: bit t <-> a[ia0 + t], b[jb0 - t] (b complemented for RC)
  uint32_t An0, An1, Bn0, Bn1;    // reservoir planes: next a at bit 0 (>>), next b at bit 31 (<<)
  uint32_t Anr, Bnr;              // raw codes of the next reservoir refill (16 bases each)
  uint32_t cm;                    // ~0: b complemented
  int64_t sa, sb; int da, db;
  int m, n, K0, ia0, jb0;
  int best, istar, jstar, dbase;  // best: H + BIAS
  int thrD1, thrD, thrN;          // W-space thresholds of anti-diagonals d-1, d and d+1
  int minL1, maxL1, minL2, maxL2;
  long long cells;
  int item;
  bool active;
};

// window + reservoirs at (ia0, jb0); `rem` blocks until the next refill
__device__ __forceinline__ void pk_reload(Band16& B, int rem, const Problem& P) {
  const int ia = B.ia0, jb = B.jb0;
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

// One anti-diagonal d of parity PAR: V (parity PAR, holds d-2) is updated in place from
// N (holds d-1).  CHECK: cells with q outside [qlo, qhi] (beyond the matrix) are dead.
template <int PAR, bool CHECK>
__device__ __forceinline__ void pk_cells(uint32_t (&V)[16], const uint32_t (&N)[16], const Band16& B, int qlo,
                                         int qhi, const Problem& P, uint32_t& kout, uint32_t& ch0, uint32_t& ch1) {
  const int thr_d = B.thrN;
  const int D1 = 32 * (B.thrD - thr_d);
  const int Ev = 32 * (B.thrD1 - B.thrD);
  const int sM = P.pkM + Ev, sU = P.pkU + Ev;            // s' + D2 - D1 for a match / a mismatch
  const uint32_t base = __byte_perm((uint32_t)sM, 0u, 0x1010);
  // sE = base + bits * kk, bits = (mismatch(lo), mismatch(hi) << 16); + 2^16 undoes the borrow
  // of a negative lo half (the hi-half product drops it mod 2^32)
  const uint32_t kk = (uint32_t)(sU - sM) + ((sU < 0 && sM >= 0) ? 0x10000u : 0u);
  const uint32_t D1p = __byte_perm((uint32_t)D1, 0u, 0x1010);
  const uint32_t mis = (B.A0 ^ B.B0) | (B.A1 ^ B.B1);     // bit t: cell t compares unequal bases
  const uint32_t two = (uint32_t)P.keym >> (KEYSH - 1);  // 2, opaque: keeps the chains on IMAD
  ch0 = 0; ch1 = 0;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    uint32_t L, R;
    if constexpr (PAR == 0) {
      L = (u == 0) ? __byte_perm(N[15], pk::DEAD2, 0x1054) : N[u == 0 ? 0 : u - 1];
      R = N[u];
    } else {
      L = N[u];
      R = (u == 15) ? __byte_perm(N[0], pk::DEAD2, 0x7632) : N[u == 15 ? 0 : u + 1];
    }
    const uint32_t nb = __vmaxs2(L, R);
    const uint32_t sh = (u == 0) ? mis : __umulhi(mis, 1u << (32 - u));
    const uint32_t sE = (sh & 0x00010001u) * kk + base;
    uint32_t v = __viaddmax_s16x2(V[u], sE, nb);
    v = __viaddmax_s16x2(v, D1p, pk::NOFLOOR);
    if constexpr (CHECK) {
      const int q0 = 2 * u + PAR, q1 = q0 + 32;
      const uint32_t cap = ((q0 >= qlo && q0 <= qhi) ? 0x7FFFu : 0x8000u) |
                           ((q1 >= qlo && q1 <= qhi) ? 0x7FFF0000u : 0x80000000u);
      v = __vmins2(v, cap);
    }
    // [31-t(lo), sign(lo) x 8, 31-t(hi), sign(hi) x 8]
    const uint32_t tcw = (u >> 1) == 0 ? pk::TCW(0) : (u >> 1) == 1 ? pk::TCW(1) : (u >> 1) == 2 ? pk::TCW(2)
                       : (u >> 1) == 3 ? pk::TCW(3) : (u >> 1) == 4 ? pk::TCW(4) : (u >> 1) == 5 ? pk::TCW(5)
                       : (u >> 1) == 6 ? pk::TCW(6) : pk::TCW(7);
    const uint32_t m = prmt(v, tcw, (u & 1) ? 0xB796u : 0xB594u);
    v = (pk::KILLC & m) | (~pk::KILLC & v & ~m);
    V[u] = v;
    if (u < 8) ch0 = ch0 * two + m;
    else ch1 = ch1 * two + m;
  }
  // argmax key tree (lo cells carry larger keys than hi cells of equal value: smaller t wins)
  uint32_t k5[6];
#pragma unroll
  for (int i = 0; i < 5; ++i) k5[i] = __vimax3_s16x2(V[3 * i], V[3 * i + 1], V[3 * i + 2]);
  k5[5] = V[15];
  kout = __vmaxs2(__vimax3_s16x2(k5[0], k5[1], k5[2]), __vimax3_s16x2(k5[3], k5[4], k5[5]));
}

template <int PAR, bool CHECK>
__device__ __forceinline__ void pk_diag(Band16& B, int d, int qlo, int qhi, const Problem& P) {
  uint32_t kk, ch0, ch1;
  if constexpr (PAR == 0) pk_cells<0, CHECK>(B.E, B.O, B, qlo, qhi, P, kk, ch0, ch1);
  else pk_cells<1, CHECK>(B.O, B.E, B, qlo, qhi, P, kk, ch0, ch1);
  const int thr_d = B.thrN;
  const int kmax = max((int)(int16_t)(kk & 0xffffu), ((int)kk) >> 16);
  const bool live = kmax >= 0;
  const int vrel = kmax >> 5;
  // ---- critical path: next threshold
  B.thrD1 = B.thrD; B.thrD = thr_d;
  B.thrN = thr_d + (live ? max(0, vrel - P.X) : 0) - P.g;
  // ---- dead bits (cell t at bit 31 - t) from the two mask chains
  const uint32_t y0 = ((ch0 - pk::CHC(0)) >> 8) * pk::INV255;   // [A8, 0, B8, -]: cells 0-7, 16-23
  const uint32_t y1 = ((ch1 - pk::CHC(1)) >> 8) * pk::INV255;   //                 cells 8-15, 24-31
  const uint32_t dbits = __byte_perm(y0, y1, 0x0426);
  const unsigned lb = ~dbits;
  const int tmin = lb ? (int)__clz(lb) : EMIN;
  const int tmax = lb ? 32 - __ffs(lb) : EMAX;
  const int ibase = (d + B.K0 + PAR) >> 1;
  const int woff = -P.g * (d - B.dbase);
  const int gv = thr_d + vrel - woff;
  const bool up = B.active && live && gv > B.best;
  const int tst = 31 - (kmax & 31);
  B.best = up ? gv : B.best;
  B.istar = up ? ibase + tst : B.istar;
  B.jstar = up ? d - ibase - tst : B.jstar;
  const int lo = max(max(0, d - B.n), min(B.minL1, B.minL2 + 1));
  const int hi = min(min(B.m, d), max(B.maxL1, B.maxL2) + 1);
  B.cells += (B.active && hi >= lo) ? (long long)(hi - lo + 1) : 0ll;
  B.minL2 = B.minL1; B.maxL2 = B.maxL1;
  B.minL1 = (tmin == EMIN) ? EMIN : ibase + tmin;
  B.maxL1 = (tmax == EMAX) ? EMAX : ibase + tmax;
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

// shift the window by 2K diagonals: cell t <- cell t + K (both parities)
template <int K>
__device__ __forceinline__ void pk_shift_arr(uint32_t (&A)[16]) {
  uint32_t T[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    if constexpr (K > 0) {
      if (u + K < 16) T[u] = A[(u + K) & 15];
      else T[u] = __byte_perm(A[(u + K - 16) & 15], pk::DEAD2, 0x7632);   // (old hi, dead)
    } else {
      if (u + K >= 0) T[u] = A[(u + K + 16) & 15];
      else T[u] = __byte_perm(A[(u + K + 16) & 15], pk::DEAD2, 0x1054);   // (dead, old lo)
    }
  }
#pragma unroll
  for (int u = 0; u < 16; ++u) A[u] = T[u];
}
template <int K>
__device__ __forceinline__ void pk_shift_k(Band16& B) { pk_shift_arr<K>(B.E); pk_shift_arr<K>(B.O); }
__device__ __forceinline__ void pk_shift_n(Band16& B, int s) {
  switch (s) {
    case 1: pk_shift_k<1>(B); break;   case -1: pk_shift_k<-1>(B); break;
    case 2: pk_shift_k<2>(B); break;   case -2: pk_shift_k<-2>(B); break;
    case 3: pk_shift_k<3>(B); break;   case -3: pk_shift_k<-3>(B); break;
    case 4: pk_shift_k<4>(B); break;   case -4: pk_shift_k<-4>(B); break;
    case 5: pk_shift_k<5>(B); break;   case -5: pk_shift_k<-5>(B); break;
    case 6: pk_shift_k<6>(B); break;   case -6: pk_shift_k<-6>(B); break;
    case 7: pk_shift_k<7>(B); break;   case -7: pk_shift_k<-7>(B); break;
    case 8: pk_shift_k<8>(B); break;   case -8: pk_shift_k<-8>(B); break;
    default: break;
  }
}

// checkpoint in the 32-bit record format of band_save (S = 32; d even: E holds d, O holds d-1)
__device__ __forceinline__ void pk_save(const Band16& B, int d, const Esc& e) {
  const int slot = atomicAdd(e.pool_tail, 1);
  if (slot >= e.cap) {
    push_item(e.fb_items, e.fb_tail, B.item);
    return;
  }
  int* rec = e.pool + (size_t)slot * e.rec_ints;
  rec[0] = B.item; rec[1] = d; rec[2] = B.K0; rec[3] = B.dbase; rec[4] = B.thrN; rec[5] = B.best;
  rec[6] = B.istar; rec[7] = B.jstar; rec[8] = B.minL1; rec[9] = B.maxL1; rec[10] = B.minL2;
  rec[11] = B.maxL2; rec[12] = B.ia0; rec[13] = B.jb0; rec[14] = 32;
  rec[15] = (int)(B.cells & 0xffffffffll); rec[16] = (int)(B.cells >> 32);
#pragma unroll
  for (int u = 0; u < 16; ++u) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int t = u + 16 * h;
      const int ve = h ? ((int)B.E[u] >> 16) : (int)(int16_t)(B.E[u] & 0xffffu);
      const int vo = h ? ((int)B.O[u] >> 16) : (int)(int16_t)(B.O[u] & 0xffffu);
      rec[HDR + 2 * t] = ve >= 0 ? B.thrD + (ve >> 5) : NEGV;
      rec[HDR + 2 * t + 1] = vo >= 0 ? B.thrD1 + (vo >> 5) : NEGV;
    }
  }
  __threadfence();
  push_item(e.q, e.q_tail, slot);
}

// end of a block of two anti-diagonals (as band_block_end<1, 32>)
__device__ __forceinline__ void pk_block_end(Band16& B, int d, int& rem, const Problem& P, int level,
                                             const Esc& esc) {
  constexpr int S = 32;
  if (d - B.dbase >= 1024) {      // keep W bounded for the 32-bit tiers' checkpoints
    const int woff = -P.g * (d - B.dbase);
    B.thrD1 -= woff; B.thrD -= woff; B.thrN -= woff;
    B.dbase = d;
  }
  if (--rem == 0) {
    rem = 16;
    if (B.active) {
      B.An0 |= even_bits16(B.Anr) << 16; B.An1 |= even_bits16(B.Anr >> 1) << 16;
      B.Bn0 |= ((__brev(even_bits16(B.Bnr)) ^ B.cm) >> 16);
      B.Bn1 |= ((__brev(even_bits16(B.Bnr >> 1)) ^ B.cm) >> 16);
      B.Anr = load16(P.PA, B.sa, B.da, B.ia0 + 64);
      B.Bnr = load16(P.PB, B.sb, B.db, B.jb0 + 33);
    }
  }
  if (!B.active) return;
  const bool e0 = (B.minL1 == EMIN), e1 = (B.minL2 == EMIN);
  if ((e0 && e1) || d >= B.m + B.n) {
    ExtOut o; o.best = B.best - BIAS; o.istar = B.istar; o.jstar = B.jstar; o.level = level;
    o.cells = B.cells; o.pad = 0;
    P.ext[B.item] = o;
    B.active = false;
    return;
  }
  int qmn = 1 << 30, qmx = -(1 << 30);
  if (!e0) { qmn = 2 * B.minL1 - d - B.K0; qmx = 2 * B.maxL1 - d - B.K0; }
  if (!e1) { qmn = min(qmn, 2 * B.minL2 - (d - 1) - B.K0); qmx = max(qmx, 2 * B.maxL2 - (d - 1) - B.K0); }
  if (qmx >= 2 * S - 2 || qmn <= 1) {
    const int s_lo = (qmx - 2 * S + 4) >> 1;
    const int s_hi = (qmn - 2) >> 1;
    if (s_lo > s_hi) {
      pk_save(B, d, esc);
      B.active = false;
      return;
    }
    int sh = (((qmn + qmx) >> 1) - S) >> 1;
    sh = min(max(sh, s_lo), s_hi);
    sh = min(max(sh, -8), 8);
    if (sh == 0) sh = s_lo > 0 ? s_lo : s_hi;
    pk_shift_n(B, sh);
    B.K0 += 2 * sh; B.ia0 += sh; B.jb0 -= sh;
    pk_reload(B, rem, P);
  }
}

// Run one extension per lane from its seed (item < 0: idle lane).  Warp-collective.
__device__ __forceinline__ void pk_run(const Problem& P, int item, int level, const Esc& esc,
                                       const Steal* st = nullptr) {
  constexpr int S = 32;
  Band16 B;
  if (item >= 0) {
    B.active = true; B.item = item;
    const Geom gm = item_geom(P, B.item);
    B.sa = gm.sa; B.sb = gm.sb; B.da = gm.da; B.db = gm.db; B.m = gm.m; B.n = gm.n;
    B.cm = (uint32_t)gm.bmask;
  } else {
    B.active = false; B.item = 0;
    B.sa = GUARD; B.sb = GUARD; B.da = 1; B.db = 1; B.m = 0; B.n = 0; B.cm = 0;
  }
  B.K0 = -S; B.ia0 = -S / 2; B.jb0 = S / 2 - 1;
#pragma unroll
  for (int u = 0; u < 16; ++u) { B.E[u] = pk::DEAD2; B.O[u] = pk::DEAD2; }
  // origin: d = 0, k = 0 -> even cell 16 = hi half of pair 0, relative to thrW_0 = BIAS - X
  B.E[0] = (pk::DEAD2 & 0xffffu) | ((uint32_t)(32 * P.X + 15) << 16);
  B.best = BIAS; B.istar = 0; B.jstar = 0; B.cells = 1; B.dbase = 0;
  B.thrD = BIAS - P.X; B.thrD1 = B.thrD; B.thrN = BIAS - P.X - P.g;
  B.minL1 = 0; B.maxL1 = 0; B.minL2 = EMIN; B.maxL2 = EMAX;
  int rem = 16;
  pk_reload(B, rem, P);
  if (B.active && B.m + B.n == 0) {
    ExtOut o; o.best = 0; o.istar = 0; o.jstar = 0; o.level = level; o.cells = 1; o.pad = 0;
    P.ext[B.item] = o;
    B.active = false;
  }
  int d = 0, blk = 0;
  while (__any_sync(FULL, B.active)) {
    if (st != nullptr && ((++blk & 31) == 0)) {
      int go = 0;
      if ((threadIdx.x & 31) == 0) go = ld_volatile(st->idle) >= st->thresh;
      go = __shfl_sync(FULL, go, 0);
      if (go && B.active) {
        const int ic = (B.minL1 == EMIN) ? B.minL2 : (B.minL1 >> 1) + (B.maxL1 >> 1);
        const int left = 2 * min(B.m - ic, B.n - (d - ic));
        if (left >= st->min_rem) {
          pk_save(B, d, st->es);
          B.active = false;
        }
      }
      if (!__any_sync(FULL, B.active)) break;
    }
    const int d2 = d + 2;
    const bool need = B.active && (d2 - B.K0 - 2 * B.n > 0 || 2 * B.m - d2 - B.K0 < 2 * S - 1);
    if (__any_sync(FULL, need)) {
      pk_diag<1, true>(B, d + 1, d + 1 - B.K0 - 2 * B.n, 2 * B.m - (d + 1) - B.K0, P);
      pk_diag<0, true>(B, d2, d2 - B.K0 - 2 * B.n, 2 * B.m - d2 - B.K0, P);
    } else {
      pk_diag<1, false>(B, d + 1, 0, 0, P);
      pk_diag<0, false>(B, d2, 0, 0, P);
    }
    d = d2;
    pk_block_end(B, d, rem, P, level, esc);
  }
}
