// xdrop_pkwide.cuh -- the S = 2048 level in the packed 16-bit mode (included by xdrop_kernels.cuh).
//
// One extension per block of TWO warps: 64 lanes x 32 cells = 2048 cells per anti-diagonal, the
// cells as packed 16-bit pairs exactly as in xdrop_pk16.cuh (pk_cells, pk_dead, pk_beyond, the same
// relative-to-threshold values, keys and checkpoint format).  What crosses the warp boundary goes
// through shared memory, once per anti-diagonal, together with the block-wide reductions:
//  * the seam cell: after an odd anti-diagonal warp 0's lane 31 publishes its last odd pair, after an
//    even one warp 1's lane 0 its first even pair (each is read by the other warp's boundary lane on
//    the next anti-diagonal; double-buffered by parity, so one barrier per anti-diagonal suffices);
//  * the group key (value, lane, cell) and the live extents: CREDUX per warp, then the two warps;
//  * window shifts, checkpoint slots and the resume minima (rare).
// It replaces the 32-bit band_cta_kernel<128, 16> (4 warps x 16 cells, one extension per 4-warp
// block) for packed batches (X + M <= 510): half the ALU work per cell, and six blocks per SM
// instead of three, so the level's extensions (X-sweep X = 100: ~900) run in one wave.
#pragma once

namespace pkw {
constexpr int G = 64;           // lanes of the group (two warps); C cells per lane is a template parameter
}

struct PkWideShared {
  uint32_t edge[2][2];     // [parity of the anti-diagonal just computed][warp]: boundary value
  int red[2][2][3];        // [parity][warp]: group key, min live cell, max live cell
  int tmp[2][2];           // block minima / shift hand-over
  uint32_t sh[2][2];       // window shift: [warp][array E/O] boundary values
  int q;                   // claimed queue index / checkpoint slot
  int redc[2][2];          // compat mode: [parity][warp] group key over real cells
};

// minima of a, b over the block (64 threads)
__device__ __forceinline__ void pkw_min2(int& a, int& b, PkWideShared& sm) {
  a = __reduce_min_sync(FULL, a);
  b = __reduce_min_sync(FULL, b);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sm.tmp[w][0] = a; sm.tmp[w][1] = b; }
  __syncthreads();
  a = min(sm.tmp[0][0], sm.tmp[1][0]);
  b = min(sm.tmp[0][1], sm.tmp[1][1]);
  __syncthreads();
}

// group state from a checkpoint record of a narrower window (pk_resume_init for the 2-warp group)
template <int C, bool CP = false>
__device__ __forceinline__ void pkw_resume_init(Band16<C>& B, int gl, int& d, const int* rec, const Problem& P,
                                                PkWideShared& sm) {
  using pkw::G;
  constexpr int NP = C / 2, S = G * C;
  pk_geom<C>(B, P, rec[0]);
  d = rec[1];
  const int s_src = rec[14];
  const int shv = S - s_src;                             // K0' = K0 - shv (even)
  B.K0 = rec[2] - shv; B.dbase = rec[3]; B.thrN = rec[4];
  B.istar = rec[6]; B.dstar = rec[6] + rec[7]; B.minL1 = rec[8]; B.maxL1 = rec[9]; B.minL2 = rec[10];
  B.maxL2 = rec[11]; B.ia0 = rec[12] - shv / 2; B.jb0 = rec[13] + shv / 2;
  B.cells = rec[15];
  if constexpr (CP) { B.lastH = rec[REC_LAST]; B.lasti = rec[REC_LAST + 1]; B.lastd = rec[REC_LAST + 2]; }
  int w_e[C], w_o[C];
#pragma unroll
  for (int t = 0; t < C; ++t) {
    const int qe = 2 * (C * gl + t) - shv, qo = qe + 1;
    w_e[t] = (qe >= 0 && qe < 2 * s_src) ? rec[HDR + qe] : NEGV;
    w_o[t] = (qo >= 0 && qo < 2 * s_src) ? rec[HDR + qo] : NEGV;
  }
  int me = 1 << 30, mo = 1 << 30;
#pragma unroll
  for (int t = 0; t < C; ++t) {
    if (w_e[t] > 0) me = min(me, w_e[t]);
    if (w_o[t] > 0) mo = min(mo, w_o[t]);
  }
  pkw_min2(me, mo, sm);
  B.thrD = min(B.thrN + P.g, me);
  B.thrD1 = min(B.thrN + 2 * P.g, mo);
  pk_set_dneed<C>(B, S);
  const int kb = pk_key_base(G, C, gl);                  // 31: keys are local (non-global)
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

// one anti-diagonal d of parity PAR for the 2-warp group (pk_diag with G = 64)
// CP: the compat mode's last-anti-diagonal maximum over real cells (pk_diag's Q29 part; the Q28
// edge rule cannot apply here: an extension reaches this level only after d >= 1,023 > X / |g| + 1)
template <int C, int PAR, bool CP = false>
__device__ __forceinline__ void pkw_diag(Band16<C>& B, int gl, int d, uint32_t by, uint32_t byr,
                                         const Problem& P, const uint32_t (&chc)[C > 16 ? 2 : 1], PkWideShared& sm) {
  using pkw::G;
  constexpr int NP = C / 2;
  const int w = gl >> 5, lane = gl & 31;
  // the other warp's boundary value of anti-diagonal d-1 (DEAD2 at the group's own edges)
  uint32_t xs = pk::DEAD2;
  if (PAR == 1 && w == 0) xs = sm.edge[0][1];            // warp 1 lane 0's even pair 0
  if (PAR == 0 && w == 1) xs = sm.edge[1][0];            // warp 0 lane 31's odd pair NP-1
  uint32_t ch[C > 16 ? 2 : 1];
  uint32_t kk;
  if constexpr (PAR == 0) kk = pk_cells<C, 0, (XDROP_PK_FMA != 0), true>(B.E, B.O, B, G, gl, by, P, ch, xs);
  else kk = pk_cells<C, 1, (XDROP_PK_FMA != 0), true>(B.O, B.E, B, G, gl, by, P, ch, xs);
  if constexpr (PAR == 1) { if (gl == 31) sm.edge[1][0] = B.O[NP - 1]; }
  else { if (gl == 32) sm.edge[0][1] = B.E[0]; }
  const int thr_d = B.thrN;
  const uint32_t kk2 = __vmaxs2(kk, __byte_perm(kk, 0u, 0x1032));
  const int kl = ((int)kk2) >> 16;
  const uint32_t dl = pk_dead<C>(ch, chc);
  const unsigned lb = ~(dl | byr) & (C == 32 ? 0xffffffffu : ((1u << C) - 1u));
  const int tmin_l = (__clz(lb) - (32 - C)) + C * gl;
  const int tmax_l = (C - __ffs(lb)) + C * gl;
  // group key: value, then the lowest lane, then the lowest local cell (reading Q8: smallest i)
  int K = (int)((uint32_t)(kl >> 5) << 11) | ((63 - gl) << 5) | (kl & 31);
  K = __reduce_max_sync(FULL, K);
  int tmin = __reduce_min_sync(FULL, lb ? tmin_l : EMIN);
  int tmax = __reduce_max_sync(FULL, lb ? tmax_l : EMAX);
  if (lane == 0) { sm.red[PAR][w][0] = K; sm.red[PAR][w][1] = tmin; sm.red[PAR][w][2] = tmax; }
  __syncthreads();
  K = max(sm.red[PAR][0][0], sm.red[PAR][1][0]);
  tmin = min(sm.red[PAR][0][1], sm.red[PAR][1][1]);
  tmax = max(sm.red[PAR][0][2], sm.red[PAR][1][2]);
  const int vrel = K >> 11;
  const int tst = C * (63 - ((K >> 5) & 63)) + 31 - (K & 31);
  const int ibase = (d + B.K0 + PAR) >> 1;
  const int mn = (tmin == EMIN) ? EMIN : ibase + tmin;
  const int mx = (tmax == EMAX) ? EMAX : ibase + tmax;
  B.thrD1 = B.thrD; B.thrD = thr_d;
  B.thrN = thr_d + max(0, vrel - P.X) - P.g;
  const bool up = vrel > P.X;
  B.istar = up ? ibase + tst : B.istar;
  B.dstar = up ? d : B.dstar;
  if constexpr (CP) {
    int vr = vrel, ts = tst;
    if (__syncthreads_or(by != 0)) {                    // block-uniform
      int kr = -32768;
#pragma unroll
      for (int u = 0; u < NP; ++u) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int tl = u + NP * h;
          const uint32_t x = PAR == 0 ? B.E[u] : B.O[u];
          const int v = h ? ((int)x >> 16) : (int)(int16_t)(x & 0xffffu);
          if (!((by >> tl) & 1u)) kr = max(kr, v);
        }
      }
      int Kr = (int)((uint32_t)(kr >> 5) << 11) | ((63 - gl) << 5) | (kr & 31);
      Kr = __reduce_max_sync(FULL, Kr);
      if (lane == 0) sm.redc[PAR][w] = Kr;
      __syncthreads();
      Kr = max(sm.redc[PAR][0], sm.redc[PAR][1]);
      vr = Kr >> 11;
      ts = C * (63 - ((Kr >> 5) & 63)) + 31 - (Kr & 31);
    }
    if (mn != EMIN) { B.lastH = thr_d + vr + P.g * (d - B.dbase); B.lasti = ibase + ts; B.lastd = d; }
  }
  const int lo = max(min(B.minL1, B.minL2 + 1), d - B.n);
  const int hi = min(max(B.maxL1, B.maxL2) + 1, B.m);
  B.cells += max(0, hi - lo + 1);
  B.minL2 = B.minL1; B.maxL2 = B.maxL1;
  B.minL1 = mn; B.maxL1 = mx;
  if constexpr (PAR == 0) {
    B.A0 = __funnelshift_r(B.A0, B.An0, 1); B.A1 = __funnelshift_r(B.A1, B.An1, 1);
    B.An0 >>= 1; B.An1 >>= 1;
    B.ia0 += 1;
  } else {
    B.B0 = __funnelshift_l(B.Bn0, B.B0, 1); B.B1 = __funnelshift_l(B.Bn1, B.B1, 1);
    B.Bn0 <<= 1; B.Bn1 <<= 1;
    B.jb0 += 1;
  }
}

// shift both parity arrays by one cell across the group (pk_shift1 with the warp boundary in smem)
template <int C>
__device__ __forceinline__ void pkw_shift1(Band16<C>& B, int gl, int dir, PkWideShared& sm) {
  constexpr int NP = C / 2;
  const int w = gl >> 5, lane = gl & 31;
  if (dir > 0) {                                          // cell t <- t + 1: lane takes the next lane's first
    if (lane == 0) { sm.sh[w][0] = B.E[0]; sm.sh[w][1] = B.O[0]; }
    __syncthreads();
    uint32_t xe = __shfl_down_sync(FULL, B.E[0], 1), xo = __shfl_down_sync(FULL, B.O[0], 1);
    if (lane == 31) {
      xe = w == 0 ? sm.sh[1][0] : pk::DEAD2;
      xo = w == 0 ? sm.sh[1][1] : pk::DEAD2;
    }
    const uint32_t le = __byte_perm(B.E[0], xe, 0x5432), lo = __byte_perm(B.O[0], xo, 0x5432);
#pragma unroll
    for (int u = 0; u < NP - 1; ++u) { B.E[u] = B.E[u + 1]; B.O[u] = B.O[u + 1]; }
    B.E[NP - 1] = le; B.O[NP - 1] = lo;
  } else {                                                // cell t <- t - 1
    if (lane == 31) { sm.sh[w][0] = B.E[NP - 1]; sm.sh[w][1] = B.O[NP - 1]; }
    __syncthreads();
    uint32_t xe = __shfl_up_sync(FULL, B.E[NP - 1], 1), xo = __shfl_up_sync(FULL, B.O[NP - 1], 1);
    if (lane == 0) {
      xe = w == 1 ? sm.sh[0][0] : pk::DEAD2;
      xo = w == 1 ? sm.sh[0][1] : pk::DEAD2;
    }
    const uint32_t fe = __byte_perm(B.E[NP - 1], xe, 0x1076), fo = __byte_perm(B.O[NP - 1], xo, 0x1076);
#pragma unroll
    for (int u = NP - 1; u >= 1; --u) { B.E[u] = B.E[u - 1]; B.O[u] = B.O[u - 1]; }
    B.E[0] = fe; B.O[0] = fo;
  }
  __syncthreads();
}

// checkpoint for the next (S = 4096, 32-bit thread-block) level in the record format of pk_save
template <int C, bool CP = false>
__device__ __forceinline__ void pkw_save(const Band16<C>& B, int gl, int d, const Esc& e, const Problem& P,
                                         PkWideShared& sm) {
  constexpr int NP = C / 2, S = pkw::G * C;
  if (gl == 0) sm.q = atomicAdd(e.pool_tail, 1);
  __syncthreads();
  const int slot = sm.q;
  __syncthreads();
  if (slot >= e.cap) {
    if (gl == 0) push_item(e.fb_items, e.fb_tail, B.item);
    return;
  }
  int* rec = e.pool + (size_t)slot * e.rec_ints;
  if (gl == 0) {
    rec[0] = B.item; rec[1] = d; rec[2] = B.K0; rec[3] = B.dbase; rec[4] = B.thrN; rec[5] = pk_best(B, d, P);
    rec[6] = B.istar; rec[7] = B.dstar - B.istar; rec[8] = B.minL1; rec[9] = B.maxL1; rec[10] = B.minL2;
    rec[11] = B.maxL2; rec[12] = B.ia0; rec[13] = B.jb0; rec[14] = S;
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
  __syncthreads();
  if (gl == 0) push_item(e.q, e.q_tail, slot);
}

// S = 2048 level: persistent over the queue of S = 1024 checkpoints (from T3 or pk_resume_kernel)
#ifndef XDROP_PKW_MINBLOCKS
#define XDROP_PKW_MINBLOCKS 6
#endif
template <int C, bool CP = false>
__global__ void __launch_bounds__(64, XDROP_PKW_MINBLOCKS)
pk_wide_kernel(Problem P, Esc src, int* queue_head, Esc esc, int level) {
  using pkw::G;
  constexpr int NP = C / 2, S = G * C;
  __shared__ PkWideShared sm;
  const int gl = threadIdx.x;
  const int n = *src.q_tail;
  for (;;) {
    if (gl == 0) {
      int q = atomicAdd(queue_head, 1);
      sm.q = q < n ? wait_entry(src.q, q) : -1;
    }
    __syncthreads();
    const int slot = sm.q;
    __syncthreads();
    if (slot < 0) return;
    const int* rec = src.pool + (size_t)slot * src.rec_ints;
    Band16<C> B;
    pk_keys<C>(B, G, gl, P.keym >> 8);
    uint32_t chc[C > 16 ? 2 : 1];
    pk_chain_consts<C>(B, chc);
    int d = 0;
    pkw_resume_init<C, CP>(B, gl, d, rec, P, sm);
    int rem = 16;
    pk_reload<C>(B, gl, rem, P);
    // the boundary values the first anti-diagonal (odd, d + 1) needs: warp 1 lane 0's even pair 0
    if (gl == 32) sm.edge[0][1] = B.E[0];
    __syncthreads();
    for (int blk = 1; B.active; ++blk) {                 // B.active is uniform over the block
      if ((blk & 31) == 0) pk_rebase<C>(B, d, P);
      const int d2 = d + 2;
      uint32_t by1 = 0, byr1 = 0, by2 = 0, byr2 = 0;
      if (d2 > B.dneed) {
        pk_beyond<C>(B, gl, d + 1, 1, by1, byr1);
        pk_beyond<C>(B, gl, d2, 0, by2, byr2);
      }
      pkw_diag<C, 1, CP>(B, gl, d + 1, by1, byr1, P, chc, sm);
      pkw_diag<C, 0, CP>(B, gl, d2, by2, byr2, P, chc, sm);
      d = d2;
      // ---- block end (pk_block_end for the group)
      if (--rem == 0) {
        rem = 16;
        B.An0 |= even_bits16(B.Anr) << 16; B.An1 |= even_bits16(B.Anr >> 1) << 16;
        B.Bn0 |= ((__brev(even_bits16(B.Bnr)) ^ B.cm) >> 16);
        B.Bn1 |= ((__brev(even_bits16(B.Bnr >> 1)) ^ B.cm) >> 16);
        B.Anr = load16(P.PA, B.sa, B.da, B.ia0 + C * gl + 64);
        B.Bnr = load16(P.PB, B.sb, B.db, B.jb0 - C * gl + 33);
      }
      const bool e0 = (B.minL1 == EMIN), e1 = (B.minL2 == EMIN);
      if ((e0 && e1) || d >= B.m + B.n) {
        if (gl == 0) {
          ExtOut o; o.best = pk_best(B, d, P) - BIAS; o.istar = B.istar; o.jstar = B.dstar - B.istar;
          if constexpr (CP) { o.best = B.lastH - BIAS; o.istar = B.lasti; o.jstar = B.lastd - B.lasti; }
          o.level = level; o.cells = B.cells; o.pad = 0;
          XDROP_CHK_ITEM(P, B.item);
          P.ext[B.item] = o;
        }
        break;
      }
      int qmn = 1 << 30, qmx = -(1 << 30);
      if (!e0) { qmn = 2 * B.minL1 - d - B.K0; qmx = 2 * B.maxL1 - d - B.K0; }
      if (!e1) { qmn = min(qmn, 2 * B.minL2 - (d - 1) - B.K0); qmx = max(qmx, 2 * B.maxL2 - (d - 1) - B.K0); }
      int dir = 0;
      bool ovf = false;
      if (qmx >= 2 * S - 2) { if (qmn >= 4) dir = 1; else ovf = true; }
      else if (qmn <= 1) { if (qmx <= 2 * S - 5) dir = -1; else ovf = true; }
      if (ovf) {
        pkw_save<C, CP>(B, gl, d, esc, P, sm);
        break;
      }
      if (dir != 0) {
        pkw_shift1<C>(B, gl, dir, sm);
        pk_rekey<NP>(B.E, pk_key_base(G, C, gl)); pk_rekey<NP>(B.O, pk_key_base(G, C, gl));
        B.K0 += 2 * dir; B.ia0 += dir; B.jb0 -= dir;
        pk_set_dneed<C>(B, S);
        pk_reload<C>(B, gl, rem, P);
        // the shifted even pair 0 of warp 1 lane 0 is what the next odd anti-diagonal reads
        if (gl == 32) sm.edge[0][1] = B.E[0];
        __syncthreads();
      }
    }
    __syncthreads();
  }
}
