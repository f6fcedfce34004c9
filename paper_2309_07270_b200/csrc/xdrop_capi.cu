// xdrop_capi.cu -- host runtime and C ABI of libxdrop.so (include/xdrop.h).
//
// Layers: L2 per-device runtime (workspaces, streams, the
// device pipeline pack -> prep/sort -> band levels -> combine), L3 multi-GPU
// scheduler (sched.h: CELLS sharding + the paper's one2all / one2one /
// opt_one2one policies, §III), L4 the C ABI.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <thread>
#include <vector>

#include "../../include/xdrop.h"
#include "sched.h"
#include "xdrop_kernels.cuh"

namespace {

using xk::ExtOut;
using xk::PairDesc;

// ----------------------------------------------------------------- device ctx
struct Buf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return 0;
    if (p) cudaFree(p);
    p = nullptr; cap = 0;
    size_t want = std::max<size_t>(bytes, 256);
    want = want + want / 4;
    if (cudaMalloc(&p, want) != cudaSuccess) { cudaGetLastError(); return XDROP_ENOMEM; }
    cap = want;
    return 0;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
  void release() { if (p) cudaFree(p); p = nullptr; cap = 0; }
};

struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  int ensure(size_t bytes) {
    if (bytes <= cap) return 0;
    if (p) cudaFreeHost(p);
    p = nullptr; cap = 0;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) { cudaGetLastError(); return XDROP_ENOMEM; }
    cap = bytes;
    return 0;
  }
  void release() { if (p) cudaFreeHost(p); p = nullptr; cap = 0; }
};

// counters block layout (ints)
enum { C_NITEMS = 0, C_HEAD0, C_DONE0, C_HEADL, C_NLONG,   // T0 queues
       C_P1, C_Q1T, C_Q1H, C_DONE1,                         // T1 record pool / queue
       C_P2, C_Q2T, C_Q2H,                                  // T2
       C_P3, C_Q3T, C_HEAD3, C_DONE2,                       // S = 1024 (launch, or T3 of the shared kernel)
       C_P4, C_Q4T, C_HEAD4,                                // CTA launch (S = 2048)
       C_P5, C_Q5T, C_HEAD5,                                // CTA launch (S = 4096)
       C_GEN, C_HEADG, C_HEADW,
       C_IDLE, C_SP, C_ST, C_SH, C_DONES,                   // tail stealing
       C_TLN,                                               // timeline records
       C_ZERO,                                              // always 0 (an empty queue's tail)
       C_WP, C_WT, C_WH, C_WD,                              // endgame steals of the shared kernel
       C_PROBE, C_PROBEFB,                                  // per-batch kernel probe: overflows, list tail
       C_MAXM,                                              // longest A-side extension (unbounded path stride)
       C_RINGO, C_HEADRW,                                   // compat: ring-kernel overflows, wide-ring head
       C_GRPO, C_HEADGRP,                                   // compat: group-kernel overflows, ring-kernel head
       C_N };
constexpr int kTimelineCap = 1 << 16;
// Per-batch choice of the packed kernel: the shared kernel when the batch's probe
// (pk_probe_kernel: kProbe evenly spaced extensions run for at most 2 * kProbeCap anti-diagonals in
// the T0 window) predicts at least kSharedT1 T0 -> T1 checkpoints for the whole batch (escalated
// work is then a large or long-running part of it: the shared kernel's T1/T2 pools, endgame steals
// and in-kernel S = 1024 tier beat the tiered kernel's per-tier loops), else the tiered kernel.
constexpr int64_t kSharedT1 = 1024;
constexpr int kGenWideSmem = 3 * xk::kGenRingWide * (int)sizeof(int);   // general_wide_kernel's rings
constexpr int kProbe = 4096;
constexpr int kProbeCap = 64;
// host mirror of the small readbacks (ints): counters at 0, bad flags at HS_BAD, level sums at HS_LVL
enum { HS_BAD = 64, HS_LVL = 80, HS_BYTES = 512 };
static_assert(int(C_N) <= int(HS_BAD) && HS_LVL + 16 <= HS_BYTES / 4, "host mirror layout: counters, bad flags, level sums");

__global__ void init_counters_kernel(int* c, int n_items) {
  for (int i = threadIdx.x; i < C_N; i += blockDim.x) c[i] = (i == C_NITEMS) ? n_items : 0;
}
__global__ void init_bad_kernel(unsigned long long* bad) {
  if (threadIdx.x < 2) bad[threadIdx.x] = ~0ull;
}

struct DevCtx {
  int dev = 0;
  int sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int occ_l0 = 1, occ_l1 = 1, occ_l2 = 1, occ_gen = 1, occ_ring = 1, occ_ringw = 1, occ_grp = 1, occ_m = 1, occ_pk = 1, occ_pkm = 1, occ_pk8 = 1, occ_pkm8 = 1, occ_pk2 = 1, occ_pkw = 1, occ_cta = 1, occ_cta1k = 1, occ_cta2k = 1;
  int shared_t3 = 1;          // shared kernel resumes S1024 records itself (XDROP_SHARED_T3=0: the CTA launch)
  int wide_pk = 1;            // S = 2048 level in the packed 2-warp kernel (XDROP_WIDE_PK=0: 32-bit CTA)
  int s1024 = 0;              // S1024 level after the band kernel: 0 warp 32x32, 1 CTA<128,8> (XDROP_S1024;
                              // measured slower: X-sweep X=50 59 -> 95 ms, the per-anti-diagonal barrier)
  int long_g = -1;         // lanes per long extension: -1 per call (4 below X = 32, 8 from it: DESIGN.md
                           // §7), XDROP_LONG_G fixes it (0 disables the long mode, 2, 4 or 8)
  float long_alpha = 2.0f; // long cut (XDROP_LONG_ALPHA; 2 measured best: E. coli 12.2 -> 11.7 ms vs 1, X-sweep and
                           // C. elegans within 1%)
  int steal_div = 8;         // stealing starts once resident warps / steal_div are idle (XDROP_STEAL_DIV)
  int steal_min = 1024;     // tail stealing: min anti-diagonals left (XDROP_STEAL_MIN; 0 disables)
  double compat_grp = 0.05;  // compat mode: warp rings first when this fraction of the probe overflows (XDROP_COMPAT_GRP)
  int compat_first = 0;      // compat mode's first kernel: 0 per batch, 1 group, 2 warp ring (XDROP_COMPAT_FIRST)
  bool compat_general = false;   // compat mode in the general path only, also when packed (XDROP_COMPAT_GENERAL)
  bool timeline = false;    // XDROP_TIMELINE: record the merged kernel's work units
  int kernel_env = 0;        // XDROP_KERNEL: 1 tiered, 2 shared, 0 per batch (probe)
  int probe_thr = 0;         // last packed call: probe threshold (0: shared forced, 2^30: tiered forced)
  int probe_choice = 0;      // last packed call: 0 probe decided, 1 tiered forced, 2 shared forced
  int age_us = 20;           // T1/T2 batch claims go partial once the oldest record waited this long (XDROP_AGE_US)
  int idle_ns = 16000;       // max poll period (exponential backoff) of escalation-only warps (XDROP_IDLE_NS)
  int t0_per_sm = 0;         // packed kernels: resident blocks per SM that take T0 work (the rest: escalations;
                             // 0: default -- all 3 of the tiered kernel, 2 of the shared kernel's 3)
  bool pk16 = true;          // packed 16-bit lane mode for T0 (XDROP_PK16=0: 32-bit lane mode)
  float endgame = 0.0f;     // endgame: T0 items left < endgame x resident lanes (XDROP_ENDGAME; off: measured no gain)
  // device workspaces
  Buf asciiA, asciiB, offA, offB, packA, packB, pairs, wcost, hist, cursor, items, ovf1, ovf2, ovf3,
      counters, bad, ext, out5, cells, scratch, level_acc, pool1, pool2, pool3, pool4, q4, pool5, q5, genl, pools, qs, tl, smcnt, ms_pairs, ms_res, ms_best, escbuf, poolw, qw, probe, ringo, grpo;
  xk::PkTier tier_host[5];          // staging of the shared packed kernel's tier descriptors (escbuf)
  // host staging (pinned)
  HostBuf h_small, h_pairs, h_res;
  cudaEvent_t ev[12] = {};
  xdrop_stats st{};
  int64_t err_index = -1;
};

int cuda_err(cudaError_t e) {
  if (e == cudaSuccess) return 0;
  if (e == cudaErrorMemoryAllocation) return XDROP_ENOMEM;
  return XDROP_ECUDA;
}

#define CK(x) do { int _r = cuda_err(x); if (_r) return _r; } while (0)
#define CKR(x) do { int _r = (x); if (_r) return _r; } while (0)

int dev_open(DevCtx& D, int dev) {
  D.dev = dev;
  CK(cudaSetDevice(dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  D.sms = prop.multiProcessorCount;
  CK(cudaStreamCreateWithFlags(&D.stream, cudaStreamNonBlocking));
  D.own_stream = true;
  for (auto& e : D.ev) CK(cudaEventCreate(&e));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_l0, xk::band_kernel<1, 32>, 128, 0));
  if (const char* e = getenv("XDROP_LONG_G")) D.long_g = atoi(e);
  if (const char* e = getenv("XDROP_LONG_ALPHA")) D.long_alpha = (float)atof(e);
  if (const char* e = getenv("XDROP_STEAL_MIN")) D.steal_min = atoi(e);
  if (const char* e = getenv("XDROP_STEAL_DIV")) D.steal_div = std::max(1, atoi(e));
  if (const char* e = getenv("XDROP_COMPAT_GRP")) D.compat_grp = atof(e);
  if (const char* e = getenv("XDROP_COMPAT_FIRST")) D.compat_first = atoi(e);
  if (const char* e = getenv("XDROP_COMPAT_GENERAL")) D.compat_general = atoi(e) != 0;
  D.timeline = getenv("XDROP_TIMELINE") != nullptr;
  if (const char* e = getenv("XDROP_ENDGAME")) D.endgame = (float)atof(e);
  if (const char* e = getenv("XDROP_PK16")) D.pk16 = atoi(e) != 0;
  if (D.long_g != -1 && D.long_g != 0 && D.long_g != 2 && D.long_g != 4 && D.long_g != 8) D.long_g = -1;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_pk8, xk::pk_tiered_kernel<8, 4>, 128, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_pkm8, xk::pk_merged_kernel<8, 4>, 128, 0));
  D.occ_pk8 = std::max(1, D.occ_pk8);
  D.occ_pkm8 = std::max(1, D.occ_pkm8);
  if (D.long_g == 2) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_m, xk::band_merged_kernel<32, 2, 16>, 128, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_pk, xk::pk_tiered_kernel<2, 16>, 128, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_pkm, xk::pk_merged_kernel<2, 16>, 128, 0));
  } else if (D.long_g == 4 || D.long_g == 8 || D.long_g == -1) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_m, xk::band_merged_kernel<32, 4, 8>, 128, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_pk, xk::pk_tiered_kernel<4, 8>, 128, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_pkm, xk::pk_merged_kernel<4, 8>, 128, 0));
  } else {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_m, xk::band_merged_kernel<32, 1, 32>, 128, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_pk, xk::pk_tiered_kernel<4, 8>, 128, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_pkm, xk::pk_merged_kernel<4, 8>, 128, 0));
  }
  D.occ_pk = std::max(1, D.occ_pk);
  D.occ_pkm = std::max(1, D.occ_pkm);
  // resident blocks per SM of the packed merged kernel: fewer co-resident warps shorten the
  // anti-diagonal chain of the longest extensions (the launch's tail); XDROP_OCC overrides
  {
    // the tiered kernel is compiled for 4 blocks per SM (128 registers) but launched with 3: measured
    // E. coli 12.0 ms vs 14.0 with 4 blocks (more co-resident warps stretch the longest extensions'
    // anti-diagonal chain, the launch's critical path) and 12.5 with 168 registers at 3 blocks
    D.occ_pk = std::min(D.occ_pk, 3);
    if (const char* e = getenv("XDROP_OCC")) {
      D.occ_pk = std::max(1, std::min(4, atoi(e)));
      D.occ_pkm = std::max(1, std::min(D.occ_pkm, atoi(e)));
    }
    if (const char* e = getenv("XDROP_T0_PER_SM")) D.t0_per_sm = std::max(0, atoi(e));
    if (const char* e = getenv("XDROP_IDLE_NS")) D.idle_ns = std::max(0, atoi(e));
    if (const char* e = getenv("XDROP_AGE_US")) D.age_us = std::max(0, atoi(e));
    if (const char* e = getenv("XDROP_KERNEL")) D.kernel_env = atoi(e);
  }
  CKR(D.smcnt.ensure(1024 * sizeof(int)));
  D.occ_m = std::max(1, D.occ_m);
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_l1, xk::band_kernel<32, 8>, 128, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_l2, xk::band_resume_kernel<32, 32>, 128, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_pk2, xk::pk_resume_kernel<32, 32>, 128, 0));
  D.occ_pk2 = std::max(1, D.occ_pk2);
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_gen, xk::general_kernel, 128, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_cta, xk::band_cta_kernel<256, 16>, 256, 0));
  D.occ_cta = std::max(1, D.occ_cta);
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_cta1k, xk::band_cta_kernel<128, 8>, 128, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_cta2k, xk::band_cta_kernel<128, 16>, 128, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_pkw, xk::pk_wide_kernel<32>, 64, 0));
  D.occ_pkw = std::max(1, D.occ_pkw);
  if (const char* e = getenv("XDROP_WIDE_PK")) D.wide_pk = atoi(e);
  D.occ_cta2k = std::max(1, D.occ_cta2k);
  D.occ_cta1k = std::max(1, D.occ_cta1k);
  if (const char* e = getenv("XDROP_SHARED_T3")) D.shared_t3 = atoi(e);
  if (const char* e = getenv("XDROP_S1024")) D.s1024 = atoi(e);
  D.occ_l0 = std::max(1, D.occ_l0); D.occ_l1 = std::max(1, D.occ_l1);
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_ring, xk::general_ring_kernel, 128, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_grp, xk::general_group_kernel, 128, 0));
  D.occ_grp = std::max(1, D.occ_grp);
  CK(cudaFuncSetAttribute(xk::general_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kGenWideSmem));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&D.occ_ringw, xk::general_wide_kernel, 256, kGenWideSmem));
  D.occ_ringw = std::max(1, D.occ_ringw);
  D.occ_l2 = std::max(1, D.occ_l2); D.occ_gen = std::max(1, D.occ_gen); D.occ_ring = std::max(1, D.occ_ring);
  CKR(D.h_small.ensure(HS_BYTES));
  return 0;
}

void dev_close(DevCtx& D) {
  cudaSetDevice(D.dev);
  if (D.stream) cudaStreamSynchronize(D.stream);
  Buf* bufs[] = {&D.asciiA, &D.asciiB, &D.offA, &D.offB, &D.packA, &D.packB, &D.pairs, &D.wcost, &D.hist,
                 &D.cursor, &D.items, &D.ovf1, &D.ovf2, &D.ovf3, &D.counters, &D.bad, &D.ext, &D.out5,
                 &D.cells, &D.scratch, &D.level_acc, &D.pool1, &D.pool2, &D.pool3, &D.pool4, &D.q4, &D.pool5, &D.q5, &D.genl, &D.pools, &D.qs, &D.tl, &D.smcnt, &D.ms_pairs, &D.ms_res, &D.ms_best, &D.escbuf, &D.poolw, &D.qw, &D.probe, &D.ringo, &D.grpo};
  for (Buf* b : bufs) b->release();
  D.h_small.release(); D.h_pairs.release(); D.h_res.release();
  for (auto& e : D.ev) if (e) cudaEventDestroy(e);
  if (D.own_stream && D.stream) cudaStreamDestroy(D.stream);
  D.stream = nullptr;
}

int64_t packed_words(int64_t len) { return (len + 2 * xk::GUARD + 15) / 16 + 2; }

int pack_pool(DevCtx& D, const char* d_seq, int64_t len, Buf& out, cudaStream_t s, int64_t& launches) {
  const int64_t nw = packed_words(len);
  CKR(out.ensure((size_t)nw * 4));
  // the kernel writes every word of the packed pool (the guard bands as 0): no memset
  const int thr = 256;
  const int64_t threads = (nw + 3) / 4;
  xk::pack_kernel<<<(unsigned)((threads + thr - 1) / thr), thr, 0, s>>>(d_seq, len, out.as<uint32_t>(), nw,
                                                                      D.bad.as<unsigned long long>());
  ++launches;
  return cuda_err(cudaGetLastError());
}

struct Flags { bool force_wide, force_general, nosort, tiered, shared, compat; };

// The device pipeline on one GPU.  All pointers are device pointers.
// out5 / cells may be the caller's buffers (device API) or D's workspaces.
int dev_pipeline(DevCtx& D, const char* seqA, const int64_t* offA, int64_t nA, int64_t lenA,
                 const char* seqB, const int64_t* offB, int64_t nB, int64_t lenB,
                 const PairDesc* pairs, int64_t n_pairs, const xdrop_params& p, int* out5,
                 long long* cells, cudaStream_t s, Flags fl, bool do_pack = true,
                 const uint32_t* prepA = nullptr, const uint32_t* prepB = nullptr) {
  // prepA / prepB: pools already 2-bit packed on this device (xdrop_pool_register); seqA / seqB are
  // then not read
  D.err_index = -1;
  D.st = xdrop_stats{};
  int64_t launches = 0;
  CK(cudaSetDevice(D.dev));
  const int64_t n_items = 2 * n_pairs;
  CKR(D.bad.ensure(16));
  CKR(D.counters.ensure(C_N * sizeof(int)));
  CKR(D.hist.ensure(xk::NBUCKET * sizeof(int)));
  CKR(D.cursor.ensure(xk::NBUCKET * sizeof(int)));
  CKR(D.wcost.ensure((size_t)std::max<int64_t>(1, n_items) * sizeof(int)));
  CKR(D.items.ensure((size_t)std::max<int64_t>(1, n_items) * sizeof(int)));
  CKR(D.ovf1.ensure((size_t)std::max<int64_t>(1, n_items) * sizeof(int)));
  CKR(D.ovf2.ensure((size_t)std::max<int64_t>(1, n_items) * sizeof(int)));
  CKR(D.ovf3.ensure((size_t)std::max<int64_t>(1, n_items) * sizeof(int)));
  CKR(D.ext.ensure((size_t)std::max<int64_t>(1, n_items) * sizeof(ExtOut)));
  CKR(D.level_acc.ensure(8 * sizeof(unsigned long long)));
  CK(cudaMemsetAsync(D.level_acc.p, 0, 8 * sizeof(unsigned long long), s));

  CK(cudaEventRecord(D.ev[0], s));
  init_bad_kernel<<<1, 32, 0, s>>>(D.bad.as<unsigned long long>());
  init_counters_kernel<<<1, 32, 0, s>>>(D.counters.as<int>(), (int)n_items);
  launches += 2;
  // a1: ingest + pack (once per call per device; sub-batches reuse it)
  if (!prepA && do_pack) CKR(pack_pool(D, seqA, lenA, D.packA, s, launches));
  const uint32_t* PA = prepA ? prepA : D.packA.as<uint32_t>();     // (after pack_pool: it may reallocate)
  const uint32_t* PB = prepB;
  if (!PB) {
    PB = PA;
    if (seqB != seqA) {
      if (do_pack) CKR(pack_pool(D, seqB, lenB, D.packB, s, launches));
      PB = D.packB.as<uint32_t>();
    }
  }
  CK(cudaEventRecord(D.ev[1], s));
#ifdef XDROP_CHECKED
  {
    const uint32_t* base[2] = {PA, PB};
    int64_t words[2] = {packed_words(lenA), packed_words(PB != PA ? lenB : lenA)};
    // mutation knob for the checker's own test: register only the leading guard band, so that
    // the first real base any kernel reads is out of bounds and must trap
    if (getenv("XDROP_CHK_SHRINK")) words[0] = words[1] = xk::GUARD / 16;
    CK(cudaMemcpyToSymbolAsync(xk::g_chk_base, base, sizeof(base), 0, cudaMemcpyHostToDevice, s));
    CK(cudaMemcpyToSymbolAsync(xk::g_chk_words, words, sizeof(words), 0, cudaMemcpyHostToDevice, s));
  }
#endif

  xk::Problem P;
  P.PA = PA; P.offA = offA; P.nA = nA;
  P.PB = PB; P.offB = offB; P.nB = nB;
  P.lenA = lenA; P.lenB = lenB;
  P.pairs = pairs; P.n_pairs = n_pairs;
  P.M = p.match; P.mu = p.mismatch; P.g = p.gap; P.X = p.xdrop; P.k = p.k;
  P.keym = 1 << xk::KEYSH;
  P.pkM = 32 * (p.match - 2 * p.gap); P.pkU = 32 * (p.mismatch - 2 * p.gap);
  // packed 16-bit lane mode (xdrop_pk16.cuh) whenever its value range holds
  const bool pk = D.pk16 && p.xdrop + p.match <= 510;
  // resident blocks per SM of the tiered (or 32-bit merged) kernel and of the shared kernel, and how
  // many of them take fresh (T0) extensions
  // lanes per long extension ("Long mode"): 4 lanes x 8 cells, or 8 x 4 from X = 32 on
  // (measured: X-sweep X = 50 / 100 49.3 / 56.6 -> 47.2 / 50.8 ms, X = 15 21.0 -> 24.3 ms)
  const int lg = D.long_g >= 0 ? D.long_g : (p.xdrop >= 32 ? 8 : 4);
  const int occ = pk ? (lg == 8 ? std::min(D.occ_pk, D.occ_pk8) : D.occ_pk) : D.occ_m;
  const int occm = lg == 8 ? std::min(D.occ_pkm, D.occ_pkm8) : D.occ_pkm;
  const int t0b = pk && D.t0_per_sm > 0 ? std::min(occ, D.t0_per_sm) : occ;
  // the shared kernel keeps one block per SM for escalated work only (measured: X-sweep X = 100
  // 67.5 -> 64.7 ms, C. elegans x0.05 57.6 -> 55.9 ms, X = 15 / 50 within 2 % better)
  const int t0bm = D.t0_per_sm > 0 ? std::min(occm, D.t0_per_sm) : std::max(1, occm - 1);
  P.ext = D.ext.as<ExtOut>();

  int* ctr = D.counters.as<int>();
  if (n_pairs > 0) {
    // a2 + a3: validate, cost estimate, length-sorted queue
    CK(cudaMemsetAsync(D.hist.p, 0, xk::NBUCKET * sizeof(int), s));
    xk::prep_kernel<<<(unsigned)((n_pairs + 255) / 256), 256, 0, s>>>(
        P, D.wcost.as<int>(), D.hist.as<int>(), D.bad.as<unsigned long long>() + 1, XDROP_MAX_READ_LEN,
        ctr + C_MAXM);
    xk::scan_kernel<<<1, 1024, 0, s>>>(D.hist.as<int>(), D.cursor.as<int>(), ctr + C_NLONG,
                                       (long long)D.sms * t0b * 128, lg ? D.long_alpha : 0.f,
                                       D.bad.as<unsigned long long>() + 1, ctr + C_NITEMS);
    xk::scatter_kernel<<<(unsigned)((n_items + 255) / 256), 256, 0, s>>>(
        D.wcost.as<int>(), n_items, D.cursor.as<int>(), D.items.as<int>(), fl.nosort ? 1 : 0);
    launches += 3;
  }
  CK(cudaEventRecord(D.ev[2], s));
  if (n_pairs > 0) {
    // a5/a6/a7: band tiers (xdrop_kernels.cuh): T0 lane (S = 32) / long multi-lane (S = 32),
    // T1 lane pair (S = 64), T2 warp (S = 256) in one persistent kernel; checkpoints of T2
    // resume in a warp with S = 1024; beyond that the unbounded kernel restarts the extension.
    int* items0 = D.items.as<int>();
    // checkpoint-record pools (never recycled within a call): every extension may escalate once per
    // tier, so T1/T2 pools hold one record per item; the wide tiers are bounded by a byte budget
    // (a full pool only sends the extension to the unbounded kernel, still exact)
    const int64_t budget = (int64_t)4 << 30;
    const int64_t cap1 = n_items, cap2 = n_items;
    const int64_t cap3 = std::min<int64_t>(n_items, budget / ((xk::HDR + 2 * 256) * 4));
    const int64_t cap4 = std::min<int64_t>(n_items, budget / 8 / ((xk::HDR + 2 * 1024) * 4));
    const int64_t cap5 = std::min<int64_t>(n_items, budget / 16 / ((xk::HDR + 2 * 2048) * 4));
    const int rec5 = xk::HDR + 2 * 2048;
    CKR(D.pool5.ensure((size_t)std::max<int64_t>(cap5, 1) * rec5 * sizeof(int)));
    CKR(D.q5.ensure((size_t)std::max<int64_t>(cap5, 1) * sizeof(int)));
    const int rec1 = xk::HDR + 2 * 32, rec2 = xk::HDR + 2 * 128, rec3 = xk::HDR + 2 * 256, rec4 = xk::HDR + 2 * 1024;
    CKR(D.pool1.ensure((size_t)std::max<int64_t>(cap1, 1) * rec1 * sizeof(int)));
    CKR(D.pool2.ensure((size_t)std::max<int64_t>(cap2, 1) * rec2 * sizeof(int)));
    CKR(D.pool3.ensure((size_t)std::max<int64_t>(cap3, 1) * rec3 * sizeof(int)));
    CKR(D.pool4.ensure((size_t)std::max<int64_t>(cap4, 1) * rec4 * sizeof(int)));
    CKR(D.q4.ensure((size_t)std::max<int64_t>(cap4, 1) * sizeof(int)));
    const int64_t caps = n_items;                          // stolen lane-mode extensions (S = 32 records)
    CKR(D.pools.ensure((size_t)std::max<int64_t>(caps, 1) * rec1 * sizeof(int)));
    CKR(D.qs.ensure((size_t)std::max<int64_t>(caps, 1) * sizeof(int)));
    CK(cudaMemsetAsync(D.qs.p, 0xff, (size_t)std::max<int64_t>(caps, 1) * sizeof(int), s));
    CKR(D.genl.ensure((size_t)std::max<int64_t>(1, n_items) * sizeof(int)));
    CK(cudaMemsetAsync(D.ovf1.p, 0xff, (size_t)n_items * sizeof(int), s));
    CK(cudaMemsetAsync(D.ovf2.p, 0xff, (size_t)n_items * sizeof(int), s));
    int* gen = D.genl.as<int>();
    xk::Esc e1{D.pool1.as<int>(), rec1, (int)cap1, ctr + C_P1, D.ovf1.as<int>(), ctr + C_Q1T, gen, ctr + C_GEN};
    xk::Esc e2{D.pool2.as<int>(), rec2, (int)cap2, ctr + C_P2, D.ovf2.as<int>(), ctr + C_Q2T, gen, ctr + C_GEN};
    xk::Esc e3{D.pool3.as<int>(), rec3, (int)cap3, ctr + C_P3, D.ovf3.as<int>(), ctr + C_Q3T, gen, ctr + C_GEN};
    xk::Esc e4{D.pool4.as<int>(), rec4, (int)cap4, ctr + C_P4, D.q4.as<int>(), ctr + C_Q4T, gen, ctr + C_GEN};
    xk::Esc e5{D.pool5.as<int>(), rec5, (int)cap5, ctr + C_P5, D.q5.as<int>(), ctr + C_Q5T, gen, ctr + C_GEN};
    xk::Esc eg{nullptr, 0, 0, ctr + C_HEADW, nullptr, nullptr, gen, ctr + C_GEN};   // always falls back
    // compat mode in the packed tiers: everything up to S = 2048 as in the default
    // mode (CP instances: the Q28 edge kill, the Q29 last-maximum), wider extensions restart in the
    // general path's rings; 32-bit cells (X + M > 510) or XDROP_COMPAT_GENERAL=1: the general path only
    const bool cpk = fl.compat && pk && !D.compat_general;
    xk::Esc e5c{nullptr, 0, 0, ctr + C_P5, nullptr, nullptr, gen, ctr + C_GEN};   // compat: S > 2048 -> gen
    if (fl.force_general) {
      // everything goes to the unbounded kernel below
    } else if (fl.compat && !cpk) {
      // compat mode: the general path in shared-memory rings; hulls wider than the ring go to the
      // unbounded kernel below (the gen list)
      CKR(D.ringo.ensure((size_t)std::max<int64_t>(1, n_items) * sizeof(int)));
      CKR(D.grpo.ensure((size_t)std::max<int64_t>(1, n_items) * sizeof(int)));
      // group kernel (8 lanes per extension) first, unless the batch is small (< 8 extensions per
      // resident ring warp) or the batch's probe (the default mode's, run in the packed T0 window)
      // finds wide hulls in >= compat_grp of its sample: then the warp-ring kernel takes it directly
      // (measured: E. coli-shaped 106 vs 190 ms with the group kernel first; X-sweep X = 15, probe
      // 8.8 %: 53 vs 93 ms with the ring first; C. elegans-shaped x0.05, probe 4.4 %: 410 vs 492 ms)
      xk::GenChoice gc{ctr + C_ZERO, 1 << 30};
      if (D.compat_first == 1) {
        // group kernel first (forced)
      } else if (D.compat_first == 2 || n_items < 8LL * D.sms * D.occ_ring * 4) {
        gc.thr = 0;      // a small batch: every extension gets its own warp at once (shorter chains)
      } else if (pk) {
        const int stride = (int)std::max<int64_t>(1, n_items / kProbe);
        const int n_probe = (int)std::min<int64_t>(kProbe, (n_items + stride - 1) / stride);
        CKR(D.probe.ensure((size_t)kProbe * sizeof(int)));
        xk::Esc ep{nullptr, 0, 0, ctr + C_PROBE, nullptr, nullptr, D.probe.as<int>(), ctr + C_PROBEFB};
        xk::pk_probe_kernel<32><<<(unsigned)((n_probe + 127) / 128), 128, 0, s>>>(P, items0, ctr + C_NITEMS, n_probe,
                                                                                  stride, kProbeCap, ep);
        ++launches;
        gc = xk::GenChoice{ctr + C_PROBE, std::max(1, (int)std::ceil(D.compat_grp * n_probe))};
      }
      xk::general_group_kernel<<<D.sms * D.occ_grp, 128, 0, s>>>(P, items0, ctr + C_NITEMS, ctr + C_HEADW,
                                                                   D.grpo.as<int>(), ctr + C_GRPO, 3, 1, gc);
      xk::general_ring_kernel<<<D.sms * D.occ_ring, 128, 0, s>>>(P, D.grpo.as<int>(), ctr + C_GRPO, ctr + C_HEADGRP,
                                                                   D.ringo.as<int>(), ctr + C_RINGO, 3, 1, gc,
                                                                   items0, ctr + C_NITEMS);
      xk::general_wide_kernel<<<D.sms * D.occ_ringw, 256, kGenWideSmem, s>>>(
          P, D.ringo.as<int>(), ctr + C_RINGO, ctr + C_HEADRW, gen, ctr + C_GEN, 3, 1);
      launches += 3;
    } else if (fl.force_wide) {
      xk::band_kernel<32, 8><<<D.sms * D.occ_l1, 128, 0, s>>>(P, items0, ctr + C_NITEMS, ctr + C_HEADW, e3, 1);
      ++launches;
    } else {
      xk::MergedCtr mc{ctr + C_HEAD0, ctr + C_DONE0, ctr + C_HEADL, ctr + C_NLONG, ctr + C_Q1H, ctr + C_DONE1,
                       ctr + C_Q2H, ctr + C_IDLE, ctr + C_SH, ctr + C_DONES, nullptr, ctr + C_TLN, 0,
                       (int)std::min<int64_t>((int64_t)(D.endgame * D.sms * t0b * 4 * 32), 1 << 30),
                       D.smcnt.as<int>(), pk ? t0b : 0, D.idle_ns, D.age_us, ctr + C_PROBE, 0};
      CK(cudaMemsetAsync(D.smcnt.p, 0, 1024 * sizeof(int), s));
      if (D.timeline) {                                   // XDROP_TIMELINE=1: per-work-unit timeline
        CKR(D.tl.ensure((size_t)3 * 8 * kTimelineCap));
        mc.tl = D.tl.as<unsigned long long>(); mc.tl_cap = kTimelineCap;
      }
      // tail stealing: when 1/8 of the resident warps are idle, lane warps hand over extensions with
      // >= 1024 anti-diagonals left (a full block pool falls back to the unbounded kernel)
      const int nwarps = D.sms * t0b * 4;
      xk::Esc es{D.pools.as<int>(), rec1, (int)caps, ctr + C_SP, D.qs.as<int>(), ctr + C_ST, gen, ctr + C_GEN};
      xk::Steal stl{ctr + C_IDLE, std::max(8, nwarps / D.steal_div), D.steal_min, es};
      if (D.steal_min <= 0) stl.thresh = 1 << 30;            // disabled
      const unsigned grid = (unsigned)(D.sms * occ), grid_m = (unsigned)(D.sms * occm);
      // the shared kernel's own occupancy, T0 blocks and steal threshold
      xk::MergedCtr mcm = mc;
      mcm.t0_per_sm = t0bm;
      xk::Steal stlm = stl;
      if (D.steal_min > 0) stlm.thresh = std::max(8, D.sms * t0bm * 4 / D.steal_div);
      // the packed kernel reads its tier descriptors from device memory where used (rare paths)
      const xk::PkTier* tiers = nullptr;
      if (pk) {
        // endgame steals (T1/T2 extensions resumed 32 lanes x 8 cells once st.thresh warps idle): at
        // most one record per resident pool group
        const int capw = D.sms * std::max(occ, occm) * 4 * 8;
        CKR(D.poolw.ensure((size_t)capw * rec3 * sizeof(int)));
        CKR(D.qw.ensure((size_t)capw * sizeof(int)));
        CK(cudaMemsetAsync(D.qw.p, 0xff, (size_t)capw * sizeof(int), s));
        xk::Esc ew{D.poolw.as<int>(), rec3, capw, ctr + C_WP, D.qw.as<int>(), ctr + C_WT, gen, ctr + C_GEN};
        CKR(D.escbuf.ensure(5 * sizeof(xk::PkTier)));
        D.tier_host[0] = xk::PkTier{es, e1, nullptr, nullptr, 0};                   // fresh (T0; src: lane steals)
        D.tier_host[1] = xk::PkTier{e1, e2, ctr + C_Q1H, ctr + C_DONE1, 1};         // T1 pool
        D.tier_host[2] = xk::PkTier{e2, e3, ctr + C_Q2H, ctr + C_DONE2, 1};         // T2 pool
        D.tier_host[3] = xk::PkTier{e3, e4, ctr + C_HEAD3, nullptr, 2};             // T3 pool (S = 1024)
        if (!D.shared_t3) D.tier_host[3].src.q_tail = ctr + C_ZERO;                  // T3 off: an empty queue
        D.tier_host[4] = xk::PkTier{ew, e3, ctr + C_WH, ctr + C_WD, 1};             // endgame steals
        CK(cudaMemcpyAsync(D.escbuf.p, D.tier_host, 5 * sizeof(xk::PkTier), cudaMemcpyHostToDevice, s));
        tiers = D.escbuf.as<xk::PkTier>();
      }
      // packed kernel per batch: forced by flag / XDROP_KERNEL, else the probe decides on
      // the device (both kernels are launched; the one not chosen exits at once, so the host never
      // waits for the probe)
      int choice = 0;             // 0 probe, 1 tiered, 2 shared
      if (pk) choice = fl.shared ? 2 : fl.tiered ? 1 : (D.kernel_env == 1 || D.kernel_env == 2) ? D.kernel_env : 0;
      if (pk && choice == 0 && n_items < kSharedT1) choice = 1;   // too few extensions to reach the threshold
      if (pk && choice == 0) {
        const int stride = (int)std::max<int64_t>(1, n_items / kProbe);
        const int n_probe = (int)std::min<int64_t>(kProbe, (n_items + stride - 1) / stride);
        CKR(D.probe.ensure((size_t)kProbe * sizeof(int)));
        xk::Esc ep{nullptr, 0, 0, ctr + C_PROBE, nullptr, nullptr, D.probe.as<int>(), ctr + C_PROBEFB};
        xk::pk_probe_kernel<32><<<(unsigned)((n_probe + 127) / 128), 128, 0, s>>>(P, items0, ctr + C_NITEMS, n_probe,
                                                                                  stride, kProbeCap, ep);
        ++launches;
        // shared iff probe overflows x (n_items / n_probe) >= kSharedT1
        mc.probe_thr = (int)std::max<int64_t>(1, (kSharedT1 * n_probe + n_items - 1) / n_items);
      } else {
        mc.probe_thr = choice == 2 ? 0 : (1 << 30);
      }
      mcm.probe_thr = mc.probe_thr;
      const bool run_tiered = pk && choice != 2, run_shared = pk && choice != 1;
      D.st.band_kernel = pk ? (choice == 2 ? 2 : 1) : 0;   // refined from the probe count after the call
      if (run_tiered && cpk)
        xk::pk_tiered_kernel<4, 8, true><<<grid, 128, 0, s>>>(P, items0, ctr + C_NITEMS, mc, e1, e2, e3, stl);
      else if (run_tiered && lg == 8)
        xk::pk_tiered_kernel<8, 4><<<grid, 128, 0, s>>>(P, items0, ctr + C_NITEMS, mc, e1, e2, e3, stl);
      else if (run_tiered && lg == 2)
        xk::pk_tiered_kernel<2, 16><<<grid, 128, 0, s>>>(P, items0, ctr + C_NITEMS, mc, e1, e2, e3, stl);
      else if (run_tiered)
        xk::pk_tiered_kernel<4, 8><<<grid, 128, 0, s>>>(P, items0, ctr + C_NITEMS, mc, e1, e2, e3, stl);
      if (run_shared && cpk)
        xk::pk_merged_kernel<4, 8, true><<<grid_m, 128, 0, s>>>(P, items0, ctr + C_NITEMS, mcm, tiers, stlm);
      else if (run_shared && lg == 8)
        xk::pk_merged_kernel<8, 4><<<grid_m, 128, 0, s>>>(P, items0, ctr + C_NITEMS, mcm, tiers, stlm);
      else if (run_shared && lg == 2)
        xk::pk_merged_kernel<2, 16><<<grid_m, 128, 0, s>>>(P, items0, ctr + C_NITEMS, mcm, tiers, stlm);
      else if (run_shared)      // lg 4, or 0 (no long mode: n_long = 0)
        xk::pk_merged_kernel<4, 8><<<grid_m, 128, 0, s>>>(P, items0, ctr + C_NITEMS, mcm, tiers, stlm);
      if (run_tiered && run_shared) ++launches;
      if (pk) {
        D.probe_thr = mc.probe_thr;
        D.probe_choice = choice;
      } else if (lg == 2) {           // 32-bit cells (X + M > 510)
        xk::band_merged_kernel<32, 2, 16><<<grid, 128, 0, s>>>(P, items0, ctr + C_NITEMS, mc, e1, e2, e3, stl);
      } else if (lg == 4 || lg == 8) {
        xk::band_merged_kernel<32, 4, 8><<<grid, 128, 0, s>>>(P, items0, ctr + C_NITEMS, mc, e1, e2, e3, stl);
      } else {
        xk::band_merged_kernel<32, 1, 32><<<grid, 128, 0, s>>>(P, items0, ctr + C_NITEMS, mc, e1, e2, e3, stl);
      }
      ++launches;
    }
    CK(cudaEventRecord(D.ev[8], s));
    CK(cudaEventRecord(D.ev[9], s));
    int* gen_items = gen;
    int* gen_count = ctr + C_GEN;
    if (fl.force_general) {
      gen_items = items0;
      gen_count = ctr + C_NITEMS;
    } else if (fl.compat && !cpk) {
      // no band levels: the ring kernel's overflows are already in the gen list
    } else if (cpk) {
      // compat in the packed tiers: the S = 1024 and the packed S = 2048 levels; wider extensions
      // restart in the general path
      xk::pk_resume_kernel<32, 32, true><<<D.sms * D.occ_pk2, 128, 0, s>>>(P, e3, ctr + C_HEAD3, e4, 2);
      xk::pk_wide_kernel<32, true><<<D.sms * D.occ_pkw, 64, 0, s>>>(P, e4, ctr + C_HEAD4, e5c, 2);
      launches += 2;
    } else {
      // S1024 level: one warp with 32 cells per lane per extension (default), or one thread block of
      // 4 warps x 32 lanes x 8 cells (XDROP_S1024=1: slower, its barrier per anti-diagonal costs more
      // than the shorter per-lane work saves)
      if (D.s1024)
        xk::band_cta_kernel<128, 8><<<D.sms * D.occ_cta1k, 128, 0, s>>>(P, e3, ctr + C_HEAD3, e4, 2);
      else if (pk)
        xk::pk_resume_kernel<32, 32><<<D.sms * D.occ_pk2, 128, 0, s>>>(P, e3, ctr + C_HEAD3, e4, 2);
      else
        xk::band_resume_kernel<32, 32><<<D.sms * D.occ_l2, 128, 0, s>>>(P, e3, ctr + C_HEAD3, e4, 2);
      // CTA levels: S = 2048 (4 warps x 32 lanes x 16 cells; twice the resident extensions of the
      // 8-warp block) checkpointing its overflows for S = 4096 (8 warps x 32 x 16)
      if (pk && D.wide_pk)        // packed S = 2048: one extension per 2-warp block (xdrop_pkwide.cuh)
        xk::pk_wide_kernel<32><<<D.sms * D.occ_pkw, 64, 0, s>>>(P, e4, ctr + C_HEAD4, e5, 2);
      else
        xk::band_cta_kernel<128, 16><<<D.sms * D.occ_cta2k, 128, 0, s>>>(P, e4, ctr + C_HEAD4, e5, 2);
      xk::band_cta_kernel<256, 16><<<D.sms * D.occ_cta, 256, 0, s>>>(P, e5, ctr + C_HEAD5, eg, 2);
      launches += 3;
    }
    CK(cudaEventRecord(D.ev[10], s));
    CK(cudaGetLastError());
    // read the validation flags and the unbounded-path count
    int* hs = reinterpret_cast<int*>(D.h_small.p);
    CK(cudaMemcpyAsync(hs, ctr, C_N * sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hs + HS_BAD, D.bad.p, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const unsigned long long* bad = reinterpret_cast<const unsigned long long*>(hs + HS_BAD);
    if (bad[0] != ~0ull) { D.err_index = (int64_t)bad[0]; return XDROP_EALPHABET; }
    if (bad[1] != ~0ull) { D.err_index = (int64_t)bad[1]; return XDROP_ESEED; }
    const int n_gen = fl.force_general ? (int)n_items : hs[C_GEN];
    const bool cgen = fl.compat && !cpk;                       // compat in the general path only
    D.st.escalated[0] = fl.force_wide || fl.force_general || cgen ? n_items : hs[C_P1];
    D.st.escalated[1] = cgen ? hs[C_GRPO] : hs[C_P2];         // compat: hulls wider than a group's ring
    if (cgen) D.st.probe_overflows = hs[C_PROBE];
    if (pk && !fl.force_wide && !fl.force_general && !cgen && D.probe_choice == 0) {
      D.st.band_kernel = hs[C_PROBE] >= D.probe_thr ? 2 : 1;   // which kernel the probe let run
      D.st.probe_overflows = hs[C_PROBE];
    }
    D.st.escalated[2] = cgen ? hs[C_RINGO] : hs[C_P3];        // compat: hulls wider than the warp's ring
    D.st.cta_items = hs[C_P4];
    D.st.cta4k_items = hs[C_P5];
    D.st.endgame_stolen = hs[C_WP];
    D.st.escalated[3] = n_gen;
    D.st.long_items = hs[C_NLONG];
    D.st.stolen = hs[C_SP];
    if (n_gen > 0 && cpk) {
      // compat in the packed tiers: the extensions wider than S = 2048 restart in the 8-warp ring
      // kernel (8,192-cell rings), whose overflows restart in the global-memory kernel below
      CKR(D.ringo.ensure((size_t)std::max<int64_t>(1, n_items) * sizeof(int)));
      xk::general_wide_kernel<<<D.sms * D.occ_ringw, 256, kGenWideSmem, s>>>(
          P, gen_items, gen_count, ctr + C_HEADRW, D.ringo.as<int>(), ctr + C_RINGO, 3, 1);
      ++launches;
      gen_items = D.ringo.as<int>();
      gen_count = ctr + C_RINGO;
    }
    if (n_gen > 0) {
      // three anti-diagonals of m + 1 values per warp (m: the batch's longest A-side extension);
      // all resident warps (the compat mode sends every extension here), scratch capped at 2 GiB
      const int64_t stride = (int64_t)std::min(std::max(hs[C_MAXM], 0), XDROP_MAX_READ_LEN) + 8;
      const int warps_per_block = 4;
      const int64_t cap = ((int64_t)2 << 30) / (3 * stride * (int64_t)sizeof(int));
      int64_t nwarps = std::min<int64_t>({(int64_t)D.sms * D.occ_gen * warps_per_block, (int64_t)n_gen, cap});
      nwarps = std::max<int64_t>(warps_per_block, (nwarps / warps_per_block) * warps_per_block);
      CKR(D.scratch.ensure((size_t)nwarps * 3 * stride * sizeof(int)));
      xk::general_kernel<<<(unsigned)(nwarps / warps_per_block), 128, 0, s>>>(
          P, gen_items, gen_count, ctr + C_HEADG, D.scratch.as<int>(), stride, 3, fl.compat ? 1 : 0);
      ++launches;
    }
  } else {
    int* hs = reinterpret_cast<int*>(D.h_small.p);
    CK(cudaMemcpyAsync(hs + HS_BAD, D.bad.p, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const unsigned long long* bad = reinterpret_cast<const unsigned long long*>(hs + HS_BAD);
    if (bad[0] != ~0ull) { D.err_index = (int64_t)bad[0]; return XDROP_EALPHABET; }
  }
  CK(cudaEventRecord(D.ev[3], s));
  if (n_pairs > 0) {
    xk::combine_kernel<<<(unsigned)((n_pairs + 255) / 256), 256, 0, s>>>(
        P, out5, cells, D.level_acc.as<unsigned long long>());
    ++launches;
    CK(cudaMemcpyAsync(reinterpret_cast<int*>(D.h_small.p) + HS_LVL, D.level_acc.p, 64, cudaMemcpyDeviceToHost, s));
  }
  CK(cudaEventRecord(D.ev[4], s));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  float ms = 0;
  cudaEventElapsedTime(&ms, D.ev[2], D.ev[3]); D.st.kernel_ms = ms;
  cudaEventElapsedTime(&ms, D.ev[0], D.ev[4]); D.st.total_ms = ms;
  cudaEventElapsedTime(&ms, D.ev[0], D.ev[1]); D.st.pack_ms = ms;
  if (n_pairs > 0) {
    cudaEventElapsedTime(&ms, D.ev[2], D.ev[8]); D.st.level_ms[0] = ms;
    cudaEventElapsedTime(&ms, D.ev[8], D.ev[9]); D.st.level_ms[1] = ms;
    cudaEventElapsedTime(&ms, D.ev[9], D.ev[10]); D.st.level_ms[2] = ms;
    cudaEventElapsedTime(&ms, D.ev[10], D.ev[3]); D.st.level_ms[3] = ms;
    const unsigned long long* acc = reinterpret_cast<const unsigned long long*>(reinterpret_cast<int*>(D.h_small.p) + HS_LVL);
    for (int l = 0; l < 4; ++l) { D.st.level_cells[l] = (int64_t)acc[l]; D.st.level_items[l] = (int64_t)acc[4 + l]; }
    D.st.cells = D.st.level_cells[0] + D.st.level_cells[1] + D.st.level_cells[2] + D.st.level_cells[3];
  }
  D.st.items = n_items;
  D.st.launches = launches;
  return 0;
}

}  // namespace

// ------------------------------------------------------------------- context
namespace {
// A read pool registered once per context (xdrop_pool_register): 2-bit packed on every device, with
// a host copy of the offsets for the host-side validation and cost estimate of each call.
struct RegPool {
  bool alive = false;
  int64_t n = 0, len = 0;
  std::vector<int64_t> off;            // host copy, n + 1 entries
  std::vector<Buf> off_d, pack_d;      // per device
};
}  // namespace

struct xdrop_ctx {
  std::vector<RegPool> pools;
  std::vector<DevCtx> devs;
  xdrop_init_opts opts{};
  std::vector<int> dev_ids;
  int64_t err_index = -1;
  xdrop_stats st{};
  bool alive = false;
  xdrop_sched_stats sched{};
  std::vector<xdrop_trace_event> trace;
};

static int validate_params(const xdrop_params* p) {
  if (!p) return XDROP_EINVAL;
  if (p->match < 1 || p->match > 32) return XDROP_EINVAL;
  if (p->mismatch > -1 || p->mismatch < -64) return XDROP_EINVAL;
  if (p->gap > -1 || p->gap < -64) return XDROP_EINVAL;
  if (p->xdrop < 0 || p->xdrop > (1 << 20)) return XDROP_EINVAL;
  if (p->k < 1 || p->k > 1024) return XDROP_EINVAL;
  return 0;
}

extern "C" int xdrop_init(const xdrop_init_opts* opts, xdrop_ctx** out_ctx) {
  if (!out_ctx) return XDROP_EINVAL;
  *out_ctx = nullptr;
  xdrop_init_opts o{};
  o.n_devices = 1;
  if (opts) o = *opts;
  if (o.n_devices < 1 || o.policy < 0 || o.policy > 3) return XDROP_EINVAL;
  if (o.n_ranks < 1) o.n_ranks = 1;
  if (o.batch_size <= 0) o.batch_size = 10000;
  if (o.subbatches <= 0) o.subbatches = 1;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) { cudaGetLastError(); return XDROP_ENODEV; }
  xdrop_ctx* ctx = new (std::nothrow) xdrop_ctx();
  if (!ctx) return XDROP_ENOMEM;
  ctx->opts = o;
  for (int i = 0; i < o.n_devices; ++i) {
    const int d = o.devices ? o.devices[i] : i % ndev;
    if (d < 0 || d >= ndev) { delete ctx; return XDROP_ENODEV; }
    ctx->dev_ids.push_back(d);
  }
  ctx->opts.devices = nullptr;
  ctx->devs.resize(o.n_devices);
  for (int i = 0; i < o.n_devices; ++i) {
    int rc = dev_open(ctx->devs[i], ctx->dev_ids[i]);
    if (rc) {
      for (int j = 0; j <= i; ++j) dev_close(ctx->devs[j]);
      delete ctx;
      return rc;
    }
  }
  ctx->alive = true;
  *out_ctx = ctx;
  return 0;
}

extern "C" int xdrop_finalize(xdrop_ctx* ctx) {
  if (!ctx) return XDROP_ESTATE;
  for (auto& rp : ctx->pools)
    for (size_t g = 0; g < rp.off_d.size() && g < ctx->devs.size(); ++g) {
      cudaSetDevice(ctx->devs[g].dev);
      rp.off_d[g].release();
      rp.pack_d[g].release();
    }
  for (auto& D : ctx->devs) dev_close(D);
  ctx->alive = false;
  delete ctx;
  return 0;
}

extern "C" const char* xdrop_strerror(int status) {
  switch (status) {
    case XDROP_OK: return "ok";
    case XDROP_EINVAL: return "invalid argument";
    case XDROP_ENOMEM: return "out of memory";
    case XDROP_ECUDA: return "CUDA error";
    case XDROP_EALPHABET: return "base outside {A,C,G,T}";
    case XDROP_ESEED: return "seed out of range or bad read id";
    case XDROP_ELENGTH: return "read too long";
    case XDROP_ESTATE: return "invalid context state";
    case XDROP_ENODEV: return "no CUDA device";
    default: return "unknown status";
  }
}

extern "C" int64_t xdrop_last_error_index(const xdrop_ctx* ctx) { return ctx ? ctx->err_index : -1; }

extern "C" int xdrop_last_stats(const xdrop_ctx* ctx, xdrop_stats* st) {
  if (!ctx || !st) return XDROP_EINVAL;
  *st = ctx->st;
  return 0;
}

static Flags flags_of(const xdrop_ctx* ctx) {
  Flags f;
  f.force_wide = (ctx->opts.flags & XDROP_FLAG_FORCE_WIDE) != 0;
  // the compat mode (Q28-Q30): the packed tiers' CP instances or the general path
  f.compat = (ctx->opts.flags & XDROP_FLAG_SEQAN_COMPAT) != 0;
  if (f.compat) f.force_wide = false;     // the 32-bit warp level has no compat instance
  f.force_general = (ctx->opts.flags & XDROP_FLAG_FORCE_GENERAL) != 0;
  f.nosort = (ctx->opts.flags & XDROP_FLAG_NO_SORT) != 0;
  f.tiered = (ctx->opts.flags & XDROP_FLAG_TIERED) != 0;
  f.shared = (ctx->opts.flags & XDROP_FLAG_SHARED) != 0;
  return f;
}

extern "C" int xdrop_align_batch_device(xdrop_ctx* ctx, const char* seqA, const int64_t* offA, int64_t nA,
                                        int64_t lenA, const char* seqB, const int64_t* offB, int64_t nB,
                                        int64_t lenB, const xdrop_pair* pairs, int64_t n_pairs,
                                        const xdrop_params* p, xdrop_result* out, int64_t* cells_out,
                                        void* stream) {
  if (!ctx || !ctx->alive) return XDROP_ESTATE;
  ctx->err_index = -1;
  int rc = validate_params(p);
  if (rc) return rc;
  if (n_pairs < 0 || nA < 0 || nB < 0 || lenA < 0 || lenB < 0) return XDROP_EINVAL;
  if (n_pairs > (int64_t)((1u << 30) - 1)) return XDROP_EINVAL;
  if (n_pairs > 0 && (!seqA || !offA || !seqB || !offB || !pairs || !out)) return XDROP_EINVAL;
  DevCtx& D = ctx->devs[0];
  cudaStream_t s = stream ? (cudaStream_t)stream : D.stream;
  rc = dev_pipeline(D, seqA, offA, nA, lenA, seqB, offB, nB, lenB, reinterpret_cast<const PairDesc*>(pairs),
                    n_pairs, *p, reinterpret_cast<int*>(out), reinterpret_cast<long long*>(cells_out), s,
                    flags_of(ctx));
  ctx->err_index = D.err_index;
  ctx->st = D.st;
  return rc;
}

// f4: best seed per candidate (device pointers)
extern "C" int xdrop_best_seed_device(xdrop_ctx* ctx, const xdrop_pair* pairs, const xdrop_result* res, int64_t n,
                                      int64_t* best, void* stream) {
  if (!ctx || !ctx->alive) return XDROP_ESTATE;
  ctx->err_index = -1;
  if (n < 0 || (n > 0 && (!pairs || !res || !best))) return XDROP_EINVAL;
  if (n == 0) return 0;
  DevCtx& D = ctx->devs[0];
  CK(cudaSetDevice(D.dev));
  cudaStream_t s = stream ? (cudaStream_t)stream : D.stream;
  xk::best_seed_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(
      reinterpret_cast<const PairDesc*>(pairs), reinterpret_cast<const int*>(res), n,
      reinterpret_cast<long long*>(best));
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));
  return 0;
}

// ---------------------------------------------------------------- host API
namespace {

struct HostBatch {
  const xdrop_seqs* A; const xdrop_seqs* B; bool same;
  const xdrop_pair* pairs; const xdrop_params* p; Flags fl;
  xdrop_result* out; int64_t* cells_out;
  int64_t n_pairs = 0;
  const RegPool* ra = nullptr; const RegPool* rb = nullptr;   // registered pools (xdrop_align_pooled)
};

// Run a subset of pairs (indices idx) on device D; pools are uploaded once per
// call per device (upload_pools), pairs/results per sub-batch.
// accumulate the counters of one pipeline run into a call's totals: counts add up, times take the
// maximum (devices run concurrently), the kernel choice is the last one
void stats_add(xdrop_stats& a, const xdrop_stats& b) {
  a.items += b.items; a.cells += b.cells; a.launches += b.launches;
  for (int l = 0; l < 4; ++l) {
    a.escalated[l] += b.escalated[l]; a.level_cells[l] += b.level_cells[l]; a.level_items[l] += b.level_items[l];
    a.level_ms[l] = std::max(a.level_ms[l], b.level_ms[l]);
  }
  a.kernel_ms = std::max(a.kernel_ms, b.kernel_ms); a.total_ms = std::max(a.total_ms, b.total_ms);
  a.pack_ms = std::max(a.pack_ms, b.pack_ms);
  a.long_items += b.long_items; a.stolen += b.stolen; a.band_kernel = b.band_kernel;
  a.cta_items += b.cta_items; a.cta4k_items += b.cta4k_items; a.endgame_stolen += b.endgame_stolen;
  a.probe_overflows += b.probe_overflows;
}

struct DevSession {
  DevCtx* D;
  const HostBatch* hb;
  bool uploaded = false;
  bool packed = false;
  xdrop_stats acc{};          // this device's counters summed over the call's turns
  int slot = 0;               // device slot of D in the context (registered pools are per slot)
  int upload() {
    if (uploaded || hb->ra) return 0;     // registered pools live on the device already
    DevCtx& d = *D;
    CK(cudaSetDevice(d.dev));
    const xdrop_seqs* A = hb->A;
    const int64_t lenA = A->offsets[A->n];
    CKR(d.asciiA.ensure((size_t)std::max<int64_t>(lenA, 1)));
    CKR(d.offA.ensure((size_t)(A->n + 1) * 8));
    CK(cudaMemcpyAsync(d.asciiA.p, A->seq, (size_t)lenA, cudaMemcpyHostToDevice, d.stream));
    CK(cudaMemcpyAsync(d.offA.p, A->offsets, (size_t)(A->n + 1) * 8, cudaMemcpyHostToDevice, d.stream));
    if (!hb->same) {
      const xdrop_seqs* B = hb->B;
      const int64_t lenB = B->offsets[B->n];
      CKR(d.asciiB.ensure((size_t)std::max<int64_t>(lenB, 1)));
      CKR(d.offB.ensure((size_t)(B->n + 1) * 8));
      CK(cudaMemcpyAsync(d.asciiB.p, B->seq, (size_t)lenB, cudaMemcpyHostToDevice, d.stream));
      CK(cudaMemcpyAsync(d.offB.p, B->offsets, (size_t)(B->n + 1) * 8, cudaMemcpyHostToDevice, d.stream));
    }
    uploaded = true;
    return 0;
  }
  // align pairs[idx[0..n)] -> out[idx[t]]; idx == nullptr means pairs[0..n) (no gather/scatter:
  // descriptors and results move straight between the caller's buffers and the device)
  int run(const int64_t* idx, int64_t n) {
    DevCtx& d = *D;
    CKR(upload());
    CKR(d.pairs.ensure((size_t)std::max<int64_t>(n, 1) * sizeof(xdrop_pair)));
    CKR(d.out5.ensure((size_t)std::max<int64_t>(n, 1) * sizeof(xdrop_result)));
    CKR(d.cells.ensure((size_t)std::max<int64_t>(n, 1) * 8));
    if (idx) {
      CKR(d.h_pairs.ensure((size_t)std::max<int64_t>(n, 1) * sizeof(xdrop_pair)));
      xdrop_pair* sub = reinterpret_cast<xdrop_pair*>(d.h_pairs.p);
      for (int64_t t = 0; t < n; ++t) sub[t] = hb->pairs[idx[t]];
      if (n > 0)
        CK(cudaMemcpyAsync(d.pairs.p, sub, (size_t)n * sizeof(xdrop_pair), cudaMemcpyHostToDevice, d.stream));
    } else if (n > 0) {
      CK(cudaMemcpyAsync(d.pairs.p, hb->pairs, (size_t)n * sizeof(xdrop_pair), cudaMemcpyHostToDevice, d.stream));
    }
    const xdrop_seqs* A = hb->A;
    const xdrop_seqs* B = hb->B;
    int rc;
    if (hb->ra) {                // registered pools: packed and resident, only the pairs moved
      const RegPool& a = *hb->ra;
      const RegPool& b = *hb->rb;
      rc = dev_pipeline(d, nullptr, a.off_d[(size_t)slot].as<int64_t>(), a.n, a.len, nullptr,
                        b.off_d[(size_t)slot].as<int64_t>(), b.n, b.len, d.pairs.as<PairDesc>(), n, *hb->p,
                        d.out5.as<int>(), d.cells.as<long long>(), d.stream, hb->fl, false,
                        a.pack_d[(size_t)slot].as<uint32_t>(), b.pack_d[(size_t)slot].as<uint32_t>());
    } else {
      const char* sA = d.asciiA.as<char>();
      const int64_t* oA = d.offA.as<int64_t>();
      const char* sB = hb->same ? sA : d.asciiB.as<char>();
      const int64_t* oB = hb->same ? oA : d.offB.as<int64_t>();
      rc = dev_pipeline(d, sA, oA, A->n, A->offsets[A->n], sB, oB, B->n, B->offsets[B->n],
                        d.pairs.as<PairDesc>(), n, *hb->p, d.out5.as<int>(), d.cells.as<long long>(),
                        d.stream, hb->fl, !packed);
    }
    if (rc == 0 || rc != XDROP_EALPHABET) packed = true;
    if (rc == 0) stats_add(acc, d.st);
    if (rc) {
      if (d.err_index >= 0 && rc != XDROP_EALPHABET && idx) d.err_index = idx[d.err_index];
      return rc;
    }
    if (n == 0) return 0;
    if (!idx) {
      CK(cudaMemcpyAsync(hb->out, d.out5.p, (size_t)n * sizeof(xdrop_result), cudaMemcpyDeviceToHost, d.stream));
      if (hb->cells_out)
        CK(cudaMemcpyAsync(hb->cells_out, d.cells.p, (size_t)n * 8, cudaMemcpyDeviceToHost, d.stream));
      CK(cudaStreamSynchronize(d.stream));
      return 0;
    }
    CKR(d.h_res.ensure((size_t)n * (sizeof(xdrop_result) + 8)));
    xdrop_result* res = reinterpret_cast<xdrop_result*>(d.h_res.p);
    int64_t* cl = reinterpret_cast<int64_t*>(res + n);
    CK(cudaMemcpyAsync(res, d.out5.p, (size_t)n * sizeof(xdrop_result), cudaMemcpyDeviceToHost, d.stream));
    CK(cudaMemcpyAsync(cl, d.cells.p, (size_t)n * 8, cudaMemcpyDeviceToHost, d.stream));
    CK(cudaStreamSynchronize(d.stream));
    for (int64_t t = 0; t < n; ++t) {
      hb->out[idx[t]] = res[t];
      if (hb->cells_out) hb->cells_out[idx[t]] = cl[t];
    }
    return 0;
  }
};

int host_validate(const xdrop_seqs* S, int64_t& err) {
  if (!S || !S->offsets || S->n < 0 || (S->n > 0 && !S->seq)) return XDROP_EINVAL;
  if (S->offsets[0] < 0) return XDROP_EINVAL;
  for (int64_t r = 0; r < S->n; ++r) {
    const int64_t L = S->offsets[r + 1] - S->offsets[r];
    if (L < 0) { err = r; return XDROP_EINVAL; }
    if (L > XDROP_MAX_READ_LEN) { err = r; return XDROP_ELENGTH; }
  }
  if (S->offsets[0] != 0) return XDROP_EINVAL;  // pools are offset from seq[0]
  return 0;
}

}  // namespace

// The host API's body (xdrop_align_batch, xdrop_align_pooled): hb holds host pools A, B (their
// offsets; with registered pools also hb.ra / hb.rb), the pairs and the outputs.
static int align_host(xdrop_ctx* ctx, HostBatch& hb) {
  const xdrop_seqs* A = hb.A;
  const xdrop_seqs* B = hb.B;
  const xdrop_pair* pairs = hb.pairs;
  const xdrop_params* p = hb.p;
  int rc = 0;
  const int64_t n_pairs = hb.n_pairs;
  const int m = (int)ctx->devs.size();
  std::vector<DevSession> sess((size_t)m);
  for (int g = 0; g < m; ++g) {
    sess[(size_t)g].D = &ctx->devs[(size_t)g]; sess[(size_t)g].hb = &hb; sess[(size_t)g].slot = g;
  }
  const bool single = m == 1 && ctx->opts.policy == XDROP_POLICY_CELLS;
  auto pool_ok = [](const xdrop_seqs* S) {
    return S && S->offsets && S->n >= 0 && (S->n == 0 || S->seq) && S->offsets[0] == 0 && S->offsets[S->n] >= 0;
  };
  if (single && pool_ok(A) && pool_ok(B)) {
    if ((rc = sess[0].upload())) return rc;
  }
  auto fail = [&](int r, int64_t e) {
    if (single) cudaStreamSynchronize(ctx->devs[0].stream);
    ctx->err_index = e;
    return r;
  };
  int64_t err = -1;
  if (!hb.ra && ((rc = host_validate(A, err)) || (B != A && (rc = host_validate(B, err))))) return fail(rc, err);
  // seeds and ids (a2), reported with the offending pair index
  for (int64_t t = 0; t < n_pairs; ++t) {
    const xdrop_pair& q = pairs[t];
    const int32_t bid = q.b_id & 0x7fffffff;   // bit 31 = XDROP_PAIR_RC
    if (q.a_id < 0 || q.a_id >= A->n || bid >= B->n) return fail(XDROP_EINVAL, t);
    const int64_t la = A->offsets[q.a_id + 1] - A->offsets[q.a_id];
    const int64_t lb = B->offsets[bid + 1] - B->offsets[bid];
    if (q.a_pos < 0 || q.b_pos < 0 || q.a_pos + (int64_t)p->k > la || q.b_pos + (int64_t)p->k > lb)
      return fail(XDROP_ESEED, t);
  }
  if (single) {   // one device: no partition, no gather
    const auto t0 = std::chrono::steady_clock::now();
    rc = sess[0].run(nullptr, n_pairs);
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    ctx->sched = xdrop_sched_stats{};
    ctx->sched.turns = 1; ctx->sched.span_ms = ms; ctx->sched.busy_ms[0] = ms; ctx->sched.max_concurrent = 1;
    ctx->sched.n_events = 1;
    ctx->trace.assign(1, xdrop_trace_event{0, 0, 0, 0, n_pairs, 0.0, ms});
    if (rc) { ctx->err_index = sess[0].D->err_index; return rc; }
    ctx->st = ctx->devs[0].st;
    return 0;
  }
  // estimated cost per pair (a3): anti-diagonals ~ min prefix + min suffix
  std::vector<int64_t> w((size_t)n_pairs);
  for (int64_t t = 0; t < n_pairs; ++t) {
    const xdrop_pair& q = pairs[t];
    const int32_t bid = q.b_id & 0x7fffffff;
    const int64_t la = A->offsets[q.a_id + 1] - A->offsets[q.a_id];
    const int64_t lb = B->offsets[bid + 1] - B->offsets[bid];
    w[(size_t)t] = std::min<int64_t>(q.a_pos, q.b_pos) + std::min<int64_t>(la - q.a_pos - p->k, lb - q.b_pos - p->k) + 1;
  }
  xdrop_sched_cfg cfg{m, ctx->opts.policy, ctx->opts.n_ranks, ctx->opts.batch_size, ctx->opts.subbatches};
  std::mutex err_mu;
  int first_rc = 0;
  int64_t first_err = -1;
  auto runner = [&](int gpu, const int64_t* idx, int64_t n) -> int {
    int r = sess[(size_t)gpu].run(idx, n);
    if (r) {
      std::lock_guard<std::mutex> lk(err_mu);
      if (!first_rc) { first_rc = r; first_err = sess[(size_t)gpu].D->err_index; }
    }
    return r;
  };
  rc = xdrop_sched_run(cfg, w.data(), n_pairs, runner, &ctx->sched, &ctx->trace);
  if (!rc) rc = first_rc;
  if (rc) { ctx->err_index = first_err; return rc; }
  // stats: every device's turns of this call, summed (times: the maximum over devices and turns)
  ctx->st = xdrop_stats{};
  for (auto& se : sess) stats_add(ctx->st, se.acc);
  return 0;
}

extern "C" int xdrop_align_batch(xdrop_ctx* ctx, const xdrop_seqs* A, const xdrop_seqs* B,
                                 const xdrop_pair* pairs, int64_t n_pairs, const xdrop_params* p,
                                 xdrop_result* out, int64_t* cells_out) {
  if (!ctx || !ctx->alive) return XDROP_ESTATE;
  ctx->err_index = -1;
  int rc = validate_params(p);
  if (rc) return rc;
  if (!A || !B || n_pairs < 0 || (n_pairs > 0 && (!pairs || !out))) return XDROP_EINVAL;
  if (n_pairs > (int64_t)((1u << 30) - 1)) return XDROP_EINVAL;
  // the read pools' H2D copy (the bulk of the call's host->device bytes) is issued first on the
  // single-device path, so the host-side validation runs while the DMA engine copies (pinned
  // caller buffers); a validation error synchronises the stream before returning
  const bool same = A == B || (A->seq == B->seq && A->offsets == B->offsets && A->n == B->n);
  HostBatch hb{A, B, same, pairs, p, flags_of(ctx), out, cells_out};
  hb.n_pairs = n_pairs;
  return align_host(ctx, hb);
}

// ------------------------------------------------------------ registered pools
extern "C" int xdrop_pool_register(xdrop_ctx* ctx, const xdrop_seqs* S, int32_t* pool_id) {
  if (!ctx || !ctx->alive) return XDROP_ESTATE;
  ctx->err_index = -1;
  if (!pool_id) return XDROP_EINVAL;
  int64_t err = -1;
  int rc = host_validate(S, err);
  if (rc) { ctx->err_index = err; return rc; }
  RegPool rp;
  rp.n = S->n;
  rp.len = S->offsets[S->n];
  rp.off.assign(S->offsets, S->offsets + S->n + 1);
  const int m = (int)ctx->devs.size();
  rp.off_d.resize((size_t)m);
  rp.pack_d.resize((size_t)m);
  auto release = [&]() { for (int g = 0; g < m; ++g) { cudaSetDevice(ctx->devs[(size_t)g].dev);
                                                         rp.off_d[(size_t)g].release(); rp.pack_d[(size_t)g].release(); } };
  // slot 0: ASCII H2D + pack (alphabet check); other slots: the packed words device-to-device
  // (NVLink peer copies on a multi-GPU node, 0.25 B per base instead of 1 B of ASCII each)
  const int64_t words = packed_words(rp.len);
  for (int g = 0; g < m && !rc; ++g) {
    DevCtx& D = ctx->devs[(size_t)g];
    if ((rc = cuda_err(cudaSetDevice(D.dev)))) break;
    if ((rc = rp.off_d[(size_t)g].ensure((size_t)(rp.n + 1) * 8))) break;
    if ((rc = rp.pack_d[(size_t)g].ensure((size_t)words * 4))) break;
    if ((rc = cuda_err(cudaMemcpyAsync(rp.off_d[(size_t)g].p, rp.off.data(), (size_t)(rp.n + 1) * 8,
                                       cudaMemcpyHostToDevice, D.stream)))) break;
    if (g == 0) {
      if ((rc = D.asciiA.ensure((size_t)std::max<int64_t>(rp.len, 1)))) break;
      if ((rc = D.bad.ensure(16))) break;
      if ((rc = cuda_err(cudaMemcpyAsync(D.asciiA.p, S->seq, (size_t)rp.len, cudaMemcpyHostToDevice, D.stream)))) break;
      init_bad_kernel<<<1, 32, 0, D.stream>>>(D.bad.as<unsigned long long>());
      int64_t launches = 0;
      if ((rc = pack_pool(D, D.asciiA.as<char>(), rp.len, rp.pack_d[0], D.stream, launches))) break;
      unsigned long long bad[2];
      if ((rc = cuda_err(cudaMemcpyAsync(bad, D.bad.p, 16, cudaMemcpyDeviceToHost, D.stream)))) break;
      if ((rc = cuda_err(cudaStreamSynchronize(D.stream)))) break;
      if (bad[0] != ~0ull) { ctx->err_index = (int64_t)bad[0]; rc = XDROP_EALPHABET; break; }
    } else {
      const DevCtx& D0 = ctx->devs[0];
      rc = cuda_err(cudaMemcpyPeerAsync(rp.pack_d[(size_t)g].p, D.dev, rp.pack_d[0].p, D0.dev, (size_t)words * 4,
                                        D.stream));
      if (!rc) rc = cuda_err(cudaStreamSynchronize(D.stream));
    }
  }
  if (rc) { release(); return rc; }
  rp.alive = true;
  for (size_t i = 0; i < ctx->pools.size(); ++i)
    if (!ctx->pools[i].alive) { ctx->pools[i] = std::move(rp); *pool_id = (int32_t)i; return 0; }
  ctx->pools.push_back(std::move(rp));
  *pool_id = (int32_t)(ctx->pools.size() - 1);
  return 0;
}

extern "C" int xdrop_pool_release(xdrop_ctx* ctx, int32_t pool_id) {
  if (!ctx || !ctx->alive) return XDROP_ESTATE;
  if (pool_id < 0 || pool_id >= (int32_t)ctx->pools.size() || !ctx->pools[(size_t)pool_id].alive) return XDROP_EINVAL;
  RegPool& rp = ctx->pools[(size_t)pool_id];
  for (size_t g = 0; g < ctx->devs.size(); ++g) {
    cudaSetDevice(ctx->devs[g].dev);
    cudaStreamSynchronize(ctx->devs[g].stream);
    rp.off_d[g].release();
    rp.pack_d[g].release();
  }
  rp = RegPool{};
  return 0;
}

extern "C" int xdrop_align_pooled(xdrop_ctx* ctx, int32_t poolA, int32_t poolB, const xdrop_pair* pairs,
                                  int64_t n_pairs, const xdrop_params* p, xdrop_result* out, int64_t* cells_out) {
  if (!ctx || !ctx->alive) return XDROP_ESTATE;
  ctx->err_index = -1;
  int rc = validate_params(p);
  if (rc) return rc;
  auto ok = [&](int32_t id) { return id >= 0 && id < (int32_t)ctx->pools.size() && ctx->pools[(size_t)id].alive; };
  if (!ok(poolA) || !ok(poolB) || n_pairs < 0 || (n_pairs > 0 && (!pairs || !out))) return XDROP_EINVAL;
  if (n_pairs > (int64_t)((1u << 30) - 1)) return XDROP_EINVAL;
  const RegPool& ra = ctx->pools[(size_t)poolA];
  const RegPool& rb = ctx->pools[(size_t)poolB];
  static const char kNoSeq = 0;        // the host bases are not needed again (validated at registration)
  xdrop_seqs A{&kNoSeq, ra.off.data(), ra.n}, B{&kNoSeq, rb.off.data(), rb.n};
  HostBatch hb{&A, poolA == poolB ? &A : &B, poolA == poolB, pairs, p, flags_of(ctx), out, cells_out};
  hb.n_pairs = n_pairs;
  hb.ra = &ra;
  hb.rb = &rb;
  return align_host(ctx, hb);
}

extern "C" int64_t xdrop_last_timeline(const xdrop_ctx* ctx, uint64_t* buf, int64_t cap) {
  if (!ctx) return XDROP_EINVAL;
  const DevCtx& D = ctx->devs[0];
  if (!D.timeline || !D.tl.p) return 0;
  int n = 0;
  if (cudaMemcpy(&n, D.counters.as<int>() + C_TLN, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess) return XDROP_ECUDA;
  n = std::min(n, kTimelineCap);
  if (buf && cap > 0)
    if (cudaMemcpy(buf, D.tl.p, (size_t)std::min<int64_t>(n, cap) * 24, cudaMemcpyDeviceToHost) != cudaSuccess) return XDROP_ECUDA;
  return n;
}

extern "C" int xdrop_last_sched_stats(const xdrop_ctx* ctx, xdrop_sched_stats* st) {
  if (!ctx || !st) return XDROP_EINVAL;
  *st = ctx->sched;
  return 0;
}

extern "C" int64_t xdrop_last_trace(const xdrop_ctx* ctx, xdrop_trace_event* buf, int64_t cap) {
  if (!ctx) return XDROP_EINVAL;
  const int64_t n = (int64_t)ctx->trace.size();
  for (int64_t t = 0; t < n && t < cap && buf; ++t) buf[t] = ctx->trace[(size_t)t];
  return n;
}

// f4 host form: the batch, then the selection kernel on the first device
extern "C" int xdrop_align_multiseed(xdrop_ctx* ctx, const xdrop_seqs* A, const xdrop_seqs* B,
                                     const xdrop_pair* pairs, int64_t n_pairs, const xdrop_params* p,
                                     xdrop_result* out, int64_t* best, int64_t* cells_out) {
  if (!ctx || !ctx->alive) return XDROP_ESTATE;
  if (n_pairs > 0 && !best) return XDROP_EINVAL;
  int rc = xdrop_align_batch(ctx, A, B, pairs, n_pairs, p, out, cells_out);
  if (rc || n_pairs == 0) return rc;
  DevCtx& D = ctx->devs[0];
  CK(cudaSetDevice(D.dev));
  cudaStream_t s = D.stream;
  CKR(D.ms_pairs.ensure((size_t)n_pairs * sizeof(xdrop_pair)));
  CKR(D.ms_res.ensure((size_t)n_pairs * sizeof(xdrop_result)));
  CKR(D.ms_best.ensure((size_t)n_pairs * sizeof(int64_t)));
  CK(cudaMemcpyAsync(D.ms_pairs.p, pairs, (size_t)n_pairs * sizeof(xdrop_pair), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(D.ms_res.p, out, (size_t)n_pairs * sizeof(xdrop_result), cudaMemcpyHostToDevice, s));
  rc = xdrop_best_seed_device(ctx, reinterpret_cast<const xdrop_pair*>(D.ms_pairs.p),
                              reinterpret_cast<const xdrop_result*>(D.ms_res.p), n_pairs,
                              reinterpret_cast<int64_t*>(D.ms_best.p), s);
  if (rc) return rc;
  CK(cudaMemcpyAsync(best, D.ms_best.p, (size_t)n_pairs * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return 0;
}
