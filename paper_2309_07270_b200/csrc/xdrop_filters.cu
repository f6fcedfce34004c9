// xdrop_filters.cu -- the candidate-pair filters next to the alignment.
//
// f2  BELLA's adaptive X-drop acceptance threshold ("An adaptive threshold is used to perform the
//     X-drop alignment", §II).  The paper gives no formula; reading Q12 fixes
//     it: with ov the overlap length the seed implies (the bases of both reads on the seed's diagonal,
//     ov = min(a_pos, b_pos) + min(|A| - a_pos, |B'| - b_pos)), mu = phi * ov the expected score of a
//     true overlap, a pair is kept iff  score >= mu - sqrt(c * mu)  (a Chernoff lower-tail bound,
//     c = 2 ln(1 / gamma) for a false-rejection probability gamma).  Evaluated in IEEE fp64 with
//     explicit round-to-nearest operations (no contraction), the same operations in the oracle, so the
//     integer decision is bit-identical on both sides.
// f4  the k-mer frequency band of ELBA's seeds (LOWER_KMER_FREQ / UPPER_KMER_FREQ, PAPER.md:227,
//     §IV-A): a seed k-mer is reliable iff lower <= its count <= upper, the count being the number
//     of positions of the pool's reads (both strands: canonical k-mers, k <= 31, no k-mer across a
//     read boundary) that hold it.  Three kernels: insert the distinct canonical seed k-mers into an
//     open-addressing table (one per pair), stream every k-mer position of the pool once (coalesced
//     ASCII reads, rolling forward / reverse-complement codes, one table probe per position, L2
//     resident table), gather each pair's count and band flag.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "../../include/xdrop.h"

namespace xf {

constexpr unsigned long long EMPTY = ~0ull;

__device__ __forceinline__ int code2(unsigned ch) {          // A0 C1 G2 T3 (either case); -1 otherwise
  const unsigned u = ch & 0xDFu;
  return u == 'A' ? 0 : u == 'C' ? 1 : u == 'G' ? 2 : u == 'T' ? 3 : -1;
}

__device__ __forceinline__ unsigned long long mix(unsigned long long x) {   // splitmix64 finaliser
  x ^= x >> 31; x *= 0x7fb5d329728ea185ull; x ^= x >> 27; x *= 0x81dadef4bc2dd44dull; x ^= x >> 33;
  return x;
}

__global__ void adaptive_kernel(const int64_t* __restrict__ offA, int64_t nA, const int64_t* __restrict__ offB,
                                int64_t nB, const xdrop_pair* __restrict__ pairs, const xdrop_result* __restrict__ res,
                                int64_t n, double phi, double c, uint8_t* __restrict__ keep,
                                unsigned long long* bad) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const xdrop_pair q = pairs[p];
  const int32_t bid = q.b_id & 0x7fffffff;
  if (q.a_id < 0 || q.a_id >= nA || bid >= nB) { atomicMin(bad, (unsigned long long)p); keep[p] = 0; return; }
  const int64_t la = offA[q.a_id + 1] - offA[q.a_id], lb = offB[bid + 1] - offB[bid];
  if (q.a_pos < 0 || q.b_pos < 0 || q.a_pos > la || q.b_pos > lb) { atomicMin(bad, (unsigned long long)p); keep[p] = 0; return; }
  const int64_t ov = min((int64_t)q.a_pos, (int64_t)q.b_pos) + min(la - q.a_pos, lb - q.b_pos);
  const double mu = __dmul_rn(phi, (double)ov);
  const double t = __dsub_rn(mu, __dsqrt_rn(__dmul_rn(c, mu)));
  keep[p] = (double)res[p].score >= t ? 1 : 0;
}

// canonical code of the k-mer of pool A at [x, x + k) (k <= 31); false on a non-ACGT base
__device__ __forceinline__ bool kmer_at(const char* __restrict__ seq, int64_t x, int k, unsigned long long& canon) {
  unsigned long long f = 0, r = 0;
  for (int t = 0; t < k; ++t) {
    const int cd = code2((unsigned char)seq[x + t]);
    if (cd < 0) return false;
    f = (f << 2) | (unsigned long long)cd;
    r |= (unsigned long long)(3 - cd) << (2 * t);
  }
  canon = f < r ? f : r;
  return true;
}

__global__ void seed_insert_kernel(const char* __restrict__ seq, const int64_t* __restrict__ off, int64_t n_reads,
                                   const xdrop_pair* __restrict__ pairs, int64_t n, int k,
                                   unsigned long long* __restrict__ keys, unsigned mask, int* __restrict__ slot_of,
                                   unsigned long long* bad) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const xdrop_pair q = pairs[p];
  if (q.a_id < 0 || q.a_id >= n_reads) { atomicMin(bad, (unsigned long long)p); slot_of[p] = -1; return; }
  const int64_t la = off[q.a_id + 1] - off[q.a_id];
  unsigned long long canon;
  if (q.a_pos < 0 || q.a_pos + (int64_t)k > la || !kmer_at(seq, off[q.a_id] + q.a_pos, k, canon)) {
    atomicMin(bad, (unsigned long long)p);
    slot_of[p] = -1;
    return;
  }
  unsigned h = (unsigned)mix(canon) & mask;
  for (;;) {
    const unsigned long long prev = atomicCAS(keys + h, EMPTY, canon);
    if (prev == EMPTY || prev == canon) break;
    h = (h + 1) & mask;
  }
  slot_of[p] = (int)h;
}

// every k-mer position of the pool: thread -> (read, chunk of CH start positions), rolling codes
constexpr int CH = 256;
__global__ void kmer_count_kernel(const char* __restrict__ seq, const int64_t* __restrict__ off,
                                  const int64_t* __restrict__ chunk0, int64_t n_reads, int k,
                                  const unsigned long long* __restrict__ keys, unsigned mask,
                                  unsigned* __restrict__ counts) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= chunk0[n_reads]) return;
  // read r of chunk g: chunk0[r] <= g < chunk0[r + 1] (binary search)
  int64_t lo = 0, hi = n_reads;
  while (hi - lo > 1) {
    const int64_t mid = (lo + hi) >> 1;
    if (chunk0[mid] <= g) lo = mid; else hi = mid;
  }
  const int64_t r = lo;
  const int64_t base = off[r], len = off[r + 1] - off[r];
  const int64_t s0 = (g - chunk0[r]) * CH;                 // first start position of this chunk
  const int64_t s1 = min(s0 + CH, len - k + 1);            // past the last
  if (s0 >= s1) return;
  const unsigned long long kmask = (k == 32) ? ~0ull : ((1ull << (2 * k)) - 1ull);
  unsigned long long f = 0, rc = 0;
  int valid = 0;                                            // trailing ACGT bases in the window
  for (int64_t x = s0; x < s1 + k - 1; ++x) {
    const int cd = code2((unsigned char)seq[base + x]);
    if (cd < 0) { valid = 0; f = 0; rc = 0; continue; }
    f = ((f << 2) | (unsigned long long)cd) & kmask;
    rc = (rc >> 2) | ((unsigned long long)(3 - cd) << (2 * (k - 1)));
    if (++valid < k) continue;
    const unsigned long long canon = f < rc ? f : rc;
    unsigned h = (unsigned)mix(canon) & mask;
    for (;;) {
      const unsigned long long key = __ldg(keys + h);
      if (key == canon) { atomicAdd(counts + h, 1u); break; }
      if (key == EMPTY) break;
      h = (h + 1) & mask;
    }
  }
}

__global__ void chunk_kernel(const int64_t* __restrict__ off, int64_t n_reads, int k, int64_t* __restrict__ nch) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n_reads) return;
  const int64_t starts = off[r + 1] - off[r] - k + 1;
  nch[r] = starts > 0 ? (starts + CH - 1) / CH : 0;
}

// exclusive prefix of nch[0..n) into chunk0[0..n] (one block of 1024: a contiguous segment per
// thread, then a shared-memory scan of the segment sums)
__global__ void __launch_bounds__(1024) chunk_scan_kernel(const int64_t* __restrict__ nch, int64_t n,
                                                          int64_t* __restrict__ chunk0) {
  __shared__ int64_t part[1024];
  const int t = threadIdx.x;
  const int64_t seg = (n + 1023) / 1024, a = min(n, t * seg), b = min(n, a + seg);
  int64_t sum = 0;
  for (int64_t i = a; i < b; ++i) sum += nch[i];
  part[t] = sum;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const int64_t v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int64_t run = part[t] - sum;
  for (int64_t i = a; i < b; ++i) { chunk0[i] = run; run += nch[i]; }
  if (t == 1023) chunk0[n] = part[1023];
}

__global__ void gather_kernel(const int* __restrict__ slot_of, int64_t n, const unsigned* __restrict__ counts,
                              int lower, int upper, int32_t* __restrict__ freq, uint8_t* __restrict__ keep) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int s = slot_of[p];
  const int f = s >= 0 ? (int)counts[s] : 0;
  if (freq) freq[p] = f;
  if (keep) keep[p] = (f >= lower && f <= upper) ? 1 : 0;
}

}  // namespace xf

namespace {
int cuda_rc(cudaError_t e) {
  if (e == cudaSuccess) return 0;
  cudaGetLastError();
  return e == cudaErrorMemoryAllocation ? XDROP_ENOMEM : XDROP_ECUDA;
}
}  // namespace

extern "C" int xdrop_adaptive_filter_device(const int64_t* offA, int64_t nA, const int64_t* offB, int64_t nB,
                                            const xdrop_pair* pairs, const xdrop_result* res, int64_t n,
                                            double phi, double c, uint8_t* keep, int64_t* err_index, void* stream) {
  if (err_index) *err_index = -1;
  if (n < 0 || nA < 0 || nB < 0 || !(phi > 0.0) || !(c >= 0.0) || phi > 1e6 || c > 1e12) return XDROP_EINVAL;
  if (n == 0) return 0;
  if (!offA || !offB || !pairs || !res || !keep) return XDROP_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* bad = nullptr;
  int rc = cuda_rc(cudaMallocAsync((void**)&bad, 8, s));
  if (rc) return rc;
  unsigned long long none = ~0ull, got = ~0ull;
  rc = cuda_rc(cudaMemcpyAsync(bad, &none, 8, cudaMemcpyHostToDevice, s));
  if (!rc) {
    xf::adaptive_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(offA, nA, offB, nB, pairs, res, n, phi, c, keep, bad);
    rc = cuda_rc(cudaGetLastError());
  }
  if (!rc) rc = cuda_rc(cudaMemcpyAsync(&got, bad, 8, cudaMemcpyDeviceToHost, s));
  if (!rc) rc = cuda_rc(cudaStreamSynchronize(s));
  cudaFreeAsync(bad, s);
  if (rc) return rc;
  if (got != ~0ull) { if (err_index) *err_index = (int64_t)got; return XDROP_ESEED; }
  return 0;
}

extern "C" int xdrop_seed_kmer_freq_device(const char* seq, const int64_t* off, int64_t n_reads, int64_t len,
                                           const xdrop_pair* pairs, int64_t n, int k, int lower, int upper,
                                           int32_t* freq, uint8_t* keep, int64_t* err_index, void* stream) {
  if (err_index) *err_index = -1;
  if (n < 0 || n_reads < 0 || len < 0 || k < 1 || k > 31 || n > (int64_t)((1u << 30) - 1)) return XDROP_EINVAL;
  if (n == 0) return 0;
  if (!seq || !off || !pairs || (!freq && !keep)) return XDROP_EINVAL;
  cudaStream_t s = (cudaStream_t)stream;
  // table: a power of two >= 2n slots (load factor <= 1/2)
  unsigned cap = 1024;
  while ((int64_t)cap < 2 * n) cap <<= 1;
  const unsigned mask = cap - 1;
  unsigned long long *keys = nullptr, *bad = nullptr;
  unsigned* counts = nullptr;
  int* slot_of = nullptr;
  int64_t *nch = nullptr, *chunk0 = nullptr;
  int rc = 0;
  auto A = [&](void** p, size_t b) { if (!rc) rc = cuda_rc(cudaMallocAsync(p, b, s)); };
  A((void**)&keys, (size_t)cap * 8);
  A((void**)&counts, (size_t)cap * 4);
  A((void**)&slot_of, (size_t)n * 4);
  A((void**)&bad, 8);
  A((void**)&nch, (size_t)std::max<int64_t>(n_reads, 1) * 8);
  A((void**)&chunk0, (size_t)(n_reads + 1) * 8);
  unsigned long long got = ~0ull;
  int64_t n_chunks = 0;
  if (!rc) rc = cuda_rc(cudaMemsetAsync(keys, 0xff, (size_t)cap * 8, s));
  if (!rc) rc = cuda_rc(cudaMemsetAsync(counts, 0, (size_t)cap * 4, s));
  if (!rc) rc = cuda_rc(cudaMemsetAsync(bad, 0xff, 8, s));
  if (!rc) {
    xf::seed_insert_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(seq, off, n_reads, pairs, n, k, keys, mask,
                                                                      slot_of, bad);
    rc = cuda_rc(cudaGetLastError());
  }
  if (!rc && n_reads > 0) {
    // chunks of CH start positions per read and their exclusive prefix, on the device; the count
    // kernel's grid is the bound len / CH + n_reads (threads past chunk0[n_reads] return)
    xf::chunk_kernel<<<(unsigned)((n_reads + 255) / 256), 256, 0, s>>>(off, n_reads, k, nch);
    xf::chunk_scan_kernel<<<1, 1024, 0, s>>>(nch, n_reads, chunk0);
    n_chunks = len / xf::CH + n_reads;
    xf::kmer_count_kernel<<<(unsigned)((n_chunks + 127) / 128), 128, 0, s>>>(seq, off, chunk0, n_reads, k,
                                                                           keys, mask, counts);
    rc = cuda_rc(cudaGetLastError());
  }
  if (!rc) {
    xf::gather_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(slot_of, n, counts, lower, upper, freq, keep);
    rc = cuda_rc(cudaGetLastError());
  }
  if (!rc) rc = cuda_rc(cudaMemcpyAsync(&got, bad, 8, cudaMemcpyDeviceToHost, s));
  if (!rc) rc = cuda_rc(cudaStreamSynchronize(s));
  for (void* p : {(void*)keys, (void*)counts, (void*)slot_of, (void*)bad, (void*)nch, (void*)chunk0})
    if (p) cudaFreeAsync(p, s);
  cudaStreamSynchronize(s);
  if (rc) return rc;
  if (got != ~0ull) { if (err_index) *err_index = (int64_t)got; return XDROP_ESEED; }
  return 0;
}
