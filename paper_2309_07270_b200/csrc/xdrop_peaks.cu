// xdrop_peaks.cu -- measured single-pipe integer issue rates of the device (the roofline
// denominators of bench.py; SURVEY.md §8(d) "P_int = measured INT32 ops/s (N10)").
//
// Each probe is a kernel whose inner loop is ONE instruction kind in 8 independent dependency
// chains per thread (4-cycle latency, 2-cycle issue per SMSP on the ALU and FMA pipes:
// B300_MICROARCH.md "Pipe rates"), 32x unrolled, with every operand register-resident so ptxas
// cannot fold or re-route it.  tools/peaks_sass.sh (cuobjdump) checks that the loop bodies are the
// named SASS instructions only.  Rates are reported per probe as
//   lane_ops_per_s  = executed thread-instructions / second (CUDA events around the launch)
//   inst_per_clk_sm = warp-instructions per SM per SM-clock (clock64 deltas of every block)
// so the caller can state both the clock-independent pipe width and the rate at the clock the
// device actually ran.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/xdrop.h"

namespace {

constexpr int kChains = 8;
constexpr int kUnroll = 32;

enum Probe { P_VMNMX3_S16X2 = 0, P_VMNMX3_S32, P_LOP3, P_IADD3, P_IMAD, P_MIX_S16X2_IMAD, P_N };

template <int OP>
__device__ __forceinline__ uint32_t op1(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  if constexpr (OP == P_VMNMX3_S16X2) {
    d = __vimax3_s16x2(a, b, c);                                     // VIMNMX3.S16x2 (ALU)
  } else if constexpr (OP == P_VMNMX3_S32) {
    d = (uint32_t)__vimax3_s32((int)a, (int)b, (int)c);               // VIMNMX3 (ALU)
  } else if constexpr (OP == P_LOP3) {
    asm volatile("lop3.b32 %0, %1, %2, %3, 0x96;" : "=r"(d) : "r"(a), "r"(b), "r"(c));   // LOP3 (ALU)
  } else if constexpr (OP == P_IADD3) {
    asm volatile("{ .reg .u32 t; add.u32 t, %1, %2; add.u32 %0, t, %3; }" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  } else {
    asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));          // IMAD (FMA)
  }
  return d;
}

template <int OP>
__global__ void __launch_bounds__(256) peak_kernel(int iters, uint32_t seed, uint32_t* sink,
                                                   long long* cycles) {
  uint32_t x[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) x[c] = seed * (c + 3) + threadIdx.x;
  const uint32_t b = seed ^ 0x9e3779b9u, cc = seed + 0x7f4a7c15u;   // run-time operands
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
      for (int c = 0; c < kChains; ++c) {
        if constexpr (OP == P_MIX_S16X2_IMAD) {
          // alternate the ALU and FMA pipes: both probes' instructions, one chain each
          x[c] = (c & 1) ? op1<P_IMAD>(x[c], b, cc) : op1<P_VMNMX3_S16X2>(x[c], b, cc);
        } else {
          x[c] = op1<OP>(x[c], b, cc);
        }
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) r ^= x[c];
  if (r == 0x12345678u) *sink = r;                                  // keeps the chains live
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int OP>
int run_probe(int sms, cudaStream_t s, uint32_t* sink, long long* cyc_d, long long* cyc_h, cudaEvent_t e0,
              cudaEvent_t e1, double* lane_ops_per_s, double* inst_per_clk_sm) {
  const int threads = 256, bps = 4, blocks = sms * bps, iters = 512;
  double best = 1e30, ipc = 0;
  for (int rep = 0; rep < 4; ++rep) {
    if (cudaEventRecord(e0, s) != cudaSuccess) return XDROP_ECUDA;
    peak_kernel<OP><<<blocks, threads, 0, s>>>(iters, 0x2545F491u + rep, sink, cyc_d);
    if (cudaEventRecord(e1, s) != cudaSuccess) return XDROP_ECUDA;
    if (cudaEventSynchronize(e1) != cudaSuccess) return XDROP_ECUDA;
    if (cudaGetLastError() != cudaSuccess) return XDROP_ECUDA;
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (cudaMemcpy(cyc_h, cyc_d, sizeof(long long) * blocks, cudaMemcpyDeviceToHost) != cudaSuccess)
      return XDROP_ECUDA;
    if (rep == 0) continue;                                            // warm-up
    long long mx = 0;
    for (int b = 0; b < blocks; ++b) mx = cyc_h[b] > mx ? cyc_h[b] : mx;
    const double warp_inst_per_sm = (double)bps * (threads / 32) * iters * kUnroll * kChains;
    if (ms < best) {
      best = ms;
      ipc = warp_inst_per_sm / (double)mx;
    }
  }
  const double lane_ops = (double)blocks * threads * iters * kUnroll * kChains;
  *lane_ops_per_s = lane_ops / (best * 1e-3);
  *inst_per_clk_sm = ipc;
  return 0;
}

}  // namespace

// out[2*p] = thread-instructions per second, out[2*p+1] = warp-instructions per SM per clock, for
// probes p = 0 VIMNMX3.S16x2, 1 VIMNMX3 (s32), 2 LOP3, 3 IADD3, 4 IMAD, 5 VIMNMX3.S16x2 + IMAD mix.
extern "C" int xdrop_alu_peaks(int device, double* out, int n_out) {
  if (!out || n_out < 2 * P_N) return XDROP_EINVAL;
  if (cudaSetDevice(device) != cudaSuccess) { cudaGetLastError(); return XDROP_ENODEV; }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return XDROP_ECUDA;
  const int sms = prop.multiProcessorCount, blocks = sms * 4;
  uint32_t* sink = nullptr;
  long long* cyc_d = nullptr;
  long long* cyc_h = new long long[blocks];
  cudaStream_t s = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  int rc = 0;
  if (cudaMalloc(&sink, 4) != cudaSuccess || cudaMalloc(&cyc_d, sizeof(long long) * blocks) != cudaSuccess ||
      cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
    rc = XDROP_ECUDA;
  if (!rc) rc = run_probe<P_VMNMX3_S16X2>(sms, s, sink, cyc_d, cyc_h, e0, e1, &out[0], &out[1]);
  if (!rc) rc = run_probe<P_VMNMX3_S32>(sms, s, sink, cyc_d, cyc_h, e0, e1, &out[2], &out[3]);
  if (!rc) rc = run_probe<P_LOP3>(sms, s, sink, cyc_d, cyc_h, e0, e1, &out[4], &out[5]);
  if (!rc) rc = run_probe<P_IADD3>(sms, s, sink, cyc_d, cyc_h, e0, e1, &out[6], &out[7]);
  if (!rc) rc = run_probe<P_IMAD>(sms, s, sink, cyc_d, cyc_h, e0, e1, &out[8], &out[9]);
  if (!rc) rc = run_probe<P_MIX_S16X2_IMAD>(sms, s, sink, cyc_d, cyc_h, e0, e1, &out[10], &out[11]);
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (s) cudaStreamDestroy(s);
  if (sink) cudaFree(sink);
  if (cyc_d) cudaFree(cyc_d);
  delete[] cyc_h;
  return rc;
}
