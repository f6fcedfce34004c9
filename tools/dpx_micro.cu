// Throughput probe of the 16x2 DP instructions vs 32-bit integer ops (8 independent chains/thread).
#include <cstdio>
#include <cuda_runtime.h>
template <int OP>
__global__ void kern(int* out, int iters, int s0) {
  int a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = threadIdx.x * 7 + c + s0;
  const int b = s0 * 3 + 1, e = s0 ^ 0x5555;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (OP == 0) a[c] = __vimax3_s32(a[c], b, e + c);
      if (OP == 1) a[c] = __vmaxs2(a[c], b + c);
      if (OP == 2) a[c] = __viaddmax_s16x2(a[c], b, e + c);
      if (OP == 3) a[c] = __vimax3_s16x2(a[c], b, e + c);
      if (OP == 4) a[c] = __byte_perm(a[c], e, 0xBB99 ^ c);
      if (OP == 5) a[c] = (a[c] & ~b) | (e & (b + c));
      if (OP == 6) a[c] = a[c] * b + e;
      if (OP == 7) a[c] = __viaddmax_s16x2_relu(a[c], b, e + c);
      if (OP == 8) a[c] = a[c] + b + c;
    }
  }
  int r = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) r ^= a[c];
  if (r == 0x12345) out[0] = r;
}
int main() {
  int* o; cudaMalloc(&o, 4);
  cudaEvent_t t0, t1; cudaEventCreate(&t0); cudaEventCreate(&t1);
  const char* nm[] = {"vimax3_s32", "vmaxs2", "viaddmax_s16x2", "vimax3_s16x2", "prmt", "lop3", "imad", "viaddmax_relu", "iadd3"};
  int iters = 20000, blocks = 148 * 8, th = 256;
  for (int op = 0; op < 9; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(t0);
      switch (op) {
        case 0: kern<0><<<blocks, th>>>(o, iters, 1); break; case 1: kern<1><<<blocks, th>>>(o, iters, 1); break;
        case 2: kern<2><<<blocks, th>>>(o, iters, 1); break; case 3: kern<3><<<blocks, th>>>(o, iters, 1); break;
        case 4: kern<4><<<blocks, th>>>(o, iters, 1); break; case 5: kern<5><<<blocks, th>>>(o, iters, 1); break;
        case 6: kern<6><<<blocks, th>>>(o, iters, 1); break; case 7: kern<7><<<blocks, th>>>(o, iters, 1); break;
        case 8: kern<8><<<blocks, th>>>(o, iters, 1); break;
      }
      cudaEventRecord(t1); cudaEventSynchronize(t1);
      float ms; cudaEventElapsedTime(&ms, t0, t1);
      double ops = double(blocks) * th * iters * 8;
      if (rep) printf("%-16s %8.3f ms  %7.2f Tops/s  %6.1f ops/clk/SM@1.965GHz\n", nm[op], ms, ops / ms / 1e9, ops / ms / 1e-3 / 148 / 1.965e9);
    }
  }
  return 0;
}
