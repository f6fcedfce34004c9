// Scratch: one packed anti-diagonal step, FMA-pipe adds vs 16x2 adds, on random realistic states.
#include <cstdio>
#include "../paper_2309_07270_b200/csrc/xdrop_kernels.cuh"
using namespace xk;
__device__ uint32_t rnd(uint32_t& s) { s ^= s << 13; s ^= s >> 17; s ^= s << 5; return s; }
template <int PAR>
__global__ void unit(Problem P, int* nbad, int* out) {
  uint32_t seed = 1234567u + 7919u * (blockIdx.x * blockDim.x + threadIdx.x);
  for (int it = 0; it < 200; ++it) {
    Band16<32> B;
    pk_keys<32>(B, 1, 0, 0);
    for (int u = 0; u < 16; ++u) {
      uint32_t e = 0, o = 0;
      for (int h = 0; h < 2; ++h) {
        const uint32_t tc = 31 - (u + 16 * h);
        uint32_t ve = (rnd(seed) % 3 == 0) ? (0xC000u | ((rnd(seed) & 7) << 5) | tc) : (((rnd(seed) % 20) << 5) | tc);
        uint32_t vo = (rnd(seed) % 3 == 0) ? (0xC000u | ((rnd(seed) & 7) << 5) | tc) : (((rnd(seed) % 20) << 5) | tc);
        e |= ve << (16 * h); o |= vo << (16 * h);
      }
      B.E[u] = e; B.O[u] = o;
    }
    B.A0 = rnd(seed); B.A1 = rnd(seed); B.B0 = rnd(seed); B.B1 = rnd(seed);
    B.thrD1 = 1000; B.thrD = B.thrD1 + 1 + rnd(seed) % 3; B.thrN = B.thrD + 1 + rnd(seed) % 3;
    Band16<32> B2 = B;
    const uint32_t by = (rnd(seed) & 1) ? 0u : rnd(seed);     // cells beyond the matrix (pk_beyond)
    uint32_t ch1[2], ch2[2];
    uint32_t k1, k2;
    if (PAR == 0) {
      k1 = pk_cells<32, 0, false>(B.E, B.O, B, 1, 0, by, P, ch1);
      k2 = pk_cells<32, 0, true>(B2.E, B2.O, B2, 1, 0, by, P, ch2);
    } else {
      k1 = pk_cells<32, 1, false>(B.O, B.E, B, 1, 0, by, P, ch1);
      k2 = pk_cells<32, 1, true>(B2.O, B2.E, B2, 1, 0, by, P, ch2);
    }
    bool bad = k1 != k2 || ch1[0] != ch2[0] || ch1[1] != ch2[1];
    for (int u = 0; u < 16; ++u) bad |= (B.E[u] != B2.E[u]) || (B.O[u] != B2.O[u]);
    if (bad) {
      const int i = atomicAdd(nbad, 1);
      if (i < 4) {
        for (int u = 0; u < 16; ++u) {
          const uint32_t a = PAR ? B.O[u] : B.E[u], b = PAR ? B2.O[u] : B2.E[u];
          if (a != b) printf("PAR %d u %d: 16x2 %08x fma %08x  thr %d %d %d\n", PAR, u, a, b, B.thrD1, B.thrD, B.thrN);
        }
        printf("keys %08x %08x ch %08x %08x / %08x %08x\n", k1, k2, ch1[0], ch1[1], ch2[0], ch2[1]);
      }
    }
  }
}
int main() {
  Problem P{}; P.M = 1; P.mu = -1; P.g = -1; P.X = 15; P.keym = 128; P.pkM = 32 * 3; P.pkU = 32 * 1;
  int* nb; cudaMallocManaged(&nb, 4); *nb = 0;
  unit<0><<<64, 128>>>(P, nb, nullptr); cudaDeviceSynchronize(); printf("PAR0 bad %d\n", *nb); *nb = 0;
  unit<1><<<64, 128>>>(P, nb, nullptr); cudaDeviceSynchronize(); printf("PAR1 bad %d\n", *nb);
  return 0;
}
