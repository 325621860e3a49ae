// throughput of 32-bit integer multiply flavours on sm_100a (independent chains)
#include <cstdio>
#include <cstdint>
template <int KIND>
__global__ void k(uint32_t *out, uint32_t a, uint32_t b, int iters) {
  uint32_t x[8];
  uint64_t y[8];
  for (int i = 0; i < 8; i++) { x[i] = threadIdx.x + i; y[i] = x[i]; }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      if (KIND == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
      if (KIND == 1) asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(y[i]) : "r"((uint32_t)y[i]), "r"(a));
      if (KIND == 2) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(x[i]) : "r"(a), "r"(b));
      if (KIND == 3) asm volatile("add.u32 %0, %0, %1;" : "+r"(x[i]) : "r"(a));
      if (KIND == 4) { double d = (double)x[i]; asm volatile("fma.rn.f64 %0, %0, %0, %0;" : "+d"(d)); x[i] = (uint32_t)(long long)d; }
      if (KIND == 5) asm volatile("mul.lo.u64 %0, %0, %1;" : "+l"(y[i]) : "l"((uint64_t)a * 77 + 3));
      if (KIND == 6) asm volatile("mul.hi.u64 %0, %0, %1;" : "+l"(y[i]) : "l"((uint64_t)a * 77 + 3));
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; i++) s ^= x[i] ^ (uint32_t)y[i];
  if (s == 0x12345) out[0] = s;
}
template <int KIND>
void run(const char *name) {
  uint32_t *o; cudaMalloc(&o, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  k<KIND><<<sms * 8, 256>>>(o, 3, 5, 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 4096;
  cudaEventRecord(a); k<KIND><<<sms * 8, 256>>>(o, 3, 5, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = (double)sms * 8 * 256 * 8 * iters;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%-12s %8.2f Gop/s  %6.1f ops/clk/SM (at %d MHz nominal)\n", name, ops / ms / 1e6, ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
}
int main() {
  run<0>("IMAD"); run<1>("IMAD.WIDE"); run<2>("IMAD.HI"); run<3>("IADD"); run<4>("DFMA(+cvt)"); run<5>("mul.lo.u64"); run<6>("mul.hi.u64");
  return 0;
}
