// FP64 throughput on sm_100a and an exact FP64 modmul (q < 2^50) vs the 64-bit Shoup modmul
#include <cstdint>
#include <cstdio>
__global__ void k_dfma(double *out, double a, double b, int iters) {
  double x[8];
  for (int i = 0; i < 8; i++) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fma(x[i], a, b);
  }
  double s = 0;
  for (int i = 0; i < 8; i++) s += x[i];
  if (s == 1.2345) out[0] = s;
}
// r = a*w mod q for a < 4q, q < 2^50, exact; w constant with wq = w/q
__device__ __forceinline__ double modmul_fp(double a, double w, double wq, double q) {
  double hi = a * w;
  double lo = fma(a, w, -hi);              // exact residual
  double qt = rint(a * wq);                 // quotient estimate
  double r = fma(-qt, q, hi) + lo;          // exact (|.| < 2^53)
  r = r < 0 ? r + q : r;
  return r >= q ? r - q : r;
}
__global__ void k_fpmod(double *out, double q, double w, int iters) {
  double x[8];
  const double wq = w / q;
  for (int i = 0; i < 8; i++) x[i] = (double)((threadIdx.x * 77 + i * 13) % 1000003);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = modmul_fp(x[i], w, wq, q);
  }
  double s = 0;
  for (int i = 0; i < 8; i++) s += x[i];
  if (s == 1.2345) out[0] = s;
}
__global__ void k_shoup(uint64_t *out, uint64_t q, uint64_t w, uint64_t wsh, int iters) {
  uint64_t x[8];
  for (int i = 0; i < 8; i++) x[i] = (threadIdx.x * 8 + i + 1) % q;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      uint64_t hi = __umul64hi(x[i], wsh);
      uint64_t r = x[i] * w - hi * q;
      x[i] = r >= q ? r - q : r;
    }
  }
  uint64_t s = 0;
  for (int i = 0; i < 8; i++) s ^= x[i];
  if (s == 12345) out[0] = s;
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *o; cudaMalloc(&o, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 2048, blocks = sms * 8, thr = 256;
  const double ops = (double)blocks * thr * 8 * iters;
  float ms;
  k_dfma<<<blocks, thr>>>(o, 1.0000001, 1e-9, 16);
  cudaEventRecord(a); k_dfma<<<blocks, thr>>>(o, 1.0000001, 1e-9, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("DFMA            %9.1f Gop/s  %6.1f /clk/SM @1965\n", ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.965e9);
  const double q = 1125899906826241.0;  // a prime-ish 50-bit value, rate test only
  k_fpmod<<<blocks, thr>>>(o, q, 987654321987.0, 16);
  cudaEventRecord(a); k_fpmod<<<blocks, thr>>>(o, q, 987654321987.0, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("fp64 modmul     %9.1f Gmodmul/s\n", ops / ms / 1e6);
  uint64_t qq = 0xfffffa000000001ull, w = 0x123456789abcdull;
  uint64_t wsh = (uint64_t)(((unsigned __int128)w << 64) / qq);
  k_shoup<<<blocks, thr>>>((uint64_t *)o, qq, w, wsh, 16);
  cudaEventRecord(a); k_shoup<<<blocks, thr>>>((uint64_t *)o, qq, w, wsh, iters); cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("u64 Shoup       %9.1f Gmodmul/s\n", ops / ms / 1e6);
  return 0;
}
