// Modular-product throughput on sm_100a: the FP64 error-free product the NTTs use,
// the 64-bit integer Shoup product, a hybrid (FP64 quotient, integer remainder), and
// FP64 + integer chains interleaved in one thread (do the two pipes overlap?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mix_rates mix_rates.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ double fp_mulmod(double a, double w, double wq, double q) {
  const double hi = a * w;
  const double lo = fma(a, w, -hi);
  return fma(-rint(a * wq), q, hi) + lo;
}
__device__ __forceinline__ double fp_reduce(double x, double q, double qinv) { return fma(-rint(x * qinv), q, x); }

// A: FP64 chains (value kept reduced so it stays exact)
__global__ void k_fp(double *out, double q, double w, int iters) {
  const double wq = w / q, qinv = 1.0 / q;
  double x[8];
  for (int i = 0; i < 8; i++) x[i] = (double)((threadIdx.x * 77 + i * 13) % 1000003);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) x[i] = fp_mulmod(x[i], w, wq, q);
  }
  double s = 0;
  for (int i = 0; i < 8; i++) s += fp_reduce(x[i], q, qinv);
  if (s == 1.2345) out[0] = s;
}
// C: integer Shoup chains
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
// B: hybrid -- quotient on the FP64 pipe, exact remainder in 64-bit integers
__global__ void k_hybrid(uint64_t *out, uint64_t q, uint64_t w, double wq, int iters) {
  int64_t x[8];
  for (int i = 0; i < 8; i++) x[i] = (int64_t)((threadIdx.x * 8 + i + 1) % q);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) {
      const int64_t qt = __double2ll_rn((double)x[i] * wq);
      int64_t r = x[i] * (int64_t)w - qt * (int64_t)q;  // exact: |r| < q (low 64 bits)
      x[i] = r < 0 ? r + (int64_t)q : r;
    }
  }
  int64_t s = 0;
  for (int i = 0; i < 8; i++) s ^= x[i];
  if (s == 12345) out[0] = (uint64_t)s;
}
// A + C interleaved: 4 FP64 chains and 4 Shoup chains per thread
__global__ void k_mix(double *out, double q, double w, uint64_t qi, uint64_t wi, uint64_t wsh, int iters) {
  const double wq = w / q, qinv = 1.0 / q;
  double x[4];
  uint64_t y[4];
  for (int i = 0; i < 4; i++) {
    x[i] = (double)((threadIdx.x * 77 + i * 13) % 1000003);
    y[i] = (threadIdx.x * 8 + i + 1) % qi;
  }
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++) {
      x[i] = fp_mulmod(x[i], w, wq, q);
      uint64_t hi = __umul64hi(y[i], wsh);
      uint64_t r = y[i] * wi - hi * qi;
      y[i] = r >= qi ? r - qi : r;
    }
  }
  double s = 0;
  uint64_t t = 0;
  for (int i = 0; i < 4; i++) {
    s += fp_reduce(x[i], q, qinv);
    t ^= y[i];
  }
  if (s == 1.2345 || t == 12345) out[0] = s + (double)t;
}

int main() {
  const uint64_t q = 562949953421313ull;  // a 49-bit prime = 1 mod 2^32 (2^49 - 2^32 + 1 is not; any odd works for rates)
  const double qd = (double)q;
  const uint64_t w = 123456789012345ull % q;
  const uint64_t wsh = (uint64_t)(((unsigned __int128)w << 64) / q);
  double *dout;
  uint64_t *uout;
  cudaMalloc(&dout, 8);
  cudaMalloc(&uout, 8);
  int dev;
  cudaGetDevice(&dev);
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, dev);
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char *name, int chains, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double ops = (double)blocks * threads * iters * chains;
    printf("{\"kernel\": \"%s\", \"modmul_per_s\": %.4g, \"ms\": %.3f}\n", name, ops / (ms * 1e-3), ms);
  };
  run("fp64_errorfree", 8, [&] { k_fp<<<blocks, threads>>>(dout, qd, (double)w, iters); });
  run("int64_shoup", 8, [&] { k_shoup<<<blocks, threads>>>(uout, q, w, wsh, iters); });
  run("hybrid_fpquot_intrem", 8, [&] { k_hybrid<<<blocks, threads>>>(uout, q, w, (double)w / qd, iters); });
  run("fp64_plus_shoup_interleaved", 8, [&] { k_mix<<<blocks, threads>>>(dout, qd, (double)w, q, w, wsh, iters); });
  return 0;
}
