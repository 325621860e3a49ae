// cgb_masks.cuh -- the MPC channel's mask stream on the device.
//
// The reference draws every server mask as MpcChannel.sample_mask(n) =
// rng.integers(0, p, n) on numpy's PCG64 (/root/reference/pkg/src/cryptogen/
// nonlinear.py:66-75, :86-87): PCG64 XSL-RR 128/64 (state <- state * M + inc,
// output from the new state), 32-bit halves taken low half first with the
// half-word buffer kept in the generator (has_uint32 / uinteger), and Lemire's
// bounded multiply with rejection: u * p = m, accept iff (m mod 2^32) >=
// (2^32 - p) mod p, value m >> 32.  A channel's successive sample_mask calls
// therefore consume ONE continuous stream of 32-bit words, and its masks are
// consecutive runs of the accepted values.
//
// On the device: every thread jumps ahead to its chunk of the 64-bit output
// stream (LCG advance by repeated squaring) and writes 32-bit values + accept
// flags; an exclusive scan of the flags numbers the accepted values; a scatter
// places accepted value k of channel c at word k % n of that channel's
// (k / n)-th item.  The host then advances each channel's numpy state by the
// number of outputs consumed (tests/test_gpu_masks.py: >= 10^6 draws per
// channel equal to numpy's).
#pragma once

#include <stdint.h>

#include <cub/device/device_scan.cuh>

namespace cgbmask {

typedef uint64_t u64;
typedef uint32_t u32;

struct U128 {
  u64 hi, lo;
};
__host__ __device__ __forceinline__ U128 mul128(U128 a, U128 b) {
#ifdef __CUDA_ARCH__
  const u64 h = __umul64hi(a.lo, b.lo);
#else
  const u64 h = (u64)(((unsigned __int128)a.lo * b.lo) >> 64);
#endif
  return {h + a.lo * b.hi + a.hi * b.lo, a.lo * b.lo};
}
__host__ __device__ __forceinline__ U128 add128(U128 a, U128 b) {
  const u64 lo = a.lo + b.lo;
  return {a.hi + b.hi + (lo < a.lo ? 1ull : 0ull), lo};
}
// numpy's PCG_DEFAULT_MULTIPLIER_128
__host__ __device__ __forceinline__ U128 pcg_mult() { return {2549297995355413924ull, 4865540595714422341ull}; }
// state after `delta` steps of state <- state * M + inc (Brown's LCG jump-ahead)
__host__ __device__ inline U128 pcg_advance(U128 state, U128 inc, u64 delta) {
  U128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = {0, 1}, acc_plus = {0, 0};
  while (delta) {
    if (delta & 1) {
      acc_mult = mul128(acc_mult, cur_mult);
      acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
    }
    cur_plus = mul128(add128(cur_mult, {0, 1}), cur_plus);
    cur_mult = mul128(cur_mult, cur_mult);
    delta >>= 1;
  }
  return add128(mul128(acc_mult, state), acc_plus);
}
__host__ __device__ __forceinline__ u64 pcg_output(U128 s) {
  const u64 x = s.hi ^ s.lo;
  const unsigned rot = (unsigned)(s.hi >> 58);
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

struct Chan {
  U128 state, inc;
  u32 has_u32, uinteger;
  u64 base;    // offset of this channel's 32-bit stream in the concatenated buffers
  u64 halves;  // stream length (32-bit words)
  u64 need;    // accepted values needed (items x n)
  u64 item0;   // offset of this channel's items in the by-channel item table
};

constexpr int GEN_CHUNK = 16;  // 64-bit outputs per thread

// one thread: GEN_CHUNK consecutive 64-bit outputs of one channel -> 2 * GEN_CHUNK halves
__global__ void k_pcg_gen(const Chan *ch, int nchan, const u64 *thread_base, u32 *val, u32 *flag, u32 p, u32 thr) {
  const u64 gt = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  // channel of this thread: thread_base[c] = first global thread of channel c
  int c = 0;
  while (c + 1 < nchan && gt >= thread_base[c + 1]) c++;
  if (gt >= thread_base[nchan]) return;
  const Chan C = ch[c];
  const u64 t = gt - thread_base[c];
  const u64 first_out = t * GEN_CHUNK;
  const u64 off = C.has_u32 ? 1 : 0;  // stream half 0 is the buffered word when present
  U128 s = pcg_advance(C.state, C.inc, first_out);
  const U128 M = pcg_mult();
  if (t == 0 && C.has_u32) {
    const u64 m = (u64)C.uinteger * p;
    val[C.base] = (u32)(m >> 32);
    flag[C.base] = (u32)m >= thr;
  }
#pragma unroll 4
  for (int k = 0; k < GEN_CHUNK; k++) {
    s = add128(mul128(s, M), C.inc);
    const u64 o = pcg_output(s);
    const u64 h = off + 2 * (first_out + k);
#pragma unroll
    for (int e = 0; e < 2; e++) {
      if (h + e >= C.halves) break;
      const u32 u = e ? (u32)(o >> 32) : (u32)o;
      const u64 m = (u64)u * p;
      val[C.base + h + e] = (u32)(m >> 32);
      flag[C.base + h + e] = (u32)m >= thr;
    }
  }
}

// accepted value k of channel c -> word k % n of item items[item0 + k / n]; records the
// stream position of the last needed value (the host advances the state from it)
__global__ void k_pcg_scatter(const Chan *ch, int nchan, const u32 *idx /*exclusive scan*/, const u32 *val,
                              const u32 *flag, u64 total, const u32 *items, int n, u64 *out /*[item][n]*/,
                              long long *last) {
  const u64 h = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= total || !flag[h]) return;
  int c = 0;
  while (c + 1 < nchan && h >= ch[c + 1].base) c++;
  const u64 k = idx[h] - idx[ch[c].base];
  if (k >= ch[c].need) return;
  out[(u64)items[ch[c].item0 + k / n] * n + (k % n)] = val[h];
  if (k + 1 == ch[c].need) last[c] = (long long)(h - ch[c].base);
}

}  // namespace cgbmask
