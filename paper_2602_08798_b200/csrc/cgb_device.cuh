// cgb_device.cuh -- device arithmetic for the sm_100a RNS-BFV backend:
// 64-bit Shoup / Barrett modular multiplication on the integer pipe,
// ChaCha20 sampling, and the shared-memory negacyclic NTT.
//
// Words are uint64 residues of primes q < 2^62 (Q: 60-bit, P/B: 61-bit).
// Every kernel here produces canonical residues in [0, q) so results are
// bit-identical to the CPU restatement in oracle/rnsbfv.c.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cgb {

typedef uint64_t u64;
typedef int64_t i64;
typedef unsigned int u32;

constexpr int MAXL = 16;        // max limbs of Q
constexpr int MAXMOD = 2 * MAXL + 3;

struct ModTab {
  u64 q;        // modulus
  u64 mu;       // floor(2^(2*bits) / q)      (Barrett)
  u64 r64;      // 2^64 mod q
  u64 ninv, ninv_sh;
  const u64 *tw, *tw_sh, *itw, *itw_sh;  // bit-reversed psi powers + Shoup companions
  int bits;
  int pad_;
};

// ---------------------------------------------------------------------------
// scalar modular arithmetic
// ---------------------------------------------------------------------------
__device__ __forceinline__ u64 add_mod(u64 a, u64 b, u64 q) {
  u64 s = a + b;
  return s >= q ? s - q : s;
}
__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }

// a * w mod q with w' = floor(w 2^64 / q); any a < 2^64, result in [0, q)
__device__ __forceinline__ u64 mul_shoup(u64 a, u64 w, u64 wsh, u64 q) {
  u64 hi = __umul64hi(a, wsh);
  u64 r = a * w - hi * q;
  return r >= q ? r - q : r;
}

// a * b mod q, a, b < q < 2^62 (Barrett with mu = floor(2^(2k)/q), k = bits(q))
__device__ __forceinline__ u64 mul_mod(u64 a, u64 b, u64 q, u64 mu, int bits) {
  u64 lo = a * b, hi = __umul64hi(a, b);
  const int s = bits - 1, s2 = bits + 1;
  u64 xs = (hi << (64 - s)) | (lo >> s);
  u64 ph = __umul64hi(xs, mu), pl = xs * mu;
  u64 qh = (ph << (64 - s2)) | (pl >> s2);
  u64 r = lo - qh * q;
  if (r >= q) r -= q;
  if (r >= q) r -= q;
  return r;
}
__device__ __forceinline__ u64 mul_mod(u64 a, u64 b, const ModTab &m) { return mul_mod(a, b, m.q, m.mu, m.bits); }

// v mod q for v < 4q
__device__ __forceinline__ u64 reduce4(u64 v, u64 q) {
  if (v >= q) v -= q;
  if (v >= q) v -= q;
  if (v >= q) v -= q;
  return v;
}
// residue in limb q of the centred representative of v in [0, qs)
__device__ __forceinline__ u64 centred_to(u64 v, u64 qs, u64 q) {
  if (v <= (qs >> 1)) return reduce4(v, q);
  u64 n = reduce4(qs - v, q);
  return n ? q - n : 0;
}

// ---------------------------------------------------------------------------
// ChaCha20 (DJB layout, 64-bit counter + 64-bit nonce)
// ---------------------------------------------------------------------------
struct ChaKey {
  u32 k[8];
};
__device__ __forceinline__ u32 rotl32(u32 x, int n) { return __funnelshift_l(x, x, n); }
#define CGB_QR(a, b, c, d)                                                      \
  a += b; d ^= a; d = rotl32(d, 16); c += d; b ^= c; b = rotl32(b, 12);         \
  a += b; d ^= a; d = rotl32(d, 8);  c += d; b ^= c; b = rotl32(b, 7);

__device__ __forceinline__ void chacha_block(const ChaKey &key, u64 ctr, u64 nonce, u32 out[16]) {
  u32 s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u, key.k[0], key.k[1], key.k[2],
               key.k[3],    key.k[4],    key.k[5],    key.k[6],    key.k[7], (u32)ctr,
               (u32)(ctr >> 32), (u32)nonce, (u32)(nonce >> 32)};
  u32 x[16];
#pragma unroll
  for (int i = 0; i < 16; i++) x[i] = s[i];
#pragma unroll
  for (int i = 0; i < 10; i++) {
    CGB_QR(x[0], x[4], x[8], x[12]) CGB_QR(x[1], x[5], x[9], x[13])
    CGB_QR(x[2], x[6], x[10], x[14]) CGB_QR(x[3], x[7], x[11], x[15])
    CGB_QR(x[0], x[5], x[10], x[15]) CGB_QR(x[1], x[6], x[11], x[12])
    CGB_QR(x[2], x[7], x[8], x[13]) CGB_QR(x[3], x[4], x[9], x[14])
  }
#pragma unroll
  for (int i = 0; i < 16; i++) out[i] = x[i] + s[i];
}

// ---------------------------------------------------------------------------
// negacyclic NTT, one CTA per (poly, limb), whole vector in shared memory.
// Forward: Cooley-Tukey, natural in -> bit-reversed out (a[k] = A(psi^(2brev(k)+1))).
// Inverse: Gentleman-Sande, bit-reversed in -> natural out, times N^-1.
// Each thread keeps E = 2^R words in registers and runs R radix-2 stages on
// them between shared-memory exchanges (logN/R exchanges in total).
// ---------------------------------------------------------------------------
constexpr int NTT_MAXSUB = 160;

struct NttJob {
  u64 *base;                 // contiguous items: base + item * item_stride
  u64 *const *items;         // or per-item pointers (device array), if non-null
  u64 item_stride;           // words
  const ModTab *mods;
  int logN;
  int nsub;                  // (poly, limb) units per item
  unsigned short sub_off[NTT_MAXSUB];  // unit offset inside the item, in units of N words
  unsigned char sub_mod[NTT_MAXSUB];   // modulus index of the unit
};

__device__ __forceinline__ int spad(int i) { return i + (i >> 4); }

template <int E, int RP, bool FWD>
__device__ __forceinline__ void ntt_phase(u64 *sm, int s0, int logN, int tid, u64 q, const u64 *__restrict__ tw,
                                          const u64 *__restrict__ twsh) {
  constexpr int K = 1 << RP;          // words per row
  constexpr int R = E / K;            // rows per thread
  const int N = 1 << logN;
  const int S = N >> s0, st = S >> RP;
  u64 x[E];
#pragma unroll
  for (int u = 0; u < R; u++) {
    int row = tid * R + u, blk = row / st, off = row - blk * st;
#pragma unroll
    for (int k = 0; k < K; k++) x[u * K + k] = sm[spad(blk * S + off + k * st)];
  }
  if (FWD) {
#pragma unroll
    for (int l = 0; l < RP; l++) {
      const int half = K >> (l + 1);
#pragma unroll
      for (int u = 0; u < R; u++) {
        int row = tid * R + u, blk = row / st;
#pragma unroll
        for (int k = 0; k < K; k++) {
          if (k & half) continue;
          int ti = (1 << (s0 + l)) + (blk << l) + (k >> (RP - l));
          u64 W = __ldg(tw + ti), Ws = __ldg(twsh + ti);
          u64 U = x[u * K + k], V = mul_shoup(x[u * K + k + half], W, Ws, q);
          x[u * K + k] = add_mod(U, V, q);
          x[u * K + k + half] = sub_mod(U, V, q);
        }
      }
    }
  } else {
#pragma unroll
    for (int l = RP - 1; l >= 0; l--) {
      const int half = K >> (l + 1);
#pragma unroll
      for (int u = 0; u < R; u++) {
        int row = tid * R + u, blk = row / st;
#pragma unroll
        for (int k = 0; k < K; k++) {
          if (k & half) continue;
          int ti = (1 << (s0 + l)) + (blk << l) + (k >> (RP - l));
          u64 W = __ldg(tw + ti), Ws = __ldg(twsh + ti);
          u64 U = x[u * K + k], V = x[u * K + k + half];
          x[u * K + k] = add_mod(U, V, q);
          x[u * K + k + half] = mul_shoup(sub_mod(U, V, q), W, Ws, q);
        }
      }
    }
  }
#pragma unroll
  for (int u = 0; u < R; u++) {
    int row = tid * R + u, blk = row / st, off = row - blk * st;
#pragma unroll
    for (int k = 0; k < K; k++) sm[spad(blk * S + off + k * st)] = x[u * K + k];
  }
}

template <int E, bool FWD>
__device__ __forceinline__ void ntt_phase_dispatch(int rp, u64 *sm, int s0, int logN, int tid, u64 q, const u64 *tw,
                                                   const u64 *twsh) {
  if (E >= 16 && rp == 4) { ntt_phase<E, (E >= 16 ? 4 : 1), FWD>(sm, s0, logN, tid, q, tw, twsh); return; }
  if (E >= 8 && rp == 3) { ntt_phase<E, (E >= 8 ? 3 : 1), FWD>(sm, s0, logN, tid, q, tw, twsh); return; }
  if (E >= 4 && rp == 2) { ntt_phase<E, (E >= 4 ? 2 : 1), FWD>(sm, s0, logN, tid, q, tw, twsh); return; }
  ntt_phase<E, 1, FWD>(sm, s0, logN, tid, q, tw, twsh);
}

template <int E, bool FWD>
__global__ void __launch_bounds__(1024) k_ntt(NttJob job) {
  extern __shared__ u64 sm[];
  constexpr int R = (E == 16) ? 4 : (E == 8) ? 3 : (E == 4) ? 2 : 1;
  const int item = blockIdx.x / job.nsub, sub = blockIdx.x - item * job.nsub;
  u64 *p = (job.items ? job.items[item] : job.base + (u64)item * job.item_stride) +
           ((u64)job.sub_off[sub] << job.logN);
  const ModTab &M = job.mods[job.sub_mod[sub]];
  const u64 q = M.q;
  const int logN = job.logN, N = 1 << logN, tid = threadIdx.x, T = blockDim.x;
  for (int i = tid; i < N; i += T) sm[spad(i)] = p[i];
  __syncthreads();
  if (FWD) {
    for (int s0 = 0; s0 < logN; s0 += R) {
      int rp = min(R, logN - s0);
      ntt_phase_dispatch<E, true>(rp, sm, s0, logN, tid, q, M.tw, M.tw_sh);
      __syncthreads();
    }
    for (int i = tid; i < N; i += T) p[i] = sm[spad(i)];
  } else {
    int nph = (logN + R - 1) / R;
    for (int ph = nph - 1; ph >= 0; ph--) {
      int s0 = ph * R, rp = min(R, logN - s0);
      ntt_phase_dispatch<E, false>(rp, sm, s0, logN, tid, q, M.itw, M.itw_sh);
      __syncthreads();
    }
    const u64 ni = M.ninv, nis = M.ninv_sh;
    for (int i = tid; i < N; i += T) p[i] = mul_shoup(sm[spad(i)], ni, nis, q);
  }
}

}  // namespace cgb
