// cgb_device.cuh -- device arithmetic for the sm_100a RNS-BFV backend:
// 64-bit Shoup / Barrett modular multiplication on the integer pipe,
// ChaCha20 sampling, and the shared-memory negacyclic NTT.
//
// Words are uint64 residues of primes q < 2^62 (Q: 60-bit, P/B: 61-bit).
// Every kernel here produces canonical residues in [0, q) so results are
// bit-identical to the CPU restatement in oracle/rnsbfv.c.
#pragma once
#include <cstdint>
#include <type_traits>
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
  const u64 *tw1, *itw1;                 // the same pairs in two-pass row-tile order (see k_ntt2)
  const u64 *ftw, *fitw, *ftw1, *fitw1;  // FP64 twiddles (w, w/q) as double pairs, same orders
  const u64 *ftw1t, *fitw1t;             // ftw1 / fitw1, levels >= 4 of each row transposed
  const u64 *ftw1tw, *fitw1tw;           // the w halves of ftw1t / fitw1t alone (w / q is one DMUL on use)
  double qd, qinv;                       // q and 1/q as doubles (FP64 NTT)
  double ninv_fp, ninv_fpq;              // N^-1 and N^-1 / q as doubles
  double itw0n_fp, itw0n_fpq;            // (last inverse stage's twiddle) * N^-1 mod q, and that / q
  int bits;
  int pad_;
};

// ---------------------------------------------------------------------------
// scalar modular arithmetic
// ---------------------------------------------------------------------------
// (A four-IMAD.WIDE high product was tried instead of __umul64hi and measured
// slower in both the NTT and the modmul-peak kernel; scripts/micro/imad_rates.cu.)
__device__ __forceinline__ u64 add_mod(u64 a, u64 b, u64 q) {
  u64 s = a + b;
  return s >= q ? s - q : s;
}
__device__ __forceinline__ u64 sub_mod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }

// x * q mod 2^64.  QS: q = k 2^32 + 1 (every ciphertext modulus of this
// backend) -> one 32-bit multiply; the plaintext modulus t takes the generic path.
template <bool QS = true>
__device__ __forceinline__ u64 mul_q(u64 x, u64 q) {
  if (QS) return x + ((u64)((u32)x * (u32)(q >> 32)) << 32);
  return x * q;
}
// a * w mod q with w' = floor(w 2^64 / q); any a < 2^64, result in [0, q)
template <bool QS = true>
__device__ __forceinline__ u64 mul_shoup(u64 a, u64 w, u64 wsh, u64 q) {
  u64 hi = __umul64hi(a, wsh);
  u64 r = a * w - mul_q<QS>(hi, q);
  return r >= q ? r - q : r;
}

// a * b mod q, a, b < q < 2^62 (Barrett with mu = floor(2^(2k)/q), k = bits(q))
__device__ __forceinline__ u64 mul_mod(u64 a, u64 b, u64 q, u64 mu, int bits) {
  u64 lo = a * b, hi = __umul64hi(a, b);
  const int s = bits - 1, s2 = bits + 1;
  u64 xs = (hi << (64 - s)) | (lo >> s);
  u64 ph = __umul64hi(xs, mu), pl = xs * mu;
  u64 qh = (ph << (64 - s2)) | (pl >> s2);
  u64 r = lo - mul_q(qh, q);
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
  if (q > (qs >> 1)) return v > (qs >> 1) ? v + (q - qs) : v;  // both halves already in [0, q)
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
// Harvey lazy butterflies: forward values live in [0, 4q), inverse in [0, 2q)
// (q < 2^62); outputs are reduced to [0, q) on the final store.
// Each thread keeps E words in registers as E/16 rows of 16 and runs up to
// 4 radix-2 stages on them between shared-memory exchanges.  Twiddles are
// (w, w') pairs read with one 16-byte load, one load per distinct twiddle.
// Optional fused load: a unit may read its input from another buffer and
// centre-lift it from a source modulus (ModUp / ModDown base conversion).
// ---------------------------------------------------------------------------
constexpr int NTT_MAXSUB = 160;

struct NttJob {
  u64 *base;                 // destination items: base + item * item_stride
  u64 *const *items;         // or per-item destination pointers (device array), if non-null
  u64 item_stride;           // words
  const u64 *src_base;       // fused-load source items (null: in place)
  u64 src_stride;
  u64 *const *src_items;     // or per-item source pointers
  const u64 *galois;         // per-item Galois element: load src[perm_g(k)] (evaluation-domain automorphism)
  int lift;                  // centre-lift from src_mod on load
  unsigned char in_raw;      // FP64 register-I/O kernels: source words are reduced doubles (a pass boundary)
  unsigned char out_raw;     //   ... store reduced doubles in [-q/2, q/2] instead of canonical u64
  const ModTab *mods;
  int logN;
  int nsub;                                // (poly, limb) units per item
  unsigned short sub_off[NTT_MAXSUB];      // unit offset inside the item, in units of N words
  unsigned short src_off[NTT_MAXSUB];      // source unit offset (fused load)
  unsigned char sub_mod[NTT_MAXSUB];       // modulus index of the unit
  unsigned char src_mod[NTT_MAXSUB];       // source modulus of the centred lift (fused load)
};

__device__ __forceinline__ int spad(int i) { return i + (i >> 4); }

// evaluation-domain automorphism X -> X^g: output word k reads input word perm_g(k)
__device__ __forceinline__ u32 perm_g(u32 k, u64 g, int logN) {
  const u32 e = 2u * (__brev(k) >> (32 - logN)) + 1u;
  const u32 se = (u32)((e * g) & ((2ull << logN) - 1));
  return __brev((se - 1) >> 1) >> (32 - logN);
}
__device__ __forceinline__ void prefetch_l2(const void *p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ void prefetch_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// Programmatic dependent launch: a kernel launched with the PDL attribute may
// start while its predecessor drains; it stages constant tables (twiddles), then
// waits for the predecessor's writes.  Without the attribute both are no-ops.
__device__ __forceinline__ void pdl_start_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ u32 smem_u32(const void *p) { return (u32)__cvta_generic_to_shared(p); }
// 16-byte asynchronous global -> shared copies (no register staging)
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// Aligned blocks of 2^b consecutive output words read an aligned block of 2^b
// input words (the automorphism acts on the top bits of brev(k) by an affine map
// and leaves the low bits' block fixed), so a gather of 4 consecutive outputs is
// ONE 32-byte sector load plus an in-register selection.
__device__ __forceinline__ u64 sel4(const u64 w[4], u32 s) {
  const u64 lo = (s & 1) ? w[1] : w[0], hi = (s & 1) ? w[3] : w[2];
  return (s & 2) ? hi : lo;
}
#ifndef CGB_GATHER_NC
#define CGB_GATHER_NC 1  // measured: the non-coherent path is marginally faster for the digit rows
#endif
// out[i] = src[perm_g(k0 + i)], i < 4, k0 a multiple of 4
__device__ __forceinline__ void gather4(const u64 *src, u32 k0, u64 g, int logN, u64 out[4]) {
  const u32 p0 = perm_g(k0, g, logN);
  u64 w[4];
#if CGB_GATHER_NC
  asm("ld.global.nc.v4.b64 {%0, %1, %2, %3}, [%4];"
      : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]) : "l"(src + (p0 & ~3u)));
#else  // the coherent L1 path: neighbouring threads' blocks stay cached
  const ulonglong2 *b = reinterpret_cast<const ulonglong2 *>(src + (p0 & ~3u));
  const ulonglong2 lo = b[0], hi = b[1];
  w[0] = lo.x, w[1] = lo.y, w[2] = hi.x, w[3] = hi.y;
#endif
  out[0] = sel4(w, p0 & 3);
#pragma unroll
  for (int i = 1; i < 4; i++) out[i] = sel4(w, perm_g(k0 + i, g, logN) & 3);
}

// source pointer of unit `sub` of `item` for a fused load (null: in place)
__device__ __forceinline__ const u64 *job_src(const NttJob &job, int item, int sub, int logN) {
  if (job.src_items) return job.src_items[item] + ((u64)job.src_off[sub] << logN);
  if (job.src_base) return job.src_base + (u64)item * job.src_stride + ((u64)job.src_off[sub] << logN);
  return nullptr;
}

// two-pass NTT tiles: one pad word per 8 (conflict-free 64-bit accesses for the
// row strides 16, 2 and 1 of the 3+3+1-stage phases and for column writes)
__device__ __forceinline__ int spad8(int i) { return i + (i >> 3); }

// lazy Shoup: a * w mod q in [0, 2q) for any a < 2^64
template <bool QS = true>
__device__ __forceinline__ u64 mul_shoup_lazy(u64 a, u64 w, u64 wsh, u64 q) {
  return a * w - mul_q<QS>(__umul64hi(a, wsh), q);
}

template <int E, int RP, bool FWD, bool QS>
__device__ __forceinline__ void ntt_phase(u64 *sm, int s0, int logN, int tid, u64 q, u64 q2,
                                          const ulonglong2 *__restrict__ tw) {
  constexpr int K = 1 << RP;   // words per row
  constexpr int R = E / K;     // rows per thread, processed one after another
  const int S = (1 << logN) >> s0, st = S >> RP;
#pragma unroll 1
  for (int u = 0; u < R; u++) {
    const int row = tid * R + u, blk = row / st;
    const int base = blk * S + (row - blk * st);
    u64 x[K];
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = sm[spad(base + k * st)];
#pragma unroll
    for (int ll = 0; ll < RP; ll++) {
      const int l = FWD ? ll : RP - 1 - ll;
      const int half = K >> (l + 1);
      ulonglong2 W;
#pragma unroll
      for (int k = 0; k < K; k++) {
        if (k & half) continue;
        // butterflies sharing twiddle group k >> (RP - l) are consecutive: one 16-byte load per group
        if ((k & ((1 << (RP - l)) - 1)) == 0) W = __ldg(tw + (1 << (s0 + l)) + (blk << l) + (k >> (RP - l)));
        u64 &X = x[k], &Y = x[k + half];
        if (FWD) {
          u64 a = X >= q2 ? X - q2 : X;
          u64 t = mul_shoup_lazy<QS>(Y, W.x, W.y, q);
          X = a + t;
          Y = a - t + q2;
        } else {
          u64 a = X + Y;
          u64 d = X - Y + q2;
          X = a >= q2 ? a - q2 : a;
          Y = mul_shoup_lazy<QS>(d, W.x, W.y, q);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; k++) sm[spad(base + k * st)] = x[k];
  }
}

template <int E, bool FWD, bool QS>
__device__ __forceinline__ void ntt_phase_dispatch(int rp, u64 *sm, int s0, int logN, int tid, u64 q, u64 q2,
                                                   const ulonglong2 *tw) {
  switch (rp) {
    case 4: if constexpr (E >= 16) { ntt_phase<E, 4, FWD, QS>(sm, s0, logN, tid, q, q2, tw); return; } break;
    case 3: if constexpr (E >= 8) { ntt_phase<E, 3, FWD, QS>(sm, s0, logN, tid, q, q2, tw); return; } break;
    case 2: if constexpr (E >= 4) { ntt_phase<E, 2, FWD, QS>(sm, s0, logN, tid, q, q2, tw); return; } break;
    default: break;
  }
  ntt_phase<E, 1, FWD, QS>(sm, s0, logN, tid, q, q2, tw);
}

// E words per thread; phases of RMAX = min(4, log2 E) stages
template <int E, bool FWD, bool QS>
__global__ void __launch_bounds__(512) k_ntt(NttJob job) {
  extern __shared__ u64 sm[];
  constexpr int RMAX = (E >= 16) ? 4 : (E == 8) ? 3 : (E == 4) ? 2 : 1;
  const int item = blockIdx.x / job.nsub, sub = blockIdx.x - item * job.nsub;
  u64 *p = (job.items ? job.items[item] : job.base + (u64)item * job.item_stride) + ((u64)job.sub_off[sub] << job.logN);
  const ModTab &M = job.mods[job.sub_mod[sub]];
  const u64 q = M.q, q2 = 2 * q;
  const int logN = job.logN, N = 1 << logN, tid = threadIdx.x, T = blockDim.x;
  {
    const u64 *src = job_src(job, item, sub, logN);
    if (!src) src = p;
    const u64 qs = job.lift ? job.mods[job.src_mod[sub]].q : 0;
    const u64 g = job.galois ? job.galois[item] : 1;
    for (int i = tid; i < N; i += T) {
      u64 v = src[g == 1 ? i : perm_g(i, g, logN)];
      sm[spad(i)] = job.lift ? centred_to(v, qs, q) : v;
    }
  }
  __syncthreads();
  const ulonglong2 *tw = reinterpret_cast<const ulonglong2 *>(FWD ? M.tw : M.itw);
  const int nph = (logN + RMAX - 1) / RMAX;
  for (int ph = 0; ph < nph; ph++) {
    const int pi = FWD ? ph : nph - 1 - ph;
    const int s0 = pi * RMAX, rp = min(RMAX, logN - s0);
    ntt_phase_dispatch<E, FWD, QS>(rp, sm, s0, logN, tid, q, q2, tw);
    __syncthreads();
  }
  if (FWD) {
    for (int i = tid; i < N; i += T) {
      u64 v = sm[spad(i)];
      v = v >= q2 ? v - q2 : v;
      p[i] = v >= q ? v - q : v;
    }
  } else {
    const u64 ni = M.ninv, nis = M.ninv_sh;
    for (int i = tid; i < N; i += T) p[i] = mul_shoup<QS>(sm[spad(i)], ni, nis, q);
  }
}

// ---------------------------------------------------------------------------
// two-pass NTT for large N = 2^a * 2^b (a = logN / 2):
//   pass 0: 2^b strided "column" sub-NTTs of 2^a points (stages 0..a-1),
//   pass 1: 2^a contiguous "row" sub-NTTs of 2^b points (stages a..logN-1).
// Forward runs pass 0 then 1; inverse runs pass 1 then 0 (GS order).  Every
// stage-s twiddle of the full transform restricted to one sub-NTT is the
// sub-NTT's own stage table, so each CTA stages exactly the (w, w') pairs
// its G sub-NTTs use in shared memory (pass 0: 2^a - 1 pairs shared by all
// columns; pass 1: 2^b - 1 pairs per row block) and works from there.
// ---------------------------------------------------------------------------
constexpr int NTT2_TILE = 2048;  // words per CTA
constexpr int NTT2_T = 256;      // threads per CTA (8 words each)

// one register phase of RP radix-2 stages starting at local stage S0 of an
// M = 2^LM point sub-NTT; each thread owns 8 words = 8/2^RP rows of 2^RP
template <int LM, int S0, int RP, bool FWD, bool QS, int E = 8>
__device__ __forceinline__ void ntt2_phase(u64 *sub, const ulonglong2 *tws, int tl, u64 q, u64 q2) {
  constexpr int K = 1 << RP, R = E / K;
  constexpr int S = (1 << LM) >> S0, ST = S >> RP;
  // word k of a row sits at spad(base) + off(k) with a compile-time off(k) when
  // the stride is a multiple of 16 or the row lies inside one 16-word block
  constexpr bool CONST_OFF = (ST % 8 == 0) || (S <= 8);
#pragma unroll
  for (int u = 0; u < R; u++) {
    const int row = tl * R + u;
    const int blk = row / ST, base = blk * S + (row & (ST - 1));
    const int pb = spad8(base);
    auto addr = [&](int k) { return CONST_OFF ? pb + k * ST + ((ST % 8 == 0) ? (k * ST) >> 3 : 0) : spad8(base + k * ST); };
    u64 x[K];
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = sub[addr(k)];
#pragma unroll
    for (int ll = 0; ll < RP; ll++) {
      const int l = FWD ? ll : RP - 1 - ll;
      const int half = K >> (l + 1);
      ulonglong2 W;
#pragma unroll
      for (int k = 0; k < K; k++) {
        if (k & half) continue;
        if ((k & ((1 << (RP - l)) - 1)) == 0) W = tws[(1 << (S0 + l)) + (blk << l) + (k >> (RP - l))];
        u64 &X = x[k], &Y = x[k + half];
        if (FWD) {
          u64 a = X >= q2 ? X - q2 : X;
          u64 t = mul_shoup_lazy<QS>(Y, W.x, W.y, q);
          X = a + t;
          Y = a - t + q2;
        } else {
          u64 a = X + Y;
          u64 d = X - Y + q2;
          X = a >= q2 ? a - q2 : a;
          Y = mul_shoup_lazy<QS>(d, W.x, W.y, q);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; k++) sub[addr(k)] = x[k];
  }
}

// all phases of one sub-NTT: phases of RMAX = log2(E) stages (the last one
// shorter), forward in increasing stage order, inverse in decreasing order
template <int LM, int E, bool FWD, bool QS, int PH = 0>
__device__ __forceinline__ void ntt2_sub(u64 *sub, const ulonglong2 *tws, int tl, u64 q, u64 q2) {
  constexpr int RMAX = E == 16 ? 4 : 3;
  constexpr int NPH = (LM + RMAX - 1) / RMAX;
  if constexpr (PH < NPH) {
    constexpr int PI = FWD ? PH : NPH - 1 - PH;
    constexpr int S0 = PI * RMAX, RP = (LM - S0 < RMAX) ? LM - S0 : RMAX;
    ntt2_phase<LM, S0, RP, FWD, QS, E>(sub, tws, tl, q, q2);
    __syncthreads();
    ntt2_sub<LM, E, FWD, QS, PH + 1>(sub, tws, tl, q, q2);
  }
}

// PASS 0: 2^LB strided columns of 2^LA points; PASS 1: 2^LA contiguous rows of 2^LB points
template <int LA, int LB, bool FWD, int PASS, bool QS, int E = 8>
__global__ void __launch_bounds__(NTT2_TILE / E) k_ntt2(NttJob job) {
  constexpr int T = NTT2_TILE / E;
  extern __shared__ u64 sm2[];
  constexpr int LOGN = LA + LB;
  constexpr int LM = PASS == 0 ? LA : LB, M = 1 << LM;
  constexpr int G = NTT2_TILE / M, LG = 11 - LM;
  constexpr int NSUBS = 1 << (PASS == 0 ? LB : LA), TILES = NSUBS / G;
  constexpr int PADM = M + (M >> 3) + 1, TPS = M / E;  // odd row pitch: conflict-free column writes
  static_assert(G * M == NTT2_TILE && (1 << LG) == G, "tile shape");
  const int unit = blockIdx.x / TILES, tile = blockIdx.x - unit * TILES;
  const int item = unit / job.nsub, sub = unit - item * job.nsub;
  u64 *p = (job.items ? job.items[item] : job.base + (u64)item * job.item_stride) + ((u64)job.sub_off[sub] << LOGN);
  const ModTab &Md = job.mods[job.sub_mod[sub]];
  const u64 q = Md.q, q2 = 2 * q;
  const int tid = threadIdx.x;
  u64 *data = sm2;
  ulonglong2 *tws = reinterpret_cast<ulonglong2 *>(sm2 + ((G * PADM + 1) & ~1));
  const ulonglong2 *gtw = reinterpret_cast<const ulonglong2 *>(
      PASS == 0 ? (FWD ? Md.tw : Md.itw) : (FWD ? Md.tw1 : Md.itw1));
  const int first = tile * G;
  // element e = tid + i*T of the tile -> (sub-NTT g, index k) and global word
  auto gidx = [&](int e, int &g, int &k) -> u64 {
    if (PASS == 0) {
      g = e & (G - 1);
      k = e >> LG;
      return ((u64)k << LB) + first + g;
    } else {
      g = e >> LM;
      k = e & (M - 1);
      return ((u64)first << LM) + e;
    }
  };
  const u64 *src = job_src(job, item, sub, LOGN);
  if (!src) src = p;
  const bool lift = job.lift != 0;
  const u64 qs = lift ? job.mods[job.src_mod[sub]].q : 0;
  const u64 gal = job.galois ? job.galois[item] : 1;
  u64 v[E];
  if (gal == 1) {
#pragma unroll
    for (int i = 0; i < E; i++) {
      int g, k;
      v[i] = __ldcs(src + gidx(tid + i * T, g, k));
    }
  } else {
#pragma unroll
    for (int i = 0; i < E; i++) {
      int g, k;
      v[i] = __ldg(src + perm_g((u32)gidx(tid + i * T, g, k), gal, LOGN));
    }
  }
  // stage twiddles while the tile loads are in flight
  if (PASS == 0) {
    for (int i = tid; i < M; i += T) tws[i] = __ldg(gtw + i);
  } else {  // row tiles: the table is pre-permuted, the CTA's pairs are contiguous
#pragma unroll
    for (int j = 0; j < E; j++) {
      const int e = tid + j * T;
      tws[e] = __ldg(gtw + ((u64)first << LM) + e);
    }
  }
#pragma unroll
  for (int i = 0; i < E; i++) {
    int g, k;
    gidx(tid + i * T, g, k);
    data[g * PADM + spad8(k)] = lift ? centred_to(v[i], qs, q) : v[i];
  }
  __syncthreads();
  {
    const int g = tid / TPS, tl = tid & (TPS - 1);
    ntt2_sub<LM, E, FWD, QS>(data + g * PADM, PASS == 0 ? tws : tws + g * M, tl, q, q2);
  }
  const bool last = FWD ? (PASS == 1) : (PASS == 0);
  const u64 ni = Md.ninv, nis = Md.ninv_sh;
#pragma unroll
  for (int i = 0; i < E; i++) {
    int g, k;
    const u64 w = gidx(tid + i * T, g, k);
    u64 x = data[g * PADM + spad8(k)];
    if (last) {
      if (FWD) {
        x = x >= q2 ? x - q2 : x;
        x = x >= q ? x - q : x;
      } else {
        x = mul_shoup<QS>(x, ni, nis, q);
      }
    }
    p[w] = x;
  }
}

template <int LA, int LB>
__host__ size_t ntt2_smem_bytes(int pass) {
  const int M = 1 << (pass == 0 ? LA : LB), G = NTT2_TILE / M, PADM = M + (M >> 3) + 1;
  return sizeof(u64) * (size_t)((G * PADM + 1) & ~1) + 16 * (size_t)(pass == 0 ? M : NTT2_TILE);
}

// ---------------------------------------------------------------------------
// FP64-pipe NTT (rings whose primes are < 2^49).  The B200 issues DFMA at the
// IMAD rate, and an exact modular product costs ~6 FP64 ops via error-free
// transformations (hi = a w, lo = fma(a, w, -hi), r = fma(-rint(a w/q), q, hi) + lo)
// against ~14 integer ops for the 64-bit Shoup product.  Values are signed
// doubles: |x| <= q/2 after a reduction, growing by < 2q per stage, reduced at
// every phase start, so every intermediate is an integer < 2^52 and exact.
// Loads and stores move canonical u64 residues, so the transform is the same
// function as the integer NTT (bit-exact against the oracle).
// ---------------------------------------------------------------------------
__device__ __forceinline__ double u2d(u64 v) {  // exact for v < 2^52
  return __longlong_as_double((long long)(v | 0x4330000000000000ull)) - 4503599627370496.0;
}
__device__ __forceinline__ double fp_reduce(double x, double q, double qinv) {  // -> [-q/2, q/2]
  return fma(-rint(x * qinv), q, x);
}
// a pass-boundary word: the reduced double's bits (the next pass loads it with r2d)
__device__ __forceinline__ u64 fp_raw(double x, double q, double qinv) {
  return (u64)__double_as_longlong(fp_reduce(x, q, qinv));
}
__device__ __forceinline__ double r2d(u64 v) { return __longlong_as_double((long long)v); }
__device__ __forceinline__ u64 fp_canon(double x, double q, double qinv) {  // -> [0, q) as u64
  double r = fp_reduce(x, q, qinv);
  r = r < 0.0 ? r + q : r;
  return (u64)__double_as_longlong(r + 4503599627370496.0) & 0xFFFFFFFFFFFFFull;
}
__device__ __forceinline__ double fp_mulmod(double a, double w, double wq, double q) {  // in (-2q, 2q)
  const double hi = a * w;
  const double lo = fma(a, w, -hi);
  return fma(-rint(a * wq), q, hi) + lo;
}

// the same product with the quotient estimated from the rounded product itself:
// rint(fl(a w) / q) instead of rint(a fl(w / q)) -- no w / q operand.  Three roundings
// (1 / q, the product, the scaling), exactly as many as fp_mulmod(a, w, w * qinv, q)
// spends when w / q has to be formed on the fly, so the same bound: |a w / q - qe| <=
// 0.5 + 3 |a w / q| 2^-53, the result an exact integer in (-2.8 q, 2.8 q) for |a| < 12 q.
__device__ __forceinline__ double fp_mulmod_q(double a, double w, double q, double qinv) {
  const double hi = a * w;
  const double lo = fma(a, w, -hi);
  return fma(-rint(hi * qinv), q, hi) + lo;
}

template <int LM, int S0, int RP, bool FWD, int E>
__device__ __forceinline__ void ntt2_phase_fp(double *sub, const double2 *tws, int tl, double q, double qinv) {
  constexpr int K = 1 << RP, R = E / K;
  constexpr int S = (1 << LM) >> S0, ST = S >> RP;
  constexpr bool CONST_OFF = (ST % 8 == 0) || (S <= 8);
#pragma unroll
  for (int u = 0; u < R; u++) {
    const int row = tl * R + u;
    const int blk = row / ST, base = blk * S + (row & (ST - 1));
    const int pb = spad8(base);
    auto addr = [&](int k) { return CONST_OFF ? pb + k * ST + ((ST % 8 == 0) ? (k * ST) >> 3 : 0) : spad8(base + k * ST); };
    double x[K];
#pragma unroll
    for (int k = 0; k < K; k++) x[k] = fp_reduce(sub[addr(k)], q, qinv);
#pragma unroll
    for (int ll = 0; ll < RP; ll++) {
      const int l = FWD ? ll : RP - 1 - ll;
      const int half = K >> (l + 1);
      double2 W;
#pragma unroll
      for (int k = 0; k < K; k++) {
        if (k & half) continue;
        if ((k & ((1 << (RP - l)) - 1)) == 0) W = tws[(1 << (S0 + l)) + (blk << l) + (k >> (RP - l))];
        double &X = x[k], &Y = x[k + half];
        if (FWD) {
          const double t = fp_mulmod(Y, W.x, W.y, q);
          Y = X - t;
          X = X + t;
        } else {  // GS: the sum is reduced so it cannot double every stage
          const double d = X - Y;
          X = fp_reduce(X + Y, q, qinv);
          Y = fp_mulmod(d, W.x, W.y, q);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < K; k++) sub[addr(k)] = x[k];
  }
}

template <int LM, int E, bool FWD, int PH = 0>
__device__ __forceinline__ void ntt2_sub_fp(double *sub, const double2 *tws, int tl, double q, double qinv) {
  constexpr int RMAX = E == 16 ? 4 : 3;
  constexpr int NPH = (LM + RMAX - 1) / RMAX;
  if constexpr (PH < NPH) {
    constexpr int PI = FWD ? PH : NPH - 1 - PH;
    constexpr int S0 = PI * RMAX, RP = (LM - S0 < RMAX) ? LM - S0 : RMAX;
    ntt2_phase_fp<LM, S0, RP, FWD, E>(sub, tws, tl, q, qinv);
    __syncthreads();
    ntt2_sub_fp<LM, E, FWD, PH + 1>(sub, tws, tl, q, qinv);
  }
}

// same tiling / fused loads as k_ntt2; every pass stores canonical u64
template <int LA, int LB, bool FWD, int PASS, int E = 8>
__global__ void __launch_bounds__(NTT2_TILE / E) k_ntt2_fp(NttJob job) {
  extern __shared__ u64 sm2[];
  constexpr int T = NTT2_TILE / E;
  constexpr int LOGN = LA + LB;
  constexpr int LM = PASS == 0 ? LA : LB, M = 1 << LM;
  constexpr int G = NTT2_TILE / M, LG = 11 - LM;
  constexpr int NSUBS = 1 << (PASS == 0 ? LB : LA), TILES = NSUBS / G;
  constexpr int PADM = M + (M >> 3) + 1, TPS = M / E;
  const int unit = blockIdx.x / TILES, tile = blockIdx.x - unit * TILES;
  const int item = unit / job.nsub, sub = unit - item * job.nsub;
  u64 *p = (job.items ? job.items[item] : job.base + (u64)item * job.item_stride) + ((u64)job.sub_off[sub] << LOGN);
  const ModTab &Md = job.mods[job.sub_mod[sub]];
  const u64 q = Md.q;
  const double qd = Md.qd, qinv = Md.qinv;
  const int tid = threadIdx.x;
  double *data = reinterpret_cast<double *>(sm2);
  double2 *tws = reinterpret_cast<double2 *>(sm2 + ((G * PADM + 1) & ~1));
  const double2 *gtw = reinterpret_cast<const double2 *>(
      PASS == 0 ? (FWD ? Md.ftw : Md.fitw) : (FWD ? Md.ftw1 : Md.fitw1));
  const int first = tile * G;
  auto gidx = [&](int e, int &g, int &k) -> u64 {
    if (PASS == 0) {
      g = e & (G - 1);
      k = e >> LG;
      return ((u64)k << LB) + first + g;
    } else {
      g = e >> LM;
      k = e & (M - 1);
      return ((u64)first << LM) + e;
    }
  };
  const u64 *src = job_src(job, item, sub, LOGN);
  if (!src) src = p;
  const bool lift = job.lift != 0;
  const u64 qs = lift ? job.mods[job.src_mod[sub]].q : 0;
  const u64 gal = job.galois ? job.galois[item] : 1;
  u64 v[E];
  if (gal == 1) {
#pragma unroll
    for (int i = 0; i < E; i++) {
      int g, k;
      v[i] = __ldcs(src + gidx(tid + i * T, g, k));
    }
  } else {
#pragma unroll
    for (int i = 0; i < E; i++) {
      int g, k;
      v[i] = __ldg(src + perm_g((u32)gidx(tid + i * T, g, k), gal, LOGN));
    }
  }
  if (PASS == 0) {
    for (int i = tid; i < M; i += T) tws[i] = __ldg(gtw + i);
  } else {
#pragma unroll
    for (int j = 0; j < E; j++) {
      const int e = tid + j * T;
      tws[e] = __ldg(gtw + ((u64)first << LM) + e);
    }
  }
#pragma unroll
  for (int i = 0; i < E; i++) {
    int g, k;
    gidx(tid + i * T, g, k);
    data[g * PADM + spad8(k)] = u2d(lift ? centred_to(v[i], qs, q) : v[i]);
  }
  __syncthreads();
  {
    const int g = tid / TPS, tl = tid & (TPS - 1);
    ntt2_sub_fp<LM, E, FWD>(data + g * PADM, PASS == 0 ? tws : tws + g * M, tl, qd, qinv);
  }
  const bool last = FWD ? (PASS == 1) : (PASS == 0);
  const double ni = Md.ninv_fp;
#pragma unroll
  for (int i = 0; i < E; i++) {
    int g, k;
    const u64 w = gidx(tid + i * T, g, k);
    double x = data[g * PADM + spad8(k)];
    if (last && !FWD) x = fp_mulmod(fp_reduce(x, qd, qinv), ni, Md.ninv_fpq, qd);
    p[w] = fp_canon(x, qd, qinv);
  }
}

// ---------------------------------------------------------------------------
// FP64 two-pass NTT, register I/O: the first phase reads global memory straight
// into registers and the last phase writes registers straight back, so a pass
// with 16 words per thread needs a single shared-memory exchange.  Pass 0
// (columns) maps consecutive threads to consecutive columns and pass 1 (rows)
// to consecutive words of a row, which keeps both ends coalesced.
// ---------------------------------------------------------------------------
// 256-bit global accesses (one full 32-byte sector per thread; sm_100 LDG/STG.256)
#ifndef CGB_LD256_SPLIT
#define CGB_LD256_SPLIT 0  // experiment: 256-bit loads as two 128-bit loads
#endif
__device__ __forceinline__ void ld256(const u64 *p, u64 *v) {
#if CGB_LD256_SPLIT
  asm volatile("ld.global.cs.v2.b64 {%0, %1}, [%2];" : "=l"(v[0]), "=l"(v[1]) : "l"(p));
  asm volatile("ld.global.cs.v2.b64 {%0, %1}, [%2];" : "=l"(v[2]), "=l"(v[3]) : "l"(p + 2));
#else
  asm volatile("ld.global.cs.v4.b64 {%0, %1, %2, %3}, [%4];"
               : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
#endif
}
__device__ __forceinline__ void st256(u64 *p, u64 a, u64 b, u64 c, u64 d) {
  asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}

// Row padding of k_ntt2_fpr's shared tile: word i of a row sits at i + (i >> fpr_psh)
// in a row of fpr_padm words.  Chosen with scripts/sim/smem_banks.py (per
// half-warp bank model, matches ncu) so the shared accesses of both phases take
// the 2-wavefront minimum of a warp of doubles (3 for the 32-point row pass).
__host__ __device__ constexpr int fpr_psh(int LM, int pass) { return LM == 8 ? 4 : (pass == 1 && LM <= 6) ? 2 : 3; }
__host__ __device__ constexpr int fpr_padm(int LM, int pass) {
  return (1 << LM) + ((1 << LM) >> fpr_psh(LM, pass)) +
         (LM == 8 ? 2 : pass == 0 ? 1 : LM == 7 ? 8 : LM == 6 ? 4 : 2);
}
template <int LA, int LB>
__host__ size_t fpr_smem_bytes(int pass) {  // data tile (+ the shared column-pass twiddles)
  const int LM = pass == 0 ? LA : LB, G = NTT2_TILE >> LM;
  return sizeof(u64) * (size_t)((G * fpr_padm(LM, pass) + 1) & ~1) + (pass == 0 ? 16 * (size_t)(1 << LM) : 0);
}

template <int LM, int S0, int RP, int E>
struct PhaseShape {
  static constexpr int K = 1 << RP, R = E / K, S = (1 << LM) >> S0, ST = S >> RP;
  static constexpr int TPS = (1 << LM) / E;  // threads per sub-NTT
  // local index (inside the sub-NTT) of register u*K + k of thread tl; a thread's
  // rows are interleaved (tl, tl + TPS, ...) so consecutive threads take consecutive
  // blocks and read consecutive twiddles
  static __device__ __forceinline__ int row(int tl, int u) { return tl + u * TPS; }
  static __device__ __forceinline__ int idx(int tl, int u, int k) {
    const int r = row(tl, u), blk = r / ST;
    return blk * S + (r & (ST - 1)) + k * ST;
  }
};
// TRANS: stage levels >= S0 of the twiddle table are stored transposed
// ([j][blk] instead of [blk][j], see k_ntt2_fpr) so threads on consecutive
// blocks read consecutive entries.
// GTW: tws is a global table (read through the read-only path) instead of shared memory
// WQ: tws holds the twiddles' w only (doubles); w/q is formed by one DMUL per use
#ifndef CGB_WQ_MULMODQ
#define CGB_WQ_MULMODQ 1  // w-only twiddles: quotient from the rounded product instead of a w * (1/q) DMUL per twiddle
#endif
// SKIPLAST: leave out the last executed stage (an inverse phase ending at stage 0, whose
// single butterfly layer the caller runs itself with N^-1 folded into both outputs)
template <int LM, int S0, int RP, bool FWD, int E, bool TRANS = false, bool GTW = false, bool WQ = false,
          bool SKIPLAST = false>
__device__ __forceinline__ void phase_regs_fp(double x[E], const double2 *tws, int tl, double q, double qinv) {
  using PS = PhaseShape<LM, S0, RP, E>;
  constexpr int K = PS::K, R = PS::R;
#pragma unroll
  for (int u = 0; u < R; u++) {
    const int blk = PS::row(tl, u) / PS::ST;
#pragma unroll
    for (int ll = 0; ll < RP; ll++) {
      if (SKIPLAST && ll == RP - 1) continue;
      const int l = FWD ? ll : RP - 1 - ll;
      const int half = K >> (l + 1);
      double2 W;
#pragma unroll
      for (int k = 0; k < K; k++) {
        if (k & half) continue;
        if ((k & ((1 << (RP - l)) - 1)) == 0) {
          const int ti = TRANS ? (1 << (S0 + l)) + ((k >> (RP - l)) << S0) + blk
                               : (1 << (S0 + l)) + (blk << l) + (k >> (RP - l));
          if constexpr (WQ) {
            const double w = GTW ? __ldg(reinterpret_cast<const double *>(tws) + ti) : reinterpret_cast<const double *>(tws)[ti];
            W = make_double2(w, (CGB_WQ_MULMODQ && !GTW) ? 0.0 : w * qinv);
          } else {
            W = GTW ? __ldg(tws + ti) : tws[ti];
          }
        }
        double &X = x[u * K + k], &Y = x[u * K + k + half];
        // staged w-only twiddles (the key switch's row kernels): the quotient comes from the rounded
        // product (fp_mulmod_q) -- the three roundings that forming w / q on the fly spends, without
        // the DMUL per twiddle.  (The register-I/O transform's row pass, twiddles through L1, measured
        // slower this way -- the longer dependent chain -- and keeps w * (1/q).)
        if (FWD) {
          const double t = (WQ && !GTW && CGB_WQ_MULMODQ) ? fp_mulmod_q(Y, W.x, q, qinv) : fp_mulmod(Y, W.x, W.y, q);
          Y = X - t;
          X = X + t;
        } else {  // X + Y left unreduced: scripts/sim/fp_bounds.py bounds a phase by 8q < 2^53
          const double d = X - Y;
          X = X + Y;
          Y = (WQ && !GTW && CGB_WQ_MULMODQ) ? fp_mulmod_q(d, W.x, q, qinv) : fp_mulmod(d, W.x, W.y, q);
        }
      }
    }
  }
}

// store epilogue of k_ntt2_fpr's last pass: NoEpi writes the transform; a fused
// consumer (e.g. the ModDown combine, cgb200.cu) receives the canonical words
// (n = 4 consecutive words, or 1) of unit `unit` of item `item` at word `pos`
struct NoEpi {
  static constexpr bool active = false;
  __device__ void store(int, int, u64, const u64 *, int) const {}
};
// an EPI may also feed the first pass of a row-first transform: `loads` = true and
// load4(item, unit, pos, out) supplies the 4 canonical words at pos (e.g. a tensor
// product computed from its operands on the fly, cgb200.cu TensorLoad)
template <class E, class = void>
struct EpiLoads {
  static constexpr bool value = false;
};
template <class E>
struct EpiLoads<E, std::void_t<decltype(E::loads)>> {
  static constexpr bool value = E::loads;
};

// Row passes (PASS 1) give each row to M / E <= 16 consecutive threads of one warp, so
// the exchange between a row pass's register phases needs only a warp-level barrier.
#ifndef CGB_FPR_WQ
#define CGB_FPR_WQ 1
#endif
#ifndef CGB_ROW_WSYNC
#define CGB_ROW_WSYNC 1
#endif
#if CGB_ROW_WSYNC
#define ROW_SYNC() __syncwarp()
#else
#define ROW_SYNC() __syncthreads()
#endif
// LM-point sub-NTT in two register phases (RA stages then LM - RA), E = 16
#ifdef CGB_FPR_MINB
#define FPR_BOUNDS __launch_bounds__(NTT2_TILE / 16, CGB_FPR_MINB)
#else
#define FPR_BOUNDS __launch_bounds__(NTT2_TILE / 16)
#endif
template <int LA, int LB, bool FWD, int PASS, class EPI = NoEpi>
__global__ void FPR_BOUNDS k_ntt2_fpr(NttJob job, EPI epi) {
  extern __shared__ u64 sm2[];
  constexpr int E = 16, T = NTT2_TILE / E;
  constexpr int LOGN = LA + LB;
  constexpr int LM = PASS == 0 ? LA : LB, M = 1 << LM;
  constexpr int G = NTT2_TILE / M, TPS = M / E;
  constexpr int NSUBS = 1 << (PASS == 0 ? LB : LA), TILES = NSUBS / G;
  constexpr int PSH = fpr_psh(LM, PASS), PADM = fpr_padm(LM, PASS);
  auto spad = [](int i) { return i + (i >> PSH); };
  constexpr int RA = 4, RB = LM - 4;  // forward: stages [0,4) then [4,LM); inverse: the reverse
  static_assert(RB >= 1 && RB <= 4, "sub-NTT of 32..256 points");
  const int unit = blockIdx.x / TILES, tile = blockIdx.x - unit * TILES;
  const int item = unit / job.nsub, sub = unit - item * job.nsub;
  const ModTab &Md = job.mods[job.sub_mod[sub]];
  const u64 q = Md.q;
  const double qd = Md.qd, qinv = Md.qinv;
  const int tid = threadIdx.x;
  double *data = reinterpret_cast<double *>(sm2);
  double2 *tws = reinterpret_cast<double2 *>(sm2 + ((G * PADM + 1) & ~1));
  // row passes read their row's twiddles from global memory through L1: the w-only table
  // (8 bytes per twiddle) halves that traffic of the LSU-bound row pass (CGB_FPR_WQ)
  constexpr bool RWQ = CGB_FPR_WQ && PASS == 1;
  const double2 *gtw = reinterpret_cast<const double2 *>(
      PASS == 0 ? (FWD ? Md.ftw : Md.fitw) : RWQ ? (FWD ? Md.ftw1tw : Md.fitw1tw) : (FWD ? Md.ftw1t : Md.fitw1t));
  const int first = tile * G;
  // thread -> (sub-NTT g, thread-in-sub tl): columns fast in pass 0, words fast in pass 1
  const int g = PASS == 0 ? (tid % G) : (tid / TPS);
  const int tl = PASS == 0 ? (tid / G) : (tid % TPS);
  auto gaddr = [&](int i) -> u64 {
    return PASS == 0 ? (((u64)i << LB) + first + g) : (((u64)(first + g) << LM) + i);
  };
  // pass 0 shares one M-entry table (staged); pass 1 reads its row's table from global
  if (PASS == 0)
    for (int i = tid; i < M; i += T) tws[i] = __ldg(gtw + i);
  pdl_start_dependents();
  pdl_wait();  // the predecessor's output is complete from here on
  u64 *p = (job.items ? job.items[item] : job.base + (u64)item * job.item_stride) + ((u64)job.sub_off[sub] << LOGN);
  // first phase straight from global memory (fused lift / automorphism)
  const u64 *src = job_src(job, item, sub, LOGN);
  if (!src) src = p;
  const bool lift = job.lift != 0;
  const u64 qs = lift ? job.mods[job.src_mod[sub]].q : 0;
  const u64 gal = job.galois ? job.galois[item] : 1;
  constexpr int S0A = FWD ? 0 : RA, RPA = FWD ? RA : RB;   // first phase (stages)
  constexpr int S0B = FWD ? RA : 0, RPB = FWD ? RB : RA;   // second phase
  using PA = PhaseShape<LM, S0A, RPA, E>;
  using PB = PhaseShape<LM, S0B, RPB, E>;
  double x[E];
  {
    u64 v[E];
    if constexpr (EpiLoads<EPI>::value) {  // the source words computed by the epilogue object
      static_assert(PASS == 1 && PA::ST == 1 && PA::K % 4 == 0, "fused loads feed a row pass in 4-word runs");
#pragma unroll
      for (int u = 0; u < PA::R; u++)
#pragma unroll
        for (int k = 0; k < PA::K; k += 4) epi.load4(item, sub, gaddr(PA::idx(tl, u, k)), &v[u * PA::K + k]);
    } else if (PASS == 1 && PA::ST == 1 && PA::K % 4 == 0 && gal == 1) {  // K consecutive words: full-sector loads
#pragma unroll
      for (int u = 0; u < PA::R; u++)
#pragma unroll
        for (int k = 0; k < PA::K; k += 4) ld256(src + gaddr(PA::idx(tl, u, k)), &v[u * PA::K + k]);
    } else if (PASS == 1 && PA::ST == 1 && PA::K % 4 == 0) {  // automorphism: one sector per 4 words
#pragma unroll
      for (int u = 0; u < PA::R; u++)
#pragma unroll
        for (int k = 0; k < PA::K; k += 4) gather4(src, (u32)gaddr(PA::idx(tl, u, k)), gal, LOGN, &v[u * PA::K + k]);
    } else {
#pragma unroll
      for (int u = 0; u < PA::R; u++)
#pragma unroll
        for (int k = 0; k < PA::K; k++) {
          const u64 a = gaddr(PA::idx(tl, u, k));
          v[u * PA::K + k] = gal == 1 ? __ldcs(src + a) : __ldg(src + perm_g((u32)a, gal, LOGN));
        }
    }
#pragma unroll
    for (int i = 0; i < E; i++) {
      x[i] = job.in_raw ? r2d(v[i]) : u2d(lift ? centred_to(v[i], qs, q) : v[i]);
      if (!FWD && RPA == 4) x[i] = fp_reduce(x[i], qd, qinv);  // a 4-stage inverse phase starts reduced
    }
  }
  if (PASS == 0 || !CGB_ROW_WSYNC) __syncthreads();  // twiddles staged (row passes read theirs from global)
  const double2 *tw_g = PASS == 0 ? tws
                        : RWQ     ? reinterpret_cast<const double2 *>(reinterpret_cast<const double *>(gtw) + ((u64)(first + g) << LM))
                                  : gtw + ((u64)(first + g) << LM);
  phase_regs_fp<LM, S0A, RPA, FWD, E, PASS == 1 && S0A == 4, PASS == 1, RWQ>(x, tw_g, tl, qd, qinv);
  double *sd = data + g * PADM;
#pragma unroll
  for (int u = 0; u < PA::R; u++)
#pragma unroll
    for (int k = 0; k < PA::K; k++) sd[spad(PA::idx(tl, u, k))] = x[u * PA::K + k];
  if (PASS == 0) __syncthreads();
  else ROW_SYNC();
#pragma unroll
  for (int u = 0; u < PB::R; u++)
#pragma unroll
    for (int k = 0; k < PB::K; k++) {
      // forward: no reduction inside a pass (|x| < 12q < 2^53, scripts/sim/fp_bounds.py)
      const double v = sd[spad(PB::idx(tl, u, k))];
      x[u * PB::K + k] = FWD ? v : fp_reduce(v, qd, qinv);
    }
  phase_regs_fp<LM, S0B, RPB, FWD, E, PASS == 1 && S0B == 4, PASS == 1, RWQ>(x, tw_g, tl, qd, qinv);
  const bool last = FWD ? (PASS == 1) : (PASS == 0);
  const double ni = Md.ninv_fp, niq = Md.ninv_fpq;
#pragma unroll
  for (int i = 0; i < E; i++) {
    if (last && !FWD) x[i] = fp_mulmod(fp_reduce(x[i], qd, qinv), ni, niq, qd);
  }
  if (PASS == 1 && PB::ST == 1 && PB::K % 4 == 0) {  // K consecutive words: full-sector stores
#pragma unroll
    for (int u = 0; u < PB::R; u++)
#pragma unroll
      for (int k = 0; k < PB::K; k += 4) {
        const double *y = &x[u * PB::K + k];
        u64 w[4];
#pragma unroll
        for (int e = 0; e < 4; e++) w[e] = job.out_raw ? fp_raw(y[e], qd, qinv) : fp_canon(y[e], qd, qinv);
        if constexpr (EPI::active) epi.store(item, job.sub_off[sub], gaddr(PB::idx(tl, u, k)), w, 4);
        else st256(p + gaddr(PB::idx(tl, u, k)), w[0], w[1], w[2], w[3]);
      }
  } else {
#pragma unroll
    for (int u = 0; u < PB::R; u++)
#pragma unroll
      for (int k = 0; k < PB::K; k++) {
        const u64 w = job.out_raw ? fp_raw(x[u * PB::K + k], qd, qinv) : fp_canon(x[u * PB::K + k], qd, qinv);
        if constexpr (EPI::active) epi.store(item, job.sub_off[sub], gaddr(PB::idx(tl, u, k)), &w, 1);
        else p[gaddr(PB::idx(tl, u, k))] = w;
      }
  }
}

}  // namespace cgb
