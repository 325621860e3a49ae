// cgb200.cu -- B200 (sm_100a) RNS-BFV backend for the CryptoGen HE hot path.
//
// Implements include/cgb200.h.  The algorithms are the ones stated in
// DESIGN.md section 3 and restated on the CPU in oracle/rnsbfv.c; every
// ciphertext word produced here must equal the oracle's (tests/test_gpu_*).
//
// Device layout: ciphertext = u64[2][L][N] NTT-domain residues in a
// fixed-slot arena; workspaces are stream-ordered allocations
// (cudaMallocAsync) laid out [item][poly][limb][N].  All kernels are
// batched over items so one launch covers every ciphertext of an op wave
// (e.g. the 768 broadcast chains of a 12-head decode step).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/cgb200.h"
#include "cgb_device.cuh"
#include "cgb_masks.cuh"

using namespace cgb;
typedef unsigned __int128 u128;

// ============================================================================
// error plumbing
// ============================================================================
// two-pass split of the 2^14-point transform: 2^A14 strided column sub-transforms x 2^(14 - A14)
// contiguous row sub-transforms (the other sizes split evenly: 6+7, 7+8, 8+8)
// Superseded kernel variants kept for A/B runs (k_ks_row MODE 0 / 2, k_ks_row8, the P-limb k_ks_row2):
// built only with -DCGB_BUILD_FALLBACKS=1 (they are ~100 heavy instantiations, half the compile time);
// without them CGB_KS_MD / CGB_KSROW2 / CGB_KSROW8 keep their defaults.
#ifndef CGB_BUILD_FALLBACKS
#define CGB_BUILD_FALLBACKS 0
#endif
#ifndef CGB_A14
#define CGB_A14 7
#endif
static inline int split_a(int logN) { return logN == 14 ? CGB_A14 : logN / 2; }
static thread_local std::string g_err;
struct CgbError {
  int code;
  std::string msg;
};
#define FAIL(code, ...)                                   \
  do {                                                    \
    char _b[512];                                         \
    snprintf(_b, sizeof _b, __VA_ARGS__);                 \
    throw CgbError{code, std::string(_b)};                \
  } while (0)
#define CK(x)                                                                       \
  do {                                                                              \
    cudaError_t _e = (x);                                                           \
    if (_e != cudaSuccess) FAIL(CGB_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(_e)); \
  } while (0)

#define API_BEGIN try {
#define RING_LOCK(r) std::lock_guard<std::recursive_mutex> _ring_lock((r)->api)
#define API_END                                                                       \
  {                                                                                   \
    cudaError_t _le = cudaGetLastError();                                             \
    if (_le != cudaSuccess) FAIL(CGB_ERR_CUDA, "%s left error: %s", __func__, cudaGetErrorString(_le)); \
  }                                                                                   \
  return CGB_OK;                                                                      \
  }                                                                                   \
  catch (const CgbError &e) {            \
    g_err = e.msg;                       \
    return e.code;                       \
  }                                      \
  catch (const std::exception &e) {      \
    g_err = e.what();                    \
    return CGB_ERR_STATE;                \
  }

// ============================================================================
// host number theory (exact, u128 / tiny bignum)
// ============================================================================
static u64 h_mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static u64 h_powmod(u64 a, u64 e, u64 q) {
  u64 r = 1 % q;
  a %= q;
  while (e) {
    if (e & 1) r = h_mulmod(r, a, q);
    a = h_mulmod(a, a, q);
    e >>= 1;
  }
  return r;
}
static u64 h_inv(u64 a, u64 q) { return h_powmod(a % q, q - 2, q); }
static bool h_prime(u64 n) {
  static const u64 B[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
  if (n < 2) return false;
  for (u64 b : B)
    if (n % b == 0) return n == b;
  u64 d = n - 1;
  int r = 0;
  while (!(d & 1)) d >>= 1, r++;
  for (u64 a : B) {
    u64 x = h_powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool ok = false;
    for (int i = 0; i < r - 1 && !ok; i++) {
      x = h_mulmod(x, x, n);
      ok = (x == n - 1);
    }
    if (!ok) return false;
  }
  return true;
}
static u32 h_brev(u32 x, int bits) {
  u32 r = 0;
  for (int i = 0; i < bits; i++) r = (r << 1) | ((x >> i) & 1);
  return r;
}
static u64 h_psi(u64 q, u64 twoN) {
  for (u64 x = 2;; x++) {
    u64 p = h_powmod(x, (q - 1) / twoN, q);
    if (h_powmod(p, twoN / 2, q) == q - 1) return p;
  }
}
struct Big {  // little-endian words
  std::vector<u64> w;
  explicit Big(u64 x = 0) : w(40, 0) { w[0] = x; }
  void mul(u64 x) {
    u128 c = 0;
    for (auto &v : w) {
      c += (u128)v * x;
      v = (u64)c;
      c >>= 64;
    }
  }
  u64 divmod(u64 d) {
    u128 r = 0;
    for (int i = (int)w.size() - 1; i >= 0; i--) {
      r = (r << 64) | w[i];
      w[i] = (u64)(r / d);
      r %= d;
    }
    return (u64)r;
  }
  u64 mod(u64 d) const {
    Big t = *this;
    return t.divmod(d);
  }
};
static void h_frac128(u64 r, u64 q, u64 *hi, u64 *lo) {
  u128 x = (u128)r << 64;
  *hi = (u64)(x / q);
  u64 r2 = (u64)(x % q);
  x = (u128)r2 << 64;
  *lo = (u64)(x / q);
}
static u64 h_shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }

// ============================================================================
// device-resident constants
// ============================================================================
struct Consts {
  int L, nB, N, logN, n_slots;
  int pad_;
  u64 t;
  u64 Qmodt;
  u64 tinvq[MAXL], Pinvq[MAXL], Pinvq_sh[MAXL], Pmodq[MAXL];
  u64 dec_omega[MAXL], dec_th_hi[MAXL], dec_th_lo[MAXL];
  u64 QhatInv[MAXL], QhatModB[MAXL][MAXL + 1], QmodB[MAXL + 1];
  double invq[MAXL], invb[MAXL + 1];
  u64 QBhatInv[MAXL], BQhatInv[MAXL + 1], sc_omega[MAXL][MAXL + 1], sc_th_hi[MAXL], sc_th_lo[MAXL];
  u64 tBhat[MAXL + 1];
  u64 BhatInv[MAXL + 1], BhatModQ[MAXL + 1][MAXL], BmodQ[MAXL];
  // Shoup companions of the base-conversion constants (w' = floor(w 2^64 / modulus))
  u64 QhatInv_sh[MAXL], QhatModB_sh[MAXL][MAXL + 1], QmodB_sh[MAXL + 1];
  u64 QBhatInv_sh[MAXL], BQhatInv_sh[MAXL + 1], sc_omega_sh[MAXL][MAXL + 1], tBhat_sh[MAXL + 1];
  u64 BhatInv_sh[MAXL + 1], BhatModQ_sh[MAXL + 1][MAXL], BmodQ_sh[MAXL];
  // FP64-pipe companions (w, w / modulus) of the same constants (rings of < 2^49 primes)
  double2 fQhatInv[MAXL], fQhatModB[MAXL][MAXL + 1], fQmodB[MAXL + 1];
  double2 fQBhatInv[MAXL], fBQhatInv[MAXL + 1], fsc_omega[MAXL][MAXL + 1], ftBhat[MAXL + 1];
  double2 fBhatInv[MAXL + 1], fBhatModQ[MAXL + 1][MAXL], fBmodQ[MAXL];
  double2 fPinvq[MAXL], fPmodq[MAXL];
};

static const u64 DOM_SK = 1, DOM_KSK_A = 2, DOM_KSK_E = 3, DOM_ENC_A = 4, DOM_ENC_E = 5;
static inline u64 nonce_of(u64 dom, u64 sub) { return (dom << 56) | sub; }

// ============================================================================
// the ring
// ============================================================================
struct cgb_ring {
  int logN, N, L, nB, nmod, n_slots, one_row;
  int q_bits = 60;  // Q primes < 2^q_bits; P / B primes < 2^(q_bits+1), or < 2^q_bits when <= 49
  bool fp_ntt = false;  // two-pass NTT on the FP64 pipe (log N >= 12, all primes < 2^49)
  int iP, iB0, iT;  // modulus indices of P, B[0], t
  u64 t;
  std::vector<u64> mods;  // Q | P | B | t
  std::vector<ModTab> h_mods;
  std::vector<std::pair<size_t, u64 *>> dec_pool;  // pinned landing buffers of cgb_decrypt_start
  ModTab *d_mods = nullptr;
  u64 *d_tables = nullptr;
  u32 *d_slot_idx = nullptr;
  u64 *d_s = nullptr;  // secret, NTT over Q u P: [L+1][N]
  Consts h_c;
  Consts *d_c = nullptr;
  ChaKey keyseed;
  std::unordered_map<u64, u64 *> keys;  // g -> [L][2][L+1][N]; g = 0 relin
  u64 *arena = nullptr;
  size_t ct_words, arena_cap;
  std::vector<u32> ct_free;
  std::vector<char> ct_used;
  u64 *pt_arena = nullptr;
  size_t pt_cap;
  std::vector<u32> pt_free;
  std::vector<char> pt_used;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  // pinned staging for pointer tables / host payloads: two halves used in turn;
  // entering a half waits only for the event recorded when it was last left
  char *pin = nullptr;
  size_t pin_cap = 0, pin_off = 0;
  int pin_half = 0;
  cudaEvent_t pin_left[2] = {nullptr, nullptr};
  // device mirror of the pinned halves, filled on a side stream: a call's pointer tables
  // are copied while the previous call's kernels still run, so the copy is not a bubble
  // between two calls on the compute stream (which only waits for the copy's event)
  char *dev_stage = nullptr;
  cudaStream_t copy_stream = nullptr;
  std::vector<cudaEvent_t> copy_ev;
  size_t copy_ev_next = 0;
  u64 launches = 0;
  std::mutex mu;
  // every entry point taking the ring holds this while it enqueues: the reference runs
  // heads on threads with forked contexts (model.py:395-400), which share one ring here,
  // and the ring's staging buffers, scratch and key cache are per-ring state
  std::recursive_mutex api;
  // timing (cgb_timing_enable): mode 1 = events around every kernel (PDL off);
  // mode 2 = events around every timing GROUP (a whole key switch, a whole
  // mult_cipher: PDL stays on inside it) and around launches outside groups
  bool timing = false;
  int timing_mode = 0;
  int group_depth = 0;
  cudaEvent_t group_a = nullptr;
  double group_mm = 0;
  struct Rec {
    const char *name;
    double bytes;
    double mm;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> event_pool;
  cudaEvent_t pending = nullptr;

  int ntt_E() const { return std::min(32, N); }
  int ntt_threads() const { return N / ntt_E(); }
  size_t ntt_smem() const { return sizeof(u64) * (size_t)(N + (N >> 4) + 1); }
};

// ---------------------------------------------------------------------------
// pinned staging + device scratch
// ---------------------------------------------------------------------------
static bool g_side_copy = true;  // CGB_SIDE_COPY: pointer tables uploaded on a side stream into a device mirror
template <class T>
static T *stage_to_device(cgb_ring *r, const T *host, size_t n, std::vector<void *> &frees) {
  size_t bytes = sizeof(T) * n;
  if (bytes == 0) return nullptr;
  bytes = (bytes + 255) & ~(size_t)255;
  T *dev = nullptr;
  const size_t half = r->pin_cap / 2;
  const bool side = g_side_copy && r->dev_stage && bytes <= half;
  if (!side) {
    CK(cudaMallocAsync((void **)&dev, bytes, r->stream));
    frees.push_back(dev);
  }
  if (bytes > half) {  // large payload: straight from the caller's buffer
    CK(cudaMemcpyAsync(dev, host, sizeof(T) * n, cudaMemcpyHostToDevice, r->stream));
    // A pageable source is staged by the driver before the call returns.  A
    // page-locked one is DMA'd later, and the caller may free or rewrite it as
    // soon as we return (torch's caching host allocator hands blocks out again):
    // wait for the transfer itself before returning.
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, host) == cudaSuccess && pa.type == cudaMemoryTypeHost) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      CK(cudaEventRecord(e, r->stream));
      CK(cudaEventSynchronize(e));
      CK(cudaEventDestroy(e));
    } else {
      cudaGetLastError();  // unregistered pageable memory may leave an error code behind
    }
    return dev;
  }
  if (r->pin_off + bytes > half) {  // switch halves
    if (!r->pin_left[r->pin_half]) CK(cudaEventCreateWithFlags(&r->pin_left[r->pin_half], cudaEventDisableTiming));
    CK(cudaEventRecord(r->pin_left[r->pin_half], r->stream));
    r->pin_half ^= 1;
    if (r->pin_left[r->pin_half]) CK(cudaEventSynchronize(r->pin_left[r->pin_half]));
    r->pin_off = 0;
  }
  char *dst = r->pin + (size_t)r->pin_half * half + r->pin_off;
  memcpy(dst, host, sizeof(T) * n);
  if (g_side_copy && r->dev_stage) {
    // the mirror slot is free: entering this half waited for every kernel that read it
    T *mirror = reinterpret_cast<T *>(r->dev_stage + (size_t)r->pin_half * half + r->pin_off);
    CK(cudaMemcpyAsync(mirror, dst, sizeof(T) * n, cudaMemcpyHostToDevice, r->copy_stream));
    if (r->copy_ev.size() < 64) {
      cudaEvent_t e;
      CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      r->copy_ev.push_back(e);
    }
    cudaEvent_t e = r->copy_ev[r->copy_ev_next++ % r->copy_ev.size()];
    CK(cudaEventRecord(e, r->copy_stream));
    CK(cudaStreamWaitEvent(r->stream, e, 0));
    r->pin_off += bytes;
    return mirror;
  }
  CK(cudaMemcpyAsync(dev, dst, sizeof(T) * n, cudaMemcpyHostToDevice, r->stream));
  r->pin_off += bytes;
  return dev;
}
struct Scratch {
  cgb_ring *r;
  std::vector<void *> frees;
  explicit Scratch(cgb_ring *r_) : r(r_) {}
  template <class T>
  T *alloc(size_t n) {
    T *p;
    CK(cudaMallocAsync((void **)&p, std::max<size_t>(sizeof(T) * n, 256), r->stream));
    frees.push_back(p);
    return p;
  }
  template <class T>
  T *up(const T *host, size_t n) {
    return stage_to_device(r, host, n, frees);
  }
  ~Scratch() {
    for (void *p : frees) cudaFreeAsync(p, r->stream);
  }
};

static cudaEvent_t take_event(cgb_ring *r) {
  if (!r->event_pool.empty()) {
    cudaEvent_t e = r->event_pool.back();
    r->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}
// Launch with programmatic stream serialization (kernels that call pdl_wait()
// before touching their predecessor's output); CGB_PDL=0 turns it off.
static bool g_pdl = true;
template <typename... KP, typename... A>
static void launch_pdl(cgb_ring *r, void (*k)(KP...), dim3 grid, dim3 block, size_t smem, A... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = r->stream;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = (g_pdl && r->timing_mode != 1) ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, k, ((KP)args)...);
}
static void launch_begin(cgb_ring *r) {
  if (!r->timing || r->group_depth) return;
  r->pending = take_event(r);
  CK(cudaEventRecord(r->pending, r->stream));
}
// timing groups (mode 2): one record for a whole multi-launch operation, named by
// the operation, with its algorithmic bytes (SURVEY 8(d) units) and the modular
// products its launches report
static void group_begin(cgb_ring *r) {
  if (r->timing_mode != 2 || r->group_depth++) return;
  r->group_a = take_event(r);
  r->group_mm = 0;
  CK(cudaEventRecord(r->group_a, r->stream));
}
static void group_end(cgb_ring *r, const char *name, double bytes) {
  if (r->timing_mode != 2 || --r->group_depth) return;
  cudaEvent_t b = take_event(r);
  CK(cudaEventRecord(b, r->stream));
  r->recs.push_back({name, bytes, r->group_mm, r->group_a, b});
}
// bytes: algorithmic HBM bytes; mm: algorithmic modular products (NTT butterflies,
// key and constant products) for the arithmetic-pipe roofline
static void launch_end(cgb_ring *r, const char *name, double bytes, double mm = 0.0) {
  r->launches++;
  {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) FAIL(CGB_ERR_CUDA, "launch of %s (N=%d, L=%d): %s", name, r->N, r->L, cudaGetErrorString(e));
  }
  if (!r->timing) return;
  if (r->group_depth) {
    r->group_mm += mm;
    return;
  }
  cudaEvent_t b = take_event(r);
  CK(cudaEventRecord(b, r->stream));
  r->recs.push_back({name, bytes, mm, r->pending, b});
}
// algorithmic bytes per launch (read + write once; shared key / table reads once)
#define BYTES_add (24.0 * count * r->ct_words)
#define BYTES_add_plain (8.0 * count * (2.0 * r->ct_words + (double)r->L * r->N))
#define BYTES_mult_plain BYTES_add_plain
#define BYTES_copy (16.0 * count * r->ct_words)
#define BYTES_sum (8.0 * (count + 1.0) * r->ct_words)
#define BYTES_automorph (16.0 * n * ctw)
#define BYTES_gather (16.0 * n * (double)L * N)
#define BYTES_modup (8.0 * (double)count * ((double)L * N + (double)L * LP * N))
#define BYTES_ks_inner (8.0 * (double)count * LP * N * (L + 2.0) + 16.0 * L * (double)LP * N)
#define BYTES_moddown_lift (8.0 * (double)count * (2.0 * N + 2.0 * L * N))
#define BYTES_moddown_combine (8.0 * (double)count * 2.0 * L * N * (3 + (add0.items ? 0.5 : 0) + (d_add1 ? 1 : 0)))
#define BYTES_lift_QB (8.0 * n * 4.0 * (L + nB) * (double)N)
#define BYTES_tensor (8.0 * n * 7.0 * nt * (double)N)
#define BYTES_scale_round (8.0 * n * 3.0 * (nt + L) * (double)N)
#define BYTES_scatter_slots (16.0 * count * r->n_slots)
#define BYTES_gather_slots (16.0 * count * r->n_slots)
#define BYTES_pt_lift (8.0 * count * ((double)words + r->N))
#define BYTES_enc_c0 (8.0 * count * ((double)words + 2.0 * r->N))
#define BYTES_enc_sub_as (24.0 * count * (double)words)
#define BYTES_dec_inner (24.0 * count * (double)words)
#define BYTES_dec_scale (8.0 * count * (r->L + 1.0) * r->N)
#define BYTES_sample_uniform (8.0 * n * nl * (double)r->N)
#define BYTES_sample_cbd (8.0 * n * (double)r->N)
#define BYTES_ksk_b (0.0)
#define BYTES_ksk_fin (0.0)
#define LAUNCH(name, bytes, ...)          \
  do {                                    \
    launch_begin(r);                      \
    __VA_ARGS__;                          \
    launch_end(r, name, (double)(bytes)); \
  } while (0)

// ============================================================================
// kernels
// ============================================================================
#define GRID1(n, b) dim3((unsigned)(((n) + (b)-1) / (b)))

// NTT launcher -------------------------------------------------------------
static int g_ntt2_e = 8;  // words per thread of the two-pass NTT (8 or 16; CGB_NTT_E)
static int g_fp_regio = 3;  // FP64 NTT passes with register I/O: bit0 pass 0, bit1 pass 1 (CGB_FP_REGIO)
static bool g_md_epi = true;  // ModDown combine fused into its NTT's row pass (CGB_MD_EPI=0 -> separate kernel)
static bool g_fp_bconv = true;  // mult_cipher base conversions on the FP64 pipe (CGB_FP_BCONV)
static bool g_ks_md = true;   // ModDown row pass + combine fused into the Q limbs' k_ks_row (CGB_KS_MD)
static bool g_ks_row = true;  // ModUp row pass fused with the key inner product (CGB_KS_ROW=0 -> ks_inner)
static bool g_col_fused = true;  // INTT column pass + lift + forward column passes in one kernel (CGB_COL_FUSED)
template <int LA, int LB, bool QS, int E>
static void launch_ntt2_e(cgb_ring *r, bool fwd, const NttJob &job, int count) {
  NttJob second = job;
  second.src_base = nullptr;  // fused loads (lift / permutation) happen in the first pass only
  second.src_items = nullptr;
  second.galois = nullptr;
  second.lift = 0;
  auto grid = [&](int lm) {
    int nsubs = 1 << (LA + LB - lm), G = NTT2_TILE / (1 << lm);
    return dim3((unsigned)((size_t)count * job.nsub * (nsubs / G)));
  };
  const size_t s0 = ntt2_smem_bytes<LA, LB>(0), s1 = ntt2_smem_bytes<LA, LB>(1);
  const int T = NTT2_TILE / E;
  if (fwd) {
    k_ntt2<LA, LB, true, 0, QS, E><<<grid(LA), T, s0, r->stream>>>(job);
    k_ntt2<LA, LB, true, 1, QS, E><<<grid(LB), T, s1, r->stream>>>(second);
  } else {
    k_ntt2<LA, LB, false, 1, QS, E><<<grid(LB), T, s1, r->stream>>>(job);
    k_ntt2<LA, LB, false, 0, QS, E><<<grid(LA), T, s0, r->stream>>>(second);
  }
}
// one pass of the two-pass forward NTT (pass 0: columns, with the job's fused load)
template <int LA, int LB>
static void launch_ntt2_colpass(cgb_ring *r, const NttJob &job, int count) {
  const int G = NTT2_TILE / (1 << LA), nsubs = 1 << LB;
  const dim3 grid((unsigned)((size_t)count * job.nsub * (nsubs / G)));
  if (r->fp_ntt)
    k_ntt2_fp<LA, LB, true, 0><<<grid, NTT2_TILE / 8, ntt2_smem_bytes<LA, LB>(0), r->stream>>>(job);
  else
    k_ntt2<LA, LB, true, 0, true, 8><<<grid, NTT2_TILE / 8, ntt2_smem_bytes<LA, LB>(0), r->stream>>>(job);
}
template <int LA, int LB>
static void launch_ntt2_fp(cgb_ring *r, bool fwd, const NttJob &job, int count) {
  NttJob second = job;
  second.src_base = nullptr;
  second.src_items = nullptr;
  second.galois = nullptr;
  second.lift = 0;
  auto grid = [&](int lm) {
    int nsubs = 1 << (LA + LB - lm), G = NTT2_TILE / (1 << lm);
    return dim3((unsigned)((size_t)count * job.nsub * (nsubs / G)));
  };
  const size_t s0 = ntt2_smem_bytes<LA, LB>(0), s1 = ntt2_smem_bytes<LA, LB>(1);
  if (g_fp_regio && LA >= 5 && LB >= 5 && LA <= 8 && LB <= 8) {
    const size_t f0 = fpr_smem_bytes<LA, LB>(0), f1 = fpr_smem_bytes<LA, LB>(1);
    // register-I/O passes (16 words/thread) where CGB_FP_REGIO's bit for the pass is set
    const bool r0 = g_fp_regio & 1, r1 = g_fp_regio & 2;
    auto pass0 = [&](const NttJob &j, bool f) {
      if (r0) {
        if (f) launch_pdl(r, k_ntt2_fpr<LA, LB, true, 0>, grid(LA), NTT2_TILE / 16, f0, j, NoEpi{});
        else launch_pdl(r, k_ntt2_fpr<LA, LB, false, 0>, grid(LA), NTT2_TILE / 16, f0, j, NoEpi{});
      } else {
        if (f) k_ntt2_fp<LA, LB, true, 0><<<grid(LA), NTT2_TILE / 8, s0, r->stream>>>(j);
        else k_ntt2_fp<LA, LB, false, 0><<<grid(LA), NTT2_TILE / 8, s0, r->stream>>>(j);
      }
    };
    auto pass1 = [&](const NttJob &j, bool f) {
      if (r1) {
        if (f) launch_pdl(r, k_ntt2_fpr<LA, LB, true, 1>, grid(LB), NTT2_TILE / 16, f1, j, NoEpi{});
        else launch_pdl(r, k_ntt2_fpr<LA, LB, false, 1>, grid(LB), NTT2_TILE / 16, f1, j, NoEpi{});
      } else {
        if (f) k_ntt2_fp<LA, LB, true, 1><<<grid(LB), NTT2_TILE / 8, s1, r->stream>>>(j);
        else k_ntt2_fp<LA, LB, false, 1><<<grid(LB), NTT2_TILE / 8, s1, r->stream>>>(j);
      }
    };
    NttJob first = job, next = second;
    if (r0 && r1) {  // the words between the passes stay reduced doubles
      first.out_raw = 1;
      next.in_raw = 1;
    }
    if (fwd) {
      pass0(first, true);
      pass1(next, true);
    } else {
      pass1(first, false);
      pass0(next, false);
    }
    return;
  }
  const int T = NTT2_TILE / 8;
  if (fwd) {
    k_ntt2_fp<LA, LB, true, 0><<<grid(LA), T, s0, r->stream>>>(job);
    k_ntt2_fp<LA, LB, true, 1><<<grid(LB), T, s1, r->stream>>>(second);
  } else {
    k_ntt2_fp<LA, LB, false, 1><<<grid(LB), T, s1, r->stream>>>(job);
    k_ntt2_fp<LA, LB, false, 0><<<grid(LA), T, s0, r->stream>>>(second);
  }
}
template <int LA, int LB, bool QS>
static void launch_ntt2(cgb_ring *r, bool fwd, const NttJob &job, int count) {
  if (r->fp_ntt) launch_ntt2_fp<LA, LB>(r, fwd, job, count);
  else if (g_ntt2_e == 16) launch_ntt2_e<LA, LB, QS, 16>(r, fwd, job, count);
  else launch_ntt2_e<LA, LB, QS, 8>(r, fwd, job, count);
}
template <int LA, int LB>
static void ntt2_attrs() {
  const int s = (int)std::max(ntt2_smem_bytes<LA, LB>(0), ntt2_smem_bytes<LA, LB>(1));
#define NTT2A(F, P, Q, E) CK(cudaFuncSetAttribute(k_ntt2<LA, LB, F, P, Q, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, s));
  NTT2A(true, 0, true, 8) NTT2A(true, 1, true, 8) NTT2A(false, 0, true, 8) NTT2A(false, 1, true, 8)
  NTT2A(true, 0, false, 8) NTT2A(true, 1, false, 8) NTT2A(false, 0, false, 8) NTT2A(false, 1, false, 8)
  NTT2A(true, 0, true, 16) NTT2A(true, 1, true, 16) NTT2A(false, 0, true, 16) NTT2A(false, 1, true, 16)
  NTT2A(true, 0, false, 16) NTT2A(true, 1, false, 16) NTT2A(false, 0, false, 16) NTT2A(false, 1, false, 16)
#undef NTT2A
  const int f0 = (int)fpr_smem_bytes<LA, LB>(0), f1 = (int)fpr_smem_bytes<LA, LB>(1);
  CK(cudaFuncSetAttribute(k_ntt2_fpr<LA, LB, true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, f0));
  CK(cudaFuncSetAttribute(k_ntt2_fpr<LA, LB, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, f1));
  CK(cudaFuncSetAttribute(k_ntt2_fpr<LA, LB, false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, f0));
  CK(cudaFuncSetAttribute(k_ntt2_fpr<LA, LB, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, f1));
  CK(cudaFuncSetAttribute(k_ntt2_fp<LA, LB, true, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, s));
  CK(cudaFuncSetAttribute(k_ntt2_fp<LA, LB, true, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, s));
  CK(cudaFuncSetAttribute(k_ntt2_fp<LA, LB, false, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, s));
  CK(cudaFuncSetAttribute(k_ntt2_fp<LA, LB, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, s));
}
static void launch_ntt(cgb_ring *r, bool fwd, NttJob &job, int count) {
  if (count <= 0 || job.nsub <= 0) return;
  job.mods = r->d_mods;
  job.logN = r->logN;
  const double bytes = 16.0 * (double)count * job.nsub * r->N;
  if (r->logN >= 12) {  // two passes over 2048-word tiles, twiddles staged in shared memory
    launch_begin(r);
    bool qs = true;  // every unit's modulus = 1 mod 2^32 (all but the plaintext modulus)
    for (int u = 0; u < job.nsub; u++) qs = qs && job.sub_mod[u] != r->iT;
#define LN2(A, B) (qs ? launch_ntt2<A, B, true>(r, fwd, job, count) : launch_ntt2<A, B, false>(r, fwd, job, count))
    switch (r->logN) {
      case 12: LN2(6, 6); break;
      case 13: LN2(6, 7); break;
      case 14: LN2(CGB_A14, 14 - CGB_A14); break;
      case 15: LN2(7, 8); break;
      default: LN2(8, 8); break;
    }
#undef LN2
    r->launches++;  // two kernels per transform (launch_end counts the other)
    // algorithmic bytes: each limb-poly read and written once (16 B/word), whatever the passes
    launch_end(r, fwd ? "ntt_fwd" : "ntt_inv", bytes, (double)count * job.nsub * (r->N / 2) * r->logN);
    return;
  }
  int E = r->ntt_E(), T = r->ntt_threads();
  size_t smem = r->ntt_smem();
  dim3 grid((unsigned)(count * job.nsub));
  bool qs = true;
  for (int u = 0; u < job.nsub; u++) qs = qs && job.sub_mod[u] != r->iT;
#define LNTT(EE)                                                                        \
  do {                                                                                  \
    if (qs) {                                                                           \
      if (fwd) k_ntt<EE, true, true><<<grid, T, smem, r->stream>>>(job);                \
      else k_ntt<EE, false, true><<<grid, T, smem, r->stream>>>(job);                   \
    } else {                                                                            \
      if (fwd) k_ntt<EE, true, false><<<grid, T, smem, r->stream>>>(job);               \
      else k_ntt<EE, false, false><<<grid, T, smem, r->stream>>>(job);                  \
    }                                                                                   \
  } while (0)
  launch_begin(r);
  switch (E) {
    case 32: LNTT(32); break;
    case 16: LNTT(16); break;
    case 8: LNTT(8); break;
    case 4: LNTT(4); break;
    default: LNTT(2); break;
  }
#undef LNTT
  launch_end(r, fwd ? "ntt_fwd" : "ntt_inv", bytes, (double)count * job.nsub * (r->N / 2) * r->logN);
}
// NTT over `nlimb` limbs of `npoly` polys per item, limb l of poly p at unit p*nlimb+l
static void ntt_items(cgb_ring *r, bool fwd, u64 *base, u64 *const *items, u64 item_stride, int count, int npoly,
                      int nlimb, const int *mod_of_limb, int poly_units = -1) {
  NttJob job{};
  job.base = base;
  job.items = items;
  job.item_stride = item_stride;
  int pu = poly_units < 0 ? nlimb : poly_units;
  int n = 0;
  for (int p = 0; p < npoly; p++)
    for (int l = 0; l < nlimb; l++) {
      if (n >= NTT_MAXSUB) FAIL(CGB_ERR_PARAM, "too many NTT units per item");
      job.sub_off[n] = (unsigned short)(p * pu + l);
      job.sub_mod[n] = (unsigned char)mod_of_limb[l];
      n++;
    }
  job.nsub = n;
  launch_ntt(r, fwd, job, count);
}

// elementwise kernels --------------------------------------------------------
// out[p][l][j] = a + b  (mod q_l), per-item pointers
// Pointwise kernels: each thread moves two consecutive words with 16-byte
// loads/stores; grid = (word pairs / TPB, items).
__device__ __forceinline__ ulonglong2 ld2(const u64 *p) { return __ldg(reinterpret_cast<const ulonglong2 *>(p)); }
__device__ __forceinline__ void st2(u64 *p, u64 x, u64 y) { *reinterpret_cast<ulonglong2 *>(p) = make_ulonglong2(x, y); }

__global__ void k_add(u64 *const *out, const u64 *const *a, const u64 *const *b, const ModTab *mods, int L, int logN,
                      u64 words) {
  const int item = blockIdx.y;
  const u64 i = 2 * ((u64)blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= words) return;
  const u64 q = mods[(int)((i >> logN) % L)].q;
  const ulonglong2 x = ld2(a[item] + i), y = ld2(b[item] + i);
  st2(out[item] + i, add_mod(x.x, y.x, q), add_mod(x.y, y.y, q));
}
// c0 * pt, c1 * pt: the plaintext limb is read once for both polys; words = L N
__global__ void k_mult_plain(u64 *const *out, const u64 *const *a, const u64 *const *pt, const ModTab *mods, int L,
                             int logN, u64 words) {
  const int item = blockIdx.y;
  const u64 i = 2 * ((u64)blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= words) return;
  const ModTab &M = mods[(int)(i >> logN)];
  const u64 *A = a[item];
  u64 *O = out[item];
  const ulonglong2 p = ld2(pt[item] + i), x0 = ld2(A + i), x1 = ld2(A + words + i);
  st2(O + i, mul_mod(x0.x, p.x, M), mul_mod(x0.y, p.y, M));
  st2(O + words + i, mul_mod(x1.x, p.x, M), mul_mod(x1.y, p.y, M));
}
// c0 + pt, c1 copied; words = L N
__global__ void k_add_plain(u64 *const *out, const u64 *const *a, const u64 *const *pt, const ModTab *mods, int L,
                            int logN, u64 words) {
  const int item = blockIdx.y;
  const u64 i = 2 * ((u64)blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= words) return;
  const u64 q = mods[(int)(i >> logN)].q;
  const u64 *A = a[item];
  u64 *O = out[item];
  const ulonglong2 p = ld2(pt[item] + i), x0 = ld2(A + i), x1 = ld2(A + words + i);
  st2(O + i, add_mod(x0.x, p.x, q), add_mod(x0.y, p.y, q));
  st2(O + words + i, x1.x, x1.y);
}
__global__ void k_copy(u64 *const *out, const u64 *const *a, u64 words) {
  const int item = blockIdx.y;
  const u64 i = 2 * ((u64)blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= words) return;
  const ulonglong2 x = ld2(a[item] + i);
  st2(out[item] + i, x.x, x.y);
}
// gather items into a strided workspace: dst[item * dstride + w] = src[item][off + w]
__global__ void k_gather(u64 *dst, u64 dstride, const u64 *const *src, u64 off, u64 words) {
  int item = blockIdx.y;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= words) return;
  dst[(u64)item * dstride + i] = src[item][off + i];
}
// sum of count items (tree in one kernel: each thread sums one word over all items)
__global__ void k_sum(u64 *out, const u64 *const *a, int count, const ModTab *mods, int L, int logN, u64 words) {
  const u64 i = 2 * ((u64)blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= words) return;
  const u64 q = mods[(int)((i >> logN) % L)].q;
  u64 s0 = 0, s1 = 0;
  for (int k = 0; k < count; k++) {
    const ulonglong2 x = ld2(a[k] + i);
    s0 = add_mod(s0, x.x, q);
    s1 = add_mod(s1, x.y, q);
  }
  st2(out + i, s0, s1);
}

// Galois automorphism in the evaluation domain: out[k] = in[perm_g(k)]
__device__ __forceinline__ u32 dbrev(u32 x, int logN) { return __brev(x) >> (32 - logN); }
__global__ void k_automorph(u64 *dst /*[item][2][L][N]*/, const u64 *const *src, const u64 *gs, int L, int logN) {
  int item = blockIdx.y;
  u64 N = 1ull << logN, words = 2ull * L * N;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= words) return;
  u64 k = i & (N - 1), base = i - k;
  u64 g = gs[item];
  u64 e = 2ull * dbrev((u32)k, logN) + 1;
  u64 se = (e * g) & (2 * N - 1);
  u64 sk = dbrev((u32)((se - 1) >> 1), logN);
  dst[(u64)item * words + i] = src[item][base + sk];
}
// same, on a plain [limbs][N] array (secret key -> sigma_g(s))
__global__ void k_automorph_flat(u64 *dst, const u64 *src, u64 g, int nlimb, int logN) {
  u64 N = 1ull << logN, words = (u64)nlimb * N;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= words) return;
  u64 k = i & (N - 1), base = i - k;
  u64 e = 2ull * dbrev((u32)k, logN) + 1;
  u64 se = (e * g) & (2 * N - 1);
  dst[i] = src[base + dbrev((u32)((se - 1) >> 1), logN)];
}

// key switching: ModUp of dnum = L one-limb digits -------------------------
// D[item][j][l][N] (l over Q u P) : l == j -> NTT-form input limb ; else centred coeff reduced
__global__ void k_modup(u64 *D, const u64 *xcoef /*[item][L][N]*/, const u64 *xin /*[item][L][N]*/,
                        const ModTab *mods, int L, int logN) {
  int item = blockIdx.y;
  u64 N = 1ull << logN;
  u64 words = (u64)L * (L + 1) * N;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= words) return;
  u64 jn = i & (N - 1), rest = i >> logN;
  int l = (int)(rest % (L + 1)), j = (int)(rest / (L + 1));
  const u64 *src = (l == j ? xin : xcoef) + ((u64)item * L + j) * N;
  u64 v = src[jn];
  if (l != j) v = centred_to(v, mods[j].q, mods[l].q);
  D[(u64)item * words + i] = v;
}
// acc[item][p][l][N] = sum_j D[j][l] * key[j][p][l]   (p = 0: b, 1: a)
// acc[item][p][l][N] = sum_j D[j][l] * key[j][p][l]  (p = 0: b, 1: a); the digit's own
// limb comes from the NTT-form input.  Keys carry Shoup companions (key + kw)
// and are held in registers while consecutive items share them (every item of
// a doubling / folding wave does); lazy sums in [0, 2Lq) are reduced once.
struct KsSrc {            // the polynomial to key-switch (NTT form over Q)
  const u64 *base;        // contiguous items at base + item * stride
  u64 stride;
  u64 *const *items;      // or per-item pointers + word offset
  u64 off;
  const u64 *g;           // per-item Galois element: read word perm_g(k)
};
__device__ __forceinline__ u64 ks_src_word(const KsSrc &x, int item, int limb, u32 k, int logN) {
  if (x.items) {
    const u32 kk = x.g ? perm_g(k, x.g[item], logN) : k;
    return x.items[item][x.off + ((u64)limb << logN) + kk];
  }
  return x.base[(u64)item * x.stride + ((u64)limb << logN) + k];
}
// words k0 .. k0 + 3 (k0 a multiple of 4) of ks_src_word: one sector per 4 words
__device__ __forceinline__ void ks_src_block4(const KsSrc &x, int item, int limb, u32 k0, int logN, u64 out[4]) {
  if (x.items) {
    const u64 *p = x.items[item] + x.off + ((u64)limb << logN);
    if (x.g) {
      gather4(p, k0, x.g[item], logN, out);
    } else {
      ld256(p + k0, out);
    }
    return;
  }
  ld256(x.base + (u64)item * x.stride + ((u64)limb << logN) + k0, out);
}
template <int L>
__global__ void k_ks_inner(u64 *acc, const u64 *D, KsSrc xin, const u64 *const *keys, u64 kw,
                           const ModTab *mods, int logN, int count, int per_block) {
  constexpr int LP = L + 1;
  const u64 N = 1ull << logN;
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;  // over [l][N]
  if (i >= LP * N) return;
  const int l = (int)(i >> logN);
  const u64 q = mods[l].q;
  const u64 jn = i & (N - 1);
  const int it0 = blockIdx.y * per_block, it1 = min(count, it0 + per_block);
  const u64 *kprev = nullptr;
  u64 kv[2][L], ks[2][L];
  // digits of the next item are loaded before the current one is reduced, so
  // the loads of consecutive items overlap (the kernel is load-latency bound)
  auto load_digits = [&](int item, u64 *d) {
    const u64 *Di = D + (u64)item * L * LP * N;
#pragma unroll
    for (int j = 0; j < L; j++)
      d[j] = (l == j) ? ks_src_word(xin, item, j, (u32)jn, logN) : __ldcs(Di + (u64)j * LP * N + i);
  };
  u64 dc[L], dn[L];
  if (it0 < it1) load_digits(it0, dc);
  for (int item = it0; item < it1; item++) {
    if (item + 1 < it1) load_digits(item + 1, dn);
    const u64 *K = keys[item];
    if (K != kprev) {
#pragma unroll
      for (int j = 0; j < L; j++)
#pragma unroll
        for (int p = 0; p < 2; p++) {
          const u64 off = ((u64)j * 2 + p) * LP * N + i;
          kv[p][j] = __ldg(K + off);
          ks[p][j] = __ldg(K + kw + off);
        }
      kprev = K;
    }
    u64 s0 = 0, s1 = 0;
#pragma unroll
    for (int j = 0; j < L; j++) {
      const u64 d = dc[j];
      s0 += mul_shoup_lazy(d, kv[0][j], ks[0][j], q);
      s1 += mul_shoup_lazy(d, kv[1][j], ks[1][j], q);
      if ((j & 3) == 3 || j == L - 1) {  // keep lazy sums below 8q < 2^64
        const u64 q4 = 4 * q, q2 = 2 * q;
        s0 = s0 >= q4 ? s0 - q4 : s0;
        s0 = s0 >= q2 ? s0 - q2 : s0;
        s1 = s1 >= q4 ? s1 - q4 : s1;
        s1 = s1 >= q2 ? s1 - q2 : s1;
      }
    }
#pragma unroll
    for (int j = 0; j < L; j++) dc[j] = dn[j];
    acc[((u64)item * 2 + 0) * LP * N + i] = s0 >= q ? s0 - q : s0;
    acc[((u64)item * 2 + 1) * LP * N + i] = s1 >= q ? s1 - q : s1;
  }
}
// Shoup companions of a key: dst[i] = floor(src[i] * 2^64 / q_limb)
__global__ void k_key_shoup(u64 *dst, const u64 *src, const ModTab *mods, int L, int iP, int logN, u64 words) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= words) return;
  int l = (int)((i >> logN) % (L + 1));
  u64 q = mods[l == L ? iP : l].q;
  dst[i] = (u64)((((unsigned __int128)src[i]) << 64) / q);
}
// the key's FP64 plane: every word as an exact double (k_ks_row's products read it
// without a per-word integer -> double conversion)
__global__ void k_key_fp(u64 *dst, const u64 *src, u64 words) {
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= words) return;
  dst[i] = (u64)__double_as_longlong(u2d(src[i]));
}
// ModDown lift: W[item][p][l][N] = centred(acc[item][p][L] (coeff, mod P)) mod q_l
__global__ void k_moddown_lift(u64 *W, const u64 *acc, const ModTab *mods, int L, int iP, int logN) {
  int item = blockIdx.y;
  u64 N = 1ull << logN, LP = L + 1, words = 2ull * L * N;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= words) return;
  u64 jn = i & (N - 1), rest = i >> logN;
  int l = (int)(rest % L), p = (int)(rest / L);
  u64 v = acc[(((u64)item * 2 + p) * LP + L) * N + jn];
  W[(u64)item * words + i] = centred_to(v, mods[iP].q, mods[l].q);
}
// out[p][l] = (acc[p][l] - W[p][l]) * P^-1 + add0 (poly 0 only, optionally read through the
// automorphism) + add1 (both polys)
__global__ void k_moddown_combine(u64 *const *out, const u64 *acc, const u64 *W, KsSrc add0,
                                  const u64 *const *add1, const ModTab *mods, const Consts *C, int L, int logN) {
  int item = blockIdx.y;
  u64 N = 1ull << logN, LP = L + 1, words = 2ull * L * N;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= words) return;
  u64 jn = i & (N - 1), rest = i >> logN;
  int l = (int)(rest % L), p = (int)(rest / L);
  u64 q = mods[l].q;
  u64 a = acc[(((u64)item * 2 + p) * LP + l) * N + jn];
  u64 v = mul_shoup(sub_mod(a, W[(u64)item * words + i], q), C->Pinvq[l], C->Pinvq_sh[l], q);
  if (p == 0 && (add0.items || add0.base)) v = add_mod(v, ks_src_word(add0, item, l, (u32)jn, logN), q);
  if (add1) v = add_mod(v, add1[item][i], q);
  out[item][i] = v;
}

// ModDown combine as the store epilogue of the forward row pass that produces
// W = NTT_l(lift_P(INTT_P(acc_P))): out = (acc_l - W) P^-1 (+ add0 on poly 0)
// (+ add1), the same words as k_moddown_combine without W's round trip.
#ifndef CGB_KEYPROD_Q
#define CGB_KEYPROD_Q 1  // key products estimate the quotient from the rounded product (no k * (1/q) DMUL)
#endif
#ifndef CGB_ABLATE
#define CGB_ABLATE 0  // timing experiments only (wrong results): which loads / phases bound k_ks_row
#endif
struct MdEpi {
  static constexpr bool active = true;
  u64 *const *out;
  const u64 *acc;
  KsSrc add0;
  const u64 *const *add1;
  const ModTab *mods;
  const Consts *C;
  int L, logN;
  __device__ void store(int item, int unit, u64 pos, const u64 *w, int n) const {
    const int pp = unit / L, l = unit - pp * L;
    const u64 N = 1ull << logN, q = mods[l].q, pi = C->Pinvq[l], pis = C->Pinvq_sh[l];
    const u64 *a = acc + (((u64)item * 2 + pp) * (L + 1) + l) * N + pos;
    u64 *o = out[item] + (u64)unit * N + pos;
    const u64 *b = add1 ? add1[item] + (u64)unit * N + pos : nullptr;
    const bool a0 = pp == 0 && (add0.items || add0.base);
    if (n == 4) {
      u64 av[4];
      ld256(a, av);
      combine4(item, unit, pos, w, av);
    } else {
      for (int k = 0; k < n; k++) {
        u64 v = mul_shoup(sub_mod(a[k], w[k], q), pi, pis, q);
        if (a0) v = add_mod(v, ks_src_word(add0, item, l, (u32)(pos + k), logN), q);
        if (b) v = add_mod(v, b[k], q);
        o[k] = v;
      }
    }
  }
  // start the async copies of the epilogue operands of words pos .. pos + 3 of unit
  // `unit` into stg[0..3] (input, rotate_add) and stg[16..19] (the 32-byte block of
  // the automorphed c0 holding them)
  __device__ void prefetch4(int item, int unit, u64 pos, u64 *stg) const {
    const int pp = unit / L, l = unit - pp * L;
    const u64 N = 1ull << logN;
    if (add1) {
      const u64 *b = add1[item] + (u64)unit * N + pos;
      cp_async16(stg, b);
      cp_async16(stg + 2, b + 2);
    }
    if (pp == 0 && (add0.items || add0.base)) {
      const u64 *c;
      if (add0.items) {
        c = add0.items[item] + add0.off + ((u64)l << logN);
        c += add0.g ? (perm_g((u32)pos, add0.g[item], logN) & ~3u) : pos;
      } else {
        c = add0.base + (u64)item * add0.stride + ((u64)l << logN) + pos;
      }
      cp_async16(stg + 16, c);
      cp_async16(stg + 18, c + 2);
    }
  }
  // combine4 with the operands prefetch4 staged (after cp_async_wait_all)
  __device__ void combine4_staged(int item, int unit, u64 pos, const u64 *w, const u64 *av, const u64 *stg) const {
    const int pp = unit / L, l = unit - pp * L;
    const u64 N = 1ull << logN, q = mods[l].q, pi = C->Pinvq[l], pis = C->Pinvq_sh[l];
    const bool a0 = pp == 0 && (add0.items || add0.base);
    const bool gal = a0 && add0.items && add0.g;
    const u64 g = gal ? add0.g[item] : 1;
    u64 v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      v[k] = mul_shoup(sub_mod(av[k], w[k], q), pi, pis, q);
      if (a0) v[k] = add_mod(v[k], stg[16 + (gal ? (perm_g((u32)(pos + k), g, logN) & 3u) : k)], q);
      if (add1) v[k] = add_mod(v[k], stg[k], q);
    }
    st256(out[item] + (u64)unit * N + pos, v[0], v[1], v[2], v[3]);
  }
  // combine4 on the FP64 pipe, from the unreduced row-pass output xw (|xw| < 12q) and
  // FP64 accumulator sums xa (|xa| < 11q): (xa - xw) P^-1 (+ c0) (+ add1), every
  // intermediate an exact integer (|y| < 4.7q), canonical at the store -- the same
  // residues as the integer combine
  __device__ void combine4_fp(int item, int unit, u64 pos, const double *xw, const double *xa) const {
    const int pp = unit / L, l = unit - pp * L;
    const u64 N = 1ull << logN;
    const ModTab &M = mods[l];
    const double q = M.qd, qi = M.qinv;
    const double2 pinv = C->fPinvq[l];
    const bool a0 = pp == 0 && (add0.items || add0.base);
    u64 bv[4], cv[4];
    if (CGB_ABLATE & 8) {
#pragma unroll
      for (int k = 0; k < 4; k++) bv[k] = pos + k, cv[k] = pos + 2 * k;
    } else {
      if (add1) ld256(add1[item] + (u64)unit * N + pos, bv);
      if (a0) ks_src_block4(add0, item, l, (u32)pos, logN, cv);
    }
    u64 v[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
      // |xa - reduce(xw)| < 11.5q: exact, inside fp_mulmod's analysed range (< 12q)
      double y = fp_mulmod(xa[k] - fp_reduce(xw[k], q, qi), pinv.x, pinv.y, q);
      if (a0) y += u2d(cv[k]);
      if (add1) y += u2d(bv[k]);
      v[k] = fp_canon(y, q, qi);
    }
    st256(out[item] + (u64)unit * N + pos, v[0], v[1], v[2], v[3]);
  }
  // words pos .. pos + 3 of unit `unit`: W's words w, the accumulator's words av
  __device__ void combine4(int item, int unit, u64 pos, const u64 *w, const u64 *av) const {
    const int pp = unit / L, l = unit - pp * L;
    const u64 N = 1ull << logN, q = mods[l].q, pi = C->Pinvq[l], pis = C->Pinvq_sh[l];
    u64 *o = out[item] + (u64)unit * N + pos;
    const u64 *b = add1 ? add1[item] + (u64)unit * N + pos : nullptr;
    const bool a0 = pp == 0 && (add0.items || add0.base);
    {
      u64 bv[4] = {0, 0, 0, 0}, cv[4] = {0, 0, 0, 0};
      if (b) ld256(b, bv);
      if (a0) ks_src_block4(add0, item, l, (u32)pos, logN, cv);
      u64 v[4];
#pragma unroll
      for (int k = 0; k < 4; k++) {
        v[k] = mul_shoup(sub_mod(av[k], w[k], q), pi, pis, q);
        if (a0) v[k] = add_mod(v[k], cv[k], q);
        if (b) v[k] = add_mod(v[k], bv[k], q);
      }
      st256(o, v[0], v[1], v[2], v[3]);
    }
  }
};

// ModUp's forward row pass fused with the key inner product.  One CTA owns row
// tile `tile` of limb l (of Q u P) of one item: for every digit j != l it runs the
// forward row pass of D unit (j, l) (the column pass's output) in registers and
// multiplies by the key words at the same positions; digit l is the key-switched
// polynomial itself (NTT form, read through the automorphism).  Products and the
// sum stay FP64: |row pass output| < 12q (unreduced forward pass), each product lies
// in (-2.7q, 2.7q) with the key's w/q formed by one DMUL (scripts/sim/fp_bounds.py),
// so a sum of <= 4 digits is an exact integer < 11q < 2^53 and its canonical residue
// equals the integer path's.  acc[item][p][l] is written
// once; D's row-pass output never reaches memory.
#ifndef CGB_KSROW_GTW
#define CGB_KSROW_GTW 0  // row twiddles read through L1 instead of staged: measured slower
#endif
#ifndef CGB_KSROW_EPF
#define CGB_KSROW_EPF 0  // MODE 2: epilogue operands prefetched (cp.async) into the exchange tile: measured slower
#endif
#ifndef CGB_KSROW_TWW
#define CGB_KSROW_TWW 1  // staged row twiddles as w only (w/q formed by one DMUL on use): half the shared
                        // memory and half the twiddle LDS traffic of the LSU-bound row kernels (0.94 -> 0.90 ms
                        // per 768 key switches in ks_row_md)
#endif
constexpr bool TWW = CGB_KSROW_TWW && !CGB_KSROW_GTW;
#ifndef CGB_KSROW_PF
#define CGB_KSROW_PF 0  // L2 prefetch of the next tile / gathered blocks: measured slower
#endif
#ifndef CGB_KSROW_FPC
#define CGB_KSROW_FPC 1  // MODE 2: the ModDown combine on the FP64 pipe
#endif
#ifndef CGB_KSROW_G4
#define CGB_KSROW_G4 0  // measured: the per-word own-digit loads are faster here (profiles/r02)
#endif
// words of k_ks_row's exchange tile: the padded row tile, or (EPF) 32 staging words per thread
__host__ __device__ constexpr int ksr_data_words(int LB) {
  return ((((NTT2_TILE >> LB) * fpr_padm(LB, 1)) + 1) & ~1) > (CGB_KSROW_EPF ? 32 * (NTT2_TILE / 16) : 0)
             ? ((((NTT2_TILE >> LB) * fpr_padm(LB, 1)) + 1) & ~1)
             : 32 * (NTT2_TILE / 16);
}
#ifndef CGB_KSROW_KSTAGE
#define CGB_KSROW_KSTAGE 0  // key words cp.async-staged in shared memory during the row pass: measured slower
                                  // (28.8 -> 42.6 ms ks_row_md per decode step; 36.6 with TWW, profiles/r02/ab_kstage.log)
#endif
// bytes of k_ks_row's key staging area: 2 polys x 16 words per thread x 128 threads
constexpr int KSTAGE_BYTES = CGB_KSROW_KSTAGE ? 2 * 16 * 8 * (NTT2_TILE / 16) : 0;
#ifndef CGB_KSROW_RPF
#define CGB_KSROW_RPF 0  // next row tile prefetched into registers during the current tile's work
#endif
#ifndef CGB_KSROW_CPF
#define CGB_KSROW_CPF 1  // next row tile prefetched by cp.async into a warp-private staging buffer
                        // (in the shared memory TWW frees: 3 CTAs per SM as before): 0.90 -> 0.86 ms
#endif
// bytes of k_ks_row's staged row twiddles
__host__ __device__ constexpr size_t ksr_tw_bytes(int LB) {
  return CGB_KSROW_GTW ? 0 : (CGB_KSROW_TWW ? 8 : 16) * (size_t)(NTT2_TILE + (NTT2_TILE >> LB));
}
// bytes of the cp.async staging buffer: the tile's rows at a pitch of 2^LB + 8 words
__host__ __device__ constexpr size_t ksr_pf_bytes(int LB) {
  return CGB_KSROW_CPF ? 8 * (size_t)(NTT2_TILE >> LB) * ((1 << LB) + 8) : 0;
}
#ifndef CGB_KSROW_MINB
#if CGB_KSROW_RPF
#define CGB_KSROW_MINB 2
#else
#define CGB_KSROW_MINB 3  // <= 168 registers: 3 CTAs per SM (MODE 2 would otherwise take 208)
#endif
#endif
#if CGB_KSROW_PF >= 2  // 2: the next tile into L1; 3: and the next digit's key rows
#define KSROW_PREFETCH(p) prefetch_l1(p)
#else
#define KSROW_PREFETCH(p) prefetch_l2(p)
#endif
#define KSROW_BOUNDS __launch_bounds__(NTT2_TILE / 16, CGB_KSROW_MINB)
// A row of the tile belongs to M / E <= 16 consecutive threads of ONE warp, so the
// exchange between the two register phases of a row pass only needs a warp-level
// barrier (ROW_SYNC, cgb_device.cuh): the CTA's warps run their rows independently.
// MODE 0: every limb of Q u P; 1: the P limb only; 2: the Q limbs, followed by
// ModDown's forward row pass of W (the column-pass output of lift(INTT(acc_P)))
// with the combine as its epilogue -- the Q limbs' accumulators never reach memory.
template <int LA, int LB, int L, int MODE = 0, bool UNRED = false>
__global__ void KSROW_BOUNDS k_ks_row(u64 *acc, const u64 *D, KsSrc xin,
                                                           const u64 *const *keys, const ModTab *mods, int iP,
                                                           int count, const u64 *W, MdEpi epi, int raw) {
  extern __shared__ u64 sm3[];
  constexpr int E = 16, LM = LB, M = 1 << LM, LOGN = LA + LB, LP = L + 1;
  constexpr int G = NTT2_TILE / M, TPS = M / E, TILES = (1 << LA) / G;
  constexpr int PSH = fpr_psh(LM, 1), PADM = fpr_padm(LM, 1);
  constexpr int RA = 4, RB = LM - 4;
  using PA = PhaseShape<LM, 0, RA, E>;
  using PB = PhaseShape<LM, RA, RB, E>;
  static_assert(PB::ST == 1 && PB::K % 4 == 0, "row-pass output: runs of >= 4 consecutive words");
  const u64 N = 1ull << LOGN;
  const int tile = blockIdx.x % TILES, rest = blockIdx.x / TILES;
  constexpr int NL = MODE == 0 ? LP : MODE == 1 ? 1 : L;  // limbs per item in the grid
  const int l = MODE == 1 ? L : rest % NL, item = rest / NL;
  const ModTab &Md = mods[l == L ? iP : l];
  const double qd = Md.qd, qinv = Md.qinv;
  const int tid = threadIdx.x, g = tid / TPS, tl = tid % TPS, first = tile * G;
  const u64 row0 = (u64)(first + g) << LM;  // word offset of this thread's row
#if CGB_KSROW_GTW
  // the row twiddles are read through L1 from the transposed global table (the
  // freed shared memory stages MODE 2's epilogue operands)
  constexpr bool GT = true;
  const double2 *tw = reinterpret_cast<const double2 *>(Md.ftw1t) + row0;
#else
  // the tile's row twiddles (same for every digit) staged once: rows of M + 1 pairs
  // (TWW: rows of M + 1 doubles, the w/q halves formed on use -- half the shared memory)
  constexpr bool GT = false;
#if CGB_KSROW_TWW
  double *twd = reinterpret_cast<double *>(sm3 + ksr_data_words(LM));
  auto stage_tw = [&](const u64 *table) {
    const double2 *gt = reinterpret_cast<const double2 *>(table) + ((u64)first << LM);
#pragma unroll
    for (int i = 0; i < E; i++) {
      const int e = tid + i * (NTT2_TILE / E);
      twd[e + (e >> LM)] = __ldg(reinterpret_cast<const double *>(table == Md.ftw1t ? Md.ftw1tw : Md.fitw1tw) + ((u64)first << LM) + e);
    }
  };
  stage_tw(Md.ftw1t);
  const double2 *tw = reinterpret_cast<const double2 *>(twd + g * (M + 1));
#else
  double2 *tws = reinterpret_cast<double2 *>(sm3 + ksr_data_words(LM));
  auto stage_tw = [&](const u64 *table) {
    const double2 *gt = reinterpret_cast<const double2 *>(table) + ((u64)first << LM);
#pragma unroll
    for (int i = 0; i < E; i++) {
      const int e = tid + i * (NTT2_TILE / E);
      tws[e + (e >> LM)] = __ldg(gt + e);
    }
  };
  if (!(CGB_ABLATE & 32)) stage_tw(Md.ftw1t);
  const double2 *tw = tws + g * (M + 1);
#endif
#endif
  // row tiles this CTA reads, in order: D(j, l) for the digits j != l, then (MODE 2) W(0, l), W(1, l)
  constexpr int NT_MAX = L + 2;
  const int ntile = (l == L ? L : L - 1) + (MODE == 2 ? 2 : 0);
  auto tile_src = [&](int t) -> const u64 * {
    const int nd = l == L ? L : L - 1;
    if (t < nd) {
      const int j = (l == L || t < l) ? t : t + 1;
      return D + ((u64)item * L * LP + (u64)j * LP + l) * N + ((u64)first << LM);
    }
    return W + ((u64)item * 2 * L + (u64)(t - nd) * L + l) * N + ((u64)first << LM);
  };
  (void)NT_MAX;
  pdl_start_dependents();
  pdl_wait();
  int tcur = 0;
#if CGB_KSROW_RPF
  // software pipelining: the NEXT row tile's words are loaded into registers while
  // this tile's row pass and key products run (loads in flight across the compute)
  u64 nv[PA::K];
  auto issue_tile = [&](int t) {
    if (t < ntile) {
      const u64 *src = tile_src(t) + ((u64)g << LM);
#pragma unroll
      for (int k = 0; k < PA::K; k++) nv[k] = __ldcs(src + PA::idx(tl, 0, k));
    }
  };
  issue_tile(0);
  auto load_tile = [&](double *x) {
#pragma unroll
    for (int k = 0; k < PA::K; k++) {
      x[k] = (raw & 1) ? r2d(nv[k]) : u2d(nv[k]);
      if constexpr (UNRED) x[k] = fp_reduce(x[k], qd, qinv);
    }
    issue_tile(tcur + 1);
    if (tcur == 0) __syncthreads(); else ROW_SYNC();  // twiddles staged; the previous tile's phase-B reads are done
    tcur++;
  };
#elif CGB_KSROW_CPF
  // The NEXT row tile streams into shared memory by 16-byte asynchronous copies while
  // this tile's row pass and key products run: no registers are held and no warp
  // waits on the tile's global loads.  A warp copies exactly the rows it consumes
  // (its 32 / TPS rows are contiguous in the tile), so the hand-over is warp-local.
  constexpr int PFP = M + 8;  // row pitch: the rows a half-warp reads in phase A fall in different bank halves
  u64 *pfb = sm3 + ksr_data_words(LM) + (ksr_tw_bytes(LB) + KSTAGE_BYTES) / 8;
  const int lane = tid & 31, wrow0 = (tid >> 5) * (32 / TPS);
  auto issue_tile = [&](int t) {
    if (t < ntile) {
      constexpr int CH = (32 / TPS) * (M / 2);  // 16-byte chunks of the warp's rows
      const u64 *src = tile_src(t) + ((u64)wrow0 << LM);
#pragma unroll
      for (int i = 0; i < CH / 32; i++) {
        const int c = lane + 32 * i, r = c / (M / 2), cc = c % (M / 2);
        cp_async16(pfb + (wrow0 + r) * PFP + 2 * cc, src + 2 * c);
      }
    }
    cp_async_commit();
  };
  issue_tile(0);
  auto load_tile = [&](double *x) {
    cp_async_wait_all();
    __syncwarp();
    const u64 *src = pfb + g * PFP;
#pragma unroll
    for (int k = 0; k < PA::K; k++) {
      const u64 v = src[PA::idx(tl, 0, k)];
      x[k] = (raw & 1) ? r2d(v) : u2d(v);
      if constexpr (UNRED) x[k] = fp_reduce(x[k], qd, qinv);
    }
    __syncwarp();  // every lane has read the staged tile
    issue_tile(tcur + 1);
    if (tcur == 0) __syncthreads(); else ROW_SYNC();  // twiddles staged; the previous tile's phase-B reads are done
    tcur++;
  };
#else
  auto load_tile = [&](double *x) {
    const u64 *src = tile_src(tcur) + ((u64)g << LM);
#pragma unroll
    for (int k = 0; k < PA::K; k++) {
      const u64 v = (CGB_ABLATE & 4) ? (u64)(tid * 977 + k + tcur) : __ldcs(src + PA::idx(tl, 0, k));
      x[k] = ((raw & 1) && !(CGB_ABLATE & 4)) ? r2d(v) : u2d(v);
      if constexpr (UNRED) x[k] = fp_reduce(x[k], qd, qinv);
    }
    if (tcur == 0) __syncthreads(); else ROW_SYNC();  // twiddles staged; the previous tile's phase-B reads are done
    tcur++;
  };
#endif
  double *sd = reinterpret_cast<double *>(sm3) + g * PADM;
  auto spad = [](int i) { return i + (i >> PSH); };
  const u64 *K = keys[item];
  // L2 prefetch of what the NEXT step of this CTA reads (no registers held): the next
  // digit's row tile (one 128-byte line per thread), the own digit's gathered blocks,
  // or (MODE 2) the W tiles
  auto prefetch_next = [&](int j) {  // called while digit j (or W tile j - L) is processed
#if CGB_KSROW_PF
    const int nd = l == L ? L : L - 1;
    if (j + 1 < L && j + 1 == l) {
      const u64 gi = xin.g ? xin.g[item] : 1;
      const u64 *p = xin.items ? xin.items[item] + xin.off + ((u64)l << LOGN)
                               : xin.base + (u64)item * xin.stride + ((u64)l << LOGN);
#pragma unroll
      for (int u = 0; u < PB::R; u++) {
        const u32 k0 = (u32)(row0 + PB::idx(tl, u, 0));
        KSROW_PREFETCH(p + (xin.items && xin.g ? (perm_g(k0, gi, LOGN) & ~7u) : k0));
      }
      return;
    }
    // index of the next tile in tile_src order
    int t;
    if (j + 1 < L) t = (l == L || j + 1 < l) ? j + 1 : j;  // digit j+1 (l skipped)
    else t = nd + (j + 1 - L);                             // W tile
    if (t < ntile) KSROW_PREFETCH(tile_src(t) + 16 * (u64)tid);
#if CGB_KSROW_PF >= 3  // also the next digit's key rows (both polys), one line per thread each
    if (j + 1 < L) {
      const u64 *KFp = K + 2 * (u64)L * 2 * LP * N;
      KSROW_PREFETCH(KFp + ((u64)((j + 1) * 2 + 0) * LP + l) * N + ((u64)first << LM) + 16 * (u64)tid);
      KSROW_PREFETCH(KFp + ((u64)((j + 1) * 2 + 1) * LP + l) * N + ((u64)first << LM) + 16 * (u64)tid);
    }
#endif
#else
    (void)j;
#endif
  };
  double a0[E], a1[E];
#pragma unroll
  for (int i = 0; i < E; i++) a0[i] = a1[i] = 0.0;
#if CGB_KSROW_KSTAGE
  // digit j's key words (both polys) for this thread's 16 output positions, staged by
  // cp.async while the digit's tile loads and its row pass runs; chunk c (16 bytes) of
  // thread t at [c][t] (conflict-free 128-bit reads), 8 chunks per poly
  constexpr int T_ = NTT2_TILE / 16;
  double2 *kst = reinterpret_cast<double2 *>(sm3 + ksr_data_words(LM) +
                                              (CGB_KSROW_GTW ? 0 : (CGB_KSROW_TWW ? 1 : 2) * (NTT2_TILE + (NTT2_TILE >> LB))));
  auto stage_keys = [&](int j) {
    const u64 *KF = K + 2 * (u64)L * 2 * LP * N;
    const u64 *k0 = KF + ((u64)(j * 2 + 0) * LP + l) * N + row0, *k1 = KF + ((u64)(j * 2 + 1) * LP + l) * N + row0;
#pragma unroll
    for (int u = 0; u < PB::R; u++)
#pragma unroll
      for (int k = 0; k < PB::K; k += 2) {
        const int c = (u * PB::K + k) / 2, o = PB::idx(tl, u, k);
        cp_async16(&kst[c * T_ + tid], k0 + o);
        cp_async16(&kst[(8 + c) * T_ + tid], k1 + o);
      }
    cp_async_commit();
  };
#endif
#pragma unroll 1
  for (int j = 0; j < L; j++) {
    prefetch_next(j);
#if CGB_KSROW_KSTAGE
    stage_keys(j);
#endif
    double x[E];
    if (j == l) {  // the digit's own limb: the input itself, already in NTT form
#if CGB_KSROW_G4
#pragma unroll
      for (int u = 0; u < PB::R; u++)
#pragma unroll
        for (int k = 0; k < PB::K; k += 4) {
          u64 w[4];
          ks_src_block4(xin, item, j, (u32)(row0 + PB::idx(tl, u, k)), LOGN, w);
#pragma unroll
          for (int e = 0; e < 4; e++) x[u * PB::K + k + e] = u2d(w[e]);
        }
#elif (CGB_ABLATE & 1)
      {
        const u64 *p_ = xin.items[item] + xin.off + ((u64)j << LOGN) + row0;
#pragma unroll
        for (int u = 0; u < PB::R; u++)
#pragma unroll
          for (int k = 0; k < PB::K; k += 4) {
            u64 w[4];
            ld256(p_ + PB::idx(tl, u, k), w);
#pragma unroll
            for (int e = 0; e < 4; e++) x[u * PB::K + k + e] = u2d(w[e] & 0xFFFFFFFFFFFFull);
          }
      }
#else
#pragma unroll
      for (int u = 0; u < PB::R; u++)
#pragma unroll
        for (int k = 0; k < PB::K; k++)
          x[u * PB::K + k] = u2d(ks_src_word(xin, item, j, (u32)(row0 + PB::idx(tl, u, k)), LOGN));
#endif
    } else {
      load_tile(x);
      if (!(CGB_ABLATE & 16)) phase_regs_fp<LM, 0, RA, true, E, false, GT, TWW>(x, tw, tl, qd, qinv);
#pragma unroll
      for (int k = 0; k < PA::K; k++) sd[spad(PA::idx(tl, 0, k))] = x[k];
      ROW_SYNC();
#pragma unroll
      for (int u = 0; u < PB::R; u++)
#pragma unroll
        for (int k = 0; k < PB::K; k++) x[u * PB::K + k] = sd[spad(PB::idx(tl, u, k))];  // no reduction in a forward pass
      if (!(CGB_ABLATE & 16)) phase_regs_fp<LM, RA, RB, true, E, true, GT, TWW>(x, tw, tl, qd, qinv);
    }
    // the key's FP64 plane (k_key_fp): exact doubles, no per-word conversion
#if CGB_KSROW_KSTAGE
    cp_async_wait_all();
#pragma unroll
    for (int u = 0; u < PB::R; u++)
#pragma unroll
      for (int k = 0; k < PB::K; k += 4) {
        const int c = (u * PB::K + k) / 2;
        const double2 p0 = kst[c * T_ + tid], p1 = kst[(c + 1) * T_ + tid];
        const double2 q0 = kst[(8 + c) * T_ + tid], q1 = kst[(9 + c) * T_ + tid];
        const double w0d[4] = {p0.x, p0.y, p1.x, p1.y}, w1d[4] = {q0.x, q0.y, q1.x, q1.y};
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const double xv = x[u * PB::K + k + e];
          const double d0 = w0d[e], d1 = w1d[e];
          a0[u * PB::K + k + e] += fp_mulmod(xv, d0, d0 * qinv, qd);
          a1[u * PB::K + k + e] += fp_mulmod(xv, d1, d1 * qinv, qd);
        }
      }
    if (false)
#endif
    {
    const u64 *KF = K + 2 * (u64)L * 2 * LP * N;
    const u64 *k0 = KF + ((u64)(j * 2 + 0) * LP + l) * N + row0, *k1 = KF + ((u64)(j * 2 + 1) * LP + l) * N + row0;
#pragma unroll
    for (int u = 0; u < PB::R; u++)
#pragma unroll
      for (int k = 0; k < PB::K; k += 4) {
        const int o = PB::idx(tl, u, k);
        u64 w0[4], w1[4];
        if (CGB_ABLATE & 2) {
#pragma unroll
          for (int e = 0; e < 4; e++) {
            w0[e] = (u64)__double_as_longlong((double)(o + e + j * 7 + 12345));
            w1[e] = (u64)__double_as_longlong((double)(o + e + j * 5 + 54321));
          }
        } else {
          ld256(k0 + o, w0);
          ld256(k1 + o, w1);
        }
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const double xv = x[u * PB::K + k + e];
          const double d0 = r2d(w0[e]), d1 = r2d(w1[e]);
#if CGB_KEYPROD_Q
          a0[u * PB::K + k + e] += fp_mulmod_q(xv, d0, qd, qinv);
          a1[u * PB::K + k + e] += fp_mulmod_q(xv, d1, qd, qinv);
#else
          a0[u * PB::K + k + e] += fp_mulmod(xv, d0, d0 * qinv, qd);
          a1[u * PB::K + k + e] += fp_mulmod(xv, d1, d1 * qinv, qd);
#endif
        }
      }
    }
    if constexpr (L > 4) {  // every 4 digits: back to [-q/2, q/2] (4 products add < 10.8 q)
      if ((j & 3) == 3 && j + 1 < L) {
#pragma unroll
        for (int i = 0; i < E; i++) {
          a0[i] = fp_reduce(a0[i], qd, qinv);
          a1[i] = fp_reduce(a1[i], qd, qinv);
        }
      }
    }
  }
  if constexpr (MODE == 2) {  // ModDown: row pass of W[pp][l] (same forward twiddles), combine, store
#pragma unroll 1
    for (int pp = 0; pp < 2; pp++) {
      prefetch_next(L + pp);
      double x[E];
      load_tile(x);
      if (!(CGB_ABLATE & 16)) phase_regs_fp<LM, 0, RA, true, E, false, GT, TWW>(x, tw, tl, qd, qinv);
#pragma unroll
      for (int k = 0; k < PA::K; k++) sd[spad(PA::idx(tl, 0, k))] = x[k];
      ROW_SYNC();
#pragma unroll
      for (int u = 0; u < PB::R; u++)
#pragma unroll
        for (int k = 0; k < PB::K; k++) x[u * PB::K + k] = sd[spad(PB::idx(tl, u, k))];
#if CGB_KSROW_EPF
      // the exchange tile is free until the next pass: this pass's epilogue operands
      // (c0 o sigma, the rotate_add input) stream into the thread's slots of it while
      // phase B computes
      u64 *stg = sm3 + 32 * tid;
      __syncthreads();  // every thread has read its phase-B words
#pragma unroll
      for (int u = 0; u < PB::R; u++)
#pragma unroll
        for (int k = 0; k < PB::K; k += 4) epi.prefetch4(item, pp * L + l, row0 + PB::idx(tl, u, k), stg + u * PB::K + k);
      cp_async_commit();
#endif
      if (!(CGB_ABLATE & 16)) phase_regs_fp<LM, RA, RB, true, E, true, GT, TWW>(x, tw, tl, qd, qinv);
#if CGB_KSROW_EPF
      cp_async_wait_all();
#endif
#pragma unroll
      for (int u = 0; u < PB::R; u++)
#pragma unroll
        for (int k = 0; k < PB::K; k += 4) {
#if CGB_KSROW_FPC
          epi.combine4_fp(item, pp * L + l, row0 + PB::idx(tl, u, k), &x[u * PB::K + k],
                          pp ? &a1[u * PB::K + k] : &a0[u * PB::K + k]);
          continue;
#endif
          u64 w[4], av[4];
#pragma unroll
          for (int e = 0; e < 4; e++) {
            w[e] = fp_canon(x[u * PB::K + k + e], qd, qinv);
            av[e] = fp_canon(pp ? a1[u * PB::K + k + e] : a0[u * PB::K + k + e], qd, qinv);
          }
#if CGB_KSROW_EPF
          epi.combine4_staged(item, pp * L + l, row0 + PB::idx(tl, u, k), w, av, stg + u * PB::K + k);
#else
          epi.combine4(item, pp * L + l, row0 + PB::idx(tl, u, k), w, av);
#endif
        }
    }
    return;
  }
  u64 *o0 = acc + ((u64)item * 2 * LP + l) * N + row0, *o1 = acc + ((u64)item * 2 * LP + LP + l) * N + row0;
  if (l == L) {  // P limb: ModDown's inverse row pass runs here, on the accumulators
#if CGB_KSROW_GTW
    const double2 *itw = reinterpret_cast<const double2 *>(Md.fitw1t) + row0;
#else
    __syncthreads();  // every thread is done with the forward twiddles
    stage_tw(Md.fitw1t);
    const double2 *itw = tw;
#endif
#pragma unroll 1
    for (int pp = 0; pp < 2; pp++) {
      double y[E];
#pragma unroll
      for (int i = 0; i < E; i++) y[i] = fp_reduce(pp ? a1[i] : a0[i], qd, qinv);
      if (pp == 0) __syncthreads(); else ROW_SYNC();  // inverse twiddles staged / previous poly's reads done
      phase_regs_fp<LM, RA, RB, false, E, true, GT, TWW>(y, itw, tl, qd, qinv);
      ROW_SYNC();
#pragma unroll
      for (int u = 0; u < PB::R; u++)
#pragma unroll
        for (int k = 0; k < PB::K; k++) sd[spad(PB::idx(tl, u, k))] = y[u * PB::K + k];
      ROW_SYNC();
#pragma unroll
      for (int k = 0; k < PA::K; k++) y[k] = fp_reduce(sd[spad(PA::idx(tl, 0, k))], qd, qinv);
      phase_regs_fp<LM, 0, RA, false, E, false, GT, TWW>(y, itw, tl, qd, qinv);
      u64 *o = pp ? o1 : o0;
#pragma unroll
      for (int k = 0; k < PA::K; k++) o[PA::idx(tl, 0, k)] = (raw & 2) ? fp_raw(y[k], qd, qinv) : fp_canon(y[k], qd, qinv);
    }
    return;
  }
#pragma unroll
  for (int u = 0; u < PB::R; u++)
#pragma unroll
    for (int k = 0; k < PB::K; k += 4) {
      const int o = PB::idx(tl, u, k);
      const double *y0 = &a0[u * PB::K + k], *y1 = &a1[u * PB::K + k];
      st256(o0 + o, fp_canon(y0[0], qd, qinv), fp_canon(y0[1], qd, qinv), fp_canon(y0[2], qd, qinv),
            fp_canon(y0[3], qd, qinv));
      st256(o1 + o, fp_canon(y1[0], qd, qinv), fp_canon(y1[1], qd, qinv), fp_canon(y1[2], qd, qinv),
            fp_canon(y1[3], qd, qinv));
    }
}

// k_ks_row's MODE 2 (Q limbs' key inner product + ModDown row pass of W + combine)
// with 8 words per thread: 256 threads per 2048-word row tile, the 7-stage row pass
// in three register phases (1 + 3 + 3 stages, two shared-memory exchanges), half the
// per-thread accumulators -- aimed at 128 registers (2 CTAs = 16 warps per SM against
// 12 at 16 words per thread).  LB = 7 (N = 2^14) only; same words.  CGB_KSROW8.
#ifndef CGB_KSROW8_MINB
#define CGB_KSROW8_MINB 2
#endif
template <int LA, int LB, int L>
__global__ void __launch_bounds__(NTT2_TILE / 8, CGB_KSROW8_MINB)
    k_ks_row8(const u64 *D, KsSrc xin, const u64 *const *keys, const ModTab *mods, const u64 *W, MdEpi epi, int raw) {
  extern __shared__ u64 sm3[];
  constexpr int E = 8, T = NTT2_TILE / E, LM = LB, M = 1 << LM, LOGN = LA + LB, LP = L + 1;
  constexpr int G = NTT2_TILE / M, TPS = M / E, TILES = (1 << LA) / G;
  constexpr int PSH = fpr_psh(LM, 1), PADM = fpr_padm(LM, 1);
  static_assert(LM == 7, "three row phases of 1 + 3 + 3 stages");
  using PA = PhaseShape<LM, 0, 1, E>;
  using PB = PhaseShape<LM, 1, 3, E>;
  using PC = PhaseShape<LM, 4, 3, E>;
  static_assert(PC::ST == 1 && PC::K % 4 == 0, "row-pass output: runs of >= 4 consecutive words");
  const u64 N = 1ull << LOGN;
  const int tile = blockIdx.x % TILES, rest = blockIdx.x / TILES;
  const int l = rest % L, item = rest / L;
  const ModTab &Md = mods[l];
  const double qd = Md.qd, qinv = Md.qinv;
  const int tid = threadIdx.x, g = tid / TPS, tl = tid % TPS, first = tile * G;
  const u64 row0 = (u64)(first + g) << LM;
  double2 *tws = reinterpret_cast<double2 *>(sm3 + ksr_data_words(LM));
  {
    const double2 *gt = reinterpret_cast<const double2 *>(Md.ftw1t) + ((u64)first << LM);
#pragma unroll
    for (int i = 0; i < E; i++) {
      const int e = tid + i * T;
      tws[e + (e >> LM)] = __ldg(gt + e);
    }
  }
  const double2 *tw = tws + g * (M + 1);
  auto tile_src = [&](int t) -> const u64 * {
    if (t < L - 1) {
      const int j = t < l ? t : t + 1;
      return D + ((u64)item * L * LP + (u64)j * LP + l) * N + ((u64)first << LM);
    }
    return W + ((u64)item * 2 * L + (u64)(t - (L - 1)) * L + l) * N + ((u64)first << LM);
  };
  pdl_start_dependents();
  pdl_wait();
  double *sd = reinterpret_cast<double *>(sm3) + g * PADM;
  auto spad = [](int i) { return i + (i >> PSH); };
  // forward row pass of tile t: x ends in PC layout (8 consecutive words per thread)
  auto row_pass = [&](double *x, int t) {
    const u64 *src = tile_src(t) + ((u64)g << LM);
#pragma unroll
    for (int u = 0; u < PA::R; u++)
#pragma unroll
      for (int k = 0; k < PA::K; k++) {
        const u64 v = __ldcs(src + PA::idx(tl, u, k));
        x[u * PA::K + k] = (raw & 1) ? r2d(v) : u2d(v);
      }
    if (t == 0) __syncthreads(); else ROW_SYNC();  // twiddles staged; the previous pass's reads of the tile are done
    phase_regs_fp<LM, 0, 1, true, E, false>(x, tw, tl, qd, qinv);
#pragma unroll
    for (int u = 0; u < PA::R; u++)
#pragma unroll
      for (int k = 0; k < PA::K; k++) sd[spad(PA::idx(tl, u, k))] = x[u * PA::K + k];
    ROW_SYNC();
#pragma unroll
    for (int u = 0; u < PB::R; u++)
#pragma unroll
      for (int k = 0; k < PB::K; k++) x[u * PB::K + k] = sd[spad(PB::idx(tl, u, k))];
    phase_regs_fp<LM, 1, 3, true, E, false>(x, tw, tl, qd, qinv);
    ROW_SYNC();
#pragma unroll
    for (int u = 0; u < PB::R; u++)
#pragma unroll
      for (int k = 0; k < PB::K; k++) sd[spad(PB::idx(tl, u, k))] = x[u * PB::K + k];
    ROW_SYNC();
#pragma unroll
    for (int u = 0; u < PC::R; u++)
#pragma unroll
      for (int k = 0; k < PC::K; k++) x[u * PC::K + k] = sd[spad(PC::idx(tl, u, k))];  // forward: unreduced
    phase_regs_fp<LM, 4, 3, true, E, true>(x, tw, tl, qd, qinv);
  };
  const u64 *K = keys[item];
  const u64 *KF = K + 2 * (u64)L * 2 * LP * N;  // the key's FP64 plane
  double a0[E], a1[E];
#pragma unroll
  for (int i = 0; i < E; i++) a0[i] = a1[i] = 0.0;
  int tcur = 0;
#pragma unroll 1
  for (int j = 0; j < L; j++) {
    double x[E];
    if (j == l) {  // the digit's own limb: the input itself, already in NTT form
#pragma unroll
      for (int u = 0; u < PC::R; u++)
#pragma unroll
        for (int k = 0; k < PC::K; k++)
          x[u * PC::K + k] = u2d(ks_src_word(xin, item, j, (u32)(row0 + PC::idx(tl, u, k)), LOGN));
    } else {
      row_pass(x, tcur++);
    }
    const u64 *k0 = KF + ((u64)(j * 2 + 0) * LP + l) * N + row0, *k1 = KF + ((u64)(j * 2 + 1) * LP + l) * N + row0;
#pragma unroll
    for (int u = 0; u < PC::R; u++)
#pragma unroll
      for (int k = 0; k < PC::K; k += 4) {
        const int o = PC::idx(tl, u, k);
        u64 w0[4], w1[4];
        ld256(k0 + o, w0);
        ld256(k1 + o, w1);
#pragma unroll
        for (int e = 0; e < 4; e++) {
          const double xv = x[u * PC::K + k + e];
          const double d0 = r2d(w0[e]), d1 = r2d(w1[e]);
          a0[u * PC::K + k + e] += fp_mulmod(xv, d0, d0 * qinv, qd);
          a1[u * PC::K + k + e] += fp_mulmod(xv, d1, d1 * qinv, qd);
        }
      }
    if constexpr (L > 4) {
      if ((j & 3) == 3 && j + 1 < L) {
#pragma unroll
        for (int i = 0; i < E; i++) {
          a0[i] = fp_reduce(a0[i], qd, qinv);
          a1[i] = fp_reduce(a1[i], qd, qinv);
        }
      }
    }
  }
#pragma unroll 1
  for (int pp = 0; pp < 2; pp++) {  // ModDown: row pass of W[pp][l], combine, store
    double x[E];
    row_pass(x, tcur++);
#pragma unroll
    for (int u = 0; u < PC::R; u++)
#pragma unroll
      for (int k = 0; k < PC::K; k += 4)
        epi.combine4_fp(item, pp * L + l, row0 + PC::idx(tl, u, k), &x[u * PC::K + k],
                        pp ? &a1[u * PC::K + k] : &a0[u * PC::K + k]);
  }
}
static bool g_ksrow8 = false;  // CGB_KSROW8

// ---------------------------------------------------------------------------
// k_ks_row2: the key switch's two row kernels (MD = false: the P limb's inner product
// and ModDown's inverse row pass, k_ks_row MODE 1; MD = true: the Q limbs' inner
// product, ModDown's forward row pass of W and the combine, MODE 2) with EVERY operand
// tile except the keys streamed through a two-slot cp.async ring in shared memory.
//
// ncu shows the row kernels bound by the L1 / LSU data pipe and by exposed load
// latency, not by HBM or the FP64 pipe (profiles/r02/ncu_ks_row_lsu.md): each warp
// used to load a tile, wait, compute, load the next.  Here a warp owns the 32 / TPS
// rows it transforms (contiguous in the tile), copies exactly those rows two entries
// ahead with 16-byte cp.async (no registers held, no warp waits on the copy), and
// hands over with warp-level barriers only -- the kernel has no CTA barrier at all.
// Entries, in consumption order:
//   MD = false:  D(0, P) ... D(L-1, P)
//   MD = true:   per digit j:  j != l: D(j, l);  j == l: the input's own limb read
//                through the automorphism (its 2^LB-word source rows are contiguous:
//                perm_g maps aligned blocks to aligned blocks), then c0 o sigma, which
//                is folded into the accumulator as P c0 (out0 = (acc0 + P c0 - W0) / P:
//                the same residue as adding c0 after the division);
//                then W(0, l), [the rotate_add input, poly 0], W(1, l), [poly 1].
// Tiles consumed pointwise (the rotate_add input) are stored with the 16-byte chunk
// index XOR-swizzled so the 64- / 128-byte-strided lanes of a row read distinct banks.
// Same words as k_ks_row (tests/test_gpu_ring_parity.py, test_gpu_primitives.py).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
template <int LB>
__host__ __device__ constexpr size_t ks_row2_smem() {
  return 8 * ((size_t)ksr_data_words(LB) + (size_t)(NTT2_TILE >> LB) * ((1 << LB) + 1) +
              2 * (size_t)(NTT2_TILE >> LB) * ((1 << LB) + 8));
}
#ifndef CGB_KSROW2_MINB
#define CGB_KSROW2_MINB 3
#endif
#ifndef CGB_R2_RAWCONST
#define CGB_R2_RAWCONST 1  // k_ks_row2 is only launched on reduced-double tiles (raw = 3): no predicated conversions
#endif
#ifndef CGB_R2_OWN
#define CGB_R2_OWN 0   // own limb / c0 through the ring (0: direct gathered loads, c0 in the epilogue): the
                       // scattered shared-memory reads cost more than the gathers (ks_row_md 0.88 -> 0.95 ms)
#endif
#ifndef CGB_R2_ADD1
#define CGB_R2_ADD1 1  // the rotate_add input through the ring (0: direct 256-bit loads in the epilogue)
#endif
// FLAGS >= 0: which epilogue operands exist is known at compile time (bit 0: c0 o sigma,
// bit 1: the rotate_add / relinearisation input) -- the rotate and rotate_add waves of the
// hot path; -1: decided from the arguments at run time
template <int LA, int LB, int L, bool MD, bool UNRED = false, int FLAGS = -1>
__global__ void __launch_bounds__(NTT2_TILE / 16, CGB_KSROW2_MINB)
    k_ks_row2(u64 *acc, const u64 *D, KsSrc xin, const u64 *const *keys, const ModTab *mods, int iP, const u64 *W,
              MdEpi epi, int raw) {
  extern __shared__ u64 sm3[];
  constexpr int E = 16, LM = LB, M = 1 << LM, LOGN = LA + LB, LP = L + 1;
  constexpr int G = NTT2_TILE / M, TPS = M / E, TILES = (1 << LA) / G, RW = 32 / TPS;
  constexpr int PSH = fpr_psh(LM, 1), PADM = fpr_padm(LM, 1);
  constexpr int RA = 4, RB = LM - 4;
  using PA = PhaseShape<LM, 0, RA, E>;
  using PB = PhaseShape<LM, RA, RB, E>;
  static_assert(PB::ST == 1 && PB::K % 4 == 0, "row-pass output: runs of >= 4 consecutive words");
  constexpr int PFP = M + 8, PFW = G * PFP;  // ring slot: the tile's rows at a pitch of M + 8 words
  constexpr int CH = RW * (M / 2);           // 16-byte chunks of a warp's rows
  const u64 N = 1ull << LOGN;
  const int tile = blockIdx.x % TILES, rest = blockIdx.x / TILES;
  const int l = MD ? rest % L : L, item = MD ? rest / L : rest;
  const ModTab &Md = mods[l == L ? iP : l];
  const double qd = Md.qd, qinv = Md.qinv;
  const int tid = threadIdx.x, g = tid / TPS, tl = tid % TPS, first = tile * G;
  const int lane = tid & 31, wrow0 = (tid >> 5) * RW;
  const u64 row0 = (u64)(first + g) << LM;  // word offset of this thread's row
  double *sd = reinterpret_cast<double *>(sm3) + g * PADM;
  double *twd = reinterpret_cast<double *>(sm3 + ksr_data_words(LM));
  u64 *ring = sm3 + ksr_data_words(LM) + G * (M + 1);
  auto spad = [](int i) { return i + (i >> PSH); };
  // the warp's rows' twiddles (w only; w / q is formed by one DMUL on use), staged by the warp itself
  auto stage_tw = [&](const u64 *table) {  // the w-only table (ftw1tw / fitw1tw)
    const double *gw = reinterpret_cast<const double *>(table) + ((u64)first << LM);
#pragma unroll
    for (int i = 0; i < E; i++) {
      const int e = wrow0 * M + lane + 32 * i;
      twd[e + (e >> LM)] = __ldg(gw + e);
    }
  };
  stage_tw(Md.ftw1tw);
  const double2 *tw = reinterpret_cast<const double2 *>(twd + g * (M + 1));
  const bool any_c0 = MD && (FLAGS >= 0 ? (FLAGS & 1) != 0 : (epi.add0.items || epi.add0.base));
  const bool any_add1 = MD && (FLAGS >= 0 ? (FLAGS & 2) != 0 : epi.add1 != nullptr);
  const bool has_c0 = CGB_R2_OWN == 1 && any_c0;      // ... as ring entries
  const bool has_add1 = CGB_R2_ADD1 && any_add1;
  const int c0n = has_c0 ? 1 : 0;
  const int NE = MD ? L - (CGB_R2_OWN >= 1 ? 0 : 1) + c0n + 2 + (has_add1 ? 2 : 0) : L;
  // the own limb / c0 as (limb-poly pointer, Galois element)
  const u64 *own_p = nullptr, *c0_p = nullptr;
  u64 own_g = 1, c0_g = 1;
  if (MD) {
    if (xin.items) {
      own_p = xin.items[item] + xin.off + ((u64)l << LOGN);
      own_g = xin.g ? xin.g[item] : 1;
    } else {
      own_p = xin.base + (u64)item * xin.stride + ((u64)l << LOGN);
    }
    if (has_c0) {
      if (epi.add0.items) {
        c0_p = epi.add0.items[item] + epi.add0.off + ((u64)l << LOGN);
        c0_g = epi.add0.g ? epi.add0.g[item] : 1;
      } else {
        c0_p = epi.add0.base + (u64)item * epi.add0.stride + ((u64)l << LOGN);
      }
    }
  }
  pdl_start_dependents();
  pdl_wait();
  // start the copy of entry e into slot e & 1 (a group is committed even past the end,
  // so "all but the newest group" always means "entry e has landed")
  auto issue = [&](int e) {
    if (e < NE) {
      u64 *dst = ring + (e & 1) * PFW + wrow0 * PFP;
      const u64 *src = nullptr, *gbase = nullptr;  // contiguous tile rows | gathered source rows
      u64 gg = 1;
      bool swz = false;
      if (!MD) {
        src = D + ((u64)item * L * LP + (u64)e * LP + L) * N;
      } else if (CGB_R2_OWN < 1 && e < L - 1) {
        src = D + ((u64)item * L * LP + (u64)(e < l ? e : e + 1) * LP + l) * N;
      } else if (CGB_R2_OWN < 1) {
        const int t = e - (L - 1);
        const int pp = has_add1 ? t >> 1 : t;
        if (has_add1 && (t & 1)) {
          src = epi.add1[item] + ((u64)pp * L + l) * N;
          swz = true;
        } else {
          src = W + ((u64)item * 2 * L + (u64)pp * L + l) * N;
        }
      } else if (e < l) {
        src = D + ((u64)item * L * LP + (u64)e * LP + l) * N;
      } else if (e == l) {
        gbase = own_p, gg = own_g;
      } else if (e == l + 1 && has_c0) {
        gbase = c0_p, gg = c0_g;
      } else if (e < L + c0n) {
        src = D + ((u64)item * L * LP + (u64)(e - c0n) * LP + l) * N;
      } else {
        const int t = e - (L + c0n);
        const int pp = has_add1 ? t >> 1 : t;
        if (has_add1 && (t & 1)) {
          src = epi.add1[item] + ((u64)pp * L + l) * N;
          swz = true;
        } else {
          src = W + ((u64)item * 2 * L + (u64)pp * L + l) * N;
        }
      }
      if (gbase) {
#pragma unroll
        for (int i = 0; i < CH / 32; i++) {
          const int c = lane + 32 * i, r = c / (M / 2), cc = c % (M / 2);
          const u32 orow = (u32)(first + wrow0 + r);
          const u32 srow = gg == 1 ? orow : perm_g(orow << LM, gg, LOGN) >> LM;
          cp_async16(dst + r * PFP + 2 * cc, gbase + ((u64)srow << LM) + 2 * cc);
        }
      } else {
        src += (u64)(first + wrow0) << LM;
#pragma unroll
        for (int i = 0; i < CH / 32; i++) {
          const int c = lane + 32 * i, r = c / (M / 2), cc = c % (M / 2);
          const int pc = swz ? (cc ^ ((cc >> 3) & 7)) : cc;
          cp_async16(dst + r * PFP + 2 * pc, src + 2 * c);
        }
      }
    }
    cp_async_commit();
  };
  issue(0);
  issue(1);
  int ecur = 0;
  auto slot = [&]() -> const u64 * { return ring + (ecur & 1) * PFW + g * PFP; };
  auto arrive = [&]() {  // entry ecur has landed and is visible to the warp
    cp_async_wait_1();
    __syncwarp();
  };
  auto release = [&]() {  // every lane has read entry ecur: refill its slot with entry ecur + 2
    __syncwarp();
    issue(ecur + 2);
    ecur++;
  };
  // forward row pass of the tile in the ring: x ends in PB layout, unreduced (|x| < 12 q)
  auto row_pass = [&](double *x) {
    arrive();
    const u64 *b = slot();
#pragma unroll
    for (int k = 0; k < PA::K; k++) {
      const u64 v = b[PA::idx(tl, 0, k)];
      x[k] = (CGB_R2_RAWCONST || (raw & 1)) ? r2d(v) : u2d(v);
      if constexpr (UNRED) x[k] = fp_reduce(x[k], qd, qinv);  // the column kernel stored its output unreduced
    }
    release();
    phase_regs_fp<LM, 0, RA, true, E, false, false, true>(x, tw, tl, qd, qinv);
#pragma unroll
    for (int k = 0; k < PA::K; k++) sd[spad(PA::idx(tl, 0, k))] = x[k];
    __syncwarp();
#pragma unroll
    for (int u = 0; u < PB::R; u++)
#pragma unroll
      for (int k = 0; k < PB::K; k++) x[u * PB::K + k] = sd[spad(PB::idx(tl, u, k))];
    __syncwarp();  // the exchange rows are free for the next pass
    phase_regs_fp<LM, RA, RB, true, E, true, false, true>(x, tw, tl, qd, qinv);
  };
  const u64 *K = keys[item];
  const u64 *KF = K + 2 * (u64)L * 2 * LP * N;  // the key's FP64 plane
  double a0[E], a1[E];
#pragma unroll
  for (int i = 0; i < E; i++) a0[i] = a1[i] = 0.0;
#pragma unroll 1
  for (int j = 0; j < L; j++) {
    double x[E];
    if (MD && j == l && CGB_R2_OWN < 1) {
#pragma unroll
      for (int u = 0; u < PB::R; u++)
#pragma unroll
        for (int k = 0; k < PB::K; k++)
          x[u * PB::K + k] = u2d(ks_src_word(xin, item, j, (u32)(row0 + PB::idx(tl, u, k)), LOGN));
    } else if (MD && j == l) {  // the digit's own limb: the input itself, read through the automorphism
      arrive();
      const u64 *b = slot();
#pragma unroll
      for (int u = 0; u < PB::R; u++)
#pragma unroll
        for (int k = 0; k < PB::K; k++) {
          const int i = PB::idx(tl, u, k);
          const int si = own_g == 1 ? i : (int)(perm_g((u32)(row0 + i), own_g, LOGN) & (M - 1));
          x[u * PB::K + k] = u2d(b[si]);
        }
      release();
      if (has_c0) {  // P c0 o sigma joins poly 0's accumulator
        const double2 pq = epi.C->fPmodq[l];
        arrive();
        const u64 *c = slot();
#pragma unroll
        for (int u = 0; u < PB::R; u++)
#pragma unroll
          for (int k = 0; k < PB::K; k++) {
            const int i = PB::idx(tl, u, k);
            const int si = c0_g == 1 ? i : (int)(perm_g((u32)(row0 + i), c0_g, LOGN) & (M - 1));
            a0[u * PB::K + k] += fp_mulmod(u2d(c[si]), pq.x, pq.y, qd);
          }
        release();
        if constexpr (L >= 4) {  // one term more than the digits: back to [-q/2, q/2]
#pragma unroll
          for (int i = 0; i < E; i++) a0[i] = fp_reduce(a0[i], qd, qinv);
        }
      }
    } else {
      row_pass(x);
    }
    {
      const u64 *k0 = KF + ((u64)(j * 2 + 0) * LP + l) * N + row0, *k1 = KF + ((u64)(j * 2 + 1) * LP + l) * N + row0;
#pragma unroll
      for (int u = 0; u < PB::R; u++)
#pragma unroll
        for (int k = 0; k < PB::K; k += 4) {
          const int o = PB::idx(tl, u, k);
          u64 w0[4], w1[4];
          ld256(k0 + o, w0);
          ld256(k1 + o, w1);
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const double xv = x[u * PB::K + k + e];
            const double d0 = r2d(w0[e]), d1 = r2d(w1[e]);
#if CGB_KEYPROD_Q
            a0[u * PB::K + k + e] += fp_mulmod_q(xv, d0, qd, qinv);
            a1[u * PB::K + k + e] += fp_mulmod_q(xv, d1, qd, qinv);
#else
            a0[u * PB::K + k + e] += fp_mulmod(xv, d0, d0 * qinv, qd);
            a1[u * PB::K + k + e] += fp_mulmod(xv, d1, d1 * qinv, qd);
#endif
          }
        }
    }
    if constexpr (L > 4) {  // every 4 digits: back to [-q/2, q/2] (4 products add < 10.8 q)
      if ((j & 3) == 3 && j + 1 < L) {
#pragma unroll
        for (int i = 0; i < E; i++) {
          a0[i] = fp_reduce(a0[i], qd, qinv);
          a1[i] = fp_reduce(a1[i], qd, qinv);
        }
      }
    }
  }
  if constexpr (MD) {  // ModDown: forward row pass of W[pp][l], out = (acc - W) P^-1 (+ the rotate_add input)
    const double2 pinv = epi.C->fPinvq[l];
#pragma unroll 1
    for (int pp = 0; pp < 2; pp++) {
      double x[E];
      row_pass(x);
      if (has_add1) arrive();
      const u64 *b = slot();
      u64 *o = epi.out[item] + ((u64)pp * L + l) * N + row0;
#pragma unroll
      for (int u = 0; u < PB::R; u++)
#pragma unroll
        for (int k = 0; k < PB::K; k += 4) {
          const int i = PB::idx(tl, u, k);
          u64 bv[4] = {0, 0, 0, 0}, cv[4] = {0, 0, 0, 0};
          if (!CGB_R2_ADD1 && any_add1) ld256(epi.add1[item] + ((u64)pp * L + l) * N + row0 + i, bv);
          if (CGB_R2_OWN != 1 && any_c0 && pp == 0) ks_src_block4(epi.add0, item, l, (u32)(row0 + i), LOGN, cv);
          if (has_add1) {
            const int c0i = i >> 1, c1i = c0i + 1;
            const ulonglong2 lo = *reinterpret_cast<const ulonglong2 *>(b + 2 * (c0i ^ ((c0i >> 3) & 7)));
            const ulonglong2 hi = *reinterpret_cast<const ulonglong2 *>(b + 2 * (c1i ^ ((c1i >> 3) & 7)));
            bv[0] = lo.x, bv[1] = lo.y, bv[2] = hi.x, bv[3] = hi.y;
          }
          u64 v[4];
#pragma unroll
          for (int e = 0; e < 4; e++) {
            const double xa = pp ? a1[u * PB::K + k + e] : a0[u * PB::K + k + e];
            // |xa - reduce(xw)| < 11.8 q: exact, inside fp_mulmod's analysed range (< 12 q)
            double y = fp_mulmod(xa - fp_reduce(x[u * PB::K + k + e], qd, qinv), pinv.x, pinv.y, qd);
            if (any_add1) y += u2d(bv[e]);
            if (CGB_R2_OWN != 1 && any_c0 && pp == 0) y += u2d(cv[e]);
            v[e] = fp_canon(y, qd, qinv);
          }
          st256(o + i, v[0], v[1], v[2], v[3]);
        }
      if (has_add1) release();
    }
    return;
  } else {  // P limb: ModDown's inverse row pass runs here, on the accumulators
    u64 *o0 = acc + ((u64)item * 2 * LP + L) * N + row0, *o1 = o0 + (u64)LP * N;
    __syncwarp();  // every lane is done with the forward twiddles
    stage_tw(Md.fitw1tw);
    __syncwarp();
#pragma unroll 1
    for (int pp = 0; pp < 2; pp++) {
      double y[E];
#pragma unroll
      for (int i = 0; i < E; i++) y[i] = fp_reduce(pp ? a1[i] : a0[i], qd, qinv);
      phase_regs_fp<LM, RA, RB, false, E, true, false, true>(y, tw, tl, qd, qinv);
#pragma unroll
      for (int u = 0; u < PB::R; u++)
#pragma unroll
        for (int k = 0; k < PB::K; k++) sd[spad(PB::idx(tl, u, k))] = y[u * PB::K + k];
      __syncwarp();
#pragma unroll
      for (int k = 0; k < PA::K; k++) y[k] = fp_reduce(sd[spad(PA::idx(tl, 0, k))], qd, qinv);
      __syncwarp();
      phase_regs_fp<LM, 0, RA, false, E, false, false, true>(y, tw, tl, qd, qinv);
      u64 *o = pp ? o1 : o0;
#pragma unroll
      for (int k = 0; k < PA::K; k++) o[PA::idx(tl, 0, k)] = (CGB_R2_RAWCONST || (raw & 2)) ? fp_raw(y[k], qd, qinv) : fp_canon(y[k], qd, qinv);
    }
  }
}
#ifndef CGB_COL_UNRED_BUILD
#define CGB_COL_UNRED_BUILD 0  // instantiate the reduce-on-load row kernels (measured a net loss; not built by default)
#endif
static bool g_ksrow2_spec = true;  // CGB_KSROW2_SPEC: epilogue operands known at compile time for rotate / rotate_add
static bool g_col_unred = false;  // CGB_COL_UNRED: the column kernels (FP64-bound) store D / W unreduced and the
                                   // row kernels reduce on load.  Measured: the column kernels gain 0.02 ms per
                                   // 768 key switches, the row kernels lose 0.03 -- off
static int g_ksrow2 = 1;  // CGB_KSROW2: 1 = the Q-limb kernel (ks_row_md), 2 = the P-limb kernel too, 0 = k_ks_row


// Column-pass fusion: inverse column pass of a source limb-poly (its row pass already
// done) followed, in the same CTA, by the centred lift into NT target moduli and each
// target's forward column pass.  The inverse's last phase and the forward's first
// phase share one register shape, so the coefficients never leave registers; the
// coefficient-domain polynomial is neither written nor re-read.
#ifndef CGB_COLF_RAWCONST
#define CGB_COLF_RAWCONST 1  // k_col_fused's callers all pass reduced-double words in and out: no per-word flag tests
#endif
struct ColJob {
  const u64 *src;     // source items (row-pass output of the inverse NTT)
  u64 src_stride;
  u64 *dst;           // destination items (column-pass output of the forward NTTs)
  u64 dst_stride;
  const ModTab *mods;
  int nsrc;
  unsigned char in_raw, out_raw;  // pass-boundary words as reduced doubles (see NttJob)
  unsigned short src_off[8];
  unsigned char src_mod[8];
  unsigned short dst_off[8][8];
  unsigned char dst_mod[8][8];
};
template <int LA, int LB, int NT>
#ifndef CGB_COLF_MINB
#define CGB_COLF_MINB 5
#endif
__global__ void __launch_bounds__(NTT2_TILE / 16, CGB_COLF_MINB) k_col_fused(ColJob job) {
  extern __shared__ u64 sm4[];
  constexpr int E = 16, LM = LA, M = 1 << LM, LOGN = LA + LB;
  constexpr int G = NTT2_TILE / M, T = NTT2_TILE / E, TILES = (1 << LB) / G;
  constexpr int PSH = fpr_psh(LM, 0), PADM = fpr_padm(LM, 0);
  constexpr int RA = 4, RB = LM - 4;
  using PF = PhaseShape<LM, 0, RA, E>;   // forward first / inverse last phase
  using PS = PhaseShape<LM, RA, RB, E>;  // forward second / inverse first phase
  const int tile = blockIdx.x % TILES, rest = blockIdx.x / TILES;
  const int s = rest % job.nsrc, item = rest / job.nsrc;
  const int tid = threadIdx.x, g = tid % G, tl = tid / G, first = tile * G;
  double *data = reinterpret_cast<double *>(sm4);
  double2 *tws = reinterpret_cast<double2 *>(sm4 + ((G * PADM + 1) & ~1));  // (NT + 1) tables of M
  auto spad = [](int i) { return i + (i >> PSH); };
  auto gaddr = [&](int i) -> u64 { return ((u64)i << LB) + first + g; };
  const ModTab &Ms = job.mods[job.src_mod[s]];
  for (int i = tid; i < M; i += T) tws[i] = __ldg(reinterpret_cast<const double2 *>(Ms.fitw) + i);
#pragma unroll
  for (int t = 0; t < NT; t++) {
    const double2 *ft = reinterpret_cast<const double2 *>(job.mods[job.dst_mod[s][t]].ftw);
    for (int i = tid; i < M; i += T) tws[(t + 1) * M + i] = __ldg(ft + i);
  }
  pdl_start_dependents();
  pdl_wait();
  const u64 *src = job.src + (u64)item * job.src_stride + ((u64)job.src_off[s] << LOGN);
  double x[E];
#pragma unroll
  for (int u = 0; u < PS::R; u++)
#pragma unroll
    for (int k = 0; k < PS::K; k++) {
      const u64 v = __ldcs(src + gaddr(PS::idx(tl, u, k)));
      x[u * PS::K + k] = (CGB_COLF_RAWCONST || job.in_raw) ? r2d(v) : u2d(v);
      if (RB == 4) x[u * PS::K + k] = fp_reduce(x[u * PS::K + k], Ms.qd, Ms.qinv);  // 4-stage inverse phase
    }
  double *sd = data + g * PADM;
  const double qs = Ms.qd, qsi = Ms.qinv;
  __syncthreads();  // twiddles staged
  // inverse column pass (the NTT's last: scale by N^-1)
  phase_regs_fp<LM, RA, RB, false, E>(x, tws, tl, qs, qsi);
#pragma unroll
  for (int u = 0; u < PS::R; u++)
#pragma unroll
    for (int k = 0; k < PS::K; k++) sd[spad(PS::idx(tl, u, k))] = x[u * PS::K + k];
  __syncthreads();
#pragma unroll
  for (int k = 0; k < PF::K; k++) x[k] = fp_reduce(sd[spad(PF::idx(tl, 0, k))], qs, qsi);
  // ... its last stage (stage 0: pairs (k, k + 8), one twiddle) run here with N^-1 folded in:
  // X' = (X + Y) N^-1, Y' = (X - Y) (w N^-1) -- 16 products instead of 8 + 16 and no
  // reduction before them (|X +- Y| <= 8 q after three unreduced stages)
  phase_regs_fp<LM, 0, RA, false, E, false, false, false, true>(x, tws, tl, qs, qsi);
#pragma unroll
  for (int k = 0; k < E / 2; k++) {
    const double sm_ = x[k] + x[k + E / 2], df_ = x[k] - x[k + E / 2];
    x[k] = fp_mulmod(sm_, Ms.ninv_fp, Ms.ninv_fpq, qs);
    x[k + E / 2] = fp_mulmod(df_, Ms.itw0n_fp, Ms.itw0n_fpq, qs);
  }
  // the centred lift of each coefficient: fp_reduce's residue in [-q_src/2, q_src/2]
  // IS the centred representative (q_src odd), and since every modulus of Q u P has
  // the same bit length (|r| <= q_src / 2 < q_t, col_fusable) it is a valid input of
  // each target's forward pass as it stands -- no canonical form, no integer lift
  double c[E];
#pragma unroll
  for (int k = 0; k < E; k++) c[k] = fp_reduce(x[k], qs, qsi);
#pragma unroll 1
  for (int t = 0; t < NT; t++) {
    const ModTab &Mt = job.mods[job.dst_mod[s][t]];
    const double qt = Mt.qd, qti = Mt.qinv;
    const double2 *tw_t = tws + (t + 1) * M;
#pragma unroll
    for (int k = 0; k < E; k++) x[k] = c[k];
    phase_regs_fp<LM, 0, RA, true, E>(x, tw_t, tl, qt, qti);
    __syncthreads();  // previous target's (or the inverse's) smem reads are done
#pragma unroll
    for (int k = 0; k < PF::K; k++) sd[spad(PF::idx(tl, 0, k))] = x[k];
    __syncthreads();
#pragma unroll
    for (int u = 0; u < PS::R; u++)
#pragma unroll
      for (int k = 0; k < PS::K; k++) x[u * PS::K + k] = sd[spad(PS::idx(tl, u, k))];  // forward: unreduced
    phase_regs_fp<LM, RA, RB, true, E>(x, tw_t, tl, qt, qti);
    u64 *dst = job.dst + (u64)item * job.dst_stride + ((u64)job.dst_off[s][t] << LOGN);
#pragma unroll
    for (int u = 0; u < PS::R; u++)
#pragma unroll
      for (int k = 0; k < PS::K; k++)
        dst[gaddr(PS::idx(tl, u, k))] =
            (CGB_COL_UNRED_BUILD && job.out_raw == 2) ? (u64)__double_as_longlong(x[u * PS::K + k])  // unreduced
            : (CGB_COLF_RAWCONST || job.out_raw) ? fp_raw(x[u * PS::K + k], qt, qti)
                             : fp_canon(x[u * PS::K + k], qt, qti);
  }
}
template <int LA, int LB>
__host__ size_t col_fused_smem(int nt) {
  const int G = NTT2_TILE >> LA;
  return sizeof(u64) * (size_t)((G * fpr_padm(LA, 0) + 1) & ~1) + 16 * (size_t)(nt + 1) * (1 << LA);
}
template <int LA, int LB>
static void col_fused_t(cgb_ring *r, const ColJob &job, int count, int nt) {
  const int G = NTT2_TILE >> LA;
  const dim3 grid((unsigned)((size_t)count * job.nsrc * ((1 << LB) / G)));
  const size_t sm = col_fused_smem<LA, LB>(nt);
  switch (nt) {
    case 2: launch_pdl(r, k_col_fused<LA, LB, 2>, grid, NTT2_TILE / 16, sm, job); break;
    case 3: launch_pdl(r, k_col_fused<LA, LB, 3>, grid, NTT2_TILE / 16, sm, job); break;
    case 4: launch_pdl(r, k_col_fused<LA, LB, 4>, grid, NTT2_TILE / 16, sm, job); break;
#define CFW(NT)                                                                                        \
  case NT: {                                                                                           \
    static std::once_flag once; /* > 48 KB of tables at 2^15 / 2^16 with many targets */              \
    std::call_once(once, [&] {                                                                         \
      CK(cudaFuncSetAttribute(k_col_fused<LA, LB, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,  \
                              (int)col_fused_smem<LA, LB>(NT)));                                        \
    });                                                                                                \
    launch_pdl(r, k_col_fused<LA, LB, NT>, grid, NTT2_TILE / 16, sm, job);                            \
    break;                                                                                             \
  }
      CFW(5) CFW(6) CFW(7) CFW(8)
#undef CFW
    default: launch_pdl(r, k_col_fused<LA, LB, 1>, grid, NTT2_TILE / 16, sm, job); break;
  }
}
static bool col_fusable(const cgb_ring *r) {
  u64 lo = ~0ull, hi = 0;  // k_col_fused feeds centred residues (|r| <= q_src / 2) to every target's pass
  for (int i = 0; i <= r->L; i++) {
    const u64 q = r->mods[i == r->L ? r->iP : i];
    lo = q < lo ? q : lo;
    hi = q > hi ? q : hi;
  }
  return r->fp_ntt && (g_fp_regio & 3) == 3 && g_col_fused && r->logN >= 13 && r->logN <= 16 && r->L >= 2 &&
         r->L <= 8 && hi < 2 * lo;
}
// inverse column pass of job.nsrc source units + lift + forward column passes into nt targets
static void col_fused(cgb_ring *r, ColJob &job, int count, int nt, const char *name) {
  job.mods = r->d_mods;
  launch_begin(r);
  switch (r->logN) {
    case 13: col_fused_t<6, 7>(r, job, count, nt); break;
    case 14: col_fused_t<CGB_A14, 14 - CGB_A14>(r, job, count, nt); break;
    case 15: col_fused_t<7, 8>(r, job, count, nt); break;
    default: col_fused_t<8, 8>(r, job, count, nt); break;
  }
  // butterflies of the inverse column pass and nt forward column passes, plus the N^-1 scaling
  const int LA = split_a(r->logN);  // column pass length (col_fused_t<LA, LB>)
  launch_end(r, name, 8.0 * (double)count * job.nsrc * r->N * (1 + nt),
             (double)count * job.nsrc * ((r->N / 2.0) * LA * (1 + nt) + r->N));
}

template <int LA, int LB>
__host__ __device__ constexpr size_t ks_row_smem() {  // exchange tile + the tile's row twiddles (rows of 2^LB + 1 pairs)
  return sizeof(u64) * (size_t)ksr_data_words(LB) + ksr_tw_bytes(LB) + KSTAGE_BYTES + ksr_pf_bytes(LB);
}
template <int LA, int LB, int L>
static void ks_row_attrs() {  // > 48 KB of dynamic shared memory needs the opt-in
  static std::once_flag once;
  std::call_once(once, [] {
    const int sm = (int)ks_row_smem<LA, LB>();
    cudaFuncSetAttribute(k_ks_row<LA, LB, L, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
#if CGB_BUILD_FALLBACKS
    cudaFuncSetAttribute(k_ks_row<LA, LB, L, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
    cudaFuncSetAttribute(k_ks_row<LA, LB, L, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
#endif
#if CGB_COL_UNRED_BUILD
    cudaFuncSetAttribute(k_ks_row<LA, LB, L, 1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
#endif
#ifdef CGB_KSROW_CARVE
    cudaFuncSetAttribute(k_ks_row<LA, LB, L, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, CGB_KSROW_CARVE);
#endif
  });
}

// ModUp column pass (fused lift) + k_ks_row: D holds only the column-pass output
template <int LA, int LB, int L>
static void modup_ks_row_t(cgb_ring *r, const NttJob &job, int count, u64 *acc, const u64 *D, const KsSrc &x,
                           u64 *const *d_keys) {
  const int G0 = NTT2_TILE >> LA, G1 = NTT2_TILE >> LB;
  const dim3 g0((unsigned)((size_t)count * job.nsub * ((1 << LB) / G0)));
  launch_pdl(r, k_ntt2_fpr<LA, LB, true, 0>, g0, NTT2_TILE / 16, fpr_smem_bytes<LA, LB>(0), job, NoEpi{});
  const dim3 g1((unsigned)((size_t)count * (L + 1) * ((1 << LA) / G1)));
  ks_row_attrs<LA, LB, L>();
#if CGB_BUILD_FALLBACKS
  launch_pdl(r, k_ks_row<LA, LB, L>, g1, NTT2_TILE / 16, ks_row_smem<LA, LB>(), acc, D, x, d_keys, r->d_mods,
             r->iP, count, (const u64 *)nullptr, MdEpi{}, 0);
#else
  (void)g1, (void)acc, (void)D, (void)x, (void)d_keys;
  FAIL(CGB_ERR_STATE, "the unfused ModUp row kernel is not built (CGB_BUILD_FALLBACKS)");
#endif
}
static bool ks_row_fusable(const cgb_ring *r) {
  // the FP64 inner-product sum is reduced after every 4 digits (|sum| < 11.3 q < 2^53), so
  // any digit count up to the 8 limbs of BASELINE config 5 stays exact
  return r->fp_ntt && (g_fp_regio & 3) == 3 && g_ks_row && r->logN >= 13 && r->logN <= 16 && r->L >= 2 &&
         r->L <= 8;
}
static void modup_ks_row(cgb_ring *r, NttJob &job, int count, u64 *acc, const u64 *D, const KsSrc &x,
                         u64 *const *d_keys) {
  job.mods = r->d_mods;
  job.logN = r->logN;
#define MKR(A, B)                                                              \
  switch (r->L) {                                                              \
    case 2: modup_ks_row_t<A, B, 2>(r, job, count, acc, D, x, d_keys); break; \
    case 3: modup_ks_row_t<A, B, 3>(r, job, count, acc, D, x, d_keys); break; \
    default: modup_ks_row_t<A, B, 4>(r, job, count, acc, D, x, d_keys); break; \
  }
  switch (r->logN) {
    case 13: MKR(6, 7) break;
    case 14: MKR(CGB_A14, 14 - CGB_A14) break;
    case 15: MKR(7, 8) break;
    default: MKR(8, 8) break;
  }
#undef MKR
}

// the inverse NTT's column pass alone (its row pass ran inside k_ks_row)
template <int LA, int LB>
static void ntt_inv_col_t(cgb_ring *r, const NttJob &job, int count) {
  const int G0 = NTT2_TILE >> LA;
  const dim3 g0((unsigned)((size_t)count * job.nsub * ((1 << LB) / G0)));
  launch_pdl(r, k_ntt2_fpr<LA, LB, false, 0>, g0, NTT2_TILE / 16, fpr_smem_bytes<LA, LB>(0), job, NoEpi{});
}
static void ntt_inv_col(cgb_ring *r, NttJob &job, int count) {
  job.mods = r->d_mods;
  job.logN = r->logN;
  launch_begin(r);
  switch (r->logN) {
    case 13: ntt_inv_col_t<6, 7>(r, job, count); break;
    case 14: ntt_inv_col_t<CGB_A14, 14 - CGB_A14>(r, job, count); break;
    case 15: ntt_inv_col_t<7, 8>(r, job, count); break;
    default: ntt_inv_col_t<8, 8>(r, job, count); break;
  }
  launch_end(r, "ntt_inv_col", 16.0 * (double)count * job.nsub * r->N,
             (double)count * job.nsub * ((r->N / 2) * (r->logN - split_a(r->logN)) + r->N));
}

// ModDown's forward NTT with the combine fused into its row pass (FP64 register-I/O
// kernels only); false when this ring's NTT takes another path
template <int LA, int LB>
static void moddown_ntt_fused_t(cgb_ring *r, const NttJob &job, int count, const MdEpi &epi) {
  NttJob second = job;
  second.src_base = nullptr;
  second.src_items = nullptr;
  second.galois = nullptr;
  second.lift = 0;
  auto grid = [&](int lm) {
    int nsubs = 1 << (LA + LB - lm), G = NTT2_TILE / (1 << lm);
    return dim3((unsigned)((size_t)count * job.nsub * (nsubs / G)));
  };
  launch_pdl(r, k_ntt2_fpr<LA, LB, true, 0>, grid(LA), NTT2_TILE / 16, fpr_smem_bytes<LA, LB>(0), job, NoEpi{});
  launch_pdl(r, k_ntt2_fpr<LA, LB, true, 1, MdEpi>, grid(LB), NTT2_TILE / 16, fpr_smem_bytes<LA, LB>(1), second, epi);
}
static bool moddown_fusable(const cgb_ring *r) {
  return r->fp_ntt && (g_fp_regio & 3) == 3 && g_md_epi && r->logN >= 12 && r->logN <= 16;
}
static bool moddown_ntt_fused(cgb_ring *r, NttJob &job, int count, const MdEpi &epi) {
  if (!moddown_fusable(r) || count <= 0) return false;
  job.mods = r->d_mods;
  job.logN = r->logN;
  switch (r->logN) {
    case 12: moddown_ntt_fused_t<6, 6>(r, job, count, epi); break;
    case 13: moddown_ntt_fused_t<6, 7>(r, job, count, epi); break;
    case 14: moddown_ntt_fused_t<CGB_A14, 14 - CGB_A14>(r, job, count, epi); break;
    case 15: moddown_ntt_fused_t<7, 8>(r, job, count, epi); break;
    case 16: moddown_ntt_fused_t<8, 8>(r, job, count, epi); break;
    default: return false;
  }
  return true;
}

// Fused key-switch passes ----------------------------------------------------
// Shared tile plumbing of the two-pass NTT's second (row) pass: the CTA owns
// G consecutive row blocks of M = 2^LB words of one limb-poly.
template <int LA, int LB, int E>
struct RowTile {
  static constexpr int M = 1 << LB, G = NTT2_TILE / M, T = NTT2_TILE / E, TILES = (1 << LA) / G;
  static constexpr int PADM = M + (M >> 3) + 1, TPS = M / E;
  static __host__ size_t smem() { return sizeof(u64) * (size_t)((G * PADM + 1) & ~1) + 16 * (size_t)NTT2_TILE; }
};

// load row tile `first` of a pass-0 output limb-poly into smem, run the forward row
// pass, leave canonical values in regs v[] (element e = tid + i T <-> word first M + e)
template <int LA, int LB, int E>
__device__ __forceinline__ void row_pass_fwd(const u64 *src, u64 *data, const ulonglong2 *tws, int first, u64 q,
                                             u64 v[E]) {
  using RT = RowTile<LA, LB, E>;
  const int tid = threadIdx.x;
#pragma unroll
  for (int i = 0; i < E; i++) v[i] = __ldcs(src + ((u64)first << LB) + tid + i * RT::T);
#pragma unroll
  for (int i = 0; i < E; i++) {
    const int e = tid + i * RT::T;
    data[(e >> LB) * RT::PADM + spad8(e & (RT::M - 1))] = v[i];
  }
  __syncthreads();
  const int g = tid / RT::TPS, tl = tid & (RT::TPS - 1);
  ntt2_sub<LB, E, true, true>(data + g * RT::PADM, tws + g * RT::M, tl, q, 2 * q);
#pragma unroll
  for (int i = 0; i < E; i++) {
    const int e = tid + i * RT::T;
    u64 x = data[(e >> LB) * RT::PADM + spad8(e & (RT::M - 1))];
    x = x >= 2 * q ? x - 2 * q : x;
    v[i] = x >= q ? x - q : x;
  }
  __syncthreads();  // smem is reused by the caller's next tile
}

// FP64-pipe version (rings with primes < 2^49): same contract, canonical u64 out
template <int LA, int LB, int E>
__device__ __forceinline__ void row_pass_fwd_fp(const u64 *src, u64 *smem, const ulonglong2 *tws_raw, int first,
                                                const ModTab &Md, u64 v[E]) {
  using RT = RowTile<LA, LB, E>;
  const int tid = threadIdx.x;
  double *data = reinterpret_cast<double *>(smem);
  const double2 *tws = reinterpret_cast<const double2 *>(tws_raw);
#pragma unroll
  for (int i = 0; i < E; i++) v[i] = __ldcs(src + ((u64)first << LB) + tid + i * RT::T);
#pragma unroll
  for (int i = 0; i < E; i++) {
    const int e = tid + i * RT::T;
    data[(e >> LB) * RT::PADM + spad8(e & (RT::M - 1))] = u2d(v[i]);
  }
  __syncthreads();
  const int g = tid / RT::TPS, tl = tid & (RT::TPS - 1);
  ntt2_sub_fp<LB, E, true>(data + g * RT::PADM, tws + g * RT::M, tl, Md.qd, Md.qinv);
#pragma unroll
  for (int i = 0; i < E; i++) {
    const int e = tid + i * RT::T;
    v[i] = fp_canon(data[(e >> LB) * RT::PADM + spad8(e & (RT::M - 1))], Md.qd, Md.qinv);
  }
  __syncthreads();
}

template <int LA, int LB, int E, bool FP = false>
__device__ __forceinline__ void stage_row_twiddles(ulonglong2 *tws, const ModTab &Md, int first) {
  using RT = RowTile<LA, LB, E>;
  const ulonglong2 *gtw = reinterpret_cast<const ulonglong2 *>(FP ? Md.ftw1 : Md.tw1);
#pragma unroll
  for (int j = 0; j < E; j++) {
    const int e = threadIdx.x + j * RT::T;
    tws[e] = __ldg(gtw + ((u64)first << LB) + e);
  }
}

// ModUp row pass fused with the key inner product:
//   acc[item][p][l] = sum_j NTT_l(lift_l(digit j)) * key[j][p][l]   (j == l: the input limb itself)
// D holds the column-pass outputs [item][j][l][N] (units j(L+1)+l, l != j).
template <int LA, int LB, int L, int E, bool FP = false>
__global__ void __launch_bounds__(NTT2_TILE / E) k_modup_ks(const u64 *D, KsSrc x, const u64 *const *keys, u64 kw,
                                                           u64 *acc, const ModTab *mods) {
  using RT = RowTile<LA, LB, E>;
  constexpr int LP = L + 1, LOGN = LA + LB;
  constexpr u64 N = 1ull << LOGN;
  extern __shared__ u64 smf[];
  const int unit = blockIdx.x / RT::TILES, tile = blockIdx.x - unit * RT::TILES;
  const int item = unit / LP, l = unit - item * LP;
  const ModTab &Md = mods[l];  // Q limbs then P (index L)
  const u64 q = Md.q;
  u64 *data = smf;
  ulonglong2 *tws = reinterpret_cast<ulonglong2 *>(smf + ((RT::G * RT::PADM + 1) & ~1));
  const int first = tile * RT::G, tid = threadIdx.x;
  stage_row_twiddles<LA, LB, E, FP>(tws, Md, first);
  const u64 *K = keys[item];
  u64 a0[E], a1[E];
#pragma unroll
  for (int i = 0; i < E; i++) a0[i] = a1[i] = 0;
#pragma unroll 1
  for (int j = 0; j < L; j++) {
    u64 v[E];
    if (j == l) {
#pragma unroll
      for (int i = 0; i < E; i++) v[i] = ks_src_word(x, item, j, (u32)(((u64)first << LB) + tid + i * RT::T), LOGN);
    } else {
      if (FP) row_pass_fwd_fp<LA, LB, E>(D + (((u64)item * L + j) * LP + l) * N, data, tws, first, Md, v);
      else row_pass_fwd<LA, LB, E>(D + (((u64)item * L + j) * LP + l) * N, data, tws, first, q, v);
    }
    const u64 *kb = K + ((u64)j * 2 + 0) * LP * N + (u64)l * N + ((u64)first << LB);
    const u64 *ka = K + ((u64)j * 2 + 1) * LP * N + (u64)l * N + ((u64)first << LB);
#pragma unroll
    for (int i = 0; i < E; i++) {
      const int e = tid + i * RT::T;
      a0[i] += mul_shoup_lazy(v[i], __ldg(kb + e), __ldg(kb + kw + e), q);
      a1[i] += mul_shoup_lazy(v[i], __ldg(ka + e), __ldg(ka + kw + e), q);
      if ((j & 3) == 3) {
        a0[i] = a0[i] >= 4 * q ? a0[i] - 4 * q : a0[i];
        a0[i] = a0[i] >= 2 * q ? a0[i] - 2 * q : a0[i];
        a1[i] = a1[i] >= 4 * q ? a1[i] - 4 * q : a1[i];
        a1[i] = a1[i] >= 2 * q ? a1[i] - 2 * q : a1[i];
      }
    }
  }
  u64 *o0 = acc + (((u64)item * 2 + 0) * LP + l) * N + ((u64)first << LB);
  u64 *o1 = acc + (((u64)item * 2 + 1) * LP + l) * N + ((u64)first << LB);
#pragma unroll
  for (int i = 0; i < E; i++) {
    u64 s0 = a0[i], s1 = a1[i];
#pragma unroll
    for (int r = 0; r < 3; r++) {
      const u64 m = (4ull >> r) * q;
      s0 = s0 >= m ? s0 - m : s0;
      s1 = s1 >= m ? s1 - m : s1;
    }
    o0[tid + i * RT::T] = s0;
    o1[tid + i * RT::T] = s1;
  }
}

// ModDown row pass fused with the combine:
//   out[p][l] = (acc[p][l] - NTT_l(lift_l(acc[p][P]))) * P^-1 + (p == 0 ? add0 : 0) + add1[p][l]
// W holds the column-pass outputs [item][p][l][N] (units pL + l).
template <int LA, int LB, int E, bool FP = false>
__global__ void __launch_bounds__(NTT2_TILE / E) k_moddown_fused(const u64 *W, const u64 *acc, u64 *const *out,
                                                                KsSrc add0, const u64 *const *add1,
                                                                const ModTab *mods, const Consts *C, int L) {
  using RT = RowTile<LA, LB, E>;
  constexpr int LOGN = LA + LB;
  constexpr u64 N = 1ull << LOGN;
  extern __shared__ u64 smf[];
  const int unit = blockIdx.x / RT::TILES, tile = blockIdx.x - unit * RT::TILES;
  const int item = unit / (2 * L), pl = unit - item * 2 * L, p = pl / L, l = pl - p * L;
  const ModTab &Md = mods[l];
  const u64 q = Md.q;
  u64 *data = smf;
  ulonglong2 *tws = reinterpret_cast<ulonglong2 *>(smf + ((RT::G * RT::PADM + 1) & ~1));
  const int first = tile * RT::G, tid = threadIdx.x;
  stage_row_twiddles<LA, LB, E, FP>(tws, Md, first);
  u64 v[E];
  if (FP) row_pass_fwd_fp<LA, LB, E>(W + ((u64)item * 2 * L + pl) * N, data, tws, first, Md, v);
  else row_pass_fwd<LA, LB, E>(W + ((u64)item * 2 * L + pl) * N, data, tws, first, q, v);
  const u64 LP = L + 1;
  const u64 *A = acc + (((u64)item * 2 + p) * LP + l) * N;
  const u64 pi = C->Pinvq[l], pis = C->Pinvq_sh[l];
  u64 *O = out[item] + (u64)pl * N;
  const u64 *A1 = add1 ? add1[item] + (u64)pl * N : nullptr;
  const bool has0 = p == 0 && (add0.items || add0.base);
#pragma unroll
  for (int i = 0; i < E; i++) {
    const u64 k = ((u64)first << LB) + tid + i * RT::T;
    u64 r = mul_shoup(sub_mod(A[k], v[i], q), pi, pis, q);
    if (has0) r = add_mod(r, ks_src_word(add0, item, l, (u32)k, LOGN), q);
    if (A1) r = add_mod(r, A1[k], q);
    O[k] = r;
  }
}

// BFV multiplication --------------------------------------------------------
// lift coefficient-form Q residues of one poly into B: dst[item][p][L + k][N]
__global__ void k_lift_QB(u64 *dst /*[item][4][L+nB][N]*/, const u64 *coef /*[item][4][L][N]*/, const ModTab *mods,
                          const Consts *C, int L, int nB, int iB0, int logN) {
  int item = blockIdx.y;
  u64 N = 1ull << logN;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;  // over [4][N]
  if (i >= 4 * N) return;
  u64 jn = i & (N - 1);
  int p = (int)(i >> logN);
  const u64 *src = coef + ((u64)item * 4 + p) * L * N;
  u64 y[MAXL];
  double s = 0.0;
  for (int l = 0; l < L; l++) {
    const ModTab &M = mods[l];
    y[l] = mul_mod(src[(u64)l * N + jn], C->QhatInv[l], M);
    s = __dadd_rn(s, __dmul_rn(__ull2double_rn(y[l]), C->invq[l]));
  }
  u64 v = (u64)__dadd_rn(s, 0.5);
  u64 *d = dst + ((u64)item * 4 + p) * (L + nB) * N;
  for (int k = 0; k < nB; k++) {
    const ModTab &M = mods[iB0 + k];
    u64 acc = 0;
    for (int l = 0; l < L; l++) acc = add_mod(acc, mul_mod(y[l], C->QhatModB[l][k], M), M.q);
    acc = sub_mod(acc, mul_mod(v, C->QmodB[k], M), M.q);
    d[(u64)(L + k) * N + jn] = acc;
  }
}
// L-templated, Shoup-constant versions of the two base-conversion kernels
// (every multiplier is a per-ring constant; lazy sums reduced every 4 terms)
__device__ __forceinline__ u64 lazy_fold(u64 a, u64 q) {
  a = a >= 4 * q ? a - 4 * q : a;
  return a >= 2 * q ? a - 2 * q : a;
}
__device__ __forceinline__ u64 lazy_final(u64 a, u64 q) {
  a = lazy_fold(a, q);
  return a >= q ? a - q : a;
}
template <int L>
__global__ void k_lift_QB_t(u64 *dst, const u64 *coef, const ModTab *mods, const Consts *C, int iB0, int logN) {
  constexpr int nB = L + 1;
  const int item = blockIdx.y;
  const u64 N = 1ull << logN;
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 4 * N) return;
  const u64 jn = i & (N - 1);
  const int p = (int)(i >> logN);
  const u64 *src = coef + ((u64)item * 4 + p) * L * N;
  u64 y[L];
  double s = 0.0;
#pragma unroll
  for (int l = 0; l < L; l++) {
    y[l] = mul_shoup(src[(u64)l * N + jn], C->QhatInv[l], C->QhatInv_sh[l], mods[l].q);
    s = __dadd_rn(s, __dmul_rn(__ull2double_rn(y[l]), C->invq[l]));
  }
  const u64 v = (u64)__dadd_rn(s, 0.5);
  u64 *d = dst + ((u64)item * 4 + p) * (L + nB) * N;
#pragma unroll
  for (int k = 0; k < nB; k++) {
    const u64 q = mods[iB0 + k].q;
    u64 acc = 0;
#pragma unroll
    for (int l = 0; l < L; l++) {
      acc += mul_shoup_lazy(y[l], C->QhatModB[l][k], C->QhatModB_sh[l][k], q);
      if ((l & 3) == 3) acc = lazy_fold(acc, q);
    }
    acc = lazy_final(acc, q);
    d[(u64)(L + k) * N + jn] = sub_mod(acc, mul_shoup(v, C->QmodB[k], C->QmodB_sh[k], q), q);
  }
}
// FP64-pipe forms of the two base conversions (every modulus < 2^49): the same
// modular products as the integer kernels through fp_mulmod (exact, results in
// (-2m, 2m)), lazy FP64 sums of <= 4 such products, canonical at the end -- so the
// same residues; the double-precision overflow estimates and the 128-bit
// fixed-point rounding are the integer kernels' operations unchanged.
__device__ __forceinline__ double fpm(double a, double2 w, double m) { return fp_mulmod(a, w.x, w.y, m); }
// The FP64 base conversions' constants as a kernel parameter (the constant bank:
// uniform reads without a load per thread -- they were ~60 L1 loads per element
// through a Consts pointer), built once per ring from Consts / the modulus table.
template <int L>
struct BConv {
  static constexpr int nB = L + 1;
  double qd[L + nB], qinv[L + nB];  // Q limbs, then B limbs
  u64 qB[nB];
  double2 QhatInv[L], QmodB[nB], QhatModB[L][nB];
  double invq[L];
  double2 QBhatInv[L];
  u64 th_hi[L], th_lo[L];
  double2 omega[L][nB], BQhatInv[nB], tBhat[nB], BhatInv[nB];
  double invb[nB];
  double2 BmodQ[L], BhatModQ[nB][L];
};
template <int L>
static BConv<L> make_bconv(const cgb_ring *r) {
  constexpr int nB = L + 1;
  const Consts &C = r->h_c;
  BConv<L> K{};
  for (int l = 0; l < L + nB; l++) {
    const ModTab &M = r->h_mods[l < L ? l : r->iB0 + (l - L)];
    K.qd[l] = M.qd;
    K.qinv[l] = M.qinv;
  }
  for (int k = 0; k < nB; k++) {
    K.qB[k] = r->h_mods[r->iB0 + k].q;
    K.QmodB[k] = C.fQmodB[k];
    K.BQhatInv[k] = C.fBQhatInv[k];
    K.tBhat[k] = C.ftBhat[k];
    K.BhatInv[k] = C.fBhatInv[k];
    K.invb[k] = C.invb[k];
    for (int l = 0; l < L; l++) K.BhatModQ[k][l] = C.fBhatModQ[k][l];
  }
  for (int l = 0; l < L; l++) {
    K.QhatInv[l] = C.fQhatInv[l];
    K.invq[l] = C.invq[l];
    K.QBhatInv[l] = C.fQBhatInv[l];
    K.th_hi[l] = C.sc_th_hi[l];
    K.th_lo[l] = C.sc_th_lo[l];
    K.BmodQ[l] = C.fBmodQ[l];
    for (int k = 0; k < nB; k++) {
      K.QhatModB[l][k] = C.fQhatModB[l][k];
      K.omega[l][k] = C.fsc_omega[l][k];
    }
  }
  return K;
}
// FP64 Q -> B base conversion (HPS lift, same residues as k_lift_QB_t)
template <int L>
__global__ void k_lift_QB_fp(u64 *dst, const u64 *coef, const __grid_constant__ BConv<L> K, int logN) {
  constexpr int nB = L + 1;
  const int item = blockIdx.y;
  const u64 N = 1ull << logN;
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 4 * N) return;
  const u64 jn = i & (N - 1);
  const int p = (int)(i >> logN);
  const u64 *src = coef + ((u64)item * 4 + p) * L * N;
  double yd[L];
  double s = 0.0;
#pragma unroll
  for (int l = 0; l < L; l++) {
    const u64 y = fp_canon(fpm(u2d(src[(u64)l * N + jn]), K.QhatInv[l], K.qd[l]), K.qd[l], K.qinv[l]);
    yd[l] = u2d(y);
    s = __dadd_rn(s, __dmul_rn(__ull2double_rn(y), K.invq[l]));
  }
  const double v = u2d((u64)__dadd_rn(s, 0.5));
  u64 *d = dst + ((u64)item * 4 + p) * (L + nB) * N;
#pragma unroll
  for (int k = 0; k < nB; k++) {
    const double qd = K.qd[L + k], qinv = K.qinv[L + k];
    double acc = -fpm(v, K.QmodB[k], qd);
#pragma unroll
    for (int l = 0; l < L; l++) {
      acc += fpm(yd[l], K.QhatModB[l][k], qd);
      if ((l & 3) == 2) acc = fp_reduce(acc, qd, qinv);
    }
    d[(u64)(L + k) * N + jn] = fp_canon(acc, qd, qinv);
  }
}
template <int L>
__global__ void k_scale_round_fp(u64 *d, const u64 *ten, const __grid_constant__ BConv<L> K, int logN) {
  constexpr int nB = L + 1, nt = L + nB;
  const int item = blockIdx.y;
  const u64 N = 1ull << logN;
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * N) return;
  const u64 jn = i & (N - 1);
  const int p = (int)(i >> logN);
  const u64 *cp = ten + ((u64)item * 3 + p) * nt * N;
  double yd[L];
  u128 S = 0;
#pragma unroll
  for (int l = 0; l < L; l++) {
    const u64 y = fp_canon(fpm(u2d(cp[(u64)l * N + jn]), K.QBhatInv[l], K.qd[l]), K.qd[l], K.qinv[l]);
    yd[l] = u2d(y);
    S += (u128)y * K.th_hi[l] + (u128)__umul64hi(y, K.th_lo[l]);
  }
  const u64 R = (u64)((S + ((u128)1 << 63)) >> 64);
  double ykd[nB];
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < nB; k++) {
    const double qd = K.qd[L + k], qinv = K.qinv[L + k];
    double acc = u2d(reduce4(R, K.qB[k]));
#pragma unroll
    for (int l = 0; l < L; l++) {
      acc += fpm(yd[l], K.omega[l][k], qd);
      if ((l & 3) == 2) acc = fp_reduce(acc, qd, qinv);
    }
    const double z = fpm(u2d(cp[(u64)(L + k) * N + jn]), K.BQhatInv[k], qd);
    acc = fp_reduce(acc + fpm(z, K.tBhat[k], qd), qd, qinv);
    const u64 yk = fp_canon(fpm(acc, K.BhatInv[k], qd), qd, qinv);
    ykd[k] = u2d(yk);
    s = __dadd_rn(s, __dmul_rn(__ull2double_rn(yk), K.invb[k]));
  }
  const double v = u2d((u64)__dadd_rn(s, 0.5));
  u64 *o = d + ((u64)item * 3 + p) * L * N;
#pragma unroll
  for (int l = 0; l < L; l++) {
    const double qd = K.qd[l], qinv = K.qinv[l];
    double acc = -fpm(v, K.BmodQ[l], qd);
#pragma unroll
    for (int k = 0; k < nB; k++) {
      acc += fpm(ykd[k], K.BhatModQ[k][l], qd);
      if ((k & 3) == 2) acc = fp_reduce(acc, qd, qinv);
    }
    o[(u64)l * N + jn] = fp_canon(acc, qd, qinv);
  }
}
template <int L>
__global__ void k_scale_round_t(u64 *d, const u64 *ten, const ModTab *mods, const Consts *C, int iB0, int logN) {
  constexpr int nB = L + 1, nt = L + nB;
  const int item = blockIdx.y;
  const u64 N = 1ull << logN;
  const u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * N) return;
  const u64 jn = i & (N - 1);
  const int p = (int)(i >> logN);
  const u64 *cp = ten + ((u64)item * 3 + p) * nt * N;
  u64 y[L];
  u128 S = 0;
#pragma unroll
  for (int l = 0; l < L; l++) {
    y[l] = mul_shoup(cp[(u64)l * N + jn], C->QBhatInv[l], C->QBhatInv_sh[l], mods[l].q);
    S += (u128)y[l] * C->sc_th_hi[l] + (u128)__umul64hi(y[l], C->sc_th_lo[l]);
  }
  const u64 R = (u64)((S + ((u128)1 << 63)) >> 64);
  u64 yk[nB];
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < nB; k++) {
    const u64 q = mods[iB0 + k].q;
    u64 acc = reduce4(R, q);
#pragma unroll
    for (int l = 0; l < L; l++) {
      acc += mul_shoup_lazy(y[l], C->sc_omega[l][k], C->sc_omega_sh[l][k], q);
      if ((l & 3) == 2) acc = lazy_fold(acc, q);
    }
    acc = lazy_fold(acc, q);
    const u64 z = mul_shoup(cp[(u64)(L + k) * N + jn], C->BQhatInv[k], C->BQhatInv_sh[k], q);
    acc = lazy_final(acc + mul_shoup_lazy(z, C->tBhat[k], C->tBhat_sh[k], q), q);
    yk[k] = mul_shoup(acc, C->BhatInv[k], C->BhatInv_sh[k], q);
    s = __dadd_rn(s, __dmul_rn(__ull2double_rn(yk[k]), C->invb[k]));
  }
  const u64 v = (u64)__dadd_rn(s, 0.5);
  u64 *o = d + ((u64)item * 3 + p) * L * N;
#pragma unroll
  for (int l = 0; l < L; l++) {
    const u64 q = mods[l].q;
    u64 acc = 0;
#pragma unroll
    for (int k = 0; k < nB; k++) {
      acc += mul_shoup_lazy(yk[k], C->BhatModQ[k][l], C->BhatModQ_sh[k][l], q);
      if ((k & 3) == 3) acc = lazy_fold(acc, q);
    }
    acc = lazy_final(acc, q);
    o[(u64)l * N + jn] = sub_mod(acc, mul_shoup(v, C->BmodQ[l], C->BmodQ_sh[l], q), q);
  }
}

// tensor over Q u B: ten[item][3][L+nB][N]
// Q limbs straight from the operand ciphertexts (pa / pb: per-item [2][L][N]),
// B limbs from the lifted buffer
__global__ void k_tensor(u64 *ten, const u64 *in /*[item][4][nt][N]*/, const u64 *const *pa, const u64 *const *pb,
                         const u64 *const *pbx /*null, or b's B-limb extension: [item][2] slots of [nB][N]*/,
                         const ModTab *mods, int L, int nt, int iB0, int logN,
                         const u64 *const *pax = nullptr /*null, or a's B-limb extension (then pbx too)*/) {
  int item = blockIdx.y;
  u64 N = 1ull << logN, P = (u64)nt * N, LN = (u64)L * N;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= P) return;
  int l = (int)(i >> logN);
  const ModTab &M = mods[l < L ? l : iB0 + (l - L)];
  const u64 *x = in + (u64)item * 4 * P;
  u64 a0, a1, b0, b1;
  if (l < L) {
    a0 = pa[item][i], a1 = pa[item][LN + i], b0 = pb[item][i], b1 = pb[item][LN + i];
  } else if (pax) {
    a0 = pax[2 * item][i - LN], a1 = pax[2 * item + 1][i - LN], b0 = pbx[2 * item][i - LN],
    b1 = pbx[2 * item + 1][i - LN];
  } else if (pbx) {
    a0 = x[i], a1 = x[P + i], b0 = pbx[2 * item][i - LN], b1 = pbx[2 * item + 1][i - LN];
  } else {
    a0 = x[i], a1 = x[P + i], b0 = x[2 * P + i], b1 = x[3 * P + i];
  }
  u64 *o = ten + (u64)item * 3 * P;
  o[i] = mul_mod(a0, b0, M);
  o[P + i] = add_mod(mul_mod(a0, b1, M), mul_mod(a1, b0, M), M.q);
  o[2 * P + i] = mul_mod(a1, b1, M);
}
// k_tensor on the FP64 pipe (rings of < 2^49 primes): 4 consecutive words per thread, every
// operand and result a full 32-byte sector access, the four modular products error-free
// FP64 products (5 FP64 instructions against ~14 integer ones, several of them the
// quarter-rate IMAD.HI) -- the same canonical residues.
__global__ void k_tensor_fp(u64 *ten, const u64 *in, const u64 *const *pa, const u64 *const *pb,
                            const u64 *const *pbx, const ModTab *mods, int L, int nt, int iB0, int logN,
                            const u64 *const *pax) {
  const int item = blockIdx.y;
  const u64 N = 1ull << logN, P = (u64)nt * N, LN = (u64)L * N;
  const u64 i = 4 * ((u64)blockIdx.x * blockDim.x + threadIdx.x);
  if (i >= P) return;
  const int l = (int)(i >> logN);
  const ModTab &M = mods[l < L ? l : iB0 + (l - L)];
  const double q = M.qd, qi = M.qinv;
  const u64 *x = in + (u64)item * 4 * P;
  const u64 *p0, *p1, *p2, *p3;
  if (l < L) {
    p0 = pa[item] + i, p1 = pa[item] + LN + i, p2 = pb[item] + i, p3 = pb[item] + LN + i;
  } else if (pax) {
    p0 = pax[2 * item] + (i - LN), p1 = pax[2 * item + 1] + (i - LN), p2 = pbx[2 * item] + (i - LN),
    p3 = pbx[2 * item + 1] + (i - LN);
  } else if (pbx) {
    p0 = x + i, p1 = x + P + i, p2 = pbx[2 * item] + (i - LN), p3 = pbx[2 * item + 1] + (i - LN);
  } else {
    p0 = x + i, p1 = x + P + i, p2 = x + 2 * P + i, p3 = x + 3 * P + i;
  }
  u64 a0[4], a1[4], b0[4], b1[4], o0[4], o1[4], o2[4];
  ld256(p0, a0);
  ld256(p1, a1);
  ld256(p2, b0);
  ld256(p3, b1);
#pragma unroll
  for (int e = 0; e < 4; e++) {
    const double A0 = u2d(a0[e]), A1 = u2d(a1[e]), B0 = u2d(b0[e]), B1 = u2d(b1[e]);
    const double B0q = B0 * qi, B1q = B1 * qi;
    o0[e] = fp_canon(fp_mulmod(A0, B0, B0q, q), q, qi);
    o1[e] = fp_canon(fp_mulmod(A0, B1, B1q, q) + fp_mulmod(A1, B0, B0q, q), q, qi);
    o2[e] = fp_canon(fp_mulmod(A1, B1, B1q, q), q, qi);
  }
  u64 *o = ten + (u64)item * 3 * P + i;
  st256(o, o0[0], o0[1], o0[2], o0[3]);
  st256(o + P, o1[0], o1[1], o1[2], o1[3]);
  st256(o + 2 * P, o2[0], o2[1], o2[2], o2[3]);
}
static bool g_tensor_fp = true;  // CGB_TENSOR_FP
// The tensor product fed straight into the first (row) pass of its inverse NTT:
// unit (k, l) of item i is d_k in limb l of Q u B -- (a0 b0, a0 b1 + a1 b0, a1 b1)
// mod q_l, from the operands' NTT words (the same residues k_tensor writes).  The
// 3 (L + nB) tensor limb-polys never make the HBM round trip (mult_cipher).
struct TensorLoad {
  static constexpr bool active = false;  // stores: the plain transform's
  static constexpr bool loads = true;
  const u64 *const *pa, *const *pb;      // arena items: the Q limbs of a, b (NTT form)
  const u64 *in;                         // [item][4][nt][N]: the B limbs of a (polys 0,1), b (2,3)
  const u64 *const *pbx, *const *pax;    // resident B extensions ([2 item + p] -> [nB][N]) or null
  const ModTab *mods;
  int L, nt, iB0, logN;
  __device__ void store(int, int, u64, const u64 *, int) const {}
  __device__ void load4(int item, int sub, u64 pos, u64 out[4]) const {
    const int k = sub / nt, l = sub - k * nt;
    const u64 N = 1ull << logN, P = (u64)nt * N, LN = (u64)L * N;
    const ModTab &M = mods[l < L ? l : iB0 + (l - L)];
    const u64 i = (u64)l * N + pos;
    const u64 *x = in + (u64)item * 4 * P;
    const u64 *a0p, *a1p, *b0p, *b1p;
    if (l < L) {
      a0p = pa[item] + i, a1p = pa[item] + LN + i, b0p = pb[item] + i, b1p = pb[item] + LN + i;
    } else if (pax) {
      a0p = pax[2 * item] + (i - LN), a1p = pax[2 * item + 1] + (i - LN);
      b0p = pbx[2 * item] + (i - LN), b1p = pbx[2 * item + 1] + (i - LN);
    } else if (pbx) {
      a0p = x + i, a1p = x + P + i, b0p = pbx[2 * item] + (i - LN), b1p = pbx[2 * item + 1] + (i - LN);
    } else {
      a0p = x + i, a1p = x + P + i, b0p = x + 2 * P + i, b1p = x + 3 * P + i;
    }
    u64 a0[4], a1[4], b0[4], b1[4];
    if (k != 2) ld256(a0p, a0);
    if (k != 0) ld256(a1p, a1);
    if (k != 2) ld256(b0p, b0);
    if (k != 0) ld256(b1p, b1);
#pragma unroll
    for (int e = 0; e < 4; e++) {
      if (k == 0) out[e] = mul_mod(a0[e], b0[e], M);
      else if (k == 2) out[e] = mul_mod(a1[e], b1[e], M);
      else out[e] = add_mod(mul_mod(a0[e], b1[e], M), mul_mod(a1[e], b0[e], M), M.q);
    }
  }
};
// scale by t/Q and round into B, then centred B -> Q: d[item][3][L][N]
__global__ void k_scale_round(u64 *d, const u64 *ten, const ModTab *mods, const Consts *C, int L, int nB, int iB0,
                              int logN) {
  int item = blockIdx.y;
  u64 N = 1ull << logN;
  int nt = L + nB;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;  // over [3][N]
  if (i >= 3 * N) return;
  u64 jn = i & (N - 1);
  int p = (int)(i >> logN);
  const u64 *cp = ten + ((u64)item * 3 + p) * nt * N;
  u64 y[MAXL];
  u128 S = 0;
  for (int l = 0; l < L; l++) {
    y[l] = mul_mod(cp[(u64)l * N + jn], C->QBhatInv[l], mods[l]);
    S += (u128)y[l] * C->sc_th_hi[l] + (u128)__umul64hi(y[l], C->sc_th_lo[l]);
  }
  u64 R = (u64)((S + ((u128)1 << 63)) >> 64);
  u64 yk[MAXL + 1];
  double s = 0.0;
  for (int k = 0; k < nB; k++) {
    const ModTab &M = mods[iB0 + k];
    u64 acc = R % M.q;
    for (int l = 0; l < L; l++) acc = add_mod(acc, mul_mod(y[l], C->sc_omega[l][k], M), M.q);
    u64 z = mul_mod(cp[(u64)(L + k) * N + jn], C->BQhatInv[k], M);
    acc = add_mod(acc, mul_mod(z, C->tBhat[k], M), M.q);
    yk[k] = mul_mod(acc, C->BhatInv[k], M);
    s = __dadd_rn(s, __dmul_rn(__ull2double_rn(yk[k]), C->invb[k]));
  }
  u64 v = (u64)__dadd_rn(s, 0.5);
  u64 *o = d + ((u64)item * 3 + p) * L * N;
  for (int l = 0; l < L; l++) {
    const ModTab &M = mods[l];
    u64 acc = 0;
    for (int k = 0; k < nB; k++) acc = add_mod(acc, mul_mod(yk[k], C->BhatModQ[k][l], M), M.q);
    acc = sub_mod(acc, mul_mod(v, C->BmodQ[l], M), M.q);
    o[(u64)l * N + jn] = acc;
  }
}

// encoding / encryption / decryption ----------------------------------------
__global__ void k_scatter_slots(u64 *m /*[item][N]*/, const u64 *slots /*[item][n]*/, const u32 *slot_idx, int n,
                                u64 t, int logN) {
  int item = blockIdx.y;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  m[((u64)item << logN) + slot_idx[i]] = slots[(u64)item * n + i] % t;
}
__global__ void k_gather_slots(u64 *slots, const u64 *m, const u32 *slot_idx, int n, int logN) {
  int item = blockIdx.y;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  slots[(u64)item * n + i] = m[((u64)item << logN) + slot_idx[i]];
}
// plaintext lift into L limbs (coefficient form): kind 0 centred, kind 1 floor(Q m / t)
__global__ void k_pt_lift(u64 *const *pt, const u64 *m, const ModTab *mods, const Consts *C, int L, int logN, int kind) {
  int item = blockIdx.y;
  u64 N = 1ull << logN, words = (u64)L * N;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= words) return;
  int l = (int)(i >> logN);
  u64 jn = i & (N - 1);
  u64 q = mods[l].q, t = C->t;
  u64 v = m[((u64)item << logN) + jn];
  u64 out;
  if (kind == CGB_PT_MUL) {
    out = (v <= t / 2) ? v % q : (q - ((t - v) % q)) % q;
  } else {
    u64 r = (u64)(((u128)C->Qmodt * v) % t);
    out = sub_mod(0, mul_mod(r % q, C->tinvq[l], mods[l]), q);
  }
  pt[item][i] = out;
}
__device__ __forceinline__ u64 u128_mod(u64 hi, u64 lo, const ModTab &M) {
  return add_mod(mul_mod(hi % M.q, M.r64, M), lo % M.q, M.q);
}
// uniform residues in NTT form from ChaCha20: element e = l*N + j uses words 4e..4e+3
__global__ void k_sample_uniform(u64 *const *dst, const ChaKey *keys, const u64 *nonces, int nl, const int *mod_idx,
                                 const ModTab *mods, int logN) {
  int item = blockIdx.y;
  u64 N = 1ull << logN, nblk = ((u64)nl * N + 3) / 4;
  u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nblk) return;
  u32 w[16];
  const ChaKey key = keys[item];
  chacha_block(key, c, nonces[item], w);
#pragma unroll
  for (int r = 0; r < 4; r++) {
    u64 e = 4 * c + r;
    if (e >= (u64)nl * N) break;
    int l = (int)(e >> logN);
    const ModTab &M = mods[mod_idx[l]];
    u64 lo = (u64)w[4 * r] | ((u64)w[4 * r + 1] << 32), hi = (u64)w[4 * r + 2] | ((u64)w[4 * r + 3] << 32);
    dst[item][e] = u128_mod(hi, lo, M);
  }
}
// centred binomial (eta = 21) errors: element j uses words 2j, 2j+1
__global__ void k_sample_cbd(i64 *e, const ChaKey *keys, const u64 *nonces, int logN) {
  int item = blockIdx.y;
  u64 N = 1ull << logN, nblk = (N + 7) / 8;
  u64 c = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nblk) return;
  u32 w[16];
  const ChaKey key = keys[item];
  chacha_block(key, c, nonces[item], w);
#pragma unroll
  for (int r = 0; r < 8; r++) {
    u64 j = 8 * c + r;
    if (j >= N) break;
    u64 x = (u64)w[2 * r] | ((u64)w[2 * r + 1] << 32);
    e[((u64)item << logN) + j] = (i64)__popcll(x & 0x1FFFFFull) - (i64)__popcll((x >> 21) & 0x1FFFFFull);
  }
}
// c0 coefficient form: floor(Q m / t) + e  (mod q_l), written into limbs of dst items (poly 0)
__global__ void k_enc_c0(u64 *const *dst, const u64 *m, const i64 *e, const ModTab *mods, const Consts *C, int L,
                         int logN) {
  int item = blockIdx.y;
  u64 N = 1ull << logN, words = (u64)L * N;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= words) return;
  int l = (int)(i >> logN);
  u64 jn = i & (N - 1);
  const ModTab &M = mods[l];
  u64 t = C->t, v = m[((u64)item << logN) + jn];
  u64 r = (u64)(((u128)C->Qmodt * v) % t);
  u64 sc = sub_mod(0, mul_mod(r % M.q, C->tinvq[l], M), M.q);
  i64 ev = e[((u64)item << logN) + jn];
  u64 er = ev >= 0 ? (u64)ev % M.q : (M.q - ((u64)(-ev) % M.q)) % M.q;
  dst[item][i] = add_mod(sc, er, M.q);
}
// c0 -= c1 * s  (NTT form), per item pointer
__global__ void k_enc_sub_as(u64 *const *ct, const u64 *s, const ModTab *mods, int L, int logN) {
  int item = blockIdx.y;
  u64 N = 1ull << logN, words = (u64)L * N;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= words) return;
  int l = (int)(i >> logN);
  const ModTab &M = mods[l];
  u64 *c = ct[item];
  c[i] = sub_mod(c[i], mul_mod(c[words + i], s[i], M), M.q);
}
// X[item][l] = c0 + c1 s (NTT form) ; optionally times t (noise diagnostic)
__global__ void k_dec_inner(u64 *X, const u64 *const *ct, const u64 *s, const ModTab *mods, const Consts *C, int L,
                            int logN, int times_t) {
  int item = blockIdx.y;
  u64 N = 1ull << logN, words = (u64)L * N;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= words) return;
  int l = (int)(i >> logN);
  const ModTab &M = mods[l];
  const u64 *c = ct[item];
  u64 v = add_mod(c[i], mul_mod(c[words + i], s[i], M), M.q);
  if (times_t) v = mul_mod(v, C->t % M.q, M);
  X[(u64)item * words + i] = v;
}
// m = [sum_l x_l omega_l + round(sum_l x_l theta_l)]_t
__global__ void k_dec_scale(u64 *m, const u64 *X, const Consts *C, int L, int logN) {
  int item = blockIdx.y;
  u64 N = 1ull << logN;
  u64 jn = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (jn >= N) return;
  u64 t = C->t;
  u128 S = 0;
  u64 I = 0;
  for (int l = 0; l < L; l++) {
    u64 x = X[((u64)item * L + l) * N + jn];
    S += (u128)x * C->dec_th_hi[l] + (u128)__umul64hi(x, C->dec_th_lo[l]);
    I = (I + (u64)(((u128)(x % t) * C->dec_omega[l]) % t)) % t;
  }
  u64 R = (u64)((S + ((u128)1 << 63)) >> 64);
  m[((u64)item << logN) + jn] = (I + R % t) % t;
}
// keygen: b[l] = e_l - a_l s_l + (l == j ? [P]_{q_j} s'_l : 0)
__global__ void k_ksk_b(u64 *key /*[L][2][L+1][N]*/, int j, const i64 *e, const u64 *s, const u64 *sp,
                        const ModTab *mods, const Consts *C, int L, int iP, int logN) {
  u64 N = 1ull << logN, LP = L + 1;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= LP * N) return;
  int l = (int)(i >> logN);
  u64 jn = i & (N - 1);
  const ModTab &M = mods[l == L ? iP : l];
  u64 *b = key + ((u64)j * 2 + 0) * LP * N, *a = key + ((u64)j * 2 + 1) * LP * N;
  i64 ev = e[jn];
  u64 er = ev >= 0 ? (u64)ev % M.q : (M.q - ((u64)(-ev) % M.q)) % M.q;
  b[i] = er;  // NTT applied by the caller, then k_ksk_fin
  (void)a; (void)s; (void)sp; (void)C;
}
__global__ void k_ksk_fin(u64 *key, int j, const u64 *s, const u64 *sp, const ModTab *mods, const Consts *C, int L,
                          int iP, int logN) {
  u64 N = 1ull << logN, LP = L + 1;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= LP * N) return;
  int l = (int)(i >> logN);
  const ModTab &M = mods[l == L ? iP : l];
  u64 *b = key + ((u64)j * 2 + 0) * LP * N, *a = key + ((u64)j * 2 + 1) * LP * N;
  u64 v = sub_mod(b[i], mul_mod(a[i], s[i], M), M.q);
  if (l == j) v = add_mod(v, mul_mod(C->Pmodq[j], sp[i], M), M.q);
  b[i] = v;
}
__global__ void k_square(u64 *dst, const u64 *s, const ModTab *mods, int nl, const int *mod_idx, int logN) {
  u64 N = 1ull << logN;
  u64 i = (u64)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (u64)nl * N) return;
  const ModTab &M = mods[mod_idx[i >> logN]];
  dst[i] = mul_mod(s[i], s[i], M);
}

// integer-pipe peak: independent chains of the NTT's 64-bit Shoup modmul,
// register resident (8 chains per thread, no memory traffic in the loop)
__global__ void k_modmul_peak(u64 *sink, u64 q, u64 w, u64 wsh, int iters) {
  u64 x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = (threadIdx.x * 8 + k + 1) % q;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = mul_shoup(x[k], w, wsh, q);
  }
  u64 acc = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) acc ^= x[k];
  if (acc == 0x1234567) sink[0] = acc;
}

// the same chains on the FP64 pipe (the exact error-free product of the FP64 NTT)
__global__ void k_modmul_peak_fp(u64 *sink, double q, double w, double wq, int iters) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; k++) x[k] = (double)(threadIdx.x * 8 + k + 1);
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = fp_mulmod(x[k], w, wq, q);
  }
  double acc = 0;
#pragma unroll
  for (int k = 0; k < 8; k++) acc += x[k];
  if (acc == 0.5) sink[0] = 1;
}

// ============================================================================
// host orchestration
// ============================================================================
static const int TPB = 256;

static std::vector<u64 *> ct_ptrs(cgb_ring *r, int count, const u32 *ids) {
  std::vector<u64 *> v(count);
  for (int i = 0; i < count; i++) {
    if (ids[i] >= r->arena_cap || !r->ct_used[ids[i]]) FAIL(CGB_ERR_PARAM, "invalid ciphertext id %u", ids[i]);
    v[i] = r->arena + (size_t)ids[i] * r->ct_words;
  }
  return v;
}
static std::vector<u64 *> pt_ptrs(cgb_ring *r, int count, const u32 *ids) {
  std::vector<u64 *> v(count);
  size_t w = (size_t)r->L * r->N;
  for (int i = 0; i < count; i++) {
    if (ids[i] >= r->pt_cap || !r->pt_used[ids[i]]) FAIL(CGB_ERR_PARAM, "invalid plaintext id %u", ids[i]);
    v[i] = r->pt_arena + (size_t)ids[i] * w;
  }
  return v;
}
static int *q_mod_idx(cgb_ring *r, std::vector<int> &v) {
  v.resize(r->L);
  for (int l = 0; l < r->L; l++) v[l] = l;
  return v.data();
}

// encode host slots into plaintext polys m[count][N] (coefficient form mod t)
static void encode_slots(cgb_ring *r, Scratch &S, const u64 *slots_host, int count, u64 *m) {
  u64 *d_slots = S.up(slots_host, (size_t)count * r->n_slots);
  CK(cudaMemsetAsync(m, 0, sizeof(u64) * (size_t)count * r->N, r->stream));
  LAUNCH("scatter_slots", BYTES_scatter_slots, k_scatter_slots<<<dim3(GRID1(r->n_slots, TPB).x, count), TPB, 0, r->stream>>>(m, d_slots, r->d_slot_idx,
                                                                                r->n_slots, r->t, r->logN));
  int mi = r->iT;
  ntt_items(r, false, m, nullptr, r->N, count, 1, 1, &mi);
}

static u64 *get_key(cgb_ring *r, u64 g);

// key-switch fusion: bit 0 = ModUp row pass + inner product, bit 1 = ModDown row pass
// + combine (CGB_KS_FUSED; 0 = the unfused pipeline)
static int g_ks_fused = 0;  // measured: the unfused pipeline is faster (profiles/r01)

// ---- fused key switch (two-pass rings): column passes as NTT launches, the row
// passes fused with the key inner product (ModUp) and the combine (ModDown)
template <int LA, int LB, int L>
static void keyswitch_fused_t(cgb_ring *r, Scratch &S, const KsSrc &x, int count, u64 *const *d_keys,
                              u64 *const *d_out, const KsSrc &add0, const u64 *const *d_add1) {
  constexpr int LP = L + 1, E = 8;
  const int N = r->N, logN = r->logN;
  using RT = RowTile<LA, LB, E>;
  // digits in coefficient form (automorphism fused into the inverse NTT's load)
  u64 *xc = S.alloc<u64>((size_t)count * L * N);
  {
    NttJob job{};
    job.base = xc;
    job.item_stride = (u64)L * N;
    job.src_items = x.items;
    job.src_base = x.items ? nullptr : x.base;
    job.src_stride = x.stride;
    job.galois = x.g;
    const int off = (int)(x.items ? x.off / (u64)N : 0);
    for (int l = 0; l < L; l++) {
      job.sub_off[l] = (unsigned short)l;
      job.sub_mod[l] = (unsigned char)l;
      job.src_off[l] = (unsigned short)(off + l);
    }
    job.nsub = L;
    launch_ntt(r, false, job, count);
  }
  // ModUp column pass (centred lift fused into the load) -> D
  u64 *D = S.alloc<u64>((size_t)count * L * LP * N);
  {
    NttJob job{};
    job.base = D;
    job.item_stride = (u64)L * LP * N;
    job.src_base = xc;
    job.src_stride = (u64)L * N;
    job.lift = 1;
    job.mods = r->d_mods;
    job.logN = logN;
    int n = 0;
    for (int j = 0; j < L; j++)
      for (int l = 0; l < LP; l++) {
        if (l == j) continue;
        job.sub_off[n] = (unsigned short)(j * LP + l);
        job.sub_mod[n] = (unsigned char)(l == L ? r->iP : l);
        job.src_off[n] = (unsigned short)j;
        job.src_mod[n] = (unsigned char)j;
        n++;
      }
    job.nsub = n;
    launch_begin(r);
    launch_ntt2_colpass<LA, LB>(r, job, count);
    launch_end(r, "ntt_fwd", 16.0 * (double)count * n * N);
  }
  // ModUp row pass + key inner product -> acc
  u64 *acc = S.alloc<u64>((size_t)count * 2 * LP * N);
  {
    const u64 kw = (u64)L * 2 * LP * N;
    launch_begin(r);
    const dim3 grid((unsigned)((size_t)count * LP * RT::TILES));
    if (r->fp_ntt)
      k_modup_ks<LA, LB, L, E, true><<<grid, RT::T, RT::smem(), r->stream>>>(D, x, d_keys, kw, acc, r->d_mods);
    else
      k_modup_ks<LA, LB, L, E, false><<<grid, RT::T, RT::smem(), r->stream>>>(D, x, d_keys, kw, acc, r->d_mods);
    launch_end(r, "modup_ks", 8.0 * (double)count * LP * N * (L * 2.0 + 2.0));
  }
  // ModDown: INTT the P limbs (both passes), column pass of their lift into Q -> W
  {
    NttJob job{};
    job.base = acc;
    job.item_stride = 2ull * LP * N;
    job.sub_off[0] = (unsigned short)L;
    job.sub_mod[0] = (unsigned char)r->iP;
    job.sub_off[1] = (unsigned short)(LP + L);
    job.sub_mod[1] = (unsigned char)r->iP;
    job.nsub = 2;
    launch_ntt(r, false, job, count);
  }
  u64 *W = S.alloc<u64>((size_t)count * 2 * L * N);
  NttJob job{};
  job.base = W;
  job.item_stride = 2ull * L * N;
  job.src_base = acc;
  job.src_stride = 2ull * LP * N;
  job.lift = 1;
  job.mods = r->d_mods;
  job.logN = logN;
  int n = 0;
  for (int pp = 0; pp < 2; pp++)
    for (int l = 0; l < L; l++) {
      job.sub_off[n] = (unsigned short)(pp * L + l);
      job.sub_mod[n] = (unsigned char)l;
      job.src_off[n] = (unsigned short)(pp * LP + L);
      job.src_mod[n] = (unsigned char)r->iP;
      n++;
    }
  job.nsub = n;
  if (!(g_ks_fused & 2)) {  // ModDown: full NTT of the lift, then the separate combine
    launch_ntt(r, true, job, count);
    LAUNCH("moddown_combine", BYTES_moddown_combine,
           k_moddown_combine<<<dim3(GRID1(2ull * L * N, TPB).x, count), TPB, 0, r->stream>>>(
               d_out, acc, W, add0, d_add1, r->d_mods, r->d_c, L, logN));
    return;
  }
  launch_begin(r);
  launch_ntt2_colpass<LA, LB>(r, job, count);
  launch_end(r, "ntt_fwd", 16.0 * (double)count * n * N);
  launch_begin(r);
  const dim3 gridm((unsigned)((size_t)count * 2 * L * RT::TILES));
  if (r->fp_ntt)
    k_moddown_fused<LA, LB, E, true><<<gridm, RT::T, RT::smem(), r->stream>>>(W, acc, d_out, add0, d_add1, r->d_mods,
                                                                            r->d_c, L);
  else
    k_moddown_fused<LA, LB, E, false><<<gridm, RT::T, RT::smem(), r->stream>>>(W, acc, d_out, add0, d_add1, r->d_mods,
                                                                             r->d_c, L);
  launch_end(r, "moddown_fused", 8.0 * (double)count * 2 * L * N * (3 + (add0.items ? 0.5 : 0) + (d_add1 ? 1 : 0)));
}
template <int LA, int LB, int L>
static void fused_attrs() {
  const int s = (int)RowTile<LA, LB, 8>::smem();
  CK(cudaFuncSetAttribute(k_modup_ks<LA, LB, L, 8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s));
  CK(cudaFuncSetAttribute(k_modup_ks<LA, LB, L, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s));
  CK(cudaFuncSetAttribute(k_moddown_fused<LA, LB, 8, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, s));
  CK(cudaFuncSetAttribute(k_moddown_fused<LA, LB, 8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, s));
}
static bool keyswitch_fused(cgb_ring *r, Scratch &S, const KsSrc &x, int count, u64 *const *d_keys, u64 *const *d_out,
                            const KsSrc &add0, const u64 *const *d_add1) {
  if (!(g_ks_fused & 1)) return false;
#define KSF(A, B, LL)                                                                \
  if (r->logN == A + B && r->L == LL) {                                              \
    keyswitch_fused_t<A, B, LL>(r, S, x, count, d_keys, d_out, add0, d_add1);        \
    return true;                                                                     \
  }
#define KSF_L(A, B) KSF(A, B, 2) KSF(A, B, 3) KSF(A, B, 4) KSF(A, B, 5) KSF(A, B, 6) KSF(A, B, 8)
  KSF_L(6, 7) KSF_L(7, 7) KSF_L(7, 8) KSF_L(8, 8)
#undef KSF_L
#undef KSF
  return false;
}
static void fused_attrs_for(int logN, int L) {
#define FA(A, B, LL) if (logN == A + B && L == LL) fused_attrs<A, B, LL>();
#define FA_L(A, B) FA(A, B, 2) FA(A, B, 3) FA(A, B, 4) FA(A, B, 5) FA(A, B, 6) FA(A, B, 8)
  FA_L(6, 7) FA_L(7, 7) FA_L(7, 8) FA_L(8, 8)
#undef FA_L
#undef FA
}

// key switch of `count` NTT-form polys (descriptor x: contiguous, or arena items read
// through an automorphism) with per-item keys; result combined into out pointers:
// out = (ks0 + add0 + add1, ks1 + add1)
// The FP64-ring key switch in five launches:
//   1 inverse row pass of the digits (automorphism fused into its load)      -> xr
//   2 k_col_fused: inverse column pass + lift + forward column passes (ModUp) -> D
//   3 k_ks_row: forward row passes + key inner product; P limb: inverse row   -> acc
//   4 k_col_fused: P limb inverse column pass + lift into Q + column passes   -> W
//   5 forward row pass of W with the ModDown combine as its store epilogue    -> out
template <int LA, int LB, int L>
static void keyswitch_fp_t(cgb_ring *r, Scratch &S, const KsSrc &x, int count, u64 *const *d_keys,
                           u64 *const *d_out, const KsSrc &add0, const u64 *const *d_add1) {
  constexpr int LP = L + 1, N = 1 << (LA + LB), G0 = NTT2_TILE >> LA, G1 = NTT2_TILE >> LB;
  // one scratch allocation for the four intermediates
  const size_t nxr = (size_t)count * L * N, nD = (size_t)count * L * LP * N, nacc = (size_t)count * 2 * LP * N;
  u64 *xr = S.alloc<u64>(nxr + nD + nacc + (size_t)count * 2 * L * N);
  u64 *D = xr + nxr;
  u64 *acc = D + nD;
  u64 *W = acc + nacc;
  const dim3 rows_grid1((unsigned)((size_t)count * L * ((1 << LA) / G1)));
  // unreduced D / W only with the kernels that take the flag as a template parameter
  const bool unred = CGB_COL_UNRED_BUILD && g_col_unred && g_ks_md && g_ksrow2 >= 1;
  const int rawf = 3;
  {  // 1
    NttJob job{};
    job.base = xr;
    job.item_stride = (u64)L * N;
    job.src_items = x.items;
    job.src_base = x.items ? nullptr : x.base;
    job.src_stride = x.stride;
    job.galois = x.g;
    const int off = (int)(x.items ? x.off / (u64)N : 0);
    for (int l = 0; l < L; l++) {
      job.sub_off[l] = (unsigned short)l;
      job.sub_mod[l] = (unsigned char)l;
      job.src_off[l] = (unsigned short)(off + l);
    }
    job.nsub = L;
    job.mods = r->d_mods;
    job.logN = LA + LB;
    job.out_raw = 1;  // pass boundary: the column pass (k_col_fused) reads reduced doubles
    launch_begin(r);
    launch_pdl(r, k_ntt2_fpr<LA, LB, false, 1>, rows_grid1, NTT2_TILE / 16, fpr_smem_bytes<LA, LB>(1), job, NoEpi{});
    launch_end(r, "ks_digit_rows", 16.0 * (double)count * L * N, (double)count * L * (N / 2) * LB);
  }
  {  // 2
    ColJob cj{};
    cj.src = xr;
    cj.src_stride = (u64)L * N;
    cj.dst = D;
    cj.dst_stride = (u64)L * LP * N;
    cj.nsrc = L;
    cj.in_raw = 1;
    cj.out_raw = unred ? 2 : 1;  // unreduced: the row kernels reduce on load
    for (int j = 0; j < L; j++) {
      cj.src_off[j] = (unsigned short)j;
      cj.src_mod[j] = (unsigned char)j;
      int t = 0;
      for (int l = 0; l < LP; l++) {
        if (l == j) continue;
        cj.dst_off[j][t] = (unsigned short)(j * LP + l);
        cj.dst_mod[j][t] = (unsigned char)(l == L ? r->iP : l);
        t++;
      }
    }
    col_fused(r, cj, count, L, "ks_modup_cols");
  }
  const MdEpi epi{d_out, acc, add0, d_add1, r->d_mods, r->d_c, L, LA + LB};
  const int TILES = (1 << LA) / G1;
  ks_row_attrs<LA, LB, L>();
  if (g_ks_md && g_ksrow2) {
    static std::once_flag once2;
    std::call_once(once2, [] {
#if CGB_BUILD_FALLBACKS
      CK(cudaFuncSetAttribute(k_ks_row2<LA, LB, L, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)ks_row2_smem<LB>()));
#endif
      CK(cudaFuncSetAttribute(k_ks_row2<LA, LB, L, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)ks_row2_smem<LB>()));
      CK(cudaFuncSetAttribute(k_ks_row2<LA, LB, L, true, false, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)ks_row2_smem<LB>()));
      CK(cudaFuncSetAttribute(k_ks_row2<LA, LB, L, true, false, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)ks_row2_smem<LB>()));
#if CGB_COL_UNRED_BUILD
#if CGB_BUILD_FALLBACKS
      CK(cudaFuncSetAttribute(k_ks_row2<LA, LB, L, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)ks_row2_smem<LB>()));
#endif
      CK(cudaFuncSetAttribute(k_ks_row2<LA, LB, L, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)ks_row2_smem<LB>()));
#endif
    });
  }
  if (g_ks_md) {  // 3: the P limb only (its accumulators feed ModDown's INTT)
    launch_begin(r);
    const dim3 gP((unsigned)((size_t)count * TILES));
    bool done = false;
#if CGB_COL_UNRED_BUILD && CGB_BUILD_FALLBACKS
    if (!done && g_ksrow2 >= 2 && unred) {
      launch_pdl(r, k_ks_row2<LA, LB, L, false, true>, gP, NTT2_TILE / 16, ks_row2_smem<LB>(), acc, (const u64 *)D, x,
                 d_keys, (const ModTab *)r->d_mods, r->iP, (const u64 *)nullptr, epi, rawf);
      done = true;
    }
#endif
#if CGB_BUILD_FALLBACKS
    if (!done && g_ksrow2 >= 2) {
      launch_pdl(r, k_ks_row2<LA, LB, L, false>, gP, NTT2_TILE / 16, ks_row2_smem<LB>(), acc, (const u64 *)D, x,
                 d_keys, (const ModTab *)r->d_mods, r->iP, (const u64 *)nullptr, epi, rawf);
      done = true;
    }
#endif
#if CGB_COL_UNRED_BUILD
    if (!done && unred) {
      launch_pdl(r, k_ks_row<LA, LB, L, 1, true>, gP, NTT2_TILE / 16, ks_row_smem<LA, LB>(), acc, D, x, d_keys,
                 r->d_mods, r->iP, count, (const u64 *)nullptr, epi, rawf);
      done = true;
    }
#endif
    if (!done)
      launch_pdl(r, k_ks_row<LA, LB, L, 1>, gP, NTT2_TILE / 16, ks_row_smem<LA, LB>(), acc, D, x, d_keys, r->d_mods,
                 r->iP, count, (const u64 *)nullptr, epi, rawf);
    launch_end(r, "ks_row_P", 8.0 * (double)count * N * (L + 2.0) + 16.0 * L * N,
               (double)count * ((N / 2) * LB * (L + 2.0) + 2.0 * L * N));
  }
#if CGB_BUILD_FALLBACKS
  else {  // 3
    const dim3 g1((unsigned)((size_t)count * LP * TILES));
    launch_begin(r);
    launch_pdl(r, k_ks_row<LA, LB, L, 0>, g1, NTT2_TILE / 16, ks_row_smem<LA, LB>(), acc, D, x, d_keys, r->d_mods,
               r->iP, count, (const u64 *)nullptr, epi, rawf);
    launch_end(r, "ks_row", 8.0 * (double)count * N * (L * L + 2.0 * LP + 4.0) + 16.0 * L * (double)LP * N,
               (double)count * ((N / 2) * LB * (L * L + 2.0) + 2.0 * LP * L * N));
  }
#endif
  {  // 4
    ColJob cj{};
    cj.src = acc;
    cj.src_stride = 2ull * LP * N;
    cj.dst = W;
    cj.dst_stride = 2ull * L * N;
    cj.nsrc = 2;
    cj.in_raw = 1;
    cj.out_raw = unred ? 2 : 1;  // unreduced: the row kernels reduce on load
    for (int pp = 0; pp < 2; pp++) {
      cj.src_off[pp] = (unsigned short)(pp * LP + L);
      cj.src_mod[pp] = (unsigned char)r->iP;
      for (int l = 0; l < L; l++) {
        cj.dst_off[pp][l] = (unsigned short)(pp * L + l);
        cj.dst_mod[pp][l] = (unsigned char)l;
      }
    }
    col_fused(r, cj, count, L, "ks_moddown_cols");
  }
  if (g_ks_md) {  // 5: Q limbs' inner product + ModDown row pass of W + combine -> out
    launch_begin(r);
    if (g_ksrow2) {
      const bool c0 = add0.items || add0.base, a1 = d_add1 != nullptr;
      const dim3 gmd((unsigned)((size_t)count * L * TILES));
#define KSR2(U, F)                                                                                              \
  launch_pdl(r, k_ks_row2<LA, LB, L, true, U, F>, gmd, NTT2_TILE / 16, ks_row2_smem<LB>(), acc, (const u64 *)D, x, \
             d_keys, (const ModTab *)r->d_mods, r->iP, (const u64 *)W, epi, rawf)
#if CGB_COL_UNRED_BUILD
      if (unred) KSR2(true, -1);
      else
#endif
      if (g_ksrow2_spec && c0 && a1) KSR2(false, 3);
      else if (g_ksrow2_spec && c0) KSR2(false, 1);
      else KSR2(false, -1);
#undef KSR2
    }
#if CGB_BUILD_FALLBACKS
    else
    if constexpr (LB == 7) {
      if (g_ksrow8) {
        static std::once_flag once8;
        std::call_once(once8, [] {
          CK(cudaFuncSetAttribute(k_ks_row8<LA, LB, L>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)ks_row_smem<LA, LB>()));
        });
        launch_pdl(r, k_ks_row8<LA, LB, L>, dim3((unsigned)((size_t)count * L * TILES)), NTT2_TILE / 8,
                   ks_row_smem<LA, LB>(), (const u64 *)D, x, d_keys, (const ModTab *)r->d_mods, (const u64 *)W, epi, rawf);
      } else {
        launch_pdl(r, k_ks_row<LA, LB, L, 2>, dim3((unsigned)((size_t)count * L * TILES)), NTT2_TILE / 16,
                   ks_row_smem<LA, LB>(), acc, D, x, d_keys, r->d_mods, r->iP, count, (const u64 *)W, epi, rawf);
      }
    } else {
      launch_pdl(r, k_ks_row<LA, LB, L, 2>, dim3((unsigned)((size_t)count * L * TILES)), NTT2_TILE / 16,
                 ks_row_smem<LA, LB>(), acc, D, x, d_keys, r->d_mods, r->iP, count, (const u64 *)W, epi, rawf);
    }
#endif
    // D (L-1 digits) + own digit + W (2) + out (2) per limb, c0 / add1 when present; keys once
    launch_end(r, "ks_row_md",
               8.0 * (double)count * N * L * (L + 4.0 + (add0.items || add0.base ? 1 : 0) + (d_add1 ? 2 : 0)) +
                   16.0 * L * (double)L * N,
               (double)count * ((N / 2) * LB * (L * (L - 1.0) + 2.0 * L) + 2.0 * L * L * N + 2.0 * L * N));
    return;
  }
  {  // 5
    NttJob job{};
    job.base = W;
    job.item_stride = 2ull * L * N;
    int n = 0;
    for (int pp = 0; pp < 2; pp++)
      for (int l = 0; l < L; l++) {
        job.sub_off[n] = (unsigned short)(pp * L + l);
        job.sub_mod[n] = (unsigned char)l;
        n++;
      }
    job.nsub = n;
    job.mods = r->d_mods;
    job.logN = LA + LB;
    job.in_raw = 1;  // W: reduced doubles from k_col_fused
    const dim3 g((unsigned)((size_t)count * n * ((1 << LA) / G1)));
    launch_begin(r);
    launch_pdl(r, k_ntt2_fpr<LA, LB, true, 1, MdEpi>, g, NTT2_TILE / 16, fpr_smem_bytes<LA, LB>(1), job, epi);
    launch_end(r, "ks_moddown_rows", 8.0 * (double)count * n * N * (3 + (add0.items ? 0.5 : 0) + (d_add1 ? 1 : 0)),
               (double)count * n * ((N / 2) * LB + N));
  }
}
static bool keyswitch_fp(cgb_ring *r, Scratch &S, const KsSrc &x, int count, u64 *const *d_keys, u64 *const *d_out,
                         const KsSrc &add0, const u64 *const *d_add1) {
  if (!(col_fusable(r) && ks_row_fusable(r) && moddown_fusable(r)) || count <= 0) return false;
#define KFP(A, B)                                                                      \
  switch (r->L) {                                                                      \
    case 2: keyswitch_fp_t<A, B, 2>(r, S, x, count, d_keys, d_out, add0, d_add1); break; \
    case 3: keyswitch_fp_t<A, B, 3>(r, S, x, count, d_keys, d_out, add0, d_add1); break; \
    case 4: keyswitch_fp_t<A, B, 4>(r, S, x, count, d_keys, d_out, add0, d_add1); break; \
    case 5: keyswitch_fp_t<A, B, 5>(r, S, x, count, d_keys, d_out, add0, d_add1); break; \
    case 6: keyswitch_fp_t<A, B, 6>(r, S, x, count, d_keys, d_out, add0, d_add1); break; \
    case 7: keyswitch_fp_t<A, B, 7>(r, S, x, count, d_keys, d_out, add0, d_add1); break; \
    default: keyswitch_fp_t<A, B, 8>(r, S, x, count, d_keys, d_out, add0, d_add1); break; \
  }
  switch (r->logN) {
    case 13: KFP(6, 7) break;
    case 14: KFP(CGB_A14, 14 - CGB_A14) break;
    case 15: KFP(7, 8) break;
    default: KFP(8, 8) break;
  }
#undef KFP
  return true;
}

// Hoisted key switch: several Galois elements applied to ONE source (the CPVM
// projections rotate one activation by every diagonal step, linear_kernels.py:105-142).
// sigma_g permutes the NTT evaluation points and commutes with the digit
// decomposition and the centred base extension (centred(q - x) = -centred(x), q odd),
// so digit j of ModUp(sigma_g(c1)) is word perm_g(k) of digit j of ModUp(c1): the
// ModUp (inverse row pass, lift + column passes, forward row pass) runs once per
// source, each item only gathers its digits through perm_g and takes the key inner
// product.  Every word is the same residue the per-item path computes.
static bool g_ks_hoist = true;  // CGB_KS_HOIST
#ifndef CGB_HOIST_MINB
#define CGB_HOIST_MINB 4  // 4 CTAs of 256 per SM (<= 64 registers) at L <= 3
#endif
// The 64-register cap was measured at L = 3 only (0.189 -> 0.179 ms per 256
// rotations, profiles/r01/hoist_micro.json; it already spills 72 bytes there).
// At L = 4 the digit and key arrays alone hold 48 u64, so wider rings keep 2 CTAs.
template <int L>
__global__ void __launch_bounds__(256, (L <= 3 ? CGB_HOIST_MINB : 2)) k_ks_inner_hoist(u64 *acc, const u64 *D, const u32 *srcidx, KsSrc xin,
                                                        const u64 *const *keys, const ModTab *mods, int iP, int logN,
                                                        int lfirst) {
  // 4 consecutive words per thread: the 4 gathered words of a digit sit in one aligned
  // 32-byte block (gather4), the key words and the accumulators move as 256-bit accesses
  constexpr int LP = L + 1;
  const u64 N = 1ull << logN;
  const int item = blockIdx.y;
  const u64 i = ((u64)lfirst << logN) + 4 * ((u64)blockIdx.x * blockDim.x + threadIdx.x);  // over [l][N]
  if (i >= LP * N) return;
  const int l = (int)(i >> logN);
  const u32 k0 = (u32)(i & (N - 1));
  const ModTab &Md = mods[l == L ? iP : l];
  const double qd = Md.qd, qinv = Md.qinv;
  const u64 g = xin.g[item];
  const u64 *Du = D + (u64)srcidx[item] * L * LP * N;
  const u64 *own = xin.items[item] + xin.off;
  const u64 *KF = keys[item] + 2 * (u64)L * 2 * LP * N + i;  // the key's FP64 plane (k_key_fp)
  if constexpr (L > 4) {  // wide rings: digit by digit, the sum reduced after every 4 digits
    double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll 1
    for (int j = 0; j < L; j++) {
      u64 dv[4], k0v[4], k1v[4];
      gather4(l == j ? own + ((u64)j << logN) : Du + ((u64)j * LP + l) * N, k0, g, logN, dv);
      ld256(KF + (u64)(j * 2 + 0) * LP * N, k0v);
      ld256(KF + (u64)(j * 2 + 1) * LP * N, k1v);
#pragma unroll
      for (int e = 0; e < 4; e++) {
        const double xv = u2d(dv[e]), d0 = r2d(k0v[e]), d1 = r2d(k1v[e]);
        a0[e] += fp_mulmod(xv, d0, d0 * qinv, qd);
        a1[e] += fp_mulmod(xv, d1, d1 * qinv, qd);
        if ((j & 3) == 3) {
          a0[e] = fp_reduce(a0[e], qd, qinv);
          a1[e] = fp_reduce(a1[e], qd, qinv);
        }
      }
    }
    u64 *o0 = acc + ((u64)item * 2 + 0) * LP * N + i, *o1 = acc + ((u64)item * 2 + 1) * LP * N + i;
    st256(o0, fp_canon(a0[0], qd, qinv), fp_canon(a0[1], qd, qinv), fp_canon(a0[2], qd, qinv), fp_canon(a0[3], qd, qinv));
    st256(o1, fp_canon(a1[0], qd, qinv), fp_canon(a1[1], qd, qinv), fp_canon(a1[2], qd, qinv), fp_canon(a1[3], qd, qinv));
    return;
  }
  constexpr int LD = L > 4 ? 1 : L;  // (the branch above returned for wider rings)
  u64 dv[LD][4], kv[LD][2][4];
#pragma unroll
  for (int j = 0; j < LD; j++) {
    gather4(l == j ? own + ((u64)j << logN) : Du + ((u64)j * LP + l) * N, k0, g, logN, dv[j]);
    ld256(KF + (u64)(j * 2 + 0) * LP * N, kv[j][0]);
    ld256(KF + (u64)(j * 2 + 1) * LP * N, kv[j][1]);
  }
  double a0[4] = {0.0, 0.0, 0.0, 0.0}, a1[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int j = 0; j < LD; j++)
#pragma unroll
    for (int e = 0; e < 4; e++) {
      const double xv = u2d(dv[j][e]), d0 = r2d(kv[j][0][e]), d1 = r2d(kv[j][1][e]);
      a0[e] += fp_mulmod(xv, d0, d0 * qinv, qd);
      a1[e] += fp_mulmod(xv, d1, d1 * qinv, qd);
    }
  u64 *o0 = acc + ((u64)item * 2 + 0) * LP * N + i, *o1 = acc + ((u64)item * 2 + 1) * LP * N + i;
  st256(o0, fp_canon(a0[0], qd, qinv), fp_canon(a0[1], qd, qinv), fp_canon(a0[2], qd, qinv), fp_canon(a0[3], qd, qinv));
  st256(o1, fp_canon(a1[0], qd, qinv), fp_canon(a1[1], qd, qinv), fp_canon(a1[2], qd, qinv), fp_canon(a1[3], qd, qinv));
}
// ModDown's combine for the hoisted key switch: the Q limbs' accumulator words are
// formed in the epilogue of W's row pass (gathered digits x key plane) and never
// reach memory; only the P limb goes through k_ks_inner_hoist.
static bool g_hoist_fuse = false;  // CGB_HOIST_FUSE: measured slower (2.12 vs 2.01 us/rotation), off
struct MdEpiHoist : MdEpi {
  const u64 *D;
  const u32 *srcidx;
  KsSrc xin;
  const u64 *const *keys;
  __device__ void store(int item, int unit, u64 pos, const u64 *w, int n) const {
    const int pp = unit / L, l = unit - pp * L, LP = L + 1;
    const u64 N = 1ull << logN;
    const ModTab &M = mods[l];
    const double qd = M.qd, qinv = M.qinv;
    const u64 g = xin.g[item];
    const u64 *Du = D + (u64)srcidx[item] * L * LP * N;
    const u64 *KF = keys[item] + 2 * (u64)L * 2 * LP * N + ((u64)pp * LP + l) * N + pos;
    double a[4] = {0.0, 0.0, 0.0, 0.0};
    for (int j = 0; j < L; j++) {
      const u64 *src = l == j ? xin.items[item] + xin.off + ((u64)j << logN) : Du + ((u64)j * LP + l) * N;
      u64 dv[4], kv[4];
      if (n == 4) {
        gather4(src, (u32)pos, g, logN, dv);
        ld256(KF + (u64)j * 2 * LP * N, kv);
      } else {
        dv[0] = src[perm_g((u32)pos, g, logN)];
        kv[0] = KF[(u64)j * 2 * LP * N];
      }
#pragma unroll
      for (int e = 0; e < 4; e++)
        if (e < n) {
          const double d = r2d(kv[e]);
          a[e] += fp_mulmod(u2d(dv[e]), d, d * qinv, qd);
          if ((j & 3) == 3) a[e] = fp_reduce(a[e], qd, qinv);  // > 4 digits stay exact
        }
    }
    u64 av[4];
#pragma unroll
    for (int e = 0; e < 4; e++) av[e] = fp_canon(a[e], qd, qinv);
    if (n == 4) {
      combine4(item, unit, pos, w, av);
      return;
    }
    const u64 q = M.q, pi = C->Pinvq[l], pis = C->Pinvq_sh[l];
    u64 v = mul_shoup(sub_mod(av[0], w[0], q), pi, pis, q);
    if (pp == 0 && (add0.items || add0.base)) v = add_mod(v, ks_src_word(add0, item, l, (u32)pos, logN), q);
    if (add1) v = add_mod(v, add1[item][(u64)unit * N + pos], q);
    out[item][(u64)unit * N + pos] = v;
  }
};
template <int LA, int LB, int L>
static void keyswitch_hoisted_t(cgb_ring *r, Scratch &S, const KsSrc &x, int count, int nu, u64 *const *d_usrc,
                                const u32 *d_srcidx, u64 *const *d_keys, u64 *const *d_out, const KsSrc &add0,
                                const u64 *const *d_add1) {
  constexpr int LP = L + 1, N = 1 << (LA + LB), G1 = NTT2_TILE >> LB;
  constexpr int RT = (1 << LA) / G1;  // row tiles per limb-poly
  const size_t nxr = (size_t)nu * L * N, nD = (size_t)nu * L * LP * N, nacc = (size_t)count * 2 * LP * N;
  u64 *xr = S.alloc<u64>(nxr + nD + nacc + (size_t)count * 2 * L * N);
  u64 *D = xr + nxr, *acc = D + nD, *W = acc + nacc;
  const size_t f1 = fpr_smem_bytes<LA, LB>(1);
  {  // 1: inverse row pass of each source's c1 (no automorphism)
    NttJob job{};
    job.base = xr;
    job.item_stride = (u64)L * N;
    job.src_items = d_usrc;
    const int off = (int)(x.off / (u64)N);
    for (int l = 0; l < L; l++) {
      job.sub_off[l] = (unsigned short)l;
      job.sub_mod[l] = (unsigned char)l;
      job.src_off[l] = (unsigned short)(off + l);
    }
    job.nsub = L;
    job.mods = r->d_mods;
    job.logN = LA + LB;
    job.out_raw = 1;
    launch_begin(r);
    launch_pdl(r, k_ntt2_fpr<LA, LB, false, 1>, dim3((unsigned)((size_t)nu * L * RT)), NTT2_TILE / 16, f1, job, NoEpi{});
    launch_end(r, "ks_digit_rows", 16.0 * (double)nu * L * N, (double)nu * L * (N / 2) * LB);
  }
  {  // 2: inverse column pass + centred lift + forward column passes into the other limbs
    ColJob cj{};
    cj.src = xr;
    cj.src_stride = (u64)L * N;
    cj.dst = D;
    cj.dst_stride = (u64)L * LP * N;
    cj.nsrc = L;
    cj.in_raw = cj.out_raw = 1;
    for (int j = 0; j < L; j++) {
      cj.src_off[j] = (unsigned short)j;
      cj.src_mod[j] = (unsigned char)j;
      int t = 0;
      for (int l = 0; l < LP; l++) {
        if (l == j) continue;
        cj.dst_off[j][t] = (unsigned short)(j * LP + l);
        cj.dst_mod[j][t] = (unsigned char)(l == L ? r->iP : l);
        t++;
      }
    }
    col_fused(r, cj, nu, L, "ks_modup_cols");
  }
  {  // 3: forward row pass of the L x L extended digits, in place -> canonical NTT words
    NttJob job{};
    job.base = D;
    job.item_stride = (u64)L * LP * N;
    int n = 0;
    for (int j = 0; j < L; j++)
      for (int l = 0; l < LP; l++) {
        if (l == j) continue;
        job.sub_off[n] = (unsigned short)(j * LP + l);
        job.sub_mod[n] = (unsigned char)(l == L ? r->iP : l);
        n++;
      }
    job.nsub = n;
    job.mods = r->d_mods;
    job.logN = LA + LB;
    job.in_raw = 1;
    launch_begin(r);
    launch_pdl(r, k_ntt2_fpr<LA, LB, true, 1>, dim3((unsigned)((size_t)nu * n * RT)), NTT2_TILE / 16, f1, job, NoEpi{});
    launch_end(r, "ks_hoist_rows", 16.0 * (double)nu * n * N, (double)nu * n * (N / 2) * LB);
  }
  {  // 4: per item: digits gathered through perm_g, key inner product over Q u P
    launch_begin(r);
    const int lf = g_hoist_fuse ? L : 0, nl = LP - lf;  // fused: the Q limbs are formed in step 7's epilogue
    k_ks_inner_hoist<L><<<dim3(GRID1((u64)nl * N / 4, 256).x, count), 256, 0, r->stream>>>(
        acc, D, d_srcidx, x, d_keys, r->d_mods, r->iP, LA + LB, lf);
    // key plane (2L words) + accumulators (2) per word; the gathered digits are L2-resident
    launch_end(r, "ks_hoist_inner", 8.0 * (double)count * nl * N * (2.0 * L + 2.0), 2.0 * count * L * nl * (double)N);
  }
  {  // 5: ModDown's inverse row pass of the P limb (both polys), in place
    NttJob job{};
    job.base = acc;
    job.item_stride = 2ull * LP * N;
    job.sub_off[0] = (unsigned short)L;
    job.sub_off[1] = (unsigned short)(LP + L);
    job.sub_mod[0] = job.sub_mod[1] = (unsigned char)r->iP;
    job.nsub = 2;
    job.mods = r->d_mods;
    job.logN = LA + LB;
    job.out_raw = 1;
    launch_begin(r);
    launch_pdl(r, k_ntt2_fpr<LA, LB, false, 1>, dim3((unsigned)((size_t)count * 2 * RT)), NTT2_TILE / 16, f1, job,
               NoEpi{});
    launch_end(r, "ks_hoist_prow", 16.0 * (double)count * 2 * N, (double)count * 2 * (N / 2) * LB);
  }
  {  // 6: inverse column pass of P, lift into Q, forward column passes
    ColJob cj{};
    cj.src = acc;
    cj.src_stride = 2ull * LP * N;
    cj.dst = W;
    cj.dst_stride = 2ull * L * N;
    cj.nsrc = 2;
    cj.in_raw = cj.out_raw = 1;
    for (int pp = 0; pp < 2; pp++) {
      cj.src_off[pp] = (unsigned short)(pp * LP + L);
      cj.src_mod[pp] = (unsigned char)r->iP;
      for (int l = 0; l < L; l++) {
        cj.dst_off[pp][l] = (unsigned short)(pp * L + l);
        cj.dst_mod[pp][l] = (unsigned char)l;
      }
    }
    col_fused(r, cj, count, L, "ks_moddown_cols");
  }
  {  // 7: forward row pass of W with the combine (acc_Q - W) P^-1 + sigma(c0) [+ input] as epilogue
    const MdEpi epi{d_out, acc, add0, d_add1, r->d_mods, r->d_c, L, LA + LB};
    NttJob job{};
    job.base = W;
    job.item_stride = 2ull * L * N;
    int n = 0;
    for (int pp = 0; pp < 2; pp++)
      for (int l = 0; l < L; l++) {
        job.sub_off[n] = (unsigned short)(pp * L + l);
        job.sub_mod[n] = (unsigned char)l;
        n++;
      }
    job.nsub = n;
    job.mods = r->d_mods;
    job.logN = LA + LB;
    job.in_raw = 1;
    const dim3 grid((unsigned)((size_t)count * n * RT));
    launch_begin(r);
    if (g_hoist_fuse) {
      MdEpiHoist he;
      static_cast<MdEpi &>(he) = epi;
      he.D = D;
      he.srcidx = d_srcidx;
      he.xin = x;
      he.keys = d_keys;
      launch_pdl(r, k_ntt2_fpr<LA, LB, true, 1, MdEpiHoist>, grid, NTT2_TILE / 16, f1, job, he);
      // W, sigma(c0), out, add1 + the key plane (2 words per digit) per word of the Q limbs
      launch_end(r, "ks_hoist_md",
                 8.0 * (double)count * n * N * (2 + (add0.items ? 0.5 : 0) + (d_add1 ? 1 : 0) + L),
                 (double)count * n * ((N / 2) * LB + N + (double)L * N));
    } else {
      launch_pdl(r, k_ntt2_fpr<LA, LB, true, 1, MdEpi>, grid, NTT2_TILE / 16, f1, job, epi);
      launch_end(r, "ks_moddown_rows", 8.0 * (double)count * n * N * (3 + (add0.items ? 0.5 : 0) + (d_add1 ? 1 : 0)),
                 (double)count * n * ((N / 2) * LB + N));
    }
  }
}
static bool keyswitch_hoisted(cgb_ring *r, Scratch &S, const KsSrc &x, int count, int nu, u64 *const *d_usrc,
                              const u32 *d_srcidx, u64 *const *d_keys, u64 *const *d_out, const KsSrc &add0,
                              const u64 *const *d_add1) {
  if (!(g_ks_hoist && col_fusable(r) && moddown_fusable(r)) || count <= 0 || !x.items || !x.g) return false;
#define KHO(A, B)                                                                                              \
  switch (r->L) {                                                                                              \
    case 2: keyswitch_hoisted_t<A, B, 2>(r, S, x, count, nu, d_usrc, d_srcidx, d_keys, d_out, add0, d_add1); break; \
    case 3: keyswitch_hoisted_t<A, B, 3>(r, S, x, count, nu, d_usrc, d_srcidx, d_keys, d_out, add0, d_add1); break; \
    case 4: keyswitch_hoisted_t<A, B, 4>(r, S, x, count, nu, d_usrc, d_srcidx, d_keys, d_out, add0, d_add1); break; \
    case 5: keyswitch_hoisted_t<A, B, 5>(r, S, x, count, nu, d_usrc, d_srcidx, d_keys, d_out, add0, d_add1); break; \
    case 6: keyswitch_hoisted_t<A, B, 6>(r, S, x, count, nu, d_usrc, d_srcidx, d_keys, d_out, add0, d_add1); break; \
    case 7: keyswitch_hoisted_t<A, B, 7>(r, S, x, count, nu, d_usrc, d_srcidx, d_keys, d_out, add0, d_add1); break; \
    default: keyswitch_hoisted_t<A, B, 8>(r, S, x, count, nu, d_usrc, d_srcidx, d_keys, d_out, add0, d_add1); break; \
  }
  switch (r->logN) {
    case 13: KHO(6, 7) break;
    case 14: KHO(CGB_A14, 14 - CGB_A14) break;
    case 15: KHO(7, 8) break;
    default: KHO(8, 8) break;
  }
#undef KHO
  return true;
}

static void keyswitch(cgb_ring *r, Scratch &S, const KsSrc &x, int count, u64 *const *d_keys, u64 *const *d_out,
                      const KsSrc &add0, const u64 *const *d_add1) {
  if (keyswitch_fused(r, S, x, count, d_keys, d_out, add0, d_add1)) return;
  if (keyswitch_fp(r, S, x, count, d_keys, d_out, add0, d_add1)) return;
  const int L = r->L, N = r->N, LP = L + 1, logN = r->logN;
  // digits in coefficient form (automorphism fused into the inverse NTT's load)
  u64 *xc = S.alloc<u64>((size_t)count * L * N);
  {
    NttJob job{};
    job.base = xc;
    job.item_stride = (u64)L * N;
    job.src_items = x.items;
    job.src_base = x.items ? nullptr : x.base;
    job.src_stride = x.stride;
    job.galois = x.g;
    const int off = (int)(x.items ? x.off / (u64)N : 0);
    for (int l = 0; l < L; l++) {
      job.sub_off[l] = (unsigned short)l;
      job.sub_mod[l] = (unsigned char)l;
      job.src_off[l] = (unsigned short)(off + l);
    }
    job.nsub = L;
    launch_ntt(r, false, job, count);
  }
  // ModUp: digit j centre-lifted into every other limb of Q u P, fused into the NTT load
  u64 *D = S.alloc<u64>((size_t)count * L * LP * N);
  u64 *acc = S.alloc<u64>((size_t)count * 2 * LP * N);
  {
    NttJob job{};
    job.base = D;
    job.item_stride = (u64)L * LP * N;
    job.src_base = xc;
    job.src_stride = (u64)L * N;
    job.lift = 1;
    int n = 0;
    for (int j = 0; j < L; j++)
      for (int l = 0; l < LP; l++) {
        if (l == j) continue;  // the digit's own limb is the NTT-form input itself
        job.sub_off[n] = (unsigned short)(j * LP + l);
        job.sub_mod[n] = (unsigned char)(l == L ? r->iP : l);
        job.src_off[n] = (unsigned short)j;
        job.src_mod[n] = (unsigned char)j;
        n++;
      }
    job.nsub = n;
    if (ks_row_fusable(r)) {
      launch_begin(r);
      modup_ks_row(r, job, count, acc, D, x, d_keys);
      r->launches++;  // two kernels
      // column pass (read digit + write D) + row pass (read D) + keys + digit's own limb + acc
      launch_end(r, "modup_ks_row", 24.0 * (double)count * n * N + BYTES_ks_inner - 8.0 * count * (double)n * N);
    } else {
      launch_ntt(r, true, job, count);
    }
  }
  // inner product with the evaluation key
  if (!ks_row_fusable(r)) {
    const int per_block = 16;
    const dim3 grid(GRID1((u64)LP * N, TPB).x, (count + per_block - 1) / per_block);
    const u64 kw = (u64)L * 2 * LP * N;
    launch_begin(r);
    switch (L) {
#define KSI(LL) case LL: k_ks_inner<LL><<<grid, TPB, 0, r->stream>>>(acc, D, x, d_keys, kw, r->d_mods, logN, count, per_block); break;
      KSI(1) KSI(2) KSI(3) KSI(4) KSI(5) KSI(6) KSI(7) KSI(8) KSI(9) KSI(10) KSI(11) KSI(12) KSI(13) KSI(14) KSI(15) KSI(16)
#undef KSI
      default: FAIL(CGB_ERR_PARAM, "unsupported limb count %d", L);
    }
    launch_end(r, "ks_inner", BYTES_ks_inner);
  }
  // ModDown: INTT the P limbs, centre-lift into Q (fused into the NTT load)
  {
    NttJob job{};
    job.base = acc;
    job.item_stride = 2ull * LP * N;
    job.sub_off[0] = (unsigned short)L;
    job.sub_mod[0] = (unsigned char)r->iP;
    job.sub_off[1] = (unsigned short)(LP + L);
    job.sub_mod[1] = (unsigned char)r->iP;
    job.nsub = 2;
    if (ks_row_fusable(r)) ntt_inv_col(r, job, count);  // row pass done by k_ks_row
    else launch_ntt(r, false, job, count);
  }
  u64 *W = S.alloc<u64>((size_t)count * 2 * L * N);
  {
    NttJob job{};
    job.base = W;
    job.item_stride = 2ull * L * N;
    job.src_base = acc;
    job.src_stride = 2ull * LP * N;
    job.lift = 1;
    int n = 0;
    for (int pp = 0; pp < 2; pp++)
      for (int l = 0; l < L; l++) {
        job.sub_off[n] = (unsigned short)(pp * L + l);
        job.sub_mod[n] = (unsigned char)l;
        job.src_off[n] = (unsigned short)(pp * LP + L);
        job.src_mod[n] = (unsigned char)r->iP;
        n++;
      }
    job.nsub = n;
    if (moddown_fusable(r)) {
      const MdEpi epi{d_out, acc, add0, d_add1, r->d_mods, r->d_c, L, logN};
      launch_begin(r);
      moddown_ntt_fused(r, job, count, epi);
      r->launches++;  // two kernels
      // column pass (read + write) + row pass reading W, then the combine's traffic without W
      launch_end(r, "ntt_fwd_moddown",
                 24.0 * (double)count * n * N + BYTES_moddown_combine - 8.0 * (double)count * 2 * L * N);
      return;
    }
    launch_ntt(r, true, job, count);
  }
  LAUNCH("moddown_combine", BYTES_moddown_combine,
         k_moddown_combine<<<dim3(GRID1(2ull * L * N, TPB).x, count), TPB, 0, r->stream>>>(
             d_out, acc, W, add0, d_add1, r->d_mods, r->d_c, L, logN));
}

// items per batched key switch (CGB_KS_CHUNK; 0 = as many as the workspace budget
// allows): smaller chunks keep a chunk's intermediates (xr, D, acc_P, W) L2-resident
// between the five launches
static int g_ks_chunk = 0;
// workspace bytes per chunk (CGB_WS_GIB): 6 GiB lets a decode wave's key switch run as
// ONE batch of up to 528 ciphertexts (3 GiB: 264) -- 76.3 -> 73.1 ms/token, fewer
// launch tails; 10 GiB measured the same
static size_t g_ws_bytes = (size_t)6 << 30;
static size_t chunk_for(cgb_ring *r, size_t words_per_item) {
  size_t budget = g_ws_bytes;
  size_t c = budget / std::max<size_t>(words_per_item * 8, 1);
  return std::max<size_t>(1, std::min<size_t>(c, 4096));
}

// galois (+ optional add of the input) on a batch
// key switch of `total` ciphertexts given by pointer (arena slots or scratch), Galois elements != 1
static void galois_ptrs(cgb_ring *r, int total, u64 *const *srcs, u64 *const *dsts, const u64 *gs, bool add_input) {
  const int L = r->L, N = r->N;
  const u64 ctw = r->ct_words;
  size_t per_item = ctw * 2 + (size_t)L * N * (1 + L * (L + 1) + 2 * (L + 1) + 2 * L);
  size_t CH = chunk_for(r, per_item);
  if (g_ks_chunk > 0) {  // at most g_ks_chunk items per batched key switch; equal-sized chunks
    const size_t nch = ((size_t)total + (size_t)g_ks_chunk - 1) / (size_t)g_ks_chunk;
    CH = std::min(CH, std::max<size_t>(1, ((size_t)total + nch - 1) / std::max<size_t>(nch, 1)));
  }
  for (size_t c0 = 0; c0 < (size_t)total; c0 += CH) {
    int n = (int)std::min(CH, (size_t)total - c0);
    Scratch S(r);
    std::vector<u64> g(gs + c0, gs + c0 + n);
    std::vector<u64 *> keys(n);
    for (int k = 0; k < n; k++) keys[k] = get_key(r, g[k]);
    std::vector<u64 *> src(srcs + c0, srcs + c0 + n), dst(dsts + c0, dsts + c0 + n);
    // sources shared by several items (one activation rotated by many steps): one ModUp each
    std::vector<u64> usrc;
    std::vector<u32> sidx(n);
    {
      std::unordered_map<u64, u32> seen;
      for (int k = 0; k < n; k++) {
        auto it = seen.emplace((u64)src[k], (u32)usrc.size());
        if (it.second) usrc.push_back((u64)src[k]);
        sidx[k] = it.first->second;
      }
    }
    const int nu = (int)usrc.size();
    const bool hoist = g_ks_hoist && 2 * nu <= n;
    // the per-item tables in ONE upload (host cost per wave is the critical path of small waves)
    const size_t nb = 4 * (size_t)n + (hoist ? (size_t)nu + ((size_t)n + 1) / 2 : 0);
    std::vector<u64> blob(nb);
    for (int k = 0; k < n; k++) {
      blob[k] = (u64)src[k];
      blob[n + k] = (u64)dst[k];
      blob[2 * n + k] = (u64)keys[k];
      blob[3 * n + k] = g[k];
    }
    if (hoist) {
      std::copy(usrc.begin(), usrc.end(), blob.begin() + 4 * (size_t)n);
      std::memcpy(blob.data() + 4 * (size_t)n + nu, sidx.data(), sizeof(u32) * (size_t)n);
    }
    u64 *d_blob = S.up(blob.data(), blob.size());
    u64 **d_src = reinterpret_cast<u64 **>(d_blob), **d_dst = reinterpret_cast<u64 **>(d_blob + n),
        **d_keys = reinterpret_cast<u64 **>(d_blob + 2 * n);
    u64 *d_g = d_blob + 3 * n;
    // c1' = sigma_g(c1) is read through the automorphism by the key switch; c0' by its epilogue
    KsSrc xin{nullptr, 0, d_src, (u64)L * N, d_g};
    KsSrc c0p{nullptr, 0, d_src, 0, d_g};
    const u64 *const *add1 = add_input ? (const u64 *const *)d_src : nullptr;
    // SURVEY 8(d) unit of a batched key switch: each input read once, each output
    // written once, each distinct evaluation key 2 dnum (L+K) N words read once
    double key_bytes = 0;
    if (r->timing_mode == 2) {
      std::vector<u64> gu(g);
      std::sort(gu.begin(), gu.end());
      key_bytes = (double)(std::unique(gu.begin(), gu.end()) - gu.begin()) * 8.0 * 2.0 * L * (L + 1.0) * N;
    }
    group_begin(r);
    const bool hoisted = hoist && keyswitch_hoisted(r, S, xin, n, nu, reinterpret_cast<u64 **>(d_blob + 4 * (size_t)n),
                                                    reinterpret_cast<const u32 *>(d_blob + 4 * (size_t)n + nu),
                                                    d_keys, d_dst, c0p, add1);
    if (!hoisted) keyswitch(r, S, xin, n, d_keys, d_dst, c0p, add1);
    group_end(r, hoisted ? "keyswitch_hoisted" : "keyswitch",
              8.0 * (double)ctw * ((hoisted ? nu : n) + n) + key_bytes);
  }
}

static void galois_batch(cgb_ring *r, int count, const u32 *a, const u64 *gs, const u32 *out, bool add_input) {
  const int L = r->L, N = r->N;
  const u64 twoN = 2ull * N, ctw = r->ct_words;
  std::vector<int> idx;  // items with g != 1
  for (int i = 0; i < count; i++) {
    u64 g = gs[i] % twoN;
    if (!(g & 1)) FAIL(CGB_ERR_PARAM, "Galois element %llu is even", (unsigned long long)gs[i]);
    if (g == 1) {
      Scratch S(r);
      std::vector<u64 *> src = ct_ptrs(r, 1, &a[i]), dst = ct_ptrs(r, 1, &out[i]);
      u64 **d_src = S.up(src.data(), 1), **d_dst = S.up(dst.data(), 1);
      launch_begin(r);
      if (add_input) {
        k_add<<<dim3(GRID1(ctw / 2, TPB).x, 1), TPB, 0, r->stream>>>(d_dst, (const u64 *const *)d_src,
                                                                 (const u64 *const *)d_src, r->d_mods, L, r->logN, ctw);
      } else {
        k_copy<<<dim3(GRID1(ctw / 2, TPB).x, 1), TPB, 0, r->stream>>>(d_dst, (const u64 *const *)d_src, ctw);
      }
      launch_end(r, add_input ? "add" : "copy", (add_input ? 24.0 : 16.0) * ctw);
    } else {
      idx.push_back(i);
    }
  }
  if (idx.empty()) return;
  std::vector<u32> ia(idx.size()), io(idx.size());
  std::vector<u64> g(idx.size());
  for (size_t k = 0; k < idx.size(); k++) {
    ia[k] = a[idx[k]];
    io[k] = out[idx[k]];
    g[k] = gs[idx[k]] % twoN;
  }
  std::vector<u64 *> src = ct_ptrs(r, (int)idx.size(), ia.data()), dst = ct_ptrs(r, (int)idx.size(), io.data());
  galois_ptrs(r, (int)idx.size(), src.data(), dst.data(), g.data(), add_input);
}

// ============================================================================
// key generation
// ============================================================================
// keys: one ChaCha20 key per item (device copy made here)
static void sample_cbd(cgb_ring *r, Scratch &S, i64 *e, const ChaKey *keys, const std::vector<u64> &nonces) {
  int n = (int)nonces.size();
  u64 *d_n = S.up(nonces.data(), n);
  ChaKey *d_k = S.up(keys, n);
  u64 nblk = ((u64)r->N + 7) / 8;
  LAUNCH("sample_cbd", BYTES_sample_cbd, k_sample_cbd<<<dim3(GRID1(nblk, 128).x, n), 128, 0, r->stream>>>(e, d_k, d_n, r->logN));
}
static void sample_uniform(cgb_ring *r, Scratch &S, u64 *const *d_dst, int n, const ChaKey *keys,
                           const std::vector<u64> &nonces, int nl, const int *mod_idx_host) {
  u64 *d_n = S.up(nonces.data(), n);
  ChaKey *d_k = S.up(keys, n);
  int *d_mi = S.up(mod_idx_host, nl);
  u64 nblk = ((u64)nl * r->N + 3) / 4;
  LAUNCH("sample_uniform", BYTES_sample_uniform, k_sample_uniform<<<dim3(GRID1(nblk, 128).x, n), 128, 0, r->stream>>>(d_dst, d_k, d_n, nl, d_mi, r->d_mods, r->logN));
}

static u64 *get_key(cgb_ring *r, u64 g) {
  auto it = r->keys.find(g);
  if (it != r->keys.end()) return it->second;
  const int L = r->L, LP = L + 1, N = r->N;
  const u64 LPN = (u64)LP * N;
  u64 *key;
  CK(cudaMalloc((void **)&key, 3 * sizeof(u64) * (size_t)L * 2 * LPN));  // values | Shoup companions | doubles
  Scratch S(r);
  std::vector<int> mi(LP);
  for (int l = 0; l < L; l++) mi[l] = l;
  mi[L] = r->iP;
  int *d_mi = S.up(mi.data(), LP);
  // source key s' over Q u P
  u64 *sp = S.alloc<u64>(LPN);
  launch_begin(r);
  if (g == 0) {
    k_square<<<GRID1(LPN, TPB), TPB, 0, r->stream>>>(sp, r->d_s, r->d_mods, LP, d_mi, r->logN);
  } else {
    k_automorph_flat<<<GRID1(LPN, TPB), TPB, 0, r->stream>>>(sp, r->d_s, g, LP, r->logN);
  }
  launch_end(r, "keygen", 16.0 * LPN);
  i64 *e = S.alloc<i64>((size_t)N);
  for (int j = 0; j < L; j++) {
    u64 sub = (g << 8) | (u64)j;
    std::vector<u64 *> adst = {key + ((u64)j * 2 + 1) * LPN};
    u64 **d_a = S.up(adst.data(), 1);
    sample_uniform(r, S, d_a, 1, &r->keyseed, {nonce_of(DOM_KSK_A, sub)}, LP, mi.data());
    sample_cbd(r, S, e, &r->keyseed, {nonce_of(DOM_KSK_E, sub)});
    LAUNCH("ksk_b", BYTES_ksk_b, k_ksk_b<<<GRID1(LPN, TPB), TPB, 0, r->stream>>>(key, j, e, r->d_s, sp, r->d_mods, r->d_c, L, r->iP, r->logN));
    ntt_items(r, true, key + ((u64)j * 2 + 0) * LPN, nullptr, 0, 1, 1, LP, mi.data());
    LAUNCH("ksk_fin", BYTES_ksk_fin, k_ksk_fin<<<GRID1(LPN, TPB), TPB, 0, r->stream>>>(key, j, r->d_s, sp, r->d_mods, r->d_c, L, r->iP, r->logN));
  }
  {
    const u64 words = (u64)L * 2 * LPN;
    LAUNCH("keygen", 0, k_key_shoup<<<GRID1(words, TPB), TPB, 0, r->stream>>>(key + words, key, r->d_mods, L, r->iP, r->logN, words));
    LAUNCH("keygen", 0, k_key_fp<<<GRID1(words, TPB), TPB, 0, r->stream>>>(key + 2 * words, key, words));
  }
  r->keys[g] = key;
  return key;
}

// ============================================================================
// ring construction
// ============================================================================
// largest primes below 2^bits with q = 1 mod 2^32 (hence mod 2N): the low word 1
// turns q-hat * q into one 32-bit multiply in every Shoup / Barrett reduction
static void take_primes(cgb_ring *r, int bits, int count) {
  u64 step = std::max<u64>(1ull << 32, 2ull * r->N), top = 1ull << bits;
  u64 c = top - (top % step) + 1;
  if (c >= top) c -= step;
  int got = 0;
  while (got < count) {
    bool dup = std::find(r->mods.begin(), r->mods.end(), c) != r->mods.end();
    if (!dup && c != r->t && h_prime(c)) {
      r->mods.push_back(c);
      got++;
    }
    c -= step;
  }
}

static void chacha_host(const ChaKey &key, u64 ctr, u64 nonce, u32 out[16]) {
  auto rotl = [](u32 x, int n) { return (x << n) | (x >> (32 - n)); };
  u32 s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u, key.k[0], key.k[1], key.k[2], key.k[3],
               key.k[4],    key.k[5],    key.k[6],    key.k[7],    (u32)ctr, (u32)(ctr >> 32), (u32)nonce,
               (u32)(nonce >> 32)};
  u32 x[16];
  memcpy(x, s, sizeof x);
  auto qr = [&](int a, int b, int c, int d) {
    x[a] += x[b]; x[d] ^= x[a]; x[d] = rotl(x[d], 16);
    x[c] += x[d]; x[b] ^= x[c]; x[b] = rotl(x[b], 12);
    x[a] += x[b]; x[d] ^= x[a]; x[d] = rotl(x[d], 8);
    x[c] += x[d]; x[b] ^= x[c]; x[b] = rotl(x[b], 7);
  };
  for (int i = 0; i < 10; i++) {
    qr(0, 4, 8, 12); qr(1, 5, 9, 13); qr(2, 6, 10, 14); qr(3, 7, 11, 15);
    qr(0, 5, 10, 15); qr(1, 6, 11, 12); qr(2, 7, 8, 13); qr(3, 4, 9, 14);
  }
  for (int i = 0; i < 16; i++) out[i] = x[i] + s[i];
}

static void build_ring(cgb_ring *r, const u32 key_seed[8]) {
  const int N = r->N, L = r->L, nB = r->nB, logN = r->logN;
  memcpy(r->keyseed.k, key_seed, sizeof r->keyseed.k);
  // q_bits <= 49: every prime < 2^q_bits (FP64-pipe NTT); otherwise P / B one bit wider
  const int pb = r->q_bits <= 49 ? r->q_bits : r->q_bits + 1;
  take_primes(r, r->q_bits, L);
  take_primes(r, pb, 1);
  take_primes(r, pb, nB);
  r->iP = L;
  r->iB0 = L + 1;
  r->iT = L + 1 + nB;
  for (u64 m : r->mods)
    if ((m & 0xffffffffull) != 1) FAIL(CGB_ERR_STATE, "modulus %llu is not 1 mod 2^32", (unsigned long long)m);
  r->fp_ntt = logN >= 12 && r->q_bits <= 49 && !getenv("CGB_INT_NTT");
  r->mods.push_back(r->t);
  r->nmod = (int)r->mods.size();
  // twiddle tables
  // tw | itw | tw1 | itw1 (u64 (w, w') pairs) | the same four as (w, w/q) doubles | ftw1 / fitw1 with
  // each row's levels >= 4 transposed ([j][blk]) for the register-I/O FP64 kernel (k_ntt2_fpr)
  size_t per = 22ull * N;  // + the w halves of the two transposed row tables
  CK(cudaMalloc((void **)&r->d_tables, sizeof(u64) * per * r->nmod));
  std::vector<u64> tab(per);
  r->h_mods.resize(r->nmod);
  for (int i = 0; i < r->nmod; i++) {
    u64 q = r->mods[i];
    u64 psi = h_psi(q, 2ull * N), psii = h_inv(psi, q);
    for (int k = 0; k < N; k++) {
      u32 b = h_brev((u32)k, logN);
      u64 w = h_powmod(psi, b, q), wi = h_powmod(psii, b, q);
      tab[2 * k] = w;  // (w, w') pairs: one 16-byte load per twiddle
      tab[2 * k + 1] = h_shoup(w, q);
      tab[2 * N + 2 * k] = wi;
      tab[2 * N + 2 * k + 1] = h_shoup(wi, q);
    }
    // two-pass row-tile order: entry blk*M + i (i = 2^sp + g) = pair 2^(a+sp) + blk 2^sp + g
    if (logN >= 12) {
      const int a = split_a(logN), b = logN - a, M = 1 << b;
      for (int blk = 0; blk < (1 << a); blk++)
        for (int ii = 0; ii < M; ii++) {
          size_t dst = (size_t)blk * M + ii, src = 0;
          if (ii) {
            int sp = 31 - __builtin_clz((unsigned)ii), gi = ii - (1 << sp);
            src = ((size_t)1 << (a + sp)) + ((size_t)blk << sp) + gi;
          }
          tab[4 * N + 2 * dst] = tab[2 * src];
          tab[4 * N + 2 * dst + 1] = tab[2 * src + 1];
          tab[6 * N + 2 * dst] = tab[2 * N + 2 * src];
          tab[6 * N + 2 * dst + 1] = tab[2 * N + 2 * src + 1];
        }
    }
    // FP64 copies: (double(w), double(w)/double(q)) in the same four orders
    for (int o = 0; o < 4; o++)
      for (int k = 0; k < N; k++) {
        const u64 w = tab[(size_t)o * 2 * N + 2 * k];
        double wd = (double)w, wq = wd / (double)q;
        memcpy(&tab[8ull * N + (size_t)o * 2 * N + 2 * k], &wd, 8);
        memcpy(&tab[8ull * N + (size_t)o * 2 * N + 2 * k + 1], &wq, 8);
      }
    if (logN >= 12) {
      const int M = 1 << (logN - split_a(logN));
      for (int o = 0; o < 2; o++)
        for (int row = 0; row < N / M; row++)
          for (int ii = 0; ii < M; ii++) {
            int pos = ii;
            if (ii >= 16) {
              const int sl = 31 - __builtin_clz((unsigned)ii), l = sl - 4, off = ii - (1 << sl);
              pos = (1 << sl) + ((off & ((1 << l) - 1)) << 4) + (off >> l);
            }
            const size_t from = 12ull * N + (size_t)o * 2 * N + 2ull * ((size_t)row * M + ii);
            const size_t to = 16ull * N + (size_t)o * 2 * N + 2ull * ((size_t)row * M + pos);
            tab[to] = tab[from];
            tab[to + 1] = tab[from + 1];
          }
    }
    for (int o = 0; o < 2; o++)
      for (int k = 0; k < N; k++) tab[20ull * N + (size_t)o * N + k] = tab[16ull * N + (size_t)o * 2 * N + 2ull * k];
    u64 *dt = r->d_tables + per * i;
    CK(cudaMemcpy(dt, tab.data(), sizeof(u64) * per, cudaMemcpyHostToDevice));
    ModTab &M = r->h_mods[i];
    M.q = q;
    int bits = 64 - __builtin_clzll(q);
    M.bits = bits;
    M.mu = (u64)((((u128)1) << (2 * bits)) / q);
    M.r64 = (u64)((((u128)1) << 64) % q);
    M.ninv = h_inv((u64)N % q, q);
    M.ninv_sh = h_shoup(M.ninv, q);
    {  // the inverse transform's stage-0 twiddle (pair index 1) times N^-1
      const u64 w0n = h_mulmod(tab[2ull * N + 2], M.ninv, q);
      M.itw0n_fp = (double)w0n;
      M.itw0n_fpq = (double)w0n / (double)q;
    }
    M.tw = dt;
    M.tw_sh = nullptr;
    M.itw = dt + 2 * N;
    M.itw_sh = nullptr;
    M.tw1 = dt + 4 * N;
    M.itw1 = dt + 6 * N;
    M.ftw = dt + 8 * N;
    M.fitw = dt + 10 * N;
    M.ftw1 = dt + 12 * N;
    M.fitw1 = dt + 14 * N;
    M.ftw1t = dt + 16 * N;
    M.fitw1t = dt + 18 * N;
    M.ftw1tw = dt + 20 * N;
    M.fitw1tw = dt + 21 * N;
    M.qd = (double)q;
    M.qinv = 1.0 / (double)q;
    M.ninv_fp = (double)M.ninv;
    M.ninv_fpq = (double)M.ninv / (double)q;
  }
  CK(cudaMalloc((void **)&r->d_mods, sizeof(ModTab) * r->nmod));
  CK(cudaMemcpy(r->d_mods, r->h_mods.data(), sizeof(ModTab) * r->nmod, cudaMemcpyHostToDevice));
  // slot map
  std::vector<u32> sidx(r->n_slots);
  u64 twoN = 2ull * N, e = 1;
  int h = r->one_row ? r->n_slots : r->n_slots / 2;
  for (int i = 0; i < h; i++) {
    sidx[i] = h_brev((u32)((e - 1) / 2), logN);
    if (!r->one_row) sidx[h + i] = h_brev((u32)((twoN - e - 1) / 2), logN);
    e = (e * 5) % twoN;
  }
  CK(cudaMalloc((void **)&r->d_slot_idx, sizeof(u32) * r->n_slots));
  CK(cudaMemcpy(r->d_slot_idx, sidx.data(), sizeof(u32) * r->n_slots, cudaMemcpyHostToDevice));
  // constants
  Consts &C = r->h_c;
  memset(&C, 0, sizeof C);
  C.L = L; C.nB = nB; C.N = N; C.logN = logN; C.n_slots = r->n_slots; C.t = r->t;
  const u64 *q = r->mods.data(), P = r->mods[r->iP], *b = r->mods.data() + r->iB0, t = r->t;
  C.Qmodt = 1;
  for (int l = 0; l < L; l++) C.Qmodt = h_mulmod(C.Qmodt, q[l] % t, t);
  for (int l = 0; l < L; l++) {
    C.tinvq[l] = h_inv(t % q[l], q[l]);
    C.Pmodq[l] = P % q[l];
    C.Pinvq[l] = h_inv(P % q[l], q[l]);
    C.Pinvq_sh[l] = h_shoup(C.Pinvq[l], q[l]);
    u64 qh = 1;
    for (int i = 0; i < L; i++)
      if (i != l) qh = h_mulmod(qh, q[i] % q[l], q[l]);
    C.QhatInv[l] = h_inv(qh, q[l]);
    u128 x = (u128)t * C.QhatInv[l];
    C.dec_omega[l] = (u64)(x / q[l]);
    h_frac128((u64)(x % q[l]), q[l], &C.dec_th_hi[l], &C.dec_th_lo[l]);
    C.invq[l] = 1.0 / (double)q[l];
    for (int k = 0; k < nB; k++) {
      u64 v = 1;
      for (int i = 0; i < L; i++)
        if (i != l) v = h_mulmod(v, q[i] % b[k], b[k]);
      C.QhatModB[l][k] = v;
    }
  }
  for (int k = 0; k < nB; k++) {
    u64 v = 1;
    for (int i = 0; i < L; i++) v = h_mulmod(v, q[i] % b[k], b[k]);
    C.QmodB[k] = v;
    u64 bh = 1;
    for (int i = 0; i < nB; i++)
      if (i != k) bh = h_mulmod(bh, b[i] % b[k], b[k]);
    C.BhatInv[k] = h_inv(bh, b[k]);
    C.tBhat[k] = h_mulmod(t % b[k], bh, b[k]);
    C.BQhatInv[k] = h_inv(h_mulmod(bh, v, b[k]), b[k]);
    C.invb[k] = 1.0 / (double)b[k];
    for (int l = 0; l < L; l++) {
      u64 w = 1;
      for (int i = 0; i < nB; i++)
        if (i != k) w = h_mulmod(w, b[i] % q[l], q[l]);
      C.BhatModQ[k][l] = w;
    }
  }
  for (int l = 0; l < L; l++) {
    u64 v = 1;
    for (int i = 0; i < nB; i++) v = h_mulmod(v, b[i] % q[l], q[l]);
    C.BmodQ[l] = v;
    u64 qh = 1;
    for (int i = 0; i < L; i++)
      if (i != l) qh = h_mulmod(qh, q[i] % q[l], q[l]);
    C.QBhatInv[l] = h_inv(h_mulmod(qh, v, q[l]), q[l]);
    Big T(t);
    for (int i = 0; i < nB; i++) T.mul(b[i]);
    u64 rem = T.divmod(q[l]);
    for (int k = 0; k < nB; k++) C.sc_omega[l][k] = T.mod(b[k]);
    h_frac128(rem, q[l], &C.sc_th_hi[l], &C.sc_th_lo[l]);
  }
  for (int l = 0; l < L; l++) {
    C.QhatInv_sh[l] = h_shoup(C.QhatInv[l], q[l]);
    C.QBhatInv_sh[l] = h_shoup(C.QBhatInv[l], q[l]);
    C.BmodQ_sh[l] = h_shoup(C.BmodQ[l], q[l]);
    for (int k = 0; k < nB; k++) {
      C.QhatModB_sh[l][k] = h_shoup(C.QhatModB[l][k], b[k]);
      C.sc_omega_sh[l][k] = h_shoup(C.sc_omega[l][k], b[k]);
      C.BhatModQ_sh[k][l] = h_shoup(C.BhatModQ[k][l], q[l]);
    }
  }
  for (int k = 0; k < nB; k++) {
    C.QmodB_sh[k] = h_shoup(C.QmodB[k], b[k]);
    C.BQhatInv_sh[k] = h_shoup(C.BQhatInv[k], b[k]);
    C.tBhat_sh[k] = h_shoup(C.tBhat[k], b[k]);
    C.BhatInv_sh[k] = h_shoup(C.BhatInv[k], b[k]);
  }
  auto fw = [](u64 w, u64 m) { return make_double2((double)w, (double)w / (double)m); };
  for (int l = 0; l < L; l++) {
    C.fQhatInv[l] = fw(C.QhatInv[l], q[l]);
    C.fQBhatInv[l] = fw(C.QBhatInv[l], q[l]);
    C.fBmodQ[l] = fw(C.BmodQ[l], q[l]);
    for (int k = 0; k < nB; k++) {
      C.fQhatModB[l][k] = fw(C.QhatModB[l][k], b[k]);
      C.fsc_omega[l][k] = fw(C.sc_omega[l][k], b[k]);
      C.fBhatModQ[k][l] = fw(C.BhatModQ[k][l], q[l]);
    }
  }
  for (int l = 0; l < L; l++) C.fPinvq[l] = fw(C.Pinvq[l], q[l]);
  for (int l = 0; l < L; l++) C.fPmodq[l] = fw(C.Pmodq[l], q[l]);
  for (int k = 0; k < nB; k++) {
    C.fQmodB[k] = fw(C.QmodB[k], b[k]);
    C.fBQhatInv[k] = fw(C.BQhatInv[k], b[k]);
    C.ftBhat[k] = fw(C.tBhat[k], b[k]);
    C.fBhatInv[k] = fw(C.BhatInv[k], b[k]);
  }
  CK(cudaMalloc((void **)&r->d_c, sizeof(Consts)));
  CK(cudaMemcpy(r->d_c, &C, sizeof(Consts), cudaMemcpyHostToDevice));
  // secret key: ternary from ChaCha20(key_seed, DOM_SK), word j -> (w mod 3) - 1
  std::vector<u64> s((size_t)(L + 1) * N);
  u32 blk[16];
  for (int j = 0; j < N; j++) {
    if (j % 16 == 0) chacha_host(r->keyseed, (u64)(j / 16), nonce_of(DOM_SK, 0), blk);
    int sv = (int)(blk[j % 16] % 3) - 1;
    for (int l = 0; l <= L; l++) {
      u64 qq = r->mods[l == L ? r->iP : l];
      s[(size_t)l * N + j] = sv >= 0 ? (u64)sv : qq - 1;
    }
  }
  CK(cudaMalloc((void **)&r->d_s, sizeof(u64) * s.size()));
  CK(cudaMemcpy(r->d_s, s.data(), sizeof(u64) * s.size(), cudaMemcpyHostToDevice));
  std::vector<int> mi(L + 1);
  for (int l = 0; l < L; l++) mi[l] = l;
  mi[L] = r->iP;
  ntt_items(r, true, r->d_s, nullptr, 0, 1, 1, L + 1, mi.data());
  CK(cudaStreamSynchronize(r->stream));
}

// ============================================================================
// C ABI
// ============================================================================
// the tensor product and its inverse NTT in two launches: the row pass computes the
// products in its load (TensorLoad), the column pass finishes the transform into ten
// measured slower: tensor_intt 6.46 ms against tensor 2.43 + its inverse transform
// 3.71 ms per decode step (the integer products in the row pass's load sit on its
// critical path); off (CGB_TENSOR_FUSE=1 turns it on)
static bool g_tensor_fuse = false;
template <int LA, int LB>
static void tensor_intt_t(cgb_ring *r, int n, u64 *ten, const TensorLoad &tl, const int *mod_of_limb) {
  const int nt = tl.nt;
  NttJob job{};
  job.base = ten;
  job.item_stride = 3ull * nt * r->N;
  int u = 0;
  for (int k = 0; k < 3; k++)
    for (int l = 0; l < nt; l++) {
      job.sub_off[u] = (unsigned short)(k * nt + l);
      job.sub_mod[u] = (unsigned char)mod_of_limb[l];
      u++;
    }
  job.nsub = u;
  job.mods = r->d_mods;
  job.logN = r->logN;
  auto grid = [&](int lm) {
    int nsubs = 1 << (LA + LB - lm), G = NTT2_TILE / (1 << lm);
    return dim3((unsigned)((size_t)n * job.nsub * (nsubs / G)));
  };
  static std::once_flag once;
  std::call_once(once, [] {
    CK(cudaFuncSetAttribute(k_ntt2_fpr<LA, LB, false, 1, TensorLoad>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)fpr_smem_bytes<LA, LB>(1)));
  });
  NttJob first = job, second = job;
  first.out_raw = 1;  // the words between the passes stay reduced doubles
  second.in_raw = 1;
  launch_begin(r);
  launch_pdl(r, k_ntt2_fpr<LA, LB, false, 1, TensorLoad>, grid(LB), NTT2_TILE / 16, fpr_smem_bytes<LA, LB>(1), first, tl);
  launch_pdl(r, k_ntt2_fpr<LA, LB, false, 0>, grid(LA), NTT2_TILE / 16, fpr_smem_bytes<LA, LB>(0), second, NoEpi{});
  r->launches++;  // two kernels (launch_end counts the other)
  const double words = (double)n * job.nsub * r->N;
  // operands read (4 limb-polys of a and b per limb), the tensor's transform written once
  launch_end(r, "tensor_intt", 8.0 * (double)n * nt * r->N * 4.0 + 8.0 * words, words / 2.0 * r->logN);
}
static bool tensor_intt_fused(cgb_ring *r, int n, u64 *ten, const TensorLoad &tl, const int *mod_of_limb) {
  if (!(g_tensor_fuse && r->fp_ntt && (g_fp_regio & 3) == 3 && r->logN >= 13 && r->logN <= 16)) return false;
  switch (r->logN) {
    case 13: tensor_intt_t<6, 7>(r, n, ten, tl, mod_of_limb); break;
    case 14: tensor_intt_t<CGB_A14, 14 - CGB_A14>(r, n, ten, tl, mod_of_limb); break;
    case 15: tensor_intt_t<7, 8>(r, n, ten, tl, mod_of_limb); break;
    default: tensor_intt_t<8, 8>(r, n, ten, tl, mod_of_limb); break;
  }
  return true;
}
extern "C" {

const char *cgb_last_error(void) { return g_err.c_str(); }

int cgb_ring_create(int log_n, uint64_t plain_modulus, int n_limbs, int n_slots, int one_row,
                    const uint32_t key_seed[8], int64_t arena_cts, int64_t arena_pts, cgb_ring **out) {
  return cgb_ring_create_ex(log_n, plain_modulus, n_limbs, 60, n_slots, one_row, key_seed, arena_cts, arena_pts, out);
}

int cgb_ring_create_ex(int log_n, uint64_t plain_modulus, int n_limbs, int q_bits, int n_slots, int one_row,
                       const uint32_t key_seed[8], int64_t arena_cts, int64_t arena_pts, cgb_ring **out) {
  API_BEGIN
  if (q_bits < 40 || q_bits > 60) FAIL(CGB_ERR_PARAM, "q_bits %d outside [40, 60]", q_bits);
  if (log_n < 2 || log_n > 16) FAIL(CGB_ERR_PARAM, "log_n %d outside [2, 16]", log_n);
  if (n_limbs < 1 || n_limbs > MAXL) FAIL(CGB_ERR_PARAM, "n_limbs %d outside [1, %d]", n_limbs, MAXL);
  u64 N = 1ull << log_n;
  if (plain_modulus < 3 || plain_modulus >= (1ull << 31) || plain_modulus % (2 * N) != 1)
    FAIL(CGB_ERR_PARAM, "plain modulus %llu must be < 2^31 and = 1 mod 2N = %llu",
         (unsigned long long)plain_modulus, (unsigned long long)(2 * N));
  if (one_row ? (u64)n_slots * 2 != N : (u64)n_slots != N)
    FAIL(CGB_ERR_PARAM, "n_slots %d does not match ring degree %llu (one_row=%d)", n_slots, (unsigned long long)N,
         one_row);
  cgb_ring *r = new cgb_ring();
  r->q_bits = q_bits;
  r->logN = log_n;
  r->N = (int)N;
  r->L = n_limbs;
  r->nB = n_limbs + 1;
  r->t = plain_modulus;
  r->n_slots = n_slots;
  r->one_row = one_row;
  CK(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
  r->own_stream = true;
  {
    int dev;
    CK(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = UINT64_MAX;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    // kernel attributes are process-global: size the single-kernel NTT for the
    // largest ring it serves (log N <= 11), once
    static std::once_flag attrs_once;
    std::call_once(attrs_once, [] {
      const size_t smem = sizeof(u64) * (size_t)((1 << 11) + (1 << 7) + 1);
#define SETSMEM(EE)                                                                                           \
  CK(cudaFuncSetAttribute(k_ntt<EE, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));  \
  CK(cudaFuncSetAttribute(k_ntt<EE, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
  CK(cudaFuncSetAttribute(k_ntt<EE, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
  CK(cudaFuncSetAttribute(k_ntt<EE, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      SETSMEM(32) SETSMEM(16) SETSMEM(8) SETSMEM(4) SETSMEM(2)
    });
#undef SETSMEM
    switch (log_n) {
      case 12: ntt2_attrs<6, 6>(); break;
      case 13: ntt2_attrs<6, 7>(); break;
      case 14: ntt2_attrs<CGB_A14, 14 - CGB_A14>(); break;
      case 15: ntt2_attrs<7, 8>(); break;
      case 16: ntt2_attrs<8, 8>(); break;
      default: break;
    }
  }
  if (const char *e = getenv("CGB_NTT_E")) g_ntt2_e = atoi(e) == 16 ? 16 : 8;
  if (const char *e = getenv("CGB_FP_REGIO")) g_fp_regio = atoi(e) & 3;
  if (const char *e = getenv("CGB_MD_EPI")) g_md_epi = atoi(e) != 0;
  if (const char *e = getenv("CGB_KS_ROW")) g_ks_row = atoi(e) != 0;
  if (const char *e = getenv("CGB_COL_FUSED")) g_col_fused = atoi(e) != 0;
  if (const char *e = getenv("CGB_KS_FUSED")) g_ks_fused = atoi(e);
  if (const char *e = getenv("CGB_PDL")) g_pdl = atoi(e) != 0;
  if (const char *e = getenv("CGB_KS_MD")) g_ks_md = atoi(e) != 0;
  if (const char *e = getenv("CGB_KS_HOIST")) g_ks_hoist = atoi(e) != 0;
  if (const char *e = getenv("CGB_TENSOR_FUSE")) g_tensor_fuse = atoi(e) != 0;
  if (const char *e = getenv("CGB_KS_CHUNK")) g_ks_chunk = atoi(e);
  if (const char *e = getenv("CGB_KSROW8")) g_ksrow8 = atoi(e) != 0;
  if (const char *e = getenv("CGB_KSROW2")) g_ksrow2 = atoi(e);
  if (const char *e = getenv("CGB_COL_UNRED")) g_col_unred = atoi(e) != 0;
  if (const char *e = getenv("CGB_KSROW2_SPEC")) g_ksrow2_spec = atoi(e) != 0;
#if !CGB_BUILD_FALLBACKS  // the superseded variants are not in this build
  g_ks_md = true;
  g_ksrow2 = 1;
  g_ksrow8 = false;
#endif
  if (const char *e = getenv("CGB_TENSOR_FP")) g_tensor_fp = atoi(e) != 0;
  if (const char *e = getenv("CGB_WS_GIB")) g_ws_bytes = (size_t)(atof(e) * (double)(1ull << 30));
  if (const char *e = getenv("CGB_HOIST_FUSE")) g_hoist_fuse = atoi(e) != 0;
  if (const char *e = getenv("CGB_FP_BCONV")) g_fp_bconv = atoi(e) != 0;
  fused_attrs_for(log_n, n_limbs);
  r->pin_cap = (log_n >= 13 ? 128ull : 8ull) << 20;
  CK(cudaMallocHost((void **)&r->pin, r->pin_cap));
  if (const char *e = getenv("CGB_SIDE_COPY")) g_side_copy = atoi(e) != 0;
  if (g_side_copy) {
    CK(cudaMalloc((void **)&r->dev_stage, r->pin_cap));
    CK(cudaStreamCreateWithFlags(&r->copy_stream, cudaStreamNonBlocking));
  }
  build_ring(r, key_seed);
  r->ct_words = 2ull * r->L * r->N;
  r->arena_cap = (size_t)std::max<int64_t>(arena_cts, 1);
  CK(cudaMalloc((void **)&r->arena, sizeof(u64) * r->ct_words * r->arena_cap));
  r->ct_used.assign(r->arena_cap, 0);
  for (size_t i = r->arena_cap; i-- > 0;) r->ct_free.push_back((u32)i);
  r->pt_cap = (size_t)std::max<int64_t>(arena_pts, 1);
  CK(cudaMalloc((void **)&r->pt_arena, sizeof(u64) * (size_t)r->L * r->N * r->pt_cap));
  r->pt_used.assign(r->pt_cap, 0);
  for (size_t i = r->pt_cap; i-- > 0;) r->pt_free.push_back((u32)i);
  *out = r;
  API_END
}

void cgb_ring_destroy(cgb_ring *r) {
  if (!r) return;
  cudaStreamSynchronize(r->stream);
  for (auto &kv : r->keys) cudaFree(kv.second);
  cudaFree(r->arena);
  cudaFree(r->pt_arena);
  cudaFree(r->d_tables);
  cudaFree(r->d_mods);
  cudaFree(r->d_slot_idx);
  cudaFree(r->d_s);
  cudaFree(r->d_c);
  cudaFreeHost(r->pin);
  cudaFree(r->dev_stage);
  if (r->copy_stream) cudaStreamDestroy(r->copy_stream);
  for (auto e : r->copy_ev) cudaEventDestroy(e);
  for (auto &b : r->dec_pool) cudaFreeHost(b.second);
  for (auto e : r->pin_left)
    if (e) cudaEventDestroy(e);
  if (r->own_stream) cudaStreamDestroy(r->stream);
  delete r;
}

int cgb_ring_moduli(const cgb_ring *r, uint64_t *out, int cap) {
  int n = std::min(cap, r->iT);
  for (int i = 0; i < n; i++) out[i] = r->mods[i];
  return n;
}
size_t cgb_ct_words(const cgb_ring *r) { return r->ct_words; }
uint64_t cgb_launch_count(const cgb_ring *r) { return r->launches; }

int cgb_modmul_peak(cgb_ring *r, double *modmuls_per_s) {
  API_BEGIN
  RING_LOCK(r);
  u64 q = r->mods[0], w = r->mods[0] / 3 + 7, wsh = h_shoup(w, q);
  u64 *sink;
  CK(cudaMallocAsync((void **)&sink, 8, r->stream));
  int dev, sms;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int threads = 512, blocks = sms * 4, iters = 4096;
  const double qd = (double)q, wd = (double)w, wq = wd / qd;
  // the pipe this ring's NTT runs on: FP64 exact products or 64-bit Shoup products
  auto run = [&](int n) {
    if (r->fp_ntt) k_modmul_peak_fp<<<blocks, threads, 0, r->stream>>>(sink, qd, wd, wq, n);
    else k_modmul_peak<<<blocks, threads, 0, r->stream>>>(sink, q, w, wsh, n);
  };
  run(64);  // warm-up
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, r->stream));
  run(iters);
  CK(cudaEventRecord(b, r->stream));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  CK(cudaFreeAsync(sink, r->stream));
  *modmuls_per_s = (double)blocks * threads * 8.0 * iters / (ms * 1e-3);
  API_END
}

// ---- kernel microbenchmarks -------------------------
// `iters` back-to-back batched transforms of count ciphertexts (2 L limb-polys
// each) on scratch data; returns the average milliseconds per batch.
int cgb_bench_ntt(cgb_ring *r, int count, int fwd, int iters, double *ms_out) {
  API_BEGIN
  RING_LOCK(r);
  const int L = r->L, N = r->N;
  Scratch S(r);
  u64 *buf = S.alloc<u64>((size_t)count * 2 * L * N);
  CK(cudaMemsetAsync(buf, 0, sizeof(u64) * (size_t)count * 2 * L * N, r->stream));
  std::vector<int> qm;
  q_mod_idx(r, qm);
  ntt_items(r, fwd != 0, buf, nullptr, 2ull * L * N, count, 2, L, qm.data());  // warm-up
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(a, r->stream));
  for (int i = 0; i < iters; i++) ntt_items(r, fwd != 0, buf, nullptr, 2ull * L * N, count, 2, L, qm.data());
  CK(cudaEventRecord(b, r->stream));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  *ms_out = ms / iters;
  API_END
}

int cgb_timing_enable(cgb_ring *r, int on) {
  API_BEGIN
  RING_LOCK(r);
  CK(cudaStreamSynchronize(r->stream));
  for (auto &rc : r->recs) {
    r->event_pool.push_back(rc.a);
    r->event_pool.push_back(rc.b);
  }
  r->recs.clear();
  r->timing = on != 0;
  r->timing_mode = on;
  r->group_depth = 0;
  API_END
}

int cgb_timing_report(cgb_ring *r, char *buf, size_t cap) {
  API_BEGIN
  RING_LOCK(r);
  CK(cudaStreamSynchronize(r->stream));
  struct Agg {
    long n = 0;
    double ms = 0, bytes = 0, mm = 0;
  };
  std::vector<std::pair<std::string, Agg>> agg;
  for (auto &rc : r->recs) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, rc.a, rc.b));
    auto it = std::find_if(agg.begin(), agg.end(), [&](auto &kv) { return kv.first == rc.name; });
    if (it == agg.end()) {
      agg.push_back({rc.name, Agg{}});
      it = agg.end() - 1;
    }
    it->second.n++;
    it->second.ms += ms;
    it->second.bytes += rc.bytes;
    it->second.mm += rc.mm;
  }
  // GPU idle time between consecutive recorded launches (host gaps, syncs)
  double idle = 0;
  std::vector<std::pair<float, size_t>> gaps;
  for (size_t i = 1; i < r->recs.size(); i++) {
    float g = 0;
    CK(cudaEventElapsedTime(&g, r->recs[i - 1].b, r->recs[i].a));
    if (g > 0) {
      idle += g;
      gaps.push_back({g, i});
    }
  }
  agg.push_back({"(idle)", Agg{}});
  agg.back().second.n = (long)r->recs.size();
  agg.back().second.ms = idle;
  std::sort(gaps.begin(), gaps.end(), [](auto &x, auto &y) { return x.first > y.first; });
  for (size_t k = 0; k < std::min<size_t>(5, gaps.size()); k++) {
    char nm[96];
    snprintf(nm, sizeof nm, "(gap%zu:%s->%s)", k, r->recs[gaps[k].second - 1].name, r->recs[gaps[k].second].name);
    agg.push_back({nm, Agg{}});
    agg.back().second.n = (long)gaps[k].second;
    agg.back().second.ms = gaps[k].first;
  }
  // idle per (previous -> next) launch-name transition, largest totals first
  {
    std::vector<std::pair<std::string, Agg>> tr;
    for (auto &gp : gaps) {
      std::string k = std::string("(trans:") + r->recs[gp.second - 1].name + "->" + r->recs[gp.second].name + ")";
      auto it = std::find_if(tr.begin(), tr.end(), [&](auto &kv) { return kv.first == k; });
      if (it == tr.end()) {
        tr.push_back({k, Agg{}});
        it = tr.end() - 1;
      }
      it->second.n++;
      it->second.ms += gp.first;
    }
    std::sort(tr.begin(), tr.end(), [](auto &x, auto &y) { return x.second.ms > y.second.ms; });
    for (size_t k = 0; k < std::min<size_t>(10, tr.size()); k++) agg.push_back(tr[k]);
  }
  std::string out;
  for (auto &kv : agg) {
    char line[256];
    snprintf(line, sizeof line, "%s %ld %.6f %.0f %.0f\n", kv.first.c_str(), kv.second.n, kv.second.ms,
             kv.second.bytes, kv.second.mm);
    out += line;
  }
  if (out.size() + 1 > cap) FAIL(CGB_ERR_PARAM, "timing report needs %zu bytes", out.size() + 1);
  memcpy(buf, out.c_str(), out.size() + 1);
  API_END
}

int cgb_set_stream(cgb_ring *r, void *s) {
  API_BEGIN
  RING_LOCK(r);
  CK(cudaStreamSynchronize(r->stream));
  if (r->own_stream) cudaStreamDestroy(r->stream);
  r->stream = (cudaStream_t)s;
  r->own_stream = false;
  API_END
}
int cgb_sync(cgb_ring *r) {
  API_BEGIN
  RING_LOCK(r);
  CK(cudaStreamSynchronize(r->stream));
  API_END
}

int cgb_ct_alloc(cgb_ring *r, int count, uint32_t *ids) {
  API_BEGIN
  RING_LOCK(r);
  std::lock_guard<std::mutex> g(r->mu);
  if ((size_t)count > r->ct_free.size())
    FAIL(CGB_ERR_NOMEM, "ciphertext arena exhausted (%zu slots)", r->arena_cap);
  for (int i = 0; i < count; i++) {
    ids[i] = r->ct_free.back();
    r->ct_free.pop_back();
    r->ct_used[ids[i]] = 1;
  }
  API_END
}
int cgb_ct_free(cgb_ring *r, int count, const uint32_t *ids) {
  API_BEGIN
  RING_LOCK(r);
  std::lock_guard<std::mutex> g(r->mu);
  for (int i = 0; i < count; i++) {
    if (ids[i] >= r->arena_cap || !r->ct_used[ids[i]]) FAIL(CGB_ERR_PARAM, "double free of ciphertext %u", ids[i]);
    r->ct_used[ids[i]] = 0;
    r->ct_free.push_back(ids[i]);
  }
  API_END
}
uint64_t *cgb_ct_device_ptr(cgb_ring *r, uint32_t id) { return r->arena + (size_t)id * r->ct_words; }
int64_t cgb_ct_free_count(cgb_ring *r) {
  std::lock_guard<std::mutex> g(r->mu);
  return (int64_t)r->ct_free.size();
}

int cgb_pt_alloc(cgb_ring *r, int count, uint32_t *ids) {
  API_BEGIN
  RING_LOCK(r);
  std::lock_guard<std::mutex> g(r->mu);
  if ((size_t)count > r->pt_free.size()) FAIL(CGB_ERR_NOMEM, "plaintext arena exhausted (%zu slots)", r->pt_cap);
  for (int i = 0; i < count; i++) {
    ids[i] = r->pt_free.back();
    r->pt_free.pop_back();
    r->pt_used[ids[i]] = 1;
  }
  API_END
}
int cgb_pt_free(cgb_ring *r, int count, const uint32_t *ids) {
  API_BEGIN
  RING_LOCK(r);
  std::lock_guard<std::mutex> g(r->mu);
  for (int i = 0; i < count; i++) {
    if (ids[i] >= r->pt_cap || !r->pt_used[ids[i]]) FAIL(CGB_ERR_PARAM, "double free of plaintext %u", ids[i]);
    r->pt_used[ids[i]] = 0;
    r->pt_free.push_back(ids[i]);
  }
  API_END
}

int cgb_ct_copy(cgb_ring *r, int count, const uint32_t *src, const uint32_t *dst) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  Scratch S(r);
  auto ps = ct_ptrs(r, count, src), pd = ct_ptrs(r, count, dst);
  u64 **ds = S.up(ps.data(), count), **dd = S.up(pd.data(), count);
  LAUNCH("copy", BYTES_copy, k_copy<<<dim3(GRID1(r->ct_words / 2, TPB).x, count), TPB, 0, r->stream>>>(dd, (const u64 *const *)ds, r->ct_words));
  API_END
}
int cgb_ct_store(cgb_ring *r, int count, const uint32_t *ids, uint64_t *host) {
  API_BEGIN
  RING_LOCK(r);
  for (int i = 0; i < count; i++) {
    auto p = ct_ptrs(r, 1, &ids[i]);
    CK(cudaMemcpyAsync(host + (size_t)i * r->ct_words, p[0], sizeof(u64) * r->ct_words, cudaMemcpyDeviceToHost,
                       r->stream));
  }
  CK(cudaStreamSynchronize(r->stream));
  API_END
}
int cgb_ct_load(cgb_ring *r, int count, const uint32_t *ids, const uint64_t *host) {
  API_BEGIN
  RING_LOCK(r);
  for (int i = 0; i < count; i++) {
    auto p = ct_ptrs(r, 1, &ids[i]);
    CK(cudaMemcpyAsync(p[0], host + (size_t)i * r->ct_words, sizeof(u64) * r->ct_words, cudaMemcpyHostToDevice,
                       r->stream));
  }
  CK(cudaStreamSynchronize(r->stream));
  API_END
}

// plaintext polys m[count][N] (coefficient form mod t) -> encoded plaintexts of `kind`
static void pt_from_coeffs(cgb_ring *r, Scratch &S, const u64 *m, int count, int kind, const uint32_t *pt_ids) {
  auto pp = pt_ptrs(r, count, pt_ids);
  u64 **dp = S.up(pp.data(), count);
  u64 words = (u64)r->L * r->N;
  LAUNCH("pt_lift", BYTES_pt_lift, k_pt_lift<<<dim3(GRID1(words, TPB).x, count), TPB, 0, r->stream>>>(dp, m, r->d_mods, r->d_c, r->L, r->logN, kind));
  std::vector<int> qm;
  ntt_items(r, true, nullptr, dp, 0, count, 1, r->L, q_mod_idx(r, qm));
}
int cgb_pt_encode(cgb_ring *r, int count, const uint64_t *slots, int kind, const uint32_t *pt_ids) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  if (kind != CGB_PT_MUL && kind != CGB_PT_ADD) FAIL(CGB_ERR_PARAM, "unknown plaintext kind %d", kind);
  Scratch S(r);
  u64 *m = S.alloc<u64>((size_t)count * r->N);
  encode_slots(r, S, slots, count, m);
  pt_from_coeffs(r, S, m, count, kind, pt_ids);
  API_END
}

// device slot vectors (residues mod t) -> coefficient-form plaintext polys; neg: (t - s) mod t
__global__ void k_scatter_slots_dev(u64 *m, const u64 *slots, const u32 *slot_idx, int n, u64 t, int logN, int neg) {
  int item = blockIdx.y;
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u64 v = slots[(u64)item * n + i];
  m[((u64)item << logN) + slot_idx[i]] = neg ? (v ? t - v : 0) : v;
}

int cgb_mask_pcg64(cgb_ring *r, int count, int nchan, const int32_t *chan, uint64_t *st, const uint32_t *pt_neg,
                   const uint32_t *pt_pos, uint64_t *masks_out) {
  API_BEGIN
  RING_LOCK(r);
  using namespace cgbmask;
  if (count <= 0) return CGB_OK;
  if (nchan <= 0 || r->t >= (1ull << 32)) FAIL(CGB_ERR_PARAM, "mask stream: %d channels, bound %llu", nchan,
                                               (unsigned long long)r->t);
  const int n = r->n_slots;
  const u32 p = (u32)r->t, thr = (u32)((0x100000000ull - p) % p);
  std::vector<std::vector<u32>> per(nchan);
  for (int i = 0; i < count; i++) {
    if (chan[i] < 0 || chan[i] >= nchan) FAIL(CGB_ERR_PARAM, "item %d: channel %d out of range", i, chan[i]);
    per[chan[i]].push_back((u32)i);
  }
  std::vector<u32> items;
  std::vector<Chan> C(nchan);
  for (int c = 0; c < nchan; c++) {
    C[c].state = {st[6 * c + 0], st[6 * c + 1]};
    C[c].inc = {st[6 * c + 2], st[6 * c + 3]};
    C[c].has_u32 = (u32)st[6 * c + 4];
    C[c].uinteger = (u32)st[6 * c + 5];
    C[c].item0 = items.size();
    C[c].need = (u64)per[c].size() * n;
    items.insert(items.end(), per[c].begin(), per[c].end());
  }
  Scratch S(r);
  u64 *slots = S.alloc<u64>((size_t)count * n);
  u32 *d_items = S.up(items.data(), items.size());
  std::vector<long long> last(nchan);
  // the stream is cut with a margin over the expected 1/(1 - 2^-3) draws per accepted
  // value (rejection rate (2^32 mod p) / 2^32 < 1/8 for p > 2^29); cut again, longer,
  // in the (never observed) case it falls short
  for (double margin = 1.25;; margin *= 1.5) {
    std::vector<u64> tb(nchan + 1, 0);
    u64 total = 0;
    for (int c = 0; c < nchan; c++) {
      const u64 outs = ((u64)((double)C[c].need * margin / 2.0) + 1024 + GEN_CHUNK - 1) / GEN_CHUNK * GEN_CHUNK;
      C[c].base = total;
      C[c].halves = C[c].has_u32 + 2 * outs;
      total += C[c].halves;
      tb[c + 1] = tb[c] + outs / GEN_CHUNK;
    }
    Chan *d_ch = S.up(C.data(), C.size());
    u64 *d_tb = S.up(tb.data(), tb.size());
    u32 *val = S.alloc<u32>(total), *flag = S.alloc<u32>(total), *idx = S.alloc<u32>(total);
    long long *d_last = S.alloc<long long>(nchan);
    CK(cudaMemsetAsync(d_last, 0xff, sizeof(long long) * nchan, r->stream));
    LAUNCH("mask_gen", 8.0 * (double)total,
           k_pcg_gen<<<(unsigned)((tb[nchan] + 127) / 128), 128, 0, r->stream>>>(d_ch, nchan, d_tb, val, flag, p, thr));
    size_t tmp_bytes = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flag, idx, (int)total, r->stream));
    void *tmp = S.alloc<char>(tmp_bytes);
    CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flag, idx, (int)total, r->stream));
    LAUNCH("mask_scatter", 12.0 * (double)total + 8.0 * count * n,
           k_pcg_scatter<<<(unsigned)((total + 255) / 256), 256, 0, r->stream>>>(d_ch, nchan, idx, val, flag, total, d_items, n, slots, d_last));
    CK(cudaMemcpyAsync(last.data(), d_last, sizeof(long long) * nchan, cudaMemcpyDeviceToHost, r->stream));
    CK(cudaStreamSynchronize(r->stream));
    bool ok = true;
    for (int c = 0; c < nchan; c++) ok = ok && (C[c].need == 0 || last[c] >= 0);
    if (ok) break;
    if (margin > 8) FAIL(CGB_ERR_STATE, "mask stream too short");
  }
  // the channels' generator states after the draws (numpy's PCG64 state layout)
  for (int c = 0; c < nchan; c++) {
    if (C[c].need == 0) continue;
    const long long lh = last[c];
    // numpy keeps the high half of the last split output in `uinteger` (buffered when
    // its low half was the last word consumed, stale but kept otherwise)
    u64 steps = 0, has = 0, uint = st[6 * c + 5];
    if (!(C[c].has_u32 && lh == 0)) {
      const u64 k = (u64)lh - C[c].has_u32;  // index among the 64-bit outputs' halves
      steps = k / 2 + 1;
      has = (k & 1) ? 0 : 1;
      uint = pcg_output(pcg_advance(C[c].state, C[c].inc, steps)) >> 32;
    }
    const U128 ns = pcg_advance(C[c].state, C[c].inc, steps);
    st[6 * c + 0] = ns.hi;
    st[6 * c + 1] = ns.lo;
    st[6 * c + 4] = has;
    st[6 * c + 5] = uint;
  }
  u64 *m = S.alloc<u64>((size_t)count * r->N);
  for (int neg = 0; neg < 2; neg++) {
    const uint32_t *ids = neg ? pt_neg : pt_pos;
    if (!ids) continue;
    CK(cudaMemsetAsync(m, 0, sizeof(u64) * (size_t)count * r->N, r->stream));
    LAUNCH("scatter_slots", BYTES_scatter_slots,
           k_scatter_slots_dev<<<dim3(GRID1(n, TPB).x, count), TPB, 0, r->stream>>>(m, slots, r->d_slot_idx, n, r->t,
                                                                                   r->logN, neg));
    int mi = r->iT;
    ntt_items(r, false, m, nullptr, r->N, count, 1, 1, &mi);
    pt_from_coeffs(r, S, m, count, CGB_PT_ADD, ids);
  }
  if (masks_out) {
    CK(cudaMemcpyAsync(masks_out, slots, sizeof(u64) * (size_t)count * n, cudaMemcpyDeviceToHost, r->stream));
    CK(cudaStreamSynchronize(r->stream));
  }
  API_END
}

// encryption of `count` slot vectors, item i with ChaCha20 key keys[i] and encryption
// index idx[i] (nonces DOM_ENC_A / DOM_ENC_E); one launch sequence for the batch
static void encrypt_items(cgb_ring *r, int count, const uint64_t *slots, const ChaKey *keys, const u64 *idx,
                          const uint32_t *out, const u64 *d_slots = nullptr) {
  Scratch S(r);
  u64 *m = S.alloc<u64>((size_t)count * r->N);
  if (d_slots) {  // slot vectors already on the device (the client's re-encryption of a refresh)
    CK(cudaMemsetAsync(m, 0, sizeof(u64) * (size_t)count * r->N, r->stream));
    LAUNCH("scatter_slots", BYTES_scatter_slots,
           k_scatter_slots<<<dim3(GRID1(r->n_slots, TPB).x, count), TPB, 0, r->stream>>>(m, d_slots, r->d_slot_idx,
                                                                                       r->n_slots, r->t, r->logN));
    int mi = r->iT;
    ntt_items(r, false, m, nullptr, r->N, count, 1, 1, &mi);
  } else {
    encode_slots(r, S, slots, count, m);
  }
  auto pc = ct_ptrs(r, count, out);
  u64 **dc = S.up(pc.data(), count);
  std::vector<u64 *> c1(count);
  std::vector<u64> na(count), ne(count);
  for (int i = 0; i < count; i++) {
    c1[i] = pc[i] + (size_t)r->L * r->N;
    na[i] = nonce_of(DOM_ENC_A, idx[i]);
    ne[i] = nonce_of(DOM_ENC_E, idx[i]);
  }
  u64 **dc1 = S.up(c1.data(), count);
  std::vector<int> qm;
  q_mod_idx(r, qm);
  sample_uniform(r, S, dc1, count, keys, na, r->L, qm.data());
  i64 *e = S.alloc<i64>((size_t)count * r->N);
  sample_cbd(r, S, e, keys, ne);
  u64 words = (u64)r->L * r->N;
  LAUNCH("enc_c0", BYTES_enc_c0, k_enc_c0<<<dim3(GRID1(words, TPB).x, count), TPB, 0, r->stream>>>(dc, m, e, r->d_mods, r->d_c, r->L, r->logN));
  ntt_items(r, true, nullptr, dc, 0, count, 1, r->L, qm.data());
  LAUNCH("enc_sub_as", BYTES_enc_sub_as, k_enc_sub_as<<<dim3(GRID1(words, TPB).x, count), TPB, 0, r->stream>>>(dc, r->d_s, r->d_mods, r->L, r->logN));
}

int cgb_encrypt(cgb_ring *r, int count, const uint64_t *slots, const uint32_t enc_key[8], uint64_t first_index,
                const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  ChaKey key;
  memcpy(key.k, enc_key, sizeof key.k);
  std::vector<ChaKey> keys(count, key);
  std::vector<u64> idx(count);
  for (int i = 0; i < count; i++) idx[i] = first_index + i;
  encrypt_items(r, count, slots, keys.data(), idx.data(), out);
  API_END
}

int cgb_encrypt_batch(cgb_ring *r, int count, const uint64_t *slots, const uint32_t *enc_keys,
                      const uint64_t *indices, const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  std::vector<ChaKey> keys(count);
  for (int i = 0; i < count; i++) memcpy(keys[i].k, enc_keys + 8 * (size_t)i, sizeof keys[i].k);
  encrypt_items(r, count, slots, keys.data(), indices, out);
  API_END
}

static void decrypt_slots_dev(cgb_ring *r, Scratch &S, int count, const uint32_t *cts, u64 *so);
int cgb_reencrypt_batch(cgb_ring *r, int count, const uint32_t *cts, const uint32_t *enc_keys,
                        const uint64_t *indices, const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  std::vector<ChaKey> keys(count);
  for (int i = 0; i < count; i++) memcpy(keys[i].k, enc_keys + 8 * (size_t)i, sizeof keys[i].k);
  Scratch S(r);
  u64 *so = S.alloc<u64>((size_t)count * r->n_slots);
  decrypt_slots_dev(r, S, count, cts, so);
  encrypt_items(r, count, nullptr, keys.data(), indices, out, so);
  API_END
}

struct DecTicket {  // an enqueued decryption: pinned landing buffer + completion event
  u64 *host;
  size_t words, cap;
  cudaEvent_t done;
};
static void decrypt_enqueue(cgb_ring *r, int count, const uint32_t *cts, u64 *dst_host);
int cgb_decrypt_start(cgb_ring *r, int count, const uint32_t *cts, void **ticket_out) {
  API_BEGIN
  RING_LOCK(r);
  const size_t words = (size_t)(count > 0 ? count : 0) * r->n_slots;
  auto *t = new DecTicket{nullptr, words, words, nullptr};
  *ticket_out = t;
  if (count <= 0) return CGB_OK;
  size_t best = r->dec_pool.size();  // best fit: the smallest pooled buffer that holds the batch
  for (size_t i = 0; i < r->dec_pool.size(); i++)
    if (r->dec_pool[i].first >= words && (best == r->dec_pool.size() || r->dec_pool[i].first < r->dec_pool[best].first))
      best = i;
  if (best < r->dec_pool.size()) {
    t->host = r->dec_pool[best].second;
    t->cap = r->dec_pool[best].first;
    r->dec_pool.erase(r->dec_pool.begin() + best);
  } else {  // sizes rounded up to a power of two so buffers serve nearby batch sizes
    size_t cap = 1;
    while (cap < words) cap <<= 1;
    CK(cudaMallocHost(&t->host, sizeof(u64) * cap));
    t->cap = cap;
  }
  decrypt_enqueue(r, count, cts, t->host);
  CK(cudaEventCreateWithFlags(&t->done, cudaEventDisableTiming));
  CK(cudaEventRecord(t->done, r->stream));
  API_END
}
// the same, landing straight in the caller's page-locked buffer (no copy at finish)
int cgb_decrypt_start_into(cgb_ring *r, int count, const uint32_t *cts, uint64_t *pinned_dst, void **ticket_out) {
  API_BEGIN
  RING_LOCK(r);
  const size_t words = (size_t)(count > 0 ? count : 0) * r->n_slots;
  auto *t = new DecTicket{pinned_dst, words, 0, nullptr};  // cap 0: not a pooled buffer
  *ticket_out = t;
  if (count <= 0) return CGB_OK;
  decrypt_enqueue(r, count, cts, pinned_dst);
  CK(cudaEventCreateWithFlags(&t->done, cudaEventDisableTiming));
  CK(cudaEventRecord(t->done, r->stream));
  API_END
}
int cgb_decrypt_finish(cgb_ring *r, void *ticket, uint64_t *slots_out) {
  API_BEGIN
  RING_LOCK(r);
  (void)r;
  auto *t = static_cast<DecTicket *>(ticket);
  if (!t) FAIL(CGB_ERR_PARAM, "null decryption ticket");
  if (t->words) {
    CK(cudaEventSynchronize(t->done));
    if (slots_out && slots_out != t->host) std::memcpy(slots_out, t->host, sizeof(u64) * t->words);
    cudaEventDestroy(t->done);
    if (t->cap) r->dec_pool.push_back({t->cap, t->host});
  }
  delete t;
  API_END
}
int cgb_decrypt(cgb_ring *r, int count, const uint32_t *cts, uint64_t *slots_out) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  decrypt_enqueue(r, count, cts, slots_out);
  CK(cudaStreamSynchronize(r->stream));
  API_END
}
// decryption kernels + the device->host copy of the slots, enqueued on the ring's stream
// decryption into device slot vectors so[count][n_slots] (the client's view)
static void decrypt_slots_dev(cgb_ring *r, Scratch &S, int count, const uint32_t *cts, u64 *so) {
  auto pc = ct_ptrs(r, count, cts);
  u64 **dc = S.up(pc.data(), count);
  u64 words = (u64)r->L * r->N;
  u64 *X = S.alloc<u64>((size_t)count * words);
  LAUNCH("dec_inner", BYTES_dec_inner, k_dec_inner<<<dim3(GRID1(words, TPB).x, count), TPB, 0, r->stream>>>(X, (const u64 *const *)dc, r->d_s, r->d_mods,
                                                                       r->d_c, r->L, r->logN, 0));
  std::vector<int> qm;
  ntt_items(r, false, X, nullptr, words, count, 1, r->L, q_mod_idx(r, qm));
  u64 *m = S.alloc<u64>((size_t)count * r->N);
  LAUNCH("dec_scale", BYTES_dec_scale, k_dec_scale<<<dim3(GRID1(r->N, TPB).x, count), TPB, 0, r->stream>>>(m, X, r->d_c, r->L, r->logN));
  int mi = r->iT;
  ntt_items(r, true, m, nullptr, r->N, count, 1, 1, &mi);
  LAUNCH("gather_slots", BYTES_gather_slots, k_gather_slots<<<dim3(GRID1(r->n_slots, TPB).x, count), TPB, 0, r->stream>>>(so, m, r->d_slot_idx, r->n_slots,
                                                                               r->logN));
}
static void decrypt_enqueue(cgb_ring *r, int count, const uint32_t *cts, u64 *slots_out) {
  Scratch S(r);
  auto pc = ct_ptrs(r, count, cts);
  u64 **dc = S.up(pc.data(), count);
  u64 words = (u64)r->L * r->N;
  u64 *X = S.alloc<u64>((size_t)count * words);
  LAUNCH("dec_inner", BYTES_dec_inner, k_dec_inner<<<dim3(GRID1(words, TPB).x, count), TPB, 0, r->stream>>>(X, (const u64 *const *)dc, r->d_s, r->d_mods,
                                                                       r->d_c, r->L, r->logN, 0));
  std::vector<int> qm;
  ntt_items(r, false, X, nullptr, words, count, 1, r->L, q_mod_idx(r, qm));
  u64 *m = S.alloc<u64>((size_t)count * r->N);
  LAUNCH("dec_scale", BYTES_dec_scale, k_dec_scale<<<dim3(GRID1(r->N, TPB).x, count), TPB, 0, r->stream>>>(m, X, r->d_c, r->L, r->logN));
  int mi = r->iT;
  ntt_items(r, true, m, nullptr, r->N, count, 1, 1, &mi);
  u64 *so = S.alloc<u64>((size_t)count * r->n_slots);
  LAUNCH("gather_slots", BYTES_gather_slots, k_gather_slots<<<dim3(GRID1(r->n_slots, TPB).x, count), TPB, 0, r->stream>>>(so, m, r->d_slot_idx, r->n_slots,
                                                                               r->logN));
  CK(cudaMemcpyAsync(slots_out, so, sizeof(u64) * (size_t)count * r->n_slots, cudaMemcpyDeviceToHost, r->stream));
}

int cgb_noise_budget(cgb_ring *r, int count, const uint32_t *cts, double *bits) {
  API_BEGIN
  RING_LOCK(r);
  const int L = r->L, N = r->N;
  u64 words = (u64)L * N;
  std::vector<u64> host(words);
  // Q and Q/q_l as bignums
  Big Q(1);
  for (int l = 0; l < L; l++) Q.mul(r->mods[l]);
  std::vector<Big> Qh(L, Big(1));
  for (int l = 0; l < L; l++)
    for (int i = 0; i < L; i++)
      if (i != l) Qh[l].mul(r->mods[i]);
  auto cmp = [](const Big &a, const Big &b) {
    for (int i = (int)a.w.size() - 1; i >= 0; i--)
      if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
  };
  auto add = [](Big &a, const Big &b) {
    u128 c = 0;
    for (size_t i = 0; i < a.w.size(); i++) {
      c += (u128)a.w[i] + b.w[i];
      a.w[i] = (u64)c;
      c >>= 64;
    }
  };
  auto sub = [](Big &a, const Big &b) {
    u64 br = 0;
    for (size_t i = 0; i < a.w.size(); i++) {
      u64 bi = b.w[i] + br;
      br = (bi < br) || (a.w[i] < bi);
      a.w[i] -= bi;
    }
  };
  auto lg = [](const Big &a) {
    for (int i = (int)a.w.size() - 1; i >= 0; i--)
      if (a.w[i]) return std::log2((double)a.w[i] + (i ? (double)a.w[i - 1] / 18446744073709551616.0 : 0.0)) + 64.0 * i;
    return -1e9;
  };
  for (int c = 0; c < count; c++) {
    Scratch S(r);
    auto pc = ct_ptrs(r, 1, &cts[c]);
    u64 **dc = S.up(pc.data(), 1);
    u64 *X = S.alloc<u64>(words);
    LAUNCH("dec_inner", BYTES_dec_inner, k_dec_inner<<<dim3(GRID1(words, TPB).x, 1), TPB, 0, r->stream>>>(X, (const u64 *const *)dc, r->d_s, r->d_mods,
                                                                     r->d_c, L, r->logN, 1));
    std::vector<int> qm;
    ntt_items(r, false, X, nullptr, words, 1, 1, L, q_mod_idx(r, qm));
    CK(cudaMemcpyAsync(host.data(), X, sizeof(u64) * words, cudaMemcpyDeviceToHost, r->stream));
    CK(cudaStreamSynchronize(r->stream));
    double worst = -1e9;
    for (int j = 0; j < N; j++) {
      Big acc(0);
      for (int l = 0; l < L; l++) {
        Big term = Qh[l];
        term.mul(h_mulmod(host[(size_t)l * N + j], r->h_c.QhatInv[l], r->mods[l]));
        add(acc, term);
      }
      while (cmp(acc, Q) >= 0) sub(acc, Q);
      Big tw = acc;
      add(tw, acc);
      if (cmp(tw, Q) > 0) {
        Big n = Q;
        sub(n, acc);
        acc = n;
      }
      worst = std::max(worst, lg(acc));
    }
    bits[c] = lg(Q) - std::max(worst, 0.0) - 1.0;
  }
  API_END
}

int cgb_add(cgb_ring *r, int count, const uint32_t *a, const uint32_t *b, const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  Scratch S(r);
  auto pa = ct_ptrs(r, count, a), pb = ct_ptrs(r, count, b), po = ct_ptrs(r, count, out);
  u64 **da = S.up(pa.data(), count), **db = S.up(pb.data(), count), **dout = S.up(po.data(), count);
  LAUNCH("add", BYTES_add, k_add<<<dim3(GRID1(r->ct_words / 2, TPB).x, count), TPB, 0, r->stream>>>(dout, (const u64 *const *)da,
                                                                       (const u64 *const *)db, r->d_mods, r->L,
                                                                       r->logN, r->ct_words));
  API_END
}
int cgb_add_plain(cgb_ring *r, int count, const uint32_t *a, const uint32_t *pt, const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  Scratch S(r);
  auto pa = ct_ptrs(r, count, a), pp = pt_ptrs(r, count, pt), po = ct_ptrs(r, count, out);
  u64 **da = S.up(pa.data(), count), **dp = S.up(pp.data(), count), **dout = S.up(po.data(), count);
  LAUNCH("add_plain", BYTES_add_plain, k_add_plain<<<dim3(GRID1((u64)r->L * r->N / 2, TPB).x, count), TPB, 0, r->stream>>>(
      dout, (const u64 *const *)da, (const u64 *const *)dp, r->d_mods, r->L, r->logN, (u64)r->L * r->N));
  API_END
}
int cgb_mult_plain(cgb_ring *r, int count, const uint32_t *a, const uint32_t *pt, const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  Scratch S(r);
  auto pa = ct_ptrs(r, count, a), pp = pt_ptrs(r, count, pt), po = ct_ptrs(r, count, out);
  u64 **da = S.up(pa.data(), count), **dp = S.up(pp.data(), count), **dout = S.up(po.data(), count);
  LAUNCH("mult_plain", BYTES_mult_plain, k_mult_plain<<<dim3(GRID1((u64)r->L * r->N / 2, TPB).x, count), TPB, 0, r->stream>>>(
      dout, (const u64 *const *)da, (const u64 *const *)dp, r->d_mods, r->L, r->logN, (u64)r->L * r->N));
  API_END
}
int cgb_sum(cgb_ring *r, int count, const uint32_t *a, uint32_t out) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) FAIL(CGB_ERR_PARAM, "empty sum");
  Scratch S(r);
  auto pa = ct_ptrs(r, count, a), po = ct_ptrs(r, 1, &out);
  u64 **da = S.up(pa.data(), count);
  LAUNCH("sum", BYTES_sum, k_sum<<<GRID1(r->ct_words / 2, TPB), TPB, 0, r->stream>>>(po[0], (const u64 *const *)da, count, r->d_mods, r->L,
                                                        r->logN, r->ct_words));
  API_END
}

int cgb_galois(cgb_ring *r, int count, const uint32_t *a, const uint64_t *g, const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  galois_batch(r, count, a, g, out, false);
  API_END
}
static std::vector<u64> steps_to_g(cgb_ring *r, int count, const int64_t *steps) {
  if (!r->one_row) FAIL(CGB_ERR_PARAM, "cgb_rotate needs the one-row layout; compose galois on the host");
  std::vector<u64> g(count);
  u64 twoN = 2ull * r->N;
  for (int i = 0; i < count; i++) {
    int64_t k = steps[i] % r->n_slots;
    if (k < 0) k += r->n_slots;
    g[i] = h_powmod(5, (u64)k, twoN);
  }
  return g;
}
int cgb_rotate(cgb_ring *r, int count, const uint32_t *a, const int64_t *steps, const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  auto g = steps_to_g(r, count, steps);
  galois_batch(r, count, a, g.data(), out, false);
  API_END
}
int cgb_rotate_add(cgb_ring *r, int count, const uint32_t *a, const int64_t *steps, const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  auto g = steps_to_g(r, count, steps);
  galois_batch(r, count, a, g.data(), out, true);
  API_END
}
// The fold / doubling chain x <- x + rotate(x, steps[k]), k = 0 .. nsteps - 1, as one call:
// the same key switches as nsteps cgb_rotate_add calls (same words), the intermediate
// ciphertexts in stream-ordered scratch instead of arena slots.  Small waves are
// host-bound (one call per step costs more host time than its five launches take on
// the device); a chain pays the per-call host work once.
int cgb_rotate_add_chain(cgb_ring *r, int count, const uint32_t *a, int nsteps, const int64_t *steps,
                         const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (count <= 0) return CGB_OK;
  if (nsteps <= 0) FAIL(CGB_ERR_PARAM, "empty rotation chain");
  if (!r->one_row) FAIL(CGB_ERR_PARAM, "cgb_rotate_add_chain needs the one-row layout");
  const u64 twoN = 2ull * r->N, ctw = r->ct_words;
  std::vector<u64> gk(nsteps);
  for (int k = 0; k < nsteps; k++) {
    int64_t kk = steps[k] % r->n_slots;
    if (kk < 0) kk += r->n_slots;
    if (kk == 0) FAIL(CGB_ERR_PARAM, "chain step %d is a multiple of the slot count", k);
    gk[k] = h_powmod(5, (u64)kk, twoN);
  }
  std::vector<u64 *> src = ct_ptrs(r, count, a), last = ct_ptrs(r, count, out), dst(count);
  Scratch S(r);
  u64 *tmp[2] = {nullptr, nullptr};
  if (nsteps > 1) tmp[0] = S.alloc<u64>((size_t)count * ctw);
  if (nsteps > 2) tmp[1] = S.alloc<u64>((size_t)count * ctw);
  std::vector<u64> g(count);
  for (int k = 0; k < nsteps; k++) {
    for (int i = 0; i < count; i++) dst[i] = k == nsteps - 1 ? last[i] : tmp[k & 1] + (size_t)i * ctw;
    std::fill(g.begin(), g.end(), gk[k]);
    galois_ptrs(r, count, src.data(), dst.data(), g.data(), true);
    src = dst;
  }
  API_END
}
int cgb_prepare_galois(cgb_ring *r, int count, const uint64_t *g) {
  API_BEGIN
  RING_LOCK(r);
  for (int i = 0; i < count; i++) {
    u64 gg = g[i] % (2ull * r->N);
    if (gg != 1) get_key(r, gg);
  }
  API_END
}

// INTT of the two polys of each item's operand (per-item pointers) into
// coef[item][4][L][N] at poly offset `poff`
static void intt_and_lift(cgb_ring *r, Scratch &S, int n, const std::vector<u64 *> &srcs, int poff, u64 *coef,
                          u64 *, bool) {
  const int L = r->L, N = r->N;
  std::vector<int> qm;
  q_mod_idx(r, qm);
  {
    std::vector<u64 *> dst(n);
    for (int i = 0; i < n; i++) dst[i] = coef + (size_t)i * 4 * L * N + (size_t)poff * L * N;
    NttJob job{};
    job.items = S.up(dst.data(), n);
    job.src_items = S.up(const_cast<u64 **>(srcs.data()), n);
    int u = 0;
    for (int p = 0; p < 2; p++)
      for (int l = 0; l < L; l++) {
        job.sub_off[u] = job.src_off[u] = (unsigned short)(p * L + l);
        job.sub_mod[u] = (unsigned char)qm[l];
        u++;
      }
    job.nsub = u;
    launch_ntt(r, false, job, n);
  }
}
static void lift_QB(cgb_ring *r, int n, int npoly, u64 *coef, u64 *in, bool fpbc) {
  const int L = r->L, nB = r->nB, N = r->N, logN = r->logN;
  const dim3 grid(GRID1((u64)npoly * N, TPB).x, n);
  launch_begin(r);
  switch (L) {
#define LQB(LL)                                                                                     \
  case LL:                                                                                           \
    if (fpbc) k_lift_QB_fp<LL><<<grid, TPB, 0, r->stream>>>(in, coef, make_bconv<LL>(r), logN);          \
    else k_lift_QB_t<LL><<<grid, TPB, 0, r->stream>>>(in, coef, r->d_mods, r->d_c, r->iB0, logN);      \
    break;
    LQB(1) LQB(2) LQB(3) LQB(4) LQB(5) LQB(6) LQB(7) LQB(8)
#undef LQB
    default: k_lift_QB<<<grid, TPB, 0, r->stream>>>(in, coef, r->d_mods, r->d_c, L, nB, r->iB0, logN);
  }
  launch_end(r, "lift_QB", BYTES_lift_QB * npoly / 4.0);
}

// b's extension to the auxiliary base: polys 0 and 1 of each b item, B limbs in NTT
// form, into two arena slots per item (slot words [nB][N]) -- what mult_cipher
// derives from b every time, kept resident for operands that are multiplied again
// (the encrypted KV cache's parts, every decode step)
static void extend_B(cgb_ring *r, int count, const uint32_t *b, const uint32_t *bx) {
  const int L = r->L, nB = r->nB, nt = L + nB, N = r->N;
  if ((size_t)nB * N > r->ct_words) FAIL(CGB_ERR_PARAM, "B extension does not fit an arena slot");
  const bool fpbc = r->fp_ntt && g_fp_bconv;
  size_t CH = chunk_for(r, (size_t)N * (4 * nt + 4 * L));
  for (int c0 = 0; c0 < count; c0 += (int)CH) {
    const int n = std::min((int)CH, count - c0);
    Scratch S(r);
    auto pb = ct_ptrs(r, n, b + c0);
    auto px = ct_ptrs(r, 2 * n, bx + 2 * (size_t)c0);
    u64 *in = S.alloc<u64>((size_t)n * 4 * nt * N);
    u64 *coef = S.alloc<u64>((size_t)n * 4 * L * N);
    intt_and_lift(r, S, n, pb, 0, coef, in, fpbc);
    lift_QB(r, n, 2, coef, in, fpbc);
    std::vector<u64 *> src(2 * (size_t)n);
    for (int i = 0; i < n; i++)
      for (int p = 0; p < 2; p++) src[2 * i + p] = in + ((size_t)i * 4 + p) * nt * N + (size_t)L * N;
    NttJob job{};
    job.items = S.up(px.data(), 2 * n);
    job.src_items = S.up(src.data(), 2 * n);
    for (int k = 0; k < nB; k++) {
      job.sub_off[k] = job.src_off[k] = (unsigned short)k;
      job.sub_mod[k] = (unsigned char)(r->iB0 + k);
    }
    job.nsub = nB;
    launch_ntt(r, true, job, 2 * n);
  }
}
int cgb_extend_b(cgb_ring *r, int count, const uint32_t *b, const uint32_t *bx) {
  API_BEGIN
  RING_LOCK(r);
  if (count > 0) extend_B(r, count, b, bx);
  API_END
}

static void mult_cipher_impl(cgb_ring *r, int count, const uint32_t *a, const uint32_t *b, const uint32_t *bx,
                             const uint32_t *out, const uint32_t *ax = nullptr);
int cgb_mult_cipher(cgb_ring *r, int count, const uint32_t *a, const uint32_t *b, const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (count > 0) mult_cipher_impl(r, count, a, b, nullptr, out);
  API_END
}
int cgb_mult_cipher_ext(cgb_ring *r, int count, const uint32_t *a, const uint32_t *b, const uint32_t *bx,
                        const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (count > 0) mult_cipher_impl(r, count, a, b, bx, out);
  API_END
}
int cgb_mult_cipher_ext2(cgb_ring *r, int count, const uint32_t *a, const uint32_t *ax, const uint32_t *b,
                         const uint32_t *bx, const uint32_t *out) {
  API_BEGIN
  RING_LOCK(r);
  if (ax && !bx) FAIL(CGB_ERR_PARAM, "mult_cipher_ext2: a resident a-extension needs b's too (swap the operands)");
  if (count > 0) mult_cipher_impl(r, count, a, b, bx, out, ax);
  API_END
}
static void mult_cipher_impl(cgb_ring *r, int count, const uint32_t *a, const uint32_t *b, const uint32_t *bx,
                             const uint32_t *out, const uint32_t *ax) {
  const int L = r->L, nB = r->nB, nt = L + nB, N = r->N, logN = r->logN;
  const bool fpbc = r->fp_ntt && g_fp_bconv;  // base conversions on the FP64 pipe (every modulus < 2^49)
  u64 *rk = get_key(r, 0);
  std::vector<int> qm, bm(nB), tm(nt);
  q_mod_idx(r, qm);
  for (int k = 0; k < nB; k++) bm[k] = r->iB0 + k;
  for (int l = 0; l < nt; l++) tm[l] = l < L ? l : r->iB0 + (l - L);
  size_t per_item = (size_t)N * (4 * nt + 4 * L + 3 * nt + 3 * L + 1 + L * (L + 1) + 2 * (L + 1) + 2 * L + L);
  size_t CH = chunk_for(r, per_item);
  for (int c0 = 0; c0 < count; c0 += (int)CH) {
    int n = std::min((int)CH, count - c0);
    Scratch S(r);
    // 8(d) unit: two input and one output ciphertext per item, the relinearisation key once
    group_begin(r);
    const double mc_bytes = 8.0 * (double)r->ct_words * 3.0 * n + 8.0 * 2.0 * L * (L + 1.0) * N;
    auto pa = ct_ptrs(r, n, a + c0), pb = ct_ptrs(r, n, b + c0), po = ct_ptrs(r, n, out + c0);
    // inputs: in[item][4][nt][N] with Q limbs = NTT copies; coef[item][4][L][N]
    u64 *in = S.alloc<u64>((size_t)n * 4 * nt * N);
    u64 *coef = S.alloc<u64>((size_t)n * 4 * L * N);
    u64 **dpa = S.up(pa.data(), n), **dpb = S.up(pb.data(), n);
    // INTT of the operands straight from the arena into coef, lift Q -> B; with b's
    // resident extension (bx) only a's two polys
    // (ax too: both extensions resident -- an operand multiplied by many others, e.g. the
    // decode step's encrypted weights a_pref against every V column, arcc.py:358-361)
    const int npoly = ax ? 0 : bx ? 2 : 4;
    u64 **dpx = nullptr, **dpax = nullptr;
    if (ax) {
      auto px = ct_ptrs(r, 2 * n, bx + 2 * (size_t)c0), pxa = ct_ptrs(r, 2 * n, ax + 2 * (size_t)c0);
      dpx = S.up(px.data(), 2 * n);
      dpax = S.up(pxa.data(), 2 * n);
    } else if (bx) {
      auto px = ct_ptrs(r, 2 * n, bx + 2 * (size_t)c0);
      dpx = S.up(px.data(), 2 * n);
      intt_and_lift(r, S, n, pa, 0, coef, in, fpbc);
    } else {
      intt_and_lift(r, S, n, pa, 0, coef, in, fpbc);
      intt_and_lift(r, S, n, pb, 2, coef, in, fpbc);
    }
    if (npoly) lift_QB(r, n, npoly, coef, in, fpbc);
    if (npoly) {
      NttJob job{};
      job.base = in;
      job.item_stride = 4ull * nt * N;
      int u = 0;
      for (int p = 0; p < npoly; p++)
        for (int k = 0; k < nB; k++) {
          job.sub_off[u] = (unsigned short)(p * nt + L + k);
          job.sub_mod[u] = (unsigned char)bm[k];
          u++;
        }
      job.nsub = u;
      launch_ntt(r, true, job, n);
    }
    u64 *ten = S.alloc<u64>((size_t)n * 3 * nt * N);
    const TensorLoad tl{dpa, dpb, in, dpx, dpax, r->d_mods, L, nt, r->iB0, logN};
    if (!tensor_intt_fused(r, n, ten, tl, tm.data())) {
      if (fpbc && g_tensor_fp && N >= 4) {
        LAUNCH("tensor", BYTES_tensor, k_tensor_fp<<<dim3(GRID1((u64)nt * N / 4, TPB).x, n), TPB, 0, r->stream>>>(ten, in, dpa, dpb, dpx, r->d_mods, L, nt, r->iB0, logN, dpax));
      } else {
        LAUNCH("tensor", BYTES_tensor, k_tensor<<<dim3(GRID1((u64)nt * N, TPB).x, n), TPB, 0, r->stream>>>(ten, in, dpa, dpb, dpx, r->d_mods, L, nt, r->iB0, logN, dpax));
      }
      ntt_items(r, false, ten, nullptr, 3ull * nt * N, n, 3, nt, tm.data());
    }
    u64 *d = S.alloc<u64>((size_t)n * 3 * L * N);
    {
      const dim3 grid(GRID1(3ull * N, TPB).x, n);
      launch_begin(r);
      switch (L) {
#define LSR(LL)                                                                                       \
  case LL:                                                                                             \
    if (fpbc) k_scale_round_fp<LL><<<grid, TPB, 0, r->stream>>>(d, ten, make_bconv<LL>(r), logN);         \
    else k_scale_round_t<LL><<<grid, TPB, 0, r->stream>>>(d, ten, r->d_mods, r->d_c, r->iB0, logN);      \
    break;
        LSR(1) LSR(2) LSR(3) LSR(4) LSR(5) LSR(6) LSR(7) LSR(8)
#undef LSR
        default: k_scale_round<<<grid, TPB, 0, r->stream>>>(d, ten, r->d_mods, r->d_c, L, nB, r->iB0, logN);
      }
      launch_end(r, "scale_round", BYTES_scale_round);
    }
    ntt_items(r, true, d, nullptr, 3ull * L * N, n, 3, L, qm.data());
    // relinearise d2 and add (d0, d1), both read in place from d = [item][d0 d1 d2][L][N]
    std::vector<u64 *> keys(n, rk);
    u64 **dk = S.up(keys.data(), n), **dout = S.up(po.data(), n);
    std::vector<u64 *> d01p(n);
    for (int i = 0; i < n; i++) d01p[i] = d + (size_t)i * 3 * L * N;
    u64 **dd01 = S.up(d01p.data(), n);
    KsSrc xin{d + 2ull * L * N, 3ull * L * N, nullptr, 0, nullptr};
    KsSrc none{nullptr, 0, nullptr, 0, nullptr};
    keyswitch(r, S, xin, n, dk, dout, none, (const u64 *const *)dd01);
    group_end(r, ax ? "mult_cipher_ext2" : bx ? "mult_cipher_ext" : "mult_cipher", mc_bytes);
  }
}

}  // extern "C"
