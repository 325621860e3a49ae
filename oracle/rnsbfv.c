/*
 * oracle/rnsbfv.c -- CPU restatement of the RNS-BFV arithmetic behind the
 * CryptoGen slot API.  TEST INFRASTRUCTURE ONLY: this file is the checker
 * that tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use.
 * The product (paper_2602_08798_b200/) never links or calls it.
 *
 * Parity status.  The reference package (cryptogen, /root/reference/pkg)
 * is a slot-level emulation: a ciphertext is an n-slot vector over Z_p
 * (backend.py:216-230) and every op is plain Z_p arithmetic
 * (backend.py:307-355).  It has no polynomials, so the POLYNOMIAL level of
 * this oracle is "parity unpinned" against the reference; what is pinned is
 * the slot level: decrypt(op(encrypt(v))) must equal the reference op on v
 * (tests/test_oracle_*.py check this against tests/golden/ vectors made by
 * tests/golden/make_golden.py from the reference itself).
 *
 * Everything here is written from textbook definitions as plain scalar C
 * with unsigned __int128; DESIGN.md section 3 states each algorithm and the
 * GPU library must reproduce every ciphertext word of it bit-exactly.
 *
 *   ring      R = Z[X]/(X^N + 1), N = 2*n_slots (one-row layout) or n_slots
 *   Q         L primes < 2^60, = 1 mod 2^32 (so = 1 mod 2N), largest first
 *   P         one special prime < 2^61 (hybrid key switching, dnum = L)
 *   B         L+1 auxiliary primes < 2^61 (BFV tensor base, HPS-style)
 *   slots     slot i <-> evaluation at psi_t^(5^i) (row 0 of the hypercube)
 *   rotate k  Galois element 5^k mod 2N (cyclic shift by k, backend.py:349)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef uint64_t u64;
typedef int64_t i64;
typedef uint32_t u32;
typedef unsigned __int128 u128;

#define MAXMODS 40
#define MAXKEYS 4096

/* ------------------------------------------------------------------ */
/* scalar modular arithmetic                                           */
/* ------------------------------------------------------------------ */
static inline u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
static inline u64 addmod(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
static inline u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
static u64 powmod(u64 a, u64 e, u64 q) {
    u64 r = 1 % q; a %= q;
    while (e) { if (e & 1) r = mulmod(r, a, q); a = mulmod(a, a, q); e >>= 1; }
    return r;
}
static u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); }
static inline u64 reduce_signed(i64 x, u64 q) {
    i64 r = x % (i64)q; return r < 0 ? (u64)(r + (i64)q) : (u64)r;
}

static int is_prime_u64(u64 n) {
    static const u64 bases[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) if (n % bases[i] == 0) return n == bases[i];
    u64 d = n - 1; int r = 0;
    while (!(d & 1)) { d >>= 1; r++; }
    for (int i = 0; i < 12; i++) {
        u64 x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int ok = 0;
        for (int k = 0; k < r - 1; k++) { x = mulmod(x, x, n); if (x == n - 1) { ok = 1; break; } }
        if (!ok) return 0;
    }
    return 1;
}

static u32 brev(u32 x, int bits) {
    u32 r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* primitive 2N-th root: psi = x^((q-1)/2N) for the smallest x >= 2 with psi^N = -1 */
static u64 find_psi(u64 q, u64 twoN) {
    for (u64 x = 2;; x++) {
        u64 psi = powmod(x, (q - 1) / twoN, q);
        if (powmod(psi, twoN / 2, q) == q - 1) return psi;
    }
}

/* ------------------------------------------------------------------ */
/* tiny bignum (little-endian u64 words) for the CRT constants         */
/* ------------------------------------------------------------------ */
#define BW 32
typedef struct { u64 w[BW]; } big;
static void big_set(big *a, u64 x) { memset(a, 0, sizeof *a); a->w[0] = x; }
static void big_mul(big *a, u64 x) {
    u128 c = 0;
    for (int i = 0; i < BW; i++) { c += (u128)a->w[i] * x; a->w[i] = (u64)c; c >>= 64; }
}
static u64 big_divmod(big *a, u64 d) { /* a /= d, returns a % d */
    u128 r = 0;
    for (int i = BW - 1; i >= 0; i--) { r = (r << 64) | a->w[i]; a->w[i] = (u64)(r / d); r %= d; }
    return (u64)r;
}
static u64 big_mod(const big *a, u64 d) { big t = *a; return big_divmod(&t, d); }
/* floor(r * 2^128 / q) for r < q, as (hi, lo) */
static void frac128(u64 r, u64 q, u64 *hi, u64 *lo) {
    u128 x = (u128)r << 64; *hi = (u64)(x / q); u64 r2 = (u64)(x % q);
    x = (u128)r2 << 64; *lo = (u64)(x / q);
}

/* ------------------------------------------------------------------ */
/* ChaCha20 (DJB layout: 64-bit block counter, 64-bit nonce)           */
/* ------------------------------------------------------------------ */
#define ROTL(x, n) (((x) << (n)) | ((x) >> (32 - (n))))
#define QR(a, b, c, d) a += b; d ^= a; d = ROTL(d, 16); c += d; b ^= c; b = ROTL(b, 12); \
                       a += b; d ^= a; d = ROTL(d, 8);  c += d; b ^= c; b = ROTL(b, 7);
static void chacha_block(const u32 key[8], u64 counter, u64 nonce, u32 out[16]) {
    u32 s[16] = {0x61707865u, 0x3320646eu, 0x79622d32u, 0x6b206574u,
                 key[0], key[1], key[2], key[3], key[4], key[5], key[6], key[7],
                 (u32)counter, (u32)(counter >> 32), (u32)nonce, (u32)(nonce >> 32)};
    u32 x[16]; memcpy(x, s, sizeof x);
    for (int i = 0; i < 10; i++) {
        QR(x[0], x[4], x[8], x[12]) QR(x[1], x[5], x[9], x[13])
        QR(x[2], x[6], x[10], x[14]) QR(x[3], x[7], x[11], x[15])
        QR(x[0], x[5], x[10], x[15]) QR(x[1], x[6], x[11], x[12])
        QR(x[2], x[7], x[8], x[13]) QR(x[3], x[4], x[9], x[14])
    }
    for (int i = 0; i < 16; i++) out[i] = x[i] + s[i];
}
/* words w[first .. first+cnt) of stream (key, nonce) */
static void chacha_words(const u32 key[8], u64 nonce, u64 first, u64 cnt, u32 *w) {
    u32 blk[16]; u64 cur = (u64)-1;
    for (u64 i = 0; i < cnt; i++) {
        u64 idx = first + i;
        if (idx / 16 != cur) { cur = idx / 16; chacha_block(key, cur, nonce, blk); }
        w[i] = blk[idx % 16];
    }
}

#define DOM_SK 1ull
#define DOM_KSK_A 2ull
#define DOM_KSK_E 3ull
#define DOM_ENC_A 4ull
#define DOM_ENC_E 5ull
static inline u64 nonce_of(u64 dom, u64 sub) { return (dom << 56) | sub; }

/* ------------------------------------------------------------------ */
/* context                                                             */
/* ------------------------------------------------------------------ */
typedef struct {
    u64 g;            /* Galois element; 0 = relinearisation key */
    u64 *b, *a;       /* [dnum][L+1][N] each, NTT form over Q u {P} */
} ksk_t;

typedef struct {
    int logN, N, L, nB, nmods, n_slots, one_row;
    u64 t;
    u64 mods[MAXMODS];          /* [0,L) Q | L: P | [L+1, L+1+nB) B */
    u64 *tw[MAXMODS], *itw[MAXMODS], ninv[MAXMODS];
    u64 *tw_t, *itw_t, ninv_t;  /* plaintext modulus NTT */
    u32 *slot_idx;              /* logical slot -> NTT_t position */
    u32 keyseed[8];
    i64 *s_coeff;               /* ternary secret, coefficient form */
    u64 *s_ntt;                 /* [L+1][N] NTT form over Q u {P} */
    /* constants */
    u64 Qmodt, tinvq[MAXMODS], Pinvq[MAXMODS], Pmodq[MAXMODS];
    u64 dec_omega[MAXMODS], dec_th_hi[MAXMODS], dec_th_lo[MAXMODS];
    u64 QhatInv[MAXMODS];               /* (Q/q_l)^-1 mod q_l */
    u64 QhatModB[MAXMODS][MAXMODS];     /* [l][k] (Q/q_l) mod b_k */
    u64 QmodB[MAXMODS];
    double invq[MAXMODS], invb[MAXMODS];
    u64 QBhatInv[MAXMODS];              /* ((Q/q_l) B)^-1 mod q_l */
    u64 BQhatInv[MAXMODS];              /* ((B/b_k) Q)^-1 mod b_k */
    u64 sc_omega[MAXMODS][MAXMODS];     /* [l][k] floor(tB/q_l) mod b_k */
    u64 sc_th_hi[MAXMODS], sc_th_lo[MAXMODS];
    u64 tBhat[MAXMODS];                 /* t (B/b_k) mod b_k */
    u64 BhatInv[MAXMODS];               /* (B/b_k)^-1 mod b_k */
    u64 BhatModQ[MAXMODS][MAXMODS];     /* [k][l] (B/b_k) mod q_l */
    u64 BmodQ[MAXMODS];
    ksk_t *keys; int nkeys;
} ora_ctx;

static void ntt_fwd_tab(const ora_ctx *c, u64 *a, const u64 *tw, u64 q) {
    int N = c->N, t = N;
    for (int m = 1; m < N; m <<= 1) {
        t >>= 1;
        for (int i = 0; i < m; i++) {
            int j1 = 2 * i * t; u64 S = tw[m + i];
            for (int j = j1; j < j1 + t; j++) {
                u64 U = a[j], V = mulmod(a[j + t], S, q);
                a[j] = addmod(U, V, q); a[j + t] = submod(U, V, q);
            }
        }
    }
}
static void ntt_inv_tab(const ora_ctx *c, u64 *a, const u64 *itw, u64 ninv, u64 q) {
    int N = c->N, t = 1;
    for (int m = N; m > 1; m >>= 1) {
        int h = m >> 1, j1 = 0;
        for (int i = 0; i < h; i++) {
            u64 S = itw[h + i];
            for (int j = j1; j < j1 + t; j++) {
                u64 U = a[j], V = a[j + t];
                a[j] = addmod(U, V, q); a[j + t] = mulmod(submod(U, V, q), S, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    for (int j = 0; j < N; j++) a[j] = mulmod(a[j], ninv, q);
}
static void ntt_m(const ora_ctx *c, int mi, u64 *a) { ntt_fwd_tab(c, a, c->tw[mi], c->mods[mi]); }
static void intt_m(const ora_ctx *c, int mi, u64 *a) { ntt_inv_tab(c, a, c->itw[mi], c->ninv[mi], c->mods[mi]); }

static void make_tables(int N, int logN, u64 q, u64 **tw, u64 **itw, u64 *ninv) {
    u64 psi = find_psi(q, 2 * (u64)N), psii = invmod(psi, q);
    *tw = malloc(sizeof(u64) * N); *itw = malloc(sizeof(u64) * N);
    for (int k = 0; k < N; k++) {
        u32 r = brev(k, logN);
        (*tw)[k] = powmod(psi, r, q); (*itw)[k] = powmod(psii, r, q);
    }
    *ninv = invmod((u64)N % q, q);
}

/* largest primes below 2^bits with q = 1 mod 2^32 (hence mod 2N), skipping ones
 * already taken; the low word 1 makes q-hat * q one 32-bit multiply on the GPU */
static int take_primes(ora_ctx *c, int bits, int count, int at) {
    u64 step = 1ull << 32, top = 1ull << bits;
    if (2 * (u64)c->N > step) step = 2 * (u64)c->N;
    u64 cand = top - (top % step) + 1;
    if (cand >= top) cand -= step;
    int got = 0;
    while (got < count) {
        int dup = 0;
        for (int i = 0; i < at + got; i++) if (c->mods[i] == cand) dup = 1;
        if (!dup && cand != c->t && is_prime_u64(cand)) { c->mods[at + got] = cand; got++; }
        cand -= step;
    }
    return at + got;
}

static void cbd_poly(const u32 key[8], u64 nonce, int N, i64 *e) {
    u32 *w = malloc(sizeof(u32) * 2 * N);
    chacha_words(key, nonce, 0, 2 * (u64)N, w);
    for (int j = 0; j < N; j++) {
        u64 x = (u64)w[2 * j] | ((u64)w[2 * j + 1] << 32);
        e[j] = (i64)__builtin_popcountll(x & 0x1FFFFFull) - (i64)__builtin_popcountll((x >> 21) & 0x1FFFFFull);
    }
    free(w);
}
static void uniform_poly(const u32 key[8], u64 nonce, int N, int nl, const u64 *mods, u64 *out) {
    u32 *w = malloc(sizeof(u32) * 4 * (size_t)N * nl);
    chacha_words(key, nonce, 0, 4 * (u64)N * nl, w);
    for (int l = 0; l < nl; l++)
        for (int j = 0; j < N; j++) {
            size_t e = 4 * ((size_t)l * N + j);
            u128 X = (u128)w[e] | ((u128)w[e + 1] << 32) | ((u128)w[e + 2] << 64) | ((u128)w[e + 3] << 96);
            out[(size_t)l * N + j] = (u64)(X % mods[l]);
        }
    free(w);
}

/* coefficient-domain automorphism X -> X^g on a signed poly */
static void auto_coeff_signed(int N, const i64 *in, u64 g, i64 *out) {
    memset(out, 0, sizeof(i64) * N);
    for (int i = 0; i < N; i++) {
        u64 j = ((u64)i * g) % (2 * (u64)N);
        if (j < (u64)N) out[j] += in[i]; else out[j - N] -= in[i];
    }
}
static void auto_coeff_mod(int N, const u64 *in, u64 g, u64 q, u64 *out) {
    for (int i = 0; i < N; i++) {
        u64 j = ((u64)i * g) % (2 * (u64)N);
        if (j < (u64)N) out[j] = in[i]; else out[j - N] = in[i] ? q - in[i] : 0;
    }
}

void *ora_create(int logN, u64 t, int L, int n_slots, int one_row, const u32 keyseed[8], int q_bits) {
    ora_ctx *c = calloc(1, sizeof(ora_ctx));
    c->logN = logN; c->N = 1 << logN; c->L = L; c->nB = L + 1; c->t = t;
    c->n_slots = n_slots; c->one_row = one_row;
    memcpy(c->keyseed, keyseed, sizeof c->keyseed);
    int N = c->N;
    /* Q primes < 2^q_bits; P and B one bit wider, or also < 2^q_bits when q_bits <= 49 */
    int pb = q_bits <= 49 ? q_bits : q_bits + 1;
    int at = take_primes(c, q_bits, L, 0);
    at = take_primes(c, pb, 1, at);
    at = take_primes(c, pb, c->nB, at);
    c->nmods = at;
    for (int i = 0; i < c->nmods; i++) make_tables(N, logN, c->mods[i], &c->tw[i], &c->itw[i], &c->ninv[i]);
    make_tables(N, logN, t, &c->tw_t, &c->itw_t, &c->ninv_t);

    /* slot map: slot i <-> exponent 5^i (row 0), row 1 = -5^c in fallback layout */
    c->slot_idx = malloc(sizeof(u32) * n_slots);
    u64 twoN = 2 * (u64)N;
    int h = one_row ? n_slots : n_slots / 2;
    u64 e = 1;
    for (int i = 0; i < h; i++) {
        c->slot_idx[i] = brev((u32)((e - 1) / 2), logN);
        if (!one_row) c->slot_idx[h + i] = brev((u32)((twoN - e - 1) / 2), logN);
        e = (e * 5) % twoN;
    }

    /* secret key */
    c->s_coeff = malloc(sizeof(i64) * N);
    u32 *w = malloc(sizeof(u32) * N);
    chacha_words(keyseed, nonce_of(DOM_SK, 0), 0, N, w);
    for (int j = 0; j < N; j++) c->s_coeff[j] = (i64)(w[j] % 3) - 1;
    free(w);
    c->s_ntt = malloc(sizeof(u64) * (size_t)(L + 1) * N);
    for (int l = 0; l <= L; l++) {
        u64 *s = c->s_ntt + (size_t)l * N;
        for (int j = 0; j < N; j++) s[j] = reduce_signed(c->s_coeff[j], c->mods[l]);
        ntt_m(c, l, s);
    }

    /* constants */
    const u64 *q = c->mods, P = c->mods[L], *b = c->mods + L + 1;
    c->Qmodt = 1; for (int l = 0; l < L; l++) c->Qmodt = mulmod(c->Qmodt, q[l] % t, t);
    for (int l = 0; l < L; l++) {
        c->tinvq[l] = invmod(t % q[l], q[l]);
        c->Pmodq[l] = P % q[l];
        c->Pinvq[l] = invmod(P % q[l], q[l]);
        u64 qh = 1; for (int i = 0; i < L; i++) if (i != l) qh = mulmod(qh, q[i] % q[l], q[l]);
        c->QhatInv[l] = invmod(qh, q[l]);
        /* decrypt scale: t*QhatInv/q = omega + theta */
        u128 x = (u128)t * c->QhatInv[l];
        c->dec_omega[l] = (u64)(x / q[l]);
        frac128((u64)(x % q[l]), q[l], &c->dec_th_hi[l], &c->dec_th_lo[l]);
        c->invq[l] = 1.0 / (double)q[l];
        for (int k = 0; k < c->nB; k++) {
            u64 v = 1; for (int i = 0; i < L; i++) if (i != l) v = mulmod(v, q[i] % b[k], b[k]);
            c->QhatModB[l][k] = v;
        }
    }
    for (int k = 0; k < c->nB; k++) {
        u64 v = 1; for (int i = 0; i < L; i++) v = mulmod(v, q[i] % b[k], b[k]);
        c->QmodB[k] = v;
        u64 bh = 1; for (int i = 0; i < c->nB; i++) if (i != k) bh = mulmod(bh, b[i] % b[k], b[k]);
        c->BhatInv[k] = invmod(bh, b[k]);
        c->tBhat[k] = mulmod(t % b[k], bh, b[k]);
        c->BQhatInv[k] = invmod(mulmod(bh, v, b[k]), b[k]);
        c->invb[k] = 1.0 / (double)b[k];
        for (int l = 0; l < L; l++) {
            u64 w2 = 1; for (int i = 0; i < c->nB; i++) if (i != k) w2 = mulmod(w2, b[i] % q[l], q[l]);
            c->BhatModQ[k][l] = w2;
        }
    }
    for (int l = 0; l < L; l++) {
        u64 v = 1; for (int i = 0; i < c->nB; i++) v = mulmod(v, b[i] % q[l], q[l]);
        c->BmodQ[l] = v;
        u64 qh = 1; for (int i = 0; i < L; i++) if (i != l) qh = mulmod(qh, q[i] % q[l], q[l]);
        c->QBhatInv[l] = invmod(mulmod(qh, v, q[l]), q[l]);
        /* scale: t*B/q_l = omega' + theta' */
        big T; big_set(&T, t);
        for (int i = 0; i < c->nB; i++) big_mul(&T, b[i]);
        u64 r = big_divmod(&T, q[l]);
        for (int k = 0; k < c->nB; k++) c->sc_omega[l][k] = big_mod(&T, b[k]);
        frac128(r, q[l], &c->sc_th_hi[l], &c->sc_th_lo[l]);
    }
    c->keys = calloc(MAXKEYS, sizeof(ksk_t));
    return c;
}

void ora_destroy(void *vc) {
    ora_ctx *c = vc;
    for (int i = 0; i < c->nmods; i++) { free(c->tw[i]); free(c->itw[i]); }
    free(c->tw_t); free(c->itw_t); free(c->slot_idx); free(c->s_coeff); free(c->s_ntt);
    for (int i = 0; i < c->nkeys; i++) { free(c->keys[i].a); free(c->keys[i].b); }
    free(c->keys); free(c);
}

int ora_moduli(void *vc, u64 *out) { ora_ctx *c = vc; memcpy(out, c->mods, sizeof(u64) * c->nmods); return c->nmods; }
void ora_secret(void *vc, i64 *out) { ora_ctx *c = vc; memcpy(out, c->s_coeff, sizeof(i64) * c->N); }
void ora_ntt(void *vc, int mi, u64 *a) { ntt_m(vc, mi, a); }
void ora_intt(void *vc, int mi, u64 *a) { intt_m(vc, mi, a); }
void ora_ntt_t(void *vc, u64 *a) { ora_ctx *c = vc; ntt_fwd_tab(c, a, c->tw_t, c->t); }
void ora_intt_t(void *vc, u64 *a) { ora_ctx *c = vc; ntt_inv_tab(c, a, c->itw_t, c->ninv_t, c->t); }

/* slots (mod t) -> plaintext polynomial coefficients in [0, t) */
void ora_encode(void *vc, const u64 *slots, u64 *m) {
    ora_ctx *c = vc;
    memset(m, 0, sizeof(u64) * c->N);
    for (int i = 0; i < c->n_slots; i++) m[c->slot_idx[i]] = slots[i] % c->t;
    ntt_inv_tab(c, m, c->itw_t, c->ninv_t, c->t);
}
void ora_decode(void *vc, const u64 *m, u64 *slots) {
    ora_ctx *c = vc;
    u64 *tmp = malloc(sizeof(u64) * c->N);
    memcpy(tmp, m, sizeof(u64) * c->N);
    ntt_fwd_tab(c, tmp, c->tw_t, c->t);
    for (int i = 0; i < c->n_slots; i++) slots[i] = tmp[c->slot_idx[i]];
    free(tmp);
}

/* floor(Q m / t) mod q_l, coefficient form */
static void scaled_msg(const ora_ctx *c, const u64 *m, int l, u64 *out) {
    u64 q = c->mods[l];
    for (int j = 0; j < c->N; j++) {
        u64 r = mulmod(c->Qmodt, m[j] % c->t, c->t);
        out[j] = submod(0, mulmod(r, c->tinvq[l], q), q);
    }
}

void ora_encrypt(void *vc, const u64 *m, const u32 enckey[8], u64 idx, u64 *ct) {
    ora_ctx *c = vc; int N = c->N, L = c->L;
    u64 *c0 = ct, *c1 = ct + (size_t)L * N;
    uniform_poly(enckey, nonce_of(DOM_ENC_A, idx), N, L, c->mods, c1);
    i64 *e = malloc(sizeof(i64) * N);
    cbd_poly(enckey, nonce_of(DOM_ENC_E, idx), N, e);
    for (int l = 0; l < L; l++) {
        u64 q = c->mods[l], *x = c0 + (size_t)l * N;
        scaled_msg(c, m, l, x);
        for (int j = 0; j < N; j++) x[j] = addmod(x[j], reduce_signed(e[j], q), q);
        ntt_m(c, l, x);
        const u64 *a = c1 + (size_t)l * N, *s = c->s_ntt + (size_t)l * N;
        for (int j = 0; j < N; j++) x[j] = submod(x[j], mulmod(a[j], s[j], q), q);
    }
    free(e);
}

void ora_decrypt(void *vc, const u64 *ct, u64 *m) {
    ora_ctx *c = vc; int N = c->N, L = c->L;
    u64 *x = malloc(sizeof(u64) * (size_t)L * N);
    for (int l = 0; l < L; l++) {
        u64 q = c->mods[l];
        const u64 *c0 = ct + (size_t)l * N, *c1 = ct + (size_t)(L + l) * N, *s = c->s_ntt + (size_t)l * N;
        u64 *xl = x + (size_t)l * N;
        for (int j = 0; j < N; j++) xl[j] = addmod(c0[j], mulmod(c1[j], s[j], q), q);
        intt_m(c, l, xl);
    }
    for (int j = 0; j < N; j++) {
        u128 S = 0; u64 I = 0;
        for (int l = 0; l < L; l++) {
            u64 xv = x[(size_t)l * N + j];
            S += (u128)xv * c->dec_th_hi[l] + (u64)(((u128)xv * c->dec_th_lo[l]) >> 64);
            I = addmod(I, mulmod(xv % c->t, c->dec_omega[l], c->t), c->t);
        }
        u64 R = (u64)((S + ((u128)1 << 63)) >> 64);
        m[j] = addmod(I, R % c->t, c->t);
    }
    free(x);
}

void ora_add(void *vc, const u64 *a, const u64 *b, u64 *out) {
    ora_ctx *c = vc; int N = c->N, L = c->L;
    for (int p = 0; p < 2; p++) for (int l = 0; l < L; l++) {
        size_t o = ((size_t)p * L + l) * N;
        for (int j = 0; j < N; j++) out[o + j] = addmod(a[o + j], b[o + j], c->mods[l]);
    }
}

void ora_add_plain(void *vc, const u64 *a, const u64 *m, u64 *out) {
    ora_ctx *c = vc; int N = c->N, L = c->L;
    memcpy(out, a, sizeof(u64) * 2 * (size_t)L * N);
    u64 *x = malloc(sizeof(u64) * N);
    for (int l = 0; l < L; l++) {
        scaled_msg(c, m, l, x); ntt_m(c, l, x);
        for (int j = 0; j < N; j++) out[(size_t)l * N + j] = addmod(out[(size_t)l * N + j], x[j], c->mods[l]);
    }
    free(x);
}

/* centered lift of a plaintext polynomial into limb l, NTT form */
static void plain_lift(const ora_ctx *c, const u64 *m, int l, u64 *x) {
    u64 q = c->mods[l], half = c->t / 2;
    for (int j = 0; j < c->N; j++) {
        u64 v = m[j] % c->t;
        x[j] = v <= half ? v % q : q - ((c->t - v) % q);
    }
    ntt_m(c, l, x);
}

void ora_mult_plain(void *vc, const u64 *a, const u64 *m, u64 *out) {
    ora_ctx *c = vc; int N = c->N, L = c->L;
    u64 *x = malloc(sizeof(u64) * N);
    for (int l = 0; l < L; l++) {
        plain_lift(c, m, l, x);
        for (int p = 0; p < 2; p++) {
            size_t o = ((size_t)p * L + l) * N;
            for (int j = 0; j < N; j++) out[o + j] = mulmod(a[o + j], x[j], c->mods[l]);
        }
    }
    free(x);
}

/* ------------------------------------------------------------------ */
/* key switching keys (hybrid, dnum = L, alpha = 1, one special prime)  */
/* ------------------------------------------------------------------ */
static ksk_t *get_key(ora_ctx *c, u64 g) {
    for (int i = 0; i < c->nkeys; i++) if (c->keys[i].g == g) return &c->keys[i];
    int N = c->N, L = c->L, nl = L + 1;
    ksk_t *k = &c->keys[c->nkeys++];
    k->g = g;
    k->a = malloc(sizeof(u64) * (size_t)L * nl * N);
    k->b = malloc(sizeof(u64) * (size_t)L * nl * N);
    /* source key s' in NTT form over Q u {P} */
    u64 *sp = malloc(sizeof(u64) * (size_t)nl * N);
    if (g == 0) {
        for (int l = 0; l < nl; l++) for (int j = 0; j < N; j++)
            sp[(size_t)l * N + j] = mulmod(c->s_ntt[(size_t)l * N + j], c->s_ntt[(size_t)l * N + j], c->mods[l]);
    } else {
        i64 *sg = malloc(sizeof(i64) * N);
        auto_coeff_signed(N, c->s_coeff, g, sg);
        for (int l = 0; l < nl; l++) {
            for (int j = 0; j < N; j++) sp[(size_t)l * N + j] = reduce_signed(sg[j], c->mods[l]);
            ntt_m(c, l, sp + (size_t)l * N);
        }
        free(sg);
    }
    i64 *e = malloc(sizeof(i64) * N);
    u64 *x = malloc(sizeof(u64) * N);
    for (int d = 0; d < L; d++) {
        u64 sub = (g << 8) | (u64)d;
        u64 *a = k->a + (size_t)d * nl * N, *b = k->b + (size_t)d * nl * N;
        uniform_poly(c->keyseed, nonce_of(DOM_KSK_A, sub), N, nl, c->mods, a);
        cbd_poly(c->keyseed, nonce_of(DOM_KSK_E, sub), N, e);
        for (int l = 0; l < nl; l++) {
            u64 q = c->mods[l];
            for (int j = 0; j < N; j++) x[j] = reduce_signed(e[j], q);
            ntt_m(c, l, x);
            for (int j = 0; j < N; j++) {
                size_t o = (size_t)l * N + j;
                u64 v = submod(x[j], mulmod(a[o], c->s_ntt[o], q), q);
                if (l == d) v = addmod(v, mulmod(c->Pmodq[d], sp[o], q), q);
                b[o] = v;
            }
        }
    }
    free(e); free(x); free(sp);
    return k;
}

/* (u0, u1) = KS(x) ; x NTT form over Q ; outputs NTT form over Q */
static void keyswitch(ora_ctx *c, const u64 *x, ksk_t *k, u64 *u0, u64 *u1) {
    int N = c->N, L = c->L, nl = L + 1;
    u64 *acc0 = calloc((size_t)nl * N, sizeof(u64)), *acc1 = calloc((size_t)nl * N, sizeof(u64));
    u64 *dig = malloc(sizeof(u64) * N), *tmp = malloc(sizeof(u64) * N);
    for (int d = 0; d < L; d++) {
        u64 qd = c->mods[d];
        memcpy(dig, x + (size_t)d * N, sizeof(u64) * N);
        intt_m(c, d, dig);
        for (int l = 0; l < nl; l++) {
            u64 q = c->mods[l];
            if (l == d) memcpy(tmp, x + (size_t)d * N, sizeof(u64) * N);
            else {
                for (int j = 0; j < N; j++) {
                    u64 v = dig[j];
                    tmp[j] = v <= qd / 2 ? v % q : submod(0, (qd - v) % q, q);
                }
                ntt_m(c, l, tmp);
            }
            const u64 *kb = k->b + ((size_t)d * nl + l) * N, *ka = k->a + ((size_t)d * nl + l) * N;
            for (int j = 0; j < N; j++) {
                size_t o = (size_t)l * N + j;
                acc0[o] = addmod(acc0[o], mulmod(tmp[j], kb[j], q), q);
                acc1[o] = addmod(acc1[o], mulmod(tmp[j], ka[j], q), q);
            }
        }
    }
    u64 P = c->mods[L];
    for (int p = 0; p < 2; p++) {
        u64 *acc = p ? acc1 : acc0, *out = p ? u1 : u0;
        memcpy(dig, acc + (size_t)L * N, sizeof(u64) * N);
        intt_m(c, L, dig);
        for (int l = 0; l < L; l++) {
            u64 q = c->mods[l];
            for (int j = 0; j < N; j++) {
                u64 v = dig[j];
                tmp[j] = v <= P / 2 ? v % q : submod(0, (P - v) % q, q);
            }
            ntt_m(c, l, tmp);
            for (int j = 0; j < N; j++)
                out[(size_t)l * N + j] = mulmod(submod(acc[(size_t)l * N + j], tmp[j], q), c->Pinvq[l], q);
        }
    }
    free(acc0); free(acc1); free(dig); free(tmp);
}

/* automorphism sigma_g + key switch back to s ; g odd, g = 1 -> copy */
void ora_galois(void *vc, const u64 *a, u64 g, u64 *out) {
    ora_ctx *c = vc; int N = c->N, L = c->L;
    size_t half = (size_t)L * N;
    g %= 2 * (u64)N;
    if (g == 1) { memcpy(out, a, sizeof(u64) * 2 * half); return; }
    u64 *c0 = malloc(sizeof(u64) * half), *c1 = malloc(sizeof(u64) * half), *tmp = malloc(sizeof(u64) * N);
    for (int p = 0; p < 2; p++) for (int l = 0; l < L; l++) {
        memcpy(tmp, a + p * half + (size_t)l * N, sizeof(u64) * N);
        intt_m(c, l, tmp);
        u64 *dst = (p ? c1 : c0) + (size_t)l * N;
        auto_coeff_mod(N, tmp, g, c->mods[l], dst);
        ntt_m(c, l, dst);
    }
    ksk_t *k = get_key(c, g);
    keyswitch(c, c1, k, out, out + half);
    for (int l = 0; l < L; l++) for (int j = 0; j < N; j++) {
        size_t o = (size_t)l * N + j;
        out[o] = addmod(out[o], c0[o], c->mods[l]);
    }
    free(c0); free(c1); free(tmp);
}

/* ------------------------------------------------------------------ */
/* BFV ciphertext product: lift Q->B, tensor over Q u B, round(t/Q .),  */
/* B->Q, relinearise                                                   */
/* ------------------------------------------------------------------ */
void ora_mult_cipher(void *vc, const u64 *A, const u64 *Bc, u64 *out) {
    ora_ctx *c = vc; int N = c->N, L = c->L, nB = c->nB, nt = L + nB;
    size_t half = (size_t)L * N;
    const u64 *q = c->mods, *b = c->mods + L + 1;
    /* four input polys over Q u B, NTT form: layout [poly][limb][N], limb < L: Q, else B */
    u64 *in = malloc(sizeof(u64) * 4 * (size_t)nt * N);
    const u64 *srcs[4] = {A, A + half, Bc, Bc + half};
    u64 *coef = malloc(sizeof(u64) * half);
    for (int p = 0; p < 4; p++) {
        u64 *dst = in + (size_t)p * nt * N;
        memcpy(coef, srcs[p], sizeof(u64) * half);
        for (int l = 0; l < L; l++) intt_m(c, l, coef + (size_t)l * N);
        memcpy(dst, srcs[p], sizeof(u64) * half);
        for (int j = 0; j < N; j++) {
            u64 y[MAXMODS]; double s = 0.0;
            for (int l = 0; l < L; l++) {
                y[l] = mulmod(coef[(size_t)l * N + j], c->QhatInv[l], q[l]);
                s = s + (double)y[l] * c->invq[l];
            }
            u64 v = (u64)(s + 0.5);
            for (int k = 0; k < nB; k++) {
                u64 acc = 0;
                for (int l = 0; l < L; l++) acc = addmod(acc, mulmod(y[l], c->QhatModB[l][k], b[k]), b[k]);
                acc = submod(acc, mulmod(v, c->QmodB[k], b[k]), b[k]);
                dst[(size_t)(L + k) * N + j] = acc;
            }
        }
        for (int k = 0; k < nB; k++) ntt_m(c, L + 1 + k, dst + (size_t)(L + k) * N);
    }
    /* tensor */
    u64 *ten = malloc(sizeof(u64) * 3 * (size_t)nt * N);
    for (int l = 0; l < nt; l++) {
        u64 mq = l < L ? q[l] : b[l - L];
        for (int j = 0; j < N; j++) {
            size_t o = (size_t)l * N + j, P = (size_t)nt * N;
            u64 a0 = in[o], a1 = in[P + o], b0 = in[2 * P + o], b1 = in[3 * P + o];
            ten[o] = mulmod(a0, b0, mq);
            ten[P + o] = addmod(mulmod(a0, b1, mq), mulmod(a1, b0, mq), mq);
            ten[2 * P + o] = mulmod(a1, b1, mq);
        }
    }
    for (int p = 0; p < 3; p++) for (int l = 0; l < nt; l++)
        intt_m(c, l < L ? l : L + 1 + (l - L), ten + ((size_t)p * nt + l) * N);
    /* scale and round into B, then B -> Q */
    u64 *d = malloc(sizeof(u64) * 3 * half);
    for (int p = 0; p < 3; p++) {
        const u64 *cp = ten + (size_t)p * nt * N;
        for (int j = 0; j < N; j++) {
            u64 y[MAXMODS]; u128 S = 0;
            for (int l = 0; l < L; l++) {
                y[l] = mulmod(cp[(size_t)l * N + j], c->QBhatInv[l], q[l]);
                S += (u128)y[l] * c->sc_th_hi[l] + (u64)(((u128)y[l] * c->sc_th_lo[l]) >> 64);
            }
            u64 R = (u64)((S + ((u128)1 << 63)) >> 64);
            u64 dk[MAXMODS];
            for (int k = 0; k < nB; k++) {
                u64 acc = R % b[k];
                for (int l = 0; l < L; l++) acc = addmod(acc, mulmod(y[l], c->sc_omega[l][k], b[k]), b[k]);
                u64 z = mulmod(cp[(size_t)(L + k) * N + j], c->BQhatInv[k], b[k]);
                acc = addmod(acc, mulmod(z, c->tBhat[k], b[k]), b[k]);
                dk[k] = acc;
            }
            /* B -> Q, centered */
            u64 yk[MAXMODS]; double s = 0.0;
            for (int k = 0; k < nB; k++) {
                yk[k] = mulmod(dk[k], c->BhatInv[k], b[k]);
                s = s + (double)yk[k] * c->invb[k];
            }
            u64 v = (u64)(s + 0.5);
            for (int l = 0; l < L; l++) {
                u64 acc = 0;
                for (int k = 0; k < nB; k++) acc = addmod(acc, mulmod(yk[k], c->BhatModQ[k][l], q[l]), q[l]);
                acc = submod(acc, mulmod(v, c->BmodQ[l], q[l]), q[l]);
                d[((size_t)p * L + l) * N + j] = acc;
            }
        }
        for (int l = 0; l < L; l++) ntt_m(c, l, d + ((size_t)p * L + l) * N);
    }
    ksk_t *rk = get_key(c, 0);
    keyswitch(c, d + 2 * half, rk, out, out + half);
    for (int p = 0; p < 2; p++) for (int l = 0; l < L; l++) for (int j = 0; j < N; j++) {
        size_t o = ((size_t)p * L + l) * N + j;
        out[o] = addmod(out[o], d[o], q[l]);
    }
    free(in); free(coef); free(ten); free(d);
}

/* invariant noise budget in bits (client-side diagnostic, like SEAL's):
 * x = t (c0 + c1 s) mod Q centered ; budget = log2(Q) - log2(max |x|) - 1 */
static int big_cmp(const big *a, const big *b) {
    for (int i = BW - 1; i >= 0; i--) if (a->w[i] != b->w[i]) return a->w[i] < b->w[i] ? -1 : 1;
    return 0;
}
static void big_add(big *a, const big *b) {
    u128 cy = 0;
    for (int i = 0; i < BW; i++) { cy += (u128)a->w[i] + b->w[i]; a->w[i] = (u64)cy; cy >>= 64; }
}
static void big_sub(big *a, const big *b) { /* a -= b, a >= b */
    u64 br = 0;
    for (int i = 0; i < BW; i++) {
        u64 bi = b->w[i] + br; br = (bi < br) || (a->w[i] < bi);
        a->w[i] -= bi;
    }
}
static double big_log2(const big *a) {
    for (int i = BW - 1; i >= 0; i--) if (a->w[i]) {
        double top = (double)a->w[i] + (i ? (double)a->w[i - 1] / 18446744073709551616.0 : 0.0);
        return log2(top) + 64.0 * i;
    }
    return -1e9;
}
double ora_noise_budget(void *vc, const u64 *ct) {
    ora_ctx *c = vc; int N = c->N, L = c->L;
    u64 *x = malloc(sizeof(u64) * (size_t)L * N);
    for (int l = 0; l < L; l++) {
        u64 q = c->mods[l];
        const u64 *c0 = ct + (size_t)l * N, *c1 = ct + (size_t)(L + l) * N, *s = c->s_ntt + (size_t)l * N;
        for (int j = 0; j < N; j++) x[(size_t)l * N + j] = mulmod(addmod(c0[j], mulmod(c1[j], s[j], q), q), c->t % q, q);
        intt_m(c, l, x + (size_t)l * N);
    }
    big Q, Qh[MAXMODS];
    big_set(&Q, 1); for (int l = 0; l < L; l++) big_mul(&Q, c->mods[l]);
    for (int l = 0; l < L; l++) { big_set(&Qh[l], 1); for (int i = 0; i < L; i++) if (i != l) big_mul(&Qh[l], c->mods[i]); }
    double worst = -1e9;
    for (int j = 0; j < N; j++) {
        big acc; big_set(&acc, 0);
        for (int l = 0; l < L; l++) {
            big term = Qh[l];
            big_mul(&term, mulmod(x[(size_t)l * N + j], c->QhatInv[l], c->mods[l]));
            big_add(&acc, &term);
        }
        while (big_cmp(&acc, &Q) >= 0) big_sub(&acc, &Q);
        big twice = acc; big_add(&twice, &acc);
        if (big_cmp(&twice, &Q) > 0) { big neg = Q; big_sub(&neg, &acc); acc = neg; }
        double lg = big_log2(&acc);
        if (lg > worst) worst = lg;
    }
    free(x);
    return big_log2(&Q) - (worst < 0 ? 0 : worst) - 1.0;
}
