/*
 * cgb200.h -- C ABI of the B200 RNS-BFV backend for the CryptoGen HE hot path.
 *
 * The reference package exposes its homomorphic substrate as the Python
 * class cryptogen.backend.Context (/root/reference/pkg/src/cryptogen/
 * backend.py:245-364) with per-op methods; every kernel above it
 * (encodings.py, linear_kernels.py, arcc.py, kv_cache.py, nonlinear.py) only
 * calls those methods.  This library is what a drop-in replacement of that
 * class binds through ctypes (INTEGRATION.md shows the binding).  Each entry
 * point below names the reference method it replaces.
 *
 * Conventions
 *  - A ring (cgb_ring) owns the parameters, the secret key, the evaluation
 *    keys and a device arena of fixed-size ciphertext slots.  Ciphertexts
 *    are named by uint32 slot ids; a ciphertext is uint64[2][L][N] in the
 *    NTT domain (poly, RNS limb over Q, coefficient).
 *  - Encoded plaintexts live in a second arena (uint64[L][N]) and are named
 *    by plaintext ids; kind CGB_PT_MUL is the centred lift used by
 *    mult_plain, CGB_PT_ADD the floor(Q m / t) scaling used by add_plain.
 *  - Batched entry points take `count` and host arrays of ids; every output
 *    id must be distinct from every input id of the same call.
 *  - Slot vectors crossing the ABI are host uint64[count][n_slots] arrays of
 *    residues mod t.
 *  - Return value 0 = success; CGB_ERR_PARAM maps to the reference's
 *    ParameterError (backend.py:45-46), everything else is a runtime error.
 *    cgb_last_error() returns the message of the last failure (thread-local).
 *  - All work is stream-ordered on the ring's stream (cgb_set_stream);
 *    calls returning host data synchronise that stream.
 */
#ifndef CGB200_H
#define CGB200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CGB_OK 0
#define CGB_ERR_PARAM 1
#define CGB_ERR_CUDA 2
#define CGB_ERR_NOMEM 3
#define CGB_ERR_STATE 4

#define CGB_PT_MUL 0
#define CGB_PT_ADD 1

typedef struct cgb_ring cgb_ring;

/* ---- lifetime ------------------------------------------------------------
 * Replaces Context.__init__ / new_context (backend.py:245-256, :367-368) for
 * the arithmetic: ring degree 2^log_n, plaintext modulus t (the reference's
 * plain_modulus, backend.py:121), n_limbs primes of Q, n_slots logical
 * slots.  one_row = 1 selects the native layout (t = 1 mod 4 n_slots,
 * N = 2 n_slots, rotation = one automorphism); 0 the two-row layout
 * (N = n_slots) whose cyclic shift the host composes from two automorphisms.
 * key_seed seeds the ChaCha20 streams of the secret and evaluation keys.
 * arena_cts / arena_pts: capacity of the ciphertext / plaintext arenas. */
int cgb_ring_create(int log_n, uint64_t plain_modulus, int n_limbs, int n_slots,
                    int one_row, const uint32_t key_seed[8], int64_t arena_cts,
                    int64_t arena_pts, cgb_ring **out);
/* as cgb_ring_create with Q primes < 2^q_bits (P and B primes < 2^(q_bits+1));
 * cgb_ring_create uses q_bits = 60 */
int cgb_ring_create_ex(int log_n, uint64_t plain_modulus, int n_limbs, int q_bits, int n_slots,
                       int one_row, const uint32_t key_seed[8], int64_t arena_cts,
                       int64_t arena_pts, cgb_ring **out);
void cgb_ring_destroy(cgb_ring *ring);
/* moduli in order Q[0..L) | P | B[0..L]; returns how many were written */
int cgb_ring_moduli(const cgb_ring *ring, uint64_t *out, int cap);
/* words of one ciphertext (2*L*N) */
size_t cgb_ct_words(const cgb_ring *ring);
const char *cgb_last_error(void);
int cgb_set_stream(cgb_ring *ring, void *cuda_stream);
int cgb_sync(cgb_ring *ring);
/* number of device kernel launches issued by this ring so far */
uint64_t cgb_launch_count(const cgb_ring *ring);
/* CUDA-event timing (clears earlier records): on = 1 times every launch (programmatic
 * dependent launch off); on = 2 times every multi-launch operation as one record
 * ("keyswitch", "keyswitch_hoisted", "mult_cipher[_ext]" with SURVEY 8(d)
 * algorithmic bytes; PDL stays on inside it) and every other launch; 0 = off */
int cgb_timing_enable(cgb_ring *ring, int on);
/* aggregate of the recorded launches, one line per kernel:
 * "<name> <launches> <total ms> <algorithmic bytes> <algorithmic modular products>\n" */
int cgb_timing_report(cgb_ring *ring, char *buf, size_t cap);
/* measured peak of the modular multiply on the pipe this ring's NTT uses
 * (register-resident independent chains over the whole GPU), per second:
 * the FP64 error-free product for rings of primes < 2^49 (FP64-pipe NTT),
 * else the 64-bit integer Shoup product */
int cgb_modmul_peak(cgb_ring *ring, double *modmuls_per_s);
/* microbenchmark: average ms of one batched forward (fwd=1) / inverse NTT over
 * count ciphertexts (2 L limb-polys each), timed over iters launches */
int cgb_bench_ntt(cgb_ring *ring, int count, int fwd, int iters, double *ms_out);

/* ---- ciphertext / plaintext storage -------------------------------------
 * Ciphertext handles replace SlotCiphertext (backend.py:216-230); the
 * reference's values are immutable and GC-owned, so the host frees ids from
 * a finalizer.  load/store move raw NTT-domain words (checkpoints, tests). */
int cgb_ct_alloc(cgb_ring *ring, int count, uint32_t *ids_out);
int cgb_ct_free(cgb_ring *ring, int count, const uint32_t *ids);
int cgb_ct_copy(cgb_ring *ring, int count, const uint32_t *src, const uint32_t *dst);
int cgb_ct_store(cgb_ring *ring, int count, const uint32_t *ids, uint64_t *host_words);
int cgb_ct_load(cgb_ring *ring, int count, const uint32_t *ids, const uint64_t *host_words);
uint64_t *cgb_ct_device_ptr(cgb_ring *ring, uint32_t id);
/* free ciphertext slots of the arena (headroom checks of optional resident data) */
int64_t cgb_ct_free_count(cgb_ring *ring);
int cgb_pt_alloc(cgb_ring *ring, int count, uint32_t *ids_out);
int cgb_pt_free(cgb_ring *ring, int count, const uint32_t *ids);
/* encode host slot vectors into plaintexts; kind CGB_PT_MUL / CGB_PT_ADD.
 * Replaces the operand handling of mult_plain / add_plain (backend.py:327-339). */
int cgb_pt_encode(cgb_ring *ring, int count, const uint64_t *slots, int kind,
                  const uint32_t *pt_ids);

/* Device-side server masks: MpcChannel.sample_mask(n_slots) (nonlinear.py:86-87,
 * rng.integers(0, t, n) on numpy's PCG64 -- its 32-bit half-word buffer and Lemire
 * rejection included) for `count` items, item i drawn from channel chan[i] (a
 * channel's items in draw order).  st holds 6 words per channel -- state_hi,
 * state_lo, inc_hi, inc_lo, has_uint32, uinteger (numpy's PCG64 state) -- and is
 * advanced in place past the draws.  Each mask r_i is encoded as an add_plain
 * plaintext into pt_pos[i] and t - r_i into pt_neg[i] (either may be NULL);
 * masks_out (optional, host count x n_slots) receives r.  Replaces the host draws
 * and uploads of _refresh_part (kv_cache.py:146-153). */
int cgb_mask_pcg64(cgb_ring *ring, int count, int nchan, const int32_t *chan, uint64_t *st,
                   const uint32_t *pt_neg, const uint32_t *pt_pos, uint64_t *masks_out);

/* ---- client role ----------------------------------------------------------
 * Context.encrypt (backend.py:307-310): symmetric RLWE encryption; the
 * randomness of ciphertext i is ChaCha20(enc_key, first_index + i). */
int cgb_encrypt(cgb_ring *ring, int count, const uint64_t *slots,
                const uint32_t enc_key[8], uint64_t first_index, const uint32_t *out);
/* cgb_encrypt over items of several contexts in one launch sequence: item i uses
 * the 8-word key enc_keys[8 i .. 8 i + 8) and encryption index indices[i] (the
 * per-context counters of Context.encrypt, backend.py:307-310, for a wave of
 * encryptions owned by different contexts) */
int cgb_encrypt_batch(cgb_ring *ring, int count, const uint64_t *slots, const uint32_t *enc_keys,
                      const uint64_t *indices, const uint32_t *out_ids);
/* The client's decrypt-then-encrypt of a refresh (kv_cache.py:150: ctx.encrypt(ctx.decrypt(masked)))
 * without the host hop: item i is decrypted to its slot vector on the device and encrypted
 * again with key enc_keys[8 i ..] at index indices[i] -- the same words as cgb_decrypt
 * followed by cgb_encrypt_batch of those slots. */
int cgb_reencrypt_batch(cgb_ring *ring, int count, const uint32_t *cts, const uint32_t *enc_keys,
                        const uint64_t *indices, const uint32_t *out_ids);
/* Context.decrypt (backend.py:312-319) */
int cgb_decrypt(cgb_ring *ring, int count, const uint32_t *cts, uint64_t *slots_out);
/* The same decryption split at the client round trip: _start enqueues it (and the
   device->host copy into library-owned pinned memory) and returns a ticket; _finish
   waits for that ticket only and copies the count x n_slots residues out.  Lets a
   caller compute on the client side of one batch while the device works on the next
   (Context.decrypt semantics per ciphertext are unchanged). */
int cgb_decrypt_start(cgb_ring *ring, int count, const uint32_t *cts, void **ticket_out);
int cgb_decrypt_finish(cgb_ring *ring, void *ticket, uint64_t *slots_out);
/* cgb_decrypt_start landing in the caller's count x n_slots buffer, which must stay
   valid until cgb_decrypt_finish(ring, ticket, NULL or that buffer); page-locked for
   the copy to stay asynchronous (a pageable buffer works, the call then returns after
   the copy) */
int cgb_decrypt_start_into(cgb_ring *ring, int count, const uint32_t *cts, uint64_t *pinned_dst, void **ticket_out);
/* client-side diagnostic: invariant noise budget in bits of each ciphertext */
int cgb_noise_budget(cgb_ring *ring, int count, const uint32_t *cts, double *bits_out);

/* ---- server role (batched) ---------------------------------------------- */
/* Context.add (backend.py:321-325) */
int cgb_add(cgb_ring *ring, int count, const uint32_t *a, const uint32_t *b, const uint32_t *out);
/* Context.add_plain (backend.py:327-332); pt of kind CGB_PT_ADD */
int cgb_add_plain(cgb_ring *ring, int count, const uint32_t *a, const uint32_t *pt, const uint32_t *out);
/* Context.mult_plain (backend.py:334-339); pt of kind CGB_PT_MUL */
int cgb_mult_plain(cgb_ring *ring, int count, const uint32_t *a, const uint32_t *pt, const uint32_t *out);
/* Context.mult_cipher (backend.py:341-347): tensor, scale-and-round, relinearise */
int cgb_mult_cipher(cgb_ring *ring, int count, const uint32_t *a, const uint32_t *b, const uint32_t *out);
/* mult_cipher with b's extension to the auxiliary base B kept resident: bx holds two
   arena slots per item (b's polys 0 and 1, the nB B limbs in NTT form, as written by
   cgb_extend_b); the result equals cgb_mult_cipher's word for word.  The encrypted KV
   cache's parts are multiplied every decode step, so their extension is computed once
   (the reference recomputes nothing -- it has no base extension: backend.py:341-347). */
int cgb_extend_b(cgb_ring *ring, int count, const uint32_t *b, const uint32_t *bx);
int cgb_mult_cipher_ext(cgb_ring *ring, int count, const uint32_t *a, const uint32_t *b, const uint32_t *bx,
                        const uint32_t *out);
/* mult_cipher with BOTH operands' base-B extensions resident (ax, bx: two arena slots
   per item each, from cgb_extend_b; ax may be NULL = cgb_mult_cipher_ext): an operand
   multiplied by many others (the decode step's encrypted attention weights against
   every V column, arcc.py:358-361; the prefill's weight rows, arcc.py:307-314) is
   extended once.  Same words as cgb_mult_cipher. */
int cgb_mult_cipher_ext2(cgb_ring *ring, int count, const uint32_t *a, const uint32_t *ax, const uint32_t *b,
                         const uint32_t *bx, const uint32_t *out);
/* Galois automorphism X -> X^g plus key switch; g = 1 copies.
 * Context.rotate (backend.py:349-355) is galois(5^k mod 2N) in the one-row layout. */
int cgb_galois(cgb_ring *ring, int count, const uint32_t *a, const uint64_t *g, const uint32_t *out);
/* Context.rotate: cyclic left shift by steps[i] (one-row layout only).
 * A batch in which ids repeat in a[] (one ciphertext rotated by many steps, e.g.
 * the diagonal CPVM, linear_kernels.py:105-142) is key-switched hoisted: one
 * ModUp per distinct source, same output words (CGB_KS_HOIST=0 disables). */
int cgb_rotate(cgb_ring *ring, int count, const uint32_t *a, const int64_t *steps, const uint32_t *out);
/* out = a + rotate(a, step): one doubling/fold step of broadcast_slot
 * (arcc.py:90-93), tile_token (encodings.py:212-215) and fold_sum
 * (linear_kernels.py:37-41), fused into one pass */
int cgb_rotate_add(cgb_ring *ring, int count, const uint32_t *a, const int64_t *steps, const uint32_t *out);
/* The rotate-and-add chain of a fold / broadcast (reference linear_kernels.py:37-41,
 * arcc.py:90-93): x <- add(x, rotate(x, steps[k])) for k = 0 .. nsteps-1 on each of the
 * count ciphertexts, out = the last x.  The same words as nsteps cgb_rotate_add calls;
 * the intermediate ciphertexts live in device scratch (no arena slots).  Every step must
 * be non-zero modulo the slot count. */
int cgb_rotate_add_chain(cgb_ring *ring, int count, const uint32_t *a, int nsteps, const int64_t *steps,
                         const uint32_t *out);
/* out = sum of count ciphertexts a[0..count) (exact mod q: order-free) */
int cgb_sum(cgb_ring *ring, int count, const uint32_t *a, uint32_t out);
/* generate (and cache) evaluation keys for Galois elements ahead of use */
int cgb_prepare_galois(cgb_ring *ring, int count, const uint64_t *g);

#ifdef __cplusplus
}
#endif
#endif /* CGB200_H */
