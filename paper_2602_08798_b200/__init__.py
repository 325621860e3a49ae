"""B200-native RNS-BFV backend for the CryptoGen (arXiv 2602.08798) HE hot path.

The package mirrors the reference package's public names (cryptogen/
__init__.py:11-88) for the hot path: the substrate (backend), the packings
(encodings), the projections' fold (linear_kernels), the CT x CT attention
kernels (arcc), the encrypted KV cache (kv_cache) and the HE <-> share
conversions (nonlinear), plus the head-batched forms
(attention_step_heads, append_token_heads, maybe_refresh_heads).
"""

from .backend import (BackendParams, Context, DecryptionFailure, GpuCiphertext, GpuContext, NoiseBudgetExhausted,
                      NoiseCosts, OpCounter, ParameterError, SlotCiphertext, Wave, default_plain_modulus, is_prime,
                      new_context)
from .encodings import (Encoding, EncodingKind, PackedMatrix, block_capacity, decode, encode, load_matrix, next_pow2,
                        pack_token_inner, save_matrix, tile_token)
from .fixedpoint import (FixedPointParams, attention_weights, causal_attention_weights, fp_decode, fp_encode,
                         fp_softmax, fp_truncate, from_signed, to_signed)
from .linear_kernels import cpmm_outer_diagonal, cpvm_inner_diagonal, fold_sum
from .nonlinear import (MpcChannel, SharePair, he_to_shares, reconstruct, share_vector, shares_to_he, truncate)
from .arcc import (ScoreLayout, ScoreVector, arcc_inner_inner, arcc_inner_outer, attention_step,
                   attention_step_heads, broadcast_slot, compact_scores, prefill_attention, prefill_attention_heads)
from .kv_cache import (KVCache, RefreshEvent, append_token, append_token_heads, cache_stats, init_cache, load_cache,
                       maybe_refresh, maybe_refresh_heads, save_cache)
