"""Heterogeneous encrypted KV cache: slot-aware append and masked refresh.

Mirrors /root/reference/pkg/src/cryptogen/kv_cache.py: ``KVCache``
(:59-78), ``init_cache`` (:86-111), ``append_token`` (:128-143) over
``_append_one`` (:114-125), ``maybe_refresh`` (:156-196) over
``_refresh_part`` (:146-153), ``cache_stats`` (:199-211) and the
checkpoint pair (:219-281).

Batched forms: ``append_token_heads`` writes the K and V tokens of every
head in one rotate / mask / add wave; ``maybe_refresh_heads`` round-trips
every selected part of every head's cache through the client in one masked
decrypt + encrypt wave.  Masks, nonces, counters and refresh events follow
the per-op order (segments prefill_K, prefill_V, auto_K, auto_V; parts in
index order; heads in list order).

``save_cache_ct`` / ``load_cache_ct`` add a ciphertext-level snapshot (raw
RNS words, no decryption) next to the reference's decrypted snapshot.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np

from .backend import ParameterError, PlainBatch, _pt_cache
from .encodings import Encoding, EncodingKind, PackedMatrix, block_capacity, load_matrix, save_matrix
from .nonlinear import MpcChannel, device_masks, device_masks_ok, draw_masks, neg_mod

__all__ = ["KVCache", "RefreshEvent", "append_token", "append_token_heads", "cache_stats", "init_cache",
           "load_cache", "load_cache_ct", "maybe_refresh", "maybe_refresh_heads", "save_cache", "save_cache_ct"]

SEGMENTS = ("prefill_K", "prefill_V", "auto_K", "auto_V")


def _chain_ids(ctxs, ops, start: dict) -> list:
    """Ids the per-op reference would give the last op of each item's chain
    when the items' chains run back to back (items in list order, each
    owner's ids counting up from ``start[id(owner)]``)."""
    nxt = dict(start)
    out = []
    for c, k in zip(ctxs, ops):
        nxt[id(c)] += k
        out.append(nxt[id(c)] - 1)
    return out


def _block_masks(n: int, pos, widths) -> PlainBatch:
    """Append masks (ones on [pos, pos + d2)) as a symbolic plaintext batch."""
    def build(keys):
        v = np.zeros((len(keys), n), dtype=np.int64)
        for i, (_, _, p0, w) in enumerate(keys):
            v[i, p0: p0 + w] = 1
        return v

    return PlainBatch([("block", n, int(p0), int(w)) for p0, w in zip(pos, widths)], build)


def _retag(handles, cids):
    for h, cid in zip(handles, cids):
        object.__setattr__(h, "id", int(cid))  # handles are immutable to users, not to their producer
    return handles


@dataclass(frozen=True)
class RefreshEvent:
    step: int
    segment: str
    part_index: int
    part_id: int
    budget_before: int
    mpc_bytes: int
    forced: bool = False


@dataclass(frozen=True)
class KVCache:
    d2: int
    B: int
    m: int
    t_auto: int
    prefill_K: PackedMatrix | None
    prefill_V: PackedMatrix | None
    auto_K: PackedMatrix
    auto_V: PackedMatrix
    refresh_log: tuple = field(default_factory=tuple)

    def segments(self):
        out = []
        if self.prefill_K is not None:
            out += [("prefill_K", self.prefill_K), ("prefill_V", self.prefill_V)]
        return out + [("auto_K", self.auto_K), ("auto_V", self.auto_V)]


def _empty_auto(d2: int, B: int) -> PackedMatrix:
    return PackedMatrix(Encoding(EncodingKind.INNER_COMPACTED, 0, d2, block=B), [], encrypted=True)


def init_cache(K_pref, V_pref, ctx, d2: int | None = None) -> KVCache:
    """kv_cache.py:86-111."""
    if (K_pref is None) != (V_pref is None):
        raise ParameterError("prefill K and V must both be present or both absent")
    if K_pref is not None:
        if K_pref.encoding.kind is not EncodingKind.OUTER or not K_pref.encrypted:
            raise ParameterError("prefill segments must be encrypted outer packings")
        if K_pref.encoding != V_pref.encoding:
            raise ParameterError(f"prefill K {K_pref.encoding} and V {V_pref.encoding} disagree")
        m, width = K_pref.encoding.rows, K_pref.encoding.cols
        if d2 is not None and d2 != width:
            raise ParameterError(f"d2 {d2} does not match prefill width {width}")
        d2 = width
    else:
        if d2 is None:
            raise ParameterError("an empty cache needs an explicit d2")
        m = 0
    B = block_capacity(ctx.params.n_slots, d2)
    return KVCache(d2, B, m, 0, K_pref, V_pref, _empty_auto(d2, B), _empty_auto(d2, B))


# ----------------------------------------------------------------------------
# append
# ----------------------------------------------------------------------------
def append_token(cache: KVCache, k_new, v_new, ctx) -> KVCache:
    """Write one token at slot offset (t_auto mod B) * d2 (kv_cache.py:128-143)."""
    return append_token_heads([cache], [k_new], [v_new], [ctx])[0]


def append_token_heads(caches, ks, vs, ctxs) -> list:
    """append_token for every head: K and V of head h are items 2h, 2h+1."""
    H = len(caches)
    c0 = ctxs[0]
    C = type(c0)
    n = c0.params.n_slots
    toks, owners, pos, fresh = [], [], [], []
    for h in range(H):
        b = caches[h].t_auto % caches[h].B
        for t in (ks[h], vs[h]):
            toks.append(t)
            owners.append(ctxs[h])
            pos.append(b * caches[h].d2)
            fresh.append(b == 0)
    pos = np.asarray(pos, np.int64)
    fresh = np.asarray(fresh)
    start = {id(c): c._next_id for c in owners}
    w = C.wave_of(toks, owners)
    moved = np.nonzero(pos)[0]
    if moved.size:
        still = np.nonzero(pos == 0)[0]
        rot = C.w_rotate(w.take(moved), -pos[moved])
        w = type(w).concat([w.take(still), rot]).take(np.argsort(np.concatenate([still, moved])))
    new = C.w_mult_plain(w, _block_masks(n, pos, [caches[h].d2 for h in np.repeat(np.arange(H), 2)]))
    # fresh blocks add onto encrypt(0); others onto the segment's last part
    fi = np.nonzero(fresh)[0]
    oi = np.nonzero(~fresh)[0]
    outs = [None] * len(toks)
    if fi.size:
        zeros = C.w_encrypt([owners[i] for i in fi], np.zeros((fi.size, n), np.int64))
        for i, hnd in zip(fi, C.w_add(zeros, new.take(fi)).handles()):
            outs[i] = hnd
    if oi.size:
        lasts = []
        for i in oi:
            cache = caches[i // 2]
            seg = cache.auto_K if i % 2 == 0 else cache.auto_V
            lasts.append(seg.parts[-1])
        base = C.wave_of(lasts, [owners[i] for i in oi])
        for i, hnd in zip(oi, C.w_add(base, new.take(oi)).handles()):
            outs[i] = hnd
    ops = [(1 if pp else 0) + 1 + (1 if fr else 0) + 1 for pp, fr in zip(pos, fresh)]
    _retag(outs, _chain_ids(owners, ops, start))
    result = []
    for h in range(H):
        cache = caches[h]
        segs = []
        for which, seg in ((0, cache.auto_K), (1, cache.auto_V)):
            parts = list(seg.parts)
            if fresh[2 * h + which]:
                parts.append(outs[2 * h + which])
            else:
                parts[-1] = outs[2 * h + which]
            segs.append(PackedMatrix(replace(seg.encoding, rows=seg.encoding.rows + 1), parts, encrypted=True))
        result.append(replace(cache, t_auto=cache.t_auto + 1, auto_K=segs[0], auto_V=segs[1]))
    return result


# ----------------------------------------------------------------------------
# refresh
# ----------------------------------------------------------------------------
def maybe_refresh(cache: KVCache, ctx, ch: MpcChannel, force: bool = False) -> KVCache:
    """Masked client round trip of every part at or below the threshold (all
    parts when forced); values unchanged, budgets reset (kv_cache.py:156-196)."""
    return maybe_refresh_heads([cache], [ctx], [ch], force)[0]


def maybe_refresh_heads(caches, ctxs, chans, force: bool = False) -> list:
    c0 = ctxs[0]
    C = type(c0)
    params = c0.params
    n, p, thr = params.n_slots, params.plain_modulus, params.refresh_threshold
    sel = []  # (head, segment name, part index, part)
    for h, cache in enumerate(caches):
        for name, seg in cache.segments():
            for i, part in enumerate(seg.parts):
                if force or part.noise_budget <= thr:
                    sel.append((h, name, i, part))
    if not sel:
        return list(caches)
    # masks drawn per part in order from each head's channel: on the device when the
    # backend can (numpy's PCG64 stream reproduced bit-exactly, nonlinear.device_masks),
    # else on the host
    item_chans = [chans[s[0]] for s in sel]
    owners = [ctxs[s[0]] for s in sel]
    start = {id(c): c._next_id for c in owners}
    wave = C.wave_of([s[3] for s in sel], owners)
    on_device = hasattr(C, "w_add_plain_ids") and device_masks_ok(item_chans)
    if on_device:
        ring = c0.ring
        _pt_cache(ring).make_room(2 * len(sel))
        pt_neg, pt_pos, _ = device_masks(ring, item_chans)
        masked = C.w_add_plain_ids(wave, pt_neg)
    else:
        r = draw_masks(item_chans, n)
        masked = C.w_add_plain(wave, neg_mod(r, p), one_shot=True, canonical=True)
    if on_device:  # the client's decrypt + re-encrypt without the host hop (same words)
        fresh = C.w_reencrypt(masked, [ctxs[s[0]] for s in sel])
    else:
        view = C.w_decrypt(masked)
        fresh = C.w_encrypt([ctxs[s[0]] for s in sel], view, canonical=True)
    for h, _, _, _ in sel:
        chans[h].transfer("refresh", n, trips=2)
    if on_device:
        restored = C.w_add_plain_ids(fresh, pt_pos)
        ring.free_pt(np.concatenate([pt_neg, pt_pos]))  # stream-ordered after their last use
    else:
        restored = C.w_add_plain(fresh, r, one_shot=True, canonical=True)
    restored = _retag(restored.handles(), _chain_ids(owners, [3] * len(sel), start))
    out = []
    for h, cache in enumerate(caches):
        mine = [(k, s) for k, s in enumerate(sel) if s[0] == h]
        if not mine:
            out.append(cache)
            continue
        ctx = ctxs[h]
        segs = {name: list(seg.parts) for name, seg in cache.segments()}
        events = []
        for k, (_, name, i, part) in mine:
            events.append(RefreshEvent(step=cache.t_auto, segment=name, part_index=i, part_id=part.id,
                                       budget_before=part.noise_budget, mpc_bytes=2 * params.ciphertext_bytes(),
                                       forced=force and part.noise_budget > thr))
            segs[name][i] = restored[k]
            ctx.counter.refresh_events += 1
        changed = {s[1] for _, s in mine}
        upd = {}
        for name, seg in cache.segments():
            if name in changed:
                upd[name] = PackedMatrix(seg.encoding, segs[name], encrypted=True, slot_period=seg.slot_period)
        out.append(replace(cache, prefill_K=upd.get("prefill_K", cache.prefill_K),
                           prefill_V=upd.get("prefill_V", cache.prefill_V),
                           auto_K=upd.get("auto_K", cache.auto_K), auto_V=upd.get("auto_V", cache.auto_V),
                           refresh_log=cache.refresh_log + tuple(events)))
    return out


def cache_stats(cache: KVCache) -> dict:
    """kv_cache.py:199-211 (K side; V mirrors)."""
    pre = len(cache.prefill_K.parts) if cache.prefill_K is not None else 0
    return {"ct_count": pre + len(cache.auto_K.parts), "prefill_ct_count": pre,
            "auto_ct_count": len(cache.auto_K.parts), "m": cache.m, "t_auto": cache.t_auto, "B": cache.B,
            "refresh_count": len(cache.refresh_log), "refresh_bytes": sum(e.mpc_bytes for e in cache.refresh_log)}


# ----------------------------------------------------------------------------
# checkpoints
# ----------------------------------------------------------------------------
def _manifest(cache: KVCache, ctx, kind: str) -> dict:
    return {"format": kind, "d2": cache.d2, "B": cache.B, "m": cache.m, "t_auto": cache.t_auto,
            "n_slots": ctx.params.n_slots, "p": ctx.params.plain_modulus, "segments": {},
            "refresh_log": [vars(e) for e in cache.refresh_log]}


def save_cache(cache: KVCache, path, ctx) -> None:
    """Decrypted snapshot in the binary matrix format (kv_cache.py:219-248)."""
    path = Path(path)
    path.mkdir(parents=True, exist_ok=True)
    man = _manifest(cache, ctx, "slots")
    C = type(ctx)
    for name, seg in cache.segments():
        vals = C.w_decrypt(C.wave_of(seg.parts, [ctx] * len(seg.parts))) if seg.parts else []
        for i in range(len(seg.parts)):
            save_matrix(path / f"{name}_{i}.bin", vals[i].reshape(1, -1), ctx.params.plain_modulus)
        man["segments"][name] = {"rows": seg.encoding.rows, "parts": len(seg.parts),
                                 "budgets": [pt.noise_budget for pt in seg.parts], "slot_period": seg.slot_period}
    (path / "manifest.json").write_text(json.dumps(man, indent=2))


def load_cache(path, ctx) -> KVCache:
    """kv_cache.py:251-281; reads both the decrypted and the ciphertext format."""
    path = Path(path)
    man = json.loads((path / "manifest.json").read_text())
    if man["n_slots"] != ctx.params.n_slots or man["p"] != ctx.params.plain_modulus:
        raise ParameterError("cache snapshot was taken under different parameters")
    d2, B = man["d2"], man["B"]
    ct_format = man.get("format") == "ciphertext"
    if ct_format:
        ring = ctx.ring
        want = {"N": ring.N, "L": ring.L, "moduli": [int(q) for q in ring.moduli]}
        if man.get("ring") != want:
            raise ParameterError("ciphertext snapshot was taken on a different ring (N, L or moduli differ)")

    def seg(name, kind, block):
        meta = man["segments"].get(name)
        if meta is None:
            return None
        parts = []
        ids = meta.get("ids") or [None] * len(meta["budgets"])
        for i, budget in enumerate(meta["budgets"]):
            if ct_format:
                words = np.load(path / f"{name}_{i}.npy")
                parts.append(ctx.load_ciphertext_words(words, budget, ids[i]))
            else:
                vals, _ = load_matrix(path / f"{name}_{i}.bin")
                parts.append(ctx.load_ciphertext(vals[0], budget))
        return PackedMatrix(Encoding(kind, meta["rows"], d2, block=block), parts, encrypted=True,
                            slot_period=meta.get("slot_period"))

    has_pre = "prefill_K" in man["segments"]
    return KVCache(d2=d2, B=B, m=man["m"], t_auto=man["t_auto"],
                   prefill_K=seg("prefill_K", EncodingKind.OUTER, None) if has_pre else None,
                   prefill_V=seg("prefill_V", EncodingKind.OUTER, None) if has_pre else None,
                   auto_K=seg("auto_K", EncodingKind.INNER_COMPACTED, B),
                   auto_V=seg("auto_V", EncodingKind.INNER_COMPACTED, B),
                   refresh_log=tuple(RefreshEvent(**e) for e in man["refresh_log"]))


def save_cache_ct(cache: KVCache, path, ctx) -> None:
    """Ciphertext-level snapshot: raw NTT-domain RNS words per part (no
    decryption, so the server can checkpoint without the client)."""
    path = Path(path)
    path.mkdir(parents=True, exist_ok=True)
    man = _manifest(cache, ctx, "ciphertext")
    ring = ctx.ring
    man["ring"] = {"N": ring.N, "L": ring.L, "moduli": [int(q) for q in ring.moduli]}
    for name, seg in cache.segments():
        words = ring.store([pt._aid for pt in seg.parts]) if seg.parts else []
        for i in range(len(seg.parts)):
            np.save(path / f"{name}_{i}.npy", words[i])
        man["segments"][name] = {"rows": seg.encoding.rows, "parts": len(seg.parts),
                                 "budgets": [pt.noise_budget for pt in seg.parts], "slot_period": seg.slot_period,
                                 "ids": [int(pt.id) for pt in seg.parts]}
    (path / "manifest.json").write_text(json.dumps(man, indent=2))


def load_cache_ct(path, ctx) -> KVCache:
    """Load a ciphertext-level snapshot (save_cache_ct): the same words, budgets
    and ids; the manifest's ring must equal ctx's ring.  load_cache reads both
    formats; this name only insists on the ciphertext one."""
    man = json.loads((Path(path) / "manifest.json").read_text())
    if man.get("format") != "ciphertext":
        raise ParameterError("not a ciphertext-level snapshot")
    return load_cache(path, ctx)
