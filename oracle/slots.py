"""Slot-level oracle: numpy restatement of the reference emulation.

TEST INFRASTRUCTURE ONLY.  Restates the op semantics of the reference's
``cryptogen.backend.Context`` (/root/reference/pkg/src/cryptogen/
backend.py:307-355: slot-wise Z_p arithmetic, ``np.roll(-k)`` rotation,
linear ledger :295-301, counters :173-213) and exposes the same batched
"wave" API as ``paper_2602_08798_b200.backend.GpuContext``, so the host
code of the hot path (arcc / kv_cache / linear_kernels / encodings) can be
checked on the CPU against golden vectors recorded from the reference
(tests/golden/, made by tests/golden/make_golden.py).

Pinned: tests/test_host_slots.py replays the reference's own
known-answer cases (tests/test_backend.py:63-110 examples, the 200-op
random program) and compares with golden values recorded from the
reference itself.
"""

from __future__ import annotations

import itertools

import numpy as np

from paper_2602_08798_b200.backend import (
    BackendParams, DecryptionFailure, NoiseBudgetExhausted, OpCounter, ParameterError,
)

_uid = itertools.count(10_000)


class SlotCiphertext:
    __slots__ = ("slots", "noise_budget", "id", "params")

    def __init__(self, slots, budget, cid, params):
        slots.setflags(write=False)
        self.slots, self.noise_budget, self.id, self.params = slots, int(budget), int(cid), params

    @property
    def n_slots(self):
        return self.params.n_slots


class SlotWave:
    __slots__ = ("ctxs", "owner", "vals", "budgets", "cids")

    def __init__(self, ctxs, owner, vals, budgets, cids=None):
        self.ctxs, self.owner, self.vals, self.budgets = ctxs, owner, vals, budgets
        self.cids = np.zeros(len(budgets), np.int64) if cids is None else cids

    def __len__(self):
        return int(self.vals.shape[0])

    def take(self, idx):
        idx = np.asarray(idx, dtype=np.int64).reshape(-1)
        return SlotWave(self.ctxs, self.owner[idx], self.vals[idx], self.budgets[idx], self.cids[idx])

    @staticmethod
    def concat(waves):
        ctxs, owners = [], []
        for w in waves:
            base = len(ctxs)
            ctxs.extend(w.ctxs)
            owners.append(w.owner + base)
        return SlotWave(ctxs, np.concatenate(owners), np.concatenate([w.vals for w in waves]),
                        np.concatenate([w.budgets for w in waves]), np.concatenate([w.cids for w in waves]))

    def handles(self):
        return [SlotCiphertext(v.copy(), b, cid, self.ctxs[o].params)
                for o, v, b, cid in zip(self.owner, self.vals, self.budgets, self.cids)]


def _owners(ctxs):
    uniq, owner, seen = [], [], {}
    for c in ctxs:
        if id(c) not in seen:
            seen[id(c)] = len(uniq)
            uniq.append(c)
        owner.append(seen[id(c)])
    return uniq, np.asarray(owner, dtype=np.int64)


class SlotContext:
    """Restates backend.py:245-364 (per-op) plus the wave API."""

    def __init__(self, params: BackendParams, seed=0):
        self.params = params
        self.counter = OpCounter()
        self._seed_seq = seed if isinstance(seed, np.random.SeedSequence) else np.random.SeedSequence(seed)
        self.rng = np.random.default_rng(self._seed_seq)
        self._next_id = next(_uid) * 1_000_000_000

    # helpers
    def _vec(self, v):
        a = np.asarray(v, dtype=np.int64)
        if a.ndim != 1 or a.shape[0] != self.params.n_slots:
            raise ParameterError(f"expected a vector of length {self.params.n_slots}, got shape {a.shape}")
        return np.mod(a, self.params.plain_modulus)

    def plain_vector(self, v):
        return self._vec(v)

    def plain_from_dense(self, v):
        a = np.asarray(v, dtype=np.int64)
        if a.shape[0] > self.params.n_slots:
            raise ParameterError("vector longer than slot count")
        out = np.zeros(self.params.n_slots, dtype=np.int64)
        out[: a.shape[0]] = a
        return np.mod(out, self.params.plain_modulus)

    def zeros(self):
        return np.zeros(self.params.n_slots, dtype=np.int64)

    def fork(self):
        return SlotContext(self.params, self._seed_seq.spawn(1)[0])

    def join(self, child):
        self.counter.merge(child.counter)

    def _emit(self, slots, budget):
        ct = SlotCiphertext(slots, budget, self._next_id, self.params)
        self._next_id += 1
        return ct

    def _check(self, *cts):
        for c in cts:
            if c.params != self.params:
                raise ParameterError("ciphertext belongs to an incompatible context")

    @staticmethod
    def _left(budget, cost):
        if budget - cost < 0:
            raise NoiseBudgetExhausted(f"operation needs {cost} bits but only {budget} remain")
        return budget - cost

    # per-op
    def encrypt(self, v):
        s = self._vec(v)
        self.counter.encrypt += 1
        return self._emit(s.copy(), self.params.initial_noise_budget)

    def decrypt(self, ct):
        self._check(ct)
        if ct.noise_budget <= 0:
            raise DecryptionFailure("noise budget exhausted: decryption would be incorrect")
        self.counter.decrypt += 1
        return ct.slots.copy()

    def add(self, a, b):
        self._check(a, b)
        bud = self._left(min(a.noise_budget, b.noise_budget), self.params.noise_costs.add)
        self.counter.add += 1
        return self._emit((a.slots + b.slots) % self.params.plain_modulus, bud)

    def add_plain(self, a, v):
        self._check(a)
        s = self._vec(v)
        bud = self._left(a.noise_budget, self.params.noise_costs.add_plain)
        self.counter.add_plain += 1
        return self._emit((a.slots + s) % self.params.plain_modulus, bud)

    def mult_plain(self, a, v):
        self._check(a)
        s = self._vec(v)
        bud = self._left(a.noise_budget, self.params.noise_costs.mult_plain)
        self.counter.mult_plain += 1
        return self._emit((a.slots * s) % self.params.plain_modulus, bud)

    def mult_cipher(self, a, b):
        self._check(a, b)
        bud = self._left(min(a.noise_budget, b.noise_budget), self.params.noise_costs.mult_cipher)
        self.counter.mult_cipher += 1
        return self._emit((a.slots * b.slots) % self.params.plain_modulus, bud)

    def rotate(self, a, k):
        self._check(a)
        bud = self._left(a.noise_budget, self.params.noise_costs.rotate)
        self.counter.rotate += 1
        return self._emit(np.roll(a.slots, -(int(k) % self.params.n_slots)), bud)

    def with_budget(self, ct, budget):
        self._check(ct)
        return SlotCiphertext(ct.slots, budget, ct.id, ct.params)

    def load_ciphertext(self, values, budget):
        return self._emit(self._vec(values).copy(), budget)

    # wave API ----------------------------------------------------------------
    @staticmethod
    def wave_of(cts, ctxs=None):
        cts = list(cts)
        if ctxs is None:
            ctxs, owner = [None], np.zeros(len(cts), np.int64)
        else:
            ctxs, owner = _owners(ctxs)
        vals = np.stack([c.slots for c in cts]) if cts else np.zeros((0, 1), np.int64)
        return SlotWave(ctxs, owner, vals.astype(np.int64), np.array([c.noise_budget for c in cts], np.int64),
                        np.array([c.id for c in cts], np.int64))

    @staticmethod
    def bind(wave, ctx):
        return SlotWave([ctx], np.zeros(len(wave), np.int64), wave.vals, wave.budgets, wave.cids)

    @staticmethod
    def _charge(wave, name, counts=None, n_emit=1):
        counts = np.bincount(wave.owner, minlength=len(wave.ctxs)) if counts is None else counts
        for c, k in zip(wave.ctxs, counts):
            if k:
                setattr(c.counter, name, getattr(c.counter, name) + int(k))
        if n_emit == 0:
            return wave.cids
        cids = np.empty(len(wave), np.int64)
        for o, c in enumerate(wave.ctxs):
            sel = np.nonzero(wave.owner == o)[0]
            if sel.size:
                cids[sel] = c._next_id + n_emit * np.arange(sel.size) + (n_emit - 1)
                c._next_id += n_emit * sel.size
        return cids

    @staticmethod
    def _spend(b, cost):
        left = b - cost
        if left.size and left.min() < 0:
            raise NoiseBudgetExhausted(f"operation needs {cost} bits")
        return left

    @staticmethod
    def w_encrypt(ctxs, vecs, canonical=False):
        uniq, owner = _owners(ctxs)
        p = uniq[0].params.plain_modulus
        w = SlotWave(uniq, owner, np.mod(np.asarray(vecs, np.int64), p),
                     np.full(len(owner), uniq[0].params.initial_noise_budget, np.int64))
        w.cids = SlotContext._charge(w, "encrypt")
        return w

    @staticmethod
    def w_decrypt(wave):
        if len(wave) and wave.budgets.min() <= 0:
            raise DecryptionFailure("noise budget exhausted: decryption would be incorrect")
        SlotContext._charge(wave, "decrypt", n_emit=0)
        return wave.vals.copy()

    @staticmethod
    def w_decrypt_start(wave):
        return SlotContext.w_decrypt(wave)

    @staticmethod
    def w_decrypt_finish(pending):
        return pending

    @staticmethod
    def w_add(wa, wb):
        c = wa.ctxs[0]
        b = SlotContext._spend(np.minimum(wa.budgets, wb.budgets), c.params.noise_costs.add)
        return SlotWave(wa.ctxs, wa.owner, (wa.vals + wb.vals) % c.params.plain_modulus, b,
                        SlotContext._charge(wa, "add"))

    @staticmethod
    def w_add_plain(wave, vecs, one_shot=False, canonical=False):
        if hasattr(vecs, "build"):
            vecs = vecs.build(vecs.keys)
        c = wave.ctxs[0]
        p = c.params.plain_modulus
        b = SlotContext._spend(wave.budgets, c.params.noise_costs.add_plain)
        return SlotWave(wave.ctxs, wave.owner, (wave.vals + np.mod(np.asarray(vecs, np.int64), p)) % p, b,
                        SlotContext._charge(wave, "add_plain"))

    @staticmethod
    def w_mult_plain(wave, vecs, one_shot=False):
        if hasattr(vecs, "build"):  # PlainBatch (symbolic rows)
            vecs = vecs.build(vecs.keys)
        c = wave.ctxs[0]
        p = c.params.plain_modulus
        b = SlotContext._spend(wave.budgets, c.params.noise_costs.mult_plain)
        return SlotWave(wave.ctxs, wave.owner, (wave.vals * np.mod(np.asarray(vecs, np.int64), p)) % p, b,
                        SlotContext._charge(wave, "mult_plain"))

    @staticmethod
    def w_mult_cipher(wa, wb, resident_b=False):
        c = wa.ctxs[0]
        b = SlotContext._spend(np.minimum(wa.budgets, wb.budgets), c.params.noise_costs.mult_cipher)
        return SlotWave(wa.ctxs, wa.owner, (wa.vals * wb.vals) % c.params.plain_modulus, b,
                        SlotContext._charge(wa, "mult_cipher"))

    @staticmethod
    def w_rotate(wave, steps, add_input=False):
        c = wave.ctxs[0]
        n = c.params.n_slots
        st = np.broadcast_to(np.asarray(steps, np.int64), (len(wave),))
        rb = SlotContext._spend(wave.budgets, c.params.noise_costs.rotate)
        b = SlotContext._spend(np.minimum(wave.budgets, rb), c.params.noise_costs.add) if add_input else rb
        idx = (np.arange(n)[None, :] + np.mod(st, n)[:, None]) % n
        rolled = np.take_along_axis(wave.vals, idx, axis=1)
        if add_input:
            SlotContext._charge(wave, "rotate", n_emit=0)
            cids = SlotContext._charge(wave, "add", n_emit=2)
            rolled = (rolled + wave.vals) % c.params.plain_modulus
        else:
            cids = SlotContext._charge(wave, "rotate")
        return SlotWave(wave.ctxs, wave.owner, rolled, b, cids)

    @staticmethod
    def w_sum(wave, groups):
        c = wave.ctxs[0]
        cost = c.params.noise_costs.add
        vals, buds, owner, cids = [], [], [], []
        for g in groups:
            g = np.asarray(g, np.int64)
            if g.size == 0:
                raise ParameterError("empty sum")
            acc = int(wave.budgets[g[0]])
            for j in g[1:]:
                acc = SlotContext._left(min(acc, int(wave.budgets[j])), cost)
            vals.append(wave.vals[g].sum(axis=0) % c.params.plain_modulus)
            buds.append(acc)
            o = wave.owner[g[0]]
            owner.append(o)
            ctx = wave.ctxs[o]
            if g.size == 1:
                cids.append(wave.cids[g[0]])
            else:
                ctx.counter.add += int(g.size - 1)
                ctx._next_id += int(g.size - 1)
                cids.append(ctx._next_id - 1)
        return SlotWave(wave.ctxs, np.asarray(owner, np.int64), np.stack(vals), np.asarray(buds, np.int64),
                        np.asarray(cids, np.int64))


def new_slot_context(params: BackendParams, seed=0) -> SlotContext:
    return SlotContext(params, seed)
