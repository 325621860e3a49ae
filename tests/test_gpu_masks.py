"""Device-drawn server masks equal the reference's host draws.

MpcChannel.sample_mask(n) is rng.integers(0, p, n) on numpy's PCG64
(/root/reference/pkg/src/cryptogen/nonlinear.py:66-75, :86-87).
cgb_mask_pcg64 reproduces that stream on the GPU (PCG64 jump-ahead, the
32-bit half-word buffer, Lemire rejection): every word of >= 10^6 draws per
channel, the generator state afterwards and the next host draws must agree.
"""
import copy

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_pcg64_masks_equal_numpy_1m_per_channel():
    from paper_2602_08798_b200 import nonlinear as nl
    from paper_2602_08798_b200._native import build
    from paper_2602_08798_b200.backend import BackendParams, GpuContext

    build()
    params = BackendParams()
    ctx = GpuContext(params, 0)
    ring, n, p = ctx.ring, params.n_slots, params.plain_modulus
    chans = [nl.MpcChannel(p, seed=s) for s in (3, 1000, 77)]
    chans[1].rng.integers(0, p, 5)  # leaves a buffered 32-bit half (has_uint32 = 1)
    assert chans[1].rng.bit_generator.state["has_uint32"] == 1
    twins = [copy.deepcopy(ch) for ch in chans]
    per = 130  # 130 x 8192 = 1.06M words per channel
    items = [chans[i % 3] for i in range(3 * per)]  # interleaved channels, each in draw order
    want = np.stack([twins[i % 3].sample_mask(n) for i in range(3 * per)])
    neg, pos, got = nl.device_masks(ring, items, want_masks=True)
    assert np.array_equal(got, want)
    for ch, tw in zip(chans, twins):
        assert ch.rng.bit_generator.state == tw.rng.bit_generator.state
        assert np.array_equal(ch.sample_mask(1001), tw.sample_mask(1001))
    # the encoded plaintexts: add_plain of r and of p - r cancel
    v = np.arange(n) % p
    ids = ring.alloc(3)
    ring.encrypt(v, np.arange(8, dtype=np.uint32), 0, ids[:1])
    ring.add_plain(ids[:1], pos[:1], ids[1:2])
    assert np.array_equal(ring.decrypt(ids[1:2])[0], (v + want[0]) % p)
    ring.add_plain(ids[1:2], neg[:1], ids[2:3])
    assert np.array_equal(ring.decrypt(ids[2:3])[0], v)
    ring.free(ids)
    ring.free_pt(np.concatenate([neg, pos]))


def test_refresh_device_masks_equal_host_masks():
    """maybe_refresh_heads with device masks == with host masks: words, ids,
    transcripts, refresh log, and the channels' next draws."""
    import os
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent / "golden"))
    import harness
    from hostapi import repo_api
    from paper_2602_08798_b200 import nonlinear as nl
    from paper_2602_08798_b200._native import build
    from paper_2602_08798_b200.backend import GpuContext

    build()
    api = repo_api()
    res = {}
    for mode in ("host", "device"):
        nl.DEVICE_MASKS = mode == "device"
        try:
            root, fp, ctxs, caches, qs, chans = harness.attention_heads(api, GpuContext, 8192, harness.P8192, 64, 8,
                                                                        3, 2, seed=4)
            cs = api.maybe_refresh_heads(caches, ctxs, chans, force=True)
        finally:
            nl.DEVICE_MASKS = True
        res[mode] = ([pt.words() for c in cs for _, seg in c.segments() for pt in seg.parts],
                     [(pt.id % 10**9, pt.noise_budget) for c in cs for _, seg in c.segments() for pt in seg.parts],
                     [c.counter.as_dict() for c in ctxs], [ch.transcript for ch in chans],
                     [ch.sample_mask(16).tolist() for ch in chans])
    for a, b in zip(res["host"][0], res["device"][0]):
        assert np.array_equal(a, b)
    assert res["host"][1:] == res["device"][1:]
