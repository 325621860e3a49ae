"""Shared-memory wavefront model of the FP64 register-I/O NTT (k_ntt2_fpr):
8-byte words, 32 x 4-byte banks, a warp of doubles served as two half-warps
(matches ncu's l1tex shared wavefront counts; ideal = 2 per warp access)."""
import itertools, sys
E = 16; TILE = 2048

def idx(LM, S0, RP, tl, u, k):
    K = 1 << RP; R = E // K; S = (1 << LM) >> S0; ST = S >> RP
    row = tl + u * ((1 << LM) // E); blk = row // ST   # rows interleaved across threads
    return blk * S + (row & (ST - 1)) + k * ST

def wavefronts(addrs):
    """8-byte accesses are served per half-warp (16 lanes x 8 B = 128 B); the
    wavefronts of each half are its worst bank's count of distinct words."""
    tot = 0
    for half in (addrs[:16], addrs[16:]):
        banks = {}
        for a in half:
            for h in (0, 1):
                w = 2 * a + h
                banks.setdefault(w % 32, set()).add(w)
        tot += max(len(v) for v in banks.values())
    return tot

def cost(LM, pas, fwd, padm, pad):
    M = 1 << LM; G = TILE // M; TPS = M // E; T = TILE // E
    RA, RB = 4, LM - 4
    phases = [(0, RA), (RA, RB)] if fwd else [(RA, RB), (0, RA)]
    tot = 0; n = 0
    for ph, (S0, RP) in enumerate(phases):  # phase 0 stores, phase 1 loads
        K = 1 << RP; R = E // K
        for w in range(T // 32):
            for u in range(R):
                for k in range(K):
                    addrs = []
                    for lane in range(32):
                        tid = w * 32 + lane
                        g, tl = (tid % G, tid // G) if pas == 0 else (tid // TPS, tid % TPS)
                        addrs.append(g * padm + pad(idx(LM, S0, RP, tl, u, k)))
                    tot += wavefronts(addrs); n += 1
    return tot / n

if __name__ == "__main__":
    for LM in (5, 6, 7, 8):
        M = 1 << LM
        for pas in (0, 1):
            res = []
            for sh in (3, 4, 5):
                for extra in range(0, 17):
                    padm = M + (M >> sh) + extra
                    c = max(cost(LM, pas, f, padm, lambda i, sh=sh: i + (i >> sh)) for f in (True, False))
                    res.append((c, sh, extra, padm))
            res.sort()
            cur = max(cost(LM, pas, f, M + (M >> 3) + 1, lambda i: i + (i >> 3)) for f in (True, False))
            print(f"LM={LM} pass={pas} current(spad8,PADM=M+M/8+1)={cur:.2f} best={res[:3]}")

def optimal_set(LM, pas):
    M = 1 << LM; out = set()
    for sh in (3, 4, 5):
        for extra in range(0, 33):
            padm = M + (M >> sh) + extra
            if max(cost(LM, pas, f, padm, lambda i, sh=sh: i + (i >> sh)) for f in (True, False)) <= 2.0:
                out.add((sh, extra))
    return out
