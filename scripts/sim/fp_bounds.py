"""Worst-case magnitude bounds of the FP64 NTT (k_ntt2_fpr / k_ks_row / k_col_fused):
every intermediate must stay an integer below 2^53 to be exact.  fp_mulmod(a, w, w/q)
returns |r| <= q (0.5 + 3 2^-53 |a|) (quotient estimate of relative error <= 3 2^-53,
covering the host-rounded w/q and the on-the-fly w * (1/q) of k_ks_row)."""
Q = 2.0 ** 49   # every prime of an FP64-NTT ring is below 2^49
LIM = 2.0 ** 53

def T(a):
    return Q * (0.5 + 3 * 2.0 ** -53 * a)

def forward(b0, stages):  # X' = X + t, Y' = X - t, t = mulmod(Y); no reduction inside
    b, worst = b0, b0
    for _ in range(stages):
        b = b + T(b)
        worst = max(worst, b)
    return worst

def inverse(b0, stages):  # X' = X + Y (not reduced), Y' = mulmod(X - Y)
    b, worst = b0, b0
    for _ in range(stages):
        worst = max(worst, 2 * b)          # X + Y and the mulmod input X - Y
        b = max(2 * b, T(2 * b))
    return worst

if __name__ == "__main__":
    ok = True
    for lm in (5, 6, 7, 8):  # forward: one pass (LM stages) from canonical [0, q)
        w = forward(Q, lm)
        print(f"forward  LM={lm}: max |x| = {w / Q:6.2f} q = 2^{__import__('math').log2(w):.2f}")
        ok &= w < LIM
    # kernel policy: an inverse phase starts from reduced values (|x| <= q/2), except a
    # phase of <= 3 stages reading canonical words straight from memory
    for st, b0, what in ((4, Q / 2, "4-stage phase from reduced"), (3, Q, "3-stage phase from canonical")):
        w = inverse(b0, st)
        print(f"inverse  {what}: max |x| = {w / Q:6.2f} q = 2^{__import__('math').log2(w):.2f}")
        ok &= w < LIM
    # k_ks_row: sum over <= 4 digits of products of forward-pass outputs (LM <= 8)
    prod = T(forward(Q, 8))
    print(f"ks_row   4-digit sum: {4 * prod / Q:6.2f} q")
    ok &= 4 * prod < LIM
    print("all below 2^53:", ok)
    raise SystemExit(0 if ok else 1)
