"""Worst-case error bound of the certified fp32 MVUE decision (csrc/s24_mvue.cu mvue_group_cert),
in units u = ulp(1) = 2^-24: absolute error bounds propagated through the reference's greedy pair
fill (sparsity.py:327-355) and cumulative sums, given |pi_fp32 - pi_float64| <= e_pi u.  Every
rounded fp32 operation on values <= 1 adds <= 1 u (<= 2 u on the pi sum, values <= 2); min / max
are 1-Lipschitz.  The kernel requires |c_j - draw| > 2^-14 = 1024 u; the bound must stay below.
python tools/mvue_bound.py"""


def bound(e_pi: float, rnd: float = 1.0, rnd2: float = 2.0) -> float:
    s = 0.5 * (4 * e_pi + 3 * rnd2)  # s = 0.5 (((p0 + p1) + p2) + p3)
    r = [e_pi] * 4
    p01 = max(r[0], r[1], s + r[2] + rnd, s + r[3] + rnd)
    r[0] += p01 + rnd; r[1] += p01 + rnd; s += p01 + rnd
    p02 = max(r[0], r[2], s + r[3] + rnd)
    r[0] += p02 + rnd; r[2] += p02 + rnd; s += p02 + rnd
    p03 = max(r[0], r[3])
    r[3] += p03 + rnd; s += p03 + rnd
    p12 = max(r[1], r[2], s + r[3] + rnd)
    r[1] += p12 + rnd; r[2] += p12 + rnd
    p13 = max(r[1], r[3])
    r[3] += p13 + rnd
    p23 = max(r[2], r[3])
    c = [p01]
    for p in (p02, p03, p12, p13, p23):
        c.append(c[-1] + p + rnd)
    draw = c[-1] + 1.0 + rnd  # uniform truncated to 24 bits (<= 1 u since c5 <= 1) + the product's rounding
    return max(c) + draw


if __name__ == "__main__":
    # pi = n * RN(1 / d) with exact n, d (binade span <= 14): two roundings -> e_pi = 2
    b = bound(2.0)
    print(f"decision error bound {b:.0f} u (margin 1024 u): {'OK' if b < 1024 else 'VIOLATED'}")
    assert b < 1024
