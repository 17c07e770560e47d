"""Brute-force check of the DMMA kernel's half-tile fragment offsets
(qg_dmma.cuh tma_frag_off / g4_frag_off, one ring stage = 64 rows x 8 k):
the per-lane closed forms equal the TMA swizzle definition for every lane,
row block, k4 step, fragment and component pair, and every quarter-warp's
128-bit loads hit 8 distinct bank groups in the 4-quaternion-group layouts
(the 32-byte-swizzle layouts keep round 1's 2-/4-way conflicts).  Also lists
every 4-set of the stage's 8 k that is conflict-free in both group layouts.

    python tools/check_g4_half_layout.py
"""
import itertools

P = [[0, 3, 4, 7], [1, 2, 5, 6]]  # k set of k4 step ks, lane kl -> P[ks][kl]


def swz128(lin):
    return lin ^ (((lin >> 7) & 7) << 4)


def swz32(lin):
    return lin ^ (((lin >> 7) & 1) << 4)


def g4_true(rc, r, k, pp):
    lin = (((r >> 2) * 8 + k) * 128 + (r & 3) * 32 + 16 * pp) if rc else ((r * 2 + (k >> 2)) * 128 + (k & 3) * 32 + 16 * pp)
    return swz128(lin)


def g4_formula(rc, rb, rho, kl, ks, i, pp):
    k = P[ks][kl]
    if rc:
        b = ((rb >> 2) + (rho >> 2)) * 1024 + k * 128 + (((2 * (rho & 3)) ^ k) << 4)
    else:
        b = (rb + rho) * 256 + (k >> 2) * 128 + (((2 * (k & 3)) ^ ((2 * rho + (k >> 2)) & 7)) << 4)
    return (b ^ (pp << 4)) + i * 2048


def t32_true(rc, r, k, pp):
    return swz32(((k * 64 + r) * 4 + 2 * pp) * 8 if rc else ((r * 8 + k) * 4 + 2 * pp) * 8)


def t32_formula(rc, r0, kl, ks, i, pp):
    if rc:
        return r0 * 32 + kl * 2048 + ks * 8192 + i * 256 + ((pp << 4) ^ (((r0 >> 2) & 1) << 4))
    return r0 * 256 + kl * 32 + i * 2048 + ks * 128 + ((pp ^ (ks & 1)) << 4)


def main():
    assert sorted(P[0] + P[1]) == list(range(8))  # a bijection of the stage's k
    for rc in (0, 1):
        for rb in range(0, 64, 8):
            for rho in range(8):
                for kl in range(4):
                    for ks in (0, 1):
                        for i in range(4):
                            for pp in (0, 1):
                                r = rb + 8 * i + rho
                                if r < 64:
                                    assert g4_formula(rc, rb, rho, kl, ks, i, pp) == g4_true(rc, r, P[ks][kl], pp)
                                if rb + rho < 64 and r < 64:
                                    assert t32_formula(rc, rb + rho, kl, ks, i, pp) == t32_true(rc, r, 4 * ks + kl, pp)
        for rb in range(0, 64, 8):
            for ks in (0, 1):
                for i in range(4):
                    for pp in (0, 1):
                        for q in range(4):
                            lanes = [l for l in range(8 * q, 8 * q + 8) if rb + 8 * i + (l >> 2) < 64]
                            if len(lanes) < 8:
                                continue
                            groups = {(g4_formula(rc, rb, l >> 2, l & 3, ks, i, pp) % 128) // 16 for l in lanes}
                            assert len(groups) == 8, (rc, rb, ks, i, pp, q)
    f = lambda k: 2 * (k & 3) ^ (k >> 2)  # noqa: E731
    good = [S for S in itertools.combinations(range(8), 4)
            if not (set(S) & {k ^ 2 for k in S}) and not ({f(k) for k in S} & {f(k) ^ 2 for k in S})]
    print("offsets match the swizzle definitions; group tiles conflict-free; conflict-free k sets:", good)


if __name__ == "__main__":
    main()
