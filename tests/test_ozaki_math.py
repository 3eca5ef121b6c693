"""Host-side checks of the integer arithmetic the Ozaki kernels rely on (ozaki.cu):
the conversion-free division by a modulus (GEMM epilogue and Garner digits) and the
integer Garner recurrence with int8 coefficients, evaluated here with numpy / Python
integers exactly as the device evaluates them."""
import math

import numpy as np

MODS = [256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193]


def sym(x, m):
    r = x % m
    return r - m if r > m - (m >> 1) - 1 else r


def magic(m):
    return (1 << 39) // m + 1


def test_moduli_are_pairwise_coprime_and_cover_the_product_range():
    for i, a in enumerate(MODS):
        for b in MODS[i + 1:]:
            assert math.gcd(a, b) == 1
    M = math.prod(MODS)
    # |P| <= K 2^106 with K <= 65535 must stay below M / 2
    assert 65535 * 2 ** 106 < M // 2


def test_magic_division_is_exact_on_the_whole_biased_range():
    """floor(u / m) == umulhi(u, magic) >> 7 for 0 <= u < 2^31: checked on the boundaries
    of every quotient step near the ends of the range and on a dense random sample."""
    rng = np.random.default_rng(0)
    for m in MODS:
        mg = np.uint64(magic(m))
        assert magic(m) < 2 ** 32
        qs = np.concatenate([np.arange(0, 4096), np.arange((2 ** 31) // m - 4096, (2 ** 31) // m + 1)])
        u = np.concatenate([qs * m, qs * m - 1, qs * m + m - 1, rng.integers(0, 2 ** 31, 2 ** 20)]).astype(np.int64)
        u = u[(u >= 0) & (u < 2 ** 31)].astype(np.uint64)
        q = ((u * mg) >> np.uint64(32)) >> np.uint64(7)
        assert np.array_equal(q, u // np.uint64(m))


def test_epilogue_reduction_matches_symmetric_residue():
    """ModStore: u = x + m floor(2^30 / m), symmetric fix-up, for |x| <= 2^30 - 2^14."""
    rng = np.random.default_rng(1)
    lim = 2 ** 30 - 2 ** 14
    x = np.concatenate([np.arange(-70000, 70000), rng.integers(-lim, lim + 1, 2 ** 20), [-lim, lim]]).astype(np.int64)
    for m in MODS:
        u = (x + m * ((1 << 30) // m)).astype(np.uint64)
        q = ((u * np.uint64(magic(m))) >> np.uint64(32)) >> np.uint64(7)
        r = (u - q * np.uint64(m)).astype(np.int64)
        r = np.where(r > m - (m >> 1) - 1, r - m, r)
        want = np.mod(x, m)
        want = np.where(want > m - (m >> 1) - 1, want - m, want)
        assert np.array_equal(r, want)


def test_integer_garner_recurrence_reconstructs_the_value():
    """dig_l = sym(r_l t_l + sum_u dig_u k[l][u]) with int8 t and k, then the balanced
    mixed-radix sum, returns the integer for values across the whole range."""
    c = [[math.prod(MODS[:u]) % MODS[l] for u in range(16)] for l in range(16)]
    inv = [pow(math.prod(MODS[:l]) % MODS[l], -1, MODS[l]) if l else 1 for l in range(16)]
    k = [[sym(-c[l][u] * inv[l], MODS[l]) for u in range(16)] for l in range(16)]
    t = [sym(inv[l], MODS[l]) for l in range(16)]
    for row in k:
        assert all(-128 <= v <= 127 for v in row)
    M = math.prod(MODS)
    rng = np.random.default_rng(2)
    vals = [0, 1, -1, M // 2 - 1, -(M // 2) + 1, 65535 * 2 ** 106, -65535 * 2 ** 106]
    vals += [int(rng.integers(-2 ** 62, 2 ** 62)) * int(rng.integers(-2 ** 62, 2 ** 62)) for _ in range(2000)]
    for v in vals:
        r = [sym(v, m) for m in MODS]
        dig = [r[0]]
        for l in range(1, 16):
            acc = r[l] * t[l] + sum(dig[u] * k[l][u] for u in range(l))
            assert abs(acc) <= 2 ** 30 - 256
            dig.append(sym(acc, MODS[l]))
            assert -128 <= dig[-1] <= 127
        total, w = 0, 1
        for l in range(16):
            total += dig[l] * w
            w *= MODS[l]
        assert total == v


def test_log2_table_in_the_kernel_source_is_rounded_down():
    """exponent_kernel's kLog2M (the moduli count decision) never overstates log2(M_L)."""
    import os
    import re
    src = open(os.path.join(os.path.dirname(__file__), "..", "paper_2012_14702_b200", "csrc", "ozaki.cu")).read()
    body = re.search(r"kLog2M\[kMods\] = \{([^}]*)\}", src).group(1)
    vals = [float(v) for v in body.replace("\n", " ").split(",")]
    assert len(vals) == 16
    for L, v in enumerate(vals, start=1):
        exact = math.log2(math.prod(MODS[:L]))
        assert v <= exact < v + 1e-5
