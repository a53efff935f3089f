"""Pins of the CPU oracle (oracle/) against what the paper, its cited sources and
mathematics fix -- never against the oracle itself.  DESIGN.md §4 lists each pin.

Each test names the plausible oracle mistake it would catch (dropped term, wrong shift
direction/amount, wrong constant, transposed halves, off-by-one iteration, ...).
"""
import hashlib

import numpy as np
import pytest

import oracle
from workloads import RAGGED_N, SPEC_GRID_I, SPEC_GRID_N

M64 = (1 << 64) - 1
M32 = (1 << 32) - 1


# ---------------------------------------------------------------- P1 / P2 / A4: values
def test_p1_wang32_values(golden):
    """P1: Wang hash of gid 0..3 and of gid^0x9E3779B9 (wang32(0) hand-traced).
    Catches a wrong multiplier, shift amount or step order in A1."""
    g = golden("survey_appendix_a.json")
    assert [oracle.wang32(x) for x in range(4)] == [int(v, 16) for v in g["wang32"]]
    assert [oracle.wang32(x ^ 0x9E3779B9) for x in range(4)] == [int(v, 16) for v in g["wang32_golden_tweak"]]


def test_p1_wang32_hand_trace():
    """P1: the hand trace of wang32(0): each intermediate was computed by
    hand there; here only the final value and the two multiplicative steps' arithmetic."""
    assert 61 * 9 == 549 and (549 ^ (549 >> 4)) == 519
    assert (519 * 0x27D4EB2D) & M32 == 0xC0A8C83B
    assert oracle.wang32(0) == 0xC0A8C83B ^ (0xC0A8C83B >> 15) == 0xC0A9496A


def _wang32_inverse(y):
    """Inverse of Wang's hash, derived step by step (each step is a bijection on u32):
    x^(x>>s) is undone by folding the shifted terms; *c is undone by *c^-1 mod 2^32;
    (x^61)^(x>>16): the high half of y is the high half of x (61 < 2^16)."""
    def unxorshr(v, s):
        x = v
        t = v >> s
        while t:
            x ^= t
            t >>= s
        return x
    y = unxorshr(y, 15)
    y = (y * pow(0x27D4EB2D, -1, 1 << 32)) & M32
    y = unxorshr(y, 4)
    y = (y * pow(9, -1, 1 << 32)) & M32
    hi = y >> 16
    lo = (y & 0xFFFF) ^ 61 ^ hi
    return (hi << 16) | lo


def test_p1_wang32_bijection_by_inverse():
    """P5 prerequisite: wang32 is a bijection on u32 (proved step by step by an inverse
    written from the algebra, not from the oracle).  Catches a non-invertible mutation and
    any reordering of the five steps."""
    r = np.random.default_rng(7)
    xs = [0, 1, 2, 61, 0xFFFF, 0x10000, M32] + [int(v) for v in r.integers(0, 1 << 32, 2000, dtype=np.uint64)]
    for x in xs:
        assert _wang32_inverse(oracle.wang32(x)) == x


def test_p2_states_gid0_3(golden):
    """P2: states for gid 0..3, k = 0..3 (seed 0).  Catches swapped hash halves (A2), a
    missing golden-ratio tweak, an extra/missing step at k = 0 (A6)."""
    g = golden("survey_appendix_a.json")["states_seed0"]
    for gid in range(4):
        want = [int(v, 16) for v in g[str(gid)]]
        assert [oracle.sample(gid, k) for k in range(4)] == want
        assert oracle.stream(4, 4)[:, gid].tolist() == want


def test_a4_seed_premix(golden):
    """A4: fmix64(0) = 0 (so seed 0 is the paper), fmix64 is a bijection (inverse built from
    the modular inverses of its two odd multipliers), and the seed=1 states of SURVEY App. A."""
    assert oracle.fmix64(0) == 0
    inv1 = pow(0xFF51AFD7ED558CCD, -1, 1 << 64)
    inv2 = pow(0xC4CEB9FE1A85EC53, -1, 1 << 64)

    def unx33(v):
        return v ^ (v >> 33)   # x ^ x>>33 is its own inverse for shifts >= 32

    r = np.random.default_rng(3)
    for z in [1, 2, M64] + [int(v) for v in r.integers(0, 1 << 63, 500, dtype=np.uint64)]:
        y = oracle.fmix64(z)
        y = unx33(y)
        y = (y * inv2) & M64
        y = unx33(y)
        y = (y * inv1) & M64
        y = unx33(y)
        assert y == z
    want = [int(v, 16) for v in golden("survey_appendix_a.json")["seed1_k0"]]
    assert [oracle.seed64(g, 1) for g in range(4)] == want
    for gid in range(4):
        assert oracle.seed64(gid, 0) == oracle.sample(gid, 0, 0)


# ---------------------------------------------------------------- P6 / P7: xorshift
def test_p6_xs_of_1(golden):
    """P6: xs(1) = 1082269761; hand trace 1 -> 1^(1<<13)=8193 -> 8193^(8193>>7)=8257
    -> 8257^(8257<<17).  Catches a wrong direction of any of the three shifts."""
    want = golden("spec_examples.json")["xs_of_1"]
    assert 1 ^ (1 << 13) == 8193 and 8193 ^ (8193 >> 7) == 8257 and 8257 ^ (8257 << 17) == want
    assert oracle.xorshift64(1) == want


def test_p7_marsaglia_published_sequence(golden):
    """P7: the cited source's published xor64() from its published seed."""
    g = golden("marsaglia_xor64.json")
    x = g["initial_state"]
    for want in g["outputs"]:
        x = oracle.xorshift64(x)
        assert x == want


# ---------------------------------------------------------------- P3 / P8: algebra
def _xs_matrix():
    """64x64 GF(2) matrix of the ORACLE's xs, column j = xs(e_j)."""
    m = np.zeros((64, 64), dtype=np.uint8)
    for j in range(64):
        v = oracle.xorshift64(1 << j)
        for i in range(64):
            m[i, j] = (v >> i) & 1
    return m


def _matpow(m, e):
    r = np.eye(64, dtype=np.int64)
    b = m.astype(np.int64)
    while e:
        if e & 1:
            r = (r @ b) & 1
        b = (b @ b) & 1
        e >>= 1
    return r


def test_p8_linearity_and_inverse():
    """P8: xs is GF(2)-linear (xs(a^b) = xs(a)^xs(b)) and invertible by the algebraic inverse
    x ^= x<<17 ^ x<<34 ^ x<<51; x ^= x>>7 ^ x>>14 ^ ... ; x ^= x<<13 ^ x<<26 ^ x<<39 ^ x<<52."""
    def inv(x):
        x ^= (x << 17) ^ (x << 34) ^ (x << 51)
        x &= M64
        y = x
        for s in range(7, 64, 7):
            y ^= x >> s
        x = y
        x ^= (x << 13) ^ (x << 26) ^ (x << 39) ^ (x << 52)
        return x & M64

    r = np.random.default_rng(11)
    vals = [int(v) for v in r.integers(0, 1 << 63, 300, dtype=np.uint64)] + [1, M64, 1 << 63]
    for a, b in zip(vals, vals[1:]):
        assert oracle.xorshift64(a ^ b) == oracle.xorshift64(a) ^ oracle.xorshift64(b)
        assert inv(oracle.xorshift64(a)) == a


def test_p3_full_period():
    """P3: Marsaglia's full-period criterion on the oracle's own xs matrix T:
    T^(2^64-1) = I and T^((2^64-1)/p) != I for every prime p | 2^64-1.
    A wrong triple/direction (e.g. the contrast (13,7,16)) fails it."""
    N = (1 << 64) - 1
    primes = [3, 5, 17, 257, 641, 65537, 6700417]
    prod = 1
    for p in primes:
        prod *= p
    assert prod == N
    T = _xs_matrix()
    eye = np.eye(64, dtype=np.int64)
    assert np.array_equal(_matpow(T, N), eye)
    for p in primes:
        assert not np.array_equal(_matpow(T, N // p), eye)


def test_p3_criterion_discriminates():
    """The P3 check is strong enough: the (13,7,16) contrast triple is NOT full period."""
    m = np.zeros((64, 64), dtype=np.uint8)
    for j in range(64):
        x = 1 << j
        x ^= (x << 13) & M64
        x ^= x >> 7
        x ^= (x << 16) & M64
        for i in range(64):
            m[i, j] = (x >> i) & 1
    N = (1 << 64) - 1
    eye = np.eye(64, dtype=np.int64)
    full = np.array_equal(_matpow(m, N), eye) and all(
        not np.array_equal(_matpow(m, N // p), eye) for p in [3, 5, 17, 257, 641, 65537, 6700417])
    assert not full


# ---------------------------------------------------------------- P4 / P5: invariants
def test_p4_nonzero_invariant():
    """P4: xs(0) = 0 (the fixed point, A3); nonzero states stay nonzero (xs invertible);
    seed64(., 0) is never 0 on a large gid range (A3 never fires for seed 0)."""
    assert oracle.xorshift64(0) == 0
    s = oracle.stream(1 << 16, 4)
    assert (s != 0).all()
    x, _ = oracle.digest(1 << 20, 1)   # touches seed64 on 2^20 gids
    assert x.shape == (1,)
    st = oracle.stream(1 << 20, 1)
    assert (st != 0).all()


def test_p5_cross_stream_distinct():
    """P5: equal-k states of distinct gids are distinct (wang32 bijective -> distinct high
    words; xs bijective keeps them distinct).  Catches e.g. hashing gid>>1."""
    s = oracle.stream(1 << 18, 3)
    for k in range(3):
        assert np.unique(s[k]).size == s.shape[1]
    assert np.unique(s[0] >> np.uint64(32)).size == s.shape[1]


def test_determinism_and_seed_distinctness():
    a = oracle.stream(513, 5, seed=9)
    b = oracle.stream(513, 5, seed=9)
    c = oracle.stream(513, 5, seed=10)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, c)


# ---------------------------------------------------------------- P9..P13: streams
def test_p9_n1_i1_bytes(golden):
    """P9: n = 1, i = 1 -> the 8 little-endian bytes of seed64(0)."""
    assert oracle.stream_bytes(1, 1).hex() == golden("spec_examples.json")["n1_i1_stream_hex"]


@pytest.mark.parametrize("n", SPEC_GRID_N + RAGGED_N[:8])
@pytest.mark.parametrize("i", SPEC_GRID_I)
def test_p10_stream_equals_random_access(n, i):
    """P10: the flat loop equals the random-access form xs^k(seed64(g)),
    byte count 8 n i (Eq. 1)."""
    s = oracle.stream(n, i, seed=5)
    assert s.shape == (i, n) and s.nbytes == 8 * n * i
    gs = sorted({0, n - 1, n // 2, n // 3})
    for k in range(i):
        for g in gs:
            assert int(s[k, g]) == oracle.sample(g, k, 5)


def test_p11_sharding_and_iteration_prefix():
    """P11 / A11: shards by global gid reassemble to the single-range stream; a shorter run
    is a prefix of a longer one (split-call equivalence is built on this)."""
    n, i = 1000, 6
    whole = oracle.stream(n, i, seed=3)
    for P in (2, 3, 4, 7):
        parts = []
        for r in range(P):
            b, e = r * n // P, (r + 1) * n // P
            parts.append(oracle.stream(n, i, seed=3, gid_begin=b, count=e - b))
        assert np.array_equal(np.concatenate(parts, axis=1), whole)
    assert np.array_equal(oracle.stream(n, 3, seed=3), whole[:3])


def test_digest_matches_stream():
    n, i = 777, 9
    s = oracle.stream(n, i, seed=2)
    x, t = oracle.digest(n, i, seed=2)
    assert np.array_equal(x, np.bitwise_xor.reduce(s, axis=1))
    assert np.array_equal(t, s.sum(axis=1, dtype=np.uint64))


def test_p12_monobit(golden):
    """P12: fraction of one-bits over the first 10^6 output bits of (4096, 8, 0)."""
    b = oracle.stream(4096, 8).astype("<u8").tobytes()[: 10**6 // 8]
    frac = float(np.unpackbits(np.frombuffer(b, np.uint8)).mean())
    lo, hi = golden("spec_examples.json")["monobit_bounds"]
    assert lo <= frac <= hi
    assert abs(frac - golden("survey_appendix_a.json")["monobit_n4096_i8_first_1e6_bits"]) < 1e-9


def test_p13_config1_digests(golden):
    """P13: config 1 (n = 1024, i = 8) sha256 / xor / sum / last word for 3 seeds,
    cross-checked with the survey's independent implementation."""
    for seed_s, d in golden("survey_appendix_a.json")["config1_n1024_i8"].items():
        s = oracle.stream(1024, 8, seed=int(seed_s))
        assert hashlib.sha256(s.astype("<u8").tobytes()).hexdigest() == d["sha256"]
        assert int(np.bitwise_xor.reduce(s.ravel())) == int(d["xor"], 16)
        assert int(s.ravel().sum(dtype=np.uint64)) == int(d["sum"], 16)
        assert int(s[-1, -1]) == int(d["last"], 16)


def test_eq1_byte_count(golden):
    """Eq. 1: N = 8 n i for the paper's command line."""
    c = golden("spec_examples.json")["paper_command_line"]
    assert 8 * c["n"] * c["i"] == c["bytes"]


def test_bounds_rejected():
    """A12: numrn in [1, 2^32], numiter >= 1, range inside [0, numrn)."""
    with pytest.raises(ValueError):
        oracle.stream(0, 1)
    with pytest.raises(ValueError):
        oracle.digest(4, 0)
    with pytest.raises(ValueError):
        oracle.digest((1 << 32) + 1, 1, count=1)
    with pytest.raises(ValueError):
        oracle.stream(10, 1, gid_begin=8, count=3)


# ---------------------------------------------------------------- NEXT-3: scrambled output
def test_star_multiplier_is_vignas_and_invertible():
    """A19: the scrambler multiplies by Vigna's xorshift64* constant M32 = 2685821657736338717
    (odd, so a bijection); multiplying by its modular inverse recovers the pinned state."""
    M = 2685821657736338717
    assert M == 0x2545F4914F6CDD1D and M % 2 == 1
    inv = pow(M, -1, 1 << 64)
    r = np.random.default_rng(4)
    for x in [0, 1, M64] + [int(v) for v in r.integers(0, 1 << 63, 200, dtype=np.uint64)]:
        y = oracle.star(x)
        assert (y * inv) & M64 == x
        assert y & 1 == x & 1          # odd multiplier keeps the lowest bit
    s = oracle.stream(777, 5, 8)
    t = oracle.stream_star(777, 5, 8)
    back = (t.astype(object) * inv) % (1 << 64)
    assert np.array_equal(back.astype(np.uint64), s)
    assert oracle.star(1) == M


# ---------------------------------------------------------------- A3: the zero-state fix-up
def _fmix64_inverse(y):
    """Inverse of the A4 premix, from the algebra: x ^ (x >> 33) is an involution on u64
    (33 >= 32) and the two odd multipliers are undone by their inverses mod 2^64."""
    def unx33(v):
        return v ^ (v >> 33)
    y = unx33(y)
    y = (y * pow(0xC4CEB9FE1A85EC53, -1, 1 << 64)) & M64
    y = unx33(y)
    y = (y * pow(0xFF51AFD7ED558CCD, -1, 1 << 64)) & M64
    return unx33(y)


def _a3_trigger():
    """A (gid, seed) whose raw composition is 0 ("if result is 0, substitute
    1"; PAPER.md P:173 needs nonzero seeds).  seed64 is 0 iff wang32(g ^ a) = 0 and
    wang32(g ^ C ^ b) = 0 with (a, b) = (lo32, hi32) of fmix64(seed) and C = 0x9E3779B9,
    i.e. g ^ a = g ^ C ^ b = w0 := wang32^-1(0).  Take a = C, b = 0: fmix64(seed) = C and
    g = w0 ^ C -- derived with the two algebraic inverses, never from the oracle."""
    C = 0x9E3779B9
    w0 = _wang32_inverse(0)
    return w0 ^ C, _fmix64_inverse(C)


def test_a3_zero_fixup_trigger():
    """A3: the zero -> 1 fix-up fires at the derived trigger, and only the A3 branch can make
    it 1: the raw composition there is 0 (both hashes 0).  Catches a dropped fix-up (0), a
    wrong substitute (0 -> gid, 0 -> anything else) and a fix-up applied to nonzero states.
    The trigger matches the one VERDICT r1 derived independently."""
    g, s = _a3_trigger()
    assert (g, s) == (2654435716, 0x236D2904C6FC2D12)
    assert _fmix64_inverse(oracle.fmix64(s)) == s and oracle.fmix64(s) == 0x9E3779B9
    m = oracle.fmix64(s)
    a, b = m & M32, m >> 32
    assert oracle.wang32(g ^ a) == 0 and oracle.wang32(g ^ 0x9E3779B9 ^ b) == 0   # raw composition = 0
    assert oracle.seed64(g, s) == 1
    # neighbours are untouched: their raw composition is nonzero and emitted as is
    for gg in (g - 1, g + 1):
        raw = (oracle.wang32(gg ^ a) << 32) | oracle.wang32(gg ^ 0x9E3779B9 ^ b)
        assert raw != 0 and oracle.seed64(gg, s) == raw
    # the stream from the fixed-up state is xs^k(1): 1, xs(1) = 1082269761, ...
    st = oracle.stream(1 << 32, 3, s, gid_begin=g - 1, count=3)
    assert st[0, 1] == 1 and st[1, 1] == 1082269761 and st[2, 1] == oracle.xorshift64(1082269761)
    r = oracle.folds(1 << 32, 1, s, gid_begin=g, count=1, last=True)
    assert r["last"][0] == 1 and r["xor"][0] == 1 and r["wsum"][0] == 2 * g + 1


# ---------------------------------------------------------------- folds: position-weighted digest, last row
def test_folds_weighted_sum_by_hand(golden):
    """The gid-weighted fold sum_g (2 g + 1) out[k][g] mod 2^64 against hand arithmetic on the
    SURVEY App. A states (n = 4, k = 0..3): catches a wrong weight, an unweighted sum, or
    weights from the handle-relative instead of the global gid."""
    g = golden("survey_appendix_a.json")["states_seed0"]
    st = [[int(v, 16) for v in g[str(gid)]] for gid in range(4)]
    r = oracle.folds(4, 4, 0)
    for k in range(4):
        assert int(r["wsum"][k]) == sum((2 * gid + 1) * st[gid][k] for gid in range(4)) & M64
        assert int(r["sum"][k]) == sum(st[gid][k] for gid in range(4)) & M64
    # a sub-range weighs by the global gid: gids 2..3 only
    r2 = oracle.folds(4, 4, 0, gid_begin=2, count=2)
    for k in range(4):
        assert int(r2["wsum"][k]) == (5 * st[2][k] + 7 * st[3][k]) & M64


def test_folds_weighted_sum_sees_a_swap():
    """The reason for the weighted fold: swapping two outputs of one iteration leaves the
    XOR and the sum unchanged but changes sum (2 g + 1) x (by 2 (a - b)(x_b - x_a))."""
    s = oracle.stream(1000, 2, 5)[1].astype(object)
    w = [2 * g + 1 for g in range(1000)]
    t = list(s)
    t[10], t[900] = t[900], t[10]
    assert sum(s) % (1 << 64) == sum(t) % (1 << 64)
    assert sum(a * b for a, b in zip(w, s)) % (1 << 64) != sum(a * b for a, b in zip(w, t)) % (1 << 64)


def test_folds_last_row_and_config1(golden):
    """last = the final iteration (App. A k = 3 column at n = 4, i = 4; the config-1 last word
    for 3 seeds), and the per-iteration folds combine to App. A's whole-stream XOR / sum."""
    g = golden("survey_appendix_a.json")
    assert [int(x) for x in oracle.folds(4, 4, 0, last=True)["last"]] == \
        [int(g["states_seed0"][str(gid)][3], 16) for gid in range(4)]
    for seed_s, d in g["config1_n1024_i8"].items():
        r = oracle.folds(1024, 8, int(seed_s), last=True)
        assert int(r["last"][-1]) == int(d["last"], 16)
        assert int(np.bitwise_xor.reduce(r["xor"])) == int(d["xor"], 16)
        assert int(r["sum"].sum(dtype=np.uint64)) == int(d["sum"], 16)
